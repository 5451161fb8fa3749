/*
 * gsi.h — C ABI of the B200-native GSI subgraph-matching library (libgsi_b200.so).
 *
 * Problem (Def. 1-3; N(v,l) at L299): given a labelled undirected data
 * graph G and a connected labelled query graph Q, enumerate every injective map
 * f : V(Q) -> V(G) with L_V(f(u)) = L_V(u) and, for every query edge (a,b,l), a data
 * edge {f(a), f(b)} labelled l (non-induced, SURVEY.md §8(c) readings A1/A2).
 *
 * Hot path: PCSR build (Def. 4, Alg. 1), signature
 * table + filter (§III-A), join-order planner (Alg. 2, Alg. 4 line 1
 * L1119), and the per-level Prealloc-Combine vertex join (Alg. 3, Alg. 4
 * L1113-1129).  Every device step runs in this library's own sm_100a kernels.
 *
 * Conventions
 *  - Ownership: every `const T*` input is a HOST pointer borrowed for the duration of the
 *    call and copied; the library never keeps it.  Handles (`gsi_graph*`, `gsi_result*`,
 *    `gsi_prepared*`) are owned by the caller and released with the matching *_free.
 *  - Errors: every entry point returns a gsi_status; on error no partial result is
 *    returned (out handles are set to NULL) and gsi_last_error() gives a thread-local
 *    message.  The library never aborts the process and never falls back to the CPU:
 *    with no usable CUDA device every compute call returns GSI_ERR_CUDA.
 *  - Concurrency: a built graph is immutable and may serve concurrent queries from
 *    different host threads on different streams.
 *  - Streams: `stream` fields take a cudaStream_t (NULL = the per-thread default stream).
 *    Calls return after the work they enqueue has completed (counts are host values).
 *  - Limits: |V| < 2^31 - 1, 2|E| < 2^31 - 1, query k <= 32 vertices, labels are int32 >= 0.
 */
#ifndef GSI_H
#define GSI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSI_MAX_K 32
#define GSI_SIG_PLANES 16        /* N = 512 bits = 16 uint32 words, K = 32 */
#define GSI_N_KCLASS 8           /* kernel classes timed when gsi_query_opts.profile = 1   */

typedef enum {
    GSI_OK = 0,
    GSI_ERR_INVALID_ARG = -1,
    GSI_ERR_VERTEX_RANGE = -2,
    GSI_ERR_LABEL_RANGE = -3,
    GSI_ERR_SELF_LOOP = -4,
    GSI_ERR_DUPLICATE_EDGE = -5,
    GSI_ERR_QUERY_DISCONNECTED = -6,
    GSI_ERR_QUERY_TOO_LARGE = -7,
    GSI_ERR_OOM = -8,
    GSI_ERR_TIMEOUT = -9,
    GSI_ERR_CUDA = -10,
    GSI_ERR_INTERNAL = -11
} gsi_status;

/* Kernel classes reported in gsi_stats (profile mode). */
enum { GSI_K_FILTER = 0, GSI_K_COMPACT = 1, GSI_K_PROBE = 2, GSI_K_JOIN = 3, GSI_K_LINK = 4,
       GSI_K_OTHER = 5 };

/* Kernel variants: gsi_stats.variant_launches[v] counts the launches of each (always, not only
 * in profile mode), so a test can prove which code path produced a result. */
#define GSI_N_KVARIANT 20
enum { GSI_V_JOIN_NEXT = 0,       /* k_join<J_NEXT>: slot tiles, compacting (Combine) write     */
       GSI_V_JOIN_COUNT = 1,      /* k_join<J_COUNT>: slot tiles, final level count (+ hash)    */
       GSI_V_JOIN_TABLE = 2,      /* k_join<J_TABLE>: slot tiles, final table                  */
       GSI_V_JOIN_CAHEAD = 3,     /* k_join<J_CAHEAD>: slot tiles, count-ahead                 */
       GSI_V_COUNT_FAST = 4,      /* k_count_fast: slot tiles, final count on shared runs      */
       GSI_V_NEXT_LEAN = 5,       /* k_next_lean: warp rows, rows at their Prealloc slots      */
       GSI_V_CAHEAD_WARP = 6,     /* k_cahead_warp: generic warp count-ahead                   */
       GSI_V_CAHEAD_LEAN = 7,     /* k_cahead_lean<*,false>: closed-form count-ahead           */
       GSI_V_FINAL_LEAN = 8,      /* k_cahead_lean<*,true>: closed-form final count            */
       GSI_V_FINAL_FP = 9,        /* k_final_fp: every final match read and hashed             */
       GSI_V_FILTER_PARTITION = 10, /* k_filter_partition: shared N(v,l0) ∩ C(u) runs          */
       GSI_V_REFILTER = 11,       /* k_refilter: a level re-pointed at shared runs             */
       GSI_V_PROBE_AHEAD = 12,    /* k_probe_ahead: per-candidate next-step locate table       */
       GSI_V_SMALL = 13,          /* k_small_query: whole query in one launch                  */
       GSI_V_TWO_STEP = 14,       /* ablation: count pass of the two-step output               */
       GSI_V_ABLATION = 15,       /* ablation engine join launches (warp per row, paper design) */
       GSI_V_FINAL_TABLE = 16,    /* k_final_table: every final match written (table mode)     */
       GSI_V_SURV_SCAN = 17,      /* k_surv_scan: table-mode Combine offsets per row           */
       GSI_V_FP_TERMS = 18 };     /* k_fp_terms: per-candidate fingerprint terms of a shared run */

/* gsi_query_opts.ablation bits (NEXT-3: the paper's join-phase study, Tables VI-VIII):
 * any bit set runs the query on the paper-style engine (one warp per row of M, Alg. 3/4) with
 * the named technique switched off; 0 = the B200 default path.  Results are identical. */
#define GSI_ABL_ENGINE   1   /* paper-style engine with PCSR, Prealloc-Combine, write cache, set ops */
#define GSI_ABL_CR       2   /* locate N(v,l) in the Compressed Representation (binary search, L674-682) */
#define GSI_ABL_TWO_STEP 4   /* two-step output (join twice: count, scan, join + write; L1635-1641) */
#define GSI_ABL_NO_WCACHE 8  /* no write cache: each lane stores its own survivor row (L1155-1158)  */
#define GSI_ABL_NAIVE_SO 16  /* naive set operation: C(u) by binary search in the candidate list,
                                 other linking lists by linear scan (L1136-1158 off)                */
#define GSI_ABL_NO_LB    32  /* no 4-layer balance (L1169-1176): every row by one warp; on, rows   */
                             /* above W2 take a block and rows above W1 an 8-CTA cluster (DSMEM)   */
#define GSI_ABL_NO_DR    64  /* no duplicate removal within the block (Alg. 5)         */

typedef struct gsi_graph gsi_graph;       /* opaque: PCSR + signature table on one device   */
typedef struct gsi_result gsi_result;     /* opaque: count, fingerprint, optional table     */
typedef struct gsi_prepared gsi_prepared; /* opaque: a validated, encoded, device-resident Q */

/* ------------------------------------------------------------------ graph build ----- */
typedef struct {
    int32_t gpn;      /* PCSR pairs per group, 2..16; default 16 = one 128 B group */
    int32_t device;   /* CUDA device ordinal; -1 = current device                               */
    void *stream;     /* cudaStream_t used for the build                                         */
} gsi_build_opts;

void gsi_build_opts_default(gsi_build_opts *opts);

/*
 * gsi_build_graph — PCSR (Def. 4, Alg. 1) for every edge label plus the column-first
 * signature table, built on the device.
 *   n        number of vertices; vertex ids are 0..n-1.
 *   vlabels  n int32 vertex labels (>= 0).
 *   m        number of undirected edges; each listed ONCE as (src[i], dst[i], elabels[i]).
 *   Parallel edges with DISTINCT labels are accepted (SURVEY.md reading A3); an exact
 *   duplicate (v,w,l) in either orientation -> GSI_ERR_DUPLICATE_EDGE; src == dst ->
 *   GSI_ERR_SELF_LOOP; ids outside [0,n) -> GSI_ERR_VERTEX_RANGE; negative labels ->
 *   GSI_ERR_LABEL_RANGE.  Edge labels are remapped densely inside the build.
 *   out      receives the graph handle (NULL on error).
 */
gsi_status gsi_build_graph(int64_t n, const int32_t *vlabels, int64_t m, const int32_t *src,
                           const int32_t *dst, const int32_t *elabels, const gsi_build_opts *opts,
                           gsi_graph **out);

/*
 * gsi_build_graph_ml — multi-label vertices and edges (§VII-B; NEXT-4).
 * A match then needs L_V(u) ⊆ L_V(f(u)) and L_E(uv) ⊆ L_E(f(u)f(v)) (L1273-1275).
 *   vls_off  n+1 int64 offsets, vls the labels: L_V(v) = vls[vls_off[v] .. vls_off[v+1]).
 *   els_off  m+1 int64 offsets, els the labels of edge e = (src[e], dst[e]).
 * Every edge label becomes one single-label parallel edge (L1283-1285); the signature
 * table hashes the vertex label sets (reading A19) and the label sets stay on
 * the device for the exact refine of C(u) (L1279-1281).  Repeated labels inside a set are
 * ignored; a label in the sets of two edges on the same vertex pair -> DUPLICATE_EDGE.
 * Query such a graph with gsi_query_prepare_ml (gsi_query_prepare refuses it).
 * Errors as gsi_build_graph; offsets that do not start at 0 or decrease -> INVALID_ARG.
 */
gsi_status gsi_build_graph_ml(int64_t n, const int64_t *vls_off, const int32_t *vls, int64_t m,
                              const int32_t *src, const int32_t *dst, const int64_t *els_off,
                              const int32_t *els, const gsi_build_opts *opts, gsi_graph **out);

/*
 * gsi_build_line_graph — edge isomorphism (§VII-A, Fig. 9; NEXT-4):
 * builds, on the device, the line graph G' of the input graph (arguments and errors as
 * gsi_build_graph): vertex i of G' is input edge i, labelled elabels[i]; every two input
 * edges sharing a vertex v give one G' edge labelled vlabels[v] (two parallel input edges
 * whose shared ends carry the same label give it once).  Then PCSR + signatures of G' as
 * gsi_build_graph.  sum_v deg(v)(deg(v)-1)/2 must stay below 2^30 -> else INVALID_ARG.
 * Query it with gsi_query_prepare_line; result rows are input edge ids per query edge.
 */
gsi_status gsi_build_line_graph(int64_t n, const int32_t *vlabels, int64_t m, const int32_t *src,
                                const int32_t *dst, const int32_t *elabels, const gsi_build_opts *opts,
                                gsi_graph **out);

typedef struct {
    int64_t n, m;                 /* |V|, |E| (undirected)                                  */
    int32_t n_elabels;            /* distinct edge labels |L_E|                             */
    int32_t gpn;
    int64_t n_groups;             /* sum_l |V(D_l)| (one group allocated per partition vertex) */
    int32_t max_chain;            /* longest overflow chain in groups  */
    int64_t overflow_groups;      /* groups whose keys spilled (Alg. 1 lines 5-8)           */
    uint64_t bytes_groups, bytes_ci, bytes_sig, bytes_total;
    int32_t device;
    float ms_build;
} gsi_graph_info;

gsi_status gsi_graph_info_get(const gsi_graph *g, gsi_graph_info *info);

/* Device buffers of a graph, for replicating it to other GPUs (NCCL broadcast). */
typedef struct {
    const char *name;   /* static string                                                  */
    void *dev_ptr;      /* device pointer owned by the graph                              */
    uint64_t bytes;
} gsi_buffer_desc;

#define GSI_MAX_BUFFERS 8
/* Fill descs[0..*ndesc) (capacity GSI_MAX_BUFFERS) and a host metadata blob (graph
 * scalars + per-label host tables) of *meta_bytes bytes (meta may be NULL to query size). */
gsi_status gsi_graph_buffers(const gsi_graph *g, gsi_buffer_desc *descs, int32_t *ndesc,
                             void *meta, uint64_t *meta_bytes);
/* Allocate an empty graph on `opts->device` with the buffer sizes / metadata produced by
 * gsi_graph_buffers on another rank; its descs (same order) can then be filled by a
 * broadcast.  The graph is usable once every buffer holds the source's bytes. */
gsi_status gsi_graph_alloc_like(const void *meta, uint64_t meta_bytes, const gsi_build_opts *opts,
                                gsi_graph **out, gsi_buffer_desc *descs, int32_t *ndesc);

void gsi_graph_free(gsi_graph *g);

/* ------------------------------------------------------------------ query ----------- */
typedef struct {
    int32_t want_table;          /* 1: materialise the match table (device, query-id order)  */
    int32_t homomorphism;        /* 1: drop the injectivity subtraction */
    int32_t filter_mode;         /* 0: signature filter (L534-552); 1: label-only C(u)        */
    int32_t e0_mode;             /* 0: per row, the shortest linking list bounds the buffer
                                    (B200 default; any linking edge bounds it, L967-981);
                                    1: the paper's min-freq linking label (Alg. 4 line 1)     */
    const int32_t *force_order;  /* test hook: k query ids (connected prefixes) or NULL        */
    const int32_t *force_first_edge; /* test hook: [k] per step j the query vertex at the
                                    other end of e0 (entry 0 ignored, -1 = planner's), or NULL */
    const int32_t *roots;        /* test hook: restrict f(pi_1) to these data vertices, or NULL */
    int64_t n_roots;
    int32_t shard_rank, shard_count; /* M-row sharding; 0/1 = whole query   */
    uint64_t shard_min_rows;     /* shard at the first level with |M_t| >= this (0 = 65536)    */
    uint64_t mem_budget_bytes;   /* device bytes the query may use (0 = 90% of free memory)    */
    double timeout_s;            /* <= 0: none.  Checked between levels.                        */
    int32_t profile;             /* 1: time every kernel with CUDA events (gsi_stats)          */
    void *stream;                /* cudaStream_t                                               */
    uint64_t chunk_slots;        /* GBA slots per chunk (0 = derived from the memory budget);
                                    a level whose |GBA| exceeds it runs depth-first in chunks  */
    int32_t partial_on_timeout;  /* 1: on timeout return GSI_OK with stats.capped = 1 and the
                                    exact count of the completed chunk prefix                  */
    int32_t fingerprint;         /* 1: compute the set fingerprint of the final rows (costs ~2k
                                    hash rounds per match); 0: fingerprint = (count, 0, 0)      */
    int32_t no_shared_lists;     /* 1: never switch a level to shared N(v,l0) ∩ C(u) lists      */
    int32_t no_count_ahead;      /* 1: enumerate every match of the last level even in count-only
                                    mode.  0 (default): when the last step has one linking edge
                                    and no fingerprint/table is wanted, the level before it counts
                                    each new row's extensions as |N(v,l0) ∩ C(u)| minus the row's
                                    own vertices in that run (Alg. 3 lines 9-10 applied to a
                                    count), so M_{k-1} is never stored and M_k never enumerated  */
    int32_t shard_pieces;        /* with shard_count > 1: the shard level's slot range is cut into
                                    shard_count x shard_pieces equal pieces (row granularity) and
                                    rank r keeps pieces r, r + shard_count, ...; 0/1 = one
                                    contiguous range per rank (concatenating the ranks' tables in
                                    rank order then gives the 1-GPU row order)                  */
    int32_t force_paths;         /* test hook, bit 0: take the shared-run paths (shared
                                    N(v,l0) ∩ C(u) runs, prefiltered next levels, probe-ahead
                                    tables, count-ahead, lean kernels) whenever the query's shape
                                    allows them, ignoring the size thresholds that normally decide
                                    — so small root-restricted runs exercise the kernels a large
                                    query uses.  Results are identical either way.               */
    int32_t small_mode;          /* 0: a query with a small first level runs all its levels in one
                                    launch (k_small_query) when it fits, else the regular path;
                                    1: always the regular per-level path                       */
    int32_t ablation;            /* GSI_ABL_* bits (0: off).  Count / fingerprint only: with
                                    want_table the call returns GSI_ERR_INVALID_ARG             */
} gsi_query_opts;

void gsi_query_opts_default(gsi_query_opts *opts);

/*
 * gsi_query — filter, plan and join Q against g (the whole hot path, §8(a) a3-a9).
 *   k                 number of query vertices (1..32), ids 0..k-1.
 *   q_vlabels         k int32.
 *   qm, q_src, q_dst, q_elabels   query edges, each listed once.
 * A disconnected Q -> GSI_ERR_QUERY_DISCONNECTED (PAPER.md L299 assumes connectivity);
 * k > 32 -> GSI_ERR_QUERY_TOO_LARGE; labels absent from G give count 0.
 */
gsi_status gsi_query(const gsi_graph *g, int32_t k, const int32_t *q_vlabels, int32_t qm,
                     const int32_t *q_src, const int32_t *q_dst, const int32_t *q_elabels,
                     const gsi_query_opts *opts, gsi_result **out);

/* Split of gsi_query: validate + encode Q once (host -> device), then run it.  A prepared
 * query is bound to its graph and may be run any number of times. */
gsi_status gsi_query_prepare(const gsi_graph *g, int32_t k, const int32_t *q_vlabels, int32_t qm,
                             const int32_t *q_src, const int32_t *q_dst, const int32_t *q_elabels,
                             gsi_prepared **out);
/* Multi-label query for a gsi_build_graph_ml graph: q_vls_off (k+1
 * int32 offsets) / q_vls the vertex label sets (at most 32 labels each), q_els_off (qm+1)
 * / q_els the edge label sets.  Validation as gsi_query_prepare.  Rows of the result are
 * data vertices in query-id order, as for single labels. */
gsi_status gsi_query_prepare_ml(const gsi_graph *g, int32_t k, const int32_t *q_vls_off, const int32_t *q_vls,
                                int32_t qm, const int32_t *q_src, const int32_t *q_dst,
                                const int32_t *q_els_off, const int32_t *q_els, gsi_prepared **out);
/* Edge-isomorphism query for a gsi_build_line_graph graph: Q (k
 * vertices, 1 <= qm <= 32 edges, connected) is transformed into its line graph on the host
 * and prepared against G'.  Result rows have qm columns: the data edge id (index into the
 * build's edge list) matched by query edge 0..qm-1. */
gsi_status gsi_query_prepare_line(const gsi_graph *g, int32_t k, const int32_t *q_vlabels, int32_t qm,
                                  const int32_t *q_src, const int32_t *q_dst, const int32_t *q_elabels,
                                  gsi_prepared **out);
gsi_status gsi_query_run(const gsi_graph *g, const gsi_prepared *q, const gsi_query_opts *opts,
                         gsi_result **out);
void gsi_prepared_free(gsi_prepared *q);

/*
 * gsi_query_run_batch — run nq prepared queries of one graph concurrently (inter-query
 * parallelism, SURVEY.md §8(e) "tiny queries"): `concurrency` (1..8) host workers, each with
 * its own CUDA stream and query workspace, take the queries in order; their kernels
 * interleave on the device.  opts applies to every query (opts->stream is ignored; a zero
 * mem_budget_bytes becomes the device budget / concurrency).  out receives nq result
 * handles in query order; on any error all are freed, out[] is NULL and the status of the
 * first failing query is returned (gsi_last_error names it).
 */
gsi_status gsi_query_run_batch(const gsi_graph *g, int32_t nq, const gsi_prepared *const *qs,
                               const gsi_query_opts *opts, int32_t concurrency, gsi_result **out);

typedef struct {
    int32_t k, levels;                /* levels = number of join levels executed            */
    int32_t order[GSI_MAX_K];         /* join order pi (query ids)                          */
    int64_t cand[GSI_MAX_K];          /* |C(u)| by query id                                 */
    uint64_t rows[GSI_MAX_K];         /* |M_t| for t = 1..k at index t-1 (this shard)        */
    uint64_t gba[GSI_MAX_K];          /* |GBA| (prealloc bound F[|M|]) producing M_{t+1}, idx t */
    uint64_t list_elems[GSI_MAX_K];   /* sum over rows and linking edges of |N(v,l)|, idx t */
    int32_t n_edges[GSI_MAX_K];       /* |ES| per step (idx t = step producing M_{t+1})     */
    int32_t first_edge[GSI_MAX_K];    /* planner's e0 other-end query id per step           */
    uint64_t count;
    int32_t shard_level;              /* level whose rows were sharded (-1: not sharded)    */
    uint64_t shard_row_begin, shard_row_end;
    float ms_total, ms_filter, ms_plan, ms_join;
    /* profile mode: per kernel class (GSI_K_*) summed device ms, launches, algorithmic bytes */
    float ms_kernel[GSI_N_KCLASS];
    uint32_t launches[GSI_N_KCLASS];
    double alg_bytes[GSI_N_KCLASS];
    uint32_t total_launches;          /* kernels this library launched for the query         */
    uint32_t n_chunks;                /* slot-range chunks executed below the memory budget   */
    int32_t capped;                   /* 1: timed out with partial_on_timeout                 */
    uint64_t h2d_bytes, d2h_bytes;    /* host<->device bytes this query copied                */
    uint32_t n_shared_lists;          /* levels that enumerated shared N(v,l0) ∩ C(u) lists   */
    float ms_host_alloc, ms_host_sync; /* host time in stream-ordered allocation / stream syncs */
    int32_t count_ahead;              /* 1: the last level was counted by the level before it    */
    uint32_t n_probe_ahead;           /* levels whose next-step locate came from a per-candidate
                                         probe-ahead table instead of a PCSR probe per new row   */
    uint32_t variant_launches[GSI_N_KVARIANT]; /* launches per kernel variant (GSI_V_*)         */
    /* profile mode, per kernel variant: summed device ms and algorithmic bytes (the bytes the
       variant must move at least once: rows, loc/F, output rows, candidates streamed from ci,
       one 32 B sector + fpos per PCSR lookup)                                   */
    float ms_variant[GSI_N_KVARIANT];
    double alg_bytes_variant[GSI_N_KVARIANT];
    int32_t small_aborted;            /* the small-query kernel stopped at this level (0: not)  */
    uint64_t abl_layer_rows[3];       /* ablation engine: rows per balance layer (warp / block /
                                         8-CTA cluster), summed over levels                      */
    uint64_t items_variant[GSI_N_KVARIANT]; /* per kernel variant: matches it produced (last
                                         level / count-ahead) or rows it stored (J_NEXT)          */
} gsi_stats;

gsi_status gsi_result_count(const gsi_result *r, uint64_t *count);
/* Order-independent set fingerprint (|R|, sum h1(row), xor h2(row)) over the final rows in
 * query-id order; computed on the device even in count-only mode. */
gsi_status gsi_result_fingerprint(const gsi_result *r, uint64_t fp[3]);
/* Device pointer to the table (nrows x k int32, query-id order), valid until free; rows
 * are strictly increasing in join-order (pi) column order. Requires want_table. */
gsi_status gsi_result_table(const gsi_result *r, const int32_t **dev_rows, uint64_t *nrows);
/* Copy the table to host memory (cap rows of k int32). */
gsi_status gsi_result_copy_table(const gsi_result *r, int32_t *host_rows, uint64_t cap);
gsi_status gsi_result_stats(const gsi_result *r, gsi_stats *stats);
void gsi_result_free(gsi_result *r);

/* ------------------------------------------------------------------ test hooks ------ */
/* Batch PCSR lookups through the join kernels' device lookup: for each (v[i], l[i]) (raw
 * edge label) writes len[i] = |N(v,l)| and groups_read[i] (chain length walked); the
 * neighbour runs are concatenated into nbrs (capacity cap) in query order. */
gsi_status gsi_debug_lookup(const gsi_graph *g, int64_t nq, const int32_t *v, const int32_t *l,
                            int64_t *len, int32_t *groups_read, int32_t *nbrs, int64_t cap);
/* Copy the column-first signature table (16 x n uint32) to host. */
gsi_status gsi_debug_signatures(const gsi_graph *g, uint32_t *planes);
/* Run only the filter kernel: bitmaps (k x ceil(n/32) uint32) and |C(u)| to host.
 * filter_mode 0 = signatures (isomorphism encoding), 1 = label only, 2 = signatures with the
 * homomorphism (distinct-key) query encoding. */
gsi_status gsi_debug_filter(const gsi_graph *g, int32_t k, const int32_t *q_vlabels, int32_t qm,
                            const int32_t *q_src, const int32_t *q_dst, const int32_t *q_elabels,
                            int32_t filter_mode, uint32_t *bitmaps, int64_t *counts);
/* Host query signatures (k x 16 uint32) as encoded by the library; distinct = 1 gives the
 * homomorphism encoding (each (edge label, neighbour label) key counted once). */
/* Test hook: C(u) bitmaps / counts of a prepared query (any kind: single-label, multi-label
 * with its refine step, line graph); mode 0 = isomorphism signatures, 2 = homomorphism. */
gsi_status gsi_debug_filter_prepared(const gsi_prepared *q, int32_t mode, uint32_t *bitmaps, int64_t *counts);
gsi_status gsi_debug_query_signatures(int32_t k, const int32_t *q_vlabels, int32_t qm,
                                      const int32_t *q_src, const int32_t *q_dst,
                                      const int32_t *q_elabels, int32_t distinct, uint32_t *qsig);

/* The hash functions of the written spec, evaluated by the library's own code
 * (host side of the __host__ __device__ functions the kernels use), for known-answer tests:
 * kind 0 = MurmurHash2 of the 4 LE bytes of (uint32)key with (uint32)seed (PCSR group f),
 * kind 1 = MurmurHash64A of the 8 LE bytes of key (signature groups), kind 2 = the fingerprint
 * finaliser mix(key) (seed ignored).  Pure host computation: needs no device.  Unknown kind -> 0. */
uint64_t gsi_debug_hash(int32_t kind, uint64_t key, uint64_t seed);

/* ------------------------------------------------------------------ memory ---------- */
/* Queries keep one device workspace per device between calls (a double-ended stack the
 * level recursion carves; re-allocating it per level cost more than the kernels).  Free an
 * idle workspace now (device -1 = current).  Graph builds do this themselves.  Never fails. */
void gsi_trim_workspace(int32_t device);

/* ------------------------------------------------------------------ misc ------------ */
const char *gsi_last_error(void);
const char *gsi_version(void);
/* Number of CUDA devices visible (0 when none); never fails. */
int32_t gsi_device_count(void);

#ifdef __cplusplus
}
#endif
#endif /* GSI_H */
