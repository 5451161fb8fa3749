/*
 * oracle.c — plain, slow, obviously-correct CPU reference for the GSI hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with paper_1906_03420_b200/csrc (the CUDA path);
 * the two implement the same written specification independently.
 *
 * What it computes (Def. 2-3; N(v,l) at L299):
 *   R(Q,G) = { f : V(Q) -> V(G) |  f injective,
 *                                   L_V(f(u)) = L_V(u) for every u,
 *                                   every query edge (a,b,l) has an undirected data
 *                                   edge {f(a), f(b)} labelled l }.
 *   (non-induced / monomorphism reading A1; a match is a mapping, reading A2.)
 *   Injectivity is the set subtraction of Alg. 3 line 10;
 *   dropping it gives homomorphism (flag `hom`).
 *
 * Algorithm: the classic backtracking search tree (Fig. 2; L430) with a
 * static BFS query order from a root query vertex (ties to the smallest id), candidates
 * from the sorted l-adjacency of the earliest-ordered already-mapped neighbour, and
 * checks for label, injectivity and every other query edge to a mapped vertex (binary
 * search in the per-vertex (label, neighbour)-sorted adjacency).  OpenMP over root
 * candidates (dynamic schedule) for timing only.
 *
 * Also here: an independent re-implementation of the signature filter specification
 * (§III-A; stored-label field L1277; N=512, K=32 at L1420; readings
 * A4/A5/A6 of SURVEY.md §8(c)) used only to compare C(u) bitmaps bit for bit, and the
 * order-independent set fingerprint of SURVEY.md §8(c).
 *
 * Parity pins: see tests/test_oracle.py (Fig. 1 reconstruction, closed forms, brute force
 * over all injective maps on tiny graphs, signature properties).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OG_MAXK 32
#define OG_MAXLS 32                /* labels per query vertex (multi-label queries)    */

/* ---------------------------------------------------------------- graph index ------ */
typedef struct {
    int64_t n, m;
    int32_t *vl;        /* vertex labels                                             */
    int64_t *off;       /* n+1 offsets into adj                                      */
    int64_t *adj;       /* packed ((uint64)label << 32) | (uint32)neighbour, sorted  */
    int64_t *eid;       /* eid[j] = input index of the edge of adjacency entry j     */
    int64_t *lsoff;     /* optional vertex label SETS (multi-label): */
    int32_t *ls;        /*   L_V(v) = ls[lsoff[v] .. lsoff[v+1]), ascending; or NULL */
} og_graph;

typedef struct { uint64_t key; int64_t eid; } og_entry;
static int cmp_entry(const void *a, const void *b) {
    uint64_t x = ((const og_entry *)a)->key, y = ((const og_entry *)b)->key;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* err: 0 ok, -1 bad arg, -2 vertex range, -3 label range, -4 self loop, -5 duplicate */
og_graph *og_build(int64_t n, const int32_t *vl, int64_t m, const int32_t *src,
                   const int32_t *dst, const int32_t *el, int32_t *err) {
    *err = 0;
    if (n < 0 || m < 0) { *err = -1; return NULL; }
    for (int64_t i = 0; i < n; i++) if (vl[i] < 0) { *err = -3; return NULL; }
    for (int64_t e = 0; e < m; e++) {
        if (src[e] < 0 || src[e] >= n || dst[e] < 0 || dst[e] >= n) { *err = -2; return NULL; }
        if (el[e] < 0) { *err = -3; return NULL; }
        if (src[e] == dst[e]) { *err = -4; return NULL; }
    }
    og_graph *g = (og_graph *)calloc(1, sizeof(og_graph));
    g->n = n; g->m = m;
    g->vl = (int32_t *)malloc(sizeof(int32_t) * (n > 0 ? n : 1));
    memcpy(g->vl, vl, sizeof(int32_t) * n);
    g->off = (int64_t *)calloc(n + 1, sizeof(int64_t));
    g->adj = (int64_t *)malloc(sizeof(int64_t) * (2 * m > 0 ? 2 * m : 1));
    g->eid = (int64_t *)malloc(sizeof(int64_t) * (2 * m > 0 ? 2 * m : 1));
    og_entry *ent = (og_entry *)malloc(sizeof(og_entry) * (2 * m > 0 ? 2 * m : 1));
    for (int64_t e = 0; e < m; e++) { g->off[src[e] + 1]++; g->off[dst[e] + 1]++; }
    for (int64_t v = 0; v < n; v++) g->off[v + 1] += g->off[v];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    memcpy(fill, g->off, sizeof(int64_t) * n);
    for (int64_t e = 0; e < m; e++) {
        uint64_t l = (uint64_t)(uint32_t)el[e] << 32;
        og_entry a = {l | (uint32_t)dst[e], e}, b = {l | (uint32_t)src[e], e};
        ent[fill[src[e]]++] = a;
        ent[fill[dst[e]]++] = b;
    }
    free(fill);
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t v = 0; v < n; v++)
        qsort(ent + g->off[v], (size_t)(g->off[v + 1] - g->off[v]), sizeof(og_entry), cmp_entry);
    for (int64_t j = 0; j < 2 * m; j++) { g->adj[j] = (int64_t)ent[j].key; g->eid[j] = ent[j].eid; }
    free(ent);
    for (int64_t v = 0; v < n && !*err; v++)
        for (int64_t j = g->off[v] + 1; j < g->off[v + 1]; j++)
            if (g->adj[j] == g->adj[j - 1]) { *err = -5; break; }
    if (*err) { free(g->vl); free(g->off); free(g->adj); free(g->eid); free(g); return NULL; }
    return g;
}

void og_free(og_graph *g) {
    if (!g) return;
    free(g->vl); free(g->off); free(g->adj); free(g->eid); free(g->lsoff); free(g->ls); free(g);
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* Attach vertex label SETS (§VII-B): L_V(v) = labs[off[v] .. off[v+1]).
 * Each set is stored ascending without repeats; every label must be >= 0.  Returns 0 or -3. */
int32_t og_set_label_sets(og_graph *g, const int64_t *off, const int32_t *labs) {
    int64_t tot = off[g->n];
    for (int64_t i = 0; i < tot; i++) if (labs[i] < 0) return -3;
    free(g->lsoff); free(g->ls);
    g->lsoff = (int64_t *)malloc(sizeof(int64_t) * (g->n + 1));
    g->ls = (int32_t *)malloc(sizeof(int32_t) * (tot > 0 ? tot : 1));
    int64_t w = 0;
    for (int64_t v = 0; v < g->n; v++) {
        g->lsoff[v] = w;
        int64_t b = off[v], c = off[v + 1] - off[v];
        memcpy(g->ls + w, labs + b, sizeof(int32_t) * c);
        qsort(g->ls + w, (size_t)c, sizeof(int32_t), cmp_i32);
        int64_t u = 0;
        for (int64_t i = 0; i < c; i++) if (u == 0 || g->ls[w + i] != g->ls[w + u - 1]) g->ls[w + u++] = g->ls[w + i];
        w += u;
    }
    g->lsoff[g->n] = w;
    return 0;
}

/* N(v,l) as a half-open index range [*b, *e) into g->adj. */
static void og_nbrs(const og_graph *g, int32_t v, int32_t l, int64_t *b, int64_t *e) {
    uint64_t lo_key = (uint64_t)(uint32_t)l << 32;
    uint64_t hi_key = lo_key | 0xFFFFFFFFull;
    int64_t lo = g->off[v], hi = g->off[v + 1];
    while (lo < hi) { int64_t mid = (lo + hi) >> 1; if ((uint64_t)g->adj[mid] < lo_key) lo = mid + 1; else hi = mid; }
    *b = lo;
    hi = g->off[v + 1];
    while (lo < hi) { int64_t mid = (lo + hi) >> 1; if ((uint64_t)g->adj[mid] <= hi_key) lo = mid + 1; else hi = mid; }
    *e = lo;
}

static int og_has_edge(const og_graph *g, int32_t v, int32_t w, int32_t l) {
    uint64_t key = ((uint64_t)(uint32_t)l << 32) | (uint32_t)w;
    int64_t lo = g->off[v], hi = g->off[v + 1];
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        uint64_t x = (uint64_t)g->adj[mid];
        if (x == key) return 1;
        if (x < key) lo = mid + 1; else hi = mid;
    }
    return 0;
}

int64_t og_degree(const og_graph *g, int32_t v) { return g->off[v + 1] - g->off[v]; }

/* Label-filtered adjacency N(v,l), ascending; returns |N(v,l)|, writes up to cap ids. */
int64_t og_neighbors(const og_graph *g, int32_t v, int32_t l, int32_t *out, int64_t cap) {
    int64_t b, e;
    og_nbrs(g, v, l, &b, &e);
    for (int64_t j = b; j < e && j - b < cap; j++) out[j - b] = (int32_t)(uint32_t)g->adj[j];
    return e - b;
}

/* ------------------------------------------------------------- fingerprint ------- */
/* SURVEY.md §8(c) 'Set fingerprint': FP(R) = (|R|, sum_rows h1(row) mod 2^64,
 * xor_rows h2(row)), rows in query-id order (DESIGN.md §3 'Fingerprint').  A row's hash
 * with seed s: S = sum over columns c of mix(s ^ (c+1) << 32 ^ (uint32)row[c]) mod 2^64,
 * h = mix(S), mix = the splitmix64 finaliser.  Sum/xor over rows: order-free.          */
#define OG_FP_SEED1 0x243F6A8885A308D3ull
#define OG_FP_SEED2 0x13198A2E03707344ull
static uint64_t og_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t og_rowhash(const int32_t *row, int32_t k, uint64_t seed) {
    uint64_t S = 0;
    for (int32_t c = 0; c < k; c++)
        S += og_mix64(seed ^ ((uint64_t)(uint32_t)(c + 1) << 32) ^ (uint64_t)(uint32_t)row[c]);
    return og_mix64(S);
}
void og_fingerprint_rows(const int32_t *rows, int64_t nrows, int32_t k, uint64_t fp[3]) {
    fp[0] = (uint64_t)nrows; fp[1] = 0; fp[2] = 0;
    for (int64_t i = 0; i < nrows; i++) {
        fp[1] += og_rowhash(rows + i * k, k, OG_FP_SEED1);
        fp[2] ^= og_rowhash(rows + i * k, k, OG_FP_SEED2);
    }
}

/* --------------------------------------------------------------- backtracker ----- */
typedef struct {
    int32_t k;
    int32_t order[OG_MAXK];          /* order[j] = query vertex at depth j                */
    int32_t depth_of[OG_MAXK];
    int32_t qlabel[OG_MAXK];
    int32_t parent[OG_MAXK];         /* depth of the earliest-ordered mapped neighbour    */
    int32_t plabel[OG_MAXK];         /* label of the (parent, u) edge used to enumerate   */
    int32_t nchk[OG_MAXK];           /* other edges to mapped vertices: (depth, label)    */
    int32_t chk_depth[OG_MAXK][2 * OG_MAXK * 4];
    int32_t chk_label[OG_MAXK][2 * OG_MAXK * 4];
    int32_t hom;
    int32_t ml;                      /* multi-label: L_V(u) ⊆ L_V(f(u))  */
    int32_t qlsn[OG_MAXK];           /* |L_V(order[j])| and its labels, ascending         */
    int32_t qls[OG_MAXK][OG_MAXLS];
} og_plan;

/* The vertex-label condition of depth j: L_V(x) = L_V(u) (Def. 2), or with label sets
 * L_V(u) ⊆ L_V(x) (the multi-label definition). */
static int og_label_ok(const og_graph *g, const og_plan *p, int32_t x, int32_t j) {
    if (!p->ml) return g->vl[x] == p->qlabel[j];
    int64_t a = g->lsoff[x], b = g->lsoff[x + 1];
    for (int32_t i = 0; i < p->qlsn[j]; i++) {
        while (a < b && g->ls[a] < p->qls[j][i]) a++;
        if (a == b || g->ls[a] != p->qls[j][i]) return 0;
        a++;
    }
    return 1;
}

/* err: -1 bad arg, -6 disconnected, -7 too large */
static int og_make_plan(int32_t k, const int32_t *qvl, int32_t qm, const int32_t *qs,
                        const int32_t *qd, const int32_t *qe, int32_t root, int32_t hom, og_plan *p) {
    if (k < 1) return -1;
    if (k > OG_MAXK) return -7;
    if (qm > 4 * OG_MAXK * OG_MAXK) return -7;
    if (root < 0 || root >= k) return -1;
    memset(p, 0, sizeof(*p));
    p->k = k; p->hom = hom;
    for (int32_t e = 0; e < qm; e++) {
        if (qs[e] < 0 || qs[e] >= k || qd[e] < 0 || qd[e] >= k || qs[e] == qd[e] || qe[e] < 0) return -1;
    }
    /* BFS order from root, neighbours visited in increasing id (ties to the smallest id). */
    int32_t seen[OG_MAXK] = {0}, head = 0, tail = 0;
    p->order[tail++] = root; seen[root] = 1;
    while (head < tail) {
        int32_t u = p->order[head++];
        for (int32_t w = 0; w < k; w++) {
            if (seen[w]) continue;
            for (int32_t e = 0; e < qm; e++)
                if ((qs[e] == u && qd[e] == w) || (qd[e] == u && qs[e] == w)) { seen[w] = 1; p->order[tail++] = w; break; }
        }
    }
    if (tail != k) return -6;
    for (int32_t j = 0; j < k; j++) { p->depth_of[p->order[j]] = j; p->qlabel[j] = qvl[p->order[j]]; }
    for (int32_t j = 0; j < k; j++) {
        int32_t u = p->order[j];
        p->parent[j] = -1; p->plabel[j] = -1; p->nchk[j] = 0;
        /* parent: earliest-ordered neighbour at a smaller depth; its smallest-label edge */
        for (int32_t e = 0; e < qm; e++) {
            int32_t o = qs[e] == u ? qd[e] : (qd[e] == u ? qs[e] : -1);
            if (o < 0) continue;
            int32_t d = p->depth_of[o];
            if (d >= j) continue;
            if (p->parent[j] < 0 || d < p->parent[j] || (d == p->parent[j] && qe[e] < p->plabel[j])) {
                p->parent[j] = d; p->plabel[j] = qe[e];
            }
        }
        for (int32_t e = 0; e < qm; e++) {
            int32_t o = qs[e] == u ? qd[e] : (qd[e] == u ? qs[e] : -1);
            if (o < 0) continue;
            int32_t d = p->depth_of[o];
            if (d >= j) continue;
            if (d == p->parent[j] && qe[e] == p->plabel[j]) continue;   /* the enumerated edge */
            if (p->nchk[j] >= 2 * OG_MAXK * 4) return -7;
            p->chk_depth[j][p->nchk[j]] = d;
            p->chk_label[j][p->nchk[j]] = qe[e];
            p->nchk[j]++;
        }
    }
    return 0;
}

typedef struct {
    int64_t count;
    uint64_t fp1, fp2;
    int32_t *rows; int64_t nrows, cap;   /* collected rows, query-id order */
    int64_t steps;
    int timed_out;
} og_acc;

static void og_emit(og_acc *a, const og_plan *p, const int32_t *f) {
    int32_t row[OG_MAXK];
    for (int32_t j = 0; j < p->k; j++) row[p->order[j]] = f[j];
    a->count++;
    a->fp1 += og_rowhash(row, p->k, OG_FP_SEED1);
    a->fp2 ^= og_rowhash(row, p->k, OG_FP_SEED2);
    if (a->cap > 0) {
        if (a->nrows == a->cap) {
            int64_t nc = a->cap * 2;
            a->rows = (int32_t *)realloc(a->rows, sizeof(int32_t) * nc * p->k);
            a->cap = nc;
        }
        memcpy(a->rows + a->nrows * p->k, row, sizeof(int32_t) * p->k);
        a->nrows++;
    }
}

static double og_now(void) {
#ifdef _OPENMP
    return omp_get_wtime();
#else
    return 0.0;
#endif
}

/* Depth-first extension of a partial map f[0..1) rooted at data vertex v0. */
static void og_search_root(const og_graph *g, const og_plan *p, int32_t v0, og_acc *a, double deadline) {
    int32_t f[OG_MAXK];
    int64_t cur[OG_MAXK], end[OG_MAXK];
    int32_t k = p->k;
    if (!og_label_ok(g, p, v0, 0)) return;
    f[0] = v0;
    if (k == 1) { og_emit(a, p, f); return; }
    int32_t j = 1;
    og_nbrs(g, f[p->parent[1]], p->plabel[1], &cur[1], &end[1]);
    while (j >= 1) {
        if (cur[j] >= end[j]) { j--; continue; }
        int32_t x = (int32_t)(uint32_t)g->adj[cur[j]++];
        if (((++a->steps) & 0xFFFF) == 0 && deadline > 0 && og_now() > deadline) { a->timed_out = 1; return; }
        if (!og_label_ok(g, p, x, j)) continue;
        int ok = 1;
        if (!p->hom)
            for (int32_t i = 0; i < j && ok; i++) if (f[i] == x) ok = 0;
        for (int32_t c = 0; c < p->nchk[j] && ok; c++)
            if (!og_has_edge(g, x, f[p->chk_depth[j][c]], p->chk_label[j][c])) ok = 0;
        if (!ok) continue;
        f[j] = x;
        if (j == k - 1) { og_emit(a, p, f); continue; }
        j++;
        og_nbrs(g, f[p->parent[j]], p->plabel[j], &cur[j], &end[j]);
    }
}

static int cmp_rows_k;
static int cmp_rows(const void *a, const void *b) {
    const int32_t *x = (const int32_t *)a, *y = (const int32_t *)b;
    for (int c = 0; c < cmp_rows_k; c++) { if (x[c] != y[c]) return x[c] < y[c] ? -1 : 1; }
    return 0;
}

/*
 * og_match: enumerate R(Q,G).
 *   root       query vertex the BFS order starts from (default 0).
 *   roots      optional subset S of data vertices: only maps with f(root) in S (root-restricted
 *              parity); NULL = all vertices.
 *   table/cap  if table != NULL, up to cap rows (k int32 each, query-id order, sorted
 *              lexicographically) are written.
 *   fp         out: (count, sum-hash, xor-hash).
 *   timeout_s  <= 0: none.  On timeout returns -9 and fp holds the partial result.
 * Returns the count (>= 0) or a negative error code.
 */
static int64_t og_match_impl(const og_graph *g, int32_t k, const int32_t *qvl, const int32_t *qlsoff,
                             const int32_t *qls, int32_t qm, const int32_t *qs, const int32_t *qd,
                             const int32_t *qe, int32_t root, const int32_t *roots, int64_t nroots,
                             int32_t nthreads, int32_t hom, int32_t *table, int64_t cap, uint64_t fp[3],
                             double timeout_s) {
    og_plan p;
    int rc = og_make_plan(k, qvl, qm, qs, qd, qe, root, hom, &p);
    if (rc) return rc;
    if (qlsoff) {   /* multi-label query: the label SETS of its vertices, in depth order */
        if (!g->lsoff) return -1;
        p.ml = 1;
        for (int32_t j = 0; j < k; j++) {
            int32_t u = p.order[j], c = qlsoff[u + 1] - qlsoff[u];
            if (c < 0 || c > OG_MAXLS) return -7;
            memcpy(p.qls[j], qls + qlsoff[u], sizeof(int32_t) * c);
            qsort(p.qls[j], (size_t)c, sizeof(int32_t), cmp_i32);
            int32_t w = 0;
            for (int32_t i = 0; i < c; i++) {
                if (p.qls[j][i] < 0) return -3;
                if (w == 0 || p.qls[j][i] != p.qls[j][w - 1]) p.qls[j][w++] = p.qls[j][i];
            }
            p.qlsn[j] = w;
        }
    }
    int64_t ncand = roots ? nroots : g->n;
    int want_rows = table != NULL;
    double deadline = timeout_s > 0 ? og_now() + timeout_s : 0;
    int64_t total = 0; uint64_t s1 = 0, s2 = 0; int timed_out = 0;
    int32_t *all = NULL; int64_t nall = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    #pragma omp parallel
    {
        og_acc a; memset(&a, 0, sizeof(a));
        if (want_rows) { a.cap = 64; a.rows = (int32_t *)malloc(sizeof(int32_t) * 64 * k); }
        #pragma omp for schedule(dynamic, 16) nowait
        for (int64_t i = 0; i < ncand; i++) {
            if (a.timed_out) continue;
            int32_t v0 = roots ? roots[i] : (int32_t)i;
            if (v0 < 0 || v0 >= g->n) continue;
            og_search_root(g, &p, v0, &a, deadline);
        }
        #pragma omp critical
        {
            total += a.count; s1 += a.fp1; s2 ^= a.fp2; timed_out |= a.timed_out;
            if (want_rows && a.nrows) {
                all = (int32_t *)realloc(all, sizeof(int32_t) * (nall + a.nrows) * k);
                memcpy(all + nall * k, a.rows, sizeof(int32_t) * a.nrows * k);
                nall += a.nrows;
            }
        }
        free(a.rows);
    }
    if (want_rows) {
        cmp_rows_k = k;
        qsort(all, (size_t)nall, sizeof(int32_t) * k, cmp_rows);
        int64_t w = nall < cap ? nall : cap;
        if (w > 0) memcpy(table, all, sizeof(int32_t) * w * k);
        free(all);
    }
    fp[0] = (uint64_t)total; fp[1] = s1; fp[2] = s2;
    return timed_out ? -9 : total;
}

int64_t og_match(const og_graph *g, int32_t k, const int32_t *qvl, int32_t qm, const int32_t *qs,
                 const int32_t *qd, const int32_t *qe, int32_t root, const int32_t *roots,
                 int64_t nroots, int32_t nthreads, int32_t hom, int32_t *table, int64_t cap,
                 uint64_t fp[3], double timeout_s) {
    return og_match_impl(g, k, qvl, NULL, NULL, qm, qs, qd, qe, root, roots, nroots, nthreads, hom, table, cap, fp,
                         timeout_s);
}

/* Multi-label vertices (§VII-B): as og_match with L_V(u) ⊆ L_V(f(u)),
 * query label sets qls[qlsoff[u] .. qlsoff[u+1]) (the graph needs og_set_label_sets).
 * Multi-label EDGES need no change here: a query edge whose label set is S asks for a data
 * edge {f(a),f(b)} carrying every l in S (L_E(uv) ⊆ L_E(f(u)f(v)), L1275), i.e. one parallel
 * single-label query edge per l (L1283-1285), which og_match already checks. */
int64_t og_match_ml(const og_graph *g, int32_t k, const int32_t *qlsoff, const int32_t *qls, int32_t qm,
                    const int32_t *qs, const int32_t *qd, const int32_t *qe, int32_t root, const int32_t *roots,
                    int64_t nroots, int32_t nthreads, int32_t hom, int32_t *table, int64_t cap, uint64_t fp[3],
                    double timeout_s) {
    int32_t zero[OG_MAXK] = {0};
    if (k < 1 || k > OG_MAXK) return k < 1 ? -1 : -7;
    return og_match_impl(g, k, zero, qlsoff, qls, qm, qs, qd, qe, root, roots, nroots, nthreads, hom, table, cap,
                         fp, timeout_s);
}

/* ------------------------------------------------------------ edge isomorphism ------ */
/* PAPER.md §VII-A L1255-1264 (Fig. 9): edge isomorphism asks that two query edges share a
 * vertex iff their images share a vertex; GSI reaches it by running vertex isomorphism on
 * line graphs.  What that computes, written on G and Q directly (reading A18):
 *   R_E(Q,G) = { h : E(Q) -> E(G) injective |  L_E(h(e)) = L_E(e) for every e, and for every
 *                two query edges e1 != e2 sharing a vertex w, h(e1) and h(e2) share a vertex
 *                v with L_V(v) = L_V(w) }.
 * Rows: h(e) for e = 0 .. |E(Q)|-1 (data edge = its index in the input edge list).
 * Backtracking over query edges in BFS order of the query's edge adjacency (from edge 0,
 * ties to the smallest id); a non-first edge enumerates the l-labelled edges incident to the
 * endpoints of its earliest-ordered adjacent edge's image, then checks injectivity and every
 * earlier adjacent edge's shared-vertex condition. */
typedef struct {
    int32_t k;                         /* |E(Q)| */
    int32_t order[OG_MAXK], depth_of[OG_MAXK];
    int32_t elab[OG_MAXK];             /* query edge label, by depth */
    int32_t parent[OG_MAXK];           /* depth of the earliest adjacent edge (-1: first) */
    int32_t plab[OG_MAXK];             /* label of one vertex it shares with that edge    */
    int32_t nchk[OG_MAXK];
    int32_t chk_depth[OG_MAXK][4 * OG_MAXK], chk_vlab[OG_MAXK][4 * OG_MAXK];
} og_eplan;

static int og_shares_label(const int32_t *ea, const int32_t *eb, const int32_t *vl, int32_t lab) {
    for (int i = 0; i < 2; i++)
        for (int j = 0; j < 2; j++)
            if (ea[i] == eb[j] && vl[ea[i]] == lab) return 1;
    return 0;
}

int64_t og_match_edges(const og_graph *g, const int32_t *gsrc, const int32_t *gdst, const int32_t *gel, int32_t qn,
                       const int32_t *qvl,
                       int32_t qm, const int32_t *qs, const int32_t *qd, const int32_t *qe, int32_t *table,
                       int64_t cap, uint64_t fp[3], double timeout_s) {
    og_eplan p;
    if (qm < 1) return -1;
    if (qm > OG_MAXK) return -7;
    for (int32_t e = 0; e < qm; e++)
        if (qs[e] < 0 || qs[e] >= qn || qd[e] < 0 || qd[e] >= qn || qs[e] == qd[e] || qe[e] < 0) return -1;
    memset(&p, 0, sizeof(p));
    p.k = qm;
    int32_t seen[OG_MAXK] = {0}, head = 0, tail = 0;
    p.order[tail++] = 0; seen[0] = 1;
    while (head < tail) {
        int32_t a = p.order[head++];
        for (int32_t b = 0; b < qm; b++) {
            if (seen[b]) continue;
            if (qs[a] == qs[b] || qs[a] == qd[b] || qd[a] == qs[b] || qd[a] == qd[b]) { seen[b] = 1; p.order[tail++] = b; }
        }
    }
    if (tail != qm) return -6;
    for (int32_t j = 0; j < qm; j++) { p.depth_of[p.order[j]] = j; p.elab[j] = qe[p.order[j]]; }
    for (int32_t j = 0; j < qm; j++) {
        int32_t b = p.order[j];
        p.parent[j] = -1;
        for (int32_t i = 0; i < j; i++) {
            int32_t a = p.order[i];
            int32_t ends_a[2] = {qs[a], qd[a]}, ends_b[2] = {qs[b], qd[b]};
            for (int x = 0; x < 2; x++)
                for (int y = 0; y < 2; y++) {
                    if (ends_a[x] != ends_b[y]) continue;
                    if (p.parent[j] < 0) { p.parent[j] = i; p.plab[j] = qvl[ends_a[x]]; }
                    p.chk_depth[j][p.nchk[j]] = i;
                    p.chk_vlab[j][p.nchk[j]] = qvl[ends_a[x]];
                    p.nchk[j]++;
                }
        }
    }
    double deadline = timeout_s > 0 ? og_now() + timeout_s : 0;
    og_acc a; memset(&a, 0, sizeof(a));
    int want_rows = table != NULL;
    if (want_rows) { a.cap = 64; a.rows = (int32_t *)malloc(sizeof(int32_t) * 64 * qm); }
    og_plan emit_plan; memset(&emit_plan, 0, sizeof(emit_plan));   /* og_emit: depth -> query edge id */
    emit_plan.k = qm;
    for (int32_t j = 0; j < qm; j++) emit_plan.order[j] = p.order[j];
    int32_t h[OG_MAXK];
    int32_t cand_v[OG_MAXK][2];        /* the two endpoints whose incident edges depth j scans */
    int64_t cur[OG_MAXK], end[OG_MAXK];
    int32_t side[OG_MAXK];
    for (int64_t e0 = 0; e0 < g->m && !a.timed_out; e0++) {
        if (gel[e0] != p.elab[0]) continue;   /* depth 0: every data edge with its label */
        h[0] = (int32_t)e0;
        if (qm == 1) { og_emit(&a, &emit_plan, h); continue; }
        int32_t j = 1;
        side[j] = 0;
        cand_v[j][0] = gsrc[h[p.parent[j]]]; cand_v[j][1] = gdst[h[p.parent[j]]];
        og_nbrs(g, cand_v[j][0], p.elab[j], &cur[j], &end[j]);
        while (j >= 1) {
            if (cur[j] >= end[j]) {
                if (side[j] == 0) {
                    side[j] = 1;
                    og_nbrs(g, cand_v[j][1], p.elab[j], &cur[j], &end[j]);
                    continue;
                }
                j--;
                continue;
            }
            int64_t pos = cur[j]++;
            int32_t x = (int32_t)g->eid[pos];
            if (((++a.steps) & 0xFFFF) == 0 && deadline > 0 && og_now() > deadline) { a.timed_out = 1; break; }
            int32_t ex[2] = {gsrc[x], gdst[x]};
            /* scanned from both endpoints of the parent image: enumerate an edge once */
            if (side[j] == 1 && (ex[0] == cand_v[j][0] || ex[1] == cand_v[j][0])) continue;
            int ok = 1;
            for (int32_t i = 0; i < j && ok; i++) if (h[i] == x) ok = 0;
            for (int32_t c = 0; c < p.nchk[j] && ok; c++) {
                int32_t y = h[p.chk_depth[j][c]];
                int32_t ey[2] = {gsrc[y], gdst[y]};
                if (!og_shares_label(ex, ey, g->vl, p.chk_vlab[j][c])) ok = 0;
            }
            if (!ok) continue;
            h[j] = x;
            if (j == qm - 1) { og_emit(&a, &emit_plan, h); continue; }
            j++;
            side[j] = 0;
            cand_v[j][0] = gsrc[h[p.parent[j]]]; cand_v[j][1] = gdst[h[p.parent[j]]];
            og_nbrs(g, cand_v[j][0], p.elab[j], &cur[j], &end[j]);
        }
    }
    if (want_rows) {
        cmp_rows_k = qm;
        qsort(a.rows, (size_t)a.nrows, sizeof(int32_t) * qm, cmp_rows);
        int64_t w = a.nrows < cap ? a.nrows : cap;
        if (w > 0) memcpy(table, a.rows, sizeof(int32_t) * w * qm);
    }
    free(a.rows);
    fp[0] = (uint64_t)a.count; fp[1] = a.fp1; fp[2] = a.fp2;
    return a.timed_out ? -9 : a.count;
}

/* ------------------------------------------------------- signature specification -- */
/* MurmurHash64A (Appleby, MurmurHash2 64-bit) over the 8 little-endian bytes of key.   */
static uint64_t og_murmur64a_u64(uint64_t key, uint64_t seed) {
    const uint64_t m = 0xc6a4a7935bd1e995ull;
    const int r = 47;
    uint64_t h = seed ^ (8ull * m);
    uint64_t k = key;
    k *= m; k ^= k >> r; k *= m;
    h ^= k; h *= m;
    h ^= h >> r; h *= m; h ^= h >> r;
    return h;
}

/* Appleby's MurmurHash2 (32-bit) and MurmurHash64A over an arbitrary byte string, restated
 * from the public-domain reference algorithm.  They pin the hash functions of the written
 * signature/PCSR spec (reading A6/A7) against external known answers: SMHasher's
 * verification value (hash the keys {}, {0}, {0,1}, ..., {0..254} with seed 256 - len, then
 * hash the concatenated results with seed 0) is 0x27864C1E for MurmurHash2 and 0x1F0D3804 for
 * MurmurHash64A.  og_murmur64a_u64 above must equal og_murmur64a_bytes on 8 LE bytes.        */
uint32_t og_murmur2_bytes(const uint8_t *data, int64_t len, uint32_t seed) {
    const uint32_t m = 0x5bd1e995u;
    uint32_t h = seed ^ (uint32_t)len;
    while (len >= 4) {
        uint32_t k = (uint32_t)data[0] | (uint32_t)data[1] << 8 | (uint32_t)data[2] << 16 | (uint32_t)data[3] << 24;
        k *= m; k ^= k >> 24; k *= m;
        h *= m; h ^= k;
        data += 4; len -= 4;
    }
    if (len == 3) h ^= (uint32_t)data[2] << 16;
    if (len >= 2) h ^= (uint32_t)data[1] << 8;
    if (len >= 1) { h ^= data[0]; h *= m; }
    h ^= h >> 13; h *= m; h ^= h >> 15;
    return h;
}
uint64_t og_murmur64a_bytes(const uint8_t *data, int64_t len, uint64_t seed) {
    const uint64_t m = 0xc6a4a7935bd1e995ull;
    uint64_t h = seed ^ ((uint64_t)len * m);
    int64_t nblk = len / 8;
    for (int64_t b = 0; b < nblk; b++) {
        uint64_t k = 0;
        for (int j = 7; j >= 0; j--) k = (k << 8) | data[8 * b + j];
        k *= m; k ^= k >> 47; k *= m;
        h ^= k; h *= m;
    }
    const uint8_t *t = data + 8 * nblk;
    int rem = (int)(len & 7);
    if (rem) {
        for (int j = rem - 1; j >= 0; j--) h ^= (uint64_t)t[j] << (8 * j);
        h *= m;
    }
    h ^= h >> 47; h *= m; h ^= h >> 47;
    return h;
}
/* SMHasher's VerificationTest: which = 0 MurmurHash2, 1 MurmurHash64A. */
uint32_t og_smhasher_verify(int32_t which) {
    uint8_t key[256], hashes[256 * 8];
    const int hb = which ? 8 : 4;
    for (int i = 0; i < 256; i++) {
        key[i] = (uint8_t)i;
        if (which) {
            uint64_t h = og_murmur64a_bytes(key, i, (uint64_t)(256 - i));
            for (int j = 0; j < 8; j++) hashes[8 * i + j] = (uint8_t)(h >> (8 * j));
        } else {
            uint32_t h = og_murmur2_bytes(key, i, (uint32_t)(256 - i));
            for (int j = 0; j < 4; j++) hashes[4 * i + j] = (uint8_t)(h >> (8 * j));
        }
    }
    if (which) return (uint32_t)og_murmur64a_bytes(hashes, 256 * hb, 0);
    return og_murmur2_bytes(hashes, 256 * hb, 0);
}
uint64_t og_murmur64a_key(uint64_t key, uint64_t seed) { return og_murmur64a_u64(key, seed); }

#define OG_SIG_SEED 0x9747B28Cull
#define OG_SIG_GROUPS 240          /* (N-K)/2 with N = 512, K = 32      */
#define OG_SIG_PLANES 16           /* 512 bits = 16 x 32-bit words                      */

static int og_sig_group(int32_t elabel, int32_t nlabel) {
    uint64_t key = ((uint64_t)(uint32_t)elabel << 32) | (uint32_t)nlabel;   /* reading A6 */
    return (int)(og_murmur64a_u64(key, OG_SIG_SEED) % OG_SIG_GROUPS);
}

/* Encode one signature from a list of (edge label, neighbour label) pairs, counted with
 * multiplicity (reading A5): group state 00 / 01 / 11 for 0 / 1 / >=2 pairs. */
static void og_encode(int32_t vlabel, int64_t npairs, const int32_t *pe, const int32_t *pn, uint32_t sig[OG_SIG_PLANES]) {
    int cnt[OG_SIG_GROUPS];
    memset(cnt, 0, sizeof(cnt));
    for (int64_t i = 0; i < npairs; i++) cnt[og_sig_group(pe[i], pn[i])]++;
    sig[0] = (uint32_t)vlabel;                                   /* stored directly, L1277 */
    for (int w = 1; w < OG_SIG_PLANES; w++) sig[w] = 0;
    for (int grp = 0; grp < OG_SIG_GROUPS; grp++) {
        uint32_t s = cnt[grp] == 0 ? 0u : (cnt[grp] == 1 ? 1u : 3u);
        sig[1 + grp / 16] |= s << (2 * (grp % 16));
    }
}

/* Data signature table, column-first: planes[w * n + v]. */
void og_signatures(const og_graph *g, uint32_t *planes) {
    int64_t n = g->n;
    #pragma omp parallel
    {
        int32_t *pe = NULL, *pn = NULL; int64_t cap = 0;
        #pragma omp for schedule(dynamic, 1024)
        for (int64_t v = 0; v < n; v++) {
            int64_t d = g->off[v + 1] - g->off[v];
            if (d > cap) { cap = d; pe = (int32_t *)realloc(pe, sizeof(int32_t) * cap); pn = (int32_t *)realloc(pn, sizeof(int32_t) * cap); }
            for (int64_t j = 0; j < d; j++) {
                uint64_t x = (uint64_t)g->adj[g->off[v] + j];
                pe[j] = (int32_t)(x >> 32);
                pn[j] = g->vl[(uint32_t)x];
            }
            uint32_t sig[OG_SIG_PLANES];
            og_encode(g->vl[v], d, pe, pn, sig);
            for (int w = 0; w < OG_SIG_PLANES; w++) planes[(int64_t)w * n + v] = sig[w];
        }
        free(pe); free(pn);
    }
}

/* Query signatures: qsig[u * 16 + w] over the query edges incident to u.  distinct != 0:
 * each (edge label, neighbour label) pair counted once — under homomorphism two query
 * neighbours with the same pair may map to one data neighbour, so
 * only the set of pairs is necessary. */
void og_query_signatures(int32_t k, const int32_t *qvl, int32_t qm, const int32_t *qs, const int32_t *qd,
                         const int32_t *qe, int32_t distinct, uint32_t *qsig) {
    int32_t pe[4 * OG_MAXK * OG_MAXK], pn[4 * OG_MAXK * OG_MAXK];
    for (int32_t u = 0; u < k; u++) {
        int64_t c = 0;
        for (int32_t e = 0; e < qm; e++) {
            int32_t l, nl;
            if (qs[e] == u) { l = qe[e]; nl = qvl[qd[e]]; }
            else if (qd[e] == u) { l = qe[e]; nl = qvl[qs[e]]; }
            else continue;
            int dup = 0;
            if (distinct)
                for (int64_t i = 0; i < c; i++) if (pe[i] == l && pn[i] == nl) dup = 1;
            if (dup) continue;
            pe[c] = l; pn[c] = nl; c++;
        }
        og_encode(qvl[u], c, pe, pn, qsig + (int64_t)u * OG_SIG_PLANES);
    }
}

/* C(u) = { v : plane0(v) == plane0(u) and plane_w(v) & plane_w(u) == plane_w(u), w=1..15 }
 * (PAPER.md L543 with reading A4).  bitmaps[u * ceil(n/32) + v/32] bit v%32.            */
void og_filter(const og_graph *g, const uint32_t *planes, int32_t k, const uint32_t *qsig,
               uint32_t *bitmaps, int64_t *counts) {
    int64_t n = g->n, words = (n + 31) / 32;
    memset(bitmaps, 0, sizeof(uint32_t) * words * k);
    for (int32_t u = 0; u < k; u++) {
        const uint32_t *s = qsig + (int64_t)u * OG_SIG_PLANES;
        int64_t c = 0;
        for (int64_t v = 0; v < n; v++) {
            int ok = planes[v] == s[0];
            for (int w = 1; w < OG_SIG_PLANES && ok; w++)
                if ((planes[(int64_t)w * n + v] & s[w]) != s[w]) ok = 0;
            if (ok) { bitmaps[(int64_t)u * words + v / 32] |= 1u << (v % 32); c++; }
        }
        counts[u] = c;
    }
}

int32_t og_sig_group_of(int32_t elabel, int32_t nlabel) { return og_sig_group(elabel, nlabel); }

/* ---------------------------------------------- multi-label signatures (§VII-B) ----- */
/* with label sets the stored-label field cannot be used, so every label
 * of v is hashed into the signature and C(u) is refined by exact label-set containment.
 * Reading A19: plane 0 = OR over l in L_V(v) of bit (MurmurHash2(l, SIG_SEED)
 * mod 32), tested by AND-containment; planes 1-15 count one (edge label, l') pair per data
 * neighbour w and per l' in L_V(w) (with multiplicity; sound: an injective f sends the pairs
 * (u', l') of u's query neighbours to distinct pairs (f(u'), l') of f(u)'s).                 */
static uint32_t og_label_bit(int32_t l) {
    uint32_t x = (uint32_t)l;
    return 1u << (og_murmur2_bytes((const uint8_t *)&x, 4, (uint32_t)OG_SIG_SEED) % 32u);
}

void og_signatures_ml(const og_graph *g, uint32_t *planes) {
    int64_t n = g->n;
    #pragma omp parallel
    {
        int32_t *pe = NULL, *pn = NULL; int64_t cap = 0;
        #pragma omp for schedule(dynamic, 1024)
        for (int64_t v = 0; v < n; v++) {
            int64_t c = 0;
            for (int64_t j = g->off[v]; j < g->off[v + 1]; j++) {
                uint64_t x = (uint64_t)g->adj[j];
                uint32_t w = (uint32_t)x;
                for (int64_t i = g->lsoff[w]; i < g->lsoff[w + 1]; i++) {
                    if (c == cap) { cap = cap ? 2 * cap : 64; pe = (int32_t *)realloc(pe, sizeof(int32_t) * cap); pn = (int32_t *)realloc(pn, sizeof(int32_t) * cap); }
                    pe[c] = (int32_t)(x >> 32); pn[c] = g->ls[i]; c++;
                }
            }
            uint32_t sig[OG_SIG_PLANES];
            og_encode(0, c, pe, pn, sig);
            sig[0] = 0;
            for (int64_t i = g->lsoff[v]; i < g->lsoff[v + 1]; i++) sig[0] |= og_label_bit(g->ls[i]);
            for (int w = 0; w < OG_SIG_PLANES; w++) planes[(int64_t)w * n + v] = sig[w];
        }
        free(pe); free(pn);
    }
}

/* Query side: single-label query edges (a multi-label query edge = one per label, L1283). */
void og_query_signatures_ml(int32_t k, const int32_t *qlsoff, const int32_t *qls, int32_t qm, const int32_t *qs,
                            const int32_t *qd, const int32_t *qe, int32_t distinct, uint32_t *qsig) {
    static const int64_t cap = 4 * OG_MAXK * OG_MAXK * OG_MAXLS;
    int32_t *pe = (int32_t *)malloc(sizeof(int32_t) * cap), *pn = (int32_t *)malloc(sizeof(int32_t) * cap);
    for (int32_t u = 0; u < k; u++) {
        int64_t c = 0;
        for (int32_t e = 0; e < qm; e++) {
            int32_t o = qs[e] == u ? qd[e] : (qd[e] == u ? qs[e] : -1);
            if (o < 0) continue;
            for (int32_t i = qlsoff[o]; i < qlsoff[o + 1]; i++) {
                int dup = 0;
                if (distinct)
                    for (int64_t t = 0; t < c; t++) if (pe[t] == qe[e] && pn[t] == qls[i]) dup = 1;
                if (dup || c == cap) continue;
                pe[c] = qe[e]; pn[c] = qls[i]; c++;
            }
        }
        uint32_t *sig = qsig + (int64_t)u * OG_SIG_PLANES;
        og_encode(0, c, pe, pn, sig);
        sig[0] = 0;
        for (int32_t i = qlsoff[u]; i < qlsoff[u + 1]; i++) sig[0] |= og_label_bit(qls[i]);
    }
    free(pe); free(pn);
}

/* C(u) = { v : plane_w(v) & plane_w(u) == plane_w(u) for w = 0..15, and L_V(u) ⊆ L_V(v) }. */
void og_filter_ml(const og_graph *g, const uint32_t *planes, int32_t k, const uint32_t *qsig, const int32_t *qlsoff,
                  const int32_t *qls, uint32_t *bitmaps, int64_t *counts) {
    int64_t n = g->n, words = (n + 31) / 32;
    memset(bitmaps, 0, sizeof(uint32_t) * words * k);
    for (int32_t u = 0; u < k; u++) {
        const uint32_t *s = qsig + (int64_t)u * OG_SIG_PLANES;
        int64_t c = 0;
        for (int64_t v = 0; v < n; v++) {
            int ok = 1;
            for (int w = 0; w < OG_SIG_PLANES && ok; w++)
                if ((planes[(int64_t)w * n + v] & s[w]) != s[w]) ok = 0;
            for (int32_t i = qlsoff[u]; i < qlsoff[u + 1] && ok; i++) {
                int found = 0;
                for (int64_t t = g->lsoff[v]; t < g->lsoff[v + 1]; t++) if (g->ls[t] == qls[i]) found = 1;
                ok = found;
            }
            if (ok) { bitmaps[(int64_t)u * words + v / 32] |= 1u << (v % 32); c++; }
        }
        counts[u] = c;
    }
}

int32_t og_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
