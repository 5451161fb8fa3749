// common.cuh — internal helpers of libgsi_b200 (CUDA path only; never shared with oracle/).
//
// * hash functions of the written specification in DESIGN.md §3 (MurmurHash2 32-bit for
//   the PCSR group function f of Alg. 1 line 4, MurmurHash64A for signature groups,
//   splitmix64 finaliser for the result fingerprint);
// * the PCSR lookup used by every kernel;
// * a single-pass decoupled look-back tile scan (status word = 2-bit flag | 62-bit value)
//   used for the Prealloc scan F (Alg. 4) and the Combine scan (Alg. 3).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/gsi.h"

namespace gsi {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;          // empty PCSR slot / GID = -1
constexpr uint32_t kPcsrSeed = 0x9747B28Cu;       // PCSR_SEED (per label: ^ dense label)
constexpr uint64_t kSigSeed = 0x9747B28Cull;      // SIG_SEED
constexpr int kSigGroups = 240;                   // (N-K)/2, N=512, K=32
constexpr int kPlanes = GSI_SIG_PLANES;
constexpr uint64_t kFpSeed1 = 0x243F6A8885A308D3ull;
constexpr uint64_t kFpSeed2 = 0x13198A2E03707344ull;

// ------------------------------------------------------------------------ hashing ---
// MurmurHash2 (Appleby), 32-bit, over the 4 little-endian bytes of x.
__host__ __device__ __forceinline__ uint32_t murmur2_u32(uint32_t x, uint32_t seed) {
    const uint32_t m = 0x5bd1e995u;
    uint32_t h = seed ^ 4u;
    uint32_t k = x * m;
    k ^= k >> 24;
    k *= m;
    h *= m;
    h ^= k;
    h ^= h >> 13;
    h *= m;
    h ^= h >> 15;
    return h;
}

// MurmurHash64A (Appleby), over the 8 little-endian bytes of key.
__host__ __device__ __forceinline__ uint64_t murmur64a_u64(uint64_t key, uint64_t seed) {
    const uint64_t m = 0xc6a4a7935bd1e995ull;
    uint64_t h = seed ^ (8ull * m);
    uint64_t k = key * m;
    k ^= k >> 47;
    k *= m;
    h ^= k;
    h *= m;
    h ^= h >> 47;
    h *= m;
    h ^= h >> 47;
    return h;
}

// Signature group of an (edge label, neighbour label) key (reading A6).
__host__ __device__ __forceinline__ int sig_group(uint32_t elabel_raw, uint32_t nlabel) {
    return (int)(murmur64a_u64(((uint64_t)elabel_raw << 32) | nlabel, kSigSeed) % kSigGroups);
}

__host__ __device__ __forceinline__ uint64_t fp_mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Set fingerprint: the hash of a final row (query-id order) is
#ifdef __CUDACC__
// The same finaliser for the per-match hot loop (bit-identical: fp_mix(z) == fp_mix_pre(z +
// kFpMixAdd)): the leading constant add is folded into the caller's per-row partial sum.
// (Moving the high words' right shifts onto the FMA pipe as IMAD.HI was measured slower:
// IMAD.HI issues at a lower rate and raised the instruction count — profiles/r2/r2e.)
constexpr uint64_t kFpMixAdd = 0x9E3779B97F4A7C15ull;
__device__ __forceinline__ uint64_t fp_mix_pre(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
#endif

// fp_mix(Σ_q fp_term(seed, q, row[q]) mod 2^64) — a per-column keyed term, summed, then
// finalised, so a row's k-1 parent terms can be summed once and each extension x costs one
// term and one finaliser.
__host__ __device__ __forceinline__ uint64_t fp_term(uint64_t seed, int q, uint32_t v) {
    return fp_mix(seed ^ ((uint64_t)(uint32_t)(q + 1) << 32) ^ (uint64_t)v);
}

// Home group of v in partition l: multiply-high range reduction of f(v) (reading A7).
__host__ __device__ __forceinline__ uint32_t pcsr_home(uint32_t v, uint32_t l_dense, uint32_t ngroups) {
    uint32_t h = murmur2_u32(v, kPcsrSeed ^ l_dense);
#ifdef __CUDA_ARCH__
    return __umulhi(h, ngroups);
#else
    return (uint32_t)(((uint64_t)h * ngroups) >> 32);
#endif
}

// ------------------------------------------------------------------ PCSR lookup ----
// Group g of a partition is gpn pairs (v, o): pairs 0..gpn-2 hold (vertex, offset into ci)
// prefix-packed, empty slots hold (kEmpty, END); pair gpn-1 is (GID, END) (Def. 4).  The run
// of slot s is ci[o_s, o_{s+1}) — for the last occupied slot o_{s+1} is END (an empty slot or
// the trailer), so a run end is always the next pair's o (DESIGN.md §3 reading A7).
struct Loc {
    uint32_t off, len;
};

template <int GPN>
__device__ __forceinline__ bool probe_group(const uint2 *__restrict__ G, uint32_t v, Loc &out, uint32_t &gid) {
    static_assert(GPN % 2 == 0, "vector path needs an even GPN");
    uint4 q[GPN / 2];
#pragma unroll
    for (int i = 0; i < GPN / 2; i++) q[i] = __ldg(reinterpret_cast<const uint4 *>(G) + i);
    uint32_t vs[GPN], os[GPN];
#pragma unroll
    for (int i = 0; i < GPN / 2; i++) {
        vs[2 * i] = q[i].x; os[2 * i] = q[i].y;
        vs[2 * i + 1] = q[i].z; os[2 * i + 1] = q[i].w;
    }
#pragma unroll
    for (int s = 0; s < GPN - 1; s++) {
        if (vs[s] == v) {
            out.off = os[s];
            out.len = os[s + 1] - os[s];
            return true;
        }
    }
    gid = vs[GPN - 1];
    return false;
}

__device__ __forceinline__ bool probe_group_generic(const uint2 *__restrict__ G, int gpn, uint32_t v, Loc &out,
                                                    uint32_t &gid) {
    for (int s = 0; s < gpn - 1; s++) {
        uint2 p = __ldg(G + s);
        if (p.x == v) {
            uint2 nx = __ldg(G + s + 1);
            out.off = p.y;
            out.len = nx.y - p.y;
            return true;
        }
        if (p.x == kEmpty) break;
    }
    gid = __ldg(G + gpn - 1).x;
    return false;
}

// Sector-wise probe of one GPN=16 group (B200: DRAM/L2 move 32 B sectors, not the 128 B
// transactions the paper sized the group for).  Pairs 4j..4j+3 form sector j.  A group is
// prefix-packed and only a FULL group can carry a GID (overflow comes from full home groups
// and every non-final chain group is full), so an empty slot ends the search.  With |V(D)|
// keys in |V(D)| groups (one-to-one hash) almost every lookup touches one sector.
__device__ __forceinline__ int probe_group16_sectored(const uint2 *__restrict__ G, uint32_t v, Loc &out,
                                                      uint32_t &gid) {
    const uint4 *G4 = reinterpret_cast<const uint4 *>(G);
#pragma unroll
    for (int sec = 0; sec < 4; sec++) {
        const uint4 a = __ldg(G4 + 2 * sec), b = __ldg(G4 + 2 * sec + 1);
        const uint32_t vs[4] = {a.x, a.z, b.x, b.z};
        const uint32_t os[4] = {a.y, a.w, b.y, b.w};
#pragma unroll
        for (int s = 0; s < 4; s++) {
            const int slot = 4 * sec + s;
            if (slot == 15) {          // trailer (GID, END)
                gid = vs[s];
                return 0;
            }
            if (vs[s] == v) {
                out.off = os[s];
                if (s < 3) out.len = os[s + 1] - os[s];
                else out.len = __ldg(G + slot + 1).y - os[s];
                return 1;
            }
            if (vs[s] == kEmpty) {
                gid = kEmpty;
                return 0;
            }
        }
    }
    gid = kEmpty;
    return 0;
}

// N(v, l) for dense label l: (offset into ci, length); len = 0 if v is not in P(G,l).
// *groups_read counts the groups visited (follow GID until found or -1).
__device__ __forceinline__ Loc pcsr_lookup(const uint2 *__restrict__ groups, int gpn, uint64_t gbase,
                                           uint32_t ngroups, uint32_t l_dense, uint32_t v, int *groups_read) {
    Loc r{0u, 0u};
    if (ngroups == 0) return r;
    uint32_t g = pcsr_home(v, l_dense, ngroups);
    int reads = 0;
    for (;;) {
        const uint2 *G = groups + (gbase + g) * (uint64_t)gpn;
        uint32_t gid = kEmpty;
        bool hit;
        reads++;
        if (gpn == 16) hit = probe_group16_sectored(G, v, r, gid);
        else if (gpn == 8) hit = probe_group<8>(G, v, r, gid);
        else hit = probe_group_generic(G, gpn, v, r, gid);
        if (hit || gid == kEmpty) break;
        g = gid;
    }
    if (groups_read) *groups_read = reads;
    return r;
}

// N independent lookups in one partition, phased so that their first-sector loads are all in
// flight together (the common case resolves from sector 0: a hit in slots 0-2, or an empty
// slot proving absence).  Anything else falls back to the full lookup.
template <int N>
__device__ __forceinline__ void pcsr_lookup_batch(const uint2 *__restrict__ groups, int gpn, uint64_t gbase,
                                                  uint32_t ngroups, uint32_t l_dense, const uint32_t (&v)[N],
                                                  const bool (&valid)[N], Loc (&out)[N]) {
    if (gpn != 16 || ngroups == 0) {
#pragma unroll
        for (int q = 0; q < N; q++)
            out[q] = valid[q] ? pcsr_lookup(groups, gpn, gbase, ngroups, l_dense, v[q], nullptr) : Loc{0u, 0u};
        return;
    }
    uint4 a[N], b[N];
#pragma unroll
    for (int q = 0; q < N; q++) {
        if (valid[q]) {
            const uint4 *G4 = reinterpret_cast<const uint4 *>(groups + (gbase + pcsr_home(v[q], l_dense, ngroups)) * 16ull);
            a[q] = __ldg(G4);
            b[q] = __ldg(G4 + 1);
        }
    }
#pragma unroll
    for (int q = 0; q < N; q++) {
        out[q] = Loc{0u, 0u};
        if (!valid[q]) continue;
        const uint32_t x = v[q];
        bool done = true;
        if (a[q].x == x) out[q] = Loc{a[q].y, a[q].w - a[q].y};
        else if (a[q].z == x) out[q] = Loc{a[q].w, b[q].y - a[q].w};
        else if (b[q].x == x) out[q] = Loc{b[q].y, b[q].w - b[q].y};
        else if (b[q].z == x) done = false;                                   // slot 3: run ends in sector 1
        else if (a[q].x == kEmpty || a[q].z == kEmpty || b[q].x == kEmpty || b[q].z == kEmpty) done = true;  // absent
        else done = false;                                                    // full sector: keep probing
        if (!done) out[q] = pcsr_lookup(groups, gpn, gbase, ngroups, l_dense, x, nullptr);
    }
}

// ------------------------------------------------------- decoupled look-back scan ---
constexpr uint64_t kFlagA = 1ull << 62;
constexpr uint64_t kFlagP = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Executed by the 32 lanes of ONE warp.  status[tile] receives (A | aggregate) immediately,
// then (P | inclusive prefix).  Returns the exclusive prefix of this tile (all lanes).
__device__ __forceinline__ unsigned long long lookback_exclusive(unsigned long long *status, uint32_t tile,
                                                                 unsigned long long aggregate) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_relaxed(&status[0], kFlagP | aggregate);
        return 0ull;
    }
    if (lane == 0) st_relaxed(&status[tile], kFlagA | aggregate);
    unsigned long long excl = 0;
    long long base = (long long)tile - 1;
    for (;;) {
        long long j = base - lane;
        unsigned long long s;
        if (j >= 0) {
            do {
                s = ld_relaxed(&status[j]);
            } while ((s >> 62) == 0);
        } else {
            s = kFlagP;   // virtual predecessor of tile 0: prefix 0
        }
        unsigned pmask = __ballot_sync(0xffffffffu, (s >> 62) == 2);
        unsigned long long val = s & kValMask;
        if (pmask) {
            int first = __ffs(pmask) - 1;
            if (lane > first) val = 0;
            excl += warp_sum_u64(val);
            break;
        }
        excl += warp_sum_u64(val);
        base -= 32;
    }
    if (lane == 0) st_relaxed(&status[tile], kFlagP | (excl + aggregate));
    return excl;
}

// Block-wide exclusive scan of one u64 per thread (blockDim.x multiple of 32, <= 1024).
// Returns the exclusive prefix; *total receives the block sum.  Uses smem[33].
__device__ __forceinline__ unsigned long long block_exclusive_scan(unsigned long long x, unsigned long long *smem,
                                                                   unsigned long long *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned long long inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) smem[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = lane < nw ? smem[lane] : 0ull;
        unsigned long long wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < nw) smem[lane] = wi - w;
        if (lane == nw - 1) smem[32] = wi;
    }
    __syncthreads();
    unsigned long long r = smem[warp] + inc - x;
    *total = smem[32];
    __syncthreads();
    return r;
}

}  // namespace gsi

// ---------------------------------------------------------------------- host side ---
namespace gsi {

void set_error(const std::string &msg);
gsi_status ensure_cr(const gsi_graph *g, cudaStream_t st);   // graph.cu: build the CR layer once
std::string gsi_last_error_str();   // this thread's last error message
size_t workspace_idle_bytes(int dev);
gsi_status cuda_fail(cudaError_t e, const char *what);

#define GSI_CUDA(call)                                            \
    do {                                                          \
        cudaError_t _e = (call);                                  \
        if (_e != cudaSuccess) return ::gsi::cuda_fail(_e, #call); \
    } while (0)

#define GSI_TRY(call)                        \
    do {                                     \
        gsi_status _s = (call);              \
        if (_s != GSI_OK) return _s;         \
    } while (0)

// Free the device's idle query workspace (query.cu); called before graph allocations.
void workspace_trim(int dev);

// Encode the query signatures on the host (same spec as the data side).
void encode_query_signatures(int32_t k, const int32_t *qvl, int32_t qm, const int32_t *qs, const int32_t *qd,
                             const int32_t *qe, uint32_t *qsig /* k*16 */, int distinct);

// ext.cu (NEXT-4): the multi-label filter (hashed-label signatures + exact label-set refine).
cudaError_t launch_filter_ml(const gsi_graph *g, const gsi_prepared *q, int hom, uint32_t *bm, long long words,
                             unsigned long long *counts, cudaStream_t st);

}  // namespace gsi

// The graph object (opaque to callers).
struct gsi_graph {
    int device = 0;
    int64_t n = 0, m = 0;
    int32_t n_labels = 0;           // dense edge labels
    int32_t gpn = 16;
    int64_t n_groups = 0;
    int32_t max_chain = 0;
    int64_t overflow_groups = 0;
    float ms_build = 0.f;
    // device buffers
    uint32_t *sig = nullptr;        // [16][n] column-first (plane-major)
    uint2 *groups = nullptr;        // [n_groups][gpn]
    int32_t *ci = nullptr;          // [2m]
    // host tables (per dense label)
    std::vector<int32_t> lab_raw;   // dense -> raw (ascending)
    std::vector<int64_t> freq;      // |E(P(G,l))|
    std::vector<int64_t> gbase;     // first group of partition l
    std::vector<uint32_t> ngroups;  // |V(D_l)|
    std::vector<uint32_t> ci_lo;    // [nl+1]: P(G,l)'s runs are ci[ci_lo[l], ci_lo[l+1])
    int dense_label(int32_t raw) const;   // -1 if absent
    // Compressed Representation, built on demand for the NEXT-3 ablation:
    // per partition l the sorted "vertex ID" layer cr_key[gbase_l .. gbase_l + ngroups_l)
    // (key = l << 32 | v) and each vertex's run cr_loc (offset into ci, length).
    mutable std::mutex cr_mu;
    mutable unsigned long long *cr_key = nullptr;
    mutable uint2 *cr_loc = nullptr;
    // NEXT-4 (ext.cu).  Multi-label vertices (§VII-B): the label SETS on
    // the device (refine step of the filter); the signatures hash them (reading A19).
    bool ml = false;
    int64_t ml_total = 0;
    int64_t *ml_off = nullptr;       // [n+1]
    int32_t *ml_labs = nullptr;      // ascending per vertex
    // Edge isomorphism (§VII-A): this graph is the line graph of an input
    // graph with line_n vertices; vertex i = input edge i.
    bool line = false;
    int64_t line_n = 0;
};

// A validated, encoded query (opaque to callers).
struct gsi_prepared {
    const gsi_graph *g = nullptr;
    int device = 0;                  // g->device at prepare time
    int k = 0;
    std::vector<int32_t> qvl, qs, qd, qe;
    std::vector<int> qe_dense;       // -1: label absent from G
    std::vector<uint32_t> qsig;      // 2 * k * 16: iso signatures, then homomorphism signatures
    uint32_t *d_qsig = nullptr;
    bool absent_label = false;
    // multi-label query (ext.cu): vertex label sets, device copy [k+1 offsets | labels]
    bool ml = false;
    std::vector<int32_t> qls;        // [k+1 offsets | labels]
    int32_t *d_qls = nullptr;
    // edge-isomorphism query (ext.cu): this is Q' = L(Q); its vertex j = query edge j
    bool line = false;
    ~gsi_prepared() {
        if (d_qsig) cudaFreeAsync(d_qsig, cudaStreamPerThread);
        if (d_qls) cudaFreeAsync(d_qls, cudaStreamPerThread);
    }
};

namespace gsi {
// vm.cu: a device table that grows in place on a reserved virtual address range.
struct TableVM {
    int device = 0, k = 1;
    unsigned long long base = 0;
    size_t reserved = 0, mapped = 0, gran = 0;
    unsigned long long used = 0;                                      // rows appended so far
    std::vector<std::pair<unsigned long long, size_t>> chunks;        // (handle, bytes)
    static TableVM *create(int device, int k);   // nullptr: VMM unavailable
    int32_t *append(unsigned long long rows);     // the next `rows` rows, mapped
    ~TableVM();
};
}  // namespace gsi

struct gsi_result {
    int device = 0;
    int k = 0;
    uint64_t count = 0;
    uint64_t fp[3] = {0, 0, 0};
    int32_t *table = nullptr;        // device, count x k, query-id order
    uint64_t nrows = 0;
    bool has_table = false;
    gsi::TableVM *vm = nullptr;      // owner of `table` when it grew in place
    gsi_stats stats;
    ~gsi_result() {
        if (vm) delete vm;
        else if (table) cudaFreeAsync(table, cudaStreamPerThread);
    }
};
