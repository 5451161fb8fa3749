// graph.cu — gsi_build_graph: PCSR (Def. 4, Alg. 1) and the
// column-first signature table (§III-A), built on the GPU.
//
// Pipeline (all device-side; CUB radix sort is used at build time only, as SURVEY.md §2d
// allows — the query path uses only this library's own kernels):
//   validate -> dense edge-label remap -> symmetrise into 2m entries (l, v, w)
//   -> stable sort by (l, v, w) -> reject exact duplicates
//   -> unique (l, v) keys = the partition vertices V(D_l); one group per key (Alg. 1 line 1)
//   -> home group f(v) (Alg. 1 lines 3-4) and per-group counts
//   -> overflow: the k-th spilled block of a partition takes the k-th empty group of that
//      partition (Alg. 1 lines 5-8; Claim 1 L724-737 guarantees enough empties)
//   -> lay out ci in group order, fill (v, o_v) pairs and the (GID, END) trailer (lines 9-14)
//   -> signatures: saturating 2-bit counters via atomicOr (reading A5).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>

#include "common.cuh"

namespace gsi {
namespace {

template <typename T>
struct DevBuf {
    T *p = nullptr;
    size_t count = 0;
    cudaStream_t s = nullptr;
    cudaError_t alloc(size_t n, cudaStream_t st) {
        s = st;
        count = n;
        return cudaMallocAsync(&p, sizeof(T) * (n ? n : 1), st);
    }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
    T *release() {
        T *r = p;
        p = nullptr;
        return r;
    }
};

constexpr int kB = 256;
inline unsigned blocks_for(int64_t n, int per = kB) {
    int64_t b = (n + per - 1) / per;
    if (b < 1) b = 1;
    if (b > (1ll << 30)) b = 1ll << 30;
    return (unsigned)b;
}

__global__ void k_validate_edges(int64_t m, int64_t n, const int32_t *src, const int32_t *dst, const int32_t *el,
                                 unsigned *flags) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        int32_t a = src[e], b = dst[e];
        unsigned f = 0;
        if (a < 0 || a >= n || b < 0 || b >= n) f |= 1;
        if (el[e] < 0) f |= 2;
        if (a == b) f |= 4;
        if (f) atomicOr(flags, f);
    }
}

__global__ void k_validate_vl(int64_t n, const int32_t *vl, unsigned *flags) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        if (vl[v] < 0) atomicOr(flags, 2u);
}

__global__ void k_entries(int64_t m, const int32_t *src, const int32_t *dst, const int32_t *el,
                          const int32_t *lab_raw, int nl, unsigned long long *key, uint32_t *val) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        int32_t l = el[e];
        int lo = 0, hi = nl;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (lab_raw[mid] < l) lo = mid + 1; else hi = mid;
        }
        unsigned long long L = (unsigned long long)lo << 32;
        key[2 * e] = L | (uint32_t)src[e];
        val[2 * e] = (uint32_t)dst[e];
        key[2 * e + 1] = L | (uint32_t)dst[e];
        val[2 * e + 1] = (uint32_t)src[e];
    }
}

__global__ void k_key_flags(int64_t E, const unsigned long long *key, const uint32_t *val, uint32_t *flag,
                            unsigned *err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
        bool newkey = i == 0 || key[i] != key[i - 1];
        if (!newkey && val[i] == val[i - 1]) atomicOr(err, 8u);   // exact duplicate (v,w,l)
        flag[i] = newkey ? 1u : 0u;
    }
}

// kid = exclusive scan of flags; write the unique keys and their run starts.
__global__ void k_unique(int64_t E, const unsigned long long *key, const uint32_t *flag, const uint32_t *kid,
                         unsigned long long *ukey, uint32_t *ustart, uint32_t K) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
        if (flag[i]) {
            ukey[kid[i]] = key[i];
            ustart[kid[i]] = (uint32_t)i;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) ustart[K] = (uint32_t)E;
}

__global__ void k_label_starts(uint32_t K, const unsigned long long *ukey, uint32_t *lstart, int nl) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < K; j += (int64_t)gridDim.x * blockDim.x) {
        uint32_t l = (uint32_t)(ukey[j] >> 32);
        if (j == 0 || (uint32_t)(ukey[j - 1] >> 32) != l) lstart[l] = (uint32_t)j;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) lstart[nl] = K;
}

__device__ __forceinline__ uint32_t label_of_group(const uint32_t *lstart, int nl, uint32_t g) {
    int lo = 0, hi = nl;   // largest l with lstart[l] <= g
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (lstart[mid] <= g) lo = mid; else hi = mid;
    }
    return (uint32_t)lo;
}

__global__ void k_home(uint32_t K, const unsigned long long *ukey, const uint32_t *lstart, uint32_t *home,
                       uint32_t *keyidx, uint32_t *cnt) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < K; j += (int64_t)gridDim.x * blockDim.x) {
        uint32_t l = (uint32_t)(ukey[j] >> 32), v = (uint32_t)ukey[j];
        uint32_t ng = lstart[l + 1] - lstart[l];
        uint32_t h = lstart[l] + pcsr_home(v, l, ng);
        home[j] = h;
        keyidx[j] = (uint32_t)j;
        atomicAdd(&cnt[h], 1u);
    }
}

__global__ void k_need_empty(uint32_t K, const uint32_t *cnt, int gpn, uint32_t *need, uint32_t *empty) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < K; g += (int64_t)gridDim.x * blockDim.x) {
        uint32_t z = cnt[g], cap = (uint32_t)(gpn - 1);
        need[g] = z > cap ? (z + cap - 1) / cap - 1 : 0u;
        empty[g] = z == 0 ? 1u : 0u;
    }
}

__global__ void k_empty_list(uint32_t K, const uint32_t *empty, const uint32_t *escan, uint32_t *elist) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < K; g += (int64_t)gridDim.x * blockDim.x)
        if (empty[g]) elist[escan[g]] = (uint32_t)g;
}

// Claim 1 check per label: total needed overflow groups <= empty groups of the label.
__global__ void k_claim1(int nl, const uint32_t *lstart, const uint32_t *nscan, const uint32_t *escan,
                         unsigned *err) {
    for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nl; l += gridDim.x * blockDim.x) {
        uint32_t a = lstart[l], b = lstart[l + 1];
        if (nscan[b] - nscan[a] > escan[b] - escan[a]) atomicOr(err, 16u);
    }
}

__device__ __forceinline__ uint32_t overflow_group(uint32_t h, uint32_t c, const uint32_t *lstart, int nl,
                                                   const uint32_t *nscan, const uint32_t *escan,
                                                   const uint32_t *elist) {
    uint32_t l = label_of_group(lstart, nl, h);
    uint32_t a = lstart[l];
    return elist[escan[a] + (nscan[h] - nscan[a]) + c];
}

// Chain links: next[home] = first overflow group, next[ov_c] = ov_{c+1} or empty.
__global__ void k_chains(uint32_t K, const uint32_t *need, const uint32_t *lstart, int nl, const uint32_t *nscan,
                         const uint32_t *escan, const uint32_t *elist, uint32_t *next, uint32_t *maxchain,
                         uint32_t *spilled) {
    for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < K; h += (int64_t)gridDim.x * blockDim.x) {
        uint32_t x = need[h];
        if (!x) continue;
        atomicMax(maxchain, x + 1);
        atomicAdd(spilled, 1u);
        uint32_t prev = (uint32_t)h;
        for (uint32_t c = 0; c < x; c++) {
            uint32_t G = overflow_group((uint32_t)h, c, lstart, nl, nscan, escan, elist);
            next[prev] = G;
            prev = G;
        }
    }
}

// Place the sorted (home, key) pairs into group slots.
__global__ void k_place(uint32_t K, const uint32_t *hs, const uint32_t *ks, const uint32_t *gpos, int gpn,
                        const uint32_t *lstart, int nl, const uint32_t *nscan, const uint32_t *escan,
                        const uint32_t *elist, uint32_t *slot_key) {
    const uint32_t cap = (uint32_t)(gpn - 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < K; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t h = hs[i], r = (uint32_t)i - gpos[h];
        uint32_t G = h, s = r;
        if (r >= cap) {
            G = overflow_group(h, r / cap - 1, lstart, nl, nscan, escan, elist);
            s = r % cap;
        }
        slot_key[(uint64_t)G * cap + s] = ks[i];
    }
}

__global__ void k_group_deg(uint32_t K, int gpn, const uint32_t *slot_key, const uint32_t *ustart, uint32_t *gdeg) {
    const uint32_t cap = (uint32_t)(gpn - 1);
    for (int64_t G = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; G < K; G += (int64_t)gridDim.x * blockDim.x) {
        uint32_t t = 0;
        for (uint32_t s = 0; s < cap; s++) {
            uint32_t j = slot_key[(uint64_t)G * cap + s];
            if (j == kEmpty) break;
            t += ustart[j + 1] - ustart[j];
        }
        gdeg[G] = t;
    }
}

__global__ void k_fill_groups(uint32_t K, int gpn, const uint32_t *slot_key, const uint32_t *ustart,
                              const unsigned long long *ukey, const uint32_t *gci, const uint32_t *gdeg,
                              const uint32_t *next, const uint32_t *lstart, int nl, uint2 *groups, uint32_t *koff) {
    const uint32_t cap = (uint32_t)(gpn - 1);
    for (int64_t G = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; G < K; G += (int64_t)gridDim.x * blockDim.x) {
        uint32_t o = gci[G];
        uint32_t end = o + gdeg[G];
        uint2 *P = groups + (uint64_t)G * gpn;
        for (uint32_t s = 0; s < cap; s++) {
            uint32_t j = slot_key[(uint64_t)G * cap + s];
            if (j == kEmpty) {
                P[s] = make_uint2(kEmpty, end);
            } else {
                P[s] = make_uint2((uint32_t)ukey[j], o);
                koff[j] = o;
                o += ustart[j + 1] - ustart[j];
            }
        }
        uint32_t nx = next[G];
        uint32_t gid = kEmpty;
        if (nx != kEmpty) gid = nx - lstart[label_of_group(lstart, nl, (uint32_t)G)];   // label-local GID
        P[cap] = make_uint2(gid, end);
    }
}

__global__ void k_scatter_ci(int64_t E, const uint32_t *kid, const uint32_t *ustart, const uint32_t *koff,
                             const uint32_t *val, int32_t *ci) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < E; p += (int64_t)gridDim.x * blockDim.x) {
        uint32_t j = kid[p];
        ci[koff[j] + ((uint32_t)p - ustart[j])] = (int32_t)val[p];
    }
}

// kid[] here is the exclusive scan of flags; for a non-first entry of a run the key id is
// kid[p] - 1 + flag[p] ... fixed up by k_kid_inclusive below.
__global__ void k_kid_inclusive(int64_t E, const uint32_t *flag, uint32_t *kid) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < E; p += (int64_t)gridDim.x * blockDim.x)
        kid[p] = kid[p] + flag[p] - 1;
}

__global__ void k_signatures(int64_t E, int64_t n, const unsigned long long *key, const uint32_t *val,
                             const int32_t *vl, const int32_t *lab_raw, uint32_t *sig) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < E; p += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long k = key[p];
        uint32_t v = (uint32_t)k;
        uint32_t lraw = (uint32_t)lab_raw[k >> 32];
        int g = sig_group(lraw, (uint32_t)vl[val[p]]);
        uint32_t *w = sig + (uint64_t)(1 + g / 16) * n + v;
        uint32_t lo = 1u << (2 * (g % 16));
        uint32_t old = atomicOr(w, lo);
        if (old & lo) atomicOr(w, lo << 1);   // second pair in the group: 01 -> 11
    }
}

// freq(l) and the ci range of partition l: its groups are contiguous and ci is laid out in
// group order, so P(G,l)'s neighbour runs are ci[gci[lstart[l]], gci[lstart[l+1]]).
__global__ void k_label_tables(int nl, const uint32_t *lstart, const uint32_t *ustart, const uint32_t *gci,
                               long long *freq, uint32_t *cilo) {
    for (int l = blockIdx.x * blockDim.x + threadIdx.x; l <= nl; l += gridDim.x * blockDim.x) {
        if (l < nl) freq[l] = (long long)(ustart[lstart[l + 1]] - ustart[lstart[l]]) / 2;
        cilo[l] = gci[lstart[l]];
    }
}

inline int bits_for(uint64_t x) {
    int b = 1;
    while (b < 64 && (1ull << b) <= x) b++;
    return b;
}

}  // namespace

// Exclusive scan of uint32 (CUB, build time only).
static gsi_status exclusive_scan_u32(const uint32_t *in, uint32_t *out, int64_t count, cudaStream_t st) {
    size_t tmp = 0;
    GSI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)count, st));
    DevBuf<unsigned char> t;
    GSI_CUDA(t.alloc(tmp, st));
    GSI_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, (int)count, st));
    return GSI_OK;
}

// ---------------------------------------------------------------- CR (ablation) -----
// The Compressed Representation of PAPER.md L674-682 ("a layer called vertex ID is added, and
// binary search is performed over this layer"), derived from the PCSR groups: every occupied
// slot (v, o_v) of partition l becomes (l << 32 | v, run), then the entries are sorted by key.
// Partition l has exactly ngroups_l keys (one group per partition vertex), so its layer is
// [gbase_l, gbase_l + ngroups_l) of the sorted arrays.
namespace {
__global__ void k_cr_emit(const uint2 *groups, int gpn, long long ngroups_total, const long long *gb, int nl,
                          unsigned long long *key, uint2 *loc, unsigned long long *ctr) {
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < ngroups_total;
         g += (long long)gridDim.x * blockDim.x) {
        int lo = 0, hi = nl;   // partition of group g: last l with gb[l] <= g
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (gb[mid] <= g) lo = mid; else hi = mid;
        }
        const uint2 *G = groups + g * (long long)gpn;
        for (int sl = 0; sl < gpn - 1; sl++) {
            const uint2 p = G[sl];
            if (p.x == kEmpty) break;
            const unsigned long long i = atomicAdd(ctr, 1ull);
            key[i] = ((unsigned long long)(uint32_t)lo << 32) | p.x;
            loc[i] = make_uint2(p.y, G[sl + 1].y - p.y);
        }
    }
}
}  // namespace

gsi_status ensure_cr(const gsi_graph *g, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g->cr_mu);
    if (g->cr_key || g->n_groups == 0) return GSI_OK;
    const long long K = g->n_groups;
    const int nl = g->n_labels;
    DevBuf<unsigned long long> k1, ctr;
    DevBuf<uint2> l1;
    DevBuf<long long> gb;
    GSI_CUDA(k1.alloc(K, st));
    GSI_CUDA(l1.alloc(K, st));
    GSI_CUDA(ctr.alloc(1, st));
    GSI_CUDA(gb.alloc(nl + 1, st));
    GSI_CUDA(cudaMemsetAsync(ctr.p, 0, 8, st));
    std::vector<long long> hgb(nl + 1);
    for (int l = 0; l < nl; l++) hgb[l] = g->gbase[l];
    hgb[nl] = K;
    GSI_CUDA(cudaMemcpyAsync(gb.p, hgb.data(), 8ull * (nl + 1), cudaMemcpyHostToDevice, st));
    k_cr_emit<<<blocks_for(K), kB, 0, st>>>(g->groups, g->gpn, K, gb.p, nl, k1.p, l1.p, ctr.p);
    unsigned long long *key = nullptr;
    uint2 *loc = nullptr;
    GSI_CUDA(cudaMalloc(&key, 8ull * K));
    GSI_CUDA(cudaMalloc(&loc, 8ull * K));
    size_t t = 0;
    GSI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t, k1.p, key, l1.p, loc, (int)K, 0, 64, st));
    DevBuf<unsigned char> tmp;
    GSI_CUDA(tmp.alloc(t, st));
    GSI_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, t, k1.p, key, l1.p, loc, (int)K, 0, 64, st));
    GSI_CUDA(cudaStreamSynchronize(st));
    g->cr_key = key;
    g->cr_loc = loc;
    return GSI_OK;
}

gsi_status build_graph_impl(int64_t n, const int32_t *h_vl, int64_t m, const int32_t *h_src, const int32_t *h_dst,
                            const int32_t *h_el, const gsi_build_opts *opts, gsi_graph **out) {
    auto t0 = std::chrono::steady_clock::now();
    int gpn = opts ? opts->gpn : 16;
    if (gpn < 2 || gpn > 16) {
        set_error("gpn must be in [2,16] (PAPER.md L700-701)");
        return GSI_ERR_INVALID_ARG;
    }
    // 2m < 2^31: the build's CUB sort / unique / scan calls take int item counts
    if (n < 0 || m < 0 || n >= (1ll << 31) - 1 || 2 * m >= (1ll << 31) - 1) {
        set_error("need 0 <= n < 2^31-1 and 0 <= 2m < 2^31-1");
        return GSI_ERR_INVALID_ARG;
    }
    if ((n > 0 && !h_vl) || (m > 0 && (!h_src || !h_dst || !h_el))) {
        set_error("null input array");
        return GSI_ERR_INVALID_ARG;
    }
    int dev = opts && opts->device >= 0 ? opts->device : -1;
    if (dev >= 0) GSI_CUDA(cudaSetDevice(dev));
    GSI_CUDA(cudaGetDevice(&dev));
    workspace_trim(dev);   // an idle query workspace must not starve the build
    cudaStream_t st = opts && opts->stream ? (cudaStream_t)opts->stream : cudaStreamPerThread;

    const int64_t E = 2 * m;
    DevBuf<int32_t> d_vl, d_src, d_dst, d_el;
    GSI_CUDA(d_vl.alloc(n, st));
    GSI_CUDA(d_src.alloc(m, st));
    GSI_CUDA(d_dst.alloc(m, st));
    GSI_CUDA(d_el.alloc(m, st));
    // host arrays (the C ABI) or device arrays (the NEXT-4 builders in ext.cu): UVA copies
    if (n) GSI_CUDA(cudaMemcpyAsync(d_vl.p, h_vl, 4 * n, cudaMemcpyDefault, st));
    if (m) {
        GSI_CUDA(cudaMemcpyAsync(d_src.p, h_src, 4 * m, cudaMemcpyDefault, st));
        GSI_CUDA(cudaMemcpyAsync(d_dst.p, h_dst, 4 * m, cudaMemcpyDefault, st));
        GSI_CUDA(cudaMemcpyAsync(d_el.p, h_el, 4 * m, cudaMemcpyDefault, st));
    }
    DevBuf<unsigned> d_flags;
    GSI_CUDA(d_flags.alloc(4, st));
    GSI_CUDA(cudaMemsetAsync(d_flags.p, 0, 16, st));
    if (m) k_validate_edges<<<blocks_for(m), kB, 0, st>>>(m, n, d_src.p, d_dst.p, d_el.p, d_flags.p);
    if (n) k_validate_vl<<<blocks_for(n), kB, 0, st>>>(n, d_vl.p, d_flags.p);
    unsigned flags = 0;
    GSI_CUDA(cudaMemcpyAsync(&flags, d_flags.p, 4, cudaMemcpyDeviceToHost, st));
    GSI_CUDA(cudaStreamSynchronize(st));
    if (flags & 1) { set_error("edge endpoint outside [0,n)"); return GSI_ERR_VERTEX_RANGE; }
    if (flags & 2) { set_error("negative vertex or edge label"); return GSI_ERR_LABEL_RANGE; }
    if (flags & 4) { set_error("self-loop (SPEC.md L34)"); return GSI_ERR_SELF_LOOP; }

    auto g = new gsi_graph();
    std::unique_ptr<gsi_graph, void (*)(gsi_graph *)> guard(g, [](gsi_graph *x) {
        if (x->sig) cudaFree(x->sig);
        if (x->groups) cudaFree(x->groups);
        if (x->ci) cudaFree(x->ci);
        delete x;
    });
    g->device = dev;
    g->n = n;
    g->m = m;
    g->gpn = gpn;

    // ---- dense edge labels: sorted unique raw labels --------------------------------
    int nl = 0;
    DevBuf<int32_t> d_labraw;
    {
        DevBuf<int32_t> sorted;
        GSI_CUDA(sorted.alloc(m, st));
        GSI_CUDA(d_labraw.alloc(m, st));
        DevBuf<int> d_nl;
        GSI_CUDA(d_nl.alloc(1, st));
        size_t t1 = 0, t2 = 0;
        GSI_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t1, d_el.p, sorted.p, (int)m, 0, 31, st));
        GSI_CUDA(cub::DeviceSelect::Unique(nullptr, t2, sorted.p, d_labraw.p, d_nl.p, (int)m, st));
        DevBuf<unsigned char> tmp;
        GSI_CUDA(tmp.alloc(std::max(t1, t2), st));
        if (m) {
            GSI_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, t1, d_el.p, sorted.p, (int)m, 0, 31, st));
            GSI_CUDA(cub::DeviceSelect::Unique(tmp.p, t2, sorted.p, d_labraw.p, d_nl.p, (int)m, st));
            GSI_CUDA(cudaMemcpyAsync(&nl, d_nl.p, 4, cudaMemcpyDeviceToHost, st));
        }
        GSI_CUDA(cudaStreamSynchronize(st));
    }
    g->n_labels = nl;
    g->lab_raw.resize(nl);
    if (nl) GSI_CUDA(cudaMemcpyAsync(g->lab_raw.data(), d_labraw.p, 4 * nl, cudaMemcpyDeviceToHost, st));

    // ---- signature plane 0 + zeroed planes ------------------------------------------
    GSI_CUDA(cudaMalloc(&g->sig, sizeof(uint32_t) * kPlanes * (n ? n : 1)));
    GSI_CUDA(cudaMemsetAsync(g->sig, 0, sizeof(uint32_t) * kPlanes * n, st));
    if (n) GSI_CUDA(cudaMemcpyAsync(g->sig, d_vl.p, 4 * n, cudaMemcpyDeviceToDevice, st));   // L1277

    if (m == 0) {
        g->ci_lo.assign(1, 0u);
        g->freq.clear();
        g->gbase.assign(1, 0);
        g->ngroups.assign(1, 0u);
        GSI_CUDA(cudaMalloc(&g->groups, 16));
        GSI_CUDA(cudaMalloc(&g->ci, 16));
        GSI_CUDA(cudaStreamSynchronize(st));
        g->ms_build = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
        *out = guard.release();
        return GSI_OK;
    }

    // ---- symmetrise and sort by (l, v, w) -------------------------------------------
    DevBuf<unsigned long long> key, key2;
    DevBuf<uint32_t> val, val2;
    GSI_CUDA(key.alloc(E, st));
    GSI_CUDA(key2.alloc(E, st));
    GSI_CUDA(val.alloc(E, st));
    GSI_CUDA(val2.alloc(E, st));
    k_entries<<<blocks_for(m), kB, 0, st>>>(m, d_src.p, d_dst.p, d_el.p, d_labraw.p, nl, key.p, val.p);
    {
        const int vbits = bits_for((uint64_t)n), kbits = 32 + bits_for((uint64_t)nl);
        size_t t1 = 0, t2 = 0;
        GSI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t1, val.p, val2.p, key.p, key2.p, (int)E, 0, vbits, st));
        GSI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t2, key2.p, key.p, val2.p, val.p, (int)E, 0, kbits, st));
        DevBuf<unsigned char> tmp;
        GSI_CUDA(tmp.alloc(std::max(t1, t2), st));
        // pass 1: by w (stable), pass 2: by (l, v) (stable) => (l, v, w) order
        GSI_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, t1, val.p, val2.p, key.p, key2.p, (int)E, 0, vbits, st));
        GSI_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, t2, key2.p, key.p, val2.p, val.p, (int)E, 0, kbits, st));
    }

    DevBuf<uint32_t> flag, kid;
    GSI_CUDA(flag.alloc(E, st));
    GSI_CUDA(kid.alloc(E, st));
    k_key_flags<<<blocks_for(E), kB, 0, st>>>(E, key.p, val.p, flag.p, d_flags.p);
    GSI_TRY(exclusive_scan_u32(flag.p, kid.p, E, st));
    uint32_t lastkid = 0, lastflag = 0;
    GSI_CUDA(cudaMemcpyAsync(&lastkid, kid.p + E - 1, 4, cudaMemcpyDeviceToHost, st));
    GSI_CUDA(cudaMemcpyAsync(&lastflag, flag.p + E - 1, 4, cudaMemcpyDeviceToHost, st));
    GSI_CUDA(cudaMemcpyAsync(&flags, d_flags.p, 4, cudaMemcpyDeviceToHost, st));
    GSI_CUDA(cudaStreamSynchronize(st));
    if (flags & 8) { set_error("duplicate (v,w,l) edge"); return GSI_ERR_DUPLICATE_EDGE; }
    const uint32_t K = lastkid + lastflag;   // sum_l |V(D_l)|
    g->n_groups = K;

    DevBuf<unsigned long long> ukey;
    DevBuf<uint32_t> ustart, lstart;
    GSI_CUDA(ukey.alloc(K, st));
    GSI_CUDA(ustart.alloc(K + 1, st));
    GSI_CUDA(lstart.alloc(nl + 1, st));
    k_unique<<<blocks_for(E), kB, 0, st>>>(E, key.p, flag.p, kid.p, ukey.p, ustart.p, K);
    k_kid_inclusive<<<blocks_for(E), kB, 0, st>>>(E, flag.p, kid.p);
    k_label_starts<<<blocks_for(K), kB, 0, st>>>(K, ukey.p, lstart.p, nl);

    // ---- group hashing, counts, overflow -------------------------------------------
    DevBuf<uint32_t> home, keyidx, cnt, hs, ks, gpos, need, empty, nscan, escan, elist, next, slot_key;
    GSI_CUDA(home.alloc(K, st));
    GSI_CUDA(keyidx.alloc(K, st));
    GSI_CUDA(cnt.alloc(K + 1, st));
    GSI_CUDA(cudaMemsetAsync(cnt.p, 0, 4ull * (K + 1), st));
    k_home<<<blocks_for(K), kB, 0, st>>>(K, ukey.p, lstart.p, home.p, keyidx.p, cnt.p);
    GSI_CUDA(hs.alloc(K, st));
    GSI_CUDA(ks.alloc(K, st));
    {
        size_t t1 = 0;
        const int hbits = bits_for(K);
        GSI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t1, home.p, hs.p, keyidx.p, ks.p, (int)K, 0, hbits, st));
        DevBuf<unsigned char> tmp;
        GSI_CUDA(tmp.alloc(t1, st));
        GSI_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, t1, home.p, hs.p, keyidx.p, ks.p, (int)K, 0, hbits, st));
    }
    GSI_CUDA(gpos.alloc(K + 1, st));
    GSI_TRY(exclusive_scan_u32(cnt.p, gpos.p, K + 1, st));
    GSI_CUDA(need.alloc(K + 1, st));
    GSI_CUDA(empty.alloc(K + 1, st));
    GSI_CUDA(cudaMemsetAsync(need.p, 0, 4ull * (K + 1), st));
    GSI_CUDA(cudaMemsetAsync(empty.p, 0, 4ull * (K + 1), st));
    k_need_empty<<<blocks_for(K), kB, 0, st>>>(K, cnt.p, gpn, need.p, empty.p);
    GSI_CUDA(nscan.alloc(K + 1, st));
    GSI_CUDA(escan.alloc(K + 1, st));
    GSI_TRY(exclusive_scan_u32(need.p, nscan.p, K + 1, st));
    GSI_TRY(exclusive_scan_u32(empty.p, escan.p, K + 1, st));
    GSI_CUDA(elist.alloc(K + 1, st));
    k_empty_list<<<blocks_for(K), kB, 0, st>>>(K, empty.p, escan.p, elist.p);
    k_claim1<<<blocks_for(nl), kB, 0, st>>>(nl, lstart.p, nscan.p, escan.p, d_flags.p);
    GSI_CUDA(next.alloc(K, st));
    GSI_CUDA(cudaMemsetAsync(next.p, 0xFF, 4ull * K, st));
    DevBuf<uint32_t> maxchain;
    GSI_CUDA(maxchain.alloc(2, st));
    GSI_CUDA(cudaMemsetAsync(maxchain.p, 0, 8, st));
    k_chains<<<blocks_for(K), kB, 0, st>>>(K, need.p, lstart.p, nl, nscan.p, escan.p, elist.p, next.p, maxchain.p,
                                           maxchain.p + 1);
    const uint64_t nslots = (uint64_t)K * (gpn - 1);
    GSI_CUDA(slot_key.alloc(nslots, st));
    GSI_CUDA(cudaMemsetAsync(slot_key.p, 0xFF, 4ull * nslots, st));
    k_place<<<blocks_for(K), kB, 0, st>>>(K, hs.p, ks.p, gpos.p, gpn, lstart.p, nl, nscan.p, escan.p, elist.p,
                                          slot_key.p);

    // ---- ci layout in group order (Alg. 1 lines 9-14) --------------------------------
    DevBuf<uint32_t> gdeg, gci, koff;
    GSI_CUDA(gdeg.alloc(K + 1, st));
    GSI_CUDA(cudaMemsetAsync(gdeg.p, 0, 4ull * (K + 1), st));
    k_group_deg<<<blocks_for(K), kB, 0, st>>>(K, gpn, slot_key.p, ustart.p, gdeg.p);
    GSI_CUDA(gci.alloc(K + 1, st));
    GSI_TRY(exclusive_scan_u32(gdeg.p, gci.p, K + 1, st));
    GSI_CUDA(koff.alloc(K, st));
    GSI_CUDA(cudaMalloc(&g->groups, sizeof(uint2) * (uint64_t)K * gpn));
    GSI_CUDA(cudaMalloc(&g->ci, sizeof(int32_t) * E));
    k_fill_groups<<<blocks_for(K), kB, 0, st>>>(K, gpn, slot_key.p, ustart.p, ukey.p, gci.p, gdeg.p, next.p,
                                                lstart.p, nl, g->groups, koff.p);
    k_scatter_ci<<<blocks_for(E), kB, 0, st>>>(E, kid.p, ustart.p, koff.p, val.p, g->ci);

    // ---- signatures (planes 1..15) ---------------------------------------------------
    k_signatures<<<blocks_for(E), kB, 0, st>>>(E, n, key.p, val.p, d_vl.p, d_labraw.p, g->sig);

    // ---- host label tables ----------------------------------------------------------
    DevBuf<long long> d_freq;
    DevBuf<uint32_t> d_cilo;
    GSI_CUDA(d_freq.alloc(nl, st));
    GSI_CUDA(d_cilo.alloc(nl + 1, st));
    k_label_tables<<<blocks_for(nl + 1), kB, 0, st>>>(nl, lstart.p, ustart.p, gci.p, d_freq.p, d_cilo.p);
    g->ci_lo.resize(nl + 1);
    GSI_CUDA(cudaMemcpyAsync(g->ci_lo.data(), d_cilo.p, 4ull * (nl + 1), cudaMemcpyDeviceToHost, st));
    std::vector<uint32_t> h_lstart(nl + 1);
    g->freq.resize(nl);
    uint32_t h_maxchain = 0, h_spilled = 0;
    GSI_CUDA(cudaMemcpyAsync(h_lstart.data(), lstart.p, 4ull * (nl + 1), cudaMemcpyDeviceToHost, st));
    GSI_CUDA(cudaMemcpyAsync(&h_spilled, maxchain.p + 1, 4, cudaMemcpyDeviceToHost, st));
    GSI_CUDA(cudaMemcpyAsync(g->freq.data(), d_freq.p, 8ull * nl, cudaMemcpyDeviceToHost, st));
    GSI_CUDA(cudaMemcpyAsync(&h_maxchain, maxchain.p, 4, cudaMemcpyDeviceToHost, st));
    GSI_CUDA(cudaMemcpyAsync(&flags, d_flags.p, 4, cudaMemcpyDeviceToHost, st));
    GSI_CUDA(cudaStreamSynchronize(st));
    GSI_CUDA(cudaGetLastError());
    if (flags & 16) { set_error("Claim 1 violated: not enough empty groups (PAPER.md L724-737)"); return GSI_ERR_INTERNAL; }
    g->gbase.resize(nl);
    g->ngroups.resize(nl);
    for (int l = 0; l < nl; l++) {
        g->gbase[l] = h_lstart[l];
        g->ngroups[l] = h_lstart[l + 1] - h_lstart[l];
    }
    g->max_chain = h_maxchain ? (int)h_maxchain : 1;
    g->overflow_groups = h_spilled;
    g->ms_build = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
    *out = guard.release();
    return GSI_OK;
}

// ------------------------------------------------------------------ debug lookup -----
namespace {
__global__ void k_debug_lookup(int64_t nq, const int32_t *v, const int32_t *ld, const uint2 *groups, int gpn,
                               const long long *gbase, const uint32_t *ngroups, uint32_t *off, uint32_t *len,
                               int32_t *reads) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq; i += (int64_t)gridDim.x * blockDim.x) {
        int l = ld[i];
        Loc r{0, 0};
        int rd = 0;
        if (l >= 0) r = pcsr_lookup(groups, gpn, (uint64_t)gbase[l], ngroups[l], (uint32_t)l, (uint32_t)v[i], &rd);
        off[i] = r.off;
        len[i] = r.len;
        reads[i] = rd;
    }
}
}  // namespace

gsi_status debug_lookup_impl(const gsi_graph *g, int64_t nq, const int32_t *v, const int32_t *l, int64_t *len,
                             int32_t *groups_read, int32_t *nbrs, int64_t cap) {
    GSI_CUDA(cudaSetDevice(g->device));
    cudaStream_t st = cudaStreamPerThread;
    std::vector<int32_t> ld(nq);
    for (int64_t i = 0; i < nq; i++) {
        if (v[i] < 0 || v[i] >= g->n) {
            set_error("lookup vertex out of range");
            return GSI_ERR_VERTEX_RANGE;
        }
        ld[i] = g->dense_label(l[i]);
    }
    int nl = g->n_labels;
    DevBuf<int32_t> dv, dl, drd;
    DevBuf<uint32_t> doff, dlen, dng;
    DevBuf<long long> dgb;
    GSI_CUDA(dv.alloc(nq, st));
    GSI_CUDA(dl.alloc(nq, st));
    GSI_CUDA(drd.alloc(nq, st));
    GSI_CUDA(doff.alloc(nq, st));
    GSI_CUDA(dlen.alloc(nq, st));
    GSI_CUDA(dgb.alloc(nl, st));
    GSI_CUDA(dng.alloc(nl, st));
    GSI_CUDA(cudaMemcpyAsync(dv.p, v, 4 * nq, cudaMemcpyHostToDevice, st));
    GSI_CUDA(cudaMemcpyAsync(dl.p, ld.data(), 4 * nq, cudaMemcpyHostToDevice, st));
    if (nl) {
        GSI_CUDA(cudaMemcpyAsync(dgb.p, g->gbase.data(), 8 * nl, cudaMemcpyHostToDevice, st));
        GSI_CUDA(cudaMemcpyAsync(dng.p, g->ngroups.data(), 4 * nl, cudaMemcpyHostToDevice, st));
    }
    if (nq) k_debug_lookup<<<blocks_for(nq), kB, 0, st>>>(nq, dv.p, dl.p, g->groups, g->gpn, dgb.p, dng.p, doff.p,
                                                         dlen.p, drd.p);
    std::vector<uint32_t> off(nq), ln(nq);
    GSI_CUDA(cudaMemcpyAsync(off.data(), doff.p, 4 * nq, cudaMemcpyDeviceToHost, st));
    GSI_CUDA(cudaMemcpyAsync(ln.data(), dlen.p, 4 * nq, cudaMemcpyDeviceToHost, st));
    if (groups_read) GSI_CUDA(cudaMemcpyAsync(groups_read, drd.p, 4 * nq, cudaMemcpyDeviceToHost, st));
    GSI_CUDA(cudaStreamSynchronize(st));
    GSI_CUDA(cudaGetLastError());
    int64_t pos = 0;
    for (int64_t i = 0; i < nq; i++) {
        if (len) len[i] = ln[i];
        if (nbrs && ln[i] && pos + (int64_t)ln[i] <= cap)
            GSI_CUDA(cudaMemcpy(nbrs + pos, g->ci + off[i], 4ull * ln[i], cudaMemcpyDeviceToHost));
        pos += ln[i];
    }
    return GSI_OK;
}

}  // namespace gsi

int gsi_graph::dense_label(int32_t raw) const {
    auto it = std::lower_bound(lab_raw.begin(), lab_raw.end(), raw);
    if (it == lab_raw.end() || *it != raw) return -1;
    return (int)(it - lab_raw.begin());
}
