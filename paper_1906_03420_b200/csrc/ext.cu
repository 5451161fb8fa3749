// ext.cu — NEXT-4 of SURVEY.md §8(f) on the same PCSR / filter / join path:
//
// * multi-label vertices and edges (§VII-B).  The match condition becomes
//   L_V(u) ⊆ L_V(f(u)) and L_E(uv) ⊆ L_E(f(u)f(v)) (L1273-1275).  Edges: every label of an
//   edge becomes one single-label parallel edge (L1283-1285, Fig. 10), on both G and Q, and
//   nothing else changes ("GSI always processes one edge at a time").  Vertices: the stored
//   label field cannot hold a set, so every label is hashed into plane 0 (AND-containment like
//   planes 1-15) and every (edge label, neighbour label) pair of every neighbour label into
//   planes 1-15 (reading A19); C(u) is then refined by exact label-set containment on the GPU
//   (L1279-1281).  The join never looks at vertex labels, so it runs unchanged; since two
//   query vertices with different label sets may now share a data vertex, every unlinked
//   earlier column is a subtraction column (the prepared query's labels are all 0).
//
// * edge isomorphism (§VII-A, Fig. 9): G is transformed into its line
//   graph G' on the device — vertex i of G' is edge i of G, labelled L_E(e_i); two edges of G
//   sharing a vertex v become an edge of G' labelled L_V(v) (a pair of parallel G edges whose
//   two shared vertices carry the same label yields one G' edge, emitted at the smaller
//   vertex) — and PCSR + signatures of G' are built exactly as for any graph.  Q' = L(Q) is
//   built on the host (|E(Q)| <= 32 vertices).  Vertex isomorphism of Q' on G' gives rows of
//   G' vertices in Q'-vertex order, i.e. data edge ids in query-edge order: the reverse
//   transformation is the identity on ids.
#include <cub/cub.cuh>

#include <algorithm>
#include <memory>
#include <tuple>
#include <vector>

#include "common.cuh"

namespace gsi {

gsi_status build_graph_impl(int64_t n, const int32_t *vl, int64_t m, const int32_t *src, const int32_t *dst,
                            const int32_t *el, const gsi_build_opts *opts, gsi_graph **out);
gsi_status prepare_impl(const gsi_graph *g, int32_t k, const int32_t *qvl, int32_t qm, const int32_t *qs,
                        const int32_t *qd, const int32_t *qe, gsi_prepared **out);

namespace {

constexpr int kB = 256;

inline unsigned blocks(int64_t n, int per = kB) {
    int64_t b = (n + per - 1) / per;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 1ll << 30));
}

template <typename T>
struct Dev {
    T *p = nullptr;
    cudaStream_t s = nullptr;
    cudaError_t alloc(size_t n, cudaStream_t st) {
        s = st;
        return cudaMallocAsync(&p, sizeof(T) * (n ? n : 1), st);
    }
    ~Dev() {
        if (p) cudaFreeAsync(p, s);
    }
};

// Host validation shared by both builders: endpoints, self-loops, labels.
gsi_status check_edges(int64_t n, int64_t m, const int32_t *src, const int32_t *dst) {
    for (int64_t e = 0; e < m; e++) {
        if (src[e] < 0 || src[e] >= n || dst[e] < 0 || dst[e] >= n) {
            set_error("edge endpoint outside [0,n)");
            return GSI_ERR_VERTEX_RANGE;
        }
        if (src[e] == dst[e]) {
            set_error("self-loop (SPEC.md L34)");
            return GSI_ERR_SELF_LOOP;
        }
    }
    return GSI_OK;
}

// ------------------------------------------------------------------ line graph --------
__global__ void k_incidence(int64_t m, const int32_t *src, const int32_t *dst, uint32_t *key, uint32_t *val,
                            uint32_t *deg) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        key[2 * e] = (uint32_t)src[e];
        val[2 * e] = (uint32_t)e;
        key[2 * e + 1] = (uint32_t)dst[e];
        val[2 * e + 1] = (uint32_t)e;
        atomicAdd(deg + src[e], 1u);
        atomicAdd(deg + dst[e], 1u);
    }
}

// Pairs of edges incident to v (i < j in ascending edge id) that become G' edges.  A pair of
// parallel edges (both ends shared) whose ends carry the same label is emitted at the smaller
// end only (its two G' edges would be identical).
__device__ __forceinline__ bool line_keep(int32_t v, int32_t oi, int32_t oj, const int32_t *vl) {
    return !(oi == oj && vl[v] == vl[oi] && v > oi);
}

__device__ __forceinline__ int32_t other_end(uint32_t e, int32_t v, const int32_t *src, const int32_t *dst) {
    const int32_t a = src[e];
    return a == v ? dst[e] : a;
}

// One warp per vertex; lane-strided rows i, inner loop over j > i.  EMIT = false: the kept
// pair count of v; EMIT = true: write the pairs at pos[v] in (i, j) order.
template <bool EMIT>
__global__ void k_line_pairs(int64_t n, const uint32_t *off, const uint32_t *inc, const int32_t *src,
                             const int32_t *dst, const int32_t *vl, unsigned long long *cnt,
                             const unsigned long long *pos, int32_t *os, int32_t *od, int32_t *ol) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = w0; v < n; v += nw) {
        const uint32_t b = off[v], d = off[v + 1] - b;
        const int32_t lab = vl[v];
        unsigned long long run = EMIT ? pos[v] : 0ull, tot = 0;
        for (uint32_t i0 = 0; i0 < d; i0 += 32) {
            const uint32_t i = i0 + lane;
            uint32_t c = 0;
            uint32_t ei = 0;
            int32_t oi = -1;
            if (i < d) {
                ei = inc[b + i];
                oi = other_end(ei, (int32_t)v, src, dst);
                for (uint32_t j = i + 1; j < d; j++)
                    c += line_keep((int32_t)v, oi, other_end(inc[b + j], (int32_t)v, src, dst), vl) ? 1u : 0u;
            }
            unsigned long long x = c, incl = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (EMIT && i < d) {
                unsigned long long p = run + incl - x;
                for (uint32_t j = i + 1; j < d; j++) {
                    const uint32_t ej = inc[b + j];
                    if (!line_keep((int32_t)v, oi, other_end(ej, (int32_t)v, src, dst), vl)) continue;
                    os[p] = (int32_t)ei;
                    od[p] = (int32_t)ej;
                    ol[p] = lab;
                    p++;
                }
            }
            const unsigned long long step = __shfl_sync(0xffffffffu, incl, 31);
            run += step;
            tot += step;
        }
        if (!EMIT && lane == 0) cnt[v] = tot;
    }
}

// ------------------------------------------------------------------ multi-label --------
__device__ __forceinline__ uint32_t label_bit(int32_t l) { return 1u << (murmur2_u32((uint32_t)l, (uint32_t)kSigSeed) & 31u); }

__global__ void k_ml_plane0(int64_t n, const int64_t *off, const int32_t *labs, uint32_t *sig) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        uint32_t s = 0;
        for (int64_t i = off[v]; i < off[v + 1]; i++) s |= label_bit(labs[i]);
        sig[v] = s;
    }
}

// Planes 1-15: one (edge label, l') pair per directed adjacency entry v -> w and per label l'
// of w, saturating 2-bit group counters (reading A5 / A19).
__global__ void k_ml_pairs(int64_t m, int64_t n, const int32_t *src, const int32_t *dst, const int32_t *el,
                           const int64_t *off, const int32_t *labs, uint32_t *sig) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < 2 * m; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = p >> 1;
        const int32_t v = (p & 1) ? dst[e] : src[e], w = (p & 1) ? src[e] : dst[e];
        for (int64_t i = off[w]; i < off[w + 1]; i++) {
            const int g = sig_group((uint32_t)el[e], (uint32_t)labs[i]);
            uint32_t *word = sig + (uint64_t)(1 + g / 16) * n + v;
            const uint32_t lo = 1u << (2 * (g % 16));
            const uint32_t old = atomicOr(word, lo);
            if (old & lo) atomicOr(word, lo << 1);
        }
    }
}

// The multi-label filter: one thread per data vertex (32 consecutive vertices per warp, so a
// plane read is one 128 B line), every query vertex tested against all 16 planes by AND-
// containment, then survivors refined by exact L_V(u) ⊆ L_V(v) (merge of two sorted lists);
// ballots form the C(u) bitmap words, popc gives |C(u)|.
__global__ void __launch_bounds__(kB) k_filter_ml(const uint32_t *__restrict__ sig, long long n, int k,
                                                  const uint32_t *__restrict__ qsig, const int32_t *__restrict__ qls,
                                                  const int64_t *__restrict__ off, const int32_t *__restrict__ labs,
                                                  uint32_t *__restrict__ bm, long long words,
                                                  unsigned long long *__restrict__ counts) {
    __shared__ uint32_t qs[GSI_MAX_K * kPlanes];
    __shared__ int32_t ql[GSI_MAX_K + 1 + GSI_MAX_K * 32];
    for (int i = threadIdx.x; i < k * kPlanes; i += blockDim.x) qs[i] = qsig[i];
    const int nl = qls[k];
    for (int i = threadIdx.x; i < k + 1 + nl; i += blockDim.x) ql[i] = qls[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned long long mycnt = 0;   // lane u < k accumulates |C(u)| of this warp
    for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w < words;
         w += ((long long)gridDim.x * blockDim.x) >> 5) {
        const long long v = w * 32 + lane;
        uint32_t s[kPlanes];
#pragma unroll
        for (int p = 0; p < kPlanes; p++) s[p] = v < n ? __ldg(sig + (long long)p * n + v) : 0u;
        for (int u = 0; u < k; u++) {
            bool ok = v < n;
#pragma unroll
            for (int p = 0; p < kPlanes; p++) ok &= (s[p] & qs[u * kPlanes + p]) == qs[u * kPlanes + p];
            if (ok) {   // refine: exact label-set containment
                long long a = off[v];
                const long long b = off[v + 1];
                for (int i = ql[u]; i < ql[u + 1] && ok; i++) {
                    const int32_t want = ql[k + 1 + i];
                    while (a < b && labs[a] < want) a++;
                    ok = a < b && labs[a] == want;
                    a++;
                }
            }
            const uint32_t word = __ballot_sync(0xffffffffu, ok);
            if (lane == 0) bm[(long long)u * words + w] = word;
            if (lane == u) mycnt += __popc(word);
        }
    }
    if (lane < k && mycnt) atomicAdd(counts + lane, mycnt);
}

// Query-side multi-label signature (same spec as the data side, reading A19): plane 0 = the
// hashed label bits of L_V(u), planes 1-15 = one pair per (query edge label, label of the
// other end); `distinct` counts each pair once (homomorphism, reading A5 / NEXT-1).
void encode_ml(int k, const std::vector<int32_t> &qls, int qm, const int32_t *qs, const int32_t *qd,
               const int32_t *qe, uint32_t *out, int distinct) {
    for (int u = 0; u < k; u++) {
        int cnt[kSigGroups] = {0};
        std::vector<unsigned long long> seen;
        for (int e = 0; e < qm; e++) {
            const int o = qs[e] == u ? qd[e] : (qd[e] == u ? qs[e] : -1);
            if (o < 0) continue;
            for (int i = qls[o]; i < qls[o + 1]; i++) {
                const int32_t l2 = qls[k + 1 + i];
                if (distinct) {
                    const unsigned long long key = ((unsigned long long)(uint32_t)qe[e] << 32) | (uint32_t)l2;
                    if (std::find(seen.begin(), seen.end(), key) != seen.end()) continue;
                    seen.push_back(key);
                }
                cnt[sig_group((uint32_t)qe[e], (uint32_t)l2)]++;
            }
        }
        uint32_t *s = out + (size_t)u * kPlanes;
        s[0] = 0;
        for (int i = qls[u]; i < qls[u + 1]; i++) s[0] |= 1u << (murmur2_u32((uint32_t)qls[k + 1 + i], (uint32_t)kSigSeed) & 31u);
        for (int w = 1; w < kPlanes; w++) s[w] = 0;
        for (int gi = 0; gi < kSigGroups; gi++) {
            const uint32_t st = cnt[gi] == 0 ? 0u : (cnt[gi] == 1 ? 1u : 3u);
            s[1 + gi / 16] |= st << (2 * (gi % 16));
        }
    }
}

// Label sets as [count+1 offsets | labels], each set ascending without repeats.
template <typename Off>
gsi_status canon_sets(int64_t count, const Off *off, const int32_t *labs, std::vector<int64_t> &o,
                      std::vector<int32_t> &l, const char *what) {
    o.assign(count + 1, 0);
    l.clear();
    if (off[0] != 0) {
        set_error(std::string(what) + ": offsets must start at 0");
        return GSI_ERR_INVALID_ARG;
    }
    for (int64_t i = 0; i < count; i++) {
        if (off[i + 1] < off[i]) {
            set_error(std::string(what) + ": offsets must be non-decreasing");
            return GSI_ERR_INVALID_ARG;
        }
        std::vector<int32_t> s(labs + off[i], labs + off[i + 1]);
        for (int32_t x : s)
            if (x < 0) {
                set_error(std::string(what) + ": negative label");
                return GSI_ERR_LABEL_RANGE;
            }
        std::sort(s.begin(), s.end());
        s.erase(std::unique(s.begin(), s.end()), s.end());
        l.insert(l.end(), s.begin(), s.end());
        o[i + 1] = (int64_t)l.size();
    }
    return GSI_OK;
}

}  // namespace

// ------------------------------------------------------------------ entry points ------
gsi_status build_line_graph_impl(int64_t n, const int32_t *vl, int64_t m, const int32_t *src, const int32_t *dst,
                                 const int32_t *el, const gsi_build_opts *opts, gsi_graph **out) {
    *out = nullptr;
    if (n < 0 || m < 0 || n >= (1ll << 31) - 1 || m >= (1ll << 31) - 1 || (n && !vl) || (m && (!src || !dst || !el))) {
        set_error("invalid graph arguments");
        return GSI_ERR_INVALID_ARG;
    }
    GSI_TRY(check_edges(n, m, src, dst));
    for (int64_t i = 0; i < n; i++)
        if (vl[i] < 0) {
            set_error("negative vertex label");
            return GSI_ERR_LABEL_RANGE;
        }
    {   // exact duplicate (v, w, l) edges are rejected as by gsi_build_graph
        std::vector<std::tuple<int32_t, int32_t, int32_t>> t((size_t)m);
        for (int64_t e = 0; e < m; e++) {
            if (el[e] < 0) {
                set_error("negative edge label");
                return GSI_ERR_LABEL_RANGE;
            }
            t[e] = std::make_tuple(std::min(src[e], dst[e]), std::max(src[e], dst[e]), el[e]);
        }
        std::sort(t.begin(), t.end());
        if (std::adjacent_find(t.begin(), t.end()) != t.end()) {
            set_error("duplicate (v,w,l) edge");
            return GSI_ERR_DUPLICATE_EDGE;
        }
    }
    int dev = opts && opts->device >= 0 ? opts->device : -1;
    if (dev >= 0) GSI_CUDA(cudaSetDevice(dev));
    cudaStream_t st = opts && opts->stream ? (cudaStream_t)opts->stream : cudaStreamPerThread;
    Dev<int32_t> d_vl, d_src, d_dst, d_el;
    GSI_CUDA(d_vl.alloc(n, st));
    GSI_CUDA(d_src.alloc(m, st));
    GSI_CUDA(d_dst.alloc(m, st));
    GSI_CUDA(d_el.alloc(m, st));
    if (n) GSI_CUDA(cudaMemcpyAsync(d_vl.p, vl, 4 * n, cudaMemcpyHostToDevice, st));
    if (m) {
        GSI_CUDA(cudaMemcpyAsync(d_src.p, src, 4 * m, cudaMemcpyHostToDevice, st));
        GSI_CUDA(cudaMemcpyAsync(d_dst.p, dst, 4 * m, cudaMemcpyHostToDevice, st));
        GSI_CUDA(cudaMemcpyAsync(d_el.p, el, 4 * m, cudaMemcpyHostToDevice, st));
    }
    // incidence lists: (v, e) sorted by v (stable, so each list is in ascending edge id)
    Dev<uint32_t> key, val, key2, val2, deg, off;
    GSI_CUDA(key.alloc(2 * m, st));
    GSI_CUDA(val.alloc(2 * m, st));
    GSI_CUDA(key2.alloc(2 * m, st));
    GSI_CUDA(val2.alloc(2 * m, st));
    GSI_CUDA(deg.alloc(n + 1, st));
    GSI_CUDA(off.alloc(n + 1, st));
    GSI_CUDA(cudaMemsetAsync(deg.p, 0, 4ull * (n + 1), st));
    if (m) k_incidence<<<blocks(m), kB, 0, st>>>(m, d_src.p, d_dst.p, key.p, val.p, deg.p);
    {
        size_t t1 = 0, t2 = 0;
        int bits = 1;
        while (bits < 32 && (1ll << bits) <= n) bits++;
        GSI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t1, key.p, key2.p, val.p, val2.p, (int)(2 * m), 0, bits, st));
        GSI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t2, deg.p, off.p, (int)(n + 1), st));
        Dev<unsigned char> tmp;
        GSI_CUDA(tmp.alloc(std::max(t1, t2), st));
        if (m) GSI_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, t1, key.p, key2.p, val.p, val2.p, (int)(2 * m), 0, bits, st));
        GSI_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, t2, deg.p, off.p, (int)(n + 1), st));
    }
    // pairs per vertex, their offsets, then the G' edges
    Dev<unsigned long long> cnt, pos;
    GSI_CUDA(cnt.alloc(n + 1, st));
    GSI_CUDA(pos.alloc(n + 1, st));
    GSI_CUDA(cudaMemsetAsync(cnt.p, 0, 8ull * (n + 1), st));
    const unsigned wb = blocks(n * 32);
    if (n) k_line_pairs<false><<<std::min(wb, 148u * 16), kB, 0, st>>>(n, off.p, val2.p, d_src.p, d_dst.p, d_vl.p, cnt.p,
                                                                         nullptr, nullptr, nullptr, nullptr);
    {
        size_t t = 0;
        GSI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t, cnt.p, pos.p, (int)(n + 1), st));
        Dev<unsigned char> tmp;
        GSI_CUDA(tmp.alloc(t, st));
        GSI_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, t, cnt.p, pos.p, (int)(n + 1), st));
    }
    unsigned long long m2 = 0;
    GSI_CUDA(cudaMemcpyAsync(&m2, pos.p + n, 8, cudaMemcpyDeviceToHost, st));
    GSI_CUDA(cudaStreamSynchronize(st));
    if (m2 >= (1ull << 30)) {
        set_error("line graph has " + std::to_string(m2) + " edges (sum of deg(v) choose 2); the build takes < 2^30");
        return GSI_ERR_INVALID_ARG;
    }
    Dev<int32_t> ls, ld, ll;
    GSI_CUDA(ls.alloc(m2, st));
    GSI_CUDA(ld.alloc(m2, st));
    GSI_CUDA(ll.alloc(m2, st));
    if (n && m2)
        k_line_pairs<true><<<std::min(wb, 148u * 16), kB, 0, st>>>(n, off.p, val2.p, d_src.p, d_dst.p, d_vl.p, nullptr,
                                                                  pos.p, ls.p, ld.p, ll.p);
    GSI_CUDA(cudaGetLastError());
    GSI_CUDA(cudaStreamSynchronize(st));
    // G' = (m vertices labelled L_E, m2 edges labelled L_V): the ordinary build
    gsi_build_opts o2{};
    if (opts) o2 = *opts;
    else {
        o2.gpn = 16;
        o2.device = -1;
    }
    o2.stream = st;
    gsi_graph *g = nullptr;
    GSI_TRY(build_graph_impl(m, d_el.p, (int64_t)m2, ls.p, ld.p, ll.p, &o2, &g));
    g->line = true;
    g->line_n = n;
    *out = g;
    return GSI_OK;
}

gsi_status build_graph_ml_impl(int64_t n, const int64_t *vls_off, const int32_t *vls, int64_t m, const int32_t *src,
                               const int32_t *dst, const int64_t *els_off, const int32_t *els,
                               const gsi_build_opts *opts, gsi_graph **out) {
    *out = nullptr;
    if (n < 0 || m < 0 || n >= (1ll << 31) - 1 || !vls_off || (m && (!src || !dst || !els_off))) {
        set_error("invalid graph arguments");
        return GSI_ERR_INVALID_ARG;
    }
    GSI_TRY(check_edges(n, m, src, dst));
    std::vector<int64_t> vo, eo;
    std::vector<int32_t> vlab, elab;
    GSI_TRY(canon_sets(n, vls_off, vls, vo, vlab, "vertex label sets"));
    if (m) GSI_TRY(canon_sets(m, els_off, els, eo, elab, "edge label sets"));
    // every label of an edge becomes one single-label (parallel) edge
    const int64_t m2 = m ? eo[m] : 0;
    if (2 * m2 >= (1ll << 31) - 1) {
        set_error("too many (edge, label) pairs");
        return GSI_ERR_INVALID_ARG;
    }
    std::vector<int32_t> s2((size_t)m2), d2((size_t)m2);
    for (int64_t e = 0; e < m; e++)
        for (int64_t i = eo[e]; i < eo[e + 1]; i++) {
            s2[i] = src[e];
            d2[i] = dst[e];
        }
    std::vector<int32_t> zero((size_t)n, 0);
    gsi_graph *g = nullptr;
    GSI_TRY(build_graph_impl(n, zero.data(), m2, s2.data(), d2.data(), elab.data(), opts, &g));
    std::unique_ptr<gsi_graph, void (*)(gsi_graph *)> guard(g, [](gsi_graph *x) { gsi_graph_free(x); });
    cudaStream_t st = opts && opts->stream ? (cudaStream_t)opts->stream : cudaStreamPerThread;
    GSI_CUDA(cudaSetDevice(g->device));
    GSI_CUDA(cudaMalloc(&g->ml_off, 8ull * (n + 1)));
    GSI_CUDA(cudaMalloc(&g->ml_labs, 4ull * std::max<int64_t>(1, (int64_t)vlab.size())));
    GSI_CUDA(cudaMemcpyAsync(g->ml_off, vo.data(), 8ull * (n + 1), cudaMemcpyHostToDevice, st));
    if (!vlab.empty()) GSI_CUDA(cudaMemcpyAsync(g->ml_labs, vlab.data(), 4ull * vlab.size(), cudaMemcpyHostToDevice, st));
    g->ml = true;
    g->ml_total = (int64_t)vlab.size();
    // signatures of the multi-label graph (reading A19) replace the single-label ones
    Dev<int32_t> ds, dd, de;
    GSI_CUDA(ds.alloc(m2, st));
    GSI_CUDA(dd.alloc(m2, st));
    GSI_CUDA(de.alloc(m2, st));
    if (m2) {
        GSI_CUDA(cudaMemcpyAsync(ds.p, s2.data(), 4ull * m2, cudaMemcpyHostToDevice, st));
        GSI_CUDA(cudaMemcpyAsync(dd.p, d2.data(), 4ull * m2, cudaMemcpyHostToDevice, st));
        GSI_CUDA(cudaMemcpyAsync(de.p, elab.data(), 4ull * m2, cudaMemcpyHostToDevice, st));
    }
    GSI_CUDA(cudaMemsetAsync(g->sig, 0, 4ull * kPlanes * n, st));
    if (n) k_ml_plane0<<<blocks(n), kB, 0, st>>>(n, g->ml_off, g->ml_labs, g->sig);
    if (m2) k_ml_pairs<<<blocks(2 * m2), kB, 0, st>>>(m2, n, ds.p, dd.p, de.p, g->ml_off, g->ml_labs, g->sig);
    GSI_CUDA(cudaGetLastError());
    GSI_CUDA(cudaStreamSynchronize(st));
    *out = guard.release();
    return GSI_OK;
}

gsi_status prepare_ml_impl(const gsi_graph *g, int32_t k, const int32_t *qvls_off, const int32_t *qvls, int32_t qm,
                           const int32_t *qs, const int32_t *qd, const int32_t *qels_off, const int32_t *qels,
                           gsi_prepared **out) {
    *out = nullptr;
    if (!g || !g->ml) {
        set_error("gsi_query_prepare_ml needs a graph from gsi_build_graph_ml");
        return GSI_ERR_INVALID_ARG;
    }
    if (k < 1 || qm < 0 || !qvls_off || (qm && (!qs || !qd || !qels_off))) {
        set_error("invalid query arguments");
        return GSI_ERR_INVALID_ARG;
    }
    if (k > GSI_MAX_K) {
        set_error("query has more than 32 vertices");
        return GSI_ERR_QUERY_TOO_LARGE;
    }
    std::vector<int64_t> vo, eo;
    std::vector<int32_t> vlab, elab;
    GSI_TRY(canon_sets(k, qvls_off, qvls, vo, vlab, "query vertex label sets"));
    if (qm) GSI_TRY(canon_sets(qm, qels_off, qels, eo, elab, "query edge label sets"));
    for (int u = 0; u < k; u++)
        if (vo[u + 1] - vo[u] > 32) {
            set_error("a query vertex has more than 32 labels");
            return GSI_ERR_QUERY_TOO_LARGE;
        }
    const int qm2 = qm ? (int)eo[qm] : 0;
    std::vector<int32_t> s2(qm2), d2(qm2);
    for (int e = 0; e < qm; e++)
        for (int64_t i = eo[e]; i < eo[e + 1]; i++) {
            s2[i] = qs[e];
            d2[i] = qd[e];
        }
    // all query vertices get label 0: the join then treats every unlinked earlier column as a
    // subtraction column (two vertices with different label sets may share a data vertex)
    std::vector<int32_t> zero(k, 0);
    gsi_prepared *p = nullptr;
    GSI_TRY(prepare_impl(g, k, zero.data(), qm2, s2.data(), d2.data(), elab.data(), &p));
    std::unique_ptr<gsi_prepared> guard(p);
    p->ml = true;
    p->qls.assign(k + 1 + vlab.size(), 0);
    for (int u = 0; u <= k; u++) p->qls[u] = (int32_t)vo[u];
    std::copy(vlab.begin(), vlab.end(), p->qls.begin() + k + 1);
    encode_ml(k, p->qls, qm2, s2.data(), d2.data(), elab.data(), p->qsig.data(), 0);
    encode_ml(k, p->qls, qm2, s2.data(), d2.data(), elab.data(), p->qsig.data() + (size_t)k * kPlanes, 1);
    GSI_CUDA(cudaSetDevice(g->device));
    GSI_CUDA(cudaMemcpyAsync(p->d_qsig, p->qsig.data(), p->qsig.size() * 4, cudaMemcpyHostToDevice, cudaStreamPerThread));
    GSI_CUDA(cudaMallocAsync(&p->d_qls, p->qls.size() * 4, cudaStreamPerThread));
    GSI_CUDA(cudaMemcpyAsync(p->d_qls, p->qls.data(), p->qls.size() * 4, cudaMemcpyHostToDevice, cudaStreamPerThread));
    GSI_CUDA(cudaStreamSynchronize(cudaStreamPerThread));
    *out = guard.release();
    return GSI_OK;
}

gsi_status prepare_line_impl(const gsi_graph *g, int32_t k, const int32_t *qvl, int32_t qm, const int32_t *qs,
                             const int32_t *qd, const int32_t *qe, gsi_prepared **out) {
    *out = nullptr;
    if (!g || !g->line) {
        set_error("gsi_query_prepare_line needs a graph from gsi_build_line_graph");
        return GSI_ERR_INVALID_ARG;
    }
    if (k < 2 || qm < 1 || !qvl || !qs || !qd || !qe) {
        set_error("edge isomorphism needs a query with at least one edge");
        return GSI_ERR_INVALID_ARG;
    }
    if (qm > GSI_MAX_K) {
        set_error("query has more than 32 edges (the vertices of its line graph)");
        return GSI_ERR_QUERY_TOO_LARGE;
    }
    if (k > 4 * GSI_MAX_K) {
        set_error("query has too many vertices");
        return GSI_ERR_QUERY_TOO_LARGE;
    }
    // Q itself: labels, endpoints, self-loops, duplicates, connectivity (every vertex on an edge)
    for (int u = 0; u < k; u++)
        if (qvl[u] < 0) {
            set_error("negative query vertex label");
            return GSI_ERR_LABEL_RANGE;
        }
    std::vector<int> seen(k, 0), stack{qs[0] >= 0 && qs[0] < k ? qs[0] : 0};
    for (int e = 0; e < qm; e++) {
        if (qs[e] < 0 || qs[e] >= k || qd[e] < 0 || qd[e] >= k) {
            set_error("query edge endpoint out of range");
            return GSI_ERR_VERTEX_RANGE;
        }
        if (qs[e] == qd[e]) {
            set_error("query self-loop");
            return GSI_ERR_SELF_LOOP;
        }
        if (qe[e] < 0) {
            set_error("negative query edge label");
            return GSI_ERR_LABEL_RANGE;
        }
        for (int f = 0; f < e; f++)
            if (qe[f] == qe[e] && ((qs[f] == qs[e] && qd[f] == qd[e]) || (qs[f] == qd[e] && qd[f] == qs[e]))) {
                set_error("duplicate query edge");
                return GSI_ERR_DUPLICATE_EDGE;
            }
    }
    seen[stack[0]] = 1;
    int reached = 1;
    while (!stack.empty()) {
        const int u = stack.back();
        stack.pop_back();
        for (int e = 0; e < qm; e++) {
            const int o = qs[e] == u ? qd[e] : (qd[e] == u ? qs[e] : -1);
            if (o >= 0 && !seen[o]) {
                seen[o] = 1;
                reached++;
                stack.push_back(o);
            }
        }
    }
    if (reached != k) {
        set_error("query graph is disconnected (PAPER.md L299 assumes connectivity)");
        return GSI_ERR_QUERY_DISCONNECTED;
    }
    // Q' = L(Q): vertex e = query edge e (label L_E(e)); for every query vertex w and pair of
    // its edges a < b, an edge (a, b) labelled L_V(w) (a parallel pair whose shared ends carry
    // the same label: once, at the smaller end — the rule of the data side)
    std::vector<int32_t> s2, d2, l2;
    for (int w = 0; w < k; w++) {
        std::vector<int> inc;
        for (int e = 0; e < qm; e++)
            if (qs[e] == w || qd[e] == w) inc.push_back(e);
        for (size_t i = 0; i < inc.size(); i++)
            for (size_t j = i + 1; j < inc.size(); j++) {
                const int a = inc[i], b = inc[j];
                const int oa = qs[a] == w ? qd[a] : qs[a], ob = qs[b] == w ? qd[b] : qs[b];
                if (oa == ob && qvl[w] == qvl[oa] && w > oa) continue;
                s2.push_back(a);
                d2.push_back(b);
                l2.push_back(qvl[w]);
            }
    }
    gsi_prepared *p = nullptr;
    GSI_TRY(prepare_impl(g, qm, qe, (int32_t)s2.size(), s2.data(), d2.data(), l2.data(), &p));
    p->line = true;
    *out = p;
    return GSI_OK;
}

cudaError_t launch_filter_ml(const gsi_graph *g, const gsi_prepared *q, int hom, uint32_t *bm, long long words,
                             unsigned long long *counts, cudaStream_t st) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
    const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>((words * 32 + kB - 1) / kB, (long long)sms * 8));
    const uint32_t *qsig = q->d_qsig + (hom ? (size_t)q->k * kPlanes : 0);
    k_filter_ml<<<grid, kB, 0, st>>>(g->sig, g->n, q->k, qsig, q->d_qls, g->ml_off, g->ml_labs, bm, words, counts);
    return cudaGetLastError();
}

}  // namespace gsi
