// query.cu — the GSI query hot path on sm_100a: signature filter (§III-A
// L534-552), join-order planner (Alg. 2), and the per-level Prealloc-Combine vertex
// join (Alg. 3, Alg. 4) re-designed for B200:
//
//   k_filter_tw     one pass over the column-first signature table tests all k query
//                   signatures: a thread per bitmap word (32 vertices), label matches queued
//                   per warp for the plane rounds, output words bit-assembled; k_filter<1>
//                   (a warp per word, ballots) for small graphs.  |C(u)|, per-group counts,
//                   and a zero-copy publication of the totals by the last CTA.
//   k_compact_*     level 1: M_1 = C(pi_1) in ascending order (Alg. 2 line 7).
//   k_probe         Prealloc (Alg. 4): one thread per row of M locates N(m_i[c_e], l_e) for
//                   every linking edge in PCSR (one 128 B group probe each, L740-753), caches
//                   (off,len), picks the buffer-bounding edge e0 and scans |N(v',l0)| into F
//                   with a single-pass decoupled look-back (the paper's CUB exclusive scan).
//   k_join          the hot kernel.  The Prealloc range [0, F[|M|]) is the GBA index space;
//                   it is cut into equal tiles of 2048 slots (exact work partition — the B200
//                   form of the 4-layer load balance of L1169-1176: a hub row's buffer is split
//                   across as many CTAs as its length needs, a tiny row shares a CTA).  Slot s
//                   of row i tests x = N(v',l0)[s-F_i]: C(u) bitmap bit (L2-resident bitset,
//                   L1150), set subtraction against the row (Alg. 3 line 10) and membership in
//                   every other linking list (binary search in the sorted run; all edges in one
//                   pass instead of one launch per edge, Alg. 3 line 4).  Survivors are compacted
//                   in slot order through shared memory (the write cache, L1155-1158) and their
//                   global position comes from the same decoupled look-back — the Combine scan of
//                   Alg. 3 line 14 fused into the join; nothing is joined twice.  The CTA then
//                   writes its contiguous block of new rows m_i || x itself (the Combine of
//                   Alg. 3 lines 15-21, coalesced), or, at the last level, counts / hashes /
//                   writes the final table in query-id order.
//   k_next_lean, k_cahead_lean, k_final_fp, k_final_table
//                   warp-centric variants on shared N(v,l0) ∩ C(u) runs.
//   k_abl_*         the paper-style ablation engine (one warp per row, NEXT-3).
//   k_small_query   every level of a small query in one launch after the host plan (M_1
//                   extracted from the filter's group counts, rows on chip).
#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <atomic>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace gsi {

// ====================================================================== device side ===
namespace {

constexpr int kThreads = 256;
#ifndef GSI_PREFILTER_RATIO
#define GSI_PREFILTER_RATIO 2   // share N(v,l0) ∩ C(u) when |GBA| >= ratio x |ci of P(G,l0)| (0: off)
#endif
#ifndef GSI_PREFILTER_AHEAD
#define GSI_PREFILTER_AHEAD 4   // ... and produce a level's rows pre-pointed when 4x its parent's slots exceed it
#endif
#ifndef GSI_PROBE_AHEAD
#define GSI_PROBE_AHEAD 2   // build a step's probe-ahead table when its slots >= 2x its partition (0: off)
#endif
#ifndef GSI_CAHEAD_WARP
#define GSI_CAHEAD_WARP 1   // count-ahead on shared lists: warp-centric kernel (0: slot tiles)
#endif
#ifndef GSI_CAHEAD_MINB
#define GSI_CAHEAD_MINB 4   // k_cahead_warp: resident blocks per SM the registers are sized for
#endif
#ifndef GSI_CAHEAD_LEAN
#define GSI_CAHEAD_LEAN 1   // lean count-ahead kernel for the common shape (0: always k_cahead_warp)
#endif
#ifndef GSI_FILTER_MINB
#define GSI_FILTER_MINB 4   // k_filter: resident blocks per SM the registers are sized for
#endif
#ifndef GSI_NEXT_LEAN
#define GSI_NEXT_LEAN 1     // lean warp-centric J_NEXT writing rows at their Prealloc slots (0: off)
#endif
#ifndef GSI_COUNT_LEAN
#define GSI_COUNT_LEAN 1    // enumerating last level on shared runs: lean warp walk (0: slot tiles)
#endif
#ifndef GSI_NEXT_STAGE
#define GSI_NEXT_STAGE 1    // k_next_lean: stage a batch's rows in shared memory, one coalesced store run
#endif
#ifndef GSI_FP_TERMS
#define GSI_FP_TERMS 1      // enumerating last level: per-candidate fingerprint term table (0: compute)
#endif
#ifndef GSI_TABLE_LEAN
#define GSI_TABLE_LEAN 1    // table-mode last level on shared runs: warp table kernel (0: slot tiles)
#endif
#ifndef GSI_CAHEAD_LONG
#define GSI_CAHEAD_LONG 1   // k_cahead_lean: rows with >= 32 candidates walked warp-cooperatively
#endif
#ifndef GSI_FP_ITEMS
#define GSI_FP_ITEMS 8      // k_filter_partition: entries per thread (tile = 256 x this)
#endif
#ifndef GSI_CAHEAD_U
#define GSI_CAHEAD_U 1      // k_cahead_warp: slots per lane per pass
#endif
#ifndef GSI_STAGE_ROWS
#define GSI_STAGE_ROWS 1    // join tile staging: rows per thread per pass (loads phased together)
#endif
#ifndef GSI_STAGE_NEXT
#define GSI_STAGE_NEXT 1    // J_NEXT: stage a row-constant next-step run per tile row
#endif
#ifndef GSI_FAST_ITEMS
#define GSI_FAST_ITEMS 16   // slots per thread of the lean count-only kernel (0: never use it)
#endif
#ifndef GSI_STAGE_BASE
#define GSI_STAGE_BASE 1  // stage per-row ci bases in the join tile
#endif
#ifndef GSI_STAGE_INJ
#define GSI_STAGE_INJ 1   // stage up to this many subtraction columns per row
#endif
#ifndef GSI_STAGE_DIV
#define GSI_STAGE_DIV 4   // stage a tile's rows when it has >= GSI_STAGE_DIV slots per row
#endif
constexpr int kJoinItems = 8;
constexpr int kJoinTile = kThreads * kJoinItems;   // 2048 GBA slots per CTA

struct StepParams {
    int t;                       // columns of M (current level)
    int E;                       // linking edges
    int per_row_e0;              // 1: per-row shortest list bounds the buffer
    int k;                       // query size (final level only)
    int col[GSI_MAX_K];          // column of linking edge e
    uint32_t lab[GSI_MAX_K];     // dense label of linking edge e
    unsigned long long gbase[GSI_MAX_K];
    uint32_t ngroups[GSI_MAX_K];
    int n_inj;
    int inj_col[GSI_MAX_K];      // columns the subtraction must test (same vertex label as u)
    int pos_of_q[GSI_MAX_K];     // final level: column (0..t) holding query vertex q
    int fp;                      // final level: accumulate the set fingerprint
    int prefiltered;             // loc / ci point at N(v,l0) ∩ C(u) (k_filter_partition): no bitmap test
    const uint32_t *fpos;        // (as the NEXT step of J_NEXT) filtered positions of P(G,l0)'s ci
    uint32_t flo, fhi;           //   ... and the partition's ci range
    int stage_base;              // join tile stages per-row ci bases in shared memory
    int stage_inj;               // ... and up to this many subtraction columns
    const Loc *pa;               // probe-ahead table of this step: pa[p] = the NEXT step's filtered
                                 //   run of x = (prefiltered ci)[p] (null: probe PCSR per new row)
    const uint32_t *cu;          // (as the counted final step of J_CAHEAD) C(u) bitmap ...
    const int32_t *fci;          //   ... and the shared N(v,l0) ∩ C(u) runs of P(G,l0)
    int stage_next;              // J_NEXT: the next step's run is row-constant (links to a parent
                                 //   column): located once per tile row into shared memory
    int no_f2;                   // J_NEXT: the next level walks rows without F (warp count-ahead):
                                 //   skip F' and its look-back chain, only total them
    int out_w;                   // J_NEXT: stored columns of a new row (count-only: live ones)
    int out_src[GSI_MAX_K];      //   ... column j = parent column out_src[j], or x if < 0
};

// Counters shared by the kernels of one query (device).
struct Counters {
    unsigned long long list_elems;   // algorithmic list elements of active rows
    unsigned long long active_rows;  // rows with a non-empty prealloc buffer
    unsigned long long count;        // final count (count-only mode) / survivors
    unsigned long long fp1, fp2;
    unsigned long long plane_loads;  // filter: signature plane words read (planes 1..15)
    unsigned long long total;        // scan totals written by the last tile
    unsigned long long total2;       // F'[|M'|] of the probe-ahead (J_NEXT)
};
constexpr unsigned long long kCtrWords = (sizeof(Counters) + 31) / 32 * 4;   // 8 B words, 32 B aligned

// Zero-copy publication of the filter's totals (the host's only wait between the filter and the
// plan): the last CTA to finish — threadFenceReduction's ticket — writes |C(u)| and the plane
// loads to mapped pinned host memory and raises a flag the host spins on, instead of a
// device-to-host copy and a stream synchronisation (~15-25 us of DMA set-up and wake-up).
// hpub: [0, k) |C(u)|, [GSI_MAX_K] plane loads, [GSI_MAX_K + 1] flag (null: not published).
__device__ __forceinline__ void filter_publish(int k, const unsigned long long *counts, const Counters *ctr,
                                               unsigned *done, unsigned long long *hpub) {
    __shared__ bool last;
    if (!hpub) return;
    __threadfence();   // this CTA's count atomics are visible device-wide before its ticket
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    volatile unsigned long long *vh = hpub;
    if (threadIdx.x < k) vh[threadIdx.x] = reinterpret_cast<volatile const unsigned long long *>(counts)[threadIdx.x];
    if (threadIdx.x == 0) vh[GSI_MAX_K] = reinterpret_cast<volatile const Counters *>(ctr)->plane_loads;
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) vh[GSI_MAX_K + 1] = 1ull;
}


// ---------------------------------------------------------------------- filter ------
// One pass over the signature table (§III-A): per data vertex v, plane 0 (its label)
// picks the query vertices u with L_V(u) = L_V(v) (A4: one hash probe, not k compares), then
// S(v) & S(u) = S(u) is tested only on the planes where S(u) has a set bit (a plane whose
// query word is 0 is contained in anything).  A warp takes FW bitmap words (32·FW vertices) per
// iteration: the plane-0 loads of all FW words are issued together, then the vertices with a
// label match — often a few percent of them — are compacted through a per-warp shared-memory
// queue into ceil(matches / 32) dense columns, so the plane tests run on full lanes instead of
// on the mostly idle lanes of FW sparse words.  The planes are tested in rounds: each round
// issues the next needed plane load of every queued vertex before testing any of them (the
// first plane tested rejects most of a label class; later planes are read for the survivors
// only).  FW = 8 with streaming loads for large graphs; FW = 1 with cached loads for small
// ones, whose signature table stays L2-resident and which need the extra warps.
template <int FW>
__global__ void __launch_bounds__(kThreads, GSI_FILTER_MINB) k_filter(const uint32_t *__restrict__ sig, long long n, int k,
                                                     const uint32_t *__restrict__ qsig, int label_only,
                                                     uint32_t *__restrict__ bitmaps, long long words,
                                                     unsigned long long *__restrict__ counts,
                                                     Counters *__restrict__ ctr,
                                                     uint16_t *__restrict__ grp, long long grp_stride,
                                                     unsigned *done, unsigned long long *hpub) {
    // grp (optional): grp[u * grp_stride + g] = |C(u)| in bitmap words [g·FW, (g+1)·FW) — a
    // summary the device-planned small path extracts M_1 = C(pi_1) from without a scan of
    // the whole bitmap (a warp's FW words are always one whole group)
    static_assert(FW == 1 || FW % 4 == 0, "the bitmap store is 16 B vectors per query vertex");
    constexpr bool kStream = FW > 1;                 // large graphs: evict-first signature reads
    constexpr int kHT = 64;                          // label -> query-vertex mask, open addressing
    constexpr int kWarps = kThreads / 32;
    __shared__ uint32_t qs[GSI_MAX_K * kPlanes];
    __shared__ uint32_t qneed[GSI_MAX_K];            // planes 1..15 where S(u) has a set bit
    __shared__ uint32_t ht_lab[kHT], ht_mask[kHT];
    __shared__ unsigned long long cnt_s[GSI_MAX_K];
    __shared__ unsigned long long loads_s;
    __shared__ uint32_t q_slot[kWarps][32 * FW];     // queued vertex: j * 32 + lane of its word
    __shared__ uint32_t q_mask[kWarps][32 * FW];     // its candidate mask, then its final mask
    for (int i = threadIdx.x; i < k * kPlanes; i += blockDim.x) qs[i] = qsig[i];
    if (threadIdx.x < GSI_MAX_K) cnt_s[threadIdx.x] = 0;
    if (threadIdx.x < kHT) {
        ht_lab[threadIdx.x] = 0xFFFFFFFFu;           // empty (labels are < 2^31)
        ht_mask[threadIdx.x] = 0u;
    }
    if (threadIdx.x == 0) loads_s = 0;
    __syncthreads();
    if (threadIdx.x < k) {
        uint32_t m = 0;
        for (int pl = 1; pl < kPlanes; pl++)
            if (qs[threadIdx.x * kPlanes + pl]) m |= 1u << pl;
        qneed[threadIdx.x] = m;
    }
    if (threadIdx.x == 0)
        for (int u = 0; u < k; u++) {
            const uint32_t L = qs[u * kPlanes];
            uint32_t h = (L * 0x9E3779B1u) >> 26;
            while (ht_lab[h] != 0xFFFFFFFFu && ht_lab[h] != L) h = (h + 1) & (kHT - 1);
            ht_lab[h] = L;
            ht_mask[h] |= 1u << u;
        }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    uint32_t *const qslot = q_slot[wid];
    uint32_t *const qmask = q_mask[wid];
    const long long warps = (long long)gridDim.x * kWarps;
    unsigned long long plane_words = 0;   // plane words this thread read (algorithmic bytes / 4)
    unsigned long long my_count = 0;      // |C(u)| partial for u = lane
    for (long long w0 = (blockIdx.x * (long long)kWarps + wid) * FW; w0 < words; w0 += warps * FW) {
        uint32_t lab[FW], mask[FW];
#pragma unroll
        for (int j = 0; j < FW; j++) {
            const long long v = (w0 + j) * 32 + lane;
            const bool in = w0 + j < words && v < n;
            lab[j] = in ? (kStream ? __ldcs(sig + v) : __ldg(sig + v)) : 0xFFFFFFFEu;   // matches no query label
        }
#pragma unroll
        for (int j = 0; j < FW; j++) {   // label field by equality (A4): one hash probe, not k compares
            uint32_t h = (lab[j] * 0x9E3779B1u) >> 26, e;
            while ((e = ht_lab[h]) != lab[j] && e != 0xFFFFFFFFu) h = (h + 1) & (kHT - 1);
            mask[j] = e == lab[j] ? ht_mask[h] : 0u;
        }
        if (!label_only) {
            // compact the label-matching vertices of the FW words into the warp's queue
            int nq = 0;
            uint32_t has = 0u;   // bit j: this lane's vertex of word j is queued (mask[j] lives in the queue)
#pragma unroll
            for (int j = 0; j < FW; j++) {
                const unsigned bal = __ballot_sync(0xffffffffu, mask[j] != 0u);
                if (mask[j]) {
                    const int p = nq + __popc(bal & lt_mask);
                    qslot[p] = (uint32_t)(j * 32 + lane);
                    qmask[p] = mask[j];
                    has |= 1u << j;
                }
                nq += __popc(bal);
            }
            __syncwarp();
            if (nq) {
                const int nc = (nq + 31) >> 5;   // dense columns of the queue
                uint32_t m[FW], rem[FW], vv[FW];   // rem: needed planes not yet tested; vertex ids < 2^31
#pragma unroll
                for (int c = 0; c < FW; c++) {
                    const int i = c * 32 + lane;
                    m[c] = 0u;
                    rem[c] = 0u;
                    vv[c] = 0u;
                    if (c < nc && i < nq) {
                        const uint32_t sl = qslot[i];
                        m[c] = qmask[i];
                        vv[c] = (uint32_t)((w0 + (sl >> 5)) * 32 + (sl & 31));
                        uint32_t t = m[c];
                        while (t) {
                            rem[c] |= qneed[__ffs(t) - 1];
                            t &= t - 1;
                        }
                    }
                }
                for (int round = 0; round < kPlanes; round++) {
                    uint32_t pv[FW];
                    int pls[FW];
                    bool any = false;
#pragma unroll
                    for (int c = 0; c < FW; c++) {
                        pls[c] = -1;
                        pv[c] = 0u;
                        if (c < nc) {
                            if (m[c] && rem[c]) {
                                pls[c] = __ffs(rem[c]) - 1;
                                const uint32_t *src = sig + (long long)pls[c] * n + vv[c];
                                pv[c] = kStream ? __ldcs(src) : __ldg(src);
                                any = true;
                            }
                        }
                    }
                    if (!__any_sync(0xffffffffu, any)) break;
#pragma unroll
                    for (int c = 0; c < FW; c++) {
                        if (pls[c] < 0) continue;
                        rem[c] &= ~(1u << pls[c]);
                        plane_words++;
                        uint32_t t = m[c];
                        while (t) {
                            const int u = __ffs(t) - 1;
                            t &= t - 1;
                            const uint32_t sq = qs[u * kPlanes + pls[c]];
                            if ((pv[c] & sq) != sq) m[c] &= ~(1u << u);   // S(v)&S(u)=S(u) fails on this plane
                        }
                    }
                }
#pragma unroll
                for (int c = 0; c < FW; c++)
                    if (c < nc && c * 32 + lane < nq) qmask[c * 32 + lane] = m[c];
                __syncwarp();
                // scatter the final masks back to the words (a queued vertex's slot is known
                // to its own lane: the p-th match of word j is the lane's own vertex)
                int base = 0;
#pragma unroll
                for (int j = 0; j < FW; j++) {
                    const bool h = (has >> j) & 1u;
                    const unsigned bal = __ballot_sync(0xffffffffu, h);
                    mask[j] = h ? qmask[base + __popc(bal & lt_mask)] : 0u;
                    base += __popc(bal);
                }
            }
            __syncwarp();   // the queue is reused by the next iteration
        }
        // lane u collects the FW bitmap words of query vertex u (ballots only for the query
        // vertices some lane matched)
        uint32_t mine[FW];
#pragma unroll
        for (int j = 0; j < FW; j++) {
            mine[j] = 0u;
            uint32_t present = __reduce_or_sync(0xffffffffu, mask[j]);
            while (present) {
                const int u = __ffs(present) - 1;
                present &= present - 1;
                const unsigned b = __ballot_sync(0xffffffffu, (mask[j] >> u) & 1u);
                if (lane == u) mine[j] = b;
            }
        }
        if (lane < k) {
            uint32_t *dst = bitmaps + (long long)lane * words + w0;
            if (FW % 4 == 0 && w0 + FW <= words && ((words & 3) == 0)) {
#pragma unroll
                for (int j = 0; j < FW; j += 4)
                    *reinterpret_cast<uint4 *>(dst + j) = make_uint4(mine[j], mine[j + 1], mine[j + 2], mine[j + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < FW; j++)
                    if (w0 + j < words) dst[j] = mine[j];
            }
            unsigned gc = 0;
#pragma unroll
            for (int j = 0; j < FW; j++) gc += __popc(mine[j]);
            my_count += gc;
            if (grp) grp[(long long)lane * grp_stride + w0 / FW] = (uint16_t)gc;
        }
    }
    if (lane < k && my_count) atomicAdd(&cnt_s[lane], my_count);
    plane_words = warp_sum_u64(plane_words);
    if (lane == 0 && plane_words) atomicAdd(&loads_s, plane_words);
    __syncthreads();
    if (threadIdx.x < k && cnt_s[threadIdx.x]) atomicAdd(&counts[threadIdx.x], cnt_s[threadIdx.x]);
    if (threadIdx.x == 0 && loads_s) atomicAdd(&ctr->plane_loads, loads_s);
    filter_publish(k, counts, ctr, done, hpub);
}

// Large graphs: one thread per bitmap word (32 consecutive vertices), so the k output words of
// a word are assembled with bit operations instead of one warp ballot per (word, query vertex).
// Phase A: the thread reads its 32 plane-0 labels (eight 16 B loads) and marks the vertices
// whose label some query vertex has (a register copy of the hash table's occupancy rejects most
// labels without a shared-memory probe).  Phase B: the warp queues the marked vertices
// (vertex id, candidate mask) in shared memory and tests the needed planes on the queue in
// rounds, 32 lanes × up to kTwCols dense columns, exactly as k_filter; a survivor sets its
// bit of every remaining u in the warp's shared output tile.  Phase C: thread w stores word w
// of every C(u) — coalesced 128 B per u across the warp — and the warp sums |C(u)| per group
// of 32 words (grp, gw = 32).
#ifndef GSI_TW_P
#define GSI_TW_P 1                               // plane loads per entry per round for queues of <= 64 (A/B r2t: 1-3 equal)
#endif
constexpr int kTwCols = 8;                       // queue columns per round (256 entries per warp)
constexpr int kTwLabelBits = 4096;               // labels below this are matched exactly by a bit test
constexpr int kTwWarps = kThreads / 32;
inline size_t filter_tw_smem(int k) { return (size_t)kTwWarps * (32 * kTwCols * 8 + (size_t)k * 32 * 4); }

__device__ __forceinline__ uint32_t ht_lookup(const uint32_t *ht_lab, const uint32_t *ht_mask, uint32_t L) {
    constexpr int kHT = 64;
    uint32_t h = (L * 0x9E3779B1u) >> 26, e;
    while ((e = ht_lab[h]) != L && e != 0xFFFFFFFFu) h = (h + 1) & (kHT - 1);
    return e == L ? ht_mask[h] : 0u;
}

// Plane rounds on a warp's queue of qn <= 32·NC label-matched vertices (k_filter_tw phase B):
// lane takes entries lane + 32c; each round issues the next P needed plane loads of every
// entry before testing any (P > 1 for short queues: the chain of dependent rounds, not the
// bytes, is their critical path); a survivor sets its bit of each remaining u in the output tile.
template <int NC, int P>
__device__ __forceinline__ void tw_rounds(const uint32_t *q_v, const uint32_t *q_m, int qn, const uint32_t *qneed,
                                          const uint32_t *qs, const uint32_t *__restrict__ sig, long long n,
                                          uint32_t *outw, long long wb, unsigned long long &plane_words) {
    const int lane = threadIdx.x & 31;
    uint32_t m[NC], need[NC], vv[NC];
#pragma unroll
    for (int c = 0; c < NC; c++) {
        const int i = c * 32 + lane;
        m[c] = 0u;
        need[c] = 0u;
        vv[c] = 0u;
        if (i < qn) {
            vv[c] = q_v[i];
            m[c] = q_m[i];
            uint32_t t = m[c];
            while (t) {
                need[c] |= qneed[__ffs(t) - 1];
                t &= t - 1;
            }
        }
    }
    for (int round = 0; round < kPlanes; round++) {
        uint32_t pv[NC][P];
        int pls[NC][P];
        bool any = false;
#pragma unroll
        for (int c = 0; c < NC; c++) {
            uint32_t rem = m[c] ? need[c] : 0u;
#pragma unroll
            for (int q = 0; q < P; q++) {
                pls[c][q] = -1;
                pv[c][q] = 0u;
                if (rem) {
                    pls[c][q] = __ffs(rem) - 1;
                    rem &= rem - 1;
                    pv[c][q] = __ldcs(sig + (long long)pls[c][q] * n + vv[c]);
                    any = true;
                }
            }
        }
        if (!__any_sync(0xffffffffu, any)) break;
#pragma unroll
        for (int c = 0; c < NC; c++)
#pragma unroll
            for (int q = 0; q < P; q++) {
                if (pls[c][q] < 0) continue;
                need[c] &= ~(1u << pls[c][q]);
                plane_words++;
                uint32_t t = m[c];
                while (t) {
                    const int u = __ffs(t) - 1;
                    t &= t - 1;
                    const uint32_t sq = qs[u * kPlanes + pls[c][q]];
                    if ((pv[c][q] & sq) != sq) m[c] &= ~(1u << u);   // S(v)&S(u)=S(u) fails on this plane
                }
            }
    }
#pragma unroll
    for (int c = 0; c < NC; c++) {
        uint32_t t = m[c];
        if (!t) continue;
        const uint32_t wl = (uint32_t)((long long)(vv[c] >> 5) - wb), bit = 1u << (vv[c] & 31);
        while (t) {
            const int u = __ffs(t) - 1;
            t &= t - 1;
            atomicOr(&outw[u * 32 + wl], bit);
        }
    }
}

__global__ void __launch_bounds__(kThreads, 4) k_filter_tw(const uint32_t *__restrict__ sig, long long n, int k,
                                                           const uint32_t *__restrict__ qsig, int label_only,
                                                           uint32_t *__restrict__ bitmaps, long long words,
                                                           unsigned long long *__restrict__ counts,
                                                           Counters *__restrict__ ctr,
                                                           uint16_t *__restrict__ grp, long long grp_stride,
                                                           unsigned *done, unsigned long long *hpub) {
    constexpr int kHT = 64;
    constexpr int kCap = 32 * kTwCols;
    __shared__ uint32_t qs[GSI_MAX_K * kPlanes];
    __shared__ uint32_t qneed[GSI_MAX_K];
    __shared__ uint32_t ht_lab[kHT], ht_mask[kHT];
    __shared__ unsigned long long occ_s;
    __shared__ uint32_t lbits[kTwLabelBits / 32];   // bit L: some query vertex has label L (L < 4096)
    __shared__ unsigned long long cnt_s[GSI_MAX_K];
    __shared__ unsigned long long loads_s;
    extern __shared__ __align__(16) uint32_t tw_dyn[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *const q_v = tw_dyn + wid * (kCap * 2);             // queued vertex ids
    uint32_t *const q_m = q_v + kCap;                             // their candidate masks
    uint32_t *const outw = tw_dyn + kTwWarps * kCap * 2 + wid * k * 32;   // [u][word in the warp]
    for (int i = threadIdx.x; i < k * kPlanes; i += blockDim.x) qs[i] = qsig[i];
    if (threadIdx.x < GSI_MAX_K) cnt_s[threadIdx.x] = 0;
    if (threadIdx.x < kHT) {
        ht_lab[threadIdx.x] = 0xFFFFFFFFu;
        ht_mask[threadIdx.x] = 0u;
    }
    if (threadIdx.x == 0) loads_s = 0;
    for (int i = lane; i < k * 32; i += 32) outw[i] = 0u;
    for (int i = threadIdx.x; i < kTwLabelBits / 32; i += blockDim.x) lbits[i] = 0u;
    __syncthreads();
    if (threadIdx.x < k && qs[threadIdx.x * kPlanes] < (uint32_t)kTwLabelBits)
        atomicOr(&lbits[qs[threadIdx.x * kPlanes] >> 5], 1u << (qs[threadIdx.x * kPlanes] & 31));
    if (threadIdx.x < k) {
        uint32_t m = 0;
        for (int pl = 1; pl < kPlanes; pl++)
            if (qs[threadIdx.x * kPlanes + pl]) m |= 1u << pl;
        qneed[threadIdx.x] = m;
    }
    if (threadIdx.x == 0) {
        unsigned long long occ = 0;
        for (int u = 0; u < k; u++) {
            const uint32_t L = qs[u * kPlanes];
            uint32_t h = (L * 0x9E3779B1u) >> 26;
            while (ht_lab[h] != 0xFFFFFFFFu && ht_lab[h] != L) h = (h + 1) & (kHT - 1);
            ht_lab[h] = L;
            ht_mask[h] |= 1u << u;
            occ |= 1ull << h;
        }
        occ_s = occ;
    }
    __syncthreads();
    const unsigned long long occ = occ_s;   // slot h empty => no query vertex has a label hashing to h
    const unsigned lt_mask = (1u << lane) - 1u;
    const long long nwarps = (long long)gridDim.x * kTwWarps;
    unsigned long long plane_words = 0, my_count = 0;
    for (long long wb = (blockIdx.x * (long long)kTwWarps + wid) * 32; wb < words; wb += nwarps * 32) {
        const long long w = wb + lane;
        const long long v0 = w * 32;
        // ---- phase A: this word's label matches
        uint32_t mb = 0u, big = 0u;
        if (w < words) {
            const uint4 *src = reinterpret_cast<const uint4 *>(sig + v0);
            const int nv = (int)min(32ll, n - v0);
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const uint4 l4 = __ldg(src + c);
                const uint32_t l[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    // exact for labels < 4096 (one shared-memory bit); larger labels are set
                    // aside and tested below against the hash table's occupancy
                    const int b = c * 4 + i;
                    const uint32_t L = l[i], Lc = min(L, (uint32_t)kTwLabelBits - 1u);
                    mb |= ((lbits[Lc >> 5] >> (Lc & 31)) & (L < (uint32_t)kTwLabelBits ? 1u : 0u)) << b;
                    big |= (L >= (uint32_t)kTwLabelBits ? 1u : 0u) << b;
                }
            }
            for (uint32_t t = big; t; t &= t - 1) {   // labels >= 4096 (rare): occupancy, then the probe below
                const int b = __ffs(t) - 1;
                const uint32_t L = __ldg(sig + v0 + b);
                if ((occ >> ((L * 0x9E3779B1u) >> 26)) & 1ull) mb |= 1u << b;
            }
            if (nv < 32) mb &= (1u << nv) - 1u;
        }
        if (label_only) {
            // C(u) by label alone: every marked vertex joins all its label's query vertices
            uint32_t rem = mb;
            while (rem) {
                const int b = __ffs(rem) - 1;
                rem &= rem - 1;
                uint32_t m = ht_lookup(ht_lab, ht_mask, __ldg(sig + v0 + b));
                while (m) {
                    const int u = __ffs(m) - 1;
                    m &= m - 1;
                    atomicOr(&outw[u * 32 + lane], 1u << b);
                }
            }
        } else {
            // ---- phase B: queue the marked vertices, test their planes in rounds
            uint32_t rem = mb;
            int qn = 0;
            for (;;) {
                const bool more = __any_sync(0xffffffffu, rem != 0u);
                if (more) {
                    const bool act = rem != 0u;
                    const unsigned bal = __ballot_sync(0xffffffffu, act);
                    if (act) {
                        const int b = __ffs(rem) - 1;
                        rem &= rem - 1;
                        const int p = qn + __popc(bal & lt_mask);
                        q_v[p] = (uint32_t)(v0 + b);
                        q_m[p] = ht_lookup(ht_lab, ht_mask, __ldg(sig + v0 + b));
                    }
                    qn += __popc(bal);
                }
                if (qn == 0 && !more) break;
                if (qn > kCap - 32 || !more) {
                    __syncwarp();
                    const int nc = (qn + 31) >> 5;   // dense columns: the rounds run on NC >= nc
                    if (nc <= 1) tw_rounds<1, GSI_TW_P>(q_v, q_m, qn, qneed, qs, sig, n, outw, wb, plane_words);
                    else if (nc <= 2) tw_rounds<2, GSI_TW_P>(q_v, q_m, qn, qneed, qs, sig, n, outw, wb, plane_words);
                    else if (nc <= 4) tw_rounds<4, 1>(q_v, q_m, qn, qneed, qs, sig, n, outw, wb, plane_words);
                    else tw_rounds<kTwCols, 1>(q_v, q_m, qn, qneed, qs, sig, n, outw, wb, plane_words);
                    __syncwarp();
                    qn = 0;
                    if (!more) break;
                }
            }
        }
        __syncwarp();
        // ---- phase C: word w of every C(u), coalesced per u; |C(u)| per 32-word group
        for (int u = 0; u < k; u++) {
            const uint32_t word = outw[u * 32 + lane];
            outw[u * 32 + lane] = 0u;
            if (w < words) bitmaps[(long long)u * words + w] = word;
            const unsigned c = __reduce_add_sync(0xffffffffu, (unsigned)__popc(word));
            if (lane == u) {
                my_count += c;
                if (grp) grp[(long long)u * grp_stride + wb / 32] = (uint16_t)c;
            }
        }
        __syncwarp();
    }
    if (lane < k && my_count) atomicAdd(&cnt_s[lane], my_count);
    plane_words = warp_sum_u64(plane_words);
    if (lane == 0 && plane_words) atomicAdd(&loads_s, plane_words);
    __syncthreads();
    if (threadIdx.x < k && cnt_s[threadIdx.x]) atomicAdd(&counts[threadIdx.x], cnt_s[threadIdx.x]);
    if (threadIdx.x == 0 && loads_s) atomicAdd(&ctr->plane_loads, loads_s);
    filter_publish(k, counts, ctr, done, hpub);
}

// Filter variant for a graph: the warp-per-word kernel (FW = 1) while one wave of the device
// still takes at most ~4 iterations per warp (small graphs: parallelism and L2 reuse), else the
// thread-per-word kernel.  Returns the group width of the per-group counts (grp).
inline int filter_fw(long long words, int sms) { return words <= (long long)sms * 8 * 8 * 4 ? 1 : 32; }

cudaError_t launch_filter(const uint32_t *sig, long long n, int k, const uint32_t *qsig, int label_only,
                          uint32_t *bm, long long words, unsigned long long *counts, Counters *ctr, uint16_t *grp,
                          long long grp_stride, int sms, cudaStream_t st, unsigned *done = nullptr,
                          unsigned long long *hpub = nullptr) {
    if (filter_fw(words, sms) == 1) {
        const long long per_cta = kThreads / 32;
        const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>((words + per_cta - 1) / per_cta,
                                                                                    (long long)sms * 8));
        k_filter<1><<<grid, kThreads, 0, st>>>(sig, n, k, qsig, label_only, bm, words, counts, ctr, grp, grp_stride,
                                               done, hpub);
    } else {
        const long long per_cta = 32ll * kTwWarps;
        const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>((words + per_cta - 1) / per_cta,
                                                                                    (long long)sms * 4));
        k_filter_tw<<<grid, kThreads, filter_tw_smem(k), st>>>(sig, n, k, qsig, label_only, bm, words, counts, ctr,
                                                                grp, grp_stride, done, hpub);
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------ level-1 compaction ----
// Tile = 256 bitmap words; M_1 ascending (Alg. 2 line 7: M = C(u_c)).
__global__ void __launch_bounds__(kThreads) k_compact_bitmap(const uint32_t *__restrict__ bm, long long words,
                                                             int32_t *__restrict__ out,
                                                             unsigned long long *status, unsigned *tile_ctr,
                                                             Counters *ctr) {
    __shared__ unsigned long long sm[33];
    __shared__ unsigned tile_s;
    __shared__ unsigned long long base_s;
    if (threadIdx.x == 0) tile_s = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const unsigned tile = tile_s;
    const long long w = (long long)tile * kThreads + threadIdx.x;
    const uint32_t word = w < words ? bm[w] : 0u;
    unsigned long long agg;
    unsigned long long ex = block_exclusive_scan((unsigned long long)__popc(word), sm, &agg);
    if (threadIdx.x < 32) {
        unsigned long long pre = lookback_exclusive(status, tile, agg);
        if (threadIdx.x == 0) base_s = pre;
    }
    __syncthreads();
    unsigned long long pos = base_s + ex;
    uint32_t x = word;
    while (x) {
        int b = __ffs(x) - 1;
        x &= x - 1;
        out[pos++] = (int32_t)(w * 32 + b);
    }
    if (tile == gridDim.x - 1 && threadIdx.x == 0) ctr->total = base_s + agg;
}

// Roots restriction (test hook / root-restricted parity): keep sorted roots that are in C(pi_1).
__global__ void __launch_bounds__(kThreads) k_compact_roots(const int32_t *__restrict__ roots, long long nroots,
                                                            const uint32_t *__restrict__ bm,
                                                            int32_t *__restrict__ out,
                                                            unsigned long long *status, unsigned *tile_ctr,
                                                            Counters *ctr) {
    __shared__ unsigned long long sm[33];
    __shared__ unsigned tile_s;
    __shared__ unsigned long long base_s;
    if (threadIdx.x == 0) tile_s = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const unsigned tile = tile_s;
    const long long i = (long long)tile * kThreads + threadIdx.x;
    int32_t v = i < nroots ? roots[i] : -1;
    bool keep = v >= 0 && ((bm[v >> 5] >> (v & 31)) & 1u);
    unsigned long long agg;
    unsigned long long ex = block_exclusive_scan(keep ? 1ull : 0ull, sm, &agg);
    if (threadIdx.x < 32) {
        unsigned long long pre = lookback_exclusive(status, tile, agg);
        if (threadIdx.x == 0) base_s = pre;
    }
    __syncthreads();
    if (keep) out[base_s + ex] = v;
    if (tile == gridDim.x - 1 && threadIdx.x == 0) ctr->total = base_s + agg;
}

// ---------------------------------------------------------------------- probe -------
// Alg. 4 for one row: locate N(v', l_e) for every linking edge of the next step (one PCSR
// group probe each), write the row's loc entries and return its buffer bound.
// In per-row mode entry 0 becomes the row's shortest list (any linking edge bounds buf_i,
// L967-981) and a row with an empty list gets a zero-size buffer.  Column c of the row is
// row[c] for c < t_parent and `newv` for c == t_parent (the vertex the join just added).
__device__ __forceinline__ void probe_row(const int32_t *__restrict__ row, int t_parent, uint32_t newv,
                                          const StepParams &P, const uint2 *__restrict__ groups, int gpn,
                                          Loc *__restrict__ L, unsigned long long &len0, unsigned long long &elems) {
    Loc first{0, 0}, best{0, 0};
    int bi = 0;
    bool anyzero = false;
    unsigned long long sum = 0;
    for (int e = 0; e < P.E; e++) {
        const int c = P.col[e];
        const uint32_t v = c < t_parent ? (uint32_t)__ldg(row + c) : newv;
        const Loc r = pcsr_lookup(groups, gpn, P.gbase[e], P.ngroups[e], P.lab[e], v, nullptr);
        L[e] = r;
        if (e == 0) {
            first = r;
            best = r;
        } else if (r.len < best.len) {
            best = r;
            bi = e;
        }
        anyzero |= r.len == 0;
        sum += r.len;
    }
    if (P.per_row_e0) {
        if (bi != 0) {
            L[0] = best;
            L[bi] = first;
        }
        len0 = anyzero ? 0ull : best.len;
        elems = anyzero ? 0ull : sum;
    } else {
        len0 = first.len;
        elems = sum;
    }
}

// The buffer bound of a candidate new row without writing anything (used to drop rows whose
// next-step buffer is empty before they are stored).
__device__ __forceinline__ void probe_row_local(const int32_t *__restrict__ row, int t_parent, uint32_t newv,
                                                const StepParams &P, const uint2 *__restrict__ groups, int gpn,
                                                Loc *L, unsigned long long &len0, unsigned long long &elems) {
    unsigned long long best = ~0ull, sum = 0, first = 0;
    bool anyzero = false;
    for (int e = 0; e < P.E; e++) {
        const int c = P.col[e];
        const uint32_t v = c < t_parent ? (uint32_t)__ldg(row + c) : newv;
        const Loc r = pcsr_lookup(groups, gpn, P.gbase[e], P.ngroups[e], P.lab[e], v, nullptr);
        if (e == 0) first = r.len;
        best = r.len < best ? r.len : best;
        anyzero |= r.len == 0;
        sum += r.len;
    }
    (void)L;
    if (P.per_row_e0) {
        len0 = anyzero ? 0ull : best;
        elems = anyzero ? 0ull : sum;
    } else {
        len0 = first;
        elems = sum;
    }
}

// Level 1: F[i] = sum_{i'<i} |N(v'_{i'}, l0)|, F[|M|] = |GBA|, by decoupled look-back.
__global__ void __launch_bounds__(kThreads) k_probe(const int32_t *__restrict__ M, long long nM, StepParams P,
                                                    const uint2 *__restrict__ groups, int gpn,
                                                    Loc *__restrict__ loc, unsigned long long *__restrict__ F,
                                                    unsigned long long *status, unsigned *tile_ctr,
                                                    Counters *ctr) {
    __shared__ unsigned long long sm[33];
    __shared__ unsigned tile_s;
    __shared__ unsigned long long base_s;
    if (threadIdx.x == 0) tile_s = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const unsigned tile = tile_s;
    const long long i = (long long)tile * kThreads + threadIdx.x;
    unsigned long long len0 = 0, elems = 0;
    if (i < nM) probe_row(M + i * P.t, P.t, 0u, P, groups, gpn, loc + i * P.E, len0, elems);
    unsigned long long agg;
    const unsigned long long ex = block_exclusive_scan(len0, sm, &agg);
    if (threadIdx.x < 32) {
        const unsigned long long pre = lookback_exclusive(status, tile, agg);
        if (threadIdx.x == 0) base_s = pre;
    }
    __syncthreads();
    if (i < nM) F[i] = base_s + ex;
    if (tile == gridDim.x - 1 && threadIdx.x == kThreads - 1) F[nM] = base_s + agg;
    const unsigned long long e1 = warp_sum_u64(elems), a1 = warp_sum_u64(len0 ? 1ull : 0ull);
    if ((threadIdx.x & 31) == 0) {
        if (e1) atomicAdd(&ctr->list_elems, e1);
        if (a1) atomicAdd(&ctr->active_rows, a1);
    }
}

// ---------------------------------------------------------------------- join --------
__device__ __forceinline__ bool in_sorted(const int32_t *__restrict__ a, uint32_t n, int32_t x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        int32_t y = __ldg(a + mid);
        if (y < x) lo = mid + 1; else hi = mid;
    }
    return lo < n && __ldg(a + lo) == x;
}

// Set fingerprint of a final row m || x: h_j = fp_mix(Σ_q fp_term(seed_j, q, row[q])).
__device__ __forceinline__ void row_hash(const int32_t *__restrict__ row, uint32_t x, const StepParams &P,
                                         unsigned long long &h1, unsigned long long &h2) {
    unsigned long long a = 0, b = 0;
    for (int q = 0; q < P.k; q++) {
        const int col = P.pos_of_q[q];
        const uint32_t val = col < P.t ? (uint32_t)__ldg(row + col) : x;
        a += fp_term(kFpSeed1, q, val);
        b += fp_term(kFpSeed2, q, val);
    }
    h1 += fp_mix(a);
    h2 ^= fp_mix(b);
}

enum JoinMode { J_COUNT = 0, J_TABLE = 1, J_NEXT = 2, J_CAHEAD = 3 };
// Slots per thread: J_NEXT carries the next-step probe state of every slot in registers, so
// it runs 1024-slot tiles; the others 2048.
#ifndef GSI_NEXT_ITEMS
#define GSI_NEXT_ITEMS 8
#endif
#ifndef GSI_COUNT_ITEMS
#define GSI_COUNT_ITEMS 8
#endif
__host__ __device__ constexpr int join_items(int mode) {
    return mode == J_NEXT ? GSI_NEXT_ITEMS : (mode == J_COUNT ? GSI_COUNT_ITEMS : 8);
}

// Duplicate removal (Alg. 5) at warp scope: consecutive rows of M
// that hold the same vertex v in the probed column (siblings share their prefix columns, and
// rows stay in lexicographic order) need the same run N(v,l) ∩ C(u).  Only the first lane of
// each run of equal v probes PCSR; the others take its result by shuffle.  Every lane of
// the warp must call this (need = false for lanes without a row).
__device__ __forceinline__ Loc warp_dedup_lookup(bool need, int32_t v, const StepParams &P2,
                                                 const uint2 *__restrict__ groups, int gpn) {
    const int lane = threadIdx.x & 31;
    const int32_t pv = __shfl_up_sync(0xffffffffu, v, 1);
    const bool head = need && (lane == 0 || pv != v);
    Loc R{0u, 0u};
    if (head) {
        R = pcsr_lookup(groups, gpn, P2.gbase[0], P2.ngroups[0], P2.lab[0], (uint32_t)v, nullptr);
        if (P2.prefiltered && R.len) {
            const uint32_t a = __ldg(P2.fpos + (R.off - P2.flo)), b = __ldg(P2.fpos + (R.off + R.len - P2.flo));
            R = Loc{a, b - a};
        }
    }
    const unsigned heads = __ballot_sync(0xffffffffu, head);
    const unsigned upto = heads & (0xffffffffu >> (31 - lane));   // heads at lanes <= this one
    const int src = upto ? 31 - __clz(upto) : lane;
    R.off = __shfl_sync(0xffffffffu, R.off, src);
    R.len = __shfl_sync(0xffffffffu, R.len, src);
    if (!need) R = Loc{0u, 0u};
    return R;
}

// The NEXT step's list of every survivor (row, x) when that step has one linking edge:
// from the probe-ahead table aligned with this step's candidates (one coalesced 8 B read),
// else one PCSR probe per survivor (batches of 4 keep the first-sector loads in flight),
// re-pointed at the next step's shared N(v,l0) ∩ C(u) run when it has one.
template <int IT>
__device__ __forceinline__ void next_step_locs(const StepParams &P, const StepParams &P2, const int32_t *__restrict__ M,
                                               const uint32_t (&rows)[IT], const uint32_t (&xs)[IT],
                                               const uint32_t (&cio)[IT], const bool (&keep)[IT],
                                               const uint2 *__restrict__ groups, int gpn, Loc (&N0)[IT],
                                               const Loc *sNext = nullptr, long long rlo = 0) {
    if (sNext) {   // row-constant: staged per tile row
#pragma unroll
        for (int it = 0; it < IT; it++) N0[it] = keep[it] ? sNext[rows[it] - rlo] : Loc{0u, 0u};
        return;
    }
    if (P.pa) {
#pragma unroll
        for (int it = 0; it < IT; it++) N0[it] = keep[it] ? P.pa[cio[it]] : Loc{0u, 0u};
        return;
    }
    const int c2 = P2.col[0];
    uint32_t v[IT];
#pragma unroll
    for (int it = 0; it < IT; it++)
        v[it] = keep[it] ? (c2 < P.t ? (uint32_t)__ldg(M + (long long)rows[it] * P.t + c2) : xs[it]) : 0u;
#pragma unroll
    for (int h = 0; h < IT; h += 4) {
        uint32_t vb[4];
        bool kb[4];
        Loc nb[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            vb[q] = v[h + q];
            kb[q] = keep[h + q];
        }
        pcsr_lookup_batch<4>(groups, gpn, P2.gbase[0], P2.ngroups[0], P2.lab[0], vb, kb, nb);
#pragma unroll
        for (int q = 0; q < 4; q++) N0[h + q] = nb[q];
    }
    if (P2.prefiltered) {   // re-point at the shared N(v,l0) ∩ C(u) run of the next step
#pragma unroll
        for (int it = 0; it < IT; it++) {
            if (!keep[it] || !N0[it].len) continue;
            const uint32_t a = __ldg(P2.fpos + (N0[it].off - P2.flo));
            const uint32_t b = __ldg(P2.fpos + (N0[it].off + N0[it].len - P2.flo));
            N0[it] = Loc{a, b - a};
        }
    }
}

// rowmap[j] = the row holding slot s0 + j*tile (j < ntiles), rowmap[ntiles] = the row
// holding slot s1-1: the first/last row of every join tile, found by one thread per tile so
// that no CTA of the join waits on a dependent search of F.
__global__ void k_tile_rows(const unsigned long long *__restrict__ F, long long nM, unsigned long long s0,
                            unsigned long long s1, unsigned ntiles, unsigned tile, uint32_t *__restrict__ rowmap) {
    const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (j > ntiles) return;
    const unsigned long long s = j < ntiles ? s0 + (unsigned long long)j * tile : s1 - 1;
    long long lo = 0, hi = nM + 1;   // largest i with F[i] <= s
    while (hi - lo > 1) {
        const long long mid = (lo + hi) >> 1;
        if (__ldg(F + mid) <= s) lo = mid; else hi = mid;
    }
    rowmap[j] = (uint32_t)lo;
}

// The fused level kernel.  Slots [s0, s1) of the Prealloc space (GBA) of this level are cut
// into 2048-slot tiles.  Per slot: the candidate x = N(v', l0)[s - F_i] of row i is kept iff
// x in C(u) (bitset, L1150), x not in m_i (Alg. 3 line 10) and x in every other linking list
// (Alg. 3 line 13).  Survivors are compacted in slot order into shared memory (the write
// cache, L1155-1158), their output offset comes from a decoupled look-back (the Combine scan
// of Alg. 3 line 14), and the CTA writes its contiguous block of new rows m_i || x with
// coalesced stores (Alg. 3 lines 15-21).
//   J_COUNT : final level, count (+ fingerprint) only.
//   J_TABLE : final level, rows written in query-id order (+ fingerprint).
//   J_NEXT  : rows of M_{t+1}.  The NEXT step's Prealloc probe runs on every survivor before
//             the compaction, so a survivor with an empty next buffer (it can never be
//             extended) is counted but not stored, and the stored rows' loc / F (second
//             look-back chain) are written here: the next level never re-reads M_{t+1} to
//             size its buffers.
template <int MODE>
#ifndef GSI_NEXT_MINB
#define GSI_NEXT_MINB 4   // A/B r2p: 4 -> join_next 358 ms vs 393 (3) over the 16 fp bench queries
#endif
__global__ void __launch_bounds__(kThreads, join_items(MODE) > 8 ? 2 : (((MODE == J_NEXT && GSI_NEXT_ITEMS > 4) || MODE == J_CAHEAD) ? GSI_NEXT_MINB : 4)) k_join(const int32_t *__restrict__ M, long long nM,
                                                   const unsigned long long *__restrict__ F,
                                                   const Loc *__restrict__ loc, const uint32_t *__restrict__ rowmap,
                                                   StepParams P, StepParams P2, const int32_t *__restrict__ ci,
                                                   const uint32_t *__restrict__ cu_bitmap,
                                                   const uint2 *__restrict__ groups, int gpn,
                                                   unsigned long long s0, unsigned long long s1,
                                                   int32_t *__restrict__ out, Loc *__restrict__ loc2,
                                                   unsigned long long *__restrict__ F2,
                                                   unsigned long long *status, unsigned long long *status2,
                                                   unsigned *tile_ctr, Counters *ctr) {
    constexpr int IT = join_items(MODE);   // slots per thread
    constexpr int TILE = IT * kThreads;    // slots per CTA
    // Dynamic shared memory (join_smem_bytes<MODE>()): before the compaction it holds the row
    // marker / row offset per slot (sR), per tile row off0 - F_i (sBase) and the subtraction
    // columns (sInj); the write cache (sx, si, sloc) reuses the same bytes afterwards.
    extern __shared__ __align__(16) unsigned char dsm[];
    // staging region (before the compaction)     | write cache (after), same bytes
    //   sR[TILE] | sBase[TILE] | sInj[P.stage_inj][TILE] | sx[TILE] | si[TILE] | sloc[TILE] (J_NEXT)
    int *sR = reinterpret_cast<int *>(dsm);
    uint32_t *sBase = reinterpret_cast<uint32_t *>(sR + TILE);
    int32_t *sInjBase = reinterpret_cast<int32_t *>(sBase + TILE);
    Loc *sNext = reinterpret_cast<Loc *>(sInjBase + (size_t)P.stage_inj * TILE);   // [TILE / GSI_STAGE_DIV]
    uint32_t *sx = reinterpret_cast<uint32_t *>(dsm);
    uint32_t *si = sx + TILE;
    Loc *sloc = reinterpret_cast<Loc *>(si + TILE);
    __shared__ unsigned wcnt[IT][kThreads / 32];
    __shared__ unsigned wbase[IT][kThreads / 32];
    __shared__ unsigned long long sm[34];
    __shared__ unsigned tile_s, agg_s;
    __shared__ unsigned long long base_s, base2_s;
    __shared__ int s_src[GSI_MAX_K];   // J_NEXT: P.out_src (stored column map of a new row)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) tile_s = atomicAdd(tile_ctr, 1u);
    if (MODE == J_NEXT && tid < GSI_MAX_K) s_src[tid] = P.out_src[tid];
    {   // zero the row-marker array with 16 B stores
        int4 *z = reinterpret_cast<int4 *>(sR);
        for (int j = tid; j < TILE / 4; j += kThreads) z[j] = make_int4(0, 0, 0, 0);
    }
    __syncthreads();
    const unsigned tile = tile_s;
    const unsigned long long tbase = s0 + (unsigned long long)tile * TILE;
    const unsigned long long tend = min(tbase + (unsigned long long)TILE, s1);
    // (no rowmap: a single tile, which may scan every row of the level)
    const long long rlo = rowmap ? (long long)__ldg(rowmap + tile) : 0ll;
    const long long rhi = rowmap ? (long long)__ldg(rowmap + tile + 1) : nM - 1;
    const long long nr = rhi - rlo + 1;
    // Stage, per row of the tile, base = off0 - F_i (so slot s reads ci[base + s]) and the
    // columns the subtraction tests, so the per-slot work touches shared memory only.
    // Staging pays when rows are long (many slots per staged row); with short rows the per-row
    // loads would sit in the serial prologue, so those tiles read the row data per slot.
    const bool staged = P.stage_base && nr * GSI_STAGE_DIV <= TILE;
    const int n_inj_st = staged ? min(P.n_inj, P.stage_inj) : 0;
    // Row of every slot of the tile without a per-slot search (load-balanced search): each row
    // overlapping the tile marks its first tile-local slot, then an inclusive max-scan over the
    // 2048 slots spreads the row offset to all its slots.
    // two rows per thread per pass, phased so that both rows' dependent loads (F -> loc / row
    // columns -> PCSR sector -> fpos) are in flight together
    constexpr int RS = GSI_STAGE_ROWS;
    // (warp-uniform trip count: the staged next-step lookups are warp-collective)
    for (long long r0 = tid; r0 - tid < nr; r0 += RS * kThreads) {
        long long rr[RS];
        bool ok[RS];
        unsigned long long a[RS], b[RS];
#pragma unroll
        for (int q = 0; q < RS; q++) {
            rr[q] = r0 + q * kThreads;
            ok[q] = rr[q] < nr;
            a[q] = ok[q] ? __ldg(F + rlo + rr[q]) : 0ull;
            b[q] = ok[q] ? __ldg(F + rlo + rr[q] + 1) : 0ull;
        }
#pragma unroll
        for (int q = 0; q < RS; q++)
            if (ok[q] && a[q] < b[q] && b[q] > tbase && a[q] < tend)
                sR[a[q] > tbase ? (unsigned)(a[q] - tbase) : 0u] = (int)rr[q];
        if (staged) {
            uint32_t off[RS], vn[RS];
            bool kn[RS];
#pragma unroll
            for (int q = 0; q < RS; q++) {
                const unsigned long long i = (unsigned long long)(rlo + (ok[q] ? rr[q] : 0));
                const int32_t *row = M + i * (unsigned)P.t;
                off[q] = ok[q] ? loc[i * (unsigned)P.E].off : 0u;
                for (int c = 0; c < n_inj_st; c++)
                    if (ok[q]) sInjBase[c * TILE + rr[q]] = __ldg(row + P.inj_col[c]);
                kn[q] = MODE == J_NEXT && P.stage_next && ok[q] && a[q] < b[q];
                vn[q] = kn[q] ? (uint32_t)__ldg(row + P2.col[0]) : 0u;
            }
            if (MODE == J_NEXT && P.stage_next) {
#pragma unroll
                for (int q = 0; q < RS; q++) {
                    // consecutive tile rows sharing the probed vertex share one lookup (Alg. 5)
                    const Loc R = warp_dedup_lookup(kn[q], kn[q] ? (int32_t)vn[q] : -1, P2, groups, gpn);
                    if (ok[q]) sNext[rr[q]] = R;
                }
            }
#pragma unroll
            for (int q = 0; q < RS; q++)
                if (ok[q]) sBase[rr[q]] = off[q] - (uint32_t)a[q];
        }
    }
    __syncthreads();
    {
        int v[IT], m = 0;
#pragma unroll
        for (int q = 0; q < IT; q++) {
            v[q] = sR[tid * IT + q];
            m = max(m, v[q]);
            v[q] = m;
        }
        int inc = m;   // inclusive max-scan of thread maxima across the block
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) inc = max(inc, __shfl_up_sync(0xffffffffu, inc, o) * (lane >= o));
        if (lane == 31) wcnt[0][warp] = (unsigned)inc;
        int prev = __shfl_up_sync(0xffffffffu, inc, 1);
        __syncthreads();
        const int wm = lane < warp ? (int)wcnt[0][lane] : 0;   // max over the preceding warps
        int carry = max(lane == 0 ? 0 : prev, 0);
        int wmax = wm;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
        carry = max(carry, wmax);
#pragma unroll
        for (int q = 0; q < IT; q++) sR[tid * IT + q] = max(v[q], carry);
    }
    __syncthreads();

    // Phased over the 8 slots of this thread so that each phase's independent loads are in
    // flight together (ci -> C(u) bit -> subtraction -> other lists -> next probe).
    bool keep[IT];
    uint32_t xs[IT];
    uint32_t rows[IT];   // row offset from rlo
    uint32_t cio[IT];
    const uint32_t tlen = (uint32_t)(tend - tbase);   // slots in this tile (<= TILE)
    if (staged) {        // tile-uniform branch: 32-bit slot arithmetic against shared memory only
        const uint32_t tb32 = (uint32_t)tbase;
#pragma unroll
        for (int it = 0; it < IT; it++) {
            const uint32_t ls = (uint32_t)(it * kThreads + tid);
            keep[it] = ls < tlen;
            const int r = sR[ls];
            rows[it] = (uint32_t)r;
            cio[it] = sBase[r] + tb32 + ls;
        }
    } else {
#pragma unroll
        for (int it = 0; it < IT; it++) {
            const uint32_t ls = (uint32_t)(it * kThreads + tid);
            keep[it] = ls < tlen;
            const int r = sR[ls];
            rows[it] = (uint32_t)r;
            const unsigned long long i = (unsigned long long)(rlo + r);
            cio[it] = keep[it] ? loc[i * (unsigned)P.E].off + (uint32_t)(tbase + ls - __ldg(F + i)) : 0u;
        }
    }
#pragma unroll
    for (int it = 0; it < IT; it++) xs[it] = keep[it] ? (uint32_t)__ldg(ci + cio[it]) : 0u;
    if (!P.prefiltered) {
#pragma unroll
        for (int it = 0; it < IT; it++) {                                // x in C(u)
            const uint32_t x = xs[it];
            if (keep[it]) keep[it] = (__ldg(cu_bitmap + (x >> 5)) >> (x & 31)) & 1u;
        }
    }
    for (int c = 0; c < P.n_inj; c++) {                                         // Alg. 3 line 10
        const int col = P.inj_col[c];
        if (c < n_inj_st) {
#pragma unroll
            for (int it = 0; it < IT; it++)
                if (keep[it]) keep[it] = sInjBase[c * TILE + rows[it]] != (int32_t)xs[it];
        } else {
#pragma unroll
            for (int it = 0; it < IT; it++)
                if (keep[it])
                    keep[it] = __ldg(M + (unsigned long long)(rlo + rows[it]) * (unsigned)P.t + col) != (int32_t)xs[it];
        }
    }
#pragma unroll
    for (int it = 0; it < IT; it++) rows[it] += (uint32_t)rlo;              // absolute row index
    if (P.E > 1) {                                                               // Alg. 3 line 13
#pragma unroll
        for (int it = 0; it < IT; it++) {
            const Loc *L = loc + (unsigned long long)rows[it] * (unsigned)P.E;
            for (int e = 1; e < P.E && keep[it]; e++) {
                const Loc Le = L[e];
                keep[it] = in_sorted(ci + Le.off, Le.len, (int32_t)xs[it]);
            }
        }
    }

    if constexpr (MODE == J_COUNT) {
        unsigned long long c = 0, h1 = 0, h2 = 0;
#pragma unroll
        for (int it = 0; it < IT; it++) {
            if (!keep[it]) continue;
            c++;
            if (P.fp) row_hash(M + (long long)rows[it] * P.t, xs[it], P, h1, h2);
        }
        c = warp_sum_u64(c);
        if (lane == 0 && c) atomicAdd(&ctr->count, c);
        if (P.fp) {
            h1 = warp_sum_u64(h1);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) h2 ^= __shfl_xor_sync(0xffffffffu, h2, o);
            if (lane == 0 && c) {
                atomicAdd(&ctr->fp1, h1);
                atomicXor(&ctr->fp2, h2);
            }
        }
    } else if constexpr (MODE == J_CAHEAD) {
        // ---- count-ahead: this level's survivors are the rows of M_{k-1}; the last step has
        // one linking edge, so the extensions of row' = m_i || x are exactly
        // (N(v,l0) ∩ C(u_k)) \ row' (Alg. 3 lines 9-10): count |run| minus the row's own
        // vertices found in the run, without storing row' or enumerating the run.
        Loc N0[IT];
        next_step_locs<IT>(P, P2, M, rows, xs, cio, keep, groups, gpn, N0);
        unsigned long long surv = 0, c = 0, bound = 0;
#pragma unroll
        for (int it = 0; it < IT; it++) {
            if (!keep[it]) continue;
            surv++;
            const Loc R = N0[it];
            bound += R.len;
            uint32_t cc = R.len;
            for (int j = 0; j < P2.n_inj && cc; j++) {
                const int col = P2.inj_col[j];
                const int32_t y = col < P.t ? __ldg(M + (long long)rows[it] * P.t + col) : (int32_t)xs[it];
                if ((__ldg(P2.cu + ((uint32_t)y >> 5)) >> (y & 31)) & 1u)
                    cc -= in_sorted(P2.fci + R.off, R.len, y) ? 1u : 0u;
            }
            c += cc;
        }
        surv = warp_sum_u64(surv);
        c = warp_sum_u64(c);
        bound = warp_sum_u64(bound);
        if (lane == 0) {
            if (c) atomicAdd(&ctr->count, c);
            if (surv) atomicAdd(&ctr->total, surv);
            if (bound) atomicAdd(&ctr->total2, bound);
        }
    } else {
        // ---- J_NEXT: next-step probe of every survivor, dead rows dropped --------------------
        Loc N0[IT];
        if constexpr (MODE == J_NEXT) {
            unsigned long long all = 0;
#pragma unroll
            for (int it = 0; it < IT; it++) all += keep[it] ? 1 : 0;
            all = warp_sum_u64(all);
            if (lane == 0 && all) atomicAdd(&ctr->count, all);      // |M_{t+1}| including dead rows
            if (P2.E == 1) {
                next_step_locs<IT>(P, P2, M, rows, xs, cio, keep, groups, gpn, N0,
                                   (P.stage_next && staged) ? sNext : nullptr, rlo);
#pragma unroll
                for (int it = 0; it < IT; it++) keep[it] = keep[it] && N0[it].len > 0;
            } else {
#pragma unroll
                for (int it = 0; it < IT; it++) {
                    if (!keep[it]) continue;
                    unsigned long long l0, el;
                    probe_row_local(M + (long long)rows[it] * P.t, P.t, xs[it], P2, groups, gpn, nullptr, l0, el);
                    keep[it] = l0 > 0;
                    N0[it] = Loc{0u, (uint32_t)l0};
                }
            }
        }
        // ---- ordered compaction into the shared-memory write cache + look-back ------------
        // (the __syncthreads below also orders every read of sR / sBase / sInj before the
        //  write cache, which reuses those bytes, is written)
        unsigned ballots[IT];
#pragma unroll
        for (int it = 0; it < IT; it++) {
            ballots[it] = __ballot_sync(0xffffffffu, keep[it]);
            if (lane == 0) wcnt[it][warp] = __popc(ballots[it]);
        }
        if constexpr (MODE == J_NEXT) {
            // the tile's next-level buffer total is known before the compaction, so both
            // look-back chains (row offsets and next F) run at the same time (warps 0 and 1)
            unsigned long long mylen = 0;
#pragma unroll
            for (int it = 0; it < IT; it++) mylen += keep[it] ? N0[it].len : 0u;
            mylen = warp_sum_u64(mylen);
            if (lane == 0) sm[warp] = mylen;
        }
        __syncthreads();
        if (warp == 0) {
            constexpr int NW = kThreads / 32;   // IT * NW (it, warp) counts in slot order: it * NW + warp
            constexpr int PER = IT * NW / 32;   // entries per lane (1 or 2)
            unsigned e[PER], pair = 0;
#pragma unroll
            for (int q = 0; q < PER; q++) {
                const int idx = PER * lane + q;
                e[q] = wcnt[idx / NW][idx % NW];
                pair += e[q];
            }
            unsigned inc = pair;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            unsigned ex = inc - pair;
#pragma unroll
            for (int q = 0; q < PER; q++) {
                const int idx = PER * lane + q;
                wbase[idx / NW][idx % NW] = ex;
                ex += e[q];
            }
            const unsigned total = __shfl_sync(0xffffffffu, inc, 31);
            const unsigned long long pre = lookback_exclusive(status, tile, total);
            if (lane == 0) {
                base_s = pre;
                agg_s = total;
            }
        } else if (MODE == J_NEXT && warp == 1) {
            unsigned long long tl = lane < kThreads / 32 ? sm[lane] : 0ull;
            tl = warp_sum_u64(tl);
            if (P.no_f2) {
                if (lane == 0 && tl) atomicAdd(&ctr->total2, tl);
            } else {
                const unsigned long long pre2 = lookback_exclusive(status2, tile, tl);
                if (lane == 0) {
                    base2_s = pre2;
                    sm[32] = tl;
                }
            }
        }
        __syncthreads();
        const unsigned lt = (1u << lane) - 1u;
#pragma unroll
        for (int it = 0; it < IT; it++) {
            if (keep[it]) {
                const unsigned lp = wbase[it][warp] + __popc(ballots[it] & lt);
                sx[lp] = xs[it];
                si[lp] = rows[it];
                if constexpr (MODE == J_NEXT) sloc[lp] = N0[it];
            }
        }
        __syncthreads();
        const unsigned long long base = base_s;
        const unsigned cnt = agg_s;

        if constexpr (MODE == J_TABLE) {
            unsigned long long h1 = 0, h2 = 0;
            if (P.fp)
                for (unsigned j = tid; j < cnt; j += kThreads) row_hash(M + (long long)si[j] * P.t, sx[j], P, h1, h2);
            h1 = warp_sum_u64(h1);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) h2 ^= __shfl_xor_sync(0xffffffffu, h2, o);
            if (lane == 0 && (h1 | h2)) {
                atomicAdd(&ctr->fp1, h1);
                atomicXor(&ctr->fp2, h2);
            }
            const int k = P.k;
            int32_t *o = out + base * (unsigned long long)k;
            for (unsigned e = tid; e < cnt * (unsigned)k; e += kThreads) {
                const unsigned r = e / k, q = e - r * k;
                const int col = P.pos_of_q[q];
                o[e] = col < P.t ? __ldg(M + (long long)si[r] * P.t + col) : (int32_t)sx[r];
            }
            if (tile == gridDim.x - 1 && tid == 0) ctr->total = base + cnt;
        } else {
            // ---- next-level loc (E' = 1: from the write cache; else probe again) -----------
            unsigned long long elems = 0;
            if (P2.E == 1) {
                for (unsigned j = tid; j < cnt; j += kThreads) {
                    const Loc r = sloc[j];
                    loc2[base + j] = r;
                    elems += r.len;
                }
            } else {
                for (unsigned j = tid; j < cnt; j += kThreads) {
                    unsigned long long l0, el;
                    probe_row(M + (long long)si[j] * P.t, P.t, sx[j], P2, groups, gpn,
                              loc2 + (base + j) * (unsigned long long)P2.E, l0, el);
                    sloc[j] = Loc{0u, (uint32_t)l0};
                    elems += el;
                }
                __syncthreads();
            }
            elems = warp_sum_u64(elems);
            if (lane == 0 && elems) atomicAdd(&ctr->list_elems, elems);
            // next F over the tile's stored rows (thread tid owns rows [8 tid, 8 tid + 8));
            // the tile's offset base2_s came from the second look-back chain above
            if (!P.no_f2) {
                unsigned long long mine = 0;
#pragma unroll
                for (int q = 0; q < IT; q++) {
                    const unsigned j = tid * IT + q;
                    if (j < cnt) mine += sloc[j].len;
                }
                const unsigned long long agg2 = sm[32];
                const unsigned long long pre2 = base2_s;
                unsigned long long dummy;
                const unsigned long long ex2 = block_exclusive_scan(mine, sm, &dummy);
                unsigned long long run = pre2 + ex2;
#pragma unroll
                for (int q = 0; q < IT; q++) {
                    const unsigned j = tid * IT + q;
                    if (j < cnt) {
                        F2[base + j] = run;
                        run += sloc[j].len;
                    }
                }
                if (tile == gridDim.x - 1 && tid == 0) {
                    ctr->total2 = pre2 + agg2;
                    F2[base + cnt] = pre2 + agg2;
                }
            }
            // ---- coalesced write of the contiguous block of new rows ------------------------
            // (the column map comes from shared memory and e / W from a multiply-high: an
            // indexed parameter read per element serialised in the constant cache and a
            // division per element dominated this loop — ncu r2x: MIO throttle 23 %)
            const int W = P.out_w;
            const unsigned mW = 0xFFFFFFFFu / (unsigned)W + 1u;   // e / W exact for e < 2^32 / W
            int32_t *o = out + base * (unsigned long long)W;
            const int Pt = P.t;
            for (unsigned e = tid; e < cnt * (unsigned)W; e += kThreads) {
                const unsigned r = W == 1 ? e : __umulhi(e, mW), c = e - r * W;
                const int src = s_src[c];
                o[e] = src >= 0 ? __ldg(M + (long long)si[r] * Pt + src) : (int32_t)sx[r];
            }
            if (tile == gridDim.x - 1 && tid == 0) ctr->total = base + cnt;
        }
    }
}

// Lean count-only final level for the common case: one linking edge, rows on shared
// N(v,l0) ∩ C(u) runs (so every candidate already passed C(u)), no fingerprint.  Per slot the
// only work left is reading the candidate and testing the subtraction columns, so the tile
// is larger (CIT slots per thread) and the per-slot state is two registers.
template <int CIT>
__global__ void __launch_bounds__(kThreads, 4) k_count_fast(const int32_t *__restrict__ M, long long nM,
                                                            const unsigned long long *__restrict__ F,
                                                            const Loc *__restrict__ loc,
                                                            const uint32_t *__restrict__ rowmap, StepParams P,
                                                            const int32_t *__restrict__ fci, unsigned long long s0,
                                                            unsigned long long s1, Counters *ctr) {
    constexpr int TILE = CIT * kThreads;
    extern __shared__ __align__(16) unsigned char dsm[];
    int *sR = reinterpret_cast<int *>(dsm);                              // row offset per slot
    uint32_t *sBase = reinterpret_cast<uint32_t *>(sR + TILE);           // off0 - F_i per row
    int32_t *sInj = reinterpret_cast<int32_t *>(sBase + TILE);           // subtraction columns
    __shared__ unsigned wmax_s[kThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned tile = blockIdx.x;
    const unsigned long long tbase = s0 + (unsigned long long)tile * TILE;
    const unsigned long long tend = min(tbase + (unsigned long long)TILE, s1);
    {
        int4 *z = reinterpret_cast<int4 *>(sR);
        for (int j = tid; j < TILE / 4; j += kThreads) z[j] = make_int4(0, 0, 0, 0);
    }
    __syncthreads();
    // (no rowmap: a single tile, which may scan every row of the level)
    const long long rlo = rowmap ? (long long)__ldg(rowmap + tile) : 0ll;
    const long long rhi = rowmap ? (long long)__ldg(rowmap + tile + 1) : nM - 1;
    const long long nr = rhi - rlo + 1;
    const bool staged = nr <= TILE;
    const int ninj = P.n_inj, nst = staged ? min(ninj, P.stage_inj) : 0;
    for (long long r = tid; r < nr; r += kThreads) {
        const unsigned long long a = __ldg(F + rlo + r), b = __ldg(F + rlo + r + 1);
        if (a < b && b > tbase && a < tend) sR[a > tbase ? (unsigned)(a - tbase) : 0u] = (int)r;
        if (staged) {
            const unsigned long long i = (unsigned long long)(rlo + r);
            sBase[r] = loc[i].off - (uint32_t)a;
            const int32_t *row = M + i * (unsigned)P.t;
            for (int c = 0; c < nst; c++) sInj[c * TILE + r] = __ldg(row + P.inj_col[c]);
        }
    }
    __syncthreads();
    {   // inclusive max-scan of the row markers over the tile (thread owns CIT consecutive slots)
        int v[CIT], m = 0;
#pragma unroll
        for (int q = 0; q < CIT; q++) {
            v[q] = sR[tid * CIT + q];
            m = max(m, v[q]);
            v[q] = m;
        }
        int inc = m;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) inc = max(inc, __shfl_up_sync(0xffffffffu, inc, o) * (lane >= o));
        if (lane == 31) wmax_s[warp] = (unsigned)inc;
        int prev = __shfl_up_sync(0xffffffffu, inc, 1);
        __syncthreads();
        int wm = lane < warp ? (int)wmax_s[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) wm = max(wm, __shfl_xor_sync(0xffffffffu, wm, o));
        const int carry = max(lane == 0 ? 0 : prev, wm);
#pragma unroll
        for (int q = 0; q < CIT; q++) sR[tid * CIT + q] = max(v[q], carry);
    }
    __syncthreads();
    const uint32_t tlen = (uint32_t)(tend - tbase), tb32 = (uint32_t)tbase;
    int32_t xs[CIT];
    uint32_t cnt = 0;
    if (staged) {
#pragma unroll
        for (int it = 0; it < CIT; it++) {
            const uint32_t ls = (uint32_t)(it * kThreads + tid);
            xs[it] = ls < tlen ? __ldg(fci + (sBase[sR[ls]] + tb32 + ls)) : -1;
        }
        unsigned dead = 0;   // bit it: slot it failed (or is past the tile end)
#pragma unroll
        for (int it = 0; it < CIT; it++)
            if (xs[it] < 0) dead |= 1u << it;
        for (int c = 0; c < ninj; c++) {
            if (c < nst) {
#pragma unroll
                for (int it = 0; it < CIT; it++)
                    if (sInj[c * TILE + sR[it * kThreads + tid]] == xs[it]) dead |= 1u << it;
            } else {
#pragma unroll
                for (int it = 0; it < CIT; it++) {
                    const uint32_t ls = (uint32_t)(it * kThreads + tid);
                    const unsigned long long i = (unsigned long long)(rlo + sR[ls]);
                    if (!((dead >> it) & 1u) && __ldg(M + i * (unsigned)P.t + P.inj_col[c]) == xs[it]) dead |= 1u << it;
                }
            }
        }
        cnt = CIT - __popc(dead);
    } else {
#pragma unroll
        for (int it = 0; it < CIT; it++) {
            const uint32_t ls = (uint32_t)(it * kThreads + tid);
            if (ls >= tlen) continue;
            const unsigned long long i = (unsigned long long)(rlo + sR[ls]);
            const int32_t x = __ldg(fci + loc[i].off + (uint32_t)(tbase + ls - __ldg(F + i)));
            bool k = true;
            for (int c = 0; c < ninj && k; c++) k = __ldg(M + i * (unsigned)P.t + P.inj_col[c]) != x;
            cnt += k ? 1u : 0u;
        }
    }
    unsigned long long c64 = warp_sum_u64(cnt);
    if (lane == 0 && c64) atomicAdd(&ctr->count, c64);
}

// Count-ahead, warp-centric (rows on shared candidate runs, which are short): a warp takes 32
// consecutive rows, scans their buffer lengths with shuffles and walks the concatenated slots
// 32 at a time; the owner of slot j is the first lane whose inclusive length exceeds j (a
// 5-step shuffle search), and the owner's row data (run offset, subtraction columns, the last
// step's row-constant subtraction vertices) travel by shuffle.  No shared memory, no block
// barriers, no F reads: per row only loc and the needed columns, per slot the candidate,
// its probe-ahead entry and the tests.  Same arithmetic as k_join<J_CAHEAD>.
constexpr int kCaReg = 4;   // subtraction columns held in registers (more are read from M)
__device__ __forceinline__ bool in_bitmap(const uint32_t *__restrict__ bm, int32_t v) {
    return (__ldg(bm + ((uint32_t)v >> 5)) >> (v & 31)) & 1u;
}
__global__ void __launch_bounds__(kThreads, GSI_CAHEAD_MINB) k_cahead_warp(const int32_t *__restrict__ M, long long r0, long long r1,
                                                             const Loc *__restrict__ loc, StepParams P, StepParams P2,
                                                             const int32_t *__restrict__ cip,
                                                             const uint32_t *__restrict__ cu_bitmap,
                                                             const uint2 *__restrict__ groups, int gpn, Counters *ctr) {
    const int lane = threadIdx.x & 31;
    const long long gw = (blockIdx.x * (long long)kThreads + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * kThreads) >> 5;
    const unsigned E = (unsigned)P.E;
    const int ninj = P.n_inj, ninj2 = P2.n_inj;
    // The last step links to a column of the parent row (not to the vertex this step adds):
    // its run R and every row-column subtraction hit are constant per row, so a survivor x
    // only costs the test "x in R" (when x itself is a subtraction column of the last step).
    const bool rowR = P2.col[0] < P.t;
    bool xinj = false;
    for (int c = 0; c < ninj2; c++) xinj |= P2.inj_col[c] >= P.t;
    unsigned long long cnt = 0, surv = 0, bound = 0;
    for (long long base = r0 + gw * 32; base < r1; base += nw * 32) {
        const long long i = base + lane;
        const bool valid = i < r1;
        const Loc L = valid ? loc[(unsigned long long)i * E] : Loc{0u, 0u};
        const int32_t *row = M + (unsigned long long)(valid ? i : r0) * (unsigned)P.t;
        int32_t inj[kCaReg], y2[kCaReg];
#pragma unroll
        for (int c = 0; c < kCaReg; c++) inj[c] = (valid && c < ninj) ? __ldg(row + P.inj_col[c]) : -1;
        Loc RR{0u, 0u};
        uint32_t rbase = 0;
#pragma unroll
        for (int c = 0; c < kCaReg; c++) y2[c] = -1;
        if (rowR) {
            const bool need = valid && L.len;
            const int32_t v = need ? __ldg(row + P2.col[0]) : -1;
            RR = warp_dedup_lookup(need, v, P2, groups, gpn);
            if (need) {
                rbase = RR.len;
                for (int c = 0; c < ninj2 && rbase; c++) {
                    if (P2.inj_col[c] >= P.t) continue;
                    const int32_t y = __ldg(row + P2.inj_col[c]);
                    if (in_bitmap(P2.cu, y) && in_sorted(P2.fci + RR.off, RR.len, y)) rbase--;
                }
            }
        } else {
            // the last step's subtraction vertices that are columns of this row: their C(u_k)
            // bit is tested once here (-1: cannot be in any candidate run)
#pragma unroll
            for (int c = 0; c < kCaReg; c++) {
                if (valid && L.len && c < ninj2 && P2.inj_col[c] < P.t) {   // (a hole row holds no vertices)
                    const int32_t y = __ldg(row + P2.inj_col[c]);
                    if (in_bitmap(P2.cu, y)) y2[c] = y;
                }
            }
        }
        uint32_t inc = L.len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const uint32_t excl = inc - L.len;
        const uint32_t T = __shfl_sync(0xffffffffu, inc, 31);
        // two slots per lane per pass (j and j + 32): their owner searches, candidate and
        // probe-ahead loads are issued together
        constexpr int U = GSI_CAHEAD_U;
        for (uint32_t j0 = 0; j0 < T; j0 += 32 * U) {
            uint32_t jj[U], pos[U], roff[U], rlen[U], rb[U];
            int oo[U];
            int32_t ri[U][kCaReg], ry[U][kCaReg];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t j = j0 + 32 * u + lane;
                int o = 0;   // owner = number of lanes whose inclusive length is <= j
#pragma unroll
                for (int st = 16; st > 0; st >>= 1) {
                    const uint32_t v = __shfl_sync(0xffffffffu, inc, o + st - 1);
                    if (v <= j) o += st;
                }
                o &= 31;
                oo[u] = o;
                jj[u] = j;
                pos[u] = __shfl_sync(0xffffffffu, L.off, o) + (j - __shfl_sync(0xffffffffu, excl, o));
                // (warp-uniform branches: only the row data this step needs travels)
#pragma unroll
                for (int c = 0; c < kCaReg; c++) {
                    ri[u][c] = -1;
                    ry[u][c] = -1;
                    if (c < ninj) ri[u][c] = __shfl_sync(0xffffffffu, inj[c], o);
                    if (!rowR && c < ninj2) ry[u][c] = __shfl_sync(0xffffffffu, y2[c], o);
                }
                roff[u] = rlen[u] = rb[u] = 0u;
                if (rowR) {
                    rb[u] = __shfl_sync(0xffffffffu, rbase, o);
                    rlen[u] = __shfl_sync(0xffffffffu, RR.len, o);
                    if (xinj) roff[u] = __shfl_sync(0xffffffffu, RR.off, o);
                }
            }
            int32_t x[U];
            Loc R[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                x[u] = jj[u] < T ? __ldg(cip + pos[u]) : -1;
                R[u] = (!rowR && P.pa && jj[u] < T) ? P.pa[pos[u]] : Loc{0u, 0u};
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (jj[u] >= T) continue;
                const unsigned long long ri_row = (unsigned long long)(base + oo[u]);
                const int32_t xv = x[u];
                bool keep = true;
                if (!P.prefiltered) keep = in_bitmap(cu_bitmap, xv);
#pragma unroll
                for (int c = 0; c < kCaReg; c++) keep &= ri[u][c] != xv;
                for (int c = kCaReg; c < ninj && keep; c++) keep = __ldg(M + ri_row * (unsigned)P.t + P.inj_col[c]) != xv;
                for (unsigned e = 1; e < E && keep; e++) {
                    const Loc Le = loc[ri_row * E + e];
                    keep = in_sorted(cip + Le.off, Le.len, xv);
                }
                if (!keep) continue;
                surv++;
                if (rowR) {
                    bound += rlen[u];
                    uint32_t cc = rb[u];
                    if (xinj && cc && in_bitmap(P2.cu, xv) && in_sorted(P2.fci + roff[u], rlen[u], xv)) cc--;
                    cnt += cc;
                    continue;
                }
                Loc Rv = R[u];
                if (!P.pa) {
                    Rv = pcsr_lookup(groups, gpn, P2.gbase[0], P2.ngroups[0], P2.lab[0], (uint32_t)xv, nullptr);
                    if (Rv.len) {
                        const uint32_t fa = __ldg(P2.fpos + (Rv.off - P2.flo));
                        const uint32_t fb = __ldg(P2.fpos + (Rv.off + Rv.len - P2.flo));
                        Rv = Loc{fa, fb - fa};
                    }
                }
                bound += Rv.len;
                uint32_t cc = Rv.len;
#pragma unroll
                for (int c = 0; c < kCaReg; c++) {
                    if (c >= ninj2 || !cc) break;
                    if (ry[u][c] >= 0 && in_sorted(P2.fci + Rv.off, Rv.len, ry[u][c])) cc--;
                }
                for (int c = kCaReg; c < ninj2 && cc; c++) {
                    const int32_t y = __ldg(M + ri_row * (unsigned)P.t + P2.inj_col[c]);
                    if (in_bitmap(P2.cu, y) && in_sorted(P2.fci + Rv.off, Rv.len, y)) cc--;
                }
                cnt += cc;
            }
        }
    }
    cnt = warp_sum_u64(cnt);
    surv = warp_sum_u64(surv);
    bound = warp_sum_u64(bound);
    if (lane == 0) {
        if (cnt) atomicAdd(&ctr->count, cnt);
        if (surv) atomicAdd(&ctr->total, surv);
        if (bound) atomicAdd(&ctr->total2, bound);
    }
}

// The common count-ahead shape, lean and in closed form: the last step links to a parent
// column (its run RR and the row-column subtraction hits against it are per row, located with
// warp duplicate removal), the vertex this step adds is not a subtraction column of the last
// step, one linking edge on shared runs (every candidate of the row's run L is already in
// C(u)), at most NINJ (<= 1) subtraction columns in this step.  Then for row m of M_{k-2}:
//   survivors  s(m) = |L| - [inj(m) in L]                      (Alg. 3 lines 9-10)
//   extensions of each survivor m || x = rb(m) = |RR| - |{y in m : y in RR}|  (constant in x)
// so the row contributes s(m) * rb(m) matches with one binary search for inj in L and one per
// last-step subtraction column in RR — no walk over the candidates.
// FINAL: the same row formula as the last level of an enumerating count (count-ahead off):
// the row's matches are the candidates of L minus the subtraction hit, s(m).
// Up to N subtraction values of a row (Alg. 3 line 10: x must differ from the row's vertices
// with u's label that are not linked to x), held in registers; -1 never equals a vertex.
constexpr int kLeanInj = 4;
template <int N>
struct Inj {
    int32_t v[N > 0 ? N : 1];
    __device__ __forceinline__ void load(const int32_t *__restrict__ row, const StepParams &P, bool on) {
#pragma unroll
        for (int c = 0; c < N; c++) v[c] = (on && c < P.n_inj) ? __ldg(row + P.inj_col[c]) : -1;
    }
    __device__ __forceinline__ bool hit(int32_t x) const {
        bool h = false;
#pragma unroll
        for (int c = 0; c < N; c++) h |= x == v[c];
        return h;
    }
    __device__ __forceinline__ Inj shfl(int src) const {
        Inj r;
#pragma unroll
        for (int c = 0; c < N; c++) r.v[c] = __shfl_sync(0xffffffffu, v[c], src);
        return r;
    }
};

template <int NINJ, bool FINAL>
__global__ void __launch_bounds__(kThreads, 4) k_cahead_lean(const int32_t *__restrict__ M, long long r0, long long r1,
                                                             const Loc *__restrict__ loc, StepParams P, StepParams P2,
                                                             const int32_t *__restrict__ cip,
                                                             const uint2 *__restrict__ groups, int gpn, Counters *ctr) {
    const int lane = threadIdx.x & 31;
    const long long gw = (blockIdx.x * (long long)kThreads + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * kThreads) >> 5;
    const int ninj2 = P2.n_inj;
    unsigned long long cnt = 0, surv = 0, bound = 0, act = 0;
    for (long long base = r0 + gw * 32; base < r1; base += nw * 32) {
        const long long i = base + lane;
        const bool valid = i < r1;
        const Loc L = valid ? loc[(unsigned long long)i] : Loc{0u, 0u};
        const int32_t *row = M + (unsigned long long)(valid ? i : r0) * (unsigned)P.t;
        const bool need = valid && L.len;
        Loc RR{1u, 1u};   // FINAL: each surviving candidate is one match
        if (!FINAL) RR = warp_dedup_lookup(need, need ? __ldg(row + P2.col[0]) : -1, P2, groups, gpn);
        uint32_t rbase = RR.len;
        for (int c = 0; c < ninj2 && rbase && !FINAL; c++) {
            const int32_t y = __ldg(row + P2.inj_col[c]);
            if (in_bitmap(P2.cu, y) && in_sorted(P2.fci + RR.off, RR.len, y)) rbase--;
        }
        uint32_t sv = need ? L.len : 0u;
        if (NINJ > 0 && need) {   // FINAL: up to kLeanInj columns, else one
            const int ninj = FINAL ? P.n_inj : 1;
            for (int c = 0; c < ninj; c++)
                if (in_sorted(cip + L.off, L.len, __ldg(row + P.inj_col[c]))) sv--;
        }
        surv += sv;
        bound += (unsigned long long)sv * RR.len;
        cnt += (unsigned long long)sv * rbase;
        act += need ? 1u : 0u;
    }
    cnt = warp_sum_u64(cnt);
    surv = warp_sum_u64(surv);
    bound = warp_sum_u64(bound);
    act = warp_sum_u64(act);
    if (lane == 0) {
        if (cnt) atomicAdd(&ctr->count, cnt);
        if (surv) atomicAdd(&ctr->total, surv);
        if (bound) atomicAdd(&ctr->total2, bound);
        if (act) atomicAdd(&ctr->active_rows, act);
    }
}

// Fingerprinted last level on shared runs (the enumerating pass: every match is read and
// hashed).  Same shape as k_cahead_lean<FINAL>: one linking edge, rows on shared
// N(v,l0) ∩ C(u) runs, at most NINJ subtraction columns.  The set fingerprint of DESIGN.md
// §3 hashes a row as fp_mix(Σ_q fp_term(seed, q, row[q])), so the k-1 terms of the parent
// row are summed once per row (by the lane that owns it) and each match x of the row costs
// its candidate read, the subtraction compare and two terms + two finalisers.  The walk is
// load-balanced like the count kernels: lane-own rows when the unit's runs are even, long
// rows (>= 32 candidates) by the whole warp, the rest by a shuffle owner search.
#ifndef GSI_FP_EVEN
#define GSI_FP_EVEN 16   // k_final_fp: lane-own rows when 32 rows' total >= GSI_FP_EVEN x the longest
#endif
#ifndef GSI_FP_MINB
#define GSI_FP_MINB 4    // k_final_fp: resident CTAs per SM the registers are sized for
#endif
template <int NINJ, bool TT>   // TT: x's terms from the per-candidate term table T (else computed)
__global__ void __launch_bounds__(kThreads, GSI_FP_MINB) k_final_fp(const int32_t *__restrict__ M, long long r0, long long r1,
                                                          const Loc *__restrict__ loc, StepParams P, int qx,
                                                          const int32_t *__restrict__ cip,
                                                          const ulonglong2 *__restrict__ T, Counters *ctr) {
    const int lane = threadIdx.x & 31;
    const long long gw = (blockIdx.x * (long long)kThreads + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * kThreads) >> 5;
    // cnt: the rows' run lengths minus the subtraction hits (counted per row, not per match)
    unsigned long long cnt = 0, h1 = 0, h2 = 0, act = 0;
    // one match m || x, x = cip[p]: the subtraction test, then the two row hashes from the
    // parent's summed terms (a1, a2) and x's terms (from T, or computed) — straight-line code
    // per match: the term-table choice is a template parameter, not a branch per match
    auto fp_match = [&](uint32_t p, const Inj<NINJ> &in, unsigned long long a1, unsigned long long a2) {
        unsigned long long t1, t2;
        if (TT) {
            if (NINJ > 0 && in.hit(__ldg(cip + p))) {
                cnt--;
                return;
            }
            const ulonglong2 tt = __ldg(T + p);
            t1 = tt.x;
            t2 = tt.y;
        } else {
            const int32_t x = __ldg(cip + p);
            if (NINJ > 0 && in.hit(x)) {
                cnt--;
                return;
            }
            t1 = fp_term(kFpSeed1, qx, (uint32_t)x);
            t2 = fp_term(kFpSeed2, qx, (uint32_t)x);
        }
        h1 += fp_mix_pre(a1 + t1);   // a1, a2 carry fp_mix's leading constant (added per row)
        h2 ^= fp_mix_pre(a2 + t2);
    };
    for (long long base = r0 + gw * 32; base < r1; base += nw * 32) {
        const long long i = base + lane;
        const bool valid = i < r1;
        const Loc L = valid ? loc[(unsigned long long)i] : Loc{0u, 0u};
        const int32_t *row = M + (unsigned long long)(valid ? i : r0) * (unsigned)P.t;
        Inj<NINJ> inj;
        inj.load(row, P, valid && L.len);
        act += (valid && L.len) ? 1u : 0u;
        cnt += valid ? L.len : 0u;
        unsigned long long s1 = kFpMixAdd, s2 = kFpMixAdd;   // the parent row's terms (every column but x)
        if (valid && L.len) {
            for (int q = 0; q < P.k; q++) {
                const int col = P.pos_of_q[q];
                if (col >= P.t) continue;
                const uint32_t v = (uint32_t)__ldg(row + col);
                s1 += fp_term(kFpSeed1, q, v);
                s2 += fp_term(kFpSeed2, q, v);
            }
        }
        uint32_t inc = L.len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const uint32_t T = __shfl_sync(0xffffffffu, inc, 31);
        const uint32_t maxlen = __reduce_max_sync(0xffffffffu, L.len);
        if (maxlen * GSI_FP_EVEN <= T) {   // even runs: every lane walks its own row
            for (uint32_t kk = 0; kk < L.len; kk++) fp_match(L.off + kk, inj, s1, s2);
            continue;
        }
        uint32_t longs = __ballot_sync(0xffffffffu, L.len >= 32);
        while (longs) {   // long rows: the whole warp, one row at a time
            const int r = __ffs(longs) - 1;
            longs &= longs - 1;
            const uint32_t off = __shfl_sync(0xffffffffu, L.off, r), len = __shfl_sync(0xffffffffu, L.len, r);
            const unsigned long long a1 = __shfl_sync(0xffffffffu, s1, r), a2 = __shfl_sync(0xffffffffu, s2, r);
            const Inj<NINJ> ri = inj.shfl(r);
            for (uint32_t kk = lane; kk < len; kk += 32) fp_match(off + kk, ri, a1, a2);
        }
        const uint32_t sl = L.len >= 32 ? 0u : L.len;   // the short rows: balanced walk
        inc = sl;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const uint32_t excl = inc - sl;
        const uint32_t T2 = __shfl_sync(0xffffffffu, inc, 31);
        for (uint32_t j0 = 0; j0 < T2; j0 += 32) {
            const uint32_t j = j0 + lane;
            int o = 0;   // owner = number of lanes whose inclusive length is <= j
#pragma unroll
            for (int st = 16; st > 0; st >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, inc, o + st - 1);
                if (v <= j) o += st;
            }
            o &= 31;
            const uint32_t pos = __shfl_sync(0xffffffffu, L.off, o) + (j - __shfl_sync(0xffffffffu, excl, o));
            const unsigned long long a1 = __shfl_sync(0xffffffffu, s1, o), a2 = __shfl_sync(0xffffffffu, s2, o);
            const Inj<NINJ> ri = inj.shfl(o);
            if (j >= T2) continue;
            fp_match(pos, ri, a1, a2);
        }
    }
    cnt = warp_sum_u64(cnt);
    act = warp_sum_u64(act);
    h1 = warp_sum_u64(h1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h2 ^= __shfl_xor_sync(0xffffffffu, h2, o);
    if (lane == 0 && cnt) {
        atomicAdd(&ctr->count, cnt);
        atomicAdd(&ctr->fp1, h1);
        atomicXor(&ctr->fp2, h2);
    }
    if (lane == 0 && act) atomicAdd(&ctr->active_rows, act);
}

// Table-mode last level on shared runs (one linking edge, at most NINJ <= 1 subtraction
// columns), pass 1: the Combine offsets of Alg. 3 line 14 in closed form per row.  Row i keeps
// s_i = |L_i| - [inj_i in L_i] matches (lines 9-10; C(u) is already applied to the shared run),
// O = exclusive scan of s over rows [r0, r0 + nrows) (decoupled look-back), O[nrows] = total.
template <int NINJ>
__global__ void __launch_bounds__(kThreads) k_surv_scan(const int32_t *__restrict__ M, long long r0, long long nrows,
                                                        const Loc *__restrict__ loc, StepParams P,
                                                        const int32_t *__restrict__ cip,
                                                        unsigned long long *__restrict__ O,
                                                        unsigned long long *status, unsigned *tile_ctr) {
    __shared__ unsigned long long sm[33];
    __shared__ unsigned tile_s;
    __shared__ unsigned long long base_s;
    if (threadIdx.x == 0) tile_s = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const unsigned tile = tile_s;
    const long long i = (long long)tile * kThreads + threadIdx.x;
    unsigned long long s = 0;
    if (i < nrows) {
        const Loc L = loc[(unsigned long long)(r0 + i)];
        s = L.len;
        if (NINJ > 0 && L.len) {
            const int32_t *row = M + (unsigned long long)(r0 + i) * (unsigned)P.t;
            for (int c = 0; c < P.n_inj; c++)
                if (in_sorted(cip + L.off, L.len, __ldg(row + P.inj_col[c]))) s--;
        }
    }
    unsigned long long agg;
    const unsigned long long ex = block_exclusive_scan(s, sm, &agg);
    if (threadIdx.x < 32) {
        const unsigned long long pre = lookback_exclusive(status, tile, agg);
        if (threadIdx.x == 0) base_s = pre;
    }
    __syncthreads();
    if (i < nrows) O[i] = base_s + ex;
    if (tile == gridDim.x - 1 && threadIdx.x == kThreads - 1) O[nrows] = base_s + agg;
}

// Table-mode last level on shared runs, pass 2: every match m_i || x written as a k-int32 row
// in query-id order at out[O_i + j] (the final M of Alg. 3 lines 15-21; the paper's output,
// 4k B per match).  A warp takes 32 consecutive rows and walks their concatenated candidates 32
// at a time (owner by shuffle search); the survivors of a batch are contiguous in the output, so
// they are compacted by ballot into a shared-memory staging tile (the write cache, L1155-1158)
// and the warp stores the batch's 32·k ints as one coalesced stream.  HBM-write-bound.
constexpr int kTabMaxK = 16;   // staging width; wider queries take the generic tile kernel
template <int NINJ, bool FP>
__global__ void __launch_bounds__(kThreads, 4) k_final_table(const int32_t *__restrict__ M, long long r0, long long r1,
                                                             const Loc *__restrict__ loc,
                                                             const unsigned long long *__restrict__ O, StepParams P,
                                                             const int32_t *__restrict__ cip,
                                                             int32_t *__restrict__ out, Counters *ctr) {
    // per warp: the unit's 32 parent rows in query-id column order (x's column unused), and
    // the batch's survivors (x, owner lane) after ballot compaction
    __shared__ __align__(16) int32_t prow_s[kThreads / 32][32 * kTabMaxK];
    __shared__ int32_t sx_s[kThreads / 32][32];
    __shared__ int32_t so_s[kThreads / 32][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int32_t *prow = prow_s[wib], *sx = sx_s[wib], *so = so_s[wib];
    const long long gw = (blockIdx.x * (long long)kThreads + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * kThreads) >> 5;
    const int k = P.k;
    int qx = 0;   // the query vertex this level adds (its column is x)
    for (int q = 0; q < k; q++)
        if (P.pos_of_q[q] >= P.t) qx = q;
    const unsigned inv_k = (65536u + (unsigned)k - 1u) / (unsigned)k;   // e / k = (e * inv_k) >> 16, e < 32k
    const unsigned lt = (1u << lane) - 1u;
    unsigned long long h1 = 0, h2 = 0;   // FP: the set fingerprint of the written rows
    for (long long base = r0 + gw * 32; base < r1; base += nw * 32) {
        const long long i = base + lane;
        const bool valid = i < r1;
        const Loc L = valid ? loc[(unsigned long long)i] : Loc{0u, 0u};
        const int32_t *row = M + (unsigned long long)(valid ? i : r0) * (unsigned)P.t;
        Inj<NINJ> inj;
        inj.load(row, P, valid && L.len);
        unsigned long long s1 = kFpMixAdd, s2 = kFpMixAdd;
        if (valid && L.len)
            for (int q = 0; q < k; q++) {
                const int col = P.pos_of_q[q];
                if (col >= P.t) continue;
                const int32_t v = __ldg(row + col);
                prow[lane * k + q] = v;
                if (FP) {
                    s1 += fp_term(kFpSeed1, q, (uint32_t)v);
                    s2 += fp_term(kFpSeed2, q, (uint32_t)v);
                }
            }
        unsigned long long ob = __shfl_sync(0xffffffffu, valid ? O[i - r0] : 0ull, 0);   // the unit's first output row
        uint32_t inc = L.len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const uint32_t excl = inc - L.len;
        const uint32_t T = __shfl_sync(0xffffffffu, inc, 31);
        __syncwarp();
        for (uint32_t j0 = 0; j0 < T; j0 += 32) {
            const uint32_t j = j0 + lane;
            int o = 0;
#pragma unroll
            for (int st = 16; st > 0; st >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, inc, o + st - 1);
                if (v <= j) o += st;
            }
            o &= 31;
            const uint32_t pos = __shfl_sync(0xffffffffu, L.off, o) + (j - __shfl_sync(0xffffffffu, excl, o));
            const Inj<NINJ> ri = inj.shfl(o);
            unsigned long long a1 = 0, a2 = 0;
            if (FP) {
                a1 = __shfl_sync(0xffffffffu, s1, o);
                a2 = __shfl_sync(0xffffffffu, s2, o);
            }
            int32_t x = -1;
            bool keep = j < T;
            if (keep) {
                x = __ldg(cip + pos);
                if (NINJ > 0) keep = !ri.hit(x);
            }
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const unsigned lp = __popc(bal & lt);
                sx[lp] = x;
                so[lp] = o;
                if (FP) {
                    h1 += fp_mix_pre(a1 + fp_term(kFpSeed1, qx, (uint32_t)x));
                    h2 ^= fp_mix_pre(a2 + fp_term(kFpSeed2, qx, (uint32_t)x));
                }
            }
            __syncwarp();
            int32_t *dst = out + ob * (unsigned long long)k;
            if ((k & 3) == 0) {   // rows of 16 B multiples: one 16 B store per 4 columns
                const unsigned k4 = (unsigned)k >> 2, inv_k4 = (65536u + k4 - 1u) / k4;
                const unsigned nf = (unsigned)__popc(bal) * k4;
                int4 *dst4 = reinterpret_cast<int4 *>(dst);
                for (unsigned f = lane; f < nf; f += 32) {
                    const unsigned r = (f * inv_k4) >> 16, q0 = (f - r * k4) * 4u;
                    int4 v = *reinterpret_cast<const int4 *>(prow + so[r] * k + q0);
                    const int d = qx - (int)q0;
                    if (d == 0) v.x = sx[r];
                    else if (d == 1) v.y = sx[r];
                    else if (d == 2) v.z = sx[r];
                    else if (d == 3) v.w = sx[r];
                    __stcs(dst4 + f, v);
                }
            } else {
                const unsigned nk = (unsigned)__popc(bal) * (unsigned)k;
                for (unsigned e = lane; e < nk; e += 32) {
                    const unsigned r = (e * inv_k) >> 16, q = e - r * (unsigned)k;
                    __stcs(dst + e, (int)q == qx ? sx[r] : prow[so[r] * k + q]);
                }
            }
            __syncwarp();
            ob += __popc(bal);
        }
        __syncwarp();   // prow is rewritten by the next unit
    }
    if (FP) {
        h1 = warp_sum_u64(h1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) h2 ^= __shfl_xor_sync(0xffffffffu, h2, o);
        if (lane == 0 && (h1 | h2)) {
            atomicAdd(&ctr->fp1, h1);
            atomicXor(&ctr->fp2, h2);
        }
    }
}

// Lean J_NEXT (count-only mode, one linking edge on shared runs in this step and the next):
// warp-centric like k_cahead_lean, and the new rows go straight to their Prealloc slots —
// row i's buffer is GBA[F_i, F_i + |N(v,l0)|) (Alg. 4), so candidate j of row i
// writes row m_i || x at slot F_i + j with no scan, and a slot whose candidate fails leaves a
// hole: its loc entry is {0, 0}, i.e. a row with an empty next buffer that the next level
// skips like any other.  The Combine compaction (Alg. 3 lines 14-21) is dropped: count-only
// levels tolerate holes, and rows stay in lexicographic order.  Slots [c0, c1) of the level
// (a chunk may cut a row); rowmap[0..1] = the rows holding slots c0 and c1 - 1.
template <int NINJ>
__global__ void __launch_bounds__(kThreads, 4) k_next_lean(const int32_t *__restrict__ M, const uint32_t *__restrict__ rowmap,
                                                           const Loc *__restrict__ loc,
                                                           const unsigned long long *__restrict__ F,
                                                           unsigned long long c0, unsigned long long c1, StepParams P,
                                                           StepParams P2, const int32_t *__restrict__ cip,
                                                           const uint32_t *__restrict__ cu_bitmap,
                                                           const uint2 *__restrict__ groups, int gpn,
                                                           int32_t *__restrict__ out, Loc *__restrict__ loc2,
                                                           Counters *ctr) {
    const int lane = threadIdx.x & 31;
    const long long gw = (blockIdx.x * (long long)kThreads + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * kThreads) >> 5;
    const long long r0 = rowmap[0], r1 = (long long)rowmap[1] + 1;
    const int W = P.out_w;
    const bool rowN = P2.col[0] < P.t;   // the next step's run is per row
#if GSI_NEXT_STAGE
    // the 32 slots of a batch are 32 consecutive Prealloc slots: their rows are staged here
    // and stored as one coalesced run (write cache); hole rows are masked out
    __shared__ int32_t nstage[kThreads / 32][32 * GSI_MAX_K];
    int32_t *sw = nstage[threadIdx.x >> 5];
    const unsigned invW = (65536u + (unsigned)max(W, 1) - 1u) / (unsigned)max(W, 1);   // e / W, e < 32 W
#endif
    unsigned long long surv = 0, kept = 0, nlen = 0;
    for (long long base = r0 + gw * 32; base < r1; base += nw * 32) {
        const long long i = base + lane;
        const bool valid = i < r1;
        Loc L = valid ? loc[(unsigned long long)i] : Loc{0u, 0u};
        unsigned long long a = valid ? F[i] : 0ull;   // first slot of the row (clipped to the chunk)
        if (valid) {
            const unsigned long long b = min(a + L.len, c1);
            const unsigned long long a2 = max(a, c0);
            L.off += (uint32_t)(a2 - a);
            L.len = b > a2 ? (uint32_t)(b - a2) : 0u;
            a = a2;
        }
        const int32_t *row = M + (unsigned long long)(valid ? i : r0) * (unsigned)P.t;
        const int32_t inj = (NINJ > 0 && valid) ? __ldg(row + P.inj_col[0]) : -1;
        Loc RN{0u, 0u};
        if (rowN) {
            const bool need = valid && L.len;
            RN = warp_dedup_lookup(need, need ? __ldg(row + P2.col[0]) : -1, P2, groups, gpn);
        }
        uint32_t inc = L.len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const uint32_t excl = inc - L.len;
        const uint32_t T = __shfl_sync(0xffffffffu, inc, 31);
        for (uint32_t j0 = 0; j0 < T; j0 += 32) {
            const uint32_t j = j0 + lane;
            int o = 0;
#pragma unroll
            for (int st = 16; st > 0; st >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, inc, o + st - 1);
                if (v <= j) o += st;
            }
            o &= 31;
            const uint32_t k = j - __shfl_sync(0xffffffffu, excl, o);
            const uint32_t pos = __shfl_sync(0xffffffffu, L.off, o) + k;
            const unsigned long long slot = __shfl_sync(0xffffffffu, a, o) + k;
            const int32_t ri = NINJ > 0 ? __shfl_sync(0xffffffffu, inj, o) : -1;
            Loc N0;
            N0.off = rowN ? __shfl_sync(0xffffffffu, RN.off, o) : 0u;
            N0.len = rowN ? __shfl_sync(0xffffffffu, RN.len, o) : 0u;
#if GSI_NEXT_STAGE
            const bool act = j < T;
#else
            if (j >= T) continue;
            const bool act = true;
#endif
            const unsigned long long ro = (unsigned long long)(base + o);
            const int32_t x = act ? __ldg(cip + pos) : -1;
            bool keep = act && (P.prefiltered || in_bitmap(cu_bitmap, x));
            if (NINJ > 0) keep &= x != ri;
            if (keep) {
                surv++;
                if (!rowN) {
                    if (P.pa) {
                        N0 = P.pa[pos];
                    } else {
                        N0 = pcsr_lookup(groups, gpn, P2.gbase[0], P2.ngroups[0], P2.lab[0], (uint32_t)x, nullptr);
                        if (N0.len) {
                            const uint32_t fa = __ldg(P2.fpos + (N0.off - P2.flo));
                            const uint32_t fb = __ldg(P2.fpos + (N0.off + N0.len - P2.flo));
                            N0 = Loc{fa, fb - fa};
                        }
                    }
                }
                keep = N0.len > 0;   // a row with an empty next buffer is counted, never stored
            }
            const unsigned long long lo = slot - c0;
            if (act) loc2[lo] = keep ? N0 : Loc{0u, 0u};
#if GSI_NEXT_STAGE
            if (keep) {
                kept++;
                nlen += N0.len;
                for (int c = 0; c < W; c++) {
                    const int src = P.out_src[c];
                    sw[lane * W + c] = src >= 0 ? __ldg(M + ro * (unsigned)P.t + src) : x;
                }
            }
            const unsigned km = __ballot_sync(0xffffffffu, keep);
            __syncwarp();
            if (km) {
                const unsigned long long lo0 = __shfl_sync(0xffffffffu, lo, 0);   // lane 0 is always active
                int32_t *dst = out + lo0 * (unsigned)W;
                const unsigned nb = min(32u, T - j0), nr = nb * (unsigned)W;
                if (km == (nb == 32u ? 0xFFFFFFFFu : (1u << nb) - 1u)) {   // every row kept: a plain copy
                    for (unsigned e = lane; e < nr; e += 32) dst[e] = sw[e];
                } else {
                    for (unsigned e = lane; e < nr; e += 32)
                        if ((km >> ((e * invW) >> 16)) & 1u) dst[e] = sw[e];
                }
            }
            __syncwarp();
#else
            if (keep) {
                kept++;
                nlen += N0.len;
                int32_t *orow = out + lo * (unsigned)W;
                for (int c = 0; c < W; c++) {
                    const int src = P.out_src[c];
                    orow[c] = src >= 0 ? __ldg(M + ro * (unsigned)P.t + src) : x;
                }
            }
#endif
        }
    }
    surv = warp_sum_u64(surv);
    kept = warp_sum_u64(kept);
    nlen = warp_sum_u64(nlen);
    if (lane == 0) {
        if (surv) atomicAdd(&ctr->count, surv);
        if (kept) atomicAdd(&ctr->active_rows, kept);
        if (nlen) {
            atomicAdd(&ctr->total2, nlen);
            atomicAdd(&ctr->list_elems, nlen);
        }
    }
}

constexpr int kFastItems = GSI_FAST_ITEMS > 0 ? GSI_FAST_ITEMS : 8;

// Dynamic shared memory of a join launch: the larger of the staging region (row markers,
// optional ci bases and subtraction columns) and the write cache.  Kept to what the step
// uses: the rest of the 228 KB SM memory stays L1 cache for the ci / bitmap / row reads.
inline size_t join_smem_bytes(int mode, const StepParams &P) {
    const size_t tile = (size_t)join_items(mode) * kThreads;
    const size_t staging = tile * 4 * (1 + (P.stage_base ? 1 : 0) + (size_t)P.stage_inj) +
                           (P.stage_next ? tile / GSI_STAGE_DIV * sizeof(Loc) : 0);
    const size_t cache = (mode == J_COUNT || mode == J_CAHEAD) ? 0 : tile * 4 * 2 + (mode == J_NEXT ? tile * 8 : 0);
    return std::max(staging, cache);
}
constexpr int kMaxJoinSmem = 6 * 4096 * 4;

// ------------------------------------------------------- shared candidate lists -----
// Duplicate removal (§VI-B, Alg. 5) taken one step further for B200: at a
// level whose rows re-scan the same neighbour lists many times (|GBA| >> |ci of P(G,l0)|),
// N(v,l0) ∩ C(u) is computed ONCE per partition run (one pass over P(G,l0)'s ci) and the
// rows then enumerate only those candidates.  fpos[o - lo] = number of kept entries of the
// partition before offset o, fci = the kept entries in ci order (runs stay sorted).
__global__ void __launch_bounds__(kThreads) k_filter_partition(const int32_t *__restrict__ ci, uint32_t lo,
                                                               uint32_t hi, const uint32_t *__restrict__ cu_bitmap,
                                                               uint32_t *__restrict__ fpos,
                                                               int32_t *__restrict__ fci,
                                                               unsigned long long *status, unsigned *tile_ctr) {
    constexpr int IT = GSI_FP_ITEMS, TILE = IT * kThreads;
    __shared__ unsigned wcnt[IT][kThreads / 32];
    __shared__ unsigned wbase[IT][kThreads / 32];
    __shared__ unsigned tile_s, agg_s;
    __shared__ unsigned long long base_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) tile_s = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const unsigned tile = tile_s;
    const uint32_t tb = lo + tile * (uint32_t)TILE;
    bool keep[IT];
    int32_t xs[IT];
    unsigned ballots[IT];
#pragma unroll
    for (int it = 0; it < IT; it++) {
        const uint32_t o = tb + it * kThreads + tid;
        keep[it] = o < hi;
        xs[it] = keep[it] ? __ldg(ci + o) : 0;
    }
#pragma unroll
    for (int it = 0; it < IT; it++)
        if (keep[it]) keep[it] = (__ldg(cu_bitmap + ((uint32_t)xs[it] >> 5)) >> (xs[it] & 31)) & 1u;
#pragma unroll
    for (int it = 0; it < IT; it++) {
        ballots[it] = __ballot_sync(0xffffffffu, keep[it]);
        if (lane == 0) wcnt[it][warp] = __popc(ballots[it]);
    }
    __syncthreads();
    if (warp == 0) {
        constexpr int NW = kThreads / 32, PER = IT * NW / 32;
        unsigned e[PER], pair = 0;
#pragma unroll
        for (int q = 0; q < PER; q++) {
            const int idx = PER * lane + q;
            e[q] = wcnt[idx / NW][idx % NW];
            pair += e[q];
        }
        unsigned inc = pair;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        unsigned ex = inc - pair;
#pragma unroll
        for (int q = 0; q < PER; q++) {
            const int idx = PER * lane + q;
            wbase[idx / NW][idx % NW] = ex;
            ex += e[q];
        }
        const unsigned total = __shfl_sync(0xffffffffu, inc, 31);
        const unsigned long long pre = lookback_exclusive(status, tile, total);
        if (lane == 0) {
            base_s = pre;
            agg_s = total;
        }
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int it = 0; it < IT; it++) {
        const uint32_t o = tb + it * kThreads + tid;
        const uint32_t pos = (uint32_t)base_s + wbase[it][warp] + __popc(ballots[it] & lt);
        if (o < hi) fpos[o - lo] = pos;
        if (keep[it]) fci[pos] = xs[it];
    }
    if (tile == gridDim.x - 1 && tid == 0) fpos[hi - lo] = (uint32_t)(base_s + agg_s);
}

// Probe-ahead table of a step on shared lists whose NEXT step has one linking edge, to the
// vertex this step adds: pa[p] = the next step's N(x,l0') ∩ C(u') run of x = fci[p].  Rows of
// a level re-scan the same candidate runs many times (that is why the runs are shared), so
// one PCSR probe per candidate replaces one per new row, and the join reads pa[p] coalesced
// next to fci[p].
__global__ void __launch_bounds__(kThreads) k_probe_ahead(const int32_t *__restrict__ fci,
                                                          const uint32_t *__restrict__ ntotal, StepParams P2,
                                                          const uint2 *__restrict__ groups, int gpn,
                                                          Loc *__restrict__ pa) {
    const uint32_t total = *ntotal;
    const uint32_t stride = gridDim.x * kThreads;
    for (uint32_t p0 = blockIdx.x * kThreads + threadIdx.x; p0 < total; p0 += 4 * stride) {
        uint32_t v[4];
        bool kb[4];
        Loc nb[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const uint32_t p = p0 + q * stride;
            kb[q] = p < total;
            v[q] = kb[q] ? (uint32_t)__ldg(fci + p) : 0u;
        }
        pcsr_lookup_batch<4>(groups, gpn, P2.gbase[0], P2.ngroups[0], P2.lab[0], v, kb, nb);
#pragma unroll
        for (int q = 0; q < 4; q++) {
            if (!kb[q]) continue;
            Loc r = nb[q];
            if (r.len) {
                const uint32_t a = __ldg(P2.fpos + (r.off - P2.flo)), b = __ldg(P2.fpos + (r.off + r.len - P2.flo));
                r = Loc{a, b - a};
            }
            pa[p0 + q * stride] = r;
        }
    }
}

// Fingerprint terms of every candidate of a shared run array (the last step's x = fci[p]):
// T[p] = (fp_term(seed1, q, x), fp_term(seed2, q, x)), q = the query vertex the step adds.
// The enumerating last level then reads 16 B per match (L2-resident: the shared runs are
// re-read by many rows) instead of computing two splitmix finalisers per match (DESIGN.md §3
// 'Fingerprint': a keyed term per column).
__global__ void __launch_bounds__(kThreads) k_fp_terms(const int32_t *__restrict__ fci, const uint32_t *__restrict__ ntotal,
                                                       int q, ulonglong2 *__restrict__ T) {
    const uint32_t total = *ntotal;
    for (uint32_t p = blockIdx.x * kThreads + threadIdx.x; p < total; p += gridDim.x * kThreads) {
        const uint32_t x = (uint32_t)__ldg(fci + p);
        T[p] = make_ulonglong2(fp_term(kFpSeed1, q, x), fp_term(kFpSeed2, q, x));
    }
}

// Re-point the rows of a level (one linking edge) at their filtered runs and rebuild F.
__global__ void __launch_bounds__(kThreads) k_refilter(Loc *__restrict__ loc, long long nM,
                                                       const uint32_t *__restrict__ fpos, uint32_t lo, uint32_t hi,
                                                       unsigned long long *__restrict__ F,
                                                       unsigned long long *status, unsigned *tile_ctr,
                                                       Counters *ctr) {
    __shared__ unsigned long long sm[33];
    __shared__ unsigned tile_s;
    __shared__ unsigned long long base_s;
    if (threadIdx.x == 0) tile_s = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const unsigned tile = tile_s;
    const long long i = (long long)tile * kThreads + threadIdx.x;
    unsigned long long len0 = 0;
    if (i < nM) {
        const Loc L = loc[i];
        Loc R{0u, 0u};
        if (L.len && L.off >= lo && L.off + L.len <= hi) {
            const uint32_t a = __ldg(fpos + (L.off - lo)), b = __ldg(fpos + (L.off + L.len - lo));
            R = Loc{a, b - a};
        }
        loc[i] = R;
        len0 = R.len;
    }
    unsigned long long agg;
    const unsigned long long ex = block_exclusive_scan(len0, sm, &agg);
    if (threadIdx.x < 32) {
        const unsigned long long pre = lookback_exclusive(status, tile, agg);
        if (threadIdx.x == 0) base_s = pre;
    }
    __syncthreads();
    if (i < nM) F[i] = base_s + ex;
    if (tile == gridDim.x - 1 && threadIdx.x == kThreads - 1) F[nM] = base_s + agg;
    const unsigned long long a1 = warp_sum_u64(len0 ? 1ull : 0ull), e1 = warp_sum_u64(len0);
    if ((threadIdx.x & 31) == 0) {
        if (a1) atomicAdd(&ctr->active_rows, a1);
        if (e1) atomicAdd(&ctr->list_elems, e1);
    }
}

// F = exclusive scan of the buffer bounds loc[i*E].len (rows that arrived without F).
__global__ void __launch_bounds__(kThreads) k_lens_scan(const Loc *__restrict__ loc, long long nM, int E,
                                                        unsigned long long *__restrict__ F,
                                                        unsigned long long *status, unsigned *tile_ctr) {
    __shared__ unsigned long long sm[33];
    __shared__ unsigned tile_s;
    __shared__ unsigned long long base_s;
    if (threadIdx.x == 0) tile_s = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const unsigned tile = tile_s;
    const long long i = (long long)tile * kThreads + threadIdx.x;
    const unsigned long long len0 = i < nM ? loc[(unsigned long long)i * E].len : 0ull;
    unsigned long long agg;
    const unsigned long long ex = block_exclusive_scan(len0, sm, &agg);
    if (threadIdx.x < 32) {
        const unsigned long long pre = lookback_exclusive(status, tile, agg);
        if (threadIdx.x == 0) base_s = pre;
    }
    __syncthreads();
    if (i < nM) F[i] = base_s + ex;
    if (tile == gridDim.x - 1 && threadIdx.x == kThreads - 1) F[nM] = base_s + agg;
}

// ------------------------------------------------------------ NEXT-3 ablations ------
// The paper's own join design (one warp per row of M, Alg. 3 / Alg. 4), with the switches of
// its join-phase study (§VII, Tables VI-VIII): the lookup structure
// (PCSR, or the Compressed Representation's binary search over a sorted vertex-ID layer,
// L674-682), the output scheme (Prealloc-Combine: survivors written once into the Prealloc'd
// GBA buffers then linked, Alg. 3 lines 14-21; or the two-step scheme of GpSM that joins twice,
// counting first, L1635-1641), the write cache (survivor rows staged in shared memory and
// written as a coalesced block, L1155-1158, or written by each lane directly) and the set
// operation (GPU-friendly: C(u) bitset + binary search, L1136-1158; or naive: C(u) by binary
// search in the sorted candidate list, other lists by linear scan).  Same R in every
// combination; used to reproduce the paper's trends on B200, never by default.
enum AblMode { AB_PC = 0, AB_COUNT = 1, AB_WRITE = 2, AB_FINAL = 3 };

__device__ __forceinline__ Loc abl_lookup(const StepParams &P, int e, uint32_t v, bool cr,
                                          const unsigned long long *__restrict__ cr_key,
                                          const uint2 *__restrict__ cr_loc, const uint2 *__restrict__ groups,
                                          int gpn) {
    if (!cr) return pcsr_lookup(groups, gpn, P.gbase[e], P.ngroups[e], P.lab[e], v, nullptr);
    const unsigned long long key = ((unsigned long long)P.lab[e] << 32) | v;
    unsigned long long lo = P.gbase[e], hi = lo + P.ngroups[e];   // lower bound in the vertex-ID layer
    while (lo < hi) {
        const unsigned long long mid = (lo + hi) >> 1;
        if (__ldg(cr_key + mid) < key) lo = mid + 1; else hi = mid;
    }
    if (lo < P.gbase[e] + P.ngroups[e] && __ldg(cr_key + lo) == key) {
        const uint2 r = __ldg(cr_loc + lo);
        return Loc{r.x, r.y};
    }
    return Loc{0u, 0u};
}

// Alg. 4: thread per row; lens[i] = the row's buffer bound (paper or per-row e0).
__global__ void k_abl_probe(const int32_t *__restrict__ M, long long nM, StepParams P, int cr,
                            const unsigned long long *__restrict__ cr_key, const uint2 *__restrict__ cr_loc,
                            const uint2 *__restrict__ groups, int gpn, Loc *__restrict__ loc, uint32_t *__restrict__ lens) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nM; i += (long long)gridDim.x * blockDim.x) {
        Loc first{0u, 0u}, best{0u, 0u};
        int bi = 0;
        bool anyzero = false;
        for (int e = 0; e < P.E; e++) {
            const Loc r = abl_lookup(P, e, (uint32_t)M[i * P.t + P.col[e]], cr != 0, cr_key, cr_loc, groups, gpn);
            loc[i * P.E + e] = r;
            if (e == 0) first = best = r;
            else if (r.len < best.len) {
                best = r;
                bi = e;
            }
            anyzero |= r.len == 0;
        }
        if (P.per_row_e0 && bi != 0) {
            loc[i * P.E] = best;
            loc[i * P.E + bi] = first;
        }
        lens[i] = P.per_row_e0 ? (anyzero ? 0u : best.len) : first.len;
    }
}

// Exclusive scan of u32 counts into u64 offsets (decoupled look-back); out[n] = total.
__global__ void __launch_bounds__(kThreads) k_scan_counts(const uint32_t *__restrict__ in, long long n,
                                                          unsigned long long *__restrict__ out,
                                                          unsigned long long *status, unsigned *tile_ctr) {
    __shared__ unsigned long long sm[33];
    __shared__ unsigned tile_s;
    __shared__ unsigned long long base_s;
    if (threadIdx.x == 0) tile_s = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const unsigned tile = tile_s;
    const long long i = (long long)tile * kThreads + threadIdx.x;
    const unsigned long long x = i < n ? in[i] : 0ull;
    unsigned long long agg;
    const unsigned long long ex = block_exclusive_scan(x, sm, &agg);
    if (threadIdx.x < 32) {
        const unsigned long long pre = lookback_exclusive(status, tile, agg);
        if (threadIdx.x == 0) base_s = pre;
    }
    __syncthreads();
    if (i < n) out[i] = base_s + ex;
    if (tile == gridDim.x - 1 && threadIdx.x == kThreads - 1) out[n] = base_s + agg;
}

// Alg. 3 with one warp per row: lanes stride over the row's buffer N(m_i[c0], l0).
//   AB_PC    : survivors into the row's Prealloc buffer gba[F_i ..], cnt[i] = survivors
//   AB_COUNT : two-step pass 1, cnt[i] only
//   AB_WRITE : two-step pass 2, rows m_i || x written at G_i (write cache: staged per warp)
//   AB_FINAL : last level, count (+ fingerprint)
// The per-candidate test of Alg. 3 (lines 9-13) in the paper-style engine.
template <bool NAIVE>
__device__ __forceinline__ bool abl_keep(int32_t x, const int32_t *__restrict__ row, long long i, const Loc *__restrict__ loc,
                                         const StepParams &P, const int32_t *__restrict__ ci,
                                         const uint32_t *__restrict__ cu_bm, const int32_t *__restrict__ cu_list,
                                         long long cu_n) {
    bool keep = NAIVE ? in_sorted(cu_list, (uint32_t)cu_n, x) : ((__ldg(cu_bm + ((uint32_t)x >> 5)) >> (x & 31)) & 1u);
    for (int q = 0; q < P.n_inj && keep; q++) keep = row[P.inj_col[q]] != x;      // line 10
    for (int e = 1; e < P.E && keep; e++) {                                      // line 13
        const Loc Le = loc[i * P.E + e];
        if (NAIVE) {
            bool f = false;
            for (uint32_t q = 0; q < Le.len && !f; q++) f = __ldg(ci + Le.off + q) == x;
            keep = f;
        } else {
            keep = in_sorted(ci + Le.off, Le.len, x);
        }
    }
    return keep;
}

// Alg. 3 with one warp per row (layer 4 of the 4-layer balance): lanes stride over the
// row's buffer N(m_i[c0], l0).  rows = the light rows of the level (null: every row).
//   AB_PC    : survivors into the row's Prealloc buffer gba[F_i ..], cnt[i] = survivors
//   AB_COUNT : two-step pass 1, cnt[i] only
//   AB_WRITE : two-step pass 2, rows m_i || x written at G_i (write cache: staged per warp)
//   AB_FINAL : last level, count (+ fingerprint)
// DR: duplicate removal within the block (Alg. 5): the 8 warps take 8 rows at a
// time; warps whose rows read the same run N(v,l0) share one input buffer in shared memory,
// filled batch by batch by the first of them, every warp then processing the batch from that
// buffer (block-synchronous, as in Alg. 5).
constexpr int kDrBatch = 128;
template <int MODE, bool WCACHE, bool NAIVE, bool DR>
__global__ void __launch_bounds__(kThreads) k_abl_join(const int32_t *__restrict__ M, long long nM,
                                                       const uint32_t *__restrict__ rows,
                                                       const Loc *__restrict__ loc,
                                                       const unsigned long long *__restrict__ off, StepParams P,
                                                       const int32_t *__restrict__ ci,
                                                       const uint32_t *__restrict__ cu_bm,
                                                       const int32_t *__restrict__ cu_list, long long cu_n,
                                                       int32_t *__restrict__ gba, uint32_t *__restrict__ cnt,
                                                       int32_t *__restrict__ out, Counters *ctr) {
    constexpr int NW = kThreads / 32;
    __shared__ int32_t stage[NW][32];
    __shared__ int32_t dbuf[DR ? NW : 1][DR ? kDrBatch : 1];
    __shared__ Loc dkey[NW];
    __shared__ int daddr[NW];
    __shared__ uint32_t dmax;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int t = P.t, W = t + 1;
    unsigned long long c_all = 0, h1 = 0, h2 = 0;
    // one row: survivors of candidates [j0, j0 + 32) read from src (global run or shared buffer)
    // candidate j of the row is src[j - sbase] (the global run, or the shared DR buffer)
    auto step32 = [&](long long i, const int32_t *row, const Loc &L0, uint32_t j0, const int32_t *src,
                      uint32_t sbase, unsigned long long base, uint32_t &c) {
        const uint32_t j = j0 + lane;
        bool keep = j < L0.len;
        const int32_t x = keep ? src[j - sbase] : 0;
        if (keep) keep = abl_keep<NAIVE>(x, row, i, loc, P, ci, cu_bm, cu_list, cu_n);
        const unsigned b = __ballot_sync(0xffffffffu, keep);
        const uint32_t pos = c + __popc(b & lt);
        if (MODE == AB_PC && keep) gba[base + pos] = x;
        if (MODE == AB_FINAL && keep) {
            c_all++;
            if (P.fp) row_hash(row, (uint32_t)x, P, h1, h2);
        }
        if (MODE == AB_WRITE) {
            if (WCACHE) {   // stage the chunk's survivors, then one coalesced block of rows
                if (keep) stage[wib][__popc(b & lt)] = x;
                __syncwarp();
                const int ns = __popc(b);
                int32_t *o = out + (base + c) * (unsigned long long)W;
                for (int e = lane; e < ns * W; e += 32) {
                    const int r = e / W, col = e - r * W;
                    o[e] = col < t ? row[col] : stage[wib][r];
                }
                __syncwarp();
            } else if (keep) {   // each lane writes its own row (strided stores)
                int32_t *o = out + (base + pos) * (unsigned long long)W;
                for (int col = 0; col < t; col++) o[col] = row[col];
                o[t] = x;
            }
        }
        c += __popc(b);
    };
    if (!DR) {
        const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
        const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
        for (long long r = gw; r < nM; r += nw) {
            const long long i = rows ? (long long)rows[r] : r;
            const Loc L0 = loc[i * P.E];
            const int32_t *row = M + i * t;
            uint32_t c = 0;
            const unsigned long long base = (MODE == AB_PC || MODE == AB_WRITE) ? off[i] : 0ull;
            for (uint32_t j0 = 0; j0 < L0.len; j0 += 32) step32(i, row, L0, j0, ci + L0.off, 0u, base, c);
            if ((MODE == AB_PC || MODE == AB_COUNT) && lane == 0) cnt[i] = c;
        }
    } else {
        for (long long g0 = (long long)blockIdx.x * NW; g0 < nM; g0 += (long long)gridDim.x * NW) {
            const long long r = g0 + wib;
            const bool valid = r < nM;
            const long long i = valid ? (rows ? (long long)rows[r] : r) : 0;
            const Loc L0 = valid ? loc[i * P.E] : Loc{0u, 0u};
            const int32_t *row = M + i * t;
            if (threadIdx.x == 0) dmax = 0;
            if (lane == 0) dkey[wib] = L0;
            __syncthreads();
            if (lane == 0) {   // Alg. 5 lines 2-5: the first warp of the block with the same run
                int a = wib;
                for (int w = 0; w < wib; w++)
                    if (dkey[w].off == L0.off && dkey[w].len == L0.len) {
                        a = w;
                        break;
                    }
                daddr[wib] = L0.len ? a : wib;
                atomicMax(&dmax, L0.len);
            }
            __syncthreads();
            const int a = daddr[wib];
            const uint32_t lmax = dmax;
            uint32_t c = 0;
            const unsigned long long base = (valid && (MODE == AB_PC || MODE == AB_WRITE)) ? off[i] : 0ull;
            for (uint32_t b0 = 0; b0 < lmax; b0 += kDrBatch) {   // Alg. 5 lines 6-10
                if (a == wib)
                    for (uint32_t q = lane; q < kDrBatch && b0 + q < L0.len; q += 32) dbuf[wib][q] = __ldg(ci + L0.off + b0 + q);
                __syncthreads();
                for (uint32_t q0 = 0; q0 < kDrBatch && b0 + q0 < L0.len; q0 += 32)
                    step32(i, row, L0, b0 + q0, dbuf[a], b0, base, c);
                __syncthreads();
            }
            if (valid && (MODE == AB_PC || MODE == AB_COUNT) && lane == 0) cnt[i] = c;
        }
    }
    if (MODE == AB_FINAL) {
        c_all = warp_sum_u64(c_all);
        h1 = warp_sum_u64(h1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) h2 ^= __shfl_xor_sync(0xffffffffu, h2, o);
        if (lane == 0 && c_all) {
            atomicAdd(&ctr->count, c_all);
            atomicAdd(&ctr->fp1, h1);
            atomicXor(&ctr->fp2, h2);
        }
    }
}

// Layers 1-2 of the 4-layer balance for the paper-style engine.  A row whose
// buffer exceeds W2 is processed by a whole block (layer 2); one above W1 by a thread-block
// CLUSTER of up to 8 CTAs (layer 1 — the B200 form of the paper's dynamically launched child
// kernel, L1172: no device-side launch, the cluster is part of the same grid).  The cluster's
// rank-0 CTA stages the row (its columns and linking-list locations) in shared memory and the
// other CTAs read it through distributed shared memory; each round, CTA r takes a contiguous
// 1024-candidate slice, compacts its survivors in order into shared memory, publishes its
// count, and reads the counts of ranks < r through DSMEM to place its survivors in the row's
// buffer (Prealloc: gba[F_i + ...]; two-step pass 2: rows at G_i + ...) — an exact in-order
// compaction with no global atomics.  rows = the level's rows of this layer.
constexpr int kSegItems = 4;
constexpr int kSegSlice = kThreads * kSegItems;
template <int MODE, bool WCACHE, bool NAIVE>
__global__ void __launch_bounds__(kThreads) k_abl_heavy(const int32_t *__restrict__ M, const uint32_t *__restrict__ rows,
                                                        long long nrows, const Loc *__restrict__ loc,
                                                        const unsigned long long *__restrict__ off, StepParams P,
                                                        const int32_t *__restrict__ ci,
                                                        const uint32_t *__restrict__ cu_bm,
                                                        const int32_t *__restrict__ cu_list, long long cu_n,
                                                        int32_t *__restrict__ gba, uint32_t *__restrict__ cnt,
                                                        int32_t *__restrict__ out, Counters *ctr) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int CL = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
    __shared__ int32_t s_row[GSI_MAX_K];
    __shared__ Loc s_loc[GSI_MAX_K];
    __shared__ int32_t s_x[kSegSlice];
    __shared__ unsigned long long s_scan[33];
    __shared__ unsigned long long s_cnt;
    const int tid = threadIdx.x, lane = tid & 31;
    const int t = P.t, W = t + 1;
    unsigned long long c_all = 0, h1 = 0, h2 = 0;
    const long long nclusters = gridDim.x / CL, cid = blockIdx.x / CL;
    for (long long r = cid; r < nrows; r += nclusters) {
        const long long i = rows[r];
        if (rank == 0) {   // stage the row once per cluster
            if (tid < t) s_row[tid] = M[i * t + tid];
            if (tid < P.E) s_loc[tid] = loc[i * P.E + tid];
        }
        cluster.sync();
        int32_t row[GSI_MAX_K];
        const int32_t *rrow = cluster.map_shared_rank(s_row, 0);   // DSMEM reads of rank 0's copy
        const Loc *rloc = cluster.map_shared_rank(s_loc, 0);
        for (int c = 0; c < t; c++) row[c] = rrow[c];
        const Loc L0 = rloc[0];
        Loc Ls[GSI_MAX_K];
        for (int e = 1; e < P.E; e++) Ls[e] = rloc[e];
        const unsigned long long base = (MODE == AB_PC || MODE == AB_WRITE) ? off[i] : 0ull;
        unsigned long long run = 0;
        for (unsigned long long r0 = 0; r0 < L0.len; r0 += (unsigned long long)CL * kSegSlice) {
            const unsigned long long s0 = r0 + (unsigned long long)rank * kSegSlice;
            int32_t xs[kSegItems];
            bool kp[kSegItems];
            uint32_t mine = 0;
#pragma unroll
            for (int it = 0; it < kSegItems; it++) {   // blocked: thread tid owns slots [4 tid, 4 tid + 4)
                const unsigned long long j = s0 + (unsigned long long)tid * kSegItems + it;
                kp[it] = j < L0.len;
                xs[it] = kp[it] ? __ldg(ci + L0.off + j) : 0;
                if (kp[it]) {
                    bool keep = NAIVE ? in_sorted(cu_list, (uint32_t)cu_n, xs[it])
                                      : ((__ldg(cu_bm + ((uint32_t)xs[it] >> 5)) >> (xs[it] & 31)) & 1u);
                    for (int q = 0; q < P.n_inj && keep; q++) keep = row[P.inj_col[q]] != xs[it];
                    for (int e = 1; e < P.E && keep; e++) {
                        if (NAIVE) {
                            bool f = false;
                            for (uint32_t q = 0; q < Ls[e].len && !f; q++) f = __ldg(ci + Ls[e].off + q) == xs[it];
                            keep = f;
                        } else {
                            keep = in_sorted(ci + Ls[e].off, Ls[e].len, xs[it]);
                        }
                    }
                    kp[it] = keep;
                }
                mine += kp[it] ? 1u : 0u;
            }
            unsigned long long tot;
            const unsigned long long ex = block_exclusive_scan(mine, s_scan, &tot);
            uint32_t p = (uint32_t)ex;
#pragma unroll
            for (int it = 0; it < kSegItems; it++)
                if (kp[it]) s_x[p++] = xs[it];
            if (tid == 0) s_cnt = tot;
            cluster.sync();   // every rank's count is published
            unsigned long long before = 0, all = 0;
            for (int q = 0; q < CL; q++) {
                const unsigned long long cq = *cluster.map_shared_rank(&s_cnt, q);
                all += cq;
                if (q < rank) before += cq;
            }
            const unsigned long long o0 = run + before;
            const unsigned n = (unsigned)tot;
            if (MODE == AB_PC)
                for (unsigned q = tid; q < n; q += kThreads) gba[base + o0 + q] = s_x[q];
            if (MODE == AB_FINAL)
                for (unsigned q = tid; q < n; q += kThreads) {
                    c_all++;
                    if (P.fp) row_hash(M + i * t, (uint32_t)s_x[q], P, h1, h2);
                }
            if (MODE == AB_WRITE) {
                int32_t *o = out + (base + o0) * (unsigned long long)W;
                if (WCACHE) {
                    for (unsigned e = tid; e < n * (unsigned)W; e += kThreads) {
                        const unsigned q = e / W, col = e - q * W;
                        o[e] = col < (unsigned)t ? row[col] : s_x[q];
                    }
                } else {
                    for (unsigned q = tid; q < n; q += kThreads) {
                        for (int col = 0; col < t; col++) o[q * W + col] = row[col];
                        o[q * W + t] = s_x[q];
                    }
                }
            }
            run += all;
            cluster.sync();   // s_x / s_cnt are reused next round
        }
        if ((MODE == AB_PC || MODE == AB_COUNT) && rank == 0 && tid == 0) cnt[i] = (uint32_t)run;
    }
    if (MODE == AB_FINAL) {
        c_all = warp_sum_u64(c_all);
        h1 = warp_sum_u64(h1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) h2 ^= __shfl_xor_sync(0xffffffffu, h2, o);
        if (lane == 0 && c_all) {
            atomicAdd(&ctr->count, c_all);
            atomicAdd(&ctr->fp1, h1);
            atomicXor(&ctr->fp2, h2);
        }
    }
}

// Stable split of a level's rows into the balance layers by buffer length: flag[i] = 1 if
// the row belongs to layer `which` (0: len <= W2, 1: W2 < len <= W1, 2: len > W1).
__global__ void k_abl_flags(const uint32_t *__restrict__ lens, long long n, uint32_t w1, uint32_t w2, int which,
                            uint32_t *__restrict__ flag) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const uint32_t l = lens[i];
        const int b = l > w1 ? 2 : (l > w2 ? 1 : 0);
        flag[i] = b == which ? 1u : 0u;
    }
}
__global__ void k_abl_gather(const uint32_t *__restrict__ flag, const unsigned long long *__restrict__ pos, long long n,
                             uint32_t *__restrict__ rows) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        if (flag[i]) rows[pos[i]] = (uint32_t)i;
}

// Combine (Alg. 3 lines 15-21): M'[G_i + j] = m_i || gba[F_i + j].  Write cache: one thread per
// output int (coalesced); off: one thread per output row.
template <bool WCACHE>
__global__ void k_abl_link(const int32_t *__restrict__ M, long long nM, const unsigned long long *__restrict__ F,
                           const unsigned long long *__restrict__ G, const int32_t *__restrict__ gba, int t,
                           unsigned long long nout, int32_t *__restrict__ out) {
    const int W = t + 1;
    const unsigned long long total = WCACHE ? nout * (unsigned long long)W : nout;
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < total;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long r = WCACHE ? e / W : e;
        long long lo = 0, hi = nM;   // last row i with G[i] <= r
        while (hi - lo > 1) {
            const long long mid = (lo + hi) >> 1;
            if (G[mid] <= r) lo = mid; else hi = mid;
        }
        const int32_t x = gba[F[lo] + (r - G[lo])];
        if (WCACHE) {
            const int col = (int)(e - r * W);
            out[e] = col < t ? M[lo * t + col] : x;
        } else {
            for (int col = 0; col < t; col++) out[r * W + col] = M[lo * t + col];
            out[r * W + t] = x;
        }
    }
}

// ------------------------------------------------------------ small-query path -----
// A query whose levels all stay small (C2-C4-shaped: |C(pi_1)| of a few to a few thousand,
// ~11 levels of tens to thousands of rows) is latency-bound on the regular path: one join
// launch and one counter read-back per level.  k_small_query runs the whole query after the
// filter inside one CTA of 1024 threads, with nothing on the host between the filter and the
// result: the join order (Alg. 2, the same greedy function the host planner calls), the steps
// and their subtraction columns are planned by one thread from |C(u)| on the device; M_1 =
// C(pi_1) is extracted in ascending order from the filter's bitmap through its per-group
// counts; then every level runs — Prealloc probe + block scan (Alg. 4), the join over the
// slot range in rounds of 1024 slots (Alg. 3 lines 2-13: C(u) bit, subtraction, the other
// linking lists), and an ordered block-scan compaction into the next level's rows (the Combine,
// Alg. 3 lines 14-21).  The host launches filter + this kernel back to back and reads one
// block back.  Rows are produced in the same lexicographic pi order as the regular path.  If
// the query does not fit (|C(pi_1)| > 4096 roots, more than 8 linking edges or subtraction
// columns in a step, a level beyond the row or slot capacity) the kernel stops and reports
// the level; the host then runs the regular path from the filter's output (identical results).
constexpr int kSmallThreads = 1024;
constexpr int kSmallMaxE = 8;
constexpr int kSmallMaxInj = 8;
constexpr unsigned long long kSmallRowCap = 1ull << 15;
constexpr unsigned long long kSmallSlotCap = 1ull << 16;
constexpr unsigned long long kSmallMaxRoots = 4096;
// Dynamic shared memory of k_small_query: two row buffers (a level's rows stay on chip when
// they fit, so the next level's row reads and the Combine writes cost shared-memory latency
// instead of L2 round trips) and the level's located lists.
constexpr int kSmallSmRows = 16384;    // int32 per row buffer (64 KB each)
constexpr int kSmallSmLoc = 2048;      // Loc entries (16 KB)
constexpr size_t kSmallDynSmem = 2 * kSmallSmRows * sizeof(int32_t) + kSmallSmLoc * sizeof(Loc);

// Alg. 2's greedy join order (reading A8 in DESIGN.md): start at the
// vertex with the smallest score |C(u)|/deg(u), then repeatedly take the connected vertex of
// smallest score, multiplying the scores of the taken vertex's neighbours by freq(l(e)) (tie:
// the smallest query id).  (A device version — warp 0 of k_small_query, lane = query vertex —
// was measured at ~37 us for a 12-vertex plan, a single warp's dependent chain of a few
// thousand instructions, against ~5 us here plus one read-back; the plan stays on the host.)
inline int plan_greedy(int k, int qm, const int *qs, const int *qd, const long long *freq_e,
                                           const long long *cand, int *order) {
    double score[GSI_MAX_K];
    uint32_t adj[GSI_MAX_K];
    int deg[GSI_MAX_K];
    for (int u = 0; u < k; u++) {
        adj[u] = 0u;
        deg[u] = 0;
    }
    for (int e = 0; e < qm; e++) {
        deg[qs[e]]++;
        deg[qd[e]]++;
        adj[qs[e]] |= 1u << qd[e];
        adj[qd[e]] |= 1u << qs[e];
    }
    for (int u = 0; u < k; u++) score[u] = deg[u] ? (double)cand[u] / deg[u] : (double)cand[u];
    uint32_t in = 0u;
    for (int i = 0; i < k; i++) {
        int best = -1;
        for (int u = 0; u < k; u++) {
            if ((in >> u) & 1u) continue;
            if (i > 0 && !(adj[u] & in)) continue;   // connected to the prefix
            if (best < 0 || score[u] < score[best]) best = u;
        }
        if (best < 0) return -1;                      // disconnected query
        order[i] = best;
        in |= 1u << best;
        for (int e = 0; e < qm; e++) {
            const int o = qs[e] == best ? qd[e] : (qd[e] == best ? qs[e] : -1);
            if (o >= 0) score[o] *= (double)freq_e[e];
        }
    }
    return 0;
}

struct SmallStep {
    int E, n_inj;
    int col[kSmallMaxE];
    uint32_t lab[kSmallMaxE];
    uint32_t ngroups[kSmallMaxE];
    unsigned long long gbase[kSmallMaxE];
    int inj_col[kSmallMaxInj];
    const uint32_t *cu;
};
struct SmallPlan {
    int k, want_table, fp, gpn;
    int pos_of_q[GSI_MAX_K];
    SmallStep st[GSI_MAX_K - 1];   // st[j]: the step joining column j + 1 (j + 1 columns before it)
    // level 1: M_1 = C(pi_1), from the filter's bitmap of pi_1 and its per-group counts
    const uint32_t *bm1;
    const uint16_t *grp1;          // [ngrp] counts of groups of gw bitmap words (16 B aligned)
    long long words, ngrp;
    int gw;
    unsigned long long nM1;        // |C(pi_1)| <= kSmallMaxRoots
};
struct SmallOut {
    unsigned long long count, fp1, fp2, nout;
    int aborted;                              // 0: done; t: level t exceeded a capacity
    unsigned long long rows[GSI_MAX_K];       // |M_t| at t - 1
    unsigned long long gba[GSI_MAX_K];        // |GBA| of level t at t
    unsigned long long elems[GSI_MAX_K];
    long long clk[GSI_MAX_K + 2];             // SM clock at: start, -, M_1 done, level t done (GSI_TRACE)
};

// Exclusive scan over the G threads of a group (G = 1024: the block, smem[33]; G = 32: a warp).
template <int G>
__device__ __forceinline__ unsigned long long group_exclusive_scan(unsigned long long x, unsigned long long *smem,
                                                                   unsigned long long *total) {
    if (G == 32) {
        const int lane = threadIdx.x & 31;
        unsigned long long inc = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        *total = __shfl_sync(0xffffffffu, inc, 31);
        return inc - x;
    }
    return block_exclusive_scan(x, smem, total);
}

// Prealloc of one small-path level (Alg. 4) by a group of G threads: locate every linking list,
// the per-row shortest list bounds the buffer (any linking edge bounds it, L967-981), F =
// exclusive scan, F[nM] = |GBA| = *T_s; *el_s = list elements of the active rows.
template <int G>
__device__ __forceinline__ void small_prealloc(const SmallStep &S, int t, unsigned long long nM, const int32_t *cur,
                                               Loc *loc, unsigned long long *Fd, const uint2 *__restrict__ groups,
                                               int gpn, unsigned long long *sm, unsigned long long *T_s,
                                               unsigned long long *el_s) {
    const int gt = threadIdx.x & (G - 1), lane = threadIdx.x & 31;
    const int E = S.E;
    if (gt == 0) *el_s = 0;
    if (G == 32) __syncwarp();
    else __syncthreads();
    unsigned long long run = 0;
    for (unsigned long long b0 = 0; b0 < nM; b0 += G) {
        const unsigned long long i = b0 + gt;
        unsigned long long len0 = 0, el = 0;
        if (i < nM) {
            Loc best{0u, 0xFFFFFFFFu}, first{0u, 0u};
            int bi = 0;
            bool anyzero = false;
            for (int e = 0; e < E; e++) {
                const uint32_t v = (uint32_t)cur[i * t + S.col[e]];
                const Loc r = pcsr_lookup(groups, gpn, S.gbase[e], S.ngroups[e], S.lab[e], v, nullptr);
                loc[i * E + e] = r;
                if (e == 0) first = r;
                if (r.len < best.len) {
                    best = r;
                    bi = e;
                }
                anyzero |= r.len == 0;
                el += r.len;
            }
            if (bi != 0) {
                loc[i * E] = best;
                loc[i * E + bi] = first;
            }
            len0 = anyzero ? 0ull : best.len;
            if (anyzero) el = 0;
        }
        unsigned long long agg;
        const unsigned long long ex = group_exclusive_scan<G>(len0, sm, &agg);
        if (i < nM) Fd[i] = run + ex;
        run += agg;
        el = warp_sum_u64(el);
        if (lane == 0 && el) atomicAdd(el_s, el);
    }
    if (gt == 0) {
        Fd[nM] = run;
        *T_s = run;
    }
}

// Join + Combine of one small-path level by a group of G threads: slots in rounds of G, the
// ordered compaction into the next level's rows (or, at the last level, the count /
// fingerprint / table).  *nout_s = rows produced (~0: over the row capacity).
template <int G>
__device__ __forceinline__ void small_join(const SmallPlan &sp, const SmallStep &S, int t, bool last,
                                           unsigned long long nM, unsigned long long T, const int32_t *cur,
                                           const Loc *loc, const unsigned long long *FF, const int32_t *__restrict__ ci,
                                           int32_t *nxt, int32_t *table, unsigned long long *sm,
                                           unsigned long long *nout_s, unsigned long long *cnt_s,
                                           unsigned long long *h1_s, unsigned long long *h2_s) {
    const int gt = threadIdx.x & (G - 1), lane = threadIdx.x & 31;
    const int E = S.E, k = sp.k;
    unsigned long long nout = 0;
    for (unsigned long long s0 = 0; s0 < T; s0 += G) {
        const unsigned long long sl = s0 + gt;
        bool keep = false;
        int32_t x = 0;
        unsigned long long row = 0;
        if (sl < T) {
            unsigned long long lo = 0, hi = nM;   // last row with F[row] <= sl
            while (hi - lo > 1) {
                const unsigned long long mid = (lo + hi) >> 1;
                if (FF[mid] <= sl) lo = mid; else hi = mid;
            }
            row = lo;
            const Loc L0 = loc[row * E];
            x = __ldg(ci + L0.off + (uint32_t)(sl - FF[row]));
            keep = (__ldg(S.cu + ((uint32_t)x >> 5)) >> (x & 31)) & 1u;              // x in C(u)
            for (int c = 0; c < S.n_inj && keep; c++) keep = cur[row * t + S.inj_col[c]] != x;   // line 10
            for (int e = 1; e < E && keep; e++) {                                       // line 13
                const Loc Le = loc[row * E + e];
                keep = in_sorted(ci + Le.off, Le.len, x);
            }
        }
        if (last && !sp.want_table) {
            unsigned long long c = keep ? 1ull : 0ull, a1 = 0, a2 = 0;
            if (keep && sp.fp) {
                for (int q = 0; q < k; q++) {
                    const int col = sp.pos_of_q[q];
                    const uint32_t val = col < t ? (uint32_t)cur[row * t + col] : (uint32_t)x;
                    a1 += fp_term(kFpSeed1, q, val);
                    a2 += fp_term(kFpSeed2, q, val);
                }
                a1 = fp_mix(a1);
                a2 = fp_mix(a2);
            }
            c = warp_sum_u64(c);
            a1 = warp_sum_u64(a1);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) a2 ^= __shfl_xor_sync(0xffffffffu, a2, o);
            if (lane == 0 && c) {
                atomicAdd(cnt_s, c);
                atomicAdd(h1_s, a1);
                atomicXor(h2_s, a2);
            }
            continue;
        }
        unsigned long long agg;
        const unsigned long long ex = group_exclusive_scan<G>(keep ? 1ull : 0ull, sm, &agg);
        if (nout + agg > kSmallRowCap) {
            if (gt == 0) *nout_s = ~0ull;
            return;
        }
        if (keep) {
            const unsigned long long p = nout + ex;
            if (last) {   // the table in query-id order (+ fingerprint)
                unsigned long long a1 = 0, a2 = 0;
                for (int q = 0; q < k; q++) {
                    const int col = sp.pos_of_q[q];
                    const int32_t val = col < t ? cur[row * t + col] : x;
                    table[p * k + q] = val;
                    a1 += fp_term(kFpSeed1, q, (uint32_t)val);
                    a2 += fp_term(kFpSeed2, q, (uint32_t)val);
                }
                if (sp.fp) {
                    atomicAdd(h1_s, fp_mix(a1));
                    atomicXor(h2_s, fp_mix(a2));
                }
            } else {
                for (int c = 0; c < t; c++) nxt[p * (t + 1) + c] = cur[row * t + c];
                nxt[p * (t + 1) + t] = x;
            }
        }
        nout += agg;
    }
    if (gt == 0) *nout_s = nout;
}

__global__ void __launch_bounds__(kSmallThreads, 1) k_small_query(const __grid_constant__ SmallPlan sp,
                                                                  const uint2 *__restrict__ groups,
                                                                  const int32_t *__restrict__ ci,
                                                                  int32_t *__restrict__ bufA, int32_t *__restrict__ bufB,
                                                                  Loc *__restrict__ locG,
                                                                  unsigned long long *__restrict__ F,
                                                                  int32_t *__restrict__ table, SmallOut *out) {
    __shared__ unsigned long long sm[34];
    __shared__ unsigned long long cnt_s, h1_s, h2_s, el_s, T_s, nout_s;
    // F of a level with fewer than kSmallFsh rows stays in shared memory: the join's per-slot
    // row search then costs shared-memory latency instead of a chain of L2 round trips
    constexpr int kSmallFsh = 4097;
    __shared__ unsigned long long Fs[kSmallFsh];
    extern __shared__ __align__(16) unsigned char small_dyn[];
    int32_t *const sA = reinterpret_cast<int32_t *>(small_dyn);
    int32_t *const sB = sA + kSmallSmRows;
    Loc *const locS = reinterpret_cast<Loc *>(sB + kSmallSmRows);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int k = sp.k;
    if (tid == 0) {
        out->clk[0] = clock64();
        cnt_s = h1_s = h2_s = 0;
    }
    // ---- level 1 (Alg. 2 line 7): M_1 = C(pi_1) ascending, from the per-group counts ------
    // Each thread sums a contiguous, 16 B aligned range of groups (vector loads, all in flight
    // at once); one block scan gives every thread its output offset and its first
    // non-empty-group index; the non-empty groups (<= |M_1|) are listed in shared memory (Fs,
    // free until level 1's Prealloc) and a warp per group writes its vertices in order.
    unsigned long long nM = sp.nM1;
    {
        const uint32_t *bm1 = sp.bm1;
        const uint16_t *g1 = sp.grp1;
        const long long ng = sp.ngrp;
        const long long per = ((ng + kSmallThreads - 1) / kSmallThreads + 7) & ~7ll;
        const long long a = tid * per, b = min(ng, a + per);
        unsigned long long sum = 0, ne = 0;
        for (long long x0 = a; x0 < b; x0 += 8) {
            const uint4 v = *reinterpret_cast<const uint4 *>(g1 + x0);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const unsigned c = x0 + i < b ? (w[i >> 1] >> (16 * (i & 1))) & 0xFFFFu : 0u;
                sum += c;
                ne += c ? 1 : 0;
            }
        }
        unsigned long long tot;
        const unsigned long long ex = block_exclusive_scan((sum << 32) | ne, sm, &tot);
        unsigned long long obase = ex >> 32, li = ex & 0xFFFFFFFFull;
        for (long long x = a; x < b && obase < (ex >> 32) + sum; x++) {
            const unsigned c = g1[x];
            if (!c) continue;
            Fs[li++] = ((unsigned long long)x << 32) | obase;
            obase += c;
        }
        __syncthreads();
        const unsigned long long nne = tot & 0xFFFFFFFFull;
        const int GW = sp.gw;
        for (unsigned long long i = warp; i < nne; i += kSmallThreads / 32) {
            const unsigned long long e = Fs[i];
            const long long w = (long long)(e >> 32) * GW + lane;
            const uint32_t word = (lane < GW && w < sp.words) ? bm1[w] : 0u;
            const unsigned c = __popc(word);
            unsigned inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            unsigned long long p = (e & 0xFFFFFFFFull) + inc - c;
            uint32_t bits = word;
            while (bits) {
                sA[p++] = (int32_t)(w * 32 + __ffs(bits) - 1);   // M_1 (<= 4096 rows) on chip
                bits &= bits - 1;
            }
        }
        __syncthreads();   // M_1 written before level 1 reads it; Fs free again
    }
    if (tid == 0) out->clk[2] = clock64();
    if (tid == 0) out->rows[0] = nM;
    // rows of the current level: a shared-memory buffer when they fit, else bufA / bufB.  A
    // level of <= 32 rows runs its Prealloc in warp 0 alone, a join of <= 256 slots likewise
    // (warp scans instead of block scans: two barriers per level instead of nine — the
    // C2/C4 queries' deep levels hold a handful of rows).
    const int32_t *cur = sA;
    for (int t = 1; t < k; t++) {
        const SmallStep &S = sp.st[t - 1];
        const int E = S.E;
        const bool last = t == k - 1;
        Loc *const loc = nM * (unsigned long long)E <= (unsigned long long)kSmallSmLoc ? locS : locG;
        unsigned long long *const Fdst = nM < kSmallFsh ? Fs : F;
        if (nM > 32) small_prealloc<kSmallThreads>(S, t, nM, cur, loc, Fdst, groups, sp.gpn, sm, &T_s, &el_s);
        else if (warp == 0) small_prealloc<32>(S, t, nM, cur, loc, Fdst, groups, sp.gpn, sm, &T_s, &el_s);
        __syncthreads();   // F, loc and T visible to the whole block
        const unsigned long long T = T_s;
        if (tid == 0) {
            out->gba[t] = T;
            out->elems[t] = el_s;
        }
        if (T > kSmallSlotCap) {
            if (tid == 0) out->aborted = t;
            return;
        }
        // the next level's rows (at most T of t + 1 columns): on chip if they fit
        int32_t *nxt;
        if (T * (unsigned long long)(t + 1) <= (unsigned long long)kSmallSmRows) nxt = cur == sA ? sB : sA;
        else nxt = cur == bufA ? bufB : bufA;
        if (T > 256) small_join<kSmallThreads>(sp, S, t, last, nM, T, cur, loc, Fdst, ci, nxt, table, sm, &nout_s, &cnt_s, &h1_s, &h2_s);
        else if (warp == 0) small_join<32>(sp, S, t, last, nM, T, cur, loc, Fdst, ci, nxt, table, sm, &nout_s, &cnt_s, &h1_s, &h2_s);
        __syncthreads();   // every row of the next level written before it is read
        const unsigned long long nout = nout_s;
        if (nout == ~0ull) {   // the next level outgrew the row capacity
            if (tid == 0) out->aborted = t + 1;
            return;
        }
        if (last) {
            if (tid == 0) {
                out->clk[2 + t] = clock64();
                const unsigned long long c = sp.want_table ? nout : cnt_s;
                out->count = c;
                out->nout = nout;
                out->rows[t] = c;
                out->fp1 = h1_s;
                out->fp2 = h2_s;
                out->aborted = 0;
            }
            return;
        }
        if (tid == 0) {
            out->rows[t] = nout;
            out->clk[2 + t] = clock64();
        }
        nM = nout;
        cur = nxt;
        if (nM == 0) break;
        __syncthreads();   // T_s / nout_s are rewritten by the next level
    }
    if (tid == 0) {   // a level came out empty: no matches (later rows stay 0)
        out->count = 0;
        out->nout = 0;
        out->aborted = 0;
    }
}

// Count + fingerprint of a table whose columns are in pi order (k = 1 queries).
__global__ void k_fp_rows(const int32_t *__restrict__ T, long long nrows, StepParams P, Counters *ctr) {
    unsigned long long h1 = 0, h2 = 0;
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < nrows; r += (long long)gridDim.x * blockDim.x) {
        unsigned long long a = 0, b = 0;
        for (int q = 0; q < P.k; q++) {
            uint32_t val = (uint32_t)T[r * P.t + P.pos_of_q[q]];
            a += fp_term(kFpSeed1, q, val);
            b += fp_term(kFpSeed2, q, val);
        }
        h1 += fp_mix(a);
        h2 ^= fp_mix(b);
    }
    h1 = warp_sum_u64(h1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h2 ^= __shfl_xor_sync(0xffffffffu, h2, o);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&ctr->fp1, h1);
        atomicXor(&ctr->fp2, h2);
    }
}

// Shard boundaries: the level's slot range [0, T = F[|M|]) is cut into NP
// equal pieces at row granularity: a_j = first row with F[i] >= ceil(j T / NP) (a_0 = 0,
// a_NP = |M|); out[j] = a_j and out[NP + 1 + j] = F[a_j] for j = 0..NP.
__global__ void k_shard_bounds(const unsigned long long *F, long long nM, int NP, long long *out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j > NP) return;
    const unsigned long long T = F[nM];
    long long a;
    if (j == 0) {
        a = 0;
    } else if (j >= NP) {
        a = nM;
    } else {
        unsigned __int128 num = (unsigned __int128)j * T + (NP - 1);
        unsigned long long target = (unsigned long long)(num / NP);
        long long lo = 0, hi = nM;   // lower_bound over F[0..nM)
        while (lo < hi) {
            long long mid = (lo + hi) >> 1;
            if (F[mid] < target) lo = mid + 1; else hi = mid;
        }
        a = lo;
    }
    out[j] = a;
    out[NP + 1 + j] = (long long)F[a];
}

}  // namespace

// ====================================================================== host side =====
void encode_query_signatures(int32_t k, const int32_t *qvl, int32_t qm, const int32_t *qs, const int32_t *qd,
                             const int32_t *qe, uint32_t *qsig, int distinct) {
    // Same written specification as the data side: plane 0 = label (L1277),
    // 240 two-bit groups.  Isomorphism counts (edge label, neighbour label) pairs with
    // multiplicity (reading A5); homomorphism may map two query neighbours with the same key
    // onto ONE data neighbour, so its query side counts distinct keys (NEXT-1).
    for (int u = 0; u < k; u++) {
        int cnt[kSigGroups];
        std::memset(cnt, 0, sizeof(cnt));
        std::vector<unsigned long long> seen;
        for (int e = 0; e < qm; e++) {
            int other = qs[e] == u ? qd[e] : (qd[e] == u ? qs[e] : -1);
            if (other < 0) continue;
            if (distinct) {
                const unsigned long long key = ((unsigned long long)(uint32_t)qe[e] << 32) | (uint32_t)qvl[other];
                bool dup = false;
                for (auto x : seen) dup |= x == key;
                if (dup) continue;
                seen.push_back(key);
            }
            cnt[sig_group((uint32_t)qe[e], (uint32_t)qvl[other])]++;
        }
        uint32_t *s = qsig + (size_t)u * kPlanes;
        s[0] = (uint32_t)qvl[u];
        for (int w = 1; w < kPlanes; w++) s[w] = 0;
        for (int gi = 0; gi < kSigGroups; gi++) {
            uint32_t st = cnt[gi] == 0 ? 0u : (cnt[gi] == 1 ? 1u : 3u);
            s[1 + gi / 16] |= st << (2 * (gi % 16));
        }
    }
}

}  // namespace gsi

namespace gsi {
namespace {

inline unsigned grid_for(unsigned long long n, int per) {
    unsigned long long b = (n + per - 1) / per;
    if (b < 1) b = 1;
    return (unsigned)std::min<unsigned long long>(b, 0x7FFFFFFFull);
}

// Per-device workspace: one plain allocation kept across queries and carved as a
// double-ended stack.  The depth-first level recursion allocates LIFO (mark()/reset() per
// chunk) from the bottom; query-lifetime buffers (shared candidate runs, probe-ahead tables)
// come from the top.  Growing the stream-ordered pool by ~1 GB per level chunk cost 7-20 ms
// of host time per allocation (physical mapping) — more than the kernels of a chunk.  A
// query owns the workspace exclusively; a concurrent query on the same device falls back to
// stream-ordered allocations.  Graph builds trim an idle workspace first.
struct Workspace {
    std::mutex mu;
    char *base = nullptr;
    size_t cap = 0;
    size_t want = 64ull << 20;   // high-water demand of the queries so far (next size)
    bool busy = false;
};
constexpr int kWsSlots = 8;        // concurrent queries per device with their own workspace
Workspace g_ws[64][kWsSlots];
// Device-wide high-water demand: every slot grows to the largest query seen on the device,
// so a heavy query never lands on a slot that only ever ran light ones (concurrent batches
// assign queries to slots dynamically).
std::atomic<size_t> g_ws_want[64];

}  // namespace

void workspace_trim(int dev) {
    if (dev < 0 || dev >= 64) return;
    for (int k = 0; k < kWsSlots; k++) {
        Workspace &W = g_ws[dev][k];
        std::lock_guard<std::mutex> lk(W.mu);
        if (W.busy) continue;
        if (W.base) cudaFree(W.base);
        W.base = nullptr;
        W.cap = 0;
        W.want = 64ull << 20;   // a new graph: learn its queries' demand afresh
    }
    g_ws_want[dev] = 0;
}

// Bytes held by the device's idle workspaces (they count as available to a new query).
size_t workspace_idle_bytes(int dev) {
    size_t idle = 0;
    if (dev < 0 || dev >= 64) return 0;
    for (int k = 0; k < kWsSlots; k++) {
        std::lock_guard<std::mutex> lk(g_ws[dev][k].mu);
        if (!g_ws[dev][k].busy) idle += g_ws[dev][k].cap;
    }
    return idle;
}

namespace {

struct Arena {
    cudaStream_t st;
    std::vector<void *> ptrs;
    double ms_alloc = 0;   // host time in allocation calls (stats.ms_host_alloc)
    char *bump = nullptr;
    size_t cap = 0, off = 0, top = 0;
    int ws_dev = -1, ws_slot = -1;   // >= 0: bump is that device's workspace slot
    size_t live_fb = 0, demand = 0;   // live fallback bytes; high-water mark of all scratch
    explicit Arena(cudaStream_t s) : st(s) {}
    void note() { demand = std::max(demand, off + (cap - top) + live_fb); }
    // Take the device workspace, (re)sized to at least `bytes`; on any failure keep going
    // with stream-ordered allocations only.
    void init_workspace(int dev, size_t budget) {
        if (dev < 0 || dev >= 64) return;
        for (int k = 0; k < kWsSlots && ws_dev < 0; k++) take_slot(dev, k, budget);
    }
    void take_slot(int dev, int slot, size_t budget) {
        Workspace &W = g_ws[dev][slot];
        std::lock_guard<std::mutex> lk(W.mu);
        if (W.busy) return;
        const size_t bytes = std::min(budget, std::max(std::max(W.want, g_ws_want[dev].load()), (size_t)64 << 20));
        const auto t0 = std::chrono::steady_clock::now();
        if (W.cap < bytes) {
            if (W.base) cudaFree(W.base);
            W.base = nullptr;
            W.cap = 0;
            cudaMemPool_t pool;   // hand pool-cached memory back to the driver first
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                cudaDeviceSynchronize();
                cudaMemPoolTrimTo(pool, 0);
            }
            if (cudaMalloc((void **)&W.base, bytes) != cudaSuccess) {
                cudaGetLastError();
                W.base = nullptr;
                return;
            }
            W.cap = bytes;
        }
        ms_alloc += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        W.busy = true;
        ws_dev = dev;
        ws_slot = slot;
        bump = W.base;
        cap = W.cap;
        off = 0;
        top = cap & ~(size_t)255;   // both stack ends stay 256 B aligned
    }
    template <typename T>
    gsi_status fallback(T **p, size_t bytes) {
        void *q = nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        cudaError_t e = cudaMallocAsync(&q, bytes, st);
        const double dt = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        ms_alloc += dt;
        if (dt > 1.0 && getenv("GSI_TRACE")) fprintf(stderr, "[alloc] pool %zu bytes %.3f ms\n", bytes, dt);
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            set_error("device memory exhausted");
            return GSI_ERR_OOM;
        }
        if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
        ptrs.push_back(q);
        sizes.push_back(bytes);
        live_fb += bytes;
        note();
        *p = (T *)q;
        return GSI_OK;
    }
    std::vector<size_t> sizes;
    template <typename T>
    gsi_status get(T **p, unsigned long long count) {   // scoped: freed by reset() / at exit
        const size_t bytes = (size_t)std::max<unsigned long long>(count, 1) * sizeof(T);
        const size_t need = (bytes + 255) & ~(size_t)255;
        if (bump && off + need <= top) {
            *p = (T *)(bump + off);
            off += need;
            note();
            return GSI_OK;
        }
        if (bump) demand = std::max(demand, off + need + (cap - top) + live_fb);
        return fallback(p, bytes);
    }
    template <typename T>
    gsi_status get_big(T **p, unsigned long long count) {   // query lifetime
        const size_t bytes = (size_t)std::max<unsigned long long>(count, 1) * sizeof(T);
        const size_t need = (bytes + 255) & ~(size_t)255;
        if (bump && top >= off + need) {
            top -= need;
            *p = (T *)(bump + top);
            note();
            return GSI_OK;
        }
        if (bump) demand = std::max(demand, off + need + (cap - top) + live_fb);
        return fallback(p, bytes);
    }
    size_t mark() const { return off; }
    void reset(size_t m) { off = m; }
    void release(void *p) {
        if (!p || (bump && (char *)p >= bump && (char *)p < bump + cap)) return;   // workspace: reset()
        for (size_t i = 0; i < ptrs.size(); i++)
            if (ptrs[i] == p) {
                cudaFreeAsync(ptrs[i], st);
                ptrs[i] = nullptr;
                live_fb -= sizes[i];
            }
    }
    ~Arena() {
        for (void *q : ptrs)
            if (q) cudaFreeAsync(q, st);
        if (ws_dev >= 0) {
            cudaStreamSynchronize(st);   // nothing in flight may still use the workspace
            Workspace &W = g_ws[ws_dev][ws_slot];
            std::lock_guard<std::mutex> lk(W.mu);
            W.busy = false;
            W.want = std::max(W.want, demand + demand / 8);
            size_t cur = g_ws_want[ws_dev].load();
            while (W.want > cur && !g_ws_want[ws_dev].compare_exchange_weak(cur, W.want)) {
            }
        }
    }
};

struct Prof {
    bool on = false;
    cudaStream_t st = nullptr;
    struct Rec {
        int cls, var;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    uint32_t launches[GSI_N_KCLASS] = {0};
    uint32_t total = 0;
    void begin(int cls, int var = -1) {
        total++;
        launches[cls]++;
        if (!on) return;
        Rec r{cls, var, nullptr, nullptr};
        host_t.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count() - host_base);
        cudaEventCreate(&r.a);
        cudaEventCreate(&r.b);
        cudaEventRecord(r.a, st);
        open_.push_back(recs.size());
        recs.push_back(r);
    }
    void end() {   // closes the innermost open begin() (launches may nest a helper launch)
        if (!on || open_.empty()) return;
        cudaEventRecord(recs[open_.back()].b, st);
        open_.pop_back();
    }
    std::vector<size_t> open_;
    cudaEvent_t base = nullptr;
    double host_base = 0;
    std::vector<double> host_t;   // host time (ms since base) of every begin(), GSI_TRACE
    void start() {
        if (!on) return;
        cudaEventCreate(&base);
        cudaEventRecord(base, st);
        host_base = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    }
    void finish(gsi_stats *s) {
        for (int c = 0; c < GSI_N_KCLASS; c++) {
            s->launches[c] = launches[c];
            s->ms_kernel[c] = 0.f;
        }
        s->total_launches = total;
        if (on && base && getenv("GSI_TRACE")) {   // GPU timeline: kernel class, start, end, gap (ms)
            float prev_end = 0.f;
            for (size_t i = 0; i < recs.size(); i++) {
                float a = 0.f, b = 0.f;
                cudaEventElapsedTime(&a, base, recs[i].a);
                cudaEventElapsedTime(&b, base, recs[i].b);
                fprintf(stderr, "[trace] %3zu cls %d host %.3f start %.3f end %.3f dur %.3f gap %.3f\n", i,
                        recs[i].cls, i < host_t.size() ? host_t[i] : -1.0, a, b, b - a, a - prev_end);
                prev_end = b;
            }
        }
        if (base) cudaEventDestroy(base);
        base = nullptr;
        for (auto &r : recs) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
                s->ms_kernel[r.cls] += ms;
                if (r.var >= 0) s->ms_variant[r.var] += ms;
            } else {
                cudaGetLastError();   // an unrecorded end event must not poison later calls
            }
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        recs.clear();
        open_.clear();
    }
    ~Prof() {
        for (auto &r : recs) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
    }
};

// stream sync with the host wait time accounted in stats.ms_host_sync
cudaError_t sync_timed(gsi_stats &S, cudaStream_t st) {
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = cudaStreamSynchronize(st);
    S.ms_host_sync += (float)std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return e;
}

cudaError_t d2h(gsi_stats &S, void *dst, const void *src, size_t bytes, cudaStream_t st) {
    S.d2h_bytes += bytes;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st);
}
cudaError_t h2d(gsi_stats &S, void *dst, const void *src, size_t bytes, cudaStream_t st) {
    S.h2d_bytes += bytes;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
}

// Keep freed stream-ordered allocations in the device pool (the default release threshold of
// 0 returns them to the driver at every synchronisation, and re-mapping tens of GB per level
// costs far more than the kernels).  Budget = free + reserved-but-unused pool memory.
std::mutex g_pool_mu;
bool g_pool_ready[64] = {false};
void ensure_pool(int dev) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (dev < 0 || dev >= 64 || g_pool_ready[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    // the join tiles use > 48 KB of dynamic shared memory (opt-in, per device)
    cudaFuncSetAttribute(k_join<J_COUNT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxJoinSmem);
    cudaFuncSetAttribute(k_join<J_TABLE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxJoinSmem);
    cudaFuncSetAttribute(k_join<J_NEXT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxJoinSmem);
    cudaFuncSetAttribute(k_join<J_CAHEAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxJoinSmem);
    cudaFuncSetAttribute(k_count_fast<kFastItems>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxJoinSmem);
    cudaFuncSetAttribute(k_small_query, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmallDynSmem);
    cudaFuncSetAttribute(k_filter_tw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)filter_tw_smem(GSI_MAX_K));
    cudaGetLastError();
    g_pool_ready[dev] = true;
}
unsigned long long available_bytes(int dev) {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    cudaMemPool_t pool;
    uint64_t reserved = 0, used = 0;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    }
    cudaGetLastError();
    return (unsigned long long)fr + (reserved > used ? reserved - used : 0);
}

// True if an idle workspace slot of the device already has the size its next query takes
// (taking it then allocates nothing, so it needs no budget).
bool workspace_fits(int dev) {
    if (dev < 0 || dev >= 64) return false;
    for (int k = 0; k < kWsSlots; k++) {
        Workspace &W = g_ws[dev][k];
        std::lock_guard<std::mutex> lk(W.mu);
        if (!W.busy) return W.cap >= std::max(std::max(W.want, g_ws_want[dev].load()), (size_t)64 << 20);
    }
    return false;
}

// A query's default memory budget: 85 % of free device memory, idle workspaces and the
// workspace the query itself holds (own_ws bytes).
unsigned long long device_budget(int dev, size_t own_ws) {
    return (unsigned long long)(0.85 * (double)(available_bytes(dev) + workspace_idle_bytes(dev) + own_ws));
}


// Pinned Counters blocks (the per-level counter read-back of a query): a process-wide
// free list, so host threads that come and go (batch workers) reuse a bounded set instead of
// leaking one page-locked allocation each.  A query holds one block for its lifetime.
std::mutex g_pinned_mu;
struct PinnedBlock {
    Counters c;                                   // per-level counters
    SmallOut so;                                  // the small path's result block
    unsigned long long rb[kCtrWords + GSI_MAX_K];   // the filter's counters and |C(u)|
    unsigned long long pub[GSI_MAX_K + 2];        // filter_publish target (mapped: device-written)
};
std::vector<PinnedBlock *> g_pinned_free;
struct PinnedCounters {
    PinnedBlock *blk = nullptr;   // nullptr if pinned memory is unavailable
    Counters *p = nullptr;        // &blk->c
    unsigned long long *dpub = nullptr;   // device address of blk->pub (mapped), or null
    PinnedCounters() {
        {
            std::lock_guard<std::mutex> lk(g_pinned_mu);
            if (!g_pinned_free.empty()) {
                blk = g_pinned_free.back();
                g_pinned_free.pop_back();
                p = &blk->c;
                map();
                return;
            }
        }
        if (cudaHostAlloc((void **)&blk, sizeof(PinnedBlock), cudaHostAllocMapped | cudaHostAllocPortable) !=
            cudaSuccess) {
            cudaGetLastError();
            blk = nullptr;
        }
        p = blk ? &blk->c : nullptr;
        map();
    }
    void map() {
        if (blk && cudaHostGetDevicePointer((void **)&dpub, blk->pub, 0) != cudaSuccess) {
            cudaGetLastError();
            dpub = nullptr;
        }
    }
    ~PinnedCounters() {
        if (!blk) return;
        std::lock_guard<std::mutex> lk(g_pinned_mu);
        g_pinned_free.push_back(blk);
    }
    PinnedCounters(const PinnedCounters &) = delete;
    PinnedCounters &operator=(const PinnedCounters &) = delete;
};

// Test / A-B switches read per query (never needed in production).
bool env_flag(const char *name) {
    const char *e = getenv(name);
    return e && e[0] == '1';
}

double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

// ------------------------------------------------------------------ prepare --------
gsi_status prepare_impl(const gsi_graph *g, int32_t k, const int32_t *qvl, int32_t qm, const int32_t *qs,
                        const int32_t *qd, const int32_t *qe, gsi_prepared **out) {
    *out = nullptr;
    if (!g || k < 1 || qm < 0 || !qvl || (qm > 0 && (!qs || !qd || !qe))) {
        set_error("invalid query arguments");
        return GSI_ERR_INVALID_ARG;
    }
    if (k > GSI_MAX_K) {
        set_error("query has more than 32 vertices");
        return GSI_ERR_QUERY_TOO_LARGE;
    }
    if (qm > 4 * GSI_MAX_K * GSI_MAX_K) {
        set_error("query has too many edges");
        return GSI_ERR_QUERY_TOO_LARGE;
    }
    for (int u = 0; u < k; u++)
        if (qvl[u] < 0) {
            set_error("negative query vertex label");
            return GSI_ERR_LABEL_RANGE;
        }
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
        for (int f = 0; f < e; f++) {
            bool same = (qs[f] == qs[e] && qd[f] == qd[e]) || (qs[f] == qd[e] && qd[f] == qs[e]);
            if (same && qe[f] == qe[e]) {
                set_error("duplicate query edge");
                return GSI_ERR_DUPLICATE_EDGE;
            }
        }
    }
    // connectivity
    {
        std::vector<int> seen(k, 0), stack{0};
        seen[0] = 1;
        int cnt = 1;
        while (!stack.empty()) {
            int u = stack.back();
            stack.pop_back();
            for (int e = 0; e < qm; e++) {
                int o = qs[e] == u ? qd[e] : (qd[e] == u ? qs[e] : -1);
                if (o >= 0 && !seen[o]) {
                    seen[o] = 1;
                    cnt++;
                    stack.push_back(o);
                }
            }
        }
        if (cnt != k) {
            set_error("query graph is disconnected (PAPER.md L299 assumes connectivity)");
            return GSI_ERR_QUERY_DISCONNECTED;
        }
    }
    auto p = std::make_unique<gsi_prepared>();
    p->g = g;
    p->device = g->device;
    p->k = k;
    p->qvl.assign(qvl, qvl + k);
    p->qs.assign(qs, qs + qm);
    p->qd.assign(qd, qd + qm);
    p->qe.assign(qe, qe + qm);
    p->qe_dense.resize(qm);
    for (int e = 0; e < qm; e++) {
        p->qe_dense[e] = g->dense_label(qe[e]);
        if (p->qe_dense[e] < 0) p->absent_label = true;
    }
    p->qsig.resize((size_t)2 * k * kPlanes);   // [iso signatures | homomorphism signatures]
    encode_query_signatures(k, qvl, qm, qs, qd, qe, p->qsig.data(), 0);
    encode_query_signatures(k, qvl, qm, qs, qd, qe, p->qsig.data() + (size_t)k * kPlanes, 1);
    GSI_CUDA(cudaSetDevice(g->device));
    // stream-ordered allocation: a plain cudaMalloc here would make the driver trim the
    // stream-ordered pool the join levels keep reserved
    GSI_CUDA(cudaMallocAsync(&p->d_qsig, p->qsig.size() * 4, cudaStreamPerThread));
    GSI_CUDA(cudaMemcpyAsync(p->d_qsig, p->qsig.data(), p->qsig.size() * 4, cudaMemcpyHostToDevice,
                             cudaStreamPerThread));
    GSI_CUDA(cudaStreamSynchronize(cudaStreamPerThread));
    *out = p.release();
    return GSI_OK;
}

// ------------------------------------------------------------------ planner --------
// Alg. 2: score(u) = |C(u)| / deg(u); first vertex = argmin; next =
// argmin among unmatched vertices adjacent to Q'; after adding u_c every neighbour's score is
// multiplied by freq(L_E(u_c u')).  Ties go to the smallest query id (reading A8).
static gsi_status plan_order(const gsi_prepared *q, const std::vector<long long> &cand,
                             const int32_t *force_order, std::vector<int> &order) {
    const gsi_graph *g = q->g;
    const int k = q->k, qm = (int)q->qs.size();
    order.clear();
    auto adjacent = [&](int a, int b) {
        for (int e = 0; e < qm; e++)
            if ((q->qs[e] == a && q->qd[e] == b) || (q->qs[e] == b && q->qd[e] == a)) return true;
        return false;
    };
    if (force_order) {
        std::vector<int> seen(k, 0);
        for (int j = 0; j < k; j++) {
            int u = force_order[j];
            if (u < 0 || u >= k || seen[u]) {
                set_error("force_order is not a permutation");
                return GSI_ERR_INVALID_ARG;
            }
            if (j > 0) {
                bool conn = false;
                for (int c = 0; c < j && !conn; c++) conn = adjacent(u, order[c]);
                if (!conn) {
                    set_error("force_order prefix is not connected");
                    return GSI_ERR_INVALID_ARG;
                }
            }
            seen[u] = 1;
            order.push_back(u);
        }
        return GSI_OK;
    }
    std::vector<long long> freq_e(qm);
    for (int e = 0; e < qm; e++) freq_e[e] = q->qe_dense[e] < 0 ? 0ll : g->freq[q->qe_dense[e]];
    order.assign(k, -1);
    if (plan_greedy(k, qm, q->qs.data(), q->qd.data(), freq_e.data(), cand.data(), order.data()) != 0) {
        set_error("query graph is not connected");
        return GSI_ERR_INVALID_ARG;
    }
    return GSI_OK;
}

struct Step {
    int u;                 // query vertex joined at this step
    int t;                 // columns of M before the step
    std::vector<int> col;  // linking edges: column
    std::vector<int> lab;  // dense label
    std::vector<int> rawlab;
    std::vector<int> other;   // query id at the other end
    int paper_e0 = 0;      // index into the edge list (Alg. 4 line 1)
};

static gsi_status build_steps(const gsi_prepared *q, const std::vector<int> &order, const int32_t *force_e0,
                              std::vector<Step> &steps) {
    const gsi_graph *g = q->g;
    const int k = q->k, qm = (int)q->qs.size();
    std::vector<int> pos(k, -1);
    for (int j = 0; j < k; j++) pos[order[j]] = j;
    // a query edge label absent from G (dense label -1) has freq 0 (the query is empty, which
    // run_impl detects after planning; it must not index freq here)
    auto freq_of = [&](int lab) -> long long { return lab < 0 ? 0ll : g->freq[lab]; };
    steps.clear();
    for (int j = 1; j < k; j++) {
        Step s;
        s.u = order[j];
        s.t = j;
        for (int e = 0; e < qm; e++) {
            int o = q->qs[e] == s.u ? q->qd[e] : (q->qd[e] == s.u ? q->qs[e] : -1);
            if (o < 0 || pos[o] >= j) continue;
            s.col.push_back(pos[o]);
            s.lab.push_back(q->qe_dense[e]);
            s.rawlab.push_back(q->qe[e]);
            s.other.push_back(o);
        }
        // e0: min freq(l); ties (min raw label id, min column) (reading A9)
        int best = 0;
        for (size_t e = 1; e < s.col.size(); e++) {
            long long fb = freq_of(s.lab[best]), fe = freq_of(s.lab[e]);
            if (fe < fb || (fe == fb && (s.rawlab[e] < s.rawlab[best] ||
                                         (s.rawlab[e] == s.rawlab[best] && s.col[e] < s.col[best]))))
                best = (int)e;
        }
        if (force_e0 && force_e0[j] >= 0) {
            int f = -1;
            for (size_t e = 0; e < s.col.size(); e++)
                if (s.other[e] == force_e0[j] && (f < 0 || freq_of(s.lab[e]) < freq_of(s.lab[f]))) f = (int)e;
            if (f < 0) {
                set_error("force_first_edge names a vertex not linked to the joined vertex");
                return GSI_ERR_INVALID_ARG;
            }
            best = f;
        }
        s.paper_e0 = best;
        steps.push_back(std::move(s));
    }
    return GSI_OK;
}

// ------------------------------------------------------------------ run -----------
// One query = filter -> plan -> level 1 -> recursive levels.  A level whose Prealloc bound
// |GBA| exceeds the chunk capacity is processed as consecutive slot ranges, each carried
// depth-first to the last level (the bound F is exact before the join runs, so the chunk
// sizes are known in advance; memory <= depth x chunk).  Chunks are taken in slot order,
// so the concatenated output keeps the 1-GPU row order.  Sharding cuts
// the slot range of one level by F into W contiguous pieces; rank r keeps piece r.
namespace {

struct QueryCtx {
    const gsi_graph *g = nullptr;
    const gsi_prepared *q = nullptr;
    gsi_query_opts opts;
    cudaStream_t st = nullptr;
    Arena *A = nullptr;
    Prof *prof = nullptr;
    Counters *ctr = nullptr;
    Counters *pinned = nullptr;   // host read-back block of this query (nullptr: pageable)
    gsi_stats *S = nullptr;
    const uint32_t *bm = nullptr;
    long long words = 0;
    std::vector<Step> steps;
    std::vector<int> order, pos_of_q;
    int W = 1, rank = 0;
    bool sharded = true;
    bool force_shared = false;   // test hook: the shared-run paths at any size (opts.force_paths & 1)
    unsigned long long shard_min = 65536;
    unsigned long long cap_slots = 0;
    double deadline = 0;
    bool capped = false;
    unsigned long long count = 0, fp1 = 0, fp2 = 0;
    std::vector<std::pair<int32_t *, unsigned long long>> pieces;   // final table pieces (device)
    TableVM *tv = nullptr;                                           // the table, grown in place (vm.cu)
    std::vector<std::pair<uint32_t *, int32_t *>> filt;             // per step: (fpos, fci) or null
    std::vector<Loc *> pa;                                           // per step: probe-ahead table or null
    std::vector<ulonglong2 *> fpt;                                   // per step: fingerprint term table or null
    std::vector<char> lean_off;                                      // per step: lean J_NEXT left too many holes
    // Zeroed once per query; every level launch takes a never-used slice for its counters and
    // look-back status words (saves a memset per level on the small-query critical path).
    unsigned long long *zpool = nullptr;
    unsigned long long zcap = 0, zoff = 0;
    // Stored columns.  Count-only mode stores in M_t only the columns a later step reads (its
    // linking columns and subtraction columns); phys[t][c] = position of logical column c in
    // a row of M_t (-1: dropped), width[t] = stored columns.  Table / fingerprint: all.
    std::vector<std::vector<int>> phys;
    std::vector<int> width;
};

// The next `rows` rows of the final table: in place at the end of the growing table (VMM), or
// a separate piece concatenated at the end when VMM is unavailable.
gsi_status table_rows(QueryCtx &C, unsigned long long rows, int32_t **dst) {
    if (C.tv) {
        *dst = C.tv->append(rows);
        return *dst ? GSI_OK : GSI_ERR_OOM;
    }
    if (cudaMallocAsync(dst, 4ull * rows * C.q->k, C.st) != cudaSuccess) {
        cudaGetLastError();
        set_error("table of " + std::to_string(rows) + " rows does not fit in device memory");
        return GSI_ERR_OOM;
    }
    C.pieces.push_back({*dst, rows});
    return GSI_OK;
}

gsi_status table_put(QueryCtx &C, const int32_t *src, unsigned long long rows) {
    int32_t *dst = nullptr;
    GSI_TRY(table_rows(C, rows, &dst));
    GSI_CUDA(cudaMemcpyAsync(dst, src, 4ull * rows * C.q->k, cudaMemcpyDeviceToDevice, C.st));
    return GSI_OK;
}

// Columns of M a step reads: linking columns and (isomorphism) the subtraction columns, i.e.
// the earlier columns with u's vertex label that are not linked (x in N(m[c],l) => x != m[c]).
static void step_reads(const QueryCtx &C, const Step &s, std::vector<int> &cols) {
    cols.assign(s.col.begin(), s.col.end());
    if (C.opts.homomorphism) return;
    for (int c = 0; c < s.t; c++) {
        if (C.q->qvl[C.order[c]] != C.q->qvl[s.u]) continue;
        bool linked = false;
        for (int lc : s.col) linked |= lc == c;
        if (!linked) cols.push_back(c);
    }
}

void plan_layout(QueryCtx &C, bool project) {
    const int k = C.q->k;
    C.phys.assign(k + 1, std::vector<int>(k + 1, -1));
    C.width.assign(k + 1, 0);
    std::vector<int> need(k + 1, 0);   // need[c] = largest step t (columns before it) reading c
    std::vector<int> cols;
    for (auto &s : C.steps) {
        step_reads(C, s, cols);
        for (int c : cols) need[c] = std::max(need[c], s.t);
    }
    for (int t = 1; t <= k; t++) {
        int w = 0;
        for (int c = 0; c < t; c++)
            if (!project || need[c] >= t) C.phys[t][c] = w++;
        C.width[t] = w;
    }
}

// Logical column c of a row of M_{lt+1} = m ‖ x read through M_lt's layout: x (c == lt) is
// the sentinel width[lt] ("the vertex being added"), others their stored position.
static int to_phys(const QueryCtx &C, int lt, int c) {
    return c == lt ? C.width[lt] : C.phys[lt][c];
}

void fill_params(QueryCtx &C, const Step &s, StepParams &P, int lt) {
    const gsi_graph *g = C.g;
    std::memset(&P, 0, sizeof(P));
    const int E = (int)s.col.size();
    P.t = s.t;
    P.E = E;
    P.k = C.q->k;
    P.per_row_e0 = C.opts.e0_mode == 0 ? 1 : 0;
    for (int qv = 0; qv < C.q->k; qv++) P.pos_of_q[qv] = C.pos_of_q[qv];
    P.fp = C.opts.fingerprint != 0;
    P.stage_base = GSI_STAGE_BASE;
    std::vector<int> eorder(E);
    for (int e = 0; e < E; e++) eorder[e] = e;
    std::swap(eorder[0], eorder[s.paper_e0]);   // paper mode: e0 first (Alg. 3 line 9)
    for (int e = 0; e < E; e++) {
        int src = eorder[e];
        P.col[e] = s.col[src];
        P.lab[e] = (uint32_t)s.lab[src];
        P.gbase[e] = (unsigned long long)g->gbase[s.lab[src]];
        P.ngroups[e] = g->ngroups[s.lab[src]];
    }
    P.n_inj = 0;
    if (!C.opts.homomorphism) {
        for (int c = 0; c < s.t; c++) {
            if (C.q->qvl[C.order[c]] != C.q->qvl[s.u]) continue;   // different label: C(u) excludes it
            bool linked = false;
            for (int e = 0; e < E; e++) linked |= P.col[e] == c;    // x in N(m[c],l) => x != m[c]
            if (!linked) P.inj_col[P.n_inj++] = c;
        }
    }
    P.stage_inj = P.stage_base ? std::min(P.n_inj, GSI_STAGE_INJ) : 0;
    // columns in the layout of M_lt (lt = s.t: this step's own level; lt = s.t - 1: the step
    // seen from the level before it, where its column s.t - 1 is that level's new vertex)
    P.t = C.width[lt];
    for (int e = 0; e < E; e++) P.col[e] = to_phys(C, lt, P.col[e]);
    for (int c = 0; c < P.n_inj; c++) P.inj_col[c] = to_phys(C, lt, P.inj_col[c]);
    // the row this step produces (J_NEXT): the columns M_{s.t+1} stores
    P.out_w = 0;
    if (lt == s.t && s.t + 1 <= C.q->k) {
        for (int c = 0; c <= s.t; c++)
            if (C.phys[s.t + 1][c] >= 0) P.out_src[P.out_w++] = c < s.t ? C.phys[s.t][c] : -1;
    }
}

// Build (once per query step) N(v,l0) ∩ C(u) for every run of P(G,l0): fpos + fci.
gsi_status ensure_filtered(QueryCtx &C, size_t si, uint32_t lab) {
    if (C.filt.size() < C.steps.size()) C.filt.assign(C.steps.size(), {nullptr, nullptr});
    if (C.filt[si].first) return GSI_OK;
    const gsi_graph *g = C.g;
    Arena &A = *C.A;
    cudaStream_t st = C.st;
    const uint32_t lo = g->ci_lo[lab], hi = g->ci_lo[lab + 1];
    uint32_t *fpos = nullptr;
    int32_t *fci = nullptr;
    GSI_TRY(A.get_big(&fpos, (unsigned long long)(hi - lo) + 1));
    GSI_TRY(A.get_big(&fci, (unsigned long long)(hi - lo)));
    const unsigned ft = grid_for(hi - lo, GSI_FP_ITEMS * kThreads);
    unsigned long long *fst = nullptr;
    GSI_TRY(A.get_big(&fst, (unsigned long long)ft + 1));
    GSI_CUDA(cudaMemsetAsync(fst, 0, 8ull * (ft + 1), st));
    const uint32_t *cu0 = C.bm + (long long)C.steps[si].u * C.words;
    C.prof->begin(GSI_K_OTHER, GSI_V_FILTER_PARTITION);
    C.S->variant_launches[GSI_V_FILTER_PARTITION]++;
    k_filter_partition<<<ft, kThreads, 0, st>>>(g->ci, lo, hi, cu0, fpos, fci, fst + 1, (unsigned *)fst);
    C.prof->end();
    C.S->alg_bytes[GSI_K_OTHER] += 12.0 * (hi - lo);
    C.S->alg_bytes_variant[GSI_V_FILTER_PARTITION] += 12.0 * (hi - lo);
    C.filt[si] = {fpos, fci};
    return GSI_OK;
}

// Probe-ahead table of step si (on shared lists; its next step links to the vertex it adds).
gsi_status ensure_probe_ahead(QueryCtx &C, size_t si, const StepParams &P, const StepParams &P2) {
    if (C.pa.size() < C.steps.size()) C.pa.assign(C.steps.size(), nullptr);
    if (C.pa[si]) return GSI_OK;
    const gsi_graph *g = C.g;
    const uint32_t lo = g->ci_lo[P.lab[0]], hi = g->ci_lo[P.lab[0] + 1];
    Loc *pa = nullptr;
    GSI_TRY(C.A->get_big(&pa, (unsigned long long)(hi - lo)));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
    const unsigned grid = std::min<unsigned>(grid_for(hi - lo, 4 * kThreads), (unsigned)sms * 8);
    C.prof->begin(GSI_K_OTHER, GSI_V_PROBE_AHEAD);
    C.S->variant_launches[GSI_V_PROBE_AHEAD]++;
    k_probe_ahead<<<grid, kThreads, 0, C.st>>>(C.filt[si].second, C.filt[si].first + (hi - lo), P2, g->groups,
                                               g->gpn, pa);
    C.prof->end();
    // read x, one PCSR sector + two fpos words per candidate, 8 B entry write
    C.S->alg_bytes[GSI_K_OTHER] += 52.0 * (hi - lo);
    C.S->alg_bytes_variant[GSI_V_PROBE_AHEAD] += 52.0 * (hi - lo);
    C.pa[si] = pa;
    return GSI_OK;
}

// Fingerprint terms of step si's shared run array (k_fp_terms), once per query.
gsi_status ensure_fp_terms(QueryCtx &C, size_t si) {
    if (C.fpt.size() < C.steps.size()) C.fpt.assign(C.steps.size(), nullptr);
    if (C.fpt[si]) return GSI_OK;
    const gsi_graph *g = C.g;
    const Step &s = C.steps[si];
    const uint32_t lab = (uint32_t)s.lab[0];
    const uint32_t lo = g->ci_lo[lab], hi = g->ci_lo[lab + 1];
    ulonglong2 *T = nullptr;
    GSI_TRY(C.A->get_big(&T, (unsigned long long)(hi - lo)));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
    const unsigned grid = std::min<unsigned>(grid_for(hi - lo, kThreads), (unsigned)sms * 8);
    C.prof->begin(GSI_K_OTHER, GSI_V_FP_TERMS);
    C.S->variant_launches[GSI_V_FP_TERMS]++;
    k_fp_terms<<<grid, kThreads, 0, C.st>>>(C.filt[si].second, C.filt[si].first + (hi - lo), s.u, T);
    C.prof->end();
    C.S->alg_bytes[GSI_K_OTHER] += 20.0 * (hi - lo);
    C.S->alg_bytes_variant[GSI_V_FP_TERMS] += 20.0 * (hi - lo);
    C.fpt[si] = T;
    return GSI_OK;
}

bool shared_lists_allowed(const QueryCtx &C, const StepParams &P) {
    return GSI_PREFILTER_RATIO > 0 && !C.opts.no_shared_lists && C.opts.e0_mode == 0 && P.E == 1;
}

// F for rows whose producer skipped it (it expected the warp count-ahead, which needs none).
gsi_status build_F(QueryCtx &C, const Loc *loc, unsigned long long nM, int E, unsigned long long **F) {
    const unsigned rt = grid_for(nM, kThreads);
    unsigned long long *rst = nullptr;
    GSI_TRY(C.A->get(F, nM + 1));
    GSI_TRY(C.A->get(&rst, (unsigned long long)rt + 1));
    GSI_CUDA(cudaMemsetAsync(rst, 0, 8ull * (rt + 1), C.st));
    C.prof->begin(GSI_K_OTHER);
    k_lens_scan<<<rt, kThreads, 0, C.st>>>(loc, (long long)nM, E, *F, rst + 1, (unsigned *)rst);
    C.prof->end();
    C.S->alg_bytes[GSI_K_OTHER] += 16.0 * nM;
    return GSI_OK;
}

bool cahead_warp_enabled() { return GSI_CAHEAD_WARP && !env_flag("GSI_CAHEAD_TILE"); }

// The warp count-ahead has the closed-form shape (k_cahead_lean): the last step links to a
// parent column, the vertex this step adds is not one of its subtraction columns, one linking
// edge here and at most one subtraction column.
bool cahead_lean(const QueryCtx &C, const StepParams &P, const StepParams &P2) {
    (void)C;
    bool xinj = false;
    for (int c = 0; c < P2.n_inj; c++) xinj |= P2.inj_col[c] >= P.t;
    return GSI_CAHEAD_LEAN && !env_flag("GSI_CAHEAD_NOLEAN") && P2.col[0] < P.t && !xinj && P.E == 1 &&
           P.n_inj <= 1;
}

// The last level of an enumerating count on shared runs is walked row-wise by the lean warp
// kernel (no F, holes allowed).
bool final_walks_rows(const QueryCtx &C, const StepParams &P, int mode) {
    return mode == J_COUNT && GSI_COUNT_LEAN && !env_flag("GSI_COUNT_NOLEAN") && P.prefiltered && P.E == 1 &&
           P.n_inj <= kLeanInj && cahead_warp_enabled();
}

// The last level of a table query on shared runs is written by the warp table kernel: one
// linking edge, at most one subtraction column, rows narrow enough for its staging tile.
bool final_writes_rows(const QueryCtx &C, const StepParams &P) {
    return GSI_TABLE_LEAN && !env_flag("GSI_TABLE_NOLEAN") && P.prefiltered && P.E == 1 && P.n_inj <= kLeanInj &&
           C.q->k <= kTabMaxK;
}

// Rows [r0, r1) of the last level of a table query (final_writes_rows): survivors per row and
// their offsets (k_surv_scan), then every match written straight into the result's table piece
// (k_final_table) — no upper-bound buffer, no compaction copy.
gsi_status final_table(QueryCtx &C, size_t si, const int32_t *M, long long r0, long long r1, const Loc *loc,
                       const StepParams &P, const int32_t *cip) {
    gsi_stats &S = *C.S;
    Arena &A = *C.A;
    cudaStream_t st = C.st;
    const int k = C.q->k;
    const unsigned long long nrows = (unsigned long long)(r1 - r0);
    if (nrows == 0) return GSI_OK;
    if (C.deadline > 0 && now_ms() > C.deadline) {
        C.capped = true;
        return GSI_OK;
    }
    const size_t mk = A.mark();
    const unsigned rt = grid_for(nrows, kThreads);
    unsigned long long *O = nullptr, *rst = nullptr;
    GSI_TRY(A.get(&O, nrows + 1));
    GSI_TRY(A.get(&rst, (unsigned long long)rt + 1));
    GSI_CUDA(cudaMemsetAsync(rst, 0, 8ull * (rt + 1), st));
    C.prof->begin(GSI_K_OTHER, GSI_V_SURV_SCAN);
    S.variant_launches[GSI_V_SURV_SCAN]++;
    if (P.n_inj == 0)
        k_surv_scan<0><<<rt, kThreads, 0, st>>>(M, r0, (long long)nrows, loc, P, cip, O, rst + 1, (unsigned *)rst);
    else
        k_surv_scan<1><<<rt, kThreads, 0, st>>>(M, r0, (long long)nrows, loc, P, cip, O, rst + 1, (unsigned *)rst);
    C.prof->end();
    S.alg_bytes_variant[GSI_V_SURV_SCAN] += 16.0 * nrows;   // loc read + O write
    S.alg_bytes[GSI_K_OTHER] += 16.0 * nrows;
    unsigned long long total = 0;
    GSI_CUDA(d2h(S, &total, O + nrows, 8, st));
    GSI_CUDA(sync_timed(S, st));
    if (total) {
        int32_t *piece = nullptr;
        {
            const gsi_status rs = table_rows(C, total, &piece);
            if (rs != GSI_OK) {
                A.reset(mk);
                return rs;
            }
        }
        Counters *lctr = nullptr;
        GSI_TRY(A.get(&lctr, 1));
        GSI_CUDA(cudaMemsetAsync(lctr, 0, sizeof(Counters), st));
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, C.g->device);
        const unsigned long long units = (nrows + 31) / 32;
        const unsigned wg = (unsigned)std::max<unsigned long long>(
            1, std::min<unsigned long long>((units + 7) / 8, (unsigned long long)sms * 8));
        C.prof->begin(GSI_K_JOIN, GSI_V_FINAL_TABLE);
        S.variant_launches[GSI_V_FINAL_TABLE]++;
        if (P.fp) {
            if (P.n_inj == 0) k_final_table<0, true><<<wg, kThreads, 0, st>>>(M, r0, r1, loc, O, P, cip, piece, lctr);
            else k_final_table<kLeanInj, true><<<wg, kThreads, 0, st>>>(M, r0, r1, loc, O, P, cip, piece, lctr);
        } else {
            if (P.n_inj == 0) k_final_table<0, false><<<wg, kThreads, 0, st>>>(M, r0, r1, loc, O, P, cip, piece, lctr);
            else k_final_table<kLeanInj, false><<<wg, kThreads, 0, st>>>(M, r0, r1, loc, O, P, cip, piece, lctr);
        }
        C.prof->end();
        GSI_CUDA(cudaGetLastError());
        // algorithmic bytes: the rows it extends (row + loc + O) and every byte it writes
        const double jb = (4.0 * P.t + 16.0) * (double)nrows + 4.0 * k * (double)total;
        S.alg_bytes_variant[GSI_V_FINAL_TABLE] += jb;
        S.items_variant[GSI_V_FINAL_TABLE] += total;
        S.alg_bytes[GSI_K_JOIN] += jb;
        if (P.fp) {
            Counters hc;
            GSI_CUDA(d2h(S, &hc, lctr, sizeof(Counters), st));
            GSI_CUDA(sync_timed(S, st));
            C.fp1 += hc.fp1;
            C.fp2 ^= hc.fp2;
        }
    }
    const int t = C.steps[si].t;
    C.count += total;
    S.rows[t] += total;
    if (S.levels < t + 1) S.levels = t + 1;
    A.reset(mk);
    return GSI_OK;
}

// The level after step si will walk its rows without F (the warp count-ahead, or the lean last
// level), so step si may skip F' and write its rows at their Prealloc slots.
bool next_walks_rows(const QueryCtx &C, size_t si, bool pf_next) {
    if (!pf_next || !C.sharded || C.opts.want_table || C.opts.e0_mode != 0 || C.opts.no_shared_lists ||
        !cahead_warp_enabled())
        return false;
    const size_t nl = si + 1;
    if (nl + 2 == C.steps.size())
        return !C.opts.no_count_ahead && !C.opts.fingerprint && C.steps[nl + 1].col.size() == 1;
    if (nl + 1 == C.steps.size()) return GSI_COUNT_LEAN && !env_flag("GSI_COUNT_NOLEAN") && C.steps[nl].col.size() == 1;
    return false;
}

// Level t = steps[si].t: M (nM x t) with its Prealloc (loc, F, |GBA| = gba) already computed
// (by k_probe for level 1, by the previous level's fused kernel otherwise).
gsi_status level(QueryCtx &C, size_t si, int32_t *M, unsigned long long nM, Loc *loc, unsigned long long *F,
                 unsigned long long gba, unsigned long long active, unsigned long long elems, bool filtered_in) {
    // (gba / active / elems are updated below if this level switches to shared candidate lists)
    const Step &s = C.steps[si];
    const int t = s.t;
    const bool last = si + 1 == C.steps.size();
    gsi_stats &S = *C.S;
    Arena &A = *C.A;
    Prof &prof = *C.prof;
    cudaStream_t st = C.st;
    const gsi_graph *g = C.g;
    StepParams P, P2;
    fill_params(C, s, P, t);
    if (!last) fill_params(C, C.steps[si + 1], P2, t);
    else std::memset(&P2, 0, sizeof(P2));
    const int E = P.E;
    if (S.levels < t) S.levels = t;
    S.gba[t] += gba;
    S.list_elems[t] += elems;
    if (nM == 0 || gba == 0) return GSI_OK;

    // ---- shared candidate lists: N(v,l0) ∩ C(u) once per partition run ----
    const int32_t *cip = g->ci;
    if (filtered_in) {   // the previous level's probe-ahead already pointed the rows at them
        P.prefiltered = 1;
        cip = C.filt[si].second;
    } else if (shared_lists_allowed(C, P)) {
        const uint32_t lo = g->ci_lo[P.lab[0]], hi = g->ci_lo[P.lab[0] + 1];
        if (hi > lo && (C.force_shared || gba >= (unsigned long long)GSI_PREFILTER_RATIO * (hi - lo))) {
            GSI_TRY(ensure_filtered(C, si, P.lab[0]));
            const unsigned rt = grid_for(nM, kThreads);
            unsigned long long *rst = nullptr;
            GSI_TRY(A.get(&rst, (unsigned long long)rt + 1 + sizeof(Counters) / 8));
            GSI_CUDA(cudaMemsetAsync(rst, 0, 8ull * (rt + 1) + sizeof(Counters), st));
            Counters *rctr = reinterpret_cast<Counters *>(rst + rt + 1);
            prof.begin(GSI_K_OTHER, GSI_V_REFILTER);
            S.variant_launches[GSI_V_REFILTER]++;
            k_refilter<<<rt, kThreads, 0, st>>>(loc, (long long)nM, C.filt[si].first, lo, hi, F, rst + 1,
                                                (unsigned *)rst, rctr);
            prof.end();
            S.alg_bytes_variant[GSI_V_REFILTER] += 32.0 * nM;   // loc read + write, two fpos words, F
            S.alg_bytes[GSI_K_OTHER] += 32.0 * nM;
            Counters hc0;
            GSI_CUDA(d2h(S, &gba, F + nM, 8, st));
            GSI_CUDA(d2h(S, &hc0, rctr, sizeof(Counters), st));
            GSI_CUDA(sync_timed(S, st));
            active = hc0.active_rows;
            elems = hc0.list_elems;
            P.prefiltered = 1;
            cip = C.filt[si].second;
            if (gba == 0) return GSI_OK;
        }
    }
    if (P.prefiltered) S.n_shared_lists++;

    // ---- count-ahead: the last step has one linking edge and only the count is wanted, so
    // this level counts the extensions of its survivors on the last step's shared lists ----
    bool cahead = false;
    if (!last && si + 2 == C.steps.size() && !C.opts.want_table && !C.opts.fingerprint &&
        !C.opts.no_count_ahead && shared_lists_allowed(C, P2)) {
        const uint32_t lo2 = g->ci_lo[P2.lab[0]], hi2 = g->ci_lo[P2.lab[0] + 1];
        cahead = hi2 > lo2 && ((C.filt.size() > si + 1 && C.filt[si + 1].first) ||
                               C.force_shared || gba * (unsigned long long)GSI_PREFILTER_AHEAD >= (unsigned long long)(hi2 - lo2));
    }

    // rows without F (see no_f2): build it unless the warp count-ahead consumes them as they are
    {
        StepParams Pl = P;   // (the last level's lean walk needs no F either)
        const bool walker = (cahead && P.prefiltered && cahead_warp_enabled()) ||
                            (last && !C.opts.want_table && final_walks_rows(C, Pl, J_COUNT));
        if (!F && (!walker || !C.sharded)) GSI_TRY(build_F(C, loc, nM, E, &F));
    }

    // ---- shard this level's slot range ----
    // W ranks x `pieces` equal slot pieces at row granularity; rank r keeps pieces r, r + W,
    // r + 2W, ... (pieces = 1: one contiguous F-weighted range, the 1-GPU row order when the
    // shards are concatenated in rank order; pieces > 1 interleave, so a query whose work is
    // concentrated in part of the level still splits evenly).
    struct Piece {
        unsigned long long s0, s1;
        long long r0, r1;
    };
    std::vector<Piece> pieces{{0ull, gba, 0ll, (long long)nM}};
    if (!C.sharded && (nM >= C.shard_min || gba > C.cap_slots || last || cahead)) {
        const int per = std::max(1, (int)C.opts.shard_pieces);
        const int NP = C.W * per;
        long long *bounds = nullptr;
        GSI_TRY(A.get(&bounds, 2ull * (NP + 1)));
        prof.begin(GSI_K_OTHER);
        k_shard_bounds<<<grid_for((unsigned long long)NP + 1, kThreads), kThreads, 0, st>>>(F, (long long)nM, NP,
                                                                                            bounds);
        prof.end();
        std::vector<long long> hb(2 * (NP + 1));
        GSI_CUDA(d2h(S, hb.data(), bounds, 8ull * hb.size(), st));
        GSI_CUDA(sync_timed(S, st));
        A.release(bounds);
        pieces.clear();
        for (int j = C.rank; j < NP; j += C.W)
            pieces.push_back({(unsigned long long)hb[NP + 1 + j], (unsigned long long)hb[NP + 1 + j + 1], hb[j],
                              hb[j + 1]});
        S.shard_level = t;
        S.shard_row_begin = (uint64_t)pieces.front().r0;
        S.shard_row_end = (uint64_t)pieces.back().r1;
        C.sharded = true;
    }

    const int mode = cahead ? J_CAHEAD : (!last ? J_NEXT : (C.opts.want_table ? J_TABLE : J_COUNT));
    const uint32_t *cu = C.bm + (long long)s.u * C.words;
    gsi_status rc = GSI_OK;
    for (const Piece &pc : pieces) {
    const unsigned long long s0 = pc.s0, s1 = pc.s1;
    const long long r_lo = pc.r0, r_hi = pc.r1;
    if (mode == J_TABLE && final_writes_rows(C, P)) {
        rc = final_table(C, si, M, r_lo, r_hi, loc, P, cip);
        if (rc != GSI_OK) break;
        continue;
    }
    const unsigned long long chunk = (mode == J_COUNT || mode == J_CAHEAD)
                                         ? std::max<unsigned long long>(s1 - s0, 1)
                                         : std::max<unsigned long long>(C.cap_slots, kJoinTile);
    for (unsigned long long c0 = s0; c0 < s1 && rc == GSI_OK; c0 += chunk) {
        if (C.deadline > 0 && now_ms() > C.deadline) {
            C.capped = true;
            break;
        }
        const size_t mk = A.mark();
        const unsigned long long c1 = std::min(s1, c0 + chunk), slots = c1 - c0;
        if (c0 != s0 || c1 != s1) S.n_chunks++;
        const bool fast = GSI_FAST_ITEMS > 0 && mode == J_COUNT && P.prefiltered && !P.fp && P.E == 1;
        const unsigned tile_slots = (unsigned)((fast ? kFastItems : join_items(mode)) * kThreads);
        const unsigned jt = grid_for(slots, tile_slots);
        // one zeroed scratch region per launch: [Counters | tile counter + status 1 | status 2]
        constexpr unsigned kCtrWords = sizeof(Counters) / 8;
        unsigned long long *status = nullptr;
        const unsigned long long swords = kCtrWords + 2ull * jt + 2;
        const bool zslice = C.zoff + swords <= C.zcap;
        if (zslice) {   // a fresh slice of the query's pre-zeroed pool
            status = C.zpool + C.zoff;
            C.zoff += (swords + 3) & ~3ull;
        } else {
            GSI_TRY(A.get(&status, swords));
            GSI_CUDA(cudaMemsetAsync(status, 0, 8ull * swords, st));
        }
        Counters *lctr = reinterpret_cast<Counters *>(status);
        unsigned *tctr = (unsigned *)(status + kCtrWords);
        unsigned long long *st1 = status + kCtrWords + 1, *st2 = status + kCtrWords + 2 + jt;
        int32_t *out = nullptr;
        Loc *loc2 = nullptr;
        unsigned long long *F2 = nullptr;
        if (mode == J_TABLE) GSI_TRY(A.get(&out, slots * (unsigned long long)C.q->k));
        if (mode == J_NEXT) {
            GSI_TRY(A.get(&out, slots * (unsigned long long)std::max(P.out_w, 1)));
            GSI_TRY(A.get(&loc2, slots * (unsigned long long)P2.E));
            // F2[0..nout] written by the kernel (allocated below unless skipped)
        }
        // next step on shared lists? (its rows are produced here, so the probe-ahead can point
        // them at N(v,l0') ∩ C(u') directly and drop rows whose filtered run is empty)
        bool pf_next = false;
        if (mode == J_CAHEAD) {
            GSI_TRY(ensure_filtered(C, si + 1, P2.lab[0]));
            P2.prefiltered = 1;
            P2.fpos = C.filt[si + 1].first;
            P2.flo = g->ci_lo[P2.lab[0]];
            P2.fhi = g->ci_lo[P2.lab[0] + 1];
            P2.fci = C.filt[si + 1].second;
            P2.cu = C.bm + (long long)C.steps[si + 1].u * C.words;
        } else if (mode == J_NEXT && shared_lists_allowed(C, P2)) {
            const uint32_t lo2 = g->ci_lo[P2.lab[0]], hi2 = g->ci_lo[P2.lab[0] + 1];
            if (hi2 > lo2 && (C.filt.size() > si + 1 && C.filt[si + 1].first ||
                              C.force_shared || slots * (unsigned long long)GSI_PREFILTER_AHEAD >= (unsigned long long)(hi2 - lo2))) {
                GSI_TRY(ensure_filtered(C, si + 1, P2.lab[0]));
                P2.prefiltered = 1;
                P2.fpos = C.filt[si + 1].first;
                P2.flo = lo2;
                P2.fhi = hi2;
                pf_next = true;
            } else {
                P2.prefiltered = 0;
            }
        }
        // probe-ahead: the next step links to the vertex this step adds, and this level's rows
        // re-scan its candidate runs often enough to pay one probe per candidate
        P.pa = nullptr;
        if ((mode == J_NEXT || mode == J_CAHEAD) && P.prefiltered && P2.prefiltered && P2.E == 1 &&
            P2.col[0] == P.t && GSI_PROBE_AHEAD > 0) {
            const uint32_t plo = g->ci_lo[P.lab[0]], phi = g->ci_lo[P.lab[0] + 1];
            if ((C.pa.size() > si && C.pa[si]) ||
                C.force_shared || slots >= (unsigned long long)GSI_PROBE_AHEAD * (unsigned long long)(phi - plo)) {
                GSI_TRY(ensure_probe_ahead(C, si, P, P2));
                P.pa = C.pa[si];
                S.n_probe_ahead++;
            }
        }
        // the next step's run is row-constant: locate it once per tile row
        P.stage_next = mode == J_NEXT && P2.E == 1 && P2.col[0] < P.t && GSI_STAGE_NEXT;
        // the next level is the count-ahead level on shared lists, walked by the warp kernel
        // (no F needed): skip F' and its look-back chain
        P.no_f2 = mode == J_NEXT && next_walks_rows(C, si, pf_next) ? 1 : 0;
        // lean J_NEXT: count-only, one linking edge here and in the next step (on shared runs),
        // and the next level is the warp count-ahead, which walks rows with holes at no cost
        // (a deeper level would pay for them: more rows, and an F to build)
        if (C.lean_off.size() < C.steps.size()) C.lean_off.assign(C.steps.size(), 0);
        const bool lean_next = P.no_f2 && GSI_NEXT_LEAN && !env_flag("GSI_NEXT_NOLEAN") && P.E == 1 && P2.E == 1 &&
                               P.n_inj <= 1 && !C.lean_off[si];
        const bool warp_ca = mode == J_CAHEAD && P.prefiltered && cahead_warp_enabled();
        const bool final_lean = final_walks_rows(C, P, mode);
        uint32_t *rowmap = nullptr;
        // first/last row of every slot tile (the warp kernels walk rows; a single tile scans
        // the level's rows itself, which saves a launch per small level)
        if (!warp_ca && !lean_next && !final_lean && (jt > 1 || nM > 2048)) {
            GSI_TRY(A.get(&rowmap, (unsigned long long)jt + 1));
            prof.begin(GSI_K_OTHER);
            k_tile_rows<<<grid_for((unsigned long long)jt + 1, kThreads), kThreads, 0, st>>>(F, (long long)nM, c0, c1, jt,
                                                                                           tile_slots, rowmap);
            prof.end();
        }
        if (mode == J_NEXT && !P.no_f2 && !lean_next) GSI_TRY(A.get(&F2, slots + 1));
        uint32_t *rows2 = nullptr;
        if (lean_next) {   // the rows holding slots c0 and c1 - 1
            GSI_TRY(A.get(&rows2, 2));
            prof.begin(GSI_K_OTHER);
            k_tile_rows<<<1, 32, 0, st>>>(F, (long long)nM, c0, c1, 1, (unsigned)std::min<unsigned long long>(slots, 0xFFFFFFFFull), rows2);
            prof.end();
        }
        Counters hc_local;
        int var;
        {
            int v;
            if (lean_next) v = GSI_V_NEXT_LEAN;
            else if (warp_ca) v = cahead_lean(C, P, P2) ? GSI_V_CAHEAD_LEAN : GSI_V_CAHEAD_WARP;
            else if (final_lean) v = P.fp ? GSI_V_FINAL_FP : GSI_V_FINAL_LEAN;
            else if (fast) v = GSI_V_COUNT_FAST;
            else if (mode == J_COUNT) v = GSI_V_JOIN_COUNT;
            else if (mode == J_CAHEAD) v = GSI_V_JOIN_CAHEAD;
            else if (mode == J_TABLE) v = GSI_V_JOIN_TABLE;
            else v = GSI_V_JOIN_NEXT;
            S.variant_launches[v]++;
            var = v;
        }
        // the enumerating last level's fingerprint terms (built once per query, before the launch)
        const ulonglong2 *fpT = nullptr;
        if (final_lean && P.fp && GSI_FP_TERMS && !env_flag("GSI_FP_NOTERMS") && C.filt.size() > si &&
            cip == C.filt[si].second) {
            GSI_TRY(ensure_fp_terms(C, si));
            fpT = C.fpt[si];
        }
        prof.begin(GSI_K_JOIN, var);
        if (lean_next) {
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
            const unsigned wg = (unsigned)std::max<unsigned long long>(
                1, std::min<unsigned long long>((slots + kThreads - 1) / kThreads, (unsigned long long)sms * 4));
            if (P.n_inj == 0)
                k_next_lean<0><<<wg, kThreads, 0, st>>>(M, rows2, loc, F, c0, c1, P, P2, cip, cu, g->groups, g->gpn, out,
                                                        loc2, lctr);
            else
                k_next_lean<1><<<wg, kThreads, 0, st>>>(M, rows2, loc, F, c0, c1, P, P2, cip, cu, g->groups, g->gpn, out,
                                                        loc2, lctr);
        } else if (warp_ca) {
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
            const unsigned long long units = ((unsigned long long)(r_hi - r_lo) + 31) / 32;
            const unsigned wg = (unsigned)std::max<unsigned long long>(
                1, std::min<unsigned long long>((units + 7) / 8, (unsigned long long)sms * 8));
            const bool lean = cahead_lean(C, P, P2);
            if (lean && P.n_inj == 0)
                k_cahead_lean<0, false><<<wg, kThreads, 0, st>>>(M, r_lo, r_hi, loc, P, P2, cip, g->groups, g->gpn, lctr);
            else if (lean)
                k_cahead_lean<1, false><<<wg, kThreads, 0, st>>>(M, r_lo, r_hi, loc, P, P2, cip, g->groups, g->gpn, lctr);
            else
                k_cahead_warp<<<wg, kThreads, 0, st>>>(M, r_lo, r_hi, loc, P, P2, cip, cu, g->groups, g->gpn, lctr);
            if (getenv("GSI_TRACE"))
                fprintf(stderr, "[cahead] t %d rows %lld slots %llu w %d rowR %d pa %d ninj %d ninj2 %d E %d\n", t,
                        r_hi - r_lo, s1 - s0, P.t, P2.col[0] < P.t, P.pa != nullptr, P.n_inj, P2.n_inj, P.E);
        } else if (final_lean) {
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
            const unsigned long long units = ((unsigned long long)(r_hi - r_lo) + 31) / 32;
            const unsigned wg = (unsigned)std::max<unsigned long long>(
                1, std::min<unsigned long long>((units + 7) / 8, (unsigned long long)sms * 8));
            if (P.fp && P.n_inj == 0) {
                if (fpT) k_final_fp<0, true><<<wg, kThreads, 0, st>>>(M, r_lo, r_hi, loc, P, s.u, cip, fpT, lctr);
                else k_final_fp<0, false><<<wg, kThreads, 0, st>>>(M, r_lo, r_hi, loc, P, s.u, cip, fpT, lctr);
            } else if (P.fp) {
                if (fpT) k_final_fp<kLeanInj, true><<<wg, kThreads, 0, st>>>(M, r_lo, r_hi, loc, P, s.u, cip, fpT, lctr);
                else k_final_fp<kLeanInj, false><<<wg, kThreads, 0, st>>>(M, r_lo, r_hi, loc, P, s.u, cip, fpT, lctr);
            } else if (P.n_inj == 0)
                k_cahead_lean<0, true><<<wg, kThreads, 0, st>>>(M, r_lo, r_hi, loc, P, P2, cip, g->groups, g->gpn, lctr);
            else
                k_cahead_lean<1, true><<<wg, kThreads, 0, st>>>(M, r_lo, r_hi, loc, P, P2, cip, g->groups, g->gpn, lctr);
        } else if (fast) {
            const size_t fsm = (size_t)tile_slots * 4 * (2 + (size_t)std::min(P.n_inj, P.stage_inj));
            k_count_fast<kFastItems><<<jt, kThreads, fsm, st>>>(M, (long long)nM, F, loc, rowmap, P, cip, c0, c1,
                                                                    lctr);
        } else if (mode == J_COUNT)
            k_join<J_COUNT><<<jt, kThreads, join_smem_bytes(J_COUNT, P), st>>>(M, (long long)nM, F, loc, rowmap, P, P2, cip, cu, g->groups,
                                                     g->gpn, c0, c1, out, loc2, F2, st1, st2, tctr, lctr);
        else if (mode == J_CAHEAD)
            k_join<J_CAHEAD><<<jt, kThreads, join_smem_bytes(J_CAHEAD, P), st>>>(M, (long long)nM, F, loc, rowmap, P, P2, cip, cu,
                                                      g->groups, g->gpn, c0, c1, out, loc2, F2, st1, st2, tctr, lctr);
        else if (mode == J_TABLE)
            k_join<J_TABLE><<<jt, kThreads, join_smem_bytes(J_TABLE, P), st>>>(M, (long long)nM, F, loc, rowmap, P, P2, cip, cu, g->groups,
                                                     g->gpn, c0, c1, out, loc2, F2, st1, st2, tctr, lctr);
        else
            k_join<J_NEXT><<<jt, kThreads, join_smem_bytes(J_NEXT, P), st>>>(M, (long long)nM, F, loc, rowmap, P, P2, cip, cu, g->groups,
                                                    g->gpn, c0, c1, out, loc2, F2, st1, st2, tctr, lctr);
        prof.end();
        // the level's counters come back through pinned memory (a pageable copy stages
        // through a driver buffer: ~10 us more per level on the small-query critical path)
        Counters *hp = C.pinned;
        GSI_CUDA(d2h(S, hp ? (void *)hp : (void *)&hc_local, lctr, sizeof(Counters), st));
        GSI_CUDA(sync_timed(S, st));
        GSI_CUDA(cudaGetLastError());
        const Counters hc = hp ? *hp : hc_local;
        if (!zslice) A.release(status);
        A.release(rowmap);
        // J_NEXT: stored rows (lean: every slot of the chunk, holes included)
        const unsigned long long nout = (mode == J_COUNT || mode == J_CAHEAD) ? hc.count : (lean_next ? slots : hc.total);
        const unsigned long long kept = lean_next ? hc.active_rows : nout;   // rows with a next buffer
        // holes cost the next level a row each: below 60 % kept, this level's later chunks
        // go back to the compacting tile kernel
        if (lean_next && kept * 5 < slots * 3 && !C.force_shared) C.lean_off[si] = 1;
        // Algorithmic bytes of this launch: what the variant must move at least
        // once — the rows of M it extends (row, loc, F), candidates streamed from ci (shared
        // N(v,l0) ∩ C(u) runs are re-read by many rows and stay in L2: not charged per slot),
        // one 32 B PCSR sector + two fpos words per lookup, and every byte it writes.
        const double frac = gba ? (double)slots / (double)gba : 0.0;
        const double rows_in = frac * (double)active;     // rows of the chunk with a non-empty buffer
        const double row_b = 4.0 * P.t + 8.0 * E + 8.0;    // row + loc + F
        const double cand_b = P.prefiltered ? 0.0 : 4.0 * (double)slots;
        constexpr double kLook = 40.0;                      // one PCSR sector + fpos pair
        const double surv_next = (double)hc.count;          // J_NEXT survivors (stored or not)
        double jb = 0.0;
        switch (var) {
        case GSI_V_NEXT_LEAN:   // rows at their Prealloc slots: loc2 for every slot, rows where kept
            jb = rows_in * row_b + cand_b + 8.0 * (double)slots + 4.0 * P.out_w * (double)kept +
                 kLook * ((P2.col[0] < P.t) ? rows_in : (P.pa ? 0.0 : surv_next)) + (P.pa ? 8.0 * surv_next : 0.0);
            break;
        case GSI_V_CAHEAD_LEAN:
        case GSI_V_FINAL_LEAN:   // closed form per row: loc of every slot, the active rows' columns
        case GSI_V_FINAL_FP:
            jb = 8.0 * (double)(r_hi - r_lo) + 4.0 * P.t * (double)hc.active_rows +
                 (var == GSI_V_CAHEAD_LEAN ? kLook * (double)hc.active_rows : 0.0);
            break;
        case GSI_V_CAHEAD_WARP:
        case GSI_V_JOIN_CAHEAD:   // rows + candidates + the last step's run per row or survivor
            jb = rows_in * row_b + cand_b + kLook * ((P2.col[0] < P.t) ? rows_in : (P.pa ? 0.0 : (double)hc.total)) +
                 (P.pa ? 8.0 * (double)hc.total : 0.0);
            break;
        case GSI_V_JOIN_NEXT: {   // + next-step locates, compacted rows, loc', F'
            double looks = 0.0;
            if (P2.E == 1) looks = (P.stage_next && !P.pa) ? rows_in : (P.pa ? 0.0 : surv_next);
            else looks = P2.E * (surv_next + (double)nout);
            jb = rows_in * row_b + cand_b + kLook * looks + (P.pa ? 8.0 * surv_next : 0.0) +
                 (double)nout * (4.0 * P.out_w + 8.0 * P2.E + (P.no_f2 ? 0.0 : 8.0));
            break;
        }
        case GSI_V_JOIN_TABLE:
            jb = rows_in * row_b + cand_b + 4.0 * C.q->k * (double)nout;
            break;
        default:   // GSI_V_JOIN_COUNT, GSI_V_COUNT_FAST
            jb = rows_in * row_b + cand_b;
        }
        if (E > 1) jb += 8.0 * rows_in * (E - 1);   // the other linking lists' locate entries
        S.alg_bytes_variant[var] += jb;
        // items: matches produced at the last level (or counted by the count-ahead), rows
        // stored by a J_NEXT level
        S.items_variant[var] += (mode == J_COUNT || mode == J_CAHEAD || mode == J_TABLE) ? (last ? nout : hc.count) : nout;
        if (mode == J_NEXT) S.rows[t] += hc.count;   // |M_{t+1}|: every survivor, stored or not
        if (mode == J_CAHEAD) {                        // survivors = |M_{t+1}|, counted = |M_{t+2}|
            S.rows[t] += hc.total;
            S.rows[t + 1] += hc.count;
            S.gba[t + 1] += hc.total2;
            if (S.levels < t + 2) S.levels = t + 2;
            S.count_ahead = 1;
            C.count += hc.count;
        }
        S.alg_bytes[GSI_K_JOIN] += jb;
        if (last) {
            C.count += nout;
            C.fp1 += hc.fp1;
            C.fp2 ^= hc.fp2;
            S.rows[t] += nout;
            if (S.levels < t + 1) S.levels = t + 1;
        }
        if (mode == J_TABLE) {
            if (nout) {
                rc = table_put(C, out, nout);
            }
            A.release(out);
        } else if (mode == J_NEXT) {
            if (nout && hc.total2) rc = level(C, si + 1, out, nout, loc2, F2, hc.total2, kept, hc.list_elems, pf_next);
            A.release(out);
            A.release(loc2);
            A.release(F2);
        }
        A.reset(mk);
    }
    if (rc != GSI_OK) break;
    }
    return rc;
}

}  // namespace

// ------------------------------------------------------------------ small path ---------
// Eligible before the filter runs: one shard, per-row e0, no test hooks.  After the plan: a
// first level of at most 4096 roots and every step within the kernel's limits (<= 8 linking
// edges and subtraction columns).  A level that outgrows the kernel's capacity stops it and the
// host takes the regular path from M_1 with the same plan.
bool small_apriori(const QueryCtx &C) {
    const gsi_query_opts &o = C.opts;
    if (o.small_mode == 1 || env_flag("GSI_SMALL_OFF") || C.W != 1 || o.e0_mode != 0) return false;
    if (o.chunk_slots || o.force_paths || o.ablation || (o.roots && o.n_roots > 0)) return false;
    return C.q->k > 1 && !C.q->absent_label;
}

bool small_eligible(const QueryCtx &C, unsigned long long nM1) {
    if (nM1 == 0 || nM1 > kSmallMaxRoots) return false;
    for (auto &s : C.steps) {
        if ((int)s.col.size() > kSmallMaxE) return false;
        int ninj = 0;
        if (!C.opts.homomorphism)
            for (int c = 0; c < s.t; c++) {
                if (C.q->qvl[C.order[c]] != C.q->qvl[s.u]) continue;
                bool linked = false;
                for (int lc : s.col) linked |= lc == c;
                ninj += linked ? 0 : 1;
            }
        if (ninj > kSmallMaxInj) return false;
    }
    return true;
}

// Every level in k_small_query (launched right after the host plan; M_1 is extracted in the
// kernel from the filter's bitmap and per-group counts), one pinned read-back.  done = false if
// a level outgrew the kernel (the caller then takes the regular path, same plan).
gsi_status run_small(QueryCtx &C, const uint16_t *grp, long long ngrp, long long ngrp_pad, int gw, SmallOut *dout,
                     SmallOut *hout, bool &done) {
    done = false;
    const gsi_graph *g = C.g;
    gsi_stats &S = *C.S;
    Arena &A = *C.A;
    const int k = C.q->k;
    const int u1 = C.order[0];
    SmallPlan plan;
    std::memset(&plan, 0, sizeof(plan));
    plan.k = k;
    plan.want_table = C.opts.want_table ? 1 : 0;
    plan.fp = C.opts.fingerprint ? 1 : 0;
    plan.gpn = g->gpn;
    for (int q = 0; q < k; q++) plan.pos_of_q[q] = C.pos_of_q[q];
    for (size_t j = 0; j < C.steps.size(); j++) {
        const Step &s = C.steps[j];
        SmallStep &T = plan.st[j];
        T.E = (int)s.col.size();
        for (int e = 0; e < T.E; e++) {
            T.col[e] = s.col[e];
            T.lab[e] = (uint32_t)s.lab[e];
            T.gbase[e] = (unsigned long long)g->gbase[s.lab[e]];
            T.ngroups[e] = g->ngroups[s.lab[e]];
        }
        T.n_inj = 0;
        if (!C.opts.homomorphism)
            for (int c = 0; c < s.t; c++) {
                if (C.q->qvl[C.order[c]] != C.q->qvl[s.u]) continue;   // C(u) excludes other labels
                bool linked = false;
                for (int lc : s.col) linked |= lc == c;                // x in N(m[c],l) => x != m[c]
                if (!linked) T.inj_col[T.n_inj++] = c;
            }
        T.cu = C.bm + (long long)s.u * C.words;
    }
    plan.bm1 = C.bm + (long long)u1 * C.words;
    plan.grp1 = grp + (long long)u1 * ngrp_pad;
    plan.words = C.words;
    plan.ngrp = ngrp;
    plan.gw = gw;
    plan.nM1 = (unsigned long long)S.cand[u1];
    int32_t *bufA = nullptr, *bufB = nullptr, *table = nullptr;
    Loc *loc = nullptr;
    unsigned long long *F = nullptr;
    const size_t mk = A.mark();
    GSI_TRY(A.get(&bufA, kSmallRowCap * (unsigned long long)k));
    GSI_TRY(A.get(&bufB, kSmallRowCap * (unsigned long long)k));
    GSI_TRY(A.get(&loc, kSmallRowCap * (unsigned long long)kSmallMaxE));
    GSI_TRY(A.get(&F, kSmallRowCap + 1));
    if (plan.want_table) GSI_TRY(A.get(&table, kSmallRowCap * (unsigned long long)k));
    C.prof->begin(GSI_K_JOIN, GSI_V_SMALL);   // dout: zeroed with the query's counter pool
    S.variant_launches[GSI_V_SMALL]++;
    k_small_query<<<1, kSmallThreads, kSmallDynSmem, C.st>>>(plan, g->groups, g->ci, bufA, bufB, loc, F, table, dout);
    C.prof->end();
    GSI_CUDA(d2h(S, hout, dout, sizeof(SmallOut), C.st));
    GSI_CUDA(sync_timed(S, C.st));
    GSI_CUDA(cudaGetLastError());
    if (hout->aborted) {
        S.small_aborted = hout->aborted;
        A.reset(mk);
        return GSI_OK;
    }
    const SmallOut &h = *hout;
    if (getenv("GSI_TRACE")) {   // device phase times (SM clock cycles -> us at the device's clock rate)
        int khz = 0;
        cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, g->device);
        const double us = khz > 0 ? 1000.0 / khz : 0.0;
        fprintf(stderr, "[small] M1 %.2f us, levels", (h.clk[2] - h.clk[0]) * us);
        for (int t = 1; t < k && h.clk[2 + t]; t++) fprintf(stderr, " %.2f", (h.clk[2 + t] - h.clk[1 + t]) * us);
        fprintf(stderr, " (rows");
        for (int t = 0; t < k; t++) fprintf(stderr, " %llu", h.rows[t]);
        fprintf(stderr, ")\n");
    }
    S.levels = 1;
    for (int t = 0; t < k; t++) {
        S.rows[t] = h.rows[t];
        S.gba[t] = h.gba[t];
        S.list_elems[t] = h.elems[t];
        if (t > 0 && h.rows[t - 1]) S.levels = t + 1;   // level t + 1 was produced
    }
    S.alg_bytes[GSI_K_COMPACT] += 4.0 * C.words + 4.0 * h.rows[0];
    C.count = h.count;
    C.fp1 = h.fp1;
    C.fp2 = h.fp2;
    if (plan.want_table && h.nout) {
        const gsi_status rs = table_put(C, table, h.nout);
        if (rs != GSI_OK) {
            A.reset(mk);
            return rs;
        }
    }
    A.reset(mk);
    done = true;
    return GSI_OK;
}

// ------------------------------------------------------------------ ablation engine ----
// Balance thresholds (reading A16: W1 = 4 W2 = 16 W3 = 4096; tunable, perf only).
uint32_t abl_w1() {
    const char *e = getenv("GSI_ABL_W1");
    return e ? (uint32_t)atol(e) : 4096u;
}
uint32_t abl_w2() {
    const char *e = getenv("GSI_ABL_W2");
    return e ? (uint32_t)atol(e) : 1024u;
}
constexpr int kAblCluster = 8;   // CTAs per heavy row (layer 1)

struct AblLayers {   // rows of each balance layer (null: every row, no balance)
    uint32_t *rows[3] = {nullptr, nullptr, nullptr};
    unsigned long long n[3] = {0, 0, 0};
};
struct AblArgs {
    const int32_t *M;
    unsigned long long nM;
    const Loc *loc;
    StepParams P;
    const int32_t *ci;
    const uint32_t *cu;
    const int32_t *cul;
    long long cun;
    Counters *ctr;
    int sms;
    bool dr;
};

// Layer 4 (warp per row, + block duplicate removal) over the light rows, layer 2 (a block per
// row) and layer 1 (an 8-CTA cluster per row) over the others.
template <int MODE, bool WC, bool NV>
gsi_status abl_layers(const AblArgs &X, const AblLayers &Ly, const unsigned long long *off, int32_t *gba,
                      uint32_t *cnt, int32_t *out, cudaStream_t st) {
    const unsigned long long nl = Ly.n[0];
    if (nl) {
        const unsigned wg = (unsigned)std::max<unsigned long long>(
            1, std::min<unsigned long long>((nl * 32 + kThreads - 1) / kThreads, (unsigned long long)X.sms * 16));
        if (X.dr)
            k_abl_join<MODE, WC, NV, true><<<wg, kThreads, 0, st>>>(X.M, (long long)nl, Ly.rows[0], X.loc, off, X.P, X.ci,
                                                                   X.cu, X.cul, X.cun, gba, cnt, out, X.ctr);
        else
            k_abl_join<MODE, WC, NV, false><<<wg, kThreads, 0, st>>>(X.M, (long long)nl, Ly.rows[0], X.loc, off, X.P, X.ci,
                                                                    X.cu, X.cul, X.cun, gba, cnt, out, X.ctr);
    }
    for (int b = 1; b <= 2; b++) {
        if (!Ly.n[b]) continue;
        const int CL = b == 2 ? kAblCluster : 1;
        const unsigned long long ncl = std::min<unsigned long long>(Ly.n[b], (unsigned long long)X.sms * 4 / CL);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(ncl * CL));
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CL;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        GSI_CUDA(cudaLaunchKernelEx(&cfg, k_abl_heavy<MODE, WC, NV>, X.M, (const uint32_t *)Ly.rows[b], (long long)Ly.n[b],
                                    X.loc, off, X.P, X.ci, X.cu, X.cul, X.cun, gba, cnt, out, X.ctr));
    }
    return GSI_OK;
}

// Every level with the paper-style kernels (one warp per row); see k_abl_join.
gsi_status run_ablation(QueryCtx &C, int32_t *M, unsigned long long nM) {
    const gsi_graph *g = C.g;
    gsi_stats &S = *C.S;
    Arena &A = *C.A;
    cudaStream_t st = C.st;
    const int ab = C.opts.ablation;
    const bool cr = ab & GSI_ABL_CR, two = ab & GSI_ABL_TWO_STEP, wc = !(ab & GSI_ABL_NO_WCACHE),
               naive = ab & GSI_ABL_NAIVE_SO, lb = !(ab & GSI_ABL_NO_LB), dr = !(ab & GSI_ABL_NO_DR);
    if (cr) GSI_TRY(ensure_cr(g, st));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
    auto scan = [&](const uint32_t *in, unsigned long long n, unsigned long long **outp) -> gsi_status {
        const unsigned tiles = grid_for(n, kThreads);
        unsigned long long *status = nullptr;
        GSI_TRY(A.get(outp, n + 1));
        GSI_TRY(A.get(&status, (unsigned long long)tiles + 1));
        GSI_CUDA(cudaMemsetAsync(status, 0, 8ull * (tiles + 1), st));
        GSI_CUDA(cudaMemsetAsync(*outp, 0, 8, st));
        C.prof->begin(GSI_K_OTHER);
        if (n) k_scan_counts<<<tiles, kThreads, 0, st>>>(in, (long long)n, *outp, status + 1, (unsigned *)status);
        C.prof->end();
        return GSI_OK;
    };
    Counters *ctr = nullptr;
    GSI_TRY(A.get(&ctr, 1));
    for (size_t si = 0; si < C.steps.size(); si++) {
        const Step &s = C.steps[si];
        const int t = s.t;
        const bool last = si + 1 == C.steps.size();
        StepParams P;
        fill_params(C, s, P, t);
        if (S.levels < t) S.levels = t;
        const uint32_t *cu = C.bm + (long long)s.u * C.words;
        int32_t *cul = nullptr;
        long long cun = 0;
        if (naive) {   // the sorted candidate list C(u) (bitmap compaction)
            cun = S.cand[s.u];
            const unsigned tiles = grid_for(C.words, kThreads);
            unsigned long long *status = nullptr;
            GSI_TRY(A.get(&cul, cun));
            GSI_TRY(A.get(&status, (unsigned long long)tiles + 1));
            GSI_CUDA(cudaMemsetAsync(status, 0, 8ull * (tiles + 1), st));
            C.prof->begin(GSI_K_COMPACT);
            k_compact_bitmap<<<tiles, kThreads, 0, st>>>(cu, C.words, cul, status + 1, (unsigned *)status, ctr);
            C.prof->end();
        }
        Loc *loc = nullptr;
        uint32_t *lens = nullptr, *cnt = nullptr;
        unsigned long long *F = nullptr, *G = nullptr;
        GSI_TRY(A.get(&loc, std::max<unsigned long long>(nM, 1) * (unsigned long long)P.E));
        GSI_TRY(A.get(&lens, nM));
        C.prof->begin(GSI_K_PROBE);
        k_abl_probe<<<grid_for(nM, kThreads), kThreads, 0, st>>>(M, (long long)nM, P, cr ? 1 : 0, g->cr_key, g->cr_loc,
                                                                  g->groups, g->gpn, loc, lens);
        C.prof->end();
        GSI_TRY(scan(lens, nM, &F));
        unsigned long long gba = 0;
        GSI_CUDA(d2h(S, &gba, F + nM, 8, st));
        GSI_CUDA(sync_timed(S, st));
        S.gba[t] += gba;
        if (gba == 0) break;
        // the 4-layer balance (layers 1, 2, 4): stable split of the rows by buffer length
        AblLayers Ly;
        Ly.n[0] = nM;
        if (lb) {
            uint32_t *flag = nullptr;
            GSI_TRY(A.get(&flag, nM));
            for (int b = 0; b < 3; b++) {
                unsigned long long *pos = nullptr;
                C.prof->begin(GSI_K_OTHER);
                k_abl_flags<<<grid_for(nM, kThreads), kThreads, 0, st>>>(lens, (long long)nM, abl_w1(), abl_w2(), b, flag);
                C.prof->end();
                GSI_TRY(scan(flag, nM, &pos));
                GSI_TRY(A.get(&Ly.rows[b], nM));
                C.prof->begin(GSI_K_OTHER);
                k_abl_gather<<<grid_for(nM, kThreads), kThreads, 0, st>>>(flag, pos, (long long)nM, Ly.rows[b]);
                C.prof->end();
                GSI_CUDA(d2h(S, &Ly.n[b], pos + nM, 8, st));
            }
            GSI_CUDA(sync_timed(S, st));
            S.abl_layer_rows[0] += Ly.n[0];
            S.abl_layer_rows[1] += Ly.n[1];
            S.abl_layer_rows[2] += Ly.n[2];
        }
        AblArgs X{M, nM, loc, P, g->ci, cu, cul, cun, ctr, sms, dr};
        if (last) {
            GSI_CUDA(cudaMemsetAsync(ctr, 0, sizeof(Counters), st));
            C.prof->begin(GSI_K_JOIN, GSI_V_ABLATION);
            S.variant_launches[GSI_V_ABLATION]++;
            if (naive) GSI_TRY((abl_layers<AB_FINAL, true, true>(X, Ly, nullptr, nullptr, nullptr, nullptr, st)));
            else GSI_TRY((abl_layers<AB_FINAL, true, false>(X, Ly, nullptr, nullptr, nullptr, nullptr, st)));
            C.prof->end();
            Counters hc;
            GSI_CUDA(d2h(S, &hc, ctr, sizeof(hc), st));
            GSI_CUDA(sync_timed(S, st));
            C.count = hc.count;
            C.fp1 = hc.fp1;
            C.fp2 = hc.fp2;
            S.rows[t] = hc.count;
            S.levels = t + 1;
            break;
        }
        GSI_TRY(A.get(&cnt, nM));
        int32_t *gbuf = nullptr, *out = nullptr;
        if (!two) GSI_TRY(A.get(&gbuf, gba));
        C.prof->begin(GSI_K_JOIN, two ? GSI_V_TWO_STEP : GSI_V_ABLATION);
        S.variant_launches[two ? GSI_V_TWO_STEP : GSI_V_ABLATION]++;
        if (two) {   // pass 1: count only
            if (naive) GSI_TRY((abl_layers<AB_COUNT, true, true>(X, Ly, nullptr, nullptr, cnt, nullptr, st)));
            else GSI_TRY((abl_layers<AB_COUNT, true, false>(X, Ly, nullptr, nullptr, cnt, nullptr, st)));
        } else {     // Prealloc: survivors into the row's buffer
            if (naive) GSI_TRY((abl_layers<AB_PC, true, true>(X, Ly, F, gbuf, cnt, nullptr, st)));
            else GSI_TRY((abl_layers<AB_PC, true, false>(X, Ly, F, gbuf, cnt, nullptr, st)));
        }
        C.prof->end();
        GSI_TRY(scan(cnt, nM, &G));
        unsigned long long nout = 0;
        GSI_CUDA(d2h(S, &nout, G + nM, 8, st));
        GSI_CUDA(sync_timed(S, st));
        S.rows[t] += nout;
        if (nout == 0) break;
        GSI_TRY(A.get(&out, nout * (unsigned long long)(t + 1)));
        C.prof->begin(GSI_K_JOIN, GSI_V_ABLATION);
        S.variant_launches[GSI_V_ABLATION]++;
        if (two) {   // pass 2: join again, write the rows
            if (naive && wc) GSI_TRY((abl_layers<AB_WRITE, true, true>(X, Ly, G, nullptr, nullptr, out, st)));
            else if (naive) GSI_TRY((abl_layers<AB_WRITE, false, true>(X, Ly, G, nullptr, nullptr, out, st)));
            else if (wc) GSI_TRY((abl_layers<AB_WRITE, true, false>(X, Ly, G, nullptr, nullptr, out, st)));
            else GSI_TRY((abl_layers<AB_WRITE, false, false>(X, Ly, G, nullptr, nullptr, out, st)));
        } else {     // Combine: link the buffers into M'
            const unsigned long long items = wc ? nout * (unsigned long long)(t + 1) : nout;
            const unsigned lg = (unsigned)std::min<unsigned long long>(grid_for(items, kThreads), (unsigned long long)sms * 32);
            if (wc) k_abl_link<true><<<lg, kThreads, 0, st>>>(M, (long long)nM, F, G, gbuf, t, nout, out);
            else k_abl_link<false><<<lg, kThreads, 0, st>>>(M, (long long)nM, F, G, gbuf, t, nout, out);
        }
        C.prof->end();
        M = out;
        nM = nout;
    }
    GSI_CUDA(cudaGetLastError());
    return GSI_OK;
}

// Plan (a4): Alg. 2 order, the steps and the stored-column layout, from |C(u)|.
gsi_status plan_query(QueryCtx &C, const std::vector<long long> &cand) {
    const gsi_prepared *q = C.q;
    const gsi_query_opts &opts = C.opts;
    gsi_stats &S = *C.S;
    const int k = q->k;
    GSI_TRY(plan_order(q, cand, opts.force_order, C.order));
    GSI_TRY(build_steps(q, C.order, opts.force_first_edge, C.steps));
    for (int j = 0; j < k; j++) S.order[j] = C.order[j];
    for (auto &s : C.steps) {
        S.n_edges[s.t] = (int)s.col.size();
        S.first_edge[s.t] = s.other[s.paper_e0];
    }
    C.pos_of_q.assign(k, 0);
    for (int j = 0; j < k; j++) C.pos_of_q[C.order[j]] = j;
    plan_layout(C, !opts.want_table && !opts.fingerprint && !opts.ablation);
    return GSI_OK;
}

// Level 1 (a5) and the levels (a6-a8) on the host-driven path, after plan_query: every query
// the small path did not take.  Leaves the count / fingerprint / table pieces in C.
gsi_status run_regular(QueryCtx &C, const std::vector<long long> &cand, unsigned long long budget, double t_start) {
    const gsi_graph *g = C.g;
    const gsi_prepared *q = C.q;
    const gsi_query_opts &opts = C.opts;
    gsi_stats &S = *C.S;
    Arena &A = *C.A;
    Prof &prof = *C.prof;
    cudaStream_t st = C.st;
    const int k = q->k;
    const long long n = g->n;
    const long long words = C.words;
    const uint32_t *bm = C.bm;
    Counters hc;

    // memory budget -> chunk capacity in GBA slots (bytes per slot per level: S,R 8 B,
    // M' 4(t+1) B, the child level's loc/F 8E+8 B), over the k-1 levels that may nest.
    {
        // (the chunk capacity depends on the budget only, never on the workspace size, so the
        // chunking of a query is reproducible)
        int maxE = 1;
        for (auto &s : C.steps) maxE = std::max(maxE, (int)s.col.size());
        const double per_slot = 8.0 + 4.0 * (k + 1) + 8.0 * maxE + 8.0;
        const double levels = std::max(1, k - 1);
        C.cap_slots = (unsigned long long)std::max(1.0, budget / (per_slot * levels));
        if (opts.chunk_slots) C.cap_slots = opts.chunk_slots;
    }
    C.shard_min = opts.shard_min_rows ? opts.shard_min_rows : 65536;
    C.sharded = C.W == 1;
    C.force_shared = (opts.force_paths & 1) != 0;
    C.deadline = opts.timeout_s > 0 ? t_start + 1000.0 * opts.timeout_s : 0;

    bool empty = q->absent_label;
    for (int u = 0; u < k; u++) empty |= cand[u] == 0;

    // ---------------- level 1 (a5) ----------------
    int32_t *M = nullptr;
    unsigned long long nM = 0;
    if (!empty) {
        unsigned long long *status = nullptr;
        const int u1 = C.order[0];
        const uint32_t *bm1 = bm + (long long)u1 * words;
        if (opts.roots && opts.n_roots > 0) {
            std::vector<int32_t> roots(opts.roots, opts.roots + opts.n_roots);
            std::sort(roots.begin(), roots.end());
            roots.erase(std::unique(roots.begin(), roots.end()), roots.end());
            roots.erase(std::remove_if(roots.begin(), roots.end(), [&](int32_t v) { return v < 0 || v >= n; }),
                        roots.end());
            long long nr = (long long)roots.size();
            int32_t *d_roots = nullptr;
            GSI_TRY(A.get(&d_roots, nr));
            if (nr) GSI_CUDA(h2d(S, d_roots, roots.data(), 4ull * nr, st));
            GSI_TRY(A.get(&M, nr));
            unsigned tiles = grid_for(nr, kThreads);
            GSI_TRY(A.get(&status, tiles + 1));
            GSI_CUDA(cudaMemsetAsync(status, 0, 8ull * (tiles + 1), st));
            prof.begin(GSI_K_COMPACT);
            k_compact_roots<<<tiles, kThreads, 0, st>>>(d_roots, nr, bm1, M, status + 1, (unsigned *)status, C.ctr);
            prof.end();
            GSI_CUDA(d2h(S, &hc, C.ctr, sizeof(Counters), st));
            GSI_CUDA(sync_timed(S, st));
            nM = hc.total;
            S.alg_bytes[GSI_K_COMPACT] += 8.0 * nr + 4.0 * nM;
        } else {
            nM = (unsigned long long)cand[u1];
            GSI_TRY(A.get(&M, nM));
            unsigned tiles = grid_for(words, kThreads);
            GSI_TRY(A.get(&status, tiles + 1));
            GSI_CUDA(cudaMemsetAsync(status, 0, 8ull * (tiles + 1), st));
            prof.begin(GSI_K_COMPACT);
            k_compact_bitmap<<<tiles, kThreads, 0, st>>>(bm1, words, M, status + 1, (unsigned *)status, C.ctr);
            prof.end();
            S.alg_bytes[GSI_K_COMPACT] += 4.0 * words + 4.0 * nM;
        }
        A.release(status);
    }

    gsi_status rc = GSI_OK;
    if (!empty && k > 1 && opts.ablation) {
        rc = run_ablation(C, M, nM);
    } else if (!empty && k == 1) {
        S.rows[0] = nM;
        S.levels = 1;
        StepParams P;
        std::memset(&P, 0, sizeof(P));
        P.k = 1;
        P.t = 1;
        GSI_CUDA(cudaMemsetAsync(C.ctr, 0, sizeof(Counters), st));
        if (nM && opts.fingerprint) {
            prof.begin(GSI_K_OTHER);
            k_fp_rows<<<grid_for(nM, kThreads), kThreads, 0, st>>>(M, (long long)nM, P, C.ctr);
            prof.end();
        }
        GSI_CUDA(d2h(S, &hc, C.ctr, sizeof(Counters), st));
        GSI_CUDA(sync_timed(S, st));
        C.count = nM;
        C.fp1 = hc.fp1;
        C.fp2 = hc.fp2;
        if (opts.want_table && nM) {
            GSI_TRY(table_put(C, M, nM));
        }
    } else if (!empty) {
        // level-1 Prealloc (Alg. 4) on M_1 = C(pi_1)
        StepParams P;
        fill_params(C, C.steps[0], P, 1);
        Loc *loc = nullptr;
        unsigned long long *F = nullptr, *status = nullptr;
        GSI_TRY(A.get(&loc, std::max<unsigned long long>(nM, 1) * (unsigned long long)P.E));
        GSI_TRY(A.get(&F, nM + 1));
        const unsigned ptiles = grid_for(nM, kThreads);
        GSI_TRY(A.get(&status, ptiles + 1));
        GSI_CUDA(cudaMemsetAsync(status, 0, 8ull * (ptiles + 1), st));
        GSI_CUDA(cudaMemsetAsync(C.ctr, 0, sizeof(Counters), st));
        GSI_CUDA(cudaMemsetAsync(F, 0, 8, st));
        if (nM) {
            prof.begin(GSI_K_PROBE);
            k_probe<<<ptiles, kThreads, 0, st>>>(M, (long long)nM, P, g->groups, g->gpn, loc, F, status + 1,
                                                 (unsigned *)status, C.ctr);
            prof.end();
        }
        unsigned long long gba = 0;
        GSI_CUDA(d2h(S, &gba, F + nM, 8, st));
        GSI_CUDA(d2h(S, &hc, C.ctr, sizeof(Counters), st));
        GSI_CUDA(sync_timed(S, st));
        A.release(status);
        S.alg_bytes[GSI_K_PROBE] += (double)nM * (20.0 * P.E + 8.0);
        S.rows[0] += nM;
        rc = level(C, 0, M, nM, loc, F, gba, hc.active_rows, hc.list_elems, false);
        A.release(loc);
        A.release(F);
    }
    if (M) A.release(M);
    return rc;
}

gsi_status run_impl(const gsi_graph *g, const gsi_prepared *q, const gsi_query_opts *opts_in, gsi_result **out) {
    *out = nullptr;
    if (!g || !q || q->g != g) {
        set_error("prepared query does not belong to this graph");
        return GSI_ERR_INVALID_ARG;
    }
    QueryCtx C;
    gsi_query_opts_default(&C.opts);
    if (opts_in) C.opts = *opts_in;
    const gsi_query_opts &opts = C.opts;
    const double t_start = now_ms();
    GSI_CUDA(cudaSetDevice(g->device));
    ensure_pool(g->device);
    if (getenv("GSI_TRACE")) fprintf(stderr, "[host] pool %.3f ms\n", now_ms() - t_start);
    cudaStream_t st = opts.stream ? (cudaStream_t)opts.stream : cudaStreamPerThread;
    const int k = q->k;
    const long long n = g->n;
    const long long words = (n + 31) / 32;
    if (opts.ablation && (opts.want_table || opts.shard_count > 1)) {
        set_error("ablation runs are count / fingerprint only and unsharded");
        return GSI_ERR_INVALID_ARG;
    }
    C.W = opts.shard_count > 1 ? opts.shard_count : 1;
    C.rank = C.W > 1 ? opts.shard_rank : 0;
    if (C.rank < 0 || C.rank >= C.W) {
        set_error("shard_rank out of range");
        return GSI_ERR_INVALID_ARG;
    }
    auto res = std::make_unique<gsi_result>();
    res->device = g->device;
    res->k = k;
    gsi_stats &S = res->stats;
    std::memset(&S, 0, sizeof(S));
    S.k = k;
    S.shard_level = -1;
    Arena A(st);
    PinnedCounters pinned;
    C.pinned = pinned.p;
    Prof prof;
    prof.on = opts.profile != 0;
    prof.st = st;
    prof.start();
    C.g = g;
    C.q = q;
    C.st = st;
    C.A = &A;
    C.prof = &prof;
    // the table grows in place (vm.cu); owned here until the result takes it
    std::unique_ptr<TableVM> tv_guard(opts.want_table ? TableVM::create(g->device, k) : nullptr);
    C.tv = tv_guard.get();
    C.S = &S;
    C.words = words;

    // device memory the query may use; the workspace grows to the demand seen so far
    // (cudaMemGetInfo costs tens of microseconds: a query that fits the workspace it takes
    // computes the budget only if it leaves the small path, in run_regular)
    unsigned long long budget = opts.mem_budget_bytes;
    if (!budget && !workspace_fits(g->device)) budget = device_budget(g->device, 0);
    const bool htrace = getenv("GSI_TRACE") != nullptr;
    if (htrace) fprintf(stderr, "[host] budget %.3f ms\n", now_ms() - t_start);
    A.init_workspace(g->device, budget ? budget : ~(size_t)0);
    if (htrace) fprintf(stderr, "[host] workspace %.3f ms\n", now_ms() - t_start);
    // One zeroed pool per query (a single memset): the query counters, |C(u)|, the small
    // path's output block, then the per-level counter / look-back slices (C.zoff).
    uint32_t *bm = nullptr;
    unsigned long long *d_counts = nullptr;
    SmallOut *d_small = nullptr;
    unsigned *d_done = nullptr;   // the filter's CTA ticket (zero-copy publication)
    {
        constexpr unsigned long long kZWords = 1ull << 17;   // 1 MB
        constexpr unsigned long long kSmallW = (sizeof(SmallOut) + 31) / 32 * 4;
        if (A.get_big(&C.zpool, kZWords) == GSI_OK && cudaMemsetAsync(C.zpool, 0, 8ull * kZWords, st) == cudaSuccess) {
            C.zcap = kZWords;
            C.ctr = reinterpret_cast<Counters *>(C.zpool);
            d_counts = C.zpool + kCtrWords;
            d_done = reinterpret_cast<unsigned *>(C.zpool + kCtrWords + 4 * ((GSI_MAX_K + 3) / 4));
            d_small = reinterpret_cast<SmallOut *>(C.zpool + kCtrWords + 4 * ((GSI_MAX_K + 3) / 4) + 4);
            C.zoff = kCtrWords + 4 * ((GSI_MAX_K + 3) / 4) + 4 + kSmallW;
        } else {
            cudaGetLastError();
            C.zpool = nullptr;
            GSI_TRY(A.get(&C.ctr, 1));
            GSI_TRY(A.get(&d_counts, k));
            GSI_TRY(A.get(&d_small, 1));
            GSI_CUDA(cudaMemsetAsync(C.ctr, 0, sizeof(Counters), st));
            GSI_CUDA(cudaMemsetAsync(d_counts, 0, 8ull * k, st));
            GSI_CUDA(cudaMemsetAsync(d_small, 0, sizeof(SmallOut), st));
        }
    }
    if (htrace) fprintf(stderr, "[host] zeroed %.3f ms\n", now_ms() - t_start);

    // ---------------- filter (a3) ----------------
    const bool small_try = small_apriori(C) && !g->ml;
    uint16_t *grp = nullptr;
    static int sms_cached[64] = {0};
    int sms = g->device >= 0 && g->device < 64 ? sms_cached[g->device] : 0;
    if (!sms) {
        sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
        if (g->device >= 0 && g->device < 64) sms_cached[g->device] = sms;
    }
    const int gw = filter_fw(words, sms);   // bitmap words per group count (= the filter's words per warp)
    const long long ngrp = (words + gw - 1) / gw;
    const long long ngrp_pad = (ngrp + 7) & ~7ll;
    GSI_TRY(A.get(&bm, (unsigned long long)words * k));
    if (small_try) GSI_TRY(A.get(&grp, (unsigned long long)ngrp_pad * k));
    C.bm = bm;
    // zero-copy publication of |C(u)| (single-label graphs, pinned block and zeroed pool)
    unsigned long long *hpub_dev = (!g->ml && d_done && pinned.dpub) ? pinned.dpub : nullptr;
    if (hpub_dev) reinterpret_cast<volatile unsigned long long *>(pinned.blk->pub)[GSI_MAX_K + 1] = 0ull;
    {
        prof.begin(GSI_K_FILTER);
        const uint32_t *qsig = q->d_qsig + (opts.homomorphism ? (size_t)k * kPlanes : 0);
        if (g->ml)   // multi-label: hashed label sets + exact refine (ext.cu)
            GSI_CUDA(launch_filter_ml(g, q, opts.homomorphism, bm, words, d_counts, st));
        else
            GSI_CUDA(launch_filter(g->sig, n, k, qsig, opts.filter_mode == 1, bm, words, d_counts, C.ctr, grp, ngrp_pad,
                                   sms, st, d_done, hpub_dev));
        prof.end();
    }
    if (htrace) fprintf(stderr, "[host] filter launched %.3f ms\n", now_ms() - t_start);
    // |C(u)| and the filter's counters back in one copy (adjacent in the zeroed pool)
    std::vector<long long> cand(k);
    unsigned long long plane_loads = 0;
    bool published = false;
    if (hpub_dev) {   // spin on the flag the filter's last CTA raises (bounded; then the copy path)
        volatile unsigned long long *pub = pinned.blk->pub;
        const auto t0 = std::chrono::steady_clock::now();
        while (pub[GSI_MAX_K + 1] == 0ull) {
            if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(2)) break;
        }
        if (pub[GSI_MAX_K + 1]) {
            std::atomic_thread_fence(std::memory_order_acquire);
            for (int u = 0; u < k; u++) cand[u] = (long long)pub[u];
            plane_loads = pub[GSI_MAX_K];
            published = true;
            S.ms_host_sync += (float)std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        }
    }
    if (!published) {
        std::vector<unsigned long long> rb_pageable;
        unsigned long long *rb = C.pinned ? pinned.blk->rb : nullptr;
        if (!rb) {
            rb_pageable.resize(kCtrWords + GSI_MAX_K);
            rb = rb_pageable.data();
        }
        if (C.zpool) {
            GSI_CUDA(d2h(S, rb, C.zpool, 8ull * (kCtrWords + k), st));
        } else {
            GSI_CUDA(d2h(S, rb, C.ctr, sizeof(Counters), st));
            GSI_CUDA(d2h(S, rb + kCtrWords, d_counts, 8ull * k, st));
        }
        GSI_CUDA(sync_timed(S, st));
        GSI_CUDA(cudaGetLastError());
        for (int u = 0; u < k; u++) cand[u] = (long long)rb[kCtrWords + u];
        plane_loads = reinterpret_cast<const Counters *>(rb)->plane_loads;
    }
    if (htrace) fprintf(stderr, "[host] read back %.3f ms\n", now_ms() - t_start);
    const double t_filter = now_ms();
    S.ms_filter = (float)(t_filter - t_start);
    for (int u = 0; u < k; u++) S.cand[u] = cand[u];
    S.alg_bytes[GSI_K_FILTER] = 4.0 * n + 4.0 * plane_loads + 4.0 * words * k;

    // ---------------- plan (a4) ----------------
    GSI_TRY(plan_query(C, cand));
    double t_plan = now_ms();
    S.ms_plan = (float)(t_plan - t_filter);
    if (htrace) fprintf(stderr, "[host] planned %.3f ms\n", t_plan - t_start);

    gsi_status rc = GSI_OK;
    bool small_done = false;
    bool all_nonempty = true;
    for (int u = 0; u < k; u++) all_nonempty &= cand[u] > 0;
    if (small_try && all_nonempty && small_eligible(C, (unsigned long long)cand[C.order[0]])) {
        // every level in one kernel, one read-back
        SmallOut hsmall_pageable;
        SmallOut *hsmall = C.pinned ? &pinned.blk->so : &hsmall_pageable;
        GSI_TRY(run_small(C, grp, ngrp, ngrp_pad, gw, d_small, hsmall, small_done));
    }
    if (!small_done) {
        if (!budget) budget = device_budget(g->device, A.ws_dev >= 0 ? A.cap : 0);
        rc = run_regular(C, cand, budget, t_start);
    }
    if (rc != GSI_OK) {
        for (auto &p : C.pieces) cudaFreeAsync(p.first, st);
        cudaStreamSynchronize(st);
        return rc;
    }
    if (C.capped && !opts.partial_on_timeout) {
        for (auto &p : C.pieces) cudaFreeAsync(p.first, st);
        cudaStreamSynchronize(st);
        set_error("query timeout");
        return GSI_ERR_TIMEOUT;
    }
    // ---------------- finalize (a9) ----------------
    res->count = C.count;
    res->fp[0] = C.count;
    res->fp[1] = C.fp1;
    res->fp[2] = C.fp2;
    S.capped = C.capped ? 1 : 0;
    if (opts.want_table) {
        res->has_table = true;
        res->nrows = C.count;
        if (C.tv) {   // grown in place: the result owns the mapping
            res->table = C.tv->used ? (int32_t *)C.tv->base : nullptr;
            res->vm = tv_guard.release();
            C.tv = nullptr;
        } else if (C.pieces.size() == 1) {
            res->table = C.pieces[0].first;
        } else if (!C.pieces.empty()) {
            GSI_CUDA(cudaMallocAsync(&res->table, 4ull * C.count * k, st));
            unsigned long long off = 0;
            for (auto &p : C.pieces) {
                GSI_CUDA(cudaMemcpyAsync(res->table + off * k, p.first, 4ull * p.second * k,
                                         cudaMemcpyDeviceToDevice, st));
                off += p.second;
                cudaFreeAsync(p.first, st);
            }
        }
        C.pieces.clear();
    }
    GSI_CUDA(sync_timed(S, st));
    prof.finish(&S);
    S.ms_host_alloc = (float)A.ms_alloc;
    S.count = res->count;
    S.ms_join = (float)(now_ms() - t_plan);
    S.ms_total = (float)(now_ms() - t_start);
    *out = res.release();
    return GSI_OK;
}

}  // namespace gsi

// ====================================================================== batch ==========
// Independent queries run concurrently: `conc` host workers, each with its own stream and
// workspace slot, pull queries in order; the device interleaves their kernels, so one
// query's host round trips (a count read back per level) and tiny levels overlap with
// another's large ones.  Each query's memory budget is the device budget / conc.
namespace gsi {
gsi_status run_batch_impl(const gsi_graph *g, int32_t nq, const gsi_prepared *const *qs,
                          const gsi_query_opts *opts_in, int32_t conc, gsi_result **out) {
    if (!g || nq < 0 || (nq > 0 && (!qs || !out))) {
        set_error("invalid batch arguments");
        return GSI_ERR_INVALID_ARG;
    }
    for (int i = 0; i < nq; i++) out[i] = nullptr;
    if (nq == 0) return GSI_OK;
    gsi_query_opts base;
    gsi_query_opts_default(&base);
    if (opts_in) base = *opts_in;
    const int T = std::max(1, std::min<int>(std::min(conc, nq), kWsSlots));
    GSI_CUDA(cudaSetDevice(g->device));
    if (!base.mem_budget_bytes)
        base.mem_budget_bytes = (unsigned long long)(0.85 * (double)(available_bytes(g->device) +
                                                                     workspace_idle_bytes(g->device)) / T);
    std::vector<gsi_status> rc(nq, GSI_OK);
    std::vector<std::string> err(nq);
    std::atomic<int> next{0};
    auto worker = [&]() {
        cudaSetDevice(g->device);
        cudaStream_t s = nullptr;
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            s = nullptr;
        }
        gsi_query_opts o = base;
        if (s) o.stream = s;
        for (;;) {
            const int i = next.fetch_add(1);
            if (i >= nq) break;
            rc[i] = run_impl(g, qs[i], &o, &out[i]);
            if (rc[i] != GSI_OK) err[i] = gsi_last_error_str();
        }
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    };
    if (T == 1) {
        worker();
    } else {
        std::vector<std::thread> th;
        for (int w = 0; w < T; w++) th.emplace_back(worker);
        for (auto &t : th) t.join();
    }
    for (int i = 0; i < nq; i++)
        if (rc[i] != GSI_OK) {
            for (int j = 0; j < nq; j++) {
                delete out[j];
                out[j] = nullptr;
            }
            set_error("query " + std::to_string(i) + " of the batch: " + err[i]);
            return rc[i];
        }
    return GSI_OK;
}
}  // namespace gsi

// ====================================================================== debug filter ===
namespace gsi {
gsi_status debug_filter_prepared_impl(const gsi_prepared *p, int32_t mode, uint32_t *bitmaps, int64_t *counts);

gsi_status debug_filter_impl(const gsi_graph *g, int32_t k, const int32_t *qvl, int32_t qm, const int32_t *qs,
                             const int32_t *qd, const int32_t *qe, int32_t mode, uint32_t *bitmaps, int64_t *counts) {
    gsi_prepared *pp = nullptr;
    GSI_TRY(prepare_impl(g, k, qvl, qm, qs, qd, qe, &pp));
    std::unique_ptr<gsi_prepared> p(pp);
    return debug_filter_prepared_impl(p.get(), mode, bitmaps, counts);
}

gsi_status debug_filter_prepared_impl(const gsi_prepared *p, int32_t mode, uint32_t *bitmaps, int64_t *counts) {
    const gsi_graph *g = p->g;
    const int k = p->k;
    GSI_CUDA(cudaSetDevice(p->device));
    cudaStream_t st = cudaStreamPerThread;
    const long long n = g->n, words = (n + 31) / 32;
    ensure_pool(p->device);
    Arena A(st);
    uint32_t *bm = nullptr;
    unsigned long long *cnt = nullptr;
    Counters *ctr = nullptr;
    GSI_TRY(A.get(&bm, (unsigned long long)words * k));
    GSI_TRY(A.get(&cnt, k));
    GSI_TRY(A.get(&ctr, 1));
    GSI_CUDA(cudaMemsetAsync(cnt, 0, 8ull * k, st));
    GSI_CUDA(cudaMemsetAsync(ctr, 0, sizeof(Counters), st));
    const uint32_t *qsig = p->d_qsig + (mode == 2 ? (size_t)k * kPlanes : 0);   // 2: homomorphism encoding
    if (g->ml)
        GSI_CUDA(launch_filter_ml(g, p, mode == 2, bm, words, cnt, st));
    else
        GSI_CUDA(launch_filter(g->sig, n, k, qsig, mode == 1, bm, words, cnt, ctr, nullptr, 0, 148, st));
    if (bitmaps && words)
        GSI_CUDA(cudaMemcpyAsync(bitmaps, bm, 4ull * words * k, cudaMemcpyDeviceToHost, st));
    std::vector<unsigned long long> hc(k);
    GSI_CUDA(cudaMemcpyAsync(hc.data(), cnt, 8ull * k, cudaMemcpyDeviceToHost, st));
    GSI_CUDA(cudaStreamSynchronize(st));
    GSI_CUDA(cudaGetLastError());
    for (int u = 0; u < k; u++)
        if (counts) counts[u] = (int64_t)hc[u];
    return GSI_OK;
}
}  // namespace gsi
