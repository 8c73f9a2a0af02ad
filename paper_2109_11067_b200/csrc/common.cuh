// common.cuh — device helpers shared by the sm_100a kernels (kernels.cu, topk.cu).
#pragma once

#include <cuda/atomic>

#include "device.cuh"

namespace mgb {
namespace dev {

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() { return (1u << lane_id()) - 1u; }
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// 128-bit lexicographic GpuConfig key (core.hpp:174-200): per normalized instance
// (slices asc, slot asc) a 15-bit field present|slices|slot|svc; shorter sorts first.
// The row's layout is the sum of its members' count patterns; within a size group the
// lower service index holds the lower slots (config_enum.hpp:140,159-163).
static __device__ __noinline__ void row_key(const DevModel& M, uint64_t row, uint64_t& hi, uint64_t& lo) {
    // members (ascending services): (service, pattern) and the pattern's packed size counts
    int svc[4], k = 0;
    uint32_t pk[4], tot = 0;
    const int sentinel = M.n * M.PP;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int code = static_cast<int>((row >> (16 * j)) & 0xFFFFull);
        if (code == sentinel) break;
        const unsigned e = M.key_code[code];
        svc[k] = static_cast<int>(e >> 8);
        pk[k] = M.pat_packed[e & 0xFFu];
        tot += pk[k];  // <= 7 instances per size: no carries between the 3-bit fields
        ++k;
    }
    const int L = M.layout_of[tot & 0x7FFFu];  // the row's layout is the sum of its members' patterns
    unsigned __int128 key = 0;
    int ninst = 0;
    for (int si = 0; si < M.n_sizes; ++si) {
        int t = 0;
        for (int j = 0; j < k; ++j) {  // within a size group the lower service holds the lower slots
            const int c = static_cast<int>((pk[j] >> (3 * si)) & 7u);
            for (int q = 0; q < c; ++q, ++t) {
                const unsigned slot = static_cast<unsigned>(M.layout_slots[(L * 5 + si) * 7 + t]);
                key = (key << 15) | ((1u << 14) | (static_cast<unsigned>(M.sizes[si]) << 11) | (slot << 8) |
                                     static_cast<unsigned>(svc[j]));
                ++ninst;
            }
        }
    }
    for (; ninst < 7; ++ninst) key <<= 15;
    hi = static_cast<uint64_t>(key >> 64);
    lo = static_cast<uint64_t>(key);
}

// Third key of candidate_preferred; reached only on exact (score, util_sum) ties.
#ifdef MGB_GREEDY_STEP_DIAG
__device__ unsigned g_sd_keys[1024];
#endif
static __device__ __noinline__ bool row_key_less(const DevModel& M, uint64_t a, uint64_t b) {
#ifdef MGB_GREEDY_STEP_DIAG
    atomicAdd(&g_sd_keys[blockIdx.x], 1u);
#endif
    uint64_t ah, al, bh, bl;
    row_key(M, a, ah, al);
    row_key(M, b, bh, bl);
    return ah != bh ? ah < bh : al < bl;
}

__device__ __forceinline__ Best none() { return Best{0.0, 0.0, kNoRow}; }

// candidate_preferred (greedy.hpp:63-67) on (score, util_sum, row); none loses to all.
__device__ __forceinline__ bool better(const DevModel& M, const Best& a, const Best& b) {
    if (a.s != b.s) return a.s > b.s;
    if (a.row == kNoRow || b.row == kNoRow || a.row == b.row) return false;
    if (a.u != b.u) return a.u > b.u;
    return row_key_less(M, a.row, b.row);
}

// util_sum (config_enum.hpp:173): ascending members from 0.0; U may be smem or global.
__device__ __forceinline__ double row_usum(const double* U, uint64_t row) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) s = __dadd_rn(s, U[(row >> (16 * j)) & 0xFFFFull]);
    return s;
}

// score (greedy.hpp:36-43) with W = need*U precomputed (0 where need <= 0).  Members are
// in ascending service order and unused positions hit a zero cell, so the sum order and
// every rounding step equal the reference's.
__device__ __forceinline__ double row_score(const double* __restrict__ W, uint64_t row) {
    double s = __dadd_rn(W[row & 0xFFFFull], W[(row >> 16) & 0xFFFFull]);
    s = __dadd_rn(s, W[(row >> 32) & 0xFFFFull]);
    return __dadd_rn(s, W[row >> 48]);
}

__device__ __forceinline__ Best shfl_xor_best(const Best& b, int off) {
    return Best{__shfl_xor_sync(0xffffffffu, b.s, off), __shfl_xor_sync(0xffffffffu, b.u, off),
                __shfl_xor_sync(0xffffffffu, b.row, off)};
}

// Lane holding the smallest config key among the `tied` lanes (rows tied on score and
// util_sum): every tied lane computes its own key once, in parallel (a call: the keys' table
// loads stay out of the caller's register budget).
static __device__ __noinline__ int warp_key_argmin(const DevModel& M, uint64_t row, bool tied) {
    const int lane = static_cast<int>(lane_id());
    uint64_t kh = ~0ull, kl = ~0ull;
    if (tied) row_key(M, row, kh, kl);
    int ln = tied ? lane : 32;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const uint64_t oh = __shfl_xor_sync(0xffffffffu, kh, off), ol = __shfl_xor_sync(0xffffffffu, kl, off);
        const int on = __shfl_xor_sync(0xffffffffu, ln, off);
        if (oh < kh || (oh == kh && (ol < kl || (ol == kl && on < ln)))) kh = oh, kl = ol, ln = on;
    }
    return ln;
}

// The warp's best under candidate_preferred, in every lane.  The butterfly orders by
// (score, util_sum) and, on equal pairs, by the raw row bits — cheap, but not the reference's
// third key — so when lanes holding DISTINCT rows tie with the winner on both, the config key
// decides among them: each tied lane computes its key once, in parallel, instead of two keys
// per tied pair at each of the five levels (tie-heavy greedy steps of slos_24 spent up to
// 25 us per step in serial key compares: tools/ab/diag.so, MGB_GREEDY_STEP_DIAG).
#ifdef MGB_OLD_WARP_BEST
__device__ __forceinline__ Best warp_best(const DevModel& M, Best b) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        Best o = shfl_xor_best(b, off);
        if (better(M, o, b)) b = o;
    }
    return b;
}
#else
__device__ __forceinline__ Best warp_best(const DevModel& M, Best b) {
    Best w = b;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const Best o = shfl_xor_best(w, off);
        if (o.s > w.s || (o.s == w.s && (o.u > w.u || (o.u == w.u && o.row < w.row)))) w = o;
    }
    if (w.row == kNoRow) return none();
    const bool tied = b.row != kNoRow && b.s == w.s && b.u == w.u;
    if (__any_sync(0xffffffffu, tied && b.row != w.row)) {
        const int src = warp_key_argmin(M, b.row, tied);
        w = Best{__shfl_sync(0xffffffffu, b.s, src), __shfl_sync(0xffffffffu, b.u, src), __shfl_sync(0xffffffffu, b.row, src)};
    }
    return w;
}
#endif

// Generation barrier across all co-resident (cooperatively launched) CTAs.  The CTA's
// writes are ordered before thread 0's arrival by bar.sync + a gpu-scope acq_rel fence
// (cumulative); the wait is an acquire load.  Data produced by other CTAs is read after the
// barrier with L2-coherent loads (ld.global.cg), never through the non-coherent path.
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> g(*gen), c(*count);
        const unsigned my = g.load(cuda::memory_order_relaxed);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (c.fetch_add(1u, cuda::memory_order_acq_rel) == nblocks - 1u) {
            c.store(0u, cuda::memory_order_relaxed);
            g.store(my + 1u, cuda::memory_order_release);
        } else {
            while (g.load(cuda::memory_order_acquire) == my) {
            }
        }
    }
    __syncthreads();
}

// ---- exact top-K by parallel ranking (topk.cu, rollout.cu)

struct Cand {
    double s, u;
    uint64_t row;
    long long pos;  // position in the candidate set: orders duplicate rows of an explicit list
};

// candidate i is preceded by j: preferred (greedy.hpp:63-67), or the same row earlier in
// the candidate list (duplicates of an explicit `from` list are both kept, mcts.hpp:59-67).
__device__ __forceinline__ bool precedes(const DevModel& M, const Cand& j, const Cand& i) {
    if (j.s != i.s) return j.s > i.s;
    if (j.row == i.row) return j.pos < i.pos;
    if (j.u != i.u) return j.u > i.u;
    return row_key_less(M, j.row, i.row);
}

// Rank the first `nc` entries of `cand` (all threads) and write the K best, in order, to
// out[0..min(K, nc)).  Ranks are distinct because `precedes` is a strict total order.
__device__ __forceinline__ void rank_select(const DevModel& M, const Cand* cand, int nc, int k, Cand* out) {
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
        const Cand ci = cand[i];
        int r = 0;
        for (int j = 0; j < nc && r < k; ++j) r += precedes(M, cand[j], ci) ? 1 : 0;
        if (r < k) out[r] = ci;
    }
}

// rank_select with a warp per candidate: the lanes compare it against 32 others at a time
// and count with a ballot (a block-wide call; same output as rank_select).
__device__ __forceinline__ void rank_select_warp(const DevModel& M, const Cand* cand, int nc, int k, Cand* out) {
    const int lane = static_cast<int>(threadIdx.x & 31u);
    const int nw = static_cast<int>(blockDim.x >> 5);
    for (int i = static_cast<int>(threadIdx.x >> 5); i < nc; i += nw) {
        const Cand ci = cand[i];
        int r = 0;
        for (int j0 = 0; j0 < nc && r < k; j0 += 32) {
            const int j = j0 + lane;
            r += __popc(__ballot_sync(0xffffffffu, j < nc && precedes(M, cand[j], ci)));
        }
        if (lane == 0 && r < k) out[r] = ci;
    }
}

// K-th largest (k <= 32) of the warp's lane values: bitonic sort descending over shuffles.
__device__ __forceinline__ double warp_kth(double v, int k) {
    const int lane = static_cast<int>(threadIdx.x & 31u);
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int j = size >> 1; j > 0; j >>= 1) {
            const double o = __shfl_xor_sync(0xffffffffu, v, j);
            const bool desc = (lane & size) == 0 || size == 32;
            const bool low = (lane & j) == 0;
            v = (low == desc) ? fmax(v, o) : fmin(v, o);
        }
    }
    return __shfl_sync(0xffffffffu, v, k - 1);
}

}  // namespace dev
}  // namespace mgb
