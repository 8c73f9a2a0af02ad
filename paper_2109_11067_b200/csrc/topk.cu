// topk.cu — K4: single-pass top-K (detail::topk_candidates, mcts.hpp:56-76) for k <= 32.
//
// The reference scores every candidate, keeps s > 0, sorts by candidate_preferred
// (greedy.hpp:63-67) and truncates to K.  That order is total, so the top-K is built
// here in one pass with a WARP-DISTRIBUTED sorted list: lane r of a warp holds the r-th
// best candidate seen so far.  Each batch of 32 rows (one per lane) is scored, filtered
// against the current K-th best with one ballot, and the few survivors are inserted by
// rank (ballot+popc) and a shfl_up shift — O(1) warp instructions per insertion and no
// per-thread serial insertion sort.  Warp lists are merged by warp 0 of each CTA through
// shared memory, CTA lists by the last CTA to finish (atomic ticket): one launch, no grid
// barrier, no cooperative launch.  MCTS calls this on every rollout-cache miss and every
// expansion, so latency is the figure of merit.
#include "common.cuh"

namespace mgb {

namespace {

constexpr int kTopkThreads = 256;
constexpr int kTopkWarps = kTopkThreads / 32;
constexpr int kRowsPerThread = 8;  // the host sizes the grid so every row has a thread slot
constexpr int kCandCap = 1024;     // per-CTA candidates above the threshold held in smem

__device__ __forceinline__ unsigned lane() { return threadIdx.x & 31u; }

// candidate_preferred on (score, util_sum, row); "none" (row == kNoRow, s == 0) loses to all.
__device__ __forceinline__ bool pref(const DevModel& M, const Best& a, const Best& b) { return dev::better(M, a, b); }
__device__ __forceinline__ Best nil() { return dev::none(); }

__device__ __forceinline__ Best shfl(const Best& b, int src) {
    return Best{__shfl_sync(0xffffffffu, b.s, src), __shfl_sync(0xffffffffu, b.u, src),
                __shfl_sync(0xffffffffu, b.row, src)};
}

__device__ __forceinline__ Best shfl_up1(const Best& b) {
    return Best{__shfl_up_sync(0xffffffffu, b.s, 1), __shfl_up_sync(0xffffffffu, b.u, 1),
                __shfl_up_sync(0xffffffffu, b.row, 1)};
}

// Offer one candidate per lane (valid lanes only) to the warp list `wl` (lane r = rank r,
// r < k).  Candidates must be distinct rows.
__device__ __forceinline__ void warp_offer(const DevModel& M, Best& wl, const Best& c, bool valid, int k) {
    const Best kth = shfl(wl, k - 1);
    unsigned todo = __ballot_sync(0xffffffffu, valid && pref(M, c, kth));
    while (todo) {
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
        const Best x = shfl(c, src);
        const bool ahead = static_cast<int>(lane()) < k && pref(M, wl, x);
        const int rank = __popc(__ballot_sync(0xffffffffu, ahead));
        if (rank >= k) continue;
        const Best up = shfl_up1(wl);
        if (static_cast<int>(lane()) > rank && static_cast<int>(lane()) < k) wl = up;
        if (static_cast<int>(lane()) == rank) wl = x;
    }
}

}  // namespace

__global__ void __launch_bounds__(kTopkThreads, 1) topk1_kernel(const __grid_constant__ Topk1Args a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const DevModel& M = a.M;
    const int nW = (M.n + 1) * M.PP;
    double* W = reinterpret_cast<double*>(smem);
    double* comp = W + nW;
    Best* wlist = reinterpret_cast<Best*>(comp + M.n + 1);  // [warps][32]
    Best* cand = wlist + kTopkWarps * 32;                    // [kCandCap]
    __shared__ double thr[kTopkThreads];
    __shared__ int n_cand;
    __shared__ uint64_t mask[4];
    __shared__ bool last;
    const int k = a.k;
    for (int i = threadIdx.x; i < M.n; i += blockDim.x) comp[i] = a.comp[i];
    if (threadIdx.x < 4) mask[threadIdx.x] = a.svc_mask ? a.svc_mask[threadIdx.x] : ~0ull;
    __syncthreads();
    for (int e = threadIdx.x; e < nW; e += blockDim.x) {  // W = need * U (greedy.hpp:38-41)
        const int svc = e / M.PP;
        double w = 0.0;
        if (svc < M.n) {
            const double need = __dadd_rn(1.0, -comp[svc]);
            if (need > 0.0) w = __dmul_rn(need, __ldg(&M.U[e]));
        }
        W[e] = w;
    }
    __syncthreads();

    // Pass 1: every thread scores its (<= kRowsPerThread) rows into registers.
    const int warp = threadIdx.x >> 5;
    const long long total = a.index ? a.n_index : a.n_rows;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    uint64_t myrow[kRowsPerThread];
    double mys[kRowsPerThread];
    double tmax = 0.0;
#pragma unroll
    for (int r = 0; r < kRowsPerThread; ++r) {
        const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x + r * stride;
        mys[r] = 0.0;
        myrow[r] = kNoRow;
        if (i < total) {
            const uint64_t row = __ldg(a.rows + (a.index ? a.index[i] : i));
            bool ok = true;
            if (a.svc_mask) {
                bool hit = false;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int svc = static_cast<int>(((row >> (16 * j)) & 0xFFFFull) / M.PP);
                    if (svc < M.n) hit |= ((mask[svc >> 6] >> (svc & 63)) & 1ull) != 0;
                }
                ok = hit;
            }
            if (ok) {  // score, greedy.hpp:36-43 (ascending members, no FMA)
                double s = __dadd_rn(W[row & 0xFFFFull], W[(row >> 16) & 0xFFFFull]);
                s = __dadd_rn(s, W[(row >> 32) & 0xFFFFull]);
                s = __dadd_rn(s, W[row >> 48]);
                if (s > 0.0) {
                    mys[r] = s;
                    myrow[r] = row;
                    tmax = fmax(tmax, s);
                }
            }
        }
    }
    // Threshold: T = the k-th largest per-thread maximum in this CTA.  At least k rows of
    // the CTA score >= T, so the CTA's exact top-k lies among its rows with s >= T.
    thr[threadIdx.x] = tmax;
    if (threadIdx.x == 0) n_cand = 0;
    __syncthreads();
    for (int k2 = 2; k2 <= kTopkThreads; k2 <<= 1)  // bitonic sort, descending
        for (int j = k2 >> 1; j > 0; j >>= 1) {
            const int t = threadIdx.x, p = t ^ j;
            if (p > t) {
                const double x = thr[t], y = thr[p];
                if (((t & k2) == 0) ? (x < y) : (x > y)) {
                    thr[t] = y;
                    thr[p] = x;
                }
            }
            __syncthreads();
        }
    const double T = thr[k - 1];
#pragma unroll
    for (int r = 0; r < kRowsPerThread; ++r)
        if (myrow[r] != kNoRow && mys[r] >= T) {
            const int at = atomicAdd(&n_cand, 1);
            if (at < kCandCap) cand[at] = Best{mys[r], 0.0, myrow[r]};
        }
    __syncthreads();
    const int nc = n_cand;
    if (warp == 0) {
        Best bl = nil();
        if (nc <= kCandCap) {  // exact top-k of the candidates (warp-distributed insertion)
            for (int b0 = 0; b0 < nc; b0 += 32) {
                const int i = b0 + static_cast<int>(lane());
                Best c = i < nc ? cand[i] : nil();
                if (i < nc) c.u = dev::row_usum(M.U, c.row);
                warp_offer(M, bl, c, i < nc, k);
            }
        }
        wlist[lane()] = bl;
    }
    if (nc > kCandCap) {  // pathological ties at T: every warp offers all its rows (exact)
        Best wl = nil();
#pragma unroll
        for (int r = 0; r < kRowsPerThread; ++r) {
            Best c{mys[r], 0.0, myrow[r]};
            const bool ok = myrow[r] != kNoRow;
            if (ok) c.u = dev::row_usum(M.U, c.row);
            warp_offer(M, wl, c, ok, k);
        }
        __syncthreads();
        wlist[warp * 32 + lane()] = wl;
    }
    __syncthreads();
    if (warp == 0) {
        Best bl = wlist[lane()];
        if (nc > kCandCap)
            for (int w = 1; w < kTopkWarps; ++w) {
                const Best c = wlist[w * 32 + lane()];
                warp_offer(M, bl, c, static_cast<int>(lane()) < k && c.row != kNoRow, k);
            }
        if (gridDim.x == 1) {
            const bool v = static_cast<int>(lane()) < k && bl.row != kNoRow;
            const unsigned valid = __ballot_sync(0xffffffffu, v);
            if (v) a.out_row[lane()] = bl.row;
            if (lane() == 0) *a.n_out = __popc(valid);
        } else {
            a.partials[blockIdx.x * 32 + lane()] = bl;
            __threadfence();
            unsigned t = 0;
            if (lane() == 0) t = atomicAdd(a.ticket, 1u);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (lane() == 0) last = (t == gridDim.x - 1);
        }
    }
    if (gridDim.x == 1) return;
    __syncthreads();
    if (!last || warp != 0) return;
    __threadfence();
    Best gl = nil();
    for (unsigned b = 0; b < gridDim.x; ++b) {  // last CTA merges the per-CTA lists
        const Best* p = &a.partials[b * 32 + lane()];
        const Best c{__ldcg(&p->s), __ldcg(&p->u), __ldcg(reinterpret_cast<const unsigned long long*>(&p->row))};
        warp_offer(M, gl, c, static_cast<int>(lane()) < k && c.row != kNoRow, k);
    }
    const bool v = static_cast<int>(lane()) < k && gl.row != kNoRow;
    const unsigned valid = __ballot_sync(0xffffffffu, v);
    if (v) a.out_row[lane()] = gl.row;
    if (lane() == 0) {
        *a.n_out = __popc(valid);
        *a.ticket = 0;
    }
}

size_t topk1_smem_bytes(int n, int PP, int) {
    return static_cast<size_t>((n + 1) * PP + n + 1) * 8 +
           static_cast<size_t>(kTopkWarps * 32 + kCandCap) * sizeof(Best);
}
int topk1_threads() { return kTopkThreads; }
int topk1_rows_per_cta() { return kTopkThreads * kRowsPerThread; }
int topk1_max_k() { return 32; }
const void* topk1_kernel_ptr(int) { return reinterpret_cast<const void*>(&topk1_kernel); }

}  // namespace mgb
