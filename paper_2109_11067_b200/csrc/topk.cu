// topk.cu — K4: single-launch top-K (detail::topk_candidates, mcts.hpp:56-76) for k <= 32.
//
// The reference scores every candidate, keeps s > 0, sorts by candidate_preferred
// (greedy.hpp:63-67) and truncates to K.  That order is total, so only the few rows that
// can reach the top K need to be ordered at all:
//   1. every thread scores its rows of the CTA's chunk and keeps its maximum;
//   2. every warp sorts its 32 per-lane maxima (bitonic, shuffles only) and takes the K-th
//      largest; the CTA threshold T is the largest such value over the warps — at least K
//      rows of the CTA score >= T, so the CTA's exact top-K lies among its rows >= T;
//   3. a second pass over the (cache-hot) chunk sends those few rows to shared memory,
//      where they are ranked IN PARALLEL (thread i counts the
//      candidates preferred to candidate i): no serial insertion, no block-wide sort;
//   4. with more than one CTA, the last CTA to finish (atomic ticket) ranks the G x K
//      per-CTA winners the same way.
// One launch, no grid barrier, no cooperative launch.  MCTS calls this on every
// rollout-cache miss and every expansion, so latency is the figure of merit.
// A CTA whose rows tie at T beyond the candidate capacity reports overflow (*n_out = -1)
// and the host re-runs the exact k-round kernel (kernels.cu) — a pathological case.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace mgb {

namespace {

constexpr int kTopkThreads = 256;
constexpr int kTopkWarps = kTopkThreads / 32;
constexpr int kCandCap = 2048;      // per-CTA candidates (and merged per-CTA winners) in smem
constexpr int kTopkMaxK = 32;

using dev::Cand;
using dev::rank_select;
using dev::warp_kth;

}  // namespace

__global__ void __launch_bounds__(kTopkThreads, 1) topk1_kernel(const __grid_constant__ Topk1Args a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const DevModel& M = a.M;
    const int nW = (M.n + 1) * M.PP;
    double* W = reinterpret_cast<double*>(smem);
    Cand* cand = reinterpret_cast<Cand*>(W + nW + 1);  // [kCandCap]
    Cand* win = cand + kCandCap;                        // [kTopkMaxK]
    __shared__ unsigned long long t_bits;
    __shared__ int n_cand, n_got, cta_scored;
    const int k = a.k;
    if (threadIdx.x == 0) {
        t_bits = 0ull;
        n_cand = 0;
        cta_scored = 0;
    }
    for (int e = threadIdx.x; e < nW; e += blockDim.x) {  // W = need * U (greedy.hpp:38-41)
        const int svc = svc_of(M, static_cast<unsigned>(e));
        double w = 0.0;
        if (svc < M.n) {
            const double need = __dadd_rn(1.0, -a.comp[svc]);
            if (need > 0.0) w = __dmul_rn(need, __ldg(&M.U[e]));
        }
        W[e] = w;
    }
    __syncthreads();

    // 1. this CTA's chunk (coalesced: consecutive threads, consecutive rows); a compact loop,
    //    so the launch does not stream a large unrolled body through the instruction cache
    const long long total = a.index ? a.n_index : a.n_rows;
    const long long lo = static_cast<long long>(blockIdx.x) * a.rows_per_cta;
    const long long hi = min(total, lo + a.rows_per_cta);
    int scored = 0;  // candidates actually scored (a service-mask filter defines the set)
    auto score_at = [&](long long i, uint64_t& row) -> double {
        row = __ldg(a.rows + (a.index ? __ldg(a.index + i) : i));
        if (a.use_mask) {
            bool hit = false;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int svc = static_cast<int>(((row >> (16 * j)) & 0xFFFFull) / M.PP);
                if (svc < M.n) hit |= ((a.svc_mask[svc >> 6] >> (svc & 63)) & 1ull) != 0;
            }
            if (!hit) return 0.0;
        }
        return dev::row_score(W, row);  // score, greedy.hpp:36-43 (ascending members, no FMA)
    };
    double tmax = 0.0;
#pragma unroll 4
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        uint64_t row;
        tmax = fmax(tmax, score_at(i, row));
        if (a.use_mask) {
            bool hit = false;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int svc = static_cast<int>(((row >> (16 * j)) & 0xFFFFull) / M.PP);
                if (svc < M.n) hit |= ((a.svc_mask[svc >> 6] >> (svc & 63)) & 1ull) != 0;
            }
            scored += hit;
        }
    }
    if (a.use_mask) {  // expand's candidate set = rows touching a sampled service (mcts.hpp:98-107)
        for (int off = 16; off > 0; off >>= 1) scored += __shfl_xor_sync(0xffffffffu, scored, off);
        if ((threadIdx.x & 31u) == 0 && scored) atomicAdd(&cta_scored, scored);  // shared: summed by rank 0
    }
    // 2. threshold: the largest per-warp K-th lane maximum (non-negative doubles order as
    //    their bit patterns, so an integer atomicMax on the bits is a max on the values)
    const double tw = warp_kth(tmax, k);
    if ((threadIdx.x & 31u) == 0) atomicMax(&t_bits, static_cast<unsigned long long>(__double_as_longlong(tw)));
    __syncthreads();
    const double T = __longlong_as_double(static_cast<long long>(t_bits));
    // 3. collect rows >= T (warp-aggregated appends; L1/L2-hot second read), then rank them
    for (long long i0 = lo; i0 < hi; i0 += blockDim.x) {
        const long long i = i0 + threadIdx.x;
        uint64_t row = 0;
        const double sc = i < hi ? score_at(i, row) : 0.0;
        const bool take = sc > 0.0 && sc >= T;
        const unsigned b = __ballot_sync(0xffffffffu, take);
        if (b) {
            int at = 0;
            if ((threadIdx.x & 31u) == 0) at = atomicAdd(&n_cand, __popc(b));
            at = __shfl_sync(0xffffffffu, at, 0) + __popc(b & dev::lanemask_lt());
            if (take && at < kCandCap) cand[at] = Cand{sc, 0.0, row, i};
        }
    }
    __syncthreads();
    const int nc_raw = n_cand;
    if (nc_raw > kCandCap && gridDim.x == 1) {  // pathological ties at T: the host re-runs the exact k-round kernel
        if (threadIdx.x == 0) *a.n_out = -1;
        return;
    }
    const int nc = min(nc_raw, kCandCap);
    for (int i = threadIdx.x; i < nc; i += blockDim.x) cand[i].u = dev::row_usum(M.U, cand[i].row);
    __syncthreads();
    const int got = nc_raw > kCandCap ? 0 : min(nc, k);
    if (nc_raw <= kCandCap) rank_select_warp(M, cand, nc, k, win);
    __syncthreads();
    if (gridDim.x == 1) {
        if (threadIdx.x < got) a.out_row[threadIdx.x] = win[threadIdx.x].row;
        if (threadIdx.x == 0) {
            *a.n_out = got;
            if (a.use_mask) *a.n_scored = static_cast<unsigned long long>(cta_scored);  // one host write
        }
        return;
    }
    // 4. cluster merge over distributed shared memory: the grid is ONE thread-block cluster;
    //    CTA 0 reads every CTA's K winners straight from their shared memory (no global
    //    round trip, no atomics), ranks those above the merge threshold and writes the answer.
    if (threadIdx.x == 0) n_got = nc_raw > kCandCap ? -1 : got;  // -1: this CTA overflowed
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    if (cluster.block_rank() == 0) {
        const int nb = static_cast<int>(cluster.num_blocks());
        __shared__ int overflow;
        if (threadIdx.x == 0) {
            n_cand = 0;
            t_bits = 0ull;
            overflow = 0;
        }
        __syncthreads();
        // merge threshold: every CTA with a full list holds K rows scoring >= its K-th score
        for (int r = threadIdx.x; r < nb; r += blockDim.x) {
            const int rg = *cluster.map_shared_rank(&n_got, r);
            if (rg < 0) overflow = 1;
            if (rg == k) {
                const Cand* rw = cluster.map_shared_rank(win, r);
                atomicMax(&t_bits, static_cast<unsigned long long>(__double_as_longlong(rw[k - 1].s)));
            }
        }
        __syncthreads();
        const double TM = __longlong_as_double(static_cast<long long>(t_bits));
        Cand* mc_list = cand;  // own candidates are no longer needed
        for (int i = threadIdx.x; i < nb * k; i += blockDim.x) {
            const int r = i / k, q = i % k;
            if (q >= *cluster.map_shared_rank(&n_got, r)) continue;
            const Cand c = cluster.map_shared_rank(win, r)[q];
            if (c.s < TM) continue;
            const int at = atomicAdd(&n_cand, 1);
            // CTA chunks are disjoint and ascending, so (CTA, rank) orders duplicates by position
            if (at < kCandCap) mc_list[at] = Cand{c.s, c.u, c.row, static_cast<long long>(i)};
        }
        __syncthreads();
        const int mc = min(n_cand, kCandCap);
        Cand* out = win + kTopkMaxK;  // spare list after this CTA's own winners
        rank_select_warp(M, mc_list, mc, k, out);
        __syncthreads();
        const int mgot = min(mc, k);
        if (threadIdx.x < mgot) a.out_row[threadIdx.x] = out[threadIdx.x].row;
        if (threadIdx.x == 0) {
            *a.n_out = (overflow || n_cand > kCandCap) ? -1 : mgot;
            if (a.use_mask) {  // one host write for the whole cluster
                unsigned long long tot = 0;
                for (int r = 0; r < nb; ++r) tot += static_cast<unsigned long long>(*cluster.map_shared_rank(&cta_scored, r));
                *a.n_scored = tot;
            }
        }
    }
    cluster.sync();  // peers' shared memory stays alive until rank 0 has read it
}

size_t topk1_smem_bytes(int n, int PP, int) {
    return static_cast<size_t>((n + 1) * PP + 1) * 8 + static_cast<size_t>(kCandCap + 2 * kTopkMaxK) * sizeof(Cand);
}
int topk1_threads() { return kTopkThreads; }
int topk1_rows_per_cta() { return 1024; }
int topk1_max_k() { return kTopkMaxK; }
int topk1_max_ctas() { return 16; }  // one thread-block cluster (non-portable size 16)
const void* topk1_kernel_ptr(int) { return reinterpret_cast<const void*>(&topk1_kernel); }

}  // namespace mgb
