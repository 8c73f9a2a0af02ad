// rollout.cu — K5: throughput-mode root-parallel MCTS rollouts, one rollout per warp.
//
// The reference's rollout (mcts.hpp:122-143) completes a partial deployment by repeatedly
// picking a uniformly random candidate among the top-K of the BASE pool under the current
// completion vector, memoized by the unsatisfied-service bitmap (completion_type_key,
// mcts.hpp:38-43; RolloutCache mcts.hpp:47-50).  Here N rollouts from one root run
// concurrently in one persistent cooperative kernel:
//   - one warp owns one rollout at a time; lane l keeps comp[l + 32 j] in registers, the
//     type key is a handful of ballots, a pick adds <= 4 utilities in the owning lanes;
//   - draws are Philox4x32-10 (philox.cuh): draw t of rollout r is philox(seed, (t, id0+r)),
//     so the result does not depend on which warp runs which rollout, or when;
//   - the key cache is a device-wide open-addressing table shared by all rollouts;
//   - rollouts advance in LOCK-STEP ROUNDS so the memoized pools are deterministic: the pool
//     of a key first seen in round d is the top-K under the completion vector of the
//     LOWEST-indexed rollout that reached the key in round d (atomicMin claim), built by one
//     CTA after a grid barrier (the same threshold + parallel-rank top-K as topk.cu);
//   - the shortest completed rollout (ties: lowest index) is replayed at the end from the
//     (immutable) cache to emit its path.
// Per round, two launches: [build the round's new pools, CTA per key] then [pick + add +
// satisfied check + key probe, warp per rollout].  The advance kernel is separate so its small
// register footprint gives full occupancy (a step is a chain of dependent L2 round trips: more
// warps in flight is what raises its rate); kernel boundaries replace the grid barriers.
// oracle/oracle.cpp (`rollouts_restated`) restates exactly this schedule on the CPU.
#include <cuda/atomic>

#include "common.cuh"
#include "philox.cuh"
#define MGB_TOPK_DENSE_PCT 100  // A/B (MIGPLAN_ROLLOUT_DENSE_PCT): by-support scans for every build
#include "topk_pair.cuh"

namespace mgb {

using namespace dev;

namespace {

constexpr int kRThreads = 512;
constexpr int kRWarps = kRThreads / 32;
constexpr int kRCandCap = 2048;
constexpr int kRMaxK = 32;
constexpr int kMaxJ = 8;  // comp registers per lane: n <= 256 (J = 2 instantiation for n <= 64)
constexpr int kAThreads = 256;  // advance kernel: small blocks, register-lean, many warps per SM
#ifndef MGB_ROLLOUT_AOCC
#define MGB_ROLLOUT_AOCC 6
#endif
constexpr int kAOcc = MGB_ROLLOUT_AOCC;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// Find (or, with `insert`, create) the slot of key kw[0..nk).  Lane-0 code.
// Returns the slot, -1 (absent, !insert) or -2 (table full).
__device__ long long probe(const RolloutArgs& a, const uint64_t* kw, int nk, bool insert, bool& created) {
    uint64_t h = 0x9e3779b97f4a7c15ull;
    for (int w = 0; w < nk; ++w) h = mix64(h ^ kw[w]);
    unsigned s = static_cast<unsigned>(h) & a.tab_mask;
    created = false;
    for (unsigned t = 0; t <= a.tab_mask; ++t, s = (s + 1) & a.tab_mask) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> tag(a.tag[s]);
        unsigned tg = tag.load(cuda::memory_order_acquire);
        if (tg == 0) {
            if (!insert) return -1;
            unsigned expect = 0;
            if (tag.compare_exchange_strong(expect, 1u, cuda::memory_order_acq_rel)) {
                for (int w = 0; w < 4; ++w) __stcg(&a.key[4ull * s + w], w < nk ? kw[w] : 0ull);
                tag.store(2u, cuda::memory_order_release);
                created = true;
                return s;
            }
            tg = expect;
        }
        while (tg == 1) {
            __nanosleep(20);
            tg = tag.load(cuda::memory_order_acquire);
        }
        bool eq = true;
        for (int w = 0; w < nk; ++w) eq &= __ldcg(&a.key[4ull * s + w]) == kw[w];
        if (eq) return s;
    }
    return -2;
}

// Unsatisfied-service bitmap (completion_type_key, mcts.hpp:38-43): bit i set when
// comp[i] < 1 - 1e-9 (core.hpp:18,217-221).  Warp-uniform result.
template <int J>
__device__ __forceinline__ bool type_key(const double (&c)[J], int n, uint64_t (&kw)[4]) {
    const int lane = static_cast<int>(threadIdx.x & 31u);
    bool any = false;
    for (int w = 0; w < 4; ++w) kw[w] = 0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
        if (32 * j >= n) break;
        const bool un = lane + 32 * j < n && c[j] < 1.0 - 1e-9;
        const unsigned b = __ballot_sync(0xffffffffu, un);
        kw[j >> 1] |= static_cast<uint64_t>(b) << (32 * (j & 1));
        any |= b != 0;
    }
    return any;
}

// Add the chosen candidate's utilities (add_util; mcts.hpp:139) in the owning lanes.
// Returns the lane's bitmask of modified slots (so only those are written back).
template <int J>
__device__ __forceinline__ unsigned add_row(const DevModel& M, uint64_t row, double (&c)[J]) {
    const int lane = static_cast<int>(threadIdx.x & 31u);
    unsigned dirty = 0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const int code = static_cast<int>((row >> (16 * m)) & 0xFFFFull);
        const int svc = svc_of(M, static_cast<unsigned>(code));
        if (svc < M.n && (svc & 31) == lane) {
            const double u = __ldg(&M.U[code]);
#pragma unroll
            for (int j = 0; j < J; ++j)
                if ((svc >> 5) == j) c[j] = __dadd_rn(c[j], u), dirty |= 1u << j;
        }
    }
    return dirty;
}

// Top-K of the base pool under `comp` (smem) by one CTA: W = need*U, threshold from the
// per-warp K-th lane maxima, parallel rank of the rows >= T (topk.cu), exact k-round
// fallback when ties at T overflow the candidate buffer.  Writes pool[0..got), returns got.
__device__ int block_topk(const RolloutArgs& a, const double* comp, double* W, Cand* cand, Cand* win,
                          unsigned* pool_out, int* sact) {
    const DevModel& M = a.M;
    __shared__ unsigned long long t_bits;
    __shared__ int n_cand;
    __shared__ Cand red[kRWarps];
    const int nW = (M.n + 1) * M.PP;
    const int k = a.k;
    for (int e = threadIdx.x; e < nW; e += blockDim.x) {
        const int svc = svc_of(M, static_cast<unsigned>(e));
        double w = 0.0;
        if (svc < M.n) {
            const double need = __dadd_rn(1.0, -comp[svc]);
            if (need > 0.0) w = __dmul_rn(need, __ldg(&M.U[e]));
        }
        W[e] = w;
    }
    __shared__ int s_nact;
    if (threadIdx.x == 0) {
        t_bits = 0ull;
        n_cand = 0;
        s_nact = 0;
    }
    __syncthreads();
    // pair pools: only supports with a member whose need is > 0 can hold a row scoring > 0
    const bool bysup = a.n_sup > 0;
    const int lane = static_cast<int>(threadIdx.x & 31u), wid = static_cast<int>(threadIdx.x >> 5);
    const int nwarps = static_cast<int>(blockDim.x >> 5);
    if (bysup) {
        for (int s0 = 0; s0 < a.n_sup; s0 += blockDim.x) {
            const int si = s0 + static_cast<int>(threadIdx.x);
            bool live = false;
            if (si < a.n_sup) {
                const unsigned e = __ldg(&a.sup_svc[si]);
                const int sa = static_cast<int>(e & 0xFFu), sb = static_cast<int>(e >> 8);
                live = comp[sa] < 1.0 || (sb != 0xFF && comp[sb] < 1.0);
            }
            const unsigned bm = __ballot_sync(0xffffffffu, live);
            int at = 0;
            if (lane == 0 && bm) at = atomicAdd(&s_nact, __popc(bm));
            at = __shfl_sync(0xffffffffu, at, 0) + __popc(bm & lanemask_lt());
            if (live) sact[at] = si;
        }
        __syncthreads();
    }
    const int nact = bysup ? s_nact : 0;
    double tmax = 0.0;
    if (bysup) {  // a warp per active support, lanes over its rows
        for (int i = wid; i < nact; i += nwarps) {
            const int si = sact[i];
            const int b = __ldg(&a.sup_begin[si]), e = __ldg(&a.sup_begin[si + 1]);
            for (int r = b + lane; r < e; r += 32) tmax = fmax(tmax, row_score(W, __ldg(a.base + r)));
        }
    } else {
        for (long long i = threadIdx.x; i < a.n_base; i += blockDim.x) tmax = fmax(tmax, row_score(W, __ldg(a.base + i)));
    }
    const double tw = warp_kth(tmax, k);
    if ((threadIdx.x & 31u) == 0) atomicMax(&t_bits, static_cast<unsigned long long>(__double_as_longlong(tw)));
    __syncthreads();
    const double T = __longlong_as_double(static_cast<long long>(t_bits));
    auto push = [&](bool valid, long long i) {  // warp-collective: the rows reaching T
        uint64_t row = 0;
        double s = 0.0;
        if (valid) {
            row = __ldg(a.base + i);
            s = row_score(W, row);
        }
        const bool take = valid && s > 0.0 && s >= T;
        const unsigned b = __ballot_sync(0xffffffffu, take);
        if (b) {
            int at = 0;
            if (lane == 0) at = atomicAdd(&n_cand, __popc(b));
            at = __shfl_sync(0xffffffffu, at, 0) + __popc(b & lanemask_lt());
            if (take && at < kRCandCap) cand[at] = Cand{s, row_usum(M.U, row), row, i};
        }
    };
    if (bysup) {
        for (int i = wid; i < nact; i += nwarps) {
            const int si = sact[i];
            const int b = __ldg(&a.sup_begin[si]), e = __ldg(&a.sup_begin[si + 1]);
            for (int r0 = b; r0 < e; r0 += 32) push(r0 + lane < e, r0 + lane);
        }
    } else {
        for (long long i0 = 0; i0 < a.n_base; i0 += blockDim.x) push(i0 + threadIdx.x < a.n_base, i0 + threadIdx.x);
    }
    __syncthreads();
    const int nc = n_cand;
    int got;
    if (nc <= kRCandCap) {
        got = min(nc, k);
        rank_select_warp(M, cand, nc, k, win);
    } else {  // exact: k rounds of "best row strictly after the previous pick"
        got = 0;
        Cand last{0.0, 0.0, kNoRow, -1};
        for (int r = 0; r < k; ++r) {
            Cand b{0.0, 0.0, kNoRow, -1};
            for (long long i = threadIdx.x; i < a.n_base; i += blockDim.x) {
                const uint64_t row = __ldg(a.base + i);
                const double s = row_score(W, row);
                if (!(s > 0.0)) continue;
                const Cand c{s, row_usum(M.U, row), row, i};
                if (r > 0 && !precedes(M, last, c)) continue;
                if (b.row == kNoRow || precedes(M, c, b)) b = c;
            }
            for (int off = 16; off > 0; off >>= 1) {
                const Cand o{__shfl_xor_sync(0xffffffffu, b.s, off), __shfl_xor_sync(0xffffffffu, b.u, off),
                             __shfl_xor_sync(0xffffffffu, b.row, off), __shfl_xor_sync(0xffffffffu, b.pos, off)};
                if (o.row != kNoRow && (b.row == kNoRow || precedes(M, o, b))) b = o;
            }
            if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = b;
            __syncthreads();
            Cand x = red[0];
            for (int w = 1; w < kRWarps; ++w)
                if (red[w].row != kNoRow && (x.row == kNoRow || precedes(M, red[w], x))) x = red[w];
            __syncthreads();
            if (x.row == kNoRow) break;
            if (threadIdx.x == 0) win[r] = x;
            last = x;
            ++got;
        }
    }
    __syncthreads();
    if (threadIdx.x < got) pool_out[threadIdx.x] = static_cast<unsigned>(win[threadIdx.x].pos);
    return got;
}

}  // namespace

// One warp-step of rollout r (see the file comment).  first: the start state (no pick).
// Pushes r to the next round's active list through the warp's buffer `wb` (32 entries).
template <int J>
struct Advancer {
    const RolloutArgs& a;
    long long* wb;
    unsigned long long *c_steps, *c_done, *c_cap, *c_fail;
    int lane, nk, nxt, nbuf = 0;

    __device__ void push_flush() {
        if (nbuf && lane == 0) {
            const unsigned long long at = atomicAdd(&a.cnt->n_act[nxt], static_cast<unsigned long long>(nbuf));
            for (int i = 0; i < nbuf; ++i) (nxt ? a.act1 : a.act0)[at + i] = wb[i];
        }
        __syncwarp();
        nbuf = 0;
    }

    __device__ void step(long long r, bool first) {
        const DevModel& M = a.M;
        const int n = M.n;
        RolloutCounters* C = a.cnt;
        double c[J];
        const double* src = first ? a.comp0 : a.comp + r * n;
#pragma unroll
        for (int j = 0; j < J; ++j) c[j] = (lane + 32 * j < n) ? src[lane + 32 * j] : 2.0;
        int L = first ? 0 : a.len[r];
        unsigned dirty = first ? ~0u : 0u;  // slots to write back (all of them for a new rollout)
        if (first && lane == 0) a.len[r] = 0;
        if (!first) {
            const unsigned slot = a.rslot[r];
            const int pn = __ldcg(&a.pool_n[slot]);
            if (pn <= 0) {  // rollout: "no candidate config serves the remaining demand" (mcts.hpp:135-136)
                if (lane == 0) {
                    a.status[r] = 3;
                    if (a.lengths) a.lengths[r] = -1;
                    atomicAdd(c_fail, 1ull);
                }
                return;
            }
            const uint64_t x = philox_u64(a.seed, static_cast<uint64_t>(a.id0 + r), static_cast<uint64_t>(L));
            const unsigned pick = __ldcg(&a.pool[static_cast<size_t>(slot) * a.k + philox_below(x, pn)]);
            dirty |= add_row(M, __ldg(a.base + pick), c);
            ++L;
            if (lane == 0) {
                a.len[r] = L;
                atomicAdd(c_steps, 1ull);
            }
        }
        uint64_t kw[4];
        if (!type_key(c, n, kw)) {  // satisfied
            if (lane == 0) {
                a.status[r] = 1;
                if (a.lengths) a.lengths[r] = L;
                atomicMin(&C->best, (static_cast<unsigned long long>(L) << 32) | static_cast<unsigned long long>(r));
                atomicAdd(c_done, 1ull);
            }
            return;
        }
        if (L >= a.max_depth) {  // rollout returns max_depth (mcts.hpp:127)
            if (lane == 0) {
                a.status[r] = 2;
                if (a.lengths) a.lengths[r] = a.max_depth;
                atomicAdd(c_cap, 1ull);
            }
            return;
        }
#pragma unroll
        for (int j = 0; j < J; ++j)
            if (lane + 32 * j < n && ((dirty >> j) & 1u)) a.comp[r * n + lane + 32 * j] = c[j];
        if (lane == 0) {
            bool created = false;
            long long slot = probe(a, kw, nk, true, created);
            if (slot < 0) {
                atomicExch(&C->status, 1);
                slot = 0;
            } else {
                if (created) {
                    const unsigned long long at = atomicAdd(&C->n_pend[nxt], 1ull);
                    (nxt ? a.pend1 : a.pend0)[at] = static_cast<unsigned>(slot);
                }
                if (__ldcg(&a.pool_n[slot]) < 0 && __ldcg(&a.claimer[slot]) > static_cast<unsigned long long>(r))
                    atomicMin(&a.claimer[slot], static_cast<unsigned long long>(r));
            }
            a.rslot[r] = static_cast<unsigned>(slot);
            wb[nbuf] = r;
        }
        if (++nbuf == 32) push_flush();
    }
};

// n <= 64: ONE LANE per rollout.  The rollout's type key (completion_type_key, mcts.hpp:38-43)
// is kept beside its completion vector, and a step touches only the <= 4 services of the picked
// config: their completions are read, the utilities added (mcts.hpp:139), their key bits
// updated (a completion only grows, so a bit only clears) — the other n - 4 completions are
// neither read nor written.  A warp advances 32 rollouts at once; the next round's active list
// takes one atomic per warp.  Same draws, pools and schedule as the lane-group steppers.
__device__ void advance_lane_step(const RolloutArgs& a, long long r, bool valid, bool first, int nxt,
                                  unsigned long long* cnt4) {
    const DevModel& M = a.M;
    const int n = M.n;
    RolloutCounters* C = a.cnt;
    const int lane = static_cast<int>(threadIdx.x & 31u);
    bool active = valid;
    int L = 0;
    uint64_t key = 0;
    if (valid && first) {  // a new rollout: the start completion and its key
        for (int i = 0; i < n; ++i) {
            const double v = a.comp0[i];
            a.comp[r * n + i] = v;
            if (v < 1.0 - 1e-9) key |= 1ull << i;
        }
        a.len[r] = 0;
    } else if (valid) {
        L = a.len[r];
        key = a.keys[r];
        const unsigned slot = a.rslot[r];
        const int pn = __ldcg(&a.pool_n[slot]);
        if (pn <= 0) {  // rollout: "no candidate config serves the remaining demand" (mcts.hpp:135-136)
            a.status[r] = 3;
            if (a.lengths) a.lengths[r] = -1;
            active = false;
        } else {
            const uint64_t x = philox_u64(a.seed, static_cast<uint64_t>(a.id0 + r), static_cast<uint64_t>(L));
            const unsigned pick = __ldcg(&a.pool[static_cast<size_t>(slot) * a.k + philox_below(x, pn)]);
            const uint64_t row = __ldg(a.base + pick);
            double* cr = a.comp + r * n;
#pragma unroll
            for (int m = 0; m < 4; ++m) {  // distinct services: the adds commute
                const unsigned code = static_cast<unsigned>((row >> (16 * m)) & 0xFFFFull);
                const int svc = svc_of(M, code);
                if (svc < n) {
                    const double v = __dadd_rn(cr[svc], __ldg(&M.U[code]));
                    cr[svc] = v;
                    if (!(v < 1.0 - 1e-9)) key &= ~(1ull << svc);
                }
            }
            ++L;
            a.len[r] = L;
        }
    }
    const bool stepped = valid && !first && active;
    bool sat = false, cap = false;
    if (active && key == 0) {  // satisfied
        a.status[r] = 1;
        if (a.lengths) a.lengths[r] = L;
        atomicMin(&C->best, (static_cast<unsigned long long>(L) << 32) | static_cast<unsigned long long>(r));
        sat = true;
        active = false;
    }
    if (active && L >= a.max_depth) {  // rollout returns max_depth (mcts.hpp:127)
        a.status[r] = 2;
        if (a.lengths) a.lengths[r] = a.max_depth;
        cap = true;
        active = false;
    }
    if (active) {
        a.keys[r] = key;
        bool created = false;
        long long slot = probe(a, &key, 1, true, created);
        if (slot < 0) {
            atomicExch(&C->status, 1);
            slot = 0;
        } else {
            if (created) {
                const unsigned long long at = atomicAdd(&C->n_pend[nxt], 1ull);
                (nxt ? a.pend1 : a.pend0)[at] = static_cast<unsigned>(slot);
            }
            if (__ldcg(&a.pool_n[slot]) < 0 && __ldcg(&a.claimer[slot]) > static_cast<unsigned long long>(r))
                atomicMin(&a.claimer[slot], static_cast<unsigned long long>(r));
        }
        a.rslot[r] = static_cast<unsigned>(slot);
    }
    // counters and the next round's active list: one shared/global atomic per warp
    const unsigned bs = __ballot_sync(0xffffffffu, stepped), bd = __ballot_sync(0xffffffffu, sat),
                   bc = __ballot_sync(0xffffffffu, cap), bf = __ballot_sync(0xffffffffu, valid && !first && !stepped),
                   ba = __ballot_sync(0xffffffffu, active);
    if (lane == 0) {
        if (bs) atomicAdd(&cnt4[0], static_cast<unsigned long long>(__popc(bs)));
        if (bd) atomicAdd(&cnt4[1], static_cast<unsigned long long>(__popc(bd)));
        if (bc) atomicAdd(&cnt4[2], static_cast<unsigned long long>(__popc(bc)));
        if (bf) atomicAdd(&cnt4[3], static_cast<unsigned long long>(__popc(bf)));
    }
    unsigned long long at = 0;
    if (lane == 0 && ba) at = atomicAdd(&C->n_act[nxt], static_cast<unsigned long long>(__popc(ba)));
    at = __shfl_sync(0xffffffffu, at, 0);
    if (active) (nxt ? a.act1 : a.act0)[at + __popc(ba & ((1u << lane) - 1u))] = r;
}

// One advance pass of a block over the active list (or, first, over every rollout): a warp
// per rollout (n > 64) or one lane per rollout (n <= 64, advance_lane_step).  Block-level counters are
// summed into the launch's RolloutCounters at the end.  Ends with a barrier.
template <int J, int NT>
__device__ void advance_pass(const RolloutArgs& a, bool first, int cur, unsigned long long n_act, long long (*wbuf)[32],
                             unsigned long long* cnt4) {
    RolloutCounters* C = a.cnt;
    if (threadIdx.x == 0) cnt4[0] = cnt4[1] = cnt4[2] = cnt4[3] = 0;
    __syncthreads();
    const int warp = static_cast<int>(threadIdx.x >> 5);
    const long long gw = static_cast<long long>(blockIdx.x) * (NT / 32) + warp;
    const long long nwarps = static_cast<long long>(gridDim.x) * (NT / 32);
    const long long* act = cur ? a.act1 : a.act0;
    if constexpr (J == 2) {  // n <= 64: a lane per rollout
        const int lane = static_cast<int>(threadIdx.x & 31u);
        for (long long i0 = 32 * gw; i0 < static_cast<long long>(n_act); i0 += 32 * nwarps) {
            const long long i = i0 + lane;
            const bool valid = i < static_cast<long long>(n_act);
            advance_lane_step(a, valid ? (first ? i : __ldcg(&act[i])) : 0, valid, first, cur ^ 1, cnt4);
        }
    } else {
        Advancer<J> adv{a, wbuf[warp], &cnt4[0], &cnt4[1], &cnt4[2], &cnt4[3], static_cast<int>(threadIdx.x & 31u),
                        (a.M.n + 63) / 64, cur ^ 1};
        for (long long i = gw; i < static_cast<long long>(n_act); i += nwarps) adv.step(first ? i : __ldcg(&act[i]), first);
        adv.push_flush();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (cnt4[0]) atomicAdd(&C->steps, cnt4[0]);
        if (cnt4[1]) atomicAdd(&C->completed, cnt4[1]);
        if (cnt4[2]) atomicAdd(&C->capped, cnt4[2]);
        if (cnt4[3]) atomicAdd(&C->failed, cnt4[3]);
    }
}

// Shared-memory tables of a pool build (same offsets in the build and persistent kernels).
struct BuildSmem {
    double *W, *comp;
    Cand *cand, *win;
    int* sact;
    float* Wf;
    unsigned char* hitc;
    __device__ BuildSmem(unsigned char* smem, const RolloutArgs& a) {
        const int n = a.M.n, nW = (n + 1) * a.M.PP;
        W = reinterpret_cast<double*>(smem);
        comp = W + nW;
        cand = reinterpret_cast<Cand*>(comp + n + 1);
        win = cand + kRCandCap;
        sact = reinterpret_cast<int*>(win + kRMaxK);  // active supports of a pool build (a.n_sup)
        Wf = reinterpret_cast<float*>(sact + (a.n_sup > 0 ? a.n_sup : 0));  // pair top-K tables
        hitc = reinterpret_cast<unsigned char*>(Wf + nW);
    }
};

// The pools of the keys created in the previous step (slots pend[0..n_pend)), CTA per key.
__device__ void build_pass(const RolloutArgs& a, const BuildSmem& sm, int cur, unsigned long long n_pend, int* s_out) {
    const DevModel& M = a.M;
    const int n = M.n;
    for (unsigned long long p = blockIdx.x; p < n_pend; p += gridDim.x) {
        const unsigned slot = __ldcg(&(cur ? a.pend1 : a.pend0)[p]);
        const long long r = static_cast<long long>(__ldcg(&a.claimer[slot]));
        for (int i = threadIdx.x; i < n; i += blockDim.x) sm.comp[i] = __ldcg(&a.comp[r * n + i]);
        __syncthreads();
        int got;
        if (a.base32) {  // pair pool: FP32-bounded two-pass top-K over the live supports (K7's)
            int scored = 0;
            got = block_topk_pair(M, a.keyrank, a.base32, a.n_base, 0, sm.comp, nullptr, a.k, M.U, sm.W, sm.Wf, sm.hitc,
                                  sm.cand, sm.win, s_out, &scored, false, SupTab{a.n_sup, a.sup_begin, a.sup_svc, sm.sact});
            if (threadIdx.x < got) a.pool[static_cast<size_t>(slot) * a.k + threadIdx.x] = static_cast<unsigned>(s_out[threadIdx.x]);
        } else {
            got = block_topk(a, sm.comp, sm.W, sm.cand, sm.win, a.pool + static_cast<size_t>(slot) * a.k, sm.sact);
        }
        if (threadIdx.x == 0) a.pool_n[slot] = got;
        __syncthreads();
    }
}

// The shortest completed rollout (ties: lowest index), replayed from the immutable cache by
// one warp: its path, pick by pick.
template <int J>
__device__ void replay_winner(const RolloutArgs& a) {
    const DevModel& M = a.M;
    const int n = M.n, nk = (n + 63) / 64;
    const int lane = static_cast<int>(threadIdx.x & 31u);
    RolloutCounters* C = a.cnt;
    const unsigned long long best = __ldcg(&C->best);
    int plen = 0;
    if (best != ~0ull && __ldcg(&C->status) == 0) {
        const long long r = static_cast<long long>(best & 0xFFFFFFFFull);
        const int L = static_cast<int>(best >> 32);
        double c[J];
#pragma unroll
        for (int j = 0; j < J; ++j) c[j] = (lane + 32 * j < n) ? a.comp0[lane + 32 * j] : 2.0;
        for (int t = 0; t < L; ++t) {
            uint64_t kw[4];
            type_key(c, n, kw);
            long long slot = 0;
            if (lane == 0) {
                bool created;
                slot = probe(a, kw, nk, false, created);
            }
            slot = __shfl_sync(0xffffffffu, slot, 0);
            const int pn = __ldcg(&a.pool_n[slot]);
            const uint64_t x = philox_u64(a.seed, static_cast<uint64_t>(a.id0 + r), static_cast<uint64_t>(t));
            const unsigned pick = __ldcg(&a.pool[static_cast<size_t>(slot) * a.k + philox_below(x, pn)]);
            if (lane == 0) a.path[t] = pick;
            add_row(M, __ldg(a.base + pick), c);
        }
        plen = L;
    }
    if (lane == 0) *a.path_len = plen;
}

// Round `round` (or the start, round < 0): every active rollout advances one step.
template <int J>
__global__ void __launch_bounds__(kAThreads, kAOcc) rollout_advance_kernel(const __grid_constant__ RolloutArgs a, int round) {
    __shared__ long long wbuf[kAThreads / 32][32];
    __shared__ unsigned long long cnt4[4];
    RolloutCounters* C = a.cnt;
    const bool first = round < 0;
    const int cur = first ? 1 : (round & 1);
    unsigned long long n_act = static_cast<unsigned long long>(a.n_roll);
    if (!first) {  // rounds enqueued past the last one (C->done) are no-ops
        n_act = __ldcg(&C->n_act[cur]);
        if (n_act == 0 || __ldcg(&C->status) != 0 || *reinterpret_cast<volatile int*>(&C->done)) return;
    }
    advance_pass<J, kAThreads>(a, first, cur, n_act, wbuf, cnt4);
}

// Round `round`: the pools of the keys first reached in the previous step (CTA per key).
// Block 0 also opens the round: the next round's lists start empty.
__global__ void __launch_bounds__(kRThreads, 1) rollout_build_kernel(const __grid_constant__ RolloutArgs a, int round) {
    extern __shared__ __align__(16) unsigned char smem[];
    const BuildSmem sm(smem, a);
    __shared__ int s_out[kRMaxK];
    RolloutCounters* C = a.cnt;
    topk_pair_counters_init();
    const int cur = round & 1, nxt = cur ^ 1;
    if (*reinterpret_cast<volatile int*>(&C->done)) return;  // enqueued past the last round
    const unsigned long long n_act = __ldcg(&C->n_act[cur]);
    const unsigned long long n_pend = __ldcg(&C->n_pend[cur]);
    if (n_act == 0 || __ldcg(&C->status) != 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) C->done = 1;
        return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // last read by the previous round's kernels
        C->n_act[nxt] = 0;
        C->n_pend[nxt] = 0;
        C->keys += n_pend;
        C->rounds = round + 1;
    }
    build_pass(a, sm, cur, n_pend, s_out);
}

template <int J>
__global__ void rollout_replay_kernel(const __grid_constant__ RolloutArgs a) {
    replay_winner<J>(a);
}

// Small batches (one advance pass per round fits one wave of the grid): the same rounds in
// ONE cooperative launch with grid barriers — per-round launches cost more than the work there
// (config #3's refills: 1,024 rollouts, ~100 rounds per call).
template <int J>
__global__ void __launch_bounds__(kRThreads, 1) rollout_persistent_kernel(const __grid_constant__ RolloutArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const BuildSmem sm(smem, a);
    __shared__ int s_out[kRMaxK];
    __shared__ long long wbuf[kRThreads / 32][32];
    __shared__ unsigned long long cnt4[4];
    RolloutCounters* C = a.cnt;
    topk_pair_counters_init();
    advance_pass<J, kRThreads>(a, true, 1, static_cast<unsigned long long>(a.n_roll), wbuf, cnt4);
    grid_barrier(&C->bar_count, &C->bar_gen, gridDim.x);
    for (int round = 0;; ++round) {
        const int cur = round & 1, nxt = cur ^ 1;
        const unsigned long long n_act = __ldcg(&C->n_act[cur]);
        const unsigned long long n_pend = __ldcg(&C->n_pend[cur]);
        if (n_act == 0 || __ldcg(&C->status) != 0) break;
        if (blockIdx.x == 0 && threadIdx.x == 0) {  // last read in round - 1, next written after the barrier below
            C->n_act[nxt] = 0;
            C->n_pend[nxt] = 0;
            C->keys += n_pend;
            C->rounds = round + 1;
        }
        build_pass(a, sm, cur, n_pend, s_out);
        grid_barrier(&C->bar_count, &C->bar_gen, gridDim.x);
        advance_pass<J, kRThreads>(a, false, cur, n_act, wbuf, cnt4);
        grid_barrier(&C->bar_count, &C->bar_gen, gridDim.x);
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) replay_winner<J>(a);
}

size_t rollout_smem_bytes(int n, int PP, int n_sup) {
    const size_t nW = static_cast<size_t>(n + 1) * PP;
    return (nW + n + 1) * 8 + static_cast<size_t>(kRCandCap + kRMaxK) * sizeof(Cand) + sizeof(int) * static_cast<size_t>(n_sup) +
           nW * 4 + nW + 16;  // + the pair top-K's Wf and mask-hit tables
}
const void* rollout_build_ptr() { return reinterpret_cast<const void*>(&rollout_build_kernel); }
const void* rollout_advance_ptr(int n) {
    return n <= 64 ? reinterpret_cast<const void*>(&rollout_advance_kernel<2>)
                   : reinterpret_cast<const void*>(&rollout_advance_kernel<kMaxJ>);
}
const void* rollout_persistent_ptr(int n) {
    return n <= 64 ? reinterpret_cast<const void*>(&rollout_persistent_kernel<2>)
                   : reinterpret_cast<const void*>(&rollout_persistent_kernel<kMaxJ>);
}
int rollout_per_warp(int n) { return n <= 64 ? 32 : 1; }
const void* rollout_replay_ptr(int n) {
    return n <= 64 ? reinterpret_cast<const void*>(&rollout_replay_kernel<2>)
                   : reinterpret_cast<const void*>(&rollout_replay_kernel<kMaxJ>);
}
int rollout_threads() { return kRThreads; }
void rollout_set_dense_pct(int pct) { cudaMemcpyToSymbol(g_mcts_dense_pct, &pct, sizeof pct); }  // this TU's copy
int rollout_advance_threads() { return kAThreads; }

namespace {
__global__ void philox_kat_kernel(uint64_t seed, uint64_t stream, uint64_t step, unsigned long long* out) {
    *out = philox_u64(seed, stream, step);
}
}  // namespace

// One Philox draw on the device code path (known-answer tests of philox.cuh, engine.cu).
const void* philox_kat_kernel_ptr() { return reinterpret_cast<const void*>(&philox_kat_kernel); }

}  // namespace mgb
