// kernels.cu — hand-written sm_100a kernels of the MIG-SERVING optimizer hot path.
//
//   K1 enum_base_kernel   build_candidate_pool  (config_enum.hpp:192-202)
//   K2/K3 greedy_kernel   fast_algo             (greedy.hpp:95-145): persistent cooperative
//                         kernel; per step a coalesced 128-bit scan of the packed rows
//                         (shared-memory resident while they fit, streamed from L2/HBM beyond)
//                         against a shared-memory need*U table, a warp-shuffle 3-key argmax,
//                         a grid-wide reduction, the completion update, maybe_extend
//                         (greedy.hpp:107-119) and the device-side extension enumerator
//                         (extend_candidate_pool, config_enum.hpp:206-211).
//   K4 topk_kernel        detail::topk_candidates (mcts.hpp:56-76) for k > 32 (the common
//                         k <= 32 case is the single-pass kernel in topk.cu).
//
// Bit-exactness: every floating add/multiply on the score path is an explicit
// __dadd_rn/__dmul_rn (and the TU is built with -fmad=false), so no FMA contraction
// changes the reference's FP64 bits (SURVEY §0 hazard 1).
#include <cooperative_groups.h>

#include "common.cuh"

namespace mgb {

using namespace dev;

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
// Streaming-row loads.  Rows are append-only and every row a step reads was completed
// before a grid barrier, so any load that bypasses L1 (L2 is the coherence point) is exact.
//   0: ld.global.cg (L2 only)   1: ld.global.nc.L1::no_allocate   2: ld.global.cs (evict-first)
// (ld.global.cs measured best for the n = 128 stress scan, profiles/: the hot loop uses it)
#define LOADM 2
__device__ __forceinline__ uint4 ld_row4(const uint4* p, int mode) {
    uint4 v;
    if (mode == 1) {
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(p));
    } else if (mode == 2) {
        asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    } else {
        v = __ldcg(p);
    }
    return v;
}

// Block-wide argmax; result valid in every thread.
__device__ Best block_best(const DevModel& M, Best b, Best* red) {
    b = warp_best(M, b);
    const unsigned w = threadIdx.x >> 5;
    if (lane_id() == 0) red[w] = b;
    __syncthreads();
    if (w == 0) {
        Best x = lane_id() < blockDim.x / 32 ? red[lane_id()] : none();
        x = warp_best(M, x);
        if (lane_id() == 0) red[0] = x;
    }
    __syncthreads();
    Best r = red[0];
    __syncthreads();
    return r;
}

// Reduce the per-CTA partials after a grid barrier (every CTA computes the same winner).
__device__ Best grid_best(const DevModel& M, const Best* partials, int G, Best* red) {
    if ((threadIdx.x >> 5) == 0) {
        Best x = none();
        for (int i = lane_id(); i < G; i += 32) {
            Best p{__ldcg(&partials[i].s), __ldcg(&partials[i].u),
                   __ldcg(reinterpret_cast<const unsigned long long*>(&partials[i].row))};
            if (better(M, p, x)) x = p;
        }
        x = warp_best(M, x);
        if (lane_id() == 0) red[0] = x;
    }
    __syncthreads();
    Best r = red[0];
    __syncthreads();
    return r;
}

// Grid-wide argmax + barrier in one: every CTA publishes its block winner and takes a
// ticket; the LAST CTA to arrive reduces the G partials and publishes the single winner
// record, then releases the generation.  Only one CTA reads the partials (instead of all G
// CTAs reading all G records — a G^2 hot-line read storm in L2), and waiters read one
// 24-byte record.  Returns the same winner in every thread of every CTA.
// Cross-rank step of the sharded greedy, run by one thread of the last CTA:
// post this rank's winner into slot [parity][rank] of EVERY rank's exchange board (peer
// memory over NVLink, or plain device memory for ranks sharing a GPU), then wait until all
// n_ranks records of this step are in the own board and reduce them in the same total
// order.  Every rank computes the same global winner.  Double-buffering by step parity is
// enough: a rank posts step t+1 only after it read all records of step t.  A watchdog turns
// a missing peer into kExchTimeout instead of a hang.
__device__ Best exchange_best(const DevModel& M, const GreedyArgs& a, Best x, unsigned long long seq, int& status) {
    const int P = a.n_ranks;
    const int par = static_cast<int>(seq & 1ull);
    for (int q = 0; q < P; ++q) {
        ExchSlot* d = a.boards[q] + par * P + a.rank;
        d->s = x.s;
        d->u = x.u;
        d->row = x.row;
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_system> f(d->seq);
        f.store(seq, cuda::memory_order_release);
    }
    ExchSlot* mine = a.boards[a.rank] + par * P;
    const unsigned long long t0 = globaltimer();
    Best g = none();
    for (int q = 0; q < P; ++q) {
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_system> f(mine[q].seq);
        while (f.load(cuda::memory_order_acquire) < seq) {
            if (globaltimer() - t0 > static_cast<unsigned long long>(a.exch_timeout_ns)) {
                status = kExchTimeout;
                return none();
            }
        }
        const Best p{*reinterpret_cast<volatile double*>(&mine[q].s), *reinterpret_cast<volatile double*>(&mine[q].u),
                     *reinterpret_cast<volatile unsigned long long*>(&mine[q].row)};
        if (better(M, p, g)) g = p;
    }
    return g;
}

namespace cg = cooperative_groups;

// The argmax of a cluster-mode group: every CTA publishes its block best in shared memory
// (double-buffered by step parity), one cluster barrier, then every CTA reduces the G
// records over DSMEM in the same order, so all agree on the winner.
__device__ Best cluster_argmax(const DevModel& M, const Best& mine, Best* xch, int parity, Best* red, int G) {
    cg::cluster_group cl = cg::this_cluster();
    if (threadIdx.x == 0) xch[parity] = mine;
    cl.sync();
    if ((threadIdx.x >> 5) == 0) {
        Best x = none();
        for (int q = lane_id(); q < G; q += 32) {
            const Best b = *cl.map_shared_rank(xch + parity, q);
            if (better(M, b, x)) x = b;
        }
        x = warp_best(M, x);
        if (lane_id() == 0) red[0] = x;
    }
    __syncthreads();
    const Best r = red[0];
    __syncthreads();
    return r;
}

// Argmax of a single-rank cooperative group without a reducing CTA: every CTA posts its
// block best (double-buffered by step parity), counts itself in, waits until all G CTAs of
// this step have arrived, then reduces the G records itself in the same order — one L2
// round trip less than "last CTA reduces, everyone reads its record".
__device__ Best grid_allreduce_argmax(const DevModel& M, const Best& mine, Best* partials, unsigned* arrive, int G,
                                      int step, Best* red, int bi) {
    Best* part = partials + (step & 1) * G;
    if (threadIdx.x == 0) {
        __stcg(&part[bi].s, mine.s);
        __stcg(&part[bi].u, mine.u);
        __stcg(reinterpret_cast<unsigned long long*>(&part[bi].row), static_cast<unsigned long long>(mine.row));
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> c(*arrive);
        c.fetch_add(1u, cuda::memory_order_release);
        const unsigned target = static_cast<unsigned>(step + 1) * static_cast<unsigned>(G);
        while (c.load(cuda::memory_order_acquire) < target) __nanosleep(16);
    }
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) {
        Best x = none();
        for (int i0 = 0; i0 < G; i0 += 128) {
            Best p[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = i0 + 32 * k + static_cast<int>(lane_id());
                p[k] = i < G ? Best{__ldcg(&part[i].s), __ldcg(&part[i].u),
                                    __ldcg(reinterpret_cast<const unsigned long long*>(&part[i].row))}
                             : none();
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (better(M, p[k], x)) x = p[k];
        }
        x = warp_best(M, x);
        if (lane_id() == 0) red[0] = x;
    }
    __syncthreads();
    const Best r = red[0];
    __syncthreads();
    return r;
}

constexpr int kKeyMaxPP = 128;  // key tables on chip up to this many patterns
constexpr int kKeyMaxLayouts = 32;  // == kMaxLayouts (model.hpp)
__device__ unsigned long long g_dep[1024], g_cta_dur[1024], g_scan[1024], g_post[1024];
__device__ unsigned long long g_arrive0, g_arrive_last, g_skew_ns, g_release_ns;
#ifdef MGB_GREEDY_STEP_DIAG
// development aid: per step, the slowest CTA's scan (ns, which CTA), the mean, and the most
// exact-path rows one CTA evaluated; CTA 0 prints the table at the end of the launch
constexpr int kDiagSteps = 4096;
__device__ unsigned long long g_sd_max[kDiagSteps], g_sd_sum[kDiagSteps], g_sd_exact[kDiagSteps], g_sd_arg[kDiagSteps], g_sd_key[kDiagSteps];
__device__ unsigned g_sd_cnt[1024];
#endif
__device__ Best grid_argmax(const DevModel& M, const Best& mine, Best* partials, Best* winrec, unsigned* count,
                            unsigned* gen, int G, Best* red, const GreedyArgs& a, unsigned long long seq,
                            int* xstatus, int bi) {
    __shared__ int s_last;
    __shared__ unsigned s_gen;
    if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> g(*gen), c(*count);
        const unsigned my = g.load(cuda::memory_order_relaxed);
        __stcg(&partials[bi].s, mine.s);
        __stcg(&partials[bi].u, mine.u);
        __stcg(reinterpret_cast<unsigned long long*>(&partials[bi].row),
               static_cast<unsigned long long>(mine.row));
        const unsigned t = c.fetch_add(1u, cuda::memory_order_acq_rel);
        s_last = t == static_cast<unsigned>(G) - 1u;
        s_gen = my;
        if (a.phase_timers) {  // diagnostics: arrival skew (last CTA vs CTA 0) and reduce+release
            const unsigned long long now = globaltimer();
            if (g_dep[blockIdx.x]) g_cta_dur[blockIdx.x] += now - g_dep[blockIdx.x];
            if (bi == 0) g_arrive0 = now;
            if (s_last) g_arrive_last = now;
        }
    }
    __syncthreads();
    if (s_last) {
        if ((threadIdx.x >> 5) == 0) {
            Best x = none();
            for (int i0 = 0; i0 < G; i0 += 128) {  // four independent partial loads in flight per lane
                Best p[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int i = i0 + 32 * k + static_cast<int>(lane_id());
                    p[k] = i < G ? Best{__ldcg(&partials[i].s), __ldcg(&partials[i].u),
                                        __ldcg(reinterpret_cast<const unsigned long long*>(&partials[i].row))}
                                 : none();
                }
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (better(M, p[k], x)) x = p[k];
            }
            x = warp_best(M, x);
            if (lane_id() == 0) {
                if (a.n_ranks > 1) {
                    int st = kOk;
                    x = exchange_best(M, a, x, seq, st);
                    if (st != kOk) atomicExch(xstatus, st);
                }
                red[0] = x;
                __stcg(&winrec->s, x.s);
                __stcg(&winrec->u, x.u);
                __stcg(reinterpret_cast<unsigned long long*>(&winrec->row), static_cast<unsigned long long>(x.row));
                cuda::atomic_ref<unsigned, cuda::thread_scope_device> g(*gen), c(*count);
                c.store(0u, cuda::memory_order_relaxed);
                g.store(s_gen + 1u, cuda::memory_order_release);
            }
        }
    } else if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> g(*gen);
        while (g.load(cuda::memory_order_acquire) == s_gen) __nanosleep(32);
        red[0] = Best{__ldcg(&winrec->s), __ldcg(&winrec->u),
                      __ldcg(reinterpret_cast<const unsigned long long*>(&winrec->row))};
        if (a.phase_timers && bi == 0) {
            const unsigned long long now = globaltimer();
            const unsigned long long t0 = *reinterpret_cast<volatile unsigned long long*>(&g_arrive0);
            const unsigned long long tl = *reinterpret_cast<volatile unsigned long long*>(&g_arrive_last);
            if (tl >= t0) g_skew_ns += tl - t0;
            if (now >= tl) g_release_ns += now - tl;
        }
    }
    if (a.phase_timers && threadIdx.x == 0) g_dep[blockIdx.x] = globaltimer();
    __syncthreads();
    const Best r = red[0];
    __syncthreads();
    return r;
}

// The thread's running argmax over one scored row (s = row_score): the 3-key order of
// candidate_preferred (greedy.hpp:63-67); util_sum and the config key only on ties.
__device__ __forceinline__ void take(const DevModel& M, const double* U, uint64_t row, double s, Best& best) {
    if (s > 0.0 && s >= best.s) {
        if (s > best.s) {
            best = Best{s, row_usum(U, row), row};
            return;
        }
        const double u = row_usum(U, row);
        if (u > best.u || (u == best.u && row != best.row && row_key_less(M, row, best.row))) best = Best{s, u, row};
    }
}

__device__ __forceinline__ void consider(const DevModel& M, const double* __restrict__ W, const double* U,
                                         uint64_t row, Best& best) {
    take(M, U, row, row_score(W, row), best);
}

// Eight rows (four 16-byte units) at once, two-level.  Level 1 gathers a 4-byte FP32
// table Wf = W rounded UP (one shared-memory wavefront serves a whole warp far more often
// than for the 8-byte W) and adds with round-up: ub >= the exact FP64 score, always (all
// terms are >= 0).  A row with ub below the thread's running best (or ub == 0) can neither
// win nor tie, so only the few survivors pay the exact FP64 gathers and adds of score()
// (greedy.hpp:36-43, bit-exact).  `floor` = the thread's best score, or the smallest
// positive double while it has none (rows must score > 0, greedy.hpp:130).
__device__ __forceinline__ float row_ub(const float* __restrict__ Wf, uint64_t row) {
    float s = __fadd_ru(Wf[row & 0xFFFFull], Wf[(row >> 16) & 0xFFFFull]);
    s = __fadd_ru(s, Wf[(row >> 32) & 0xFFFFull]);
    return __fadd_ru(s, Wf[row >> 48]);
}

// Upper bound of one row from its two 32-bit halves (codes 0,1 in lo; 2,3 in hi): 32-bit
// field extraction only, no 64-bit shifts on the hot path.  Codes are < 2^14 (model.cpp), so
// x << 2 holds BOTH codes' byte offsets into Wf (4 * code < 2^16 in each half): one shift
// serves two gathers, and each offset is one mask or one shift (3 ALU ops per half instead of
// a shift and a mask per code).
__device__ __forceinline__ float wf_at(const float* __restrict__ Wf, unsigned byte_off) {
    return *reinterpret_cast<const float*>(reinterpret_cast<const char*>(Wf) + byte_off);
}
__device__ __forceinline__ float ub2(const float* __restrict__ Wf, unsigned lo, unsigned hi) {
    const unsigned l = lo << 2, h = hi << 2;
    float s = __fadd_ru(wf_at(Wf, l & 0xFFFFu), wf_at(Wf, l >> 16));
    s = __fadd_ru(s, wf_at(Wf, h & 0xFFFFu));
    return __fadd_ru(s, wf_at(Wf, h >> 16));
}

__device__ __forceinline__ void consider8(const DevModel& M, const double* __restrict__ W, const float* __restrict__ Wf,
                                          const double* U, const uint4& v0, const uint4& v1, const uint4& v2,
                                          const uint4& v3, Best& best, double floor = 0.0) {
    // FP32 floor rounded DOWN: ub >= best.s implies ub >= ff, so no row that can win or tie
    // is skipped; with no best yet, ff = the smallest positive float (rows must score > 0).
    // `floor` is a score some row of the warp already has: a row below it cannot be the argmax
    // (it may still tie it, so the compare stays >=).
    const double fl = fmax(best.s, floor);
    const float ff = fl > 0.0 ? __double2float_rd(fl) : 1.40129846e-45f;
    const float ub[8] = {ub2(Wf, v0.x, v0.y), ub2(Wf, v0.z, v0.w), ub2(Wf, v1.x, v1.y), ub2(Wf, v1.z, v1.w),
                         ub2(Wf, v2.x, v2.y), ub2(Wf, v2.z, v2.w), ub2(Wf, v3.x, v3.y), ub2(Wf, v3.z, v3.w)};
    bool hit = false;
#pragma unroll
    for (int j = 0; j < 8; ++j) hit |= ub[j] >= ff;
    if (hit) {
        const uint64_t r[8] = {(static_cast<uint64_t>(v0.y) << 32) | v0.x, (static_cast<uint64_t>(v0.w) << 32) | v0.z,
                               (static_cast<uint64_t>(v1.y) << 32) | v1.x, (static_cast<uint64_t>(v1.w) << 32) | v1.z,
                               (static_cast<uint64_t>(v2.y) << 32) | v2.x, (static_cast<uint64_t>(v2.w) << 32) | v2.z,
                               (static_cast<uint64_t>(v3.y) << 32) | v3.x, (static_cast<uint64_t>(v3.w) << 32) | v3.z};
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (static_cast<double>(ub[j]) >= (fl > 0.0 ? fl : 4.9406564584124654e-324) && r[j] != best.row) {
#ifdef MGB_GREEDY_STEP_DIAG
                atomicAdd(&g_sd_cnt[blockIdx.x], 1u);
#endif
                take(M, U, r[j], row_score(W, r[j]), best);
            }
    }
}

__device__ __forceinline__ void consider2(const DevModel& M, const double* __restrict__ W, const double* U,
                                          const uint4& v, Best& best) {
    consider(M, W, U, (static_cast<uint64_t>(v.y) << 32) | v.x, best);
    consider(M, W, U, (static_cast<uint64_t>(v.w) << 32) | v.z, best);
}

// The streaming part of a greedy step's scan (units u, u + GT, ... < NU, four per thread per
// iteration).  Measured alternatives (tools/gpu_ab.sh, n = 128): a non-inlined copy with its
// own register budget, a 1024-thread CTA at 64 registers, and a max-reduced FP32 bound with
// a separate exact path were all slower than this inlined, software-pipelined loop.
__device__ __forceinline__ Best scan_stream(const DevModel& M, const double* W, const float* Wf, const double* U,
                                         const uint4* rows4, long long u, long long NU, long long GT, int prefetch,
                                         int pipeline, Best best, double wfloor) {
    if (pipeline && u + 3 * GT < NU) {
        // software-pipelined: the next 4 units are loaded before this 4 are scored, so every
        // warp keeps its loads in flight while it computes
        uint4 n0 = ld_row4(rows4 + u, LOADM), n1 = ld_row4(rows4 + u + GT, LOADM),
              n2 = ld_row4(rows4 + u + 2 * GT, LOADM), n3 = ld_row4(rows4 + u + 3 * GT, LOADM);
        for (; u + 3 * GT < NU; u += 4 * GT) {
            if (threadIdx.x < 4 && prefetch > 0) {
                const long long pu = u - threadIdx.x + (prefetch * 4 + threadIdx.x) * GT;
                if (pu + static_cast<long long>(blockDim.x) <= NU)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rows4 + pu),
                                 "r"(static_cast<unsigned>(blockDim.x * 16))
                                 : "memory");
            }
            const uint4 v0 = n0, v1 = n1, v2 = n2, v3 = n3;
            if (u + 7 * GT < NU) {
                n0 = ld_row4(rows4 + u + 4 * GT, LOADM);
                n1 = ld_row4(rows4 + u + 5 * GT, LOADM);
                n2 = ld_row4(rows4 + u + 6 * GT, LOADM);
                n3 = ld_row4(rows4 + u + 7 * GT, LOADM);
            }
            consider8(M, W, Wf, U, v0, v1, v2, v3, best, wfloor);
        }
    }
    for (; u + 3 * GT < NU; u += 4 * GT) {
        // Bulk L2 prefetch, `prefetch` iterations ahead: one thread per CTA pulls the CTA's next
        // stripes (contiguous: unit index = cta * blockDim + thread) into L2, so the loads
        // below hit L2 instead of waiting on HBM latency.
        if (threadIdx.x < 4 && prefetch > 0) {
            const long long pu = u - threadIdx.x + (prefetch * 4 + threadIdx.x) * GT;
            if (pu + static_cast<long long>(blockDim.x) <= NU)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rows4 + pu),
                             "r"(static_cast<unsigned>(blockDim.x * 16))
                             : "memory");
        }
        // rows appended during this launch: L2-coherent loads (never the non-coherent path)
        const uint4 v0 = ld_row4(rows4 + u, LOADM), v1 = ld_row4(rows4 + u + GT, LOADM),
                    v2 = ld_row4(rows4 + u + 2 * GT, LOADM), v3 = ld_row4(rows4 + u + 3 * GT, LOADM);
        consider8(M, W, Wf, U, v0, v1, v2, v3, best, wfloor);
    }
    for (; u < NU; u += GT) consider2(M, W, U, __ldcg(rows4 + u), best);
    return best;
}

// W[e] = need * U[e] for need = 1 - comp[svc] > 0, else 0 (greedy.hpp:38-41).
__device__ __forceinline__ double w_of(const double* comp, const double* U, int svc, int e, int n) {
    if (svc >= n) return 0.0;
    const double need = __dadd_rn(1.0, -comp[svc]);
    return need > 0.0 ? __dmul_rn(need, U[e]) : 0.0;
}

__device__ __forceinline__ long long binom(long long a, int q) {
    if (a < q) return 0;
    if (q == 1) return a;
    if (q == 2) return a * (a - 1) / 2;
    return a * (a - 1) * (a - 2) / 6;
}

// colex unranking of a q-subset (q <= 3) of {0..m-1}; out ascending.
__device__ __forceinline__ void unrank(long long r, int q, int m, int* out) {
    for (int c = q; c >= 1; --c) {
        int lo = c - 1, hi = m - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (binom(mid, c) <= r) lo = mid;
            else hi = mid - 1;
        }
        out[c - 1] = lo;
        r -= binom(lo, c);
    }
}

// ---- TMA ring (cp.async.bulk + mbarrier) for the streaming part of the scan
constexpr int kWarpChunk = 128;    // units per warp slot (4 per lane: one consider8)
constexpr int kStageUnits = 32 * kWarpChunk;  // one stage: a 2 KB slot for each of up to 32 warps
constexpr int kMaxStages = 8;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "MBAR_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra MBAR_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// One elected thread: expect `bytes` on `bar`, then bulk-copy them global -> shared (TMA).
__device__ __forceinline__ void tma_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

struct GreedySmem {  // byte offsets into dynamic shared memory
    int W, Wf, U, comp, best, evmask, evof, evsvc, xlist, cache, ring, total;
};

__host__ __device__ inline GreedySmem greedy_layout(int n, int PP, int cache_units, int stages) {
    GreedySmem s;
    const int nW = (n + 1) * PP;
    int o = 0;
    s.W = o;
    o += nW * 8;
    s.Wf = o;
    o += ((nW * 4 + 15) / 16) * 16;
    s.U = o;
    o += nW * 8;
    s.comp = o;
    o += (n + 1) * 8;
    s.best = o;
    o += (n + 1) * 8;
    s.evmask = o;
    o += (n + 1) * 4 * 8;
    s.evof = o;
    o += (n + 1) * 2;
    s.evsvc = o;
    o += (n + 1) * 2;
    s.xlist = o;
    o += 256;
    o = (o + 15) & ~15;
    s.cache = o;
    o += cache_units * 16;
    o = (o + 127) & ~127;
    s.ring = o;
    o += stages * kStageUnits * 16;
    s.total = o;
    return s;
}

}  // namespace

// ---------------------------------------------------------------- K1: base pool rows
// One warp per support (<= max_mix members, ascending service index); valid templates
// are written at a host-computed offset in template order (deterministic pool order).
__global__ void __launch_bounds__(256) enum_base_kernel(const __grid_constant__ DevModel M,
                                                        const uint32_t* __restrict__ supports,
                                                        const long long* __restrict__ offsets, int n_supports,
                                                        uint64_t* __restrict__ rows) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (warp >= n_supports) return;
    const uint32_t sp = supports[warp];
    int s[4], k = 0;
    for (int j = 0; j < 4; ++j) {
        int v = (sp >> (8 * j)) & 0xFF;
        if (v == 0xFF) break;
        s[k++] = v;
    }
    long long base = offsets[warp];
    const int nt = M.n_tmpl[k];
    for (int t0 = 0; t0 < nt; t0 += 32) {
        const int t = t0 + static_cast<int>(lane_id());
        bool ok = t < nt;
        uint64_t row = 0;
        if (ok) {
            uint64_t tp = M.tmpl[k][t];
            for (int j = 0; j < 4; ++j) {
                uint64_t code;
                if (j < k) {
                    int p = static_cast<int>((tp >> (8 * (j + 1))) & 0xFF);
                    ok &= (M.pat_mask[p] & ~M.feas_mask[s[j]]) == 0;
                    code = static_cast<uint64_t>(s[j] * M.PP + p);
                } else {
                    code = static_cast<uint64_t>(M.n * M.PP);
                }
                row |= code << (16 * j);
            }
        }
        unsigned b = __ballot_sync(0xffffffffu, ok);
        if (ok) rows[base + __popc(b & lanemask_lt())] = row;
        base += __popc(b);
    }
}

// ---------------------------------------------------------------- K2+K3: persistent greedy
// Working set = arena rows [0, n_base + ext_count): the base pool (copied in by the host)
// followed by extension rows appended on the device.  Rows are processed in 16-byte units
// (two rows) assigned grid-stride; the first `cache_units / blockDim` units of every
// thread live in this CTA's shared memory once complete, so a working set of up to
// ~148 x 200 KB is scanned on-chip every step and only the excess streams from L2/HBM.
// One launch may carry several independent instances ("groups"): the ranks of a sharded
// greedy that share one GPU run as CTA ranges of ONE cooperative grid, so their per-step
// exchange never depends on two kernels being co-scheduled.  bi / G are the CTA index and
// CTA count of this CTA's instance.
template <int NT>
__global__ void __launch_bounds__(NT, 1) greedy_kernel(const __grid_constant__ GreedyLaunch GL) {
    constexpr int NW = NT / 32;
#ifdef MGB_GREEDY_PRINT_PHASES
    const unsigned long long t_entry = globaltimer();
#endif
    extern __shared__ __align__(16) unsigned char smem[];
    const int grp = static_cast<int>(blockIdx.x) / GL.ctas_per_group;
    const GreedyArgs& a = GL.g[grp];
    const int G = GL.ctas_per_group;
    const int bi = static_cast<int>(blockIdx.x) - grp * G;
    const DevModel& M = a.M;
    const int n = M.n, PP = M.PP;
    const int nW = (n + 1) * PP;
    const GreedySmem L = greedy_layout(n, PP, a.cache_units, a.ring_stages);
    double* W = reinterpret_cast<double*>(smem + L.W);
    float* Wf = reinterpret_cast<float*>(smem + L.Wf);
    double* U = reinterpret_cast<double*>(smem + L.U);
    double* comp = reinterpret_cast<double*>(smem + L.comp);
    double* best_single = reinterpret_cast<double*>(smem + L.best);
    uint64_t* ev_mask = reinterpret_cast<uint64_t*>(smem + L.evmask);
    short* ev_of = reinterpret_cast<short*>(smem + L.evof);
    short* ev_svc = reinterpret_cast<short*>(smem + L.evsvc);
    uint8_t* xlist = smem + L.xlist;
    uint4* cache = reinterpret_cast<uint4*>(smem + L.cache);
    uint4* ring = reinterpret_cast<uint4*>(smem + L.ring);
    __shared__ __align__(8) unsigned long long wbar[kMaxStages][NW];  // per-warp TMA slots
    const int S = a.ring_stages;
    if (lane_id() == 0 && S > 0) {
        for (int q = 0; q < S; ++q) mbar_init(&wbar[q][threadIdx.x >> 5], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __shared__ Best red[NW];
    __shared__ Best xch[2];  // cluster mode: this CTA's block best, by step parity
    __shared__ uint64_t unsat[4];
    __shared__ int s_events, s_first_new, s_done, s_m, s_status;
    __shared__ long long s_rows;
    if (threadIdx.x == 0) s_status = kOk;

    for (int e = threadIdx.x; e < nW; e += blockDim.x) U[e] = __ldg(&M.U[e]);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        comp[i] = a.comp0[i];
        best_single[i] = M.best_single[i];
        ev_of[i] = -1;
    }
    if (threadIdx.x == 0) s_events = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < nW; e += blockDim.x) {
        W[e] = w_of(comp, U, e / PP, e, n);
        Wf[e] = __double2float_ru(W[e]);
    }

    // maybe_extend (greedy.hpp:107-119), warp 0, identical in every CTA.
    auto maybe_extend = [&]() {
        if ((threadIdx.x >> 5) == 0) {
            uint64_t um[4] = {0, 0, 0, 0};
            const int chunks = (n + 31) / 32;
            for (int c = 0; c < chunks; ++c) {
                int i = c * 32 + static_cast<int>(lane_id());
                bool un = i < n && comp[i] < 1.0 - 1e-9;
                unsigned b = __ballot_sync(0xffffffffu, un);
                um[c >> 1] |= static_cast<uint64_t>(b) << (32 * (c & 1));
            }
            int ev = s_events;
            const int first = ev;
            for (int c = 0; c < chunks; ++c) {
                int i = c * 32 + static_cast<int>(lane_id());
                bool e = i < n && ((um[i >> 6] >> (i & 63)) & 1ull) && ev_of[i] < 0 &&
                         __dadd_rn(1.0, -comp[i]) < best_single[i];
                unsigned b = __ballot_sync(0xffffffffu, e);
                if (e) {
                    int pos = ev + __popc(b & lanemask_lt());
                    ev_of[i] = static_cast<short>(pos);
                    ev_svc[pos] = static_cast<short>(i);
                    for (int w = 0; w < 4; ++w) ev_mask[pos * 4 + w] = um[w];
                    if (bi == 0) a.ev_svc[pos] = i;
                }
                ev += __popc(b);
            }
            __syncwarp();  // every lane has read s_events / unsat before lane 0 rewrites them
            if (lane_id() == 0) {
                for (int w = 0; w < 4; ++w) unsat[w] = um[w];
                s_first_new = first;
                s_events = ev;
                s_done = (um[0] | um[1] | um[2] | um[3]) == 0ull;
            }
        }
        __syncthreads();
    };

    // Device-side extend_candidate_pool for the events recorded since `first`
    // (config_enum.hpp:206-211 with must_include = i, allowed = unsat, max_mix = 4):
    // every support S, max_mix < |S| <= 4, i in S subset-of unsat, not covered by an earlier
    // event e' (i_e' in S subset-of unsat_e'), times every feasible template.
    // Two levels per warp: the 32 lanes unrank and coverage-test 32 supports at once; then
    // the warp walks the surviving supports (ballot order) and its lanes take that support's
    // templates, so each support is unranked once and the appends stay warp-aggregated.
    auto extend_new = [&](int first, int last) {
        const int ln = static_cast<int>(lane_id());
        const long long gw = static_cast<long long>(bi) * NW + (threadIdx.x >> 5);
        const long long GW = static_cast<long long>(G) * NW;
        for (int e = first; e < last; ++e) {
            __syncthreads();
            const int ie = ev_svc[e];
            const uint64_t* me = ev_mask + e * 4;
            if ((threadIdx.x >> 5) == 0) {
                int m = 0;
                for (int c = 0; c < (n + 31) / 32; ++c) {
                    int i = c * 32 + ln;
                    bool in = i < n && i != ie && ((me[i >> 6] >> (i & 63)) & 1ull);
                    unsigned b = __ballot_sync(0xffffffffu, in);
                    if (in) xlist[m + __popc(b & lanemask_lt())] = static_cast<uint8_t>(i);
                    m += __popc(b);
                }
                if (ln == 0) s_m = m;
            }
            __syncthreads();
            const int m = s_m;
            // sharded greedy: support (event e, size k, colex rank r) belongs to rank
            // (r + k + e) mod P, so each rank unranks only its own supports r = off[k] + j*P
            const int P = a.n_ranks > 1 ? a.n_ranks : 1;
            long long cnt[5] = {0, 0, 0, 0, 0};
            int off[5] = {0, 0, 0, 0, 0};
            long long total = 0;
            for (int k = M.max_mix + 1; k <= 4; ++k) {
                const long long B = binom(m, k - 1);
                off[k] = P > 1 ? ((a.rank - k - e) % P + P) % P : 0;
                cnt[k] = B > off[k] ? (B - off[k] + P - 1) / P : 0;
                total += cnt[k];
            }
            // batch width: 32 supports per warp when there is work for every warp's lanes,
            // fewer (down to 1) for small events so every warp of the grid gets a share
            const long long bw = min(32ll, max(1ll, (total + GW - 1) / GW));
            for (long long base = gw * bw; base < total; base += GW * bw) {
                // level 1: lane = one support
                const long long g = base + ln;
                bool live = ln < bw && g < total;
                int k = M.max_mix + 1;
                unsigned packed = 0xFFFFFFFFu;  // members, ascending, one byte each (0xFF unused)
                if (live) {
                    long long rem = g;
                    while (rem >= cnt[k]) rem -= cnt[k++];
                    const long long r = off[k] + rem * P;
                    int idx[3];
                    unrank(r, k - 1, m, idx);
                    int S[4];
                    int q = 0, placed = 0;
                    for (int j = 0; j < k - 1; ++j) {
                        int v = xlist[idx[j]];
                        if (!placed && ie < v) {
                            S[q++] = ie;
                            placed = 1;
                        }
                        S[q++] = v;
                    }
                    if (!placed) S[q++] = ie;
                    for (int j = 0; j < k && live; ++j) {  // covered by an earlier event?
                        int ev = ev_of[S[j]];
                        if (ev >= 0 && ev < e) {
                            const uint64_t* mk = ev_mask + ev * 4;
                            bool sub = true;
                            for (int x = 0; x < k; ++x) sub &= ((mk[S[x] >> 6] >> (S[x] & 63)) & 1ull) != 0;
                            if (sub) live = false;
                        }
                    }
                    packed = 0;
                    for (int j = 0; j < 4; ++j) packed |= static_cast<unsigned>(j < k ? S[j] : 0xFF) << (8 * j);
                }
                // level 2: the warp takes each surviving support's templates.  A support's rows
                // are appended as ONE contiguous run (one atomic for all its feasible templates,
                // in template order): the scan's lanes then gather the Wf codes of one support's
                // consecutive templates — few distinct shared-memory banks per gather — instead of
                // interleaved 32-row pieces of several supports (bank conflicts, ncu r02).
                unsigned todo = __ballot_sync(0xffffffffu, live);
                while (todo) {
                    const int src = __ffs(todo) - 1;
                    todo &= todo - 1;
                    const unsigned sp = __shfl_sync(0xffffffffu, packed, src);
                    const int kk = __shfl_sync(0xffffffffu, k, src);
                    int S[4];
                    for (int j = 0; j < 4; ++j) S[j] = static_cast<int>((sp >> (8 * j)) & 0xFFu);
                    const int nt = M.n_tmpl[kk];
                    auto make = [&](int t, uint64_t& row) {
                        bool ok = t < nt;
                        row = 0;
                        if (ok) {
                            const uint64_t tp = M.tmpl[kk][t];
                            for (int j = 0; j < 4; ++j) {
                                uint64_t code;
                                if (j < kk) {
                                    int p = static_cast<int>((tp >> (8 * (j + 1))) & 0xFF);
                                    ok &= (M.pat_mask[p] & ~M.feas_mask[S[j]]) == 0;
                                    code = static_cast<uint64_t>(S[j] * PP + p);
                                } else {
                                    code = static_cast<uint64_t>(n * PP);
                                }
                                row |= code << (16 * j);
                            }
                        }
                        return ok;
                    };
#ifdef MIGPLAN_EXT_PIECES
                    for (int t0 = 0; t0 < nt; t0 += 32) {
                        uint64_t row;
                        const bool ok = make(t0 + ln, row);
                        const unsigned b = __ballot_sync(0xffffffffu, ok);
                        if (b) {
                            unsigned long long at = 0;
                            if (ln == 0) at = atomicAdd(&a.st->ext_count, static_cast<unsigned long long>(__popc(b)));
                            at = __shfl_sync(0xffffffffu, at, 0);
                            if (a.n_base + static_cast<long long>(at + __popc(b)) > a.cap) {
                                if (ln == 0) atomicExch(&a.st->status, static_cast<int>(kExtOverflow));
                            } else if (ok) {
                                a.rows[a.n_base + static_cast<long long>(at) + __popc(b & lanemask_lt())] = row;
                            }
                        }
                    }
#else
                    int cnt = 0;
                    for (int t0 = 0; t0 < nt; t0 += 32) {
                        uint64_t row;
                        cnt += __popc(__ballot_sync(0xffffffffu, make(t0 + ln, row)));
                    }
                    if (cnt == 0) continue;
                    unsigned long long at = 0;
                    if (ln == 0) at = atomicAdd(&a.st->ext_count, static_cast<unsigned long long>(cnt));
                    at = __shfl_sync(0xffffffffu, at, 0);
                    if (a.n_base + static_cast<long long>(at + cnt) > a.cap) {
                        if (ln == 0) atomicExch(&a.st->status, static_cast<int>(kExtOverflow));
                        continue;
                    }
                    for (int t0 = 0; t0 < nt; t0 += 32) {
                        uint64_t row;
                        const bool ok = make(t0 + ln, row);
                        const unsigned b = __ballot_sync(0xffffffffu, ok);
                        if (ok) a.rows[a.n_base + static_cast<long long>(at) + __popc(b & lanemask_lt())] = row;
                        at += __popc(b);
                    }
#endif
                }
            }
        }
    };

    unsigned* bc = &a.st->bar_count;
    unsigned* bg = &a.st->bar_gen;
    int status = kOk;

    // Rows in the working set and the overflow status change only at extension events:
    // read them once after each extension barrier instead of every step.
    long long N = a.n_base;
    auto extend_and_sync = [&]() {
        extend_new(s_first_new, s_events);
        if (GL.cluster)
            cg::this_cluster().sync();  // release/acquire at cluster scope: the appended rows
        else
            grid_barrier(bc, bg, G);
        if (threadIdx.x == 0) {
            s_status = *reinterpret_cast<volatile int*>(&a.st->status);
            s_rows = a.n_base + static_cast<long long>(*reinterpret_cast<volatile unsigned long long*>(&a.st->ext_count));
        }
        __syncthreads();
        N = s_rows;
    };
    maybe_extend();
    if (s_events > s_first_new) extend_and_sync();

    const uint4* rows4 = reinterpret_cast<const uint4*>(a.rows);
    const long long GT = static_cast<long long>(G) * blockDim.x;
    // The thread's first unit; its units are my0 + k * GT.  Streaming scans give each CTA 512
    // contiguous units per stride (the bulk L2 prefetch fetches them); when the whole working
    // set lives in the row caches, 32-unit blocks are dealt round-robin over the CTAs instead,
    // so every CTA holds a slice of each pool region (base rows, each extension event) and the
    // per-step scan work is balanced.
    const long long my0 = a.interleave ? (static_cast<long long>(threadIdx.x >> 5) * G + bi) * 32 + (threadIdx.x & 31)
                                       : static_cast<long long>(bi) * blockDim.x + threadIdx.x;
    const int J = a.cache_units / static_cast<int>(blockDim.x);  // cached units per thread
    int cj = 0;                                                  // units of mine cached so far

    int step = 0;
    unsigned long long t_win = 0;   // diagnostics (phase timers)
    uint64_t prev_row = kNoRow;     // this thread's best row of the previous step
    unsigned long long kchunk = 0;  // TMA ring chunks consumed by this CTA (all steps)
    unsigned long long last_seq = a.exch_seq0;
    long long rows_total = 0;
    const bool timer = a.phase_timers && bi == 0 && threadIdx.x == 0;
    unsigned long long ph[5] = {0, 0, 0, 0, 0};
    unsigned long long tp = timer ? globaltimer() : 0;
    auto mark = [&](int k) {
        if (timer) {
            unsigned long long t = globaltimer();
            ph[k] += t - tp;
            tp = t;
        }
    };
#ifdef MGB_GREEDY_PRINT_PHASES
    const unsigned long long t_loop = globaltimer();
#endif
    while (!s_done) {
        if (s_status != kOk) {
            status = s_status;
            break;
        }
        if (step >= a.cap_steps) {
            status = kStepOverflow;
            break;
        }
        mark(4);
        unsigned long long t_scan0 = 0;
        if (a.phase_timers && threadIdx.x == 0) {  // diagnostics: per-CTA scan and post-argmax time
            t_scan0 = globaltimer();
            if (t_win) g_post[blockIdx.x] += t_scan0 - t_win;
        }
        const long long NU = N >> 1;  // complete 16-byte units
        while (cj < J && my0 + cj * GT < NU) {  // pull newly complete units of mine on-chip
            cache[cj * blockDim.x + threadIdx.x] = __ldcg(rows4 + my0 + cj * GT);
            ++cj;
        }
        // Start from this thread's previous best row, re-scored: it is one of the thread's own
        // rows (the working set only grows), so the argmax is unchanged, and its score is a
        // high floor from the first row on (scores only fall as the completion rises), so the
        // FP32 filter sends almost no row down the exact path.
        Best best = none();
        if (prev_row != kNoRow) {
            const double s0 = row_score(W, prev_row);
            if (s0 > 0.0) best = Best{s0, row_usum(U, prev_row), prev_row};
        }
        double wfloor = best.s;  // the warp's best re-scored row: a common floor for its lanes
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) wfloor = fmax(wfloor, __shfl_xor_sync(0xffffffffu, wfloor, off));
        {
            int j = 0;
            for (; j + 3 < cj; j += 4) {
                const uint4 v0 = cache[(j + 0) * blockDim.x + threadIdx.x];
                const uint4 v1 = cache[(j + 1) * blockDim.x + threadIdx.x];
                const uint4 v2 = cache[(j + 2) * blockDim.x + threadIdx.x];
                const uint4 v3 = cache[(j + 3) * blockDim.x + threadIdx.x];
                consider8(M, W, Wf, U, v0, v1, v2, v3, best, wfloor);
            }
            for (; j < cj; ++j) consider2(M, W, U, cache[j * blockDim.x + threadIdx.x], best);
            long long u = my0 + static_cast<long long>(cj) * GT;
            if (S > 0) {
                // Rows beyond the on-chip cache, TMA-staged per WARP: the streamed region is cut
                // into 2 KB warp-chunks (128 units: one consider8 per lane) dealt round-robin over
                // the grid's warps; each warp keeps S chunks in flight in its own shared-memory
                // slots (lane 0 issues cp.async.bulk, a per-warp mbarrier completes on the bytes),
                // so the bytes in flight live in the TMA engine, not in registers, and no warp
                // ever waits for another (no CTA-wide ring barrier).
                const int w = static_cast<int>(threadIdx.x >> 5), ln = static_cast<int>(lane_id());
                const long long base_u = static_cast<long long>(J) * GT;
                const long long n_ch = NU > base_u ? (NU - base_u + kWarpChunk - 1) / kWarpChunk : 0;
                const long long gw = static_cast<long long>(bi) * NW + w, GW = static_cast<long long>(G) * NW;
                const long long my_n = n_ch > gw ? (n_ch - gw + GW - 1) / GW : 0;
                uint4* wr = ring + w * kWarpChunk;  // slot q of this warp: wr + q * kStageUnits
                auto issue = [&](long long i) {     // lane 0
                    const unsigned long long kk = kchunk + static_cast<unsigned long long>(i);
                    const int slot = static_cast<int>(kk % S);
                    const long long u0 = base_u + (gw + i * GW) * kWarpChunk;
                    const long long cnt = min(static_cast<long long>(kWarpChunk), NU - u0);
                    tma_load(wr + static_cast<long long>(slot) * kStageUnits, rows4 + u0, static_cast<unsigned>(cnt * 16),
                             &wbar[slot][w]);
                };
                if (ln == 0 && my_n > 0) {
                    asm volatile("fence.proxy.async.global;" ::: "memory");  // rows appended this launch
                    for (long long i = 0; i < my_n && i < S; ++i) issue(i);
                }
                const uint64_t pad = static_cast<uint64_t>(n * PP) * 0x0001000100010001ull;  // 4 sentinel codes
                const uint4 padv = make_uint4(static_cast<unsigned>(pad), static_cast<unsigned>(pad >> 32),
                                              static_cast<unsigned>(pad), static_cast<unsigned>(pad >> 32));
                for (long long i = 0; i < my_n; ++i) {
                    const unsigned long long kk = kchunk + static_cast<unsigned long long>(i);
                    const int slot = static_cast<int>(kk % S);
                    mbar_wait(&wbar[slot][w], static_cast<unsigned>((kk / S) & 1ull));
                    const long long u0 = base_u + (gw + i * GW) * kWarpChunk;
                    const int cnt = static_cast<int>(min(static_cast<long long>(kWarpChunk), NU - u0));
                    const uint4* st = wr + static_cast<long long>(slot) * kStageUnits;
                    const uint4 v0 = ln < cnt ? st[ln] : padv;
                    const uint4 v1 = ln + 32 < cnt ? st[ln + 32] : padv;
                    const uint4 v2 = ln + 64 < cnt ? st[ln + 64] : padv;
                    const uint4 v3 = ln + 96 < cnt ? st[ln + 96] : padv;
                    consider8(M, W, Wf, U, v0, v1, v2, v3, best, wfloor);
                    __syncwarp();  // every lane has consumed its slot data: the slot may be refilled
                    if (ln == 0 && i + S < my_n) issue(i + S);
                }
                kchunk += static_cast<unsigned long long>(my_n);
                u = NU;  // everything beyond the cache was streamed
            }
            if (u < NU)
                best = scan_stream(M, W, Wf, U, rows4, u, NU, GT, a.prefetch, a.pipeline, best, wfloor);
            if ((N & 1) && my0 == 0) consider(M, W, U, __ldcg(a.rows + N - 1), best);
        }
        prev_row = best.row;
        const Best bb = block_best(M, best, red);
        if (a.phase_timers && threadIdx.x == 0) g_scan[blockIdx.x] += globaltimer() - t_scan0;
#ifdef MGB_GREEDY_STEP_DIAG
        if (threadIdx.x == 0 && step < kDiagSteps) {
            const unsigned long long dt = globaltimer() - t_scan0;
            atomicMax(&g_sd_max[step], dt);
            atomicAdd(&g_sd_sum[step], dt);
            const unsigned c = atomicExch(&g_sd_cnt[blockIdx.x], 0u);
            atomicMax(&g_sd_exact[step], static_cast<unsigned long long>(c));
            atomicMax(&g_sd_arg[step], (dt << 12) | blockIdx.x);
            const unsigned kc = atomicExch(&g_sd_keys[blockIdx.x], 0u);
            atomicMax(&g_sd_key[step], static_cast<unsigned long long>(kc));
        }
#endif
        mark(0);
        last_seq = a.exch_seq0 + static_cast<unsigned long long>(step) + 1ull;
        const Best win = GL.cluster               ? cluster_argmax(M, bb, xch, step & 1, red, G)
                         : a.n_ranks == 1
                             ? grid_allreduce_argmax(M, bb, a.partials, &a.st->arrive, G, step, red, bi)
                             : grid_argmax(M, bb, a.partials, a.partials + G, bc, bg, G, red, a, last_seq,
                                           &a.st->status, bi);
        mark(1);
        if (a.phase_timers && threadIdx.x == 0) t_win = globaltimer();
        if (win.row == kNoRow) {
            const int xs = *reinterpret_cast<volatile int*>(&a.st->status);
            status = xs != kOk ? xs : kNoPositive;
            break;
        }
        rows_total += N;
        if (threadIdx.x == 0) {
            for (int j = 0; j < 4; ++j) {
                int code = static_cast<int>((win.row >> (16 * j)) & 0xFFFFull);
                int svc = code / PP;
                if (svc < n) comp[svc] = __dadd_rn(comp[svc], U[code]);
            }
            if (bi == 0) {
                a.pick_row[step] = win.row;
                a.pick_score[step] = win.s;
                a.pick_rows[step] = N;
            }
        }
        __syncthreads();
        // only the winner's (<= 4) services changed: refresh their W rows
        for (int e = threadIdx.x; e < 4 * PP; e += blockDim.x) {
            const int j = e / PP, p = e - j * PP;
            const int svc = static_cast<int>((win.row >> (16 * j)) & 0xFFFFull) / PP;
            if (svc < n) {
                W[svc * PP + p] = w_of(comp, U, svc, svc * PP + p, n);
                Wf[svc * PP + p] = __double2float_ru(W[svc * PP + p]);
            }
        }
        ++step;
        mark(2);
        maybe_extend();  // ends with __syncthreads (also publishes the W refresh)
        mark(3);
        if (s_events > s_first_new) extend_and_sync();
    }
    mark(4);
#ifdef MGB_GREEDY_PRINT_PHASES
    const unsigned long long t_end = globaltimer();
#endif
    if (GL.cluster) cg::this_cluster().sync();  // peers may still read this CTA's xch over DSMEM
    if (bi == 0) {  // one coalesced copy of the plan to host-mapped memory
        for (int i = threadIdx.x; i < step; i += blockDim.x) {
            a.host_pick_row[i] = a.pick_row[i];
            a.host_pick_score[i] = a.pick_score[i];
            a.host_pick_rows[i] = a.pick_rows[i];
        }
    }
    if (bi == 0 && threadIdx.x == 0) {
        if (status != kOk) atomicExch(&a.st->status, status);
        __threadfence();
        GreedyState* o = a.out;  // host-mapped: the host reads it after one stream sync
        for (int k = 0; k < 5; ++k) o->phase_ns[k] = ph[k];
        o->n_steps = step;
        o->last_seq = last_seq;
        o->n_events = s_events;
        o->rows_scored = rows_total;
        o->ext_count = *reinterpret_cast<volatile unsigned long long*>(&a.st->ext_count);
        o->status = *reinterpret_cast<volatile int*>(&a.st->status);
        __threadfence_system();
#ifdef MGB_GREEDY_STEP_DIAG
        for (int q = 0; q < step && q < kDiagSteps; ++q) {
            printf("[step %d] rows %lld scan max %.2f us (cta %llu) mean %.2f us, max exact rows/cta %llu, max key compares/cta %llu\n", q,
                   a.pick_rows[q], g_sd_max[q] / 1e3, g_sd_arg[q] & 4095ull, g_sd_sum[q] / 1e3 / G, g_sd_exact[q], g_sd_key[q]);
            g_sd_max[q] = g_sd_sum[q] = g_sd_exact[q] = g_sd_arg[q] = g_sd_key[q] = 0;
        }
#endif
#ifdef MGB_GREEDY_PRINT_PHASES
        const unsigned long long t_exit = globaltimer();
        printf("[greedy cta0] prologue %.1f us (events %d), loop %.1f us (%d steps), epilogue %.1f us, G %d\n",
               (t_loop - t_entry) / 1e3, s_events, (t_end - t_loop) / 1e3, step, (t_exit - t_end) / 1e3, G);
#endif
    }
}

// ---------------------------------------------------------------- K4 (k > 32): top-K
// k rounds of "argmax among rows strictly less preferred than the previous pick";
// because candidate_preferred is a total order this yields the reference's sorted
// top-K (mcts.hpp:68-71) without materialising or sorting all scores.
__global__ void __launch_bounds__(kThreads, 1) topk_kernel(const __grid_constant__ TopkArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const DevModel& M = a.M;
    const int nW = (M.n + 1) * M.PP;
    double* W = reinterpret_cast<double*>(smem);
    double* comp = W + nW;
    __shared__ Best red[kWarps];
    __shared__ uint64_t mask[4];
    for (int i = threadIdx.x; i < M.n; i += blockDim.x) comp[i] = a.comp[i];
    if (threadIdx.x < 4) mask[threadIdx.x] = a.svc_mask ? a.svc_mask[threadIdx.x] : ~0ull;
    __syncthreads();
    for (int e = threadIdx.x; e < nW; e += blockDim.x) W[e] = w_of(comp, M.U, e / M.PP, e, M.n);
    __syncthreads();
    const int G = gridDim.x;
    const long long total = a.index ? a.n_index : a.n_rows;
    const long long stride = static_cast<long long>(G) * blockDim.x;
    Best last = none();
    int got = 0;
    for (int r = 0; r < a.k; ++r) {
        Best best = none();
        for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
            const uint64_t row = __ldg(a.rows + (a.index ? a.index[i] : i));
            if (a.svc_mask) {
                bool hit = false;
                for (int j = 0; j < 4; ++j) {
                    int svc = static_cast<int>(((row >> (16 * j)) & 0xFFFFull) / M.PP);
                    if (svc < M.n) hit |= ((mask[svc >> 6] >> (svc & 63)) & 1ull) != 0;
                }
                if (!hit) continue;
            }
            const double s = row_score(W, row);
            if (!(s > 0.0)) continue;
            if (r > 0 && s >= last.s) {
                Best c{s, row_usum(M.U, row), row};
                if (!better(M, last, c)) continue;
                if (best.row == kNoRow || better(M, c, best)) best = c;
                continue;
            }
            if (s >= best.s) {
                Best c{s, row_usum(M.U, row), row};
                if (best.row == kNoRow || better(M, c, best)) best = c;
            }
        }
        best = block_best(M, best, red);
        Best* part = a.partials + (r & 1) * G;
        if (threadIdx.x == 0) part[blockIdx.x] = best;
        grid_barrier(a.bar, a.bar + 1, G);
        const Best win = grid_best(M, part, G, red);
        if (win.row == kNoRow) break;
        if (blockIdx.x == 0 && threadIdx.x == 0) a.out_row[r] = win.row;
        last = win;
        ++got;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.n_out = got;
}

// ---------------------------------------------------------------- launch helpers
size_t greedy_smem_bytes(int n, int PP, int cache_units, int stages) {
    return static_cast<size_t>(greedy_layout(n, PP, cache_units, stages).total);
}
int greedy_chunk_bytes() { return kStageUnits * 16; }

size_t topk_smem_bytes(int n, int PP) { return static_cast<size_t>((n + 1) * PP + n) * 8 + 16; }

const void* greedy_kernel_ptr() { return reinterpret_cast<const void*>(&greedy_kernel<kThreads>); }

// Set-up of a grouped greedy launch in ONE kernel (blockIdx.y = instance): each instance's
// GreedyState zeroed and its arena seeded with the base pool — instead of a memset and a
// device-to-device copy enqueued per instance (host API time dominated the GA refills' set-up).
__global__ void greedy_batch_init_kernel(const __grid_constant__ GreedyLaunch GL, const uint64_t* base, long long n_base) {
    const GreedyArgs& a = GL.g[blockIdx.y];
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i < static_cast<int>(sizeof(GreedyState)); i += blockDim.x)
            reinterpret_cast<unsigned char*>(a.st)[i] = 0;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_base;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        a.rows[i] = base[i];
}
void launch_greedy_batch_init(const GreedyLaunch& L, const uint64_t* base, long long n_base, cudaStream_t st) {
    const int bx = static_cast<int>(std::min<long long>(64, std::max<long long>(1, (n_base + 255) / 256)));
    greedy_batch_init_kernel<<<dim3(bx, L.n_groups), 256, 0, st>>>(L, base, n_base);
}
const void* topk_kernel_ptr() { return reinterpret_cast<const void*>(&topk_kernel); }
const void* enum_base_kernel_ptr() { return reinterpret_cast<const void*>(&enum_base_kernel); }
int kernel_threads() { return kThreads; }

void greedy_read_diag(unsigned long long* skew_ns, unsigned long long* release_ns) {
    cudaMemcpyFromSymbol(skew_ns, g_skew_ns, 8);
    cudaMemcpyFromSymbol(release_ns, g_release_ns, 8);
    static unsigned long long d[1024];
    for (int which = 0; which < 2; ++which) {
        cudaMemcpyFromSymbol(d, which ? g_post : g_scan, sizeof d);
        unsigned long long mn = ~0ull, mx = 0, sum = 0;
        int cnt = 0, amx = 0, amn = 0;
        for (int i = 0; i < 1024; ++i)
            if (d[i]) {
                if (d[i] > mx) mx = d[i], amx = i;
                if (d[i] < mn) mn = d[i], amn = i;
                sum += d[i];
                ++cnt;
            }
        if (cnt)
            fprintf(stderr, "[greedy] per-CTA %s total: min %.3f ms (cta %d) avg %.3f max %.3f ms (cta %d)\n",
                    which ? "post-argmax" : "scan", mn * 1e-6, amn, sum * 1e-6 / cnt, mx * 1e-6, amx);
    }
    cudaMemcpyFromSymbol(d, g_cta_dur, sizeof d);
    unsigned long long mn = ~0ull, mx = 0, sum = 0;
    int cnt = 0, amx = 0, amn = 0;
    for (int i = 0; i < 1024; ++i)
        if (d[i]) {
            if (d[i] > mx) mx = d[i], amx = i;
            if (d[i] < mn) mn = d[i], amn = i;
            sum += d[i];
            ++cnt;
        }
    if (cnt)
        fprintf(stderr, "[greedy] per-CTA scan total: min %.3f ms (cta %d) avg %.3f max %.3f ms (cta %d)\n", mn * 1e-6, amn,
                sum * 1e-6 / cnt, mx * 1e-6, amx);
}

}  // namespace mgb
