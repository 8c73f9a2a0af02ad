// topk_pair.cuh — the block-wide exact top-K over 32-bit pair rows (max_mix <= 2) shared by
// K7 (mcts.cu: expansions and rollout-cache misses) and K5 (rollout.cu: pool builds): both are
// detail::topk_candidates (mcts.hpp:56-76) under one completion vector.  Internal linkage: each
// including translation unit gets its own shared counters and diagnostics.
#pragma once

#include "common.cuh"

namespace mgb {

using namespace dev;

namespace {

#ifndef MGB_MCTS_THREADS
#define MGB_MCTS_THREADS 512
#endif
constexpr int kMThreads = MGB_MCTS_THREADS;  // a power-of-two number of warps (the top-K merge tree)
constexpr int kMWarps = kMThreads / 32;
constexpr int kMCandCap = 512;  // above-threshold rows per top-K (ties beyond: exact k-round path)
constexpr int kMMaxK = 32;

__device__ unsigned g_mcts_fallbacks = 0;  // diagnostics: exact-path top-Ks (MIGPLAN_MCTS_TIMERS)
// diagnostics (MctsLaunch::timers): top-K phase cycles seen by thread 0 — tables, pass 1 +
// threshold, pass 2, rank + output — then Σ candidates and calls
__device__ unsigned long long g_tk[12];  // [6]: pass-2 rescans; [8..10]: pair top-K warps' scan end, max/mean/min

// Candidates here carry pos | keyrank[pos] << 32: the config-order tie-break (core.hpp:174-200)
// becomes one integer compare instead of decoding both rows.
__device__ __forceinline__ bool precedes_kr(const Cand& j, const Cand& i) {
    if (j.s != i.s) return j.s > i.s;
    if (j.row == i.row) return static_cast<unsigned>(j.pos) < static_cast<unsigned>(i.pos);
    if (j.u != i.u) return j.u > i.u;
    return (j.pos >> 32) < (i.pos >> 32);
}
__device__ __forceinline__ long long pack_pos(const unsigned* keyrank, long long pos) {
    return pos | (static_cast<long long>(keyrank[pos]) << 32);
}
__device__ __forceinline__ int pos_of(const Cand& c) { return static_cast<int>(c.pos & 0xffffffffll); }

// rank_select (common.cuh) with a warp per candidate and the packed key rank.
__device__ __forceinline__ void rank_select_kr(const Cand* cand, int nc, int k, Cand* out) {
    const int lane = static_cast<int>(threadIdx.x & 31u);
    const int nw = static_cast<int>(blockDim.x >> 5);
    for (int i = static_cast<int>(threadIdx.x >> 5); i < nc; i += nw) {
        const Cand ci = cand[i];
        int r = 0;
        for (int j0 = 0; j0 < nc && r < k; j0 += 32) {
            const int j = j0 + lane;
            bool p = false;
            if (j < nc) {  // the score decides unless it ties: load the rest only then
                const double sj = cand[j].s;
                p = sj != ci.s ? sj > ci.s : precedes_kr(cand[j], ci);
            }
            r += __popc(__ballot_sync(0xffffffffu, p));
        }
        if (lane == 0 && r < k) out[r] = ci;
    }
}

// block_topk_bound over rows of at most two members (max_mix <= 2), stored as their low 32
// bits: two bound gathers and 4 bytes per row instead of four gathers and 8 bytes.  The
// omitted members are sentinels (W = 0, U = 0), so every exact score and util_sum is the
// 64-bit row's bit for bit.
__device__ __forceinline__ float ub_pair(const float* Wf, unsigned x) { return __fadd_ru(Wf[x & 0xFFFFu], Wf[x >> 16]); }
__device__ __forceinline__ bool hit_pair(const unsigned char* hitc, unsigned x) {
    return (hitc[x & 0xFFFFu] | hitc[x >> 16]) != 0;
}
// The base pool's supports (contiguous row ranges in K1 order) and an active-list buffer; n = 0
// scans every row.
struct SupTab {
    int n;
    const int* begin;
    const unsigned short* svc;
    int* act;
    int dense_pct = -1;  // dense scan above this % of live rows (-1: g_mcts_dense_pct)
};

// block_topk_pair's block-wide counters: zero at kernel start (mcts_kernel) and re-zeroed by
// every call before its closing barrier, so a call needs no opening barrier for them.
__shared__ int tp_ncand, tp_nhit, tp_nact, tp_actrows;
#ifdef MGB_MCTS_SKEW
__shared__ long long tp_c0, tp_dmax, tp_dmin, tp_dsum;  // development aid: warps' scan-end skew
#endif
__device__ __forceinline__ void topk_pair_counters_init() {
    if (threadIdx.x == 0) tp_ncand = tp_nhit = tp_nact = tp_actrows = 0;
}
#ifndef MGB_TOPK_DENSE_PCT
#define MGB_TOPK_DENSE_PCT 60  // K7 (rows on chip); rollout.cu's pool builds (rows in L2) use 100
#endif
__device__ int g_mcts_dense_pct = MGB_TOPK_DENSE_PCT;  // dense scan when live rows exceed this % of the pool

// Inlined into mcts_kernel: as a call, the ABI's register saves around each call site pushed
// the 128-register kernel into spilling on the search's serial paths (measured: the GA
// context's searches 17.4 vs 19.4 ms per two_phase inlined vs called).
#ifdef MGB_TOPK_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
int block_topk_pair(const DevModel& M, const unsigned* keyrank, const unsigned* base, long long nb,
                               long long pos0, const double* comp, const uint64_t* mask, int k, const double* U,
                               double* W, float* Wf, unsigned char* hitc, Cand* cand, Cand* win, int* out, int* scored,
                               bool tm, SupTab sup) {
    __shared__ Cand red[kMWarps];
    long long c0 = 0, c1 = 0;
    auto mark = [&](int slot) {
        if (tm && threadIdx.x == 0) {
            c1 = clock64();
            if (slot >= 0) atomicAdd(&g_tk[slot], static_cast<unsigned long long>(c1 - c0));
            c0 = c1;
        }
    };
    mark(-1);
    const int lane = static_cast<int>(threadIdx.x & 31u);
    const int wid = static_cast<int>(threadIdx.x >> 5), nwarps = static_cast<int>(blockDim.x >> 5);
    const int nW = (M.n + 1) * M.PP;
    const unsigned sent = static_cast<unsigned>(M.n * M.PP);
    const uint64_t hiS = static_cast<uint64_t>(sent | (sent << 16)) << 32;
#ifdef MGB_MCTS_SKEW
    if (tm && threadIdx.x == 0) {
        tp_c0 = c0;
        tp_dmax = tp_dsum = 0;
        tp_dmin = 1ll << 62;
    }
#endif
    // ---- tables (W = need * U, its FP32 round-up, mask hits) and the live supports: one barrier
    for (int e = threadIdx.x; e < nW; e += blockDim.x) {
        const int svc = svc_of(M, static_cast<unsigned>(e));
        double w = 0.0;
        if (svc < M.n) {
            const double need = __dadd_rn(1.0, -comp[svc]);
            if (need > 0.0) w = __dmul_rn(need, U[e]);
        }
        W[e] = w;
        Wf[e] = __double2float_ru(w);
        if (mask) hitc[e] = svc < M.n && ((mask[svc >> 6] >> (svc & 63)) & 1ull) != 0;
    }
    // Supports that can hold a candidate: a member with need > 0 (rows of the others all score
    // 0), or, with a mask, a sampled member (every row of such a support touches it).
    const int dense_pct = sup.dense_pct >= 0 ? sup.dense_pct : g_mcts_dense_pct;
    const bool sup_pass = sup.n > 0 && dense_pct < 100;
    if (sup_pass) {
        int hitrows = 0;
        for (int s0 = 0; s0 < sup.n; s0 += blockDim.x) {
            const int si = s0 + static_cast<int>(threadIdx.x);
            bool live = false;
            if (si < sup.n) {
                const unsigned e = sup.svc[si];
                const int sa = static_cast<int>(e & 0xFFu), sb2 = static_cast<int>(e >> 8);
                if (mask)
                    live = ((mask[sa >> 6] >> (sa & 63)) & 1ull) ||
                           (sb2 != 0xFF && ((mask[sb2 >> 6] >> (sb2 & 63)) & 1ull));
                else
                    live = comp[sa] < 1.0 || (sb2 != 0xFF && comp[sb2] < 1.0);
            }
            const unsigned bm = __ballot_sync(0xffffffffu, live);
            int at = 0;
            if (lane == 0 && bm) at = atomicAdd(&tp_nact, __popc(bm));
            at = __shfl_sync(0xffffffffu, at, 0) + __popc(bm & lanemask_lt());
            if (live) {
                sup.act[at] = si;
                hitrows += sup.begin[si + 1] - sup.begin[si];
            }
        }
        for (int off = 16; off > 0; off >>= 1) hitrows += __shfl_xor_sync(0xffffffffu, hitrows, off);
        if (lane == 0 && hitrows) atomicAdd(&tp_actrows, hitrows);
    }
    __syncthreads();
    // few live rows: a warp per live support; most rows live: the dense 8-rows-per-iteration scan
    const bool bysup = sup_pass && 100ll * tp_actrows <= static_cast<long long>(dense_pct) * nb;
    const int nact = bysup ? tp_nact : 0;
    mark(0);
    const uint4* base4 = reinterpret_cast<const uint4*>(base);  // 4 rows per 16 bytes
    const long long nq = nb >> 2;
    const long long B = blockDim.x;
    // the thread's two largest bounds with their rows, and its third largest bound: a thread
    // whose third bound is below the threshold has at most these two candidate rows
    float umax = 0.0f, u2 = 0.0f, u3 = 0.0f;
    unsigned x1 = 0u, x2 = 0u;
    int p1 = -1, p2 = -1;
    int hits = 0;
    auto insert = [&](float u, unsigned x, int pos) {
        if (u > u3) {
            if (u > u2) {
                u3 = u2;
                if (u > umax) {
                    u2 = umax, x2 = x1, p2 = p1;
                    umax = u, x1 = x, p1 = pos;
                } else {
                    u2 = u, x2 = x, p2 = pos;
                }
            } else {
                u3 = u;
            }
        }
    };
    const bool dmask = mask && !bysup;
    // 8 rows: bounds (0 off the mask), and the insertion only when one beats the third bound
    auto bound8 = [&](const unsigned (&x)[8], int r0, int r1) {
        float ub[8];
        float mx = 0.0f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            ub[j] = ub_pair(Wf, x[j]);
            if (dmask) {
                const bool h = hit_pair(hitc, x[j]);
                hits += h;
                if (!h) ub[j] = 0.0f;
            }
            mx = fmaxf(mx, ub[j]);
        }
        if (mx > u3) {
#pragma unroll
            for (int j = 0; j < 8; ++j) insert(ub[j], x[j], j < 4 ? r0 + j : r1 + j - 4);
        }
    };
    const unsigned sp = sent | (sent << 16);
    if (bysup) {  // a warp per active support, lanes over its rows (two rounds per load batch)
        for (int i = wid; i < nact; i += nwarps) {
            const int si = sup.act[i];
            const int b = sup.begin[si], e = sup.begin[si + 1];
            for (int r0 = b; r0 < e; r0 += 64) {
                const int ra = r0 + lane, rb = ra + 32;
                const unsigned xa = ra < e ? base[ra] : sp, xb = rb < e ? base[rb] : sp;
                const float ua = ub_pair(Wf, xa), ubb = ub_pair(Wf, xb);
                if (fmaxf(ua, ubb) > u3) {
                    insert(ua, xa, static_cast<int>(pos0) + ra);
                    insert(ubb, xb, static_cast<int>(pos0) + rb);
                }
            }
        }
        if (mask && threadIdx.x == 0) tp_nhit = tp_actrows;  // every row of a live support touches the mask
    } else {
        long long p = threadIdx.x;
        for (; p + B < nq; p += 2 * B) {
            const uint4 v0 = base4[p], v1 = base4[p + B];
            const unsigned x[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
            bound8(x, static_cast<int>(pos0 + 4 * p), static_cast<int>(pos0 + 4 * (p + B)));
        }
        for (; p < nq; p += B) {
            const uint4 v = base4[p];
            const unsigned x[8] = {v.x, v.y, v.z, v.w, sp, sp, sp, sp};
            bound8(x, static_cast<int>(pos0 + 4 * p), 0);
        }
        if (threadIdx.x < (nb & 3)) {
            const unsigned x[8] = {base[4 * nq + threadIdx.x], sp, sp, sp, sp, sp, sp, sp};
            bound8(x, static_cast<int>(pos0 + 4 * nq + threadIdx.x), 0);
        }
        if (dmask) {
            for (int off = 16; off > 0; off >>= 1) hits += __shfl_xor_sync(0xffffffffu, hits, off);
            if (lane == 0 && hits) atomicAdd(&tp_nhit, hits);
        }
    }
#ifdef MGB_MCTS_SKEW
    if (tm && lane == 0) {
        const long long d = clock64() - tp_c0;
        atomicMax(reinterpret_cast<unsigned long long*>(&tp_dmax), static_cast<unsigned long long>(d));
        atomicMin(reinterpret_cast<unsigned long long*>(&tp_dmin), static_cast<unsigned long long>(d));
        atomicAdd(reinterpret_cast<unsigned long long*>(&tp_dsum), static_cast<unsigned long long>(d));
    }
#endif
    mark(7);
    // the listed rows' config-order key ranks, in flight while the threshold is found
    const unsigned kr1 = p1 >= 0 ? __ldg(keyrank + p1) : 0u, kr2 = p2 >= 0 ? __ldg(keyrank + p2) : 0u;
    // U_K: the K-th largest of the warps' four largest lane maxima (bounds are >= 0, so their
    // bits order like the values).  These are bounds of distinct rows, so K rows have a bound
    // >= U_K; with four per warp it is within a few ranks of the K-th largest lane maximum.
    __shared__ unsigned wtop[kMWarps * 4];
    {
        unsigned mine = __float_as_uint(umax);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const unsigned m = __reduce_max_sync(0xffffffffu, mine);
            const unsigned eq = __ballot_sync(0xffffffffu, mine == m);
            if (lane == 0) wtop[wid * 4 + r] = m;
            if (lane == __ffs(eq) - 1) mine = 0u;
        }
    }
    __syncthreads();
    unsigned tk_bits = 0u;
    {  // every warp: K rounds of max-and-remove over the nwarps * 4 values (no second barrier)
        const int nv = nwarps * 4;
        unsigned v0 = lane < nv ? wtop[lane] : 0u, v1 = lane + 32 < nv ? wtop[lane + 32] : 0u;
#ifndef MGB_TK_ROUNDS  // MGB_TK_ROUNDS: the K max-and-remove rounds (A/B)
        // the 64 values sorted descending by a warp bitonic network (element lane in v0, lane + 32
        // in v1; 21 compare-exchange stages instead of K dependent max-and-remove rounds); the K-th
        // largest (with multiplicity, as the rounds give it) is then element K - 1 (K <= 32)
#pragma unroll
        for (int size = 2; size <= 64; size <<= 1) {
#pragma unroll
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                if (stride == 32) {
                    const unsigned hi = max(v0, v1), lo = min(v0, v1);
                    v0 = hi, v1 = lo;
                } else {
                    const unsigned o0 = __shfl_xor_sync(0xffffffffu, v0, stride);
                    const unsigned o1 = __shfl_xor_sync(0xffffffffu, v1, stride);
                    const bool lower = (lane & stride) == 0;
                    const bool desc0 = (lane & size) == 0, desc1 = ((lane + 32) & size) == 0;
                    v0 = lower == desc0 ? max(v0, o0) : min(v0, o0);
                    v1 = lower == desc1 ? max(v1, o1) : min(v1, o1);
                }
            }
        }
        const unsigned kv = __shfl_sync(0xffffffffu, k <= 32 ? v0 : v1, (k - 1) & 31);
        tk_bits = k > 0 ? kv : 0u;
#else
        for (int r = 0; r < k; ++r) {
            const unsigned m = __reduce_max_sync(0xffffffffu, max(v0, v1));
            tk_bits = m;
            const unsigned e0 = __ballot_sync(0xffffffffu, v0 == m);
            if (e0) {
                if (lane == __ffs(e0) - 1) v0 = 0u;
            } else {
                const unsigned e1 = __ballot_sync(0xffffffffu, v1 == m);
                if (lane == __ffs(e1) - 1) v1 = 0u;
            }
        }
#endif
    }
    mark(1);
    const double LB = __dmul_rd(static_cast<double>(__uint_as_float(tk_bits)), 1.0 - 0x1p-20);
    const float LB_f = __double2float_rd(LB);
    // one compaction per up to 8 rows: the lane's taken rows, a warp scan, one atomic per warp;
    // each candidate's config-order key rank is fetched here (its latency overlaps the scan)
    auto emit = [&](const unsigned (&x)[8], const double (&sc)[8], const long long (&pk)[8], unsigned tk) {
        const int cnt = __popc(tk);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        if (total == 0) return;
        int at = 0;
        if (lane == 31) at = atomicAdd(&tp_ncand, total);
        at = __shfl_sync(0xffffffffu, at, 31) + incl - cnt;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if ((tk >> j) & 1u) {
                if (at < kMCandCap) {
                    const uint64_t row = x[j] | hiS;
                    cand[at] = Cand{sc[j], row_usum(U, row), row, pk[j]};
                }
                ++at;
            }
        }
    };
    const uint4 padv = make_uint4(sp, sp, sp, sp);
    // lanes with a third bound reaching LB rescan all their rows; the others offer their two
    // listed rows (exact scores only where a bound reaches LB)
    const bool rescan = u3 > 0.0f && u3 >= LB_f;
    {
        const unsigned xs[8] = {x1, x2, sp, sp, sp, sp, sp, sp};
        double sc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const long long ps[8] = {p1 | static_cast<long long>(kr1) << 32, p2 | static_cast<long long>(kr2) << 32, 0, 0, 0, 0, 0, 0};
        unsigned tk = 0;
        if (!rescan) {
            if (umax > 0.0f && umax >= LB_f) {
                sc[0] = __dadd_rn(W[x1 & 0xFFFFu], W[x1 >> 16]);
                if (sc[0] > 0.0 && sc[0] >= LB) tk |= 1u;
            }
            if (u2 > 0.0f && u2 >= LB_f) {
                sc[1] = __dadd_rn(W[x2 & 0xFFFFu], W[x2 >> 16]);
                if (sc[1] > 0.0 && sc[1] >= LB) tk |= 2u;
            }
        }
        if (__any_sync(0xffffffffu, tk != 0)) emit(xs, sc, ps, tk);
    }
    auto exact8 = [&](const unsigned (&x)[8], const int (&pos)[8], bool masked) {  // rescans: key ranks loaded here
        float ub[8];
        float mx = 0.0f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            ub[j] = ub_pair(Wf, x[j]);
            if (masked && !hit_pair(hitc, x[j])) ub[j] = 0.0f;
            mx = fmaxf(mx, ub[j]);
        }
        if (!__any_sync(0xffffffffu, mx > 0.0f && mx >= LB_f)) return;
        double sc[8];
        unsigned tk = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            sc[j] = 0.0;
            if (ub[j] > 0.0f && ub[j] >= LB_f) {
                sc[j] = __dadd_rn(W[x[j] & 0xFFFFu], W[x[j] >> 16]);
                if (sc[j] > 0.0 && sc[j] >= LB) tk |= 1u << j;
            }
        }
        long long pk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) pk[j] = (tk >> j) & 1u ? pack_pos(keyrank, pos[j]) : 0ll;
        emit(x, sc, pk, tk);
    };
    if (bysup && __any_sync(0xffffffffu, rescan)) {  // the same rows as pass 1, two per lane per call
        for (int i = wid; i < nact; i += nwarps) {
            const int si = sup.act[i];
            const int b = sup.begin[si], e = sup.begin[si + 1];
            for (int r0 = b; r0 < e; r0 += 64) {
                const int ra = r0 + lane, rb = ra + 32;
                const unsigned x[8] = {rescan && ra < e ? base[ra] : sp, rescan && rb < e ? base[rb] : sp, sp, sp, sp, sp, sp, sp};
                const int ps[8] = {static_cast<int>(pos0) + ra, static_cast<int>(pos0) + rb, 0, 0, 0, 0, 0, 0};
                exact8(x, ps, false);
            }
        }
    } else if (!bysup && __any_sync(0xffffffffu, rescan)) {
        const long long nq2 = (nq + 2 * B - 1) / (2 * B) * (2 * B);
        for (long long p0 = threadIdx.x; p0 < nq2; p0 += 2 * B) {
            const uint4 v0 = rescan && p0 < nq ? base4[p0] : padv;
            const uint4 v1 = rescan && p0 + B < nq ? base4[p0 + B] : padv;
            const unsigned x[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
            const int r0 = static_cast<int>(pos0 + 4 * p0), r1 = static_cast<int>(pos0 + 4 * (p0 + B));
            const int ps[8] = {r0, r0 + 1, r0 + 2, r0 + 3, r1, r1 + 1, r1 + 2, r1 + 3};
            exact8(x, ps, mask != nullptr);
        }
        if (nb & 3) {  // the last rows, warp 0 (the scan needs the whole warp)
            if (wid == 0) {
                const int t = static_cast<int>(threadIdx.x);
                const unsigned x[8] = {rescan && t < (nb & 3) ? base[4 * nq + t] : sp, sp, sp, sp, sp, sp, sp, sp};
                const int ps[8] = {static_cast<int>(pos0 + 4 * nq) + t, 0, 0, 0, 0, 0, 0, 0};
                exact8(x, ps, mask != nullptr);
            }
        }
    }
    __syncthreads();
    mark(2);
    const int nc = tp_ncand;
    int got;
    if (nc <= kMCandCap) {
        got = min(nc, k);
        rank_select_kr(cand, nc, k, win);
    } else {  // pathological ties: exact k rounds of "best row strictly after the previous"
        if (threadIdx.x == 0) atomicAdd(&g_mcts_fallbacks, 1u);
        got = 0;
        Cand last{0.0, 0.0, kNoRow, -1};
        for (int r = 0; r < k; ++r) {
            Cand b{0.0, 0.0, kNoRow, -1};
            for (long long i = threadIdx.x; i < nb; i += blockDim.x) {
                const unsigned x = base[i];
                if (mask && !hit_pair(hitc, x)) continue;
                const double sc = __dadd_rn(W[x & 0xFFFFu], W[x >> 16]);
                if (!(sc > 0.0)) continue;
                const uint64_t row = x | hiS;
                const Cand c{sc, row_usum(U, row), row, pack_pos(keyrank, pos0 + i)};
                if (r > 0 && !precedes_kr(last, c)) continue;
                if (b.row == kNoRow || precedes_kr(c, b)) b = c;
            }
            for (int off = 16; off > 0; off >>= 1) {
                const Cand o{__shfl_xor_sync(0xffffffffu, b.s, off), __shfl_xor_sync(0xffffffffu, b.u, off),
                             __shfl_xor_sync(0xffffffffu, b.row, off), __shfl_xor_sync(0xffffffffu, b.pos, off)};
                if (o.row != kNoRow && (b.row == kNoRow || precedes_kr(o, b))) b = o;
            }
            if (lane == 0) red[wid] = b;
            __syncthreads();
            Cand x = red[0];
            for (int w = 1; w < kMWarps; ++w)
                if (red[w].row != kNoRow && (x.row == kNoRow || precedes_kr(red[w], x))) x = red[w];
            __syncthreads();
            if (x.row == kNoRow) break;
            if (threadIdx.x == 0) win[r] = x;
            last = x;
            ++got;
        }
    }
    __syncthreads();
    if (out && threadIdx.x < got) out[threadIdx.x] = pos_of(win[threadIdx.x]);
    if (threadIdx.x == 0) {
        *scored = mask ? tp_nhit : static_cast<int>(nb);
        tp_ncand = tp_nhit = tp_nact = tp_actrows = 0;  // the next call's counters
    }
    __syncthreads();
    mark(3);
    if (tm && threadIdx.x == 0) {
        atomicAdd(&g_tk[4], static_cast<unsigned long long>(nc));
        atomicAdd(&g_tk[5], 1ull);
#ifdef MGB_MCTS_SKEW
        atomicAdd(&g_tk[8], static_cast<unsigned long long>(tp_dmax));
        atomicAdd(&g_tk[9], static_cast<unsigned long long>(tp_dsum / nwarps));
        atomicAdd(&g_tk[10], static_cast<unsigned long long>(tp_dmin));
#endif
        atomicAdd(&g_tk[11], static_cast<unsigned long long>(bysup));
    }
    return got;
}

}  // namespace
}  // namespace mgb
