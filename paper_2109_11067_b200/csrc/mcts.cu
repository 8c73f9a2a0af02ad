// mcts.cu — K7: device-resident parity-mode mcts_solve (mcts.hpp:148-252).
//
// One CTA runs one whole search: UCB1 selection (strict >, first unvisited child), expansion
// (partial Fisher-Yates over the unsatisfied services, top-K of the base rows touching a
// sampled service), the random child, the memoized rollout (RolloutCache keyed by the
// unsatisfied bitmap, top-K of the whole base pool on a miss), backpropagation, and the final
// visit-count descent — with the reference's std::mt19937_64 stream reproduced on the device
// (thread 0), so under a matched seed the tree, every trace line and the answer are the
// reference's.  The host runs the two fast_algo calls around it (fast_ref before, the
// descent completion after) on the greedy kernel, and replays the trace.
// Every top-K is one block-wide pass: FP32 round-up bounds (Wf) filter the rows, exact FP64
// scores only where a bound reaches the thread's running best, threshold from the per-warp
// K-th best exact maxima, parallel rank of the survivors (common.cuh).
// log(visits) comes from a host table (std::log), so the UCB arithmetic is bit-exact; the
// divisions, sqrt and adds are correctly rounded on both sides (no FMA).
#include <cooperative_groups.h>

#include "common.cuh"
#include "topk_pair.cuh"

namespace cg = cooperative_groups;

namespace mgb {

using namespace dev;

namespace {


constexpr int kMaxServicesDev = 256;  // >= kMaxServices (model.hpp)
constexpr unsigned char kExpanded = 1, kLeaf = 2;
constexpr int kL1Empty = -2, kL1Pending = -3;
constexpr int kLogSmem = 256;  // log(visits) entries kept on chip (selection reads one per level)

struct Mt64 {  // std::mt19937_64 (w 64, n 312, m 156, r 31)
    uint64_t mt[312];
    uint64_t out[312];  // the current block's outputs, tempered when the block is twisted
    int idx;
};

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    return y ^ (y >> 43);
}

__device__ void mt_seed(Mt64& g, uint64_t s) {
    g.mt[0] = s;
    for (int i = 1; i < 312; ++i) g.mt[i] = 6364136223846793005ull * (g.mt[i - 1] ^ (g.mt[i - 1] >> 62)) + static_cast<uint64_t>(i);
    g.idx = 312;
}

__device__ uint64_t mt_next(Mt64& g) {
    if (g.idx >= 312) {  // serial twist (the rollout walk twists warp-parallel ahead of time)
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (g.mt[i] & 0xFFFFFFFF80000000ull) | (g.mt[(i + 1) % 312] & 0x7FFFFFFFull);
            uint64_t xa = x >> 1;
            if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
            g.mt[i] = g.mt[(i + 156) % 312] ^ xa;
        }
        for (int i = 0; i < 312; ++i) g.out[i] = mt_temper(g.mt[i]);
        g.idx = 0;
    }
    return g.out[g.idx++];
}

// pick_index (util.hpp:39-47) constants for n <= kPickTab: the rejection limit
// UINT64_MAX - UINT64_MAX % n, 2^32 mod n and Lemire's fastmod multiplier ceil(2^64 / n), so
// r % n = ((r >> 32) % n * (2^32 % n) + (r & 0xffffffff) % n) % n costs three multiplies.
constexpr int kPickTab = 256;
struct PickTab {
    uint64_t lim[kPickTab + 1];
    uint64_t fm[kPickTab + 1];
    unsigned p32[kPickTab + 1];
};
__device__ void pick_tab_init(PickTab& t) {
    for (int m = threadIdx.x; m <= kPickTab; m += blockDim.x) {
        if (m < 2) {
            t.lim[m] = ~0ull;
            t.fm[m] = 0;
            t.p32[m] = 0;
            continue;
        }
        const unsigned mu = static_cast<unsigned>(m);
        const unsigned p32 = static_cast<unsigned>((1ull << 32) % mu);
        const unsigned rmax = ((0xFFFFFFFFu % mu) * p32 + 0xFFFFFFFFu % mu) % mu;  // UINT64_MAX mod m
        t.lim[m] = ~0ull - rmax;
        t.fm[m] = ~0ull / mu + 1;
        t.p32[m] = p32;
    }
}
__device__ __forceinline__ unsigned fastmod32(unsigned x, uint64_t fm, unsigned d) {
    return static_cast<unsigned>(__umul64hi(fm * x, d));
}

__device__ uint64_t mt_pick(Mt64& g, uint64_t n, const PickTab* t = nullptr) {  // pick_index, util.hpp:39-47
    if (n <= 1) return 0;
    if (t && n <= static_cast<uint64_t>(kPickTab)) {
        const unsigned m = static_cast<unsigned>(n);
        const uint64_t limit = t->lim[m], fm = t->fm[m];
        uint64_t r;
        do {
            r = mt_next(g);
        } while (r >= limit);
        const unsigned a = fastmod32(static_cast<unsigned>(r >> 32), fm, m), b = fastmod32(static_cast<unsigned>(r), fm, m);
        return fastmod32(a * t->p32[m] + b, fm, m);
    }
    if (n < (1ull << 16)) {  // the same arithmetic with 32-bit remainders (the search's n are small)
        const unsigned m = static_cast<unsigned>(n);
        const unsigned p32 = static_cast<unsigned>((1ull << 32) % m);            // 2^32 mod m
        const unsigned rmax = ((0xFFFFFFFFu % m) * p32 + 0xFFFFFFFFu % m) % m;  // UINT64_MAX mod m
        const uint64_t limit = ~0ull - rmax;
        uint64_t r;
        do {
            r = mt_next(g);
        } while (r >= limit);
        const unsigned hi = static_cast<unsigned>(r >> 32), lo = static_cast<unsigned>(r);
        return ((hi % m) * p32 + lo % m) % m;
    }
    const uint64_t limit = ~0ull - (~0ull % n);
    uint64_t r;
    do {
        r = mt_next(g);
    } while (r >= limit);
    return r % n;
}

// The mt19937_64 twist of all 312 words by one warp (a generator that is exhausted, idx = 312):
// the first 156 words read only old words, the rest read the first half's new words and, for
// the last one, the new word 0 — the sequential loop's dependences, two read-then-write phases.
__device__ void mt_twist_warp(Mt64& g) {
    const int lane = static_cast<int>(threadIdx.x & 31u);
    auto f = [&](int i) {
        const uint64_t x = (g.mt[i] & 0xFFFFFFFF80000000ull) | (g.mt[(i + 1) % 312] & 0x7FFFFFFFull);
        uint64_t xa = x >> 1;
        if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
        return g.mt[(i + 156) % 312] ^ xa;
    };
    uint64_t v[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = lane + 32 * k;
        if (i < 156) v[k] = f(i);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = lane + 32 * k;
        if (i < 156) g.mt[i] = v[k];
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = 156 + lane + 32 * k;
        if (i < 312) v[k] = f(i);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = 156 + lane + 32 * k;
        if (i < 312) g.mt[i] = v[k];
    }
    __syncwarp();
    for (int i = lane; i < 312; i += 32) g.out[i] = mt_temper(g.mt[i]);
    if (lane == 0) g.idx = 0;
    __syncwarp();
}

// row touches a masked service: per-code flags built with the W table (4 byte lookups)
__device__ __forceinline__ bool row_hits(const unsigned char* hitc, uint64_t row) {
    return (hitc[row & 0xFFFFull] | hitc[(row >> 16) & 0xFFFFull] | hitc[(row >> 32) & 0xFFFFull] |
            hitc[row >> 48]) != 0;
}

__device__ __forceinline__ float ub_row(const float* Wf, uint64_t row) {
    float s = __fadd_ru(Wf[row & 0xFFFFull], Wf[(row >> 16) & 0xFFFFull]);
    s = __fadd_ru(s, Wf[(row >> 32) & 0xFFFFull]);
    return __fadd_ru(s, Wf[row >> 48]);
}

// detail::topk_candidates (mcts.hpp:56-76) over the base rows (mask: rows touching a masked
// service, else all), block-wide.  Writes base-pool indices in preference order to out[],
// returns their count.  Ends with a barrier.

__device__ __forceinline__ float ub_half(const float* Wf, unsigned lo, unsigned hi) {
    float s = __fadd_ru(Wf[lo & 0xFFFFu], Wf[lo >> 16]);
    s = __fadd_ru(s, Wf[hi & 0xFFFFu]);
    return __fadd_ru(s, Wf[hi >> 16]);
}
__device__ __forceinline__ bool hit_half(const unsigned char* hitc, unsigned lo, unsigned hi) {
    return (hitc[lo & 0xFFFFu] | hitc[lo >> 16] | hitc[hi & 0xFFFFu] | hitc[hi >> 16]) != 0;
}

// Bitonic sort of the warp's lane values, descending (lane q ends with the q-th largest).
__device__ __forceinline__ float warp_sort_desc_f(float v) {
    const int lane = static_cast<int>(threadIdx.x & 31u);
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int j = size >> 1; j > 0; j >>= 1) {
            const float o = __shfl_xor_sync(0xffffffffu, v, j);
            const bool desc = (lane & size) == 0 || size == 32;
            const bool low = (lane & j) == 0;
            v = (low == desc) ? fmaxf(v, o) : fminf(v, o);
        }
    }
    return v;
}

// warp_kth (common.cuh) on floats: half the shuffles of the double version.
__device__ __forceinline__ float warp_kth_f(float v, int k) {
    const int lane = static_cast<int>(threadIdx.x & 31u);
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int j = size >> 1; j > 0; j >>= 1) {
            const float o = __shfl_xor_sync(0xffffffffu, v, j);
            const bool desc = (lane & size) == 0 || size == 32;
            const bool low = (lane & j) == 0;
            v = (low == desc) ? fmaxf(v, o) : fminf(v, o);
        }
    }
    return __shfl_sync(0xffffffffu, v, k - 1);
}

// The candidates' key ranks (pos | keyrank[pos] << 32), fetched in one parallel round trip
// after compaction instead of one dependent global load per push.
__device__ __forceinline__ void fill_keyrank(const unsigned* keyrank, Cand* cand, int nc) {
    for (int i = threadIdx.x; i < nc; i += blockDim.x) cand[i].pos = pack_pos(keyrank, cand[i].pos);
}

// The same top-K with an FP32-only first pass: every thread's largest bound ub, the K-th
// largest of a warp's lane maxima (max over warps) U_K, then LB = U_K (1 - 2^-20) is a lower
// bound of the K-th exact score: K rows have ub >= U_K, and ub over-estimates an exact score
// by < 4.01 * 2^-23 relative (4 round-up conversions/adds of non-negative terms), so those K
// rows score >= LB.  Pass 2 scores exactly only rows whose bound reaches LB; the candidates
// (exact score >= LB) contain every row of the top-K.
__device__ __noinline__ int block_topk_bound(const DevModel& M, const unsigned* keyrank, const uint64_t* base, long long nb,
                                long long pos0, const double* comp, const uint64_t* mask, int k, const double* U,
                                double* W, float* Wf, unsigned char* hitc, Cand* cand, Cand* win, int* out, int* scored,
                                bool tm) {
    __shared__ unsigned t_fbits;
    __shared__ int n_cand, n_hit;
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
    const int nW = (M.n + 1) * M.PP;
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
    if (threadIdx.x == 0) {
        t_fbits = 0u;
        n_cand = 0;
        n_hit = 0;
    }
    __syncthreads();
    mark(0);
    const uint4* base2 = reinterpret_cast<const uint4*>(base);
    const long long np = nb >> 1;
    const long long B = blockDim.x;
    // pass 1: FP32 bounds only (no exact scores, no divergence)
    float umax = 0.0f;
    int hits = 0;
    long long p = threadIdx.x;
    for (; p + 3 * B < np; p += 4 * B) {
        const uint4 v[4] = {base2[p], base2[p + B], base2[p + 2 * B], base2[p + 3 * B]};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float u0 = ub_half(Wf, v[q].x, v[q].y), u1 = ub_half(Wf, v[q].z, v[q].w);
            if (mask) {
                const bool h0 = hit_half(hitc, v[q].x, v[q].y), h1 = hit_half(hitc, v[q].z, v[q].w);
                hits += h0 + h1;
                if (!h0) u0 = 0.0f;
                if (!h1) u1 = 0.0f;
            }
            umax = fmaxf(umax, fmaxf(u0, u1));
        }
    }
    for (; p < np; p += B) {
        const uint4 v = base2[p];
        float u0 = ub_half(Wf, v.x, v.y), u1 = ub_half(Wf, v.z, v.w);
        if (mask) {
            const bool h0 = hit_half(hitc, v.x, v.y), h1 = hit_half(hitc, v.z, v.w);
            hits += h0 + h1;
            if (!h0) u0 = 0.0f;
            if (!h1) u1 = 0.0f;
        }
        umax = fmaxf(umax, fmaxf(u0, u1));
    }
    if ((nb & 1) && threadIdx.x == 0) {
        const uint64_t r = base[nb - 1];
        const unsigned lo = static_cast<unsigned>(r), hi = static_cast<unsigned>(r >> 32);
        if (!mask || hit_half(hitc, lo, hi)) {
            hits += mask ? 1 : 0;
            umax = fmaxf(umax, ub_half(Wf, lo, hi));
        }
    }
    if (mask) {
        for (int off = 16; off > 0; off >>= 1) hits += __shfl_xor_sync(0xffffffffu, hits, off);
        if ((threadIdx.x & 31u) == 0) atomicAdd(&n_hit, hits);
    }
    const float uk = warp_kth_f(umax, k);
    if ((threadIdx.x & 31u) == 0) atomicMax(&t_fbits, __float_as_uint(uk));  // non-negative floats
    __syncthreads();
    mark(1);
    const double LB = __dmul_rd(static_cast<double>(__uint_as_float(t_fbits)), 1.0 - 0x1p-20);
    const float LB_f = __double2float_rd(LB);
    // pass 2: exact scores where the bound reaches LB; candidates score >= LB (> 0)
    auto visit2 = [&](unsigned lo, unsigned hi, long long pos) {
        bool take = false;
        double sc = 0.0;
        const uint64_t row = (static_cast<uint64_t>(hi) << 32) | lo;
        const float ub = ub_half(Wf, lo, hi);
        if (ub > 0.0f && ub >= LB_f && (!mask || hit_half(hitc, lo, hi))) {
            sc = row_score(W, row);
            take = sc > 0.0 && sc >= LB;
        }
        const unsigned b = __ballot_sync(0xffffffffu, take);
        if (b) {
            int at = 0;
            if ((threadIdx.x & 31u) == 0) at = atomicAdd(&n_cand, __popc(b));
            at = __shfl_sync(0xffffffffu, at, 0) + __popc(b & lanemask_lt());
            if (take && at < kMCandCap) cand[at] = Cand{sc, row_usum(U, row), row, pack_pos(keyrank, pos)};
        }
    };
    const unsigned sent = static_cast<unsigned>(M.n * M.PP) * 0x00010001u;
    const uint4 padv = make_uint4(sent, sent, sent, sent);
    const long long np4 = (np + 4 * B - 1) / (4 * B) * (4 * B);
    for (long long p0 = threadIdx.x; p0 < np4; p0 += 4 * B) {
        uint4 v[4];
        float mx = 0.0f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const long long pp = p0 + q * B;
            v[q] = pp < np ? base2[pp] : padv;
            mx = fmaxf(mx, fmaxf(ub_half(Wf, v[q].x, v[q].y), ub_half(Wf, v[q].z, v[q].w)));
        }
        if (!__any_sync(0xffffffffu, mx > 0.0f && mx >= LB_f)) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const long long pp = p0 + q * B;
            visit2(v[q].x, v[q].y, pos0 + 2 * pp);
            visit2(v[q].z, v[q].w, pos0 + 2 * pp + 1);
        }
    }
    if (nb & 1) {
        if ((threadIdx.x >> 5) == 0) {
            const uint64_t r = threadIdx.x == 0 ? base[nb - 1]
                                                : static_cast<uint64_t>(M.n * M.PP) * 0x0001000100010001ull;
            visit2(static_cast<unsigned>(r), static_cast<unsigned>(r >> 32), pos0 + nb - 1);
        }
    }
    __syncthreads();
    mark(2);
    const int nc = n_cand;
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
                const uint64_t row = base[i];
                if (mask && !row_hits(hitc, row)) continue;
                const double s = row_score(W, row);
                if (!(s > 0.0)) continue;
                const Cand c{s, row_usum(U, row), row, pack_pos(keyrank, pos0 + i)};
                if (r > 0 && !precedes_kr(last, c)) continue;
                if (b.row == kNoRow || precedes_kr(c, b)) b = c;
            }
            for (int off = 16; off > 0; off >>= 1) {
                const Cand o{__shfl_xor_sync(0xffffffffu, b.s, off), __shfl_xor_sync(0xffffffffu, b.u, off),
                             __shfl_xor_sync(0xffffffffu, b.row, off), __shfl_xor_sync(0xffffffffu, b.pos, off)};
                if (o.row != kNoRow && (b.row == kNoRow || precedes_kr(o, b))) b = o;
            }
            if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = b;
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
    if (threadIdx.x == 0) *scored = mask ? n_hit : static_cast<int>(nb);
    __syncthreads();
    mark(3);
    if (tm && threadIdx.x == 0) {
        atomicAdd(&g_tk[4], static_cast<unsigned long long>(nc));
        atomicAdd(&g_tk[5], 1ull);
    }
    return got;
}

__device__ __forceinline__ bool comp_satisfied(const double* c, int n) {  // core.hpp:217-221
    for (int i = 0; i < n; ++i)
        if (c[i] < 1.0 - 1e-9) return false;
    return true;
}

__device__ __forceinline__ void add_row_util(const DevModel& M, const double* U, uint64_t row, double* c) {
    for (int j = 0; j < 4; ++j) {  // rollout / expand add (mcts.hpp:112,139)
        const int code = static_cast<int>((row >> (16 * j)) & 0xFFFFull);
        const int svc = svc_of(M, static_cast<unsigned>(code));
        if (svc < M.n) c[svc] = __dadd_rn(c[svc], U[code]);
    }
}

}  // namespace

// NK: 64-bit words of the rollout-cache key (the unsatisfied bitmap): 1 for n <= 64, else 4 —
// the walk keeps the key in registers, so the narrow variant frees 12 of them.
template <int NK>
__global__ void __launch_bounds__(kMThreads, 1) mcts_kernel(const __grid_constant__ MctsLaunch L) {
    extern __shared__ __align__(16) unsigned char smem[];
    // One search per thread-block CLUSTER: rank 0 runs the search; every rank scans its slice
    // of the base pool for each top-K and rank 0 merges the slices' winners over DSMEM.
    cg::cluster_group cl = cg::this_cluster();
    const int C = static_cast<int>(cl.num_blocks());
    const int rank = static_cast<int>(cl.block_rank());
    const MctsSolveArgs& a = L.s[blockIdx.x / C];
    const DevModel& M = L.M;
    const int n = M.n, K = L.topk;
    const int nW = (n + 1) * M.PP;
    // a multiple of 2 rows (4 with 32-bit pair rows): 16-byte vectors stay aligned
    const long long chunk = L.pair ? (((L.n_base + C - 1) / C + 3) & ~3ll) : (((L.n_base + C - 1) / C + 1) & ~1ll);
    const long long lo = min(L.n_base, static_cast<long long>(rank) * chunk);
    const long long hi = min(L.n_base, lo + chunk);
    // dynamic shared memory: tables (same offsets in every rank: peers read `cur`, `win` and
    // the request over DSMEM), then rank 0's node metadata, then this rank's slice of the pool
    size_t off = 0;
    auto carve = [&](size_t bytes) {
        unsigned char* p = smem + off;
        off = (off + bytes + 15) & ~size_t{15};
        return p;
    };
    double* W = reinterpret_cast<double*>(carve(sizeof(double) * nW));
    double* Us = reinterpret_cast<double*>(carve(sizeof(double) * nW));
    double* cur = reinterpret_cast<double*>(carve(sizeof(double) * (n + 1)));
    Cand* cand = reinterpret_cast<Cand*>(carve(sizeof(Cand) * kMCandCap));
    Cand* win = reinterpret_cast<Cand*>(carve(sizeof(Cand) * 2 * kMMaxK));  // [0,K) local, [K,2K) merged
    float* Wf = reinterpret_cast<float*>(carve(sizeof(float) * nW));
    unsigned char* hitc = carve(nW);
    unsigned char* csvc = carve(nW);
    const int MN = a.max_nodes;
    double* nval = a.node_value;
    int *nvis = a.node_visits, *nfirst = a.node_first, *nnch = a.node_nch, *ncand = a.node_cand;
    unsigned char* nflags = a.node_flags;
    if (L.node_smem) {  // selection walks these every iteration: keep them on chip
        nval = reinterpret_cast<double*>(carve(sizeof(double) * MN));
        nvis = reinterpret_cast<int*>(carve(sizeof(int) * MN));
        nfirst = reinterpret_cast<int*>(carve(sizeof(int) * MN));
        nnch = reinterpret_cast<int*>(carve(sizeof(int) * MN));
        ncand = reinterpret_cast<int*>(carve(sizeof(int) * MN));
        nflags = carve(MN);
    }
    const uint64_t* rows = L.base;  // whole pool (rank 0's adds); slice for the top-K scans
    const uint64_t* slice = L.base + lo;
    const unsigned* slice32 = nullptr;  // pair rows: low halves only (L.pair)
    // pair top-K over 32-bit rows: on chip when they fit, else from global memory (L.base32)
    const bool pair = L.pair && (L.rows_smem || (L.base32 && C == 1));
    if (pair && !L.rows_smem) {
        slice32 = L.base32 + lo;
    } else if (pair) {
        unsigned* r = reinterpret_cast<unsigned*>(carve(sizeof(unsigned) * chunk));
        for (long long i = threadIdx.x; i < hi - lo; i += blockDim.x) r[i] = static_cast<unsigned>(__ldg(L.base + lo + i));
        slice32 = r;
    } else if (L.rows_smem) {
        uint64_t* r = reinterpret_cast<uint64_t*>(carve(sizeof(uint64_t) * chunk));
        for (long long i = threadIdx.x; i < hi - lo; i += blockDim.x) r[i] = __ldg(L.base + lo + i);
        slice = r;
    }
    const unsigned sent16 = static_cast<unsigned>(n * M.PP);
    const uint64_t hiS = static_cast<uint64_t>(sent16 | (sent16 << 16)) << 32;
    int* sbeg = nullptr;
    unsigned short* ssvc = nullptr;
    int* sact = nullptr;
    const int nsup = L.n_sup;
    if (nsup) {  // supports of the base pool (C == 1: the slice is the whole pool)
        sbeg = reinterpret_cast<int*>(carve(sizeof(int) * (nsup + 1)));
        ssvc = reinterpret_cast<unsigned short*>(carve(sizeof(unsigned short) * nsup));
        sact = reinterpret_cast<int*>(carve(sizeof(int) * nsup));
        for (int i = threadIdx.x; i <= nsup; i += blockDim.x) sbeg[i] = L.sup_begin[i];
        for (int i = threadIdx.x; i < nsup; i += blockDim.x) ssvc[i] = L.sup_svc[i];
    }
    // rows in global memory (L2 latency): scanning only the live supports always pays (A/B gen48:
    // 121 vs 141 ms per 200-iteration search); rows on chip: the dense scan above 60% live rows
    const SupTab sup{nsup, sbeg, ssvc, sact, pair && !L.rows_smem ? 100 : -1};
    for (int e = threadIdx.x; e < nW; e += blockDim.x) {
        Us[e] = __ldg(&M.U[e]);
        csvc[e] = static_cast<unsigned char>(svc_of(M, static_cast<unsigned>(e)));  // service of a code (n for the sentinel row)
    }
    __shared__ int s_exit, s_usemask, n_got, s_hits;
    __shared__ uint64_t s_mask[4];
    if (threadIdx.x == 0) {
        s_exit = 0;
        s_usemask = 0;
    }
    topk_pair_counters_init();
    __syncthreads();
    if (rank != 0) {  // helper: serve rank 0's top-K requests until it posts exit
        for (;;) {
            cl.sync();  // request posted
            if (*cl.map_shared_rank(&s_exit, 0)) {
                cl.sync();  // rank 0 stays resident until every helper has read the flag
                break;
            }
            const double* rc = cl.map_shared_rank(cur, 0);
            for (int i = threadIdx.x; i < n; i += blockDim.x) cur[i] = rc[i];
            if (threadIdx.x < 4) s_mask[threadIdx.x] = cl.map_shared_rank(s_mask, 0)[threadIdx.x];
            if (threadIdx.x == 0) s_usemask = *cl.map_shared_rank(&s_usemask, 0);
            __syncthreads();
            int sc = 0;
            const int got = pair ? block_topk_pair(M, L.keyrank, slice32, hi - lo, lo, cur, s_usemask ? s_mask : nullptr, K, Us, W, Wf,
                                                   hitc, cand, win, nullptr, &sc, L.timers != 0, SupTab{})
                                 : block_topk_bound(M, L.keyrank, slice, hi - lo, lo, cur, s_usemask ? s_mask : nullptr, K, Us, W, Wf,
                                             hitc, cand, win, nullptr, &sc, L.timers != 0);
            if (threadIdx.x == 0) {
                n_got = got;
                s_hits = sc;
            }
            cl.sync();  // winners published
        }
        return;
    }
    // rank 0: the top-K of the whole pool under `cur` (mask: rows touching a sampled service)
    auto cluster_topk = [&](bool usemask, int* out, int* scored) -> int {
        if (C == 1) {  // one CTA: its own top-K is the answer (no merge, no cluster barriers)
            __syncthreads();
            return pair ? block_topk_pair(M, L.keyrank, slice32, hi - lo, lo, cur, usemask ? s_mask : nullptr, K, Us, W,
                                          Wf, hitc, cand, win, out, scored, L.timers != 0, sup)
                        : block_topk_bound(M, L.keyrank, slice, hi - lo, lo, cur, usemask ? s_mask : nullptr, K, Us,
                                        W, Wf, hitc, cand, win, out, scored, L.timers != 0);
        }
        if (threadIdx.x == 0) s_usemask = usemask ? 1 : 0;
        __syncthreads();
        cl.sync();
        int sc = 0;
        const int got0 = pair ? block_topk_pair(M, L.keyrank, slice32, hi - lo, lo, cur, usemask ? s_mask : nullptr, K, Us, W, Wf,
                                                hitc, cand, win, nullptr, &sc, L.timers != 0, SupTab{})
                               : block_topk_bound(M, L.keyrank, slice, hi - lo, lo, cur, usemask ? s_mask : nullptr, K, Us, W, Wf, hitc,
                                          cand, win, nullptr, &sc, L.timers != 0);
        if (threadIdx.x == 0) {
            n_got = got0;
            s_hits = sc;
        }
        cl.sync();
        __shared__ unsigned long long m_bits;
        __shared__ int m_n, m_scored;
        if (threadIdx.x == 0) {
            m_bits = 0ull;
            m_n = 0;
            m_scored = 0;
        }
        __syncthreads();
        for (int r = threadIdx.x; r < C; r += blockDim.x) {  // merge threshold: full lists' K-th scores
            const int g = *cl.map_shared_rank(&n_got, r);
            atomicAdd(&m_scored, *cl.map_shared_rank(&s_hits, r));
            if (g == K) atomicMax(&m_bits, static_cast<unsigned long long>(__double_as_longlong(cl.map_shared_rank(win, r)[K - 1].s)));
        }
        __syncthreads();
        const double TM = __longlong_as_double(static_cast<long long>(m_bits));
        for (int i = threadIdx.x; i < C * K; i += blockDim.x) {
            const int r = i / K, q = i % K;
            if (q >= *cl.map_shared_rank(&n_got, r)) continue;
            const Cand c = cl.map_shared_rank(win, r)[q];
            if (c.s < TM) continue;
            cand[atomicAdd(&m_n, 1)] = c;  // <= C * K <= kMCandCap
        }
        __syncthreads();
        const int mc = m_n;
        rank_select_kr(cand, mc, K, win + kMMaxK);
        __syncthreads();
        const int got = min(mc, K);
        if (threadIdx.x < got) out[threadIdx.x] = pos_of(win[kMMaxK + threadIdx.x]);
        if (threadIdx.x == 0) *scored = m_scored;
        __syncthreads();
        return got;
    };
    __shared__ Mt64 g;
    __shared__ PickTab s_pick;
    pick_tab_init(s_pick);
    __shared__ double s_log[kLogSmem];
    for (int v = threadIdx.x; v < kLogSmem && v < L.budget + 2; v += blockDim.x) s_log[v] = L.logtab[v];
    __shared__ int s_node, s_leaf, s_expand, s_take, s_nch, s_done, s_est, s_miss, s_slot, s_abort, s_steps;
    __shared__ int s_edges, s_path, s_best, s_have, s_nodes, s_builds, s_iters, s_scored, s_expands;
    __shared__ long long s_expand_rows, s_wcyc;  // s_wcyc, s_wsteps: walk cycles and steps (timers)
    __shared__ int s_wsteps, s_wprobes, s_wentries;
    __shared__ long long s_wpcyc;
    __shared__ int s_out[kMMaxK];
    __shared__ int s_unsat[kMaxServicesDev];  // expand: the node's unsatisfied services
    // on-chip level of the rollout cache (dynamic shared memory, filled to 3/4): per slot the
    // key's nk words, the pool size and the pool as (base index, low 32 row bits)
    __shared__ int l1_used, s_l1new;
    const int l1_slots = rank == 0 ? L.l1_slots : 0, nk = (n + 63) >> 6;
    uint64_t* l1k = reinterpret_cast<uint64_t*>(carve(sizeof(uint64_t) * l1_slots * nk));
    int* l1n = reinterpret_cast<int*>(carve(sizeof(int) * l1_slots));
    uint2* l1p = reinterpret_cast<uint2*>(carve(sizeof(uint2) * l1_slots * K));
    for (int q = threadIdx.x; q < l1_slots; q += blockDim.x) l1n[q] = kL1Empty;
    if (threadIdx.x == 0) l1_used = 0;
    // rows by pool index for the utility adds: the on-chip copy when it holds the whole pool
    const uint64_t* prow = (C == 1 && L.rows_smem && !pair) ? slice : rows;
    const unsigned* prow32 = (C == 1 && pair) ? slice32 : nullptr;
    auto rowat = [&](int idx) -> uint64_t { return prow32 ? (prow32[idx] | hiS) : prow[idx]; };
    const int max_depth = 2 * a.l_ref;
    const int tid = threadIdx.x;
    long long t_sel = 0, t_exp = 0, t_miss = 0, t_roll = 0, t_topk = 0, tc = 0;  // thread-0 clock64 phase split
    const bool timers = L.timers != 0;
    auto tick = [&](long long& acc) {
        if (timers && tid == 0) {
            const long long t = clock64();
            acc += t - tc;
            tc = t;
        }
    };
    if (tid == 0) tc = clock64();

    // root (mcts.hpp:157-160)
    if (tid == 0) {
        mt_seed(g, a.seed);
        s_nodes = 1;
        s_have = 0;
        s_best = 0;
        s_abort = 0;
        s_builds = 0;
        s_iters = 0;
        s_expands = 0;
        s_expand_rows = 0;
        s_wcyc = 0;
        s_wsteps = 0;
        s_wprobes = 0;
        s_wentries = 0;
        s_wpcyc = 0;
        nvis[0] = 0;
        nval[0] = 0.0;
        nnch[0] = 0;
        nfirst[0] = 0;
        ncand[0] = -1;
    }
    for (int i = tid; i < n; i += blockDim.x) a.node_comp[i] = a.comp0[i];  // pinned host staging (mapped)
    for (unsigned i = tid; i <= a.tab_mask; i += blockDim.x) a.tag[i] = 0;    // the global rollout-cache level
    __syncthreads();
    if (tid == 0) nflags[0] = comp_satisfied(a.node_comp, n) ? kLeaf : 0;
    __syncthreads();

    const int lane = tid & 31, warp = tid >> 5;
    for (int iter = 0; iter < L.budget && !s_abort; ++iter) {
        // ---- selection (mcts.hpp:183-191): UCB1, first unvisited child, strict >.  Warp 0, a
        // lane per child: the first unvisited child, else the first maximum.
        if (warp == 0) {
            int node = 0, edges = 0, path = 1;
            if (lane == 0) a.pathnodes[0] = 0;
            while ((nflags[node] & kExpanded) && !(nflags[node] & kLeaf) && nnch[node] > 0) {
                const int nch = nnch[node], f0 = nfirst[node];
                const int nv = max(1, nvis[node]);
                const double log_n = nv < kLogSmem ? s_log[nv] : L.logtab[nv];
                int pick = -1, bq = -1;
                double bv = -1.0;
                for (int q0 = 0; q0 < nch; q0 += 32) {
                    const int q = q0 + lane;
                    double val = -1.0;
                    bool unvisited = false;
                    if (q < nch) {
                        const int v = nvis[f0 + q];
                        unvisited = v == 0;
                        if (!unvisited) {
                            const double dv = static_cast<double>(v);
                            val = __dadd_rn(__ddiv_rn(nval[f0 + q], dv),
                                            __dmul_rn(L.ucb_c, __dsqrt_rn(__ddiv_rn(log_n, dv))));
                        }
                    }
                    const unsigned um = __ballot_sync(0xffffffffu, unvisited);
                    if (um) {
                        pick = q0 + __ffs(um) - 1;
                        break;
                    }
                    int qq = q < nch ? q : 0x7fffffff;
                    for (int off = 16; off > 0; off >>= 1) {
                        const double ov = __shfl_xor_sync(0xffffffffu, val, off);
                        const int oq = __shfl_xor_sync(0xffffffffu, qq, off);
                        if (ov > val || (ov == val && oq < qq)) val = ov, qq = oq;
                    }
                    if (val > bv) bv = val, bq = qq;  // strict: an earlier round wins ties
                }
                if (pick < 0) pick = bq;
                node = f0 + pick;
                if (lane == 0) {
                    a.edges[edges] = ncand[node];
                    a.pathnodes[path] = node;
                }
                ++edges;
                ++path;
            }
            if (lane == 0) {
                s_edges = edges;
                s_path = path;
                s_node = node;
                s_leaf = (nflags[node] & kLeaf) != 0;
                s_expand = !s_leaf && !(nflags[node] & kExpanded);
                s_est = 0;
            }
        }
        __syncthreads();
        tick(t_sel);
        if (s_leaf) {  // mcts.hpp:193-198
            if (tid == 0 && (!s_have || s_edges < s_best)) {
                for (int q = 0; q < s_edges; ++q) a.best_out[q] = a.edges[q];
                s_best = s_edges;
                s_have = 1;
            }
        } else {
            if (s_expand) {  // expand (mcts.hpp:89-116)
                if (warp == 0) {  // the node's completion into `cur`, its unsatisfied services in order
                    // (ballot compaction, on chip), then lane 0's partial Fisher-Yates
                    const double* nc = a.node_comp + static_cast<long long>(s_node) * n;
                    int m = 0;
                    for (int i0 = 0; i0 < n; i0 += 32) {
                        const int i = i0 + lane;
                        const double v = i < n ? nc[i] : 2.0;
                        if (i < n) cur[i] = v;
                        const bool u = i < n && v < 1.0 - 1e-9;
                        const unsigned bm = __ballot_sync(0xffffffffu, u);
                        if (u) s_unsat[m + __popc(bm & lanemask_lt())] = i;
                        m += __popc(bm);
                    }
                    __syncwarp();
                    if (lane == 0) {
                        const int take = min(L.pick_services, m);
                        for (int i = 0; i < take; ++i) {
                            const int j = i + static_cast<int>(mt_pick(g, static_cast<uint64_t>(m - i), &s_pick));
                            const int t = s_unsat[i];
                            s_unsat[i] = s_unsat[j];
                            s_unsat[j] = t;
                        }
                        for (int w = 0; w < 4; ++w) s_mask[w] = 0;
                        for (int i = 0; i < take; ++i) s_mask[s_unsat[i] >> 6] |= 1ull << (s_unsat[i] & 63);
                        s_take = take;
                    }
                }
                __syncthreads();
                tick(t_exp);
                const int got = s_take > 0 ? cluster_topk(true, s_out, &s_scored) : 0;
                tick(t_topk);
                if (tid == 0 && s_take > 0) {
                    ++s_expands;
                    s_expand_rows += s_scored;
                }
                // the children: a warp each (copy, add the config's utility, satisfied flag)
                const int first = s_nodes;
                const bool fits = first + got <= a.max_nodes;
                if (fits) {
                    for (int q = warp; q < got; q += kMWarps) {
                        const int c = first + q;
                        double* cc = a.node_comp + static_cast<long long>(c) * n;
                        const uint64_t row = rowat(s_out[q]);
                        bool uns = false;
                        for (int i = lane; i < n; i += 32) {  // parent + the config's utility (expand, mcts.hpp:109-113)
                            double v = cur[i];
#pragma unroll
                            for (int m = 0; m < 4; ++m) {
                                const int code = static_cast<int>((row >> (16 * m)) & 0xFFFFull);
                                if (csvc[code] == i) v = __dadd_rn(v, Us[code]);
                            }
                            cc[i] = v;
                            uns |= v < 1.0 - 1e-9;
                        }
                        const bool sat = !__any_sync(0xffffffffu, uns);
                        if (lane == 0) {
                            ncand[c] = s_out[q];
                            nvis[c] = 0;
                            nval[c] = 0.0;
                            nnch[c] = 0;
                            nfirst[c] = 0;
                            nflags[c] = sat ? kLeaf : 0;
                        }
                    }
                }
                __syncthreads();
                if (tid == 0) {
                    if (!fits) {
                        s_abort = 3;  // node storage exhausted (host sizes it from the budget)
                    } else {
                        nfirst[s_node] = first;
                        nnch[s_node] = got;
                        nflags[s_node] |= kExpanded;
                        s_nodes += got;
                    }
                }
                __syncthreads();
                tick(t_exp);
                if (s_abort) break;
            }
            // random child (mcts.hpp:202-207)
            __shared__ int s_child_row;
            if (tid == 0) {
                const int nch = nnch[s_node];
                s_child_row = -1;
                if (nch > 0) {
                    const int c = nfirst[s_node] + static_cast<int>(mt_pick(g, static_cast<uint64_t>(nch), &s_pick));
                    a.edges[s_edges++] = ncand[c];
                    a.pathnodes[s_path++] = c;
                    s_node = c;
                    s_child_row = ncand[c];
                }
                s_steps = 0;
                s_done = 0;
            }
            __syncthreads();
            if (s_expand) {
                // expanded in this iteration: `cur` still holds the parent's completion, and the
                // child's is the same adds the expansion made (bit for bit), without re-reading it
                if (s_child_row >= 0 && warp == 0) {
                    const uint64_t row = rowat(s_child_row);
                    for (int i = lane; i < n; i += 32) {
                        double v = cur[i];
#pragma unroll
                        for (int m = 0; m < 4; ++m) {
                            const int code = static_cast<int>((row >> (16 * m)) & 0xFFFFull);
                            if (csvc[code] == i) v = __dadd_rn(v, Us[code]);
                        }
                        cur[i] = v;
                    }
                }
            } else {
                for (int i = tid; i < n; i += blockDim.x) cur[i] = a.node_comp[static_cast<long long>(s_node) * n + i];
            }
            __syncthreads();
            // rollout (mcts.hpp:122-143) with the RolloutCache keyed by the unsatisfied bitmap:
            // warp 0 steps alone through cache hits; the block joins for a miss's top-K
            for (;;) {
                if (warp == 0) {
                    // Warp 0 walks; its state is warp-uniform registers: the unsatisfied bitmap (the
                    // type key), the cache entry it maps to (re-probed only when the key changes:
                    // most steps satisfy no service), the pick constants of that entry's size and
                    // the mt19937_64 position.  n <= 32: lane i keeps cur[i] in a register.
                    const bool regc = n <= 32;
                    double creg = regc && lane < n ? cur[lane] : 2.0;
                    int r_steps = *reinterpret_cast<volatile int*>(&s_steps);
                    int midx = *reinterpret_cast<volatile int*>(&g.idx);
                    uint64_t kw[NK];
#pragma unroll
                    for (int w = 0; w < NK; ++w) kw[w] = ~0ull;
                    bool have = false, inl1 = false;
                    int pn = 0, slot = 0;  // the entry: pool size, L1 slot (inl1) or global slot
#ifndef MGB_PICK_SERIAL
                    // picks of the next 32 draws for pool size sb_n, one per lane (lane j: draw
                    // sb_i0 + j), computed off the walk's serial chain; sb_stop marks lanes whose draw
                    // is rejected by pick_index or lies past the buffer: those steps take the serial path
                    int sb_n = -1, sb_i0 = 0;
                    unsigned sb_pick = 0u, sb_stop = 0u;
#endif
                    const int steps0 = r_steps;
                    const long long wc0 = timers ? clock64() : 0;
                    __syncwarp();
                    if (lane == 0) s_miss = 0;
                    for (;;) {
                        uint64_t kn[NK];
#pragma unroll
                        for (int w = 0; w < NK; ++w) kn[w] = 0ull;
                        if (regc) {
                            kn[0] = __ballot_sync(0xffffffffu, lane < n && creg < 1.0 - 1e-9);
                        } else {
#pragma unroll
                            for (int c = 0; c < 2 * NK; ++c) {  // static indices: kn stays in registers
                                const int i = 32 * c + lane;
                                if (32 * c < n) {
                                    const unsigned bm = __ballot_sync(0xffffffffu, i < n && cur[i] < 1.0 - 1e-9);
                                    kn[c >> 1] |= static_cast<uint64_t>(bm) << (32 * (c & 1));
                                }
                            }
                        }
                        int st = 0;  // 1 done, 2 miss, 3 abort
                        uint64_t any = 0ull, diff = 0ull;
#pragma unroll
                        for (int w = 0; w < NK; ++w) {
                            any |= kn[w];
                            diff |= kn[w] ^ kw[w];
                        }
                        if (!any || r_steps >= max_depth) {  // satisfied / depth cap
                            if (lane == 0) {
                                s_done = 1;
                                s_est = any ? max_depth : r_steps;
                            }
                            st = 1;
                        } else if (!have || diff) {
                            const long long pc0 = timers ? clock64() : 0;
#pragma unroll
                            for (int w = 0; w < NK; ++w) kw[w] = kn[w];
                            have = false;
                            // the cache's own hash (not reference-visible): one multiply
                            uint64_t h = kw[0];
#pragma unroll
                            for (int w = 1; w < NK; ++w) h ^= kw[w] << (16 * w) | kw[w] >> (64 - 16 * w);
                            h *= 0x9e3779b97f4a7c15ull;
                            h ^= h >> 29;
                            // level 1: the on-chip copy, probed 32 slots at a time (linear probing:
                            // the key lies before the first empty slot)
                            int l1 = -1;
                            // while the on-chip level has never refused a key (it is filled to 3/4)
                            // it holds every key of this search: an L1 miss is a cache miss
                            const bool l1_all = l1_slots && *reinterpret_cast<volatile int*>(&l1_used) < l1_slots * 3 / 4;
                            if (l1_slots) {
                                const unsigned q0 = static_cast<unsigned>(h >> 32) & (l1_slots - 1);
                                for (int b0 = 0; b0 < l1_slots; b0 += 32) {
                                    const unsigned q = (q0 + b0 + lane) & (l1_slots - 1);
                                    const int qn = l1n[q];
                                    bool match = qn != kL1Empty;
#pragma unroll
                                    for (int w = 0; w < NK; ++w)
                                        if (w < nk) match = match && l1k[q * nk + w] == kw[w];
                                    const unsigned bm = __ballot_sync(0xffffffffu, match);
                                    if (bm) {
                                        l1 = static_cast<int>((q0 + b0 + __ffs(bm) - 1) & (l1_slots - 1));
                                        break;
                                    }
                                    if (__ballot_sync(0xffffffffu, qn == kL1Empty)) break;
                                }
                            }
                            if (l1 >= 0) {
                                inl1 = true;
                                pn = l1n[l1];
                                slot = l1;
                            } else if (l1_all) {  // miss, inserted on chip only (no global round trips)
                                inl1 = false;
                                st = 2;
                                if (lane == 0) {
                                    unsigned q = static_cast<unsigned>(h >> 32) & (l1_slots - 1);
                                    while (l1n[q] != kL1Empty) q = (q + 1) & (l1_slots - 1);
#pragma unroll
                                    for (int w = 0; w < NK; ++w)
                                        if (w < nk) l1k[q * nk + w] = kw[w];
                                    l1n[q] = kL1Pending;
                                    ++l1_used;
                                    s_miss = 1;
                                    s_slot = -1;
                                    s_l1new = static_cast<int>(q);
                                }
                            } else {  // level 2: the global table (keys the full L1 refused), 32 slots a probe
                                inl1 = false;
                                int found = -1, empty_at = -1;
                                for (unsigned t0 = 0;; t0 += 32) {
                                    if (t0 > a.tab_mask) {
                                        if (lane == 0) s_abort = 2;  // cache full
                                        st = 3;
                                        break;
                                    }
                                    const unsigned sl = (static_cast<unsigned>(h) + t0 + lane) & a.tab_mask;
                                    const bool used = a.tag[sl] != 0;
                                    bool match = used;
#pragma unroll
                                    for (int w = 0; w < NK; ++w)
                                        if (w < nk) match = match && a.key[4ull * sl + w] == kw[w];
                                    const unsigned mm = __ballot_sync(0xffffffffu, match), em = __ballot_sync(0xffffffffu, !used);
                                    const unsigned fmask = mm & (em ? ((em & (0u - em)) - 1u) : 0xffffffffu);  // before the first empty
                                    if (fmask) {
                                        found = static_cast<int>((static_cast<unsigned>(h) + t0 + __ffs(fmask) - 1) & a.tab_mask);
                                        break;
                                    }
                                    if (em) {
                                        empty_at = static_cast<int>((static_cast<unsigned>(h) + t0 + __ffs(em) - 1) & a.tab_mask);
                                        break;
                                    }
                                }
                                if (st == 0 && found < 0) {  // miss: insert; the block builds the pool
                                    st = 2;
                                    if (lane == 0) {
                                        a.tag[empty_at] = 1;
#pragma unroll
                                        for (int w = 0; w < 4; ++w) a.key[4ull * empty_at + w] = w < NK ? kw[w] : 0ull;
                                        int l1new = -1;
                                        if (l1_slots && l1_used < l1_slots * 3 / 4) {  // mirror the new key on chip
                                            unsigned q = static_cast<unsigned>(h >> 32) & (l1_slots - 1);
                                            while (l1n[q] != kL1Empty) q = (q + 1) & (l1_slots - 1);
#pragma unroll
                                            for (int w = 0; w < NK; ++w)
                                                if (w < nk) l1k[q * nk + w] = kw[w];
                                            l1n[q] = kL1Pending;
                                            ++l1_used;
                                            l1new = static_cast<int>(q);
                                        }
                                        s_miss = 1;
                                        s_slot = empty_at;
                                        s_l1new = l1new;
                                    }
                                } else if (st == 0) {
                                    slot = found;
                                    pn = a.pool_n[found];
                                }
                            }
                            if (st == 0) {
                                if (pn <= 0) {
                                    if (lane == 0) s_abort = 1;  // "rollout: no candidate config serves the remaining demand"
                                    st = 3;
                                } else {
                                    have = true;
                                }
                            }
                            if (timers && lane == 0) {
                                ++s_wprobes;
                                s_wpcyc += clock64() - pc0;
                            }
                        }
                        if (st) {
                            if (midx >= 312) {  // twist here, warp-parallel, not in lane 0's next mt_next
                                mt_twist_warp(g);
                                midx = 0;
                            }
                            if (lane == 0) {
                                s_steps = r_steps;
                                g.idx = midx;
                                if (timers) {
                                    ++s_wentries;
                                    s_wsteps += r_steps - steps0;
                                    s_wcyc += clock64() - wc0;
                                }
                            }
                            if (regc && lane < n) cur[lane] = creg;
                            break;
                        }
                        // a uniform pick from the cached pool (pick_index, util.hpp:39-47), every lane
                        unsigned pk = 0;
#ifndef MGB_PICK_SERIAL
                        bool picked = false;
                        if (pn > 1) {
                            int off = midx - sb_i0;
                            if (pn != sb_n || off < 0 || off >= 32) {  // (re)fill the batch at midx
                                if (midx >= 312) {
                                    mt_twist_warp(g);
                                    midx = 0;
                                }
                                const uint64_t lim = s_pick.lim[pn], fm = s_pick.fm[pn];
                                const unsigned p32 = s_pick.p32[pn], m = static_cast<unsigned>(pn);
                                const int j = midx + lane;
                                const uint64_t r = j < 312 ? g.out[j] : ~0ull;
                                const unsigned ra = fastmod32(static_cast<unsigned>(r >> 32), fm, m), rb = fastmod32(static_cast<unsigned>(r), fm, m);
                                sb_pick = fastmod32(ra * p32 + rb, fm, m);
                                sb_stop = __ballot_sync(0xffffffffu, j >= 312 || r >= lim);
                                sb_n = pn;
                                sb_i0 = midx;
                                off = 0;
                            }
                            pk = __shfl_sync(0xffffffffu, sb_pick, off);
                            if (!((sb_stop >> off) & 1u)) {
                                ++midx;
                                picked = true;
                            } else {
                                sb_n = -1;  // the serial path below twists or rejects: refill after it
                            }
                        }
                        if (pn > 1 && !picked) {
#else
                        if (pn > 1) {  // pick_index constants (mt_pick), read beside the draw
#endif
                            const uint64_t lim = s_pick.lim[pn], fm = s_pick.fm[pn];
                            const unsigned p32 = s_pick.p32[pn];
                            uint64_t r;
                            do {
                                if (midx >= 312) {
                                    mt_twist_warp(g);
                                    midx = 0;
                                }
                                r = g.out[midx++];
                            } while (r >= lim);
                            const unsigned m = static_cast<unsigned>(pn);
                            const unsigned ra = fastmod32(static_cast<unsigned>(r >> 32), fm, m), rb = fastmod32(static_cast<unsigned>(r), fm, m);
                            pk = fastmod32(ra * p32 + rb, fm, m);
                        }
                        int idx;
                        uint64_t row;
                        if (inl1) {
                            const uint2 e = l1p[slot * K + pk];
                            idx = static_cast<int>(e.x);
                            row = pair ? (static_cast<uint64_t>(e.y) | hiS) : rowat(idx);
                        } else {
                            idx = static_cast<int>(a.pool[static_cast<long long>(slot) * K + pk]);
                            row = rowat(idx);
                        }
                        if (lane == 0) a.picked[r_steps] = idx;
                        ++r_steps;
                        if (regc) {  // rollout add (mcts.hpp:139) in the owning lanes
#ifndef MGB_WALK_ADD4
                            // a row's members are distinct services: a lane owns at most one of them,
                            // so select its term and add once (one FP64 add on the chain, not four)
                            int own = -1;
#pragma unroll
                            for (int m = 0; m < 4; ++m) {
                                const int code = static_cast<int>((row >> (16 * m)) & 0xFFFFull);
                                if (csvc[code] == lane) own = code;
                            }
                            if (own >= 0) creg = __dadd_rn(creg, Us[own]);
#else
#pragma unroll
                            for (int m = 0; m < 4; ++m) {
                                const int code = static_cast<int>((row >> (16 * m)) & 0xFFFFull);
                                if (csvc[code] == lane) creg = __dadd_rn(creg, Us[code]);
                            }
#endif
                        } else {
                            if (lane < 4) {  // distinct services: the adds commute
                                const int code = static_cast<int>((row >> (16 * lane)) & 0xFFFFull);
                                const int svc = csvc[code];
                                if (svc < n) cur[svc] = __dadd_rn(cur[svc], Us[code]);
                            }
                            __syncwarp();
                        }
                    }
                }
                __syncthreads();
                tick(t_roll);
                if (s_done || s_abort) break;
                // cache miss: top-K of the whole base pool (mcts.hpp:129-133); warp 0 then
                // finds the key again and picks from the new pool
                const int got = cluster_topk(false, s_out, &s_scored);
                tick(t_topk);
                if (tid < got) {
                    if (s_slot >= 0) a.pool[static_cast<long long>(s_slot) * K + tid] = static_cast<unsigned>(s_out[tid]);
                    if (s_l1new >= 0)
                        l1p[static_cast<long long>(s_l1new) * K + tid] =
                            make_uint2(static_cast<unsigned>(s_out[tid]), static_cast<unsigned>(rowat(s_out[tid])));
                }
                if (tid == 0) {
                    if (s_slot >= 0) a.pool_n[s_slot] = got;
                    if (s_l1new >= 0) l1n[s_l1new] = got;
                    ++s_builds;
                }
                __syncthreads();
                tick(t_miss);
            }
            if (s_abort) break;
            if (tid == 0) {  // mcts.hpp:210-218
                const bool complete = (nflags[s_node] & kLeaf) || s_steps == s_est;
                if (complete && s_est < max_depth) {
                    const int len = s_edges + s_steps;
                    if (!s_have || len < s_best) {
                        for (int q = 0; q < s_edges; ++q) a.best_out[q] = a.edges[q];
                        for (int q = 0; q < s_steps; ++q) a.best_out[s_edges + q] = a.picked[q];
                        s_best = len;
                        s_have = 1;
                    }
                }
            }
        }
        if (tid == 0) {  // backpropagation + trace (mcts.hpp:220-226)
            const int total = s_edges + s_est;
            const double reward = total > 0 ? fmin(1.0, __ddiv_rn(static_cast<double>(a.l_ref), static_cast<double>(total)))
                                            : 1.0;
            for (int q = 0; q < s_path; ++q) {
                const int nd = a.pathnodes[q];
                nvis[nd] += 1;
                nval[nd] = __dadd_rn(nval[nd], reward);
            }
            a.trace[4 * iter + 0] = iter;
            a.trace[4 * iter + 1] = s_edges;
            a.trace[4 * iter + 2] = s_est;
            a.trace[4 * iter + 3] = s_have ? s_best : -1;
            s_iters = iter + 1;
        }
        __syncthreads();
    }
    // visit-count descent (mcts.hpp:230-238); the host completes it with fast_algo
    if (tid == 0) {
        int node = 0, dl = 0;
        if (!s_abort)
            while ((nflags[node] & kExpanded) && !(nflags[node] & kLeaf) && nnch[node] > 0) {
                int pick = 0;
                for (int q = 1; q < nnch[node]; ++q)
                    if (nvis[nfirst[node] + q] > nvis[nfirst[node] + pick]) pick = q;
                node = nfirst[node] + pick;
                a.descent_out[dl++] = ncand[node];
            }
        for (int i = 0; i < n; ++i) a.descent_comp[i] = a.node_comp[static_cast<long long>(node) * n + i];
        a.out[0] = s_abort;
        a.out[1] = s_have ? s_best : -1;
        a.out[2] = dl;
        a.out[3] = (nflags[node] & kLeaf) ? 1 : 0;
        a.out[4] = s_builds;
        a.out[5] = s_nodes;
        a.out[6] = s_iters;
        a.out[7] = s_expands;
        reinterpret_cast<long long*>(a.out)[5] = t_sel;   // out[10..11]
        reinterpret_cast<long long*>(a.out)[6] = t_exp;   // out[12..13]
        reinterpret_cast<long long*>(a.out)[7] = t_miss;  // out[14..15]
        reinterpret_cast<long long*>(a.out)[8] = t_topk;  // out[16..17]
        reinterpret_cast<long long*>(a.out)[9] = t_roll;  // out[18..19]
        a.out[20] = static_cast<int>(g_mcts_fallbacks);
        a.out[21] = s_wsteps;
        reinterpret_cast<long long*>(a.out)[11] = s_wcyc;  // out[22..23]
        a.out[24] = s_wprobes;
        a.out[25] = s_wentries;
        reinterpret_cast<long long*>(a.out)[13] = s_wpcyc;  // out[26..27]
        reinterpret_cast<long long*>(a.out)[4] = s_expand_rows;  // out[8..9]
    }
    if (threadIdx.x == 0) s_exit = 1;  // release the helper ranks
    __syncthreads();
    cl.sync();
    cl.sync();  // ... and keep this shared memory alive until they have read the flag
}

// Dynamic shared memory of mcts_kernel (must mirror its carve order).
size_t mcts_smem_bytes(int n, int PP, int max_nodes, long long n_base, bool node_smem, bool rows_smem, bool pair,
                       int n_sup) {
    // n_base: rows of ONE rank's slice
    const size_t nW = static_cast<size_t>(n + 1) * PP;
    size_t off = 0;
    auto carve = [&](size_t bytes) { off = (off + bytes + 15) & ~size_t{15}; };
    carve(8 * nW);
    carve(8 * nW);
    carve(8 * static_cast<size_t>(n + 1));
    carve(sizeof(Cand) * kMCandCap);
    carve(sizeof(Cand) * 2 * kMMaxK);
    carve(4 * nW);
    carve(nW);
    carve(nW);
    if (node_smem) {
        carve(8 * static_cast<size_t>(max_nodes));
        for (int i = 0; i < 4; ++i) carve(4 * static_cast<size_t>(max_nodes));
        carve(static_cast<size_t>(max_nodes));
    }
    if (rows_smem) carve((pair ? 4 : 8) * static_cast<size_t>(n_base));
    if (n_sup) {  // support offsets, services, the active list
        carve(4 * static_cast<size_t>(n_sup + 1));
        carve(2 * static_cast<size_t>(n_sup));
        carve(4 * static_cast<size_t>(n_sup));
    }
    return off;
}
void mcts_read_topk_timers(unsigned long long* h) { cudaMemcpyFromSymbol(h, g_tk, sizeof g_tk); }
void mcts_set_dense_pct(int pct) { cudaMemcpyToSymbol(g_mcts_dense_pct, &pct, sizeof pct); }
const void* mcts_kernel_ptr(int n) {
    return n <= 64 ? reinterpret_cast<const void*>(&mcts_kernel<1>) : reinterpret_cast<const void*>(&mcts_kernel<4>);
}
int mcts_threads() { return kMThreads; }

}  // namespace mgb
