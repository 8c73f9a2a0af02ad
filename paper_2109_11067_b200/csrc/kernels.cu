// kernels.cu — hand-written sm_100a kernels of the MIG-SERVING optimizer hot path.
//
//   K1 enum_base_kernel   build_candidate_pool  (config_enum.hpp:192-202)
//   K2/K3 greedy_kernel   fast_algo             (greedy.hpp:95-145): persistent cooperative
//                         kernel; per step a coalesced 128-bit scan of the packed rows with
//                         a shared-memory need*U table, a warp-shuffle 3-key argmax, a
//                         grid-wide reduction, the completion update, maybe_extend
//                         (greedy.hpp:107-119) and the device-side extension enumerator
//                         (extend_candidate_pool, config_enum.hpp:206-211).
//   K4 topk_kernel        detail::topk_candidates (mcts.hpp:56-76)
//
// Bit-exactness: every floating add/multiply on the score path is an explicit
// __dadd_rn/__dmul_rn (and the TU is built with -fmad=false), so no FMA contraction
// changes the reference's FP64 bits (SURVEY §0 hazard 1).
#include <cuda/atomic>

#include "device.cuh"

namespace mgb {

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() { return (1u << lane_id()) - 1u; }

// Sense-free generation barrier across all (co-resident, cooperatively launched) CTAs.
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> g(*gen), c(*count);
        unsigned my = g.load(cuda::memory_order_relaxed);
        __threadfence();
        if (c.fetch_add(1u, cuda::memory_order_acq_rel) == nblocks - 1u) {
            c.store(0u, cuda::memory_order_relaxed);
            g.fetch_add(1u, cuda::memory_order_release);
        } else {
            while (g.load(cuda::memory_order_acquire) == my) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

// 128-bit lexicographic GpuConfig key (core.hpp:174-200): per normalized instance
// (slices asc, slot asc) a 15-bit field present|slices|slot|svc; shorter sorts first.
__device__ __noinline__ void row_key(const DevModel& M, uint64_t row, uint64_t& hi, uint64_t& lo) {
    int svc[4], pat[4], k = 0;
    const int sentinel = M.n * M.PP;
    for (int j = 0; j < 4; ++j) {
        int code = static_cast<int>((row >> (16 * j)) & 0xFFFFull);
        if (code == sentinel) break;
        svc[k] = code / M.PP;
        pat[k] = code % M.PP;
        ++k;
    }
    int tot[5] = {0, 0, 0, 0, 0};
    for (int j = 0; j < k; ++j)
        for (int s = 0; s < 5; ++s) tot[s] += M.pat_count[pat[j] * 5 + s];
    int L = 0;
    for (int l = 0; l < M.n_layouts; ++l) {
        bool eq = true;
        for (int s = 0; s < 5; ++s) eq &= M.layout_count[l * 5 + s] == tot[s];
        if (eq) {
            L = l;
            break;
        }
    }
    unsigned __int128 key = 0;
    int ninst = 0;
    for (int si = 0; si < M.n_sizes; ++si) {
        int j = 0, used = 0;
        for (int t = 0; t < tot[si]; ++t) {
            while (used >= M.pat_count[pat[j] * 5 + si]) {
                ++j;
                used = 0;
            }
            unsigned slot = static_cast<unsigned>(M.layout_slots[(L * 5 + si) * 7 + t]);
            unsigned f = (1u << 14) | (static_cast<unsigned>(M.sizes[si]) << 11) | (slot << 8) |
                         static_cast<unsigned>(svc[j]);
            key = (key << 15) | f;
            ++used;
            ++ninst;
        }
    }
    for (; ninst < 7; ++ninst) key <<= 15;
    hi = static_cast<uint64_t>(key >> 64);
    lo = static_cast<uint64_t>(key);
}

__device__ __forceinline__ bool row_key_less(const DevModel& M, uint64_t a, uint64_t b) {
    uint64_t ah, al, bh, bl;
    row_key(M, a, ah, al);
    row_key(M, b, bh, bl);
    return ah != bh ? ah < bh : al < bl;
}

// util_sum (config_enum.hpp:173): ascending members, starting from 0.0.
__device__ __forceinline__ double row_usum(const DevModel& M, uint64_t row) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) s = __dadd_rn(s, __ldg(&M.U[(row >> (16 * j)) & 0xFFFFull]));
    return s;
}

// candidate_preferred (greedy.hpp:63-67) on (score, util_sum, config) records.
__device__ __noinline__ bool better(const DevModel& M, const Best& a, const Best& b) {
    if (a.s != b.s) return a.s > b.s;
    if (a.row == kNoRow || b.row == kNoRow || a.row == b.row) return false;
    if (a.u != b.u) return a.u > b.u;
    return row_key_less(M, a.row, b.row);
}

__device__ __noinline__ Best consider_slow(const DevModel& M, uint64_t row, double s, Best best) {
    double u = row_usum(M, row);
    Best c{s, u, row};
    return (best.row == kNoRow || better(M, c, best)) ? c : best;
}

// score (greedy.hpp:36-43) with W = need*U precomputed per step (0 where need <= 0).
__device__ __forceinline__ double row_score(const double* __restrict__ W, uint64_t row) {
    double s = __dadd_rn(W[row & 0xFFFFull], W[(row >> 16) & 0xFFFFull]);
    s = __dadd_rn(s, W[(row >> 32) & 0xFFFFull]);
    return __dadd_rn(s, W[row >> 48]);
}

__device__ __forceinline__ void consider(const DevModel& M, const double* __restrict__ W, uint64_t row,
                                         Best& best) {
    double s = row_score(W, row);
    if (s > 0.0 && s >= best.s) best = consider_slow(M, row, s, best);
}

__device__ __forceinline__ Best shfl_best(const Best& b, int off) {
    Best o;
    o.s = __shfl_xor_sync(0xffffffffu, b.s, off);
    o.u = __shfl_xor_sync(0xffffffffu, b.u, off);
    o.row = __shfl_xor_sync(0xffffffffu, b.row, off);
    return o;
}

__device__ __forceinline__ Best warp_best(const DevModel& M, Best b) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        Best o = shfl_best(b, off);
        if (better(M, o, b)) b = o;
    }
    return b;
}

__device__ __forceinline__ Best none() { return Best{0.0, 0.0, kNoRow}; }

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
            Best p;
            p.s = __ldcg(&partials[i].s);
            p.u = __ldcg(&partials[i].u);
            p.row = __ldcg(reinterpret_cast<const unsigned long long*>(&partials[i].row));
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

// Scan rows[0, nrows) grid-stride with 4 x 128-bit loads in flight per thread.
__device__ __forceinline__ void scan_rows(const DevModel& M, const double* __restrict__ W,
                                          const uint64_t* __restrict__ rows, long long nrows, Best& best) {
    const uint4* v = reinterpret_cast<const uint4*>(rows);
    const long long nv = nrows >> 1;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < nv; i += 4 * stride) {
        uint4 a = __ldg(v + i), b = __ldg(v + i + stride), c = __ldg(v + i + 2 * stride),
              d = __ldg(v + i + 3 * stride);
        consider(M, W, (static_cast<uint64_t>(a.y) << 32) | a.x, best);
        consider(M, W, (static_cast<uint64_t>(a.w) << 32) | a.z, best);
        consider(M, W, (static_cast<uint64_t>(b.y) << 32) | b.x, best);
        consider(M, W, (static_cast<uint64_t>(b.w) << 32) | b.z, best);
        consider(M, W, (static_cast<uint64_t>(c.y) << 32) | c.x, best);
        consider(M, W, (static_cast<uint64_t>(c.w) << 32) | c.z, best);
        consider(M, W, (static_cast<uint64_t>(d.y) << 32) | d.x, best);
        consider(M, W, (static_cast<uint64_t>(d.w) << 32) | d.z, best);
    }
    for (; i < nv; i += stride) {
        uint4 a = __ldg(v + i);
        consider(M, W, (static_cast<uint64_t>(a.y) << 32) | a.x, best);
        consider(M, W, (static_cast<uint64_t>(a.w) << 32) | a.z, best);
    }
    if ((nrows & 1) && blockIdx.x == 0 && threadIdx.x == 0) consider(M, W, __ldg(rows + nrows - 1), best);
}

// W[e] = need * U[e] for need = 1 - comp[svc] > 0, else 0 (greedy.hpp:38-41).
__device__ __forceinline__ void build_W(const DevModel& M, const double* comp, double* W) {
    const int nW = (M.n + 1) * M.PP;
    for (int e = threadIdx.x; e < nW; e += blockDim.x) {
        int svc = e / M.PP;
        double w = 0.0;
        if (svc < M.n) {
            double need = __dadd_rn(1.0, -comp[svc]);
            if (need > 0.0) w = __dmul_rn(need, __ldg(&M.U[e]));
        }
        W[e] = w;
    }
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

}  // namespace

// ---------------------------------------------------------------- K1: base pool rows
// One warp per support (<= max_mix members, ascending service index); valid templates
// are written at a host-computed offset in template order (deterministic pool order).
__global__ void __launch_bounds__(256) enum_base_kernel(const __grid_constant__ DevModel M, const uint32_t* __restrict__ supports,
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
__global__ void __launch_bounds__(kThreads, 1) greedy_kernel(const __grid_constant__ GreedyArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const DevModel& M = a.M;
    const int n = M.n;
    const int nW = (n + 1) * M.PP;
    const int G = gridDim.x;
    double* W = reinterpret_cast<double*>(smem);
    double* comp = W + nW;
    double* best_single = comp + n;
    uint64_t* ev_mask = reinterpret_cast<uint64_t*>(best_single + n);  // n events x 4 words
    short* ev_of = reinterpret_cast<short*>(ev_mask + 4 * (n + 1));
    short* ev_svc = ev_of + n;
    uint8_t* xlist = reinterpret_cast<uint8_t*>(ev_svc + n + 1);
    __shared__ Best red[kWarps];
    __shared__ uint64_t unsat[4];
    __shared__ int s_events, s_first_new, s_done, s_m;

    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        comp[i] = a.comp0[i];
        best_single[i] = M.best_single[i];
        ev_of[i] = -1;
    }
    if (threadIdx.x == 0) s_events = 0;
    __syncthreads();

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
                    if (blockIdx.x == 0) a.ev_svc[pos] = i;
                }
                ev += __popc(b);
            }
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
    auto extend_new = [&](int first, int last) {
        for (int e = first; e < last; ++e) {
            __syncthreads();
            const int ie = ev_svc[e];
            const uint64_t* me = ev_mask + e * 4;
            if ((threadIdx.x >> 5) == 0) {
                int m = 0;
                for (int c = 0; c < (n + 31) / 32; ++c) {
                    int i = c * 32 + static_cast<int>(lane_id());
                    bool in = i < n && i != ie && ((me[i >> 6] >> (i & 63)) & 1ull);
                    unsigned b = __ballot_sync(0xffffffffu, in);
                    if (in) xlist[m + __popc(b & lanemask_lt())] = static_cast<uint8_t>(i);
                    m += __popc(b);
                }
                if (lane_id() == 0) s_m = m;
            }
            __syncthreads();
            const int m = s_m;
            long long seg[5] = {0, 0, 0, 0, 0};
            long long total = 0;
            for (int k = M.max_mix + 1; k <= 4; ++k) {
                seg[k] = binom(m, k - 1) * M.n_tmpl[k];
                total += seg[k];
            }
            const long long stride = static_cast<long long>(G) * blockDim.x;
            for (long long base = static_cast<long long>(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u);
                 base < total; base += stride) {
                long long g = base + lane_id();
                bool ok = g < total;
                uint64_t row = 0;
                if (ok) {
                    int k = M.max_mix + 1;
                    long long rem = g;
                    while (rem >= seg[k]) rem -= seg[k++];
                    const int nt = M.n_tmpl[k];
                    const long long r = rem / nt;
                    const int t = static_cast<int>(rem - r * nt);
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
                    // covered by an earlier extension event?
                    for (int j = 0; j < k && ok; ++j) {
                        int ev = ev_of[S[j]];
                        if (ev >= 0 && ev < e) {
                            const uint64_t* mk = ev_mask + ev * 4;
                            bool sub = true;
                            for (int x = 0; x < k; ++x) sub &= ((mk[S[x] >> 6] >> (S[x] & 63)) & 1ull) != 0;
                            if (sub) ok = false;
                        }
                    }
                    const uint64_t tp = M.tmpl[k][t];
                    for (int j = 0; j < 4; ++j) {
                        uint64_t code;
                        if (j < k) {
                            int p = static_cast<int>((tp >> (8 * (j + 1))) & 0xFF);
                            ok &= (M.pat_mask[p] & ~M.feas_mask[S[j]]) == 0;
                            code = static_cast<uint64_t>(S[j] * M.PP + p);
                        } else {
                            code = static_cast<uint64_t>(n * M.PP);
                        }
                        row |= code << (16 * j);
                    }
                }
                const unsigned b = __ballot_sync(0xffffffffu, ok);
                if (b) {
                    unsigned long long at = 0;
                    if (lane_id() == 0) at = atomicAdd(&a.st->ext_count, static_cast<unsigned long long>(__popc(b)));
                    at = __shfl_sync(0xffffffffu, at, 0);
                    if (at + __popc(b) > static_cast<unsigned long long>(a.ext_cap)) {
                        if (lane_id() == 0) atomicExch(&a.st->status, static_cast<int>(kExtOverflow));
                    } else if (ok) {
                        a.ext_rows[at + __popc(b & lanemask_lt())] = row;
                    }
                }
            }
        }
    };

    unsigned* bc = &a.st->bar_count;
    unsigned* bg = &a.st->bar_gen;
    int status = kOk;

    maybe_extend();
    if (s_events > s_first_new) {
        extend_new(s_first_new, s_events);
        grid_barrier(bc, bg, G);
    }
    int step = 0;
    long long rows_total = 0;
    while (!s_done) {
        if (*reinterpret_cast<volatile int*>(&a.st->status) != kOk) {
            status = *reinterpret_cast<volatile int*>(&a.st->status);
            break;
        }
        if (step >= a.cap_steps) {
            status = kStepOverflow;
            break;
        }
        build_W(M, comp, W);
        __syncthreads();
        const long long n_ext =
            static_cast<long long>(*reinterpret_cast<volatile unsigned long long*>(&a.st->ext_count));
        Best best = none();
        scan_rows(M, W, a.base_rows, a.n_base, best);
        scan_rows(M, W, a.ext_rows, n_ext, best);
        best = block_best(M, best, red);
        Best* part = a.partials + (step & 1) * G;
        if (threadIdx.x == 0) part[blockIdx.x] = best;
        grid_barrier(bc, bg, G);
        const Best win = grid_best(M, part, G, red);
        if (win.row == kNoRow) {
            status = kNoPositive;
            break;
        }
        rows_total += a.n_base + n_ext;
        if (threadIdx.x == 0) {
            for (int j = 0; j < 4; ++j) {
                int code = static_cast<int>((win.row >> (16 * j)) & 0xFFFFull);
                int svc = code / M.PP;
                if (svc < n) comp[svc] = __dadd_rn(comp[svc], __ldg(&M.U[code]));
            }
            if (blockIdx.x == 0) {
                a.pick_row[step] = win.row;
                a.pick_score[step] = win.s;
                a.pick_rows[step] = a.n_base + n_ext;
            }
        }
        __syncthreads();
        ++step;
        maybe_extend();
        if (s_events > s_first_new) {
            extend_new(s_first_new, s_events);
            grid_barrier(bc, bg, G);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.st->n_steps = step;
        a.st->n_events = s_events;
        a.st->rows_scored = rows_total;
        if (status != kOk) atomicExch(&a.st->status, status);
    }
}

// ---------------------------------------------------------------- K4: top-K
// K rounds of "argmax among rows strictly less preferred than the previous pick";
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
    build_W(M, comp, W);
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
                Best c{s, row_usum(M, row), row};
                if (!better(M, last, c)) continue;
                if (best.row == kNoRow || better(M, c, best)) best = c;
                continue;
            }
            if (s >= best.s) best = consider_slow(M, row, s, best);
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
size_t greedy_smem_bytes(int n, int PP) {
    size_t b = static_cast<size_t>((n + 1) * PP) * 8;  // W
    b += static_cast<size_t>(n) * 8 * 2;              // comp + best_single
    b += static_cast<size_t>(n + 1) * 4 * 8;          // event masks
    b += static_cast<size_t>(n) * 2 + static_cast<size_t>(n + 1) * 2;  // ev_of, ev_svc
    b += 256 + 16;                                    // xlist
    return (b + 15) & ~static_cast<size_t>(15);
}

size_t topk_smem_bytes(int n, int PP) { return static_cast<size_t>((n + 1) * PP + n) * 8 + 16; }

const void* greedy_kernel_ptr() { return reinterpret_cast<const void*>(&greedy_kernel); }
const void* topk_kernel_ptr() { return reinterpret_cast<const void*>(&topk_kernel); }
const void* enum_base_kernel_ptr() { return reinterpret_cast<const void*>(&enum_base_kernel); }
int kernel_threads() { return kThreads; }

}  // namespace mgb
