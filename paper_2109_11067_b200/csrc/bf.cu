// bf.cu — exhaustive minimum-GPU search (brute_force_optimum, bench.hpp:160-219) on the device.
//
// The reference's test oracle: iterative deepening over config multisets (nondecreasing pool
// indices), a child kept only if it scores > 0 under the current completion, pruned by the
// admissible bound ceil((1 - c_i) / best_any_i - 1e-12) (bench.hpp:176-184).  Here every depth
// d runs as launches over chunks of DFS prefixes in lexicographic order: the prefix (i1 <= i2)
// of rank t is owned by a thread (d <= 2) or a warp whose lanes split its level-3 children
// (d >= 3), and the rest of the search below runs sequentially.  The rows are the pool in the
// reference's emission order (the host permutes them, engine.cu Engine::brute_force).  The
// reference's DFS visits the prefixes in rank order and stops at its first solution, so its
// result is the smallest solving rank's first solution (atomicMin + a replay launch), and
// its node count is exactly 1 (root) + Σ_{t <= t*} cnt[t] where cnt[t] counts the nodes the
// reference enters inside prefix t's subtree (a level-1 node is charged to its (i1, i1)
// prefix).  The budget is therefore enforced exactly as the reference's ++nodes > budget:
// a thread whose own count passes the remaining budget records its rank (overrun), and the
// host throws iff that rank precedes the stopping rank or the exact prefix sum passes it.
// Threads whose rank exceeds an already-found solution stop early (their counts are moot).
#include "common.cuh"

namespace mgb {

using namespace dev;

namespace {

constexpr int kBfThreads = 256;

__device__ __forceinline__ int bf_code(const uint4& row, int j) {  // member j's u16 code
    const unsigned w = j < 4 ? (j < 2 ? row.x : row.y) : (j < 6 ? row.z : row.w);
    return static_cast<int>((w >> (16 * (j & 1))) & 0xFFFFu);
}

__device__ __forceinline__ bool bf_positive(const DevModel& M, const uint4& row, const double* c) {
    for (int j = 0; j < kBfCodes; ++j) {  // score > 0 <=> a member with need > 0 and utility > 0 (greedy.hpp:36-43)
        const int code = bf_code(row, j);
        const int svc = code / M.PP;
        if (svc >= M.n) break;  // members are packed in front of the sentinels
        if (__dadd_rn(1.0, -c[svc]) > 0.0 && M.U[code] > 0.0) return true;
    }
    return false;
}

__device__ __forceinline__ void bf_add(const DevModel& M, const uint4& row, double* c) {
    for (int j = 0; j < kBfCodes; ++j) {
        const int code = bf_code(row, j);
        const int svc = code / M.PP;
        if (svc >= M.n) break;
        c[svc] = __dadd_rn(c[svc], M.U[code]);
    }
}

__device__ __forceinline__ bool bf_satisfied(const double* c, int n) {
    for (int i = 0; i < n; ++i)
        if (c[i] < 1.0 - 1e-9) return false;
    return true;
}

__device__ __forceinline__ int bf_bound(const double* c, const double* best_any, int n) {  // bench.hpp:176-184
    int need = 0;
    for (int i = 0; i < n; ++i) {
        const double residual = __dadd_rn(1.0, -c[i]);
        if (residual > 1e-9)
            need = max(need, static_cast<int>(ceil(__dadd_rn(__ddiv_rn(residual, best_any[i]), -1e-12))));
    }
    return need;
}

// Sequential DFS below the node at `depth` (picks idx[0..depth-1], completion st[depth]),
// children from pool index next0 on, in the reference's order (bench.hpp:197-205).  Counts
// entered nodes into `nodes`; returns the found length (0: none).  Stops (stop = true) when
// `base + nodes` passes the remaining budget (over = true) or a smaller rank has already
// solved this depth.
__device__ __forceinline__ int bf_dfs(const BfArgs& a, double (*st)[kBfMaxN], long long* idx, int depth,
                                      long long next0, unsigned long long base, unsigned long long& nodes,
                                      bool& stop, bool& over, unsigned long long t) {
    const DevModel& M = a.M;
    const int n = M.n, d = a.depth, top = depth;
    const long long P = a.n_rows;
    volatile unsigned long long* best_key = a.best_key;
    long long next[kBfMaxDepth + 1];
    next[depth] = next0;
    while (depth >= top) {
        if (base + nodes > a.remaining) {
            stop = over = true;
            return 0;
        }
        if ((nodes & 255ull) == 255ull && *best_key < t) {
            stop = true;
            return 0;
        }
        const long long i = next[depth]++;
        if (i >= P) {
            --depth;
            continue;
        }
        const uint4 row = a.rows[i];
        if (!bf_positive(M, row, st[depth])) continue;
        ++nodes;
        for (int k = 0; k < n; ++k) st[depth + 1][k] = st[depth][k];
        bf_add(M, row, st[depth + 1]);
        idx[depth] = i;
        if (bf_satisfied(st[depth + 1], n)) return depth + 1;
        if (depth + 1 == d || bf_bound(st[depth + 1], a.best_any, n) > d - (depth + 1)) continue;
        ++depth;
        next[depth] = i;
    }
    return 0;
}

// Walk the prefix of rank t (one or two picks): every pick must score > 0 where it is taken
// (bench.hpp:198).  Returns true when the search continues below it.
__device__ __forceinline__ bool bf_prefix(const BfArgs& a, long long t, double (*st)[kBfMaxN], long long* idx,
                                          int pl, unsigned long long& nodes, int& found) {
    const DevModel& M = a.M;
    const int n = M.n, d = a.depth;
    const long long P = a.n_rows;
    if (pl == 1) {
        idx[0] = t;
    } else {  // unrank t -> (i1, i2), i1 <= i2 < P; row i1 starts at i1*P - i1*(i1-1)/2
        long long lo = 0, hi = P - 1;
        while (lo < hi) {
            const long long mid = (lo + hi + 1) >> 1;
            if (mid * P - mid * (mid - 1) / 2 <= t) lo = mid;
            else hi = mid - 1;
        }
        idx[0] = lo;
        idx[1] = lo + (t - (lo * P - lo * (lo - 1) / 2));
    }
    for (int i = 0; i < n; ++i) st[0][i] = 0.0;
    for (int q = 0; q < pl; ++q) {
        const uint4 row = a.rows[idx[q]];
        if (!bf_positive(M, row, st[q])) return false;
        if (q > 0 || pl == 1 || idx[1] == idx[0]) ++nodes;  // a level-1 node is charged once
        for (int i = 0; i < n; ++i) st[q + 1][i] = st[q][i];
        bf_add(M, row, st[q + 1]);
        if (bf_satisfied(st[q + 1], n)) {  // bench.hpp:192-196
            found = q + 1;
            return false;
        }
        if (q + 1 == d || bf_bound(st[q + 1], a.best_any, n) > d - (q + 1)) return false;
    }
    return true;
}

}  // namespace

// Depth 1-2 (and the replay of any depth): one thread per prefix.
__global__ void __launch_bounds__(kBfThreads) bf_kernel(const __grid_constant__ BfArgs a) {
    const long long t = a.replay >= 0 ? a.replay : a.rank0 + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (a.replay >= 0 && (blockIdx.x | threadIdx.x)) return;
    if (a.replay < 0 && t >= a.rank_end) return;
    const unsigned long long tk = static_cast<unsigned long long>(t);
    const int pl = min(a.depth, 2);
    double st[kBfMaxDepth + 1][kBfMaxN];  // st[k] = completion after k picks
    long long idx[kBfMaxDepth];
    unsigned long long nodes = 0;
    int found = 0;
    bool stop = false, over = false;
    if (bf_prefix(a, t, st, idx, pl, nodes, found) && *reinterpret_cast<volatile unsigned long long*>(a.best_key) >= tk)
        found = bf_dfs(a, st, idx, pl, idx[pl - 1], 0, nodes, stop, over, tk);
    if (over || nodes > a.remaining) atomicMin(a.overrun, tk);
    if (a.replay >= 0) {
        for (int q = 0; q < found; ++q) a.tuple[q] = idx[q];
        a.tuple[kBfMaxDepth] = found;
        return;
    }
    a.cnt[t - a.rank0] = nodes;
    if (found && !stop) atomicMin(a.best_key, tk);
}

// Depth >= 3: one warp per two-pick prefix; the 32 lanes take its level-3 children in
// rounds of 32 consecutive pool indices and search below them.  A round's first solving
// lane (lowest index) is the prefix's first solution in the reference's order, and the
// prefix's node count is everything before it: the lanes below it plus its own partial.
__global__ void __launch_bounds__(kBfThreads) bf_warp_kernel(const __grid_constant__ BfArgs a) {
    const int lane = threadIdx.x & 31;
    const long long w = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const long long t = a.replay >= 0 ? a.replay : a.rank0 + w;
    if (a.replay >= 0 && w) return;
    if (a.replay < 0 && t >= a.rank_end) return;
    const unsigned long long tk = static_cast<unsigned long long>(t);
    const DevModel& M = a.M;
    const int n = M.n, d = a.depth;
    const long long P = a.n_rows;
    volatile unsigned long long* best_key = a.best_key;
    double st[kBfMaxDepth + 1][kBfMaxN];
    long long idx[kBfMaxDepth];
    unsigned long long total = 0;  // the prefix's reference-order node count (warp-uniform)
    int found = 0;
    bool stop = false, over = false;
    const bool go = bf_prefix(a, t, st, idx, 2, total, found) && *best_key >= tk;
    if (go) {
        for (long long b = idx[1]; b < P; b += 32) {
            const long long i = b + lane;
            unsigned long long nodes = 0;
            int f = 0;
            bool lstop = false, lover = false;
            if (i < P) {
                const uint4 row = a.rows[i];
                if (bf_positive(M, row, st[2])) {
                    nodes = 1;
                    for (int k = 0; k < n; ++k) st[3][k] = st[2][k];
                    bf_add(M, row, st[3]);
                    idx[2] = i;
                    if (bf_satisfied(st[3], n)) f = 3;
                    else if (d > 3 && bf_bound(st[3], a.best_any, n) <= d - 3)
                        f = bf_dfs(a, st, idx, 3, i, total, nodes, lstop, lover, tk);
                    if (total + nodes > a.remaining) lover = true;
                }
            }
            const unsigned fm = __ballot_sync(0xffffffffu, f != 0);
            const unsigned om = __ballot_sync(0xffffffffu, lover);
            const unsigned sm = __ballot_sync(0xffffffffu, lstop && !lover);
            const unsigned upto = fm ? ((fm & (0u - fm)) << 1) - 1u : 0xffffffffu;  // lanes <= first solver
            if (om & upto) {
                over = true;
                break;
            }
            if (sm & upto) {  // a smaller rank solved: this prefix's count is moot
                stop = true;
                break;
            }
            unsigned long long c = (upto >> lane) & 1u ? nodes : 0ull;
            for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            total += c;
            if (fm) {
                const int wl = __ffs(fm) - 1;
                found = __shfl_sync(0xffffffffu, f, wl);
                if (a.replay >= 0 && lane == wl) {
                    for (int q = 0; q < found; ++q) a.tuple[q] = idx[q];
                    a.tuple[kBfMaxDepth] = found;
                }
                break;
            }
            if (total > a.remaining) {
                over = true;
                break;
            }
            if (*best_key < tk) {
                stop = true;
                break;
            }
        }
    }
    if (lane) return;
    if (over || total > a.remaining) atomicMin(a.overrun, tk);
    if (a.replay >= 0) {
        if (!go || found < 3) {  // solved inside the prefix
            for (int q = 0; q < found; ++q) a.tuple[q] = idx[q];
            a.tuple[kBfMaxDepth] = found;
        }
        return;
    }
    a.cnt[t - a.rank0] = total;
    if (found && !stop && !over) atomicMin(a.best_key, tk);
}

// *a.sum += Σ cnt[0 .. min(best_key, rank_end - 1) - rank0]: the reference's node count for
// this launch's part of the DFS.
__global__ void __launch_bounds__(kBfThreads) bf_sum_kernel(const __grid_constant__ BfArgs a) {
    const unsigned long long bk = *a.best_key;
    const long long last = bk < static_cast<unsigned long long>(a.rank_end) ? static_cast<long long>(bk) : a.rank_end - 1;
    const long long m = last - a.rank0 + 1;
    unsigned long long s = 0;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        s += a.cnt[i];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(a.sum, s);
}

// ---- the pool (build_candidate_pool(services, profiles, rules, min(n, 7)), bench.hpp:164-165)
namespace {

__device__ __forceinline__ long long bf_multichoose(int m, int r) {  // C(m + r - 1, r): r-sequences over m symbols
    long long c = 1;
    for (int i = 1; i <= r; ++i) c = c * (m + i - 1) / i;  // exact: c * (m+i-1) is divisible by i
    return c;
}

// Decode flat index t into its config (fill_group / materialize, config_enum.hpp:131-183);
// false when a service is infeasible at its size or the support exceeds max_mix.
__device__ bool bf_enum_row(const BfEnumArgs& e, long long t, uint4& out) {
    int li = 0;
    while (t >= e.lay_off[li + 1]) ++li;
    long long r = t - e.lay_off[li];
    const int G = e.n_groups[li];
    long long dig[5];
    for (int g = G - 1; g >= 0; --g) {
        dig[g] = r % e.g_cnt[li][g];
        r /= e.g_cnt[li][g];
    }
    unsigned mask = 0;
    unsigned cnt[kBfMaxN];  // per service: instance counts, 3 bits per size index
    for (int g = 0; g < G; ++g) {
        const int len = e.g_len[li][g], z = e.g_size[li][g];
        long long q = dig[g];
        int v = 0;
        for (int p = 0; p < len; ++p) {  // lexicographic unrank of a nondecreasing sequence
            const int rem = len - p - 1;
            for (;; ++v) {
                const long long c = bf_multichoose(e.n - v, rem);
                if (q < c) break;
                q -= c;
            }
            if (!((e.feas_mask[v] >> z) & 1u)) return false;  // config_enum.hpp:142
            if (!((mask >> v) & 1u)) cnt[v] = 0;
            mask |= 1u << v;
            cnt[v] += 1u << (3 * z);
        }
    }
    if (__popc(mask) > e.max_mix) return false;  // config_enum.hpp:145
    unsigned short code[kBfCodes];
    int k = 0;
    for (unsigned m = mask; m; m &= m - 1) {  // members in ascending service order
        const int v = __ffs(m) - 1;
        const int pat = e.pat_of[cnt[v]];
        if (pat == 0xFF) *e.error = 1;
        code[k++] = static_cast<unsigned short>(v * e.PP + pat);
    }
    for (; k < kBfCodes; ++k) code[k] = static_cast<unsigned short>(e.n * e.PP);
    out = make_uint4(code[0] | static_cast<unsigned>(code[1]) << 16, code[2] | static_cast<unsigned>(code[3]) << 16,
                     code[4] | static_cast<unsigned>(code[5]) << 16, code[6] | static_cast<unsigned>(code[7]) << 16);
    return true;
}

}  // namespace

// mode 0: block_cnt[b] = valid configs among indices [256 b, 256 b + 256); mode 1: write them,
// in index order, from block_cnt[b] (the exclusive scan) on.
__global__ void __launch_bounds__(256) bf_enum_kernel(const __grid_constant__ BfEnumArgs e, int mode) {
    const long long t = static_cast<long long>(blockIdx.x) * 256 + threadIdx.x;
    uint4 row;
    const bool ok = t < e.lay_off[e.n_layouts] && bf_enum_row(e, t, row);
    __shared__ unsigned wcnt[8];
    const unsigned bm = __ballot_sync(0xffffffffu, ok);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) wcnt[w] = __popc(bm);
    __syncthreads();
    if (mode == 0) {
        if (threadIdx.x == 0) {
            unsigned c = 0;
            for (int i = 0; i < 8; ++i) c += wcnt[i];
            e.block_cnt[blockIdx.x] = c;
        }
        return;
    }
    if (!ok) return;
    unsigned pos = e.block_cnt[blockIdx.x] + __popc(bm & ((1u << lane) - 1u));
    for (int i = 0; i < w; ++i) pos += wcnt[i];
    e.rows[pos] = row;
}

// In-place exclusive scan of block_cnt[0..nb) by one CTA; block_cnt[nb] = total.
__global__ void __launch_bounds__(1024) bf_scan_kernel(unsigned* c, int nb) {
    __shared__ unsigned wsum[32];
    __shared__ unsigned carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int b0 = 0; b0 < nb; b0 += 1024) {
        const int i = b0 + threadIdx.x;
        const unsigned v = i < nb ? c[i] : 0u;
        unsigned x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        if (w == 0) {
            unsigned s = wsum[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            wsum[lane] = s;
        }
        __syncthreads();
        const unsigned incl = x + (w ? wsum[w - 1] : 0u) + carry;
        if (i < nb) c[i] = incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry = incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) c[nb] = carry;
}

// best_any[i] = max over the pool of the utility configs give service i (bench.hpp:167-171);
// utilities are >= 0, so their bit patterns order like the values.
__global__ void __launch_bounds__(256) bf_best_any_kernel(const DevModel M, const uint4* rows, long long P,
                                                          unsigned long long* best_bits) {
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < P;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const uint4 row = rows[i];
        for (int j = 0; j < kBfCodes; ++j) {
            const int code = bf_code(row, j);
            const int svc = code / M.PP;
            if (svc >= M.n) break;
            atomicMax(best_bits + svc, static_cast<unsigned long long>(__double_as_longlong(M.U[code])));
        }
    }
}

const void* bf_kernel_ptr() { return reinterpret_cast<const void*>(&bf_kernel); }
const void* bf_warp_kernel_ptr() { return reinterpret_cast<const void*>(&bf_warp_kernel); }
const void* bf_sum_kernel_ptr() { return reinterpret_cast<const void*>(&bf_sum_kernel); }
int bf_threads() { return kBfThreads; }
const void* bf_enum_kernel_ptr() { return reinterpret_cast<const void*>(&bf_enum_kernel); }
const void* bf_scan_kernel_ptr() { return reinterpret_cast<const void*>(&bf_scan_kernel); }
const void* bf_best_any_kernel_ptr() { return reinterpret_cast<const void*>(&bf_best_any_kernel); }

}  // namespace mgb
