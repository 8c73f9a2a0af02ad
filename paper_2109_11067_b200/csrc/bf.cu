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

__device__ __forceinline__ bool bf_positive(const DevModel& M, uint64_t row, const double* c) {
    for (int j = 0; j < 4; ++j) {  // score > 0 <=> a member with need > 0 and utility > 0 (greedy.hpp:36-43)
        const int code = static_cast<int>((row >> (16 * j)) & 0xFFFFull);
        const int svc = code / M.PP;
        if (svc < M.n && __dadd_rn(1.0, -c[svc]) > 0.0 && M.U[code] > 0.0) return true;
    }
    return false;
}

__device__ __forceinline__ void bf_add(const DevModel& M, uint64_t row, double* c) {
    for (int j = 0; j < 4; ++j) {
        const int code = static_cast<int>((row >> (16 * j)) & 0xFFFFull);
        const int svc = code / M.PP;
        if (svc < M.n) c[svc] = __dadd_rn(c[svc], M.U[code]);
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
        const uint64_t row = a.rows[i];
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
        const uint64_t row = a.rows[idx[q]];
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
                const uint64_t row = a.rows[i];
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

const void* bf_kernel_ptr() { return reinterpret_cast<const void*>(&bf_kernel); }
const void* bf_warp_kernel_ptr() { return reinterpret_cast<const void*>(&bf_warp_kernel); }
const void* bf_sum_kernel_ptr() { return reinterpret_cast<const void*>(&bf_sum_kernel); }
int bf_threads() { return kBfThreads; }

}  // namespace mgb
