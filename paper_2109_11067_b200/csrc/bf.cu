// bf.cu — exhaustive minimum-GPU search (brute_force_optimum, bench.hpp:160-219) on the device.
//
// The reference's test oracle: iterative deepening over config multisets (nondecreasing pool
// indices), a child kept only if it scores > 0 under the current completion, pruned by the
// admissible bound ceil((1 - c_i) / best_any_i - 1e-12) (bench.hpp:176-184).  Here every depth
// d runs as launches over chunks of DFS prefixes in lexicographic order: thread t owns the
// prefix (i1 <= i2) of rank t and runs the rest of the search below it sequentially.  The
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

}  // namespace

__global__ void __launch_bounds__(kBfThreads) bf_kernel(const __grid_constant__ BfArgs a) {
    const DevModel& M = a.M;
    const int n = M.n, d = a.depth;
    const long long P = a.n_rows;
    const long long t = a.replay >= 0 ? a.replay : a.rank0 + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (a.replay >= 0 && (blockIdx.x | threadIdx.x)) return;
    if (a.replay < 0 && t >= a.rank_end) return;
    volatile unsigned long long* best_key = a.best_key;
    const int pl = min(d, 2);
    long long idx[kBfMaxDepth];
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
    double st[kBfMaxDepth + 1][kBfMaxN];  // st[k] = completion after k picks
    for (int i = 0; i < n; ++i) st[0][i] = 0.0;
    unsigned long long nodes = 0;
    int found = 0;  // length of the solution found (0: none)
    bool stop = false;
    // the prefix is a DFS path: every pick must score > 0 where it is taken (bench.hpp:198)
    bool ok = true;
    for (int q = 0; q < pl && ok; ++q) {
        const uint64_t row = a.rows[idx[q]];
        if (!bf_positive(M, row, st[q])) {
            ok = false;
            break;
        }
        if (q > 0 || pl == 1 || idx[1] == idx[0]) ++nodes;  // level-1 node: charged once
        for (int i = 0; i < n; ++i) st[q + 1][i] = st[q][i];
        bf_add(M, row, st[q + 1]);
        if (bf_satisfied(st[q + 1], n)) {  // bench.hpp:192-196
            found = q + 1;
            ok = false;
        } else if (q + 1 == d || bf_bound(st[q + 1], a.best_any, n) > d - (q + 1)) {
            ok = false;
        }
    }
    if (ok && pl < d && *best_key < static_cast<unsigned long long>(t)) ok = false;
    if (ok) {  // sequential DFS below the prefix, in the reference's child order
        long long next[kBfMaxDepth + 1];
        int depth = pl;
        next[depth] = idx[pl - 1];
        while (depth >= pl) {
            if (nodes > a.remaining) {
                atomicMin(a.overrun, static_cast<unsigned long long>(t));
                stop = true;
                break;
            }
            if ((nodes & 255ull) == 255ull && *best_key < static_cast<unsigned long long>(t)) {
                stop = true;
                break;
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
            if (bf_satisfied(st[depth + 1], n)) {
                found = depth + 1;
                break;
            }
            if (depth + 1 == d || bf_bound(st[depth + 1], a.best_any, n) > d - (depth + 1)) continue;
            ++depth;
            next[depth] = i;
        }
    }
    if (!stop && nodes > a.remaining) atomicMin(a.overrun, static_cast<unsigned long long>(t));
    if (a.replay >= 0) {
        for (int q = 0; q < found; ++q) a.tuple[q] = idx[q];
        a.tuple[kBfMaxDepth] = found;
        return;
    }
    a.cnt[t - a.rank0] = nodes;
    if (found && !stop) atomicMin(a.best_key, static_cast<unsigned long long>(t));
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
const void* bf_sum_kernel_ptr() { return reinterpret_cast<const void*>(&bf_sum_kernel); }
int bf_threads() { return kBfThreads; }

}  // namespace mgb
