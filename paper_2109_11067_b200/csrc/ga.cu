// ga.cu — K6: one GA generation over a whole population on the device (throughput mode).
//
// The reference's two_phase (ga.hpp:126-179) breeds ceil(P/2) children per round on host
// threads: child i = crossover(mutate(pop[i])) with a sequential mt19937_64 stream seeded by
// mix_seed(seed, (round << 20) + i).  Here every child is one CTA:
//   ga_breed_kernel   mutate (ga.hpp:83-113): equal-size (service, batch) swaps over the
//                     GPU-major instance refs; crossover (ga.hpp:51-66): erase ceil(f*n) GPUs
//                     by a partial Fisher-Yates, survivors kept in order, and their residual
//                     completion (count-based sums, core.hpp:245-269, bit-exact);
//   (greedy_kernel    the refill, FastProcedure (greedy.hpp:160-164): all children's
//                     fast_algo runs as CTA groups of ONE launch, engine.cu greedy_batch)
//   ga_finish_kernel  child = survivors + refill, evaluate_chromosome (ga.hpp:38-46):
//                     completion, validity, slack; a failed refill returns the mutated parent.
// Draw t of child i in round r is Philox4x32-10(key = seed, counter = (t, (r << 20) + i)),
// index = floor(draw * n / 2^64) (philox.cuh) — identical on host (oracle/oracle.cpp).
#include "common.cuh"
#include "philox.cuh"

namespace mgb {

using namespace dev;

namespace {

constexpr int kGaThreads = 256;
constexpr int kGaMaxSizes = 5;
constexpr unsigned char kNoSvc = 0xFF;

__device__ __forceinline__ int genome_layout(uint64_t g) { return static_cast<int>(g & 0xFFull); }
__device__ __forceinline__ int genome_svc(uint64_t g, int k) { return static_cast<int>((g >> (8 * (k + 1))) & 0xFFull); }

// Instances of layout L in normalized order: size index ascending, slot ascending.
__device__ __forceinline__ int layout_sizes(const DevModel& M, int L, int* si_of) {
    int k = 0;
    for (int si = 0; si < M.n_sizes; ++si)
        for (int t = 0; t < M.layout_count[L * 5 + si]; ++t) si_of[k++] = si;
    return k;
}

// Packed candidate row -> genome (Model::decode order: within a size, lower service index
// takes the lower slots, config_enum.hpp:140,159-163).
__device__ uint64_t row_genome(const DevModel& M, uint64_t row) {
    int svc[4], pat[4], k = 0;
    const int sentinel = M.n * M.PP;
    for (int j = 0; j < 4; ++j) {
        const int code = static_cast<int>((row >> (16 * j)) & 0xFFFFull);
        if (code == sentinel) break;
        svc[k] = svc_of(M, static_cast<unsigned>(code));
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
    uint64_t g = static_cast<uint64_t>(L);
    int pos = 0;
    for (int si = 0; si < M.n_sizes; ++si)
        for (int j = 0; j < k; ++j)
            for (int c = 0; c < M.pat_count[pat[j] * 5 + si]; ++c) g |= static_cast<uint64_t>(svc[j]) << (8 * (1 + pos++));
    for (; pos < 7; ++pos) g |= static_cast<uint64_t>(kNoSvc) << (8 * (1 + pos));
    return g;
}

// completion_of (core.hpp:291-302, detail::sum_rates): instance counts per (service, size),
// then per service total = sum over sizes ascending of count * thr, divided once by req.
// cnt: n * 5 ints of shared memory.  Writes comp[0..n).  Block-wide.
__device__ void completion(const DevModel& M, const uint64_t* gpus, int len, int* cnt, double* comp) {
    for (int i = threadIdx.x; i < M.n * kGaMaxSizes; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    for (int g = threadIdx.x; g < len; g += blockDim.x) {
        const uint64_t x = gpus[g];
        int si_of[7];
        const int ni = layout_sizes(M, genome_layout(x), si_of);
        for (int k = 0; k < ni; ++k) {
            const int s = genome_svc(x, k);
            if (s < M.n) atomicAdd(&cnt[s * kGaMaxSizes + si_of[k]], 1);
        }
    }
    __syncthreads();
    for (int s = threadIdx.x; s < M.n; s += blockDim.x) {
        double total = 0.0;
        for (int si = 0; si < M.n_sizes; ++si) {
            const int c = cnt[s * kGaMaxSizes + si];
            if (c) total = __dadd_rn(total, __dmul_rn(static_cast<double>(c), M.thr[s * kGaMaxSizes + si]));
        }
        comp[s] = __ddiv_rn(total, M.req[s]);
    }
    __syncthreads();
}

// Ordered compaction helper: exclusive prefix of one int per thread (block-wide).
__device__ int block_excl_scan(int v, int* tmp, int& total) {
    tmp[threadIdx.x] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0;
        for (int t = 0; t < static_cast<int>(blockDim.x); ++t) {
            const int x = tmp[t];
            tmp[t] = run;
            run += x;
        }
        tmp[blockDim.x] = run;
    }
    __syncthreads();
    const int r = tmp[threadIdx.x];
    total = tmp[blockDim.x];
    __syncthreads();
    return r;
}

}  // namespace

__global__ void __launch_bounds__(kGaThreads) ga_breed_kernel(const __grid_constant__ GaBreedArgs a) {
    const DevModel& M = a.M;
    const int c = blockIdx.x;
    const int L = a.pop_len[c];
    const uint64_t* parent = a.pop + static_cast<long long>(c) * a.L_cap;
    uint64_t* work = a.work + static_cast<long long>(c) * a.L_cap;
    uint64_t* child = a.child + static_cast<long long>(c) * a.L_cap;
    unsigned* scratch = a.scratch + static_cast<long long>(c) * 8 * a.L_cap;
    extern __shared__ __align__(16) unsigned char smem[];
    int* cnt = reinterpret_cast<int*>(smem);                    // n * 5
    int* tmp = cnt + M.n * kGaMaxSizes;                         // blockDim + 1
    int* per = tmp + kGaThreads + 1;                            // blockDim * 5
    __shared__ int seg[kGaMaxSizes + 1], total_of[kGaMaxSizes], elig[kGaMaxSizes], n_elig;
    __shared__ unsigned long long draws;
    const uint64_t stream = (static_cast<uint64_t>(a.round) << 20) + static_cast<uint64_t>(c);
    auto draw_below = [&](uint64_t n) { return philox_below(philox_u64(a.seed, stream, draws++), n); };

    for (int g = threadIdx.x; g < L; g += blockDim.x) work[g] = parent[g];
    // ---- mutate: refs by size in GPU-major, normalized-instance order (ga.hpp:88-96)
    const int chunk = (L + blockDim.x - 1) / blockDim.x;
    const int g0 = min(L, static_cast<int>(threadIdx.x) * chunk), g1 = min(L, g0 + chunk);
    int mine[kGaMaxSizes] = {0, 0, 0, 0, 0};
    for (int g = g0; g < g1; ++g) {
        int si_of[7];
        const int ni = layout_sizes(M, genome_layout(parent[g]), si_of);
        for (int k = 0; k < ni; ++k) mine[si_of[k]]++;
    }
    for (int si = 0; si < kGaMaxSizes; ++si) per[threadIdx.x * kGaMaxSizes + si] = mine[si];
    __syncthreads();
    if (threadIdx.x < kGaMaxSizes) {  // per size: exclusive prefix over threads
        const int si = threadIdx.x;
        int run = 0;
        for (int t = 0; t < static_cast<int>(blockDim.x); ++t) {
            const int x = per[t * kGaMaxSizes + si];
            per[t * kGaMaxSizes + si] = run;
            run += x;
        }
        total_of[si] = run;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int o = 0;
        n_elig = 0;
        for (int si = 0; si < kGaMaxSizes; ++si) {
            seg[si] = o;
            o += total_of[si];
            if (total_of[si] >= 2) elig[n_elig++] = si;  // sizes with >= 2 refs, ascending (ga.hpp:92-94)
        }
        seg[kGaMaxSizes] = o;
        draws = 0;
    }
    __syncthreads();
    {
        int at[kGaMaxSizes];
        for (int si = 0; si < kGaMaxSizes; ++si) at[si] = seg[si] + per[threadIdx.x * kGaMaxSizes + si];
        for (int g = g0; g < g1; ++g) {
            int si_of[7];
            const int ni = layout_sizes(M, genome_layout(parent[g]), si_of);
            for (int k = 0; k < ni; ++k) scratch[at[si_of[k]]++] = (static_cast<unsigned>(g) << 3) | static_cast<unsigned>(k);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && n_elig > 0) {  // ga.hpp:97-111
        for (int pair = 0; pair < a.mutation_pairs; ++pair) {
            for (int attempt = 0; attempt < 64; ++attempt) {
                const int si = elig[draw_below(static_cast<uint64_t>(n_elig))];
                const unsigned ra = scratch[seg[si] + draw_below(static_cast<uint64_t>(total_of[si]))];
                const unsigned rb = scratch[seg[si] + draw_below(static_cast<uint64_t>(total_of[si]))];
                const int ga = static_cast<int>(ra >> 3), ka = static_cast<int>(ra & 7u);
                const int gb = static_cast<int>(rb >> 3), kb = static_cast<int>(rb & 7u);
                const int sa = genome_svc(work[ga], ka), sb = genome_svc(work[gb], kb);
                if (sa == sb) continue;
                const uint64_t ma = 0xFFull << (8 * (ka + 1)), mb = 0xFFull << (8 * (kb + 1));
                work[ga] = (work[ga] & ~ma) | (static_cast<uint64_t>(sb) << (8 * (ka + 1)));
                work[gb] = (work[gb] & ~mb) | (static_cast<uint64_t>(sa) << (8 * (kb + 1)));
                break;
            }
        }
    }
    __syncthreads();
    // ---- crossover: erase ceil(f * n) GPUs by a partial Fisher-Yates (ga.hpp:53-66)
    const int erase = L == 0 ? 0 : static_cast<int>(ceil(__dmul_rn(a.erase_fraction, static_cast<double>(L))));
    if (erase == 0) {  // crossover returns its (mutated) parent (ga.hpp:55)
        if (threadIdx.x == 0) a.n_surv[c] = -1;
        return;
    }
    for (int i = threadIdx.x; i < L; i += blockDim.x) scratch[i] = static_cast<unsigned>(i);
    __syncthreads();
    if (threadIdx.x == 0)
        for (int i = 0; i < erase; ++i) {
            const int j = i + static_cast<int>(draw_below(static_cast<uint64_t>(L - i)));
            const unsigned t = scratch[i];
            scratch[i] = scratch[j];
            scratch[j] = t;
        }
    __syncthreads();
    unsigned* gone = scratch + a.L_cap;  // erased flags
    for (int i = threadIdx.x; i < L; i += blockDim.x) gone[i] = 0u;
    __syncthreads();
    for (int i = threadIdx.x; i < erase; i += blockDim.x) gone[scratch[i]] = 1u;
    __syncthreads();
    int keep = 0;
    for (int g = g0; g < g1; ++g) keep += gone[g] == 0u;
    int n_surv = 0;
    int at = block_excl_scan(keep, tmp, n_surv);
    for (int g = g0; g < g1; ++g)
        if (gone[g] == 0u) child[at++] = work[g];
    __syncthreads();
    if (threadIdx.x == 0) a.n_surv[c] = n_surv;
    // residual = completion_of(survivors) (ga.hpp:70)
    completion(M, child, n_surv, cnt, a.residual + static_cast<long long>(c) * M.n);
}

__global__ void __launch_bounds__(kGaThreads) ga_finish_kernel(const __grid_constant__ GaFinishArgs a) {
    const DevModel& M = a.M;
    const int c = blockIdx.x;
    const uint64_t* work = a.work + static_cast<long long>(c) * a.L_cap;
    uint64_t* child = a.child + static_cast<long long>(c) * a.L_cap;
    extern __shared__ __align__(16) unsigned char smem[];
    int* cnt = reinterpret_cast<int*>(smem);
    double* comp = reinterpret_cast<double*>(cnt + ((M.n * kGaMaxSizes + 1) & ~1));
    __shared__ int len, ok;
    __shared__ double slack;
    const int ns = a.n_surv[c];
    const int rn = a.refill_n[c];
    const int wl = a.child_len[c];  // the parent's (= mutated parent's) length, set by the host
    if (threadIdx.x == 0) {
        len = (ns < 0 || rn < 0 || ns + rn > a.L_cap) ? -1 : ns + rn;
        ok = 1;
    }
    __syncthreads();
    if (len >= 0) {
        const uint64_t* rows = a.refill[c];
        for (int i = threadIdx.x; i < rn; i += blockDim.x) child[ns + i] = row_genome(M, rows[i]);
        __syncthreads();
        completion(M, child, len, cnt, comp);
        for (int s = threadIdx.x; s < M.n; s += blockDim.x)
            if (comp[s] < 1.0 - 1e-9) ok = 0;  // evaluate_chromosome: validity (ga.hpp:40-41)
        __syncthreads();
    }
    if (len < 0 || !ok) {  // PlanningError inside crossover: return the parent (ga.hpp:74-76)
        for (int g = threadIdx.x; g < wl; g += blockDim.x) child[g] = work[g];
        __syncthreads();
        if (threadIdx.x == 0) len = wl;
        __syncthreads();
        completion(M, child, len, cnt, comp);
    }
    if (threadIdx.x == 0) {  // slack_of (core.hpp:232-236), service order
        double s = 0.0;
        for (int i = 0; i < M.n; ++i) s = __dadd_rn(s, fmax(0.0, __dadd_rn(comp[i], -1.0)));
        slack = s;
        a.child_len[c] = len;
        a.child_slack[c] = slack;
    }
}

size_t ga_breed_smem_bytes(int n) {
    return static_cast<size_t>(n * kGaMaxSizes + kGaThreads + 1 + kGaThreads * kGaMaxSizes) * sizeof(int);
}
size_t ga_finish_smem_bytes(int n) {
    return static_cast<size_t>(((n * kGaMaxSizes + 1) & ~1)) * sizeof(int) + static_cast<size_t>(n) * sizeof(double) + 16;
}
const void* ga_breed_kernel_ptr() { return reinterpret_cast<const void*>(&ga_breed_kernel); }
const void* ga_finish_kernel_ptr() { return reinterpret_cast<const void*>(&ga_finish_kernel); }
int ga_threads() { return kGaThreads; }

}  // namespace mgb
