// keyrank.cu — rank of every base row in the config order (core.hpp:174-200), built on the
// device once per context (lazily, at its first MCTS search): the 128-bit row keys
// (common.cuh row_key), a merge sort of (key, index) pairs, and a scatter.  The MCTS top-Ks
// break their last ties on this rank (mcts.cu precedes_kr).
//
// The sort is this file's own: every CTA bitonic-sorts a 2,048-pair tile in shared memory,
// then log2(P / 2048) merge passes each place every output element directly — a thread
// finds its element's split between the two input runs by a binary search on the co-rank
// (merge path) — ping-ponging between two buffers.  Keys are distinct (every base row is a
// distinct configuration), so no stability rule is needed.
#include "common.cuh"

namespace mgb {

using namespace dev;

namespace {

struct KeyIdx {
    uint64_t hi, lo;
    unsigned idx, pad;
};

__device__ __forceinline__ bool key_less(const KeyIdx& a, const KeyIdx& b) {
    return a.hi != b.hi ? a.hi < b.hi : a.lo < b.lo;
}

constexpr int kTile = 2048;
constexpr int kTileThreads = 1024;

__global__ void keyrank_keys_kernel(const __grid_constant__ DevModel M, const uint64_t* rows, long long P, KeyIdx* out) {
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < P;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        uint64_t hi, lo;
        row_key(M, rows[i], hi, lo);
        out[i] = KeyIdx{hi, lo, static_cast<unsigned>(i), 0u};
    }
}

// One tile of kTile pairs per CTA, sorted ascending in shared memory (bitonic network; the
// tail of the last tile is padded with +infinity keys that sort after every real key).
__global__ void __launch_bounds__(kTileThreads) keyrank_tile_kernel(KeyIdx* v, long long P) {
    __shared__ KeyIdx t[kTile];
    const long long base = static_cast<long long>(blockIdx.x) * kTile;
    for (int i = threadIdx.x; i < kTile; i += blockDim.x)
        t[i] = base + i < P ? v[base + i] : KeyIdx{~0ull, ~0ull, 0xFFFFFFFFu, 0u};
    __syncthreads();
    for (int size = 2; size <= kTile; size <<= 1) {
        for (int j = size >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < kTile; i += blockDim.x) {
                const int p = i ^ j;
                if (p > i) {
                    const bool up = (i & size) == 0;
                    if (key_less(t[p], t[i]) == up) {
                        const KeyIdx x = t[i];
                        t[i] = t[p];
                        t[p] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < kTile; i += blockDim.x)
        if (base + i < P) v[base + i] = t[i];
}

// Merge pass: runs of `run` sorted pairs, merged pairwise into runs of 2 * run.  Output
// element t of a merged pair takes A[i] or B[t - i], where i = the number of A elements
// among the first t outputs (binary search on the merge path).
__global__ void keyrank_merge_kernel(const KeyIdx* in, KeyIdx* out, long long P, long long run) {
    for (long long g = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; g < P;
         g += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long a0 = g / (2 * run) * (2 * run);
        const long long b0 = min(a0 + run, P);
        const long long la = b0 - a0, lb = min(b0 + run, P) - b0;
        const long long t = g - a0;
        const KeyIdx* A = in + a0;
        const KeyIdx* B = in + b0;
        long long lo = max(0ll, t - lb), hi = min(t, la);
        while (lo < hi) {  // smallest i with A[i] > B[t - i - 1]
            const long long mid = (lo + hi) >> 1;
            if (key_less(A[mid], B[t - mid - 1])) lo = mid + 1;
            else hi = mid;
        }
        const long long i = lo, j = t - lo;
        out[g] = (j >= lb || (i < la && key_less(A[i], B[j]))) ? A[i] : B[j];
    }
}

__global__ void keyrank_scatter_kernel(const KeyIdx* sorted, long long P, unsigned* rank) {
    for (long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; r < P;
         r += static_cast<long long>(gridDim.x) * blockDim.x)
        rank[sorted[r].idx] = static_cast<unsigned>(r);
}

}  // namespace

// Scratch bytes build_keyrank needs for P rows (two (key, index) buffers).
size_t keyrank_scratch_bytes(long long P) { return 2 * sizeof(KeyIdx) * static_cast<size_t>(P > 0 ? P : 1) + 256; }

// rank[i] = position of rows[i] in the config order; returns the CUDA status.  Launches the
// key kernel, the tile sort, the merge passes and a scatter on `stream` and synchronizes it.
cudaError_t build_keyrank(const DevModel& M, const uint64_t* rows, long long P, unsigned* rank, void* scratch,
                          size_t scratch_bytes, cudaStream_t stream, int* launches) {
    if (P <= 0) return cudaSuccess;
    if (scratch_bytes < keyrank_scratch_bytes(P)) return cudaErrorInvalidValue;
    KeyIdx* a = static_cast<KeyIdx*>(scratch);
    KeyIdx* b = a + P;
    const unsigned grid = static_cast<unsigned>(std::min<long long>((P + 255) / 256, 4096));
    keyrank_keys_kernel<<<grid, 256, 0, stream>>>(M, rows, P, a);
    const unsigned tiles = static_cast<unsigned>((P + kTile - 1) / kTile);
    keyrank_tile_kernel<<<tiles, kTileThreads, 0, stream>>>(a, P);
    int n = 2;
    for (long long run = kTile; run < P; run *= 2, ++n) {
        keyrank_merge_kernel<<<grid, 256, 0, stream>>>(a, b, P, run);
        std::swap(a, b);
    }
    keyrank_scatter_kernel<<<grid, 256, 0, stream>>>(a, P, rank);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (launches) *launches += n + 1;
    return e;
}

}  // namespace mgb
