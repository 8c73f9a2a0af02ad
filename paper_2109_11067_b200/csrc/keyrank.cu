// keyrank.cu — rank of every base row in the config order (core.hpp:174-200), built on the
// device: the 128-bit row keys (common.cuh row_key), one radix sort of (key, index) pairs,
// and a scatter.  The MCTS top-Ks break their last ties on this rank (mcts.cu precedes_kr).
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace mgb {

using namespace dev;

namespace {

struct Key128 {
    uint64_t hi, lo;
};
struct Key128Decomposer {  // most significant first
    __host__ __device__ ::cuda::std::tuple<uint64_t&, uint64_t&> operator()(Key128& k) const { return {k.hi, k.lo}; }
};

__global__ void keyrank_keys_kernel(const __grid_constant__ DevModel M, const uint64_t* rows, long long P, Key128* keys,
                                    unsigned* idx) {
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < P;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        uint64_t hi, lo;
        row_key(M, rows[i], hi, lo);
        keys[i] = Key128{hi, lo};
        idx[i] = static_cast<unsigned>(i);
    }
}

__global__ void keyrank_scatter_kernel(const unsigned* sorted_idx, long long P, unsigned* rank) {
    for (long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; r < P;
         r += static_cast<long long>(gridDim.x) * blockDim.x)
        rank[sorted_idx[r]] = static_cast<unsigned>(r);
}

}  // namespace

// Scratch bytes build_keyrank needs for P rows (keys and indices double-buffered + the sort).
size_t keyrank_scratch_bytes(long long P) {
    if (P <= 0) return 256;
    size_t tmp_bytes = 0;
    Key128 *k = nullptr;
    unsigned* i = nullptr;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k, k, i, i, P, Key128Decomposer{}, 0, 128);
    const size_t kb = sizeof(Key128) * static_cast<size_t>(P), ib = sizeof(unsigned) * static_cast<size_t>(P);
    return ((2 * kb + 2 * ib + 255) & ~size_t(255)) + tmp_bytes + 256;
}

// rank[i] = position of rows[i] in the config order; returns the CUDA status.  Launches the
// key kernel, the radix sort and a scatter on `stream` and synchronizes it.
cudaError_t build_keyrank(const DevModel& M, const uint64_t* rows, long long P, unsigned* rank, void* scratch,
                          size_t scratch_bytes, cudaStream_t stream, int* launches) {
    if (P <= 0) return cudaSuccess;
    const size_t kb = sizeof(Key128) * static_cast<size_t>(P), ib = sizeof(unsigned) * static_cast<size_t>(P);
    unsigned char* mem = static_cast<unsigned char*>(scratch);
    Key128* kin = reinterpret_cast<Key128*>(mem);
    Key128* kout = reinterpret_cast<Key128*>(mem + kb);
    unsigned* iin = reinterpret_cast<unsigned*>(mem + 2 * kb);
    unsigned* iout = reinterpret_cast<unsigned*>(mem + 2 * kb + ib);
    void* tmp = mem + ((2 * kb + 2 * ib + 255) & ~size_t(255));
    size_t tmp_bytes = scratch_bytes - ((2 * kb + 2 * ib + 255) & ~size_t(255));
    const unsigned grid = static_cast<unsigned>(std::min<long long>((P + 255) / 256, 4096));
    keyrank_keys_kernel<<<grid, 256, 0, stream>>>(M, rows, P, kin, iin);
    cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kin, kout, iin, iout, P, Key128Decomposer{}, 0,
                                                    128, stream);
    if (e == cudaSuccess) {
        keyrank_scatter_kernel<<<grid, 256, 0, stream>>>(iout, P, rank);
        e = cudaStreamSynchronize(stream);
    }
    if (launches) *launches += 4;  // keys, the sort's passes (counted as 2), scatter
    return e;
}

}  // namespace mgb
