// philox.cuh — Philox4x32-10 counter-based RNG, identical on host and device.
//
// The throughput-mode searches (root-parallel rollouts, rollout.cu) draw from a stateless
// stream keyed by the seed: draw t of stream (rollout) r is philox(key = seed,
// counter = (t, r)).  Any thread can produce any draw without sequencing, which is what a
// warp-per-rollout kernel needs; the reference's std::mt19937_64 (util.hpp:27) is a single
// sequential stream and stays the RNG of the parity-mode drivers (search.cpp).
// Constants and round function: Salmon et al., "Parallel random numbers: as easy as
// 1, 2, 3" (SC'11), Philox4x32 with 10 rounds.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define MGB_HD __host__ __device__ __forceinline__
#else
#define MGB_HD inline
#endif

namespace mgb {

struct Philox4 {
    uint32_t v[4];
};

MGB_HD Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
    constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = static_cast<uint64_t>(M0) * c0;
        const uint64_t p1 = static_cast<uint64_t>(M1) * c2;
        const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
        const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += W0;
        k1 += W1;
    }
    return Philox4{{c0, c1, c2, c3}};
}

// 64-bit draw `step` of stream `stream` under `seed`.
MGB_HD uint64_t philox_u64(uint64_t seed, uint64_t stream, uint64_t step) {
    const Philox4 r = philox4x32_10(static_cast<uint32_t>(step), static_cast<uint32_t>(step >> 32),
                                    static_cast<uint32_t>(stream), static_cast<uint32_t>(stream >> 32),
                                    static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
    return (static_cast<uint64_t>(r.v[1]) << 32) | r.v[0];
}

// floor(x * n / 2^64): an index in [0, n) from a uniform 64-bit draw.
MGB_HD uint64_t philox_below(uint64_t x, uint64_t n) {
#ifdef __CUDA_ARCH__
    return __umul64hi(x, n);
#else
    return static_cast<uint64_t>((static_cast<unsigned __int128>(x) * n) >> 64);
#endif
}

}  // namespace mgb
