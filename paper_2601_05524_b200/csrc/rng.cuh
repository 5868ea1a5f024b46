// The reference's deterministic RNG on the device: specpar::Rng is std::mt19937_64 (rng.hpp:19-30),
// uniform() takes the top 53 bits of one word (rng.hpp:23), derive_rng seeds from splitmix64 of the
// (seed, round, lane) triple (rng.hpp:8-13, 33-35).  Shared by the verifier entry points (verify.cu)
// and the sampled decode loop (sampling.cu); every draw is bit-identical to the reference's.
#pragma once
#include <cstdint>

#include "verify.cuh"

namespace dbl {

__host__ __device__ inline void mt_seed(DevRng& g, uint64_t seed) {
    g.mt[0] = seed;
    for (int i = 1; i < 312; ++i) g.mt[i] = 6364136223846793005ULL * (g.mt[i - 1] ^ (g.mt[i - 1] >> 62)) + i;
    g.idx = 312;
}

__device__ inline uint64_t mt_next(DevRng& g) {
    if (g.idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (g.mt[i] & 0xFFFFFFFF80000000ULL) | (g.mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g.mt[i] = g.mt[(i + 156) % 312] ^ xa;
        }
        g.idx = 0;
    }
    uint64_t y = g.mt[g.idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

__device__ inline double mt_uniform(DevRng& g) { return static_cast<double>(mt_next(g) >> 11) * 0x1.0p-53; }

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d49bb133111ebULL;
    return x ^ (x >> 31);
}

// derive_rng's seed (rng.hpp:33-35)
__host__ __device__ inline uint64_t derived_seed(uint64_t seed, uint64_t round, uint64_t lane) {
    return splitmix64(seed ^ splitmix64(round * 4 + lane + 1));
}

}  // namespace dbl
