// field.cuh -- counter-based synthetic "HPC field" for the sharded configs (SURVEY.md 8d,
// "Generators for large configs": synth::generator is one sequential mt19937_64 stream,
// synthetic.hpp:111, so a 64 GiB input cannot be produced shard by shard with it).
//
// Value x (absolute index) depends on (seed, x) only, so any rank or CTA produces any
// range directly, on the host and on the device with identical integer arithmetic:
//
//   h      = splitmix64 finaliser of (x + (seed + 1) * 0x9E3779B97F4A7C15)
//   noise  = (h % 127) - 63                                  units
//   tri(P, A) = A * t / (P / 2),  t = x mod P folded to [0, P/2]
//   units  = tri(65536, 50000) + tri(1048573, 400000) - 225000 + noise
//   value  = (T)units / 10^dp  (one IEEE division: inverse_scale, numeric.hpp:159-162)
//
// Two triangle waves (a smooth field sampled on a grid) plus small noise: deltas stay
// within a few hundred units, as in the 2-dp sensor walk (ratio ~0.13).
#pragma once
#include <cstdint>

#ifndef FB_HD
#define FB_HD __host__ __device__ __forceinline__
#endif

namespace fb200 {

FB_HD uint64_t field_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

FB_HD int64_t field_tri(uint64_t x, uint64_t period, int64_t amp) {
    const uint64_t half = period / 2;
    const uint64_t r = x % period;
    const uint64_t t = r < half ? r : period - r;
    return amp * (int64_t)t / (int64_t)half;
}

FB_HD int64_t field_units(uint64_t seed, uint64_t x) {
    const uint64_t h = field_mix(x + (seed + 1) * 0x9E3779B97F4A7C15ull);
    const int64_t noise = (int64_t)(h % 127u) - 63;
    return field_tri(x, 65536u, 50000) + field_tri(x, 1048573u, 400000) - 225000 + noise;
}

}  // namespace fb200
