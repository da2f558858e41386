// synth.cuh — the SURVEY §8d synthetic workload generator on the device.
//
// Integer-exact twin of oracle/lookup_oracle.cpp's generator (the oracle is
// the checker; tests compare both bit-for-bit). The hash is the reference's
// splitmix64 finalizer mix64 (rng.hpp:13-19).
#pragma once

#include <cstdint>

namespace sp {

constexpr uint64_t kTagLen = 0x6c656e5f62616773ULL;  // "len_bags"
constexpr uint64_t kTagIdx = 0x6964785f726f7773ULL;  // "idx_rows"
constexpr uint64_t kTagW = 0x77656967687473ULL;      // "weights"
constexpr uint64_t kTagG = 0x6772616469656e74ULL;    // "gradient"

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t h3(uint64_t seed, uint64_t tag,
                                                uint64_t a, uint64_t b) {
  return mix64(mix64(mix64(seed ^ tag) ^ a) ^ b);
}

// Threshold on the low 32 hash bits for "hot" draws (probability hot_mass).
__host__ __device__ __forceinline__ uint64_t hot_threshold(double hot_mass) {
  if (!(hot_mass > 0.0)) return 0;
  if (hot_mass >= 1.0) return 1ULL << 32;
  return static_cast<uint64_t>(hot_mass * 4294967296.0);
}

// Bag length: uniform integer in [0, lmax], lmax = floor(2 pf).
__host__ __device__ __forceinline__ int64_t bag_len(uint64_t seed, int32_t t,
                                                    int64_t b, int64_t lmax) {
  if (lmax <= 0) return 0;
  const uint64_t h = h3(seed, kTagLen, static_cast<uint64_t>(t),
                        static_cast<uint64_t>(b));
  return static_cast<int64_t>(h % static_cast<uint64_t>(lmax + 1));
}

// Row of draw j of bag (t, b); `base` = h3(seed, kTagIdx, t, b).
__host__ __device__ __forceinline__ int64_t bag_index(uint64_t base, int64_t j,
                                                      int64_t rows,
                                                      uint64_t thr) {
  const uint64_t h = mix64(base ^ static_cast<uint64_t>(j));
  const uint64_t lo = h & 0xffffffffULL;
  const uint64_t hi = h >> 32;
  if (lo < thr) {
    const uint64_t k = hi & 1023ULL;
    if (rows <= 1024) return static_cast<int64_t>(k % static_cast<uint64_t>(rows));
    return static_cast<int64_t>(k * static_cast<uint64_t>(rows / 1024));
  }
  return static_cast<int64_t>(hi % static_cast<uint64_t>(rows));
}

// w = 0.5 + 0.5 u, u = k 2^-23 (exact in fp32); `base` = h3(seed,kTagW,t,row).
__host__ __device__ __forceinline__ float weight_from_base(uint64_t base,
                                                           int32_t col) {
  const uint64_t h = mix64(base ^ static_cast<uint64_t>(col));
  return 0.5f + static_cast<float>(h >> 41) * 0x1.0p-24f;
}

// dL/dpooled in [-1, 1): k 2^-23 - 1 (exact in fp32).
__host__ __device__ __forceinline__ float grad_value(uint64_t seed, int64_t bag,
                                                     int64_t gcol) {
  const uint64_t h = h3(seed, kTagG, static_cast<uint64_t>(bag),
                        static_cast<uint64_t>(gcol));
  return static_cast<float>(h >> 40) * 0x1.0p-23f - 1.0f;
}

}  // namespace sp
