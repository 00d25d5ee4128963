// Counter-based RNG, bit-identical to the reference's rng.hpp:37-89 (host and
// device): every draw is a pure function of (seed, purpose, indices).
#pragma once

#include <cmath>
#include <cstdint>
#include <string>

namespace mglp {

enum RngPurpose : uint64_t { kRngInit = 1, kRngData = 2, kRngDropout = 3, kRngTestOnly = 6 };

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
__host__ __device__ inline uint64_t derive(uint64_t seed, uint64_t a, uint64_t b, uint64_t c,
                                           uint64_t d) {
  uint64_t s = splitmix64(seed ^ 0x243f6a8885a308d3ULL);
  s = splitmix64(s ^ a);
  s = splitmix64(s ^ b);
  s = splitmix64(s ^ c);
  s = splitmix64(s ^ d);
  return s;
}
// uniform integer in [0, n): multiply-shift, the high 64 bits of bits * n
// (rng.hpp:68-72, unsigned __int128 on the host, __umul64hi on the device)
__host__ __device__ inline uint64_t uniform_index(uint64_t bits, uint64_t n) {
#ifdef __CUDA_ARCH__
  return __umul64hi(bits, n);
#else
  return (uint64_t)(((unsigned __int128)bits * n) >> 64);
#endif
}
inline double u01(uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }
inline double gaussian(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  const uint64_t k1 = derive(seed, a, b, c, d);
  const uint64_t k2 = splitmix64(k1 ^ 0x452821e638d01377ULL);
  double x1 = u01(k1);
  const double x2 = u01(k2);
  if (x1 <= 0.0) x1 = 0x1.0p-53;
  return std::sqrt(-2.0 * std::log(x1)) * std::cos(6.283185307179586 * x2);
}
inline double truncated_gaussian(double stddev, uint64_t seed, uint64_t a, uint64_t b,
                                 uint64_t c) {
  for (uint64_t attempt = 0;; ++attempt) {
    const double g = gaussian(seed, a, b, c, attempt);
    if (g >= -2.0 && g <= 2.0) return g * stddev;
  }
}
inline uint64_t fnv1a(const std::string& s) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (char ch : s) {
    h ^= static_cast<unsigned char>(ch);
    h *= 0x100000001b3ULL;
  }
  return h;
}

}  // namespace mglp
