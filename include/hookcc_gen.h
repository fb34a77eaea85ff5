// Counter-based graph generators shared by the device kernels and the host
// library (one definition, compiled for both sides).
//
// The reference generators (proj/include/hookcc/generators.hpp:14-87) draw
// from one sequential std::mt19937_64 stream: RMAT-24 takes 137 s and
// RMAT-28 about 40 min on one core, and they cannot be split across
// threads.  The "rmatx"/"erx" twins keep the same models — per-level
// quadrant choice with probabilities (a, b, c, d) applied un-perturbed and
// ids unpermuted (generators.hpp:28-62); endpoints uniform with replacement
// (generators.hpp:14-26) — but draw each random word from a counter
// (splitmix64 of seed and position), so edge i depends only on (seed, i)
// and any range can be generated in parallel.  oracle/hookcc_oracle.c
// restates them independently (this header is shared by the device kernels
// and the host C++ API) for the bit-exact parity tests.
//
//   word(key, c)  = mix64(key + (c + 1) * 0x9E3779B97F4A7C15)
//   key           = mix64(seed ^ 0x5851F42D4C957F2D)
//   rmatx edge i  : level l (MSB first) uses the 32-bit half (l & 1) of
//                   word(key, i * 16 + l / 2); p < ta -> (0,0),
//                   p < tab -> (0,1), p < tabc -> (1,0), else (1,1);
//                   thresholds are floor(x * 2^32) of the cumulative sums.
//   erx edge i    : w = word(key, i); u = lo32(w) * n >> 32,
//                   v = hi32(w) * n >> 32.
//   grid          : identical to generators.hpp:71-87 (row edges, then
//                   column edges).
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define HCC_HD __host__ __device__ __forceinline__
#else
#define HCC_HD inline
#endif

namespace hcc {

HCC_HD uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

HCC_HD uint64_t gen_key(uint64_t seed) {
  return mix64(seed ^ 0x5851F42D4C957F2Dull);
}

HCC_HD uint64_t gen_word(uint64_t key, uint64_t ctr) {
  return mix64(key + (ctr + 1) * 0x9E3779B97F4A7C15ull);
}

HCC_HD void rmatx_edge(uint64_t key, uint64_t i, uint32_t scale, uint32_t ta,
                       uint32_t tab, uint32_t tabc, uint32_t* u_out,
                       uint32_t* v_out) {
  uint32_t u = 0, v = 0;
  uint64_t w = 0;
  for (uint32_t l = 0; l < scale; ++l) {
    if ((l & 1u) == 0) w = gen_word(key, i * 16ull + (l >> 1));
    uint32_t p = (l & 1u) ? (uint32_t)(w >> 32) : (uint32_t)w;
    u <<= 1;
    v <<= 1;
    if (p < ta) {
    } else if (p < tab) {
      v |= 1u;
    } else if (p < tabc) {
      u |= 1u;
    } else {
      u |= 1u;
      v |= 1u;
    }
  }
  *u_out = u;
  *v_out = v;
}

HCC_HD void erx_edge(uint64_t key, uint64_t i, uint64_t n, uint32_t* u_out,
                     uint32_t* v_out) {
  uint64_t w = gen_word(key, i);
  *u_out = (uint32_t)(((w & 0xffffffffull) * n) >> 32);
  *v_out = (uint32_t)(((w >> 32) * n) >> 32);
}

HCC_HD void grid_edge(uint64_t rows, uint64_t cols, uint64_t i,
                      uint32_t* u_out, uint32_t* v_out) {
  const uint64_t row_edges = rows * (cols - 1);
  if (i < row_edges) {
    uint64_t r = i / (cols - 1), c = i % (cols - 1);
    uint64_t id = r * cols + c;
    *u_out = (uint32_t)id;
    *v_out = (uint32_t)(id + 1);
  } else {
    uint64_t j = i - row_edges;
    uint64_t r = j / cols, c = j % cols;
    uint64_t id = r * cols + c;
    *u_out = (uint32_t)id;
    *v_out = (uint32_t)(id + cols);
  }
}

// Position-keyed checksum term; the checksum of an edge stream is the
// wrapping sum of these over i (order-dependent, parallel-friendly).
HCC_HD uint64_t checksum_term(uint64_t i, uint32_t u, uint32_t v) {
  return mix64((i * 0x9E3779B97F4A7C15ull) ^
               (((uint64_t)u << 32) | (uint64_t)v));
}

// floor(x * 2^32) clamped to [0, 2^32 - 1]; x is a cumulative probability.
inline uint32_t prob_threshold(double x) {
  if (!(x > 0.0)) return 0u;
  if (x >= 1.0) return 0xffffffffu;
  double t = x * 4294967296.0;
  if (t >= 4294967295.0) return 0xffffffffu;
  return (uint32_t)t;
}

}  // namespace hcc
