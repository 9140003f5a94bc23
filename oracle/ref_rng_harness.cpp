// Test-infrastructure harness around the REFERENCE's own draw code.
//
// Compiled by oracle/Makefile straight from /root/reference/proj/core/include
// (ridgepath/rng.hpp is header-only and needs only <random>/<cmath>; the rest
// of the reference needs Eigen, which is absent, so only the draw contract is
// built from reference sources).  The output goes to oracle/_ref/ and is used
// only by tests/ and tests/golden/make_golden.py to pin oracle/rp_oracle.c.
//
// The draw loops below restate the reference's consumption order:
//   Gaussian    sketch.cpp:94-95 (row-major, scale * normal())
//   Count/SJLT  sketch.cpp:119-124 (per block, per row: uniform_index then sign)
//   SRHT        sketch.cpp:62-79 (signs, then partial Fisher-Yates)
#include <cmath>
#include <cstdint>
#include <numeric>
#include <utility>
#include <vector>

#include "ridgepath/rng.hpp"

using ridgepath::SeededRng;

extern "C" {

void ref_fill_u64(std::uint64_t seed, std::uint64_t skip, std::int64_t count, std::uint64_t* out) {
  SeededRng r(seed);
  for (std::uint64_t i = 0; i < skip; ++i) r.next_u64();
  for (std::int64_t i = 0; i < count; ++i) out[i] = r.next_u64();
}

void ref_fill_uniform01(std::uint64_t seed, std::int64_t count, double* out) {
  SeededRng r(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = r.uniform01();
}

void ref_fill_uniform_index(std::uint64_t seed, std::uint64_t bound, std::int64_t count,
                            std::uint64_t* out) {
  SeededRng r(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = r.uniform_index(bound);
}

void ref_fill_sign(std::uint64_t seed, std::int64_t count, double* out) {
  SeededRng r(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = r.sign();
}

void ref_fill_normals(std::uint64_t seed, std::int64_t count, double scale, double* out) {
  SeededRng r(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = scale * r.normal();
}

void ref_count_draws(std::uint64_t seed, std::int64_t n, std::int64_t rows_per_block, int blocks,
                     double entry, std::int64_t* h, double* sgn) {
  SeededRng r(seed);
  for (int b = 0; b < blocks; ++b)
    for (std::int64_t j = 0; j < n; ++j) {
      h[b * n + j] = static_cast<std::int64_t>(r.uniform_index(static_cast<std::uint64_t>(rows_per_block)));
      sgn[b * n + j] = r.sign() * entry;
    }
}

void ref_srht_draws(std::uint64_t seed, std::int64_t n, std::int64_t m, double* signs,
                    std::int64_t* rows) {
  SeededRng r(seed);
  std::int64_t npad = 1;
  while (npad < n) npad <<= 1;
  for (std::int64_t i = 0; i < n; ++i) signs[i] = r.sign();
  std::vector<std::int64_t> pool(static_cast<std::size_t>(npad));
  std::iota(pool.begin(), pool.end(), std::int64_t{0});
  for (std::int64_t i = 0; i < m; ++i) {
    const std::int64_t j =
        i + static_cast<std::int64_t>(r.uniform_index(static_cast<std::uint64_t>(npad - i)));
    std::swap(pool[i], pool[j]);
    rows[i] = pool[i];
  }
}

}  // extern "C"
