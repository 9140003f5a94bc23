/*
 * rp_oracle.c -- CPU restatement of the reference's draw contract and of the
 * integer/byte-exact parts of the sketch families.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2210_12212_b200/ links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it, as the checker.
 *
 * Every function cites the reference line it restates:
 *   ref = /root/reference/proj/core
 *   - SeededRng                     ref/include/ridgepath/rng.hpp:17-61
 *   - std::mt19937_64               ISO C++ [rand.eng.mers] + [rand.predef] (w=64, n=312, m=156, r=31,
 *                                   a=0xb5026f5aa96619e9, u=29, d=0x5555555555555555, s=17,
 *                                   b=0x71d67fffeda60000, t=37, c=0xfff7eee000000000, l=43,
 *                                   f=6364136223846793005); pinned by the standard's 10000th-output check.
 *   - draw_srht                     ref/src/sketch.cpp:62-79
 *   - fwht_select / apply_srht      ref/src/sketch.cpp:25-48, 138-173
 *   - apply_count_blocks            ref/src/sketch.cpp:114-136
 *   - realize_dense (Gaussian)      ref/src/sketch.cpp:250-262
 *
 * Box-Muller uses the host libm (glibc), exactly as the reference does
 * (std::log / std::sin / std::cos on doubles resolve to the same glibc symbols).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x000000007FFFFFFFULL

typedef struct {
  uint64_t mt[MT_N];
  int mti;
  double cached;
  int have_cached;
} or_rng;

/* std::mt19937_64 seeding: x0 = seed, xi = f*(x_{i-1} ^ (x_{i-1} >> 62)) + i. */
void or_rng_init(or_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = MT_N;
  r->cached = 0.0;
  r->have_cached = 0;
}

static void or_twist(or_rng* r) {
  for (int i = 0; i < MT_N; ++i) {
    const uint64_t y = (r->mt[i] & MT_UM) | (r->mt[(i + 1) % MT_N] & MT_LM);
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
  }
  r->mti = 0;
}

/* SeededRng::next_u64 (rng.hpp:23). */
uint64_t or_next_u64(or_rng* r) {
  if (r->mti >= MT_N) or_twist(r);
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* SeededRng::uniform01 (rng.hpp:26-28): ((x >> 11) + 1) * 2^-53, in (0, 1]. */
double or_uniform01(or_rng* r) {
  return (double)((or_next_u64(r) >> 11) + 1) * 0x1.0p-53;
}

/* SeededRng::uniform_index (rng.hpp:32-37): rejection on x >= n*floor((2^64-1)/n). */
uint64_t or_uniform_index(or_rng* r, uint64_t n) {
  const uint64_t limit = n * (~(uint64_t)0 / n);
  uint64_t x = or_next_u64(r);
  while (x >= limit) x = or_next_u64(r);
  return x % n;
}

/* SeededRng::sign (rng.hpp:40): +1 iff the top bit is set. */
double or_sign(or_rng* r) { return (or_next_u64(r) >> 63) ? 1.0 : -1.0; }

/* SeededRng::normal (rng.hpp:43-55): Box-Muller, cos returned first, sin cached. */
double or_normal(or_rng* r) {
  if (r->have_cached) {
    r->have_cached = 0;
    return r->cached;
  }
  const double u1 = or_uniform01(r);
  const double u2 = or_uniform01(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double two_pi = 6.283185307179586476925286766559;
  r->cached = rad * sin(two_pi * u2);
  r->have_cached = 1;
  return rad * cos(two_pi * u2);
}

/* ---- bulk helpers (used through ctypes) ---------------------------------- */

/* count outputs of next_u64 after discarding `skip` outputs. */
void or_fill_u64(uint64_t seed, uint64_t skip, int64_t count, uint64_t* out) {
  or_rng r;
  or_rng_init(&r, seed);
  for (uint64_t i = 0; i < skip; ++i) or_next_u64(&r);
  for (int64_t i = 0; i < count; ++i) out[i] = or_next_u64(&r);
}

void or_fill_uniform01(uint64_t seed, int64_t count, double* out) {
  or_rng r;
  or_rng_init(&r, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = or_uniform01(&r);
}

void or_fill_uniform_index(uint64_t seed, uint64_t bound, int64_t count, uint64_t* out) {
  or_rng r;
  or_rng_init(&r, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = or_uniform_index(&r, bound);
}

/* out[i] = scale * normal() for i < count: the row-major realization order of
 * random_dense (tests/test_support.hpp:15-21) and of the Gaussian sketch
 * (sketch.cpp:94-95, 257-260). */
void or_fill_normals(uint64_t seed, int64_t count, double scale, double* out) {
  or_rng r;
  or_rng_init(&r, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = scale * or_normal(&r);
}

/* The Gaussian sketch realization for a rectangular window of S:
 * entries (r, j) for r in [r0, r0+rc), j in [j0, j0+jc) of the m x n operator,
 * written row-major into out (rc x jc).  scale = fl(1/fl(sqrt(m))) (sketch.cpp:86). */
void or_gaussian_window(uint64_t seed, int64_t m, int64_t n, int64_t r0, int64_t rc,
                        int64_t j0, int64_t jc, double* out) {
  or_rng r;
  or_rng_init(&r, seed);
  const double scale = 1.0 / sqrt((double)m);
  for (int64_t row = 0; row < r0 + rc; ++row) {
    for (int64_t j = 0; j < n; ++j) {
      const double v = scale * or_normal(&r);
      if (row >= r0 && j >= j0 && j < j0 + jc) out[(row - r0) * jc + (j - j0)] = v;
    }
  }
}

/* CountSketch / SJLT draws (sketch.cpp:119-124): for block b, for row j
 * ascending: h = uniform_index(rows_per_block), sgn = sign() * entry.
 * Outputs are indexed [b*n + j]. */
void or_count_draws(uint64_t seed, int64_t n, int64_t rows_per_block, int blocks,
                    double entry, int64_t* h, double* sgn) {
  or_rng r;
  or_rng_init(&r, seed);
  for (int b = 0; b < blocks; ++b) {
    for (int64_t j = 0; j < n; ++j) {
      h[(int64_t)b * n + j] = (int64_t)or_uniform_index(&r, (uint64_t)rows_per_block);
      sgn[(int64_t)b * n + j] = or_sign(&r) * entry;
    }
  }
}

/* apply_count_blocks, dense A (column-major n x d, leading dim lda) ->
 * out (column-major m x d), sketch.cpp:126-128.  Accumulation per output row
 * runs over j ascending, exactly as the reference loop. */
void or_count_apply_dense(uint64_t seed, int64_t m, int64_t n, int64_t d, int blocks,
                          double entry, const double* a, int64_t lda, double* out) {
  or_rng r;
  or_rng_init(&r, seed);
  const int64_t rpb = m / blocks;
  memset(out, 0, sizeof(double) * (size_t)(m * d));
  for (int b = 0; b < blocks; ++b) {
    const int64_t base = (int64_t)b * rpb;
    for (int64_t j = 0; j < n; ++j) {
      const int64_t hh = (int64_t)or_uniform_index(&r, (uint64_t)rpb);
      const double s = or_sign(&r) * entry;
      for (int64_t c = 0; c < d; ++c) out[c * m + base + hh] += s * a[c * lda + j];
    }
  }
}

/* apply_count_blocks, CSR A (sketch.cpp:129-133). */
void or_count_apply_csr(uint64_t seed, int64_t m, int64_t n, int64_t d, int blocks,
                        double entry, const int64_t* off, const int64_t* cols,
                        const double* vals, double* out) {
  or_rng r;
  or_rng_init(&r, seed);
  const int64_t rpb = m / blocks;
  memset(out, 0, sizeof(double) * (size_t)(m * d));
  for (int b = 0; b < blocks; ++b) {
    const int64_t base = (int64_t)b * rpb;
    for (int64_t j = 0; j < n; ++j) {
      const int64_t hh = (int64_t)or_uniform_index(&r, (uint64_t)rpb);
      const double s = or_sign(&r) * entry;
      for (int64_t p = off[j]; p < off[j + 1]; ++p) out[cols[p] * m + base + hh] += s * vals[p];
    }
  }
}

/* ---- SRHT ------------------------------------------------------------------ */

int64_t or_hadamard_pad(int64_t n) {
  uint64_t v = (uint64_t)(n < 1 ? 1 : n);
  uint64_t p = 1;
  while (p < v) p <<= 1;
  return (int64_t)p;
}

/* draw_srht (sketch.cpp:62-79): n signs in row order, then m partial
 * Fisher-Yates picks over [0, npad), kept in draw order.  The pool is the
 * identity permutation materialized lazily. */
void or_srht_draws(uint64_t seed, int64_t n, int64_t m, double* signs, int64_t* rows) {
  or_rng r;
  or_rng_init(&r, seed);
  const int64_t npad = or_hadamard_pad(n);
  for (int64_t i = 0; i < n; ++i) signs[i] = or_sign(&r);
  int64_t* pool = (int64_t*)malloc(sizeof(int64_t) * (size_t)npad);
  for (int64_t i = 0; i < npad; ++i) pool[i] = i;
  for (int64_t i = 0; i < m; ++i) {
    const int64_t j = i + (int64_t)or_uniform_index(&r, (uint64_t)(npad - i));
    const int64_t t = pool[i];
    pool[i] = pool[j];
    pool[j] = t;
    rows[i] = pool[i];
  }
  free(pool);
}

typedef struct {
  int64_t first;  /* output index in [0, npad) */
  int64_t second; /* slot in [0, m) */
} or_pair;

static int or_pair_cmp(const void* x, const void* y) {
  const or_pair* a = (const or_pair*)x;
  const or_pair* b = (const or_pair*)y;
  if (a->first != b->first) return a->first < b->first ? -1 : 1;
  if (a->second != b->second) return a->second < b->second ? -1 : 1;
  return 0;
}

/* fwht_select (sketch.cpp:25-48): butterfly at stride len/2 first, then
 * recurse into the halves that contain a requested output. */
static void or_fwht_select(double* x, int64_t len, const or_pair* tb, const or_pair* te,
                           int64_t base, double scale, double* out) {
  if (tb == te) return;
  if (len == 1) {
    for (const or_pair* t = tb; t != te; ++t) out[t->second] = x[0] * scale;
    return;
  }
  const int64_t h = len / 2;
  for (int64_t i = 0; i < h; ++i) {
    const double a = x[i];
    const double b = x[i + h];
    x[i] = a + b;
    x[i + h] = a - b;
  }
  const int64_t mid = base + h;
  const or_pair* split = tb;
  while (split != te && split->first < mid) ++split;
  or_fwht_select(x, h, tb, split, base, scale, out);
  or_fwht_select(x + h, h, split, te, mid, scale, out);
}

/* apply_srht (sketch.cpp:138-173) for dense column-major A or CSR A.
 * If offs != NULL the CSR arrays are used (column gather through the CSR
 * transpose: stored entries get sign*value, every other slot stays +0.0). */
void or_srht_apply(uint64_t seed, int64_t m, int64_t n, int64_t d, const double* a, int64_t lda,
                   const int64_t* off, const int64_t* cols, const double* vals, double* out) {
  const int64_t npad = or_hadamard_pad(n);
  double* signs = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)m);
  or_srht_draws(seed, n, m, signs, rows);
  const double scale = 1.0 / sqrt((double)m);
  or_pair* targets = (or_pair*)malloc(sizeof(or_pair) * (size_t)m);
  for (int64_t r = 0; r < m; ++r) {
    targets[r].first = rows[r];
    targets[r].second = r;
  }
  qsort(targets, (size_t)m, sizeof(or_pair), or_pair_cmp);
  double* col = (double*)malloc(sizeof(double) * (size_t)npad);
  for (int64_t c = 0; c < d; ++c) {
    for (int64_t i = 0; i < npad; ++i) col[i] = 0.0;
    if (!off) {
      for (int64_t i = 0; i < n; ++i) col[i] = signs[i] * a[c * lda + i];
    } else {
      for (int64_t r = 0; r < n; ++r)
        for (int64_t p = off[r]; p < off[r + 1]; ++p)
          if (cols[p] == c) col[r] = signs[r] * vals[p];
    }
    or_fwht_select(col, npad, targets, targets + m, 0, scale, out + c * m);
  }
  free(col);
  free(targets);
  free(rows);
  free(signs);
}
