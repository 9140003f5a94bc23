// HBM-bound passes over a dense column-major operator with few right-hand
// sides: x = M^T y (the linear term c = A^T b, path_solver.cpp:295) and the
// fused single-pass Gram product  z = M^T (M w)  (matrix.cpp:168-172) that
// reads every element of M once.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace rpb {

constexpr int kNarrowMax = 16;

// x (d x k, ld d) = A^T y (y: n x k, ld n) for column-major A (n x d, lda),
// k <= kNarrowMax.  One warp per column of A; the per-column reduction order
// is fixed (independent of k), so results are deterministic and column-stable.
void atv_narrow(const double* a, int64_t lda, int64_t n, int64_t d, const double* y, int64_t k, double* x,
                cudaStream_t stream);

// z (d x k) = A^T (A w) for column-major A (n x d) and k <= 8 in ONE pass over
// A: each CTA stages a block of R rows (all d columns) in shared memory,
// forms y_blk = A_blk w, then accumulates A_blk^T y_blk; per-CTA partials are
// reduced in a fixed order.  Returns false if d is too wide for the staging.
bool gram_fused(const double* a, int64_t lda, int64_t n, int64_t d, const double* w, int64_t k, double* z,
                cudaStream_t stream);

}  // namespace rpb
