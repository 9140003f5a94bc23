// Batched SPD inverse on the FP64 tensor cores: blocked Cholesky (potrf),
// triangular inverse (trtri) and P = L^{-T} L^{-1}.
//
// Replaces the reference's thin_svd + Preconditioner weights
// (matrix.cpp:213-234, preconditioner.cpp:12-65): (SA^T SA + l0 I)^{-1} and
// (l0 I + SA SA^T)^{-1} are formed explicitly per interval shift, so that the
// per-generation preconditioner application is one batched DMMA GEMM.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace rpb {

// For b < batch: H_b (n x n, column-major, leading dim ld, stride `stride`;
// lower triangle read, strict upper triangle must be zero) is overwritten
// (scratch); out_b = H_b^{-1} (full symmetric).  Throws FactorFailure if some
// H_b is not numerically positive definite.
// chain_high_priority: the critical chain's stream (diagonal kernels, panel
// solves) is created at the device's highest stream priority, so its CTAs
// are placed ahead of the trailing updates' and of any overlapped work.
void spd_inverse_batched(double* h, int64_t n, int64_t ld, int64_t stride, int64_t batch, double* out,
                         int64_t ldo, int64_t stride_o, cudaStream_t stream, bool chain_high_priority = false);

// H_b = lower(G) + shift_b * I for b < batch (G shared, n x n), strict upper
// triangle zero -- the input spd_inverse_batched expects.
void shifted_copies(const double* g, int64_t n, const double* d_shifts, int64_t batch, double* h, cudaStream_t stream);

}  // namespace rpb
