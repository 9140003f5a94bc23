// d-vector kernels of the iterative baselines (warm CG / warm IHS,
// ref/proj/core/src/baselines.cpp:120-224) and the spectral sums
// (spectrum.cu).  Element-wise arithmetic follows the reference's Eigen
// expressions operation by operation (no FMA contraction); dot products use a
// fixed two-stage reduction, so every result is deterministic.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace rpb {

constexpr int kDotParts = 296;  // partial sums of vec_dot (fixed: order never depends on the device)

// *out = x . y  (device scalar); part holds kDotParts doubles of scratch.
void vec_dot(const double* x, const double* y, int64_t n, double* part, double* out, cudaStream_t s);

// grad = (g + lam * x) - atb           (gram_apply(a, x) + lambda * x - atb, baselines.cpp:196)
void ihs_grad(const double* g, const double* x, double lam, const double* atb, int64_t n, double* grad,
              cudaStream_t s);
// xs = xs - tau * pg; *flag = 1 if any entry is non-finite (baselines.cpp:200-202)
void ihs_step(double* xs, const double* pg, double tau, int64_t n, int* flag, cudaStream_t s);
// r = (atb - g) - lam * x; p = r      (baselines.cpp:140-141)
void cg_init(const double* atb, const double* g, const double* x, double lam, int64_t n, double* r, double* p,
             cudaStream_t s);
// q = g + lam * p                      (baselines.cpp:147)
void cg_q(const double* g, const double* p, double lam, int64_t n, double* q, cudaStream_t s);
// alpha = *rr / *pq; x += alpha p; r -= alpha q   (baselines.cpp:148-150)
void cg_update(double* x, double* r, const double* p, const double* q, const double* rr, const double* pq, int64_t n,
               cudaStream_t s);
// p = r + (*rr_next / *rr) p           (baselines.cpp:152)
void cg_direction(double* p, const double* r, const double* rr_next, const double* rr, int64_t n, cudaStream_t s);

// dst = src, src a device-mapped (pinned) host buffer read over PCIe by the kernel
void copy_mapped(const double* src, int64_t n, double* dst, cudaStream_t s);
// r = r - b  (the residual apply(a, x) - b, adaptive.cpp:64-66)
void residual_in_place(double* r, const double* b, int64_t n, cudaStream_t s);
// g[i + j ld] = g[j + i ld] for i < j (copy the lower triangle onto the upper)
void mirror_lower(double* g, int64_t n, int64_t ld, cudaStream_t s);
// out (d x cols, ld d) = columns c0 .. c0+cols-1 of the d x d identity.
void identity_block(double* out, int64_t d, int64_t cols, int64_t c0, cudaStream_t s);
// out (r x r, ld r) = upper triangle of a (r x r block at a, ld lda), zeros below.
void upper_triangle(const double* a, int64_t lda, int64_t r, double* out, cudaStream_t s);
// svd_path's diagonal solve (baselines.cpp:66-68): z[i, t] = (sigma_i utb_i) / (sigma_i^2 + lambda_t),
// z is r x T (ld r); no contraction, the reference's operation order.
void svd_scale(const double* sigma, const double* utb, int64_t r, const double* lambda, int64_t T, double* z,
               cudaStream_t s);

}  // namespace rpb
