// Elementwise / gather kernels of the binomial-basis recursion
// (path_solver.cpp:27-53), the Horner composition (path_solver.cpp:64-74) and
// the sparse Gram pieces (matrix.cpp:140-166).
//
// Layouts.  NB = L*K independent recursions ("problems") b = l*K + r for
// interval l and right-hand side r.  gen / tilde are dim x (kmax*NB)
// column-major with column j*NB + b = basis term j of problem b, so that the
// first g*NB columns are exactly the block W = gen[:, :g] of every problem and
// one Gram product serves all of them.  The preconditioner works on the
// interval-major layout im[l] = dim x (kmax*K) with column j*K + r.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "gemm_f64.h"

namespace rpb {

struct BasisDims {
  int64_t dim = 0;
  int64_t L = 0;     // intervals in this batch
  int64_t K = 0;     // right-hand sides
  int64_t kmax = 0;  // max budget over the intervals
  int64_t nb() const { return L * K; }
};

// args_im[l][:, j*K + r] = tau_l * Y[:, j*NB + b] + (j >= 1 ? gen[:, (j-1)*NB + b] : 0) for j < g
// args_im[l][:, g*K + r] = gen[:, (g-1)*NB + b]
// y is the Gram product (possibly as deferred split-K partials).
void build_args(const BasisDims& d, int64_t g, const Partials& y, const double* gen, const double* d_tau,
                double* args_im, cudaStream_t stream);

// args_im[l][:, K + r] = gen[:, b] (the generation-1 argument column; the
// fused recursion epilogue writes the later ones, see gemm_f64.h).
void seed_args(const BasisDims& d, const double* gen, double* args_im, cudaStream_t stream);
// args_im[l][:, (g+1)*K + r] = gen[:, g*NB + b] (next generation's last argument
// column; what the fused update epilogue writes).
void seed_next_args(const BasisDims& d, int64_t g, const double* gen, double* args_im, cudaStream_t stream);

// gen[:, j*NB+b] -= applied[l][:, j*K+r] (j < g); gen[:, g*NB+b] = -applied[l][:, g*K+r];
// flags[l] |= any non-finite in gen[:, 0..g]; tilde[:, j*NB+b] += gen[:, j*NB+b] (j <= g).
// Problems whose interval has k_l <= g are left untouched.
// applied: batch l = interval, column j*K + r (possibly deferred partials).
void update_gen(const BasisDims& d, int64_t g, const Partials& applied, const int* d_k, double* gen, double* tilde,
                int* d_flags, cudaStream_t stream);

// x[:, t*K + r] = tau_l * Horner(tilde of problem l*K + r, tau_l * lambda_t) for t < T,
// where l = d_interval[t].  Reference: compose_horner, path_solver.cpp:64-74.
void compose(const BasisDims& d, const double* tilde, const double* d_tau, const int* d_k, const double* d_lambda,
             const int* d_interval, int64_t T, double* x, cudaStream_t stream);

// Composition as a product (north_star 6): for interval l with cnt[l] grid
// points starting at position off[l] of d_lambda, the k x tmax coefficient
// block  coef[l][j + c*kmax] = tau_l (tau_l lambda_{off[l]+c})^j  (j < k_l,
// c < cnt[l]; zero elsewhere), so that  x(lambda) = U_l coef[l]  with U_l the
// interval's dim x kmax basis.  compose_gather copies the cnt[l]*K columns of
// each interval's padded dim x (tmax*K) result block to x[:, (off[l]+c)*K + r].
void compose_coeffs(const BasisDims& d, const double* d_tau, const int* d_k, const double* d_lambda, const int* d_off,
                    const int* d_cnt, int64_t tmax, double* coef, cudaStream_t stream);
void compose_gather(const BasisDims& d, const double* xpad, const int* d_off, const int* d_cnt, int64_t tmax, double* x,
                    cudaStream_t stream);

// out_l = (args_l - t3_l) / lambda0_l for l < L (Woodbury preconditioner tail);
// each operand is dim x cols contiguous per interval at its own interval
// stride (s_args = 0 broadcasts one input).
void woodbury_tail(int64_t dim, int64_t cols, int64_t L, int64_t s_args, const double* args, int64_t s_t3,
                   const double* t3, const double* d_lambda0, int64_t s_out, double* out, cudaStream_t stream);

// Feature-sharded Woodbury tail: rows [f0, f0 + rows) of out_l = (args_l -
// t3_l) / lambda0_l, written into this rank's pack block (ld blk, column
// l*cols + c) for the all-gather.  args: interval stride s_args (0 =
// broadcast), ld `ld_args`; t3: rows x (L*cols), ld rows.
void woodbury_tail_rows(int64_t f0, int64_t rows, int64_t cols, int64_t L, const double* args, int64_t ld_args,
                        int64_t s_args, const double* t3, const double* d_lambda0, double* pack, int64_t blk,
                        cudaStream_t stream);
// Unpack an all-gathered row-block matrix: recv holds world blocks of
// blk x N (ld blk), block r = rows [r*blk, min(dim, (r+1)*blk)); column
// j = l*cols + c goes to out[l*s_out + c*dim + row].
void gather_row_blocks(const double* recv, int64_t blk, int64_t dim, int64_t cols, int64_t L, double* out,
                       int64_t s_out, cudaStream_t stream);

// Loss pieces (path_solver.cpp:425-454).  For output column j of R
// (rows x cols, ld ldr): out[j] = sum_r (R[r, j] - B[r, j % K])^2 (B may be
// null: plain sum of squares), summed over rows in a fixed order.
void column_sq_norms(const double* r, int64_t rows, int64_t cols, int64_t ldr, const double* b, int64_t K,
                     int64_t ldb, double* out, cudaStream_t stream);
// loss[t] = 0.5 * sum_k rn[t K + k] + 0.5 * lambda[t] * sum_k xn[t K + k]  (lambda/xn may be null)
void combine_losses(const double* rn, const double* xn, const double* lambda, int64_t T, int64_t K, double* loss,
                    cudaStream_t stream);

// Row-major helpers for the CSR Gram.
void transpose(const double* in, int64_t rows, int64_t cols, int64_t ldi, double* out, int64_t ldo,
               cudaStream_t stream);  // out (cols x rows, col-major) = in^T (in: rows x cols col-major)
// y_rm (n x c, row-major) = CSR(M) * x_rm (D x c, row-major): per row, entries in stored order.
void spmm_csr_rm(const int64_t* off, const int32_t* col, const double* val, int64_t n, int64_t c, const double* x_rm,
                 double* y_rm, cudaStream_t stream);

// Scale-and-copy helpers.
void copy_cols(const double* src, int64_t rows, int64_t cols, int64_t lds, double* dst, int64_t ldd,
               cudaStream_t stream);
void fill(double* dst, int64_t count, double v, cudaStream_t stream);

}  // namespace rpb
