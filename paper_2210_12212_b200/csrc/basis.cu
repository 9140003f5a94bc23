// Recursion epilogues, Horner composition and sparse Gram helpers.
#include <algorithm>

#include "basis.h"
#include "common.h"

namespace rpb {
namespace {

unsigned grid_for(int64_t work, int threads = 256) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, threads), 148 * 32)));
}

__device__ __forceinline__ double sum_partials(const Partials& P, int64_t b, int64_t i, int64_t j) {
  const double* q = P.p + b * P.batch_stride + i + j * P.ld;
  double v = q[0];
  for (int s = 1; s < P.split; ++s) v += q[s * P.split_stride];
  return v;
}

// Column-indexed grids: blockIdx.y = output column, threads over rows, so the
// column bookkeeping (j, b, l, r) is done once per block, not per element.
__global__ void build_args_kernel(BasisDims d, int64_t g, Partials y, const double* __restrict__ gen,
                                  const double* __restrict__ tau, double* __restrict__ args, int64_t col0) {
  // (launched with programmatic dependent launch between the Gram GEMM and the
  // preconditioner GEMM: let the latter start early, wait for the former)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t nb = d.L * d.K;
  const int64_t col = blockIdx.y + col0;  // = j*NB + b
  const int64_t j = col / nb, b = col - j * nb;
  const int64_t l = b / d.K, r = b - l * d.K;
  const double tl = tau[l];
  double* out = args + (l * d.kmax * d.K + j * d.K + r) * d.dim;
  const double* prev = gen + ((j - 1) * nb + b) * d.dim;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < d.dim;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double v;
    if (j < g) {
      v = __dmul_rn(tl, sum_partials(y, 0, i, col));
      if (j >= 1) v = __dadd_rn(v, prev[i]);
    } else {
      v = gen[i + ((g - 1) * nb + b) * d.dim];
    }
    out[i] = v;
  }
}

__global__ void update_kernel(BasisDims d, int64_t g, Partials applied, const int* __restrict__ kb,
                              double* __restrict__ gen, double* __restrict__ tilde, int* __restrict__ flags, int64_t col0) {
  const int64_t nb = d.L * d.K;
  const int64_t col = blockIdx.y + col0;
  const int64_t j = col / nb, b = col - j * nb;
  const int64_t l = b / d.K, r = b - l * d.K;
  if (g >= kb[l]) return;  // this interval's loop has ended (path_solver.cpp:39)
  double* gp = gen + col * d.dim;
  double* tp = tilde + col * d.dim;
  bool bad = false;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < d.dim;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double a = sum_partials(applied, l, i, j * d.K + r);
    const double v = (j < g) ? __dsub_rn(gp[i], a) : -a;
    gp[i] = v;
    bad |= !isfinite(v);
    tp[i] = __dadd_rn(tp[i], v);
  }
  if (bad) flags[l] = 1;
}

__global__ void seed_args_kernel(BasisDims d, const double* __restrict__ gen, double* __restrict__ args, int64_t col0,
                                 int64_t g) {
  const int64_t b = blockIdx.y + col0;  // problem
  const int64_t l = b / d.K, r = b - l * d.K;
  double* out = args + (l * d.kmax * d.K + (g + 1) * d.K + r) * d.dim;
  const double* src = gen + (g * d.L * d.K + b) * d.dim;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < d.dim;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = src[i];
}

__global__ void compose_kernel(BasisDims d, const double* __restrict__ tilde, const double* __restrict__ tau,
                               const int* __restrict__ kb, const double* __restrict__ lambda,
                               const int* __restrict__ interval, int64_t T, double* __restrict__ x, int64_t col0) {
  const int64_t nb = d.L * d.K;
  const int64_t col = blockIdx.y + col0;  // t*K + r
  const int64_t t = col / d.K, r = col - t * d.K;
  const int l = interval[t];
  const int64_t b = l * d.K + r;
  const double ta = tau[l];
  const double tt = __dmul_rn(ta, lambda[t]);
  const int k = kb[l];
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < d.dim;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double v = tilde[i + ((k - 1) * nb + b) * d.dim];
    for (int j = k - 2; j >= 0; --j) v = __dadd_rn(tilde[i + (j * nb + b) * d.dim], __dmul_rn(tt, v));
    x[i + col * d.dim] = __dmul_rn(v, ta);
  }
}

// One thread per (interval l, grid slot c): the column of powers, in j order.
__global__ void compose_coeffs_kernel(BasisDims d, const double* __restrict__ tau, const int* __restrict__ kb,
                                      const double* __restrict__ lambda, const int* __restrict__ off,
                                      const int* __restrict__ cnt, int64_t tmax, double* __restrict__ coef) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= d.L * tmax) return;
  const int64_t l = idx / tmax, c = idx - l * tmax;
  double* col = coef + (l * tmax + c) * d.kmax;
  const bool live = c < cnt[l];
  const double ta = tau[l];
  const double tt = live ? __dmul_rn(ta, lambda[off[l] + c]) : 0.0;
  const int k = kb[l];
  double pw = ta;
  for (int j = 0; j < d.kmax; ++j) {
    col[j] = (live && j < k) ? pw : 0.0;
    pw = __dmul_rn(pw, tt);
  }
}

// Grid: x = dim chunks, y = padded column (l, c, r); dead slots return at once.
__global__ void compose_gather_kernel(BasisDims d, const double* __restrict__ xpad, const int* __restrict__ off,
                                      const int* __restrict__ cnt, int64_t tmax, double* __restrict__ x, int64_t col0) {
  const int64_t col = blockIdx.y + col0;  // (l*tmax + c)*K + r
  const int64_t r = col % d.K, lc = col / d.K, l = lc / tmax, c = lc - l * tmax;
  if (c >= cnt[l]) return;
  const double* src = xpad + col * d.dim;
  double* dst = x + ((off[l] + c) * d.K + r) * d.dim;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < d.dim;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

__global__ void woodbury_tail_kernel(int64_t dim, int64_t cols, int64_t L, const double* __restrict__ args,
                                     int64_t s_args, const double* __restrict__ t3, int64_t s_t3,
                                     const double* __restrict__ lambda0, double* __restrict__ out, int64_t s_out) {
  const int64_t per = dim * cols;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < per * L;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t l = idx / per, e = idx % per;
    out[l * s_out + e] = __ddiv_rn(__dsub_rn(args[l * s_args + e], t3[l * s_t3 + e]), lambda0[l]);
  }
}

__global__ void woodbury_tail_rows_kernel(int64_t f0, int64_t rows, int64_t cols, int64_t L,
                                          const double* __restrict__ args, int64_t ld_args, int64_t s_args,
                                          const double* __restrict__ t3, const double* __restrict__ lambda0,
                                          double* __restrict__ pack, int64_t blk) {
  const int64_t N = cols * L;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < rows * N;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = idx % rows, j = idx / rows, l = j / cols, c = j - l * cols;
    pack[j * blk + r] =
        __ddiv_rn(__dsub_rn(args[l * s_args + c * ld_args + f0 + r], t3[j * rows + r]), lambda0[l]);
  }
}

__global__ void gather_row_blocks_kernel(const double* __restrict__ recv, int64_t blk, int64_t dim, int64_t cols,
                                         int64_t L, double* __restrict__ out, int64_t s_out) {
  const int64_t N = cols * L;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < dim * N;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = idx % dim, j = idx / dim, r = row / blk, l = j / cols, c = j - l * cols;
    out[l * s_out + c * dim + row] = recv[r * blk * N + j * blk + (row - r * blk)];
  }
}

__global__ void transpose_kernel(const double* __restrict__ in, int64_t rows, int64_t cols, int64_t ldi,
                                 double* __restrict__ out, int64_t ldo, int64_t cblk0) {
  __shared__ double tile[32][33];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32, c0 = (static_cast<int64_t>(blockIdx.y) + cblk0) * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + threadIdx.x, c = c0 + k;
    if (r < rows && c < cols) tile[k][threadIdx.x] = in[r + c * ldi];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + threadIdx.x, r = r0 + k;
    if (r < rows && c < cols) out[c + r * ldo] = tile[threadIdx.x][k];
  }
}

// One warp per row; lanes stride over the c right-hand sides.
__global__ void spmm_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ col,
                            const double* __restrict__ val, int64_t n, int64_t c, const double* __restrict__ x,
                            double* __restrict__ y) {
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t row = warp; row < n; row += nwarps) {
    const int64_t p0 = off[row], p1 = off[row + 1];
    for (int64_t cc = lane; cc < c; cc += 32) {
      double acc = 0.0;
      for (int64_t p = p0; p < p1; ++p) acc = __dadd_rn(acc, __dmul_rn(val[p], x[static_cast<int64_t>(col[p]) * c + cc]));
      y[row * c + cc] = acc;
    }
  }
}

__global__ void copy_cols_kernel(const double* __restrict__ src, int64_t rows, int64_t cols, int64_t lds,
                                 double* __restrict__ dst, int64_t ldd) {
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < rows * cols;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx % rows, j = idx / rows;
    dst[i + j * ldd] = src[i + j * lds];
  }
}

__global__ void fill_kernel(double* __restrict__ dst, int64_t count, double v) {
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < count;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[idx] = v;
}

// One CTA per column: strided per-thread sums (rows in a fixed order), then a
// fixed shared-memory tree.
__global__ void __launch_bounds__(256) column_sq_kernel(const double* __restrict__ r, int64_t rows, int64_t ldr,
                                                        const double* __restrict__ b, int64_t K, int64_t ldb,
                                                        double* __restrict__ out, int64_t col0) {
  __shared__ double red[256];
  const int64_t j = blockIdx.x + col0;
  const double* rc = r + j * ldr;
  const double* bc = b ? b + (j % K) * ldb : nullptr;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < rows; i += 256) {
    const double v = bc ? __dsub_rn(rc[i], bc[i]) : rc[i];
    acc = fma(v, v, acc);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int h = 128; h >= 1; h >>= 1) {
    if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[j] = red[0];
}

__global__ void combine_losses_kernel(const double* __restrict__ rn, const double* __restrict__ xn,
                                      const double* __restrict__ lambda, int64_t T, int64_t K,
                                      double* __restrict__ loss) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < T;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s = 0.0, q = 0.0;
    for (int64_t k = 0; k < K; ++k) {
      s += rn[t * K + k];
      if (xn) q += xn[t * K + k];
    }
    loss[t] = lambda && xn ? 0.5 * s + 0.5 * lambda[t] * q : 0.5 * s;
  }
}

}  // namespace

void column_sq_norms(const double* r, int64_t rows, int64_t cols, int64_t ldr, const double* b, int64_t K,
                     int64_t ldb, double* out, cudaStream_t stream) {
  for (int64_t c0 = 0; c0 < cols; c0 += (int64_t{1} << 30)) {
    const int64_t cn = std::min<int64_t>(int64_t{1} << 30, cols - c0);
    column_sq_kernel<<<static_cast<unsigned>(cn), 256, 0, stream>>>(r, rows, ldr, b, K, ldb, out, c0);
    RP_LAUNCH_CHECK();
  }
}

void combine_losses(const double* rn, const double* xn, const double* lambda, int64_t T, int64_t K, double* loss,
                    cudaStream_t stream) {
  if (T <= 0) return;
  combine_losses_kernel<<<grid_for(T), 256, 0, stream>>>(rn, xn, lambda, T, K, loss);
  RP_LAUNCH_CHECK();
}

// Launches `launch(grid, col0)` over column chunks of at most 65535 (grid.y limit).
template <class F>
void for_col_chunks(int64_t rows, int64_t cols, F launch) {
  const unsigned gx = static_cast<unsigned>(std::min<int64_t>(ceil_div(rows, 256), 64));
  for (int64_t c0 = 0; c0 < cols; c0 += 65535) {
    const int64_t cn = std::min<int64_t>(65535, cols - c0);
    launch(dim3(gx, static_cast<unsigned>(cn)), c0);
    RP_LAUNCH_CHECK();
  }
}

void build_args(const BasisDims& d, int64_t g, const Partials& y, const double* gen, const double* d_tau,
                double* args_im, cudaStream_t stream) {
  for_col_chunks(d.dim, (g + 1) * d.nb(), [&](dim3 grid, int64_t c0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(256);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    RP_CUDA(cudaLaunchKernelEx(&cfg, build_args_kernel, d, g, y, gen, d_tau, args_im, c0));
  });
}

void seed_args(const BasisDims& d, const double* gen, double* args_im, cudaStream_t stream) {
  if (d.kmax < 2) return;
  for_col_chunks(d.dim, d.nb(), [&](dim3 grid, int64_t c0) {
    seed_args_kernel<<<grid, 256, 0, stream>>>(d, gen, args_im, c0, 0);
  });
}

void seed_next_args(const BasisDims& d, int64_t g, const double* gen, double* args_im, cudaStream_t stream) {
  for_col_chunks(d.dim, d.nb(), [&](dim3 grid, int64_t c0) {
    seed_args_kernel<<<grid, 256, 0, stream>>>(d, gen, args_im, c0, g);
  });
}

void update_gen(const BasisDims& d, int64_t g, const Partials& applied, const int* d_k, double* gen, double* tilde,
                int* d_flags, cudaStream_t stream) {
  for_col_chunks(d.dim, (g + 1) * d.nb(), [&](dim3 grid, int64_t c0) {
    update_kernel<<<grid, 256, 0, stream>>>(d, g, applied, d_k, gen, tilde, d_flags, c0);
  });
}

void compose(const BasisDims& d, const double* tilde, const double* d_tau, const int* d_k, const double* d_lambda,
             const int* d_interval, int64_t T, double* x, cudaStream_t stream) {
  if (T <= 0) return;
  for_col_chunks(d.dim, d.K * T, [&](dim3 grid, int64_t c0) {
    compose_kernel<<<grid, 256, 0, stream>>>(d, tilde, d_tau, d_k, d_lambda, d_interval, T, x, c0);
  });
}

void compose_coeffs(const BasisDims& d, const double* d_tau, const int* d_k, const double* d_lambda, const int* d_off,
                    const int* d_cnt, int64_t tmax, double* coef, cudaStream_t stream) {
  if (d.L <= 0 || tmax <= 0) return;
  compose_coeffs_kernel<<<grid_for(d.L * tmax), 256, 0, stream>>>(d, d_tau, d_k, d_lambda, d_off, d_cnt, tmax, coef);
  RP_LAUNCH_CHECK();
}

void compose_gather(const BasisDims& d, const double* xpad, const int* d_off, const int* d_cnt, int64_t tmax, double* x,
                    cudaStream_t stream) {
  if (d.L <= 0 || tmax <= 0) return;
  for_col_chunks(d.dim, d.L * tmax * d.K, [&](dim3 grid, int64_t c0) {
    compose_gather_kernel<<<grid, 256, 0, stream>>>(d, xpad, d_off, d_cnt, tmax, x, c0);
  });
}

void woodbury_tail(int64_t dim, int64_t cols, int64_t L, int64_t s_args, const double* args, int64_t s_t3,
                   const double* t3, const double* d_lambda0, int64_t s_out, double* out, cudaStream_t stream) {
  if (dim <= 0 || cols <= 0 || L <= 0) return;
  woodbury_tail_kernel<<<grid_for(dim * cols * L), 256, 0, stream>>>(dim, cols, L, args, s_args, t3, s_t3, d_lambda0,
                                                                     out, s_out);
  RP_LAUNCH_CHECK();
}

void woodbury_tail_rows(int64_t f0, int64_t rows, int64_t cols, int64_t L, const double* args, int64_t ld_args,
                        int64_t s_args, const double* t3, const double* d_lambda0, double* pack, int64_t blk,
                        cudaStream_t stream) {
  if (rows <= 0 || cols <= 0 || L <= 0) return;
  woodbury_tail_rows_kernel<<<grid_for(rows * cols * L), 256, 0, stream>>>(f0, rows, cols, L, args, ld_args, s_args,
                                                                          t3, d_lambda0, pack, blk);
  RP_LAUNCH_CHECK();
}

void gather_row_blocks(const double* recv, int64_t blk, int64_t dim, int64_t cols, int64_t L, double* out,
                       int64_t s_out, cudaStream_t stream) {
  if (dim <= 0 || cols <= 0 || L <= 0) return;
  gather_row_blocks_kernel<<<grid_for(dim * cols * L), 256, 0, stream>>>(recv, blk, dim, cols, L, out, s_out);
  RP_LAUNCH_CHECK();
}

void transpose(const double* in, int64_t rows, int64_t cols, int64_t ldi, double* out, int64_t ldo,
               cudaStream_t stream) {
  // (grid.y is limited to 65535 blocks: column blocks go in chunks)
  const int64_t cblks = ceil_div(cols, 32);
  for (int64_t cb = 0; cb < cblks; cb += 65535) {
    dim3 grid(static_cast<unsigned>(ceil_div(rows, 32)), static_cast<unsigned>(std::min<int64_t>(65535, cblks - cb)));
    transpose_kernel<<<grid, dim3(32, 8), 0, stream>>>(in, rows, cols, ldi, out, ldo, cb);
    RP_LAUNCH_CHECK();
  }
}

void spmm_csr_rm(const int64_t* off, const int32_t* col, const double* val, int64_t n, int64_t c, const double* x_rm,
                 double* y_rm, cudaStream_t stream) {
  if (n <= 0 || c <= 0) return;
  spmm_kernel<<<grid_for(n * 32, 256), 256, 0, stream>>>(off, col, val, n, c, x_rm, y_rm);
  RP_LAUNCH_CHECK();
}

void copy_cols(const double* src, int64_t rows, int64_t cols, int64_t lds, double* dst, int64_t ldd,
               cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return;
  copy_cols_kernel<<<grid_for(rows * cols), 256, 0, stream>>>(src, rows, cols, lds, dst, ldd);
  RP_LAUNCH_CHECK();
}

void fill(double* dst, int64_t count, double v, cudaStream_t stream) {
  if (count <= 0) return;
  fill_kernel<<<grid_for(count), 256, 0, stream>>>(dst, count, v);
  RP_LAUNCH_CHECK();
}

}  // namespace rpb
