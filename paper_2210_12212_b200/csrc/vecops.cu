// d-vector kernels, see vecops.h.
#include "vecops.h"

#include <algorithm>

#include "common.h"

namespace rpb {
namespace {

unsigned blocks_for(int64_t work) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, 256), 148 * 16)));
}

#define RP_GRID_STRIDE(i, n)                                                                     \
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < (n); \
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)

__global__ void dot_partials_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t count,
                                    double* __restrict__ part) {
  __shared__ double sh[256];
  const int64_t per = (count + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = min(count, lo + per);
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) acc = __fma_rn(x[i], y[i], acc);
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void sum_partials_kernel(const double* __restrict__ part, int count, double* __restrict__ out) {
  __shared__ double sh[32];
  // 32 lanes sum fixed strided subsets, then lane 0 adds them in lane order
  double acc = 0.0;
  for (int i = threadIdx.x; i < count; i += 32) acc += part[i];
  sh[threadIdx.x] = acc;
  __syncwarp();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < 32; ++i) s += sh[i];
    *out = s;
  }
}

__global__ void ihs_grad_kernel(const double* __restrict__ g, const double* __restrict__ x, double lam,
                                const double* __restrict__ atb, int64_t n, double* __restrict__ grad) {
  RP_GRID_STRIDE(i, n) grad[i] = __dsub_rn(__dadd_rn(g[i], __dmul_rn(lam, x[i])), atb[i]);
}

__global__ void ihs_step_kernel(double* __restrict__ xs, const double* __restrict__ pg, double tau, int64_t n,
                                int* __restrict__ flag) {
  bool bad = false;
  RP_GRID_STRIDE(i, n) {
    const double v = __dsub_rn(xs[i], __dmul_rn(tau, pg[i]));
    xs[i] = v;
    bad |= !isfinite(v);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 1;
}

__global__ void cg_init_kernel(const double* __restrict__ atb, const double* __restrict__ g,
                               const double* __restrict__ x, double lam, int64_t n, double* __restrict__ r,
                               double* __restrict__ p) {
  RP_GRID_STRIDE(i, n) {
    const double v = __dsub_rn(__dsub_rn(atb[i], g[i]), __dmul_rn(lam, x[i]));
    r[i] = v;
    p[i] = v;
  }
}

__global__ void cg_q_kernel(const double* __restrict__ g, const double* __restrict__ p, double lam, int64_t n,
                            double* __restrict__ q) {
  RP_GRID_STRIDE(i, n) q[i] = __dadd_rn(g[i], __dmul_rn(lam, p[i]));
}

__global__ void cg_update_kernel(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                                 const double* __restrict__ q, const double* __restrict__ rr,
                                 const double* __restrict__ pq, int64_t n) {
  const double alpha = __ddiv_rn(*rr, *pq);
  RP_GRID_STRIDE(i, n) {
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
    r[i] = __dsub_rn(r[i], __dmul_rn(alpha, q[i]));
  }
}

__global__ void cg_direction_kernel(double* __restrict__ p, const double* __restrict__ r,
                                    const double* __restrict__ rr_next, const double* __restrict__ rr, int64_t n) {
  const double beta = __ddiv_rn(*rr_next, *rr);
  RP_GRID_STRIDE(i, n) p[i] = __dadd_rn(r[i], __dmul_rn(beta, p[i]));
}

__global__ void identity_block_kernel(double* __restrict__ out, int64_t d, int64_t cols, int64_t c0) {
  RP_GRID_STRIDE(e, d * cols) {
    const int64_t i = e % d, j = e / d;
    out[e] = i == c0 + j ? 1.0 : 0.0;
  }
}

__global__ void residual_kernel(double* __restrict__ r, const double* __restrict__ b, int64_t n) {
  RP_GRID_STRIDE(i, n) r[i] = __dsub_rn(r[i], b[i]);
}

__global__ void mirror_lower_kernel(double* __restrict__ g, int64_t n, int64_t ld) {
  __shared__ double tile[32][33];
  const int64_t bi = blockIdx.y, bj = blockIdx.x;  // source tile (rows bi, cols bj), bi >= bj
  if (bi < bj) return;
  const int64_t r0 = bi * 32, c0 = bj * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + threadIdx.x, c = c0 + k;
    if (r < n && c < n) tile[k][threadIdx.x] = g[r + c * ld];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = c0 + threadIdx.x, c = r0 + k;  // destination (r, c) = source (c, r)
    if (r < n && c < n && r < c) g[r + c * ld] = tile[threadIdx.x][k];
  }
}

__global__ void copy_mapped_kernel(const double* __restrict__ src, int64_t n, double* __restrict__ dst) {
  RP_GRID_STRIDE(i, n) dst[i] = src[i];
}

}  // namespace

void copy_mapped(const double* src, int64_t n, double* dst, cudaStream_t s) {
  if (n <= 0) return;
  copy_mapped_kernel<<<blocks_for(n), 256, 0, s>>>(src, n, dst);
  RP_LAUNCH_CHECK();
}

void mirror_lower(double* g, int64_t n, int64_t ld, cudaStream_t s) {
  if (n <= 1) return;
  const unsigned t = static_cast<unsigned>(ceil_div(n, 32));
  mirror_lower_kernel<<<dim3(t, t), dim3(32, 8), 0, s>>>(g, n, ld);
  RP_LAUNCH_CHECK();
}

void residual_in_place(double* r, const double* b, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  residual_kernel<<<blocks_for(n), 256, 0, s>>>(r, b, n);
  RP_LAUNCH_CHECK();
}

void identity_block(double* out, int64_t d, int64_t cols, int64_t c0, cudaStream_t s) {
  identity_block_kernel<<<blocks_for(d * cols), 256, 0, s>>>(out, d, cols, c0);
  RP_LAUNCH_CHECK();
}

void vec_dot(const double* x, const double* y, int64_t n, double* part, double* out, cudaStream_t s) {
  dot_partials_kernel<<<kDotParts, 256, 0, s>>>(x, y, n, part);
  RP_LAUNCH_CHECK();
  sum_partials_kernel<<<1, 32, 0, s>>>(part, kDotParts, out);
  RP_LAUNCH_CHECK();
}

void ihs_grad(const double* g, const double* x, double lam, const double* atb, int64_t n, double* grad,
              cudaStream_t s) {
  ihs_grad_kernel<<<blocks_for(n), 256, 0, s>>>(g, x, lam, atb, n, grad);
  RP_LAUNCH_CHECK();
}

void ihs_step(double* xs, const double* pg, double tau, int64_t n, int* flag, cudaStream_t s) {
  ihs_step_kernel<<<blocks_for(n), 256, 0, s>>>(xs, pg, tau, n, flag);
  RP_LAUNCH_CHECK();
}

void cg_init(const double* atb, const double* g, const double* x, double lam, int64_t n, double* r, double* p,
             cudaStream_t s) {
  cg_init_kernel<<<blocks_for(n), 256, 0, s>>>(atb, g, x, lam, n, r, p);
  RP_LAUNCH_CHECK();
}

void cg_q(const double* g, const double* p, double lam, int64_t n, double* q, cudaStream_t s) {
  cg_q_kernel<<<blocks_for(n), 256, 0, s>>>(g, p, lam, n, q);
  RP_LAUNCH_CHECK();
}

void cg_update(double* x, double* r, const double* p, const double* q, const double* rr, const double* pq, int64_t n,
               cudaStream_t s) {
  cg_update_kernel<<<blocks_for(n), 256, 0, s>>>(x, r, p, q, rr, pq, n);
  RP_LAUNCH_CHECK();
}

void cg_direction(double* p, const double* r, const double* rr_next, const double* rr, int64_t n, cudaStream_t s) {
  cg_direction_kernel<<<blocks_for(n), 256, 0, s>>>(p, r, rr_next, rr, n);
  RP_LAUNCH_CHECK();
}

__global__ void upper_triangle_kernel(const double* __restrict__ a, int64_t lda, int64_t r, double* __restrict__ out) {
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < r * r;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx % r, j = idx / r;
    out[idx] = i <= j ? a[i + j * lda] : 0.0;
  }
}

void upper_triangle(const double* a, int64_t lda, int64_t r, double* out, cudaStream_t s) {
  if (r <= 0) return;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(r * r, 256), 148 * 16));
  upper_triangle_kernel<<<blocks, 256, 0, s>>>(a, lda, r, out);
  RP_LAUNCH_CHECK();
}

__global__ void svd_scale_kernel(const double* __restrict__ sigma, const double* __restrict__ utb, int64_t r,
                                 const double* __restrict__ lambda, int64_t T, double* __restrict__ z) {
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < r * T;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx % r, t = idx / r;
    const double sg = sigma[i];
    z[idx] = __ddiv_rn(__dmul_rn(sg, utb[i]), __dadd_rn(__dmul_rn(sg, sg), lambda[t]));
  }
}

void svd_scale(const double* sigma, const double* utb, int64_t r, const double* lambda, int64_t T, double* z,
               cudaStream_t s) {
  if (r <= 0 || T <= 0) return;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(r * T, 256), 148 * 16));
  svd_scale_kernel<<<blocks, 256, 0, s>>>(sigma, utb, r, lambda, T, z);
  RP_LAUNCH_CHECK();
}

}  // namespace rpb
