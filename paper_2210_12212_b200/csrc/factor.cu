// Batched SPD inverse: potrf (right-looking, 64-wide panels) -> trtri
// (recursive doubling) -> P = L^{-T} L^{-1}; the O(n^3) parts run as DMMA GEMMs.
#include <algorithm>
#include <string>
#include <vector>

#include "common.h"
#include "factor.h"
#include "gemm_f64.h"

namespace rpb {
namespace {

constexpr int NB = 64;

// Unblocked Cholesky of the kb x kb diagonal block at (k0, k0) of each matrix:
// one warp per matrix, lane l owns rows l and l + 32 (no block barriers).  The
// finished column j is copied to a separate array so the trailing update's
// loads never alias its stores (lets the compiler pipeline the loop).
__global__ void __launch_bounds__(32) potrf_diag(double* h, int64_t ld, int64_t stride, int64_t k0, int kb,
                                                 int* info) {
  __shared__ double T[NB][NB + 1];
  __shared__ double colj[NB];
  double* A = h + blockIdx.x * stride + k0 + k0 * ld;
  const int lane = threadIdx.x;
#pragma unroll 8
  for (int j = 0; j < kb; ++j) {
    if (lane < kb) T[lane][j] = A[lane + j * ld];
    if (lane + 32 < kb) T[lane + 32][j] = A[lane + 32 + j * ld];
  }
  __syncwarp();
  int bad = 0;
  for (int j = 0; j < kb; ++j) {
    double d = T[j][j];
    if (!(d > 0.0) || !isfinite(d)) {
      if (!bad) bad = j + 1;
      d = 1.0;  // keep going; the caller reports the failure
    }
    const double piv = sqrt(d);
    const double inv = 1.0 / piv;
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int r = lane + 32 * h2;
      if (r >= j && r < kb) {
        const double v = (r == j) ? piv : T[r][j] * inv;
        T[r][j] = v;
        colj[r] = v;
      }
    }
    __syncwarp();
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int r = lane + 32 * h2;
      if (r > j && r < kb) {
        const double lrj = colj[r];
        double* row = &T[r][0];
        int c = j + 1;
        for (; c + 3 <= r; c += 4) {
          const double c0 = colj[c], c1 = colj[c + 1], c2 = colj[c + 2], c3 = colj[c + 3];
          const double t0 = row[c], t1 = row[c + 1], t2 = row[c + 2], t3 = row[c + 3];
          row[c] = t0 - lrj * c0;
          row[c + 1] = t1 - lrj * c1;
          row[c + 2] = t2 - lrj * c2;
          row[c + 3] = t3 - lrj * c3;
        }
        for (; c <= r; ++c) row[c] -= lrj * colj[c];
      }
    }
    __syncwarp();
  }
  if (bad && lane == 0 && info[blockIdx.x] == 0) info[blockIdx.x] = static_cast<int>(k0 + bad);
#pragma unroll 8
  for (int j = 0; j < kb; ++j) {
    if (lane < kb && lane >= j) A[lane + j * ld] = T[lane][j];
    if (lane + 32 < kb && lane + 32 >= j) A[lane + 32 + j * ld] = T[lane + 32][j];
  }
}

// Panel solve X * L11^T = B for the rows below the diagonal block; one thread
// per row, 128 rows per CTA; four independent partial sums per dot product.
__global__ void __launch_bounds__(128) potrf_trsm(double* h, int64_t ld, int64_t stride, int64_t k0, int kb,
                                                  int64_t rows) {
  extern __shared__ double dsm[];
  double(*L)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm);
  double(*X)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm + NB * (NB + 1));
  double* base = h + blockIdx.y * stride;
  const double* L11 = base + k0 + k0 * ld;
  const int t = threadIdx.x;
#pragma unroll 8
  for (int j = 0; j < kb; ++j)
    if (t < kb) L[t][j] = L11[t + j * ld];
  const int64_t r0 = k0 + kb + static_cast<int64_t>(blockIdx.x) * 128;
  const int nr = static_cast<int>((k0 + kb + rows - r0) < 128 ? (k0 + kb + rows - r0) : 128);
  double* B = base + k0 * ld;  // column k0 of the matrix
#pragma unroll 8
  for (int j = 0; j < kb; ++j)
    if (t < nr) X[t][j] = B[r0 + t + j * ld];
  __syncthreads();
  if (t < nr) {
    for (int j = 0; j < kb; ++j) {
      double s0 = X[t][j], s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int i = 0;
      for (; i + 3 < j; i += 4) {
        s0 -= X[t][i] * L[j][i];
        s1 -= X[t][i + 1] * L[j][i + 1];
        s2 -= X[t][i + 2] * L[j][i + 2];
        s3 -= X[t][i + 3] * L[j][i + 3];
      }
      for (; i < j; ++i) s0 -= X[t][i] * L[j][i];
      X[t][j] = ((s0 + s1) + (s2 + s3)) / L[j][j];
    }
  }
  __syncthreads();
#pragma unroll 8
  for (int j = 0; j < kb; ++j)
    if (t < nr) B[r0 + t + j * ld] = X[t][j];
}

// In-place inverse of each nb x nb lower-triangular diagonal block; zeroes the
// strict upper triangle of the whole matrix on the way.
__global__ void __launch_bounds__(64) trtri_diag(double* h, int64_t n, int64_t ld, int64_t stride) {
  extern __shared__ double dsm[];
  double(*L)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm);
  double(*X)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm + NB * (NB + 1));
  const int64_t k0 = static_cast<int64_t>(blockIdx.x) * NB;
  const int kb = static_cast<int>((n - k0) < NB ? (n - k0) : NB);
  double* A = h + blockIdx.y * stride + k0 + k0 * ld;
  {
    const int i = threadIdx.x;
#pragma unroll 8
    for (int j = 0; j < kb; ++j)
      if (i < kb) L[i][j] = (i >= j) ? A[i + j * ld] : 0.0;
  }
  __syncthreads();
  const int c = threadIdx.x;
  if (c < kb) {
    X[c][c] = 1.0 / L[c][c];
    for (int i = 0; i < c; ++i) X[i][c] = 0.0;
    for (int i = c + 1; i < kb; ++i) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int k = c;
      for (; k + 3 < i; k += 4) {
        s0 += L[i][k] * X[k][c];
        s1 += L[i][k + 1] * X[k + 1][c];
        s2 += L[i][k + 2] * X[k + 2][c];
        s3 += L[i][k + 3] * X[k + 3][c];
      }
      for (; k < i; ++k) s0 += L[i][k] * X[k][c];
      X[i][c] = -((s0 + s1) + (s2 + s3)) / L[i][i];
    }
  }
  __syncthreads();
  {
    const int i = threadIdx.x;
#pragma unroll 8
    for (int j = 0; j < kb; ++j)
      if (i < kb) A[i + j * ld] = X[i][j];
  }
}

__global__ void zero_upper(double* h, int64_t n, int64_t ld, int64_t stride) {
  double* A = h + blockIdx.y * stride;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < n * n;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    if (i < j) A[i + j * ld] = 0.0;
  }
}

__global__ void shifted_copy_kernel(const double* __restrict__ g, int64_t n, const double* __restrict__ shifts,
                                    double* __restrict__ h) {
  const int64_t b = blockIdx.y;
  const double s = shifts[b];
  double* H = h + b * n * n;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < n * n;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = idx % n, j = idx / n;
    H[idx] = (i == j) ? g[idx] + s : (i > j ? g[idx] : 0.0);
  }
}

unsigned grid1(int64_t work) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, 256), 148 * 8)));
}

}  // namespace

void shifted_copies(const double* g, int64_t n, const double* d_shifts, int64_t batch, double* h, cudaStream_t stream) {
  dim3 grid(grid1(n * n), static_cast<unsigned>(batch));
  shifted_copy_kernel<<<grid, 256, 0, stream>>>(g, n, d_shifts, h);
  RP_LAUNCH_CHECK();
}

void spd_inverse_batched(double* h, int64_t n, int64_t ld, int64_t stride, int64_t batch, double* out, int64_t ldo,
                         int64_t stride_o, cudaStream_t stream) {
  require(n >= 1 && batch >= 1, "spd_inverse: empty problem");
  DBuf<int> info(static_cast<size_t>(batch), stream);
  RP_CUDA(cudaMemsetAsync(info.get(), 0, sizeof(int) * batch, stream));
  // 1) Cholesky, lower.
  for (int64_t k0 = 0; k0 < n; k0 += NB) {
    const int kb = static_cast<int>(std::min<int64_t>(NB, n - k0));
    potrf_diag<<<static_cast<unsigned>(batch), 32, 0, stream>>>(h, ld, stride, k0, kb, info.get());
    RP_LAUNCH_CHECK();
    const int64_t rows = n - k0 - kb;
    if (rows <= 0) break;
    dim3 tg(static_cast<unsigned>(ceil_div(rows, 128)), static_cast<unsigned>(batch));
    constexpr int kTrsmSmem = (NB + 128) * (NB + 1) * 8;
    static bool attr = false;
    if (!attr) {
      RP_CUDA(cudaFuncSetAttribute(potrf_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrsmSmem));
      attr = true;
    }
    potrf_trsm<<<tg, 128, kTrsmSmem, stream>>>(h, ld, stride, k0, kb, rows);
    RP_LAUNCH_CHECK();
    GemmArgs g;  // A22 -= A21 A21^T (lower)
    g.opa = Op::N;
    g.opb = Op::T;
    g.m = rows;
    g.n = rows;
    g.k = kb;
    g.alpha = -1.0;
    g.beta = 1.0;
    g.a = h + (k0 + kb) + k0 * ld;
    g.lda = ld;
    g.stride_a = stride;
    g.b = g.a;
    g.ldb = ld;
    g.stride_b = stride;
    g.c = h + (k0 + kb) + (k0 + kb) * ld;
    g.ldc = ld;
    g.stride_c = stride;
    g.batch = batch;
    g.lower_only = true;
    g.split_k = 1;
    dgemm(g, stream);
  }
  // 2) Triangular inverse in place.
  {
    // (the strict upper triangle is already zero: shifted_copies writes it so
    // and potrf only touches the lower triangle)
    dim3 dg(static_cast<unsigned>(ceil_div(n, NB)), static_cast<unsigned>(batch));
    constexpr int kDiagSmem = 2 * NB * (NB + 1) * 8;
    static bool attr = false;
    if (!attr) {
      RP_CUDA(cudaFuncSetAttribute(trtri_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, kDiagSmem));
      attr = true;
    }
    trtri_diag<<<dg, 64, kDiagSmem, stream>>>(h, n, ld, stride);
    RP_LAUNCH_CHECK();
    DBuf<double> tmp;
    for (int64_t s = NB; s < n; s *= 2) {
      const int64_t pairs_full = n / (2 * s);
      // full pairs: blocks [i*2s, i*2s+s) and [i*2s+s, i*2s+2s)
      auto combine = [&](int64_t first, int64_t npairs, int64_t s2) {
        if (npairs <= 0 || s2 <= 0) return;
        const size_t need = static_cast<size_t>(npairs * batch * s2 * s);
        if (tmp.size() < need) tmp.alloc(need, stream);
        const int64_t pstride = 2 * s * (ld + 1);
        double* base = h + first * 2 * s * (ld + 1);
        // T = L21 * L11^{-1}   (s2 x s)
        GemmArgs g1;
        g1.m = s2;
        g1.n = s;
        g1.k = s;
        g1.a = base + s;  // L21 at (i*2s + s, i*2s)
        g1.lda = ld;
        g1.stride_a = pstride;
        g1.stride_a2 = stride;
        g1.b = base;  // L11^{-1}
        g1.ldb = ld;
        g1.stride_b = pstride;
        g1.stride_b2 = stride;
        g1.c = tmp.get();
        g1.ldc = s2;
        g1.stride_c = s2 * s;
        g1.stride_c2 = s2 * s * npairs;
        g1.batch = npairs;
        g1.batch2 = batch;
        g1.split_k = 1;
        dgemm(g1, stream);
        // X21 = -L22^{-1} * T  -> written over L21
        GemmArgs g2;
        g2.m = s2;
        g2.n = s;
        g2.k = s2;
        g2.alpha = -1.0;
        g2.a = base + s + s * ld;  // L22^{-1}
        g2.lda = ld;
        g2.stride_a = pstride;
        g2.stride_a2 = stride;
        g2.b = tmp.get();
        g2.ldb = s2;
        g2.stride_b = s2 * s;
        g2.stride_b2 = s2 * s * npairs;
        g2.c = base + s;
        g2.ldc = ld;
        g2.stride_c = pstride;
        g2.stride_c2 = stride;
        g2.batch = npairs;
        g2.batch2 = batch;
        g2.split_k = 1;
        dgemm(g2, stream);
      };
      combine(0, pairs_full, s);
      const int64_t tail0 = pairs_full * 2 * s;
      if (tail0 + s < n) combine(pairs_full, 1, n - tail0 - s);
    }
  }
  // 3) out = L^{-T} L^{-1} (symmetric).
  {
    GemmArgs g;
    g.opa = Op::T;
    g.opb = Op::N;
    g.m = n;
    g.n = n;
    g.k = n;
    g.a = h;
    g.lda = ld;
    g.stride_a = stride;
    g.b = h;
    g.ldb = ld;
    g.stride_b = stride;
    g.c = out;
    g.ldc = ldo;
    g.stride_c = stride_o;
    g.batch = batch;
    g.lower_only = true;
    g.mirror = true;
    g.tri_k = true;  // L^{-1} is lower triangular
    g.split_k = 1;
    dgemm(g, stream);
  }
  std::vector<int> hinfo(static_cast<size_t>(batch));
  RP_CUDA(cudaMemcpyAsync(hinfo.data(), info.get(), sizeof(int) * batch, cudaMemcpyDeviceToHost, stream));
  RP_CUDA(cudaStreamSynchronize(stream));
  for (int64_t b = 0; b < batch; ++b)
    if (hinfo[b])
      throw FactorFailure("factorization: shifted sketched Gram is not positive definite (matrix " +
                          std::to_string(b) + ", column " + std::to_string(hinfo[b]) + ")");
}

}  // namespace rpb
