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

// Unblocked Cholesky of the kb x kb diagonal block at (k0, k0) of each matrix.
// 256 threads: thread t owns row r = t % 64 and the columns c = t / 64 (mod 4)
// of the trailing update; every thread recomputes the pivot (no broadcast
// barrier), two barriers per column.
__global__ void __launch_bounds__(256) potrf_diag(double* h, int64_t ld, int64_t stride, int64_t k0, int kb,
                                                  int* info) {
  __shared__ double T[NB][NB + 1];
  double* A = h + blockIdx.x * stride + k0 + k0 * ld;
  const int r = threadIdx.x & (NB - 1);
  const int part = threadIdx.x >> 6;  // 0..3
#pragma unroll
  for (int jj = 0; jj < NB / 4; ++jj) {
    const int j = part + 4 * jj;
    if (j < kb && r < kb) T[r][j] = A[r + j * ld];
  }
  __syncthreads();
  int bad = 0;
  for (int j = 0; j < kb; ++j) {
    double d = T[j][j];
    if (!(d > 0.0) || !isfinite(d)) {
      if (!bad) bad = j + 1;
      d = 1.0;  // keep going; the caller reports the failure
    }
    const double piv = sqrt(d);
    if (part == 0 && r >= j && r < kb) T[r][j] = (r == j) ? piv : T[r][j] / piv;
    __syncthreads();
    if (r > j && r < kb) {
      const double lrj = T[r][j];
      const int c0 = j + 1 + ((part - (j + 1)) & 3);  // first c > j with c % 4 == part
      for (int c = c0; c <= r; c += 4) T[r][c] -= lrj * T[c][j];
    }
    __syncthreads();
  }
  if (bad && threadIdx.x == 0 && info[blockIdx.x] == 0) info[blockIdx.x] = static_cast<int>(k0 + bad);
  // L11^{-1} by columns: four threads per column c split each dot product
  // X[i][c] = -(sum_{k=c}^{i-1} L[i][k] X[k][c]) / L[i][i].  X (lower) is kept
  // transposed in the unused strict upper triangle of T (X[i][c] at T[c][i]),
  // its diagonal in xd.
  __shared__ double xd[NB];
  {
    const int c = threadIdx.x >> 2, q = threadIdx.x & 3;
    const bool live = c < kb;
    const double xcc = live ? 1.0 / T[c][c] : 0.0;
    if (live && q == 0) xd[c] = xcc;
    // uniform trip count across the warp (the shuffles need every lane)
    for (int i = 1; i < NB; ++i) {
      const bool act = live && i > c && i < kb;
      double sum = 0.0;
      if (act)
        for (int k = c + q; k < i; k += 4) sum += T[i][k] * (k == c ? xcc : T[c][k]);
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      if (act && q == 0) T[c][i] = -sum / T[i][i];
      __syncwarp();
    }
  }
  __syncthreads();
  // the diagonal block now holds L11^{-1} (zero above the diagonal): the
  // panel solve becomes a GEMM and the later triangular inverse starts from it
#pragma unroll
  for (int jj = 0; jj < NB / 4; ++jj) {
    const int j = part + 4 * jj;
    if (j < kb && r < kb) A[r + j * ld] = (r > j) ? T[j][r] : (r == j ? xd[r] : 0.0);
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
    potrf_diag<<<static_cast<unsigned>(batch), 256, 0, stream>>>(h, ld, stride, k0, kb, info.get());
    RP_LAUNCH_CHECK();
    const int64_t rows = n - k0 - kb;
    if (rows <= 0) break;
    {
      // Panel: A21 <- A21 * L11^{-T}.  In place is safe: N = kb <= 64 fits one
      // 128x64 tile, so each CTA owns whole rows and reads its full A tile
      // before the epilogue writes them.
      GemmArgs t;
      t.opa = Op::N;
      t.opb = Op::T;
      t.m = rows;
      t.n = kb;
      t.k = kb;
      t.a = h + (k0 + kb) + k0 * ld;
      t.lda = ld;
      t.stride_a = stride;
      t.b = h + k0 + k0 * ld;  // L11^{-1}
      t.ldb = ld;
      t.stride_b = stride;
      t.c = h + (k0 + kb) + k0 * ld;
      t.ldc = ld;
      t.stride_c = stride;
      t.batch = batch;
      t.split_k = 1;
      t.force_tile = 6;  // 128 x 64
      dgemm(t, stream);
    }
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
    // (the diagonal blocks already hold their inverses, written by potrf_diag)
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
