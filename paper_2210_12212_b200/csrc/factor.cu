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

// Cholesky of the kb x kb diagonal block at (k0, k0) of each matrix, then its
// triangular inverse, written back in place (the panel solve becomes a GEMM
// and the later trtri starts from the diagonal inverses).  256 threads:
// thread (r = t % 64, p = t / 64) keeps row r's columns c = 4 cc + p in
// registers; L's columns are published in shared memory one per step.  Rows
// and columns >= kb are padded with the identity.
__global__ void __launch_bounds__(256) potrf_diag(double* h, int64_t ld, int64_t stride, int64_t k0, int kb,
                                                  int* info) {
  __shared__ double Ls[NB][NB + 1];  // Ls[c][r] = L(r, c)
  __shared__ double xrow[NB];
  __shared__ double piv_s;
  double* A = h + blockIdx.x * stride + k0 + k0 * ld;
  const int r = threadIdx.x & (NB - 1);
  const int part = threadIdx.x >> 6;  // 0..3
  double t[NB / 4];
  {
    // all 16 loads issued unconditionally (clamped addresses), then selected
    const int rc = min(r, kb - 1);
    double v[NB / 4];
#pragma unroll
    for (int cc = 0; cc < NB / 4; ++cc) v[cc] = A[rc + static_cast<int64_t>(min(4 * cc + part, kb - 1)) * ld];
#pragma unroll
    for (int cc = 0; cc < NB / 4; ++cc) {
      const int c = 4 * cc + part;
      t[cc] = (r < kb && c < kb) ? (c <= r ? v[cc] : 0.0) : (r == c ? 1.0 : 0.0);
    }
  }
  // The step loops stay rolled (small code: the kernel is latency bound, and a
  // fully unrolled 64-step body runs out of instruction cache); t[jc] with a
  // run-time jc is read and written through selects.
  int bad = 0;
#pragma unroll 1
  for (int j = 0; j < NB; ++j) {
    const int jc = j >> 2, jp = j & 3;
    double tj = t[0];
#pragma unroll
    for (int cc = 1; cc < NB / 4; ++cc) tj = (cc == jc) ? t[cc] : tj;
    if (part == jp && r == j) piv_s = tj;
    __syncthreads();
    double dpiv = piv_s;
    if (!(dpiv > 0.0) || !isfinite(dpiv)) {
      if (!bad) bad = j + 1;
      dpiv = 1.0;  // keep going; the caller reports the failure
    }
    const double piv = sqrt(dpiv);
    const double rpiv = 1.0 / piv;
    if (part == jp && r >= j) {
      const double l = (r == j) ? piv : tj * rpiv;
#pragma unroll
      for (int cc = 0; cc < NB / 4; ++cc) t[cc] = (cc == jc) ? l : t[cc];
      Ls[j][r] = l;
    }
    if (r < j && part == 0) Ls[j][r] = 0.0;
    __syncthreads();
    if (r > j) {
      const double lr = Ls[j][r];
#pragma unroll
      for (int cc = 0; cc < NB / 4; ++cc) {
        const int c = 4 * cc + part;
        if (c > j && c <= r) t[cc] -= lr * Ls[j][c];
      }
    }
  }
  if (bad && threadIdx.x == 0 && bad <= kb && info[blockIdx.x] == 0) info[blockIdx.x] = static_cast<int>(k0 + bad);
  // X = L^{-1} row by row: X(j, :) = (e_j - sum_{i<j} L(j, i) X(i, :)) / L(j, j).
  double x[NB / 4];
#pragma unroll
  for (int cc = 0; cc < NB / 4; ++cc) x[cc] = (4 * cc + part == r) ? 1.0 : 0.0;
#pragma unroll 1
  for (int j = 0; j < NB; ++j) {
    if (r == j) {
      const double rdjj = 1.0 / Ls[j][j];
#pragma unroll
      for (int cc = 0; cc < NB / 4; ++cc) {
        x[cc] = x[cc] * rdjj;
        xrow[4 * cc + part] = x[cc];
      }
    }
    __syncthreads();
    if (r > j) {
      const double lrj = Ls[j][r];
#pragma unroll
      for (int cc = 0; cc < NB / 4; ++cc)
        if (4 * cc + part <= j) x[cc] -= lrj * xrow[4 * cc + part];
    }
    __syncthreads();
  }
#pragma unroll
  for (int cc = 0; cc < NB / 4; ++cc) {
    const int c = 4 * cc + part;
    if (r < kb && c < kb) A[r + c * ld] = (c <= r) ? x[cc] : 0.0;
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
  // 1) Cholesky, lower, right-looking with one panel of lookahead: after the
  // panel solve of block k, the next block column is updated on `stream`
  // (then block k+1 is factored there) while the rest of the trailing matrix
  // is updated on an auxiliary stream -- the latency-bound diagonal kernels
  // (one CTA per matrix) overlap the big trailing GEMMs.  All GEMMs here run
  // unsplit, so they share no workspace.
  // The critical chain (diagonal kernels, panel solves, next-column updates)
  // runs on a high-priority stream so its CTAs are scheduled ahead of the
  // trailing-update CTAs as SMs free up.
  const cudaStream_t user = stream;
  int prio_lo = 0, prio_hi = 0;
  RP_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  cudaStream_t aux = nullptr, hi = nullptr;
  RP_CUDA(cudaStreamCreateWithPriority(&aux, cudaStreamNonBlocking, prio_lo));
  RP_CUDA(cudaStreamCreateWithPriority(&hi, cudaStreamNonBlocking, prio_hi));
  std::vector<cudaEvent_t> events;
  auto new_event = [&]() {
    cudaEvent_t e;
    RP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    events.push_back(e);
    return e;
  };
  {
    cudaEvent_t start = new_event();
    RP_CUDA(cudaEventRecord(start, user));
    RP_CUDA(cudaStreamWaitEvent(hi, start, 0));
  }
  stream = hi;
  auto syrk_update = [&](int64_t row0, int64_t m, int64_t ncols, int64_t k0, int kb, cudaStream_t st) {
    // C(row0.., row0..row0+ncols) -= A21(row0.., :) A21(row0..row0+ncols, :)^T, lower part
    GemmArgs g;
    g.opa = Op::N;
    g.opb = Op::T;
    g.m = m;
    g.n = ncols;
    g.k = kb;
    g.alpha = -1.0;
    g.beta = 1.0;
    g.a = h + row0 + k0 * ld;
    g.lda = ld;
    g.stride_a = stride;
    g.b = g.a;
    g.ldb = ld;
    g.stride_b = stride;
    g.c = h + row0 + row0 * ld;
    g.ldc = ld;
    g.stride_c = stride;
    g.batch = batch;
    g.lower_only = true;
    g.split_k = 1;
    dgemm(g, st);
  };
  cudaEvent_t prev_rest = nullptr;  // trailing update of the previous panel (aux stream)
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
    const int64_t r0 = k0 + kb;
    const int64_t nxt = std::min<int64_t>(NB, rows), rest = rows - nxt;
    cudaEvent_t rest_done = nullptr;
    if (rest > 0) {  // columns beyond the next block: aux stream
      cudaEvent_t panel_done = new_event();
      RP_CUDA(cudaEventRecord(panel_done, stream));
      RP_CUDA(cudaStreamWaitEvent(aux, panel_done, 0));
      syrk_update(r0 + nxt, rest, rest, k0, kb, aux);
      rest_done = new_event();
      RP_CUDA(cudaEventRecord(rest_done, aux));
    }
    // the next block column (all rows below the diagonal) on the main stream;
    // it also needs the previous panel's update of those columns
    if (prev_rest) RP_CUDA(cudaStreamWaitEvent(stream, prev_rest, 0));
    syrk_update(r0, rows, nxt, k0, kb, stream);
    prev_rest = rest_done;
  }
  if (prev_rest) RP_CUDA(cudaStreamWaitEvent(stream, prev_rest, 0));
  {
    cudaEvent_t done = new_event();
    RP_CUDA(cudaEventRecord(done, hi));
    RP_CUDA(cudaStreamWaitEvent(user, done, 0));
  }
  stream = user;
  for (cudaEvent_t e : events) RP_CUDA(cudaEventDestroy(e));  // (released once complete)
  RP_CUDA(cudaStreamDestroy(aux));
  RP_CUDA(cudaStreamDestroy(hi));
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
