// Batched SPD inverse: potrf (right-looking, 64-wide panels) -> trtri
// (recursive doubling) -> P = L^{-T} L^{-1}; the O(n^3) parts run as DMMA GEMMs.
#include <algorithm>
#include <cstdlib>
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

// Same contract as potrf_diag, blocked by 4 columns: per block of four a
// single thread factors the 4 x 4 diagonal block (and inverts it), every
// thread solves its row of the 64 x 4 panel against it, then applies the
// rank-4 trailing update as four sequential rank-1 steps (the unblocked
// kernel's order).  The triangular inverse runs as block forward
// substitution with the stored 4 x 4 inverses.  3 + 2 barriers per four
// columns instead of 2 + 2 per column.
__global__ void __launch_bounds__(256) potrf_diag4(double* h, int64_t ld, int64_t stride, int64_t k0, int kb,
                                                   int* info) {
  __shared__ double Ls[NB][NB + 1];    // Ls[c][r] = L(r, c), r >= c
  __shared__ double Pn[NB][5];         // the current 64 x 4 panel, Pn[r][s] = A(r, j0 + s)
  __shared__ double invD[NB / 4][4][4];  // inverses of the 4 x 4 diagonal blocks of L
  __shared__ double Yb[4][NB + 1];     // block forward substitution: right-hand rows / solved rows
  __shared__ double Xb[4][NB + 1];
  __shared__ int bad_s;
  double* A = h + blockIdx.x * stride + k0 + k0 * ld;
  const int r = threadIdx.x & (NB - 1);
  const int part = threadIdx.x >> 6;  // 0..3
  double t[NB / 4];
  {
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
  if (threadIdx.x == 0) bad_s = 0;
#pragma unroll 1
  for (int q = 0; q < NB / 4; ++q) {
    const int j0 = 4 * q;
    double tq = t[0];
#pragma unroll
    for (int cc = 1; cc < NB / 4; ++cc) tq = (cc == q) ? t[cc] : tq;
    Pn[r][part] = tq;  // A(r, j0 + part) after the previous blocks' updates
    __syncthreads();
    if (threadIdx.x == 0) {  // 4 x 4 Cholesky of the diagonal block, then its inverse
      double L4[4][4] = {};
      for (int a = 0; a < 4; ++a) {
        double d = Pn[j0 + a][a];
        for (int b = 0; b < a; ++b) d -= L4[a][b] * L4[a][b];
        if (!(d > 0.0) || !isfinite(d)) {
          if (!bad_s) bad_s = j0 + a + 1;
          d = 1.0;  // keep going; the caller reports the failure
        }
        L4[a][a] = sqrt(d);
        const double rp = 1.0 / L4[a][a];
        for (int i = a + 1; i < 4; ++i) {
          double v = Pn[j0 + i][a];
          for (int b = 0; b < a; ++b) v -= L4[i][b] * L4[a][b];
          L4[i][a] = v * rp;
        }
      }
      double I4[4][4] = {};
      for (int a = 0; a < 4; ++a) {
        I4[a][a] = 1.0 / L4[a][a];
        for (int i = a + 1; i < 4; ++i) {
          double v = 0.0;
          for (int b = a; b < i; ++b) v += L4[i][b] * I4[b][a];
          I4[i][a] = -v / L4[i][i];
        }
      }
      for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
          invD[q][a][b] = I4[a][b];
          if (b <= a) Ls[j0 + b][j0 + a] = L4[a][b];
        }
    }
    __syncthreads();
    // panel rows below the block: L(r, j0 + part) = sum_{s <= part} A(r, j0 + s) (L44^{-1})(part, s)
    if (r >= j0 + 4) {
      double l = 0.0;
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2)
        if (s2 <= part) l += Pn[r][s2] * invD[q][part][s2];
      Ls[j0 + part][r] = l;
    }
    __syncthreads();
    if (r >= j0) {
      // this thread's column j0 + part of L (the diagonal block from Ls)
      const double l = (r >= j0 + 4) ? Ls[j0 + part][r] : (part <= r - j0 ? Ls[j0 + part][r] : 0.0);
#pragma unroll
      for (int cc = 0; cc < NB / 4; ++cc) t[cc] = (cc == q) ? l : t[cc];
    }
    if (r >= j0 + 4) {  // rank-4 trailing update, four rank-1 steps in column order
      double lr[4];
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) lr[s2] = Ls[j0 + s2][r];
#pragma unroll
      for (int cc = 0; cc < NB / 4; ++cc) {
        const int c = 4 * cc + part;
        if (cc > q && c <= r) {
#pragma unroll
          for (int s2 = 0; s2 < 4; ++s2) t[cc] -= lr[s2] * Ls[j0 + s2][c];
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int bad = bad_s;
    if (bad && bad <= kb && info[blockIdx.x] == 0) info[blockIdx.x] = static_cast<int>(k0 + bad);
  }
  // X = L^{-1} by block forward substitution: y(r, :) = e_r - sum_{i < j0} L(r, i) X(i, :)
  // for the rows of the current block, X_J = L_JJ^{-1} y_J.
  double x[NB / 4];
#pragma unroll
  for (int cc = 0; cc < NB / 4; ++cc) x[cc] = (4 * cc + part == r) ? 1.0 : 0.0;
#pragma unroll 1
  for (int q = 0; q < NB / 4; ++q) {
    const int j0 = 4 * q;
    if (r >= j0 && r < j0 + 4) {
#pragma unroll
      for (int cc = 0; cc < NB / 4; ++cc) Yb[r - j0][4 * cc + part] = x[cc];
    }
    __syncthreads();
    if (r >= j0 && r < j0 + 4) {
      const int a = r - j0;
#pragma unroll
      for (int cc = 0; cc < NB / 4; ++cc) {
        const int c = 4 * cc + part;
        double v = 0.0;
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2)
          if (s2 <= a) v += invD[q][a][s2] * Yb[s2][c];
        x[cc] = v;
        Xb[a][c] = v;
      }
    }
    __syncthreads();
    if (r >= j0 + 4) {
      double lr[4];
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) lr[s2] = Ls[j0 + s2][r];
#pragma unroll
      for (int cc = 0; cc < NB / 4; ++cc) {
        const int c = 4 * cc + part;
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2) x[cc] -= lr[s2] * Xb[s2][c];
      }
    }
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

// RP_POTRF_DIAG=1 selects the unblocked diagonal kernel (A/B).
bool blocked_diag() {
  static const bool on = [] {
    const char* e = std::getenv("RP_POTRF_DIAG");
    return !(e && e[0] == '1');
  }();
  return on;
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
                         int64_t stride_o, cudaStream_t stream, bool chain_high_priority) {
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
  // runs on its own stream, optionally at the highest stream priority.
  const cudaStream_t user = stream;
  cudaStream_t aux = nullptr, hi = nullptr;
  static const bool one_stream = [] {  // RP_FACTOR_ONE_STREAM=1: no lookahead streams (concurrency probe)
    const char* e = std::getenv("RP_FACTOR_ONE_STREAM");
    return e && e[0] == '1';
  }();
  if (one_stream) {
    aux = hi = user;
  } else {
    RP_CUDA(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
    int lo_p = 0, hi_p = 0;
    if (chain_high_priority) RP_CUDA(cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p));
    RP_CUDA(cudaStreamCreateWithPriority(&hi, cudaStreamNonBlocking, chain_high_priority ? hi_p : 0));
  }
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
  // (round 2 ran the chain's GEMMs on the cp.async kernel to keep one TMA
  // grid on the GPU at a time; with the stage-release fence of gemm_f64.cu
  // concurrent TMA grids are exact, profiles/r02_tma_release_race.txt)
  static const bool chain_cp_async = [] {  // RP_FACTOR_CHAIN_TMA=0: cp.async kernel on the critical chain (A/B)
    const char* e = std::getenv("RP_FACTOR_CHAIN_TMA");
    return e && e[0] == '0';
  }();
  const bool chain_no_tma = !one_stream && chain_cp_async;
  // C(rowc.., colc..colc+ncols) -= A21(rowc.., :) A21(colc..colc+ncols, :)^T over m rows; `lower`: a block
  // with rowc == colc, only its part on and below the diagonal
  auto panel_update = [&](int64_t rowc, int64_t colc, int64_t m, int64_t ncols, bool lower, int64_t k0, int kb,
                          cudaStream_t st) {
    GemmArgs g;
    g.opa = Op::N;
    g.opb = Op::T;
    g.m = m;
    g.n = ncols;
    g.k = kb;
    g.alpha = -1.0;
    g.beta = 1.0;
    g.a = h + rowc + k0 * ld;
    g.lda = ld;
    g.stride_a = stride;
    g.b = h + colc + k0 * ld;
    g.ldb = ld;
    g.stride_b = stride;
    g.c = h + rowc + colc * ld;
    g.ldc = ld;
    g.stride_c = stride;
    g.batch = batch;
    g.lower_only = lower;
    g.split_k = 1;
    g.no_tma = chain_no_tma && st != aux;
    dgemm(g, st);
  };
  cudaEvent_t prev_rest = nullptr;  // trailing update of the previous panel (aux stream)
  cudaEvent_t prev_col = nullptr;   // previous panel's update of this block column below its diagonal block (aux)
  for (int64_t k0 = 0; k0 < n; k0 += NB) {
    const int kb = static_cast<int>(std::min<int64_t>(NB, n - k0));
    if (blocked_diag())
      potrf_diag4<<<static_cast<unsigned>(batch), 256, 0, stream>>>(h, ld, stride, k0, kb, info.get());
    else
      potrf_diag<<<static_cast<unsigned>(batch), 256, 0, stream>>>(h, ld, stride, k0, kb, info.get());
    RP_LAUNCH_CHECK();
    const int64_t rows = n - k0 - kb;
    if (rows <= 0) break;
    if (prev_col) RP_CUDA(cudaStreamWaitEvent(stream, prev_col, 0));  // (the rows the panel solve reads)
    prev_col = nullptr;
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
      t.no_tma = chain_no_tma;
      dgemm(t, stream);
    }
    const int64_t r0 = k0 + kb;
    const int64_t nxt = std::min<int64_t>(NB, rows), rest = rows - nxt;
    cudaEvent_t rest_done = nullptr;
    if (rest > 0) {
      // aux stream: first the next block column below its diagonal block (the
      // next panel solve's input), then the columns beyond it
      cudaEvent_t panel_done = new_event();
      RP_CUDA(cudaEventRecord(panel_done, stream));
      RP_CUDA(cudaStreamWaitEvent(aux, panel_done, 0));
      panel_update(r0 + nxt, r0, rest, nxt, false, k0, kb, aux);
      prev_col = new_event();
      RP_CUDA(cudaEventRecord(prev_col, aux));
      panel_update(r0 + nxt, r0 + nxt, rest, rest, true, k0, kb, aux);
      rest_done = new_event();
      RP_CUDA(cudaEventRecord(rest_done, aux));
    }
    // chain: only the next diagonal block (the next potrf_diag's input); it
    // also needs the previous panel's update of that block (aux)
    if (prev_rest) RP_CUDA(cudaStreamWaitEvent(stream, prev_rest, 0));
    panel_update(r0, r0, nxt, nxt, true, k0, kb, stream);
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
  if (!one_stream) {
    release_workspace(aux);  // (the GEMMs above run unsplit; this only guards a recycled handle)
    release_workspace(hi);
    RP_CUDA(cudaStreamDestroy(aux));
    RP_CUDA(cudaStreamDestroy(hi));
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
        g1.tri_b = true;  // L11^{-1} is lower triangular: column j only needs k >= j
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
        g2.tri_a_lower = true;  // L22^{-1} is lower triangular: row i only needs k <= i
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
