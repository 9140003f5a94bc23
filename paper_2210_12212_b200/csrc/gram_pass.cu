// HBM-bound narrow passes over a dense column-major operator (see gram_pass.h).
//
// Algorithmic bytes: atv_narrow reads A once (8 n d bytes) plus y; gram_fused
// reads A once for z = A^T (A w) -- the reference evaluates the same product
// as two passes, apply_transpose(a, apply(a, x)) (matrix.cpp:168-172).
#include <algorithm>

#include "common.h"
#include "gram_pass.h"

namespace rpb {
namespace {

constexpr int kChunkRows = 8192;  // rows per warp task in atv_narrow

template <int K>
__device__ __forceinline__ void warp_reduce(double (&acc)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
}

// One warp per (column c, row chunk q): partial[q][c + k d] = sum over the
// chunk's rows of A[i, c] y[i, k].  Lane l handles rows l, l + 32, ... (two per
// step, unrolled), then a fixed xor-tree reduction.
template <int K>
__global__ void __launch_bounds__(256) atv_partial_kernel(const double* __restrict__ a, int64_t lda, int64_t n,
                                                          int64_t d, const double* __restrict__ y, int64_t chunks,
                                                          double* __restrict__ part) {
  const int64_t task = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (task >= d * chunks) return;
  const int64_t c = task % d, q = task / d;
  const int64_t r0 = q * kChunkRows, r1 = min(n, r0 + kChunkRows);
  const double* col = a + c * lda;
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  int64_t i = r0 + lane;
  for (; i + 96 < r1; i += 128) {
    const double a0 = __ldg(col + i), a1 = __ldg(col + i + 32), a2 = __ldg(col + i + 64), a3 = __ldg(col + i + 96);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double* yk = y + k * n;
      acc[k] = fma(a0, yk[i], acc[k]);
      acc[k] = fma(a1, yk[i + 32], acc[k]);
      acc[k] = fma(a2, yk[i + 64], acc[k]);
      acc[k] = fma(a3, yk[i + 96], acc[k]);
    }
  }
  for (; i < r1; i += 32) {
    const double a0 = __ldg(col + i);
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = fma(a0, y[i + k * n], acc[k]);
  }
  warp_reduce<K>(acc);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) part[q * d * K + c + k * d] = acc[k];
  }
}

__global__ void sum_chunks_kernel(const double* __restrict__ part, int64_t chunks, int64_t total,
                                  double* __restrict__ x) {
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s = part[idx];
    for (int64_t q = 1; q < chunks; ++q) s += part[q * total + idx];
    x[idx] = s;
  }
}

// ---- fused single-pass Gram: z = A^T (A w) ------------------------------------

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}

// Persistent CTAs; CTA b handles row blocks b, b + grid, ...  Each row block
// (R rows x d columns, R*8-byte segments of every column) is staged in shared
// memory with cp.async (double-buffered), y_blk = A_blk w is formed from it,
// and z_cta += A_blk^T y_blk accumulates in registers (columns t, t+256, ...).
template <int K>
__global__ void __launch_bounds__(256) gram_fused_kernel(const double* __restrict__ a, int64_t lda, int64_t n,
                                                         int64_t d, int R, const double* __restrict__ w,
                                                         double* __restrict__ ws, int cols_per_thread) {
  extern __shared__ __align__(16) double sm[];
  double* buf[2] = {sm, sm + static_cast<int64_t>(R) * d};
  double* yblk = sm + 2 * static_cast<int64_t>(R) * d;  // [R][K]
  double* red = yblk + R * K;                           // [256][K] partial dots
  const int t = threadIdx.x;
  const int64_t nblocks = (n + R - 1) / R;
  const bool vec = (R % 2 == 0) && (lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(a) & 15) == 0);

  auto stage = [&](int64_t blk, double* dst) {
    const int64_t r0 = blk * R;
    const int rr = static_cast<int>((n - r0) < R ? (n - r0) : R);
    if (vec && rr == R) {
      const int per_col = R / 2;
      for (int64_t e = t; e < d * per_col; e += blockDim.x) {
        const int64_t c = e / per_col;
        const int h = static_cast<int>(e - c * per_col);
        cp_async16(dst + c * R + 2 * h, a + c * lda + r0 + 2 * h);
      }
    } else {
      for (int64_t e = t; e < d * R; e += blockDim.x) {
        const int64_t c = e / R;
        const int r = static_cast<int>(e - c * R);
        if (r < rr)
          cp_async8(dst + c * R + r, a + c * lda + r0 + r);
        else
          dst[c * R + r] = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };

  double z[8][K];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int k = 0; k < K; ++k) z[j][k] = 0.0;

  int64_t blk = blockIdx.x;
  int cur = 0;
  if (blk < nblocks) stage(blk, buf[0]);
  for (; blk < nblocks; blk += gridDim.x) {
    const int64_t nxt = blk + gridDim.x;
    if (nxt < nblocks) {
      stage(nxt, buf[cur ^ 1]);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    const double* A = buf[cur];
    // y_blk[r][k] = sum_c A[r, c] w[c, k]: thread t -> row r = t % R, column
    // slice q = t / R (fixed slices, fixed reduction order below).
    const int slices = blockDim.x / R;
    {
      const int r = t % R, q = t / R;
      double acc[K];
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] = 0.0;
      if (q < slices) {
        for (int64_t c = q; c < d; c += slices) {
          const double v = A[c * R + r];
#pragma unroll
          for (int k = 0; k < K; ++k) acc[k] = fma(v, __ldg(w + c + k * d), acc[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) red[t * K + k] = acc[k];
    }
    __syncthreads();
    if (t < R) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double s = red[t * K + k];
        for (int q = 1; q < slices; ++q) s += red[(q * R + t) * K + k];
        yblk[t * K + k] = s;
      }
    }
    __syncthreads();
    // z[c] += sum_r A[r, c] y_blk[r]
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t c = t + static_cast<int64_t>(j) * blockDim.x;
      if (j >= cols_per_thread || c >= d) break;
      const double* col = A + c * R;
      for (int r = 0; r < R; ++r) {
        const double v = col[r];
#pragma unroll
        for (int k = 0; k < K; ++k) z[j][k] = fma(v, yblk[r * K + k], z[j][k]);
      }
    }
    __syncthreads();
    cur ^= 1;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t c = t + static_cast<int64_t>(j) * blockDim.x;
    if (j >= cols_per_thread || c >= d) break;
#pragma unroll
    for (int k = 0; k < K; ++k) ws[static_cast<int64_t>(blockIdx.x) * d * K + c + k * d] = z[j][k];
  }
}

template <int K>
void atv_launch(const double* a, int64_t lda, int64_t n, int64_t d, const double* y, double* x, cudaStream_t s) {
  const int64_t chunks = ceil_div(n, kChunkRows);
  const int64_t warps = d * chunks;
  DBuf<double> part(static_cast<size_t>(chunks * d * K), s);
  atv_partial_kernel<K><<<static_cast<unsigned>(ceil_div(warps * 32, 256)), 256, 0, s>>>(a, lda, n, d, y, chunks,
                                                                                          part.get());
  RP_LAUNCH_CHECK();
  sum_chunks_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(d * K, 256), 1184)), 256, 0, s>>>(
      part.get(), chunks, d * K, x);
  RP_LAUNCH_CHECK();
}

template <int K>
bool fused_launch(const double* a, int64_t lda, int64_t n, int64_t d, const double* w, double* z, cudaStream_t s) {
  // rows per block: R * d * 8 * 2 (double buffer) <= ~200 KB, R a multiple of 4
  int R = static_cast<int>(std::min<int64_t>(32, (200 * 1024) / (16 * d)));
  R &= ~3;
  if (R < 4 || d > 256 * 8) return false;
  const int cols_per_thread = static_cast<int>(ceil_div(d, 256));
  const int64_t nblocks = ceil_div(n, R);
  const int grid = static_cast<int>(std::min<int64_t>(nblocks, 148));
  const size_t smem = sizeof(double) * (2 * static_cast<size_t>(R) * d + R * K + 256 * K);
  RP_CUDA(cudaFuncSetAttribute(gram_fused_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  DBuf<double> ws(static_cast<size_t>(grid) * d * K, s);
  gram_fused_kernel<K><<<grid, 256, smem, s>>>(a, lda, n, d, R, w, ws.get(), cols_per_thread);
  RP_LAUNCH_CHECK();
  sum_chunks_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(d * K, 256), 1184)), 256, 0, s>>>(
      ws.get(), grid, d * K, z);
  RP_LAUNCH_CHECK();
  return true;
}

}  // namespace

void atv_narrow(const double* a, int64_t lda, int64_t n, int64_t d, const double* y, int64_t k, double* x,
                cudaStream_t stream) {
  require(k >= 1 && k <= kNarrowMax, "atv_narrow: 1 <= k <= 16");
  if (d <= 0) return;
  // Process columns of y in groups of the instantiated widths; each output
  // column's arithmetic is the same whatever group it falls in.
  int64_t j = 0;
  while (j < k) {
    const int64_t left = k - j;
    const double* yj = y + j * n;
    double* xj = x + j * d;
    if (left >= 8) {
      atv_launch<8>(a, lda, n, d, yj, xj, stream);
      j += 8;
    } else if (left >= 4) {
      atv_launch<4>(a, lda, n, d, yj, xj, stream);
      j += 4;
    } else if (left >= 2) {
      atv_launch<2>(a, lda, n, d, yj, xj, stream);
      j += 2;
    } else {
      atv_launch<1>(a, lda, n, d, yj, xj, stream);
      j += 1;
    }
  }
}

bool gram_fused(const double* a, int64_t lda, int64_t n, int64_t d, const double* w, int64_t k, double* z,
                cudaStream_t stream) {
  if (k < 1 || k > 8 || d <= 0 || n <= 0) return false;  // widths 1-4 and 8 are instantiated
  switch (k) {
    case 1: return fused_launch<1>(a, lda, n, d, w, z, stream);
    case 2: return fused_launch<2>(a, lda, n, d, w, z, stream);
    case 3: return fused_launch<3>(a, lda, n, d, w, z, stream);
    case 4: return fused_launch<4>(a, lda, n, d, w, z, stream);
    case 8: return fused_launch<8>(a, lda, n, d, w, z, stream);
    default: return false;
  }
}

}  // namespace rpb
