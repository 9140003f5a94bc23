// GEMM tile/split tuner: times every tile shape of paper_2210_12212_b200's
// DMMA GEMM on the shapes the IHS-BIN path issues.  Build + run on the GPU:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2210_12212_b200/csrc \
//        tools/gemm_tune.cu -o gpurun_out/gemm_tune && gpurun_out/gemm_tune
#include "../paper_2210_12212_b200/csrc/gemm_f64.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

using namespace rpb;

// (operands in [-0.5, 0.5): every tile must reproduce the auto tile's bits -- same k order per element)
__global__ void tune_fill(double* x, size_t n, unsigned long long seed) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    unsigned long long z = (i + 1) * 0x9E3779B97F4A7C15ull + seed;
    z ^= z >> 29, z *= 0xBF58476D1CE4E5B9ull, z ^= z >> 32;
    x[i] = static_cast<double>(z >> 11) * 0x1.0p-53 - 0.5;
  }
}
__global__ void tune_diff(const double* x, const double* y, size_t n, unsigned long long* bad) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    if (__double_as_longlong(x[i]) != __double_as_longlong(y[i])) atomicAdd(bad, 1ull);
}

struct Shape {
  const char* name;
  Op opa, opb;
  int64_t m, n, k, batch;
  bool lower, col_stable;
  int split = 0;  // > 0: forced (the recursion's P product runs unsplit, fused epilogue)
};

int main(int argc, char** argv) {
  // optional: gemm_tune SHAPE TILE -> one shape/tile, few iterations (for ncu)
  const int only_shape = argc > 2 ? atoi(argv[1]) : -1, only_tile = argc > 2 ? atoi(argv[2]) : -9;
  std::vector<Shape> shapes = {
      {"GW g=1   (1024x32x1024)", Op::N, Op::N, 1024, 32, 1024, 1, false, true},
      {"GW g=8   (1024x256x1024)", Op::N, Op::N, 1024, 256, 1024, 1, false, true},
      {"GW g=32  (1024x1024x1024)", Op::N, Op::N, 1024, 1024, 1024, 1, false, true},
      {"GW g=63  (1024x2016x1024)", Op::N, Op::N, 1024, 2016, 1024, 1, false, true},
      {"P  g=1   32x(1024x2x1024)", Op::N, Op::N, 1024, 2, 1024, 32, false, true, 1},
      {"P  g=15  32x(1024x16x1024)", Op::N, Op::N, 1024, 16, 1024, 32, false, true, 1},
      {"P  g=31  32x(1024x32x1024)", Op::N, Op::N, 1024, 32, 1024, 32, false, true, 1},
      {"P  g=35  32x(1024x36x1024)", Op::N, Op::N, 1024, 36, 1024, 32, false, true, 1},
      {"P  g=41  32x(1024x42x1024)", Op::N, Op::N, 1024, 42, 1024, 32, false, true, 1},
      {"P  g=47  32x(1024x48x1024)", Op::N, Op::N, 1024, 48, 1024, 32, false, true, 1},
      {"P  g=55  32x(1024x56x1024)", Op::N, Op::N, 1024, 56, 1024, 32, false, true, 1},
      {"P  g=63  32x(1024x64x1024)", Op::N, Op::N, 1024, 64, 1024, 32, false, true, 1},
      // quantization / overhead probes of the recursion's P product: 16 x batch CTAs of 64 x 64 on 296 slots
      {"P  N=64 batch 37 (2 full waves)", Op::N, Op::N, 1024, 64, 1024, 37, false, true, 1},
      {"P  N=64 batch 74 (4 full waves)", Op::N, Op::N, 1024, 64, 1024, 74, false, true, 1},
      {"P  N=64 batch 32, K = 4096", Op::N, Op::N, 1024, 64, 4096, 32, false, true, 1},
      {"SYRK A^T A (1024,65536)", Op::T, Op::N, 1024, 1024, 65536, 1, true, false},
      {"SYRK A^T A (2048,262144) [C3/4]", Op::T, Op::N, 2048, 2048, 262144, 1, true, false},
      {"square 4096^3", Op::N, Op::N, 4096, 4096, 4096, 1, false, false},
      {"sketch S^T A 2048x1024x65536", Op::T, Op::N, 2048, 1024, 65536, 1, false, false},
  };
  cudaStream_t s;
  cudaStreamCreate(&s);
  size_t maxe = 0;
  for (auto& sh : shapes)
    maxe = std::max(maxe, (size_t)std::max({sh.m * sh.k * sh.batch, sh.k * sh.n * sh.batch, sh.m * sh.n * sh.batch}));
  double *a, *b, *c, *cref;
  unsigned long long* bad;
  cudaMalloc(&a, maxe * 8);
  cudaMalloc(&b, maxe * 8);
  cudaMalloc(&c, maxe * 8);
  cudaMalloc(&cref, maxe * 8);
  cudaMalloc(&bad, 8);
  tune_fill<<<148 * 8, 256>>>(a, maxe, 1);
  tune_fill<<<148 * 8, 256>>>(b, maxe, 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (size_t si = 0; si < shapes.size(); ++si) {
    auto& sh = shapes[si];
    if (only_shape >= 0 && static_cast<int>(si) != only_shape) continue;
    printf("%-32s", sh.name);
    for (int tile = -1; tile < kNumTiles; ++tile) {
      if (only_tile != -9 && tile != only_tile) continue;
      GemmArgs g;
      g.opa = sh.opa;
      g.opb = sh.opb;
      g.m = sh.m;
      g.n = sh.n;
      g.k = sh.k;
      g.a = a;
      g.lda = sh.opa == Op::N ? sh.m : sh.k;
      g.stride_a = sh.m * sh.k;
      g.b = b;
      g.ldb = sh.opb == Op::N ? sh.k : sh.n;
      g.stride_b = sh.k * sh.n;
      g.c = c;
      g.ldc = sh.m;
      g.stride_c = sh.m * sh.n;
      g.batch = sh.batch;
      g.lower_only = sh.lower;
      g.col_stable = sh.col_stable;
      g.split_k = sh.split;
      g.force_tile = tile;
      for (int w = 0; w < 3; ++w) dgemm(g, s);
      cudaEventRecord(e0, s);
      const int iters = only_shape >= 0 ? 2 : 10;
      for (int it = 0; it < iters; ++it) dgemm(g, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * sh.m * sh.n * sh.k * sh.batch * (sh.lower ? 0.5 : 1.0);
      // bits against the auto tile (lower_only shapes leave the upper triangle untouched: same in both)
      const size_t ce = static_cast<size_t>(sh.m * sh.n * sh.batch);
      unsigned long long hb = 0;
      if (tile < 0) {
        cudaMemcpyAsync(cref, c, ce * 8, cudaMemcpyDeviceToDevice, s);
      } else {
        cudaMemsetAsync(bad, 0, 8, s);
        tune_diff<<<148 * 4, 256, 0, s>>>(c, cref, ce, bad);
        cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, s);
      }
      cudaStreamSynchronize(s);
      printf(" %s%6.1f%s", tile < 0 ? "auto:" : "", fl / (ms / iters * 1e-3) / 1e12, hb ? "!" : "");
    }
    printf("   TF/s [auto, 128x128, 64x64, 128x32, 64x32, 128x16, 64x128, 128x64, 64x128w4, 128x64w4, 64x128k32, 128x64k32, 64x48, 128x48, 128x{24,40,48,56,64}, 32x{16..64 step 8} 4x1 warps, 32x{32,48,64} 2x2 warps]; ! = bits differ from auto\n");
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
