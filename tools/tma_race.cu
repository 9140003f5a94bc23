// Concurrency probe for the TMA GEMM: the same GEMM sequences run serially
// and then concurrently on two streams (one host thread), results compared
// bitwise.  Build + run on the GPU:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda -I paper_2210_12212_b200/csrc \
//        tools/tma_race.cu -o gpurun_out/tma_race && gpurun_out/tma_race
// Modes (argv[1]): 0 = both TMA, 1 = side stream cp.async, 2 = split_k forced 1 on both,
//   argv[3] = 0: both streams at one priority (default: side low, chain high)
//                  3 = no lower_only on the side SYRK, 4 = the path's SYRK layout (A^T A, tile 3, split 4)
#include "../paper_2210_12212_b200/csrc/gemm_f64.cu"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

using namespace rpb;

static void fill(double* d, size_t n, unsigned seed) {
  std::vector<double> h(n);
  uint64_t x = seed * 0x9E3779B97F4A7C15ull + 1;
  for (auto& v : h) {
    x ^= x << 13, x ^= x >> 7, x ^= x << 17;
    v = static_cast<double>(x >> 11) * 0x1.0p-53 - 0.5;
  }
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int reps = argc > 2 ? atoi(argv[2]) : 10;
  const int64_t n = 65536, d = 1024, mm = 2048;
  double *A, *S, *G, *Gref, *W, *X, *Y, *Yref;
  cudaMalloc(&A, n * d * 8);
  cudaMalloc(&S, mm * d * 8);
  cudaMalloc(&G, d * d * 8);
  cudaMalloc(&Gref, d * d * 8);
  cudaMalloc(&W, d * 2048 * 8);
  cudaMalloc(&X, 32 * d * 64 * 8);
  cudaMalloc(&Y, 40 * d * 2048 * 8);
  cudaMalloc(&Yref, 40 * d * 2048 * 8);
  fill(A, n * d, 1);
  fill(S, mm * d, 2);
  fill(W, d * 2048, 3);
  fill(X, 32 * d * 64, 4);
  cudaStream_t s1, s2;
  int lo, hi;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  const bool prio = !(argc > 3 && atoi(argv[3]) == 0);  // argv[3] = 0: both streams at the default priority
  cudaStreamCreateWithPriority(&s1, cudaStreamNonBlocking, prio ? lo : 0);
  cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, prio ? hi : 0);

  auto side = [&](double* out, cudaStream_t st) {  // the side-stream Gram SYRK
    GemmArgs g;
    g.opa = Op::N, g.opb = Op::T, g.m = d, g.n = d, g.k = n;
    g.a = A, g.lda = d, g.b = A, g.ldb = d, g.c = out, g.ldc = d;
    if (mode == 4) {  // the path's layout: A n x d column-major, G = A^T A, 64 x 32 tile, split 4, mirrored
      g.opa = Op::T, g.opb = Op::N, g.lda = n, g.ldb = n;
      g.force_tile = 3, g.split_k = 4, g.mirror = true;
    }
    g.lower_only = mode != 3;
    g.no_tma = mode == 1;
    if (mode == 2) g.split_k = 1;
    dgemm(g, st);
  };
  auto chain = [&](double* out, cudaStream_t st) {  // basis-like GEMMs on the critical stream
    for (int i = 0; i < 40; ++i) {
      GemmArgs g;
      const int64_t cols = 32 + 48 * (i % 40);
      g.m = d, g.n = cols, g.k = d;
      g.a = S, g.lda = d, g.b = W, g.ldb = d, g.c = out + i * d * 2048, g.ldc = d;
      if (mode == 2) g.split_k = 1;
      dgemm(g, st);
    }
  };
  side(Gref, s1);
  chain(Yref, s2);
  cudaDeviceSynchronize();
  int bad_g = 0, bad_y = 0;
  std::vector<double> h1(d * d), h2(d * d);
  std::vector<double> y1(40 * d * 2048), y2(40 * d * 2048);
  cudaMemcpy(h1.data(), Gref, d * d * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(y1.data(), Yref, y1.size() * 8, cudaMemcpyDeviceToHost);
  for (int r = 0; r < reps; ++r) {
    cudaMemset(G, 0, d * d * 8);
    cudaMemset(Y, 0, y1.size() * 8);
    cudaDeviceSynchronize();
    side(G, s1);
    chain(Y, s2);
    cudaDeviceSynchronize();
    cudaMemcpy(h2.data(), G, d * d * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(y2.data(), Y, y2.size() * 8, cudaMemcpyDeviceToHost);
    int64_t dg = 0, dy = 0;
    for (int64_t j = 0; j < d; ++j)
      for (int64_t i = j; i < d; ++i) dg += memcmp(&h1[j * d + i], &h2[j * d + i], 8) != 0;
    for (size_t i = 0; i < y1.size(); ++i) dy += memcmp(&y1[i], &y2[i], 8) != 0;
    bad_g += dg != 0, bad_y += dy != 0;
    printf("rep %d: gram mismatches %lld, chain mismatches %lld\n", r, (long long)dg, (long long)dy);
  }
  printf("mode %d%s: %d/%d gram runs differ, %d/%d chain runs differ; err %s\n", mode,
         prio ? " (side low / chain high priority)" : " (one priority)", bad_g, reps, bad_y, reps,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
