// Concurrency probe: the C2 SRHT sketch on a high-priority stream next to the
// Gram SYRK (lower + mirror, auto tile) on a low-priority stream, each
// compared bitwise with its serial result.  Links the library's objects:
//   make -C paper_2210_12212_b200 && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//     -I paper_2210_12212_b200/csrc -I include tools/sketch_race.cu paper_2210_12212_b200/build/{gemm_f64,draws,sketch,mt_host}.o \
//     -lcuda -o gpurun_out/sketch_race && gpurun_out/sketch_race [side_no_tma] [reps] [force_tile]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "gemm_f64.h"
#include "sketch.h"

using namespace rpb;

int main(int argc, char** argv) {
  const bool side_no_tma = argc > 1 && atoi(argv[1]) != 0;
  const int reps = argc > 2 ? atoi(argv[2]) : 6;
  const int tile = argc > 3 ? atoi(argv[3]) : -1;
  const int64_t n = 65536, d = 1024, m = 2048;
  std::vector<double> h(n * d);
  uint64_t x = 88172645463325252ull;
  for (auto& v : h) {
    x ^= x << 13, x ^= x >> 7, x ^= x << 17;
    v = static_cast<double>(x >> 11) * 0x1.0p-53 - 0.5;
  }
  double *A, *G, *SA;
  cudaMalloc(&A, n * d * 8);
  cudaMalloc(&G, d * d * 8);
  cudaMalloc(&SA, m * d * 8);
  cudaMemcpy(A, h.data(), n * d * 8, cudaMemcpyHostToDevice);
  int lo, hi;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaStream_t s_side, s_hi;
  cudaStreamCreateWithPriority(&s_side, cudaStreamNonBlocking, lo);
  cudaStreamCreateWithPriority(&s_hi, cudaStreamNonBlocking, hi);
  OpView op;
  op.n_global = n, op.row0 = 0, op.n_loc = n, op.d = d, op.a = A, op.ld = n;
  SketchSpecC spec;
  spec.kind = kSrht, spec.m = m, spec.n = n, spec.s = 1, spec.seed = 12345;
  auto syrk = [&](cudaStream_t st) {
    GemmArgs g;
    g.opa = op.op_mt(), g.opb = op.op_m(), g.m = d, g.n = d, g.k = n;
    g.a = A, g.lda = n, g.b = A, g.ldb = n, g.c = G, g.ldc = d;
    g.lower_only = true, g.mirror = true, g.no_tma = side_no_tma, g.force_tile = tile;
    dgemm(g, st);
  };
  std::vector<double> g0(d * d), s0(m * d), g1(d * d), s1(m * d);
  syrk(s_side);
  cudaDeviceSynchronize();
  sketch_apply(spec, op, SA, s_hi);
  cudaDeviceSynchronize();
  cudaMemcpy(g0.data(), G, d * d * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(s0.data(), SA, m * d * 8, cudaMemcpyDeviceToHost);
  int bad_g = 0, bad_s = 0;
  for (int r = 0; r < reps; ++r) {
    cudaMemset(G, 0, d * d * 8);
    cudaMemset(SA, 0, m * d * 8);
    cudaDeviceSynchronize();
    syrk(s_side);
    sketch_apply(spec, op, SA, s_hi);
    cudaDeviceSynchronize();
    cudaMemcpy(g1.data(), G, d * d * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(s1.data(), SA, m * d * 8, cudaMemcpyDeviceToHost);
    int64_t dg = 0, ds = 0, first = -1;
    for (int64_t i = 0; i < d * d; ++i)
      if (memcmp(&g0[i], &g1[i], 8)) {
        if (first < 0) first = i;
        ++dg;
      }
    for (int64_t i = 0; i < m * d; ++i) ds += memcmp(&s0[i], &s1[i], 8) != 0;
    bad_g += dg != 0, bad_s += ds != 0;
    printf("rep %d: G mismatches %lld (first at row %lld col %lld), SA mismatches %lld\n", r, (long long)dg,
           (long long)(first >= 0 ? first % d : -1), (long long)(first >= 0 ? first / d : -1), (long long)ds);
  }
  printf("side_no_tma %d tile %d: %d/%d G differ, %d/%d SA differ; %s\n", side_no_tma, tile, bad_g, reps, bad_s, reps,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
