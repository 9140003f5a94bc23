// Microbenchmark: DMMA m8n8k4 fed from shared memory (the GEMM warp-tile inner
// loop without global loads or barriers), to separate the operand-feed cost
// from the pipeline/barrier cost of dgemm_kernel.
#include <cstdio>
#include <cuda_runtime.h>

template <int FM, int FN>
__global__ void dmma_lds(double* out, int iters) {
  __shared__ double sm[2][16][132];  // [A|B][k][mn]
  for (int i = threadIdx.x; i < 2 * 16 * 132; i += blockDim.x) (&sm[0][0][0])[i] = i * 1e-3;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r8 = lane >> 2, k4 = lane & 3;
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0;
  const int wo = (warp & 1) * 8 * FM;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kk = 0; kk < 16; kk += 4) {
      double af[FM], bf[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = sm[0][kk + k4][wo + i * 8 + r8];
#pragma unroll
      for (int j = 0; j < FN; ++j) bf[j] = sm[1][kk + k4][wo + j * 8 + r8];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[i][j][0]), "+d"(acc[i][j][1]) : "d"(af[i]), "d"(bf[j]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 12345.678) out[0] = s;
}

template <int FM, int FN>
void run(const char* name, int warps, int blocks_per_sm) {
  double* d;
  cudaMalloc(&d, 64);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * blocks_per_sm, iters = 4000;
  dmma_lds<FM, FN><<<blocks, warps * 32>>>(d, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  dmma_lds<FM, FN><<<blocks, warps * 32>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * 8 * 8 * 4 * FM * FN * 4.0 * iters * blocks * warps;
  printf("%-10s warps/blk=%2d blk/SM=%d: %.2f TFLOP/s\n", name, warps, blocks_per_sm, fl / ms / 1e9);
  cudaFree(d);
}

int main() {
  run<4, 4>("4x4", 8, 2);
  run<4, 4>("4x4", 4, 4);
  run<4, 8>("4x8", 4, 2);
  run<4, 8>("4x8", 8, 2);
  run<8, 4>("8x4", 4, 2);
  run<2, 4>("2x4", 8, 3);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
