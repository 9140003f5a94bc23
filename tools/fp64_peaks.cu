// Microbenchmark: FP64 pipe peaks on sm_100a (DFMA, DMMA m8n8k4, DMMA m16n8k16).
// Used once to pick the FP64 roofline denominator and the GEMM micro-kernel shape.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = fma(r[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += r[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma884_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma16816_loop(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 + i;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 148; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int warps : {4, 8, 16}) {
    int blocks = sms * 4, threads = warps * 32 / 4 * 4; (void)threads;
    int iters = 20000;
    // DFMA: 16 chains per thread
    dfma_loop<<<blocks, warps * 32>>>(d, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, warps * 32>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * iters * (double)blocks * warps * 32;
    printf("DFMA     warps/blk=%2d blocks=%d: %.2f TFLOP/s\n", warps, blocks, fl / ms / 1e9);
    dmma884_loop<<<blocks, warps * 32>>>(d, 100);
    cudaEventRecord(e0);
    dmma884_loop<<<blocks, warps * 32>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * warps;
    printf("DMMA884  warps/blk=%2d blocks=%d: %.2f TFLOP/s\n", warps, blocks, fl / ms / 1e9);
    dmma16816_loop<<<blocks, warps * 32>>>(d, 100);
    cudaEventRecord(e0);
    dmma16816_loop<<<blocks, warps * 32>>>(d, iters / 4);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * 8 * 16 * 4 * (double)(iters / 4) * blocks * warps;
    printf("DMMA16816 warps/blk=%2d blocks=%d: %.2f TFLOP/s\n", warps, blocks, fl / ms / 1e9);
  }
  cudaError_t err = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}
