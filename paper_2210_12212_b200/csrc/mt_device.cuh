// Device-side std::mt19937_64 building blocks (see mt19937.h for conventions).
#pragma once

#include <cstdint>

#include "mt19937.h"

namespace rpb {
namespace mt {

__device__ __forceinline__ uint64_t d_temper(uint64_t x) {
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

__device__ __forceinline__ uint64_t d_twist(uint64_t x0, uint64_t x1, uint64_t xm) {
  const uint64_t y = (x0 & kUpper) | (x1 & kLower);
  return xm ^ (y >> 1) ^ ((y & 1ULL) ? kMatrixA : 0ULL);
}

// SeededRng::uniform01 (rng.hpp:26-28).
__device__ __forceinline__ double d_uniform01(uint64_t w) {
  return static_cast<double>((w >> 11) + 1) * 0x1.0p-53;
}

// Block-cooperative generator.  Needs blockDim.x >= 156 and 2 x 312 words of
// shared memory.  After step(), cur[0..311] holds the untempered outputs
// q..q+311 (= the new window W_{q+312}) and prev() the old window W_q.
struct BlockGen {
  uint64_t* cur;
  uint64_t* nxt;

  __device__ void init(uint64_t* smem2x312) {
    cur = smem2x312;
    nxt = smem2x312 + kN;
  }
  __device__ void load(const uint64_t* g) {
    for (int i = threadIdx.x; i < kN; i += blockDim.x) cur[i] = g[i];
    __syncthreads();
  }
  __device__ void step() {
    const int t = threadIdx.x;
    if (t < kM) nxt[t] = d_twist(cur[t], cur[t + 1], cur[t + kM]);
    __syncthreads();
    if (t < kM) {
      const int k = t + kM;
      nxt[k] = d_twist(cur[k], (k + 1 < kN) ? cur[k + 1] : nxt[0], nxt[k - kM]);
    }
    __syncthreads();
    uint64_t* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
  // Window at relative position s in [0, 312] of the last step: prev[s..] ++ cur[..s).
  __device__ void save(uint64_t* g, int s) const {
    for (int i = threadIdx.x; i < kN; i += blockDim.x) g[i] = (i + s < kN) ? nxt[i + s] : cur[i + s - kN];
  }
};

}  // namespace mt
}  // namespace rpb
