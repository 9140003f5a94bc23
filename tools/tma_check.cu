// Minimal TMA / mbarrier pipeline checker (no GEMM): the same producer-warp /
// consumer-warp ring as dgemm_tma_kernel (4-D tensor maps, boxes 4 elements
// wider than the tile, SWIZZLE_NONE, one elected producer lane, "full" /
// "empty" mbarriers), but the consumers VERIFY every element of every stage
// against the value its global coordinate must hold, and log what they saw
// instead.  Two instances with different arrays run on two streams (optionally
// at different priorities), or in two processes time-sharing the GPU, to tell
// a pipeline bug of ours from a platform effect:
//   * a mismatch whose value belongs to the OTHER array     -> descriptor mix-up
//   * a mismatch whose value is the stage's previous tile   -> read before the copy landed (RAW)
//   * a mismatch whose value is the stage's next tile       -> overwritten before the read (WAR)
// Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda -I paper_2210_12212_b200/csrc \
//        tools/tma_check.cu -o gpurun_out/tma_check && gpurun_out/tma_check [reps] [prio 0/1] [passes]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2210_12212_b200/csrc/tma_util.cuh"

namespace rpb {
namespace tma {
PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}
}  // namespace tma
}  // namespace rpb

using namespace rpb;

constexpr int BM = 64, BK = 16, STAGES = 4, WARPS = 4;
constexpr int LD = BM + 4;
constexpr int STAGE = LD * BK;  // doubles

struct Bad {
  unsigned long long got, want;
  int tile, kt, idx, warp, inst;
};

// value of element (row r, column c) of instance `inst`
__host__ __device__ inline unsigned long long value_of(int inst, long long r, long long c, long long rows) {
  return (static_cast<unsigned long long>(inst + 1) << 56) | static_cast<unsigned long long>(c * rows + r);
}

__global__ void fill_kernel(unsigned long long* x, long long rows, long long cols, int inst) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < rows * cols;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    x[i] = value_of(inst, i % rows, i / rows, rows);
}

// X is rows x cols column-major (inner = rows).  CTA b walks the row tile
// m0 = (b % tiles_m) * BM over all columns, BK columns per stage, `passes` times.
__global__ void __launch_bounds__((WARPS + 1) * 32)
    tma_check_kernel(const __grid_constant__ CUtensorMap map, long long rows, long long cols, int inst, int passes,
                     unsigned long long* nbad, Bad* log, int log_cap) {
  extern __shared__ __align__(128) double smem_raw[];
  double* smem = smem_raw + (((128u - (tma::smem_u32(smem_raw) & 127u)) & 127u) >> 3);
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tiles_m = static_cast<int>(rows / BM);
  const int m0 = (blockIdx.x % tiles_m) * BM;
  const int ktiles = static_cast<int>(cols / BK) * passes;
  const int kper = static_cast<int>(cols / BK);
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], WARPS);
    }
    tma::fence_barrier_init();
  }
  __syncthreads();
  constexpr uint32_t kBytes = STAGE * 8;
  if (warp == WARPS) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kt = 0; kt < ktiles; ++kt) {
        tma::mbar_wait(&empty[stage], phase ^ 1);
        tma::mbar_arrive_expect_tx(&full[stage], kBytes);
        tma::load_4d(smem + stage * STAGE, &map, m0, (kt % kper) * BK, 0, 0, &full[stage]);
        if (++stage == STAGES) stage = 0, phase ^= 1;
      }
    }
  } else {
    int stage = 0;
    uint32_t phase = 0;
    unsigned long long bad = 0;
    for (int kt = 0; kt < ktiles; ++kt) {
      tma::mbar_wait(&full[stage], phase);
      const unsigned long long* st = reinterpret_cast<const unsigned long long*>(smem + stage * STAGE);
      // every warp checks the whole stage (like the GEMM: every warp reads A or B rows of the stage)
      for (int idx = lane; idx < BM * BK; idx += 32) {
        const int r = idx % BM, c = idx / BM;
        const unsigned long long got = st[c * LD + r];
        const unsigned long long want = value_of(inst, m0 + r, static_cast<long long>(kt % kper) * BK + c, rows);
        if (got != want) {
          const unsigned long long slot = atomicAdd(nbad, 1ull);
          if (slot < static_cast<unsigned long long>(log_cap))
            log[slot] = Bad{got, want, static_cast<int>(blockIdx.x), kt, idx, warp, inst};
          ++bad;
        }
      }
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&empty[stage]);
      if (++stage == STAGES) stage = 0, phase ^= 1;
    }
    (void)bad;
  }
}

static bool make_map(CUtensorMap* map, const void* base, long long rows, long long cols) {
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols), 1, 1};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(rows) * 8, static_cast<cuuint64_t>(rows * cols) * 8,
                                 static_cast<cuuint64_t>(rows * cols) * 8};
  const cuuint32_t box[4] = {LD, BK, 1, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return tma::encoder()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 20;
  const bool prio = argc > 2 ? atoi(argv[2]) != 0 : true;
  const int passes = argc > 3 ? atoi(argv[3]) : 8;
  const long long rows = 1024, cols = 65536;  // 512 MB each: larger than L2
  unsigned long long *X[2], *nbad;
  Bad* log;
  const int cap = 64;
  for (int i = 0; i < 2; ++i) {
    cudaMalloc(&X[i], rows * cols * 8);
    fill_kernel<<<148 * 8, 256>>>(X[i], rows, cols, i);
  }
  cudaMalloc(&nbad, 8);
  cudaMalloc(&log, sizeof(Bad) * cap);
  cudaMemset(nbad, 0, 8);
  int lo, hi;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaStream_t s[2];
  cudaStreamCreateWithPriority(&s[0], cudaStreamNonBlocking, prio ? lo : 0);
  cudaStreamCreateWithPriority(&s[1], cudaStreamNonBlocking, prio ? hi : 0);
  CUtensorMap map[2];
  for (int i = 0; i < 2; ++i)
    if (!make_map(&map[i], X[i], rows, cols)) {
      printf("tensor map encode failed\n");
      return 1;
    }
  const int smem = STAGES * STAGE * 8 + 128;
  cudaFuncSetAttribute(tma_check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaDeviceSynchronize();
  unsigned long long total = 0;
  for (int r = 0; r < reps; ++r) {
    // instance 0 (low priority): one long grid, 3 CTAs per SM worth of tiles;
    // instance 1 (high priority): a chain of short grids, like the recursion's GEMMs
    tma_check_kernel<<<16 * 32, (WARPS + 1) * 32, smem, s[0]>>>(map[0], rows, cols, 0, passes, nbad, log, cap);
    for (int q = 0; q < 40; ++q)
      tma_check_kernel<<<16 * (2 + q % 12), (WARPS + 1) * 32, smem, s[1]>>>(map[1], rows, cols / 64, 1, 1, nbad, log,
                                                                            cap);
    cudaDeviceSynchronize();
    unsigned long long h = 0;
    cudaMemcpy(&h, nbad, 8, cudaMemcpyDeviceToHost);
    if (h != total) {
      printf("rep %d: %llu new mismatches\n", r, h - total);
      total = h;
    }
  }
  printf("tma_check%s: %llu mismatching words in %d reps; err %s\n", prio ? " (low/high priority)" : " (one priority)",
         total, reps, cudaGetErrorString(cudaGetLastError()));
  if (total) {
    std::vector<Bad> hl(cap);
    cudaMemcpy(hl.data(), log, sizeof(Bad) * cap, cudaMemcpyDeviceToHost);
    for (int i = 0; i < cap && i < static_cast<int>(total); ++i)
      printf("  inst %d cta %d kt %d warp %d idx %d (r %d, c %d): got %016llx want %016llx\n", hl[i].inst, hl[i].tile,
             hl[i].kt, hl[i].warp, hl[i].idx, hl[i].idx % BM, hl[i].idx / BM, hl[i].got, hl[i].want);
  }
  return 0;
}
