// HBM-bound narrow passes over a dense column-major operator (see gram_pass.h).
//
// Algorithmic bytes: atv_narrow reads A once (8 n d bytes) plus y; gram_fused
// reads A once for z = A^T (A w) -- the reference evaluates the same product
// as two passes, apply_transpose(a, apply(a, x)) (matrix.cpp:168-172).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "common.h"
#include "gram_pass.h"

namespace rpb {
namespace {

constexpr int kChunkRows = 8192;  // rows per warp task in atv_narrow
constexpr int kRB = 64;           // rows per atv step: 2 per lane, one 16-byte load per column

template <int K>
__device__ __forceinline__ void warp_reduce(double (&acc)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
}

// One warp per (column c, row chunk q): partial[q][c + k d] = sum over the
// chunk's rows of A[i, c] y[i, k].  Lane l loads rows 2l, 2l+1 of every
// 64-row step (16-byte loads, eight steps in flight), then the xor tree.
template <int K>
__global__ void __launch_bounds__(256) atv_partial_kernel(const double* __restrict__ a, int64_t lda, int64_t n,
                                                          int64_t d, const double* __restrict__ y, int64_t chunks,
                                                          double* __restrict__ part, bool vec) {
  const int64_t task = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (task >= d * chunks) return;
  const int64_t c = task % d, q = task / d;
  const int64_t r0 = q * kChunkRows, r1 = min(n, r0 + kChunkRows);
  const double* col = a + c * lda;
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  int64_t i = r0;
  if (vec) {
    constexpr int U = 8;
    for (; i + U * kRB <= r1; i += U * kRB) {
      double2 av[U];
#pragma unroll
      for (int u = 0; u < U; ++u) av[u] = __ldg(reinterpret_cast<const double2*>(col + i + u * kRB + 2 * lane));
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const double2 yv = __ldg(reinterpret_cast<const double2*>(y + k * n + i + u * kRB + 2 * lane));
          acc[k] = fma(av[u].x, yv.x, acc[k]);
          acc[k] = fma(av[u].y, yv.y, acc[k]);
        }
    }
  }
  for (; i < r1; i += kRB) {
    const int64_t ra = i + 2 * lane, rb = ra + 1;
    const double a0 = ra < r1 ? __ldg(col + ra) : 0.0, a1 = rb < r1 ? __ldg(col + rb) : 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double y0 = ra < r1 ? y[k * n + ra] : 0.0, y1 = rb < r1 ? y[k * n + rb] : 0.0;
      acc[k] = fma(a0, y0, acc[k]);
      acc[k] = fma(a1, y1, acc[k]);
    }
  }
  warp_reduce<K>(acc);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) part[q * d * K + c + k * d] = acc[k];
  }
}

// Deterministic sum over the chunk partials, two fixed levels: 16 threads per
// output each sum the chunks g, g + 16, g + 32, ... (in order), then the 16
// group sums are added in group order.  256 threads = 16 outputs x 16 groups.
__global__ void __launch_bounds__(256) sum_chunks_tree_kernel(const double* __restrict__ part, int64_t chunks,
                                                              int64_t total, double* __restrict__ x) {
  __shared__ double red[16][17];
  // (launched programmatically after the pass that writes `part`: resident early, waits here for that grid;
  // a no-op under a plain launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int o = threadIdx.x & 15, g = threadIdx.x >> 4;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * 16 + o;
  double s = 0.0;
  if (idx < total) {
    int64_t q = g;
    if (q < chunks) s = part[q * total + idx];
    for (q += 16; q < chunks; q += 16) s += part[q * total + idx];
  }
  red[g][o] = s;
  __syncthreads();
  if (g == 0 && idx < total) {
    double t = red[0][o];
    for (int h = 1; h < 16 && h < chunks; ++h) t += red[h][o];
    x[idx] = t;
  }
}

__global__ void sum_chunks_kernel(const double* __restrict__ part, int64_t chunks, int64_t total,
                                  double* __restrict__ x) {
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // sum in chunk order; loads issued eight at a time (latency overlap)
    double s = part[idx];
    int64_t q = 1;
    for (; q + 8 <= chunks; q += 8) {
      double t8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) t8[u] = part[(q + u) * total + idx];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += t8[u];
    }
    for (; q < chunks; ++q) s += part[q * total + idx];
    x[idx] = s;
  }
}

// ---- TMA-staged column passes: z = A^T (A w)  and  x = A^T y ----------------
//
// A (n x d, column-major) is cut into 32-row blocks; persistent CTAs (one per
// SM) own blocks b, b + grid, ...  A producer warp streams 16 KB tiles of A
// through a shared-memory ring with 2-D TMA (cp.async.bulk.tensor, completion
// on mbarriers), so the memory stream runs ahead of the math with no
// registers held; sixteen consumer warps work on each tile.  Two tile shapes:
//   "row" tiles  32 rows x  64 columns, plain layout   (y_b = A_b w: lane = row,
//                warp = 4 columns; y partials stay in registers)
//   "col" tiles  16 rows x 128 columns, 128B-swizzled (z += A_b^T y_b: 4 lanes
//                per column, 4 rows each; the swizzle makes the transposed
//                128-bit reads conflict-free; z accumulates in shared memory)
// GRAM (z = A^T A w): the row tiles of block b+1 (from HBM, L2 evict_last)
// are interleaved with the col tiles of block b (the same bytes, re-read one
// block later from L2, evict_first), so the HBM stream never pauses and no
// per-row-block cross-lane reduction is needed for z.  The L2 working set is
// one block per SM (148 x 32 x d x 8 B, 39 MB at d = 1024).
// ATV  (x = A^T y): col tiles only, from HBM.
// Sums run in a fixed order (rows within a lane, xor tree over 4 lanes, blocks
// in CTA order, CTA partials in CTA order, then the n % 32 tail): the result
// is deterministic and each output column's arithmetic is independent of K.

constexpr int kPR = 32;                    // rows per block
constexpr int kPWarps = 16;                // consumer warps
constexpr int kRowTileCols = 128;          // row tile: 32 x 128
constexpr int kColTileRows = 16;           // col tile: 16 x 256
constexpr int kColTileCols = 256;
constexpr int kRowU = kRowTileCols / kPWarps;        // row-tile columns per warp (8)
constexpr int kColG = kColTileCols / (kPWarps * 8);  // col-tile column groups per warp (2)
constexpr int kPMaxStages = 6;
constexpr int kPStageDoubles = 4096;       // 32 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Orders this thread's earlier shared-memory reads (generic proxy) before the
// TMA refill of the stage (async proxy): issued by every consumer lane before
// the stage is released -- an mbarrier arrive or a CTA barrier alone lets the
// refill overtake loads still in flight (gemm_f64.cu, stage release).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}
// One 2-D TMA box into a ring stage (elements past the end are zero-filled).
__device__ __forceinline__ void tma_box(double* dst, const CUtensorMap* map, int row0, int col0, uint64_t* bar,
                                        uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(row0), "r"(col0), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kPWarps * 32) : "memory"); }
template <int NW>
__device__ __forceinline__ void consumer_sync_n() { asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory"); }

// The tile sequence of one CTA, shared by producer and consumers.
//   GRAM: row tiles of block 0; then for each block i, interleaved:
//         col tile s of block i (s < Q2), row tile s of block i+1 (s < Q1)
//   ATV:  col tiles of each block
struct TileSeq {
  int q1, q2;  // row tiles / col tiles per block
  __device__ TileSeq(int64_t d)
      : q1(static_cast<int>((d + kRowTileCols - 1) / kRowTileCols)),
        q2(static_cast<int>(2 * ((d + kColTileCols - 1) / kColTileCols))) {}
};

// Ring bookkeeping.
struct RingPos {
  int stage = 0;
  uint32_t phase = 0;
  __device__ void next(int stages) {
    if (++stage == stages) {
      stage = 0;
      phase ^= 1;
    }
  }
};

template <int K, bool GRAM>
__global__ void __launch_bounds__((kPWarps + 1) * 32, 1)
    colpass_kernel(const __grid_constant__ CUtensorMap rowmap, const __grid_constant__ CUtensorMap colmap, int64_t n,
                   int64_t nfull, int64_t d, const double* __restrict__ v, double* __restrict__ ws, int stages) {
  extern __shared__ __align__(1024) double sm_raw[];
  // 1024-byte aligned ring (the 128B swizzle pattern is defined on address bits 4-9)
  // (offset arithmetic on the shared array keeps the accesses LDS/STS)
  double* ring = sm_raw + (((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u) >> 3);
  double* zs = ring + stages * kPStageDoubles;  // [d][K]
  double* ypart = zs + d * K;                   // [kPWarps][32][K]
  double* ycur = ypart + kPWarps * kPR * K;     // [K][kPR + 1] (padded: conflict-free)
  __shared__ __align__(8) uint64_t full[kPMaxStages], empty[kPMaxStages];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const TileSeq seq(d);
  const int64_t my_blocks = blockIdx.x < nfull ? (nfull - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto block_row = [&](int64_t i) { return (blockIdx.x + i * gridDim.x) * kPR; };
  if (t == 0) {
    for (int s2 = 0; s2 < stages; ++s2) {
      mbar_init(&full[s2], 1);
      mbar_init(&empty[s2], kPWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int64_t e = t; e < d * K; e += blockDim.x) zs[e] = 0.0;
  __syncthreads();

  if (wid == kPWarps) {  // producer
    if (lane != 0) return;
    uint64_t pol_last, pol_first;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
    RingPos rp;
    auto put = [&](const CUtensorMap* map, int64_t row, int64_t col, uint64_t pol) {
      mbar_wait(&empty[rp.stage], rp.phase ^ 1);
      mbar_arrive_expect_tx(&full[rp.stage], kPStageDoubles * 8);
      tma_box(ring + rp.stage * kPStageDoubles, map, static_cast<int>(row), static_cast<int>(col), &full[rp.stage],
              pol);
      rp.next(stages);
    };
    if (GRAM) {
      if (my_blocks > 0)
        for (int64_t s2 = 0; s2 < seq.q1; ++s2) put(&rowmap, block_row(0), s2 * kRowTileCols, pol_last);
      for (int64_t i = 0; i < my_blocks; ++i) {
        const bool more = i + 1 < my_blocks;
        for (int64_t s2 = 0; s2 < max(seq.q1, seq.q2); ++s2) {
          if (s2 < seq.q2)
            put(&colmap, block_row(i) + kColTileRows * (s2 & 1), kColTileCols * (s2 >> 1), pol_first);
          if (more && s2 < seq.q1) put(&rowmap, block_row(i + 1), s2 * kRowTileCols, pol_last);
        }
      }
    } else {
      for (int64_t i = 0; i < my_blocks; ++i)
        for (int64_t s2 = 0; s2 < seq.q2; ++s2)
          put(&colmap, block_row(i) + kColTileRows * (s2 & 1), kColTileCols * (s2 >> 1), pol_first);
    }
    return;
  }

  RingPos rp;
  const int d32 = static_cast<int>(d);
  double acc[K];  // y partial of row `lane` over this warp's columns
  // row tile s of some block: acc += A[rows, c] w[c]
  auto row_tile = [&](int s2) {
    mbar_wait(&full[rp.stage], rp.phase);
    const double* st = ring + rp.stage * kPStageDoubles + (wid * kRowU) * kPR + lane;
    double av[kRowU];
#pragma unroll
    for (int u = 0; u < kRowU; ++u) av[u] = st[u * kPR];
    const int cbase = s2 * kRowTileCols + wid * kRowU;
#pragma unroll
    for (int u = 0; u < kRowU; ++u) {
      if (cbase + u < d32)
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = fma(av[u], __ldg(v + cbase + u + k * d32), acc[k]);
    }
    // release the stage only once its values are consumed (the arrive does
    // not wait for this warp's outstanding shared-memory loads)
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[rp.stage]);
    rp.next(stages);
  };
  // col tile s of the block whose y is in ycur: z[c] += A[rows, c] . y[rows];
  // 4 lanes per column (rq = rows 4rq..4rq+3), kColG column groups per warp
  const int rq = lane & 3;
  auto col_tile = [&](int s2) {
    mbar_wait(&full[rp.stage], rp.phase);
    const int rb = kColTileRows * (s2 & 1) + 4 * rq;
    double pv[kColG][K];
#pragma unroll
    for (int g2 = 0; g2 < kColG; ++g2) {
      const int cl = g2 * (kPWarps * 8) + wid * 8 + (lane >> 2);
      const double* st = ring + rp.stage * kPStageDoubles + cl * kColTileRows;
      const double2 x0 = *reinterpret_cast<const double2*>(st + (((2 * rq) ^ (cl & 7)) << 1));
      const double2 x1 = *reinterpret_cast<const double2*>(st + (((2 * rq + 1) ^ (cl & 7)) << 1));
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const double* yk = ycur + k * (kPR + 1) + rb;
        double p = x0.x * yk[0];
        p = fma(x0.y, yk[1], p);
        p = fma(x1.x, yk[2], p);
        p = fma(x1.y, yk[3], p);
        pv[g2][k] = p;
      }
    }
    fence_proxy_async_smem();
    __syncwarp();  // (stage values consumed: release it)
    if (lane == 0) mbar_arrive(&empty[rp.stage]);
    rp.next(stages);
    // sum over the 4 lanes of each column: xor 2, then xor 1; with K >= 2 as
    // a reduce-scatter (each lane keeps half the values at each step)
#pragma unroll
    for (int g2 = 0; g2 < kColG; ++g2) {
      const int c = kColTileCols * (s2 >> 1) + g2 * (kPWarps * 8) + wid * 8 + (lane >> 2);
      double* q = pv[g2];
      if (K == 1) {
        q[0] += __shfl_xor_sync(0xffffffffu, q[0], 2);
        q[0] += __shfl_xor_sync(0xffffffffu, q[0], 1);
        if (rq == 0 && c < d32) zs[c] += q[0];
      } else {
        constexpr int H = K / 2;
        {
          const bool up = lane & 2;
#pragma unroll
          for (int i2 = 0; i2 < H; ++i2) {
            const double send = up ? q[i2] : q[i2 + H];
            const double keep = up ? q[i2 + H] : q[i2];
            q[i2] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
          }
        }
        constexpr int Q4 = (H / 2 > 0) ? H / 2 : 1;
        if (H >= 2) {
          const bool up = lane & 1;
#pragma unroll
          for (int i2 = 0; i2 < Q4; ++i2) {
            const double send = up ? q[i2] : q[i2 + Q4];
            const double keep = up ? q[i2 + Q4] : q[i2];
            q[i2] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
          }
          const int base = ((lane & 2) ? H : 0) + ((lane & 1) ? Q4 : 0);
          if (c < d32)
#pragma unroll
            for (int i2 = 0; i2 < Q4; ++i2) zs[c * K + base + i2] += q[i2];
        } else {  // K == 2
          q[0] += __shfl_xor_sync(0xffffffffu, q[0], 1);
          if ((lane & 1) == 0 && c < d32) zs[c * K + ((lane & 2) ? 1 : 0)] += q[0];
        }
      }
    }
  };
  auto reduce_y = [&]() {  // ycur = sum of the warps' y partials, warp order
#pragma unroll
    for (int k = 0; k < K; ++k) ypart[(wid * kPR + lane) * K + k] = acc[k];
    consumer_sync();  // (also: every col tile of the previous block is done)
    if (wid == 0) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double sacc = ypart[lane * K + k];
        for (int w2 = 1; w2 < kPWarps; ++w2) sacc += ypart[(w2 * kPR + lane) * K + k];
        ycur[k * (kPR + 1) + lane] = sacc;
      }
    }
    consumer_sync();
  };

  if (GRAM) {
    if (my_blocks > 0) {
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] = 0.0;
      for (int s2 = 0; s2 < seq.q1; ++s2) row_tile(s2);
      reduce_y();
    }
    for (int64_t i = 0; i < my_blocks; ++i) {
      const bool more = i + 1 < my_blocks;
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] = 0.0;
      for (int s2 = 0; s2 < max(seq.q1, seq.q2); ++s2) {
        if (s2 < seq.q2) col_tile(s2);
        if (more && s2 < seq.q1) row_tile(s2);
      }
      if (more) reduce_y();
    }
  } else {
    for (int64_t i = 0; i < my_blocks; ++i) {
      consumer_sync();  // previous block's col tiles are done with ycur
      if (wid == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) ycur[k * (kPR + 1) + lane] = __ldg(v + k * n + block_row(i) + lane);
      consumer_sync();
      for (int s2 = 0; s2 < seq.q2; ++s2) col_tile(s2);
    }
  }
  consumer_sync();
  for (int64_t e = t; e < d * K; e += kPWarps * 32) {
    const int64_t c = e / K;
    const int k = static_cast<int>(e - c * K);
    ws[static_cast<int64_t>(blockIdx.x) * d * K + c + k * d] = zs[e];
  }
}

// ---- Gram pass on the FP64 tensor cores: z = A^T (A W), W up to 8 columns ------
//
// The column pass above is issue-bound beyond one right-hand column (each
// element of A costs 2K FMAs plus their operand loads on the SIMT pipes).
// Here both products run as DMMA m8n8k4 (W padded to 8 columns), so an
// element of A costs 1/16 of a warp instruction whatever K <= 8 is, and every
// block of A is read from HBM exactly once:
//   * persistent CTAs (one per SM) own contiguous runs of 8-row blocks; a
//     producer warp streams each block (8 rows x all d columns, 64-byte
//     column segments) into a shared-memory ring with 2-D TMA boxes of
//     8 x 256, 64B-swizzled (both fragment patterns below are then
//     conflict-free);
//   * the CTA's NW warps (8; 16 with RP_GRAM_DMMA_WARPS=16) own d/NW columns
//     each.  y pass:
//     y_blk^T (K x 8 rows) = W^T A_blk^T with W^T as the register-resident A
//     operand and the stage as the B operand, four accumulator chains;
//   * the NW partial y tiles meet in shared memory (one barrier per block,
//     summed in warp order), then the z pass
//     z[cols] (8 cols x K) += A_blk^T y_blk reads the same stage again as the
//     A operand: z stays in registers for the whole kernel;
//   * per-CTA z partials are summed in CTA order (sum_chunks_tree_kernel).
// Fixed summation orders throughout: deterministic.  Bound: HBM (8 n d
// bytes) as long as the DMMA pipe keeps up: 2 DMMA (512 flops each) per
// 32 elements = 32 flops per 8 bytes, i.e. ~70 % of the DMMA peak at the
// HBM roof on B200.

constexpr int kGRows = 8;     // rows per block
constexpr int kGWarpsMax = 16;  // warps per CTA (template NW: 8 or 16)
constexpr int kGBox = 256;    // columns per TMA box

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Index (in doubles) of element (row r < 8, stage column c) in a 64B-swizzled
// stage: the 16-byte chunk (byte-offset bits 4-5, = r >> 1) is XORed with
// byte-offset bits 7-8 (= (c >> 1) & 3), i.e. r ^ (c & 6) -- written so that
// the unrolled fragment offsets fold into immediates.
__device__ __forceinline__ int sw64(int c, int r) { return c * kGRows + (r ^ (c & 6)); }
// Partial y tile layout: element (K, row) at (row >> 2) * 32 + (row & 3) + 4 K,
// so the reduction's reads (lane = 4 K + (row & 3)) are 32 consecutive doubles.
__device__ __forceinline__ int ypos(int k, int row) { return (row >> 2) * 32 + (row & 3) + 4 * k; }
// Column order inside each 8-column block: {0, 1, 4, 5, 2, 3, 6, 7}.  A 64-bit
// shared load is served per half-warp; with this order the 16 (column, row)
// pairs of each half-warp fall on 16 different 8-byte banks of the swizzled
// stage, for both fragment patterns (y pass: 4 columns x 4 rows; z pass:
// 4 columns x 4 rows).
__device__ __forceinline__ int perm8(int g) { return (g & 1) | ((g & 2) << 1) | ((g & 4) >> 1); }

template <int NT, int NW>  // NW warps, 256 * NT / NW * 8 ... columns per warp = 256 * NT / NW
__global__ void __launch_bounds__(NW * 32, 1)
    gram_dmma_kernel(const __grid_constant__ CUtensorMap map, int64_t n, int64_t d, int K,
                     const double* __restrict__ w, double* __restrict__ ws, int stages) {
  constexpr int kGWarps = NW;
  constexpr int CPW = 256 * NT / NW;  // columns per warp (multiple of 8)
  static_assert(CPW % 8 == 0, "columns per warp");
  constexpr int KS = CPW / 4;        // k-steps of the y pass (also W fragments)
  constexpr int MT = CPW / 8;        // 8-column tiles of the z pass
  constexpr int DPAD = CPW * kGWarps;  // = 256 * NT
  constexpr int STAGE = DPAD * kGRows;  // doubles
  extern __shared__ __align__(1024) double sm_raw[];
  double* ring = sm_raw + (((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u) >> 3);
  double* ypart = ring + stages * STAGE;  // [2][kGWarps][64]
  __shared__ __align__(8) uint64_t full[kPMaxStages];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  // (the partial-sum kernel behind this pass is launched programmatically: its blocks may take the SMs'
  // free slots early; they wait for this grid's completion before reading the partials)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t nb = (n + kGRows - 1) / kGRows;
  const int64_t b0 = (static_cast<int64_t>(blockIdx.x) * nb) / gridDim.x;
  const int64_t cnt = (static_cast<int64_t>(blockIdx.x + 1) * nb) / gridDim.x - b0;
  uint64_t pol = 0;
  // Thread 0 issues the TMA boxes (no producer warp: 8 warps = 2 per SM
  // sub-partition leave 255 registers per thread for the W fragments and the
  // z accumulators).  Block j lives in stage j % stages; it is refilled with
  // block j + stages once every warp is past the block barrier of block j + 1.
  auto issue = [&](int64_t j) {
    const int st = static_cast<int>(j % stages);
    mbar_arrive_expect_tx(&full[st], STAGE * 8);
    for (int c0 = 0; c0 < DPAD; c0 += kGBox)
      tma_box(ring + st * STAGE + c0 * kGRows, &map, static_cast<int>((b0 + j) * kGRows), c0, &full[st], pol);
  };
  if (t == 0) {
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (int s2 = 0; s2 < stages; ++s2) mbar_init(&full[s2], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int64_t j = 0; j < stages && j < cnt; ++j) issue(j);
  }
  __syncthreads();

  const int g4 = lane >> 2, q4 = lane & 3;
  const int cw = wid * CPW;  // this warp's first column
  // W^T fragments (A operand of the y pass): lane (m = K index g4, k = column q4)
  double wf[KS];
#pragma unroll
  for (int i = 0; i < KS; ++i) {
    const int c = cw + 8 * (i >> 1) + perm8(q4 + 4 * (i & 1));  // k-step i: columns {0,1,4,5} or {2,3,6,7}
    wf[i] = (g4 < K && c < d) ? __ldg(w + c + static_cast<int64_t>(g4) * d) : 0.0;
  }
  double zacc[MT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i) zacc[i][0] = zacc[i][1] = 0.0;
  // Software-pipelined: iteration j runs the z pass of block j interleaved
  // with the y pass of block j + 1 (independent DMMA streams), then one CTA
  // barrier publishes y(j + 1) and frees block j's stage for block j + stages.
  // Partial y tiles are stored [row][K] (8 doubles per row), so the reads of
  // the reduction below are 32 consecutive doubles (conflict-free).
  auto y_pass_store = [&](int64_t jb) {
    const double* sg = ring + static_cast<int>(jb % stages) * STAGE;
    double ya[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) ya[u][0] = ya[u][1] = 0.0;
#pragma unroll
    for (int i = 0; i < KS; ++i) dmma(ya[i & 3][0], ya[i & 3][1], wf[i], sg[sw64(cw + 8 * (i >> 1) + perm8(q4 + 4 * (i & 1)), g4)]);
    double* yp = ypart + (static_cast<int>(jb & 1) * kGWarps + wid) * 64;
    yp[ypos(g4, 2 * q4)] = (ya[0][0] + ya[1][0]) + (ya[2][0] + ya[3][0]);
    yp[ypos(g4, 2 * q4 + 1)] = (ya[0][1] + ya[1][1]) + (ya[2][1] + ya[3][1]);
  };
  auto y_sum = [&](int64_t jb, double (&yb)[2]) {  // y (k = row, n = K) summed over the warps in order
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double* base = ypart + static_cast<int>(jb & 1) * kGWarps * 64 + ypos(g4, 4 * h + q4);  // = h*32 + lane
      double sacc = base[0];
#pragma unroll
      for (int w2 = 1; w2 < kGWarps; ++w2) sacc += base[w2 * 64];
      yb[h] = sacc;
    }
  };
  double yb[2] = {0.0, 0.0};
  if (cnt > 0) {
    mbar_wait(&full[0], 0);
    y_pass_store(0);
    __syncthreads();
    y_sum(0, yb);
  }
  for (int64_t j = 0; j < cnt; ++j) {
    const double* sg = ring + static_cast<int>(j % stages) * STAGE;
    const bool more = j + 1 < cnt;
    if (more) {
      mbar_wait(&full[(j + 1) % stages], static_cast<uint32_t>(((j + 1) / stages) & 1));
      const double* sn = ring + static_cast<int>((j + 1) % stages) * STAGE;
      double ya[4][2];
#pragma unroll
      for (int u = 0; u < 4; ++u) ya[u][0] = ya[u][1] = 0.0;
      // z pass of block j (2 MT = KS DMMAs) interleaved with the y pass of block j + 1 (KS DMMAs)
#pragma unroll
      for (int i = 0; i < KS; ++i) {
        dmma(ya[i & 3][0], ya[i & 3][1], wf[i], sn[sw64(cw + 8 * (i >> 1) + perm8(q4 + 4 * (i & 1)), g4)]);
        const int it = i >> 1, hh = i & 1;
        dmma(zacc[it][0], zacc[it][1], sg[sw64(cw + 8 * it + perm8(g4), 4 * hh + q4)], yb[hh]);
      }
      double* yp = ypart + (static_cast<int>((j + 1) & 1) * kGWarps + wid) * 64;
      yp[ypos(g4, 2 * q4)] = (ya[0][0] + ya[1][0]) + (ya[2][0] + ya[3][0]);
      yp[ypos(g4, 2 * q4 + 1)] = (ya[0][1] + ya[1][1]) + (ya[2][1] + ya[3][1]);
    } else {
#pragma unroll
      for (int i = 0; i < KS; ++i) {
        const int it = i >> 1, hh = i & 1;
        dmma(zacc[it][0], zacc[it][1], sg[sw64(cw + 8 * it + perm8(g4), 4 * hh + q4)], yb[hh]);
      }
    }
    // every warp is done with block j: its stage takes block j + stages
    fence_proxy_async_smem();
    __syncthreads();
    if (t == 0 && j + stages < cnt) issue(j + stages);
    if (more) y_sum(j + 1, yb);
  }
  // this CTA's z partial: lane holds z[col = cw + 8i + perm8(g4)][K = 2 q4 + e]
  double* out = ws + static_cast<int64_t>(blockIdx.x) * d * K;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int c = cw + 8 * i + perm8(g4);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int k = 2 * q4 + e;
      if (c < d && k < K) out[c + static_cast<int64_t>(k) * d] = zacc[i][e];
    }
  }
}

// The last n % 32 rows (one CTA): the same sums, written as one more partial.
template <int K, bool GRAM>
__global__ void __launch_bounds__(256) colpass_tail_kernel(const double* __restrict__ a, int64_t lda, int64_t n,
                                                           int64_t r0, int64_t d, const double* __restrict__ v,
                                                           double* __restrict__ out) {
  __shared__ double yt[kPR][K];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int rows = static_cast<int>(n - r0);
  if (GRAM) {  // y_tail[r] = sum_c A[r, c] w[c]: one warp per row
    for (int r = wid; r < rows; r += blockDim.x / 32) {
      double acc[K];
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] = 0.0;
      for (int64_t c = lane; c < d; c += 32) {
        const double x = a[c * lda + r0 + r];
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = fma(x, v[c + k * d], acc[k]);
      }
      warp_reduce<K>(acc);
      if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) yt[r][k] = acc[k];
    }
  } else if (t < rows) {
#pragma unroll
    for (int k = 0; k < K; ++k) yt[t][k] = v[k * n + r0 + t];
  }
  __syncthreads();
  for (int64_t c = t; c < d; c += blockDim.x) {
    double acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = 0.0;
    for (int r = 0; r < rows; ++r) {
      const double x = a[c * lda + r0 + r];
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] = fma(x, yt[r][k], acc[k]);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) out[c + k * d] = acc[k];
  }
}

// Launches the column pass; false if the operator is not 16-byte aligned.
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static std::once_flag once;
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Tensor map of the column-major operator: dims (rows n, columns d), box
// rows x cols; the smem image is [column][row].
bool operator_tensor_map(CUtensorMap* map, const double* a, int64_t lda, int64_t n, int64_t d, int box_rows,
                         int box_cols, bool swizzle128, bool swizzle64 = false) {
  auto enc = tensor_map_encoder();
  if (!enc || n >= (int64_t{1} << 31) || d >= (int64_t{1} << 31)) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(d)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(lda) * sizeof(double)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(box_cols)};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(a), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE,
             swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : (swizzle64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE),
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int K, bool GRAM>
bool colpass_launch(const double* a, int64_t lda, int64_t n, int64_t d, const double* v, double* out, cudaStream_t s) {
  if (lda % 2 != 0 || reinterpret_cast<uintptr_t>(a) % 16 != 0 || d <= 0 || n <= 0) return false;
  CUtensorMap rowmap, colmap;
  if (!operator_tensor_map(&rowmap, a, lda, n, d, kPR, kRowTileCols, false) ||
      !operator_tensor_map(&colmap, a, lda, n, d, kColTileRows, kColTileCols, true))
    return false;
  const size_t fixed = sizeof(double) * (static_cast<size_t>(d) * K + kPWarps * kPR * K + (kPR + 1) * K);
  const size_t budget = 220 * 1024;
  constexpr size_t stage_bytes = kPStageDoubles * sizeof(double);
  if (fixed + 3 * stage_bytes + 1024 > budget || d >= (int64_t{1} << 30)) return false;
  const int stages = static_cast<int>(std::min<size_t>(kPMaxStages, (budget - fixed - 1024) / stage_bytes));
  const size_t smem = fixed + static_cast<size_t>(stages) * stage_bytes + 1024;  // (+ alignment slack)
  int dev = 0, sms = 0;
  RP_CUDA(cudaGetDevice(&dev));
  RP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t nfull = n / kPR;
  const bool tail = n % kPR != 0;
  const int grid = static_cast<int>(std::min<int64_t>(nfull, sms));
  const int64_t parts = grid + (tail ? 1 : 0);
  DBuf<double> ws(static_cast<size_t>(parts) * d * K, s);
  if (grid > 0) {
    ensure_dynamic_smem(colpass_kernel<K, GRAM>, smem);
    colpass_kernel<K, GRAM><<<grid, (kPWarps + 1) * 32, smem, s>>>(rowmap, colmap, n, nfull, d, v, ws.get(), stages);
    RP_LAUNCH_CHECK();
  }
  if (tail) {
    colpass_tail_kernel<K, GRAM><<<1, 256, 0, s>>>(a, lda, n, nfull * kPR, d, v, ws.get() + grid * d * K);
    RP_LAUNCH_CHECK();
  }
  sum_chunks_tree_kernel<<<static_cast<unsigned>(ceil_div(d * K, 16)), 256, 0, s>>>(ws.get(), parts, d * K, out);
  RP_LAUNCH_CHECK();
  return true;
}

template <int K>
void atv_launch(const double* a, int64_t lda, int64_t n, int64_t d, const double* y, double* x, cudaStream_t s) {
  const int64_t chunks = ceil_div(n, kChunkRows);
  const int64_t warps = d * chunks;
  DBuf<double> part(static_cast<size_t>(chunks * d * K), s);
  const bool vec = (lda % 2 == 0) && (n % 2 == 0) && ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(y)) % 16 == 0);
  atv_partial_kernel<K><<<static_cast<unsigned>(ceil_div(warps * 32, 256)), 256, 0, s>>>(a, lda, n, d, y, chunks,
                                                                                          part.get(), vec);
  RP_LAUNCH_CHECK();
  sum_chunks_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(d * K, 256), 1184)), 256, 0, s>>>(
      part.get(), chunks, d * K, x);
  RP_LAUNCH_CHECK();
}


// The DMMA Gram pass (k <= 8 columns, d <= 5 * 256): false if it does not apply.
template <int NT, int NW>
bool gram_dmma_launch_nt(const double* a, int64_t lda, int64_t n, int64_t d, const double* w, int64_t k, double* z,
                         cudaStream_t s) {
  constexpr int kGWarps = NW;
  constexpr int DPAD = 256 * NT;
  CUtensorMap map;
  if (!operator_tensor_map(&map, a, lda, n, d, kGRows, kGBox, false, true)) return false;
  constexpr size_t stage_bytes = static_cast<size_t>(DPAD) * kGRows * sizeof(double);
  const size_t fixed = 2 * kGWarps * 64 * sizeof(double) + 1024;
  const size_t budget = 225 * 1024;
  const int stages = static_cast<int>(std::min<size_t>(kPMaxStages, (budget - fixed) / stage_bytes));
  if (stages < 3) return false;  // (block j uses one stage, block j - 1 is refilled, one in flight)
  const size_t smem = fixed + static_cast<size_t>(stages) * stage_bytes;
  int dev = 0, sms = 0;
  RP_CUDA(cudaGetDevice(&dev));
  RP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t nb = (n + kGRows - 1) / kGRows;
  const int grid = static_cast<int>(std::min<int64_t>(nb, sms));
  DBuf<double> ws(static_cast<size_t>(grid) * d * k, s);
  ensure_dynamic_smem(gram_dmma_kernel<NT, NW>, smem);
  gram_dmma_kernel<NT, NW><<<grid, NW * 32, smem, s>>>(map, n, d, static_cast<int>(k), w, ws.get(), stages);
  RP_LAUNCH_CHECK();
  {
    // the CTA-partial sum starts its blocks while the pass drains (programmatic dependent launch)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(ceil_div(d * k, 16)));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const double* part = ws.get();
    const int64_t chunks = grid, total = d * k;
    RP_CUDA(cudaLaunchKernelEx(&cfg, sum_chunks_tree_kernel, part, chunks, total, z));
  }
  RP_LAUNCH_CHECK();
  return true;
}

bool gram_dmma_launch(const double* a, int64_t lda, int64_t n, int64_t d, const double* w, int64_t k, double* z,
                      cudaStream_t s) {
  if (k < 1 || k > 8 || n <= 0 || d <= 0 || lda % 2 != 0 || reinterpret_cast<uintptr_t>(a) % 16 != 0) return false;
  // (RP_GRAM_DMMA_WARPS=16: sixteen warps per CTA instead of eight -- A/B;
  // measured 0.63 vs 0.73 of HBM on the C2 operator, profiles/r02_gram_pass_dmma.txt)
  static const bool w8 = [] {
    const char* e = std::getenv("RP_GRAM_DMMA_WARPS");
    return !(e && std::atoi(e) == 16);
  }();
  switch (ceil_div(d, 256)) {
    case 1: return w8 ? gram_dmma_launch_nt<1, 8>(a, lda, n, d, w, k, z, s) : gram_dmma_launch_nt<1, 16>(a, lda, n, d, w, k, z, s);
    case 2: return w8 ? gram_dmma_launch_nt<2, 8>(a, lda, n, d, w, k, z, s) : gram_dmma_launch_nt<2, 16>(a, lda, n, d, w, k, z, s);
    case 3: return w8 ? gram_dmma_launch_nt<3, 8>(a, lda, n, d, w, k, z, s) : gram_dmma_launch_nt<3, 16>(a, lda, n, d, w, k, z, s);
    case 4: return w8 ? gram_dmma_launch_nt<4, 8>(a, lda, n, d, w, k, z, s) : gram_dmma_launch_nt<4, 16>(a, lda, n, d, w, k, z, s);
    default: return false;
  }
}

// Smallest column count sent to the DMMA pass (RP_GRAM_DMMA_MIN, default 1:
// every width where it applies, so a column's bits do not depend on how many
// columns are batched with it).
int64_t gram_dmma_min() {
  static const int64_t v = [] {
    const char* e = std::getenv("RP_GRAM_DMMA_MIN");
    return e ? std::atoll(e) : int64_t{1};
  }();
  return v;
}

}  // namespace

namespace {
// One group of kw columns through the column pass (false: does not fit).
template <bool GRAM>
bool colpass_group(int64_t kw, const double* a, int64_t lda, int64_t n, int64_t d, const double* v, double* out,
                   cudaStream_t s) {
  switch (kw) {
    case 8: return colpass_launch<8, GRAM>(a, lda, n, d, v, out, s);
    case 4: return colpass_launch<4, GRAM>(a, lda, n, d, v, out, s);
    case 2: return colpass_launch<2, GRAM>(a, lda, n, d, v, out, s);
    default: return colpass_launch<1, GRAM>(a, lda, n, d, v, out, s);
  }
}
// Columns j .. k-1 in groups of 8/4/2/1, each group as wide as fits the
// shared-memory budget (a column's arithmetic does not depend on its group).
// Returns the number of columns done (< k only if a single column fails).
template <bool GRAM>
int64_t colpass_columns(const double* a, int64_t lda, int64_t n, int64_t d, const double* v, int64_t v_ld,
                        int64_t k, double* out, cudaStream_t s) {
  int64_t j = 0;
  while (j < k) {
    int64_t kw = k - j >= 8 ? 8 : k - j >= 4 ? 4 : k - j >= 2 ? 2 : 1;
    while (kw >= 1 && !colpass_group<GRAM>(kw, a, lda, n, d, v + j * v_ld, out + j * d, s)) kw /= 2;
    if (kw < 1) break;
    j += kw;
  }
  return j;
}
}  // namespace

void atv_narrow(const double* a, int64_t lda, int64_t n, int64_t d, const double* y, int64_t k, double* x,
                cudaStream_t stream) {
  require(k >= 1 && k <= kNarrowMax, "atv_narrow: 1 <= k <= 16");
  if (d <= 0) return;
  int64_t j = 0;
  if (n % 2 == 0 && reinterpret_cast<uintptr_t>(y) % 16 == 0)
    j = colpass_columns<false>(a, lda, n, d, y, n, k, x, stream);
  // (unaligned operators: one warp per column and row chunk)
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
  if (k < 1 || k > 8 || d <= 0 || n <= 0) return false;
  if (k >= gram_dmma_min() && gram_dmma_launch(a, lda, n, d, w, k, z, stream)) return true;
  return colpass_columns<true>(a, lda, n, d, w, d, k, z, stream) == k;
}

}  // namespace rpb
