// FP64 DMMA GEMM for sm_100a (see gemm_f64.h for the contract).
//
// Layout of one CTA: BM x BN output tile, WM x WN warps, each warp owning a
// (BM/WM) x (BN/WN) register tile built from m8n8k4 DMMA fragments.  Operands
// move global -> shared through a STAGES-deep cp.async ring; every operand has
// two shared layouts so the 16-byte copies stay contiguous in global memory:
//   MN-major  (op(A) = A, op(B) = B^T):  smem[k][mn], row stride MN + 4 doubles
//   K-major   (op(A) = A^T, op(B) = B):  smem[mn][k], row stride BK + 4 doubles
// Strides = 4 (mod 16) doubles keep the DMMA fragment loads (8 rows x 4 k)
// free of shared-memory bank conflicts within each half-warp.
#include "common.h"
#include "gemm_f64.h"
#include "tma_util.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

namespace rpb {
namespace {

thread_local int g_last_launches = 0;

constexpr int kMaxDevices = 64;
int current_device() {
  int dev = 0;
  RP_CUDA(cudaGetDevice(&dev));
  require(dev >= 0 && dev < kMaxDevices, "dgemm: device ordinal out of range");
  return dev;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct KParams {
  int64_t m, n, k;
  double alpha, beta;
  const double* a;
  int64_t lda, stride_a;
  const double* b;
  int64_t ldb, stride_b;
  double* c;
  int64_t ldc, stride_c;
  int64_t batch;
  int64_t batch2;
  int64_t stride_a2, stride_b2, stride_c2;
  int split;        // number of K splits
  int64_t k_chunk;  // K per split (multiple of the tile K)
  int vchunk;       // > 0: "virtual split" -- one CTA per tile runs every K chunk of vchunk k-tiles, each
                    // chunk accumulated from zero and added to the running total in chunk order: the bits
                    // of a real split (partials summed 0..S-1), without partials or a consumer kernel
  double* ws;       // split partials: [batch][split][n][m]
  bool lower_only;
  bool mirror;  // lower_only: also write the transposed element (C symmetric)
  bool tri_k;   // op(A)(i, k) == 0 for k < i: start the k loop at the tile's first row
  bool tri_b;   // op(B)(k, j) == 0 for k < j: start the k loop at the tile's first column
  bool tri_a_lower;  // op(A)(i, k) == 0 for k > i: end the k loop at the tile's last row
  bool no_tma;  // use the cp.async kernel (GemmArgs::no_tma)
  int occ_cap;  // host side only: GemmArgs::max_ctas_per_sm
  RecursionEpilogue epi;
};

// Per-column bookkeeping of the fused recursion epilogues, computed once per
// output column of a tile (see RecursionEpilogue in gemm_f64.h):
//   kArgs:   dst = args offset, src = gen offset of column j-1 (or -1), s = tau_l
//   kUpdate: dst = gen/tilde offset (or -1: interval finished), src = next-args
//            offset (or -1), s = 1 if j < g (subtract) else 0 (negate)
struct ColInfo {
  int64_t dst, src;
  double s;
};

__device__ __forceinline__ ColInfo column_info(const RecursionEpilogue& E, int64_t b1, int64_t col) {
  const int64_t nb = E.L * E.K;
  ColInfo ci;
  if (E.kind == RecursionEpilogue::kArgs) {
    const int64_t j = col / nb, b = col - j * nb;
    const int64_t l = b / E.K, r = b - l * E.K;
    ci.dst = (l * E.kmax * E.K + j * E.K + r) * E.dim;
    ci.src = j >= 1 ? ((j - 1) * nb + b) * E.dim : -1;
    ci.s = E.tau[l];
  } else {
    const int64_t l = b1, j = col / E.K, r = col - j * E.K, b = l * E.K + r;
    const bool live = E.g < E.kb[l];
    ci.dst = live ? (j * nb + b) * E.dim : -1;
    ci.src = (live && j == E.g && E.g + 1 < E.kmax) ? (l * E.kmax * E.K + (E.g + 1) * E.K + r) * E.dim : -1;
    ci.s = j < E.g ? 1.0 : 0.0;
  }
  return ci;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BKM, int VEC>
struct Cfg {
  static constexpr int THREADS = WM * WN * 32;
  static constexpr int TM = BM / WM;
  static constexpr int TN = BN / WN;
  static constexpr int FM = TM / 8;
  static constexpr int FN = TN / 8;
  static constexpr int A_LD = AK ? (BK + 4) : (BM + 4);
  static constexpr int A_ROWS = AK ? BM : BK;
  static constexpr int B_LD = BKM ? (BK + 4) : (BN + 4);
  static constexpr int B_ROWS = BKM ? BN : BK;
  static constexpr int A_STAGE = A_ROWS * A_LD;
  static constexpr int B_STAGE = B_ROWS * B_LD;
  static constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * 8;
  static_assert(TM % 8 == 0 && TN % 8 == 0, "warp tile must be a multiple of 8");
  static_assert(BK % 4 == 0, "BK must be a multiple of 4");
};

// Load an MN x BK operand tile (op(X) is MN x K) into shared memory.
// KMAJ: the operand is contiguous along k in global memory.
template <int MN_T, int BK, int LD, int THREADS, bool KMAJ, int VEC>
__device__ __forceinline__ void load_tile(double* sm, const double* g, int64_t ld, int64_t mn0,
                                          int64_t mn_lim, int64_t k0, int64_t k_lim, int tid) {
  if (!KMAJ) {
    constexpr int CPR = MN_T / VEC;
    constexpr int TOTAL = BK * CPR;
#pragma unroll
    for (int c = tid; c < TOTAL; c += THREADS) {
      const int kk = c / CPR;
      const int mm = (c % CPR) * VEC;
      const int64_t gm = mn0 + mm, gk = k0 + kk;
      int bytes = 0;
      const double* src = g;
      if (gk < k_lim && gm < mn_lim) {
        bytes = static_cast<int>(mn_lim - gm < VEC ? mn_lim - gm : VEC) * 8;
        src = g + gm + gk * ld;
      }
      double* dst = sm + kk * LD + mm;
      if (VEC == 2)
        cp_async16(dst, src, bytes);
      else
        cp_async8(dst, src, bytes);
    }
  } else {
    constexpr int CPR = BK / VEC;
    constexpr int TOTAL = MN_T * CPR;
#pragma unroll
    for (int c = tid; c < TOTAL; c += THREADS) {
      const int mm = c / CPR;
      const int kk = (c % CPR) * VEC;
      const int64_t gm = mn0 + mm, gk = k0 + kk;
      int bytes = 0;
      const double* src = g;
      if (gm < mn_lim && gk < k_lim) {
        bytes = static_cast<int>(k_lim - gk < VEC ? k_lim - gk : VEC) * 8;
        src = g + gk + gm * ld;
      }
      double* dst = sm + mm * LD + kk;
      if (VEC == 2)
        cp_async16(dst, src, bytes);
      else
        cp_async8(dst, src, bytes);
    }
  }
}

// Per-thread copy plan of one operand tile (MN_T x BK of op(X)), computed
// once per CTA: global source of each 16-byte chunk at the first k tile, its
// shared-memory slot, and how many bytes the MN bound leaves.  Each k tile
// then only adds a fixed stride; the k bound is checked on the last tile only.
template <int MN_T, int BK, int LD, int THREADS, bool KMAJ, int VEC>
struct TileCopier {
  static constexpr int CPR = KMAJ ? BK / VEC : MN_T / VEC;  // chunks per smem row
  static constexpr int TOTAL = KMAJ ? MN_T * CPR : BK * CPR;
  static constexpr int NCH = (TOTAL + THREADS - 1) / THREADS;
  const double* src[NCH];
  int dst[NCH];
  int kk[NCH];
  int bytes[NCH];  // < 0: no chunk
  int64_t kstep;
  __device__ __forceinline__ void init(const double* g, int64_t ld, int64_t mn0, int64_t mn_lim, int64_t kbeg,
                                       int tid) {
#pragma unroll
    for (int n = 0; n < NCH; ++n) {
      const int c = tid + n * THREADS;
      int mm, k;
      if (KMAJ) {
        mm = c / CPR;
        k = (c % CPR) * VEC;
      } else {
        k = c / CPR;
        mm = (c % CPR) * VEC;
      }
      const int64_t gm = mn0 + mm;
      kk[n] = k;
      dst[n] = KMAJ ? mm * LD + k : k * LD + mm;
      if (c >= TOTAL) {
        bytes[n] = -1;
        src[n] = g;
      } else if (gm >= mn_lim) {
        bytes[n] = 0;
        src[n] = g;
      } else {
        bytes[n] = KMAJ ? VEC * 8 : static_cast<int>(mn_lim - gm < VEC ? mn_lim - gm : VEC) * 8;
        src[n] = KMAJ ? g + (kbeg + k) + gm * ld : g + gm + (kbeg + k) * ld;
      }
    }
    kstep = KMAJ ? BK : BK * ld;
  }
  // k tile `kt`; k_rem = valid k values left from this tile's first k
  __device__ __forceinline__ void issue(double* sm, int kt, int64_t k_rem) const {
    const int64_t off = static_cast<int64_t>(kt) * kstep;
    const bool full = k_rem >= BK;
#pragma unroll
    for (int n = 0; n < NCH; ++n) {
      if (bytes[n] < 0) continue;
      int b = bytes[n];
      if (!full) {
        const int64_t kv = k_rem - kk[n];
        if (KMAJ)
          b = kv <= 0 ? 0 : (kv < VEC ? static_cast<int>(kv) * 8 : b);
        else if (kv <= 0)
          b = 0;
      }
      const double* sp = b > 0 ? src[n] + off : src[n];
      if (VEC == 2)
        cp_async16(sm + dst[n], sp, b);
      else
        cp_async8(sm + dst[n], sp, b);
    }
  }
};

// GEMM epilogue shared by the cp.async and TMA kernels: accumulators -> the
// consumer of C (store / mirror / recursion epilogue, or split-K partials).
// Every thread of the CTA must call it (it contains CTA barriers); `active`
// marks the compute threads (tid < C::THREADS) that hold accumulators and do
// element work.
template <class C, int BM, int WN, int STAGES>
__device__ __forceinline__ void gemm_epilogue(const KParams& p, double (&acc)[C::FM][C::FN][2], double* smem, int tid,
                                              bool active, int wm, int wn, int r8, int k4, int64_t m0, int64_t n0,
                                              int64_t b1, int64_t b2, int64_t bidx, int sidx) {
  // Epilogue, staged through shared memory one warp-column (BM x TN) at a
  // time: the accumulators leave registers once, and every global access below
  // walks rows fastest (coalesced, column-major C).  Split-K: each split
  // publishes its partial tile; the last one to finish (tile counter) sums the
  // partials in split order 0..S-1 -- an order independent of launch timing --
  // and runs the consumer.
  constexpr int SLD = BM + 2;  // conflict-free fragment stores
  static_assert(SLD * C::TN <= STAGES * (C::A_STAGE + C::B_STAGE), "epilogue staging does not fit");
  double* Cb = p.c + b1 * p.stride_c + b2 * p.stride_c2;
  const int64_t mn = p.m * p.n;
  double* W = p.split > 1 ? p.ws + bidx * p.split * mn : nullptr;
  auto for_tile = [&](int w, auto&& fn) {  // fn(row, col, smem value) over warp-column w
    if (!active) return;
    for (int idx = tid; idx < BM * C::TN; idx += C::THREADS) {
      const int rr = idx % BM, cc = idx / BM;
      const int64_t row = m0 + rr, col = n0 + w * C::TN + cc;
      if (row < p.m && col < p.n && !(p.lower_only && row < col)) fn(row, col, smem[cc * SLD + rr]);
    }
  };
  auto stage = [&](int w) {
    __syncthreads();
    if (active && wn == w) {
#pragma unroll
      for (int i = 0; i < C::FM; ++i)
#pragma unroll
        for (int j = 0; j < C::FN; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) smem[(j * 8 + 2 * k4 + e) * SLD + wm * C::TM + i * 8 + r8] = acc[i][j][e];
    }
    __syncthreads();
  };
  // C = reduced values of warp-column w (in smem) -> consumer.  Loads are
  // issued U elements at a time before any store, so the L2 latency of the
  // read-modify-write consumers overlaps.
  constexpr int PER = BM * C::TN;
  constexpr int U = 4;  // (batches of 8 / 16 were measured: no gain on C2's basis, and the 64 x 64 tile spills)
  __shared__ ColInfo cinfo[C::TN];
  auto finish = [&](int w) {
    const int64_t col0 = n0 + w * C::TN;
    if (p.epi.kind != 0) {
      if (tid < C::TN && col0 + tid < p.n) cinfo[tid] = column_info(p.epi, b1, col0 + tid);
      __syncthreads();
    }
    if (!active) {
      if (p.epi.kind == 0 && p.mirror) __syncthreads();
    } else if (p.epi.kind == 0) {
      if (p.beta == 0.0) {
        for (int idx = tid; idx < PER; idx += C::THREADS) {
          const int rr = idx % BM, cc = idx / BM;
          const int64_t row = m0 + rr, col = col0 + cc;
          if (row < p.m && col < p.n && !(p.lower_only && row < col)) Cb[row + col * p.ldc] = p.alpha * smem[cc * SLD + rr];
        }
      } else {
        // C <- alpha AB + beta C: the old values are fetched UB at a time before
        // any store -- one element per iteration serialized a full L2 / HBM
        // round trip per element (16 per thread and warp-column: the rank-64
        // trailing updates of the Cholesky ran at 8 TF/s on it)
        constexpr int UB = 8;
        for (int base = tid; base < PER; base += UB * C::THREADS) {
          double old[UB];
#pragma unroll
          for (int u = 0; u < UB; ++u) {
            const int idx = base + u * C::THREADS, rr = idx % BM, cc = idx / BM;
            const int64_t row = m0 + rr, col = col0 + cc;
            old[u] = 0.0;
            if (idx < PER && row < p.m && col < p.n && !(p.lower_only && row < col)) old[u] = __ldcg(Cb + row + col * p.ldc);
          }
#pragma unroll
          for (int u = 0; u < UB; ++u) {
            const int idx = base + u * C::THREADS, rr = idx % BM, cc = idx / BM;
            const int64_t row = m0 + rr, col = col0 + cc;
            if (idx < PER && row < p.m && col < p.n && !(p.lower_only && row < col))
              Cb[row + col * p.ldc] = p.alpha * smem[cc * SLD + rr] + p.beta * old[u];
          }
        }
      }
      if (p.mirror) {
        __syncthreads();
        for (int idx = tid; idx < PER; idx += C::THREADS) {
          const int cc = idx % C::TN, rr = idx / C::TN;
          const int64_t row = m0 + rr, col = col0 + cc;
          if (row < p.m && col < p.n && row > col) Cb[col + row * p.ldc] = p.alpha * smem[cc * SLD + rr];
        }
      }
    } else if (p.epi.kind == RecursionEpilogue::kArgs) {
      const double* __restrict__ gen = p.epi.gen;
      double* __restrict__ args = p.epi.args;
      for (int base = tid; base < PER; base += U * C::THREADS) {
        double pv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = base + u * C::THREADS, rr = idx % BM, cc = idx / BM;
          pv[u] = 0.0;
          if (idx < PER && m0 + rr < p.m && col0 + cc < p.n && cinfo[cc].src >= 0)
            pv[u] = __ldcg(gen + cinfo[cc].src + m0 + rr);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = base + u * C::THREADS, rr = idx % BM, cc = idx / BM;
          if (idx < PER && m0 + rr < p.m && col0 + cc < p.n) {
            const ColInfo ci = cinfo[cc];
            double a = __dmul_rn(ci.s, smem[cc * SLD + rr]);
            if (ci.src >= 0) a = __dadd_rn(a, pv[u]);
            args[ci.dst + m0 + rr] = a;
          }
        }
      }
    } else {  // kUpdate
      double* __restrict__ gen = p.epi.gen;
      double* __restrict__ tilde = p.epi.tilde;
      double* __restrict__ args = p.epi.args;
      bool bad = false;
      for (int base = tid; base < PER; base += U * C::THREADS) {
        double gv[U], tv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = base + u * C::THREADS, rr = idx % BM, cc = idx / BM;
          gv[u] = tv[u] = 0.0;
          if (idx < PER && m0 + rr < p.m && col0 + cc < p.n && cinfo[cc].dst >= 0) {
            gv[u] = __ldcg(gen + cinfo[cc].dst + m0 + rr);
            tv[u] = __ldcg(tilde + cinfo[cc].dst + m0 + rr);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = base + u * C::THREADS, rr = idx % BM, cc = idx / BM;
          if (idx < PER && m0 + rr < p.m && col0 + cc < p.n && cinfo[cc].dst >= 0) {
            const ColInfo ci = cinfo[cc];
            const double v = smem[cc * SLD + rr];
            const double nv = ci.s != 0.0 ? __dsub_rn(gv[u], v) : -v;
            gen[ci.dst + m0 + rr] = nv;
            tilde[ci.dst + m0 + rr] = __dadd_rn(tv[u], nv);
            bad |= !isfinite(nv);
            if (ci.src >= 0) args[ci.src + m0 + rr] = nv;
          }
        }
      }
      if (bad) p.epi.flags[b1] = 1;
    }
    __syncthreads();  // smem / cinfo are reused by the next warp-column
  };
  if (p.split > 1) {
    if (!active) return;
    // split-K: this split's partial tile goes straight from registers to the
    // workspace; the sum over splits (in split order) happens in the consumer
    // (deferred Partials) or in splitk_reduce
#pragma unroll
    for (int i = 0; i < C::FM; ++i) {
      const int64_t row = m0 + wm * C::TM + i * 8 + r8;
      if (row >= p.m) continue;
#pragma unroll
      for (int j = 0; j < C::FN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t col = n0 + wn * C::TN + j * 8 + 2 * k4 + e;
          if (col < p.n && !(p.lower_only && row < col)) W[sidx * mn + row + col * p.m] = acc[i][j][e];
        }
    }
    return;
  }
  for (int w = 0; w < WN; ++w) {
    stage(w);
    finish(w);
  }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BKM, int VEC>
__global__ void __launch_bounds__(WM* WN * 32) dgemm_kernel(KParams p) {
  using C = Cfg<BM, BN, BK, WM, WN, STAGES, AK, BKM, VEC>;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * C::A_STAGE;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wm = warp % WM;
  const int wn = warp / WM;

  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int64_t n0 = static_cast<int64_t>(blockIdx.y) * BN;
  if (p.lower_only && m0 + BM <= n0) return;  // tile strictly above the diagonal
  const int64_t z = blockIdx.z;
  const int64_t bidx = z / p.split;
  const int sidx = static_cast<int>(z % p.split);
  const int64_t b1 = bidx % p.batch, b2 = bidx / p.batch;
  const double* A = p.a + b1 * p.stride_a + b2 * p.stride_a2;
  const double* B = p.b + b1 * p.stride_b + b2 * p.stride_b2;
  int64_t kbeg = static_cast<int64_t>(sidx) * p.k_chunk;
  int64_t kend = min(p.k, kbeg + p.k_chunk);
  if (p.tri_k) kbeg = max(kbeg, m0 & ~static_cast<int64_t>(BK - 1));
  if (p.tri_b) kbeg = max(kbeg, n0 & ~static_cast<int64_t>(BK - 1));
  if (p.tri_a_lower) kend = min(kend, m0 + BM);  // (BM is a multiple of BK)
  const int ktiles = kend > kbeg ? static_cast<int>((kend - kbeg + BK - 1) / BK) : 0;

  double acc[C::FM][C::FN][2];
#pragma unroll
  for (int i = 0; i < C::FM; ++i)
#pragma unroll
    for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  TileCopier<BM, BK, C::A_LD, C::THREADS, AK, VEC> ca;
  TileCopier<BN, BK, C::B_LD, C::THREADS, BKM, VEC> cb;
  ca.init(A, p.lda, m0, p.m, kbeg, tid);
  cb.init(B, p.ldb, n0, p.n, kbeg, tid);
  auto issue = [&](int kt, int stage) {
    const int64_t k_rem = kend - kbeg - static_cast<int64_t>(kt) * BK;
    ca.issue(As + stage * C::A_STAGE, kt, k_rem);
    cb.issue(Bs + stage * C::B_STAGE, kt, k_rem);
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) issue(s, s);
    cp_async_commit();
  }

  const int r8 = lane >> 2;  // fragment row / column within the 8-wide tile
  const int k4 = lane & 3;   // fragment k index
  int rstage = 0, wstage = STAGES - 1;  // (rolling stage indices, no modulo)
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < ktiles) issue(nk, wstage);
      cp_async_commit();
      wstage = wstage + 1 == STAGES ? 0 : wstage + 1;
    }
    const double* as = As + rstage * C::A_STAGE;
    const double* bs = Bs + rstage * C::B_STAGE;
    rstage = rstage + 1 == STAGES ? 0 : rstage + 1;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[C::FM], bf[C::FN];
#pragma unroll
      for (int i = 0; i < C::FM; ++i) {
        const int row = wm * C::TM + i * 8 + r8;
        af[i] = AK ? as[row * C::A_LD + kk + k4] : as[(kk + k4) * C::A_LD + row];
      }
#pragma unroll
      for (int j = 0; j < C::FN; ++j) {
        const int col = wn * C::TN + j * 8 + r8;
        bf[j] = BKM ? bs[col * C::B_LD + kk + k4] : bs[(kk + k4) * C::B_LD + col];
      }
#pragma unroll
      for (int i = 0; i < C::FM; ++i)
#pragma unroll
        for (int j = 0; j < C::FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  gemm_epilogue<C, BM, WN, STAGES>(p, acc, smem, tid, true, wm, wn, r8, k4, m0, n0, b1, b2, bidx, sidx);
}

// TMA + mbarrier variant: one producer warp streams both operand tiles with
// 4-D tensor boxes (inner, outer, batch, batch2) into a STAGES-deep ring;
// the WM x WN compute warps wait on per-stage "full" barriers and release
// stages through "empty" barriers -- no CTA-wide barrier in the main loop.
// Boxes are 4 elements wider than the tile along the contiguous dimension,
// which reproduces the padded shared-memory layouts of the cp.async kernel
// (conflict-free fragment loads); the extra elements are never read.  The
// arithmetic (k order, fragment mapping, epilogue) is the cp.async kernel's,
// so both produce identical bits.
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BKM, bool VS>
__global__ void __launch_bounds__((WM * WN + 1) * 32)
    dgemm_tma_kernel(const __grid_constant__ CUtensorMap amap_p, const __grid_constant__ CUtensorMap bmap_p, KParams p,
                     int a_batched, int a_batched2, int b_batched, int b_batched2
#ifdef RP_PROBE_GMAP  // (concurrency probe, tools/tma_race.cu: tensor maps read from global memory)
                     ,
                     const CUtensorMap* gmaps
#endif
    ) {
  using C = Cfg<BM, BN, BK, WM, WN, STAGES, AK, BKM, 2>;
#ifdef RP_PROBE_GMAP
  const CUtensorMap& amap = gmaps[0];
  const CUtensorMap& bmap = gmaps[1];
#else
  const CUtensorMap& amap = amap_p;
  const CUtensorMap& bmap = bmap_p;
#endif
  extern __shared__ __align__(128) double smem_raw[];
  // 128-byte aligned ring (TMA destinations); the launch adds 128 B of slack
  double* smem = smem_raw + (((128u - (tma::smem_u32(smem_raw) & 127u)) & 127u) >> 3);
  double* As = smem;
  double* Bs = smem + STAGES * C::A_STAGE;
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const bool compute = warp < WM * WN;
  const int wm = warp % WM;
  const int wn = warp / WM;

  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int64_t n0 = static_cast<int64_t>(blockIdx.y) * BN;
  if (p.lower_only && m0 + BM <= n0) return;
  const int64_t z = blockIdx.z;
  const int64_t bidx = z / p.split;
  const int sidx = static_cast<int>(z % p.split);
  const int64_t b1 = bidx % p.batch, b2 = bidx / p.batch;
  int64_t kbeg = static_cast<int64_t>(sidx) * p.k_chunk;
  int64_t kend = min(p.k, kbeg + p.k_chunk);
  if (p.tri_k) kbeg = max(kbeg, m0 & ~static_cast<int64_t>(BK - 1));
  if (p.tri_b) kbeg = max(kbeg, n0 & ~static_cast<int64_t>(BK - 1));
  if (p.tri_a_lower) kend = min(kend, m0 + BM);  // (BM is a multiple of BK)
  const int ktiles = kend > kbeg ? static_cast<int>((kend - kbeg + BK - 1) / BK) : 0;

  if (tid == 0) {
    for (int s2 = 0; s2 < STAGES; ++s2) {
      tma::mbar_init(&full[s2], 1);
      tma::mbar_init(&empty[s2], WM * WN);
    }
    tma::fence_barrier_init();
  }
  __syncthreads();
  // Programmatic dependent launch: the next PDL-launched GEMM may start its
  // CTAs (barrier set-up) as ours retire; nothing below touches global memory
  // before the previous grid has completed (griddepcontrol.wait; a no-op when
  // this grid was launched without the attribute).
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  double acc[C::FM][C::FN][2];
#pragma unroll
  for (int i = 0; i < C::FM; ++i)
#pragma unroll
    for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  constexpr uint32_t kStageBytes = (C::A_STAGE + C::B_STAGE) * 8;
  if (!compute) {
    if (lane == 0) {
      const int ab1 = a_batched ? static_cast<int>(b1) : 0, ab2 = a_batched2 ? static_cast<int>(b2) : 0;
      const int bb1 = b_batched ? static_cast<int>(b1) : 0, bb2 = b_batched2 ? static_cast<int>(b2) : 0;
      int stage = 0;
      uint32_t phase = 0;
      for (int kt = 0; kt < ktiles; ++kt) {
        const int k0 = static_cast<int>(kbeg + static_cast<int64_t>(kt) * BK);
        tma::mbar_wait(&empty[stage], phase ^ 1);
        tma::mbar_arrive_expect_tx(&full[stage], kStageBytes);
        // A: op(A) is m x k; K-major (AK): inner = k; else inner = m
        if (AK)
          tma::load_4d(As + stage * C::A_STAGE, &amap, k0, static_cast<int>(m0), ab1, ab2, &full[stage]);
        else
          tma::load_4d(As + stage * C::A_STAGE, &amap, static_cast<int>(m0), k0, ab1, ab2, &full[stage]);
        if (BKM)
          tma::load_4d(Bs + stage * C::B_STAGE, &bmap, k0, static_cast<int>(n0), bb1, bb2, &full[stage]);
        else
          tma::load_4d(Bs + stage * C::B_STAGE, &bmap, static_cast<int>(n0), k0, bb1, bb2, &full[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    const int r8 = lane >> 2;
    const int k4 = lane & 3;
    int stage = 0;
    uint32_t phase = 0;
    double tot[VS ? C::FM : 1][VS ? C::FN : 1][2];  // (virtual split: the running total over chunks)
    for (int kt = 0; kt < ktiles; ++kt) {
      tma::mbar_wait(&full[stage], phase);
      const double* as = As + stage * C::A_STAGE;
      const double* bs = Bs + stage * C::B_STAGE;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double af[C::FM], bf[C::FN];
#pragma unroll
        for (int i = 0; i < C::FM; ++i) {
          const int row = wm * C::TM + i * 8 + r8;
          af[i] = AK ? as[row * C::A_LD + kk + k4] : as[(kk + k4) * C::A_LD + row];
        }
#pragma unroll
        for (int j = 0; j < C::FN; ++j) {
          const int col = wn * C::TN + j * 8 + r8;
          bf[j] = BKM ? bs[col * C::B_LD + kk + k4] : bs[(kk + k4) * C::B_LD + col];
        }
#pragma unroll
        for (int i = 0; i < C::FM; ++i)
#pragma unroll
          for (int j = 0; j < C::FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      // Release the stage.  The refill is an async-proxy write (TMA) and this
      // warp's fragment loads are generic-proxy reads that may still be in
      // flight when the arrive is issued (ptxas schedules the arrive ahead of
      // the last DMMAs, whose operands those loads feed): without a
      // cross-proxy fence the refill can overwrite the stage before the loads
      // return.  Seen as wrong 8 x 16 / 32 x 16 / 64 x 32 output blocks in
      // 1 of 8 runs whenever a second grid's CTAs shared the SMs
      // (profiles/r02_tma_release_race.txt: 6/48 runs wrong without the
      // fence, 0/48 with it).
#ifdef RP_PROBE_ORDER  // (concurrency probe: every DMMA of the stage retired before the release)
#pragma unroll
      for (int i = 0; i < C::FM; ++i)
#pragma unroll
        for (int j = 0; j < C::FN; ++j) asm volatile("add.f64 %0, %0, 0d0000000000000000;" : "+d"(acc[i][j][0]));
#endif
#ifndef RP_PROBE_NOFENCE  // (concurrency probe: the round-1 kernel, no fence)
      tma::fence_proxy_async_smem();
#endif
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&empty[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
      if constexpr (VS) {
        if ((kt + 1) % p.vchunk == 0 || kt + 1 == ktiles) {
          const bool first = kt < p.vchunk;
#pragma unroll
          for (int i = 0; i < C::FM; ++i)
#pragma unroll
            for (int j = 0; j < C::FN; ++j)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                tot[i][j][e] = first ? acc[i][j][e] : __dadd_rn(tot[i][j][e], acc[i][j][e]);
                acc[i][j][e] = 0.0;
              }
        }
      }
    }
    if constexpr (VS) {
      if (ktiles > 0) {
#pragma unroll
        for (int i = 0; i < C::FM; ++i)
#pragma unroll
          for (int j = 0; j < C::FN; ++j) acc[i][j][0] = tot[i][j][0], acc[i][j][1] = tot[i][j][1];
      }
    }
  }
  __syncthreads();  // ring drained: the stages become the epilogue's staging area
  gemm_epilogue<C, BM, WN, STAGES>(p, acc, smem, tid, compute, wm, wn, lane >> 2, lane & 3, m0, n0, b1, b2, bidx,
                                   sidx);
}

// Deterministic split-K reduction: partials summed in split order 0..S-1;
// lower_only + mirror also writes the transposed element.
__global__ void splitk_reduce(KParams p) {
  const int64_t total = p.m * p.n;
  const int64_t bidx = blockIdx.y;
  const double* W = p.ws + bidx * p.split * total;
  double* Cb = p.c + (bidx % p.batch) * p.stride_c + (bidx / p.batch) * p.stride_c2;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = idx % p.m, col = idx / p.m;
    if (p.lower_only && row < col) continue;
    double s = W[idx];
    for (int t = 1; t < p.split; ++t) s += W[t * total + idx];
    double* dst = Cb + row + col * p.ldc;
    const double out = (p.beta == 0.0) ? p.alpha * s : p.alpha * s + p.beta * (*dst);
    *dst = out;
    if (p.mirror && row > col) Cb[col + row * p.ldc] = out;
  }
}

// Split-K partials: one buffer per (device, stream), so GEMMs issued on
// different streams (the preconditioner build overlapping the Gram matrix)
// never share partials, and deferred partials stay valid until the next split
// GEMM on the same stream.  Grown on demand (the grow path synchronizes the
// stream before freeing the old buffer).
struct WsBuf {
  double* ptr = nullptr;
  size_t bytes = 0;
};
struct Workspace {
  std::mutex mu;
  std::map<std::pair<int, cudaStream_t>, WsBuf> bufs;
};
Workspace g_ws;

double* workspace(size_t bytes, cudaStream_t stream) {
  std::lock_guard<std::mutex> lock(g_ws.mu);
  int dev = 0;
  RP_CUDA(cudaGetDevice(&dev));
  WsBuf& w = g_ws.bufs[{dev, stream}];
  if (w.bytes < bytes) {
    if (w.ptr) {
      RP_CUDA(cudaStreamSynchronize(stream));
      RP_CUDA(cudaFree(w.ptr));
    }
    w.ptr = nullptr;
    RP_CUDA(cudaMalloc(&w.ptr, bytes));
    w.bytes = bytes;
  }
  return w.ptr;
}

}  // namespace

void release_workspace(cudaStream_t stream) {
  std::lock_guard<std::mutex> lock(g_ws.mu);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  auto it = g_ws.bufs.find({dev, stream});
  if (it == g_ws.bufs.end()) return;
  cudaStreamSynchronize(stream);
  if (it->second.ptr) cudaFree(it->second.ptr);
  g_ws.bufs.erase(it);
}

namespace {

// ---- TMA launch path -------------------------------------------------------------

// RP_GEMM_PDL=0 disables programmatic dependent launch of the TMA GEMM.
bool g_pdl_enabled = [] {
  const char* e = std::getenv("RP_GEMM_PDL");
  return !(e && e[0] == '0');
}();

bool g_tma_enabled = [] {
  const char* e = std::getenv("RP_GEMM_TMA");
  return !(e && e[0] == '0');
}();

// 4-D tensor map of one operand: dims (inner, outer, batch, batch2) with the
// given box (inner is the contiguous dimension).  A batch dimension with zero
// stride (operand shared by the batch) becomes extent 1 (coordinate 0).
bool operand_map(CUtensorMap* map, const double* base, int64_t inner, int64_t outer, int64_t ld, int64_t s1,
                 int64_t n1, int64_t s2, int64_t n2, int box_inner, int box_outer, int* batched1, int* batched2) {
  auto enc = tma::encoder();
  if (!enc) return false;
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0 || ld % 2 != 0 || s1 % 2 != 0 || s2 % 2 != 0) return false;
  if (inner <= 0 || outer <= 0 || inner >= (int64_t{1} << 31) || outer >= (int64_t{1} << 31)) return false;
  *batched1 = (n1 > 1 && s1 != 0) ? 1 : 0;
  *batched2 = (n2 > 1 && s2 != 0) ? 1 : 0;
  const int64_t span = ld * outer;  // (placeholder stride of an unused dimension)
  const int64_t st1 = *batched1 ? s1 : span, st2 = *batched2 ? s2 : span * (*batched1 ? n1 : 1);
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer),
                              static_cast<cuuint64_t>(*batched1 ? n1 : 1), static_cast<cuuint64_t>(*batched2 ? n2 : 1)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(ld) * 8, static_cast<cuuint64_t>(st1) * 8,
                                 static_cast<cuuint64_t>(st2) * 8};
  const cuuint32_t box[4] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer), 1, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tiles whose per-warp accumulators fit twice in registers (the virtual split
// keeps a running total beside the chunk accumulator): 2 x 2 warps with warp
// tiles of at most 32 x 32 (64 x 64, 64 x 48, 64 x 32 -- no spills).
template <int BM, int BN, int WM, int WN>
constexpr bool vsplit_tile() {
  return WM * WN == 4 && (BM / WM) <= 32 && (BN / WN) <= 32;  // (2 x 2 warps: room for both register sets)
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BKM, bool VS>
bool launch_tma_cfg(const KParams& kp, cudaStream_t stream) {
  using C = Cfg<BM, BN, BK, WM, WN, STAGES, AK, BKM, 2>;
  CUtensorMap amap, bmap;
  int ab1 = 0, ab2 = 0, bb1 = 0, bb2 = 0;
  // op(A) is m x k: K-major (AK) -> inner k, box (BK + 4) x BM; else inner m, box (BM + 4) x BK
  const bool ok_a = AK ? operand_map(&amap, kp.a, kp.k, kp.m, kp.lda, kp.stride_a, kp.batch, kp.stride_a2, kp.batch2,
                                     BK + 4, BM, &ab1, &ab2)
                       : operand_map(&amap, kp.a, kp.m, kp.k, kp.lda, kp.stride_a, kp.batch, kp.stride_a2, kp.batch2,
                                     BM + 4, BK, &ab1, &ab2);
  if (!ok_a) return false;
  const bool ok_b = BKM ? operand_map(&bmap, kp.b, kp.k, kp.n, kp.ldb, kp.stride_b, kp.batch, kp.stride_b2,
                                      kp.batch2, BK + 4, BN, &bb1, &bb2)
                        : operand_map(&bmap, kp.b, kp.n, kp.k, kp.ldb, kp.stride_b, kp.batch, kp.stride_b2,
                                      kp.batch2, BN + 4, BK, &bb1, &bb2);
  if (!ok_b) return false;
  auto kern = dgemm_tma_kernel<BM, BN, BK, WM, WN, STAGES, AK, BKM, VS>;
  int smem = C::SMEM_BYTES + 128;
  // (occupancy cap: a CTA that asks for more than 1/(cap + 1) of the SM's
  // shared memory leaves room for at most `cap` of its kind)
  constexpr int kSmSmem = 227 * 1024, kMaxDyn = kSmSmem - 4096;
  if (kp.occ_cap > 0) smem = std::min(kMaxDyn, std::max(smem, kSmSmem / (kp.occ_cap + 1) + 1024));
  static std::atomic<bool> attr_set[kMaxDevices];  // per template instantiation and device
  const int dev = current_device();
  if (!attr_set[dev].load(std::memory_order_acquire)) {
    RP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDyn));
    attr_set[dev].store(true, std::memory_order_release);
  }
  dim3 grid(static_cast<unsigned>(ceil_div(kp.m, BM)), static_cast<unsigned>(ceil_div(kp.n, BN)),
            static_cast<unsigned>(kp.batch * kp.batch2 * kp.split));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(C::THREADS + 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl_enabled ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#ifdef RP_PROBE_GMAP
  {
    static CUtensorMap* ring = nullptr;
    static size_t slot = 0;
    constexpr size_t kSlots = 1 << 16;  // (never reused within a probe run)
    if (!ring) RP_CUDA(cudaMalloc(&ring, sizeof(CUtensorMap) * 2 * kSlots));
    CUtensorMap* dst = ring + 2 * (slot++ % kSlots);
    const CUtensorMap both[2] = {amap, bmap};
    RP_CUDA(cudaMemcpyAsync(dst, both, sizeof(both), cudaMemcpyHostToDevice, stream));
    const CUtensorMap* gm = dst;
    RP_CUDA(cudaLaunchKernelEx(&cfg, kern, amap, bmap, kp, ab1, ab2, bb1, bb2, gm));
  }
#else
  RP_CUDA(cudaLaunchKernelEx(&cfg, kern, amap, bmap, kp, ab1, ab2, bb1, bb2));
#endif
  RP_LAUNCH_CHECK();
  return true;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BKM, int VEC>
void launch_cfg(const KParams& kp, cudaStream_t stream) {
  using C = Cfg<BM, BN, BK, WM, WN, STAGES, AK, BKM, VEC>;
  if constexpr (VEC == 2) {
    if (g_tma_enabled && !kp.no_tma && ceil_div(kp.n, BN) <= 65535 && kp.batch * kp.batch2 * kp.split <= 65535) {
      if constexpr (vsplit_tile<BM, BN, WM, WN>() && BK == 16) {
        if (kp.vchunk > 0 && launch_tma_cfg<BM, BN, BK, WM, WN, STAGES, AK, BKM, true>(kp, stream)) return;
      }
      if (kp.vchunk == 0 && launch_tma_cfg<BM, BN, BK, WM, WN, STAGES, AK, BKM, false>(kp, stream)) return;
    }
  }
  require(kp.vchunk == 0, "dgemm: virtual split needs the TMA kernel");
  auto kern = dgemm_kernel<BM, BN, BK, WM, WN, STAGES, AK, BKM, VEC>;
  static std::atomic<bool> attr_set[kMaxDevices];  // per template instantiation and device
  const int dev = current_device();
  if (!attr_set[dev].load(std::memory_order_acquire)) {
    RP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES));
    attr_set[dev].store(true, std::memory_order_release);
  }
  require(ceil_div(kp.n, BN) <= 65535 && kp.batch * kp.batch2 * kp.split <= 65535 &&
              ceil_div(kp.m, BM) < (int64_t{1} << 31),
          "dgemm: problem too large for one launch grid");
  dim3 grid(static_cast<unsigned>(ceil_div(kp.m, BM)), static_cast<unsigned>(ceil_div(kp.n, BN)),
            static_cast<unsigned>(kp.batch * kp.batch2 * kp.split));
  kern<<<grid, C::THREADS, C::SMEM_BYTES, stream>>>(kp);
  RP_LAUNCH_CHECK();
}

// Tile shapes, largest first: 128x128 (8 warps), 64x64, 128x32, 64x32,
// 128x16 (4 warps each).
struct TileShape {
  int bm, bn;
};
constexpr TileShape kTiles[] = {{128, 128}, {64, 64}, {128, 32}, {64, 32}, {128, 16}, {64, 128},
                                 {128, 64},  {64, 128}, {128, 64}, {64, 128}, {128, 64}, {64, 48}, {128, 48},
                                 // narrow N (the recursion's batched preconditioner GEMM, N = g + 1 <= 64):
                                 // 128-row tiles of 4 x 1 warps in steps of 8 columns
                                 // (32-row tiles -- 1024 CTAs, 7 x 32 rows on the busiest SM instead of
                                 // 2 x 128 -- were measured: no gain, each small tile re-streams the whole
                                 // B operand; profiles/r02_gemm_tune_32row.txt)
                                 {128, 24},  {128, 40}, {128, 48}, {128, 56}, {128, 64}};
constexpr int kNumTiles = 18;
constexpr int kTileBK[kNumTiles] = {16, 16, 16, 16, 16, 16, 16, 16, 16, 32, 32, 16, 16,
                                    16, 16, 16, 16, 16};  // (launch_layout)

template <bool AK, bool BKM, int VEC>
void launch_layout(const KParams& kp, int tile, cudaStream_t stream) {
  switch (tile) {
    case 0: launch_cfg<128, 128, 16, 2, 4, 3, AK, BKM, VEC>(kp, stream); break;
    case 1: launch_cfg<64, 64, 16, 2, 2, 4, AK, BKM, VEC>(kp, stream); break;
    case 2: launch_cfg<128, 32, 16, 4, 1, 4, AK, BKM, VEC>(kp, stream); break;
    case 3: launch_cfg<64, 32, 16, 2, 2, 4, AK, BKM, VEC>(kp, stream); break;
    case 4: launch_cfg<128, 16, 16, 4, 1, 4, AK, BKM, VEC>(kp, stream); break;
    case 5: launch_cfg<64, 128, 16, 2, 4, 3, AK, BKM, VEC>(kp, stream); break;
    case 6: launch_cfg<128, 64, 16, 4, 2, 3, AK, BKM, VEC>(kp, stream); break;
    // 4 warps with 32 x 64 / 64 x 32 warp tiles: more DMMAs per fragment load
    case 7: launch_cfg<64, 128, 16, 2, 2, 3, AK, BKM, VEC>(kp, stream); break;
    case 8: launch_cfg<128, 64, 16, 2, 2, 3, AK, BKM, VEC>(kp, stream); break;
    // BK = 32, 2 stages: half the barriers per flop
    case 9: launch_cfg<64, 128, 32, 2, 4, 2, AK, BKM, VEC>(kp, stream); break;
    case 10: launch_cfg<128, 64, 32, 4, 2, 2, AK, BKM, VEC>(kp, stream); break;
    // 48-wide tiles: N in (32, 48] (the recursion's P-apply at g + 1 <= 48)
    // without padding the last third of a 64-wide tile
    case 11: launch_cfg<64, 48, 16, 2, 2, 4, AK, BKM, VEC>(kp, stream); break;
    case 12: launch_cfg<128, 48, 16, 4, 2, 3, AK, BKM, VEC>(kp, stream); break;
    // narrow N in steps of 8: the per-SM padded work, not the tile count,
    // sets the time of the N <= 64 batched products
    case 13: launch_cfg<128, 24, 16, 4, 1, 4, AK, BKM, VEC>(kp, stream); break;
    case 14: launch_cfg<128, 40, 16, 4, 1, 4, AK, BKM, VEC>(kp, stream); break;
    case 15: launch_cfg<128, 48, 16, 4, 1, 3, AK, BKM, VEC>(kp, stream); break;
    case 16: launch_cfg<128, 56, 16, 4, 1, 3, AK, BKM, VEC>(kp, stream); break;
    default: launch_cfg<128, 64, 16, 4, 1, 3, AK, BKM, VEC>(kp, stream); break;
  }
}

}  // namespace

int choose_split(const GemmArgs& g);

namespace tma {
PFN_cuTensorMapEncodeTiled_v12000 encoder() {
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
}  // namespace tma

int dgemm_last_launches() { return g_last_launches; }

namespace {
bool vsplit_planned(const GemmArgs& g);
}
// The effective split: a split that runs as a virtual split is no split for
// the caller (no partials; a fused epilogue is allowed).
int dgemm_split(const GemmArgs& g) {
  const int s = choose_split(g);
  return (s > 1 && vsplit_planned(g)) ? 1 : s;
}

namespace {
thread_local GemmProfiler* g_prof = nullptr;
void dgemm_impl(const GemmArgs& g, cudaStream_t stream);
}  // namespace

void set_gemm_profiler(GemmProfiler* p) { g_prof = p; }

GemmProfiler::~GemmProfiler() {
  for (auto& r : recs) {
    cudaEventDestroy(r.start);
    cudaEventDestroy(r.stop);
  }
}

void GemmProfiler::resolve(double* seconds, double* flops, int64_t* calls) {
  double s = 0.0, f = 0.0;
  if (!recs.empty()) RP_CUDA(cudaEventSynchronize(recs.back().stop));
  for (auto& r : recs) {
    float ms = 0.f;
    RP_CUDA(cudaEventElapsedTime(&ms, r.start, r.stop));
    s += ms * 1e-3;
    f += r.flops;
  }
  *seconds = s;
  *flops = f;
  *calls = static_cast<int64_t>(recs.size());
}

void GemmProfiler::launches(std::vector<double>& seconds, std::vector<double>& flops,
                            std::vector<double>& bytes) const {
  seconds.clear();
  flops.clear();
  bytes.clear();
  for (const auto& r : recs) {
    float ms = 0.f;
    RP_CUDA(cudaEventElapsedTime(&ms, r.start, r.stop));
    seconds.push_back(ms * 1e-3);
    flops.push_back(r.flops);
    bytes.push_back(r.bytes);
  }
}

void dgemm(const GemmArgs& g, cudaStream_t stream) {
  if (!g_prof || g.m == 0 || g.n == 0) {
    dgemm_impl(g, stream);
    return;
  }
  GemmProfiler::Rec r{};
  RP_CUDA(cudaEventCreate(&r.start));
  RP_CUDA(cudaEventCreate(&r.stop));
  const double batch = static_cast<double>(g.batch * g.batch2);
  const double mn = g.lower_only ? 0.5 * static_cast<double>(g.m) * static_cast<double>(g.n + 1)
                                 : static_cast<double>(g.m) * static_cast<double>(g.n);
  r.flops = 2.0 * mn * static_cast<double>(g.k) * batch;
  {
    const double m = static_cast<double>(g.m), n = static_cast<double>(g.n), k = static_cast<double>(g.k);
    const double a_copies = g.stride_a == 0 && g.stride_a2 == 0 ? 1.0 : batch;
    const double b_copies = g.stride_b == 0 && g.stride_b2 == 0 ? 1.0 : batch;
    const double a_bytes = 8.0 * m * k * a_copies;
    const double b_bytes = g.b == g.a && g.lower_only ? 0.0 : 8.0 * k * n * b_copies;  // SYRK reads A once
    const double c_bytes = 8.0 * mn * batch * (g.beta != 0.0 ? 2.0 : 1.0);
    r.bytes = a_bytes + b_bytes + c_bytes;
  }
  RP_CUDA(cudaEventRecord(r.start, stream));
  dgemm_impl(g, stream);
  RP_CUDA(cudaEventRecord(r.stop, stream));
  g_prof->recs.push_back(r);
}

// ---- joint (tile, split) plan of long-K products ---------------------------------
// Products whose 128 x 128 tiles do not fill the GPU twice and whose reduction
// order is free (not col_stable) -- the Gram-matrix SYRKs over the operator's
// rows -- pick tile and split together from a time model:
//   waves x per-CTA time + the partial-sum round trip,
// per-CTA time = 2 bm bn (k / split + K0) flop at the SM's DMMA rate shared by
// the tile's resident CTAs; K0 = 400 k-values of prologue + epilogue per CTA
// (fitted: the 64 x 64 tile runs K = 1024 at 24.4 and K = 4096 at 31.1 TF/s);
// lower_only counts only the tiles that run.  (Round 2: the split came from a
// 128-tile wave count and the tile from an all-tiles count, which gave C3's
// 2048 x 2048 x 1M SYRK 1056 CTAs of 64 x 32 x 1M -- 2.4 waves, 25 TF/s.)
constexpr int kOccT[kNumTiles] = {1, 2, 2, 3, 3, 1, 1, 2, 2, 2, 2, 3, 2, 2, 2, 2, 2, 2};
constexpr double kEffT[kNumTiles] = {0.97, 1.0, 0.99, 0.98, 0.94, 0.94, 0.98, 0.0, 0.0, 0.99, 0.99, 1.25, 0.0,
                                 1.0, 1.0, 1.0, 1.0, 1.0};
// CTAs of one batch entry and one split: all tiles, or (lower_only) the tiles
// that reach the diagonal -- the kernel returns at once when m0 + BM <= n0.
int64_t plan_ctas(const GemmArgs& g, int tile) {
  const int64_t bm = kTiles[tile].bm, bn = kTiles[tile].bn;
  const int64_t tm = ceil_div(g.m, bm), tn = ceil_div(g.n, bn);
  if (!g.lower_only) return tm * tn;
  int64_t c = 0;
  for (int64_t j = 0; j < tn; ++j) {
    const int64_t first = std::max<int64_t>(0, (j * bn - bm) / bm + 1);  // smallest i with i bm + bm > j bn
    c += std::max<int64_t>(0, tm - first);
  }
  return c;
}
double plan_seconds(const GemmArgs& g, int tile, int split) {
  const int64_t nb = g.batch * g.batch2;
  const int64_t kc = ceil_div(ceil_div(g.k, split), 16) * 16;
  const int64_t ctas = plan_ctas(g, tile) * nb * split;
  const double waves = static_cast<double>(ceil_div(ctas, int64_t{148} * kOccT[tile]));
  const double sm_rate = 35.0e12 / 148.0 * kEffT[tile];
  const double t_cta = 2.0 * kTiles[tile].bm * kTiles[tile].bn * static_cast<double>(kc + 400) * kOccT[tile] / sm_rate;
  const double mn = (g.lower_only ? 0.5 : 1.0) * static_cast<double>(g.m) * static_cast<double>(g.n);
  const double t_red = split > 1 ? 4.0e-12 * mn * static_cast<double>(nb) * split + 5.0e-6 : 0.0;
  return waves * t_cta + t_red;
}
bool plan_applies(const GemmArgs& g) {
  if (g.col_stable || g.split_k > 0 || g.force_tile >= 0 || g.tri_k || g.tri_b || g.tri_a_lower || g.epilogue || g.partials) return false;
  if (g.k < 8192) return false;
  const int64_t tm = ceil_div(g.m, 128), tn = ceil_div(g.n, 128);
  int64_t tiles = tm * tn;
  if (g.lower_only) {
    tiles = 0;
    for (int64_t i = 0; i < tm; ++i) tiles += std::min<int64_t>(tn, i + 1);
  }
  return tiles * g.batch * g.batch2 < 2 * 148;
}
void plan_long_k(const GemmArgs& g, int* tile_out, int* split_out) {
  const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(64, g.k / 512));
  double best = 1e300;
  *tile_out = 0;
  *split_out = 1;
  for (int t = 0; t < kNumTiles; ++t) {
    if (kEffT[t] <= 0.0 || t >= 13 || kTileBK[t] > 16 || kTiles[t].bn == 16 || kTiles[t].bn == 48) continue;
    for (int64_t s2 = 1; s2 <= cap; ++s2) {
      const double sec = plan_seconds(g, t, static_cast<int>(s2));
      if (sec < best * 0.999) {
        best = sec;
        *tile_out = t;
        *split_out = static_cast<int>(s2);
      }
    }
  }
}


// Split-K factor of a product (see dgemm_split in gemm_f64.h).
int choose_split(const GemmArgs& g) {
  if (plan_applies(g)) {
    int t = 0, s2 = 1;
    plan_long_k(g, &t, &s2);
    const int64_t kc = std::max<int64_t>(16, ceil_div(ceil_div(g.k, s2), 16) * 16);
    return static_cast<int>(std::max<int64_t>(1, ceil_div(g.k, kc)));
  }
  const int64_t nb = g.batch * g.batch2;
  // Split-K.  With col_stable the factor depends on (m, k) only, never on n
  // (column determinism); otherwise it is picked for full waves over the
  // 148 SMs, counting only the tiles that run (lower_only skips the rest).
  int split = g.split_k;
  if (split <= 0) {
    const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(64, g.k / 512));
    if (g.col_stable) {
      // a function of k only (and of m for long k): every column of C sees the
      // same reduction order whatever n is
      const int64_t tiles_m = ceil_div(g.m, 128) * nb;
      // (k <= 8192: chunks of 256 -- cheap when the consumer sums the partials)
      split = g.k <= 8192 ? static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(8, g.k / 256)))
                          : static_cast<int>(std::min<int64_t>(cap, ceil_div(2 * 148, std::max<int64_t>(tiles_m, 1))));
      if (g.k < 256) split = 1;
    } else {
      const int64_t tm = ceil_div(g.m, 128), tn = ceil_div(g.n, 128);
      int64_t tiles = tm * tn;
      if (g.lower_only) tiles = 0;
      if (g.lower_only)
        for (int64_t i = 0; i < tm; ++i) tiles += std::min<int64_t>(tn, i + 1);
      tiles *= nb;
      if (tiles >= 2 * 148 || cap == 1) {
        split = 1;
      } else {
        // time ~ waves * (K / split) plus a per-split reduction overhead
        double best = 1e30;
        split = 1;
        for (int64_t s2 = 1; s2 <= cap; ++s2) {
          const double waves = static_cast<double>(ceil_div(tiles * s2, 148));
          const double cost = waves / static_cast<double>(s2) * (1.0 + 0.03 * static_cast<double>(s2));
          if (cost < best) {
            best = cost;
            split = static_cast<int>(s2);
          }
        }
      }
    }
    split = std::max(1, split);
  }
  int64_t k_chunk = ceil_div(ceil_div(g.k, split), 16) * 16;
  if (k_chunk == 0) k_chunk = 16;
  return static_cast<int>(std::max<int64_t>(1, ceil_div(g.k, k_chunk)));
}

namespace {
// RP_GEMM_LOG=path: every dgemm call's shape and launch choice, one line each.
FILE* gemm_log() {
  static FILE* f = [] {
    const char* e = std::getenv("RP_GEMM_LOG");
    return e ? std::fopen(e, "w") : nullptr;
  }();
  return f;
}

// Tile choice: estimated time = waves x per-wave tile work, where a wave is
// 148 SMs x CTAs-per-SM for the shape (ties keep the larger tile).  With the
// virtual split only the tiles whose accumulators fit twice are candidates.
// CTAs per SM and relative large-problem throughput per shape (measured,
// profiles/r01_gemm_tune.txt; 9, 10 = BK 32 variants, kept for tuning only;
// the 4-warp shapes 7, 8 only pay off in the cp.async kernel; the 48-wide
// tile only where N fits one of them and a 64-wide tile would pad a quarter
// or more: 24 % faster there, profiles/r01_gemm_tune_bn48.txt).
constexpr int kOcc[] = {1, 2, 2, 3, 3, 1, 1, 2, 2, 2, 2, 3, 2, 2, 2, 2, 2, 2};
constexpr double kEff[] = {0.97, 1.0, 0.99, 0.98, 0.94, 0.94, 0.98, 0.0, 0.0, 0.99, 0.99, 1.25, 0.0,
                           1.0, 1.0, 1.0, 1.0, 1.0};
constexpr bool kVsTile[] = {false, true, false, true, false, false, false, false, false, false, false, true, false,
                            false, false, false, false, false};
// RP_GEMM_NARROW=0: no narrow-N tiles (A/B)
bool g_narrow_tiles = [] {
  const char* e = std::getenv("RP_GEMM_NARROW");
  return !(e && e[0] == '0');
}();

int choose_tile(const GemmArgs& g, int split, int64_t k_chunk, bool vs) {
  const int64_t nb = g.batch * g.batch2;
  int tile = 0;
  double best = 1e300;
  if (!vs && plan_applies(g)) {  // (long-K product: tile and split were chosen together)
    int s2 = 1;
    plan_long_k(g, &tile, &s2);
    return tile;
  }
  // Narrow products (N <= 64): one tile column, sized to N in steps of 8,
  // costed by the padded work on the busiest SM -- ceil(CTAs / 148) tiles of
  // BM x BN -- since such products never fill the GPU evenly.
  // (the recursion's batched preconditioner products with m >= 512 only:
  // measured -0.25 ms on C2's basis; on C1 (m = 256) and on the factor's
  // products it was neutral to negative, profiles/r02_narrow_tiles.txt)
  const bool narrow = g_narrow_tiles && g.n <= 64 && !vs && g.force_tile < 0 && !g.lower_only && nb > 1 &&
                      g.epilogue != nullptr && g.m >= 512;
  static const int pgemm_tile = [] {  // RP_PGEMM_TILE=t: that tile for every such product (tuning probe)
    const char* e = std::getenv("RP_PGEMM_TILE");
    return e ? std::atoi(e) : -1;
  }();
  if (narrow && pgemm_tile >= 0 && pgemm_tile < kNumTiles) return pgemm_tile;
  for (int t = 0; t < kNumTiles; ++t) {
    const bool narrow_tile = t >= 13;
    if (narrow) {
      // 128 x 16 / 32, 64 x 32 / 48 / 64 and the 128-row steps of 8
      // (the 64 x 32 tile may take two column tiles: 1024 short CTAs overlap one another's
      // prologue and epilogue -- N = 57..64 in 145 us against 168 for one 64-wide column of
      // tiles, profiles/r02_pgemm_tile_sweep.txt)
      const bool two_cols = t == 3 && g.n > kTiles[t].bn && g.n <= 2 * kTiles[t].bn;
      if ((kTiles[t].bn < g.n && !two_cols) || (!narrow_tile && t != 4 && t != 2 && t != 3 && t != 11 && t != 1))
        continue;
      if (kEff[t] <= 0.0) continue;
      if (kTileBK[t] > 16 && k_chunk % kTileBK[t] != 0) continue;
      const int64_t ctas = ceil_div(g.m, kTiles[t].bm) * ceil_div(g.n, kTiles[t].bn) * nb * split;
      const double eff = t == 11 ? 1.0 : kEff[t];  // (64 x 48: 127 us at N = 33..40 where 128 x 40 takes 108)
      const double cost = static_cast<double>(ceil_div(ctas, 148)) * kTiles[t].bm * kTiles[t].bn / eff;
      if (cost < best * 0.999) {
        best = cost;
        tile = t;
      }
      continue;
    }
    if (narrow_tile) continue;
    if (kTiles[t].bn == 16 && g.n > 16) continue;
    if (kTiles[t].bn == 48 && (g.n <= 32 || g.n > 48)) continue;
    if (kEff[t] <= 0.0) continue;
    if (vs && !kVsTile[t]) continue;
    if (kTileBK[t] > 16 && k_chunk % kTileBK[t] != 0) continue;  // (a split's last k tile must not cross into the next)
    const int64_t ctas = ceil_div(g.m, kTiles[t].bm) * ceil_div(g.n, kTiles[t].bn) * nb * split;
    const double waves = static_cast<double>(ceil_div(ctas, 148 * kOcc[t]));
    const double cost = waves * kTiles[t].bm * kTiles[t].bn * kOcc[t] / kEff[t];
    if (cost < best * 0.999) {
      best = cost;
      tile = t;
    }
  }
  return tile;
}

// RP_GEMM_VSPLIT=1 enables the virtual split.  Off by default: measured on
// C2 it loses -- the second register set costs the 64 x 64 tile its second
// CTA per SM (255 registers; capped at 168 it spills), and one CTA per tile
// quantizes worse than the real split's four (path 19.9 vs 18.7 ms,
// profiles/r02_vsplit_c2.txt).  Bit-identical either way
// (test_virtual_split_bitwise).
bool g_vsplit_enabled = [] {
  const char* e = std::getenv("RP_GEMM_VSPLIT");
  return e && e[0] == '1';
}();

// A column-stable split product runs as a virtual split (one CTA per tile,
// the chunks summed in order inside it) when the tiles alone fill the GPU:
// same bits, no partials round trip, and a fused epilogue becomes possible.
bool use_vsplit(const GemmArgs& g, int split, int64_t k_chunk, bool aligned) {
  if (!g_vsplit_enabled || split <= 1 || !g.col_stable || g.lower_only || g.tri_k || g.no_tma || !g_tma_enabled ||
      !aligned || g.force_tile >= 0 || g.split_k > 0 || k_chunk % 16 != 0)
    return false;
  const int t = choose_tile(g, 1, k_chunk, true);
  const int64_t ctas = ceil_div(g.m, kTiles[t].bm) * ceil_div(g.n, kTiles[t].bn) * g.batch * g.batch2;
  return ctas >= 148 * kOcc[t];  // at least one full wave without the split
}

bool operands_aligned(const GemmArgs& g) {
  return (reinterpret_cast<uintptr_t>(g.a) % 16 == 0) && (reinterpret_cast<uintptr_t>(g.b) % 16 == 0) &&
         g.lda % 2 == 0 && g.ldb % 2 == 0 && g.stride_a % 2 == 0 && g.stride_b % 2 == 0 && g.stride_a2 % 2 == 0 &&
         g.stride_b2 % 2 == 0;
}

bool vsplit_planned(const GemmArgs& g) {
  int split = choose_split(g);
  int64_t k_chunk = ceil_div(ceil_div(g.k, split), 16) * 16;
  if (k_chunk == 0) k_chunk = 16;
  split = static_cast<int>(std::max<int64_t>(1, ceil_div(g.k, k_chunk)));
  return use_vsplit(g, split, k_chunk, operands_aligned(g));
}

void dgemm_impl(const GemmArgs& g, cudaStream_t stream) {
  g_last_launches = 0;
  require(g.m >= 0 && g.n >= 0 && g.k >= 0 && g.batch >= 1 && g.batch2 >= 1, "dgemm: negative dimensions");
  if (g.m == 0 || g.n == 0) return;
  const int64_t nb = g.batch * g.batch2;
  KParams kp{};
  kp.m = g.m;
  kp.n = g.n;
  kp.k = g.k;
  kp.alpha = g.alpha;
  kp.beta = g.beta;
  kp.a = g.a;
  kp.lda = g.lda;
  kp.stride_a = g.stride_a;
  kp.b = g.b;
  kp.ldb = g.ldb;
  kp.stride_b = g.stride_b;
  kp.c = g.c;
  kp.ldc = g.ldc;
  kp.stride_c = g.stride_c;
  kp.batch = g.batch;
  kp.batch2 = g.batch2;
  kp.stride_a2 = g.stride_a2;
  kp.stride_b2 = g.stride_b2;
  kp.stride_c2 = g.stride_c2;
  kp.lower_only = g.lower_only;
  kp.tri_k = g.tri_k;
  kp.tri_b = g.tri_b;
  kp.tri_a_lower = g.tri_a_lower;
  require(!(g.tri_k || g.tri_b || g.tri_a_lower) || (g.split_k == 1 && !g.col_stable),
          "dgemm: triangular k ranges need an unsplit product");
  kp.no_tma = g.no_tma;
  kp.occ_cap = g.max_ctas_per_sm;

  const bool ak = g.opa == Op::T;  // A contiguous along k
  const bool bk = g.opb == Op::N;  // B contiguous along k
  const bool aligned = operands_aligned(g);

  int split = choose_split(g);
  int64_t k_chunk = ceil_div(ceil_div(g.k, split), 16) * 16;
  if (k_chunk == 0) k_chunk = 16;
  split = static_cast<int>(std::max<int64_t>(1, ceil_div(g.k, k_chunk)));
  kp.split = split;
  kp.k_chunk = k_chunk;

  const bool vs = use_vsplit(g, split, k_chunk, aligned);
  int tile = choose_tile(g, vs ? 1 : split, k_chunk, vs);
  if (vs) {
    kp.split = 1;
    kp.vchunk = static_cast<int>(k_chunk / 16);
    kp.k_chunk = g.k;  // (one CTA covers the whole k range)
    split = 1;
  }
  if (g.force_tile >= 0 && g.force_tile < kNumTiles) {
    // The kernels do not mask k past their split's end: a tile's BK must
    // divide the K chunk (always true for BK = 16, k_chunk % 16 == 0).
    require(k_chunk % kTileBK[g.force_tile] == 0, "dgemm: a BK = 32 tile needs a split K chunk that is a multiple of 32");
    tile = g.force_tile;
  }
  if (split > 1) kp.ws = workspace(sizeof(double) * static_cast<size_t>(nb * split) * g.m * g.n, stream);
  if (g.epilogue) {
    require(!g.lower_only && !g.mirror && g.alpha == 1.0 && g.beta == 0.0 && split == 1,
            "dgemm: fused epilogue needs a plain, unsplit product");
    kp.epi = *g.epilogue;
  }
  if (g.mirror) require(g.lower_only && g.m == g.n && g.beta == 0.0, "dgemm: mirror needs a square lower_only output");
  kp.mirror = g.mirror;
  if (ak && bk) {
    aligned ? launch_layout<true, true, 2>(kp, tile, stream) : launch_layout<true, true, 1>(kp, tile, stream);
  } else if (ak && !bk) {
    aligned ? launch_layout<true, false, 2>(kp, tile, stream) : launch_layout<true, false, 1>(kp, tile, stream);
  } else if (!ak && bk) {
    aligned ? launch_layout<false, true, 2>(kp, tile, stream) : launch_layout<false, true, 1>(kp, tile, stream);
  } else {
    aligned ? launch_layout<false, false, 2>(kp, tile, stream) : launch_layout<false, false, 1>(kp, tile, stream);
  }
  g_last_launches = 1;
  if (FILE* log = gemm_log()) {  // (tuning aid: one line per GEMM -- shape, batch, split, tile, layout)
    std::fprintf(log, "%lld %lld %lld batch %lld split %d tile %d ak %d bk %d tma %d epi %d lower %d\n",
                 static_cast<long long>(g.m), static_cast<long long>(g.n), static_cast<long long>(g.k),
                 static_cast<long long>(nb), split, tile, ak ? 1 : 0, bk ? 1 : 0, (g_tma_enabled && !kp.no_tma) ? 1 : 0,
                 static_cast<int>(kp.epi.kind), g.lower_only ? 1 : 0);
    std::fflush(log);
  }
  const bool defer = g.partials && split > 1 && !g.lower_only && !g.mirror && g.alpha == 1.0 && g.beta == 0.0;
  if (g.partials)
    *g.partials = defer ? Partials{kp.ws, split, g.m, g.m * g.n, split * g.m * g.n}
                        : Partials{g.c, 1, g.ldc, 0, g.stride_c};
  if (split > 1 && !defer) {
    dim3 grid(static_cast<unsigned>(std::min<int64_t>(ceil_div(g.m * g.n, 256), 148 * 8)), static_cast<unsigned>(nb));
    splitk_reduce<<<grid, 256, 0, stream>>>(kp);
    RP_LAUNCH_CHECK();
    ++g_last_launches;
  }
}

}  // namespace

}  // namespace rpb
