// FP64 tensor-core GEMM (DMMA via mma.sync.m8n8k4.f64) for sm_100a.
//
// tcgen05/UMMA has no f64 kind, so FP64 tensor work on Blackwell is the
// warp-level DMMA path; this kernel stages operands global->shared with a
// multi-stage cp.async pipeline and keeps accumulators in registers.
//
// C = alpha * op(A) * op(B) + beta * C, column-major, optional strided batch.
// Every output element is reduced over k in a fixed order that depends only on
// (K, split) -- never on N -- so a column of C is bit-identical whether it is
// computed alone or inside a wider batch (the property the reference pins in
// test_path_solver.cpp "matrix basis equals independent vector runs").
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace rpb {

enum class Op { N, T };

struct GemmArgs {
  Op opa = Op::N, opb = Op::N;
  int64_t m = 0, n = 0, k = 0;
  double alpha = 1.0, beta = 0.0;
  const double* a = nullptr;
  int64_t lda = 0, stride_a = 0;
  const double* b = nullptr;
  int64_t ldb = 0, stride_b = 0;
  double* c = nullptr;
  int64_t ldc = 0, stride_c = 0;
  int64_t batch = 1;
  // Optional second batch dimension (batch index = b1 + batch * b2).
  int64_t batch2 = 1;
  int64_t stride_a2 = 0, stride_b2 = 0, stride_c2 = 0;
  // Only the lower triangle (row >= col) of each output tile is meaningful and
  // tiles strictly above the diagonal are skipped (SYRK: C = A^T A).  The upper
  // triangle is filled by a mirror pass when `mirror` is set.
  bool lower_only = false;
  bool mirror = false;
  // op(A)(i, k) == 0 for k < i (A^T of a lower-triangular matrix): each output
  // tile skips the k range below its first row.  Requires split_k == 1.
  bool tri_k = false;
  // op(B)(k, j) == 0 for k < j (B lower triangular as a k x n matrix): each
  // output tile starts its k range at its first column.  Requires split_k == 1.
  bool tri_b = false;
  // op(A)(i, k) == 0 for k > i (A lower triangular as an m x k matrix): each
  // output tile ends its k range at its last row.  Requires split_k == 1.
  bool tri_a_lower = false;
  // Use the cp.async kernel instead of the TMA one (A/B switch).
  bool no_tma = false;
  // At most this many CTAs of the launch per SM (0 = the kernel's natural
  // occupancy): the TMA kernel pads its dynamic shared memory so that the
  // rest of every SM stays free for another stream's kernels (the Gram SYRK
  // overlapping the latency-bound Cholesky chain).
  int max_ctas_per_sm = 0;
  // Deterministic split-K factor; 0 = heuristic.  With col_stable the
  // heuristic looks at (m, k) only, so column j of C does not depend on n.
  int split_k = 0;
  bool col_stable = false;
    // Deferred split-K: when the chosen split is > 1 the partial products are
  // left in `*partials` (see Partials) for the consumer to sum in split order,
  // and no reduction kernel runs.  Ignored for lower_only / mirror.
  struct Partials* partials = nullptr;
  // Tuning hook: force a tile shape index (see gemm_f64.cu kTiles), -1 = auto.
  int force_tile = -1;
  // Fused consumer of C (replaces the plain store; see RecursionEpilogue).
  const struct RecursionEpilogue* epilogue = nullptr;
};

// Epilogues of the binomial-basis recursion (path_solver.cpp:37-49) fused
// into the GEMM that produces their input, so each generation is two kernels.
// Problems b = l*K + r (interval l, right-hand side r); gen / tilde are
// dim x (kmax*NB) with column j*NB + b; args is interval-major
// (dim x kmax*K per interval, column j*K + r).  See basis.h.
//   kArgs   C = G * gen[:, :g*NB] (column j*NB + b):
//           args[l][:, j*K + r] = tau_l * C + (j >= 1 ? gen[:, (j-1)*NB + b] : 0)
//   kUpdate C_l = P_l * args[l][:, :(g+1)*K] (batch l, column j*K + r), for
//           intervals with g < k_l:  gen[:, j*NB+b] = (j < g ? gen - C : -C),
//           tilde += gen, flags[l] |= non-finite, and the next generation's
//           last argument column args[l][:, (g+1)*K + r] = gen[:, g*NB + b].
// Element-wise arithmetic is the standalone kernels' (build_args / update_gen),
// so both routes give identical bits.
struct RecursionEpilogue {
  enum Kind { kArgs = 1, kUpdate = 2 };
  int kind = 0;
  int64_t dim = 0, L = 0, K = 0, kmax = 0, g = 0;
  const double* tau = nullptr;
  const int* kb = nullptr;
  double* gen = nullptr;
  double* tilde = nullptr;
  double* args = nullptr;
  int* flags = nullptr;
};

// Where a GEMM result lives when its reduction is deferred.  Element (i, j) of
// batch b is  sum_{s < split} p[b * batch_stride + s * split_stride + i + j * ld]
// (summed in s order -- bitwise what the split-K reduction kernel computes).
struct Partials {
  const double* p = nullptr;
  int split = 1;
  int64_t ld = 0;
  int64_t split_stride = 0;
  int64_t batch_stride = 0;
};

// Launches on `stream`.  `workspace` (may be null) is used for split-K partials;
// when null and a split is wanted, an internal cached buffer is used.
void dgemm(const GemmArgs& g, cudaStream_t stream);

// Frees the split-K workspace cached for `stream` (after synchronizing it).
// Owners of streams call it before destroying them, so no workspace outlives
// its stream and a recycled stream handle never inherits a stale entry.
void release_workspace(cudaStream_t stream);

// The split-K factor dgemm() would use for `g` (1 = no split: a fused
// epilogue is only allowed then).
int dgemm_split(const GemmArgs& g);

// Number of kernel launches issued by the last dgemm() call on this thread.
int dgemm_last_launches();

// Optional per-thread GEMM profiler: while installed, every dgemm() call is
// bracketed by CUDA events on its stream and its algorithmic flops recorded.
struct GemmProfiler {
  struct Rec {
    cudaEvent_t start, stop;
    double flops;
    double bytes;  // algorithmic operand bytes: A and B read once, C written (and read when beta != 0)
  };
  std::vector<Rec> recs;
  ~GemmProfiler();
  // Synchronizes on the last event and returns (seconds, flops, calls).
  void resolve(double* seconds, double* flops, int64_t* calls);
  // Per-launch (seconds, flops, bytes), in launch order (after resolve).
  void launches(std::vector<double>& seconds, std::vector<double>& flops, std::vector<double>& bytes) const;
};
void set_gemm_profiler(GemmProfiler* p);

}  // namespace rpb
