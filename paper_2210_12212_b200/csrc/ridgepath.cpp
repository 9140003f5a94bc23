// Host orchestration of the IHS-BIN path on the device, and the C ABI
// (include/ridgepath_b200.h).
//
// Mirrors path_solver.cpp: run_path (:147-190), plan_intervals (:85-108),
// build_interval_basis_matrix with the tau/2 retry (:110-141), ihs_basis_core
// (:27-53), compose_horner (:64-74) and the ihs_bin_path / ihs_bin_path_matrix
// / dual_path wrappers (:289-351); spectrum.cpp's scalar tuning is restated
// verbatim on the host (same glibc libm), so the plans are bit-identical.
//
// Device design (B200): every interval and right-hand side of the path runs
// its recursion in lockstep -- one Gram product and one batched preconditioner
// GEMM per generation for the whole path (L*K problems) instead of L*K*(k-1)
// sequential products.  The Gram operator is either a pass over the data
// (M^T (M W), two DMMA GEMMs or two sparse products) or, when cheaper, the
// precomputed Gram matrix G = M^T M (one DMMA SYRK) applied as G W.
#include <cusolverDn.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <limits>
#include <chrono>
#include <string_view>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <optional>
#include <string>
#include <vector>

#include "basis.h"
#include "common.h"
#include "draws.h"
#include "factor.h"
#include "gemm_f64.h"
#include "gram_pass.h"
#include "mt19937.h"
#include "operator.h"
#include "ridgepath_b200.h"
#include "sketch.h"
#include "sparse_gram.h"
#include "spectrum.h"
#include "vecops.h"

namespace rpb {

// ---------------------------------------------------------------------------
// Scalar tuning, restated from spectrum.cpp (host, bit-identical).
// ---------------------------------------------------------------------------

struct Rho {
  double rho1 = 1.0, rho2 = 1.0;
  int provenance = 3;
};

void rho_validate(const Rho& r) {  // spectrum.cpp:71-76
  require(r.rho2 > 0.0, "rho bounds: rho2 must be positive");
  require(r.rho1 >= r.rho2, "rho bounds: rho1 must be >= rho2");
  if (r.provenance == 3) require(r.rho1 == 1.0 && r.rho2 == 1.0, "identity rho bounds must be (1,1)");
}

std::vector<double> log_grid(double lo, double hi, int count) {  // spectrum.cpp:38-53
  require(count >= 1, "log_grid: count must be >= 1");
  require(lo > 0.0 && hi >= lo, "log_grid: bad range");
  std::vector<double> g(static_cast<size_t>(count));
  if (count == 1) {
    g[0] = lo;
    return g;
  }
  const double lr = std::log(hi / lo);
  for (int i = 0; i < count; ++i) g[i] = lo * std::exp(lr * static_cast<double>(i) / (count - 1));
  g.front() = lo;
  g.back() = hi;
  return g;
}

rp_rate_params tune_interval(double lambda_lo, double lambda_hi, const Rho& rho, std::optional<double> sigma_d,
                             double eps) {  // spectrum.cpp:171-203
  require(lambda_lo > 0.0, "tune_interval: lambda_lo must be positive");
  require(lambda_lo <= lambda_hi, "tune_interval: interval ordering violated");
  require(eps > 0.0 && eps < 1.0, "tune_interval: eps not in (0,1)");
  rho_validate(rho);
  const double shift = sigma_d ? (*sigma_d) * (*sigma_d) : 0.0;
  require(shift >= 0.0, "tune_interval: sigma_d must be nonnegative");
  const double lo = lambda_lo + shift;
  const double hi = lambda_hi + shift;
  rp_rate_params out{};
  out.lambda0 = std::sqrt(lo * hi) - shift;
  out.kappa = rho.rho1 * hi / (rho.rho2 * lo);
  out.alpha = 2.0 * std::sqrt(lo * hi) / (lo / rho.rho1 + hi / rho.rho2);
  const double rate = (out.kappa - 1.0) / (out.kappa + 1.0);
  out.contraction = rate * rate;
  if (out.contraction <= 0.0) {
    out.k = 2;
  } else {
    const double per_step = -std::log(rate);
    const double raw = std::ceil(std::log(1.0 / eps) / per_step);
    out.k = static_cast<int>(std::clamp(raw, 2.0, 64.0));
  }
  return out;
}

int auto_interval_count(double lo, double hi) {  // spectrum.cpp:205-211
  require(lo > 0.0 && lo < hi, "interval_split: need 0 < lambda_min < lambda_max");
  return std::max(1, static_cast<int>(std::floor(2.0 * std::log(hi / lo))));
}

std::vector<std::pair<double, double>> interval_split(double lo, double hi, std::optional<int> num) {
  require(lo > 0.0 && lo < hi, "interval_split: need 0 < lambda_min < lambda_max");  // spectrum.cpp:213-233
  const int count = num ? *num : auto_interval_count(lo, hi);
  require(count >= 1, "interval_split: L must be >= 1");
  const double log_beta = std::log(hi / lo);
  std::vector<double> edges(static_cast<size_t>(count) + 1);
  for (int i = 0; i <= count; ++i) edges[i] = lo * std::exp(log_beta * static_cast<double>(i) / count);
  edges.front() = lo;
  edges.back() = hi;
  std::vector<std::pair<double, double>> out;
  for (int i = 0; i < count; ++i) out.emplace_back(edges[i], edges[i + 1]);
  return out;
}

struct PathCfg {
  double lambda_min = 0, lambda_max = 0;
  std::vector<double> lambdas;
  double epsilon = 1e-6;
  std::optional<int> num_intervals;
  void validate() const {  // spectrum.cpp:20-36
    require(lambda_min > 0.0 && lambda_max > 0.0, "path config: lambda bounds must be positive");
    require(lambda_min < lambda_max, "path config: lambda_min must be below lambda_max");
    require(!lambdas.empty(), "path config: empty evaluation grid");
    require(epsilon > 0.0 && epsilon < 1.0, "path config: epsilon not in (0,1)");
    double prev = lambda_min;
    for (double l : lambdas) {
      require(l >= prev, "path config: grid must be sorted ascending");
      prev = l;
    }
    require(lambdas.front() >= lambda_min && lambdas.back() <= lambda_max,
            "path config: grid must lie within [lambda_min, lambda_max]");
    if (num_intervals) require(*num_intervals >= 1, "path config: L must be >= 1");
  }
};

struct IntervalPlan {
  double lo = 0, hi = 0;
  rp_rate_params params{};
  std::vector<int64_t> grid;  // indices into cfg.lambdas
};

std::vector<IntervalPlan> plan_intervals(const PathCfg& cfg, const Rho& rho, std::optional<double> sigma_d) {
  const auto splits = interval_split(cfg.lambda_min, cfg.lambda_max, cfg.num_intervals);  // path_solver.cpp:85-108
  std::vector<IntervalPlan> plans;
  size_t cursor = 0;
  for (size_t i = 0; i < splits.size(); ++i) {
    IntervalPlan p;
    p.lo = splits[i].first;
    p.hi = splits[i].second;
    p.params = tune_interval(p.lo, p.hi, rho, sigma_d, cfg.epsilon);
    const bool last = (i + 1 == splits.size());
    while (cursor < cfg.lambdas.size() && (last || cfg.lambdas[cursor] <= p.hi)) {
      p.grid.push_back(static_cast<int64_t>(cursor));
      ++cursor;
    }
    plans.push_back(std::move(p));
  }
  return plans;
}

// ---------------------------------------------------------------------------
// NCCL, loaded at run time (the library does not link a specific NCCL; in a
// PyTorch process the already-loaded libnccl.so.2 is reused).
// ---------------------------------------------------------------------------

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.handle) break;
    }
    if (api.handle) {
      api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(api.handle, "ncclGetUniqueId"));
      api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(api.handle, "ncclCommInitRank"));
      api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(api.handle, "ncclAllReduce"));
      api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(api.handle, "ncclAllGather"));
      api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(api.handle, "ncclCommDestroy"));
      api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(api.handle, "ncclGetErrorString"));
    }
  }
  if (!api.handle || !api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.AllGather)
    throw NcclFailure("NCCL (libnccl.so.2) could not be loaded");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw NcclFailure(std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "error"));
}

// ---------------------------------------------------------------------------
// Context
// ---------------------------------------------------------------------------

// Chunked asynchronous upload of a host operator (RP_HOST_STREAM).  Chunks
// are enqueued on the context's copy stream a few at a time (`enqueue`), so
// the small host<->device copies the consumer issues meanwhile are never
// queued behind the whole transfer; one event per chunk.
struct Upload {
  std::vector<cudaEvent_t> ev;   // per chunk (created up front, recorded when enqueued)
  int64_t chunk = 0;             // columns per chunk
  int64_t next = 0;              // first chunk not yet enqueued
  const double* src = nullptr;   // host source (column-major, leading dim lda)
  int64_t lda = 0, rows = 0, cols = 0;
  double* dst = nullptr;         // device destination (leading dim rows)
  cudaStream_t copy = nullptr;
  Upload() = default;
  Upload(const Upload&) = delete;
  Upload& operator=(const Upload&) = delete;
  Upload(Upload&& o) noexcept { *this = std::move(o); }
  Upload& operator=(Upload&& o) noexcept {
    if (this != &o) {
      release();
      ev = std::move(o.ev);
      chunk = o.chunk;
      next = o.next;
      src = o.src;
      lda = o.lda;
      rows = o.rows;
      cols = o.cols;
      dst = o.dst;
      copy = o.copy;
      o.ev.clear();
      o.next = 0;
    }
    return *this;
  }
  ~Upload() { release(); }
  void release() {
    for (auto e : ev) cudaEventDestroy(e);
    ev.clear();
  }
  int64_t chunks() const { return static_cast<int64_t>(ev.size()); }
  // Enqueue chunks [next, min(upto, chunks)).
  void enqueue(int64_t upto) {
    for (; next < std::min<int64_t>(upto, chunks()); ++next) {
      const int64_t c0 = next * chunk, cc = std::min(chunk, cols - c0);
      if (cc > 0 && rows > 0)
        RP_CUDA(cudaMemcpy2DAsync(dst + c0 * rows, sizeof(double) * rows, src + c0 * lda, sizeof(double) * lda,
                                  sizeof(double) * rows, static_cast<size_t>(cc), cudaMemcpyHostToDevice, copy));
      RP_CUDA(cudaEventRecord(ev[static_cast<size_t>(next)], copy));
    }
  }
};

constexpr int64_t kUploadDepth = 2;  // chunks kept in flight ahead of the consumer

struct OperatorStore {
  double free_after_alloc = 0.0;  // free device bytes when a streamed upload's buffer was allocated
  bool set = false;
  bool sparse = false;
  int shard = 0;  // 0 none, 1 rows, 2 cols
  int64_t n = 0, d = 0;          // global shape of A
  int64_t off0 = 0, n_local = 0; // shard offset / extent (rows or cols)
  // dense
  const double* a = nullptr;
  int64_t lda = 0;
  DBuf<double> owned;
  // csr (+csc) of the local block
  DBuf<int64_t> csr_off, csc_off;
  DBuf<int32_t> csr_col, csc_row;
  DBuf<double> csr_val, csc_val;
  int64_t nnz = 0;
  // per-panel CSC of the primal / dual operator (sparse Gram passes), built lazily
  PanelCsc panels_primal, panels_dual;
  Upload up;  // pending chunked upload (RP_HOST_STREAM)

  // Primal operator M = A (rows local).
  OpView primal() const {
    OpView v;
    require(set, "no operator set");
    require(shard != 2, "this operator is column-sharded: use the dual route");
    v.n_global = n;
    v.row0 = shard == 1 ? off0 : 0;
    v.n_loc = shard == 1 ? n_local : n;
    v.d = d;
    v.sparse = sparse;
    if (!sparse) {
      v.a = a;
      v.ld = lda;
      v.trans = false;
    } else {
      v.csr_off = csr_off.get();
      v.csr_col = csr_col.get();
      v.csr_val = csr_val.get();
      v.csc_off = csc_off.get();
      v.csc_row = csc_row.get();
      v.csc_val = csc_val.get();
      v.nnz = nnz;
    }
    return v;
  }
  // Dual operator M = A^T (rows of M = columns of A).
  OpView dual() const {
    OpView v;
    require(set, "no operator set");
    require(shard != 1, "this operator is row-sharded: use the primal route");
    v.n_global = d;
    v.row0 = shard == 2 ? off0 : 0;
    v.n_loc = shard == 2 ? n_local : d;
    v.d = n;
    v.sparse = sparse;
    if (!sparse) {
      v.a = a;
      v.ld = lda;
      v.trans = true;
    } else {
      v.csr_off = csc_off.get();
      v.csr_col = csc_row.get();
      v.csr_val = csc_val.get();
      v.csc_off = csr_off.get();
      v.csc_row = csr_col.get();
      v.csc_val = csr_val.get();
      v.nnz = nnz;
    }
    return v;
  }
};

}  // namespace rpb

struct rp_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t copy = nullptr;  // upload stream of RP_HOST_STREAM operators (created on first use)
  cudaStream_t side = nullptr;  // side stream: the Gram matrix overlapping the sketch and the preconditioner build
  cudaStream_t hi = nullptr;    // second stream: the sketch while the Gram matrix is in flight
  cudaStream_t basis2 = nullptr;  // second stream of the two-group basis recursion (option "basis_streams")
  // option "basis_streams": 1 = one recursion over all intervals, 2 = two interval groups on two streams,
  // interleaved generation by generation (exact; measured: no gain -- C2 -0.1 ms, C4 7.73 vs 7.72 s, the
  // sparse Gram passes and the other group's GEMMs each fill every SM and take turns instead of overlapping)
  int basis_streams = 1;
  rpb::OperatorStore op;
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  // host-side communicator (rp_comm_init_host): collectives through caller callbacks
  rp_host_allreduce_fn host_allreduce = nullptr;
  rp_host_allgather_fn host_allgather = nullptr;
  void* host_user = nullptr;
  double* host_stage = nullptr;  // pinned staging buffer of the host collectives
  size_t host_stage_count = 0;
  int gram_mode = -1;
  bool profile = false;
  double last_device_seconds = 0.0;  // profile: device time of the last product call
  bool fuse_update = true;           // option "fuse_update": recursion update in the P GEMM epilogue
  bool stable_columns = true;        // option "stable_columns": column-stable GEMMs inside the path
  bool compose_gemm = true;          // option "compose_gemm": x(lambda) as a DMMA GEMM (0: Horner kernel, the reference's order)
  int gram_overlap_tile = -1;  // option "gram_overlap_tile": GEMM tile of the overlapped Gram SYRK (-1 = auto)
  // option "gram_overlap_tma": 1 = the overlapped SYRK on the TMA kernel (0: cp.async, A/B switch)
  bool gram_overlap_tma = true;
  int gram_overlap_split = 0;     // option "gram_overlap_split": split-K of the overlapped SYRK (0 = auto; probe)
  int gram_overlap_occ = 0;       // option "gram_overlap_occ": at most this many CTAs of that SYRK per SM (0 = no cap)
  bool sketch_on_hi = true;       // option "sketch_on_hi": sketch on its own stream while the SYRK runs
  // option "stream_priorities": the sketch stream and the Cholesky chain's
  // stream run at the highest stream priority, so their CTAs are placed
  // ahead of the overlapped Gram SYRK's.  (Rounds 1-2 rejected priorities:
  // the wrong results they exposed were the TMA GEMM's stage-release race,
  // fixed in gemm_f64.cu -- DESIGN.md, concurrency finding.)
  bool stream_priorities = true;  // (C2: 18.5 -> 17.9 ms; exact in every stress run)
  // option "gram_overlap": Gram SYRK on a side stream, overlapping the sketch
  // and the precond build; bit-identical to the single-stream path
  // (tools/race_stress.py, concurrency finding).
  bool gram_overlap = true;
  int gram_after_sketch = 0;  // option "gram_after_sketch": start that SYRK after the sketch (1) or after the linear term too (2)
  int64_t upload_chunk_bytes = 32 << 20;  // option "upload_chunk_bytes": column chunk of RP_HOST_STREAM uploads
  std::vector<double> prof_seconds, prof_flops, prof_bytes;  // per-GEMM profile of the last profiled path
  int64_t csr_panel_rows = 65536;    // option "csr_panel_rows": row panel of the sparse Gram passes
  int64_t csr_one_panel_bytes = 48 << 20;  // option "csr_one_panel_bytes": M W up to this size runs as one panel
  int64_t csr_chunk = 128;           // option "csr_chunk": right-hand columns per sparse Gram sweep (<= 128)
  // option "feature_shard": with several ranks, the Woodbury preconditioner
  // (m < d) is sharded over the d features (all-reduce of SA in,
  // all-gather of the output rows) and its shifted m x m factors over the
  // intervals (all-gather of the inverses); 0 = every rank applies it whole
  bool feature_shard = true;
  bool csr_l2_persist = false;  // option "csr_l2_persist": sparse Gram running sums as an L2-persisting window
  int csr_blocks_per_sm = 0;  // option "csr_blocks_per_sm": cap of the sparse passes' 256-thread blocks per SM (0 = none)
  std::string err;
};

struct rp_precond {
  int device = 0;
  int64_t m = 0, d = 0;
  bool woodbury = false;
  double lambda0 = 0;
  std::shared_ptr<rpb::DBuf<double>> sa;    // m x d
  std::shared_ptr<rpb::DBuf<double>> gram;  // d x d or m x m
  std::shared_ptr<rpb::DBuf<double>> inv;  // P (d x d) or (l0 I + SA SA^T)^{-1} (m x m)
};

namespace rpb {

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    RP_CUDA(cudaGetDevice(&prev));
    if (prev != dev) RP_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// Order the context's stream after a pending chunked upload (every generic
// reader of the operator goes through op_primal / op_dual).
void wait_upload(rp_ctx* ctx) {
  Upload& up = ctx->op.up;
  if (up.ev.empty()) return;
  up.enqueue(up.chunks());
  RP_CUDA(cudaStreamWaitEvent(ctx->stream, up.ev.back(), 0));
}
OpView op_primal(rp_ctx* ctx) {
  wait_upload(ctx);
  return ctx->op.primal();
}
OpView op_dual(rp_ctx* ctx) {
  wait_upload(ctx);
  return ctx->op.dual();
}

// True when the context's collectives do something (NCCL or host callbacks).
bool has_comm(const rp_ctx* ctx) { return ctx->comm != nullptr || ctx->host_allreduce != nullptr; }

double* host_stage(rp_ctx* ctx, size_t count) {
  if (ctx->host_stage_count < count) {
    if (ctx->host_stage) RP_CUDA(cudaFreeHost(ctx->host_stage));
    ctx->host_stage = nullptr;
    ctx->host_stage_count = 0;
    RP_CUDA(cudaMallocHost(&ctx->host_stage, count * sizeof(double)));
    ctx->host_stage_count = count;
  }
  return ctx->host_stage;
}

// Sum over ranks of buf[0..count), in place, stream-ordered on `st` (default:
// the context's stream).
void allreduce(rp_ctx* ctx, double* buf, int64_t count, cudaStream_t st = nullptr) {
  if (count <= 0) return;
  cudaStream_t s = st ? st : ctx->stream;
  if (ctx->host_allreduce) {
    double* h = host_stage(ctx, static_cast<size_t>(count));
    RP_CUDA(cudaMemcpyAsync(h, buf, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
    RP_CUDA(cudaStreamSynchronize(s));
    if (ctx->host_allreduce(ctx->host_user, h, count) != 0) throw NcclFailure("host allreduce callback failed");
    RP_CUDA(cudaMemcpyAsync(buf, h, sizeof(double) * count, cudaMemcpyHostToDevice, s));
    RP_CUDA(cudaStreamSynchronize(s));
    return;
  }
  if (!ctx->comm) return;
  nccl_check(nccl().AllReduce(buf, buf, static_cast<size_t>(count), ncclFloat64, ncclSum, ctx->comm, s),
             "ncclAllReduce");
}

// recv[r * count ...] = rank r's send[0..count) (recv holds world * count).
void allgather(rp_ctx* ctx, const double* send, int64_t count, double* recv, cudaStream_t st = nullptr) {
  cudaStream_t s = st ? st : ctx->stream;
  if (count <= 0) return;
  if (ctx->world == 1 || (!ctx->comm && !ctx->host_allgather)) {
    require(ctx->world == 1, "allgather: no communicator");
    if (recv != send)
      RP_CUDA(cudaMemcpyAsync(recv, send, sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
    return;
  }
  if (ctx->host_allgather) {
    const size_t total = static_cast<size_t>(count) * static_cast<size_t>(ctx->world + 1);
    double* h = host_stage(ctx, total);
    double* hr = h + count;
    RP_CUDA(cudaMemcpyAsync(h, send, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
    RP_CUDA(cudaStreamSynchronize(s));
    if (ctx->host_allgather(ctx->host_user, h, count, hr) != 0) throw NcclFailure("host allgather callback failed");
    RP_CUDA(cudaMemcpyAsync(recv, hr, sizeof(double) * count * ctx->world, cudaMemcpyHostToDevice, s));
    RP_CUDA(cudaStreamSynchronize(s));
    return;
  }
  nccl_check(nccl().AllGather(send, recv, static_cast<size_t>(count), ncclFloat64, ctx->comm, s), "ncclAllGather");
}

// ---- operator products -------------------------------------------------------

// y (n_loc x cols) = M_local x (D x cols)
void op_apply(rp_ctx* ctx, const OpView& op, const double* x, int64_t cols, double* y) {
  cudaStream_t s = ctx->stream;
  if (!op.sparse) {
    GemmArgs g;
    g.opa = op.op_m();
    g.m = op.n_loc;
    g.n = cols;
    g.k = op.d;
    g.a = op.a;
    g.lda = op.ld;
    g.b = x;
    g.ldb = op.d;
    g.c = y;
    g.ldc = op.n_loc;
    g.col_stable = true;
    dgemm(g, s);
  } else {
    DBuf<double> xr(static_cast<size_t>(op.d * cols), s), yr(static_cast<size_t>(op.n_loc * cols), s);
    transpose(x, op.d, cols, op.d, xr.get(), cols, s);
    spmm_csr_rm(op.csr_off, op.csr_col, op.csr_val, op.n_loc, cols, xr.get(), yr.get(), s);
    transpose(yr.get(), cols, op.n_loc, cols, y, op.n_loc, s);
  }
}

// x (D x cols) = M_local^T y (n_loc x cols), summed over ranks
void op_apply_t(rp_ctx* ctx, const OpView& op, const double* y, int64_t cols, double* x, bool reduce = true) {
  cudaStream_t s = ctx->stream;
  if (!op.sparse && !op.trans && cols <= kNarrowMax) {
    // one HBM pass over the operator (gram_pass.cu)
    atv_narrow(op.a, op.ld, op.n_loc, op.d, y, cols, x, s);
  } else if (!op.sparse) {
    GemmArgs g;
    g.opa = op.op_mt();
    g.m = op.d;
    g.n = cols;
    g.k = op.n_loc;
    g.a = op.a;
    g.lda = op.ld;
    g.b = y;
    g.ldb = op.n_loc;
    g.c = x;
    g.ldc = op.d;
    g.col_stable = true;
    dgemm(g, s);
  } else {
    DBuf<double> yr(static_cast<size_t>(op.n_loc * cols), s), xr(static_cast<size_t>(op.d * cols), s);
    transpose(y, op.n_loc, cols, op.n_loc, yr.get(), cols, s);
    spmm_csr_rm(op.csc_off, op.csc_row, op.csc_val, op.d, cols, yr.get(), xr.get(), s);
    transpose(xr.get(), cols, op.d, cols, x, op.d, s);
  }
  if (reduce) allreduce(ctx, x, op.d * cols);
}

struct GramOp {
  rp_ctx* ctx = nullptr;
  OpView op;
  bool matrix = false;
  // The fused single-pass kernel serves narrow standalone products
  // (rp_gram_apply); the recursion keeps one code path for every width so a
  // column's bits do not depend on how many problems are batched with it.
  bool allow_fused = false;
  // Column-stable products (a column's bits independent of the batch width,
  // the reference's matrix-vs-vector contract): on for the basis API, optional
  // for the path (option "stable_columns"), where the split-K factor may then
  // follow the problem's width.
  bool col_stable = true;
  DBuf<double> G;  // D x D when matrix
  DBuf<double> tmp;

  // Y (D x cols) = M^T (M W)  (matrix.cpp:168-172) or G W.  With `out`
  // the split-K reduction of G W may be left to the consumer.
  void apply(const double* W, int64_t cols, double* Y, Partials* out = nullptr,
             const RecursionEpilogue* epi = nullptr) {
    cudaStream_t s = ctx->stream;
    if (cols <= 0) return;
    if (out) *out = Partials{Y, 1, op.d, 0, 0};
    require(!epi || matrix, "gram: fused epilogue needs the Gram matrix");
    if (matrix) {
      GemmArgs g;
      g.m = op.d;
      g.n = cols;
      g.k = op.d;
      g.a = G.get();
      g.lda = op.d;
      g.b = W;
      g.ldb = op.d;
      g.c = Y;
      g.ldc = op.d;
      g.col_stable = col_stable;
      g.partials = out;
      if (epi && dgemm_split(g) > 1) {
        // split-K product: the partials stay deferred and the recursion's
        // standalone argument kernel consumes them
        require(out != nullptr && Y != nullptr, "gram: split product needs an output buffer");
        dgemm(g, s);
        BasisDims bd{epi->dim, epi->L, epi->K, epi->kmax};
        build_args(bd, epi->g, *out, epi->gen, epi->tau, epi->args, s);
        return;
      }
      g.epilogue = epi;
      dgemm(g, s);
      return;
    }
    if (allow_fused && !op.sparse && !op.trans && cols <= 8 && gram_fused(op.a, op.ld, op.n_loc, op.d, W, cols, Y, s)) {
      allreduce(ctx, Y, op.d * cols);  // fused single pass over the operator
      return;
    }
    if (op.sparse) {
      // L2-blocked two passes per row panel (sparse_gram.cu): bit-identical to
      // apply followed by apply_transpose, without the n x cols intermediate
      // (a narrow product whose whole M W fits in L2 runs as one panel on the
      // operator's plain CSC: same bits, no panel structure needed)
      const bool one_panel =
          static_cast<double>(op.n_loc) * static_cast<double>(cols) * 8.0 <= static_cast<double>(ctx->csr_one_panel_bytes);
      const PanelView pv = one_panel ? single_panel(op.n_loc, op.d, op.csc_off, op.csc_row, op.csc_val)
                                     : view_of(panel_csc(ctx, op));
      sparse_gram(op.csr_off, op.csr_col, op.csr_val, pv, W, op.d, cols, Y, op.d, ctx->csr_chunk, s,
                  ctx->csr_l2_persist, ctx->csr_blocks_per_sm);
      allreduce(ctx, Y, op.d * cols);
      return;
    }
    const size_t need = static_cast<size_t>(op.n_loc * cols);
    if (tmp.size() < need) tmp.alloc(need, s);
    op_apply(ctx, op, W, cols, tmp.get());
    op_apply_t(ctx, op, tmp.get(), cols, Y, true);
  }

  static const PanelCsc& panel_csc(rp_ctx* ctx, const OpView& op) {
    OperatorStore& st = ctx->op;
    PanelCsc& pc = op.csr_off == st.csr_off.get() ? st.panels_primal : st.panels_dual;
    if (!pc.matches(op.n_loc, op.d, op.nnz, ctx->csr_panel_rows))
      build_panel_csc(op.csr_off, op.csr_col, op.csr_val, op.n_loc, op.d, op.nnz, ctx->csr_panel_rows, pc,
                      ctx->stream);
    return pc;
  }

  // Streamed build (RP_HOST_STREAM uploads): block rows of the lower triangle
  // as the operator's column chunks land, then mirror and all-reduce.
  void begin_matrix() {
    require(!op.sparse && !op.trans, "gram matrix rows need a dense primal operator");
    G.alloc(static_cast<size_t>(op.d * op.d), ctx->stream);
  }
  void matrix_rows(int64_t c0, int64_t c1) {  // G[c0:c1, 0:c1] = M[:, c0:c1]^T M[:, 0:c1]
    GemmArgs g;
    g.opa = Op::T;
    g.m = c1 - c0;
    g.n = c1;
    g.k = op.n_loc;
    g.a = op.a + c0 * op.ld;
    g.lda = op.ld;
    g.b = op.a;
    g.ldb = op.ld;
    g.c = G.get() + c0;
    g.ldc = op.d;
    dgemm(g, ctx->stream);
  }
  void end_matrix() {
    mirror_lower(G.get(), op.d, op.d, ctx->stream);
    allreduce(ctx, G.get(), op.d * op.d);
    matrix = true;
  }

  void build_matrix(cudaStream_t st = nullptr) {
    cudaStream_t s = st ? st : ctx->stream;
    require(!op.sparse, "gram matrix mode needs a dense operator");
    G.alloc(static_cast<size_t>(op.d * op.d), s);
    GemmArgs g;  // G = M^T M (lower + mirror)
    g.opa = op.op_mt();
    g.opb = op.op_m();
    g.m = op.d;
    g.n = op.d;
    g.k = op.n_loc;
    g.a = op.a;
    g.lda = op.ld;
    g.b = op.a;
    g.ldb = op.ld;
    g.c = G.get();
    g.ldc = op.d;
    g.lower_only = true;
    g.mirror = true;
    // (tuning hook for the overlapped build; forcing 128 x 128 tiles, which
    // leave shared memory for the Cholesky chain's kernels on every SM,
    // measured slower than the auto choice: 19.16 vs 18.96 ms on C2)
    if (st && ctx->gram_overlap_tile >= 0) g.force_tile = ctx->gram_overlap_tile;
    if (st && !ctx->gram_overlap_tma) g.no_tma = true;
    if (st && ctx->gram_overlap_split > 0) g.split_k = ctx->gram_overlap_split;
    if (st && ctx->gram_overlap_occ > 0) g.max_ctas_per_sm = ctx->gram_overlap_occ;
    dgemm(g, s);
    allreduce(ctx, G.get(), op.d * op.d, s);
    matrix = true;
  }
};

// ---- preconditioner ------------------------------------------------------------

// P_l for a batch of shifts.  m >= d: P_l = (SA^T SA + l0 I)^{-1} explicitly;
// m < d: Woodbury with W_l = (l0 I + SA SA^T)^{-1}: P v = (v - SA^T W_l SA v) / l0.
// Same operator as preconditioner.cpp:12-65 (projection or shift form).
struct PrecondBatch {
  int64_t m = 0, d = 0, L = 0;
  bool woodbury = false;
  bool col_stable = true;  // (see GramOp::col_stable)
  // feature sharding (Woodbury, several ranks): this rank applies SA[:, f0:f1],
  // rows split in blocks of `blk` (the last rank's block may be short)
  bool fshard = false;
  int64_t f0 = 0, f1 = 0, blk = 0;
  bool allow_fshard = true;  // false when the ranks build different interval sets (collectives would not match)
  const double* sa = nullptr;  // m x d
  std::vector<double> lambda0;
  DBuf<double> d_lambda0;
  DBuf<double> inv_owned;
  const double* inv = nullptr;  // L x (n x n), n = d or m
  int64_t n() const { return woodbury ? m : d; }

  void build(rp_ctx* ctx, const double* sa_, const double* gram /* n x n, may be null */, int64_t m_, int64_t d_,
             const std::vector<double>& l0) {
    cudaStream_t s = ctx->stream;
    m = m_;
    d = d_;
    sa = sa_;
    woodbury = m < d;
    L = static_cast<int64_t>(l0.size());
    lambda0 = l0;
    for (double v : l0) require(v > 0.0, "preconditioner: shift must be positive");
    const int64_t nn = n();
    fshard = woodbury && allow_fshard && ctx->feature_shard && ctx->world > 1 && has_comm(ctx);
    if (fshard) {
      blk = ceil_div(d, ctx->world);
      f0 = std::min<int64_t>(d, blk * ctx->rank);
      f1 = std::min<int64_t>(d, f0 + blk);
    }
    DBuf<double> gbuf;
    if (!gram && fshard) {
      // SA SA^T = sum over ranks of SA[:, f0:f1] SA[:, f0:f1]^T
      gbuf.alloc(static_cast<size_t>(nn * nn), s);
      if (f1 > f0) {
        GemmArgs g;
        g.opa = Op::N;
        g.opb = Op::T;
        g.m = nn;
        g.n = nn;
        g.k = f1 - f0;
        g.a = sa + f0 * m;
        g.lda = m;
        g.b = sa + f0 * m;
        g.ldb = m;
        g.c = gbuf.get();
        g.ldc = nn;
        g.lower_only = true;
        g.mirror = true;
        dgemm(g, s);
      } else {
        fill(gbuf.get(), nn * nn, 0.0, s);
      }
      allreduce(ctx, gbuf.get(), nn * nn);
      gram = gbuf.get();
    }
    if (!gram) {
      gbuf.alloc(static_cast<size_t>(nn * nn), s);
      GemmArgs g;
      g.opa = woodbury ? Op::N : Op::T;
      g.opb = woodbury ? Op::T : Op::N;
      g.m = nn;
      g.n = nn;
      g.k = woodbury ? d : m;
      g.a = sa;
      g.lda = m;
      g.b = sa;
      g.ldb = m;
      g.c = gbuf.get();
      g.ldc = nn;
      g.lower_only = true;
      g.mirror = true;
      dgemm(g, s);
      gram = gbuf.get();
    }
    d_lambda0.alloc(static_cast<size_t>(L), s);
    RP_CUDA(cudaMemcpyAsync(d_lambda0.get(), lambda0.data(), sizeof(double) * L, cudaMemcpyHostToDevice, s));
    if (fshard && L > 1) {
      // the shifted m x m factors split over the ranks by interval, then
      // all-gathered: rank r inverts shifts [r*lb, min(L, (r+1)*lb))
      const int64_t lb = ceil_div(L, ctx->world);
      const int64_t s0 = std::min<int64_t>(L, lb * ctx->rank), s1 = std::min<int64_t>(L, s0 + lb);
      DBuf<double> mine(static_cast<size_t>(lb * nn * nn), s);
      if (s1 > s0) {
        DBuf<double> h(static_cast<size_t>((s1 - s0) * nn * nn), s);
        shifted_copies(gram, nn, d_lambda0.get() + s0, s1 - s0, h.get(), s);
        spd_inverse_batched(h.get(), nn, nn, nn * nn, s1 - s0, mine.get(), nn, nn * nn, s, ctx->stream_priorities);
      }
      inv_owned.alloc(static_cast<size_t>(ctx->world * lb * nn * nn), s);
      allgather(ctx, mine.get(), lb * nn * nn, inv_owned.get());
      inv = inv_owned.get();  // (rank blocks are consecutive shifts: the first L blocks are shifts 0..L-1)
      return;
    }
    DBuf<double> h(static_cast<size_t>(L * nn * nn), s);
    shifted_copies(gram, nn, d_lambda0.get(), L, h.get(), s);
    inv_owned.alloc(static_cast<size_t>(L * nn * nn), s);
    inv = inv_owned.get();
    spd_inverse_batched(h.get(), nn, nn, nn * nn, L, inv_owned.get(), nn, nn * nn, s, ctx->stream_priorities);
  }

  // A view of shifts [l0, l1) (no copy of the factors).
  PrecondBatch slice(rp_ctx* ctx, int64_t l0, int64_t l1) const {
    PrecondBatch v;
    v.m = m;
    v.d = d;
    v.L = l1 - l0;
    v.woodbury = woodbury;
    v.col_stable = col_stable;
    v.sa = sa;
    v.fshard = fshard;
    v.f0 = f0;
    v.f1 = f1;
    v.blk = blk;
    v.lambda0.assign(lambda0.begin() + l0, lambda0.begin() + l1);
    v.d_lambda0.alloc(static_cast<size_t>(v.L), ctx->stream);
    RP_CUDA(cudaMemcpyAsync(v.d_lambda0.get(), v.lambda0.data(), sizeof(double) * v.L, cudaMemcpyHostToDevice,
                            ctx->stream));
    RP_CUDA(cudaStreamSynchronize(ctx->stream));
    v.inv = inv + l0 * n() * n();
    return v;
  }
  PrecondBatch single(rp_ctx* ctx, int64_t l) const { return slice(ctx, l, l + 1); }

  // out_l (d x cols) = P_l in_l for l < L; in/out strided by `sin`/`sout`
  // (sin = 0 broadcasts one input to every interval).
  void apply(rp_ctx* ctx, const double* in, int64_t sin, int64_t cols, double* out, int64_t sout,
             Partials* part = nullptr, const RecursionEpilogue* epi = nullptr) const {
    cudaStream_t s = ctx->stream;
    if (cols <= 0) return;
    if (part) *part = Partials{out, 1, d, 0, sout};
    require(!epi || !woodbury, "preconditioner: fused epilogue needs the explicit inverse");
    if (!woodbury) {
      GemmArgs g;
      g.m = d;
      g.n = cols;
      g.k = d;
      g.a = inv;
      g.lda = d;
      g.stride_a = d * d;
      g.b = in;
      g.ldb = d;
      g.stride_b = sin;
      g.c = out;
      g.ldc = d;
      g.stride_c = sout;
      g.batch = L;
      g.col_stable = true;
      g.partials = part;
      if (epi && !ctx->fuse_update) {
        // split product + the standalone update kernel
        require(out != nullptr, "preconditioner: split product needs an output buffer");
        Partials pa;
        g.partials = &pa;
        dgemm(g, s);
        BasisDims bd{epi->dim, epi->L, epi->K, epi->kmax};
        update_gen(bd, epi->g, pa, epi->kb, epi->gen, epi->tilde, epi->flags, s);
        if (epi->g + 1 < epi->kmax) seed_next_args(bd, epi->g, epi->gen, epi->args, s);
        return;
      }
      if (epi) g.split_k = 1;  // (the L-way batch fills the GPU; a fused epilogue needs no split)
      g.epilogue = epi;
      dgemm(g, s);
      return;
    }
    // Woodbury: SA is shared by every interval, so the two SA products run as
    // single GEMMs over all L * cols columns (SA streamed once per call); only
    // the m x m middle factor is batched per interval.  A broadcast input is
    // multiplied by SA once.
    const bool bcast = sin == 0;
    if (fshard) {
      apply_feature_sharded(ctx, in, sin, cols, out, sout);
      return;
    }
    const double* src = in;
    DBuf<double> inb;
    if (!bcast && sin != d * cols) {
      inb.alloc(static_cast<size_t>(L * d * cols), s);
      for (int64_t l = 0; l < L; ++l) copy_cols(in + l * sin, d, cols, d, inb.get() + l * d * cols, d, s);
      src = inb.get();
    }
    const int64_t n1 = bcast ? cols : L * cols;
    DBuf<double> t1(static_cast<size_t>(m * n1), s), t2(static_cast<size_t>(L * m * cols), s);
    DBuf<double> t3(static_cast<size_t>(L * d * cols), s);
    GemmArgs g1;  // t1 = SA [in_0 .. in_{L-1}]
    g1.m = m;
    g1.n = n1;
    g1.k = d;
    g1.a = sa;
    g1.lda = m;
    g1.b = src;
    g1.ldb = d;
    g1.c = t1.get();
    g1.ldc = m;
    g1.col_stable = true;
    dgemm(g1, s);
    GemmArgs g2;  // t2_l = W_l t1_l
    g2.m = m;
    g2.n = cols;
    g2.k = m;
    g2.a = inv;
    g2.lda = m;
    g2.stride_a = m * m;
    g2.b = t1.get();
    g2.ldb = m;
    g2.stride_b = bcast ? 0 : m * cols;
    g2.c = t2.get();
    g2.ldc = m;
    g2.stride_c = m * cols;
    g2.batch = L;
    g2.col_stable = true;
    dgemm(g2, s);
    GemmArgs g3;  // t3 = SA^T [t2_0 .. t2_{L-1}]
    g3.opa = Op::T;
    g3.m = d;
    g3.n = L * cols;
    g3.k = m;
    g3.a = sa;
    g3.lda = m;
    g3.b = t2.get();
    g3.ldb = m;
    g3.c = t3.get();
    g3.ldc = d;
    g3.col_stable = true;
    dgemm(g3, s);
    // out_l = (in_l - t3_l) / l0_l
    woodbury_tail(d, cols, L, sin, in, d * cols, t3.get(), d_lambda0.get(), sout, out, s);
  }

  // Woodbury apply with the features split over the ranks:
  //   t1   = sum_p SA[:, f_p] in[f_p, :]          local GEMM + all-reduce (m x L*cols)
  //   t2_l = W_l t1_l                             replicated m x m batch
  //   t3_p = SA[:, f_p]^T t2                      local GEMM (|f_p| x L*cols)
  //   out[f_p, :] = (in[f_p, :] - t3_p) / l0_l    local, then all-gather of the row blocks
  // Per call: one all-reduce of 8*m*L*cols bytes and one all-gather of
  // 8*d*L*cols bytes; the 4*m*d*L*cols SA flops are split over the ranks.
  void apply_feature_sharded(rp_ctx* ctx, const double* in, int64_t sin, int64_t cols, double* out,
                             int64_t sout) const {
    cudaStream_t s = ctx->stream;
    const bool bcast = sin == 0;
    const int64_t dl = f1 - f0;
    const double* src = in;
    DBuf<double> inb;
    if (!bcast && sin != d * cols) {
      inb.alloc(static_cast<size_t>(L * d * cols), s);
      for (int64_t l = 0; l < L; ++l) copy_cols(in + l * sin, d, cols, d, inb.get() + l * d * cols, d, s);
      src = inb.get();
    }
    const int64_t n1 = bcast ? cols : L * cols;
    DBuf<double> t1(static_cast<size_t>(m * n1), s), t2(static_cast<size_t>(L * m * cols), s);
    if (dl > 0) {
      GemmArgs g1;  // t1 = SA[:, f0:f1] in[f0:f1, :]
      g1.m = m;
      g1.n = n1;
      g1.k = dl;
      g1.a = sa + f0 * m;
      g1.lda = m;
      g1.b = src + f0;
      g1.ldb = d;
      g1.c = t1.get();
      g1.ldc = m;
      g1.col_stable = true;
      dgemm(g1, s);
    } else {
      fill(t1.get(), m * n1, 0.0, s);
    }
    allreduce(ctx, t1.get(), m * n1);
    GemmArgs g2;  // t2_l = W_l t1_l
    g2.m = m;
    g2.n = cols;
    g2.k = m;
    g2.a = inv;
    g2.lda = m;
    g2.stride_a = m * m;
    g2.b = t1.get();
    g2.ldb = m;
    g2.stride_b = bcast ? 0 : m * cols;
    g2.c = t2.get();
    g2.ldc = m;
    g2.stride_c = m * cols;
    g2.batch = L;
    g2.col_stable = true;
    dgemm(g2, s);
    DBuf<double> t3(static_cast<size_t>(std::max<int64_t>(dl, 1) * L * cols), s);
    DBuf<double> pack(static_cast<size_t>(blk * L * cols), s);
    if (dl > 0) {
      GemmArgs g3;  // t3 = SA[:, f0:f1]^T [t2_0 .. t2_{L-1}]
      g3.opa = Op::T;
      g3.m = dl;
      g3.n = L * cols;
      g3.k = m;
      g3.a = sa + f0 * m;
      g3.lda = m;
      g3.b = t2.get();
      g3.ldb = m;
      g3.c = t3.get();
      g3.ldc = dl;
      g3.col_stable = true;
      dgemm(g3, s);
      woodbury_tail_rows(f0, dl, cols, L, in, d, sin, t3.get(), d_lambda0.get(), pack.get(), blk, s);
    }
    DBuf<double> recv(static_cast<size_t>(ctx->world * blk * L * cols), s);
    allgather(ctx, pack.get(), blk * L * cols, recv.get());
    gather_row_blocks(recv.get(), blk, d, cols, L, out, sout, s);
  }
};

// ---- basis recursion (path_solver.cpp:27-53), batched over intervals x RHS ----

struct BasisRun {
  BasisDims dims;
  DBuf<double> gen, tilde;
  std::vector<double> tau;
  std::vector<int> k;
  DBuf<double> d_tau;
  DBuf<int> d_k;
  std::vector<int> diverged;  // per interval
};

// The recursion as a resumable object: begin() (gen_0 = P c), step(g) for
// g = 1 .. kmax-1, finish() (divergence flags to the host, asynchronously).
// Every launch goes to `stream`.
struct BasisStepper {
  rp_ctx* ctx;
  GramOp& gram;
  const PrecondBatch& P;
  BasisRun& out;
  cudaStream_t stream;
  int64_t K = 0, L = 0, dim = 0, NB = 0, stride_im = 0;
  int kmax = 1;
  BasisDims dims{};
  DBuf<int> flags;
  DBuf<double> args, y, applied;
  RecursionEpilogue e{};
  bool fused = false;

  // (the library's building blocks launch on ctx->stream: point it at ours)
  struct Use {
    rp_ctx* c;
    cudaStream_t prev;
    Use(rp_ctx* c_, cudaStream_t s) : c(c_), prev(c_->stream) { c->stream = s; }
    ~Use() { c->stream = prev; }
  };

  BasisStepper(rp_ctx* ctx_, GramOp& gram_, const PrecondBatch& P_, BasisRun& out_, cudaStream_t st)
      : ctx(ctx_), gram(gram_), P(P_), out(out_), stream(st) {}

  void begin(const double* c, int64_t K_, const std::vector<double>& tau, const std::vector<int>& ks) {
    Use u(ctx, stream);
    cudaStream_t s = stream;
    K = K_;
    L = P.L;
    dim = P.d;
    for (int kv : ks) {
      require(kv >= 1, "ihs_basis: k must be >= 1");
      kmax = std::max(kmax, kv);
    }
    for (double t : tau) require(t > 0.0, "ihs_basis: tau must be positive");
    dims = BasisDims{dim, L, K, kmax};
    out.dims = dims;
    out.tau = tau;
    out.k = ks;
    NB = dims.nb();
    out.gen.alloc(static_cast<size_t>(dim * kmax * NB), s);
    out.tilde.alloc(static_cast<size_t>(dim * kmax * NB), s);
    out.d_tau.alloc(static_cast<size_t>(L), s);
    out.d_k.alloc(static_cast<size_t>(L), s);
    RP_CUDA(cudaMemcpyAsync(out.d_tau.get(), tau.data(), sizeof(double) * L, cudaMemcpyHostToDevice, s));
    RP_CUDA(cudaMemcpyAsync(out.d_k.get(), ks.data(), sizeof(int) * L, cudaMemcpyHostToDevice, s));
    flags.alloc(static_cast<size_t>(L), s);
    RP_CUDA(cudaMemsetAsync(flags.get(), 0, sizeof(int) * L, s));
    // gen_0 = P c (every interval, every RHS), tilde_0 = gen_0.
    P.apply(ctx, c, 0, K, out.gen.get(), K * dim);
    fill(out.tilde.get(), dim * kmax * NB, 0.0, s);
    copy_cols(out.gen.get(), dim, NB, dim, out.tilde.get(), dim, s);
    if (kmax > 1) {
      stride_im = dim * kmax * K;
      args.alloc(static_cast<size_t>(L * stride_im), s);
      y.alloc(static_cast<size_t>(dim * (kmax - 1) * NB), s);  // (used when the Gram product is split)
      applied.alloc(static_cast<size_t>(L * stride_im), s);
      fused = gram.matrix && !P.woodbury;
      if (fused) {
        // Two kernels per generation: the Gram GEMM builds the preconditioner
        // arguments in its epilogue, the preconditioner GEMM updates gen/tilde
        // (and seeds the next generation's last argument column) in its own.
        seed_args(dims, out.gen.get(), args.get(), s);
        e.dim = dim;
        e.L = L;
        e.K = K;
        e.kmax = kmax;
        e.tau = out.d_tau.get();
        e.kb = out.d_k.get();
        e.gen = out.gen.get();
        e.tilde = out.tilde.get();
        e.args = args.get();
        e.flags = flags.get();
      }
    }
  }

  void step(int64_t g) {
    if (g >= kmax) return;
    Use u(ctx, stream);
    cudaStream_t s = stream;
    nvtxRangePushA("generation");
    if (fused) {
      Partials py;
      e.g = g;
      e.kind = RecursionEpilogue::kArgs;
      gram.apply(out.gen.get(), g * NB, y.get(), &py, &e);
      e.kind = RecursionEpilogue::kUpdate;
      P.apply(ctx, args.get(), stride_im, (g + 1) * K, applied.get(), stride_im, nullptr, &e);
    } else {
      Partials py, pa;
      gram.apply(out.gen.get(), g * NB, y.get(), &py);
      build_args(dims, g, py, out.gen.get(), out.d_tau.get(), args.get(), s);
      P.apply(ctx, args.get(), stride_im, (g + 1) * K, applied.get(), stride_im, &pa);
      update_gen(dims, g, pa, out.d_k.get(), out.gen.get(), out.tilde.get(), flags.get(), s);
    }
    nvtxRangePop();
  }

  void finish() {
    out.diverged.assign(static_cast<size_t>(L), 0);
    RP_CUDA(cudaMemcpyAsync(out.diverged.data(), flags.get(), sizeof(int) * L, cudaMemcpyDeviceToHost, stream));
  }
};

void run_basis(rp_ctx* ctx, GramOp& gram, const PrecondBatch& P, const double* c, int64_t K,
               const std::vector<double>& tau, const std::vector<int>& ks, BasisRun& out) {
  BasisStepper b(ctx, gram, P, out, ctx->stream);
  b.begin(c, K, tau, ks);
  for (int64_t g = 1; g < b.kmax; ++g) b.step(g);
  b.finish();
  RP_CUDA(cudaStreamSynchronize(ctx->stream));
}

// ---- helpers for host/device buffers -------------------------------------------

struct InBuf {
  const double* ptr = nullptr;
  DBuf<double> owned;
  InBuf(const double* p, size_t count, int where, cudaStream_t s, bool zero_copy = false) {
    if (where == RP_DEVICE || count == 0) {
      ptr = p;
      return;
    }
    owned.alloc(count, s);
    ptr = owned.get();
    if (zero_copy) {
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer) {
        copy_mapped(static_cast<const double*>(at.devicePointer), static_cast<int64_t>(count), owned.get(), s);
        return;
      }
      cudaGetLastError();
    }
    RP_CUDA(cudaMemcpyAsync(owned.get(), p, count * sizeof(double), cudaMemcpyHostToDevice, s));
  }
};

struct OutBuf {
  double* dev = nullptr;
  double* host = nullptr;
  size_t count = 0;
  DBuf<double> owned;
  cudaStream_t s;
  OutBuf(double* p, size_t n, int where, cudaStream_t st) : count(n), s(st) {
    if (where == RP_DEVICE) {
      dev = p;
    } else {
      host = p;
      owned.alloc(n ? n : 1, st);
      dev = owned.get();
    }
  }
  void finish() {
    if (host && count) RP_CUDA(cudaMemcpyAsync(host, dev, count * sizeof(double), cudaMemcpyDeviceToHost, s));
    RP_CUDA(cudaStreamSynchronize(s));
  }
};

Rho to_rho(const rp_rho_bounds* r) {
  require(r != nullptr, "rho bounds: null");
  Rho o;
  o.rho1 = r->rho1;
  o.rho2 = r->rho2;
  o.provenance = r->provenance;
  return o;
}

SketchSpecC to_spec(const rp_sketch_spec* s) {
  require(s != nullptr, "sketch spec: null");
  SketchSpecC o;
  o.kind = s->kind;
  o.m = s->m;
  o.n = s->n;
  o.s = s->s;
  o.seed = s->seed;
  return o;
}

PathCfg to_cfg(const rp_path_config* c) {
  require(c != nullptr, "path config: null");
  PathCfg o;
  o.lambda_min = c->lambda_min;
  o.lambda_max = c->lambda_max;
  require(c->num_lambdas >= 0, "path config: negative grid size");
  if (c->num_lambdas > 0) {
    require(c->lambdas != nullptr, "path config: null grid");
    o.lambdas.assign(c->lambdas, c->lambdas + c->num_lambdas);
  }
  o.epsilon = c->epsilon;
  if (c->num_intervals > 0) o.num_intervals = c->num_intervals;
  return o;
}

// NVTX ranges (header-only NVTX 3: free unless a profiler is attached).  The
// reference's timing sites (path_solver.cpp:12-16, 153-189) become ranges a
// profiler timeline shows: one per path, one per phase, one per generation.
struct NvtxPhases {
  bool open = false;
  explicit NvtxPhases(const char* whole) { nvtxRangePushA(whole); }
  void next(const char* name) {
    if (open) nvtxRangePop();
    nvtxRangePushA(name);
    open = true;
  }
  ~NvtxPhases() {
    if (open) nvtxRangePop();
    nvtxRangePop();
  }
};

// Composition of T grid points (sorted by interval: itv ascending) into
// x[:, t*K + r].  Default: one FP64 DMMA GEMM batched over (interval, right-hand
// side) -- x(lambda) = U_l (dim x kmax) times the interval's kmax x tmax block of
// coefficients tau_l (tau_l lambda)^j, padded to the largest interval and
// gathered (north_star 6).  Option "compose_gemm" = 0: the reference's Horner
// order, one thread per entry (compose_horner, path_solver.cpp:64-74).
void compose_points(rp_ctx* ctx, const BasisRun& R, const std::vector<int>& itv, const double* d_lam, const int* d_itv,
                    int64_t Tn, double* x) {
  cudaStream_t s = ctx->stream;
  const BasisDims& d = R.dims;
  bool sorted = true;
  for (size_t i = 1; i < itv.size(); ++i) sorted = sorted && itv[i - 1] <= itv[i];
  if (!ctx->compose_gemm || !sorted || d.kmax < 2) {
    compose(d, R.tilde.get(), R.d_tau.get(), R.d_k.get(), d_lam, d_itv, Tn, x, s);
    return;
  }
  std::vector<int> off(static_cast<size_t>(d.L), 0), cnt(static_cast<size_t>(d.L), 0);
  for (int64_t t = 0; t < Tn; ++t) {
    if (cnt[itv[t]] == 0) off[itv[t]] = static_cast<int>(t);
    ++cnt[itv[t]];
  }
  int64_t tmax = 1;
  for (int c : cnt) tmax = std::max<int64_t>(tmax, c);
  tmax = (tmax + 7) & ~int64_t{7};  // (whole 8-column DMMA fragments; keeps the operand strides even)
  DBuf<int> d_off(static_cast<size_t>(d.L), s), d_cnt(static_cast<size_t>(d.L), s);
  RP_CUDA(cudaMemcpyAsync(d_off.get(), off.data(), sizeof(int) * d.L, cudaMemcpyHostToDevice, s));
  RP_CUDA(cudaMemcpyAsync(d_cnt.get(), cnt.data(), sizeof(int) * d.L, cudaMemcpyHostToDevice, s));
  DBuf<double> coef(static_cast<size_t>(d.L * tmax * d.kmax), s);
  DBuf<double> xpad(static_cast<size_t>(d.L * tmax * d.K * d.dim), s);
  compose_coeffs(d, R.d_tau.get(), R.d_k.get(), d_lam, d_off.get(), d_cnt.get(), tmax, coef.get(), s);
  GemmArgs g;  // batch = interval l, batch2 = right-hand side r
  g.m = d.dim;
  g.n = tmax;
  g.k = d.kmax;
  g.a = R.tilde.get();           // U_{l,r}: column j at ((j*NB + l*K + r) * dim)
  g.lda = d.nb() * d.dim;
  g.stride_a = d.K * d.dim;
  g.stride_a2 = d.dim;
  g.b = coef.get();              // kmax x tmax per interval, shared by the right-hand sides
  g.ldb = d.kmax;
  g.stride_b = d.kmax * tmax;
  g.stride_b2 = 0;
  g.c = xpad.get();              // column (l*tmax + c)*K + r
  g.ldc = d.K * d.dim;
  g.stride_c = tmax * d.K * d.dim;
  g.stride_c2 = d.dim;
  g.batch = d.L;
  g.batch2 = d.K;
  g.split_k = 1;
  dgemm(g, s);
  compose_gather(d, xpad.get(), d_off.get(), d_cnt.get(), tmax, x, s);
  RP_CUDA(cudaStreamSynchronize(s));  // (off / cnt are host vectors of this frame)
}

// ---- run_path (path_solver.cpp:147-190) ------------------------------------------

struct Events {
  std::vector<cudaEvent_t> ev;
  explicit Events(int n) : ev(static_cast<size_t>(n)) {
    for (auto& e : ev) RP_CUDA(cudaEventCreate(&e));
  }
  ~Events() {
    for (auto& e : ev) cudaEventDestroy(e);
  }
  double secs(int a, int b) const {
    float ms = 0.f;
    RP_CUDA(cudaEventElapsedTime(&ms, ev[a], ev[b]));
    return ms * 1e-3;
  }
};

void run_path(rp_ctx* ctx, bool dual, const double* b_in, int64_t K, const PathCfg& cfg, const SketchSpecC& spec,
              const Rho& rho, std::optional<double> sigma_d, double* x_out, int where, rp_timings* tm) {
  cudaStream_t s = ctx->stream;
  const int64_t launches0 = launch_counter().load();
  std::unique_ptr<GemmProfiler> prof;
  if (ctx->profile) {
    prof = std::make_unique<GemmProfiler>();
    set_gemm_profiler(prof.get());
  }
  struct ProfReset {
    ~ProfReset() { set_gemm_profiler(nullptr); }
  } prof_reset;
  const auto host_t0 = std::chrono::steady_clock::now();
  cfg.validate();
  rho_validate(rho);
  require(K >= 1, "path: empty right-hand side");
  // A dense primal operator still landing in chunks (RP_HOST_STREAM) is
  // consumed chunk by chunk below; every other case waits for the upload.
  // (a Gaussian sketch is streamed when its local S, m x n_loc doubles, can stay resident: it is drawn
  // once and applied to each column block as that lands)
  bool gauss_resident = false;
  if (spec.kind == kGaussian && !dual && ctx->op.set && !ctx->op.sparse && ctx->op.shard != 2 &&
      ctx->op.up.chunks() > 1 && ctx->op.up.next < ctx->op.up.chunks()) {  // (only when an upload is streaming)
    const double need = 8.0 * static_cast<double>(spec.m) * static_cast<double>(ctx->op.shard == 1 ? ctx->op.n_local : ctx->op.n);
    gauss_resident = need <= 0.45 * ctx->op.free_after_alloc;
  }
  const bool stream_in = !dual && ctx->op.set && !ctx->op.sparse && ctx->op.shard != 2 &&
                         ctx->op.up.chunks() > 1 && ctx->op.up.next < ctx->op.up.chunks() &&
                         (spec.kind != kGaussian || gauss_resident);
  const OpView op = stream_in ? ctx->op.primal() : (dual ? op_dual(ctx) : op_primal(ctx));
  // ihs_bin_path: spec.n == A.rows; dual_path: spec.n == A.cols (path_solver.cpp:294, 333-334)
  require(spec.n == op.n_global, dual ? "dual_path: spec.n must equal A.cols (the dual operator is A^T)"
                                      : "ihs_bin_path: spec.n must equal A.rows");
  const int64_t dim = op.d;
  const int64_t b_rows = dual ? op.d : op.n_loc;  // dual: b has A.rows = op.d entries per column
  // Host -> device copy of b (timed as copy).
  double copy_secs = 0.0;
  auto tc0 = std::chrono::steady_clock::now();
  // (while an upload streams, a pinned host b is read by a kernel through its
  // mapped address instead of queueing a copy behind the transfer)
  InBuf b(b_in, static_cast<size_t>(b_rows * K), where, s, stream_in);
  if (where == RP_HOST) RP_CUDA(cudaStreamSynchronize(s));
  copy_secs += std::chrono::duration<double>(std::chrono::steady_clock::now() - tc0).count();

  Events ev(8);
  RP_CUDA(cudaEventRecord(ev.ev[0], s));
  NvtxPhases nv(dual ? "ridgepath: dual_path" : "ridgepath: ihs_bin_path");
  nv.next("sketch + linear term (+ Gram matrix)");
  // 2) Plans (host, bit-identical to the reference).
  const auto plans = plan_intervals(cfg, rho, sigma_d);
  const int64_t L = static_cast<int64_t>(plans.size());
  // Gram operator: pass over M, or G = M^T M when cheaper.
  GramOp gram;
  gram.ctx = ctx;
  gram.op = op;
  int kmax = 2;
  for (const auto& p : plans) kmax = std::max(kmax, p.params.k);
  bool use_matrix = false;
  {
    const double cols_total = static_cast<double>(L * K) * (static_cast<double>(kmax) * (kmax - 1) / 2.0);
    const double nnz = op.sparse ? static_cast<double>(op.nnz) : static_cast<double>(op.n_loc) * op.d;
    const double pass = 4.0 * nnz * cols_total;
    const double matrix = static_cast<double>(op.n_loc) * op.d * op.d + 2.0 * op.d * op.d * cols_total;
    use_matrix = !op.sparse && matrix < pass && static_cast<double>(op.d) * op.d * 8.0 <= 16.0 * (1 << 30);
    if (ctx->gram_mode == 0) use_matrix = false;
    if (ctx->gram_mode == 1) {
      require(!op.sparse, "gram_mode=1 needs a dense operator");
      use_matrix = true;
    }
  }
  DBuf<double> sa(static_cast<size_t>(spec.m * dim), s);
  DBuf<double> cbuf(static_cast<size_t>(dim * K), s);
  cudaEvent_t gram_done = nullptr;  // side-stream Gram matrix (see below)
  if (stream_in) {
    // Chunked consumption of the upload: as column block [c0, c1) of A lands,
    // sketch its columns, form rows c0..c1 of c = A^T b and block row
    // G[c0:c1, 0:c1] of the Gram matrix (lower part; mirrored at the end).
    const Upload& up = ctx->op.up;
    // upload chunks consumed per step: one, or -- Gaussian sketch, whose block product streams all of S --
    // as many as make the block at least 128 columns wide
    const int64_t nchunks = static_cast<int64_t>(up.ev.size());
    const int64_t group = spec.kind == kGaussian ? std::max<int64_t>(1, ceil_div(128, std::max<int64_t>(up.chunk, 1))) : 1;
    DBuf<double> ctmp(static_cast<size_t>(std::min<int64_t>(up.chunk * group, dim) * K), s);
    if (use_matrix) gram.begin_matrix();
    Upload& upm = ctx->op.up;
    const bool planned = spec.kind == kCountSketch || spec.kind == kSjlt || spec.kind == kSrht || spec.kind == kGaussian;
    SketchPlan plan;  // draws / SRHT tables / Gaussian S once, applied per column block
    if (planned) {
      upm.enqueue(kUploadDepth * group);  // (the first blocks travel while the plan is drawn)
      sketch_plan(spec, op, plan, s);
    }
    for (int64_t j = 0; j < nchunks; j += group) {
      const int64_t j1 = std::min(nchunks, j + group);
      const int64_t c0 = j * up.chunk, cc = std::min(up.chunk * (j1 - j), dim - c0);
      upm.enqueue(j1 + kUploadDepth * group);
      RP_CUDA(cudaStreamWaitEvent(s, up.ev[static_cast<size_t>(j1 - 1)], 0));  // (copy-stream order: the block is whole)
      OpView sub = op;
      sub.a = op.a + c0 * op.ld;
      sub.d = cc;
      if (planned)
        sketch_apply_planned(plan, sub, sa.get() + c0 * spec.m, s);
      else
        sketch_apply(spec, sub, sa.get() + c0 * spec.m, s);
      op_apply_t(ctx, sub, b.ptr, K, ctmp.get(), false);
      copy_cols(ctmp.get(), cc, K, cc, cbuf.get() + c0, dim, s);
      if (use_matrix) gram.matrix_rows(c0, c0 + cc);
    }
    allreduce(ctx, sa.get(), spec.m * dim);
    RP_CUDA(cudaEventRecord(ev.ev[1], s));
    allreduce(ctx, cbuf.get(), dim * K);
    RP_CUDA(cudaEventRecord(ev.ev[5], s));
    if (use_matrix) gram.end_matrix();
  } else {
    // The Gram matrix (a throughput-bound SYRK over A) runs on the context's
    // side stream from the start, overlapping the HBM-bound sketch and the
    // latency-bound preconditioner build; the basis waits for both.  (All
    // streams at one priority: preempting a CTA of the TMA SYRK corrupts it
    // -- DESIGN.md, concurrency finding.)
    // (single process only: with a communicator the Gram all-reduce would be
    // in flight on a second stream next to the sketch all-reduce)
    // (only for Gram matrices up to 4096^2, the measured range)
    const bool side_gram = use_matrix && ctx->gram_overlap && !has_comm(ctx) && op.d <= 4096;
    auto launch_side_gram = [&]() {
      if (!ctx->side) {
        RP_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
      }
      RP_CUDA(cudaEventCreateWithFlags(&gram_done, cudaEventDisableTiming));
      RP_CUDA(cudaEventRecord(gram_done, s));
      RP_CUDA(cudaStreamWaitEvent(ctx->side, gram_done, 0));
      gram.build_matrix(ctx->side);
      RP_CUDA(cudaEventRecord(gram_done, ctx->side));
    };
    if (side_gram && !ctx->gram_after_sketch) launch_side_gram();
    // 1) Sketch (once), summed over ranks.  While the Gram SYRK occupies the
    //    side stream, the sketch -- on the critical path to the
    //    preconditioner -- runs on a second stream of the context.
    if (gram_done && ctx->sketch_on_hi) {
      if (!ctx->hi) {
        int lo_p = 0, hi_p = 0;
        if (ctx->stream_priorities) RP_CUDA(cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p));
        RP_CUDA(cudaStreamCreateWithPriority(&ctx->hi, cudaStreamNonBlocking, ctx->stream_priorities ? hi_p : 0));
      }
      cudaEvent_t fork;
      RP_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
      RP_CUDA(cudaEventRecord(fork, s));
      RP_CUDA(cudaStreamWaitEvent(ctx->hi, fork, 0));
      sketch_apply(spec, op, sa.get(), ctx->hi);
      RP_CUDA(cudaEventRecord(fork, ctx->hi));
      RP_CUDA(cudaStreamWaitEvent(s, fork, 0));
      RP_CUDA(cudaEventDestroy(fork));
    } else {
      sketch_apply(spec, op, sa.get(), s);
    }
    allreduce(ctx, sa.get(), spec.m * dim);
    if (side_gram && ctx->gram_after_sketch == 1) launch_side_gram();
    RP_CUDA(cudaEventRecord(ev.ev[1], s));
    // 3) Linear term: c = M^T b (primal) or c = b (dual).
    if (!dual) {
      op_apply_t(ctx, op, b.ptr, K, cbuf.get(), true);
    } else {
      copy_cols(b.ptr, dim, K, dim, cbuf.get(), dim, s);
    }
    if (side_gram && ctx->gram_after_sketch == 2) launch_side_gram();
    RP_CUDA(cudaEventRecord(ev.ev[5], s));
  }
  if (use_matrix && !gram.matrix) gram.build_matrix();  // (gram_overlap off)
  RP_CUDA(cudaEventRecord(ev.ev[6], s));
  nv.next("preconditioners (batched factorization)");
  // 4) Interval ownership.  With the Gram matrix every rank holds the whole
  //    operator state (SA, c, G are all-reduced), so the intervals -- which are
  //    independent (path_solver.cpp:168-186) -- are split round-robin and the
  //    composed x(lambda) summed.  In pass mode every generation needs every
  //    rank's rows, so all ranks run all intervals.
  const bool split = ctx->world > 1 && gram.matrix;
  std::vector<int64_t> own;
  for (int64_t l = 0; l < L; ++l)
    if (!split || l % ctx->world == ctx->rank) own.push_back(l);
  const int64_t Lo = static_cast<int64_t>(own.size());
  // Preconditioners for the owned shifts (shared sketch, one reshift per
  // interval: path_solver.cpp:164-170).
  PrecondBatch P;
  std::vector<double> l0s, taus;
  std::vector<int> ks;
  for (int64_t l : own) {
    l0s.push_back(plans[l].params.lambda0);
    taus.push_back(plans[l].params.alpha);
    ks.push_back(plans[l].params.k);
  }
  P.col_stable = ctx->stable_columns;
  P.allow_fshard = !split;
  gram.col_stable = ctx->stable_columns;
  if (Lo > 0) P.build(ctx, sa.get(), nullptr, spec.m, dim, l0s);
  if (gram_done) {
    RP_CUDA(cudaStreamWaitEvent(s, gram_done, 0));
    RP_CUDA(cudaEventDestroy(gram_done));  // (released once complete)
  }
  RP_CUDA(cudaEventRecord(ev.ev[2], s));
  nv.next("interval bases (all intervals, lock-step generations)");
  if (const char* dir = std::getenv("RP_DUMP_DIR")) {  // concurrency probe: the set-up products, raw bits
    RP_CUDA(cudaDeviceSynchronize());
    auto dump = [&](const char* name, const double* p, int64_t count) {
      if (!p || count <= 0) return;
      std::vector<double> h(static_cast<size_t>(count));
      RP_CUDA(cudaMemcpy(h.data(), p, sizeof(double) * count, cudaMemcpyDeviceToHost));
      const std::string path = std::string(dir) + "/" + name + ".bin";
      if (FILE* f = std::fopen(path.c_str(), "wb")) {
        std::fwrite(h.data(), sizeof(double), h.size(), f);
        std::fclose(f);
      }
    };
    dump("sa", sa.get(), spec.m * dim);
    dump("c", cbuf.get(), dim * K);
    if (gram.matrix) dump("gram", gram.G.get(), dim * dim);
    if (Lo > 0) dump("inv0", P.inv, P.n() * P.n());
  }
  // 5) Bases for all owned intervals at once; diverged intervals are retried
  //    at tau/2 (path_solver.cpp:132-140).
  BasisRun run2;
  // the first attempt's bases: one run over all owned intervals, or two runs
  // over the two halves on two streams (part p of `runs` covers own positions
  // [pbeg[p], pend[p]); in Gram-matrix mode the split was measured at -0.1 ms
  // on C2, so there it is opt-in; its round-2 run-to-run differences on C3
  // were the TMA stage-release race, fixed since)
  std::vector<BasisRun> runs(1);
  std::vector<int64_t> pbeg{0}, pend{Lo};
  std::vector<int64_t> retry;             // positions in `own`
  std::vector<int> retry_slot(static_cast<size_t>(Lo), -1);
  int failed = 0;
  if (Lo > 0) {
    // Option "basis_streams" = 2: two interval groups on two streams
    // (BasisStepper), interleaved generation by generation: exact (every
    // group runs the one-stream arithmetic on its own intervals).
    const bool two_ok = Lo >= 2 && !has_comm(ctx) && (gram.matrix || op.sparse);
    const bool two = two_ok && ctx->basis_streams == 2;
    if (!two) {
      run_basis(ctx, gram, P, cbuf.get(), K, taus, ks, runs[0]);
    } else {
      if (!ctx->basis2) RP_CUDA(cudaStreamCreateWithFlags(&ctx->basis2, cudaStreamNonBlocking));
      // (the lazily built panel structure of the sparse Gram passes: once, here, before the second stream reads it)
      if (!gram.matrix && op.sparse) (void)GramOp::panel_csc(ctx, op);
      const int64_t h = (Lo + 1) / 2;
      runs.resize(2);
      pbeg = {0, h};
      pend = {h, Lo};
      const PrecondBatch PA = P.slice(ctx, 0, h), PB = P.slice(ctx, h, Lo);
      cudaEvent_t fork;
      RP_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
      RP_CUDA(cudaEventRecord(fork, s));
      RP_CUDA(cudaStreamWaitEvent(ctx->basis2, fork, 0));
      {
        BasisStepper A(ctx, gram, PA, runs[0], s), B(ctx, gram, PB, runs[1], ctx->basis2);
        A.begin(cbuf.get(), K, std::vector<double>(taus.begin(), taus.begin() + h),
                std::vector<int>(ks.begin(), ks.begin() + h));
        B.begin(cbuf.get(), K, std::vector<double>(taus.begin() + h, taus.end()),
                std::vector<int>(ks.begin() + h, ks.end()));
        for (int64_t g = 1; g < std::max(A.kmax, B.kmax); ++g) {
          A.step(g);
          B.step(g);
        }
        A.finish();
        B.finish();
        RP_CUDA(cudaEventRecord(fork, ctx->basis2));  // (the steppers' buffers are freed on their streams)
      }
      RP_CUDA(cudaStreamWaitEvent(s, fork, 0));
      RP_CUDA(cudaStreamSynchronize(s));
      RP_CUDA(cudaStreamSynchronize(ctx->basis2));
      RP_CUDA(cudaEventDestroy(fork));
    }
    for (size_t q = 0; q < runs.size(); ++q)
      for (int64_t i = pbeg[q]; i < pend[q]; ++i)
        if (runs[q].diverged[static_cast<size_t>(i - pbeg[q])]) retry.push_back(i);
    if (!retry.empty()) {
      PrecondBatch P2;
      std::vector<double> l0r, taur;
      std::vector<int> kr;
      for (size_t j = 0; j < retry.size(); ++j) {
        l0r.push_back(l0s[retry[j]]);
        taur.push_back(taus[retry[j]] / 2.0);
        kr.push_back(ks[retry[j]]);
        retry_slot[retry[j]] = static_cast<int>(j);
      }
      P2.col_stable = ctx->stable_columns;
      P2.allow_fshard = !split;
      P2.build(ctx, sa.get(), nullptr, spec.m, dim, l0r);
      run_basis(ctx, gram, P2, cbuf.get(), K, taur, kr, run2);
      for (int v : run2.diverged) failed |= v;
    }
  }
  if (ctx->world > 1) {  // every rank must agree before anyone throws
    DBuf<double> f(1, s);
    const double fv = failed;
    RP_CUDA(cudaMemcpyAsync(f.get(), &fv, sizeof(double), cudaMemcpyHostToDevice, s));
    allreduce(ctx, f.get(), 1);
    double tot = 0;
    RP_CUDA(cudaMemcpyAsync(&tot, f.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
    RP_CUDA(cudaStreamSynchronize(s));
    failed = tot > 0.0;
  }
  if (failed) throw SolverFailure("interval basis diverged twice, even at tau/2");
  RP_CUDA(cudaEventRecord(ev.ev[3], s));
  nv.next("compose x(lambda) + recovery");
  // 6) Compose x(lambda) for every owned grid point (Horner,
  //    path_solver.cpp:64-74).
  const int64_t T = static_cast<int64_t>(cfg.lambdas.size());
  DBuf<double> xs(static_cast<size_t>(dim * K * T), s);
  if (split) fill(xs.get(), dim * K * T, 0.0, s);
  const size_t nparts = runs.size();
  for (size_t pass = 0; pass <= nparts; ++pass) {
    const bool retry_pass = pass == nparts;
    BasisRun& R = retry_pass ? run2 : runs[pass];
    if (retry_pass && retry.empty()) break;
    std::vector<double> lam;
    std::vector<int> itv;
    std::vector<int64_t> tidx;
    const int64_t i0 = retry_pass ? 0 : pbeg[pass], i1 = retry_pass ? Lo : pend[pass];
    for (int64_t i = i0; i < i1; ++i) {
      const bool mine = retry_pass ? retry_slot[i] >= 0 : retry_slot[i] < 0;
      if (!mine) continue;
      for (int64_t t : plans[own[i]].grid) {
        lam.push_back(cfg.lambdas[t]);
        itv.push_back(retry_pass ? retry_slot[i] : static_cast<int>(i - i0));
        tidx.push_back(t);
      }
    }
    if (lam.empty()) continue;
    const int64_t Tn = static_cast<int64_t>(lam.size());
    DBuf<double> d_lam(static_cast<size_t>(Tn), s);
    DBuf<int> d_itv(static_cast<size_t>(Tn), s);
    RP_CUDA(cudaMemcpyAsync(d_lam.get(), lam.data(), sizeof(double) * Tn, cudaMemcpyHostToDevice, s));
    RP_CUDA(cudaMemcpyAsync(d_itv.get(), itv.data(), sizeof(int) * Tn, cudaMemcpyHostToDevice, s));
    // grid points of one batch are contiguous in t when no interval is skipped
    const bool contiguous = tidx.back() - tidx.front() + 1 == Tn;
    if (contiguous) {
      compose_points(ctx, R, itv, d_lam.get(), d_itv.get(), Tn, xs.get() + tidx.front() * dim * K);
    } else {
      DBuf<double> tmp(static_cast<size_t>(dim * K * Tn), s);
      compose_points(ctx, R, itv, d_lam.get(), d_itv.get(), Tn, tmp.get());
      for (int64_t i = 0; i < Tn; ++i)
        copy_cols(tmp.get() + i * dim * K, dim, K, dim, xs.get() + tidx[i] * dim * K, dim, s);
    }
    RP_CUDA(cudaStreamSynchronize(s));
  }
  if (split) allreduce(ctx, xs.get(), dim * K * T);  // exact: every entry has one non-zero term
  // 7) Dual recovery v = A^T z = M_local z (path_solver.cpp:342).
  const int64_t out_rows = dual ? op.n_loc : dim;
  OutBuf xo(x_out, static_cast<size_t>(out_rows * K * T), where, s);
  if (dual) {
    op_apply(ctx, op, xs.get(), K * T, xo.dev);
  } else {
    RP_CUDA(cudaMemcpyAsync(xo.dev, xs.get(), sizeof(double) * dim * K * T, cudaMemcpyDeviceToDevice, s));
  }
  RP_CUDA(cudaEventRecord(ev.ev[4], s));
  RP_CUDA(cudaEventSynchronize(ev.ev[4]));
  tc0 = std::chrono::steady_clock::now();
  xo.finish();
  copy_secs += std::chrono::duration<double>(std::chrono::steady_clock::now() - tc0).count();
  if (tm) {
    std::memset(tm, 0, sizeof(*tm));
    tm->sketch_seconds = ev.secs(0, 1);
    tm->factor_seconds = ev.secs(1, 2);
    tm->basis_seconds = ev.secs(2, 3);
    tm->eval_seconds = ev.secs(3, 4);
    tm->setup_seconds = ev.secs(0, 3);
    tm->total_seconds = ev.secs(0, 4);
    tm->copy_seconds = copy_secs;
    tm->retries = static_cast<int32_t>(retry.size());
    tm->gram_mode = gram.matrix ? 1 : 0;
    tm->launches = launch_counter().load() - launches0;
    tm->linear_seconds = ev.secs(1, 5);
    tm->gram_seconds = ev.secs(5, 6);
    tm->precond_seconds = ev.secs(6, 2);
    if (prof) {
      prof->resolve(&tm->gemm_seconds, &tm->gemm_flops, &tm->gemm_calls);
      prof->launches(ctx->prof_seconds, ctx->prof_flops, ctx->prof_bytes);
    }
  }
  (void)host_t0;
}

rp_status status_of(rp_ctx* ctx, const std::exception& e, rp_status code) {
  if (ctx) ctx->err = e.what();
  return code;
}

}  // namespace rpb

// ============================================================================
// C ABI
// ============================================================================

using namespace rpb;

namespace {

thread_local std::string g_err_noctx;

// Optional lock per device (RP_DEVICE_LOCK=1), held for the whole of every
// context call, so that contexts sharing a GPU in one process never overlap
// their device work.  Rounds 1-2 needed it (concurrent grids exposed the TMA
// GEMM's stage-release race, concurrency finding); since the fix
// contexts driven from different threads run concurrently and the lock is
// off by default.  Recursive: a call may use another entry point.
std::recursive_mutex& device_mutex(int dev) {
  static std::recursive_mutex m[64];
  return m[static_cast<unsigned>(dev) % 64];
}

template <class F>
rp_status guarded(rp_ctx* ctx, F&& f) {
  try {
    std::optional<DeviceGuard> guard;
    std::unique_lock<std::recursive_mutex> lock;
    static const bool use_lock = [] {  // RP_DEVICE_LOCK=1: serialize the calls of contexts that share a GPU
      const char* e = std::getenv("RP_DEVICE_LOCK");
      return e && e[0] == '1';
    }();
    if (ctx) {
      if (use_lock) lock = std::unique_lock<std::recursive_mutex>(device_mutex(ctx->device));
      guard.emplace(ctx->device);
    }
    f();
    return RP_OK;
  } catch (const ParseFailure& e) {
    if (!ctx) g_err_noctx = e.what();
    return status_of(ctx, e, RP_EPARSE);
  } catch (const InvalidArgument& e) {
    if (!ctx) g_err_noctx = e.what();
    return status_of(ctx, e, RP_EINVAL);
  } catch (const BasisDiverged& e) {
    return status_of(ctx, e, RP_EDIVERGED);
  } catch (const SolverFailure& e) {
    return status_of(ctx, e, RP_ESOLVER);
  } catch (const FactorFailure& e) {
    return status_of(ctx, e, RP_ESVD);
  } catch (const NcclFailure& e) {
    if (!ctx) g_err_noctx = e.what();
    return status_of(ctx, e, RP_ENCCL);
  } catch (const CudaFailure& e) {
    if (!ctx) g_err_noctx = e.what();
    const bool oom = std::string(e.what()).find("allocation") != std::string::npos;
    return status_of(ctx, e, oom ? RP_ENOMEM : RP_ECUDA);
  } catch (const std::invalid_argument& e) {
    if (!ctx) g_err_noctx = e.what();
    return status_of(ctx, e, RP_EINVAL);
  } catch (const std::exception& e) {
    if (!ctx) g_err_noctx = e.what();
    return status_of(ctx, e, RP_ECUDA);
  }
}

void copy_out_i64(int64_t* dst, const int32_t* src_dev, int64_t n, int where, cudaStream_t s) {
  std::vector<int32_t> tmp(static_cast<size_t>(n));
  RP_CUDA(cudaMemcpyAsync(tmp.data(), src_dev, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  RP_CUDA(cudaStreamSynchronize(s));
  std::vector<int64_t> wide(tmp.begin(), tmp.end());
  if (where == RP_DEVICE)
    RP_CUDA(cudaMemcpyAsync(dst, wide.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
  else
    std::memcpy(dst, wide.data(), sizeof(int64_t) * n);
  RP_CUDA(cudaStreamSynchronize(s));
}

template <class T>
void copy_out(T* dst, const T* src_dev, int64_t n, int where, cudaStream_t s) {
  if (n <= 0) return;
  RP_CUDA(cudaMemcpyAsync(dst, src_dev, sizeof(T) * n, where == RP_DEVICE ? cudaMemcpyDeviceToDevice
                                                                          : cudaMemcpyDeviceToHost, s));
  RP_CUDA(cudaStreamSynchronize(s));
}

void set_csr_impl(rp_ctx* ctx, int64_t n_global, int64_t row0, int64_t n_local, int64_t d, const int64_t* offsets,
                  const int64_t* cols, const double* vals, int where, int shard) {
  require(n_local >= 0 && d >= 0 && n_global >= n_local, "csr: negative dimensions");
  require(d < (int64_t{1} << 31) && n_local < (int64_t{1} << 31), "csr: dimensions exceed int32 indices");
  cudaStream_t s = ctx->stream;
  // Row offsets are validated on the host (n + 1 values); the entries never
  // visit the host: invariants, int32 columns and the CSC mirror (a stable
  // radix sort by column keeps the rows of a column ascending, as the
  // reference's counting pass does) are built on the device.
  std::vector<int64_t> off(static_cast<size_t>(n_local + 1));
  if (where == RP_DEVICE) {
    RP_CUDA(cudaMemcpy(off.data(), offsets, sizeof(int64_t) * (n_local + 1), cudaMemcpyDeviceToHost));
  } else {
    std::memcpy(off.data(), offsets, sizeof(int64_t) * (n_local + 1));
  }
  require(off.front() == 0, "csr: row_offsets must start at 0");
  for (int64_t i = 0; i < n_local; ++i) require(off[i] <= off[i + 1], "csr: row_offsets must be monotone");
  const int64_t nnz = off.back();
  require(nnz < (int64_t{1} << 31), "csr: more than 2^31 entries");
  OperatorStore o;  // (built aside: a rejected matrix leaves the context's operator as it was)
  o.sparse = true;
  o.n = n_global;
  o.d = d;
  o.shard = shard;
  o.off0 = row0;
  o.n_local = n_local;
  o.nnz = nnz;
  o.csr_off.alloc(off.size(), s);
  o.csr_col.alloc(static_cast<size_t>(std::max<int64_t>(nnz, 1)), s);
  o.csr_val.alloc(static_cast<size_t>(std::max<int64_t>(nnz, 1)), s);
  RP_CUDA(cudaMemcpyAsync(o.csr_off.get(), off.data(), sizeof(int64_t) * off.size(), cudaMemcpyHostToDevice, s));
  if (nnz > 0) {
    DBuf<int64_t> c64;
    const int64_t* d_c64 = cols;
    if (where != RP_DEVICE) {
      c64.alloc(static_cast<size_t>(nnz), s);
      RP_CUDA(cudaMemcpyAsync(c64.get(), cols, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, s));
      d_c64 = c64.get();
    }
    RP_CUDA(cudaMemcpyAsync(o.csr_val.get(), vals, sizeof(double) * nnz,
                            where == RP_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    DBuf<long long> flag(1, s);
    const long long none = std::numeric_limits<long long>::max();
    RP_CUDA(cudaMemcpyAsync(flag.get(), &none, sizeof(none), cudaMemcpyHostToDevice, s));
    csr_validate_convert(o.csr_off.get(), d_c64, o.csr_val.get(), n_local, d, o.csr_col.get(), flag.get(), s);
    long long seen = none;
    RP_CUDA(cudaMemcpyAsync(&seen, flag.get(), sizeof(seen), cudaMemcpyDeviceToHost, s));
    RP_CUDA(cudaStreamSynchronize(s));
    if (seen != none) {
      switch (static_cast<int>(seen & 3)) {
        case 1: throw InvalidArgument("csr: column index out of range");
        case 2: throw InvalidArgument("csr: column indices must be strictly increasing within a row");
        default: throw InvalidArgument("csr: non-finite value");
      }
    }
  }
  {
    PanelCsc mirror;  // one panel over all rows = the CSC of the shard
    build_panel_csc(o.csr_off.get(), o.csr_col.get(), o.csr_val.get(), n_local, d, nnz, std::max<int64_t>(n_local, 1),
                    mirror, s);
    o.csc_off = std::move(mirror.off);
    o.csc_row = std::move(mirror.row);
    o.csc_val = std::move(mirror.val);
  }
  RP_CUDA(cudaStreamSynchronize(s));
  o.set = true;
  wait_upload(ctx);
  ctx->op = std::move(o);
}

void set_dense_impl(rp_ctx* ctx, int64_t n, int64_t d, int shard, int64_t off0, int64_t n_local, const double* a,
                    int64_t lda, int where) {
  require(n >= 0 && d >= 0 && n_local >= 0, "dense: negative dimensions");
  const int64_t rows = shard == 1 ? n_local : n;
  const int64_t cols = shard == 2 ? n_local : d;
  require(lda >= std::max<int64_t>(rows, 1), "dense: leading dimension too small");
  cudaStream_t s = ctx->stream;
  OperatorStore& o = ctx->op;
  wait_upload(ctx);  // the old buffer is freed on this stream: after its upload
  o = OperatorStore();
  o.sparse = false;
  o.n = n;
  o.d = d;
  o.shard = shard;
  o.off0 = off0;
  o.n_local = n_local;
  if (where == RP_DEVICE) {
    o.a = a;
    o.lda = lda;
  } else if (where == RP_HOST_STREAM) {
    // Column chunks of ~upload_chunk_bytes (32 MiB) on the copy stream, one event each.
    o.owned.alloc(static_cast<size_t>(std::max<int64_t>(rows * cols, 1)), s);
    {
      // free device memory once the operator's buffer exists (asked here, before the copies start: the query
      // takes ~10 ms beside a running upload); the streamed Gaussian sketch budgets its resident S with it
      size_t free_b = 0, total_b = 0;
      RP_CUDA(cudaStreamSynchronize(s));
      RP_CUDA(cudaMemGetInfo(&free_b, &total_b));
      o.free_after_alloc = static_cast<double>(free_b);
    }
    if (!ctx->copy) RP_CUDA(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
    cudaEvent_t alloc_done;
    RP_CUDA(cudaEventCreateWithFlags(&alloc_done, cudaEventDisableTiming));
    RP_CUDA(cudaEventRecord(alloc_done, s));
    RP_CUDA(cudaStreamWaitEvent(ctx->copy, alloc_done, 0));
    RP_CUDA(cudaEventDestroy(alloc_done));
    const int64_t chunk = std::max<int64_t>(1, ctx->upload_chunk_bytes / std::max<int64_t>(1, rows * 8));
    Upload& up = o.up;
    up.chunk = chunk;
    up.src = a;
    up.lda = lda;
    up.rows = rows;
    up.cols = cols;
    up.dst = o.owned.get();
    up.copy = ctx->copy;
    up.next = 0;
    up.ev.resize(static_cast<size_t>(std::max<int64_t>(1, ceil_div(cols, chunk))));
    for (auto& e : up.ev) RP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    up.enqueue(1);  // the consumer keeps kUploadDepth chunks in flight from here on
    o.a = o.owned.get();
    o.lda = std::max<int64_t>(rows, 1);
  } else {
    o.owned.alloc(static_cast<size_t>(std::max<int64_t>(rows * cols, 1)), s);
    RP_CUDA(cudaMemcpy2DAsync(o.owned.get(), sizeof(double) * rows, a, sizeof(double) * lda, sizeof(double) * rows,
                              static_cast<size_t>(cols), cudaMemcpyHostToDevice, s));
    RP_CUDA(cudaStreamSynchronize(s));
    o.a = o.owned.get();
    o.lda = std::max<int64_t>(rows, 1);
  }
  o.set = true;
}

}  // namespace

extern "C" {

const char* rp_version(void) { return "ridgepath-b200 0.1 (sm_100a)"; }

int64_t rp_launch_count(void) { return launch_counter().load(); }

rp_status rp_create(rp_ctx** out, int device) {
  if (!out) return RP_EINVAL;
  *out = nullptr;
  rp_ctx* ctx = new rp_ctx();
  ctx->device = device;
  const rp_status st = guarded(nullptr, [&] {
    int count = 0;
    RP_CUDA(cudaGetDeviceCount(&count));
    require(device >= 0 && device < count, "rp_create: no such CUDA device");
    DeviceGuard g(device);
    RP_CUDA(cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking));
    ctx->stream = ctx->own;
    // Keep stream-ordered allocations cached across calls (the default release
    // threshold of 0 returns every freed block to the driver at each sync).
    cudaMemPool_t pool;
    RP_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = UINT64_MAX;
    RP_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    mt::init_tables();
  });
  if (st != RP_OK) {
    delete ctx;
    return st;
  }
  *out = ctx;
  return RP_OK;
}

void rp_destroy(rp_ctx* ctx) {
  if (!ctx) return;
  {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(ctx->device);
    if (!ctx->op.up.ev.empty()) cudaStreamWaitEvent(ctx->stream, ctx->op.up.ev.back(), 0);
    cudaStreamSynchronize(ctx->stream);
    ctx->op = OperatorStore();
    if (ctx->copy) cudaStreamDestroy(ctx->copy);
    if (ctx->side) {
      release_workspace(ctx->side);
      cudaStreamSynchronize(ctx->side);
      cudaStreamDestroy(ctx->side);
    }
    if (ctx->hi) {
      release_workspace(ctx->hi);
      cudaStreamSynchronize(ctx->hi);
      cudaStreamDestroy(ctx->hi);
    }
    if (ctx->basis2) {
      release_workspace(ctx->basis2);
      cudaStreamSynchronize(ctx->basis2);
      cudaStreamDestroy(ctx->basis2);
    }
    if (ctx->comm && nccl().CommDestroy) nccl().CommDestroy(ctx->comm);
    if (ctx->host_stage) cudaFreeHost(ctx->host_stage);
    if (ctx->own) {
      release_workspace(ctx->own);
      cudaStreamDestroy(ctx->own);
    }
    cudaSetDevice(prev);
  }
  delete ctx;
}

const char* rp_last_error(const rp_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err_noctx.c_str(); }

rp_status rp_set_stream(rp_ctx* ctx, void* stream) {
  if (!ctx) return RP_EINVAL;
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own;
  return RP_OK;
}

rp_status rp_synchronize(rp_ctx* ctx) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] { RP_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

rp_status rp_set_option(rp_ctx* ctx, const char* key, int64_t value) {
  if (!ctx || !key) return RP_EINVAL;
  return guarded(ctx, [&] {
    const std::string k(key);
    if (k == "gram_mode") {
      require(value >= -1 && value <= 1, "gram_mode must be -1, 0 or 1");
      ctx->gram_mode = static_cast<int>(value);
    } else if (k == "profile") {
      ctx->profile = value != 0;
    } else if (k == "fuse_update") {
      ctx->fuse_update = value != 0;
    } else if (k == "compose_gemm") {
      ctx->compose_gemm = value != 0;
    } else if (k == "stable_columns") {
      ctx->stable_columns = value != 0;
    } else if (k == "csr_panel_rows") {
      require(value >= 1 && value < (int64_t{1} << 31), "csr_panel_rows must be in [1, 2^31)");
      ctx->csr_panel_rows = value;
    } else if (k == "gram_overlap_split") {
      require(value >= 0 && value <= 64, "gram_overlap_split must be in [0, 64]");
      ctx->gram_overlap_split = static_cast<int>(value);
    } else if (k == "csr_blocks_per_sm") {
      require(value >= 0 && value <= 8, "csr_blocks_per_sm must be in [0, 8]");
      ctx->csr_blocks_per_sm = static_cast<int>(value);
    } else if (k == "csr_l2_persist") {
      ctx->csr_l2_persist = value != 0;
    } else if (k == "basis_streams") {
      require(value == 1 || value == 2, "basis_streams must be 1 or 2");
      ctx->basis_streams = static_cast<int>(value);
    } else if (k == "feature_shard") {
      ctx->feature_shard = value != 0;
    } else if (k == "stream_priorities") {
      if (ctx->stream_priorities != (value != 0) && ctx->hi) {  // (recreated at the new priority on next use)
        RP_CUDA(cudaStreamSynchronize(ctx->hi));
        release_workspace(ctx->hi);
        RP_CUDA(cudaStreamDestroy(ctx->hi));
        ctx->hi = nullptr;
      }
      ctx->stream_priorities = value != 0;
    } else if (k == "sketch_on_hi") {
      ctx->sketch_on_hi = value != 0;
    } else if (k == "gram_overlap_tma") {
      ctx->gram_overlap_tma = value != 0;
    } else if (k == "gram_overlap_tile") {
      require(value >= -1 && value < 13, "gram_overlap_tile must be in [-1, 12]");
      ctx->gram_overlap_tile = static_cast<int>(value);
    } else if (k == "gram_overlap_occ") {
      require(value >= 0 && value <= 4, "gram_overlap_occ must be in [0, 4]");
      ctx->gram_overlap_occ = static_cast<int>(value);
    } else if (k == "gram_after_sketch") {
      require(value >= 0 && value <= 2, "gram_after_sketch must be 0, 1 or 2");
      ctx->gram_after_sketch = static_cast<int>(value);
    } else if (k == "gram_overlap") {
      ctx->gram_overlap = value != 0;
    } else if (k == "upload_chunk_bytes") {
      require(value >= 1, "upload_chunk_bytes must be >= 1");
      ctx->upload_chunk_bytes = value;
    } else if (k == "csr_one_panel_bytes") {
      require(value >= 0, "csr_one_panel_bytes must be >= 0");
      ctx->csr_one_panel_bytes = value;
    } else if (k == "csr_chunk") {
      require(value >= 1 && value <= 128, "csr_chunk must be in [1, 128]");
      ctx->csr_chunk = value;
    } else {
      throw InvalidArgument("unknown option: " + k);
    }
  });
}

rp_status rp_last_gemm_profile(rp_ctx* ctx, double* seconds, double* flops, double* bytes, int64_t cap,
                               int64_t* count) {
  if (!ctx || !count) return RP_EINVAL;
  return guarded(ctx, [&] {
    const int64_t n = static_cast<int64_t>(ctx->prof_seconds.size());
    *count = n;
    for (int64_t i = 0; i < std::min(n, cap); ++i) {
      if (seconds) seconds[i] = ctx->prof_seconds[i];
      if (flops) flops[i] = ctx->prof_flops[i];
      if (bytes) bytes[i] = ctx->prof_bytes[i];
    }
  });
}

rp_status rp_comm_unique_id(void* id128) {
  return guarded(nullptr, [&] {
    require(id128 != nullptr, "unique id: null buffer");
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(id128, &id, 128);
  });
}

rp_status rp_comm_init(rp_ctx* ctx, int rank, int world, const void* id128) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    require(world >= 1 && rank >= 0 && rank < world, "comm: bad rank/world");
    ctx->rank = rank;
    ctx->world = world;
    // world 1 without an id: no communicator (collectives are no-ops); with an
    // id, a one-rank NCCL communicator (the collectives then run through NCCL)
    if (world == 1 && id128 == nullptr) return;
    require(id128 != nullptr, "comm: null unique id");
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    nccl_check(nccl().CommInitRank(&ctx->comm, world, id, rank), "ncclCommInitRank");
  });
}

rp_status rp_comm_init_host(rp_ctx* ctx, int rank, int world, rp_host_allreduce_fn allreduce_fn,
                            rp_host_allgather_fn allgather_fn, void* user) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    require(world >= 1 && rank >= 0 && rank < world, "comm: bad rank/world");
    require(allreduce_fn != nullptr && allgather_fn != nullptr, "comm: null host callback");
    require(ctx->comm == nullptr, "comm: the context already has an NCCL communicator");
    ctx->rank = rank;
    ctx->world = world;
    ctx->host_allreduce = allreduce_fn;
    ctx->host_allgather = allgather_fn;
    ctx->host_user = user;
  });
}

rp_status rp_set_dense(rp_ctx* ctx, int64_t n, int64_t d, const double* a, int64_t lda, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] { set_dense_impl(ctx, n, d, 0, 0, n, a, lda, where); });
}

rp_status rp_set_dense_rows(rp_ctx* ctx, int64_t n_global, int64_t row0, int64_t n_local, int64_t d, const double* a,
                            int64_t lda, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    require(row0 >= 0 && row0 + n_local <= n_global, "dense rows: shard out of range");
    set_dense_impl(ctx, n_global, d, 1, row0, n_local, a, lda, where);
  });
}

rp_status rp_set_dense_cols(rp_ctx* ctx, int64_t n, int64_t d_global, int64_t col0, int64_t d_local, const double* a,
                            int64_t lda, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    require(col0 >= 0 && col0 + d_local <= d_global, "dense cols: shard out of range");
    set_dense_impl(ctx, n, d_global, 2, col0, d_local, a, lda, where);
  });
}

rp_status rp_set_csr(rp_ctx* ctx, int64_t n, int64_t d, const int64_t* offsets, const int64_t* cols,
                     const double* vals, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] { set_csr_impl(ctx, n, 0, n, d, offsets, cols, vals, where, 0); });
}

rp_status rp_set_csr_rows(rp_ctx* ctx, int64_t n_global, int64_t row0, int64_t n_local, int64_t d,
                          const int64_t* offsets, const int64_t* cols, const double* vals, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    require(row0 >= 0 && row0 + n_local <= n_global, "csr rows: shard out of range");
    set_csr_impl(ctx, n_global, row0, n_local, d, offsets, cols, vals, where, 1);
  });
}

// With the profile option, brackets the device work of one product call with
// CUDA events (the C-ABI call itself synchronizes, so host timing would add
// the round trip): rp_last_device_seconds() returns it.
struct DeviceTimer {
  rp_ctx* ctx;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  explicit DeviceTimer(rp_ctx* c) : ctx(c) {
    if (!ctx->profile) return;
    RP_CUDA(cudaEventCreate(&e0));
    RP_CUDA(cudaEventCreate(&e1));
    RP_CUDA(cudaEventRecord(e0, ctx->stream));
  }
  void stop() {
    if (!e0) return;
    RP_CUDA(cudaEventRecord(e1, ctx->stream));
    RP_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    RP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    ctx->last_device_seconds = ms * 1e-3;
  }
  ~DeviceTimer() {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  }
};

rp_status rp_apply(rp_ctx* ctx, const double* x, int64_t ncols, double* y, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    const OpView op = op_primal(ctx);
    require(ncols >= 0, "apply: dimension mismatch");
    InBuf in(x, static_cast<size_t>(op.d * ncols), where, ctx->stream);
    OutBuf out(y, static_cast<size_t>(op.n_loc * ncols), where, ctx->stream);
    if (ncols > 0) op_apply(ctx, op, in.ptr, ncols, out.dev);
    out.finish();
  });
}

rp_status rp_apply_transpose(rp_ctx* ctx, const double* y, int64_t ncols, double* x, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    const OpView op = op_primal(ctx);
    require(ncols >= 0, "apply_transpose: dimension mismatch");
    InBuf in(y, static_cast<size_t>(op.n_loc * ncols), where, ctx->stream);
    OutBuf out(x, static_cast<size_t>(op.d * ncols), where, ctx->stream);
    DeviceTimer timer(ctx);
    if (ncols > 0) op_apply_t(ctx, op, in.ptr, ncols, out.dev, true);
    timer.stop();
    out.finish();
  });
}

rp_status rp_gram_apply(rp_ctx* ctx, const double* x, int64_t ncols, double* outp, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    const OpView op = op_primal(ctx);
    require(ncols >= 0, "gram_apply: dimension mismatch");
    InBuf in(x, static_cast<size_t>(op.d * ncols), where, ctx->stream);
    OutBuf out(outp, static_cast<size_t>(op.d * ncols), where, ctx->stream);
    GramOp g;
    g.ctx = ctx;
    g.op = op;
    g.allow_fused = true;
    DeviceTimer timer(ctx);
    if (ncols > 0) g.apply(in.ptr, ncols, out.dev);
    timer.stop();
    out.finish();
  });
}

rp_status rp_last_device_seconds(rp_ctx* ctx, double* seconds) {
  if (!ctx || !seconds) return RP_EINVAL;
  *seconds = ctx->last_device_seconds;
  return RP_OK;
}

rp_status rp_losses(rp_ctx* ctx, const double* b, int64_t K, int64_t T, const double* x, const double* lambda,
                    double* lossp, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    const OpView op = op_primal(ctx);
    require(K >= 1 && T >= 0, "losses: dimension mismatch");
    cudaStream_t s = ctx->stream;
    InBuf xb(x, static_cast<size_t>(op.d * K * T), where, s);
    InBuf bb(b, static_cast<size_t>(op.n_loc * K), where, s);
    InBuf lb(lambda, lambda ? static_cast<size_t>(T) : 0, where, s);
    OutBuf out(lossp, static_cast<size_t>(T), where, s);
    if (T > 0) {
      DBuf<double> rn(static_cast<size_t>(T * K), s), xn(static_cast<size_t>(T * K), s);
      // residuals in chunks of solutions (R: n_local x chunk*K, <= ~1 GiB)
      const int64_t per = std::max<int64_t>(1, (int64_t{1} << 27) / std::max<int64_t>(1, op.n_loc * K));
      DBuf<double> r(static_cast<size_t>(op.n_loc * K * std::min<int64_t>(per, T)), s);
      for (int64_t t0 = 0; t0 < T; t0 += per) {
        const int64_t tc = std::min<int64_t>(per, T - t0);
        op_apply(ctx, op, xb.ptr + t0 * op.d * K, tc * K, r.get());
        column_sq_norms(r.get(), op.n_loc, tc * K, op.n_loc, bb.ptr, K, op.n_loc, rn.get() + t0 * K, s);
      }
      allreduce(ctx, rn.get(), T * K);  // row shards: sum the partial squared norms
      if (lb.ptr) column_sq_norms(xb.ptr, op.d, T * K, op.d, nullptr, 1, 0, xn.get(), s);
      combine_losses(rn.get(), lb.ptr ? xn.get() : nullptr, lb.ptr, T, K, out.dev, s);
    }
    out.finish();
  });
}

rp_status rp_sketch_apply(rp_ctx* ctx, const rp_sketch_spec* specp, int transpose_op, double* sa, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    const SketchSpecC spec = to_spec(specp);
    const OpView op = transpose_op ? op_dual(ctx) : op_primal(ctx);
    validate_spec(spec);
    require(op.n_global == spec.n, "sketch_apply: spec.n must match A.rows");
    OutBuf out(sa, static_cast<size_t>(spec.m * op.d), where, ctx->stream);
    sketch_apply(spec, op, out.dev, ctx->stream);
    allreduce(ctx, out.dev, spec.m * op.d);
    out.finish();
  });
}

rp_status rp_precond_build(rp_ctx* ctx, const double* sa, int64_t m, int64_t d, double lambda0, int where,
                           rp_precond** outp) {
  if (!ctx || !outp) return RP_EINVAL;
  *outp = nullptr;
  return guarded(ctx, [&] {
    if (lambda0 <= 0.0) throw InvalidArgument("preconditioner: shift must be positive");
    require(m >= 1 && d >= 1, "preconditioner: empty sketch");
    cudaStream_t s = ctx->stream;
    auto p = std::make_unique<rp_precond>();
    p->device = ctx->device;
    p->m = m;
    p->d = d;
    p->lambda0 = lambda0;
    p->woodbury = m < d;
    p->sa = std::make_shared<DBuf<double>>(static_cast<size_t>(m * d), s);
    if (where == RP_DEVICE)
      RP_CUDA(cudaMemcpyAsync(p->sa->get(), sa, sizeof(double) * m * d, cudaMemcpyDeviceToDevice, s));
    else
      RP_CUDA(cudaMemcpyAsync(p->sa->get(), sa, sizeof(double) * m * d, cudaMemcpyHostToDevice, s));
    PrecondBatch P;
    P.build(ctx, p->sa->get(), nullptr, m, d, {lambda0});
    p->inv = std::make_shared<DBuf<double>>(std::move(P.inv_owned));
    RP_CUDA(cudaStreamSynchronize(s));
    *outp = p.release();
  });
}

rp_status rp_precond_reshift(rp_ctx* ctx, const rp_precond* p, double lambda0, rp_precond** outp) {
  if (!ctx || !p || !outp) return RP_EINVAL;
  *outp = nullptr;
  return guarded(ctx, [&] {
    if (lambda0 <= 0.0) throw InvalidArgument("preconditioner: shift must be positive");
    auto q = std::make_unique<rp_precond>();
    q->device = p->device;
    q->m = p->m;
    q->d = p->d;
    q->lambda0 = lambda0;
    q->woodbury = p->woodbury;
    q->sa = p->sa;
    PrecondBatch P;
    P.build(ctx, q->sa->get(), nullptr, q->m, q->d, {lambda0});
    q->inv = std::make_shared<DBuf<double>>(std::move(P.inv_owned));
    RP_CUDA(cudaStreamSynchronize(ctx->stream));
    *outp = q.release();
  });
}

void rp_precond_destroy(rp_precond* p) {
  if (!p) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  p->inv.reset();
  p->sa.reset();
  cudaDeviceSynchronize();
  cudaSetDevice(prev);
  delete p;
}

namespace {

PrecondBatch view_of(rp_ctx* ctx, const rp_precond* p) {
  PrecondBatch P;
  P.m = p->m;
  P.d = p->d;
  P.L = 1;
  P.woodbury = p->woodbury;
  P.sa = p->sa->get();
  P.inv = p->inv->get();
  P.lambda0 = {p->lambda0};
  P.d_lambda0.alloc(1, ctx->stream);
  RP_CUDA(cudaMemcpyAsync(P.d_lambda0.get(), &p->lambda0, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  return P;
}

void precond_apply_borrowed(rp_ctx* ctx, const rp_precond* p, const double* in, int64_t cols, double* out) {
  const PrecondBatch P = view_of(ctx, p);
  P.apply(ctx, in, p->d * cols, cols, out, p->d * cols);
}

void basis_core(rp_ctx* ctx, const rp_precond* p, const OpView& op, const double* c_dev, int64_t K, double tau, int k,
                double* terms_out, int where) {
  require(op.d == p->d, "ihs_basis: preconditioner dimension mismatch");
  GramOp gram;
  gram.ctx = ctx;
  gram.op = op;
  if (ctx->gram_mode == 1) gram.build_matrix();
  const PrecondBatch P = view_of(ctx, p);
  BasisRun run;
  run_basis(ctx, gram, P, c_dev, K, {tau}, {k}, run);
  if (run.diverged[0]) throw BasisDiverged("basis recursion diverged (step too large)");
  // terms_out block j = tilde[:, j*K : (j+1)*K]  (NB = K for one interval)
  const int64_t dim = op.d;
  OutBuf out(terms_out, static_cast<size_t>(dim * K * k), where, ctx->stream);
  copy_cols(run.tilde.get(), dim, K * k, dim, out.dev, dim, ctx->stream);
  out.finish();
}

}  // namespace

rp_status rp_precond_apply(rp_ctx* ctx, const rp_precond* p, const double* v, int64_t ncols, double* outp,
                           int where) {
  if (!ctx || !p) return RP_EINVAL;
  return guarded(ctx, [&] {
    require(ncols >= 0, "preconditioner apply: dimension mismatch");
    InBuf in(v, static_cast<size_t>(p->d * ncols), where, ctx->stream);
    OutBuf out(outp, static_cast<size_t>(p->d * ncols), where, ctx->stream);
    if (ncols > 0) precond_apply_borrowed(ctx, p, in.ptr, ncols, out.dev);
    out.finish();
  });
}

rp_status rp_ihs_basis(rp_ctx* ctx, const rp_precond* p, const double* b, int64_t K, double tau, int32_t k,
                       double* terms_out, int where) {
  if (!ctx || !p) return RP_EINVAL;
  return guarded(ctx, [&] {
    require(K >= 1, "ihs_basis_matrix: empty right-hand side");
    require(k >= 1, "ihs_basis: k must be >= 1");
    require(tau > 0.0, "ihs_basis: tau must be positive");
    const OpView op = op_primal(ctx);
    InBuf bb(b, static_cast<size_t>(op.n_loc * K), where, ctx->stream);
    DBuf<double> c(static_cast<size_t>(op.d * K), ctx->stream);
    op_apply_t(ctx, op, bb.ptr, K, c.get(), true);
    basis_core(ctx, p, op, c.get(), K, tau, k, terms_out, where);
  });
}

rp_status rp_ihs_basis_core(rp_ctx* ctx, const rp_precond* p, const double* c, int64_t K, double tau, int32_t k,
                            int transpose_op, double* terms_out, int where) {
  if (!ctx || !p) return RP_EINVAL;
  return guarded(ctx, [&] {
    require(K >= 1, "ihs_basis_matrix: empty right-hand side");
    require(k >= 1, "ihs_basis: k must be >= 1");
    require(tau > 0.0, "ihs_basis: tau must be positive");
    const OpView op = transpose_op ? op_dual(ctx) : op_primal(ctx);
    require(op.d == p->d, "ihs_basis: operator/right-hand-side mismatch");
    InBuf cc(c, static_cast<size_t>(op.d * K), where, ctx->stream);
    basis_core(ctx, p, op, cc.ptr, K, tau, k, terms_out, where);
  });
}

rp_status rp_ihs_compose(rp_ctx* ctx, const double* terms, int64_t dim, int64_t K, int32_t k, double tau, double lambda,
                         double* x_out, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    require(k >= 1 && dim >= 0 && K >= 1, "ihs_compose: bad basis shape");
    cudaStream_t s = ctx->stream;
    InBuf tb(terms, static_cast<size_t>(dim * K * k), where, s);
    OutBuf out(x_out, static_cast<size_t>(dim * K), where, s);
    BasisDims d{dim, 1, K, k};
    DBuf<double> dt(1, s), dl(1, s);
    DBuf<int> dk(1, s), di(1, s);
    const int kk = k, zero = 0;
    RP_CUDA(cudaMemcpyAsync(dt.get(), &tau, sizeof(double), cudaMemcpyHostToDevice, s));
    RP_CUDA(cudaMemcpyAsync(dl.get(), &lambda, sizeof(double), cudaMemcpyHostToDevice, s));
    RP_CUDA(cudaMemcpyAsync(dk.get(), &kk, sizeof(int), cudaMemcpyHostToDevice, s));
    RP_CUDA(cudaMemcpyAsync(di.get(), &zero, sizeof(int), cudaMemcpyHostToDevice, s));
    if (dim > 0) compose(d, tb.ptr, dt.get(), dk.get(), dl.get(), di.get(), 1, out.dev, s);
    out.finish();
  });
}

rp_status rp_ihs_bin_path(rp_ctx* ctx, const double* b, int64_t K, const rp_path_config* cfg,
                          const rp_sketch_spec* spec, const rp_rho_bounds* rho, const double* sigma_d, double* x_out,
                          int where, rp_timings* timings) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    std::optional<double> sd;
    if (sigma_d) sd = *sigma_d;
    run_path(ctx, false, b, K, to_cfg(cfg), to_spec(spec), to_rho(rho), sd, x_out, where, timings);
  });
}

rp_status rp_dual_path(rp_ctx* ctx, const double* b, int64_t K, const rp_path_config* cfg, const rp_sketch_spec* spec,
                       const rp_rho_bounds* rho, const double* sigma_d, double* x_out, int where,
                       rp_timings* timings) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    std::optional<double> sd;
    if (sigma_d) sd = *sigma_d;
    run_path(ctx, true, b, K, to_cfg(cfg), to_spec(spec), to_rho(rho), sd, x_out, where, timings);
  });
}

rp_status rp_log_grid(double lambda_min, double lambda_max, int32_t count, double* out) {
  return guarded(nullptr, [&] {
    const auto g = log_grid(lambda_min, lambda_max, count);
    std::copy(g.begin(), g.end(), out);
  });
}

rp_status rp_tune_interval(double lambda_lo, double lambda_hi, const rp_rho_bounds* rho, const double* sigma_d,
                           double eps, rp_rate_params* out) {
  return guarded(nullptr, [&] {
    std::optional<double> sd;
    if (sigma_d) sd = *sigma_d;
    *out = tune_interval(lambda_lo, lambda_hi, to_rho(rho), sd, eps);
  });
}

int32_t rp_auto_interval_count(double lambda_min, double lambda_max) {
  int32_t v = -1;
  guarded(nullptr, [&] { v = auto_interval_count(lambda_min, lambda_max); });
  return v;
}

rp_status rp_interval_split(double lambda_min, double lambda_max, int32_t num_intervals, double* edges_out,
                            int32_t* count_out) {
  return guarded(nullptr, [&] {
    std::optional<int> num;
    if (num_intervals > 0) num = num_intervals;
    const auto sp = interval_split(lambda_min, lambda_max, num);
    *count_out = static_cast<int32_t>(sp.size());
    if (edges_out)
      for (size_t i = 0; i < sp.size(); ++i) {
        edges_out[2 * i] = sp[i].first;
        edges_out[2 * i + 1] = sp[i].second;
      }
  });
}

// ---- comparison baselines (baselines.cpp:80-226) --------------------------------
//
// The reference's speed/accuracy baselines for the IHS-BIN path, run on the
// same device operator.  warm_cg / warm_ihs are sequential per lambda (warm
// starts along the descending sweep); their per-iteration Gram product is the
// narrow fused pass (gram_pass.cu) for dense operators and the one-panel
// sparse pass for CSR.  Scalars stay on the device; the host reads the one
// convergence scalar per iteration.

namespace rpb {

std::vector<size_t> descending_order(const std::vector<double>& grid) {  // baselines.cpp:40-47
  std::vector<size_t> idx(grid.size());
  std::iota(idx.begin(), idx.end(), size_t{0});
  std::stable_sort(idx.begin(), idx.end(), [&](size_t i, size_t j) { return grid[i] > grid[j]; });
  return idx;
}

struct BaselineRun {
  std::vector<int32_t> iterations;
  std::vector<double> seconds;
  double setup_seconds = 0.0, total_seconds = 0.0;
};

double read_scalar(const double* dev, cudaStream_t s) {
  double v = 0.0;
  RP_CUDA(cudaMemcpyAsync(&v, dev, sizeof(double), cudaMemcpyDeviceToHost, s));
  RP_CUDA(cudaStreamSynchronize(s));
  return v;
}

double host_seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// warm_cg_path (baselines.cpp:120-162); x_out: d x T on the device.
void run_warm_cg(rp_ctx* ctx, const double* b, const PathCfg& cfg, double* x_out, BaselineRun& run) {
  cudaStream_t s = ctx->stream;
  const auto t_total = std::chrono::steady_clock::now();
  const OpView op = op_primal(ctx);
  const int64_t d = op.d;
  GramOp gram;
  gram.ctx = ctx;
  gram.op = op;
  gram.allow_fused = true;
  DBuf<double> atb(static_cast<size_t>(d), s), x(static_cast<size_t>(d), s), r(static_cast<size_t>(d), s),
      p(static_cast<size_t>(d), s), q(static_cast<size_t>(d), s), g(static_cast<size_t>(d), s),
      part(kDotParts, s), sc(4, s);
  op_apply_t(ctx, op, b, 1, atb.get(), true);
  vec_dot(atb.get(), atb.get(), d, part.get(), sc.get(), s);
  const double rhs_norm = std::sqrt(read_scalar(sc.get(), s));
  run.setup_seconds = host_seconds_since(t_total);
  const int64_t cap = 10 * d;
  const double tol = cfg.epsilon * (rhs_norm > 0.0 ? rhs_norm : 1.0);
  const size_t T = cfg.lambdas.size();
  run.iterations.assign(T, 0);
  run.seconds.assign(T, 0.0);
  fill(x.get(), d, 0.0, s);
  for (size_t idx : descending_order(cfg.lambdas)) {
    const double lam = cfg.lambdas[idx];
    const auto t_eval = std::chrono::steady_clock::now();
    gram.apply(x.get(), 1, g.get());
    cg_init(atb.get(), g.get(), x.get(), lam, d, r.get(), p.get(), s);
    vec_dot(r.get(), r.get(), d, part.get(), sc.get(), s);
    double rr = read_scalar(sc.get(), s);
    int slot = 0;  // sc[0] / sc[2] hold rr and rr_next in turn, sc[1] = p.q
    int32_t iters = 0;
    while (std::sqrt(rr) > tol) {
      if (iters >= cap) throw SolverFailure("warm_cg_path: iteration cap (10 d) reached");
      double* rr_dev = sc.get() + slot;
      double* rr_next_dev = sc.get() + (2 - slot);
      gram.apply(p.get(), 1, g.get());
      cg_q(g.get(), p.get(), lam, d, q.get(), s);
      vec_dot(p.get(), q.get(), d, part.get(), sc.get() + 1, s);
      cg_update(x.get(), r.get(), p.get(), q.get(), rr_dev, sc.get() + 1, d, s);
      vec_dot(r.get(), r.get(), d, part.get(), rr_next_dev, s);
      cg_direction(p.get(), r.get(), rr_next_dev, rr_dev, d, s);
      rr = read_scalar(rr_next_dev, s);
      slot = 2 - slot;
      ++iters;
    }
    RP_CUDA(cudaMemcpyAsync(x_out + static_cast<int64_t>(idx) * d, x.get(), sizeof(double) * d,
                            cudaMemcpyDeviceToDevice, s));
    RP_CUDA(cudaStreamSynchronize(s));
    run.iterations[idx] = iters;
    run.seconds[idx] = host_seconds_since(t_eval);
  }
  run.total_seconds = host_seconds_since(t_total);
}

// warm_ihs_path (baselines.cpp:164-224); x_out: d x T on the device.
void run_warm_ihs(rp_ctx* ctx, const double* b, const PathCfg& cfg, const SketchSpecC& spec, const Rho& rho,
                  double* x_out, BaselineRun& run) {
  cudaStream_t s = ctx->stream;
  const auto t_total = std::chrono::steady_clock::now();
  const OpView op = op_primal(ctx);
  const int64_t d = op.d;
  DBuf<double> sa(static_cast<size_t>(spec.m * d), s);
  sketch_apply(spec, op, sa.get(), s);
  allreduce(ctx, sa.get(), spec.m * d);
  GramOp gram;
  gram.ctx = ctx;
  gram.op = op;
  gram.allow_fused = true;
  DBuf<double> atb(static_cast<size_t>(d), s), x(static_cast<size_t>(d), s), xs(static_cast<size_t>(d), s),
      g(static_cast<size_t>(d), s), grad(static_cast<size_t>(d), s), pg(static_cast<size_t>(d), s),
      part(kDotParts, s), sc(2, s);
  DBuf<int> flag(1, s);
  op_apply_t(ctx, op, b, 1, atb.get(), true);
  vec_dot(atb.get(), atb.get(), d, part.get(), sc.get(), s);
  const double rhs_norm = std::sqrt(read_scalar(sc.get(), s));
  // P for the swept shifts, factored in batches (reshift per lambda, :189)
  const std::vector<size_t> order = descending_order(cfg.lambdas);
  const int64_t nn = spec.m < d ? spec.m : d;
  const int64_t per_batch =
      std::max<int64_t>(1, std::min<int64_t>(64, (int64_t{1} << 31) / std::max<int64_t>(1, nn * nn * 8)));
  run.setup_seconds = host_seconds_since(t_total);
  const double tau_nominal = 2.0 / (1.0 / rho.rho1 + 1.0 / rho.rho2);
  const double tol = cfg.epsilon * (rhs_norm > 0.0 ? rhs_norm : 1.0);
  const int cap = 1000;
  const size_t T = cfg.lambdas.size();
  run.iterations.assign(T, 0);
  run.seconds.assign(T, 0.0);
  fill(x.get(), d, 0.0, s);
  PrecondBatch P;
  P.col_stable = true;
  int64_t batch0 = -1;
  for (size_t pos = 0; pos < T; ++pos) {
    const size_t idx = order[pos];
    const double lam = cfg.lambdas[idx];
    const auto t_eval = std::chrono::steady_clock::now();
    if (batch0 < 0 || static_cast<int64_t>(pos) >= batch0 + P.L) {
      batch0 = static_cast<int64_t>(pos);
      std::vector<double> shifts;
      for (size_t q = pos; q < T && static_cast<int64_t>(shifts.size()) < per_batch; ++q)
        shifts.push_back(cfg.lambdas[order[q]]);
      P.build(ctx, sa.get(), nullptr, spec.m, d, shifts);
    }
    const PrecondBatch Pl = P.single(ctx, static_cast<int64_t>(pos) - batch0);
    double tau = tau_nominal;
    RP_CUDA(cudaMemcpyAsync(xs.get(), x.get(), sizeof(double) * d, cudaMemcpyDeviceToDevice, s));
    RP_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), s));
    int32_t iters = 0;
    bool retried = false;
    while (true) {
      gram.apply(xs.get(), 1, g.get());
      ihs_grad(g.get(), xs.get(), lam, atb.get(), d, grad.get(), s);
      vec_dot(grad.get(), grad.get(), d, part.get(), sc.get(), s);
      struct {
        double nrm2;
        int bad;
      } h{};
      RP_CUDA(cudaMemcpyAsync(&h.nrm2, sc.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
      RP_CUDA(cudaMemcpyAsync(&h.bad, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
      RP_CUDA(cudaStreamSynchronize(s));
      if (h.bad) {  // the previous step left a non-finite iterate (:201-208)
        if (retried) throw SolverFailure("warm_ihs_path: diverged twice, even at tau/2");
        retried = true;
        tau /= 2.0;
        RP_CUDA(cudaMemcpyAsync(xs.get(), x.get(), sizeof(double) * d, cudaMemcpyDeviceToDevice, s));
        RP_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), s));
        iters = 0;
        continue;
      }
      if (std::sqrt(h.nrm2) <= tol) break;
      if (iters >= cap) throw SolverFailure("warm_ihs_path: iteration cap reached");
      Pl.apply(ctx, grad.get(), d, 1, pg.get(), d);
      ihs_step(xs.get(), pg.get(), tau, d, flag.get(), s);
      ++iters;
    }
    RP_CUDA(cudaMemcpyAsync(x.get(), xs.get(), sizeof(double) * d, cudaMemcpyDeviceToDevice, s));
    RP_CUDA(cudaMemcpyAsync(x_out + static_cast<int64_t>(idx) * d, x.get(), sizeof(double) * d,
                            cudaMemcpyDeviceToDevice, s));
    RP_CUDA(cudaStreamSynchronize(s));
    run.iterations[idx] = iters;
    run.seconds[idx] = host_seconds_since(t_eval);
  }
  run.total_seconds = host_seconds_since(t_total);
}

// direct_path (baselines.cpp:80-118): G = A^T A once, then (G + lambda I)^{-1} A^T b
// for batches of lambdas (batched Cholesky + triangular inverse on the tensor cores).
void run_direct(rp_ctx* ctx, const double* b, const PathCfg& cfg, double* x_out, BaselineRun& run) {
  cudaStream_t s = ctx->stream;
  const auto t_total = std::chrono::steady_clock::now();
  const OpView op = op_primal(ctx);
  const int64_t d = op.d;
  require(static_cast<double>(d) * d * 8.0 <= 32.0 * (1ull << 30), "direct_path: A^T A exceeds 32 GiB");
  DBuf<double> G;
  if (!op.sparse) {
    GramOp gram;
    gram.ctx = ctx;
    gram.op = op;
    gram.build_matrix();
    G = std::move(gram.G);
  } else {  // apply_transpose(a, apply(a, I)) (baselines.cpp:93), in column blocks
    G.alloc(static_cast<size_t>(d * d), s);
    GramOp gram;
    gram.ctx = ctx;
    gram.op = op;
    const int64_t blk = std::min<int64_t>(d, 1024);
    DBuf<double> eye(static_cast<size_t>(d * blk), s);
    for (int64_t c0 = 0; c0 < d; c0 += blk) {
      const int64_t cb = std::min(blk, d - c0);
      identity_block(eye.get(), d, cb, c0, s);
      gram.apply(eye.get(), cb, G.get() + c0 * d);
    }
  }
  DBuf<double> atb(static_cast<size_t>(d), s);
  op_apply_t(ctx, op, b, 1, atb.get(), true);
  RP_CUDA(cudaStreamSynchronize(s));
  run.setup_seconds = host_seconds_since(t_total);
  const int64_t T = static_cast<int64_t>(cfg.lambdas.size());
  const int64_t per = std::max<int64_t>(1, std::min<int64_t>(T, (int64_t{1} << 31) / std::max<int64_t>(1, d * d * 8)));
  run.iterations.assign(static_cast<size_t>(T), 0);
  run.seconds.assign(static_cast<size_t>(T), 0.0);
  DBuf<double> h(static_cast<size_t>(per * d * d), s), inv(static_cast<size_t>(per * d * d), s),
      shifts(static_cast<size_t>(per), s);
  for (int64_t t0 = 0; t0 < T; t0 += per) {
    const auto t_eval = std::chrono::steady_clock::now();
    const int64_t tc = std::min(per, T - t0);
    RP_CUDA(cudaMemcpyAsync(shifts.get(), cfg.lambdas.data() + t0, sizeof(double) * tc, cudaMemcpyHostToDevice, s));
    shifted_copies(G.get(), d, shifts.get(), tc, h.get(), s);
    try {
      spd_inverse_batched(h.get(), d, d, d * d, tc, inv.get(), d, d * d, s);
    } catch (const FactorFailure&) {
      throw SolverFailure("direct_path: Cholesky factorization failed");
    }
    GemmArgs gx;  // x_t = (G + lambda_t I)^{-1} A^T b
    gx.m = d;
    gx.n = 1;
    gx.k = d;
    gx.a = inv.get();
    gx.lda = d;
    gx.stride_a = d * d;
    gx.b = atb.get();
    gx.ldb = d;
    gx.stride_b = 0;
    gx.c = x_out + t0 * d;
    gx.ldc = d;
    gx.stride_c = d;
    gx.batch = tc;
    dgemm(gx, s);
    RP_CUDA(cudaStreamSynchronize(s));
    const double secs = host_seconds_since(t_eval) / static_cast<double>(tc);
    for (int64_t t = t0; t < t0 + tc; ++t) run.seconds[static_cast<size_t>(t)] = secs;
  }
  run.total_seconds = host_seconds_since(t_total);
}

// ---- cuSOLVER, loaded at run time (svd_path's dense QR and SVD) -------------
// A plain library factorization, like cuBLAS for a plain GEMM: svd_path is a
// comparison baseline, not the hot path.  Loaded on first use so the library
// keeps no link-time dependency on a specific cuSOLVER.
struct CusolverApi {
  void* lib = nullptr;
  decltype(&cusolverDnCreate) Create = nullptr;
  decltype(&cusolverDnDestroy) Destroy = nullptr;
  decltype(&cusolverDnSetStream) SetStream = nullptr;
  decltype(&cusolverDnDgeqrf_bufferSize) GeqrfSize = nullptr;
  decltype(&cusolverDnDgeqrf) Geqrf = nullptr;
  decltype(&cusolverDnDormqr_bufferSize) OrmqrSize = nullptr;
  decltype(&cusolverDnDormqr) Ormqr = nullptr;
  decltype(&cusolverDnDgesvd_bufferSize) GesvdSize = nullptr;
  decltype(&cusolverDnDgesvd) Gesvd = nullptr;
};

CusolverApi& cusolver() {
  static CusolverApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libcusolver.so.11", "libcusolver.so", "/usr/local/cuda/lib64/libcusolver.so.11"}) {
      api.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.lib) break;
    }
    if (!api.lib) return;
    auto sym = [](const char* n) { return dlsym(api.lib, n); };
    api.Create = reinterpret_cast<decltype(api.Create)>(sym("cusolverDnCreate"));
    api.Destroy = reinterpret_cast<decltype(api.Destroy)>(sym("cusolverDnDestroy"));
    api.SetStream = reinterpret_cast<decltype(api.SetStream)>(sym("cusolverDnSetStream"));
    api.GeqrfSize = reinterpret_cast<decltype(api.GeqrfSize)>(sym("cusolverDnDgeqrf_bufferSize"));
    api.Geqrf = reinterpret_cast<decltype(api.Geqrf)>(sym("cusolverDnDgeqrf"));
    api.OrmqrSize = reinterpret_cast<decltype(api.OrmqrSize)>(sym("cusolverDnDormqr_bufferSize"));
    api.Ormqr = reinterpret_cast<decltype(api.Ormqr)>(sym("cusolverDnDormqr"));
    api.GesvdSize = reinterpret_cast<decltype(api.GesvdSize)>(sym("cusolverDnDgesvd_bufferSize"));
    api.Gesvd = reinterpret_cast<decltype(api.Gesvd)>(sym("cusolverDnDgesvd"));
  });
  if (!api.lib || !api.Create || !api.Geqrf || !api.Ormqr || !api.Gesvd)
    throw CudaFailure("svd_path: cuSOLVER (libcusolver.so.11) could not be loaded");
  return api;
}

void cusolver_check(cusolverStatus_t st, const char* what) {
  if (st != CUSOLVER_STATUS_SUCCESS) throw CudaFailure(std::string(what) + ": cuSOLVER status " + std::to_string(st));
}

// svd_path (baselines.cpp:51-78): one thin SVD of A, then for every lambda
// x = V diag(sigma / (sigma^2 + lambda)) U^T b.  The thin SVD is formed as a
// Householder QR of A (or of A^T when n < d) followed by the SVD of the small
// triangular factor -- A = Q R, R = U_R S V^T, so U^T b = U_R^T (Q^T b)[0:d] --
// which is backward stable in A like the reference's JacobiSVD.  All T
// solutions come out of one GEMM V Z, Z = the scaled r x T matrix.
void run_svd(rp_ctx* ctx, const double* b, const PathCfg& cfg, double* x_out, BaselineRun& run) {
  cudaStream_t s = ctx->stream;
  const auto t_total = std::chrono::steady_clock::now();
  require(ctx->world == 1, "svd_path: needs the whole operator on one device");
  const OpView op = op_primal(ctx);
  const int64_t n = op.n_loc, d = op.d, r = std::min(n, d);
  const int64_t T = static_cast<int64_t>(cfg.lambdas.size());
  require(n < (int64_t{1} << 31) && d < (int64_t{1} << 31) && n * d * 8.0 <= 64.0 * (1ull << 30),
          "svd_path: A exceeds the dense factorization limits");
  CusolverApi& cs = cusolver();
  cusolverDnHandle_t h = nullptr;
  cusolver_check(cs.Create(&h), "cusolverDnCreate");
  struct HandleGuard {
    CusolverApi& cs;
    cusolverDnHandle_t h;
    ~HandleGuard() { cs.Destroy(h); }
  } guard{cs, h};
  cusolver_check(cs.SetStream(h, s), "cusolverDnSetStream");
  const bool tall = n >= d;
  // F: the matrix whose QR is taken -- A (n x d) when tall, else A^T (d x n).
  const int64_t fm = tall ? n : d, fn = r;
  DBuf<double> F(static_cast<size_t>(fm * fn), s);
  if (tall) {
    densify(op, F.get(), n, s);
  } else {
    DBuf<double> a(static_cast<size_t>(n * d), s);
    densify(op, a.get(), n, s);
    transpose(a.get(), n, d, n, F.get(), d, s);
  }
  DBuf<double> tau(static_cast<size_t>(r), s);
  DBuf<int> info(1, s);
  int lwork = 0;
  cusolver_check(cs.GeqrfSize(h, static_cast<int>(fm), static_cast<int>(fn), F.get(), static_cast<int>(fm), &lwork),
                 "geqrf_bufferSize");
  int lw_svd = 0;
  cusolver_check(cs.GesvdSize(h, static_cast<int>(r), static_cast<int>(r), &lw_svd), "gesvd_bufferSize");
  DBuf<double> work(static_cast<size_t>(std::max(lwork, lw_svd) + 1), s);
  cusolver_check(cs.Geqrf(h, static_cast<int>(fm), static_cast<int>(fn), F.get(), static_cast<int>(fm), tau.get(),
                          work.get(), std::max(lwork, lw_svd), info.get()),
                 "geqrf");
  // the r x r triangle: R (tall) or R^T (wide: A = R^T Q^T)
  DBuf<double> tri(static_cast<size_t>(r * r), s), R(static_cast<size_t>(r * r), s);
  upper_triangle(F.get(), fm, r, tall ? R.get() : tri.get(), s);
  if (!tall) transpose(tri.get(), r, r, r, R.get(), r, s);
  DBuf<double> sigma(static_cast<size_t>(r), s), U(static_cast<size_t>(r * r), s), VT(static_cast<size_t>(r * r), s),
      rwork(static_cast<size_t>(r), s);
  cusolver_check(cs.Gesvd(h, 'A', 'A', static_cast<int>(r), static_cast<int>(r), R.get(), static_cast<int>(r),
                          sigma.get(), U.get(), static_cast<int>(r), VT.get(), static_cast<int>(r), work.get(),
                          std::max(lwork, lw_svd), rwork.get(), info.get()),
                 "gesvd");
  int hinfo = 0;
  RP_CUDA(cudaMemcpyAsync(&hinfo, info.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  // U^T b: tall -> U_R^T (Q^T b)[0:r]; wide -> U^T b (A = U S (Q W)^T)
  DBuf<double> qb(static_cast<size_t>(n), s), utb(static_cast<size_t>(r), s);
  RP_CUDA(cudaMemcpyAsync(qb.get(), b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  if (tall) {
    int lw_q = 0;
    cusolver_check(cs.OrmqrSize(h, CUBLAS_SIDE_LEFT, CUBLAS_OP_T, static_cast<int>(n), 1, static_cast<int>(r), F.get(),
                                static_cast<int>(n), tau.get(), qb.get(), static_cast<int>(n), &lw_q),
                   "ormqr_bufferSize");
    DBuf<double> wq(static_cast<size_t>(lw_q + 1), s);
    cusolver_check(cs.Ormqr(h, CUBLAS_SIDE_LEFT, CUBLAS_OP_T, static_cast<int>(n), 1, static_cast<int>(r), F.get(),
                            static_cast<int>(n), tau.get(), qb.get(), static_cast<int>(n), wq.get(), lw_q, info.get()),
                   "ormqr");
  }
  {
    GemmArgs g;  // utb = U^T qb[0:r]
    g.opa = Op::T;
    g.m = r;
    g.n = 1;
    g.k = r;
    g.a = U.get();
    g.lda = r;
    g.b = qb.get();
    g.ldb = r;
    g.c = utb.get();
    g.ldc = r;
    dgemm(g, s);
  }
  RP_CUDA(cudaStreamSynchronize(s));
  if (hinfo != 0) throw SolverFailure("svd_path: the SVD did not converge");
  run.setup_seconds = host_seconds_since(t_total);
  const auto t_eval = std::chrono::steady_clock::now();
  DBuf<double> lam(static_cast<size_t>(T), s), Z(static_cast<size_t>(r * T), s);
  RP_CUDA(cudaMemcpyAsync(lam.get(), cfg.lambdas.data(), sizeof(double) * T, cudaMemcpyHostToDevice, s));
  svd_scale(sigma.get(), utb.get(), r, lam.get(), T, Z.get(), s);
  GemmArgs g;  // x = V_R Z (tall) or W Z, then Q (wide)
  g.opa = Op::T;
  g.m = r;
  g.n = T;
  g.k = r;
  g.a = VT.get();
  g.lda = r;
  g.b = Z.get();
  g.ldb = r;
  g.ldc = d;
  if (tall) {
    g.c = x_out;
    dgemm(g, s);
  } else {
    fill(x_out, d * T, 0.0, s);
    g.c = x_out;
    dgemm(g, s);
    int lw_q = 0;
    cusolver_check(cs.OrmqrSize(h, CUBLAS_SIDE_LEFT, CUBLAS_OP_N, static_cast<int>(d), static_cast<int>(T),
                                static_cast<int>(r), F.get(), static_cast<int>(d), tau.get(), x_out,
                                static_cast<int>(d), &lw_q),
                   "ormqr_bufferSize");
    DBuf<double> wq(static_cast<size_t>(lw_q + 1), s);
    cusolver_check(cs.Ormqr(h, CUBLAS_SIDE_LEFT, CUBLAS_OP_N, static_cast<int>(d), static_cast<int>(T),
                            static_cast<int>(r), F.get(), static_cast<int>(d), tau.get(), x_out, static_cast<int>(d),
                            wq.get(), lw_q, info.get()),
                   "ormqr");
  }
  RP_CUDA(cudaStreamSynchronize(s));
  const double secs = host_seconds_since(t_eval) / static_cast<double>(std::max<int64_t>(T, 1));
  run.iterations.assign(static_cast<size_t>(T), 0);
  run.seconds.assign(static_cast<size_t>(T), secs);
  run.total_seconds = host_seconds_since(t_total);
}

// adaptive_sketch_dim (adaptive.cpp:53-135): sketched Newton steps at
// lambda_min with Armijo backtracking, doubling m under a fresh seed when the
// progress measure d.grad stalls.  Every vector lives on the device; the
// objective is one pass over the operator plus two dots.
void run_adaptive(rp_ctx* ctx, const double* b, double lambda_min, const rp_adaptive_config& cfg,
                  const SketchSpecC& tmpl, const double* x0, double* x_out, rp_adaptive_result& res,
                  std::vector<rp_adaptive_step>& trace) {
  cudaStream_t s = ctx->stream;
  const OpView op = op_primal(ctx);
  const int64_t d = op.d, nl = op.n_loc;
  // AdaptiveConfig::validate / initial_m / cap_m (adaptive.cpp:19-37)
  const int64_t m0 = cfg.m_initial > 0 ? cfg.m_initial : std::max<int64_t>(16, d / 64);
  const int64_t m_cap = cfg.m_cap > 0 ? cfg.m_cap : d;
  require(lambda_min > 0.0, "adaptive: lambda_min must be positive");
  require(cfg.gamma1 > 0.0 && cfg.gamma1 < 1.0, "adaptive: gamma1 not in (0,1)");
  require(cfg.gamma2 > 0.0 && cfg.gamma2 < 1.0, "adaptive: gamma2 not in (0,1)");
  require(cfg.gamma3 > 0.0 && cfg.gamma3 < 1.0, "adaptive: gamma3 not in (0,1)");
  require(cfg.epsilon > 0.0, "adaptive: epsilon must be positive");
  require(m0 >= 1, "adaptive: m_initial must be >= 1");
  require(m_cap <= d, "adaptive: m_cap must not exceed d");
  require(m0 <= m_cap, "adaptive: m_initial above m_cap");
  require(cfg.iteration_cap >= 1, "adaptive: iteration cap must be >= 1");
  require(tmpl.n == op.n_global, "sketch_apply: spec.n must match A.rows");
  GramOp gram;
  gram.ctx = ctx;
  gram.op = op;
  gram.allow_fused = true;
  auto vec = [&](int64_t n) { return DBuf<double>(static_cast<size_t>(std::max<int64_t>(n, 1)), s); };
  DBuf<double> atb = vec(d), x = vec(d), xt = vec(d), xn = vec(d), g = vec(d), grad = vec(d), gradn = vec(d),
               dir = vec(d), dirn = vec(d), r = vec(nl), part(kDotParts, s), sc(4, s);
  DBuf<int> flag(1, s);
  op_apply_t(ctx, op, b, 1, atb.get(), true);
  auto dot = [&](const double* u, const double* v, int64_t n, bool reduce) {
    vec_dot(u, v, n, part.get(), sc.get(), s);
    if (reduce) allreduce(ctx, sc.get(), 1);
    return read_scalar(sc.get(), s);
  };
  auto objective = [&](const double* xv) {  // 0.5 ||A x - b||^2 + 0.5 lambda ||x||^2
    op_apply(ctx, op, xv, 1, r.get());
    residual_in_place(r.get(), b, nl, s);
    const double rr = dot(r.get(), r.get(), nl, true);
    const double xx = dot(xv, xv, d, false);
    return 0.5 * rr + 0.5 * lambda_min * xx;
  };
  auto gradient = [&](const double* xv, double* out) {  // gram_apply(a, x) + lambda x - atb
    gram.apply(xv, 1, g.get());
    ihs_grad(g.get(), xv, lambda_min, atb.get(), d, out, s);
  };
  auto axpy_to = [&](const double* xv, double step, const double* dv, double* out) {  // out = x - step d
    RP_CUDA(cudaMemcpyAsync(out, xv, sizeof(double) * d, cudaMemcpyDeviceToDevice, s));
    ihs_step(out, dv, step, d, flag.get(), s);
  };
  PrecondBatch P;
  DBuf<double> sa;
  auto make_pre = [&](int64_t m, int resample) {
    SketchSpecC spec = tmpl;
    spec.m = m;
    spec.seed = tmpl.seed + 0x9e3779b97f4a7c15ull * static_cast<uint64_t>(resample);
    if (spec.kind == kIdentity) spec.m = spec.n;
    if (spec.kind == kSjlt && spec.m % spec.s != 0) spec.m += spec.s - spec.m % spec.s;
    validate_spec(spec);
    sa.alloc(static_cast<size_t>(spec.m * d), s);
    sketch_apply(spec, op, sa.get(), s);
    allreduce(ctx, sa.get(), spec.m * d);
    P.build(ctx, sa.get(), nullptr, spec.m, d, {lambda_min});
  };
  res = rp_adaptive_result{};
  res.m = m0;
  if (x0)
    RP_CUDA(cudaMemcpyAsync(x.get(), x0, sizeof(double) * d, cudaMemcpyDeviceToDevice, s));
  else
    fill(x.get(), d, 0.0, s);
  make_pre(res.m, 0);
  gradient(x.get(), grad.get());
  P.apply(ctx, grad.get(), d, 1, dir.get(), d);
  double progress = dot(dir.get(), grad.get(), d, false);
  int loop_guard = 0;
  while (progress >= cfg.epsilon) {
    if (res.iterations >= cfg.iteration_cap || ++loop_guard > 4 * cfg.iteration_cap) break;
    // armijo_step (adaptive.cpp:39-51)
    require(progress > 0.0, "armijo: direction is not a descent direction");
    const double fx = objective(x.get());
    double step = 1.0;
    bool found = false;
    for (int j = 0; j <= 50; ++j) {
      axpy_to(x.get(), step, dir.get(), xt.get());
      if (objective(xt.get()) <= fx - cfg.gamma2 * step * progress) {
        found = true;
        break;
      }
      step *= cfg.gamma1;
    }
    if (!found) throw SolverFailure("armijo: no acceptable step within 50 backtracks");
    axpy_to(x.get(), step, dir.get(), xn.get());
    gradient(xn.get(), gradn.get());
    P.apply(ctx, gradn.get(), d, 1, dirn.get(), d);
    const double progress_next = dot(dirn.get(), gradn.get(), d, false);
    rp_adaptive_step rec{};
    rec.m = res.m;
    rec.f_before = objective(x.get());
    rec.f_after = objective(xn.get());
    rec.step = step;
    rec.progress = progress;
    if (progress_next >= cfg.gamma3 * progress && res.m < m_cap) {
      res.m = std::min(2 * res.m, m_cap);
      ++res.doublings;
      rec.doubled = 1;
      make_pre(res.m, res.doublings);
      gradient(x.get(), grad.get());
      P.apply(ctx, grad.get(), d, 1, dir.get(), d);
      progress = dot(dir.get(), grad.get(), d, false);
    } else {
      std::swap(x, xn);
      std::swap(grad, gradn);
      std::swap(dir, dirn);
      progress = progress_next;
      ++res.iterations;
    }
    trace.push_back(rec);
  }
  res.converged = progress < cfg.epsilon ? 1 : 0;
  res.stalled_at_cap = (!res.converged && res.m >= m_cap) ? 1 : 0;
  res.trace_len = static_cast<int64_t>(trace.size());
  RP_CUDA(cudaMemcpyAsync(x_out, x.get(), sizeof(double) * d, cudaMemcpyDeviceToDevice, s));
  RP_CUDA(cudaStreamSynchronize(s));
}

void finish_baseline(const BaselineRun& run, int32_t* iterations, double* seconds, double* setup_total) {
  if (iterations) std::copy(run.iterations.begin(), run.iterations.end(), iterations);
  if (seconds) std::copy(run.seconds.begin(), run.seconds.end(), seconds);
  if (setup_total) {
    setup_total[0] = run.setup_seconds;
    setup_total[1] = run.total_seconds;
  }
}

}  // namespace rpb

rp_status rp_warm_cg_path(rp_ctx* ctx, const double* b, const rp_path_config* cfgp, double* x_out, int where,
                          int32_t* iterations, double* seconds, double* setup_total) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    const PathCfg cfg = to_cfg(cfgp);
    cfg.validate();
    const OpView op = op_primal(ctx);
    InBuf bb(b, static_cast<size_t>(op.n_loc), where, ctx->stream);
    OutBuf out(x_out, static_cast<size_t>(op.d * cfg.lambdas.size()), where, ctx->stream);
    BaselineRun run;
    run_warm_cg(ctx, bb.ptr, cfg, out.dev, run);
    out.finish();
    finish_baseline(run, iterations, seconds, setup_total);
  });
}

rp_status rp_warm_ihs_path(rp_ctx* ctx, const double* b, const rp_path_config* cfgp, const rp_sketch_spec* specp,
                           const rp_rho_bounds* rhop, double* x_out, int where, int32_t* iterations, double* seconds,
                           double* setup_total) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    const PathCfg cfg = to_cfg(cfgp);
    cfg.validate();
    const Rho rho = to_rho(rhop);
    rho_validate(rho);
    const SketchSpecC spec = to_spec(specp);
    const OpView op = op_primal(ctx);
    require(spec.n == op.n_global, "warm_ihs_path: spec.n must equal A.rows");
    validate_spec(spec);
    InBuf bb(b, static_cast<size_t>(op.n_loc), where, ctx->stream);
    OutBuf out(x_out, static_cast<size_t>(op.d * cfg.lambdas.size()), where, ctx->stream);
    BaselineRun run;
    run_warm_ihs(ctx, bb.ptr, cfg, spec, rho, out.dev, run);
    out.finish();
    finish_baseline(run, iterations, seconds, setup_total);
  });
}

rp_status rp_adaptive_sketch_dim(rp_ctx* ctx, const double* b, double lambda_min, const rp_adaptive_config* cfg,
                                 const rp_sketch_spec* spec_template, const double* x0, double* x_out, int where,
                                 rp_adaptive_result* result, rp_adaptive_step* trace, int64_t trace_cap) {
  if (!ctx || !cfg || !result) return RP_EINVAL;
  return guarded(ctx, [&] {
    const SketchSpecC tmpl = to_spec(spec_template);
    const OpView op = op_primal(ctx);
    require(trace_cap >= 0, "adaptive: negative trace capacity");
    InBuf bb(b, static_cast<size_t>(op.n_loc), where, ctx->stream);
    InBuf xb(x0, x0 ? static_cast<size_t>(op.d) : 0, where, ctx->stream);
    OutBuf out(x_out, static_cast<size_t>(op.d), where, ctx->stream);
    std::vector<rp_adaptive_step> tr;
    run_adaptive(ctx, bb.ptr, lambda_min, *cfg, tmpl, x0 ? xb.ptr : nullptr, out.dev, *result, tr);
    out.finish();
    if (trace)
      for (int64_t i = 0; i < std::min<int64_t>(trace_cap, static_cast<int64_t>(tr.size())); ++i) trace[i] = tr[i];
  });
}

rp_status rp_svd_path(rp_ctx* ctx, const double* b, const rp_path_config* cfgp, double* x_out, int where,
                      double* seconds, double* setup_total) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    const PathCfg cfg = to_cfg(cfgp);
    cfg.validate();
    const OpView op = op_primal(ctx);
    InBuf bb(b, static_cast<size_t>(op.n_loc), where, ctx->stream);
    OutBuf out(x_out, static_cast<size_t>(op.d * cfg.lambdas.size()), where, ctx->stream);
    BaselineRun run;
    run_svd(ctx, bb.ptr, cfg, out.dev, run);
    out.finish();
    finish_baseline(run, nullptr, seconds, setup_total);
  });
}

rp_status rp_direct_path(rp_ctx* ctx, const double* b, const rp_path_config* cfgp, double* x_out, int where,
                         double* seconds, double* setup_total) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    const PathCfg cfg = to_cfg(cfgp);
    cfg.validate();
    const OpView op = op_primal(ctx);
    InBuf bb(b, static_cast<size_t>(op.n_loc), where, ctx->stream);
    OutBuf out(x_out, static_cast<size_t>(op.d * cfg.lambdas.size()), where, ctx->stream);
    BaselineRun run;
    run_direct(ctx, bb.ptr, cfg, out.dev, run);
    out.finish();
    finish_baseline(run, nullptr, seconds, setup_total);
  });
}

// ---- plug-in envelope (derive_rho, ridgepath_main.cpp:218-279) -------------------

static void to_c_rho(const RhoResult& r, rp_rho_bounds* out) {
  out->rho1 = r.rho1;
  out->rho2 = r.rho2;
  out->provenance = r.provenance;
}

rp_status rp_derive_rho(rp_ctx* ctx, const rp_sketch_spec* specp, int transpose_op, double lambda_min,
                        double lambda_max, rp_rho_bounds* out, rp_spectrum_info* info) {
  if (!ctx || !out) return RP_EINVAL;
  return guarded(ctx, [&] {
    const SketchSpecC spec = to_spec(specp);
    require(lambda_min > 0.0 && lambda_max >= lambda_min, "derive_rho: bad lambda range");
    rp_spectrum_info inf{};
    const double lambda0 = std::sqrt(lambda_min * lambda_max);
    inf.lambda0 = lambda0;
    if (spec.kind == RP_SKETCH_IDENTITY) {
      to_c_rho(RhoResult{}, out);
      if (info) *info = inf;
      return;
    }
    const OpView op = transpose_op ? op_dual(ctx) : op_primal(ctx);
    validate_spec(spec);
    require(op.n_global == spec.n, "sketch_apply: spec.n must match A.rows");
    cudaStream_t s = ctx->stream;
    DBuf<double> sa(static_cast<size_t>(spec.m * op.d), s);
    sketch_apply(spec, op, sa.get(), s);
    allreduce(ctx, sa.get(), spec.m * op.d);
    const SketchedSpectrum sp = sketched_spectrum(sa.get(), spec.m, op.d, lambda0, s);
    double de = 0.0, dn = 0.0;
    const RhoResult r = envelope_from_spectrum(spec.kind, spec.m, spec.n, sp, lambda0, &de, &dn);
    to_c_rho(r, out);
    inf.effective_dimension = de;
    inf.sigma_max_sq = sp.sigma_max_sq;
    inf.dnorm_sq = dn;
    inf.lanczos_steps = sp.lanczos_steps;
    if (info) *info = inf;
  });
}

rp_status rp_effective_dimension(const double* sigma, int64_t count, double lambda0, double* out) {
  return guarded(nullptr, [&] {
    require(out != nullptr && (sigma != nullptr || count == 0), "effective_dimension: null buffer");
    *out = effective_dimension(sigma, count, lambda0);
  });
}

rp_status rp_rho_gaussian(double rho, double eta, double dnorm_sq, int64_t m, rp_rho_bounds* out,
                          double* success_probability) {
  return guarded(nullptr, [&] {
    require(out != nullptr, "rho_gaussian: null output");
    std::optional<int64_t> mm;
    if (m > 0) mm = m;
    const RhoResult r = rho_gaussian(rho, eta, dnorm_sq, mm);
    to_c_rho(r, out);
    if (success_probability) *success_probability = r.success_probability ? *r.success_probability : std::nan("");
  });
}

rp_status rp_rho_srht(double rho, double dnorm_sq, int64_t n, double de, rp_rho_bounds* out, int64_t* recommended_m) {
  return guarded(nullptr, [&] {
    require(out != nullptr, "rho_srht: null output");
    std::optional<std::pair<int64_t, double>> nd;
    if (n > 0) nd = std::make_pair(n, de);
    const RhoResult r = rho_srht(rho, dnorm_sq, nd);
    to_c_rho(r, out);
    if (recommended_m) *recommended_m = r.recommended_m ? *r.recommended_m : -1;
  });
}

rp_status rp_rho_sjlt(double eps, double alpha, double delta, double de, rp_rho_bounds* out, int64_t* recommended_m,
                      int32_t* recommended_s) {
  return guarded(nullptr, [&] {
    require(out != nullptr, "rho_sjlt: null output");
    std::optional<std::tuple<double, double, double>> adde;
    if (alpha > 0.0) adde = std::make_tuple(alpha, delta, de);
    const RhoResult r = rho_sjlt(eps, adde);
    to_c_rho(r, out);
    if (recommended_m) *recommended_m = r.recommended_m ? *r.recommended_m : -1;
    if (recommended_s) *recommended_s = r.recommended_s ? *r.recommended_s : -1;
  });
}

rp_status rp_draw_u64(rp_ctx* ctx, uint64_t seed, uint64_t skip, int64_t count, uint64_t* out, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    require(count >= 0, "draw: negative count");
    DBuf<uint64_t> d(static_cast<size_t>(std::max<int64_t>(count, 1)), ctx->stream);
    draw_words(seed, skip, count, WordMode::Raw, d.get(), ctx->stream);
    copy_out(out, d.get(), count, where, ctx->stream);
  });
}

rp_status rp_draw_uniform01(rp_ctx* ctx, uint64_t seed, int64_t count, double* out, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    require(count >= 0, "draw: negative count");
    DBuf<double> d(static_cast<size_t>(std::max<int64_t>(count, 1)), ctx->stream);
    draw_words(seed, 0, count, WordMode::Uniform01, d.get(), ctx->stream);
    copy_out(out, d.get(), count, where, ctx->stream);
  });
}

rp_status rp_draw_sign(rp_ctx* ctx, uint64_t seed, int64_t count, double* out, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    require(count >= 0, "draw: negative count");
    DBuf<double> d(static_cast<size_t>(std::max<int64_t>(count, 1)), ctx->stream);
    draw_words(seed, 0, count, WordMode::Sign, d.get(), ctx->stream);
    copy_out(out, d.get(), count, where, ctx->stream);
  });
}

rp_status rp_draw_uniform_index(rp_ctx* ctx, uint64_t seed, uint64_t bound, int64_t count, uint64_t* out, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    require(count >= 0, "draw: negative count");
    DBuf<uint64_t> d(static_cast<size_t>(std::max<int64_t>(count, 1)), ctx->stream);
    draw_uniform_index(seed, bound, count, d.get(), ctx->stream);
    copy_out(out, d.get(), count, where, ctx->stream);
  });
}

rp_status rp_draw_normals(rp_ctx* ctx, uint64_t seed, int64_t first, int64_t count, double scale, double* out,
                          int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    require(count >= 0 && first >= 0, "draw: negative count");
    if (count == 0) return;
    DBuf<uint64_t> st(312, ctx->stream);
    DBuf<int64_t> cur(1, ctx->stream);
    DBuf<double> d(static_cast<size_t>(count), ctx->stream);
    GaussRows g;
    g.d_states = st.get();
    g.d_cursor = cur.get();
    gauss_rows_init(seed, 1, first, 0, g, ctx->stream);
    gauss_rows_next(g, count, scale, d.get(), count, ctx->stream);
    copy_out(out, d.get(), count, where, ctx->stream);
  });
}

rp_status rp_gaussian_window(rp_ctx* ctx, uint64_t seed, int64_t m, int64_t n, int64_t r0, int64_t rc, int64_t j0,
                             int64_t jc, double* out, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    require(m >= 1 && n >= 1 && r0 >= 0 && rc >= 0 && j0 >= 0 && jc >= 0 && r0 + rc <= m && j0 + jc <= n,
            "gaussian window: out of range");
    if (rc == 0 || jc == 0) return;
    DBuf<uint64_t> st(static_cast<size_t>(rc) * 312, ctx->stream);
    DBuf<int64_t> cur(static_cast<size_t>(rc), ctx->stream);
    DBuf<double> d(static_cast<size_t>(rc * jc), ctx->stream);
    GaussRows g;
    g.d_states = st.get();
    g.d_cursor = cur.get();
    gauss_rows_init(seed, rc, r0 * n + j0, n, g, ctx->stream);
    gauss_rows_next(g, jc, 1.0 / std::sqrt(static_cast<double>(m)), d.get(), jc, ctx->stream);
    copy_out(out, d.get(), rc * jc, where, ctx->stream);
  });
}

rp_status rp_count_draws(rp_ctx* ctx, const rp_sketch_spec* specp, int64_t* h_out, double* sign_out, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    const SketchSpecC spec = to_spec(specp);
    validate_spec(spec);
    require(spec.kind == kCountSketch || spec.kind == kSjlt, "count draws: not a CountSketch/SJLT spec");
    const int blocks = spec.kind == kSjlt ? spec.s : 1;
    const double entry = spec.kind == kSjlt ? 1.0 / std::sqrt(static_cast<double>(spec.s)) : 1.0;
    const int64_t total = spec.n * blocks;
    DBuf<int32_t> h(static_cast<size_t>(total), ctx->stream);
    DBuf<double> sg(static_cast<size_t>(total), ctx->stream);
    draw_count(spec.seed, spec.n, spec.m / blocks, blocks, entry, h.get(), sg.get(), ctx->stream);
    copy_out_i64(h_out, h.get(), total, where, ctx->stream);
    copy_out(sign_out, sg.get(), total, where, ctx->stream);
  });
}

rp_status rp_srht_draws(rp_ctx* ctx, const rp_sketch_spec* specp, double* signs_out, int64_t* rows_out, int where) {
  if (!ctx) return RP_EINVAL;
  return guarded(ctx, [&] {
    const SketchSpecC spec = to_spec(specp);
    validate_spec(spec);
    require(spec.kind == kSrht, "srht draws: not an SRHT spec");
    DBuf<double> sg(static_cast<size_t>(spec.n), ctx->stream);
    DBuf<int64_t> rows(static_cast<size_t>(spec.m), ctx->stream);
    draw_srht(spec.seed, spec.n, spec.m, sg.get(), rows.get(), ctx->stream);
    copy_out(signs_out, sg.get(), spec.n, where, ctx->stream);
    copy_out(rows_out, rows.get(), spec.m, where, ctx->stream);
  });
}

int rp_mt_selfcheck(uint64_t seed, uint64_t offset) {
  // Outputs offset..offset+3 from the jumped window must equal direct
  // generation; for large offsets "direct" starts from an independent jump to
  // offset - 1000 followed by 1000 ordinary steps.
  try {
    mt::init_tables();
    using W = std::vector<uint64_t>;
    auto step_outputs = [](const W& window, int64_t skip, int count) {
      W x(window);
      W out;
      for (int64_t k = 0; static_cast<int64_t>(out.size()) < count; ++k) {
        const uint64_t y = (x[k] & mt::kUpper) | (x[k + 1] & mt::kLower);
        x.push_back(x[k + mt::kM] ^ (y >> 1) ^ ((y & 1ULL) ? mt::kMatrixA : 0ULL));
        if (k >= skip) {
          uint64_t v = x.back();
          v ^= (v >> 29) & 0x5555555555555555ULL;
          v ^= (v << 17) & 0x71D67FFFEDA60000ULL;
          v ^= (v << 37) & 0xFFF7EEE000000000ULL;
          v ^= (v >> 43);
          out.push_back(v);
        }
      }
      return out;
    };
    uint64_t w0[mt::kN], w1[mt::kN];
    mt::seed_window(seed, w0);
    mt::host_jump(w0, mt::xpow(offset), w1);
    const W got = step_outputs(W(w1, w1 + mt::kN), 0, 4);
    W want(4);
    if (offset <= (uint64_t{1} << 22)) {
      mt::host_outputs(seed, offset, 4, want.data());
    } else {
      uint64_t w2[mt::kN];
      mt::host_jump(w0, mt::xpow(offset - 1000), w2);
      want = step_outputs(W(w2, w2 + mt::kN), 1000, 4);
    }
    return got == want ? 0 : 1;
  } catch (...) {
    return 2;
  }
}

// ---- data formats either side of the path (data_io.cpp) ----------------------

namespace {

// parse_real (data_io.cpp:23-39): std::stod semantics -- strtod on the whole
// token, ERANGE (overflow or underflow) is "out of range", then finite only.
double libsvm_real(const std::string& tok, int64_t line, int64_t col) {
  auto fail = [&](const std::string& what) -> double {
    throw ParseFailure("line " + std::to_string(line) + ", column " + std::to_string(col) + ": " + what, line, col);
  };
  const char* b = tok.c_str();
  char* end = nullptr;
  errno = 0;
  const double v = std::strtod(b, &end);
  if (end == b) return fail("malformed number '" + tok + "'");
  if (errno == ERANGE) return fail("number out of range '" + tok + "'");
  if (static_cast<size_t>(end - b) != tok.size()) return fail("trailing characters in number '" + tok + "'");
  if (!std::isfinite(v)) return fail("non-finite value '" + tok + "'");
  return v;
}

struct Libsvm {
  std::vector<int64_t> offsets{0}, cols;
  std::vector<double> values, labels;
  int64_t max_index = 0;
};

// parse_libsvm (data_io.cpp:50-127): one record per line; '#' starts a
// comment; blank lines are skipped; "label idx:value ..." with 1-based,
// strictly increasing indices.  Errors carry 1-based line and column.
Libsvm parse_libsvm_text(const char* text, int64_t len) {
  Libsvm out;
  int64_t line_no = 0;
  int64_t pos0 = 0;
  auto is_space = [](char c) { return std::isspace(static_cast<unsigned char>(c)) != 0; };
  while (pos0 < len) {
    int64_t eol = pos0;
    while (eol < len && text[eol] != '\n') ++eol;
    ++line_no;
    std::string_view line(text + pos0, static_cast<size_t>(eol - pos0));
    pos0 = eol + 1;
    if (const auto hash = line.find('#'); hash != std::string_view::npos) line = line.substr(0, hash);
    size_t pos = 0;
    auto next_token = [&](int64_t* col) {
      while (pos < line.size() && is_space(line[pos])) ++pos;
      const size_t start = pos;
      while (pos < line.size() && !is_space(line[pos])) ++pos;
      *col = static_cast<int64_t>(start) + 1;
      return std::string(line.substr(start, pos - start));
    };
    int64_t col = 0;
    const std::string label = next_token(&col);
    if (label.empty()) continue;
    out.labels.push_back(libsvm_real(label, line_no, col));
    int64_t prev = 0;
    for (;;) {
      const std::string tok = next_token(&col);
      if (tok.empty()) break;
      auto fail = [&](const std::string& what) {
        throw ParseFailure("line " + std::to_string(line_no) + ", column " + std::to_string(col) + ": " + what,
                           line_no, col);
      };
      const size_t colon = tok.find(':');
      if (colon == std::string::npos || colon == 0 || colon + 1 == tok.size())
        fail("expected index:value, got '" + tok + "'");
      const std::string idx_part = tok.substr(0, colon);
      int64_t idx = 0;
      const auto [ptr, ec] = std::from_chars(idx_part.data(), idx_part.data() + idx_part.size(), idx);
      if (ec != std::errc{} || ptr != idx_part.data() + idx_part.size())
        fail("malformed feature index '" + idx_part + "'");
      if (idx < 1) fail("feature index must be >= 1, got " + std::to_string(idx));
      if (idx <= prev) fail("non-increasing feature index " + std::to_string(idx));
      const double v = libsvm_real(tok.substr(colon + 1), line_no, col + static_cast<int64_t>(colon) + 1);
      out.cols.push_back(idx - 1);
      out.values.push_back(v);
      prev = idx;
      out.max_index = std::max(out.max_index, idx);
    }
    out.offsets.push_back(static_cast<int64_t>(out.values.size()));
  }
  return out;
}

// format_double (data_io.cpp:338-342)
std::string format_g17(double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

}  // namespace

rp_status rp_libsvm_parse(const char* text, int64_t len, int64_t feature_override, int64_t* rows, int64_t* cols,
                          int64_t* nnz, int64_t* offsets, int64_t* col_indices, double* values, double* labels,
                          int64_t* err_line, int64_t* err_col) {
  if (err_line) *err_line = 0;
  if (err_col) *err_col = 0;
  return guarded(nullptr, [&] {
    require(len >= 0 && (text || len == 0) && rows && cols && nnz, "parse_libsvm: null argument");
    Libsvm p;
    try {
      p = parse_libsvm_text(text, len);
    } catch (const ParseFailure& e) {
      if (err_line) *err_line = e.line;
      if (err_col) *err_col = e.column;
      throw;
    }
    if (feature_override >= 0 && feature_override < p.max_index)
      throw InvalidArgument("parse_libsvm: declared dimension " + std::to_string(feature_override) +
                            " below max index " + std::to_string(p.max_index));
    *rows = static_cast<int64_t>(p.labels.size());
    *cols = feature_override >= 0 ? feature_override : p.max_index;
    *nnz = static_cast<int64_t>(p.values.size());
    if (offsets) std::copy(p.offsets.begin(), p.offsets.end(), offsets);
    if (col_indices) std::copy(p.cols.begin(), p.cols.end(), col_indices);
    if (values) std::copy(p.values.begin(), p.values.end(), values);
    if (labels) std::copy(p.labels.begin(), p.labels.end(), labels);
  });
}

rp_status rp_write_csv(int64_t nresults, const char* const* solvers, const int64_t* npoints, const double* lambdas,
                       const double* train_loss, const double* test_loss, const uint8_t* has_test,
                       const double* seconds, char* out, int64_t cap, int64_t* needed) {
  return guarded(nullptr, [&] {
    require(nresults >= 0 && needed && (nresults == 0 || (solvers && npoints)), "write_csv: null argument");
    struct Row {
      double lambda;
      const char* solver;
      int64_t i;
    };
    std::vector<Row> rows;
    int64_t at = 0;
    for (int64_t r = 0; r < nresults; ++r) {
      require(npoints[r] >= 0 && solvers[r], "write_csv: bad result");
      for (int64_t j = 0; j < npoints[r]; ++j, ++at) rows.push_back({lambdas[at], solvers[r], at});
    }
    // (data_io.cpp:353-356: stable, by lambda then solver name)
    std::stable_sort(rows.begin(), rows.end(), [](const Row& a, const Row& b) {
      if (a.lambda != b.lambda) return a.lambda < b.lambda;
      return std::strcmp(a.solver, b.solver) < 0;
    });
    std::string s = "lambda,train_loss,test_loss,time_s,solver\n";
    for (const Row& row : rows) {
      s += format_g17(row.lambda) + ',' + format_g17(train_loss[row.i]) + ',';
      if (has_test && has_test[row.i]) s += format_g17(test_loss[row.i]);
      s += ',' + format_g17(seconds[row.i]) + ',' + row.solver + '\n';
    }
    *needed = static_cast<int64_t>(s.size()) + 1;
    if (out && cap > 0) {
      const size_t n = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
      std::memcpy(out, s.data(), n);
      out[n] = '\0';
    }
  });
}

}  // extern "C"
