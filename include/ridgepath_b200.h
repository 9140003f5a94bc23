/*
 * ridgepath_b200.h -- C ABI of the B200-native IHS-BIN ridge-path engine.
 *
 * Drop-in boundary for the reference's proj/core solver API (namespace
 * ridgepath::, /root/reference/proj/core/include/ridgepath/).  Every entry point
 * below names the reference interface it replaces.  Plain pointers and sizes
 * only: dense matrices are column-major (Eigen::MatrixXd's layout,
 * matrix.hpp:10), CSR uses the reference's int64 offsets/columns
 * (matrix.hpp:16-50).  `where` says whether a buffer lives in host memory
 * (RP_HOST, copied in/out inside the call) or in device memory on the
 * context's GPU (RP_DEVICE, used in place; results are ready when the call
 * returns unless stated otherwise).  Device buffers are read and written on
 * the context's stream (its own non-blocking stream unless rp_set_stream
 * selects the caller's): a caller producing inputs on another stream must
 * order them first (rp_set_stream to that stream, or a synchronization).
 *
 * Errors: every function returns rp_status; the message of the last failure on
 * a context is available from rp_last_error().  Status codes map the
 * reference's exceptions 1:1:
 *   std::invalid_argument          -> RP_EINVAL
 *   BasisDivergedError             -> RP_EDIVERGED (path_solver.hpp:18-21)
 *   SolverError                    -> RP_ESOLVER   (path_solver.hpp:23-27)
 *   thin_svd non-convergence       -> RP_ESVD      (matrix.cpp:227-228); here:
 *                                     shifted sketched Gram not SPD
 * plus RP_ECUDA / RP_ENCCL / RP_ENOMEM for device-side failures.
 *
 * Threading: a context is single-owner (like SeededRng); calls on
 * one context must come from one host thread.  Distinct contexts hold
 * independent state and may be driven from different threads concurrently;
 * calls are synchronous.  (RP_DEVICE_LOCK=1 in the environment serializes
 * the calls of contexts that share a GPU, e.g. to keep one call's phase
 * timings free of another's work.)
 */
#ifndef RIDGEPATH_B200_H
#define RIDGEPATH_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define RP_API __attribute__((visibility("default")))
#else
#define RP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rp_ctx rp_ctx;
typedef struct rp_precond rp_precond;

typedef enum {
  RP_OK = 0,
  RP_EINVAL = 1,
  RP_EDIVERGED = 2,
  RP_ESOLVER = 3,
  RP_ESVD = 4,
  RP_ECUDA = 5,
  RP_ENCCL = 6,
  RP_ENOMEM = 7,
  RP_EPARSE = 8 /* ParseError (data_io.hpp): rp_last_error(NULL) = "line L, column C: ..." */
} rp_status;

enum { RP_HOST = 0, RP_DEVICE = 1, RP_HOST_STREAM = 2 };
/* RP_HOST_STREAM (rp_set_dense / rp_set_dense_rows / rp_set_dense_cols only):
 * the operator is uploaded asynchronously, in column chunks on an internal
 * copy stream, and the call returns at once.  The next call that reads the
 * operator waits for it -- rp_ihs_bin_path on a dense primal operator with an
 * SRHT / CountSketch / SJLT / identity sketch instead consumes the chunks as
 * they land (sketch columns, A^T b rows and Gram-matrix block rows), so the
 * PCIe transfer overlaps that work.  The host buffer must stay valid and
 * unmodified until that next call returns; pinned memory is needed for the
 * overlap (pageable memory degrades to a synchronous copy). */

/* SketchKind, sketch.hpp:10 (same order). */
typedef enum {
  RP_SKETCH_GAUSSIAN = 0,
  RP_SKETCH_COUNTSKETCH = 1,
  RP_SKETCH_SJLT = 2,
  RP_SKETCH_SRHT = 3,
  RP_SKETCH_IDENTITY = 4
} rp_sketch_kind;

/* SketchSpec, sketch.hpp:17-29. */
typedef struct {
  int32_t kind; /* rp_sketch_kind */
  int32_t s;    /* SJLT column sparsity */
  int64_t m;    /* sketch rows */
  int64_t n;    /* input rows (rows of the operator) */
  uint64_t seed;
} rp_sketch_spec;

/* PathConfig, spectrum.hpp:14-22.  num_intervals <= 0 selects the automatic
 * split (std::nullopt). */
typedef struct {
  double lambda_min;
  double lambda_max;
  const double* lambdas; /* host */
  int64_t num_lambdas;
  double epsilon;
  int32_t num_intervals;
} rp_path_config;

/* RhoBounds, spectrum.hpp:32-40; provenance follows RhoProvenance
 * (0 Gaussian, 1 Sjlt, 2 Srht, 3 Identity, 4 Manual). */
typedef struct {
  double rho1;
  double rho2;
  int32_t provenance;
} rp_rho_bounds;

/* RateParams, spectrum.hpp:43-49. */
typedef struct {
  double lambda0;
  double alpha;
  double kappa;
  double contraction;
  int32_t k;
} rp_rate_params;

/* Timings of the last path call (RegPathResult setup/total seconds,
 * path_solver.hpp:58-62, split per phase; device-timed with CUDA events). */
typedef struct {
  double setup_seconds;   /* sketch + factor + all interval bases */
  double eval_seconds;    /* compose (+ dual recovery) */
  double total_seconds;   /* setup + eval (excludes host<->device copies) */
  double sketch_seconds;
  double factor_seconds;  /* c = M^T b, Gram matrix, shifted inverses */
  double basis_seconds;
  double copy_seconds;    /* host<->device copies inside the call */
  int32_t retries;        /* intervals rebuilt at tau/2 */
  int32_t gram_mode;      /* 0 = pass over the operator, 1 = Gram matrix */
  int64_t launches;       /* kernels launched by the call */
  /* With rp_set_option(ctx, "profile", 1): every FP64 DMMA GEMM of the call
   * bracketed by CUDA events on the call's stream. */
  double gemm_seconds;    /* summed GEMM kernel time */
  double gemm_flops;      /* algorithmic flops of those GEMMs */
  int64_t gemm_calls;
  /* factor_seconds split: c = M^T b, Gram matrix G = M^T M, preconditioners */
  double linear_seconds;
  double gram_seconds;
  double precond_seconds;
} rp_timings;

/* ---- context -------------------------------------------------------------- */
RP_API const char* rp_version(void);
RP_API rp_status rp_create(rp_ctx** out, int device);
RP_API void rp_destroy(rp_ctx* ctx);
RP_API const char* rp_last_error(const rp_ctx* ctx);
/* Run the context's work on an external CUDA stream (cudaStream_t), or NULL
 * for the context's own stream. */
RP_API rp_status rp_set_stream(rp_ctx* ctx, void* stream);
RP_API rp_status rp_synchronize(rp_ctx* ctx);
/* Options: "gram_mode" (-1 auto, 0 pass, 1 matrix); "profile" (0/1);
 * "stream_priorities" (default 1: sketch and Cholesky-chain streams at the
 * highest stream priority); "gram_overlap" (default 1: Gram matrix SYRK on a
 * side stream); tuning knobs listed in DESIGN.md. */
RP_API rp_status rp_set_option(rp_ctx* ctx, const char* key, int64_t value);
RP_API int64_t rp_launch_count(void);

/* ---- multi-GPU (one process per GPU, NCCL over NVLink) -------------------- */
/* Per-GEMM records of the last path call made with option "profile" = 1:
 * device seconds (CUDA events on the call's stream), algorithmic flops and
 * algorithmic operand bytes, in launch order.  *count = number of records;
 * the first `cap` are copied (any output pointer may be NULL). */
RP_API rp_status rp_last_gemm_profile(rp_ctx* ctx, double* seconds, double* flops, double* bytes, int64_t cap,
                                      int64_t* count);

/* Multi-GPU (one process per GPU): rank 0 makes the id, every rank joins.
 * world = 1 with id128 = NULL leaves the context without a communicator
 * (collectives are no-ops); with an id it builds a one-rank NCCL communicator,
 * so the collective code path runs on a single GPU too. */
RP_API rp_status rp_comm_unique_id(void* id128);
RP_API rp_status rp_comm_init(rp_ctx* ctx, int rank, int world, const void* id128);

/* Host-side communicator: the context's collectives run through caller
 * callbacks on host memory instead of NCCL (an MPI / gloo / shared-memory
 * transport of the caller's choosing, or several ranks sharing one GPU).  Each
 * collective synchronizes the context's stream, copies the operand to a pinned
 * staging buffer, calls the callback from the calling thread and copies the
 * result back.  A callback returns 0 on success; anything else fails the call
 * with RP_ENCCL.
 *   allreduce: buf[0..count) <- sum over ranks, in place;
 *   allgather: recv[r*count .. (r+1)*count) <- rank r's send[0..count). */
typedef int (*rp_host_allreduce_fn)(void* user, double* buf, int64_t count);
typedef int (*rp_host_allgather_fn)(void* user, const double* send, int64_t count, double* recv);
RP_API rp_status rp_comm_init_host(rp_ctx* ctx, int rank, int world, rp_host_allreduce_fn allreduce,
                                   rp_host_allgather_fn allgather, void* user);

/* ---- data operator ----------------------------------------------------------
 * Matrix, matrix.hpp:54-73.  The context keeps one operator A (n x d).  With
 * several ranks each passes its shard: rows [row0, row0 + n_local) of the
 * n_global x d matrix (primal route, row-sharded).  The dual route column-
 * shards A: pass the local column block with rp_set_dense_cols. */
RP_API rp_status rp_set_dense(rp_ctx* ctx, int64_t n, int64_t d, const double* a, int64_t lda, int where);
RP_API rp_status rp_set_dense_rows(rp_ctx* ctx, int64_t n_global, int64_t row0, int64_t n_local, int64_t d,
                            const double* a, int64_t lda, int where);
RP_API rp_status rp_set_dense_cols(rp_ctx* ctx, int64_t n, int64_t d_global, int64_t col0, int64_t d_local,
                            const double* a, int64_t lda, int where);
RP_API rp_status rp_set_csr(rp_ctx* ctx, int64_t n, int64_t d, const int64_t* offsets, const int64_t* cols,
                     const double* vals, int where);
RP_API rp_status rp_set_csr_rows(rp_ctx* ctx, int64_t n_global, int64_t row0, int64_t n_local, int64_t d,
                          const int64_t* offsets, const int64_t* cols, const double* vals, int where);

/* ---- building blocks -------------------------------------------------------
 * apply / apply_transpose / gram_apply (matrix.hpp:81-92): y = A x,
 * x = A^T y, out = A^T (A x) for `ncols` column-major right-hand sides. */
RP_API rp_status rp_apply(rp_ctx* ctx, const double* x, int64_t ncols, double* y, int where);
RP_API rp_status rp_apply_transpose(rp_ctx* ctx, const double* y, int64_t ncols, double* x, int where);
RP_API rp_status rp_gram_apply(rp_ctx* ctx, const double* x, int64_t ncols, double* out, int where);
/* With rp_set_option(ctx, "profile", 1): device seconds (CUDA events on the
 * context stream) of the last rp_apply_transpose / rp_gram_apply call. */
RP_API rp_status rp_last_device_seconds(rp_ctx* ctx, double* seconds);

/* losses / losses_matrix (ref/src/path_solver.cpp:425-454) for T solutions at
 * once, against the context's operator (primal view):
 *   loss[t] = 0.5 ||A X_t - B||_F^2 + 0.5 lambda[t] ||X_t||_F^2
 * X_t = x + t*d*K (d x K, column-major), B: n_local x K (this rank's rows),
 * lambda may be NULL (no regularization term: the reference's test loss).
 * With several ranks (row shards) every rank receives the global sum.
 * x, b, lambda and loss all live on `where`. */
RP_API rp_status rp_losses(rp_ctx* ctx, const double* b, int64_t K, int64_t T, const double* x,
                           const double* lambda, double* loss, int where);

/* sketch_apply (sketch.hpp:43): SA (m x d) of the context's operator;
 * `transpose_op` = 1 sketches A^T instead (the dual route's operator). */
RP_API rp_status rp_sketch_apply(rp_ctx* ctx, const rp_sketch_spec* spec, int transpose_op, double* sa, int where);

/* Preconditioner::build / reshift / apply (preconditioner.hpp:24-34).
 * P = (SA^T SA + lambda0 I)^{-1}, explicit for m >= d, Woodbury for m < d. */
RP_API rp_status rp_precond_build(rp_ctx* ctx, const double* sa, int64_t m, int64_t d, double lambda0, int where,
                           rp_precond** out);
RP_API rp_status rp_precond_reshift(rp_ctx* ctx, const rp_precond* p, double lambda0, rp_precond** out);
RP_API rp_status rp_precond_apply(rp_ctx* ctx, const rp_precond* p, const double* v, int64_t ncols, double* out,
                           int where);
RP_API void rp_precond_destroy(rp_precond* p);

/* ihs_basis / ihs_basis_matrix (path_solver.hpp:89-96): c = A^T b, then the
 * recursion; terms_out is k blocks of d x K (column-major, block j at
 * j*d*K).  ihs_basis_core takes c directly (path_solver.cpp:27-53). */
RP_API rp_status rp_ihs_basis(rp_ctx* ctx, const rp_precond* p, const double* b, int64_t K, double tau, int32_t k,
                       double* terms_out, int where);
RP_API rp_status rp_ihs_basis_core(rp_ctx* ctx, const rp_precond* p, const double* c, int64_t K, double tau, int32_t k,
                            int transpose_op, double* terms_out, int where);
/* ihs_compose / ihs_compose_matrix (path_solver.hpp:98-101): tau * sum_j (tau lambda)^j u_j. */
RP_API rp_status rp_ihs_compose(rp_ctx* ctx, const double* terms, int64_t dim, int64_t K, int32_t k, double tau,
                         double lambda, double* x_out, int where);

/* ---- end-to-end paths ------------------------------------------------------
 * ihs_bin_path / ihs_bin_path_matrix (path_solver.hpp:109-121) for K = 1 / K > 1:
 * b is n x K; x_out receives the d x K solution for every grid lambda, point t
 * at x_out + t*d*K.  dual_path (path_solver.hpp:134-139), matrix B handled as
 * K independent dual paths: x_out is d x K per lambda (the local column block
 * when A is column-sharded).  sigma_d may be NULL (std::nullopt). */
RP_API rp_status rp_ihs_bin_path(rp_ctx* ctx, const double* b, int64_t K, const rp_path_config* cfg,
                          const rp_sketch_spec* spec, const rp_rho_bounds* rho, const double* sigma_d,
                          double* x_out, int where, rp_timings* timings);
RP_API rp_status rp_dual_path(rp_ctx* ctx, const double* b, int64_t K, const rp_path_config* cfg, const rp_sketch_spec* spec,
                       const rp_rho_bounds* rho, const double* sigma_d, double* x_out, int where,
                       rp_timings* timings);

/* ---- host scalar tuning (spectrum.hpp; bit-identical to the reference) ---- */
RP_API rp_status rp_log_grid(double lambda_min, double lambda_max, int32_t count, double* out);
RP_API rp_status rp_tune_interval(double lambda_lo, double lambda_hi, const rp_rho_bounds* rho, const double* sigma_d,
                           double eps, rp_rate_params* out);
RP_API int32_t rp_auto_interval_count(double lambda_min, double lambda_max);
RP_API rp_status rp_interval_split(double lambda_min, double lambda_max, int32_t num_intervals, double* edges_out,
                            int32_t* count_out);

/* ---- comparison baselines (baselines.hpp; baselines.cpp:80-226) ----------
 * warm_cg_path, warm_ihs_path and direct_path on the context's operator with a
 * vector b (n entries; the local rows when row-sharded).  x_out is d x T
 * column-major in grid order.  iterations / seconds (host, T entries each,
 * nullable) are PathPoint::iterations / ::seconds; setup_total (host, 2
 * entries, nullable) receives RegPathResult setup_seconds and total_seconds.
 * Iteration caps and divergence raise RP_ESOLVER (SolverError) as in the
 * reference; direct_path's failed Cholesky is RP_ESOLVER too.
 * rp_svd_path replaces svd_path (baselines.hpp:15, baselines.cpp:51-78): the
 * thin SVD of A as a Householder QR + SVD of the triangular factor (cuSOLVER,
 * loaded at run time), one process only (RP_EINVAL with a communicator). */
RP_API rp_status rp_warm_cg_path(rp_ctx* ctx, const double* b, const rp_path_config* cfg, double* x_out, int where,
                                 int32_t* iterations, double* seconds, double* setup_total);
RP_API rp_status rp_warm_ihs_path(rp_ctx* ctx, const double* b, const rp_path_config* cfg, const rp_sketch_spec* spec,
                                  const rp_rho_bounds* rho, double* x_out, int where, int32_t* iterations,
                                  double* seconds, double* setup_total);
RP_API rp_status rp_direct_path(rp_ctx* ctx, const double* b, const rp_path_config* cfg, double* x_out, int where,
                                double* seconds, double* setup_total);
RP_API rp_status rp_svd_path(rp_ctx* ctx, const double* b, const rp_path_config* cfg, double* x_out, int where,
                             double* seconds, double* setup_total);

/* ---- adaptive sketch dimension (adaptive.hpp; adaptive.cpp:19-137) --------
 * AdaptiveConfig / AdaptiveStep / AdaptiveResult; m_initial, m_cap = 0 select
 * the reference defaults max(16, d/64) and d.  The trace holds every step
 * (trace_len); the first trace_cap entries are copied to `trace` (nullable).
 * x0 (nullable, d entries) and x_out (d entries) live on `where`. */
typedef struct {
  double gamma1;   /* backtracking factor (0.5) */
  double gamma2;   /* sufficient-decrease fraction (1e-4) */
  double gamma3;   /* stall threshold (0.9) */
  double epsilon;  /* progress tolerance (1e-8) */
  int64_t m_initial;
  int64_t m_cap;
  int32_t iteration_cap; /* (200) */
} rp_adaptive_config;

typedef struct {
  int64_t m;
  double f_before;
  double f_after;
  double step;
  double progress;
  int32_t doubled;
} rp_adaptive_step;

typedef struct {
  int64_t m;
  int32_t iterations;
  int32_t doublings;
  int32_t converged;
  int32_t stalled_at_cap;
  int64_t trace_len;
} rp_adaptive_result;

RP_API rp_status rp_adaptive_sketch_dim(rp_ctx* ctx, const double* b, double lambda_min, const rp_adaptive_config* cfg,
                                        const rp_sketch_spec* spec_template, const double* x0, double* x_out,
                                        int where, rp_adaptive_result* result, rp_adaptive_step* trace,
                                        int64_t trace_cap);

/* ---- plug-in envelope (derive_rho, tools/ridgepath_main.cpp:218-279) ------
 * The reference CLI derives (rho1, rho2) from the sketched spectrum when
 * --rho1/--rho2 are absent: sketch A, thin SVD of SA, effective dimension at
 * lambda0 = sqrt(lambda_min * lambda_max), then the family's envelope
 * (spectrum.cpp:87-169).  rp_derive_rho does the same on the device for the
 * context's operator (transpose_op = 1: A^T, the dual route) without an SVD:
 * ||D||_F^2 = tr(H (H + lambda0 I)^{-1}) and s_max^2 = lambda_max(H) by
 * Lanczos, H = SA^T SA or SA SA^T.  Identity sketches return identity bounds
 * without sketching, as the reference does. */
typedef struct {
  double effective_dimension; /* d_e at lambda0 */
  double sigma_max_sq;        /* s_max(SA)^2 */
  double dnorm_sq;            /* s_max^2 / (s_max^2 + lambda0) */
  double lambda0;
  int32_t lanczos_steps;
} rp_spectrum_info;

RP_API rp_status rp_derive_rho(rp_ctx* ctx, const rp_sketch_spec* spec, int transpose_op, double lambda_min,
                               double lambda_max, rp_rho_bounds* out, rp_spectrum_info* info);
/* effective_dimension (spectrum.hpp:51-52; spectrum.cpp:87-103), host. */
RP_API rp_status rp_effective_dimension(const double* sigma, int64_t count, double lambda0, double* out);
/* rho_gaussian (spectrum.cpp:105-128); m <= 0 = std::nullopt.  success_probability
 * may be NULL; it is set to NaN when m is absent. */
RP_API rp_status rp_rho_gaussian(double rho, double eta, double dnorm_sq, int64_t m, rp_rho_bounds* out,
                                 double* success_probability);
/* rho_srht (spectrum.cpp:130-148); n <= 0 = std::nullopt; recommended_m (nullable) = -1 when absent. */
RP_API rp_status rp_rho_srht(double rho, double dnorm_sq, int64_t n, double de, rp_rho_bounds* out,
                             int64_t* recommended_m);
/* rho_sjlt (spectrum.cpp:150-169); alpha <= 0 = std::nullopt; recommendations = -1 when absent. */
RP_API rp_status rp_rho_sjlt(double eps, double alpha, double delta, double de, rp_rho_bounds* out,
                             int64_t* recommended_m, int32_t* recommended_s);

/* ---- draw contract (rng.hpp / sketch.cpp draw loops), device-generated ---- */
RP_API rp_status rp_draw_u64(rp_ctx* ctx, uint64_t seed, uint64_t skip, int64_t count, uint64_t* out, int where);
RP_API rp_status rp_draw_uniform01(rp_ctx* ctx, uint64_t seed, int64_t count, double* out, int where);
RP_API rp_status rp_draw_sign(rp_ctx* ctx, uint64_t seed, int64_t count, double* out, int where);
RP_API rp_status rp_draw_uniform_index(rp_ctx* ctx, uint64_t seed, uint64_t bound, int64_t count, uint64_t* out,
                                int where);
/* normals #first .. #first+count-1 of SeededRng(seed).normal(), times scale */
RP_API rp_status rp_draw_normals(rp_ctx* ctx, uint64_t seed, int64_t first, int64_t count, double scale, double* out,
                          int where);
/* Gaussian sketch window S[r0:r0+rc, j0:j0+jc] (row-major rc x jc). */
RP_API rp_status rp_gaussian_window(rp_ctx* ctx, uint64_t seed, int64_t m, int64_t n, int64_t r0, int64_t rc, int64_t j0,
                             int64_t jc, double* out, int where);
RP_API rp_status rp_count_draws(rp_ctx* ctx, const rp_sketch_spec* spec, int64_t* h_out, double* sign_out, int where);
RP_API rp_status rp_srht_draws(rp_ctx* ctx, const rp_sketch_spec* spec, double* signs_out, int64_t* rows_out, int where);

/* Host-only self-check of the jump-ahead engine: 0 on success. */
RP_API int rp_mt_selfcheck(uint64_t seed, uint64_t offset);

/* ---- data formats either side of the path (data_io.hpp; data_io.cpp) ------
 * rp_libsvm_parse replaces parse_libsvm (data_io.cpp:50-127) on an in-memory
 * text of `len` bytes: call once with NULL arrays for rows / cols / nnz, then
 * with offsets (rows + 1), col_indices (nnz, 0-based), values (nnz) and labels
 * (rows).  feature_override < 0 = none (cols = max index), else the declared
 * dimension (RP_EINVAL if below the max index).  Malformed input returns
 * RP_EPARSE with the 1-based line / column in err_line / err_col (nullable).
 * rp_write_csv replaces write_csv (data_io.cpp:344-364): results r = 0 ..
 * nresults-1 with npoints[r] points each, the point arrays concatenated in
 * result order; rows sorted stably by lambda then solver name, 17 significant
 * digits, empty test_loss where has_test[i] == 0 (has_test nullable = none).
 * *needed = bytes incl. the terminating NUL; out (cap bytes) may be NULL. */
RP_API rp_status rp_libsvm_parse(const char* text, int64_t len, int64_t feature_override, int64_t* rows,
                                 int64_t* cols, int64_t* nnz, int64_t* offsets, int64_t* col_indices, double* values,
                                 double* labels, int64_t* err_line, int64_t* err_col);
RP_API rp_status rp_write_csv(int64_t nresults, const char* const* solvers, const int64_t* npoints,
                              const double* lambdas, const double* train_loss, const double* test_loss,
                              const uint8_t* has_test, const double* seconds, char* out, int64_t cap,
                              int64_t* needed);

#ifdef __cplusplus
}
#endif

#endif /* RIDGEPATH_B200_H */
