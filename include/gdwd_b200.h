/*
 * gdwd_b200 -- C ABI of the B200-native sGS-ADMM hot path for generalized
 * Distance Weighted Discrimination (arXiv 2305.12019).
 *
 * The reference (pkg/src/gdwd, pure Python on numpy/scipy) has no FFI; the
 * entry points below are the seams a maintainer binds (ctypes stub in
 * INTEGRATION.md) to replace its hot path.  Each declaration cites the
 * reference interface it stands in for.
 *
 * Conventions
 *   - plain pointers + sizes; host pointers are borrowed for the call only;
 *     device memory is owned by the context.
 *   - all arithmetic is fp64; Z~ is the scaled d x n data matrix of
 *     ProblemData (reference solver.py:60-71), samples as columns.
 *   - return value: GDWD_OK (0) or one of the GDWD_ERR_* codes; codes map 1:1
 *     onto the reference's exceptions; gdwd_last_error() has the message.
 *   - one context per host thread; a context is not re-entrant.
 */
#ifndef GDWD_B200_H
#define GDWD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  GDWD_OK = 0,
  GDWD_ERR_CUDA = 1,         /* RuntimeError (device / launch failure)                  */
  GDWD_ERR_VALUE = 2,        /* ValueError (solver.py:73-87,118-124)                   */
  GDWD_ERR_INDEFINITE = 3,   /* IndefiniteMatrixError (linalg/cholesky.py:12,47-48)     */
  GDWD_ERR_SCHUR = 4,        /* DegenerateSchurError (subsolvers.py:38,249-252)        */
  GDWD_ERR_LANCZOS = 5,      /* LanczosConvergenceError (linalg/lanczos.py:25-30)      */
  GDWD_ERR_ASSERT = 6,       /* AssertionError: r left the positive orthant (solver.py:319-320) */
  GDWD_ERR_UNSUPPORTED = 7,  /* feature not available on this path                     */
  GDWD_ERR_ABORTED = 8       /* the per-iteration callback asked to stop               */
};

enum { GDWD_BACKEND_AUTO = 0, GDWD_BACKEND_DIRECT = 1, GDWD_BACKEND_SMW2 = 2, GDWD_BACKEND_ITERATIVE = 3 };

typedef struct gdwd_ctx gdwd_ctx;

/* SolverConfig (reference solver.py:101-124).  NaN in sigma0 / epsilon_c
 * means "reference default" (solver.py:440-445). */
typedef struct {
  int32_t max_iter;
  int32_t backend;            /* GDWD_BACKEND_* (Backend enum, solver.py:48-57) */
  int32_t use_sgs;
  int32_t psqmr_switch_steps;
  int32_t ell;
  int32_t seed;
  int32_t use_graph;          /* capture the iteration body in a CUDA graph (DIRECT/SMW2) */
  int32_t poll_every;         /* host polls the device stop flag every k iterations      */
  int32_t smw_gram_space;     /* SMW2 with n <= d: iterate in n-coefficient space, K = Z~^T Z~ */
  int32_t persistent;         /* Gram-space SMW2: run iterations in one cooperative kernel */
  int32_t iter_gram;          /* ITERATIVE, dense: PSQMR operator A v from the d x d Gram
                                 Z~ Z~^T (formed once on the FP64 tensor cores) instead of two
                                 passes over X; 0 auto (d <= n/4 and it fits), 1 on, -1 off */
  double steplength;
  double tol_feas;
  double tol_cgap;
  double tol_cap;
  double sigma0;
  double epsilon_c;
  double mu;
} gdwd_config;

/* SolveResult scalars (reference solver.py:170-183). */
typedef struct {
  int32_t iterations;
  int32_t converged;
  int32_t backend;            /* resolved backend */
  int32_t psqmr_total;
  int32_t double_count;
  int32_t status;
  double beta;
  double sigma;
  double eps_c;
  double setup_ms;            /* factorisation / preconditioner build, device time */
  double loop_ms;             /* iteration loop, device time                        */
  double resid[11];           /* KKTResiduals fields, reference order (solver.py:143-155) */
} gdwd_result;

/* callback(state, residuals) of sgs_admm_solve (solver.py:546-547): called on
 * the host after each iteration with the 11 KKT values; the iterates can be
 * fetched with gdwd_get_state from inside the callback.  Nonzero return
 * aborts the solve (GDWD_ERR_ABORTED). */
typedef int (*gdwd_iter_cb)(void* user, int32_t iter, const double* resid11, double sigma, double beta);

/* all-reduce (sum, in place, across the sample shards) of `count` host
 * doubles; nonzero return aborts.  Used by gdwd_comm_init_host. */
typedef int (*gdwd_allreduce_cb)(void* user, double* buf, int64_t count);

/* context ------------------------------------------------------------------*/
int gdwd_ctx_create(int32_t device, gdwd_ctx** out);
void gdwd_ctx_destroy(gdwd_ctx* ctx);
const char* gdwd_last_error(const gdwd_ctx* ctx);
/* sizeof(gdwd_config), sizeof(gdwd_result) as compiled (binding layout check) */
void gdwd_abi_sizes(int64_t* config_bytes, int64_t* result_bytes);
int gdwd_version(void);

/* data ----------------------------------------------------------------------
 * Dense Z~: the CSC values array of a fully stored d x n matrix, i.e. the
 * row-major [n][d] sample matrix (SparseMatrixCSC, linalg/sparse.py:20-57). */
int gdwd_upload_dense(gdwd_ctx* ctx, const double* samples, int64_t d, int64_t n);
/* gdwd_upload_dense overlaps the copy with the one-time factorisation where
 * the regime allows (unsharded contexts): a pageable source is staged by host
 * threads through a pooled page-locked ring while earlier blocks are in
 * flight; in the sample-space regimes the Gram, its Cholesky factor and
 * inverse advance block by block under the copy (see gdwd_upload_hint); in
 * DIRECT's own regime (n >= 4d) the d x d Gram Z~ Z~^T (subsolvers.py:76) is
 * summed block by block.  Results match the plain path to rounding (other
 * summation order; deterministic run to run). */
/* Optional, before gdwd_upload_dense: the backend (GDWD_BACKEND_*) and mu the
 * coming solve will use (SolverConfig, solver.py:101-124).  In the
 * sample-space regimes (n <= d, n <= 2500) a page-locked upload then forms
 * the n x n Gram (subsolvers.py:109), its Cholesky factor and explicit
 * inverse (cholesky.py:46,60-61) block by block while the samples are still
 * being copied; a solve with another mu refactors from the Gram.  Default:
 * AUTO, mu = 1.  GDWD_BACKEND_ITERATIVE (also passed for the shards of a
 * multi-GPU solve): plain copy, nothing is formed during the upload. */
int gdwd_upload_hint(gdwd_ctx* ctx, int32_t backend, double mu);
/* Sparse Z~ in the reference's CSC layout (int64 colptr/rowidx). */
int gdwd_upload_csc(gdwd_ctx* ctx, const int64_t* colptr, const int64_t* rowidx, const double* values,
                    int64_t d, int64_t n);
/* On-device synthetic data (configs too large for host memory): raw samples
 * x_i = ytrue_i * shift * 1[j < signal_k] + N(0, I) for global sample indices
 * offset .. offset+n-1 (counter-based, shard-consistent; kind 0 = two
 * Gaussians).  Then scale in place to Z~ = X diag(y) / z_scale
 * (scale_problem, solver.py:253-285).  gdwd_frobenius_sq reports ||X||_F^2
 * after generation and ||Z~||_F^2 after scaling. */
int gdwd_generate_dense(gdwd_ctx* ctx, int32_t kind, uint64_t seed, int64_t d, int64_t n, int64_t offset,
                        int64_t signal_k, double shift);
int gdwd_scale_dense(gdwd_ctx* ctx, const double* y, double z_scale);
/* copy the (local) dense samples back as row-major [n][d] (tests, proxies) */
int gdwd_download_dense(gdwd_ctx* ctx, double* samples);
/* ||Z~||_F^2, reduced on the device at upload (frobenius_norm, sparse.py:63). */
int gdwd_frobenius_sq(gdwd_ctx* ctx, double* out);
/* ProblemData vectors and scalars (solver.py:60-71); all length n. */
int gdwd_set_problem(gdwd_ctx* ctx, const double* y, const double* e, const double* weights, double C,
                     double q, double z_scale);

/* sample sharding -------------------------------------------
 * Each rank uploads its contiguous block of samples (columns of Z~) and its
 * y/e/weights, then joins a communicator; every later product with Z~
 * all-reduces its d-partial and n-sums (one bundle per reduction point) and
 * d-space work is replicated.  n_global is the total sample count.  SMW2 is
 * not sharded (its n x n Gram couples all samples). */
int gdwd_comm_unique_id(uint8_t* out128);  /* ncclGetUniqueId, on one rank */
int gdwd_comm_init_nccl(gdwd_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t* id128, int64_t n_global);
int gdwd_comm_init_host(gdwd_ctx* ctx, int32_t nranks, int32_t rank, gdwd_allreduce_cb cb, void* user,
                        int64_t n_global);
/* Sum of a host vector over the shards of the attached communicator (identity
 * when unsharded): the host-side n-sums such as the global train error
 * (solver.py:558-559). */
int gdwd_allreduce_host(gdwd_ctx* ctx, double* buf, int64_t count);

/* operator seams ------------------------------------------------------------
 * Z~ v  (scipy csc_matvec at solver.py:496,508,517,300; subsolvers.py:146) */
int gdwd_matvec(gdwd_ctx* ctx, const double* v_n, double* out_d);
/* Z~^T v (scipy csr_matvec at solver.py:501,530,322; subsolvers.py:140)   */
int gdwd_matvec_t(gdwd_ctx* ctx, const double* v_d, double* out_n);

/* scoring a trained model (decision_values / predict / train_error,
 * solver.py:610-642) over the uploaded samples X (raw, d x n, as uploaded by
 * gdwd_upload_dense / gdwd_upload_csc): scores = beta + X^T w, w of the
 * uploaded length d (callers pad or truncate the composite weights, as
 * decision_values does).  scores (n) may be NULL.  If y (n) is not NULL,
 * *wrong receives the number of samples with y_i * sgn(score_i) <= 0 (a zero
 * score counts as wrong for both classes).  One fused pass over X. */
int gdwd_score(gdwd_ctx* ctx, const double* w, double beta, const double* y, double* scores, int64_t* wrong);

/* kkt_residuals (solver.py:311-340) of an iterate (r, xi, alpha: n; w, u: d;
 * beta) for the uploaded problem: out11 = [eta_c1, eta_c2, eta_c3, eta_p1,
 * eta_p2, eta_p3, eta_d1, eta_d2, eta_gap, obj_primal, obj_dual].
 * GDWD_ERR_ASSERT if some r_i <= 0 (solver.py:319-320). */
int gdwd_kkt_residuals(gdwd_ctx* ctx, const double* r, const double* xi, const double* alpha, const double* w,
                       const double* u, double beta, double mu, double* out11);

/* the distance statistic of compute_penalty_C (solver.py:193-232): over the
 * uploaded raw samples, the median Euclidean distance between the samples
 * ia[0..na) and ib[0..nb) (the two classes after the caller's seeded
 * subsampling, solver.py:208-213), exact-zero distances dropped; Gram on the
 * FP64 tensor cores, exact median by radix selection.  *positives receives
 * the number of positive distances (0: all zero, *median = 0). */
int gdwd_between_class_median(gdwd_ctx* ctx, const int64_t* ia, int64_t na, const int64_t* ib, int64_t nb,
                              double* median, int64_t* positives);

/* LIBSVM ingest (ingest.py:102-211), native and multi-threaded -----------------
 * gdwd_libsvm_parse: parse a file (path) or an in-memory buffer (text, len)
 * with the reference grammar; on a malformed line returns GDWD_ERR_VALUE with
 * *err_line (1-based; 0 = "no samples in input") and the reference's message
 * in err_msg.  Samples become CSC columns, exact zeros dropped; labels are
 * NaN on unlabeled lines (label mapping to {-1,+1} is the caller's,
 * ingest.py:90-99).  threads <= 0: all host cores. */
typedef struct gdwd_libsvm gdwd_libsvm;
int gdwd_libsvm_parse(const char* path, const char* text, int64_t text_len, int32_t require_labels,
                      int32_t threads, gdwd_libsvm** out, int64_t* err_line, char* err_msg, int64_t err_cap);
int gdwd_libsvm_sizes(const gdwd_libsvm* p, int64_t* n, int64_t* d, int64_t* nnz, int32_t* unlabeled);
int gdwd_libsvm_copy(const gdwd_libsvm* p, int64_t* colptr, int64_t* rowidx, double* values, double* labels,
                     int64_t* label_lines);
void gdwd_libsvm_free(gdwd_libsvm* p);
/* preprocess (ingest.py:185-211) of a CSC matrix: kept features (max-abs > 0)
 * with their max-abs scales, entries divided by their feature's max-abs
 * (zero quotients pruned) and rows renumbered.  Output capacities: kept_ids,
 * scales: d; new_colptr: n + 1; new_rowidx, new_values: nnz (may be NULL to
 * query *new_nnz).  GDWD_ERR_VALUE when every feature is zero
 * (*kept_count = 0) or on a non-finite / out-of-range entry. */
int gdwd_preprocess_csc(int64_t d, int64_t n, const int64_t* colptr, const int64_t* rowidx, const double* values,
                        int32_t threads, int64_t* kept_count, int64_t* kept_ids, double* scales, int64_t* new_colptr,
                        int64_t* new_rowidx, double* new_values, int64_t* new_nnz);

/* the solver ----------------------------------------------------------------
 * sgs_admm_solve (solver.py:392-602).  sigma_schedule (nullable, test hook):
 * sigma of iteration k for 1 <= k < sched_len replaces update_sigma. */
int gdwd_solve(gdwd_ctx* ctx, const gdwd_config* cfg, const double* sigma_schedule, int64_t sched_len,
               gdwd_iter_cb cb, void* user, gdwd_result* out);
/* The same solve in three calls, so a caller (the benchmark) can time an
 * exact number of iterations on device-resident state: _begin does the setup
 * (factorisation / preconditioner, initial iterates, CUDA-graph capture),
 * _iterate runs up to `count` more iterations (fewer if the stopping rule
 * fires), _end evaluates the last iteration's stop test and fills `out`. */
int gdwd_solve_begin(gdwd_ctx* ctx, const gdwd_config* cfg, const double* sigma_schedule, int64_t sched_len);
int gdwd_solve_iterate(gdwd_ctx* ctx, int32_t count, gdwd_iter_cb cb, void* user, int32_t* iters_done,
                       int32_t* stopped);
int gdwd_solve_end(gdwd_ctx* ctx, gdwd_result* out);
/* Device time (ms, CUDA events on the solve's stream, synchronised on both
 * sides) of `count` further iterations of the current solve. */
int gdwd_time_iterations(gdwd_ctx* ctx, int32_t count, double* ms, int32_t* iters_done);
/* Per-kernel profiling: with profiling on, iterations run without the CUDA
 * graph and every launch is bracketed by events; gdwd_get_profile writes
 * "tag launches total_ms" lines and the launch counter. */
int gdwd_set_profile(gdwd_ctx* ctx, int32_t enable);
int gdwd_get_profile(gdwd_ctx* ctx, char* buf, int64_t buflen, int64_t* launches);
int gdwd_reset_counters(gdwd_ctx* ctx);
/* Start vector of the Lanczos run that builds the proximal backend when
 * PSQMR exceeds psqmr_switch_steps (lanczos.py:85: default_rng(seed)
 * .standard_normal(d), normalised by the library). */
int gdwd_set_lanczos_start(gdwd_ctx* ctx, const double* v, int64_t d);
/* End-of-iteration iterates (SolverState, solver.py:127-140); any pointer may
 * be NULL.  n-vectors: r, xi, alpha, ztw; d-vectors: w, u, rho. */
int gdwd_get_state(gdwd_ctx* ctx, double* r, double* xi, double* alpha, double* w, double* u, double* rho,
                   double* ztw, double* beta);
/* Per-iteration history rows of 16 doubles: the 11 KKT fields, sigma, beta,
 * reused (0/1), psqmr steps, eps_k.  Returns rows written in *rows. */
int gdwd_get_history(gdwd_ctx* ctx, double* hist, int64_t max_rows, int64_t* rows);

/* standalone kernels (unit-test seams) -------------------------------------*/
/* newton_r_sweep (subsolvers.py:321-364); scalar_form bit 0 gives newton_r
 * (subsolvers.py:283-318) per coordinate, iters (nullable) its counts; bit 1
 * runs one warp per coordinate (the persistent kernel's warp-parallel
 * bisection; same roots and counts). */
int gdwd_newton_sweep(int32_t device, int64_t n, const double* a, double sigma, double q, const double* weights,
                      const double* r_init, double tol, int32_t max_newton, int32_t scalar_form, double* out,
                      int32_t* iters);
/* cholesky_factorize + explicit inverse (linalg/cholesky.py:25-66): S (m x m
 * SPD, row-major) -> S^{-1}.  GDWD_ERR_INDEFINITE on a non-positive pivot. */
int gdwd_chol_inverse(int32_t device, const double* S, int64_t m, double* inv_out);
/* the same inverse by the row-block (bordered) chain of the pipelined upload,
 * `block` rows at a time */
int gdwd_chol_inverse_bordered(int32_t device, const double* S, int64_t m, int32_t block, double* inv_out);
/* Gram of a row-major [rows][cols] matrix X on the FP64 tensor cores:
 * sum_over_rows=1: X^T X (cols x cols, "Z Z^T" of subsolvers.py:76)
 * sum_over_rows=0: X X^T (rows x rows, "Z^T Z" of subsolvers.py:109)
 * result = gram / div + shift * I. */
/* device time (ms, mean of reps) of the one-time FP64 DMMA Gram of the
 * resident dense Z~ (bench: the Gram's tensor-pipe roofline) */
int gdwd_time_gram(gdwd_ctx* ctx, int32_t reps, double* ms);
int gdwd_gram(int32_t device, const double* X, int64_t rows, int64_t cols, int32_t sum_over_rows, double div,
              double shift, double* out);
/* the n x n Gram K = Z~^T Z~ (subsolvers.py:109) and G^{-1} = (K/mu^2 + I)^{-1}
 * (cholesky.py:46,60-61) that a page-locked gdwd_upload_dense formed during
 * the copy; row-major n x n outputs (nullable); *have: bit 0 = K is
 * available, bit 1 = G^{-1} is. */
int gdwd_get_upload_factor(gdwd_ctx* ctx, double* K_out, double* Ginv_out, int32_t* have);
/* psqmr (linalg/psqmr.py:27-95) with a dense symmetric operator A (m x m,
 * row-major) and diagonal preconditioner M (nullable = identity); x0 nullable.
 * info[4] = {iterations, converged, breakdown, 0}; *resnorm = final |res|. */
int gdwd_psqmr_dense(int32_t device, const double* A, int64_t m, const double* b, const double* M, double tol,
                     int32_t max_iter, const double* x0, double* x_out, int32_t* info, double* resnorm);

#ifdef __cplusplus
}
#endif
#endif /* GDWD_B200_H */
