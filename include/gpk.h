/*
 * gpk.h — C-ABI of the B200-native matrix-free GP kernel operator and its
 * iterative solvers (arXiv 2405.18457 hot path).
 *
 * Drop-in boundary: every entry point replaces one call of the reference C++
 * API in /root/reference/proj/core/include/gpiter/ (cited per function). The
 * reference passes Eigen::MatrixXd (column-major FP64) by const reference and
 * returns by value; here the same matrices cross as plain column-major FP64
 * host pointers plus sizes, so a C++ shim (include/gpiter_b200.hpp) or a
 * ctypes/cgo binding can wrap them without copies of its own. No torch or
 * CUDA types appear in any signature; device pointers in the *_device calls
 * are plain `void*`/typed pointers into memory the caller obtained from the
 * same device.
 *
 * Errors: every call returns a gpk_status; gpk_last_error() gives the message
 * (thread-local). The C++ shim maps GPK_EINVAL -> std::invalid_argument,
 * GPK_ERANGE -> std::out_of_range, GPK_ENUMERIC -> std::runtime_error,
 * exactly the reference's conventions (kernel.cpp:134-135, 201-203;
 * solvers.cpp:108-112; pivoted_cholesky.cpp:47-49). Solver breakdown /
 * divergence is NOT an error: it is reported through gpk_solver_report
 * .aborted/.abort_reason as in solvers.cpp:65-71 and 173-177.
 *
 * Numerics: kernel evaluation and the K.V contraction run in FP32 on the GPU
 * with FP64 accumulation across column tiles; all solver state, reductions,
 * preconditioner and block factors are FP64.
 */
#ifndef GPK_H_
#define GPK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GPK_OK = 0,
  GPK_EINVAL = 1,   /* std::invalid_argument */
  GPK_ERANGE = 2,   /* std::out_of_range */
  GPK_ENUMERIC = 3, /* std::runtime_error (numerical failure) */
  GPK_ECUDA = 4,    /* CUDA runtime / library failure */
  GPK_ENCCL = 5
} gpk_status;

typedef struct gpk_ctx gpk_ctx;
typedef struct gpk_operator gpk_operator;
typedef struct gpk_batch gpk_batch;
typedef struct gpk_precond gpk_precond;
typedef struct gpk_rff_basis gpk_rff_basis;

/* SolverKind (linear_system.hpp:12). */
enum { GPK_CG = 0, GPK_AP = 1, GPK_SGD = 2 };

/* SolverConfig (linear_system.hpp:14-28), same fields and defaults. */
typedef struct {
  int kind;
  double tolerance;        /* 0.01 */
  int max_epochs;          /* 50 */
  int block_size;          /* 1000 (AP) */
  int batch_size;          /* 500 (SGD) */
  double learning_rate;    /* 30 (SGD) */
  double momentum;         /* 0.9 (SGD) */
  int preconditioner_rank; /* 100 (CG) */
  int warm_start;
  uint64_t seed;           /* SGD batch sampling */
  uint64_t substream;
} gpk_solver_config;

/* SolverReport (linear_system.hpp:30-40). */
typedef struct {
  int iterations;
  double epochs_consumed;
  double mean_residual_norm;
  double probe_residual_norm;
  int reached_tolerance;
  int residuals_estimated;
  int aborted;
  char abort_reason[128];
  double wall_seconds;
} gpk_solver_report;

/* ---- context -------------------------------------------------------- */
const char* gpk_last_error(void);
const char* gpk_version(void);
/* One context per GPU (one process per GPU in multi-GPU runs). */
gpk_status gpk_ctx_create(int device, gpk_ctx** out);
gpk_status gpk_ctx_destroy(gpk_ctx* ctx);
gpk_status gpk_ctx_synchronize(gpk_ctx* ctx);
/* Makes the context stream wait for all work issued so far on the context's
 * auxiliary stream (the AP block factorisations the optimiser starts for the
 * next step), so an event recorded on the stream afterwards covers both. */
gpk_status gpk_ctx_join(gpk_ctx* ctx);
/* Number of this library's kernel launches issued on the context so far. */
gpk_status gpk_ctx_launch_count(gpk_ctx* ctx, long long* out);
/* The CUDA stream (cudaStream_t) all work of this context is issued on. */
gpk_status gpk_ctx_stream(gpk_ctx* ctx, void** stream_out);
/* Operator-kernel counters, accumulated on the device by every executed
 * (non-skipped) K.V launch: out[0] = kernel evals x RHS, out[1] = algorithmic
 * FP32 flops (entries * (2m + 3d + 6)), out[2] = profiled K.V launches,
 * out[3] = summed CUDA-event duration of those launches in ms (only while
 * profiling is on). gpk_ctx_reset_stats zeroes them. */
gpk_status gpk_ctx_set_profiling(gpk_ctx* ctx, int enable);
/* Operator kernel: 0 = FP32 SIMT (kv_slab_kernel), 1 = tcgen05 3xTF32
 * (kv_tc_kernel; K evaluated into TMEM, contraction on the tensor cores). */
gpk_status gpk_ctx_set_operator_kernel(gpk_ctx* ctx, int kernel);
gpk_status gpk_ctx_reset_stats(gpk_ctx* ctx);
/* out5: [evals x RHS, FP32-equivalent operator flops (2m + 3d + 6 per kernel
 * entry), profiled operator launches, profiled operator ms, flops executed on
 * the FP32 pipe (3d + 6 per entry on the tcgen05 kernel, whose 2m-flop
 * contraction runs on the tensor cores; all of them on the SIMT kernel)]. */
gpk_status gpk_ctx_stats(gpk_ctx* ctx, double* out5);

/* ---- multi-GPU (row-sharded; one process per GPU) ----------------------
 * Rank 0 calls gpk_comm_unique_id and ships the 128 bytes to every rank out
 * of band (e.g. a torch.distributed broadcast); each rank then calls
 * gpk_ctx_init_comm on its own context. Afterwards gpk_optimiser_* / gpk_optimise
 * on that context shard the n rows: rank r owns rows [r*S, min(n, (r+1)*S)),
 * S = 32-row-aligned ceil(n / nranks) (gpk_shard_rows), holds only those rows of
 * the solver state, and exchanges the packed search direction (all-gather
 * over NVLink) and per-column partial sums (all-gathered, then summed in rank
 * order so every rank takes bitwise identical decisions). X is replicated. */
gpk_status gpk_comm_unique_id(unsigned char* id128);
gpk_status gpk_ctx_init_comm(gpk_ctx* ctx, const unsigned char* id128, int nranks, int rank);
gpk_status gpk_shard_rows(int n, int nranks, int rank, int* row0, int* row1);

/* ---- KernelOperator (kernel.hpp:37-97) --------------------------------
 * gpk_operator_create replaces KernelOperator(shared_ptr<const Dataset>,
 * Hyperparameters, KernelOperatorOptions) (kernel.hpp:39-40, kernel.cpp:83-109):
 * inputs is the Dataset's n x d column-major FP64 matrix; raw is the
 * Hyperparameters raw vector [l_1..l_d, signal, noise] (hyperparameters.hpp:19-49).
 * The inputs are uploaded once; gpk_operator_set_hyperparameters re-prescales
 * on the device for the next outer step without re-uploading. */
gpk_status gpk_operator_create(gpk_ctx* ctx, const double* inputs, int n, int d,
                               const double* raw, gpk_operator** out);
gpk_status gpk_operator_set_hyperparameters(gpk_operator* op, const double* raw);
/* KernelOperatorOptions::dense_cache (kernel.hpp:27-30): FP64 products for
 * full H V (the reference holds H in FP64). Here H is never materialised:
 * entries are evaluated in FP64 on the fly (GPK_DENSE_KV64=0: cached FP64
 * matrix + DGEMM, as the reference). Single-rank operators only. */
gpk_status gpk_operator_set_dense_cache(gpk_operator* op, int enable);
gpk_status gpk_operator_destroy(gpk_operator* op);
gpk_status gpk_operator_size(const gpk_operator* op, int* n, int* d);

/* H V, V n x m (kernel.cpp:133-152). */
gpk_status gpk_apply(gpk_operator* op, const double* v, int m, double* out);
/* H[rows, :] V (kernel.cpp:154-168). */
gpk_status gpk_apply_rows(gpk_operator* op, const int* rows, int count, const double* v, int m,
                          double* out);
/* H[:, c0:c0+len] U, U len x m (kernel.cpp:170-177). */
gpk_status gpk_apply_columns(gpk_operator* op, int c0, int len, const double* u, int m, double* out);
/* Dense H[r0:r0+rows, c0:c0+cols] (kernel.cpp:179-184), evaluated in FP64. */
gpk_status gpk_dense_block(gpk_operator* op, int r0, int rows, int c0, int cols, double* out);
/* (dH/dtheta_k) V for parameter k of [l_1..l_d, signal, noise] in FP64, V n x m
 * column-major (derivative_apply, kernel.hpp:71, kernel.cpp:200-236):
 * GPK_ERANGE for k outside [0, d+2) as the reference's std::out_of_range. */
gpk_status gpk_derivative_apply(gpk_operator* op, int k, const double* v, int m, double* out);
/* Column i of K (no noise) in FP64 (kernel.cpp:188-194); diag(K) (196-198). */
gpk_status gpk_kernel_column(gpk_operator* op, int i, double* out);
gpk_status gpk_kernel_diagonal(gpk_operator* op, double* out);
/* sum_j u_j^T (dH/dtheta_k) w_j for all k, for npairs (U,W) pairs sharing one
 * pass over the kernel tiles (kernel.cpp:238-272). u[p], w[p] are n x cols[p]
 * column-major; out is npairs x (d+2), row p = pair p. */
gpk_status gpk_derivative_quadratic_forms_many(gpk_operator* op, int npairs, const double* const* u,
                                               const double* const* w, const int* cols, double* out);

/* Device-resident operator product (the solvers' hot path):
 * out[r][j] (FP64, row-major, leading dim ldo) = sum_c H[r, c] v[c][j], with
 * v FP32 row-major [n][ldv], ldv == gpk_rhs_ld(m), pad columns zero.
 * Stream-ordered on the context stream; no synchronisation. */
int gpk_rhs_ld(int m);
gpk_status gpk_apply_device(gpk_operator* op, const float* v, int m, double* out, int ldo);

/* ---- PivotedCholeskyPreconditioner (pivoted_cholesky.hpp:13-32) ------- */
gpk_status gpk_precond_create(gpk_operator* op, int rank, gpk_precond** out);
gpk_status gpk_precond_destroy(gpk_precond* p);
gpk_status gpk_precond_info(const gpk_precond* p, int* achieved_rank, int* stopped_early);
/* factor: n x achieved_rank column-major; pivots: achieved_rank ints. */
gpk_status gpk_precond_factor(gpk_precond* p, double* factor, int* pivots);
/* P^-1 V (pivoted_cholesky.cpp:53-58). */
gpk_status gpk_precond_apply(gpk_precond* p, const double* v, int m, double* out);

/* ---- LinearSystemBatch (linear_system.hpp:45-68) ----------------------- */
gpk_status gpk_batch_create(gpk_operator* op, const double* targets, int m, gpk_batch** out);
gpk_status gpk_batch_destroy(gpk_batch* b);
/* Sets the initial iterate bit for bit (linear_system.cpp:24-30). */
gpk_status gpk_batch_warm_start(gpk_batch* b, const double* previous_solutions);
/* Same, from the solutions another batch of identical shape holds on device. */
gpk_status gpk_batch_warm_start_from(gpk_batch* b, const gpk_batch* previous);
gpk_status gpk_batch_refresh_residuals(gpk_batch* b);
/* which: 0 targets, 1 solutions, 2 residuals (n x m column-major); 3 scales (m). */
gpk_status gpk_batch_get(gpk_batch* b, int which, double* out);
gpk_status gpk_batch_set(gpk_batch* b, int which, const double* in);
/* termination_check (linear_system.cpp:47-53). */
gpk_status gpk_termination_check(gpk_batch* b, double tolerance, double* mean_norm,
                                 double* probe_norm, int* done);

/* ---- solvers (solvers.hpp:10-25) -------------------------------------- */
/* precond may be NULL (identity), as in solve_cg(batch, config, nullptr). */
gpk_status gpk_solve_cg(gpk_batch* b, const gpk_solver_config* c, gpk_precond* precond,
                        gpk_solver_report* report);
gpk_status gpk_solve_ap(gpk_batch* b, const gpk_solver_config* c, gpk_solver_report* report);
gpk_status gpk_solve_sgd(gpk_batch* b, const gpk_solver_config* c, gpk_solver_report* report);
/* Dispatch; builds the CG preconditioner internally (solvers.cpp:186-202). */
gpk_status gpk_solve(gpk_batch* b, const gpk_solver_config* c, gpk_solver_report* report);
/* Minibatch indices SGD iteration t of a solve with config c would use
 * (rng.cpp:108-126 on stream (seed, kSolver=6, substream)); out: count x b. */
gpk_status gpk_sgd_batches(gpk_ctx* ctx, int n, const gpk_solver_config* c, int first, int count,
                           int* out);

/* ---- gradient estimators (gradients.hpp:41-48) ------------------------ */
/* values, quadratic_term, trace_term: d+2 each (any may be NULL). */
gpk_status gpk_estimate_gradient_pathwise(gpk_operator* op, const double* v_y, const double* zhat,
                                          int s, double* values, double* quadratic_term,
                                          double* trace_term);
gpk_status gpk_estimate_gradient_standard(gpk_operator* op, const double* v_y,
                                          const double* solutions, const double* probes, int s,
                                          double* values, double* quadratic_term,
                                          double* trace_term);
/* The pathwise estimator on a batch's device-resident solutions (column 0 =
 * v_y, columns 1..s = zhat): the outer loop's call (outer_loop.cpp:198-201). */
gpk_status gpk_batch_gradient_pathwise(gpk_batch* b, double* values, double* quadratic_term,
                                       double* trace_term);

/* ---- RFF prior sampling (rff.hpp:27-54) ------------------------------- */
gpk_status gpk_rff_basis_build(gpk_ctx* ctx, int d, int m_pairs, int sample_count, uint64_t seed,
                               uint64_t substream, gpk_rff_basis** out);
gpk_status gpk_rff_basis_destroy(gpk_rff_basis* b);
/* base_frequencies m_pairs x d, weights 2 m_pairs x sample_count (col-major). */
gpk_status gpk_rff_basis_get(const gpk_rff_basis* b, double* base_frequencies, double* weights);
/* pathwise_targets (rff.cpp:64-79) at the operator's inputs and
 * hyperparameters; prior, noise, xi: n x s column-major (any may be NULL). */
gpk_status gpk_pathwise_targets(gpk_operator* op, gpk_rff_basis* basis, int s, uint64_t seed,
                                uint64_t substream, double* prior, double* noise, double* xi);

/* ---- posterior predictions (posterior.hpp:14-51) ---------------------- */
/* k(P, X) V for query points P (p x d, column-major), V n x m: cross_kernel_apply
 * (kernel.hpp:24-26, kernel.cpp:72-81); no noise term. out: p x m. */
gpk_status gpk_cross_apply(gpk_operator* op, const double* points, int p, const double* v, int m, double* out);
/* posterior mean k(P, X) v_y (posterior.cpp:11-17). out: p. */
gpk_status gpk_predict_mean(gpk_operator* op, const double* points, int p, const double* v_y, double* out);
/* pathwise posterior samples f_j(P) + k(P, X)(v_y - zhat_j), j < s, with f_j the
 * RFF prior draws of `basis` (posterior.cpp:19-27; basis NULL = zero prior).
 * zhat: n x s; out: p x s. */
gpk_status gpk_sample_posterior(gpk_operator* op, gpk_rff_basis* basis, const double* points, int p,
                                const double* v_y, const double* zhat, int s, double* out);
/* test_metrics (posterior.cpp:29-59): out4 = {rmse, llh, rmse_raw, llh_raw};
 * llh entries are NaN unless s >= 2 and a basis is given. */
gpk_status gpk_test_metrics(gpk_operator* op, gpk_rff_basis* basis, const double* points, int p,
                            const double* targets, const double* v_y, const double* zhat, int s, double target_scale,
                            double* out4);

/* ---- outer loop (outer_loop.hpp:37-90, optimise) ----------------------- */
typedef struct {
  int estimator;          /* 0 standard, 1 pathwise */
  gpk_solver_config solver;
  int warm_start;
  int steps;
  double learning_rate;   /* Adam, 0.1 */
  int probe_count;        /* s */
  int rff_pairs;
  int probe_distribution; /* 0 gaussian, 1 rademacher */
  uint64_t probe_seed, feature_seed, solver_seed;
  double init_value;      /* constrained init of every parameter */
  int divergence_policy;  /* 0 skip-and-halve, 1 abort */
  int prior_mode;         /* pathwise prior: 0 random features, 1 exact dense
                             (jittered Cholesky draws, n <= 4096; outer_loop.cpp:140-153) */
} gpk_outer_config;

/* One row per outer step (TraceRecord, trace.hpp:10-27, plus the full
 * gradient vector): constrained[d+2], gradient[d+2], then mean_norm,
 * probe_norm, epochs, grad_inf_norm, iterations, diverged, step_seconds,
 * solver_seconds. Row stride = 2*(d+2)+8 doubles. */
gpk_status gpk_optimise(gpk_ctx* ctx, const double* inputs, const double* targets, int n, int d,
                        const gpk_outer_config* config, const double* init_constrained,
                        double* trace, int* rows_written, double* final_raw, int* aborted);

/* The same outer loop as a resumable object: the dataset is uploaded once at
 * create; each gpk_optimiser_step call runs up to `steps` further outer
 * steps on the device-resident state (warm-start solutions, RFF basis, noise
 * draws, Adam moments) and writes one trace row per step taken. */
typedef struct gpk_optimiser gpk_optimiser;
gpk_status gpk_optimiser_create(gpk_ctx* ctx, const double* inputs, const double* targets, int n, int d,
                                const gpk_outer_config* config, const double* init_constrained,
                                gpk_optimiser** out);
gpk_status gpk_optimiser_step(gpk_optimiser* o, int steps, double* trace, int* rows_written);
/* raw: d+2 current raw hyperparameters; step: steps taken; aborted: run aborted. */
gpk_status gpk_optimiser_state(gpk_optimiser* o, double* raw, int* step, int* aborted);
gpk_status gpk_optimiser_destroy(gpk_optimiser* o);

/* ---- BASELINE.json synthetic data (not a reference API) ----------------
 * X ~ N(0, I) (uniform = 0) or U[-1, 1]^d (uniform = 1); y = sum_{k<4}
 * sin(x . w_k), w_k ~ N(0, I/d), plus N(0, noise^2); features and targets
 * standardised with the reference formula (data_io.cpp:148-168); draws from
 * Philox streams (seed, kSynthetic = 7, substream 0/1/2). Output FP32,
 * x row-major n x d. Bit-identical to oracle/gpiter_oracle.cpp's generator. */
gpk_status gpk_sinsum_dataset(int n, int d, int uniform, double noise, uint64_t seed, float* x_rowmajor,
                              float* y);

/* write_trace_csv (trace.cpp:20-44) for rows of gpk_optimise's trace: same
 * header, columns and shortest round-trip doubles (test columns empty). */
gpk_status gpk_write_trace_csv(const char* path, const double* trace, int rows, int d);

/* ---- exact marginal likelihood (row f4; exact.cpp, outer_loop.cpp:248-296)
 * optimise_exact: Adam on the exact MLL gradient (dense FP64 H, cuSOLVER
 * Cholesky + inverse, one fused pass sum_ij W_ij dH_ij/dtheta with
 * W = (alpha alpha^T - H^-1)/2). inputs column-major n x d; init_constrained
 * null = all 1.0; trajectory (nullable) steps x (d+2) constrained, row-major;
 * final_raw d+2. init_heuristic: the mean of optimise_exact fits on the
 * `subset` nearest rows (stable sort of squared distances) of n_centroids
 * centroids drawn from (seed, kCentroids = 9); subset >= n fits all rows. */
gpk_status gpk_optimise_exact(gpk_ctx* ctx, const double* inputs, const double* targets, int n, int d,
                              const double* init_constrained, int steps, double learning_rate, double* trajectory,
                              double* final_raw);
gpk_status gpk_init_heuristic(gpk_ctx* ctx, const double* inputs, const double* targets, int n, int d, int n_centroids,
                              int subset, uint64_t seed, int adam_steps, double learning_rate, double* constrained);

/* Batched SPD inverse used for the AP diagonal blocks (host buffers, batch
 * column-major dim x dim matrices). mode 1: recursive Schur complement with
 * strided-batched DGEMMs (the solver's default); mode 0: cuSOLVER
 * potrfBatched + two batched triangular solves. GPK_ENUMERIC if a matrix is
 * not positive definite. Exposed for testing the block solves. */
gpk_status gpk_spd_inverse(gpk_ctx* ctx, const double* mats, int dim, int batch, int mode, double* inv);

#ifdef __cplusplus
}
#endif
#endif /* GPK_H_ */
