// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// FP64 CPU restatement ("oracle") of the reference gpiter library
// (/root/reference/proj/core/src/*.cpp), written without Eigen because Eigen3
// is absent from this image (the reference cannot be built
// here). Every function cites the reference file:line it restates. Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
// may load this code; the product path (paper_2405_18457_b200/) never does.
//
// Parity pins: the Philox4x64-10 known-answer blocks, the Matérn-3/2 KATs and
// the softplus KAT of proj/tests/test_rng.cpp:10-38 / test_kernel.cpp:18-55,
// plus the reference's property tests restated in tests/test_oracle.py.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace oracle {

// Column-major dense matrix with the storage order of Eigen::MatrixXd.
struct Mat {
  int rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int r, int c, double v = 0.0) : rows(r), cols(c), a(static_cast<size_t>(r) * c, v) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(j) * rows + i]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(j) * rows + i]; }
  double* col(int j) { return a.data() + static_cast<size_t>(j) * rows; }
  const double* col(int j) const { return a.data() + static_cast<size_t>(j) * rows; }
  size_t size() const { return a.size(); }
  bool all_finite() const;
};
using Vec = std::vector<double>;

// ---- rng (proj/core/src/rng.cpp, proj/core/include/gpiter/rng.hpp) --------
std::array<uint64_t, 4> philox4x64(const std::array<uint64_t, 4>& counter,
                                   const std::array<uint64_t, 2>& key);

class RandomStream {
 public:
  RandomStream(uint64_t seed, uint64_t stream_id, uint64_t substream = 0)
      : key_{seed, stream_id}, counter_{0, substream, 0, 0} {}
  uint64_t next_u64();
  double next_double();
  double next_gaussian();
  uint64_t next_below(uint64_t bound);
  void fill_gaussian(double* data, size_t count);
  void fill_rademacher(double* data, size_t count);
  std::vector<int> permutation(int n);
  std::vector<int> sample_without_replacement(int n, int k);

 private:
  void refill();
  std::array<uint64_t, 2> key_;
  std::array<uint64_t, 4> counter_;
  std::array<uint64_t, 4> buffer_{};
  int buffer_pos_ = 4;
  double cached_gaussian_ = 0.0;
  bool has_cached_gaussian_ = false;
};

namespace streams {
constexpr uint64_t kSplit = 1, kProbes = 2, kFrequencies = 3, kWeights = 4, kNoiseDraws = 5,
                   kSolver = 6, kSynthetic = 7, kPriorSample = 8, kCentroids = 9;
}

// ---- hyperparameters (proj/core/src/hyperparameters.cpp) ------------------
double softplus(double x);
double softplus_inverse(double y);
double sigmoid(double x);

struct Hyper {
  Vec raw;  // [l_1..l_d, signal, noise], unconstrained
  int input_dim() const { return static_cast<int>(raw.size()) - 2; }
  int count() const { return static_cast<int>(raw.size()); }
  Vec constrained() const;
  Vec lengthscales() const;
  double signal_scale() const { return softplus(raw[raw.size() - 2]); }
  double noise_scale() const { return softplus(raw[raw.size() - 1]); }
  double noise_variance() const { double s = noise_scale(); return s * s; }
  static Hyper from_raw(Vec raw);
  static Hyper from_constrained(const Vec& c);
  static Hyper constant(int d, double v);
  void validate() const;
};

// ---- kernel operator (proj/core/src/kernel.cpp) ---------------------------
double matern32(const double* x, const double* x2, int d, const Hyper& hp);

struct Dataset {
  Mat inputs;  // n x d
  Vec targets;
  int n() const { return inputs.rows; }
  int dim() const { return inputs.cols; }
};

class KernelOperator {
 public:
  KernelOperator(const Dataset* data, Hyper hp, int block_rows = 1024, int threads = 1);
  int size() const { return n_; }
  const Hyper& params() const { return hp_; }
  const Dataset& data() const { return *data_; }
  Mat apply(const Mat& v) const;
  Mat apply_rows(const std::vector<int>& rows, const Mat& v) const;
  Mat apply_columns(int c0, int len, const Mat& u) const;
  Mat dense_block(int r0, int rows, int c0, int cols) const;
  Vec kernel_column(int i) const;
  Vec kernel_diagonal() const { return Vec(n_, signal_variance_); }
  Mat derivative_apply(int k, const Mat& v) const;
  std::vector<Vec> derivative_quadratic_forms_many(
      const std::vector<std::pair<const Mat*, const Mat*>>& pairs) const;
  double signal_variance() const { return signal_variance_; }
  double noise_variance() const { return noise_variance_; }
  int threads() const { return threads_; }
  int dim() const { return d_; }
  const double* scaled_inputs() const { return xs_.data(); }  // row-major n x d
  const Vec& inverse_lengthscales() const { return inv_ls_; }

 private:
  void fill_rows(int row0, int count, double* out) const;
  void fill_row(int i, double* out) const;
  const Dataset* data_;
  Hyper hp_;
  int block_rows_, threads_;
  int n_ = 0, d_ = 0;
  Vec inv_ls_;
  std::vector<double> xs_;  // scaled inputs, row-major n x d (values == Eigen col-major copy)
  std::vector<double> xst_;  // the same, dimension-major d x n
  double signal_variance_ = 0.0, noise_variance_ = 0.0;
};

// ---- linear systems + solvers (linear_system.cpp, solvers.cpp) ------------
enum SolverKind { CG = 0, AP = 1, SGD = 2 };

struct SolverConfig {
  int kind = CG;
  double tolerance = 0.01;
  int max_epochs = 50;
  int block_size = 1000;
  int batch_size = 500;
  double learning_rate = 30.0;
  double momentum = 0.9;
  int preconditioner_rank = 100;
  bool warm_start = false;
  uint64_t seed = 0;
  uint64_t substream = 0;
  void validate() const;
};

struct SolverReport {
  int iterations = 0;
  double epochs_consumed = 0.0;
  double mean_residual_norm = 0.0;
  double probe_residual_norm = 0.0;
  bool reached_tolerance = false;
  bool residuals_estimated = false;
  bool aborted = false;
  std::string abort_reason;
  double wall_seconds = 0.0;
};

struct LinearSystemBatch {
  static constexpr double kNormEpsilon = 1e-12;
  const KernelOperator* op = nullptr;
  Mat targets, solutions, residuals;
  Vec scales;
  LinearSystemBatch(const KernelOperator& op, Mat targets);
  int columns() const { return targets.cols; }
  int probe_count() const { return columns() - 1; }
  void warm_start(const Mat& prev);
  void refresh_residuals();
  double mean_residual_norm() const;
  double probe_residual_norm() const;
};

struct TerminationStatus { double mean_norm = 0, probe_norm = 0; bool done = false; };
TerminationStatus termination_check(const LinearSystemBatch& b, double tol);

// Dense Cholesky (lower), stands in for Eigen::LLT.
struct LLT {
  int n = 0;
  Mat L;
  bool ok = false;
  void compute(const Mat& a);
  Mat solve(const Mat& b) const;
};

class PivotedCholesky {
 public:
  PivotedCholesky(const KernelOperator& op, int rank);
  int achieved_rank() const { return achieved_rank_; }
  bool stopped_early() const { return stopped_early_; }
  const Mat& factor() const { return factor_; }
  const std::vector<int>& pivots() const { return pivots_; }
  Mat apply(const Mat& v) const;

 private:
  Mat factor_;
  LLT small_;
  double noise_variance_ = 0.0;
  int achieved_rank_ = 0;
  bool stopped_early_ = false;
  std::vector<int> pivots_;
};

SolverReport solve_cg(LinearSystemBatch& b, const SolverConfig& c, const PivotedCholesky* p);
SolverReport solve_ap(LinearSystemBatch& b, const SolverConfig& c);
SolverReport solve_sgd(LinearSystemBatch& b, const SolverConfig& c,
                       std::vector<std::vector<int>>* batches_out = nullptr, int record = 0);
SolverReport solve(LinearSystemBatch& b, const SolverConfig& c);

// ---- gradients (gradients.cpp) --------------------------------------------
struct GradientEstimate { Vec values, quadratic_term, trace_term; };
Mat gen_standard_probes(int n, int s, uint64_t seed, int distribution, uint64_t substream);
GradientEstimate estimate_gradient_standard(const KernelOperator& op, const Vec& v_y,
                                            const Mat& solutions, const Mat& probes);
GradientEstimate estimate_gradient_pathwise(const KernelOperator& op, const Vec& v_y,
                                            const Mat& zhat);

// ---- rff (rff.cpp) -------------------------------------------------------
struct RffBasis {
  Mat base_frequencies;  // P x d
  Mat weights;           // 2P x S
  uint64_t seed = 0;
  int pairs() const { return base_frequencies.rows; }
};
RffBasis build_rff_basis(int d, int m_pairs, int sample_count, uint64_t seed, uint64_t substream);
Mat rff_features(const RffBasis& basis, const Hyper& hp, const Mat& points);
struct PathwiseTargets { Mat prior_values, noise, xi; };
// rff.cpp:81-91: xi = prior + sigma * eps, eps from (seed, kNoiseDraws, substream)
PathwiseTargets pathwise_targets_from_prior(const Mat& prior_values, const Hyper& hp, uint64_t seed,
                                            uint64_t substream);
// exact.cpp:52-61: lower Cholesky factor of K + jitter * mean(diag K) I, jitter
// 1e-10, 1e-9, ..., 1e-6 (first success); throws beyond 1e-6
Mat jittered_kernel_cholesky(const Mat& kernel_matrix);
constexpr int kDefaultDenseCap = 4096;  // exact.hpp:24
class KernelOperator;
// ExactDense prior values (outer_loop.cpp:149-152): L W with L the jittered
// Cholesky factor of dense(H) - sigma^2 I and W the n x s weights.
Mat exact_dense_prior(const KernelOperator& op, const Hyper& hp, const Mat& weights);
PathwiseTargets pathwise_targets(const RffBasis& basis, const Hyper& hp, const Dataset& data,
                                 int s, uint64_t seed, uint64_t substream);

// ---- posterior (kernel.cpp:57-81, rff.cpp:56-62, posterior.cpp:11-59) ----
// k(P, X) V for m columns, row tiles of block_rows (cross_kernel_apply).
Mat cross_kernel_apply(const Mat& points, const Mat& inputs, const Hyper& hp, const Mat& v, int block_rows = 1024,
                       int threads = 1);
// prior sample j at points: rff_features(points) W[:, j] (evaluate_prior), all j < s.
Mat evaluate_prior_all(const RffBasis& basis, const Hyper& hp, const Mat& points, int s);
// f_j(P) + k(P, X)(v_y - zhat_j) for every j < s (sample_posterior); prior may be empty (zero prior).
Mat sample_posterior_all(const Mat& prior, const Mat& points, const Mat& inputs, const Hyper& hp, const Vec& v_y,
                         const Mat& zhat, int threads = 1);
struct TestMetrics { double rmse = 0, llh = 0, rmse_raw = 0, llh_raw = 0; bool has_llh = false; };
TestMetrics test_metrics(const Mat& prior, const Mat& points, const Vec& targets, const Mat& inputs, const Hyper& hp,
                         const Vec& v_y, const Mat& zhat, double target_scale, int threads = 1);

// ---- outer loop (outer_loop.cpp:39-246) ----------------------------------
struct OuterConfig {
  int estimator = 1;  // 0 standard, 1 pathwise
  SolverConfig solver;
  bool warm_start = false;
  int steps = 100;
  double learning_rate = 0.1;
  int probe_count = 64;
  int rff_pairs = 1000;
  int probe_distribution = 0;  // 0 gaussian, 1 rademacher
  uint64_t probe_seed = 0, feature_seed = 0, solver_seed = 0;
  Vec init_constrained;  // empty: all init_value
  double init_value = 1.0;
  int divergence_policy = 0;  // 0 skip-and-halve, 1 abort
  int prior_mode = 0;         // 0 random features, 1 exact dense (outer_loop.cpp:134-154)
};

struct TraceRow {
  int step = 0;
  Vec constrained;
  Vec gradient;  // full constrained gradient (the reference logs only its inf-norm)
  double mean_residual_norm = 0, probe_residual_norm = 0, epochs = 0, grad_inf_norm = 0;
  int iterations = 0;
  bool solver_diverged = false;
};

struct OuterResult {
  Hyper hp;
  std::vector<TraceRow> trace;
  bool aborted = false;
  std::string abort_reason;
};

OuterResult optimise(const Dataset& train, const OuterConfig& config, int threads = 1,
                     int block_rows = 1024);

// ---- exact dense reference (exact.cpp), test scaffolding only -------------
struct DenseProblem { Hyper hp; Mat h; LLT chol; std::vector<Mat> dh; };
DenseProblem build_dense_problem(const Dataset& data, const Hyper& hp);
double exact_mll(const DenseProblem& dense, const Vec& y);
Vec exact_gradient(const DenseProblem& dense, const Vec& y);

// outer_loop.cpp:248-262: Adam on the exact marginal likelihood
struct ExactTrajectory { Hyper hp; std::vector<Vec> constrained_per_step; };
ExactTrajectory optimise_exact(const Dataset& data, const Hyper& init, int steps, double learning_rate);
// outer_loop.cpp:264-296: average of optimise_exact fits on the `subset`
// nearest rows (stable sort by squared distance) of n_centroids centroids
// drawn from (seed, kCentroids = 9, 0); subset >= n fits the whole set.
Hyper init_heuristic(const Dataset& data, int n_centroids, int subset, uint64_t seed, int adam_steps,
                     double learning_rate);

// ---- BASELINE.json synthetic sin-sum generator (not in the reference) -----
// X ~ N(0,I) (uniform=false) or U[-1,1]^d; y = sum_{k<4} sin(x.w_k), w_k ~ N(0, I/d),
// + N(0, noise^2); y standardised with the reference formula
// (proj/core/src/data_io.cpp:148-168: mean, population std, clamp 0 -> 1).
// Inputs are rounded to FP32 (the dataset file format); targets too.
void make_sinsum_dataset(int n, int d, bool uniform, double noise, uint64_t seed,
                         std::vector<float>& x_rowmajor, std::vector<float>& y);

// ---- oracle-at-scale hook (oracle/gpu/, test infrastructure) -------------
// The CPU oracle leaves this null. liboracle_gpu.so (the same restatement
// linked with oracle/gpu/oracle_gpu.cu) sets it, and the O(n^2) passes below
// then run as naive FP64 CUDA restatements of the same loops (same sums, not
// the same summation order), so the BASELINE configurations C4/C5 whose CPU
// cost is 1e13..1e15 flops per epoch can be run through the unchanged
// optimise / solve_* / estimator code. Each hook returns false to decline
// (the CPU code then runs).
struct OracleBackend {
  // out = H[rows, :] v, rows == nullptr: all n rows (kernel.cpp:133-168)
  bool (*apply)(const KernelOperator& op, const int* rows, int count, const Mat& v, Mat& out);
  // derivative_quadratic_forms_many (kernel.cpp:238-272)
  bool (*quad_forms)(const KernelOperator& op, const std::vector<std::pair<const Mat*, const Mat*>>& pairs,
                     std::vector<Vec>& out);
  // rff prior values rff_features(X) W[:, :s] (rff.cpp:64-73)
  bool (*prior)(const RffBasis& basis, const Hyper& hp, const Dataset& data, int s, Mat& prior);
  // solve_sgd (solvers.cpp:147-184) with the n x m state device-resident
  bool (*solve_sgd)(LinearSystemBatch& b, const SolverConfig& c, SolverReport& rep,
                    std::vector<std::vector<int>>* batches_out, int record);
};
extern const OracleBackend* g_backend;
// Test knob: stop solve_sgd after this many iterations (-1: the epoch budget only).
extern int g_sgd_iteration_cap;
// Sensitivity knobs for apply() (the full H.V product; tests only):
// g_apply_order 1 sums each output in descending column order; g_apply_noise
// eps multiplies every output entry by 1 + eps u, u uniform in [-1, 1).
extern int g_apply_order;
extern double g_apply_noise;

}  // namespace oracle
