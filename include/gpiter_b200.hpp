// gpiter_b200.hpp — header-only C++ drop-in for the reference's hot-path API
// (/root/reference/proj/core/include/gpiter/{kernel,linear_system,solvers,
// pivoted_cholesky,gradients,rff,outer_loop}.hpp) implemented over the C-ABI
// in gpk.h. Same class and function names, same argument meaning, same
// exception types (std::invalid_argument / std::out_of_range /
// std::runtime_error); matrices are column-major FP64 like Eigen::MatrixXd.
// A caller that used gpiter::KernelOperator / solve_cg / ... switches by
// including this header and linking libgpk.so; Eigen is not required (Matrix
// below is a minimal column-major container; an Eigen::MatrixXd's data()
// pointer can be passed to the raw-pointer overloads directly).
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gpk.h"

namespace gpiter_b200 {

inline void check(gpk_status st) {
  if (st == GPK_OK) return;
  const std::string msg = gpk_last_error();
  switch (st) {
    case GPK_EINVAL: throw std::invalid_argument(msg);
    case GPK_ERANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
  }
}

// Column-major FP64 matrix (storage order of Eigen::MatrixXd).
struct Matrix {
  int rows = 0, cols = 0;
  std::vector<double> a;
  Matrix() = default;
  Matrix(int r, int c, double v = 0.0) : rows(r), cols(c), a(static_cast<size_t>(r) * c, v) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(j) * rows + i]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(j) * rows + i]; }
  double* data() { return a.data(); }
  const double* data() const { return a.data(); }
};
using Vector = std::vector<double>;

class Context {
 public:
  explicit Context(int device = 0) { check(gpk_ctx_create(device, &ctx_)); }
  ~Context() { gpk_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  gpk_ctx* get() const { return ctx_; }

 private:
  gpk_ctx* ctx_ = nullptr;
};

// Hyperparameters (hyperparameters.hpp:19-49): raw [l_1..l_d, signal, noise].
struct Hyperparameters {
  Vector raw;
  int input_dim() const { return static_cast<int>(raw.size()) - 2; }
  int count() const { return static_cast<int>(raw.size()); }
};

// KernelOperatorOptions (kernel.hpp:27-30); block_rows has no meaning here
// (no tile of H is materialised), dense_cache selects FP64 full products.
struct KernelOperatorOptions {
  int block_rows = 1024;
  bool dense_cache = false;
};

// KernelOperator (kernel.hpp:37-97). `inputs` is the Dataset's n x d matrix.
class KernelOperator {
 public:
  KernelOperator(Context& ctx, const Matrix& inputs, const Hyperparameters& hp,
                 KernelOperatorOptions options = {})
      : hp_(hp) {
    if (static_cast<int>(hp.raw.size()) != inputs.cols + 2)
      throw std::invalid_argument("KernelOperator: dataset dimension does not match hyperparameters");
    check(gpk_operator_create(ctx.get(), inputs.data(), inputs.rows, inputs.cols, hp.raw.data(), &op_));
    n_ = inputs.rows;
    if (options.dense_cache) check(gpk_operator_set_dense_cache(op_, 1));
  }
  ~KernelOperator() { gpk_operator_destroy(op_); }
  KernelOperator(const KernelOperator&) = delete;
  KernelOperator& operator=(const KernelOperator&) = delete;

  int size() const { return n_; }
  int param_count() const { return hp_.count(); }
  const Hyperparameters& params() const { return hp_; }
  gpk_operator* get() const { return op_; }

  Matrix apply(const Matrix& v) const {
    if (v.rows != n_) throw std::invalid_argument("KernelOperator::apply: dimension mismatch");
    Matrix out(n_, v.cols);
    check(gpk_apply(op_, v.data(), v.cols, out.data()));
    return out;
  }
  Matrix apply_rows(const std::vector<int>& rows, const Matrix& v) const {
    Matrix out(static_cast<int>(rows.size()), v.cols);
    check(gpk_apply_rows(op_, rows.data(), static_cast<int>(rows.size()), v.data(), v.cols, out.data()));
    return out;
  }
  Matrix apply_columns(int c0, int len, const Matrix& u) const {
    if (u.rows != len) throw std::invalid_argument("KernelOperator::apply_columns: height mismatch");
    Matrix out(n_, u.cols);
    check(gpk_apply_columns(op_, c0, len, u.data(), u.cols, out.data()));
    return out;
  }
  Matrix dense_block(int r0, int rows, int c0, int cols) const {
    Matrix out(rows, cols);
    check(gpk_dense_block(op_, r0, rows, c0, cols, out.data()));
    return out;
  }
  Matrix dense() const { return dense_block(0, n_, 0, n_); }
  // kernel.hpp:71 -- std::out_of_range for a parameter index outside [0, d + 2)
  Matrix derivative_apply(int k, const Matrix& v) const {
    if (v.rows != n_) throw std::invalid_argument("KernelOperator::derivative_apply: dimension mismatch");
    Matrix out(n_, v.cols);
    check(gpk_derivative_apply(op_, k, v.data(), v.cols, out.data()));
    return out;
  }
  Vector kernel_column(int i) const {
    Vector out(n_);
    check(gpk_kernel_column(op_, i, out.data()));
    return out;
  }
  Vector kernel_diagonal() const {
    Vector out(n_);
    check(gpk_kernel_diagonal(op_, out.data()));
    return out;
  }
  std::vector<Vector> derivative_quadratic_forms_many(
      const std::vector<std::pair<const Matrix*, const Matrix*>>& pairs) const {
    std::vector<const double*> u, w;
    std::vector<int> cols;
    for (const auto& p : pairs) {
      if (p.first->rows != n_ || p.second->rows != n_ || p.first->cols != p.second->cols)
        throw std::invalid_argument("derivative_quadratic_forms: shape mismatch");
      u.push_back(p.first->data());
      w.push_back(p.first == p.second ? p.first->data() : p.second->data());
      cols.push_back(p.first->cols);
    }
    std::vector<double> out(pairs.size() * hp_.count());
    check(gpk_derivative_quadratic_forms_many(op_, static_cast<int>(pairs.size()), u.data(), w.data(), cols.data(),
                                              out.data()));
    std::vector<Vector> res;
    for (size_t p = 0; p < pairs.size(); ++p)
      res.emplace_back(out.begin() + p * hp_.count(), out.begin() + (p + 1) * hp_.count());
    return res;
  }
  Vector derivative_quadratic_forms(const Matrix& u, const Matrix& w) const {
    return derivative_quadratic_forms_many({{&u, &w}}).front();
  }

 private:
  gpk_operator* op_ = nullptr;
  Hyperparameters hp_;
  int n_ = 0;
};

// PivotedCholeskyPreconditioner (pivoted_cholesky.hpp:13-32).
class PivotedCholeskyPreconditioner {
 public:
  PivotedCholeskyPreconditioner(const KernelOperator& op, int rank) : n_(op.size()) {
    check(gpk_precond_create(op.get(), rank, &p_));
  }
  ~PivotedCholeskyPreconditioner() { gpk_precond_destroy(p_); }
  PivotedCholeskyPreconditioner(const PivotedCholeskyPreconditioner&) = delete;
  PivotedCholeskyPreconditioner& operator=(const PivotedCholeskyPreconditioner&) = delete;
  int achieved_rank() const {
    int r = 0, s = 0;
    check(gpk_precond_info(p_, &r, &s));
    return r;
  }
  bool stopped_early() const {
    int r = 0, s = 0;
    check(gpk_precond_info(p_, &r, &s));
    return s != 0;
  }
  Matrix factor() const {
    Matrix f(n_, achieved_rank());
    check(gpk_precond_factor(p_, f.data(), nullptr));
    return f;
  }
  Matrix apply(const Matrix& v) const {
    Matrix out(v.rows, v.cols);
    check(gpk_precond_apply(p_, v.data(), v.cols, out.data()));
    return out;
  }
  gpk_precond* get() const { return p_; }

 private:
  gpk_precond* p_ = nullptr;
  int n_;
};

enum class SolverKind { CG = GPK_CG, AP = GPK_AP, SGD = GPK_SGD };

// SolverConfig / SolverReport (linear_system.hpp:14-40).
struct SolverConfig {
  SolverKind kind = SolverKind::CG;
  double tolerance = 0.01;
  int max_epochs = 50;
  int block_size = 1000;
  int batch_size = 500;
  double learning_rate = 30.0;
  double momentum = 0.9;
  int preconditioner_rank = 100;
  bool warm_start = false;
  std::uint64_t seed = 0;
  std::uint64_t substream = 0;
  gpk_solver_config c() const {
    return gpk_solver_config{static_cast<int>(kind), tolerance, max_epochs, block_size, batch_size, learning_rate,
                             momentum, preconditioner_rank, warm_start ? 1 : 0, seed, substream};
  }
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
  static SolverReport from(const gpk_solver_report& r) {
    SolverReport o;
    o.iterations = r.iterations;
    o.epochs_consumed = r.epochs_consumed;
    o.mean_residual_norm = r.mean_residual_norm;
    o.probe_residual_norm = r.probe_residual_norm;
    o.reached_tolerance = r.reached_tolerance != 0;
    o.residuals_estimated = r.residuals_estimated != 0;
    o.aborted = r.aborted != 0;
    o.abort_reason = r.abort_reason;
    o.wall_seconds = r.wall_seconds;
    return o;
  }
};

// LinearSystemBatch (linear_system.hpp:45-68): device-resident targets,
// solutions and residuals; the accessors copy to the host.
class LinearSystemBatch {
 public:
  LinearSystemBatch(const KernelOperator& op, const Matrix& targets) : n_(op.size()), m_(targets.cols) {
    if (targets.rows != op.size())
      throw std::invalid_argument("LinearSystemBatch: target height does not match operator");
    check(gpk_batch_create(op.get(), targets.data(), targets.cols, &b_));
  }
  ~LinearSystemBatch() { gpk_batch_destroy(b_); }
  LinearSystemBatch(const LinearSystemBatch&) = delete;
  LinearSystemBatch& operator=(const LinearSystemBatch&) = delete;
  int columns() const { return m_; }
  int probe_count() const { return m_ - 1; }
  void warm_start(const Matrix& previous) {
    if (previous.rows != n_ || previous.cols != m_)
      throw std::invalid_argument("LinearSystemBatch::warm_start: shape mismatch");
    check(gpk_batch_warm_start(b_, previous.data()));
  }
  void refresh_residuals() { check(gpk_batch_refresh_residuals(b_)); }
  Matrix targets() const { return get(0); }
  Matrix solutions() const { return get(1); }
  Matrix residuals() const { return get(2); }
  Vector scales() const {
    Vector s(m_);
    check(gpk_batch_get(b_, 3, s.data()));
    return s;
  }
  gpk_batch* get() const { return b_; }

 private:
  Matrix get(int which) const {
    Matrix out(n_, m_);
    check(gpk_batch_get(b_, which, out.data()));
    return out;
  }
  gpk_batch* b_ = nullptr;
  int n_, m_;
};

struct TerminationStatus {
  double mean_norm = 0.0, probe_norm = 0.0;
  bool done = false;
};
inline TerminationStatus termination_check(const LinearSystemBatch& b, double tolerance) {
  TerminationStatus s;
  int done = 0;
  check(gpk_termination_check(b.get(), tolerance, &s.mean_norm, &s.probe_norm, &done));
  s.done = done != 0;
  return s;
}

// solvers.hpp:10-25
inline SolverReport solve_cg(LinearSystemBatch& b, const SolverConfig& c,
                             const PivotedCholeskyPreconditioner* precond = nullptr) {
  gpk_solver_report r{};
  const gpk_solver_config cc = c.c();
  check(gpk_solve_cg(b.get(), &cc, precond ? precond->get() : nullptr, &r));
  return SolverReport::from(r);
}
inline SolverReport solve_ap(LinearSystemBatch& b, const SolverConfig& c) {
  gpk_solver_report r{};
  const gpk_solver_config cc = c.c();
  check(gpk_solve_ap(b.get(), &cc, &r));
  return SolverReport::from(r);
}
inline SolverReport solve_sgd(LinearSystemBatch& b, const SolverConfig& c) {
  gpk_solver_report r{};
  const gpk_solver_config cc = c.c();
  check(gpk_solve_sgd(b.get(), &cc, &r));
  return SolverReport::from(r);
}
inline SolverReport solve(LinearSystemBatch& b, const SolverConfig& c) {
  gpk_solver_report r{};
  const gpk_solver_config cc = c.c();
  check(gpk_solve(b.get(), &cc, &r));
  return SolverReport::from(r);
}

// gradients.hpp:34-48
struct GradientEstimate {
  Vector values, quadratic_term, trace_term;
};
inline GradientEstimate estimate_gradient_pathwise(const KernelOperator& op, const Vector& v_y, const Matrix& zhat) {
  if (zhat.rows != op.size()) throw std::invalid_argument("estimate_gradient_pathwise: shape mismatch");
  GradientEstimate g;
  const int k = op.param_count();
  g.values.resize(k);
  g.quadratic_term.resize(k);
  g.trace_term.resize(k);
  check(gpk_estimate_gradient_pathwise(op.get(), v_y.data(), zhat.data(), zhat.cols, g.values.data(),
                                       g.quadratic_term.data(), g.trace_term.data()));
  return g;
}
inline GradientEstimate estimate_gradient_standard(const KernelOperator& op, const Vector& v_y,
                                                   const Matrix& solutions, const Matrix& probes) {
  if (solutions.rows != op.size() || probes.rows != op.size() || solutions.cols != probes.cols)
    throw std::invalid_argument("estimate_gradient_standard: shape mismatch");
  GradientEstimate g;
  const int k = op.param_count();
  g.values.resize(k);
  g.quadratic_term.resize(k);
  g.trace_term.resize(k);
  check(gpk_estimate_gradient_standard(op.get(), v_y.data(), solutions.data(), probes.data(), solutions.cols,
                                       g.values.data(), g.quadratic_term.data(), g.trace_term.data()));
  return g;
}

// rff.hpp:27-54
class RffBasis {
 public:
  RffBasis(Context& ctx, int input_dim, int m_pairs, int sample_count, std::uint64_t seed,
           std::uint64_t substream = 0)
      : d_(input_dim), pairs_(m_pairs), samples_(sample_count) {
    check(gpk_rff_basis_build(ctx.get(), input_dim, m_pairs, sample_count, seed, substream, &b_));
  }
  ~RffBasis() { gpk_rff_basis_destroy(b_); }
  RffBasis(const RffBasis&) = delete;
  RffBasis& operator=(const RffBasis&) = delete;
  int pairs() const { return pairs_; }
  int input_dim() const { return d_; }
  int sample_count() const { return samples_; }
  gpk_rff_basis* get() const { return b_; }

 private:
  gpk_rff_basis* b_ = nullptr;
  int d_, pairs_, samples_;
};

struct PathwiseTargets {
  Matrix prior_values, noise, xi;
};
inline PathwiseTargets pathwise_targets(const RffBasis& basis, const KernelOperator& op, int s, std::uint64_t seed,
                                        std::uint64_t substream = 0) {
  PathwiseTargets t{Matrix(op.size(), s), Matrix(op.size(), s), Matrix(op.size(), s)};
  check(gpk_pathwise_targets(op.get(), basis.get(), s, seed, substream, t.prior_values.data(), t.noise.data(),
                             t.xi.data()));
  return t;
}

}  // namespace gpiter_b200
