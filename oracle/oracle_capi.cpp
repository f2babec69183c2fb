// TEST INFRASTRUCTURE — NOT PRODUCT CODE. Flat C entry points over the FP64
// oracle for ctypes (tests/, smoke(), bench.py's CPU arms only). All matrices
// are column-major FP64 (Eigen::MatrixXd layout) unless stated otherwise.
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "gpiter_oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

Dataset make_data(const double* x, const double* y, int n, int d) {
  Dataset ds;
  ds.inputs = Mat(n, d);
  std::memcpy(ds.inputs.a.data(), x, sizeof(double) * n * d);
  ds.targets.assign(n, 0.0);
  if (y) std::memcpy(ds.targets.data(), y, sizeof(double) * n);
  return ds;
}
Mat make_mat(const double* p, int r, int c) {
  Mat m(r, c);
  if (p) std::memcpy(m.a.data(), p, sizeof(double) * r * c);
  return m;
}
Hyper make_hp(const double* raw, int d) { return Hyper::from_raw(Vec(raw, raw + d + 2)); }
void put(const Mat& m, double* out) { std::memcpy(out, m.a.data(), sizeof(double) * m.size()); }

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

struct ReportC {
  int iterations;
  double epochs_consumed, mean_residual_norm, probe_residual_norm;
  int reached_tolerance, residuals_estimated, aborted;
  char abort_reason[128];
  double wall_seconds;
};
void fill_report(const SolverReport& r, ReportC* out) {
  out->iterations = r.iterations;
  out->epochs_consumed = r.epochs_consumed;
  out->mean_residual_norm = r.mean_residual_norm;
  out->probe_residual_norm = r.probe_residual_norm;
  out->reached_tolerance = r.reached_tolerance;
  out->residuals_estimated = r.residuals_estimated;
  out->aborted = r.aborted;
  std::strncpy(out->abort_reason, r.abort_reason.c_str(), 127);
  out->abort_reason[127] = 0;
  out->wall_seconds = r.wall_seconds;
}

struct SolverConfigC {
  int kind;
  double tolerance;
  int max_epochs, block_size, batch_size;
  double learning_rate, momentum;
  int preconditioner_rank, warm_start;
  unsigned long long seed, substream;
};
SolverConfig to_cfg(const SolverConfigC* c) {
  SolverConfig s;
  s.kind = c->kind;
  s.tolerance = c->tolerance;
  s.max_epochs = c->max_epochs;
  s.block_size = c->block_size;
  s.batch_size = c->batch_size;
  s.learning_rate = c->learning_rate;
  s.momentum = c->momentum;
  s.preconditioner_rank = c->preconditioner_rank;
  s.warm_start = c->warm_start != 0;
  s.seed = c->seed;
  s.substream = c->substream;
  return s;
}
}  // namespace

extern "C" {

void oracle_set_sgd_iteration_cap(int cap) { g_sgd_iteration_cap = cap; }
void oracle_set_apply_sensitivity(int order, double noise) {
  g_apply_order = order;
  g_apply_noise = noise;
}

const char* oracle_last_error() { return g_err.c_str(); }

void oracle_philox(const unsigned long long* counter, const unsigned long long* key, unsigned long long* out) {
  const auto r = philox4x64({counter[0], counter[1], counter[2], counter[3]}, {key[0], key[1]});
  for (int i = 0; i < 4; ++i) out[i] = r[i];
}

// Draws `count` items of `kind` (0 u64, 1 double, 2 gaussian, 3 below(bound), 4 rademacher)
// from RandomStream(seed, stream, substream).
void oracle_stream_draw(unsigned long long seed, unsigned long long stream, unsigned long long substream,
                        int kind, unsigned long long bound, long long count, void* out) {
  RandomStream s(seed, stream, substream);
  for (long long i = 0; i < count; ++i) {
    switch (kind) {
      case 0: static_cast<unsigned long long*>(out)[i] = s.next_u64(); break;
      case 1: static_cast<double*>(out)[i] = s.next_double(); break;
      case 2: static_cast<double*>(out)[i] = s.next_gaussian(); break;
      case 3: static_cast<unsigned long long*>(out)[i] = s.next_below(bound); break;
      default: static_cast<double*>(out)[i] = (s.next_u64() & 1u) ? 1.0 : -1.0; break;
    }
  }
}

// `rounds` successive Floyd samples of k from n on one stream, concatenated.
int oracle_sample_without_replacement(unsigned long long seed, unsigned long long stream,
                                      unsigned long long substream, int n, int k, int rounds, int* out) {
  return guarded([&] {
    RandomStream s(seed, stream, substream);
    for (int r = 0; r < rounds; ++r) {
      const auto v = s.sample_without_replacement(n, k);
      std::memcpy(out + static_cast<size_t>(r) * k, v.data(), sizeof(int) * k);
    }
  });
}

int oracle_permutation(unsigned long long seed, unsigned long long stream, int n, int* out) {
  return guarded([&] {
    RandomStream s(seed, stream, 0);
    const auto v = s.permutation(n);
    std::memcpy(out, v.data(), sizeof(int) * n);
  });
}

double oracle_softplus(double x) { return softplus(x); }
int oracle_softplus_inverse(double y, double* out) { return guarded([&] { *out = softplus_inverse(y); }); }
double oracle_sigmoid(double x) { return sigmoid(x); }

int oracle_matern32(const double* x, const double* x2, int d, const double* raw, double* out) {
  return guarded([&] { *out = matern32(x, x2, d, make_hp(raw, d)); });
}

int oracle_apply(const double* x, int n, int d, const double* raw, const double* v, int m, double* out,
                 int block_rows, int threads) {
  return guarded([&] {
    const Dataset ds = make_data(x, nullptr, n, d);
    KernelOperator op(&ds, make_hp(raw, d), block_rows, threads);
    put(op.apply(make_mat(v, n, m)), out);
  });
}

int oracle_apply_rows(const double* x, int n, int d, const double* raw, const int* rows, int count,
                      const double* v, int m, double* out, int threads) {
  return guarded([&] {
    const Dataset ds = make_data(x, nullptr, n, d);
    KernelOperator op(&ds, make_hp(raw, d), 1024, threads);
    put(op.apply_rows(std::vector<int>(rows, rows + count), make_mat(v, n, m)), out);
  });
}

int oracle_apply_columns(const double* x, int n, int d, const double* raw, int c0, int len,
                         const double* u, int m, double* out, int threads) {
  return guarded([&] {
    const Dataset ds = make_data(x, nullptr, n, d);
    KernelOperator op(&ds, make_hp(raw, d), 1024, threads);
    put(op.apply_columns(c0, len, make_mat(u, len, m)), out);
  });
}

int oracle_dense_block(const double* x, int n, int d, const double* raw, int r0, int rows, int c0,
                       int cols, double* out) {
  return guarded([&] {
    const Dataset ds = make_data(x, nullptr, n, d);
    KernelOperator op(&ds, make_hp(raw, d));
    put(op.dense_block(r0, rows, c0, cols), out);
  });
}

int oracle_kernel_column(const double* x, int n, int d, const double* raw, int i, double* out) {
  return guarded([&] {
    const Dataset ds = make_data(x, nullptr, n, d);
    KernelOperator op(&ds, make_hp(raw, d));
    const Vec c = op.kernel_column(i);
    std::memcpy(out, c.data(), sizeof(double) * n);
  });
}

int oracle_derivative_apply(const double* x, int n, int d, const double* raw, int k, const double* v,
                            int m, double* out) {
  return guarded([&] {
    const Dataset ds = make_data(x, nullptr, n, d);
    KernelOperator op(&ds, make_hp(raw, d));
    put(op.derivative_apply(k, make_mat(v, n, m)), out);
  });
}

// Two pairs (U1,W1) (U2,W2), the shape `assemble` uses; out = 2*(d+2).
int oracle_quad_forms(const double* x, int n, int d, const double* raw, const double* u1,
                      const double* w1, int m1, const double* u2, const double* w2, int m2,
                      double* out, int threads) {
  return guarded([&] {
    const Dataset ds = make_data(x, nullptr, n, d);
    KernelOperator op(&ds, make_hp(raw, d), 1024, threads);
    const Mat U1 = make_mat(u1, n, m1), W1 = make_mat(w1, n, m1);
    const Mat U2 = make_mat(u2, n, m2), W2 = make_mat(w2, n, m2);
    const auto f = op.derivative_quadratic_forms_many({{&U1, &W1}, {&U2, &W2}});
    for (int k = 0; k < d + 2; ++k) {
      out[k] = f[0][k];
      out[d + 2 + k] = f[1][k];
    }
  });
}

// Builds the preconditioner, returns factor (n x rank_out col-major; caller
// allocates n x rank), pivots, and P^-1 v for v (n x m).
int oracle_precond(const double* x, int n, int d, const double* raw, int rank, const double* v, int m,
                   double* pv, double* factor, int* pivots, int* achieved) {
  return guarded([&] {
    const Dataset ds = make_data(x, nullptr, n, d);
    KernelOperator op(&ds, make_hp(raw, d));
    PivotedCholesky pc(op, rank);
    *achieved = pc.achieved_rank();
    if (factor) put(pc.factor(), factor);
    if (pivots) std::memcpy(pivots, pc.pivots().data(), sizeof(int) * pc.pivots().size());
    if (v && pv) put(pc.apply(make_mat(v, n, m)), pv);
  });
}

// Runs one solver call. targets n x m; warm (nullable) n x m initial
// solutions; outputs solutions and residuals n x m. precond_rank < 0 means
// "dispatch through solve()" (CG builds its own preconditioner); >= 0 calls
// solve_cg with that explicit rank (0 => rank-0 preconditioner object).
int oracle_solve(const double* x, int n, int d, const double* raw, const double* targets, int m,
                 const double* warm, const SolverConfigC* cfg, int explicit_rank, double* solutions,
                 double* residuals, ReportC* report, int threads, int* sgd_batches, int record) {
  return guarded([&] {
    const Dataset ds = make_data(x, nullptr, n, d);
    KernelOperator op(&ds, make_hp(raw, d), 1024, threads);
    LinearSystemBatch b(op, make_mat(targets, n, m));
    if (warm) b.warm_start(make_mat(warm, n, m));
    const SolverConfig c = to_cfg(cfg);
    SolverReport r;
    std::vector<std::vector<int>> batches;
    if (c.kind == CG && explicit_rank >= 0) {
      PivotedCholesky pc(op, explicit_rank);
      r = solve_cg(b, c, &pc);
    } else if (c.kind == CG && explicit_rank == -2) {
      r = solve_cg(b, c, nullptr);
    } else if (c.kind == SGD && sgd_batches) {
      r = solve_sgd(b, c, &batches, record);
      for (size_t t = 0; t < batches.size(); ++t)
        std::memcpy(sgd_batches + t * batches[t].size(), batches[t].data(), sizeof(int) * batches[t].size());
    } else {
      r = solve(b, c);
    }
    put(b.solutions, solutions);
    put(b.residuals, residuals);
    fill_report(r, report);
  });
}

int oracle_termination_check(const double* targets, const double* residuals, int n, int m, double tol,
                             double* mean, double* probe, int* done) {
  return guarded([&] {
    // Norms only; the operator is not touched.
    Dataset ds = make_data(std::vector<double>(n, 0.0).data(), nullptr, n, 1);
    KernelOperator op(&ds, Hyper::constant(1, 1.0));
    LinearSystemBatch b(op, make_mat(targets, n, m));
    b.residuals = make_mat(residuals, n, m);
    const auto st = termination_check(b, tol);
    *mean = st.mean_norm;
    *probe = st.probe_norm;
    *done = st.done;
  });
}

// out: values, quadratic_term, trace_term (each d+2).
int oracle_gradient(const double* x, int n, int d, const double* raw, const double* v_y,
                    const double* zhat, int s, const double* probes, double* out, int threads) {
  return guarded([&] {
    const Dataset ds = make_data(x, nullptr, n, d);
    KernelOperator op(&ds, make_hp(raw, d), 1024, threads);
    const Vec vy(v_y, v_y + n);
    const GradientEstimate g = probes ? estimate_gradient_standard(op, vy, make_mat(zhat, n, s), make_mat(probes, n, s))
                                      : estimate_gradient_pathwise(op, vy, make_mat(zhat, n, s));
    for (int k = 0; k < d + 2; ++k) {
      out[k] = g.values[k];
      out[d + 2 + k] = g.quadratic_term[k];
      out[2 * (d + 2) + k] = g.trace_term[k];
    }
  });
}

int oracle_standard_probes(int n, int s, unsigned long long seed, int distribution,
                           unsigned long long substream, double* out) {
  return guarded([&] { put(gen_standard_probes(n, s, seed, distribution, substream), out); });
}

int oracle_rff_basis(int d, int pairs, int samples, unsigned long long seed, unsigned long long substream,
                     double* freq, double* weights) {
  return guarded([&] {
    const RffBasis b = build_rff_basis(d, pairs, samples, seed, substream);
    put(b.base_frequencies, freq);
    put(b.weights, weights);
  });
}

int oracle_rff_features(int d, int pairs, int samples, unsigned long long seed, const double* raw,
                        const double* points, int p, double* out) {
  return guarded([&] {
    const RffBasis b = build_rff_basis(d, pairs, samples, seed, 0);
    put(rff_features(b, make_hp(raw, d), make_mat(points, p, d)), out);
  });
}

// prior, noise, xi: n x s each (nullable).
int oracle_pathwise_targets(const double* x, int n, int d, const double* raw, int pairs, int samples,
                            int s, unsigned long long seed, unsigned long long substream, double* prior,
                            double* noise, double* xi) {
  return guarded([&] {
    const Dataset ds = make_data(x, nullptr, n, d);
    const RffBasis b = build_rff_basis(d, pairs, samples, seed, substream);
    const PathwiseTargets t = pathwise_targets(b, make_hp(raw, d), ds, s, seed, substream);
    if (prior) put(t.prior_values, prior);
    if (noise) put(t.noise, noise);
    if (xi) put(t.xi, xi);
  });
}

struct OuterConfigC {
  int estimator;
  SolverConfigC solver;
  int warm_start, steps;
  double learning_rate;
  int probe_count, rff_pairs, probe_distribution;
  unsigned long long probe_seed, feature_seed, solver_seed;
  double init_value;
  int divergence_policy;
  int prior_mode;
};

// Per step row of `trace` (stride 2*(d+2)+8): constrained[d+2], gradient[d+2],
// mean, probe, epochs, grad_inf, iterations, diverged, solver_seconds(0), pad.
int oracle_optimise(const double* x, const double* y, int n, int d, const OuterConfigC* cfg,
                    const double* init_constrained, double* trace, int* rows_out, double* final_raw,
                    int* aborted, int threads) {
  return guarded([&] {
    const Dataset ds = make_data(x, y, n, d);
    OuterConfig oc;
    oc.estimator = cfg->estimator;
    oc.solver = to_cfg(&cfg->solver);
    oc.warm_start = cfg->warm_start != 0;
    oc.steps = cfg->steps;
    oc.learning_rate = cfg->learning_rate;
    oc.probe_count = cfg->probe_count;
    oc.rff_pairs = cfg->rff_pairs;
    oc.probe_distribution = cfg->probe_distribution;
    oc.probe_seed = cfg->probe_seed;
    oc.feature_seed = cfg->feature_seed;
    oc.solver_seed = cfg->solver_seed;
    oc.init_value = cfg->init_value;
    oc.divergence_policy = cfg->divergence_policy;
    oc.prior_mode = cfg->prior_mode;
    if (init_constrained) oc.init_constrained.assign(init_constrained, init_constrained + d + 2);
    const OuterResult r = optimise(ds, oc, threads);
    const int P = d + 2, stride = 2 * P + 8;
    for (size_t t = 0; t < r.trace.size(); ++t) {
      double* row = trace + t * stride;
      const TraceRow& tr = r.trace[t];
      for (int k = 0; k < P; ++k) row[k] = tr.constrained[k];
      for (int k = 0; k < P; ++k) row[P + k] = tr.gradient.empty() ? 0.0 : tr.gradient[k];
      row[2 * P + 0] = tr.mean_residual_norm;
      row[2 * P + 1] = tr.probe_residual_norm;
      row[2 * P + 2] = tr.epochs;
      row[2 * P + 3] = tr.grad_inf_norm;
      row[2 * P + 4] = tr.iterations;
      row[2 * P + 5] = tr.solver_diverged;
      row[2 * P + 6] = 0.0;
      row[2 * P + 7] = 0.0;
    }
    *rows_out = static_cast<int>(r.trace.size());
    for (int k = 0; k < P; ++k) final_raw[k] = r.hp.raw[k];
    *aborted = r.aborted;
  });
}

int oracle_exact(const double* x, const double* y, int n, int d, const double* raw, double* mll,
                 double* grad) {
  return guarded([&] {
    const Dataset ds = make_data(x, y, n, d);
    const DenseProblem dp = build_dense_problem(ds, make_hp(raw, d));
    *mll = exact_mll(dp, ds.targets);
    const Vec g = exact_gradient(dp, ds.targets);
    std::memcpy(grad, g.data(), sizeof(double) * g.size());
  });
}

// optimise_exact: trajectory (steps x (d+2) constrained, row-major), final raw (d+2).
int oracle_optimise_exact(const double* x, const double* y, int n, int d, const double* init_constrained, int steps,
                          double learning_rate, double* trajectory, double* final_raw) {
  return guarded([&] {
    const Dataset ds = make_data(x, y, n, d);
    const Hyper init = init_constrained ? Hyper::from_constrained(Vec(init_constrained, init_constrained + d + 2))
                                        : Hyper::constant(d, 1.0);
    const ExactTrajectory tr = optimise_exact(ds, init, steps, learning_rate);
    for (int t = 0; t < steps; ++t)
      std::memcpy(trajectory + static_cast<size_t>(t) * (d + 2), tr.constrained_per_step[t].data(),
                  sizeof(double) * (d + 2));
    std::memcpy(final_raw, tr.hp.raw.data(), sizeof(double) * (d + 2));
  });
}

// init_heuristic: constrained (d+2) of the averaged fit.
int oracle_init_heuristic(const double* x, const double* y, int n, int d, int n_centroids, int subset,
                          unsigned long long seed, int adam_steps, double learning_rate, double* constrained) {
  return guarded([&] {
    const Dataset ds = make_data(x, y, n, d);
    const Vec c = init_heuristic(ds, n_centroids, subset, seed, adam_steps, learning_rate).constrained();
    std::memcpy(constrained, c.data(), sizeof(double) * (d + 2));
  });
}

// k(P, X) V (p x m), P p x d, X n x d, V n x m.
int oracle_cross_apply(const double* points, int p, const double* x, int n, int d, const double* raw, const double* v,
                       int m, double* out, int threads) {
  return guarded([&] {
    put(cross_kernel_apply(make_mat(points, p, d), make_mat(x, n, d), make_hp(raw, d), make_mat(v, n, m), 1024, threads),
        out);
  });
}

// ExactDense prior values (n x s): weights from (seed, kPriorSample, substream).
int oracle_exact_prior(const double* x, int n, int d, const double* raw, int s, unsigned long long seed,
                       unsigned long long substream, double* out) {
  return guarded([&] {
    const Dataset ds = make_data(x, nullptr, n, d);
    const Hyper hp = make_hp(raw, d);
    KernelOperator op(&ds, hp);
    Mat w(n, s);
    RandomStream st(seed, streams::kPriorSample, substream);
    st.fill_gaussian(w.a.data(), w.size());
    put(exact_dense_prior(op, hp, w), out);
  });
}

// RFF prior at points (p x s) for basis (d, pairs, samples, seed, substream).
int oracle_prior_at(int d, int pairs, int samples, unsigned long long seed, unsigned long long substream,
                    const double* raw, const double* points, int p, int s, double* out) {
  return guarded([&] {
    const RffBasis b = build_rff_basis(d, pairs, samples, seed, substream);
    put(evaluate_prior_all(b, make_hp(raw, d), make_mat(points, p, d), s), out);
  });
}

// samples (p x s) and metrics {rmse, llh, rmse_raw, llh_raw, has_llh}; prior p x s (nullable = zero prior).
int oracle_posterior(const double* points, int p, const double* x, int n, int d, const double* raw, const double* v_y,
                     const double* zhat, int s, const double* prior, const double* test_targets, double target_scale,
                     double* samples, double* metrics, int threads) {
  return guarded([&] {
    const Mat P = make_mat(points, p, d), X = make_mat(x, n, d);
    const Hyper hp = make_hp(raw, d);
    const Vec vy(v_y, v_y + n);
    const Mat Z = make_mat(zhat, n, s);
    const Mat pr = prior ? make_mat(prior, p, s) : Mat();
    if (samples) put(sample_posterior_all(pr, P, X, hp, vy, Z, threads), samples);
    if (metrics && test_targets) {
      const TestMetrics mt = test_metrics(pr, P, Vec(test_targets, test_targets + p), X, hp, vy, Z, target_scale,
                                          threads);
      metrics[0] = mt.rmse;
      metrics[1] = mt.llh;
      metrics[2] = mt.rmse_raw;
      metrics[3] = mt.llh_raw;
      metrics[4] = mt.has_llh;
    }
  });
}

void oracle_sinsum_dataset(int n, int d, int uniform, double noise, unsigned long long seed, float* x_rowmajor,
                           float* y) {
  std::vector<float> xv, yv;
  make_sinsum_dataset(n, d, uniform != 0, noise, seed, xv, yv);
  std::memcpy(x_rowmajor, xv.data(), sizeof(float) * xv.size());
  std::memcpy(y, yv.data(), sizeof(float) * yv.size());
}

}  // extern "C"
