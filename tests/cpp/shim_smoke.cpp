// Exercises include/gpiter_b200.hpp the way the reference's own tests use
// gpiter (proj/tests/test_kernel.cpp, test_solvers.cpp): builds an operator,
// applies it, solves a batch with CG/AP/SGD and evaluates the pathwise
// gradient. Prints one JSON object; tests/test_cpp_shim.py checks it against
// the oracle on the GPU box.
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "gpiter_b200.hpp"

using namespace gpiter_b200;

int main() {
  const int n = 512, d = 3, s = 4;
  Context ctx(0);
  Matrix x(n, d);
  // deterministic inputs: x(i, k) = sin(0.37 i + 1.3 k)
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) x(i, k) = std::sin(0.37 * i + 1.3 * k);
  Hyperparameters hp;
  for (int k = 0; k < d + 2; ++k) hp.raw.push_back(k == d + 1 ? -1.0 : 0.5);
  KernelOperator op(ctx, x, hp);
  Matrix v(n, s + 1);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= s; ++j) v(i, j) = std::cos(0.11 * i * (j + 1));
  const Matrix hv = op.apply(v);
  bool threw = false;
  try {
    op.apply(Matrix(n - 1, 1));
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  std::printf("{\"hv00\": %.17g, \"hv_last\": %.17g, \"threw_invalid_argument\": %d", hv(0, 0), hv(n - 1, s), threw);
  const char* names[3] = {"cg", "ap", "sgd"};
  for (int kind = 0; kind < 3; ++kind) {
    LinearSystemBatch batch(op, v);
    SolverConfig c;
    c.kind = static_cast<SolverKind>(kind);
    c.tolerance = 0.01;
    c.max_epochs = 200;
    c.block_size = 64;
    c.batch_size = 64;
    c.learning_rate = 2.0;
    c.seed = 4;
    const SolverReport r = solve(batch, c);
    std::printf(", \"%s_iterations\": %d, \"%s_mean\": %.17g, \"%s_probe\": %.17g", names[kind], r.iterations,
                names[kind], r.mean_residual_norm, names[kind], r.probe_residual_norm);
    if (kind == 0) {
      const Matrix sol = batch.solutions();
      Vector vy(n);
      Matrix z(n, s);
      for (int i = 0; i < n; ++i) {
        vy[i] = sol(i, 0);
        for (int j = 0; j < s; ++j) z(i, j) = sol(i, j + 1);
      }
      const GradientEstimate g = estimate_gradient_pathwise(op, vy, z);
      std::printf(", \"grad\": [");
      for (int k = 0; k < d + 2; ++k) std::printf("%s%.17g", k ? ", " : "", g.values[k]);
      std::printf("], \"cg_solutions\": [");
      for (int i = 0; i < n; ++i)
        for (int j = 0; j <= s; ++j) std::printf("%s%.17g", (i || j) ? ", " : "", sol(i, j));
      std::printf("]");
    }
  }
  std::printf("}\n");
  return 0;
}
