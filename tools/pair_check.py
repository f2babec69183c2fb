"""Runs one short SGD solve (d = 3, 65 RHS, b = 512) and prints its report and
solution checksums, for comparing the paired slab (GPK_SGD_PAIR=1, default)
with the one-CTA slab (GPK_SGD_PAIR=0) in separate processes.

usage: python tools/pair_check.py n epochs [lr]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18457_b200 as G  # noqa: E402


def main():
    n, epochs = int(sys.argv[1]), int(sys.argv[2])
    lr = float(sys.argv[3]) if len(sys.argv) > 3 else 10.0
    d, m, b = 3, 65, 512
    ctx = G.Context(0)
    X32, _ = G.sinsum_dataset(n, d, True, 0.05, 0)
    raw = np.array([G.gpiter.softplus_inverse(v) for v in [1.0] * d + [1.0, 0.05]])
    op = G.KernelOperator(X32.astype(np.float64), G.Hyperparameters.from_raw(raw), ctx)
    T = np.asfortranarray(np.random.default_rng(0).standard_normal((n, m)))
    batch = G.LinearSystemBatch(op, T)
    rep = G.solve_sgd(batch, G.SolverConfig(kind=2, tolerance=1e-9, max_epochs=epochs, batch_size=b,
                                            learning_rate=lr, momentum=0.9, seed=4))
    S = batch.solutions
    out = dict(n=n, pair=os.environ.get("GPK_SGD_PAIR", "1"), iterations=rep.iterations,
               mean_residual_norm=rep.mean_residual_norm, aborted=rep.aborted,
               sol_sum=float(np.sum(S)), sol_abs=float(np.sum(np.abs(S))), col0=[float(v) for v in S[:4, 0]])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
