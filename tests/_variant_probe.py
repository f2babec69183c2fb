"""Subprocess probe for test_gpu_parity.test_operator_variants_match_oracle:
operator products of the tcgen05 kernel under the launch variant the
environment selects (GPK_KV_DEEP, GPK_TGRAM, GPK_TGRAM_MIN_D are read when the
library creates its context / operators), against the FP64 oracle. Prints one
JSON line of max column-relative errors."""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
from _problems import default_test_raw, gp_problem  # noqa: E402
from oracle import oracle as O  # noqa: E402
import paper_2405_18457_b200 as G  # noqa: E402


# the caller compares every entry with the operator tolerance (2e-5): gradient
# errors (bar 1e-4) are rescaled to it
OP_TOL_OVER_GRAD_TOL = 2e-5 / 1e-4


def colrel(a, b):
    return max(np.max(np.abs(a[:, j] - b[:, j])) / max(np.max(np.abs(b[:, j])), 1e-300) for j in range(b.shape[1]))


def main():
    ctx = G.Context(0)
    out = {}
    for n, d, m in [(2048, 3, 65), (1500, 11, 33), (2048, 20, 65), (2048, 26, 65), (1000, 32, 80), (777, 17, 17)]:
        X, _ = gp_problem(n, d, 31 * n + d)
        raw = default_test_raw(d, O)
        V = np.asfortranarray(np.random.default_rng(d).standard_normal((n, m)))
        op = G.KernelOperator(X, G.Hyperparameters.from_raw(raw), ctx)
        out[f"{n}x{d}x{m}"] = float(colrel(op.apply(V), O.apply(X, raw, V, threads=8)))
    if os.environ.get("GPK_KV_PANEL_MB"):
        # column panels (forced at any size): n x 8 NPAD bytes of images > 2 panels
        n, d, m = 5000, 11, 65
        X, _ = gp_problem(n, d, 31 * n + d)
        raw = default_test_raw(d, O)
        V = np.asfortranarray(np.random.default_rng(d).standard_normal((n, m)))
        op = G.KernelOperator(X, G.Hyperparameters.from_raw(raw), ctx)
        out[f"panels {n}x{d}x{m}"] = float(colrel(op.apply(V), O.apply(X, raw, V, threads=8)))
    if os.environ.get("GPK_GRAD_WAVE"):
        # gradient pass with the row-wave tile schedule (forced; the size rule picks it from 8 rows per CTA):
        # more tile rows than one wave of CTAs would need n > 19000, so this checks the partial-wave bookkeeping
        for n, d, s in [(1500, 3, 16), (1300, 20, 64)]:
            X, _ = gp_problem(n, d, 4 * n)
            raw = default_test_raw(d, O)
            rng = np.random.default_rng(n)
            vy, Z = rng.standard_normal(n), rng.standard_normal((n, s))
            op = G.KernelOperator(X, G.Hyperparameters.from_raw(raw), ctx)
            g = G.estimate_gradient_pathwise(op, vy, Z)
            r = O.gradient(X, raw, vy, Z, threads=8)
            err = 0.0
            for key in ("quadratic_term", "trace_term"):
                a, b = getattr(g, key), r[key]
                err = max(err, float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-3 * np.max(np.abs(b))))))
            out[f"grad wave {n}x{d}x{s}"] = err * OP_TOL_OVER_GRAD_TOL
    print(json.dumps(out))


if __name__ == "__main__":
    main()
