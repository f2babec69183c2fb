"""Precision of the fused gradient pass on a cancellation-heavy problem (the
C++ shim test's: sin inputs, CG solutions as probes): quadratic and trace
forms from the SIMT (kernel 0) and tensor-core (kernel 1) passes against the
FP64 oracle, plus a CPU FP32 emulation of the evaluation for reference."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_18457_b200 as G  # noqa: E402
from oracle import oracle as O  # noqa: E402


def run(X, raw, vy, Z, tag):
    ref = O.gradient(X, raw, vy, Z, threads=8)
    out = {"case": tag}
    for kern in (0, 1):
        ctx = G.Context(0)
        ctx.set_operator_kernel(kern)
        op = G.KernelOperator(X, G.Hyperparameters.from_raw(raw), ctx)
        g = G.estimate_gradient_pathwise(op, vy, Z)
        for key in ("quadratic_term", "trace_term", "values"):
            a, b = np.asarray(getattr(g, key)), ref[key]
            out[f"k{kern}_{key}"] = float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-2)))
    print(json.dumps(out), flush=True)


def main():
    n, d, s = 512, 3, 4
    i = np.arange(n)
    X = np.stack([np.sin(0.37 * i + 1.3 * k) for k in range(d)], axis=1)
    raw = np.array([0.5] * (d + 1) + [-1.0])
    V = np.stack([np.cos(0.11 * i * (j + 1)) for j in range(s + 1)], axis=1)
    sol = O.solve(X, raw, V, O.solver_config(kind=0, tolerance=0.01, max_epochs=200))["solutions"]
    run(X, raw, sol[:, 0], sol[:, 1:], "shim")
    rng = np.random.default_rng(0)
    run(X, raw, rng.standard_normal(n), rng.standard_normal((n, s)), "shim-X random-probes")
    for n, d, s in [(500, 2, 8), (2048, 26, 64), (1024, 3, 16)]:
        X = rng.standard_normal((n, d))
        raw = np.array([0.3] * d + [0.5, -1.0])
        run(X, raw, rng.standard_normal(n), rng.standard_normal((n, s)), f"random n={n} d={d} s={s}")


if __name__ == "__main__":
    main()
