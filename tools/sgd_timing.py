"""Times one SGD solve at BASELINE configs[3]'s shape (C4: n=393216, d=3,
s=64 probes + mean = 65 RHS, batch 512, lr 10, momentum 0.9) on the device,
with the operator's own profiling events giving the K.V share.

usage: python tools/sgd_timing.py [n] [epochs]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18457_b200 as G  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 393216
    epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    d, m, b = 3, 65, 512
    ctx = G.Context(0)
    X32, y32 = G.sinsum_dataset(n, d, True, 0.05, 0)
    X = X32.astype(np.float64)
    raw = np.array([G.gpiter.softplus_inverse(v) for v in [1.0] * d + [1.0, 0.05]])
    op = G.KernelOperator(X, G.Hyperparameters.from_raw(raw), ctx)
    rng = np.random.default_rng(0)
    T = np.asfortranarray(rng.standard_normal((n, m)))
    cfg = G.SolverConfig(kind=2, tolerance=1e-9, max_epochs=epochs, batch_size=b, learning_rate=float(os.environ.get("SGD_LR", "10")), momentum=0.9,
                         seed=4)
    # warm-up solve (allocations, module load)
    G.solve_sgd(G.LinearSystemBatch(op, T), G.SolverConfig(kind=2, tolerance=1e-9, max_epochs=1, batch_size=b,
                                                           learning_rate=10.0, seed=4))
    batch = G.LinearSystemBatch(op, T)
    ctx.synchronize()
    ctx.reset_stats()
    ctx.set_profiling(True)
    t = time.perf_counter()
    rep = G.solve_sgd(batch, cfg)
    ctx.synchronize()
    wall = time.perf_counter() - t
    st = ctx.stats()
    it = rep.iterations
    out = {"n": n, "d": d, "m": m, "batch": b, "iterations": it, "wall_s": wall, "us_per_iteration": wall / it * 1e6,
           "kv_us_per_iteration": st["kv_ms"] / max(1, st["kv_launches"]) * 1e3, "kv_launches": st["kv_launches"],
           "kv_tflops": st["flops"] / (st["kv_ms"] / 1e3) / 1e12 if st["kv_ms"] else None,
           "mean_residual_norm": rep.mean_residual_norm, "aborted": rep.aborted}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
