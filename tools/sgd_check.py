"""Quick check of the SGD path against the CPU oracle on a small problem
(solutions, tracked residual norms, iteration count), then one C4-size SGD
epoch timed: python tools/sgd_check.py"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_18457_b200 as G  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    ctx = G.Context(0)
    for (n, d, m, b, ep, lr) in [(2048, 3, 65, 512, 3, 10.0), (3000, 5, 17, 256, 2, 5.0), (1536, 11, 65, 128, 2, 3.0)]:
        X32, _ = O.sinsum_dataset(n, d, True, 0.05, 0)
        X = np.asfortranarray(X32.astype(np.float64))
        raw = O.raw_from_constrained([1.0] * d + [1.0, 0.1])
        T = np.asfortranarray(np.random.default_rng(n).standard_normal((n, m)))
        cfg = dict(kind=2, tolerance=1e-9, max_epochs=ep, batch_size=b, learning_rate=lr, momentum=0.9, seed=4)
        ref = O.solve(X, raw, T, O.solver_config(**cfg), threads=8)
        op = G.KernelOperator(X, G.Hyperparameters.from_raw(raw), ctx)
        batch = G.LinearSystemBatch(op, T)
        rep = G.solve_sgd(batch, G.SolverConfig(**cfg))
        sol = batch.solutions
        err = np.max(np.abs(sol - ref["solutions"])) / np.max(np.abs(ref["solutions"]))
        print(f"n={n} d={d} m={m} b={b}: iters {rep.iterations}/{ref['iterations']} "
              f"mean {rep.mean_residual_norm:.9f}/{ref['mean_residual_norm']:.9f} "
              f"probe {rep.probe_residual_norm:.9f}/{ref['probe_residual_norm']:.9f} sol rel {err:.2e}", flush=True)
    n = 393216
    X32, _ = G.sinsum_dataset(n, 3, True, 0.05, 0)
    op = G.KernelOperator(X32.astype(np.float64), G.Hyperparameters.from_constrained([1.0] * 3 + [1.0, 0.1]), ctx)
    T = np.asfortranarray(np.random.default_rng(0).standard_normal((n, 65)))
    cfg = G.SolverConfig(kind=2, tolerance=1e-9, max_epochs=1, batch_size=512, learning_rate=10.0, momentum=0.9, seed=4)
    G.solve_sgd(G.LinearSystemBatch(op, T), cfg)
    batch = G.LinearSystemBatch(op, T)
    ctx.synchronize()
    t = time.perf_counter()
    rep = G.solve_sgd(batch, cfg)
    ctx.synchronize()
    dt = time.perf_counter() - t
    print(f"C4 epoch: {rep.iterations} iterations {dt:.3f} s = {dt / rep.iterations * 1e6:.1f} us/iteration", flush=True)
    ctx.reset_stats()
    ctx.set_profiling(True)
    G.solve_sgd(G.LinearSystemBatch(op, T), cfg)
    st = ctx.stats()
    print(f"slab {st['kv_ms'] / max(1, st['kv_launches']) * 1e3:.1f} us/launch over {st['kv_launches']} launches, "
          f"{st['flops'] / (st['kv_ms'] / 1e3) / 1e12:.1f} TF F_KV", flush=True)


if __name__ == "__main__":
    main()
