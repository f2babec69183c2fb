"""Times one AP solve at the C2 shape (n=16384, d=26, 65 RHS, block 512,
tol 0.01) with the device profiling events: per-iteration wall time and the
K.V kernel share. GPK_FUSED_AP=0 selects the unfused slab + reduce path."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18457_b200 as G  # noqa: E402


def main():
    n, d, m = 16384, 26, 65
    ctx = G.Context(0)
    X32, y32 = G.sinsum_dataset(n, d, False, 0.1, 0)
    raw = np.array([G.gpiter.softplus_inverse(v) for v in [1.0] * d + [1.0, 0.1]])
    op = G.KernelOperator(X32.astype(np.float64), G.Hyperparameters.from_raw(raw), ctx)
    rng = np.random.default_rng(0)
    T = np.asfortranarray(rng.standard_normal((n, m)))
    cfg = G.SolverConfig(kind=1, tolerance=0.01, max_epochs=50, block_size=512)
    G.solve_ap(G.LinearSystemBatch(op, T), cfg)
    batch = G.LinearSystemBatch(op, T)
    ctx.synchronize()
    ctx.reset_stats()
    ctx.set_profiling(True)
    t = time.perf_counter()
    rep = G.solve_ap(batch, cfg)
    ctx.synchronize()
    wall = time.perf_counter() - t
    st = ctx.stats()
    print(json.dumps({"fused": os.environ.get("GPK_FUSED_AP", "1"), "iterations": rep.iterations, "wall_s": wall,
                      "us_per_iteration": wall / max(1, rep.iterations) * 1e6,
                      "kv_us": st["kv_ms"] / max(1, st["kv_launches"]) * 1e3, "kv_launches": st["kv_launches"],
                      "mean": rep.mean_residual_norm, "probe": rep.probe_residual_norm}))


if __name__ == "__main__":
    main()
