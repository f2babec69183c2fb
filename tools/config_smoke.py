"""One or more outer steps of each BASELINE configuration (C1-C5) on one GPU
through the device optimiser: seconds per marginal-likelihood step, solver
iterations/epochs, device-counted evals x RHS per second. Configurations and
seeds are bench.py's (synthetic sin-sum data, BASELINE init).

usage: python tools/config_smoke.py [C1 C2 ...] [--steps K]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2405_18457_b200 as G  # noqa: E402


def main():
    argv = sys.argv[1:]
    steps = 2
    if "--steps" in argv:
        i = argv.index("--steps")
        steps = int(argv[i + 1])
        argv = argv[:i] + argv[i + 2:]
    args = argv
    names = args or ["C1", "C2", "C3", "C4", "C5"]
    ctx = G.Context(0)
    for name in names:
        c = bench.CONFIGS[name]
        X32, y32 = G.sinsum_dataset(c["n"], c["d"], c["uniform"], c["noise"], bench.SEEDS["data"])
        X, y = X32.astype(np.float64), y32.astype(np.float64)
        opt = G.Optimiser(ctx, X, y, bench.outer_config(G, name, steps), init_constrained=bench.init_constrained(c))
        rows = []
        for k in range(steps):
            ctx.synchronize()
            ctx.reset_stats()
            t = time.perf_counter()
            tr = opt.step(1)
            ctx.synchronize()
            dt = time.perf_counter() - t
            st = ctx.stats()
            rows.append({"step": k, "seconds": dt, "iterations": int(tr["iterations"][0]),
                         "epochs": float(tr["epochs"][0]), "evals_x_rhs_per_s": st["evals_x_rhs"] / dt,
                         "mean_norm": float(tr["mean_residual_norm"][0])})
        print(json.dumps({"config": bench.workload_config(name)["workload"], "steps": rows}), flush=True)


if __name__ == "__main__":
    main()
