"""Runs `steps` marginal-likelihood steps of a BASELINE workload through the
device optimiser (bench.py's configuration), for launch lists and ncu
captures: python tools/one_step.py [C4] [steps]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2405_18457_b200 as G  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    c = bench.CONFIGS[name]
    ctx = G.Context(0)
    X32, y32 = G.sinsum_dataset(c["n"], c["d"], c["uniform"], c["noise"], bench.SEEDS["data"])
    X, y = X32.astype(np.float64), y32.astype(np.float64)
    opt = G.Optimiser(ctx, X, y, bench.outer_config(G, name, steps), init_constrained=bench.init_constrained(c))
    for k in range(steps):
        t = time.perf_counter()
        tr = opt.step(1)
        ctx.synchronize()
        print(name, "step", k, "s", round(time.perf_counter() - t, 4), "iters", int(tr["iterations"][0]),
              "mean", float(tr["mean_residual_norm"][0]), flush=True)
    opt.close()


if __name__ == "__main__":
    main()
