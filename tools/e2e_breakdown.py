"""Where the end-to-end (host buffers, public API) time of the C2 bench goes:
optimiser creation, first step (cold start, no warm start yet), later steps."""
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
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    c = bench.CONFIGS[name]
    ctx = G.Context(0)
    X32, y32 = G.sinsum_dataset(c["n"], c["d"], c["uniform"], c["noise"], bench.SEEDS["data"])
    X, y = X32.astype(np.float64), y32.astype(np.float64)
    for rep in range(2):
        ctx.synchronize()
        t0 = time.perf_counter()
        opt = G.Optimiser(ctx, X, y, bench.outer_config(G, name, 8), init_constrained=bench.init_constrained(c))
        ctx.synchronize()
        t1 = time.perf_counter()
        steps = []
        for k in range(8):
            ts = time.perf_counter()
            tr = opt.step(1)
            ctx.synchronize()
            steps.append({"ms": (time.perf_counter() - ts) * 1e3, "iterations": int(tr["iterations"][0])})
        opt.close()
        ctx.synchronize()
        t2 = time.perf_counter()
        print(json.dumps({"rep": rep, "create_ms": (t1 - t0) * 1e3, "steps": steps, "close_ms": (t2 - t1) * 1e3 -
                          sum(s["ms"] for s in steps)}), flush=True)




def optimise_calls():
    name = "C2"
    c = bench.CONFIGS[name]
    ctx = G.Context(0)
    X32, y32 = G.sinsum_dataset(c["n"], c["d"], c["uniform"], c["noise"], bench.SEEDS["data"])
    X, y = X32.astype(np.float64), y32.astype(np.float64)
    for rep in range(3):
        ctx.reset_stats()
        ctx.synchronize()
        t0 = time.perf_counter()
        res = G.optimise(ctx, X, y, bench.outer_config(G, name, 8), init_constrained=bench.init_constrained(c))
        ctx.synchronize()
        dt = time.perf_counter() - t0
        st = ctx.stats()
        print(json.dumps({"optimise_rep": rep, "seconds": dt, "evals": st["evals_x_rhs"],
                          "e2e_value": st["evals_x_rhs"] / dt, "iterations": res["iterations"].tolist(),
                          "step_seconds": res["step_seconds"].tolist()}), flush=True)


if __name__ == "__main__":
    main()
    optimise_calls()
