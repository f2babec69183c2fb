"""Runs the first `steps` outer steps of a BASELINE config through the public
optimise() call on the GPU and saves the trajectory (gpurun_out/<cfg>_<steps>_gpu.npz)
for comparison with tools/make_golden.py's oracle trajectory.

usage: python tools/traj_gpu.py C3 2"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2405_18457_b200 as G  # noqa: E402


def main():
    name, steps = sys.argv[1], int(sys.argv[2])
    c = bench.CONFIGS[name]
    ctx = G.Context(0)
    X32, y32 = G.sinsum_dataset(c["n"], c["d"], c["uniform"], c["noise"], bench.SEEDS["data"])
    r = G.optimise(ctx, X32.astype(np.float64), y32.astype(np.float64), bench.outer_config(G, name, steps),
                   init_constrained=bench.init_constrained(c))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.savez(os.path.join(ROOT, "gpurun_out", f"{name.lower()}_{steps}_gpu.npz"),
             **{k: np.asarray(v) for k, v in r.items()})
    print(name, "iterations", list(np.asarray(r["iterations"])), "seconds", list(np.asarray(r["step_seconds"])))


if __name__ == "__main__":
    main()
