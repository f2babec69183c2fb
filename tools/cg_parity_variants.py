"""CG parity attribution: one operator variant of the
product against the CPU oracle's C1 / C3 fixtures (tests/golden/c1.npz: 10
steps, c3.npz: 2 steps). The variant is chosen by the environment (each knob
is read once per process):

  GPK_TGRAM=0          FP32 distance loops instead of tensor-core Gram distances
  GPK_FLUSH_CHUNKS=k   FP32 TMEM accumulation over k x 32 columns (default 16)
  GPK_DENSE_CAP=0      C1 on the matrix-free operator instead of the FP64 cache
  kernel=simt (argv)   the FP32 SIMT operator kernel

usage: python tools/cg_parity_variants.py C1|C3 [simt] -> one JSON line"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2405_18457_b200 as G  # noqa: E402


def main():
    name = sys.argv[1]
    simt = "simt" in sys.argv[2:]
    steps = {"C1": 10, "C3": 2}[name]
    g = np.load(os.path.join(ROOT, "tests", "golden", name.lower() + ".npz"))
    c = bench.CONFIGS[name]
    ctx = G.Context(0)
    if simt:
        ctx.set_operator_kernel(0)
    X32, y32 = G.sinsum_dataset(c["n"], c["d"], c["uniform"], c["noise"], 0)
    r = G.optimise(ctx, X32.astype(np.float64), y32.astype(np.float64), bench.outer_config(G, name, steps),
                   init_constrained=bench.init_constrained(c))
    gg = g["traj_gradient"]
    out = {"config": name, "variant": {k: os.environ.get(k) for k in ("GPK_TGRAM", "GPK_FLUSH_CHUNKS", "GPK_DENSE_CAP")},
           "kernel": "simt" if simt else "tcgen05",
           "iterations": r["iterations"].tolist(), "oracle_iterations": g["traj_iterations"].tolist(),
           "mean_norm_rel": (np.abs(r["mean_residual_norm"] - g["traj_mean_residual_norm"]) /
                             g["traj_mean_residual_norm"]).tolist(),
           "probe_norm_rel": (np.abs(r["probe_residual_norm"] - g["traj_probe_residual_norm"]) /
                              g["traj_probe_residual_norm"]).tolist(),
           "gradient_rel_componentwise": (np.abs(r["gradient"] - gg) / np.abs(gg)).max(axis=1).tolist(),
           "gradient_rel_of_max": (np.abs(r["gradient"] - gg).max(axis=1) / np.abs(gg).max(axis=1)).tolist(),
           "trajectory_rel": float(np.max(np.abs(r["constrained"] - g["traj_constrained"]) / g["traj_constrained"]))}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
