"""Fixtures for the two BASELINE configurations the CPU oracle cannot run in
full (C4: SGD, n = 393216; C5: CG, n = 1835008), made by the oracle-at-scale
(oracle/gpu/oracle_gpu.cu: the FP64 restatement with its O(n^2) passes as naive
FP64 CUDA kernels). Run on a GPU box:

    python tools/make_golden_scale.py [validate] [c4] [c5]

validate  the oracle-at-scale against the CPU oracle's committed C1/C3
          trajectories (tests/golden/c1.npz, c3.npz): prints the differences
          (FP64 vs FP64, different summation order) -> gpurun_out/scale_validate.json
c4        tests/golden/c4_scale.npz: an 8-iteration SGD replay (the CPU test
          re-runs it with the CPU oracle) and the first 2 optimiser steps of C4
c5        tests/golden/c5_scale.npz: the first optimiser step of C5
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
OUT = os.path.join(ROOT, "gpurun_out")
REPLAY_ITERS = 8


def data(name):
    c = bench.CONFIGS[name]
    X32, y32 = O.sinsum_dataset(c["n"], c["d"], c["uniform"], c["noise"], bench.SEEDS["data"])
    return np.asfortranarray(X32.astype(np.float64)), y32.astype(np.float64)


def ocfg(name, steps):
    c = bench.CONFIGS[name]
    sc = O.solver_config(kind=c["kind"], tolerance=0.01, max_epochs=c["max_epochs"], block_size=c["block"],
                         batch_size=c["batch"], learning_rate=c["lr_sgd"], momentum=0.9, preconditioner_rank=100)
    return O.outer_config(estimator=1, solver=sc, warm_start=True, steps=steps, learning_rate=0.1,
                          probe_count=c["s"], rff_pairs=c["rff_pairs"], probe_seed=2, feature_seed=3, solver_seed=4)


def traj(name, steps):
    X, y = data(name)
    c = bench.CONFIGS[name]
    t = time.perf_counter()
    r = O.optimise(X, y, ocfg(name, steps), init_constrained=bench.init_constrained(c), threads=os.cpu_count())
    r["seconds"] = time.perf_counter() - t
    return r


def sgd_replay(iters):
    """C4 shape, cold SGD solve on seeded Gaussian targets, `iters` iterations."""
    X, _ = data("C4")
    n, m = X.shape[0], 65
    raw = O.raw_from_constrained(bench.init_constrained(bench.CONFIGS["C4"]))
    T = np.asfortranarray(O.stream_draw(11, 2, 0, "gaussian", n * m).reshape((n, m), order="F"))
    cfg = O.solver_config(kind=2, tolerance=0.01, max_epochs=10, batch_size=512, learning_rate=10.0, momentum=0.9,
                          seed=4)
    O.set_sgd_iteration_cap(iters)
    try:
        r = O.solve(X, raw, T, cfg, threads=os.cpu_count(), record_batches=iters)
    finally:
        O.set_sgd_iteration_cap(-1)
    rows = np.unique(r["batches"].reshape(-1))[:512]
    out = {"replay_rows": rows.astype(np.int32), "replay_solutions": r["solutions"][rows],
           "replay_colsum": r["solutions"].sum(axis=0), "replay_mean_residual_norm": r["mean_residual_norm"],
           "replay_probe_residual_norm": r["probe_residual_norm"], "replay_iterations": r["iterations"],
           "replay_raw": raw}
    # the same solve over its whole 10-epoch budget (7680 iterations)
    f = O.solve(X, raw, T, cfg, threads=os.cpu_count())
    sample = np.arange(0, n, 769, dtype=np.int32)
    out.update({"full_rows": sample, "full_solutions": f["solutions"][sample], "full_colsum": f["solutions"].sum(axis=0),
                "full_mean_residual_norm": f["mean_residual_norm"], "full_probe_residual_norm": f["probe_residual_norm"],
                "full_iterations": f["iterations"]})
    return out


def pack(prefix, r):
    keys = ["constrained", "gradient", "mean_residual_norm", "probe_residual_norm", "epochs", "iterations",
            "final_raw"]
    return {f"{prefix}_{k}": np.asarray(r[k]) for k in keys}


def main():
    what = sys.argv[1:] or ["validate", "c4", "c5"]
    os.makedirs(OUT, exist_ok=True)
    with O.gpu_backend(0):
        if "validate" in what:
            rep = {}
            for name, steps in (("C1", 10), ("C3", 2)):
                g = np.load(os.path.join(GOLD, name.lower() + ".npz"))
                r = traj(name, steps)
                gg = g["traj_gradient"]
                rep[name] = {
                    "seconds": r["seconds"],
                    "iterations_gpu_oracle": r["iterations"].tolist(),
                    "iterations_cpu_oracle": g["traj_iterations"].tolist(),
                    "mean_norm_rel": (np.abs(r["mean_residual_norm"] - g["traj_mean_residual_norm"]) /
                                      g["traj_mean_residual_norm"]).tolist(),
                    "probe_norm_rel": (np.abs(r["probe_residual_norm"] - g["traj_probe_residual_norm"]) /
                                       g["traj_probe_residual_norm"]).tolist(),
                    "gradient_rel_of_max": (np.abs(r["gradient"] - gg).max(axis=1) / np.abs(gg).max(axis=1)).tolist(),
                    "trajectory_rel": float(np.max(np.abs(r["constrained"] - g["traj_constrained"]) /
                                                   g["traj_constrained"]))}
                print(name, json.dumps(rep[name]), flush=True)
            # sensitivity of the C3 step to operator rounding: the FP64 oracle
            # with every H.V entry perturbed by a relative 1e-12 / 1e-7
            for noise in (1e-12, 1e-7):
                O.set_apply_sensitivity(0, noise)
                g = np.load(os.path.join(GOLD, "c3.npz"))
                r = traj("C3", 2)
                O.set_apply_sensitivity(0, 0.0)
                gg = g["traj_gradient"]
                rep[f"C3_noise_{noise:g}"] = {
                    "iterations": r["iterations"].tolist(),
                    "mean_norm_rel": (np.abs(r["mean_residual_norm"] - g["traj_mean_residual_norm"]) /
                                      g["traj_mean_residual_norm"]).tolist(),
                    "probe_norm_rel": (np.abs(r["probe_residual_norm"] - g["traj_probe_residual_norm"]) /
                                       g["traj_probe_residual_norm"]).tolist(),
                    "gradient_rel_of_max": (np.abs(r["gradient"] - gg).max(axis=1) / np.abs(gg).max(axis=1)).tolist()}
                print(f"C3 noise {noise:g}", json.dumps(rep[f"C3_noise_{noise:g}"]), flush=True)
            json.dump(rep, open(os.path.join(OUT, "scale_validate.json"), "w"), indent=1)
        if "c4" in what:
            out = sgd_replay(REPLAY_ITERS)
            print("c4 replay", out["replay_iterations"], out["replay_mean_residual_norm"], flush=True)
            r = traj("C4", 2)
            print("c4 traj", r["seconds"], r["iterations"], r["mean_residual_norm"], flush=True)
            out.update(pack("traj", r))
            np.savez_compressed(os.path.join(GOLD, "c4_scale.npz"), **out)
            np.savez_compressed(os.path.join(OUT, "c4_scale.npz"), **out)
        if "c5" in what:
            r = traj("C5", 1)
            print("c5 traj", r["seconds"], r["iterations"], r["mean_residual_norm"], flush=True)
            out = pack("traj", r)
            np.savez_compressed(os.path.join(GOLD, "c5_scale.npz"), **out)
            np.savez_compressed(os.path.join(OUT, "c5_scale.npz"), **out)


if __name__ == "__main__":
    main()
