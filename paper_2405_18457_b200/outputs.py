"""Run outputs of the GPU optimiser in the reference tool's formats (SURVEY
row f2): the trace CSV (trace.cpp, via gpk_write_trace_csv), summary.json of
`gpiter train` (/root/reference/proj/tools/gpiter_cli.cpp:118-143) and the
`compare-oracle` pair differences.csv + compare_oracle.json
(gpiter_cli.cpp:230-280), so the parity evidence of a GPU run is
byte-comparable with the reference tool's.

compare_oracle runs both trajectories on the GPU: the iterative pathwise /
standard optimiser (gpk_optimise) and Adam on the exact marginal likelihood
(gpk_optimise_exact, dense FP64 Cholesky), as the reference command does with
its CPU paths.
"""
from __future__ import annotations

import json
import math
import os

import numpy as np

from . import gpiter as G

SCHEMA_VERSION = 1  # RunConfig::kSchemaVersion (config.hpp)
HIST_EDGES = ["<=1e-8", "1e-8..1e-7", "1e-7..1e-6", "1e-6..1e-5", "1e-5..1e-4", "1e-4..1e-3", "1e-3..1e-2",
              "1e-2..1e-1", "1e-1..1", ">1"]


def format_double(value: float) -> str:
    """Shortest %.{15,16,17}g form that parses back exactly (trace.cpp:7-18)."""
    for precision in (15, 16, 17):
        text = "%.*g" % (precision, value)
        if float(text) == value:
            return text
    return "%.17g" % value


def histogram_bin(diff: float) -> int:
    """log10 bins from <= 1e-8 up (gpiter_cli.cpp:255-257)."""
    if diff <= 1e-8:
        return 0
    return min(9, 1 + int(math.floor(math.log10(diff) + 8.0)))


def write_differences(out_dir, iterative_constrained, exact_constrained):
    """differences.csv + the compare_oracle.json payload (gpiter_cli.cpp:247-278)."""
    a = np.atleast_2d(np.asarray(iterative_constrained, dtype=np.float64))
    b = np.atleast_2d(np.asarray(exact_constrained, dtype=np.float64))
    steps = min(a.shape[0], b.shape[0])
    hist = [0] * 10
    max_abs = 0.0
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "differences.csv"), "w", newline="\n") as f:
        f.write("step,coordinate,iterative,exact,abs_diff\n")
        for t in range(steps):
            for k in range(a.shape[1]):
                diff = abs(a[t, k] - b[t, k])
                max_abs = max(max_abs, diff)
                hist[histogram_bin(diff)] += 1
                f.write(f"{t},{k},{format_double(a[t, k])},{format_double(b[t, k])},{format_double(diff)}\n")
    return {"max_abs_diff": max_abs, "histogram_bin_edges": HIST_EDGES, "histogram_counts": hist}


def compare_oracle(ctx, inputs, targets, config: G.OuterConfig, out_dir, dense_cache_cap=4096):
    """`gpiter compare-oracle` on the GPU: iterative trajectory vs the exact-MLL
    Adam trajectory from the same constant initialisation, n <= dense cap."""
    X = np.asarray(inputs, dtype=np.float64)
    n, d = X.shape
    if n > dense_cache_cap:
        raise ValueError(f"compare-oracle needs n <= {dense_cache_cap}, got {n}")
    iterative = G.optimise(ctx, X, targets, config)
    init = [config.init_value] * (d + 2)
    exact_traj, _ = G.optimise_exact(ctx, X, targets, config.steps, config.learning_rate, init_constrained=init)
    out = {"steps": config.steps}
    out.update(write_differences(out_dir, iterative["constrained"], exact_traj))
    with open(os.path.join(out_dir, "compare_oracle.json"), "w") as f:
        f.write(json.dumps(out, indent=2) + "\n")
    return out


def write_summary(path, result: dict, config: G.OuterConfig, n_train: int, n_test: int = 0,
                  standardisation=None, solver_seconds=None, total_seconds=None, input_dim=None):
    """summary.json of `gpiter train` (gpiter_cli.cpp:118-143) for an optimise()
    result dict (gpiter.optimise / Optimiser.step traces concatenated)."""
    P = len(result["final_raw"]) if "final_raw" in result else result["constrained"].shape[1]
    d = input_dim if input_dim is not None else P - 2
    final_c = [G.softplus(float(v)) for v in result["final_raw"]] if "final_raw" in result else \
        list(result["constrained"][-1])
    epochs = np.asarray(result["epochs"], dtype=np.float64)
    diverged = np.asarray(result["solver_diverged"], dtype=bool)
    summary = {
        "schema_version": SCHEMA_VERSION,
        "config": {"estimator": "pathwise" if config.estimator == 1 else "standard",
                   "solver": {0: "cg", 1: "ap", 2: "sgd"}[config.solver.kind],
                   "tolerance": config.solver.tolerance, "max_epochs": config.solver.max_epochs,
                   "block_size": config.solver.block_size, "batch_size": config.solver.batch_size,
                   "sgd_learning_rate": config.solver.learning_rate, "momentum": config.solver.momentum,
                   "preconditioner_rank": config.solver.preconditioner_rank, "warm_start": bool(config.warm_start),
                   "steps": config.steps, "learning_rate": config.learning_rate, "probe_count": config.probe_count,
                   "rff_pairs": config.rff_pairs, "seeds": {"probes": config.probe_seed, "features": config.feature_seed,
                                                           "solver": config.solver_seed}},
        "n_train": int(n_train),
        "n_test": int(n_test),
        "hyperparameters": {"lengthscales": final_c[:d], "signal_scale": final_c[d], "noise_scale": final_c[d + 1]},
        "aborted": bool(result.get("aborted", False)),
        "steps_completed": int(len(epochs)),
        "total_epochs": float(epochs.sum()),
        "diverged_steps": int(diverged.sum()),
    }
    if standardisation is not None:
        summary["standardisation"] = standardisation
    if solver_seconds is None and "solver_seconds" in result:
        solver_seconds = float(np.sum(result["solver_seconds"]))
    if total_seconds is None and "step_seconds" in result:
        total_seconds = float(np.sum(result["step_seconds"]))
    summary["solver_seconds"] = solver_seconds
    summary["total_seconds"] = total_seconds
    with open(path, "w") as f:
        f.write(json.dumps(summary, indent=2) + "\n")
    return summary
