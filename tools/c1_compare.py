"""C1 (BASELINE configs[0]) 10-step trajectory on the GPU against tests/golden/c1.npz: iteration counts,
residual norms and per-step gradient errors (GPK_DENSE_KV64=0 selects the cached-matrix DGEMM path)."""
import numpy as np, sys, os
sys.path.insert(0, os.getcwd())
import paper_2405_18457_b200 as G
g = np.load("tests/golden/c1.npz")
ctx = G.Context(0)
X32, y32 = G.sinsum_dataset(4096, 8, False, 0.1, 0)
sc = G.SolverConfig(kind=0, tolerance=0.01, max_epochs=50, preconditioner_rank=100)
oc = G.OuterConfig(estimator=1, solver=sc, warm_start=True, steps=10, learning_rate=0.1, probe_count=16,
                   rff_pairs=512, probe_seed=2, feature_seed=3, solver_seed=4)
r = G.optimise(ctx, X32.astype(np.float64), y32.astype(np.float64), oc, init_constrained=[1.0] * 8 + [1.0, 0.1])
print("gpu iters   ", list(r["iterations"]))
print("oracle iters", list(g["traj_iterations"]))
print("traj rel", np.max(np.abs(r["constrained"] - g["traj_constrained"]) / g["traj_constrained"]))
for k in ["mean_residual_norm", "probe_residual_norm"]:
    print(k, np.max(np.abs(r[k] - g["traj_" + k]) / g["traj_" + k]))
gg = g["traj_gradient"]; print("grad rel", np.max(np.abs(r["gradient"] - gg) / np.abs(gg).max(axis=1, keepdims=True)))
print("step seconds", list(np.round(r["step_seconds"], 5)))
print("grad rel-of-max per step", [f"{v:.2e}" for v in (np.abs(r["gradient"] - gg) / np.abs(gg).max(axis=1, keepdims=True)).max(axis=1)])
print("mean norm rel per step", [f"{v:.2e}" for v in np.abs(r["mean_residual_norm"] - g["traj_mean_residual_norm"]) / g["traj_mean_residual_norm"]])
