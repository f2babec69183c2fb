import numpy as np, sys, os
sys.path.insert(0, os.getcwd())
import paper_2405_18457_b200 as G
ctx = G.Context(0)
X32, y32 = G.sinsum_dataset(16384, 26, False, 0.1, 0)
sc = G.SolverConfig(kind=1, tolerance=0.01, max_epochs=50, block_size=512)
oc = G.OuterConfig(estimator=1, solver=sc, warm_start=True, steps=20, learning_rate=0.1, probe_count=64,
                   rff_pairs=1024, probe_seed=2, feature_seed=3, solver_seed=4)
r = G.optimise(ctx, X32.astype(np.float64), y32.astype(np.float64), oc, init_constrained=[1.0] * 26 + [1.0, 0.1])
np.savez("gpurun_out/c2_20_gpu.npz", **{k: np.asarray(v) for k, v in r.items()})
print({k: np.asarray(v).shape for k, v in r.items()})
print("iterations", list(np.asarray(r["iterations"])))
