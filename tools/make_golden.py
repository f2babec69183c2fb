"""Generates tests/golden/*.npz from the FP64 oracle (oracle/, the restated
reference) at the BASELINE.json configurations. Inputs are regenerated from
the BASELINE sin-sum generator (seed 0), bit-identical in the oracle and in
libgpk, so fixtures hold only outputs.

usage: python tools/make_golden.py [c1 c2 c4 c5 ...]   (default: c1 c4 c5)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
THREADS = os.cpu_count() or 8

CFG = {
    "c1": dict(n=4096, d=8, uniform=False, noise=0.1, s=16, pairs=512, kind=0, steps=10, max_epochs=50, block=1000,
               batch=500, lr_sgd=30.0),
    "c2": dict(n=16384, d=26, uniform=False, noise=0.1, s=64, pairs=1024, kind=1, steps=2, max_epochs=50, block=512,
               batch=500, lr_sgd=30.0),
    "c3": dict(n=43008, d=20, uniform=False, noise=0.1, s=64, pairs=1000, kind=0, steps=2, max_epochs=10, block=1000,
               batch=500, lr_sgd=30.0),
    "c4": dict(n=393216, d=3, uniform=True, noise=0.05, s=64, pairs=1000, kind=2, steps=30, max_epochs=10, block=1000,
               batch=512, lr_sgd=10.0),
    "c5": dict(n=1835008, d=11, uniform=False, noise=0.1, s=64, pairs=2048, kind=0, steps=15, max_epochs=5,
               block=1000, batch=500, lr_sgd=30.0),
}
# BASELINE.json: init lengthscales 1, signal 1, noise 0.1
INIT_CONSTRAINED = lambda d: [1.0] * d + [1.0, 0.1]  # noqa: E731
INIT = lambda d: O.raw_from_constrained(INIT_CONSTRAINED(d))  # noqa: E731


def dataset(c):
    X32, y32 = O.sinsum_dataset(c["n"], c["d"], c["uniform"], c["noise"], 0)
    return np.asfortranarray(X32.astype(np.float64)), y32.astype(np.float64)


def rhs(n, m, seed=11):
    return np.asfortranarray(O.stream_draw(seed, 2, 0, "gaussian", n * m).reshape((n, m), order="F"))


def slab(name, rows=256):
    """H.V on the first `rows` rows at the init hyperparameters, V = Philox(11, 2) gaussians."""
    c = CFG[name]
    X, _ = dataset(c)
    m = c["s"] + 1
    V = rhs(c["n"], m)
    raw = INIT(c["d"])
    t = time.time()
    hv = O.apply_rows(X, raw, np.arange(rows, dtype=np.int32), V, threads=THREADS)
    print(f"{name}: slab {rows}x{c['n']}x{m} in {time.time() - t:.1f}s", flush=True)
    return {"hv_rows": hv, "raw": raw, "rows": rows}


def trajectory(name, steps=None):
    c = CFG[name]
    X, y = dataset(c)
    sc = O.solver_config(kind=c["kind"], tolerance=0.01, max_epochs=c["max_epochs"], block_size=c["block"],
                         batch_size=c["batch"], learning_rate=c["lr_sgd"], momentum=0.9, preconditioner_rank=100)
    oc = O.outer_config(estimator=1, solver=sc, warm_start=True, steps=steps or c["steps"], learning_rate=0.1,
                        probe_count=c["s"], rff_pairs=c["pairs"], probe_seed=2, feature_seed=3, solver_seed=4)
    t = time.time()
    r = O.optimise(X, y, oc, init_constrained=INIT_CONSTRAINED(c["d"]), threads=THREADS)
    print(f"{name}: {len(r['iterations'])} steps in {time.time() - t:.1f}s, iterations {list(r['iterations'])}",
          flush=True)
    return {k: np.asarray(v) for k, v in r.items()}


def main(names):
    os.makedirs(OUT, exist_ok=True)
    for name in names:
        c = CFG[name]
        out = {}
        if name in ("c1",):
            X, _ = dataset(c)
            m = c["s"] + 1
            V = rhs(c["n"], m)
            raw = INIT(c["d"])
            out["hv_full_colsum"] = O.apply(X, raw, V, threads=THREADS).sum(axis=0)
        out.update(slab(name))
        if name == "c4":
            b = c["batch"]
            out["sgd_batches"] = O.sample_without_replacement(4, 6, 0, c["n"], b, 4)
        if name in ("c1", "c2", "c3"):
            out.update({"traj_" + k: v for k, v in trajectory(name).items()})
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
        print(f"wrote tests/golden/{name}.npz", flush=True)


def main_full_c2():
    """BASELINE configs[1] at its stated step count (20 Adam steps): the
    oracle's constrained trajectory and per-step solver counts/norms only."""
    out = {"traj_" + k: v for k, v in trajectory("c2", steps=20).items()}
    np.savez_compressed(os.path.join(OUT, "c2_20.npz"), **out)
    print("wrote tests/golden/c2_20.npz", flush=True)


if __name__ == "__main__":
    if sys.argv[1:] == ["c2_20"]:
        main_full_c2()
    else:
        main(sys.argv[1:] or ["c1", "c4", "c5"])
