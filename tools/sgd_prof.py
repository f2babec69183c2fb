"""Per-role barrier-wait split of the 64-column SGD slab kernel at C4 (one
epoch, 768 launches) from the instrumented build (tools/sgd_prof.sh):
  GPK_LIB_PATH=paper_2405_18457_b200/build/prof/libgpk.so python tools/sgd_prof.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18457_b200 as G  # noqa: E402
from paper_2405_18457_b200 import _lib  # noqa: E402

NAMES = ["prod st_empty", "build st_full", "build b_empty", "build bar.sync", "mma b_full", "mma d_empty",
         "mma a_full", "eval d_full", "eval st_full", "eval a_empty", "prod total", "build total", "mma total",
         "eval total", "build build"]
BW = int(os.environ.get("GPK_SGD_BW", "8"))
WARPS = {0: 1, 1: BW, 2: BW, 3: BW, 4: 1, 5: 1, 6: 1, 7: 16, 8: 16, 9: 16, 10: 1, 11: BW, 12: 1, 13: 16, 14: BW}


def main():
    n, d, m, b = 393216, 3, 65, 512
    ctx = G.Context(0)
    X32, _ = G.sinsum_dataset(n, d, True, 0.05, 0)
    raw = np.array([G.gpiter.softplus_inverse(v) for v in [1.0] * d + [1.0, 0.05]])
    op = G.KernelOperator(X32.astype(np.float64), G.Hyperparameters.from_raw(raw), ctx)
    T = np.asfortranarray(np.random.default_rng(0).standard_normal((n, m)))
    lib = _lib.load()
    f = lib.gpk_debug_sgd_prof
    f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    buf = (C.c_ulonglong * 16)()
    cfg = G.SolverConfig(kind=2, tolerance=1e-9, max_epochs=1, batch_size=b, learning_rate=float(os.environ.get("SGD_LR", "10")), momentum=0.9, seed=4)
    G.solve_sgd(G.LinearSystemBatch(op, T), cfg)
    f(buf, 1)
    G.solve_sgd(G.LinearSystemBatch(op, T), cfg)
    f(buf, 1)
    v = np.array(buf[:16], dtype=np.float64)
    for i, name in enumerate(NAMES):
        tot = v[10 + (0 if i == 0 else 1 if i < 4 else 2 if i < 7 else 3)] if i < 10 else v[11] if i == 14 else v[i]
        per_warp = v[i] / WARPS[i]
        print(f"{name:16s} {v[i]:.4e} cycles  {100 * v[i] / tot:5.1f}% of role  {per_warp / 148 / 768:9.0f} per warp-launch")


if __name__ == "__main__":
    main()
