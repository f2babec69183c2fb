"""The C++ drop-in shim (include/gpiter_b200.hpp) compiles against the C-ABI
(CPU), and on a GPU its results match the FP64 oracle (gpu)."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "shim_smoke.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "shim_smoke")


def build_shim():
    subprocess.run(["g++", "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"), SRC,
                    "-L" + os.path.join(ROOT, "paper_2405_18457_b200"), "-lgpk",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_2405_18457_b200"), "-o", BIN], check=True)


def test_shim_compiles_and_links():
    build_shim()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_shim_matches_oracle(oracle):
    if not os.path.exists(BIN):
        build_shim()
    out = json.loads(subprocess.run([BIN], capture_output=True, text=True, check=True).stdout)
    n, d, s = 512, 3, 4
    i = np.arange(n)
    X = np.stack([np.sin(0.37 * i + 1.3 * k) for k in range(d)], axis=1)
    raw = np.array([0.5] * (d + 1) + [-1.0])
    V = np.stack([np.cos(0.11 * i * (j + 1)) for j in range(s + 1)], axis=1)
    hv = oracle.apply(X, raw, V)
    assert abs(out["hv00"] - hv[0, 0]) <= 2e-5 * np.max(np.abs(hv[:, 0]))
    assert abs(out["hv_last"] - hv[-1, s]) <= 2e-5 * np.max(np.abs(hv[:, s]))
    assert out["threw_invalid_argument"] == 1
    for kind, name in enumerate(("cg", "ap", "sgd")):
        cfg = oracle.solver_config(kind=kind, tolerance=0.01, max_epochs=200, block_size=64, batch_size=64,
                                   learning_rate=2.0, seed=4)
        r = oracle.solve(X, raw, V, cfg)
        assert abs(out[f"{name}_iterations"] - r["iterations"]) <= 1, name
    # the gradient of the shim's own CG solutions (row-major n x (s+1)). This
    # problem is an FP32 stress case: its trace/quadratic sums cancel by ~4e5
    # (sum of |terms| / |sum|), so any FP32 evaluation of the forms (SIMT pass
    # 7e-4, tensor-core pass ~5e-3; tools/grad_precision.py, profiles/) misses
    # 1e-4 here; the pass is pinned at 1e-4 on ordinary inputs by
    # test_gpu_parity.py::test_quadratic_forms_match_oracle. This test checks
    # the C++ plumbing (signs, ordering, scaling of every component).
    sol = np.array(out["cg_solutions"]).reshape(n, s + 1)
    g = oracle.gradient(X, raw, sol[:, 0], sol[:, 1:])["values"]
    assert np.max(np.abs(np.array(out["grad"]) - g) / np.maximum(np.abs(g), 1e-2)) <= 1e-2
