"""The C-ABI library loads on CPU-only hosts and exports every entry point
include/gpk.h declares (no compute calls: no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gpk.h")
LIB = os.path.join(ROOT, "paper_2405_18457_b200", "libgpk.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(gpk_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_reference_surface():
    syms = declared_symbols()
    for must in ("gpk_apply", "gpk_apply_rows", "gpk_apply_columns", "gpk_dense_block", "gpk_kernel_column",
                 "gpk_derivative_quadratic_forms_many", "gpk_solve_cg", "gpk_solve_ap", "gpk_solve_sgd", "gpk_solve",
                 "gpk_precond_create", "gpk_precond_apply", "gpk_estimate_gradient_pathwise",
                 "gpk_pathwise_targets", "gpk_rff_basis_build", "gpk_optimise", "gpk_termination_check"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-C", os.path.dirname(LIB)], check=True)
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_python_mirror_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2405_18457_b200 import Context
    with pytest.raises(Exception):
        Context(0)
