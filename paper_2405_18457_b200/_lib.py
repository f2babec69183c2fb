"""Loads libgpk.so (the sm_100a CUDA kernels + C-ABI, built in-tree).

There is no fallback: if the shared library is missing or the GPU is not an
sm_100 part, every call fails loudly with GpkError.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgpk.so")
# development A/B: GPK_LIB_PATH points at another in-tree build of the same C-ABI
LIB_PATH = os.environ.get("GPK_LIB_PATH", LIB_PATH)
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "gpk.h")

GPK_OK, GPK_EINVAL, GPK_ERANGE, GPK_ENUMERIC, GPK_ECUDA, GPK_ENCCL = range(6)


class GpkError(RuntimeError):
    pass


class SolverConfigC(C.Structure):
    _fields_ = [("kind", C.c_int), ("tolerance", C.c_double), ("max_epochs", C.c_int),
                ("block_size", C.c_int), ("batch_size", C.c_int), ("learning_rate", C.c_double),
                ("momentum", C.c_double), ("preconditioner_rank", C.c_int), ("warm_start", C.c_int),
                ("seed", C.c_uint64), ("substream", C.c_uint64)]


class SolverReportC(C.Structure):
    _fields_ = [("iterations", C.c_int), ("epochs_consumed", C.c_double),
                ("mean_residual_norm", C.c_double), ("probe_residual_norm", C.c_double),
                ("reached_tolerance", C.c_int), ("residuals_estimated", C.c_int), ("aborted", C.c_int),
                ("abort_reason", C.c_char * 128), ("wall_seconds", C.c_double)]


class OuterConfigC(C.Structure):
    _fields_ = [("estimator", C.c_int), ("solver", SolverConfigC), ("warm_start", C.c_int),
                ("steps", C.c_int), ("learning_rate", C.c_double), ("probe_count", C.c_int),
                ("rff_pairs", C.c_int), ("probe_distribution", C.c_int), ("probe_seed", C.c_uint64),
                ("feature_seed", C.c_uint64), ("solver_seed", C.c_uint64), ("init_value", C.c_double),
                ("divergence_policy", C.c_int), ("prior_mode", C.c_int)]


_lib = None
dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
vp = C.c_void_p


def _sig(lib):
    H = vp  # opaque handles
    spec = {
        "gpk_last_error": (C.c_char_p, []),
        "gpk_version": (C.c_char_p, []),
        "gpk_rhs_ld": (C.c_int, [C.c_int]),
        "gpk_ctx_create": (C.c_int, [C.c_int, C.POINTER(H)]),
        "gpk_ctx_destroy": (C.c_int, [H]),
        "gpk_ctx_synchronize": (C.c_int, [H]),
        "gpk_ctx_join": (C.c_int, [H]),
        "gpk_ctx_launch_count": (C.c_int, [H, C.POINTER(C.c_longlong)]),
        "gpk_ctx_stream": (C.c_int, [H, C.POINTER(vp)]),
        "gpk_ctx_set_profiling": (C.c_int, [H, C.c_int]),
        "gpk_ctx_set_operator_kernel": (C.c_int, [H, C.c_int]),
        "gpk_ctx_reset_stats": (C.c_int, [H]),
        "gpk_ctx_stats": (C.c_int, [H, dp]),
        "gpk_operator_create": (C.c_int, [H, dp, C.c_int, C.c_int, dp, C.POINTER(H)]),
        "gpk_operator_set_hyperparameters": (C.c_int, [H, dp]),
        "gpk_operator_set_dense_cache": (C.c_int, [H, C.c_int]),
        "gpk_operator_destroy": (C.c_int, [H]),
        "gpk_operator_size": (C.c_int, [H, ip, ip]),
        "gpk_apply": (C.c_int, [H, dp, C.c_int, dp]),
        "gpk_apply_rows": (C.c_int, [H, ip, C.c_int, dp, C.c_int, dp]),
        "gpk_apply_columns": (C.c_int, [H, C.c_int, C.c_int, dp, C.c_int, dp]),
        "gpk_dense_block": (C.c_int, [H, C.c_int, C.c_int, C.c_int, C.c_int, dp]),
        "gpk_derivative_apply": (C.c_int, [H, C.c_int, dp, C.c_int, dp]),
        "gpk_kernel_column": (C.c_int, [H, C.c_int, dp]),
        "gpk_kernel_diagonal": (C.c_int, [H, dp]),
        "gpk_derivative_quadratic_forms_many": (C.c_int, [H, C.c_int, C.POINTER(dp), C.POINTER(dp), ip, dp]),
        "gpk_apply_device": (C.c_int, [H, vp, C.c_int, vp, C.c_int]),
        "gpk_precond_create": (C.c_int, [H, C.c_int, C.POINTER(H)]),
        "gpk_precond_destroy": (C.c_int, [H]),
        "gpk_precond_info": (C.c_int, [H, ip, ip]),
        "gpk_precond_factor": (C.c_int, [H, dp, ip]),
        "gpk_precond_apply": (C.c_int, [H, dp, C.c_int, dp]),
        "gpk_batch_create": (C.c_int, [H, dp, C.c_int, C.POINTER(H)]),
        "gpk_batch_destroy": (C.c_int, [H]),
        "gpk_batch_warm_start": (C.c_int, [H, dp]),
        "gpk_batch_warm_start_from": (C.c_int, [H, H]),
        "gpk_batch_refresh_residuals": (C.c_int, [H]),
        "gpk_batch_get": (C.c_int, [H, C.c_int, dp]),
        "gpk_batch_set": (C.c_int, [H, C.c_int, dp]),
        "gpk_termination_check": (C.c_int, [H, C.c_double, dp, dp, ip]),
        "gpk_solve_cg": (C.c_int, [H, C.POINTER(SolverConfigC), H, C.POINTER(SolverReportC)]),
        "gpk_solve_ap": (C.c_int, [H, C.POINTER(SolverConfigC), C.POINTER(SolverReportC)]),
        "gpk_solve_sgd": (C.c_int, [H, C.POINTER(SolverConfigC), C.POINTER(SolverReportC)]),
        "gpk_solve": (C.c_int, [H, C.POINTER(SolverConfigC), C.POINTER(SolverReportC)]),
        "gpk_sgd_batches": (C.c_int, [H, C.c_int, C.POINTER(SolverConfigC), C.c_int, C.c_int, ip]),
        "gpk_estimate_gradient_pathwise": (C.c_int, [H, dp, dp, C.c_int, dp, dp, dp]),
        "gpk_estimate_gradient_standard": (C.c_int, [H, dp, dp, dp, C.c_int, dp, dp, dp]),
        "gpk_batch_gradient_pathwise": (C.c_int, [H, dp, dp, dp]),
        "gpk_rff_basis_build": (C.c_int, [H, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.POINTER(H)]),
        "gpk_rff_basis_destroy": (C.c_int, [H]),
        "gpk_rff_basis_get": (C.c_int, [H, dp, dp]),
        "gpk_pathwise_targets": (C.c_int, [H, H, C.c_int, C.c_uint64, C.c_uint64, dp, dp, dp]),
        "gpk_optimise": (C.c_int, [H, dp, dp, C.c_int, C.c_int, C.POINTER(OuterConfigC), dp, dp, ip, dp, ip]),
        "gpk_optimiser_create": (C.c_int, [H, dp, dp, C.c_int, C.c_int, C.POINTER(OuterConfigC), dp,
                                           C.POINTER(H)]),
        "gpk_optimiser_step": (C.c_int, [H, C.c_int, dp, ip]),
        "gpk_optimiser_state": (C.c_int, [H, dp, ip, ip]),
        "gpk_optimiser_destroy": (C.c_int, [H]),
        "gpk_comm_unique_id": (C.c_int, [C.POINTER(C.c_ubyte)]),
        "gpk_ctx_init_comm": (C.c_int, [H, C.POINTER(C.c_ubyte), C.c_int, C.c_int]),
        "gpk_shard_rows": (C.c_int, [C.c_int, C.c_int, C.c_int, ip, ip]),
        "gpk_cross_apply": (C.c_int, [H, dp, C.c_int, dp, C.c_int, dp]),
        "gpk_predict_mean": (C.c_int, [H, dp, C.c_int, dp, dp]),
        "gpk_sample_posterior": (C.c_int, [H, H, dp, C.c_int, dp, dp, C.c_int, dp]),
        "gpk_test_metrics": (C.c_int, [H, H, dp, C.c_int, dp, dp, dp, C.c_int, C.c_double, dp]),
        "gpk_write_trace_csv": (C.c_int, [C.c_char_p, dp, C.c_int, C.c_int]),
        "gpk_spd_inverse": (C.c_int, [vp, dp, C.c_int, C.c_int, C.c_int, dp]),
        "gpk_optimise_exact": (C.c_int, [vp, dp, dp, C.c_int, C.c_int, dp, C.c_int, C.c_double, dp, dp]),
        "gpk_init_heuristic": (C.c_int, [vp, dp, dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int,
                                         C.c_double, dp]),
        "gpk_sinsum_dataset": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64,
                                         C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    }
    for name, (res, args) in spec.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def load():
    """Returns the loaded libgpk CDLL; raises GpkError if it is not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise GpkError(f"libgpk.so not found at {LIB_PATH}; run __graft_entry__.build() "
                           "(make -C paper_2405_18457_b200)")
        lib = C.CDLL(LIB_PATH)
        _sig(lib)
        _lib = lib
    return _lib


def check(rc):
    if rc != GPK_OK:
        msg = load().gpk_last_error().decode()
        if rc == GPK_EINVAL:
            raise ValueError(msg)
        if rc == GPK_ERANGE:
            raise IndexError(msg)
        if rc == GPK_ENUMERIC:
            raise ArithmeticError(msg)
        raise GpkError(msg)
