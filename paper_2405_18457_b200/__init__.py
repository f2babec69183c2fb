"""B200-native matrix-free GP kernel operator and iterative solvers
(arXiv 2405.18457 hot path): CUDA sm_100a kernels behind a C-ABI (include/gpk.h),
with a host mirror of the reference gpiter API in :mod:`.gpiter`."""
from ._lib import GpkError, LIB_PATH, load  # noqa: F401
from .gpiter import (  # noqa: F401
    AP, CG, SGD, Context, GradientEstimate, Hyperparameters, KernelOperator, LinearSystemBatch, Optimiser, OuterConfig,
    PivotedCholeskyPreconditioner, RffBasis, SolverConfig, SolverReport, build_rff_basis, estimate_gradient_pathwise,
    estimate_gradient_standard, optimise, pathwise_targets, sgd_batches, sinsum_dataset, solve, solve_ap, solve_cg, solve_sgd,
    termination_check)
from .gpiter import cross_kernel_apply, predict_mean, sample_posterior, test_metrics  # noqa: F401
