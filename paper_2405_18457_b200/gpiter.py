"""Host-side mirror of the reference gpiter C++ API over the libgpk C-ABI.

Names, argument meanings and error behaviour follow
/root/reference/proj/core/include/gpiter/*.hpp (cited per class); matrices are
numpy arrays in the reference's column-major FP64 convention. Every compute
call runs on the GPU through libgpk.so; nothing here computes on the CPU.

Error mapping (include/gpk.h): std::invalid_argument -> ValueError,
std::out_of_range -> IndexError, std::runtime_error -> ArithmeticError.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math

import numpy as np

from . import _lib
from ._lib import OuterConfigC, SolverConfigC, SolverReportC, check

CG, AP, SGD = 0, 1, 2


def _f64(a, ndim=2):
    a = np.asarray(a, dtype=np.float64)
    if ndim == 2 and a.ndim == 1:
        a = a[:, None]
    return np.asfortranarray(a)


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


# ---- hyperparameters (hyperparameters.hpp:19-49) -------------------------
def softplus(x):
    return x + math.log1p(math.exp(-x)) if x > 0 else math.log1p(math.exp(x))


def softplus_inverse(y):
    if y <= 0:
        raise ValueError("softplus_inverse: argument must be positive")
    return y + math.log(-math.expm1(-y))


def sigmoid(x):
    if x >= 0:
        return 1.0 / (1.0 + math.exp(-x))
    e = math.exp(x)
    return e / (1.0 + e)


class Hyperparameters:
    """Raw vector [l_1..l_d, signal, noise]; constrained = softplus(raw)."""

    def __init__(self, raw):
        raw = np.asarray(raw, dtype=np.float64).copy()
        if raw.size < 3:
            raise ValueError("Hyperparameters: need at least d=1 plus scales")
        self.raw = raw

    @staticmethod
    def from_raw(raw):
        return Hyperparameters(raw)

    @staticmethod
    def from_constrained(c):
        return Hyperparameters([softplus_inverse(float(v)) for v in c])

    @staticmethod
    def constant(d, value):
        return Hyperparameters.from_constrained([value] * (d + 2))

    def input_dim(self):
        return self.raw.size - 2

    def count(self):
        return self.raw.size

    def constrained(self):
        return np.array([softplus(v) for v in self.raw])

    def lengthscales(self):
        return self.constrained()[:-2]

    def signal_scale(self):
        return softplus(self.raw[-2])

    def noise_scale(self):
        return softplus(self.raw[-1])

    def noise_variance(self):
        return self.noise_scale() ** 2

    @staticmethod
    def signal_index(d):
        return d

    @staticmethod
    def noise_index(d):
        return d + 1


# ---- context --------------------------------------------------------------
class Context:
    """One CUDA device + stream (one process per GPU)."""

    def __init__(self, device=0):
        self._lib = _lib.load()
        h = C.c_void_p()
        check(self._lib.gpk_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    def synchronize(self):
        check(self._lib.gpk_ctx_synchronize(self.handle))

    def join(self):
        """Stream-orders the auxiliary stream's pending work before later work (gpk_ctx_join)."""
        check(self._lib.gpk_ctx_join(self.handle))

    def launch_count(self):
        v = C.c_longlong()
        check(self._lib.gpk_ctx_launch_count(self.handle, C.byref(v)))
        return v.value

    def stream(self):
        v = C.c_void_p()
        check(self._lib.gpk_ctx_stream(self.handle, C.byref(v)))
        return v.value

    def init_comm(self, unique_id: bytes, nranks: int, rank: int):
        """Joins the NCCL communicator (one process per GPU); see gpk_ctx_init_comm."""
        buf = (C.c_ubyte * 128).from_buffer_copy(unique_id)
        check(self._lib.gpk_ctx_init_comm(self.handle, buf, nranks, rank))

    def set_operator_kernel(self, kernel: int):
        """0 = FP32 SIMT operator kernel, 1 = tcgen05 3xTF32 operator kernel."""
        check(self._lib.gpk_ctx_set_operator_kernel(self.handle, int(kernel)))

    def set_profiling(self, enable: bool):
        check(self._lib.gpk_ctx_set_profiling(self.handle, int(enable)))

    def reset_stats(self):
        check(self._lib.gpk_ctx_reset_stats(self.handle))

    def stats(self):
        """K.V operator counters: evals x RHS, FP32-equivalent flops (2m+3d+6 per entry), profiled
        launches, profiled ms, flops on the FP32 pipe (3d+6 per entry on the tcgen05 kernel)."""
        out = np.zeros(5)
        check(self._lib.gpk_ctx_stats(self.handle, _p(out)))
        return {"evals_x_rhs": out[0], "flops": out[1], "kv_launches": int(out[2]), "kv_ms": out[3],
                "fp32_pipe_flops": out[4]}

    def close(self):
        if getattr(self, "handle", None):
            self._lib.gpk_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx = None


def default_context():
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ---- KernelOperator (kernel.hpp:37-97) ------------------------------------
class KernelOperator:
    def __init__(self, inputs, hp: Hyperparameters, ctx: Context | None = None, dense_cache: bool = False):
        self.ctx = ctx or default_context()
        self._lib = self.ctx._lib
        X = _f64(inputs)
        n, d = X.shape
        if hp.input_dim() != d:
            raise ValueError("KernelOperator: dataset dimension does not match hyperparameters")
        self.n, self.d = n, d
        self.hp = hp
        self.inputs = X
        h = C.c_void_p()
        check(self._lib.gpk_operator_create(self.ctx.handle, _p(X), n, d, _p(hp.raw), C.byref(h)))
        self.handle = h
        if dense_cache:  # KernelOperatorOptions::dense_cache: FP64 full products
            check(self._lib.gpk_operator_set_dense_cache(h, 1))

    def size(self):
        return self.n

    def param_count(self):
        return self.hp.count()

    def params(self):
        return self.hp

    def set_hyperparameters(self, hp: Hyperparameters):
        check(self._lib.gpk_operator_set_hyperparameters(self.handle, _p(np.ascontiguousarray(hp.raw))))
        self.hp = hp

    def apply(self, v):
        V = _f64(v)
        if V.shape[0] != self.n:
            raise ValueError("KernelOperator::apply: dimension mismatch")
        out = np.empty(V.shape, order="F")
        check(self._lib.gpk_apply(self.handle, _p(V), V.shape[1], _p(out)))
        return out

    def apply_rows(self, rows, v):
        V = _f64(v)
        r = np.ascontiguousarray(rows, dtype=np.int32)
        out = np.empty((r.size, V.shape[1]), order="F")
        check(self._lib.gpk_apply_rows(self.handle, r.ctypes.data_as(C.POINTER(C.c_int)), r.size, _p(V),
                                       V.shape[1], _p(out)))
        return out

    def apply_columns(self, c0, length, u):
        U = _f64(u)
        if U.shape[0] != length:
            raise ValueError("KernelOperator::apply_columns: height mismatch")
        out = np.empty((self.n, U.shape[1]), order="F")
        check(self._lib.gpk_apply_columns(self.handle, c0, length, _p(U), U.shape[1], _p(out)))
        return out

    def dense_block(self, r0, rows, c0, cols):
        out = np.empty((rows, cols), order="F")
        check(self._lib.gpk_dense_block(self.handle, r0, rows, c0, cols, _p(out)))
        return out

    def dense(self):
        return self.dense_block(0, self.n, 0, self.n)

    def derivative_apply(self, k, v):
        """(dH/dtheta_k) V (kernel.hpp:71): lengthscales k < d, signal k = d, noise k = d + 1."""
        V = _f64(v)
        out = np.empty(V.shape, order="F")
        check(self._lib.gpk_derivative_apply(self.handle, int(k), _p(V), V.shape[1], _p(out)))
        return out

    def kernel_column(self, i):
        out = np.empty(self.n)
        check(self._lib.gpk_kernel_column(self.handle, i, _p(out)))
        return out

    def kernel_diagonal(self):
        out = np.empty(self.n)
        check(self._lib.gpk_kernel_diagonal(self.handle, _p(out)))
        return out

    def derivative_quadratic_forms_many(self, pairs):
        mats = [(_f64(u), _f64(w)) for u, w in pairs]
        for u, w in mats:
            if u.shape[0] != self.n or w.shape[0] != self.n or u.shape[1] != w.shape[1]:
                raise ValueError("derivative_quadratic_forms: shape mismatch")
        k = len(mats)
        U = (C.POINTER(C.c_double) * k)(*[_p(u) for u, _ in mats])
        W = (C.POINTER(C.c_double) * k)(*[_p(w) if w is not u else _p(u) for u, w in mats])
        # identical objects signal U == W to the library (symmetric pass)
        for i, (u, w) in enumerate(pairs):
            if u is w:
                W[i] = U[i]
        cols = (C.c_int * k)(*[u.shape[1] for u, _ in mats])
        out = np.empty((k, self.d + 2))
        check(self._lib.gpk_derivative_quadratic_forms_many(self.handle, k, U, W, cols, _p(out)))
        return [out[i].copy() for i in range(k)]

    def derivative_quadratic_forms(self, u, w):
        return self.derivative_quadratic_forms_many([(u, w)])[0]

    def close(self):
        if getattr(self, "handle", None):
            self._lib.gpk_operator_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- PivotedCholeskyPreconditioner (pivoted_cholesky.hpp:13-32) ----------
class PivotedCholeskyPreconditioner:
    def __init__(self, op: KernelOperator, rank: int):
        self.op = op
        self._lib = op._lib
        h = C.c_void_p()
        check(self._lib.gpk_precond_create(op.handle, rank, C.byref(h)))
        self.handle = h
        self.rank = rank

    def achieved_rank(self):
        a, s = C.c_int(), C.c_int()
        check(self._lib.gpk_precond_info(self.handle, C.byref(a), C.byref(s)))
        return a.value

    def stopped_early(self):
        a, s = C.c_int(), C.c_int()
        check(self._lib.gpk_precond_info(self.handle, C.byref(a), C.byref(s)))
        return bool(s.value)

    def factor(self):
        r = self.achieved_rank()
        out = np.zeros((self.op.n, max(r, 1)), order="F")
        piv = np.zeros(max(r, 1), dtype=np.int32)
        check(self._lib.gpk_precond_factor(self.handle, _p(out), piv.ctypes.data_as(C.POINTER(C.c_int))))
        return out[:, :r]

    def pivots(self):
        r = self.achieved_rank()
        piv = np.zeros(max(r, 1), dtype=np.int32)
        check(self._lib.gpk_precond_factor(self.handle, None, piv.ctypes.data_as(C.POINTER(C.c_int))))
        return piv[:r]

    def apply(self, v):
        V = _f64(v)
        out = np.empty(V.shape, order="F")
        check(self._lib.gpk_precond_apply(self.handle, _p(V), V.shape[1], _p(out)))
        return out

    def close(self):
        if getattr(self, "handle", None):
            self._lib.gpk_precond_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- SolverConfig / SolverReport (linear_system.hpp:14-40) ----------------
@dataclasses.dataclass
class SolverConfig:
    kind: int = CG
    tolerance: float = 0.01
    max_epochs: int = 50
    block_size: int = 1000
    batch_size: int = 500
    learning_rate: float = 30.0
    momentum: float = 0.9
    preconditioner_rank: int = 100
    warm_start: bool = False
    seed: int = 0
    substream: int = 0

    def c(self):
        return SolverConfigC(self.kind, self.tolerance, self.max_epochs, self.block_size, self.batch_size,
                             self.learning_rate, self.momentum, self.preconditioner_rank, int(self.warm_start),
                             self.seed, self.substream)


@dataclasses.dataclass
class SolverReport:
    iterations: int
    epochs_consumed: float
    mean_residual_norm: float
    probe_residual_norm: float
    reached_tolerance: bool
    residuals_estimated: bool
    aborted: bool
    abort_reason: str
    wall_seconds: float

    @staticmethod
    def from_c(r: SolverReportC):
        return SolverReport(r.iterations, r.epochs_consumed, r.mean_residual_norm, r.probe_residual_norm,
                            bool(r.reached_tolerance), bool(r.residuals_estimated), bool(r.aborted),
                            r.abort_reason.decode(), r.wall_seconds)


# ---- LinearSystemBatch (linear_system.hpp:45-68) --------------------------
class LinearSystemBatch:
    kNormEpsilon = 1e-12

    def __init__(self, op: KernelOperator, targets):
        T = _f64(targets)
        if T.shape[0] != op.n:
            raise ValueError("LinearSystemBatch: target height does not match operator")
        self.op = op
        self._lib = op._lib
        self.m = T.shape[1]
        h = C.c_void_p()
        check(self._lib.gpk_batch_create(op.handle, _p(T), self.m, C.byref(h)))
        self.handle = h

    def columns(self):
        return self.m

    def probe_count(self):
        return self.m - 1

    def _get(self, which):
        out = np.empty((self.op.n, self.m), order="F") if which < 3 else np.empty(self.m)
        check(self._lib.gpk_batch_get(self.handle, which, _p(out)))
        return out

    def _set(self, which, a):
        A = _f64(a)
        check(self._lib.gpk_batch_set(self.handle, which, _p(A)))

    @property
    def targets(self):
        return self._get(0)

    @property
    def solutions(self):
        return self._get(1)

    @property
    def residuals(self):
        return self._get(2)

    @residuals.setter
    def residuals(self, value):
        self._set(2, value)

    @property
    def scales(self):
        return self._get(3)

    def warm_start(self, previous):
        P = _f64(previous)
        if P.shape != (self.op.n, self.m):
            raise ValueError("LinearSystemBatch::warm_start: shape mismatch")
        check(self._lib.gpk_batch_warm_start(self.handle, _p(P)))

    def refresh_residuals(self):
        check(self._lib.gpk_batch_refresh_residuals(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            self._lib.gpk_batch_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclasses.dataclass
class TerminationStatus:
    mean_norm: float
    probe_norm: float
    done: bool


def termination_check(batch: LinearSystemBatch, tolerance: float) -> TerminationStatus:
    mean, probe, done = C.c_double(), C.c_double(), C.c_int()
    check(batch._lib.gpk_termination_check(batch.handle, tolerance, C.byref(mean), C.byref(probe), C.byref(done)))
    return TerminationStatus(mean.value, probe.value, bool(done.value))


# ---- solvers (solvers.hpp:10-25) -----------------------------------------
def _run(fn, batch, config, *extra):
    rep = SolverReportC()
    cfg = config.c()
    check(fn(batch.handle, C.byref(cfg), *extra, C.byref(rep)))
    return SolverReport.from_c(rep)


def solve_cg(batch, config, precond: PivotedCholeskyPreconditioner | None = None):
    return _run(batch._lib.gpk_solve_cg, batch, config, precond.handle if precond is not None else None)


def solve_ap(batch, config):
    return _run(batch._lib.gpk_solve_ap, batch, config)


def solve_sgd(batch, config):
    return _run(batch._lib.gpk_solve_sgd, batch, config)


def solve(batch, config):
    return _run(batch._lib.gpk_solve, batch, config)


def sgd_batches(ctx: Context, n: int, config: SolverConfig, first: int, count: int):
    b = min(config.batch_size, n)
    out = np.empty((count, b), dtype=np.int32)
    cfg = config.c()
    check(ctx._lib.gpk_sgd_batches(ctx.handle, n, C.byref(cfg), first, count,
                                   out.ctypes.data_as(C.POINTER(C.c_int))))
    return out


# ---- gradients (gradients.hpp:41-48) --------------------------------------
@dataclasses.dataclass
class GradientEstimate:
    values: np.ndarray
    quadratic_term: np.ndarray
    trace_term: np.ndarray


def estimate_gradient_pathwise(op: KernelOperator, v_y, zhat) -> GradientEstimate:
    Z = _f64(zhat)
    if Z.shape[0] != op.n:
        raise ValueError("estimate_gradient_pathwise: shape mismatch")
    vy = np.ascontiguousarray(v_y, dtype=np.float64).reshape(-1)
    k = op.d + 2
    v, q, t = np.empty(k), np.empty(k), np.empty(k)
    check(op._lib.gpk_estimate_gradient_pathwise(op.handle, _p(vy), _p(Z), Z.shape[1], _p(v), _p(q), _p(t)))
    return GradientEstimate(v, q, t)


def estimate_gradient_standard(op: KernelOperator, v_y, solutions, probes) -> GradientEstimate:
    S, P = _f64(solutions), _f64(probes)
    if S.shape[0] != op.n or P.shape[0] != op.n or S.shape[1] != P.shape[1]:
        raise ValueError("estimate_gradient_standard: shape mismatch")
    vy = np.ascontiguousarray(v_y, dtype=np.float64).reshape(-1)
    k = op.d + 2
    v, q, t = np.empty(k), np.empty(k), np.empty(k)
    check(op._lib.gpk_estimate_gradient_standard(op.handle, _p(vy), _p(S), _p(P), S.shape[1], _p(v), _p(q), _p(t)))
    return GradientEstimate(v, q, t)


# ---- RFF (rff.hpp:27-54) ---------------------------------------------------
class RffBasis:
    def __init__(self, ctx: Context, d, m_pairs, sample_count, seed, substream=0):
        self.ctx = ctx
        self._lib = ctx._lib
        h = C.c_void_p()
        check(self._lib.gpk_rff_basis_build(ctx.handle, d, m_pairs, sample_count, seed, substream, C.byref(h)))
        self.handle = h
        self.d, self.m_pairs, self.samples, self.seed = d, m_pairs, sample_count, seed

    def pairs(self):
        return self.m_pairs

    def sample_count(self):
        return self.samples

    def arrays(self):
        f = np.empty((self.m_pairs, self.d), order="F")
        w = np.empty((2 * self.m_pairs, self.samples), order="F")
        check(self._lib.gpk_rff_basis_get(self.handle, _p(f), _p(w)))
        return f, w

    def close(self):
        if getattr(self, "handle", None):
            self._lib.gpk_rff_basis_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_rff_basis(ctx, input_dim, m_pairs, sample_count, seed, substream=0):
    return RffBasis(ctx, input_dim, m_pairs, sample_count, seed, substream)


@dataclasses.dataclass
class PathwiseTargets:
    prior_values: np.ndarray
    noise: np.ndarray
    xi: np.ndarray


def pathwise_targets(basis: RffBasis, op: KernelOperator, s, seed, substream=0) -> PathwiseTargets:
    n = op.n
    prior, noise, xi = (np.empty((n, s), order="F") for _ in range(3))
    check(op._lib.gpk_pathwise_targets(op.handle, basis.handle, s, seed, substream, _p(prior), _p(noise), _p(xi)))
    return PathwiseTargets(prior, noise, xi)


# ---- outer loop (outer_loop.hpp:37-90) ------------------------------------
@dataclasses.dataclass
class OuterConfig:
    estimator: int = 1  # 0 standard, 1 pathwise
    solver: SolverConfig = dataclasses.field(default_factory=SolverConfig)
    warm_start: bool = False
    steps: int = 100
    learning_rate: float = 0.1
    probe_count: int = 64
    rff_pairs: int = 1000
    probe_distribution: int = 0
    probe_seed: int = 0
    feature_seed: int = 0
    solver_seed: int = 0
    init_value: float = 1.0
    divergence_policy: int = 0
    prior_mode: int = 0  # pathwise prior: 0 random features, 1 exact dense (n <= 4096)

    def c(self):
        return OuterConfigC(self.estimator, self.solver.c(), int(self.warm_start), self.steps, self.learning_rate,
                            self.probe_count, self.rff_pairs, self.probe_distribution, self.probe_seed,
                            self.feature_seed, self.solver_seed, self.init_value, self.divergence_policy,
                            self.prior_mode)


def optimise(ctx: Context, inputs, targets, config: OuterConfig, init_constrained=None):
    """Returns dict of per-step trace arrays plus final raw hyperparameters."""
    X = _f64(inputs)
    y = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1)
    n, d = X.shape
    P = d + 2
    stride = 2 * P + 8
    trace = np.zeros((max(config.steps, 1), stride))
    rows, aborted = C.c_int(), C.c_int()
    final_raw = np.empty(P)
    ic = np.ascontiguousarray(init_constrained, dtype=np.float64) if init_constrained is not None else None
    cfg = config.c()
    check(ctx._lib.gpk_optimise(ctx.handle, _p(X), _p(y), n, d, C.byref(cfg), _p(ic), _p(trace), C.byref(rows),
                                _p(final_raw), C.byref(aborted)))
    t = trace[: rows.value]
    return {"constrained": t[:, :P], "gradient": t[:, P:2 * P], "mean_residual_norm": t[:, 2 * P],
            "probe_residual_norm": t[:, 2 * P + 1], "epochs": t[:, 2 * P + 2], "grad_inf_norm": t[:, 2 * P + 3],
            "iterations": t[:, 2 * P + 4].astype(int), "solver_diverged": t[:, 2 * P + 5].astype(bool),
            "step_seconds": t[:, 2 * P + 6], "solver_seconds": t[:, 2 * P + 7], "final_raw": final_raw,
            "aborted": bool(aborted.value)}


def _trace_dict(t, P):
    return {"constrained": t[:, :P], "gradient": t[:, P:2 * P], "mean_residual_norm": t[:, 2 * P],
            "probe_residual_norm": t[:, 2 * P + 1], "epochs": t[:, 2 * P + 2], "grad_inf_norm": t[:, 2 * P + 3],
            "iterations": t[:, 2 * P + 4].astype(int), "solver_diverged": t[:, 2 * P + 5].astype(bool),
            "step_seconds": t[:, 2 * P + 6], "solver_seconds": t[:, 2 * P + 7]}


class Optimiser:
    """Resumable optimise(): dataset uploaded once, steps run on device-resident state."""

    def __init__(self, ctx: Context, inputs, targets, config: OuterConfig, init_constrained=None):
        self.ctx = ctx
        self._lib = ctx._lib
        X = _f64(inputs)
        y = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1)
        self.n, self.d = X.shape
        self.P = self.d + 2
        ic = np.ascontiguousarray(init_constrained, dtype=np.float64) if init_constrained is not None else None
        cfg = config.c()
        h = C.c_void_p()
        check(self._lib.gpk_optimiser_create(ctx.handle, _p(X), _p(y), self.n, self.d, C.byref(cfg), _p(ic),
                                             C.byref(h)))
        self.handle = h

    def step(self, steps=1):
        trace = np.zeros((max(steps, 1), 2 * self.P + 8))
        rows = C.c_int()
        check(self._lib.gpk_optimiser_step(self.handle, steps, _p(trace), C.byref(rows)))
        return _trace_dict(trace[: rows.value], self.P)

    def state(self):
        raw = np.empty(self.P)
        step, ab = C.c_int(), C.c_int()
        check(self._lib.gpk_optimiser_state(self.handle, _p(raw), C.byref(step), C.byref(ab)))
        return {"raw": raw, "step": step.value, "aborted": bool(ab.value)}

    def close(self):
        if getattr(self, "handle", None):
            self._lib.gpk_optimiser_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sinsum_dataset(n, d, uniform=False, noise=0.1, seed=0):
    """BASELINE.json synthetic data (X float32 n x d row-major, y float32 n)."""
    lib = _lib.load()
    x = np.empty((n, d), dtype=np.float32)
    y = np.empty(n, dtype=np.float32)
    check(lib.gpk_sinsum_dataset(n, d, int(uniform), noise, seed, x.ctypes.data_as(C.POINTER(C.c_float)),
                                 y.ctypes.data_as(C.POINTER(C.c_float))))
    return x, y


# ---- posterior predictions (posterior.hpp:14-51) ----------------------------
def cross_kernel_apply(op: KernelOperator, points, v):
    """k(P, X) V without the noise term (kernel.cpp:72-81)."""
    P, V = _f64(points), _f64(v)
    out = np.empty((P.shape[0], V.shape[1]), order="F")
    check(op._lib.gpk_cross_apply(op.handle, _p(P), P.shape[0], _p(V), V.shape[1], _p(out)))
    return out


def predict_mean(op: KernelOperator, points, v_y):
    P = _f64(points)
    vy = np.ascontiguousarray(v_y, dtype=np.float64).reshape(-1)
    out = np.empty(P.shape[0])
    check(op._lib.gpk_predict_mean(op.handle, _p(P), P.shape[0], _p(vy), _p(out)))
    return out


def sample_posterior(op: KernelOperator, basis, points, v_y, zhat):
    """All pathwise posterior samples f_j(P) + k(P,X)(v_y - zhat_j) (posterior.cpp:19-27); basis None = zero prior."""
    P, Z = _f64(points), _f64(zhat)
    vy = np.ascontiguousarray(v_y, dtype=np.float64).reshape(-1)
    out = np.empty((P.shape[0], Z.shape[1]), order="F")
    check(op._lib.gpk_sample_posterior(op.handle, basis.handle if basis is not None else None, _p(P), P.shape[0],
                                       _p(vy), _p(Z), Z.shape[1], _p(out)))
    return out


def test_metrics(op: KernelOperator, basis, points, targets, v_y, zhat, target_scale=1.0):
    """posterior.cpp:29-59 -> dict(rmse, llh, rmse_raw, llh_raw); llh None without >= 2 samples and a basis."""
    P, Z = _f64(points), _f64(zhat)
    t = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1)
    vy = np.ascontiguousarray(v_y, dtype=np.float64).reshape(-1)
    out = np.empty(4)
    check(op._lib.gpk_test_metrics(op.handle, basis.handle if basis is not None else None, _p(P), P.shape[0], _p(t),
                                   _p(vy), _p(Z), Z.shape[1], target_scale, _p(out)))
    llh = None if np.isnan(out[1]) else out[1]
    return {"rmse": out[0], "llh": llh, "rmse_raw": out[2], "llh_raw": None if llh is None else out[3]}


def write_trace_csv(path, trace: dict, input_dim: int):
    """write_trace_csv (trace.cpp:20-44) for a trace dict returned by optimise()/Optimiser.step()."""
    P = input_dim + 2
    rows = len(trace["iterations"])
    t = np.zeros((max(rows, 1), 2 * P + 8))
    t[:rows, :P] = trace["constrained"]
    t[:rows, P:2 * P] = trace["gradient"]
    t[:rows, 2 * P + 0] = trace["mean_residual_norm"]
    t[:rows, 2 * P + 1] = trace["probe_residual_norm"]
    t[:rows, 2 * P + 2] = trace["epochs"]
    t[:rows, 2 * P + 3] = trace["grad_inf_norm"]
    t[:rows, 2 * P + 4] = trace["iterations"]
    t[:rows, 2 * P + 5] = trace["solver_diverged"]
    t[:rows, 2 * P + 6] = trace.get("step_seconds", np.zeros(rows))
    t[:rows, 2 * P + 7] = trace.get("solver_seconds", np.zeros(rows))
    check(_lib.load().gpk_write_trace_csv(str(path).encode(), _p(np.ascontiguousarray(t)), rows, input_dim))


def spd_inverse(ctx: Context, mats, mode: int = 1):
    """Batched SPD inverse of the AP diagonal-block solver (mats: batch x dim x dim).
    mode 1: recursive Schur complement on strided-batched DGEMMs (default in the
    solver); mode 0: cuSOLVER potrfBatched + batched triangular solves."""
    mats = np.asarray(mats, dtype=np.float64)
    if mats.ndim == 2:
        mats = mats[None]
    batch, dim, _ = mats.shape
    src = np.ascontiguousarray(np.transpose(mats, (0, 2, 1)))  # column-major per matrix
    out = np.empty_like(src)
    check(ctx._lib.gpk_spd_inverse(ctx.handle, _p(src), dim, batch, int(mode), _p(out)))
    return np.transpose(out, (0, 2, 1)).copy()


def optimise_exact(ctx: Context, inputs, targets, steps: int, learning_rate: float = 0.1, init_constrained=None):
    """optimise_exact (outer_loop.cpp:248-262) on the device: Adam on the exact
    marginal likelihood. Returns (trajectory steps x (d+2) constrained, final raw)."""
    X = _f64(inputs)
    y = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1)
    n, d = X.shape
    traj = np.empty((steps, d + 2))
    raw = np.empty(d + 2)
    init = np.ascontiguousarray(init_constrained, dtype=np.float64) if init_constrained is not None else None
    check(ctx._lib.gpk_optimise_exact(ctx.handle, _p(X), _p(y), n, d, _p(init), steps, learning_rate, _p(traj),
                                      _p(raw)))
    return traj, raw


def init_heuristic(ctx: Context, inputs, targets, n_centroids: int, subset: int, seed: int, adam_steps: int,
                   learning_rate: float = 0.1):
    """init_heuristic (outer_loop.cpp:264-296) on the device: constrained d+2."""
    X = _f64(inputs)
    y = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1)
    n, d = X.shape
    out = np.empty(d + 2)
    check(ctx._lib.gpk_init_heuristic(ctx.handle, _p(X), _p(y), n, d, n_centroids, subset, seed, adam_steps,
                                      learning_rate, _p(out)))
    return out

