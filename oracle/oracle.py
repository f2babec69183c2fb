"""TEST INFRASTRUCTURE — NOT PRODUCT CODE.

ctypes binding of the FP64 C++ oracle (oracle/gpiter_oracle.cpp), a restatement
of /root/reference/proj/core/src/*.cpp without Eigen. Only tests/,
__graft_entry__.smoke() and bench.py's CPU arms import this module; the product
package (paper_2405_18457_b200) never does.

Matrices cross the boundary column-major FP64 (the reference's Eigen layout);
numpy arrays are converted with ``np.asfortranarray``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
u64p = C.POINTER(C.c_ulonglong)


class SolverConfigC(C.Structure):
    _fields_ = [("kind", C.c_int), ("tolerance", C.c_double), ("max_epochs", C.c_int),
                ("block_size", C.c_int), ("batch_size", C.c_int), ("learning_rate", C.c_double),
                ("momentum", C.c_double), ("preconditioner_rank", C.c_int), ("warm_start", C.c_int),
                ("seed", C.c_ulonglong), ("substream", C.c_ulonglong)]


class ReportC(C.Structure):
    _fields_ = [("iterations", C.c_int), ("epochs_consumed", C.c_double),
                ("mean_residual_norm", C.c_double), ("probe_residual_norm", C.c_double),
                ("reached_tolerance", C.c_int), ("residuals_estimated", C.c_int),
                ("aborted", C.c_int), ("abort_reason", C.c_char * 128), ("wall_seconds", C.c_double)]


class OuterConfigC(C.Structure):
    _fields_ = [("estimator", C.c_int), ("solver", SolverConfigC), ("warm_start", C.c_int),
                ("steps", C.c_int), ("learning_rate", C.c_double), ("probe_count", C.c_int),
                ("rff_pairs", C.c_int), ("probe_distribution", C.c_int),
                ("probe_seed", C.c_ulonglong), ("feature_seed", C.c_ulonglong),
                ("solver_seed", C.c_ulonglong), ("init_value", C.c_double),
                ("divergence_policy", C.c_int), ("prior_mode", C.c_int)]


def build():
    """Compile the oracle (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def use_timing_build():
    """Switch this process to the -march=native -ffast-math timing build (bench.py's
    CPU arms only; parity checks always use the strict build). Compiled on the
    host that runs it, into a directory keyed on its CPU model and flags."""
    global _LIB_PATH
    if _lib is not None:
        raise RuntimeError("oracle: choose the build before the first call")
    import hashlib
    import platform
    try:
        info = open("/proc/cpuinfo").read()
        key = [ln for ln in info.splitlines() if ln.startswith(("model name", "flags"))][:2]
    except OSError:
        key = [platform.processor()]
    tag = hashlib.sha1("\n".join(key).encode()).hexdigest()[:12]
    out = os.path.join(_HERE, "build", "native-" + tag)
    subprocess.run(["make", "-s", "-C", _HERE, "native", f"NATIVE_OUT={out}"], check=True)
    _LIB_PATH = os.path.join(out, "liboracle.so")
    return _LIB_PATH


_gpu_lib = None


class gpu_backend:
    """Context manager: oracle calls inside run through oracle/build/liboracle_gpu.so,
    the same restatement with its O(n^2) passes (apply, apply_rows, quadratic forms,
    RFF prior, solve_sgd) as naive FP64 CUDA kernels (oracle/gpu/oracle_gpu.cu) --
    the oracle-at-scale for C4/C5. Needs a GPU; test infrastructure only."""

    def __init__(self, device=0):
        self.device = device

    def __enter__(self):
        global _lib, _gpu_lib
        if _gpu_lib is None:
            path = os.path.join(_HERE, "build", "liboracle_gpu.so")
            if not os.path.exists(path):
                subprocess.run(["make", "-s", "-C", _HERE, "gpu"], check=True)
            _gpu_lib = C.CDLL(path)
            _gpu_lib.oracle_last_error.restype = C.c_char_p
            _gpu_lib.oracle_softplus.restype = C.c_double
            _gpu_lib.oracle_softplus.argtypes = [C.c_double]
            _gpu_lib.oracle_sigmoid.restype = C.c_double
            _gpu_lib.oracle_sigmoid.argtypes = [C.c_double]
        if _gpu_lib.oracle_gpu_enable(self.device, 1) != 0:
            raise RuntimeError("oracle_gpu_enable failed (no GPU?)")
        self._saved = lib()
        _lib = _gpu_lib
        return self

    def __exit__(self, *exc):
        global _lib
        _lib = self._saved
        return False


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.oracle_last_error.restype = C.c_char_p
        _lib.oracle_softplus.restype = C.c_double
        _lib.oracle_softplus.argtypes = [C.c_double]
        _lib.oracle_sigmoid.restype = C.c_double
        _lib.oracle_sigmoid.argtypes = [C.c_double]
    return _lib


class OracleError(Exception):
    pass


def _check(rc):
    if rc != 0:
        msg = lib().oracle_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        if rc == 2:
            raise IndexError(msg)
        raise OracleError(msg)


def _f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return a.ctypes.data_as(dp) if a is not None else None


def solver_config(kind=0, tolerance=0.01, max_epochs=50, block_size=1000, batch_size=500,
                  learning_rate=30.0, momentum=0.9, preconditioner_rank=100, warm_start=False,
                  seed=0, substream=0):
    return SolverConfigC(kind, tolerance, max_epochs, block_size, batch_size, learning_rate,
                         momentum, preconditioner_rank, int(warm_start), seed, substream)


# ---- rng ----------------------------------------------------------------
def philox(counter, key):
    c = (C.c_ulonglong * 4)(*counter)
    k = (C.c_ulonglong * 2)(*key)
    out = (C.c_ulonglong * 4)()
    lib().oracle_philox(c, k, out)
    return [int(x) for x in out]


def stream_draw(seed, stream, substream, kind, count, bound=1):
    """kind: 'u64' | 'double' | 'gaussian' | 'below' | 'rademacher'."""
    code = {"u64": 0, "double": 1, "gaussian": 2, "below": 3, "rademacher": 4}[kind]
    out = np.empty(count, dtype=np.uint64 if code in (0, 3) else np.float64)
    lib().oracle_stream_draw(C.c_ulonglong(seed), C.c_ulonglong(stream), C.c_ulonglong(substream),
                             code, C.c_ulonglong(bound), C.c_longlong(count), out.ctypes.data_as(C.c_void_p))
    return out


def sample_without_replacement(seed, stream, substream, n, k, rounds=1):
    out = np.empty((rounds, k), dtype=np.int32)
    _check(lib().oracle_sample_without_replacement(C.c_ulonglong(seed), C.c_ulonglong(stream),
                                                   C.c_ulonglong(substream), n, k, rounds,
                                                   out.ctypes.data_as(ip)))
    return out


def permutation(seed, stream, n):
    out = np.empty(n, dtype=np.int32)
    _check(lib().oracle_permutation(C.c_ulonglong(seed), C.c_ulonglong(stream), n, out.ctypes.data_as(ip)))
    return out


def softplus(x):
    return lib().oracle_softplus(x)


def softplus_inverse(y):
    out = C.c_double()
    _check(lib().oracle_softplus_inverse(C.c_double(y), C.byref(out)))
    return out.value


def sigmoid(x):
    return lib().oracle_sigmoid(x)


def raw_from_constrained(c):
    return np.array([softplus_inverse(float(v)) for v in c])


# ---- kernel operator ------------------------------------------------------
def matern32(x, x2, raw):
    x, x2, raw = _f(x), _f(x2), _f(raw)
    out = C.c_double()
    _check(lib().oracle_matern32(_p(x), _p(x2), x.size, _p(raw), C.byref(out)))
    return out.value


def apply(X, raw, V, block_rows=1024, threads=1):
    X, raw, V = _f(X), _f(raw), _f(V)
    if V.ndim == 1:
        V = V[:, None]
    n, d = X.shape
    out = np.empty((n, V.shape[1]), order="F")
    _check(lib().oracle_apply(_p(X), n, d, _p(raw), _p(V), V.shape[1], _p(out), block_rows, threads))
    return out


def apply_rows(X, raw, rows, V, threads=1):
    X, raw, V = _f(X), _f(raw), _f(V)
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    n, d = X.shape
    out = np.empty((rows.size, V.shape[1]), order="F")
    _check(lib().oracle_apply_rows(_p(X), n, d, _p(raw), rows.ctypes.data_as(ip), rows.size, _p(V),
                                   V.shape[1], _p(out), threads))
    return out


def apply_columns(X, raw, c0, length, U, threads=1):
    X, raw, U = _f(X), _f(raw), _f(U)
    n, d = X.shape
    out = np.empty((n, U.shape[1]), order="F")
    _check(lib().oracle_apply_columns(_p(X), n, d, _p(raw), c0, length, _p(U), U.shape[1], _p(out), threads))
    return out


def dense_block(X, raw, r0, rows, c0, cols):
    X, raw = _f(X), _f(raw)
    n, d = X.shape
    out = np.empty((rows, cols), order="F")
    _check(lib().oracle_dense_block(_p(X), n, d, _p(raw), r0, rows, c0, cols, _p(out)))
    return out


def dense(X, raw):
    n = X.shape[0]
    return dense_block(X, raw, 0, n, 0, n)


def kernel_column(X, raw, i):
    X, raw = _f(X), _f(raw)
    n, d = X.shape
    out = np.empty(n)
    _check(lib().oracle_kernel_column(_p(X), n, d, _p(raw), i, _p(out)))
    return out


def derivative_apply(X, raw, k, V):
    X, raw, V = _f(X), _f(raw), _f(V)
    n, d = X.shape
    out = np.empty((n, V.shape[1]), order="F")
    _check(lib().oracle_derivative_apply(_p(X), n, d, _p(raw), k, _p(V), V.shape[1], _p(out)))
    return out


def quad_forms(X, raw, U1, W1, U2, W2, threads=1):
    X, raw = _f(X), _f(raw)
    U1, W1, U2, W2 = (_f(a) if a.ndim == 2 else _f(a[:, None]) for a in (U1, W1, U2, W2))
    n, d = X.shape
    out = np.empty(2 * (d + 2))
    _check(lib().oracle_quad_forms(_p(X), n, d, _p(raw), _p(U1), _p(W1), U1.shape[1], _p(U2), _p(W2),
                                   U2.shape[1], _p(out), threads))
    return out[: d + 2], out[d + 2:]


def precond(X, raw, rank, V=None):
    X, raw = _f(X), _f(raw)
    n, d = X.shape
    factor = np.empty((n, max(rank, 1)), order="F")
    piv = np.empty(max(rank, 1), dtype=np.int32)
    ach = C.c_int()
    pv = None
    m = 0
    if V is not None:
        V = _f(V if V.ndim == 2 else V[:, None])
        m = V.shape[1]
        pv = np.empty((n, m), order="F")
    _check(lib().oracle_precond(_p(X), n, d, _p(raw), rank, _p(V), m, _p(pv), _p(factor),
                                piv.ctypes.data_as(ip), C.byref(ach)))
    r = ach.value
    fac = np.asfortranarray(factor.reshape(-1, order="F")[: n * r].reshape((n, r), order="F"))
    return {"factor": fac, "pivots": piv[:r].copy(), "achieved_rank": r, "apply": pv}


def solve(X, raw, targets, config, warm=None, explicit_rank=-1, threads=1, record_batches=0):
    X, raw, T = _f(X), _f(raw), _f(targets)
    n, d = X.shape
    m = T.shape[1]
    sol = np.empty((n, m), order="F")
    res = np.empty((n, m), order="F")
    rep = ReportC()
    W = _f(warm) if warm is not None else None
    batches = None
    if record_batches:
        b = min(config.batch_size, n)
        batches = np.zeros((record_batches, b), dtype=np.int32)
    _check(lib().oracle_solve(_p(X), n, d, _p(raw), _p(T), m, _p(W), C.byref(config), explicit_rank,
                              _p(sol), _p(res), C.byref(rep), threads,
                              batches.ctypes.data_as(ip) if batches is not None else None,
                              record_batches))
    out = {"solutions": sol, "residuals": res, "iterations": rep.iterations,
           "epochs_consumed": rep.epochs_consumed, "mean_residual_norm": rep.mean_residual_norm,
           "probe_residual_norm": rep.probe_residual_norm,
           "reached_tolerance": bool(rep.reached_tolerance),
           "residuals_estimated": bool(rep.residuals_estimated), "aborted": bool(rep.aborted),
           "abort_reason": rep.abort_reason.decode(), "wall_seconds": rep.wall_seconds}
    if batches is not None:
        out["batches"] = batches
    return out


def set_sgd_iteration_cap(cap):
    """Test knob: solve_sgd stops after `cap` iterations (-1: epoch budget only)."""
    lib().oracle_set_sgd_iteration_cap(int(cap))


def set_apply_sensitivity(order=0, noise=0.0):
    """Test knobs of KernelOperator::apply: order 1 sums in descending column
    order, noise eps perturbs every output entry by a factor 1 + eps u, u ~ U[-1, 1)."""
    lib().oracle_set_apply_sensitivity(int(order), C.c_double(noise))


def termination_check(targets, residuals, tol):
    T, R = _f(targets), _f(residuals)
    mean, probe, done = C.c_double(), C.c_double(), C.c_int()
    _check(lib().oracle_termination_check(_p(T), _p(R), T.shape[0], T.shape[1], C.c_double(tol),
                                          C.byref(mean), C.byref(probe), C.byref(done)))
    return mean.value, probe.value, bool(done.value)


def gradient(X, raw, v_y, zhat, probes=None, threads=1):
    X, raw, vy, Z = _f(X), _f(raw), _f(v_y), _f(zhat)
    P = _f(probes) if probes is not None else None
    n, d = X.shape
    out = np.empty(3 * (d + 2))
    _check(lib().oracle_gradient(_p(X), n, d, _p(raw), _p(vy), _p(Z), Z.shape[1], _p(P), _p(out), threads))
    k = d + 2
    return {"values": out[:k], "quadratic_term": out[k:2 * k], "trace_term": out[2 * k:]}


def standard_probes(n, s, seed, distribution=0, substream=0):
    out = np.empty((n, s), order="F")
    _check(lib().oracle_standard_probes(n, s, C.c_ulonglong(seed), distribution, C.c_ulonglong(substream), _p(out)))
    return out


def rff_basis(d, pairs, samples, seed, substream=0):
    freq = np.empty((pairs, d), order="F")
    w = np.empty((2 * pairs, samples), order="F")
    _check(lib().oracle_rff_basis(d, pairs, samples, C.c_ulonglong(seed), C.c_ulonglong(substream), _p(freq), _p(w)))
    return freq, w


def rff_features(d, pairs, samples, seed, raw, points):
    raw, P = _f(raw), _f(points)
    out = np.empty((P.shape[0], 2 * pairs), order="F")
    _check(lib().oracle_rff_features(d, pairs, samples, C.c_ulonglong(seed), _p(raw), _p(P), P.shape[0], _p(out)))
    return out


def pathwise_targets(X, raw, pairs, samples, s, seed, substream=0):
    X, raw = _f(X), _f(raw)
    n, d = X.shape
    prior, noise, xi = (np.empty((n, s), order="F") for _ in range(3))
    _check(lib().oracle_pathwise_targets(_p(X), n, d, _p(raw), pairs, samples, s, C.c_ulonglong(seed),
                                         C.c_ulonglong(substream), _p(prior), _p(noise), _p(xi)))
    return {"prior_values": prior, "noise": noise, "xi": xi}


def optimise(X, y, config: OuterConfigC, init_constrained=None, threads=1):
    X, y = _f(X), _f(y)
    n, d = X.shape
    P = d + 2
    stride = 2 * P + 8
    trace = np.zeros((max(config.steps, 1), stride))
    rows, aborted = C.c_int(), C.c_int()
    final_raw = np.empty(P)
    ic = _f(init_constrained) if init_constrained is not None else None
    _check(lib().oracle_optimise(_p(X), _p(y), n, d, C.byref(config), _p(ic), _p(trace), C.byref(rows),
                                 _p(final_raw), C.byref(aborted), threads))
    t = trace[: rows.value]
    return {"constrained": t[:, :P], "gradient": t[:, P:2 * P], "mean_residual_norm": t[:, 2 * P],
            "probe_residual_norm": t[:, 2 * P + 1], "epochs": t[:, 2 * P + 2],
            "grad_inf_norm": t[:, 2 * P + 3], "iterations": t[:, 2 * P + 4].astype(int),
            "solver_diverged": t[:, 2 * P + 5].astype(bool), "final_raw": final_raw,
            "aborted": bool(aborted.value)}


def outer_config(estimator=1, solver=None, warm_start=False, steps=100, learning_rate=0.1,
                 probe_count=64, rff_pairs=1000, probe_distribution=0, probe_seed=0, feature_seed=0,
                 solver_seed=0, init_value=1.0, divergence_policy=0, prior_mode=0):
    return OuterConfigC(estimator, solver if solver is not None else solver_config(), int(warm_start),
                        steps, learning_rate, probe_count, rff_pairs, probe_distribution, probe_seed,
                        feature_seed, solver_seed, init_value, divergence_policy, prior_mode)


def exact(X, y, raw):
    X, y, raw = _f(X), _f(y), _f(raw)
    n, d = X.shape
    mll = C.c_double()
    grad = np.empty(d + 2)
    _check(lib().oracle_exact(_p(X), _p(y), n, d, _p(raw), C.byref(mll), _p(grad)))
    return mll.value, grad


def sinsum_dataset(n, d, uniform=False, noise=0.1, seed=0):
    """BASELINE.json generator; returns (X float32 n x d row-major, y float32 n)."""
    x = np.empty((n, d), dtype=np.float32)
    y = np.empty(n, dtype=np.float32)
    lib().oracle_sinsum_dataset(n, d, int(uniform), C.c_double(noise), C.c_ulonglong(seed),
                                x.ctypes.data_as(C.POINTER(C.c_float)), y.ctypes.data_as(C.POINTER(C.c_float)))
    return x, y


# ---- posterior (posterior.cpp) ---------------------------------------------
def cross_apply(points, X, raw, V, threads=1):
    P, X, raw, V = _f(points), _f(X), _f(raw), _f(V)
    if V.ndim == 1:
        V = V[:, None]
    out = np.empty((P.shape[0], V.shape[1]), order="F")
    _check(lib().oracle_cross_apply(_p(P), P.shape[0], _p(X), X.shape[0], X.shape[1], _p(raw), _p(V), V.shape[1],
                                    _p(out), threads))
    return out


def optimise_exact(X, y, steps, learning_rate=0.1, init_constrained=None):
    """outer_loop.cpp:248-262: returns (trajectory steps x (d+2) constrained, final raw)."""
    X, y = _f(X), _f(y)
    n, d = X.shape
    traj = np.empty((steps, d + 2))
    raw = np.empty(d + 2)
    init = _f(init_constrained) if init_constrained is not None else None
    _check(lib().oracle_optimise_exact(_p(X), _p(y), n, d, _p(init), steps, C.c_double(learning_rate), _p(traj),
                                       _p(raw)))
    return traj, raw


def init_heuristic(X, y, n_centroids, subset, seed, adam_steps, learning_rate=0.1):
    """outer_loop.cpp:264-296: constrained hyperparameters (d+2)."""
    X, y = _f(X), _f(y)
    n, d = X.shape
    out = np.empty(d + 2)
    _check(lib().oracle_init_heuristic(_p(X), _p(y), n, d, n_centroids, subset, C.c_ulonglong(seed), adam_steps,
                                       C.c_double(learning_rate), _p(out)))
    return out


def exact_prior(X, raw, s, seed, substream=0):
    """ExactDense prior values L W (outer_loop.cpp:140-153), W from (seed, 8, substream)."""
    X, raw = _f(X), _f(raw)
    n, d = X.shape
    out = np.empty((n, s), order="F")
    _check(lib().oracle_exact_prior(_p(X), n, d, _p(raw), s, C.c_ulonglong(seed), C.c_ulonglong(substream), _p(out)))
    return out


def prior_at(d, pairs, samples, seed, raw, points, s, substream=0):
    raw, P = _f(raw), _f(points)
    out = np.empty((P.shape[0], s), order="F")
    _check(lib().oracle_prior_at(d, pairs, samples, C.c_ulonglong(seed), C.c_ulonglong(substream), _p(raw), _p(P),
                                 P.shape[0], s, _p(out)))
    return out


def posterior(points, X, raw, v_y, zhat, prior=None, test_targets=None, target_scale=1.0, threads=1):
    P, X, raw, vy, Z = _f(points), _f(X), _f(raw), _f(v_y), _f(zhat)
    pr = _f(prior) if prior is not None else None
    tt = _f(test_targets) if test_targets is not None else None
    p, s = P.shape[0], Z.shape[1]
    samples = np.empty((p, s), order="F")
    metrics = np.zeros(5)
    _check(lib().oracle_posterior(_p(P), p, _p(X), X.shape[0], X.shape[1], _p(raw), _p(vy), _p(Z), s, _p(pr), _p(tt),
                                  C.c_double(target_scale), _p(samples), _p(metrics), threads))
    return {"samples": samples, "rmse": metrics[0], "llh": metrics[1] if metrics[4] else None,
            "rmse_raw": metrics[2], "llh_raw": metrics[3] if metrics[4] else None}
