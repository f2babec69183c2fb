"""GPU parity: the CUDA path (through the C-ABI, via the Python mirror of the
reference API) against the FP64 oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): FP32 operator products and gradients
within 1e-4 relative (we test tighter where the kernel allows: operator
products 2e-5 of the column max); FP64 paths (dense blocks, kernel columns,
preconditioner, RFF prior) to ~1e-10; integer work (SGD minibatches,
preconditioner pivots) bit-exact; solver residual norms within 1e-4
relative; iteration counts within +-1.
"""
import numpy as np
import pytest

from _problems import default_test_raw, gp_problem

pytestmark = pytest.mark.gpu

OP_TOL = 2e-5


@pytest.fixture(scope="module")
def G():
    import paper_2405_18457_b200 as G
    return G


KERNELS = [0, 1]  # 0: FP32 SIMT operator kernel, 1: tcgen05 3xTF32 operator kernel


@pytest.fixture(params=KERNELS, ids=["simt", "tcgen05"])
def kctx(request, gpk_ctx):
    gpk_ctx.set_operator_kernel(request.param)
    yield gpk_ctx
    gpk_ctx.set_operator_kernel(1)


def colrel(a, b):
    """max over columns of max|a-b| / max|b|."""
    a, b = np.atleast_2d(a.T).T, np.atleast_2d(b.T).T
    return max(np.max(np.abs(a[:, j] - b[:, j])) / max(np.max(np.abs(b[:, j])), 1e-300) for j in range(b.shape[1]))


def make_op(G, ctx, X, raw):
    return G.KernelOperator(X, G.Hyperparameters.from_raw(raw), ctx)


@pytest.mark.parametrize("n,d,m", [(300, 3, 1), (1000, 8, 17), (2048, 26, 65), (777, 20, 65), (513, 1, 9),
                                   (1500, 11, 33), (4096, 3, 65),
                                   # Gram-form distance tiles (d >= 21), incl. d = 32 (image width 36)
                                   (900, 21, 17), (1100, 24, 65), (640, 32, 33), (1000, 31, 80)])
def test_apply_matches_oracle(G, kctx, oracle, n, d, m):
    X, _ = gp_problem(n, d, 1000 + n)
    raw = default_test_raw(d, oracle)
    V = np.asfortranarray(np.random.default_rng(n).standard_normal((n, m)))
    op = make_op(G, kctx, X, raw)
    got = op.apply(V)
    ref = oracle.apply(X, raw, V, threads=8)
    assert colrel(got, ref) <= OP_TOL


@pytest.mark.parametrize("n,d,m", [(4096, 8, 17), (1000, 3, 5), (777, 13, 33), (600, 20, 65), (300, 16, 9),
                                   (129, 1, 1)])
def test_apply_dense_cache_fp64_matches_oracle(G, gpk_ctx, oracle, n, d, m):
    """KernelOperatorOptions::dense_cache (kernel.hpp:27-30): full products in
    FP64 with entries evaluated on the fly (kv64 kernels; H never held), to
    FP64 rounding of the oracle's ascending-column sums; the C1 optimiser
    (n <= dense_cache_cap) runs this operator."""
    X, _ = gp_problem(n, d, 2000 + n)
    raw = default_test_raw(d, oracle)
    V = np.asfortranarray(np.random.default_rng(n + 1).standard_normal((n, m)))
    op = G.KernelOperator(X, G.Hyperparameters.from_raw(raw), gpk_ctx, dense_cache=True)
    got = op.apply(V)
    ref = oracle.apply(X, raw, V, threads=8)
    assert colrel(got, ref) <= 1e-12
    assert np.array_equal(op.apply(V), got)  # deterministic


def test_apply_identity_is_dense(G, kctx, oracle):
    n, d = 64, 3
    X, _ = gp_problem(n, d, 101)
    raw = default_test_raw(d, oracle)
    op = make_op(G, kctx, X, raw)
    H = oracle.dense(X, raw)
    assert np.max(np.abs(op.apply(np.eye(n)) - H)) <= 1e-6
    assert np.max(np.abs(op.dense() - H)) <= 1e-12
    assert np.max(np.abs(op.apply(np.zeros((n, 5))))) == 0.0


def test_apply_rejects_bad_input(G, gpk_ctx, oracle):
    X, _ = gp_problem(50, 2, 3)
    op = make_op(G, gpk_ctx, X, default_test_raw(2, oracle))
    with pytest.raises(ValueError):
        op.apply(np.full((50, 2), np.nan))
    with pytest.raises(ValueError):
        op.apply(np.ones((49, 2)))
    with pytest.raises(ValueError):
        G.KernelOperator(X, G.Hyperparameters.from_constrained([1.0, 1.0, -1.0, 1.0]), gpk_ctx)


def test_apply_is_deterministic(G, kctx, oracle):
    X, _ = gp_problem(3000, 5, 7)
    op = make_op(G, kctx, X, default_test_raw(5, oracle))
    V = np.random.default_rng(0).standard_normal((3000, 65))
    assert np.array_equal(op.apply(V), op.apply(V))


@pytest.mark.parametrize("n,d,m,b", [(2000, 3, 65, 512), (600, 8, 17, 37), (50, 2, 3, 5), (700, 24, 17, 61)])
def test_apply_rows_matches_oracle(G, kctx, oracle, n, d, m, b):
    X, _ = gp_problem(n, d, 2 * n)
    raw = default_test_raw(d, oracle)
    V = np.asfortranarray(np.random.default_rng(1).standard_normal((n, m)))
    rows = np.sort(np.random.default_rng(2).choice(n, b, replace=False)).astype(np.int32)
    op = make_op(G, kctx, X, raw)
    assert colrel(op.apply_rows(rows, V), oracle.apply_rows(X, raw, rows, V, threads=8)) <= OP_TOL
    with pytest.raises(IndexError):
        op.apply_rows([n], V)


@pytest.mark.parametrize("n,d,m,c0,ln", [(2048, 26, 65, 512, 512), (1000, 4, 17, 990, 10), (300, 2, 5, 0, 300)])
def test_apply_columns_matches_oracle(G, kctx, oracle, n, d, m, c0, ln):
    X, _ = gp_problem(n, d, 3 * n)
    raw = default_test_raw(d, oracle)
    U = np.asfortranarray(np.random.default_rng(1).standard_normal((ln, m)))
    op = make_op(G, kctx, X, raw)
    assert colrel(op.apply_columns(c0, ln, U), oracle.apply_columns(X, raw, c0, ln, U, threads=8)) <= OP_TOL


def test_dense_block_and_kernel_column_fp64(G, gpk_ctx, oracle):
    n, d = 300, 4
    X, _ = gp_problem(n, d, 5)
    raw = default_test_raw(d, oracle)
    op = make_op(G, gpk_ctx, X, raw)
    assert np.max(np.abs(op.dense_block(5, 12, 7, 20) - oracle.dense_block(X, raw, 5, 12, 7, 20))) <= 1e-13
    assert np.max(np.abs(op.kernel_column(17) - oracle.kernel_column(X, raw, 17))) <= 1e-13
    s2 = G.gpiter.softplus(raw[-2]) ** 2
    assert np.all(op.kernel_diagonal() == s2)


@pytest.mark.parametrize("n,d,m", [(300, 4, 3), (700, 11, 17), (257, 2, 65)])
def test_derivative_apply_matches_oracle(G, gpk_ctx, oracle, n, d, m):
    """derivative_apply(k, V) (kernel.hpp:71, kernel.cpp:200-236) for every
    parameter, FP64 on the device, against the oracle's restatement."""
    X, _ = gp_problem(n, d, 3 * n)
    raw = default_test_raw(d, oracle)
    V = np.asfortranarray(np.random.default_rng(m).standard_normal((n, m)))
    op = make_op(G, gpk_ctx, X, raw)
    for k in range(d + 2):
        got, ref = op.derivative_apply(k, V), oracle.derivative_apply(X, raw, k, V)
        assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref)), k
    with pytest.raises(IndexError):
        op.derivative_apply(d + 2, V)


@pytest.mark.parametrize("n,d,s", [(500, 2, 8), (1200, 20, 64), (2048, 26, 64), (700, 3, 16), (300, 3, 80),
                                   (129, 5, 2)])
def test_quadratic_forms_match_oracle(G, kctx, oracle, n, d, s):
    """tcgen05 context: G = Z Z^T on the tensor cores (grad_tc_kernel, s <= 64;
    s = 80 takes the SIMT pass); simt context: grad_kernel throughout."""
    X, _ = gp_problem(n, d, 4 * n)
    raw = default_test_raw(d, oracle)
    rng = np.random.default_rng(n)
    vy = rng.standard_normal(n)
    Z = rng.standard_normal((n, s))
    op = make_op(G, kctx, X, raw)
    g = G.estimate_gradient_pathwise(op, vy, Z)
    r = oracle.gradient(X, raw, vy, Z, threads=8)
    for key in ("quadratic_term", "trace_term"):
        a, b = getattr(g, key), r[key]
        assert np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-3 * np.max(np.abs(b)))) <= 1e-4, key
    # standard estimator (U != W, non-symmetric pass)
    P = rng.standard_normal((n, s))
    gs = G.estimate_gradient_standard(op, vy, Z, P)
    rs = oracle.gradient(X, raw, vy, Z, probes=P, threads=8)
    b = rs["trace_term"]
    assert np.max(np.abs(gs.trace_term - b) / np.maximum(np.abs(b), 1e-3 * np.max(np.abs(b)))) <= 1e-4


def test_gradient_zero_inputs(G, gpk_ctx, oracle):
    X, _ = gp_problem(20, 1, 85)
    op = make_op(G, gpk_ctx, X, default_test_raw(1, oracle))
    g = G.estimate_gradient_pathwise(op, np.zeros(20), np.zeros((20, 4)))
    assert np.max(np.abs(g.values)) == 0.0 and np.max(np.abs(g.trace_term)) == 0.0


@pytest.mark.parametrize("n,d,rank", [(400, 3, 100), (1000, 8, 50), (40, 1, 40), (300, 2, 0)])
def test_preconditioner_matches_oracle(G, gpk_ctx, oracle, n, d, rank):
    X, _ = gp_problem(n, d, 5 * n)
    raw = default_test_raw(d, oracle)
    op = make_op(G, gpk_ctx, X, raw)
    pc = G.PivotedCholeskyPreconditioner(op, rank)
    V = np.random.default_rng(3).standard_normal((n, 5))
    ref = oracle.precond(X, raw, rank, V)
    assert pc.achieved_rank() == ref["achieved_rank"]
    if rank:
        assert np.array_equal(pc.pivots(), ref["pivots"])
        assert np.max(np.abs(pc.factor() - ref["factor"])) <= 1e-10
    assert colrel(pc.apply(V), ref["apply"]) <= 1e-9


def _targets(oracle, n, s, seed, y):
    T = np.empty((n, s + 1), order="F")
    T[:, 0] = y
    T[:, 1:] = oracle.stream_draw(seed, 2, 0, "gaussian", n * s).reshape((n, s), order="F")
    return T


@pytest.mark.parametrize("kind,n,d,s,extra", [
    (0, 1024, 8, 16, dict(preconditioner_rank=100)),
    (0, 2048, 20, 64, dict(preconditioner_rank=100)),
    (1, 1024, 8, 16, dict(block_size=128)),
    (1, 2048, 26, 64, dict(block_size=512)),
    (2, 1024, 3, 16, dict(batch_size=128, learning_rate=10.0, max_epochs=5)),
])
def test_solvers_match_oracle(G, kctx, oracle, kind, n, d, s, extra):
    X, y = gp_problem(n, d, 6 * n + kind)
    raw = oracle.raw_from_constrained([1.0] * d + [1.0, 0.1 if kind < 2 else 0.5])
    T = _targets(oracle, n, s, 11, y)
    cfg = dict(kind=kind, tolerance=0.01, max_epochs=50, seed=4, substream=1)
    cfg.update(extra)
    ref = oracle.solve(X, raw, T, oracle.solver_config(**cfg), threads=8)
    op = make_op(G, kctx, X, raw)
    batch = G.LinearSystemBatch(op, T)
    rep = G.solve(batch, G.SolverConfig(**cfg))
    assert not rep.aborted
    assert abs(rep.iterations - ref["iterations"]) <= 1
    assert rep.reached_tolerance == ref["reached_tolerance"] or abs(rep.iterations - ref["iterations"]) == 1
    if rep.iterations == ref["iterations"]:
        assert abs(rep.mean_residual_norm - ref["mean_residual_norm"]) <= 1e-4 * ref["mean_residual_norm"]
        assert abs(rep.probe_residual_norm - ref["probe_residual_norm"]) <= 1e-4 * ref["probe_residual_norm"]


def test_cg_pre_solved_terminates_immediately(G, gpk_ctx, oracle):  # test_solvers.cpp:113-127
    n, d = 300, 2
    X, y = gp_problem(n, d, 305)
    raw = oracle.raw_from_constrained([1.0, 1.0, 1.0, 0.4])
    T = _targets(oracle, n, 2, 306, y)
    direct = np.linalg.solve(oracle.dense(X, raw), T)
    op = make_op(G, gpk_ctx, X, raw)
    b = G.LinearSystemBatch(op, T)
    b.warm_start(direct)
    # tolerance 1e-4: the exact FP64 solution has an FP32-operator residual of ~1e-6..1e-5
    rep = G.solve_cg(b, G.SolverConfig(tolerance=1e-4, max_epochs=50))
    assert rep.iterations == 0 and rep.reached_tolerance
    assert np.array_equal(b.solutions, direct)


def test_cg_converges_to_dense_solution(G, gpk_ctx, oracle):
    n, d = 400, 3
    X, y = gp_problem(n, d, 307)
    raw = oracle.raw_from_constrained([1.0, 1.0, 1.0, 1.0, 0.5])
    T = _targets(oracle, n, 4, 308, y)
    direct = np.linalg.solve(oracle.dense(X, raw), T)
    op = make_op(G, gpk_ctx, X, raw)
    b = G.LinearSystemBatch(op, T)
    pc = G.PivotedCholeskyPreconditioner(op, 50)
    rep = G.solve_cg(b, G.SolverConfig(tolerance=1e-5, max_epochs=200), pc)
    assert rep.reached_tolerance
    err = max(np.linalg.norm(b.solutions[:, j] - direct[:, j]) / np.linalg.norm(direct[:, j]) for j in range(5))
    assert err <= 1e-4


def test_sgd_zero_lr_and_divergence(G, gpk_ctx, oracle):  # test_solvers.cpp:268-283, 331-343
    n = 256
    X, y = gp_problem(n, 2, 331)
    raw = oracle.raw_from_constrained([1.0, 1.0, 1.0, 0.4])
    T = _targets(oracle, n, 2, 332, y)
    op = make_op(G, gpk_ctx, X, raw)
    b = G.LinearSystemBatch(op, T)
    rep = G.solve_sgd(b, G.SolverConfig(kind=2, tolerance=1e-12, max_epochs=1, batch_size=16, learning_rate=0.0))
    assert np.max(np.abs(b.solutions)) == 0.0 and np.array_equal(b.residuals, T) and rep.residuals_estimated
    b2 = G.LinearSystemBatch(op, T)
    rep2 = G.solve_sgd(b2, G.SolverConfig(kind=2, tolerance=1e-10, max_epochs=50, batch_size=16,
                                          learning_rate=1e6))
    assert rep2.aborted and "divergence" in rep2.abort_reason
    # the oracle diverges too; the GPU's FP32 operator images overflow at
    # ~3.4e38 rather than FP64's ~1.8e308, so it can only stop earlier
    o2 = oracle.solve(X, raw, T, oracle.solver_config(kind=2, tolerance=1e-10, max_epochs=50, batch_size=16,
                                                      learning_rate=1e6))
    assert o2["aborted"] and rep2.iterations <= o2["iterations"]


@pytest.mark.parametrize("d", [2, 20])  # d = 2: lazy-momentum slab kernel; d = 20: full-state SGD path
def test_sgd_divergence_iteration_count(G, gpk_ctx, oracle, d):  # solvers.cpp:168-177
    """A non-finite iterate aborts in the iteration that formed it (t + 1
    updates reported, as solve_sgd does), on every SGD code path."""
    n = 256
    X, y = gp_problem(n, d, 333)
    raw = oracle.raw_from_constrained([1.0] * d + [1.0, 0.4])
    T = _targets(oracle, n, 2, 334, y)
    T[5, 1] = np.inf
    op = make_op(G, gpk_ctx, X, raw)
    cfg = dict(kind=2, tolerance=1e-10, max_epochs=5, batch_size=16, learning_rate=1.0)
    ref = oracle.solve(X, raw, T, oracle.solver_config(**cfg))
    b = G.LinearSystemBatch(op, T)
    rep = G.solve_sgd(b, G.SolverConfig(**cfg))
    assert ref["aborted"] and rep.aborted
    assert rep.iterations == ref["iterations"], (rep.iterations, ref["iterations"])
    assert rep.epochs_consumed == ref["epochs_consumed"]


def test_sgd_minibatches_bit_exact(G, gpk_ctx, oracle):
    n, b, rounds = 393216, 512, 6
    cfg = G.SolverConfig(kind=2, batch_size=b, seed=4, substream=7)
    got = G.sgd_batches(gpk_ctx, n, cfg, 0, rounds)
    ref = oracle.sample_without_replacement(4, 6, 7, n, b, rounds)
    assert np.array_equal(got, ref)
    got2 = G.sgd_batches(gpk_ctx, n, cfg, 3, 2)
    assert np.array_equal(got2, ref[3:5])
    small = G.sgd_batches(gpk_ctx, 97, G.SolverConfig(kind=2, batch_size=31, seed=5, substream=0), 0, 20)
    assert np.array_equal(small, oracle.sample_without_replacement(5, 6, 0, 97, 31, 20))


def test_epoch_budget_law(G, gpk_ctx, oracle):  # test_solvers.cpp:345-364
    n = 512
    X, y = gp_problem(n, 2, 349)
    raw = oracle.raw_from_constrained([1.0, 1.0, 1.0, 0.05])
    T = _targets(oracle, n, 3, 350, y)
    op = make_op(G, gpk_ctx, X, raw)
    for kind, per in ((0, 1.0), (1, 33 / n), (2, 20 / n)):
        b = G.LinearSystemBatch(op, T)
        rep = G.solve(b, G.SolverConfig(kind=kind, tolerance=1e-14, max_epochs=3, block_size=33, batch_size=20,
                                         learning_rate=1.0))
        assert rep.epochs_consumed <= 3.0 + per + 1e-12


@pytest.mark.parametrize("n,d,pairs,s", [(600, 3, 64, 8), (2048, 26, 1024, 64)])
def test_pathwise_targets_match_oracle(G, gpk_ctx, oracle, n, d, pairs, s):
    X, _ = gp_problem(n, d, 7 * n)
    raw = default_test_raw(d, oracle)
    op = make_op(G, gpk_ctx, X, raw)
    basis = G.build_rff_basis(gpk_ctx, d, pairs, s, 3)
    f, w = basis.arrays()
    rf, rw = oracle.rff_basis(d, pairs, s, 3)
    assert np.array_equal(f, rf) and np.array_equal(w, rw)  # host Philox/Box-Muller port: bit-exact
    t = G.pathwise_targets(basis, op, s, 3)
    r = oracle.pathwise_targets(X, raw, pairs, s, s, 3)
    assert np.max(np.abs(t.noise - r["noise"])) <= 1e-12
    assert np.max(np.abs(t.prior_values - r["prior_values"])) <= 1e-10 * max(1, np.max(np.abs(r["prior_values"])))
    assert np.max(np.abs(t.xi - r["xi"])) <= 1e-10 * max(1, np.max(np.abs(r["xi"])))


def test_optimise_trajectory_matches_oracle(G, kctx, oracle):
    """C1-shaped run at reduced n: pathwise + warm start + CG, 10 Adam steps."""
    n, d = 1024, 8
    X32, y32 = oracle.sinsum_dataset(n, d, seed=0)
    X, y = X32.astype(np.float64), y32.astype(np.float64)
    scfg = dict(kind=0, tolerance=0.01, max_epochs=50, preconditioner_rank=100)
    ocfg = dict(estimator=1, warm_start=True, steps=10, learning_rate=0.1, probe_count=16, rff_pairs=512,
                probe_seed=2, feature_seed=3, solver_seed=4)
    ref = oracle.optimise(X, y, oracle.outer_config(solver=oracle.solver_config(**scfg), **ocfg), threads=8)
    got = G.optimise(kctx, X, y, G.OuterConfig(solver=G.SolverConfig(**scfg), **ocfg))
    assert np.max(np.abs(got["constrained"] - ref["constrained"]) / ref["constrained"]) <= 1e-3
    assert np.max(np.abs(got["iterations"] - ref["iterations"])) <= 1
    same = got["iterations"] == ref["iterations"]
    g, rg = got["gradient"][same], ref["gradient"][same]
    assert np.max(np.abs(g - rg) / np.maximum(np.abs(rg), 1e-2 * np.max(np.abs(rg)))) <= 1e-3


@pytest.mark.parametrize("solver", ["cg", "sgd"])
def test_sharded_optimiser_world1_matches_plain(G, gpk_ctx, oracle, solver):
    """The row-sharded optimiser (NCCL communicator, all-gathered packed
    directions / SGD gradient partials and partial sums) on a 1-rank
    communicator reproduces the plain single-GPU run bit for bit (n above
    the dense-cache cap, so both run the tcgen05 operator)."""
    from paper_2405_18457_b200 import parallel as P
    n, d = 4224, 8
    X32, y32 = G.sinsum_dataset(n, d, False, 0.1, 0)
    X, y = X32.astype(np.float64), y32.astype(np.float64)
    scfg = dict(kind=0, tolerance=0.01, max_epochs=50, preconditioner_rank=100) if solver == "cg" else \
        dict(kind=2, tolerance=0.01, max_epochs=10, batch_size=256, learning_rate=10.0, momentum=0.9)
    ocfg = dict(estimator=1, warm_start=True, steps=4, learning_rate=0.1, probe_count=16, rff_pairs=256,
                probe_seed=2, feature_seed=3, solver_seed=4)
    plain = G.optimise(gpk_ctx, X, y, G.OuterConfig(solver=G.SolverConfig(**scfg), **ocfg))
    ctx1 = G.Context(0)
    ctx1.init_comm(P.comm_unique_id(), 1, 0)
    sharded = G.optimise(ctx1, X, y, G.OuterConfig(solver=G.SolverConfig(**scfg), **ocfg))
    for key in ("constrained", "gradient", "mean_residual_norm", "probe_residual_norm", "iterations"):
        assert np.array_equal(plain[key], sharded[key]), key


@pytest.mark.parametrize("n,d,block", [(2048, 8, 512), (1000, 3, 200), (700, 5, 64), (1500, 20, 333)])
def test_ap_block_inverse_paths_agree(G, oracle, n, d, block, monkeypatch):
    """AP diagonal-block inverses: the recursive Schur-complement DGEMM path
    (default) and the cuSOLVER potrf + triangular-solve path give the same
    solve (same iteration count; solutions equal to FP64 rounding)."""
    X, y = gp_problem(n, d, 9 * n)
    raw = oracle.raw_from_constrained([1.0] * d + [1.0, 0.2])
    T = _targets(oracle, n, 8, 9 * n + 1, y)
    cfg = G.SolverConfig(kind=1, tolerance=0.01, max_epochs=50, block_size=block)
    out = []
    for mode in ("1", "0"):
        monkeypatch.setenv("GPK_SPD_INVERSE", mode)
        ctx = G.Context(0)
        op = make_op(G, ctx, X, raw)
        b = G.LinearSystemBatch(op, T)
        rep = G.solve_ap(b, cfg)
        out.append((rep.iterations, b.solutions.copy()))
        ctx.close()
    (i1, v1), (i0, v0) = out
    # both inverses are exact to FP64 rounding (test_spd_inverse_both_paths);
    # the solves may then differ by the rounding the AP iteration carries
    assert abs(i1 - i0) <= 1
    if i1 == i0:
        assert np.max(np.abs(v1 - v0)) <= 1e-6 * np.max(np.abs(v0))


@pytest.mark.parametrize("dim,batch", [(64, 3), (200, 4), (333, 2), (512, 5), (97, 1)])
def test_spd_inverse_both_paths(G, gpk_ctx, oracle, dim, batch):
    """Both AP block-inverse paths against numpy on kernel blocks H[blk, blk]."""
    rng = np.random.default_rng(dim)
    mats = []
    for k in range(batch):
        X = rng.standard_normal((dim, 4))
        raw = oracle.raw_from_constrained([0.7, 1.0, 1.3, 0.9, 1.0, 0.1 + 0.1 * k])
        mats.append(oracle.dense(X, raw))
    mats = np.stack(mats)
    for mode in (1, 0):
        inv = G.gpiter.spd_inverse(gpk_ctx, mats, mode)
        for k in range(batch):
            ref = np.linalg.inv(mats[k])
            assert np.max(np.abs(inv[k] - ref)) <= 1e-9 * np.max(np.abs(ref)), (mode, k)
            assert np.max(np.abs(mats[k] @ inv[k] - np.eye(dim))) <= 1e-9


def test_spd_inverse_rejects_indefinite(G, gpk_ctx):
    A = np.eye(80)
    A[40, 40] = -1.0
    for mode in (1, 0):
        with pytest.raises(ArithmeticError, match="not positive definite"):
            G.gpiter.spd_inverse(gpk_ctx, A, mode)


def test_ap_non_pd_block_raises_before_any_update(G, gpk_ctx, oracle):  # solvers.cpp:104-113
    """Duplicated points and noise 1e-12 make the diagonal blocks numerically
    indefinite: the oracle's factor_for throws; the device solve stops before
    its first update (solutions untouched) and raises the same error."""
    n = 256
    X = np.zeros((n, 2))
    X[:, 0] = np.repeat(np.arange(4), 64) * 5.0
    raw = oracle.raw_from_constrained([1.0, 1.0, 1.0, 1e-12])
    T = np.asfortranarray(np.random.default_rng(0).standard_normal((n, 3)))
    cfg = dict(kind=1, block_size=64, tolerance=1e-6, max_epochs=5)
    with pytest.raises(Exception, match="not positive definite"):
        oracle.solve(X, raw, T, oracle.solver_config(**cfg))
    op = make_op(G, gpk_ctx, X, raw)
    W = np.asfortranarray(np.random.default_rng(1).standard_normal((n, 3)))
    b = G.LinearSystemBatch(op, T)
    b.warm_start(W)
    with pytest.raises(ArithmeticError, match="not positive definite"):
        G.solve(b, G.SolverConfig(**cfg))
    assert np.array_equal(b.solutions, W)


def test_optimise_exact_dense_prior_matches_oracle(G, gpk_ctx, oracle):
    """ExactDense pathwise prior (outer_loop.cpp:140-153): device jittered
    cuSOLVER Cholesky + TRMM of the stream-8 weights against the oracle."""
    n, d = 600, 3
    X, y = gp_problem(n, d, 611)
    scfg = dict(kind=0, tolerance=0.01, max_epochs=100, preconditioner_rank=50)
    ocfg = dict(estimator=1, warm_start=True, steps=3, learning_rate=0.1, probe_count=8, rff_pairs=32,
                probe_seed=2, feature_seed=3, solver_seed=4, prior_mode=1)
    r = G.optimise(gpk_ctx, X, y, G.OuterConfig(solver=G.SolverConfig(**scfg), **ocfg))
    ref = oracle.optimise(X, y, oracle.outer_config(solver=oracle.solver_config(**scfg), **ocfg), threads=8)
    assert np.max(np.abs(r["constrained"] - ref["constrained"]) / ref["constrained"]) <= 1e-3
    assert np.all(np.abs(r["iterations"] - ref["iterations"]) <= 1)
    # the prior differs from the random-feature one
    ocfg["prior_mode"] = 0
    r0 = G.optimise(gpk_ctx, X, y, G.OuterConfig(solver=G.SolverConfig(**scfg), **ocfg))
    assert not np.array_equal(r0["gradient"][0], r["gradient"][0])


@pytest.mark.parametrize("n,d,steps", [(300, 2, 15), (700, 5, 8)])
def test_optimise_exact_matches_oracle(G, gpk_ctx, oracle, n, d, steps):
    """Row f4: Adam on the exact MLL (cuSOLVER Cholesky/inverse + fused FP64 dH pass)."""
    X, y = gp_problem(n, d, 13 * n)
    traj, raw = G.gpiter.optimise_exact(gpk_ctx, X, y, steps, 0.1)
    rtraj, rraw = oracle.optimise_exact(X, y, steps, 0.1)
    assert np.max(np.abs(traj - rtraj) / rtraj) <= 1e-8
    assert np.max(np.abs(raw - rraw)) <= 1e-8 * np.max(np.abs(rraw))
    # one exact gradient against the oracle's dense restatement
    _, g = oracle.exact(X, y, rraw)
    _, rraw1 = oracle.optimise_exact(X, y, 1, 0.1, init_constrained=[oracle.softplus(v) for v in rraw])
    _, graw1 = G.gpiter.optimise_exact(gpk_ctx, X, y, 1, 0.1, init_constrained=[oracle.softplus(v) for v in rraw])
    assert np.max(np.abs(graw1 - rraw1)) <= 1e-8 * np.max(np.abs(rraw1))


def test_init_heuristic_matches_oracle(G, gpk_ctx, oracle):
    X, y = gp_problem(900, 3, 4321)
    got = G.gpiter.init_heuristic(gpk_ctx, X, y, 3, 200, 11, 10, 0.1)
    ref = oracle.init_heuristic(X, y, 3, 200, 11, 10, 0.1)
    assert np.max(np.abs(got - ref) / ref) <= 1e-8
    whole = G.gpiter.init_heuristic(gpk_ctx, X[:150], y[:150], 1, 150, 7, 10, 0.1)
    _, raw = oracle.optimise_exact(X[:150], y[:150], 10, 0.1)
    assert np.max(np.abs(whole - [oracle.softplus(v) for v in raw])) <= 1e-8


@pytest.mark.parametrize("n,d,m", [(4096, 26, 65), (2100, 3, 17)])
def test_apply_streamk_matches_oracle(G, oracle, n, d, m, monkeypatch):
    """The stream-K operator launch (GPK_KV_STREAMK=1, deep mode forced): one
    persistent CTA per SM over (row tile, chunk) units, partial slots per tile."""
    monkeypatch.setenv("GPK_KV_STREAMK", "1")
    monkeypatch.setenv("GPK_KV_DEEP", "1")
    ctx = G.Context(0)
    X, _ = gp_problem(n, d, 77 + n)
    raw = default_test_raw(d, oracle)
    V = np.asfortranarray(np.random.default_rng(n).standard_normal((n, m)))
    got = make_op(G, ctx, X, raw).apply(V)
    ctx.close()
    ref = oracle.apply(X, raw, V, threads=8)
    assert colrel(got, ref) <= OP_TOL


@pytest.mark.parametrize("env", [{"GPK_KV_DEEP": "1", "GPK_TGRAM_MIN_D": "1"},  # deep launch, Gram MMAs at every d
                                 {"GPK_KV_DEEP": "1", "GPK_TGRAM": "0"},        # deep launch, FP32 distances
                                 {"GPK_KV_DEEP": "0", "GPK_TGRAM_MIN_D": "1"},  # two CTAs per SM (no Gram MMAs)
                                 {"GPK_KV_DEEP": "1", "GPK_KV_PANEL_MB": "1"},  # column panels of large products
                                 {"GPK_KV_DEEP": "1", "GPK_FLUSH_CHUNKS": "2"},  # double-buffered D, short groups
                                 {"GPK_GRAD_WAVE": "1"}],                       # gradient pass in row waves
                         ids=["deep-gram", "deep-fp32", "shallow", "panels", "dbuf-short-groups", "grad-wave"])
def test_operator_variants_match_oracle(env):
    """The launch variants the size heuristics pick at BASELINE sizes (one CTA
    per SM with tensor-core Gram distances for the C2 refresh and the AP
    solver), forced at oracle-checkable sizes in a fresh process."""
    import json
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, os.path.join(here, "_variant_probe.py")], env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    errs = json.loads(r.stdout.strip().splitlines()[-1])
    assert max(errs.values()) <= OP_TOL, errs


def test_optimiser_buffers_are_reused(G, gpk_ctx):
    """Device buffers come from the stream-ordered pool (GPK_DEVICE_POOL): a
    destroyed optimiser's buffers serve the next one, so repeated
    create/step/destroy cycles do not grow device memory, and destroy does not
    synchronise-and-unmap every buffer."""
    import time
    import pynvml  # not torch: importing torch after libgpk has loaded the system NCCL breaks torch's own
    pynvml.nvmlInit()
    dev = pynvml.nvmlDeviceGetHandleByIndex(0)
    X32, y32 = G.sinsum_dataset(4096, 8, False, 0.1, 0)
    X, y = X32.astype(np.float64), y32.astype(np.float64)
    sc = G.SolverConfig(kind=0, tolerance=0.01, max_epochs=20, preconditioner_rank=100)
    oc = G.OuterConfig(estimator=1, solver=sc, warm_start=True, steps=2, learning_rate=0.1, probe_count=16,
                       rff_pairs=256, probe_seed=2, feature_seed=3, solver_seed=4)
    used, close_s = [], []
    for _ in range(4):
        opt = G.Optimiser(gpk_ctx, X, y, oc, init_constrained=[1.0] * 8 + [1.0, 0.1])
        opt.step(2)
        gpk_ctx.synchronize()
        t = time.perf_counter()
        opt.close()
        close_s.append(time.perf_counter() - t)
        used.append(pynvml.nvmlDeviceGetMemoryInfo(dev).used)
    assert max(used[1:]) - used[1] <= 64 << 20, used
    assert min(close_s[1:]) < 5e-3, close_s
