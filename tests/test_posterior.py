"""Posterior predictions: the oracle restatement
against the reference's own posterior tests (proj/tests/test_posterior.cpp,
CPU) and the CUDA path against the oracle (gpu)."""
import numpy as np
import pytest

from _problems import default_test_raw, gp_problem


def _setup(oracle, n, d, seed):
    X, y = gp_problem(n, d, seed)
    raw = default_test_raw(d, oracle)
    H = oracle.dense(X, raw)
    return X, y, raw, H, np.linalg.solve(H, y)


def test_oracle_mean_matches_dense_and_decays(oracle):  # test_posterior.cpp:34-56
    X, y, raw, H, vy = _setup(oracle, 100, 2, 201)
    P = np.array([[0.2, -0.5], [1.3, 0.4], [-0.8, -0.1], [2.0, 1.0]])
    kpx = np.array([[oracle.matern32(p, x, raw) for x in X] for p in P])
    assert np.max(np.abs(oracle.cross_apply(P, X, raw, vy)[:, 0] - kpx @ vy)) <= 1e-12
    assert abs(oracle.cross_apply(np.array([[60.0, 60.0]]), X, raw, vy)[0, 0]) <= 1e-8
    assert np.max(np.abs(oracle.cross_apply(P, X, raw, np.zeros(100)))) == 0.0


def test_oracle_samples_reduce_to_mean_without_randomness(oracle):  # test_posterior.cpp:58-76
    X, y, raw, H, vy = _setup(oracle, 60, 2, 203)
    P = np.array([[0.0, 0.0], [0.7, -0.7], [-1.2, 0.5]])
    r = oracle.posterior(P, X, raw, vy, np.zeros((60, 3)))
    mean = oracle.cross_apply(P, X, raw, vy)[:, 0]
    assert np.max(np.abs(r["samples"][:, 1] - mean)) == 0.0


def test_oracle_metrics_closed_form(oracle):
    X, y, raw, H, vy = _setup(oracle, 50, 1, 211)
    P = X[:10]
    mean = oracle.cross_apply(P, X, raw, vy)[:, 0]
    r = oracle.posterior(P, X, raw, vy, np.zeros((50, 1)), test_targets=mean + 0.5, target_scale=2.0)
    assert abs(r["rmse"] - 0.5) <= 1e-12 and abs(r["rmse_raw"] - 1.0) <= 1e-12 and r["llh"] is None


@pytest.mark.gpu
def test_gpu_posterior_matches_oracle(gpk_ctx, oracle):
    import paper_2405_18457_b200 as G
    n, d, s, p, pairs = 3000, 6, 16, 777, 256
    X, y = gp_problem(n, d, 17)
    raw = default_test_raw(d, oracle)
    P, _ = gp_problem(p, d, 18)
    rng = np.random.default_rng(3)
    vy, Z = rng.standard_normal(n), rng.standard_normal((n, s))
    op = G.KernelOperator(X, G.Hyperparameters.from_raw(raw), gpk_ctx)
    got = G.predict_mean(op, P, vy)
    ref = oracle.cross_apply(P, X, raw, vy, threads=8)[:, 0]
    assert np.max(np.abs(got - ref)) <= 2e-5 * np.max(np.abs(ref))
    V = rng.standard_normal((n, 65))
    gv = G.cross_kernel_apply(op, P, V)
    rv = oracle.cross_apply(P, X, raw, V, threads=8)
    assert max(np.max(np.abs(gv[:, j] - rv[:, j])) / np.max(np.abs(rv[:, j])) for j in range(65)) <= 2e-5
    basis = G.build_rff_basis(gpk_ctx, d, pairs, s, 3)
    prior = oracle.prior_at(d, pairs, s, 3, raw, P, s)
    gs = G.sample_posterior(op, basis, P, vy, Z)
    rs = oracle.posterior(P, X, raw, vy, Z, prior=prior, threads=8)["samples"]
    assert np.max(np.abs(gs - rs)) <= 2e-5 * np.max(np.abs(rs))
    t = rng.standard_normal(p)
    gm = G.test_metrics(op, basis, P, t, vy, Z, target_scale=1.7)
    rm = oracle.posterior(P, X, raw, vy, Z, prior=prior, test_targets=t, target_scale=1.7, threads=8)
    for k in ("rmse", "rmse_raw", "llh", "llh_raw"):
        assert abs(gm[k] - rm[k]) <= 1e-4 * abs(rm[k]), k
    # no prior, zero probe solutions: every sample is the posterior mean (the
    # wider right-hand side runs a different kernel instance: FP32 rounding)
    gz = G.sample_posterior(op, None, P[:3], vy, np.zeros((n, 3)))
    assert np.max(np.abs(gz[:, 1] - got[:3])) <= 2e-5 * np.max(np.abs(got))
    assert np.array_equal(gz[:, 0], gz[:, 1]) and np.array_equal(gz[:, 1], gz[:, 2])


@pytest.mark.gpu
def test_gpu_cross_kernel_gram_form_matches_oracle(gpk_ctx, oracle):
    """k(P, X) V for d >= 21, where the tensor-core operator takes distances in
    Gram form from the points' own (x, |x|^2) image (no kernel diagonal)."""
    import paper_2405_18457_b200 as G
    n, d, p = 1500, 24, 333
    X, y = gp_problem(n, d, 21)
    raw = default_test_raw(d, oracle)
    P, _ = gp_problem(p, d, 22)
    P[:5] = X[:5]  # coincident points: r = 0 through the Gram form
    rng = np.random.default_rng(5)
    op = G.KernelOperator(X, G.Hyperparameters.from_raw(raw), gpk_ctx)
    V = rng.standard_normal((n, 65))
    gv = G.cross_kernel_apply(op, P, V)
    rv = oracle.cross_apply(P, X, raw, V, threads=8)
    assert max(np.max(np.abs(gv[:, j] - rv[:, j])) / np.max(np.abs(rv[:, j])) for j in range(65)) <= 2e-5


@pytest.mark.gpu
def test_gpu_compare_oracle_outputs(gpk_ctx, tmp_path):
    """`gpiter compare-oracle` on the GPU (gpiter_cli.cpp:230-280): the iterative
    pathwise trajectory against Adam on the exact marginal likelihood from the
    same initialisation; both written in the reference tool's formats."""
    import json

    from oracle import oracle as O
    from paper_2405_18457_b200 import gpiter, outputs
    X32, y32 = O.sinsum_dataset(512, 3, False, 0.1, 0)
    sc = gpiter.SolverConfig(kind=0, tolerance=1e-4, max_epochs=200, preconditioner_rank=50)
    cfg = gpiter.OuterConfig(estimator=1, solver=sc, warm_start=True, steps=5, learning_rate=0.1, probe_count=64,
                             rff_pairs=1024, probe_seed=2, feature_seed=3, solver_seed=4, init_value=1.0)
    out = outputs.compare_oracle(gpk_ctx, X32.astype(np.float64), y32.astype(np.float64), cfg, tmp_path)
    assert json.loads((tmp_path / "compare_oracle.json").read_text()) == out
    assert sum(out["histogram_counts"]) == 5 * 5
    # Adam's first steps are sign-driven: both trajectories move together
    assert out["max_abs_diff"] < 0.05
