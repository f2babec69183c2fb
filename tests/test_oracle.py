"""Pins the FP64 oracle (oracle/, a restatement of the reference without Eigen)
against the reference's own known-answer tests and property tests
(/root/reference/proj/tests/*.cpp, restated case by case; file:line cited).
CPU only."""
import numpy as np
import pytest

from _problems import default_test_raw, gp_problem


# ---- test_rng.cpp ------------------------------------------------------
def test_philox_known_answers(oracle):  # test_rng.cpp:10-38
    assert oracle.philox([1, 0, 0, 0], [0, 0]) == [0x02f4ba6408e4d89b, 0x3dd62b0b9ca8c5b2, 0x1c8667a55d902e79,
                                                   0x907d7a052fd5b4dc]
    assert oracle.philox([2, 0, 0, 0], [0, 0]) == [0x809bf322883987c3, 0x471128b9e807f7dd, 0xf250ba0dbec065b7,
                                                   0xfc6ed66767a457bc]
    assert oracle.philox([43, 0, 0, 0], [0x123456789abcdef0, 0]) == [0x65c23bbfdb8a827e, 0x95b606d9172b3a83,
                                                                     0xfee9691c17f52a9d, 0x17f169d5594179a1]
    ones = 0xffffffffffffffff
    assert oracle.philox([0, 0, 0, 0], [ones, ones]) == [0x44b7493d1acfc229, 0x6636af8e997921dd,
                                                         0x3f73e132b5b3780e, 0x605644dde03b01b1]


def test_philox_matches_numpy_philox(oracle):
    # independent implementation: numpy's Philox evaluates at counter + 1
    g = np.random.Philox(key=np.array([7, 2], dtype=np.uint64), counter=np.array([5, 3, 0, 0], dtype=np.uint64))
    ref = [int(x) for x in g.random_raw(4)]
    assert oracle.philox([6, 3, 0, 0], [7, 2]) == ref


def test_streams_deterministic_and_independent(oracle):  # test_rng.cpp:40-56
    a = oracle.stream_draw(7, 2, 0, "u64", 100)
    b = oracle.stream_draw(7, 2, 0, "u64", 100)
    assert np.array_equal(a, b)
    c = oracle.stream_draw(7, 4, 0, "u64", 8)
    d = oracle.stream_draw(7, 2, 1, "u64", 8)
    assert not np.array_equal(c, a[:8]) and not np.array_equal(d, a[:8])


def test_gaussian_moments(oracle):  # test_rng.cpp:58-72
    g = oracle.stream_draw(3, 2, 0, "gaussian", 200000)
    assert abs(g.mean()) < 0.01
    assert abs((g ** 2).mean() - 1.0) < 0.02
    assert abs((g ** 4).mean() - 3.0) < 0.15


def test_permutation(oracle):  # test_rng.cpp:74-83
    p = oracle.permutation(11, 1, 500)
    assert np.array_equal(np.sort(p), np.arange(500))
    assert not np.array_equal(oracle.permutation(12, 1, 500), p)


def test_sample_without_replacement_sorted_distinct(oracle):  # test_rng.cpp:85-95
    s = oracle.sample_without_replacement(5, 6, 0, 97, 31, rounds=20)
    for row in s:
        assert np.all(np.diff(row) > 0) and row[0] >= 0 and row[-1] < 97


def test_floyd_restatement(oracle):
    # rng.cpp:108-126 restated in Python from raw u64 draws
    n, k, rounds = 1000, 37, 5
    u = oracle.stream_draw(9, 6, 3, "u64", k * rounds)
    got = oracle.sample_without_replacement(9, 6, 3, n, k, rounds)
    for r in range(rounds):
        taken, chosen = set(), []
        for q, j in enumerate(range(n - k, n)):
            t = int(u[r * k + q]) % (j + 1)
            pick = j if t in taken else t
            taken.add(pick)
            chosen.append(pick)
        assert np.array_equal(sorted(chosen), got[r])


def test_uniform_ints_cover_range(oracle):  # test_rng.cpp:97-101
    v = oracle.stream_draw(9, 6, 0, "below", 10000, bound=10)
    assert np.all(np.bincount(v.astype(int), minlength=10) > 800)


# ---- test_kernel.cpp ---------------------------------------------------
def test_softplus_round_trip(oracle):  # test_kernel.cpp:18-25
    for nu in (-30.0, -5.0, -0.3, 0.0, 0.7, 12.0, 30.0):
        assert abs(oracle.softplus_inverse(oracle.softplus(nu)) - nu) <= 1e-10 * max(1, abs(nu))
    assert abs(oracle.softplus_inverse(1.0) - 0.5413248546129181) <= 1e-14
    assert oracle.sigmoid(0.0) == 0.5


def test_matern_closed_form(oracle):  # test_kernel.cpp:27-55
    raw = oracle.raw_from_constrained([1.0, 1.0, 1.0])
    assert abs(oracle.matern32([0.3], [0.3], raw) - 1.0) <= 1e-15
    assert abs(oracle.matern32([0.3], [1.3], raw) - 0.48335772459650765) <= 1e-15
    with pytest.raises(ValueError):
        oracle.matern32([0.3], [np.nan], raw)
    raw2 = oracle.raw_from_constrained([0.5, 2.0, 1.5, 0.1])
    r = np.sqrt(2.0)
    expect = 1.5 ** 2 * (1 + np.sqrt(3) * r) * np.exp(-np.sqrt(3) * r)
    assert abs(oracle.matern32([0, 0], [0.5, 2.0], raw2) - expect) <= 1e-14 * expect


def _dense_reference(X, raw, oracle):
    n = X.shape[0]
    H = np.empty((n, n))
    for i in range(n):
        for j in range(n):
            H[i, j] = oracle.matern32(X[i], X[j], raw)
    sigma = oracle.softplus(raw[-1])
    return H + sigma ** 2 * np.eye(n)


def test_hmatvec_dense_and_block_size_independent(oracle):  # test_kernel.cpp:57-98
    n, d = 64, 3
    X, _ = gp_problem(n, d, 101)
    raw = default_test_raw(d, oracle)
    Href = _dense_reference(X, raw, oracle)
    assert np.max(np.abs(oracle.apply(X, raw, np.eye(n)) - Href)) <= 1e-12
    assert np.max(np.abs(oracle.dense(X, raw) - Href)) <= 1e-12
    assert np.max(np.abs(oracle.apply(X, raw, np.zeros((n, 5))))) == 0.0
    V = np.asfortranarray(oracle.stream_draw(55, 2, 0, "gaussian", n * 7).reshape((n, 7), order="F"))
    base = oracle.apply(X, raw, V)
    for block in (1, 5, 8, 17, 64, 200):
        assert np.array_equal(oracle.apply(X, raw, V, block_rows=block), base)
    assert np.array_equal(oracle.apply(X, raw, V, threads=4), base)


def test_operator_symmetric_positive_definite(oracle):  # test_kernel.cpp:100-117
    n = 80
    X, _ = gp_problem(n, 2, 7)
    raw = default_test_raw(2, oracle)
    sigma2 = oracle.softplus(raw[-1]) ** 2
    g = oracle.stream_draw(8, 2, 0, "gaussian", 10 * n).reshape(10, n)
    for r in range(5):
        u, v = g[2 * r], g[2 * r + 1]
        left = u @ oracle.apply(X, raw, v)[:, 0]
        right = oracle.apply(X, raw, u)[:, 0] @ v
        assert abs(left - right) <= 1e-8 * abs(left)
        assert v @ oracle.apply(X, raw, v)[:, 0] >= sigma2 * (v @ v) * (1 - 1e-12)


def test_slabs_agree_with_dense(oracle):  # test_kernel.cpp:119-141
    n = 50
    X, _ = gp_problem(n, 2, 13)
    raw = default_test_raw(2, oracle)
    H = oracle.dense(X, raw)
    V = np.asfortranarray(np.random.default_rng(1).standard_normal((n, 3)))
    rows = [0, 7, 13, 29, 49]
    assert np.max(np.abs(oracle.apply_rows(X, raw, rows, V) - H[rows] @ V)) <= 1e-12
    U = np.asfortranarray(np.random.default_rng(2).standard_normal((10, 3)))
    assert np.max(np.abs(oracle.apply_columns(X, raw, 20, 10, U) - H[:, 20:30] @ U)) <= 1e-10
    assert np.array_equal(oracle.dense_block(X, raw, 5, 12, 7, 20), H[5:17, 7:27])


def test_derivative_matches_finite_differences(oracle):  # test_kernel.cpp:143-177
    n, d = 50, 3
    X, _ = gp_problem(n, d, 23)
    c = np.array([0.8 + 0.1 * i for i in range(d)] + [1.2, 0.4])
    raw = oracle.raw_from_constrained(c)
    V = np.asfortranarray(np.random.default_rng(2).standard_normal((n, 2)))
    eps = 1e-5
    for k in range(d + 2):
        up, dn = c.copy(), c.copy()
        up[k] += eps
        dn[k] -= eps
        fd = (oracle.apply(X, oracle.raw_from_constrained(up), V) -
              oracle.apply(X, oracle.raw_from_constrained(dn), V)) / (2 * eps)
        an = oracle.derivative_apply(X, raw, k, V)
        assert np.max(np.abs(an - fd)) / max(1.0, np.max(np.abs(fd))) <= 1e-5
    noise = oracle.derivative_apply(X, raw, d + 1, V)
    assert np.array_equal(noise, (2.0 * oracle.softplus(raw[-1])) * V)
    with pytest.raises(IndexError):
        oracle.derivative_apply(X, raw, d + 2, V)


def test_quadratic_forms_match_explicit(oracle):  # test_kernel.cpp:179-198
    n, d = 40, 2
    X, _ = gp_problem(n, d, 31)
    raw = default_test_raw(d, oracle)
    rng = np.random.default_rng(3)
    U, W = rng.standard_normal((n, 4)), rng.standard_normal((n, 4))
    f1, f2 = oracle.quad_forms(X, raw, U, W, U, U)
    for k in range(d + 2):
        dhw = oracle.derivative_apply(X, raw, k, W)
        assert abs(f1[k] - np.sum(U * dhw)) <= 1e-10 * max(1.0, abs(f1[k]))
        dhu = oracle.derivative_apply(X, raw, k, U)
        assert abs(f2[k] - np.sum(U * dhu)) <= 1e-10 * max(1.0, abs(f2[k]))
    g1, _ = oracle.quad_forms(X, raw, U, W, U, U, threads=4)
    assert np.array_equal(g1, f1)


# ---- test_pivoted_cholesky.cpp ------------------------------------------
def test_precond_full_rank_inverts(oracle):  # test_pivoted_cholesky.cpp:10-23
    n = 20
    X, _ = gp_problem(n, 2, 41)
    raw = default_test_raw(2, oracle)
    b = np.random.default_rng(1).standard_normal(n)
    pc = oracle.precond(X, raw, n, b)
    direct = np.linalg.solve(oracle.dense(X, raw), b)
    assert np.linalg.norm(pc["apply"][:, 0] - direct) / np.linalg.norm(direct) <= 1e-8


def test_precond_rank_zero(oracle):  # test_pivoted_cholesky.cpp:25-33
    n = 15
    X, _ = gp_problem(n, 1, 43)
    raw = default_test_raw(1, oracle)
    b = np.linspace(-1, 1, n)
    pc = oracle.precond(X, raw, 0, b)
    assert np.array_equal(pc["apply"][:, 0], b / oracle.softplus(raw[-1]) ** 2)


def test_precond_spd_and_low_rank(oracle):  # test_pivoted_cholesky.cpp:35-66
    n = 40
    X, _ = gp_problem(n, 1, 53)
    raw = default_test_raw(1, oracle)
    full = oracle.precond(X, raw, n)
    K = oracle.dense(X, raw) - oracle.softplus(raw[-1]) ** 2 * np.eye(n)
    L = full["factor"]
    assert np.max(np.abs(L @ L.T - K)) <= 1e-8
    X2, _ = gp_problem(30, 2, 47)
    raw2 = default_test_raw(2, oracle)
    rng = np.random.default_rng(5)
    for _ in range(5):
        u, v = rng.standard_normal(30), rng.standard_normal(30)
        pu = oracle.precond(X2, raw2, 10, u)["apply"][:, 0]
        pv = oracle.precond(X2, raw2, 10, v)["apply"][:, 0]
        assert abs(u @ pv - pu @ v) <= 1e-10 * max(1, abs(u @ pv))
        assert v @ pv > 0


# ---- test_solvers.cpp -----------------------------------------------------
def _problem(n, d, s, seed, oracle, noise=0.4):
    X, y = gp_problem(n, d, seed)
    c = [1.0] * d + [1.0, noise]
    raw = oracle.raw_from_constrained(c)
    T = np.empty((n, s + 1), order="F")
    T[:, 0] = y
    if s:
        T[:, 1:] = oracle.stream_draw(seed + 1, 2, 0, "gaussian", n * s).reshape((n, s), order="F")
    direct = np.linalg.solve(oracle.dense(X, raw), T)
    return X, raw, T, direct


def _worst(sol, direct):
    return max(np.linalg.norm(sol[:, j] - direct[:, j]) / np.linalg.norm(direct[:, j]) for j in range(sol.shape[1]))


def test_termination_follows_both_norms(oracle):  # test_solvers.cpp:57-85
    X, raw, T, _ = _problem(20, 2, 2, 301, oracle)
    R = np.zeros_like(T)
    assert oracle.termination_check(T, R, 0.01) == (0.0, 0.0, True)
    scales = np.linalg.norm(T, axis=0) + 1e-12
    R[:, 0] = 0.005 * T[:, 0] / np.linalg.norm(T[:, 0]) * scales[0]
    for j in (1, 2):
        R[:, j] = 0.02 * T[:, j] / np.linalg.norm(T[:, j]) * scales[j]
    mean, probe, done = oracle.termination_check(T, R, 0.01)
    assert abs(mean - 0.005) <= 1e-9 * 0.005 and abs(probe - 0.02) <= 1e-9 * 0.02 and not done
    assert abs(oracle.termination_check(T, T, 0.01)[1] - 1.0) <= 1e-9


def test_cg_pre_solved_terminates_immediately(oracle):  # test_solvers.cpp:113-127
    X, raw, T, direct = _problem(30, 2, 2, 305, oracle)
    cfg = oracle.solver_config(kind=0, tolerance=1e-6, max_epochs=50)
    r = oracle.solve(X, raw, T, cfg, warm=direct, explicit_rank=-2)
    assert r["iterations"] == 0 and r["reached_tolerance"]
    assert np.array_equal(r["solutions"], direct)


def test_cg_matches_dense(oracle):  # test_solvers.cpp:129-141
    X, raw, T, direct = _problem(200, 3, 4, 307, oracle)
    r = oracle.solve(X, raw, T, oracle.solver_config(kind=0, tolerance=1e-10, max_epochs=200), explicit_rank=0)
    assert r["reached_tolerance"] and _worst(r["solutions"], direct) <= 1e-6
    assert r["epochs_consumed"] == r["iterations"]


def test_cg_preconditioner_helps(oracle):  # test_solvers.cpp:143-159
    X, raw, T, _ = _problem(150, 2, 4, 309, oracle, noise=0.1)
    cfg = oracle.solver_config(kind=0, tolerance=1e-8, max_epochs=300)
    plain = oracle.solve(X, raw, T, cfg, explicit_rank=-2)
    pre = oracle.solve(X, raw, T, cfg, explicit_rank=50)
    assert pre["reached_tolerance"] and pre["iterations"] < plain["iterations"]


def test_ap_single_block_is_direct(oracle):  # test_solvers.cpp:197-210
    X, raw, T, direct = _problem(50, 2, 3, 319, oracle)
    r = oracle.solve(X, raw, T, oracle.solver_config(kind=1, tolerance=1e-8, max_epochs=10, block_size=50))
    assert r["iterations"] == 1 and r["reached_tolerance"] and _worst(r["solutions"], direct) <= 1e-8


def test_ap_honest_residuals(oracle):  # test_solvers.cpp:212-226
    X, raw, T, _ = _problem(200, 2, 4, 321, oracle)
    # budget 400 (the reference uses 200 on its own GP-prior data; this seeded instance converges slower)
    r = oracle.solve(X, raw, T, oracle.solver_config(kind=1, tolerance=0.01, max_epochs=400, block_size=50))
    assert r["reached_tolerance"]
    R = T - oracle.apply(X, raw, r["solutions"])
    mean, probe, _ = oracle.termination_check(T, R, 0.011)
    assert mean <= 0.011 and probe <= 0.011
    assert r["epochs_consumed"] == pytest.approx(r["iterations"] * 50 / 200)


def test_sgd_zero_lr_noop(oracle):  # test_solvers.cpp:268-283
    X, raw, T, _ = _problem(64, 2, 2, 331, oracle)
    r = oracle.solve(X, raw, T, oracle.solver_config(kind=2, tolerance=1e-12, max_epochs=1, batch_size=16,
                                                     learning_rate=0.0))
    assert np.max(np.abs(r["solutions"])) == 0.0 and np.array_equal(r["residuals"], T)
    assert r["residuals_estimated"]


def test_sgd_full_batch_is_gradient_descent(oracle):  # test_solvers.cpp:285-307 (bit for bit)
    X, raw, T, _ = _problem(32, 1, 1, 337, oracle)
    cfg = oracle.solver_config(kind=2, tolerance=1e-12, max_epochs=7, batch_size=32, learning_rate=3.0, momentum=0.0)
    r = oracle.solve(X, raw, T, cfg)
    v = np.zeros((32, 2), order="F")
    step = 3.0 / 32.0
    for _ in range(7):
        g = oracle.apply_rows(X, raw, list(range(32)), v) - T
        v = v - step * g
    assert np.array_equal(r["solutions"], v)


def test_sgd_divergence_reported(oracle):  # test_solvers.cpp:331-343
    X, raw, T, _ = _problem(64, 2, 2, 347, oracle)
    r = oracle.solve(X, raw, T, oracle.solver_config(kind=2, tolerance=1e-10, max_epochs=50, batch_size=16,
                                                     learning_rate=1e6))
    assert r["aborted"] and "divergence" in r["abort_reason"]


def test_epoch_budget_law(oracle):  # test_solvers.cpp:345-364
    X, raw, T, _ = _problem(128, 2, 3, 349, oracle, noise=0.05)
    for kind, per in ((0, 1.0), (1, 33 / 128), (2, 20 / 128)):
        cfg = oracle.solver_config(kind=kind, tolerance=1e-14, max_epochs=3, block_size=33, batch_size=20,
                                   learning_rate=1.0)
        r = oracle.solve(X, raw, T, cfg)
        assert r["epochs_consumed"] <= 3.0 + per + 1e-12


def test_solver_oracle_equivalence(oracle):  # test_solvers.cpp:391-409
    X, raw, T, direct = _problem(150, 2, 3, 359, oracle, noise=0.7)
    for kind in (0, 1, 2):
        cfg = oracle.solver_config(kind=kind, tolerance=1e-8, max_epochs=4000, block_size=40, batch_size=30,
                                   learning_rate=4.0, preconditioner_rank=30, seed=11)
        r = oracle.solve(X, raw, T, cfg)
        assert r["reached_tolerance"] and _worst(r["solutions"], direct) <= 1e-4


# ---- test_gradients.cpp / exact ----------------------------------------
def test_gradients_zero_inputs(oracle):  # test_gradients.cpp:60-71
    X, _ = gp_problem(20, 1, 85)
    raw = default_test_raw(1, oracle)
    g = oracle.gradient(X, raw, np.zeros(20), np.zeros((20, 4)))
    assert np.max(np.abs(g["values"])) == 0.0 and np.max(np.abs(g["trace_term"])) == 0.0


def test_deterministic_basis_gives_exact_gradient(oracle):  # test_gradients.cpp:34-58
    n, d = 60, 2
    X, y = gp_problem(n, d, 83)
    raw = default_test_raw(d, oracle)
    H = oracle.dense(X, raw)
    probes = np.sqrt(n) * np.eye(n)
    sols = np.linalg.solve(H, probes)
    vy = np.linalg.solve(H, y)
    g = oracle.gradient(X, raw, vy, sols, probes=probes)
    _, exact = oracle.exact(X, y, raw)
    assert np.allclose(g["values"], exact, rtol=1e-6, atol=1e-9)
    assert np.array_equal(g["values"], 0.5 * g["quadratic_term"] - 0.5 * g["trace_term"])


def test_exact_gradient_matches_fd_of_mll(oracle):  # test_outer_loop.cpp:21-48 (constrained space)
    n, d = 40, 2
    X, y = gp_problem(n, d, 401)
    c = np.array([0.8, 0.9, 1.2, 0.4])
    raw = oracle.raw_from_constrained(c)
    _, grad = oracle.exact(X, y, raw)
    eps = 1e-5
    for k in range(d + 2):
        up, dn = raw.copy(), raw.copy()
        up[k] += eps
        dn[k] -= eps
        fd = (oracle.exact(X, y, up)[0] - oracle.exact(X, y, dn)[0]) / (2 * eps)
        assert abs(grad[k] * oracle.sigmoid(raw[k]) - fd) <= 1e-5 * max(1, abs(fd))


# ---- test_rff.cpp --------------------------------------------------------
def test_rff_basis_deterministic(oracle):  # test_rff.cpp:12-19
    a = oracle.rff_basis(3, 64, 4, 99)
    b = oracle.rff_basis(3, 64, 4, 99)
    c = oracle.rff_basis(3, 64, 4, 100)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and not np.array_equal(a[0], c[0])


def test_rff_feature_norm_is_signal_variance(oracle):  # test_rff.cpp:21-32
    raw = default_test_raw(2, oracle)
    pts = np.array([[0.0, 0.0], [1.5, -2.0], [0.3, 0.3], [-4.0, 1.0]])
    phi = oracle.rff_features(2, 128, 1, 7, raw, pts)
    s2 = oracle.softplus(raw[-2]) ** 2
    assert np.allclose((phi ** 2).sum(1), s2, rtol=1e-12)


def test_rff_lengthscale_scaling_equivalence(oracle):  # test_rff.cpp:112-131
    c = np.array([0.9, 1.1, 0.2])
    raw = oracle.raw_from_constrained(c)
    c2 = c.copy()
    c2[0] *= 3.0
    raw2 = oracle.raw_from_constrained(c2)
    pts = np.array([[-1.0], [0.2], [0.8], [2.5]])
    a = oracle.rff_features(1, 256, 1, 11, raw, pts)
    b = oracle.rff_features(1, 256, 1, 11, raw2, 3.0 * pts)
    assert np.max(np.abs(a - b)) <= 1e-12


def test_pathwise_targets_construction(oracle):  # test_rff.cpp:133-167
    n, s = 30, 6
    X, _ = gp_problem(n, 2, 61)
    c = np.array([0.8, 0.9, 1.2, 0.4])
    raw = oracle.raw_from_constrained(c)
    a = oracle.pathwise_targets(X, raw, 128, s, s, 17)
    b = oracle.pathwise_targets(X, raw, 128, s, s, 17)
    assert np.array_equal(a["xi"], b["xi"])
    assert np.array_equal(a["xi"], a["prior_values"] + oracle.softplus(raw[-1]) * a["noise"])
    c2 = c.copy()
    c2[3] = 0.9
    d2 = oracle.pathwise_targets(X, oracle.raw_from_constrained(c2), 128, s, s, 17)
    assert np.array_equal(d2["prior_values"], a["prior_values"]) and np.array_equal(d2["noise"], a["noise"])


# ---- test_outer_loop.cpp ---------------------------------------------------
def test_optimise_reproducible(oracle):  # test_outer_loop.cpp:59-81
    X, y = gp_problem(60, 2, 405)
    cfg = oracle.outer_config(estimator=1, warm_start=True, steps=5, probe_count=8, rff_pairs=64,
                              solver=oracle.solver_config(kind=0, tolerance=1e-6, max_epochs=100,
                                                          preconditioner_rank=20))
    a = oracle.optimise(X, y, cfg)
    b = oracle.optimise(X, y, cfg)
    assert np.array_equal(a["final_raw"], b["final_raw"])
    assert np.array_equal(a["constrained"], b["constrained"])


def test_optimise_divergence_policy(oracle):  # test_outer_loop.cpp:149-169
    X, y = gp_problem(60, 1, 413)
    cfg = oracle.outer_config(estimator=0, steps=3, probe_count=4,
                              solver=oracle.solver_config(kind=2, batch_size=15, learning_rate=1e8, max_epochs=20))
    r = oracle.optimise(X, y, cfg)
    assert not r["aborted"] and r["solver_diverged"][0]
    assert np.array_equal(r["constrained"][1], r["constrained"][0])
    cfg.divergence_policy = 1
    r2 = oracle.optimise(X, y, cfg)
    assert r2["aborted"] and len(r2["constrained"]) == 1


def test_sinsum_generator_standardised(oracle):
    X, y = oracle.sinsum_dataset(4096, 8, seed=0)
    assert X.dtype == np.float32 and y.dtype == np.float32
    assert abs(float(y.astype(np.float64).mean())) < 1e-6 and abs(float(y.astype(np.float64).std()) - 1) < 1e-5
    assert np.allclose(X.astype(np.float64).mean(0), 0, atol=1e-6)
    X2, _ = oracle.sinsum_dataset(4096, 8, seed=0)
    assert np.array_equal(X, X2)


def test_exact_dense_prior_restates_jittered_cholesky(oracle):  # outer_loop.cpp:140-153, exact.cpp:52-61
    """ExactDense prior = L W, L the first successful Cholesky of
    dense(H) - s2 I + jitter mean(diag) I (jitter 1e-10 ...), W from stream 8."""
    rng = np.random.default_rng(21)
    n, d, s = 150, 3, 5
    X = rng.standard_normal((n, d))
    raw = oracle.raw_from_constrained([0.8, 1.2, 1.0, 1.3, 0.2])
    got = oracle.exact_prior(X, raw, s, seed=3, substream=0)
    K = oracle.dense(X, raw)
    sig2 = oracle.softplus(raw[-1]) ** 2
    K[np.diag_indices(n)] -= sig2
    md = np.mean(np.diag(K))
    L = None
    for jit in (1e-10, 1e-9, 1e-8, 1e-7, 1e-6):
        try:
            L = np.linalg.cholesky(K + jit * md * np.eye(n))
            break
        except np.linalg.LinAlgError:
            continue
    W = oracle.stream_draw(3, 8, 0, "gaussian", n * s).reshape((n, s), order="F")
    ref = L @ W
    assert np.max(np.abs(got - ref)) <= 1e-9 * np.max(np.abs(ref))


def test_optimise_exact_dense_prior_mode(oracle):
    X, y = gp_problem(120, 2, 433)
    cfg = oracle.outer_config(estimator=1, warm_start=True, steps=3, probe_count=4, rff_pairs=16,
                              solver=oracle.solver_config(kind=0, tolerance=1e-3, max_epochs=100), prior_mode=1,
                              feature_seed=5)
    r = oracle.optimise(X, y, cfg)
    assert len(r["constrained"]) == 3 and np.all(np.isfinite(r["constrained"]))
    r2 = oracle.optimise(X, y, cfg)
    assert np.array_equal(r["constrained"], r2["constrained"])  # deterministic
    cfg.prior_mode = 0
    r3 = oracle.optimise(X, y, cfg)
    assert not np.array_equal(r["gradient"][0], r3["gradient"][0])  # a different prior


def test_init_heuristic_falls_back_to_whole_dataset(oracle):  # test_outer_loop.cpp:170-178
    X, y = gp_problem(40, 1, 415)
    _, raw = oracle.optimise_exact(X, y, 30, 0.1)
    direct = np.array([oracle.softplus(r) for r in raw])
    averaged = oracle.init_heuristic(X, y, 1, 40, 7, 30, 0.1)
    assert np.max(np.abs(averaged - direct)) <= 1e-12


def test_init_heuristic_averages_per_cluster_optima(oracle):  # test_outer_loop.cpp:180-211
    per = 60
    rng = np.random.default_rng(417)

    def cluster(center, ls, seed):
        Xc, _ = gp_problem(per, 1, seed)
        Xc = Xc * ls + center  # lengthscale-like spread, far-apart centres
        yc = np.sin(Xc[:, 0] / ls) + 0.1 * rng.standard_normal(per)
        return Xc, yc

    XL, yL = cluster(0.0, 0.4, 7)
    XR, yR = cluster(40.0, 2.5, 4007)
    X = np.vstack([XL, XR])
    y = np.concatenate([yL, yR])
    lsL = oracle.softplus(oracle.optimise_exact(XL, yL, 60, 0.1)[1][0])
    lsR = oracle.softplus(oracle.optimise_exact(XR, yR, 60, 0.1)[1][0])
    ls = oracle.init_heuristic(X, y, 6, per, 11, 60, 0.1)[0]
    assert min(lsL, lsR) - 1e-9 <= ls <= max(lsL, lsR) + 1e-9


def test_optimise_exact_trajectory_starts_at_init(oracle):
    X, y = gp_problem(50, 2, 419)
    traj, raw = oracle.optimise_exact(X, y, 5, 0.1)
    assert np.allclose(traj[0], 1.0)
    assert traj.shape == (5, 4) and np.all(np.isfinite(raw))
