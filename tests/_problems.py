"""Shared test problem generators (imported by tests as `_problems`)."""
import numpy as np


def gp_problem(n, d, seed, noise=0.4, lengthscale=1.0):
    """Seeded GP-like test problem: N(0,I) inputs, smooth targets + noise."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d))
    w = rng.standard_normal((d, 3)) / np.sqrt(d)
    y = np.sin(X @ w).sum(1) + noise * rng.standard_normal(n)
    return np.asfortranarray(X), y


def default_test_raw(d, oracle):
    """proj/tests/support/test_problems.hpp:31-37: l_i = 0.8+0.1 i, s = 1.2, sigma = 0.4."""
    c = [0.8 + 0.1 * i for i in range(d)] + [1.2, 0.4]
    return oracle.raw_from_constrained(c)
