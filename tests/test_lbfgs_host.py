"""The L-BFGS two-loop recursion (reference optimize.py:310-335) equals the explicit BFGS
inverse-Hessian recursion H+ = (I - r s y^T) H (I - r y s^T) + r s s^T from H0."""
import numpy as np

from paper_2107_03285_b200.optimize import direction_lbfgs


def _explicit(history, g, H0):
    H = H0.copy()
    n = len(g)
    for s, y, rho in history:
        V = np.eye(n) - rho * np.outer(y, s)
        H = V.T @ H @ V + rho * np.outer(s, s)
    return -H @ g


def test_two_loop_matches_explicit_bfgs():
    rng = np.random.default_rng(0)
    n = 12
    A = rng.standard_normal((n, n))
    A = A @ A.T + n * np.eye(n)                       # SPD model Hessian: s.y > 0
    hist = []
    for _ in range(5):
        s = rng.standard_normal(n)
        y = A @ s
        hist.append((s, y, 1.0 / (s @ y)))
    g = rng.standard_normal(n)
    s, y, _ = hist[-1]
    gamma = (s @ y) / (y @ y)
    np.testing.assert_allclose(direction_lbfgs(hist, g), _explicit(hist, g, gamma * np.eye(n)), rtol=1e-12, atol=1e-14)
    M = rng.standard_normal((n, n))
    M = M @ M.T + np.eye(n)
    np.testing.assert_allclose(direction_lbfgs(hist, g, lambda q: M @ q), _explicit(hist, g, M), rtol=1e-11, atol=1e-13)
    np.testing.assert_array_equal(direction_lbfgs([], g), -g)              # empty history, gamma = 1
