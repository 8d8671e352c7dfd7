"""Block-substitution Gauss-Newton (reference optimize.py:201-209,
sensitivity.py:269-284) and the unsymmetric sparse solve it needs, against the reference's
own outputs (tests/golden/ref_bgn.npz, written by make_golden_formats.py).

Reference tests mirrored: test_sensitivity.py:324-333 and test_optimizers.py:112-119 (BGN =
SGN to 1e-8 on the spring bar 6x3, w_reg 0), test_acceptance.py:57-62 (criterion 2)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
SIZES = [(6, 3), (11, 3)]


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(os.path.join(GOLD, "ref_bgn.npz")))


@pytest.mark.parametrize("nw,nh", SIZES)
def test_unsymmetric_factor_matches_reference(cuda, gold, nw, nh):
    """dc/dp is square and unsymmetric: the device factors its saddle form and matches the
    reference's SuperLU solves, plain and transposed."""
    from paper_2107_03285_b200 import CscMatrix, factor_sparse
    k = f"{nw}x{nh}"
    n = gold[f"gp_indptr_{k}"].size - 1
    gp = CscMatrix(n, n, gold[f"gp_indptr_{k}"], gold[f"gp_indices_{k}"], gold[f"gp_data_{k}"])
    fac = factor_sparse(gp)
    rhs = gold[f"gp_rhs_{k}"]
    x = fac.solve(rhs)
    xt = fac.solve(rhs, transpose=True)
    assert _rel(x, gold[f"gp_sol_{k}"]) <= 1e-10
    assert _rel(xt, gold[f"gp_solT_{k}"]) <= 1e-10
    a = gp.to_scipy()
    assert np.linalg.norm(a @ x - rhs) <= 1e-11 * np.linalg.norm(rhs)
    assert np.linalg.norm(a.T @ xt - rhs) <= 1e-11 * np.linalg.norm(rhs)
    # several right-hand sides at once (columns)
    both = fac.solve(np.stack([rhs, 2.0 * rhs], axis=1))
    np.testing.assert_allclose(both[:, 1], 2.0 * both[:, 0], rtol=1e-10, atol=1e-14 * np.abs(x).max())
    assert fac.fill_nnz > 0


def test_unsymmetric_random(cuda):
    """A random diagonally-weighted unsymmetric sparse matrix vs a dense solve."""
    import scipy.sparse as sp
    from paper_2107_03285_b200 import CscMatrix, factor_sparse
    rng = np.random.default_rng(3)
    n = 300
    a = sp.random(n, n, density=0.02, random_state=rng, format="csc") + sp.diags(2.0 + rng.random(n))
    a = a.tocsc()
    m = CscMatrix.from_scipy(a)
    b = rng.standard_normal(n)
    x = factor_sparse(m).solve(b)
    ref = np.linalg.solve(a.toarray(), b)
    assert _rel(x, ref) <= 1e-10


@pytest.mark.parametrize("nw,nh", SIZES)
def test_bgn_matches_reference(cuda, gold, nw, nh):
    from paper_2107_03285_b200 import OptimizerConfig, direction_bgn, direction_sgn
    from paper_2107_03285_b200.problems import build_spring_bar
    k = f"{nw}x{nh}"
    prob = build_spring_bar(nw, nh, w_reg=0.0)
    x, p = gold[f"x_{k}"], gold[f"p_{k}"]
    d_b = direction_bgn(prob, x, p, OptimizerConfig())
    assert _rel(d_b.dp, gold[f"dp_bgn_{k}"]) <= 1e-8
    # BGN = SGN (reference test_optimizers.py:112-119)
    d_s = direction_sgn(prob, x, p, OptimizerConfig())
    assert _rel(d_b.dp, d_s.dp) <= 1e-8
    assert _rel(d_s.dp, gold[f"dp_sgn_{k}"]) <= 1e-8


def test_bgn_minimize_trajectory(cuda, gold):
    from paper_2107_03285_b200 import OptimizerConfig, minimize
    from paper_2107_03285_b200.problems import build_spring_bar
    prob = build_spring_bar(6, 3, w_reg=0.0)
    ref = gold["traj_bgn_f"]
    run = minimize(prob, prob.default_parameters(),
                   OptimizerConfig(method="bgn", max_iterations=len(ref) - 1, gradient_tolerance=1e-12))
    f = run.f_values()
    assert len(f) == len(ref)
    np.testing.assert_allclose(f, ref, rtol=1e-7, atol=1e-14 * ref[0])


def test_gd_direction_is_negative_gradient(cuda):
    from paper_2107_03285_b200 import OptimizerConfig, direction_gd
    from paper_2107_03285_b200.problems import build_spring_bar
    g = dict(np.load(os.path.join(GOLD, "spring_bar_5x3.npz")))
    prob = build_spring_bar(5, 3)
    sd = direction_gd(prob, g["x"], g["p"], OptimizerConfig())
    assert _rel(sd.dp, -g["grad"]) <= 1e-10
