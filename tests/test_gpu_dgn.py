"""Dense Gauss-Newton on the device vs the reference / oracle DGN and the
SGN = DGN identity (the paper's Theorem 1; reference checks.py:71-128)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("name,nw,nh,wreg", [("spring_bar_5x3.npz", 5, 3, 0.0), ("spring_bar_16x4.npz", 16, 4, 0.0),
                                             ("spring_bar_11x3.npz", 11, 3, 0.0)])
def test_dgn_matches_reference(cuda, name, nw, nh, wreg):
    from paper_2107_03285_b200 import OptimizerConfig, direction_dgn
    from paper_2107_03285_b200.problems import build_spring_bar
    g = dict(np.load(os.path.join(GOLD, name)))
    prob = build_spring_bar(nw, nh, w_reg=wreg)
    p = g["p"]
    sd = direction_dgn(prob, g["x"], p, OptimizerConfig())
    assert _rel(sd.dp, g["dp_dgn"]) <= 1e-8
    assert sd.relative_residual <= 1e-10
    assert sd.extra["sens_matrix_s"] > 0 and "dense_factor_s" in sd.extra


def test_dgn_equals_sgn_sheet(cuda):
    """Theorem 1 on config 1: the dense and the sparse Gauss-Newton steps coincide."""
    from oracle import sgn_cpu
    from oracle.configs import oracle_sheet
    from paper_2107_03285_b200 import OptimizerConfig, adjoint_gradient, direction_dgn, direction_sgn
    from paper_2107_03285_b200.problems import build_sheet
    prob, p0 = build_sheet(1)
    x = prob.simulate(p0)
    g = adjoint_gradient(prob, x, p0)
    dgn = direction_dgn(prob, x, p0, OptimizerConfig(), grad=g)
    sgn = direction_sgn(prob, x, p0, OptimizerConfig(), grad=g)
    assert _rel(dgn.dp, sgn.dp) <= 1e-6 * (1 + 0 * np.linalg.norm(sgn.dp))
    oprob, _ = oracle_sheet(1)
    ref = sgn_cpu.direction_dgn(oprob, x, p0)
    assert _rel(dgn.dp, ref.dp) <= 1e-8


def test_dgn_minimize_trajectory(cuda):
    from paper_2107_03285_b200 import OptimizerConfig, minimize
    from paper_2107_03285_b200.problems import build_spring_bar
    g = dict(np.load(os.path.join(GOLD, "spring_bar_11x3.npz")))
    prob = build_spring_bar(11, 3)
    run = minimize(prob, prob.default_parameters(),
                   OptimizerConfig(method="dgn", max_iterations=len(g["traj_f"]) - 1, gradient_tolerance=1e-12))
    n = min(len(run.f_values()), len(g["traj_f"]))
    # SGN and DGN take the same steps (Theorem 1): the reference SGN trajectory is the target
    np.testing.assert_allclose(run.f_values()[:n], g["traj_f"][:n], rtol=1e-7, atol=1e-14 * g["traj_f"][0])


@pytest.mark.parametrize("nw,nh", [(5, 3), (11, 3)])
def test_cg_gn_matches_reference(cuda, nw, nh):
    """Matrix-free CG on the reduced GN operator (reference optimize.py:212-232) with device
    operator applications: at cg_eta 1e-10 it reproduces the reference dp; at the default
    1e-3 both stop at the same tolerance (same iterates up to rounding)."""
    from paper_2107_03285_b200 import OptimizerConfig, direction_cg_gn
    from paper_2107_03285_b200.problems import build_spring_bar
    g = dict(np.load(os.path.join(GOLD, "ref_cg_gn.npz")))
    prob = build_spring_bar(nw, nh)
    x, p, grad = g[f"x_{nw}x{nh}"], g[f"p_{nw}x{nh}"], g[f"g_{nw}x{nh}"]
    tight = direction_cg_gn(prob, x, p, OptimizerConfig(cg_eta=1e-10), grad=grad)
    assert tight.relative_residual <= 1e-10
    assert _rel(tight.dp, g[f"dp_{nw}x{nh}_1e-10"]) <= 1e-8
    loose = direction_cg_gn(prob, x, p, OptimizerConfig(), grad=grad)
    assert loose.relative_residual <= 1e-3
    assert _rel(loose.dp, g[f"dp_{nw}x{nh}_0.001"]) <= 1e-6
