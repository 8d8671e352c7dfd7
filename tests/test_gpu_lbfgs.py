"""SGN-initialised L-BFGS on the device."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _identity(prob, p):
    from paper_2107_03285_b200 import OptimizerConfig, adjoint_gradient, direction_sgn
    from paper_2107_03285_b200.optimize import _direction_lbfgs_sgn
    cfg = OptimizerConfig()
    x = prob.simulate(p)
    g = adjoint_gradient(prob, x, p)
    a = direction_sgn(prob, x, p, cfg, grad=g).dp
    b = _direction_lbfgs_sgn(prob, x, p, cfg, g, []).dp
    return float(np.max(np.abs(a - b)))


def test_empty_history_is_sgn_bitwise_device_problems(cuda):
    """reference checks.py:213-226: worst == 0.0 (bitwise identical systems)."""
    from paper_2107_03285_b200.problems import build_sheet, build_spring_bar
    prob = build_spring_bar(5, 3)
    assert _identity(prob, prob.default_parameters()) == 0.0
    prob, p0 = build_sheet(1)
    assert _identity(prob, p0) == 0.0


def test_empty_history_is_sgn_bitwise_plugin_problem(cuda):
    from oracle.problems import SpringBarOracle
    prob = SpringBarOracle(5, 3)
    assert _identity(prob, prob.default_parameters()) == 0.0


@pytest.mark.parametrize("method", ["lbfgs_sgn", "lbfgs"])
def test_trajectory_matches_reference(cuda, method):
    from paper_2107_03285_b200 import OptimizerConfig, minimize
    from paper_2107_03285_b200.problems import build_spring_bar
    g = dict(np.load(os.path.join(GOLD, "ref_lbfgs_11x3.npz")))
    prob = build_spring_bar(11, 3)
    run = minimize(prob, prob.default_parameters(),
                   OptimizerConfig(method=method, max_iterations=6, gradient_tolerance=1e-12))
    ref_f = g[f"{method}_f"]
    n = min(len(run.f_values()), len(ref_f))
    assert n == len(ref_f)
    np.testing.assert_allclose(run.f_values()[:n], ref_f[:n], rtol=1e-8, atol=1e-14 * ref_f[0])
