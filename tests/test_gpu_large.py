"""BASELINE configs 2 and 3 at full size against the reference solver's own outputs
(tests/golden/large_c{2,3}.npz: the oracle problems driven through the unmodified reference
direction_sgn / adjoint_gradient / minimize by tests/golden/make_golden_large.py).

The reference's minimize raises NoConvergence once a direction's refinement stalls above
1e-10 (optimize.py:389 -> linear_solvers.py:168); the goldens hold the iterations it
completed, and the device run is compared over exactly those."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def _problem(config):
    if config == 2:
        from paper_2107_03285_b200.problems import build_sheet
        return build_sheet(2)
    from paper_2107_03285_b200.problems import build_beam
    prob, p0, _ = build_beam(0)
    return prob, p0


@pytest.mark.parametrize("config,dp_tol", [(2, 1e-8), (3, 2e-6)])
def test_full_size_direction_matches_reference(cuda, config, dp_tol):
    """dp tolerance: config 2 at the north-star 1e-8.  Config 3's dp is defined only to
    ~1e-7 by ANY solver meeting the 1e-10 residual contract: the reference's own SGN and
    DGN directions differ by 6.9e-7 on this point, and its refinement floors at 1.8e-12
    (SGN at 1e-11 is still 1.1e-7 from DGN): 1881 parameters against 363 target dofs leave
    a reduced Hessian whose null space is held only by the 1e-6 |p|^2 regularizer
    (DESIGN.md section 7)."""
    from paper_2107_03285_b200 import OptimizerConfig, adjoint_gradient, direction_sgn
    gold = np.load(os.path.join(GOLDEN, f"large_c{config}.npz"))
    prob, p0 = _problem(config)
    np.testing.assert_array_equal(p0, gold["p"])
    x = prob.simulate(p0)
    assert _rel(x, gold["x"]) <= 1e-9
    xg = gold["x"]
    assert _rel(adjoint_gradient(prob, xg, p0), gold["grad"]) <= 1e-9
    assert abs(prob.objective(xg, p0) - float(gold["f0"])) <= 1e-12 * abs(float(gold["f0"]))
    sd = direction_sgn(prob, xg, p0, OptimizerConfig())
    assert sd.relative_residual <= 1e-10
    assert _rel(sd.dp, gold["dp"]) <= dp_tol


@pytest.mark.parametrize("config", [2, 3])
def test_full_size_trajectory_matches_reference(cuda, config):
    from paper_2107_03285_b200 import OptimizerConfig, minimize
    gold = np.load(os.path.join(GOLDEN, f"large_c{config}.npz"))
    ref_f = gold["traj_f"]
    prob, p0 = _problem(config)
    prob._x_warm = None
    cfg = OptimizerConfig(max_iterations=len(ref_f) - 1, gradient_tolerance=1e-12)
    run = minimize(prob, p0, cfg)
    f = run.f_values()
    assert f.size == ref_f.size, (f.size, ref_f.size, run.termination)
    # config 3: dp is defined only to ~1e-7 (test above), which the line search turns into
    # ~2e-6 on f near the end (measured 1.9e-6 at iteration 9 of 11)
    rtol = 1e-8 if config == 2 else 5e-6
    np.testing.assert_allclose(f, ref_f, rtol=rtol, atol=0)
    alpha, ref_alpha = np.array([r.step_length for r in run.records]), gold["traj_alpha"]
    if config == 2:
        np.testing.assert_array_equal(alpha, ref_alpha)
    else:
        # the same ~1e-7 dp ambiguity can move an Armijo test across its threshold once
        # the decrease is small: one backtrack more or less on the final iteration only
        # (measured: 9.5e-7 vs 1.9e-6 at iteration 11)
        np.testing.assert_array_equal(alpha[:-1], ref_alpha[:-1])
        assert alpha[-1] / ref_alpha[-1] in (0.5, 1.0, 2.0), (alpha[-1], ref_alpha[-1])
