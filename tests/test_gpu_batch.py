"""Batched instances (BASELINE config 5 machinery) on one device.

Every kernel processes instance b identically whatever the batch size, so batched results
must equal single-instance results bitwise; directions must match the CPU oracle to 1e-8.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def test_batched_sheet_matches_single_instances_and_oracle(cuda):
    from oracle import sgn_cpu
    from oracle.configs import oracle_sheet
    from paper_2107_03285_b200 import OptimizerConfig, direction_sgn
    from paper_2107_03285_b200.problems import BatchedDesign, build_sheet, sheet_spec
    inst = [1, 2, 3]
    specs = [sheet_spec(1, 0, k) for k in inst]
    bd = BatchedDesign(specs)
    X, status = bd.simulate(bd.p0)
    assert np.all(status == 1)
    bd.load(X, bd.p0)
    res, its = bd.directions()
    sol = bd.engine.sol.cpu().numpy()
    n_x, n_p = bd.n_x, bd.n_p
    for b, k in enumerate(inst):
        prob, p0 = build_sheet(1, 0, k)
        np.testing.assert_array_equal(p0, bd.p0[b])
        x1 = prob.simulate(p0)
        np.testing.assert_array_equal(x1, X[b])                     # batched == single, bitwise
        sd = direction_sgn(prob, x1, p0, OptimizerConfig())
        np.testing.assert_array_equal(sd.dp, sol[b, n_x:n_x + n_p])
        oprob, _ = oracle_sheet(1, 0, k)
        ref = sgn_cpu.direction_sgn(oprob, x1, p0)
        assert _rel(sd.dp, ref.dp) <= 1e-8
    assert np.all(res <= 1e-10)


def test_batched_c2_instances_shape_and_residual(cuda):
    from paper_2107_03285_b200.problems import build_sheet_batch
    bd = build_sheet_batch(2, 0, instances=[1, 2])
    X, status = bd.simulate(bd.p0)
    assert np.all(status == 1)
    bd.load(X, bd.p0)
    res, its = bd.directions()
    assert np.all(res <= 1e-10)
    assert bd.engine.sol.shape == (2, 2 * bd.n_x + bd.n_p)


def test_wide_batch_paths_match_single_instances(cuda):
    """Batches of >= 8 take runs of 4 instances per factorization grab and the 4-CTA/SM
    solve kernel; results stay bitwise equal to single-instance runs."""
    from paper_2107_03285_b200 import OptimizerConfig, direction_sgn
    from paper_2107_03285_b200.problems import BatchedDesign, build_sheet, sheet_spec
    inst = list(range(1, 9))
    bd = BatchedDesign([sheet_spec(1, 0, k) for k in inst])
    X, status = bd.simulate(bd.p0)
    assert np.all(status == 1)
    bd.load(X, bd.p0)
    res, its = bd.directions()
    assert np.all(res <= 1e-10)
    sol = bd.engine.sol.cpu().numpy()
    n_x, n_p = bd.n_x, bd.n_p
    for b in (0, 4, 7):
        prob, p0 = build_sheet(1, 0, inst[b])
        x1 = prob.simulate(p0)
        np.testing.assert_array_equal(x1, X[b])
        sd = direction_sgn(prob, x1, p0, OptimizerConfig())
        np.testing.assert_array_equal(sd.dp, sol[b, n_x:n_x + n_p])
