"""Host-side checks of the block-substitution path (no GPU): the n_p == n_c precondition
raises before any device work (reference test_sensitivity.py:316-321), the method registry
names the reference's methods, and the saddle form of an unsymmetric matrix is exact."""
import numpy as np
import pytest


class _NonSquare:
    n_x, n_p, n_c = 2, 1, 2


def test_block_solve_rejects_non_square():
    from paper_2107_03285_b200 import CscMatrix, solve_block_gn
    from paper_2107_03285_b200.errors import NonSquareParamJacobian
    with pytest.raises(NonSquareParamJacobian):
        solve_block_gn(_NonSquare(), np.zeros(2), np.zeros(1), CscMatrix.identity(2))


def test_methods_registry():
    from paper_2107_03285_b200.optimize import _DIRECTION_FUNCS, METHODS
    for m in ("sgn", "dgn", "bgn", "cg_gn", "gd"):
        assert m in METHODS and m in _DIRECTION_FUNCS
    assert "lbfgs" in METHODS and "lbfgs_sgn" in METHODS


def test_saddle_form():
    import scipy.sparse as sp
    from paper_2107_03285_b200 import CscMatrix
    from paper_2107_03285_b200.linear_solvers import _augmented, _is_symmetric
    rng = np.random.default_rng(0)
    a = (sp.random(20, 20, density=0.2, random_state=rng) + sp.eye(20)).tocsc()
    m = CscMatrix.from_scipy(a)
    assert not _is_symmetric(m)
    aug = _augmented(m).to_scipy().toarray()
    assert _is_symmetric(_augmented(m))
    np.testing.assert_array_equal(aug[20:, :20], a.toarray())
    np.testing.assert_array_equal(aug[:20, 20:], a.toarray().T)
    assert not aug[:20, :20].any() and not aug[20:, 20:].any()
    assert _is_symmetric(CscMatrix.from_scipy((a + a.T).tocsc()))
