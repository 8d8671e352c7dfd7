"""Device factorization / refined KKT solve vs dense CPU references.

Mirrors the reference's solver tests (reference pkg/tests/test_linear_solvers.py:31-126)
plus larger mesh-like KKT systems that exercise multi-level trees, multi-panel fronts and
the DMMA Schur updates.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from kkt_fixtures import grid_laplacian, kkt_system

pytestmark = pytest.mark.gpu


class _K:
    def __init__(self, m, n_x, n_p):
        self.matrix, self.n_x, self.n_p, self.n_c = m, n_x, n_p, n_x


def test_factor_identity_fill_and_solve(cuda):
    from paper_2107_03285_b200 import CscMatrix, factor_sparse
    f = factor_sparse(CscMatrix.identity(10))
    assert f.fill_nnz == 10
    b = np.arange(10.0)
    np.testing.assert_array_equal(f.solve(b), b)


def test_factor_diagonal(cuda):
    from paper_2107_03285_b200 import CscMatrix, factor_sparse
    x = factor_sparse(CscMatrix.from_dense(np.diag([2.0, 4.0, 8.0]))).solve(np.array([2.0, 4.0, 8.0]))
    np.testing.assert_allclose(x, np.ones(3), rtol=0, atol=1e-15)


@pytest.mark.parametrize("n,seed", [(50, 0), (300, 1)])
def test_factor_spd_matches_dense(cuda, n, seed):
    from paper_2107_03285_b200 import CscMatrix, factor_sparse
    rng = np.random.default_rng(seed)
    a = sp.random(n, n, density=0.05, random_state=rng, data_rvs=rng.standard_normal)
    spd = (a.T @ a + sp.identity(n)).tocsc()
    b = rng.standard_normal(n)
    x = factor_sparse(CscMatrix.from_scipy(spd)).solve(b)
    expect = np.linalg.solve(spd.toarray(), b)
    assert np.linalg.norm(x - expect) <= 1e-10 * np.linalg.norm(expect)


@pytest.mark.parametrize("nx,ny", [(20, 20), (45, 40)])
def test_factor_grid_generic_mode(cuda, nx, ny):
    from paper_2107_03285_b200 import CscMatrix, factor_sparse
    g = grid_laplacian(nx, ny, 2, seed=3)
    b = np.random.default_rng(4).standard_normal(g.shape[0])
    x = factor_sparse(CscMatrix.from_scipy(g)).solve(b)
    expect = sp.linalg.spsolve(g, b)
    assert np.linalg.norm(x - expect) <= 1e-10 * np.linalg.norm(expect)


def test_structurally_singular_reports_pivot(cuda):
    from paper_2107_03285_b200 import CscMatrix, SingularMatrix, factor_sparse
    with pytest.raises(SingularMatrix) as exc:
        factor_sparse(CscMatrix.from_dense(np.diag([1.0, 0.0, 3.0])))
    assert exc.value.pivot_index == 1


def test_numerically_singular_raises(cuda):
    from paper_2107_03285_b200 import CscMatrix, SingularMatrix, factor_sparse
    m = CscMatrix.from_scipy(sp.csc_matrix(np.array([[1.0, 1.0], [1.0, 1.0]])))
    with pytest.raises(SingularMatrix):
        factor_sparse(m)


@pytest.mark.parametrize("shape", [(3, 3, 1, 2, 1e-2), (6, 5, 2, 7, 1e-2), (12, 10, 2, 9, 0.0),
                                   (30, 25, 2, 40, 1e-3), (70, 60, 2, 100, 1e-4)])
def test_kkt_refined_matches_dense(cuda, shape):
    from paper_2107_03285_b200 import CscMatrix, StabilizationConfig, solve_kkt_stabilized
    nx, ny, dof, n_p, cd = shape
    K, n_x, n_p, rhs = kkt_system(nx, ny, dof, n_p, cd, seed=sum(shape[:4]))
    sol, rep = solve_kkt_stabilized(_K(CscMatrix.from_scipy(K), n_x, n_p), rhs, StabilizationConfig())
    if K.shape[0] <= 3000:
        expect = np.linalg.solve(K.toarray(), rhs)
    else:
        expect = sp.linalg.spsolve(K.tocsc(), rhs)
    assert rep.relative_residual <= 1e-10
    assert np.linalg.norm(K @ sol - rhs) <= 1e-10 * np.linalg.norm(rhs)
    dp, dp_e = sol[n_x:n_x + n_p], expect[n_x:n_x + n_p]
    assert np.linalg.norm(dp - dp_e) <= 1e-8 * np.linalg.norm(dp_e)


def test_zero_rhs_returns_zero(cuda):
    from paper_2107_03285_b200 import CscMatrix, solve_kkt_stabilized
    K, n_x, n_p, rhs = kkt_system(5, 4, 2, 3, 1e-2)
    sol, rep = solve_kkt_stabilized(_K(CscMatrix.from_scipy(K), n_x, n_p), np.zeros_like(rhs))
    assert np.all(sol == 0.0) and rep.relative_residual == 0.0 and rep.refine_iterations == 0


def test_no_convergence_when_refinement_disabled(cuda):
    from paper_2107_03285_b200 import (CscMatrix, NoConvergence, StabilizationConfig,
                                       solve_kkt_stabilized)
    K, n_x, n_p, rhs = kkt_system(8, 7, 2, 5, 1e-2, seed=11)
    cfg = StabilizationConfig(eps_x=1e-2, eps_lambda=1e-2, max_refine_iters=0)
    with pytest.raises(NoConvergence) as exc:
        solve_kkt_stabilized(_K(CscMatrix.from_scipy(K), n_x, n_p), rhs, cfg)
    assert exc.value.best is not None and exc.value.best.shape == rhs.shape


def test_zero_stabilization_is_plain_solve(cuda):
    from paper_2107_03285_b200 import CscMatrix, StabilizationConfig, solve_kkt_stabilized
    K, n_x, n_p, rhs = kkt_system(6, 6, 2, 4, 1e-2, seed=5)
    cfg = StabilizationConfig(eps_x=0.0, eps_lambda=0.0)
    sol, rep = solve_kkt_stabilized(_K(CscMatrix.from_scipy(K), n_x, n_p), rhs, cfg)
    expect = np.linalg.solve(K.toarray(), rhs)
    assert rep.refine_iterations == 0
    np.testing.assert_allclose(sol, expect, rtol=1e-9, atol=1e-12 * np.abs(expect).max())


@pytest.mark.parametrize("n,seed", [(40, 0), (200, 3)])
def test_symmetric_indefinite_zero_diagonal(cuda, n, seed):
    """Nonsingular symmetric indefinite input with zero diagonal entries: SuperLU pivots past
    them (reference linear_solvers.py:87); the device falls back to the saddle form."""
    from paper_2107_03285_b200 import CscMatrix, factor_sparse
    rng = np.random.default_rng(seed)
    a = sp.random(n, n, density=0.08, random_state=rng, data_rvs=rng.standard_normal)
    m = (a + a.T + sp.diags(rng.standard_normal(n))).tolil()
    for i in range(0, n, 3):
        m[i, i] = 0.0                                       # zero pivots in any static order
    m = m.tocsc()
    dense = m.toarray()
    assert abs(np.linalg.det(dense)) > 0
    b = rng.standard_normal(n)
    f = factor_sparse(CscMatrix.from_scipy(m))
    x = f.solve(b)
    ref = np.linalg.solve(dense, b)
    assert np.linalg.norm(dense @ x - b) <= 1e-10 * np.linalg.norm(b)
    assert np.linalg.norm(x - ref) <= 1e-8 * np.linalg.norm(ref) * max(1.0, np.linalg.cond(dense) * 1e-6)


def test_cta_hand_over_option_keeps_the_factorization(cuda):
    """sgn_factor_set_retire: CTAs past the kept share leave at the top levels; the task
    order per tile is unchanged, so the factor and the solve are bitwise the same."""
    import torch
    from paper_2107_03285_b200.device import DeviceFactor, symbolic_for
    g = grid_laplacian(60, 50, 2, seed=5).tocsc()
    g.sort_indices()
    sym = symbolic_for(g.shape[0], g.indptr, g.indices)
    fac = DeviceFactor(sym, 1)
    vals = torch.as_tensor(g.data, dtype=torch.float64, device="cuda").reshape(1, -1)
    b = torch.as_tensor(np.random.default_rng(6).standard_normal(g.shape[0]), device="cuda").reshape(1, -1)
    x0, x1 = torch.empty_like(b), torch.empty_like(b)
    fac.numeric(vals)
    fac.check()
    fac.solve(b, x0)
    full = fac.set_grid(0)
    task = fac.set_retire(max(1, full // 4), 4)
    assert task >= 0                                   # a hand-over point exists (top levels of <= 4 fronts)
    fac.numeric(vals)
    fac.check()
    fac.solve(b, x1)
    assert fac.set_retire(0, 0) == -1
    torch.cuda.synchronize()
    assert torch.equal(x0, x1)
    expect = sp.linalg.spsolve(g, b[0].cpu().numpy())
    assert np.linalg.norm(x1[0].cpu().numpy() - expect) <= 1e-10 * np.linalg.norm(expect)
