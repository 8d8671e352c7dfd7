"""No kernel reads device memory it has not written in the same factorization / solve.

Every scratch buffer of a factor (fronts, solve panels Z, pivot-block scratch, solve
vectors, chunk partials) is filled with NaN before factoring; results must still match
dense references exactly as without poisoning.  Guards the class of bug where a zero
operand multiplied unwritten memory (0 x NaN = NaN) and corrupted Z only when recycled
device memory happened to hold NaN.  Sizes are chosen so pivot blocks end off the
32-grid (partial last tiles) in generic and pair mode, multi-level trees and a root front.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from kkt_fixtures import grid_laplacian, kkt_system

pytestmark = pytest.mark.gpu


def _poisoned_solve(m, b, n_x=0, n_p=0, eps=(0.0, 0.0)):
    import torch
    from paper_2107_03285_b200._lib import check, lib
    from paper_2107_03285_b200.device import DeviceFactor, symbolic_for
    from paper_2107_03285_b200.linear_solvers import _symmetric_pattern
    from paper_2107_03285_b200.sparse import CscMatrix
    M = CscMatrix.from_scipy(m.tocsc())
    indptr, indices, src = _symmetric_pattern(M)
    n = M.rows
    sym = symbolic_for(n, indptr, indices, n_x, n_p, n_x)
    fac = DeviceFactor(sym, 1)
    vals = torch.as_tensor(np.where(src >= 0, M.data[np.maximum(src, 0)], 0.0), device="cuda").reshape(1, -1)
    bt = torch.as_tensor(b, device="cuda").reshape(1, -1)
    x = torch.empty_like(bt)
    out = []
    for _ in range(2):                                   # poison, factor, solve -- twice
        check(lib().sgn_debug_poison(fac._h, float("nan")))
        fac.numeric(vals, *eps)
        fac.check()
        fac.solve(bt, x)
        torch.cuda.synchronize()
        out.append(x.cpu().numpy()[0].copy())
    np.testing.assert_array_equal(out[0], out[1])      # deterministic despite the poison
    return out[0]


@pytest.mark.parametrize("nx,ny,dof", [(19, 13, 2), (27, 11, 1), (7, 5, 2)])
def test_generic_mode_under_poison(cuda, nx, ny, dof):
    g = grid_laplacian(nx, ny, dof, seed=5)
    b = np.random.default_rng(6).standard_normal(g.shape[0])
    x = _poisoned_solve(g, b)
    expect = sp.linalg.spsolve(g.tocsc(), b)
    assert np.all(np.isfinite(x))
    assert np.linalg.norm(x - expect) <= 1e-10 * np.linalg.norm(expect)


@pytest.mark.parametrize("nx,ny,n_p", [(6, 5, 7), (13, 9, 38), (21, 17, 45)])
def test_pair_mode_under_poison(cuda, nx, ny, n_p):
    K, n_x, npar, _ = kkt_system(nx=nx, ny=ny, dof=2, n_p=n_p, seed=2)
    n = K.shape[0]
    eps = 1e-6
    shift = np.r_[np.full(n_x, eps), np.zeros(npar), np.full(n - n_x - npar, -eps)]
    Ks = (K + sp.diags(shift)).tocsc()
    b = np.random.default_rng(8).standard_normal(n)
    x = _poisoned_solve(K, b, n_x, npar, (eps, eps))
    expect = np.linalg.solve(Ks.toarray(), b)
    assert np.all(np.isfinite(x))
    assert np.linalg.norm(x - expect) <= 1e-9 * np.linalg.norm(expect)
