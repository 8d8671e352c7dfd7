"""Unrefined direct-solve residuals of the device LDL^T (pair mode) -- debugging aid."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np, torch
from kkt_fixtures import kkt_system
from paper_2107_03285_b200.linear_solvers import _DeviceSystem
from paper_2107_03285_b200.sparse import CscMatrix
from paper_2107_03285_b200.problems import build_sheet


def resid(K, n_x, n_p, rhs, eps):
    s = _DeviceSystem(CscMatrix.from_scipy(K), n_x, n_p, n_x)
    s.factorize(eps, eps)
    x = s.solve_host(rhs)
    import scipy.sparse as sp
    Ks = K + sp.diags(np.r_[np.full(n_x, eps), np.zeros(n_p), np.full(n_x, -eps)])
    return np.linalg.norm(Ks @ x - rhs) / np.linalg.norm(rhs)


for shape in [(6, 5, 2, 7, 1e-2), (30, 25, 2, 40, 1e-3), (70, 60, 2, 100, 1e-4)]:
    K, n_x, n_p, rhs = kkt_system(*shape, seed=1)
    print(shape, "eps0", resid(K, n_x, n_p, rhs, 0.0), "eps1e-6", resid(K, n_x, n_p, rhs, 1e-6))
for cfg in (1, 2):
    prob, p0 = build_sheet(cfg)
    x = prob.X0 if False else prob.plan.X0.ravel()[prob.plan.free_dofs]
    K = prob.kkt_matrix(x, p0).to_scipy()
    rhs = np.random.default_rng(0).standard_normal(K.shape[0])
    print("sheet", cfg, "eps0", resid(K, prob.n_x, prob.n_p, rhs, 0.0), "eps1e-6", resid(K, prob.n_x, prob.n_p, rhs, 1e-6))
