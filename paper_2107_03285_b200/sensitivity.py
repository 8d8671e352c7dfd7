"""Drop-in derivative machinery of the SGN path (reference sensitivity.py).

Same names and signatures as the reference (pkg/src/sgnopt/sensitivity.py):
``EquilibriumProblem`` (29-120), ``GnBlocks`` (123-137), ``KktSystem`` (140-157),
``gn_blocks`` (205-216), ``kkt_from_blocks`` (245-256), ``assemble_sgn`` (259-266),
``adjoint_gradient`` (194-198).

* GPU-native problems (``problems.ElasticDesignProblem``, carrying ``.engine``): the
  adjoint gradient comes from a device LDL^T of dc/dx (the reference's SuperLU of dc/dx,
  sensitivity.py:160-164) and one solve, g = f_p + G_p^T lambda; inside a direction it
  runs on a side stream next to the KKT factorization (``engine.sgn_solve_stages``).
* Plugin problems (user subclasses evaluated on the host): Jacobians come from the
  problem's own evaluators and the stacked KKT is solved on the device (``HostKKT``).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .errors import CapabilityMissing
from .sparse import CscMatrix, stack_kkt_blocks

__all__ = ["EquilibriumProblem", "GnBlocks", "KktSystem", "gn_blocks", "kkt_from_blocks",
           "assemble_sgn", "adjoint_gradient", "solve_block_gn"]


class EquilibriumProblem:
    """Problem contract c(x, p) = 0, n_c == n_x (sensitivity.py:29-120)."""

    n_x: int
    n_p: int

    @property
    def n_c(self) -> int:
        return self.n_x

    @property
    def name(self) -> str:
        return type(self).__name__

    def simulate(self, p, x_init=None):
        raise NotImplementedError

    def constraints(self, x, p):
        raise NotImplementedError

    def constraint_jac_x(self, x, p) -> CscMatrix:
        raise NotImplementedError

    def constraint_jac_p(self, x, p) -> CscMatrix:
        raise NotImplementedError

    def residuals(self, x, p):
        raise CapabilityMissing("residuals")

    def weights(self):
        raise CapabilityMissing("weights")

    def residual_jac_x(self, x, p) -> CscMatrix:
        raise CapabilityMissing("residual_jac_x")

    def residual_jac_p(self, x, p) -> CscMatrix:
        raise CapabilityMissing("residual_jac_p")

    def objective(self, x, p) -> float:
        r = self.residuals(x, p)
        return float(0.5 * self.weights() @ (r * r))

    def objective_grad_x(self, x, p):
        return self.residual_jac_x(x, p).to_scipy().T @ (self.weights() * self.residuals(x, p))

    def objective_grad_p(self, x, p):
        return self.residual_jac_p(x, p).to_scipy().T @ (self.weights() * self.residuals(x, p))

    def bounds(self):
        return None


@dataclass
class GnBlocks:
    """A = J_x^T W J_x, B = J_p^T W J_x, C = J_p^T W J_p (sensitivity.py:123-137)."""

    A: CscMatrix
    B: CscMatrix
    C: CscMatrix


@dataclass
class KktSystem:
    """Assembled saddle point + rhs + block sizes (sensitivity.py:140-157)."""

    matrix: CscMatrix
    rhs: np.ndarray
    n_x: int
    n_p: int
    n_c: int

    def split(self, solution):
        n_x, n_p = self.n_x, self.n_p
        return solution[:n_x], solution[n_x:n_x + n_p], solution[n_x + n_p:]


def _is_device_problem(prob) -> bool:
    return hasattr(prob, "engine") and hasattr(prob, "plan")


def _sym(m) -> CscMatrix:
    return CscMatrix.from_scipy((m + m.T) * 0.5)


def gn_blocks(prob, x, p) -> GnBlocks:
    """Weighted Gauss-Newton blocks (sensitivity.py:205-216)."""
    w = sp.diags(prob.weights(), format="csc")
    jx = prob.residual_jac_x(x, p).to_scipy()
    jp = prob.residual_jac_p(x, p).to_scipy()
    wjx = w @ jx
    return GnBlocks(A=_sym(jx.T @ wjx), B=CscMatrix.from_scipy(jp.T @ wjx), C=_sym(jp.T @ (w @ jp)))


def kkt_from_blocks(blocks: GnBlocks, dcdx: CscMatrix, dcdp: CscMatrix, grad_p) -> KktSystem:
    """Stack blocks; rhs = (0, -grad_p, 0) (sensitivity.py:245-256)."""
    matrix = stack_kkt_blocks(blocks.A, blocks.B, blocks.C, dcdx, dcdp)
    n_x, n_p, n_c = dcdx.cols, dcdp.cols, dcdx.rows
    rhs = np.zeros(2 * n_x + n_p)
    rhs[n_x:n_x + n_p] = -np.asarray(grad_p, dtype=np.float64)
    return KktSystem(matrix=matrix, rhs=rhs, n_x=n_x, n_p=n_p, n_c=n_c)


def _host_kkt(prob, x, p, blocks=None):
    """Plugin path: host-assembled KKT + device solve stages (engine.HostKKT)."""
    from .engine import HostKKT
    from .linear_solvers import StabilizationConfig
    blocks = blocks or gn_blocks(prob, x, p)
    dcdx, dcdp = prob.constraint_jac_x(x, p), prob.constraint_jac_p(x, p)
    K = stack_kkt_blocks(blocks.A, blocks.B, blocks.C, dcdx, dcdp)
    hk = HostKKT(K, dcdx.cols, dcdp.cols, StabilizationConfig())
    hk.set_fvec(prob.objective_grad_x(x, p), prob.objective_grad_p(x, p))
    return hk, K


def adjoint_gradient(prob, x, p, factor=None):
    """Total gradient df/dp by the adjoint method (sensitivity.py:194-198), on the device."""
    from .engine import adjoint_gradient_stage, sgn_solve_stages
    if _is_device_problem(prob):
        eng = prob.engine
        prob._load(x, p)
        eng.assemble()
        adjoint_gradient_stage(eng)
        return eng.grad[0].cpu().numpy()
    hk, _ = _host_kkt(prob, x, p)
    sgn_solve_stages(hk, None, need_direction=False)
    return hk.grad[0].cpu().numpy()


def assemble_sgn(prob, x, p, blocks: GnBlocks | None = None) -> KktSystem:
    """SGN saddle point at (x, p) (sensitivity.py:259-266); values assembled on the device
    for GPU-native problems, the gradient from the device adjoint solve."""
    g = adjoint_gradient(prob, x, p)
    if _is_device_problem(prob):
        K = prob.kkt_matrix(x, p)
        n_x, n_p = prob.n_x, prob.n_p
        rhs = np.zeros(2 * n_x + n_p)
        rhs[n_x:n_x + n_p] = -g
        return KktSystem(K, rhs, n_x, n_p, n_x)
    blocks = blocks or gn_blocks(prob, x, p)
    return kkt_from_blocks(blocks, prob.constraint_jac_x(x, p), prob.constraint_jac_p(x, p), g)


def solve_block_gn(prob, x, p, A: CscMatrix) -> np.ndarray:
    """Block-substitution Gauss-Newton step for B = C = 0 (sensitivity.py:269-284):
    dp = (dc/dp)^{-1} (dc/dx) A^{-1} (df/dx)^T -- two device factorizations (A symmetric
    LDL^T; the square unsymmetric dc/dp through its saddle form, ``SparseFactorization``)."""
    from .errors import NonSquareParamJacobian
    from .linear_solvers import factor_sparse
    if prob.n_p != prob.n_c:
        raise NonSquareParamJacobian(f"block solve needs n_p == n_c, got n_p={prob.n_p}, n_c={prob.n_c}")
    dy = factor_sparse(A).solve(prob.objective_grad_x(x, p))
    rhs = prob.constraint_jac_x(x, p).to_scipy() @ dy
    return factor_sparse(prob.constraint_jac_p(x, p)).solve(rhs)

