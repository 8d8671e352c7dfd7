"""CPU restatement of the reference SGN solver path (oracle; test infrastructure only).

Each function restates one reference routine (reference = /root/reference/pkg/src/sgnopt)
on SciPy/NumPy, the same third-party numerics the reference uses (scipy SuperLU via
``splu`` with its default COLAMD ordering; sparsetools products).  Problems follow the
reference contract (sensitivity.py:29-120) and return matrices as ``Csc`` below, which
duck-types the reference's ``CscMatrix`` (``rows``/``cols``/``shape``/``indptr``/
``indices``/``data``/``to_scipy``/``to_dense``) so the same problem objects also run
through the real reference solver in tests/golden/make_golden.py.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


class OracleSingular(Exception):
    def __init__(self, msg, pivot_index=-1):
        super().__init__(msg)
        self.pivot_index = pivot_index


class OracleNoConvergence(Exception):
    def __init__(self, msg, residual=float("nan"), iterations=0, best=None):
        super().__init__(msg)
        self.residual, self.iterations, self.best = residual, iterations, best


class Csc:
    """Minimal CSC container with the reference CscMatrix interface (sparse.py:63-135)."""

    def __init__(self, m):
        m = sp.csc_matrix(m, copy=True)
        m.sum_duplicates()
        m.sort_indices()
        self._m = m
        self.rows, self.cols = m.shape
        self.indptr = m.indptr.astype(np.int64)
        self.indices = m.indices.astype(np.int64)
        self.data = m.data

    shape = property(lambda self: (self.rows, self.cols))
    nnz = property(lambda self: int(self.indptr[-1]))

    def to_scipy(self):
        return self._m

    def to_dense(self):
        return self._m.toarray()

    def transpose(self):
        return Csc(self._m.T)

    def diagonal(self):
        return self._m.diagonal()


def csc_structural(rows, cols, vals, shape) -> Csc:
    """Triplets -> CSC with duplicates summed and stored zeros kept (sparse.py:138-146)."""
    return Csc(sp.coo_matrix((vals, (rows, cols)), shape=shape).tocsc())


# -- sparse.py:165-194 ---------------------------------------------------------------
def stack_kkt(A, B, C, Gx, Gp) -> Csc:
    n_x, n_p = A.rows, C.rows
    assert Gx.rows == n_x, "need n_c == n_x"
    K = sp.bmat([[A.to_scipy(), B.to_scipy().T, Gx.to_scipy().T],
                 [B.to_scipy(), C.to_scipy(), Gp.to_scipy().T],
                 [Gx.to_scipy(), Gp.to_scipy(), None]], format="csc")
    return Csc(K)


# -- linear_solvers.py:61-102 ----------------------------------------------------------
class LuFactor:
    def __init__(self, m):
        a = m.to_scipy() if hasattr(m, "to_scipy") else sp.csc_matrix(m)
        n = a.shape[0]
        cnt = np.diff(a.indptr)
        if np.any(cnt == 0):
            j = int(np.flatnonzero(cnt == 0)[0])
            raise OracleSingular(f"empty column {j}", j)
        present = np.zeros(n, bool)
        present[a.indices] = True
        if not present.all():
            r = int(np.flatnonzero(~present)[0])
            raise OracleSingular(f"empty row {r}", r)
        try:
            self._lu = spla.splu(sp.csc_matrix(a))
        except RuntimeError as exc:
            raise OracleSingular(str(exc)) from exc
        self.n = n
        self.fill_nnz = int(self._lu.nnz) - n

    def solve(self, b, transpose=False):
        return self._lu.solve(np.asarray(b, dtype=np.float64), trans="T" if transpose else "N")


# -- linear_solvers.py:105-127 ---------------------------------------------------------
def rel_residual(a, x, b, bnorm):
    return 0.0 if bnorm == 0.0 else float(np.linalg.norm(b - a @ x) / bnorm)


def stabilized(K: Csc, n_x, n_p, n_c, eps_x, eps_l) -> Csc:
    if eps_x == 0.0 and eps_l == 0.0:
        return K
    d = np.concatenate([np.full(n_x, eps_x), np.zeros(n_p), np.full(n_c, -eps_l)])
    return Csc(K.to_scipy() + sp.diags(d, format="csc"))


@dataclass
class Stab:
    eps_x: float = 1e-6
    eps_lambda: float = 1e-6
    refine_tolerance: float = 1e-10
    max_refine_iters: int = 50


# -- linear_solvers.py:178-211 ---------------------------------------------------------
def bicgstab_refine(a, b, x0, M: LuFactor, tol, max_iters):
    bnorm = float(np.linalg.norm(b))
    x = x0.copy()
    r = M.solve(b - a @ x)
    rh = r.copy()
    rho = alpha = omega = 1.0
    v = np.zeros_like(b)
    p = np.zeros_like(b)
    best_x, best_res = x.copy(), rel_residual(a, x, b, bnorm)
    for it in range(1, max_iters + 1):
        rho_new = float(rh @ r)
        if rho_new == 0.0 or omega == 0.0:
            return best_x, best_res, it - 1
        beta = (rho_new / rho) * (alpha / omega)
        rho = rho_new
        p = r + beta * (p - omega * v)
        v = M.solve(a @ p)
        den = float(rh @ v)
        if den == 0.0:
            return best_x, best_res, it - 1
        alpha = rho / den
        s = r - alpha * v
        t = M.solve(a @ s)
        tt = float(t @ t)
        omega = float(t @ s) / tt if tt > 0.0 else 0.0
        x = x + alpha * p + omega * s
        r = s - omega * t
        res = rel_residual(a, x, b, bnorm)
        if res < best_res:
            best_x, best_res = x.copy(), res
        if res <= tol:
            return x, res, it
    return best_x, best_res, max_iters


# -- linear_solvers.py:130-175 ---------------------------------------------------------
def solve_kkt_stabilized(K: Csc, n_x, n_p, n_c, rhs, cfg: Stab = Stab()):
    dim = 2 * n_x + n_p
    rhs = np.asarray(rhs, dtype=np.float64)
    assert K.rows == dim and rhs.shape == (dim,)
    a = K.to_scipy()
    t0 = time.perf_counter()
    M = LuFactor(stabilized(K, n_x, n_p, n_c, cfg.eps_x, cfg.eps_lambda))
    t_f = time.perf_counter() - t0
    t1 = time.perf_counter()
    bnorm = float(np.linalg.norm(rhs))
    if bnorm == 0.0:
        return np.zeros(dim), dict(res=0.0, iters=0, factor_s=t_f, solve_s=time.perf_counter() - t1)
    x = M.solve(rhs)
    res = rel_residual(a, x, rhs, bnorm)
    iters = 0
    if res > cfg.refine_tolerance:
        x, res, iters = bicgstab_refine(a, rhs, x, M, cfg.refine_tolerance, cfg.max_refine_iters)
        if res > cfg.refine_tolerance:
            raise OracleNoConvergence(f"stalled at {res:.3e}", res, iters, x)
    return x, dict(res=res, iters=iters, factor_s=t_f, solve_s=time.perf_counter() - t1)


# -- sensitivity.py:83-93, 181-216, 245-266 ----------------------------------------------
def objective(prob, x, p):
    r = prob.residuals(x, p)
    return float(0.5 * prob.weights() @ (r * r))


def objective_grads(prob, x, p):
    wr = prob.weights() * prob.residuals(x, p)
    return (prob.residual_jac_x(x, p).to_scipy().T @ wr,
            prob.residual_jac_p(x, p).to_scipy().T @ wr)


def adjoint_gradient(prob, x, p, factor: LuFactor | None = None):
    Gx = prob.constraint_jac_x(x, p)
    if factor is None:
        factor = LuFactor(Gx)
    fx, fp = objective_grads(prob, x, p)
    lam = -factor.solve(fx, transpose=True)
    return fp + prob.constraint_jac_p(x, p).to_scipy().T @ lam


def gn_blocks(prob, x, p):
    w = sp.diags(prob.weights(), format="csc")
    jx = prob.residual_jac_x(x, p).to_scipy()
    jp = prob.residual_jac_p(x, p).to_scipy()
    wjx = w @ jx
    sym = lambda m: Csc((m + m.T) * 0.5)
    return sym(jx.T @ wjx), Csc(jp.T @ wjx), sym(jp.T @ (w @ jp))


def assemble_sgn(prob, x, p):
    """(K, rhs) of the SGN saddle point at (x, p) (sensitivity.py:245-266)."""
    A, B, C = gn_blocks(prob, x, p)
    Gx = prob.constraint_jac_x(x, p)
    Gp = prob.constraint_jac_p(x, p)
    g = adjoint_gradient(prob, x, p, LuFactor(Gx))
    K = stack_kkt(A, B, C, Gx, Gp)
    n_x, n_p = Gx.cols, Gp.cols
    rhs = np.zeros(2 * n_x + n_p)
    rhs[n_x:n_x + n_p] = -g
    return K, rhs, g


@dataclass
class Direction:
    dp: np.ndarray
    dx: np.ndarray | None = None
    dlam: np.ndarray | None = None
    res: float = float("nan")
    iters: int = 0
    timings: dict = field(default_factory=dict)


# -- optimize.py:155-165 ---------------------------------------------------------------
def direction_sgn(prob, x, p, cfg: Stab = Stab()) -> Direction:
    t0 = time.perf_counter()
    K, rhs, _ = assemble_sgn(prob, x, p)
    t_a = time.perf_counter() - t0
    n_x, n_p = prob.n_x, prob.n_p
    sol, rep = solve_kkt_stabilized(K, n_x, n_p, n_x, rhs, cfg)
    return Direction(sol[n_x:n_x + n_p], sol[:n_x], sol[n_x + n_p:], rep["res"], rep["iters"],
                     dict(assemble_s=t_a, factor_s=rep["factor_s"], solve_s=rep["solve_s"]))


# -- optimize.py:168-198 + sensitivity.py:167-178, 232-242 -----------------------------
def direction_dgn(prob, x, p) -> Direction:
    Gx = prob.constraint_jac_x(x, p)
    F = LuFactor(Gx)
    S = -F.solve(prob.constraint_jac_p(x, p).to_dense())
    A, B, C = gn_blocks(prob, x, p)
    bs = B.to_scipy() @ S
    H = S.T @ (A.to_scipy() @ S) + bs + bs.T + C.to_dense()
    H = 0.5 * (H + H.T)
    g = adjoint_gradient(prob, x, p, F)
    import scipy.linalg as sla
    dp = sla.cho_solve(sla.cho_factor(H, lower=True), -g)
    return Direction(dp)


# -- forward.py:135-203 (static equilibrium Newton) -------------------------------------
def solve_static(energy, gradient, hessian, x0, tol, max_iters=200):
    """Damped Newton on the free coordinates (x0 = free-coordinate start)."""
    x = np.asarray(x0, dtype=np.float64).copy()
    for _ in range(max_iters):
        g = gradient(x)
        if np.linalg.norm(g, np.inf) <= tol:
            return x
        e0 = energy(x)
        if not (np.isfinite(e0) and np.all(np.isfinite(g))):
            # every Armijo comparison with a non-finite e0 / slope is false: the 8 escalations
            # below would all fail and raise (forward.py:155-164) -- fail now, same outcome
            raise OracleNoConvergence("static: line search failed (non-finite energy)", float("nan"))
        K = hessian(x).tocsc()
        step = _reg_newton_step(K, g)
        accepted = False
        for _ in range(8):
            alpha, x_new = _energy_backtrack(energy, x, step, g, e0)
            if alpha is not None:
                x, accepted = x_new, True
                break
            step = _reg_newton_step(K, g, bias=True)
        if not accepted:
            raise OracleNoConvergence("static: line search failed", float(np.linalg.norm(g, np.inf)))
    raise OracleNoConvergence("static: no convergence", float(np.linalg.norm(gradient(x), np.inf)), max_iters)


def _reg_newton_step(K, g, bias=False):
    n = K.shape[0]
    tau0 = 1e-6 * abs(K.diagonal().sum()) / max(n, 1) + 1e-12
    tau = tau0 * 1e6 if bias else 0.0
    for _ in range(60):
        try:
            m = K if tau == 0.0 else (K + tau * sp.identity(n, format="csc")).tocsc()
            d = LuFactor(Csc(m)).solve(-g)
            if g @ d < 0 and np.all(np.isfinite(d)):
                return d
        except OracleSingular:
            pass
        tau = tau0 if tau == 0.0 else tau * 10.0
    return -g


def _energy_backtrack(energy, x, step, g, e0, c1=1e-4, factor=0.5, max_bt=60):
    slope = float(g @ step)
    slack = 4e-15 * abs(e0)
    alpha = 1.0
    for _ in range(max_bt):
        xt = x + alpha * step
        et = energy(xt)
        if np.isfinite(et) and et <= e0 + c1 * alpha * slope + slack:
            return alpha, xt
        alpha *= factor
    return None, None


# -- optimize.py:353-420, 468-488 (SGN outer loop with Armijo backtracking) ------------
def minimize_sgn(prob, p0, max_iterations=20, gradient_tolerance=1e-12, c1=1e-4, factor=0.5,
                 max_backtracks=60, cfg: Stab = Stab()):
    p = np.asarray(p0, dtype=np.float64).copy()
    x = prob.simulate(p)
    f = objective(prob, x, p)
    g = adjoint_gradient(prob, x, p)
    fs, gn, alphas = [f], [float(np.linalg.norm(g))], [0.0]
    term = "max_iterations"
    for _ in range(max_iterations):
        if np.linalg.norm(g) <= gradient_tolerance:
            term = "gradient_tolerance"
            break
        dp = direction_sgn(prob, x, p, cfg).dp
        if np.linalg.norm(dp) == 0.0:
            term = "stationary"
            break
        if g @ dp >= 0.0:
            term = "no_descent"
            break
        alpha, ok = 1.0, False
        for _ in range(max_backtracks + 1):
            pt = p + alpha * dp
            slope = float(g @ (pt - p))
            if slope < 0.0:
                try:
                    xt = prob.simulate(pt, x_init=x)
                except (OracleNoConvergence, RuntimeError):
                    xt = None
                if xt is not None:
                    ft = objective(prob, xt, pt)
                    if np.isfinite(ft) and ft <= f + c1 * slope:
                        ok = True
                        break
            alpha *= factor
        if not ok:
            term = "line_search_failure"
            break
        p, x, f = pt, xt, ft
        g = adjoint_gradient(prob, x, p)
        fs.append(f)
        gn.append(float(np.linalg.norm(g)))
        alphas.append(alpha)
    return dict(f=np.array(fs), grad_norm=np.array(gn), alpha=np.array(alphas), p=p, x=x,
                termination=term)
