"""Drop-in SGN search direction and outer loop (reference optimize.py), GPU-resident.

Same names/signatures/records as the reference (pkg/src/sgnopt/optimize.py):
``OptimizerConfig`` (63-80), ``SearchDirection`` (83-98), ``IterationRecord`` /
``OptimizerRun`` (101-137), ``direction_sgn`` (155-165), ``minimize`` (353-420),
``_line_search`` (468-488), ``_DIRECTION_FUNCS`` (338-346, "sgn" entry).

For GPU-native problems one direction is: device assembly -> device LDL^T -> device
adjoint gradient -> device refined KKT solve; the forward statics of the line search
run on the device too (problems.ElasticDesignProblem.simulate).  Only scalars (f,
slopes, norms) cross to the host for the Armijo decisions.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .errors import (CapabilityMissing, ForwardSimFailure, InfeasiblePoint, NoConvergence, NotPositiveDefinite,
                     NumericalBlowup)
from .linear_solvers import StabilizationConfig, solve_kkt_stabilized
from .sensitivity import _host_kkt, _is_device_problem, adjoint_gradient, gn_blocks

__all__ = ["METHODS", "CSV_HEADER", "OptimizerConfig", "SearchDirection", "IterationRecord",
           "OptimizerRun", "direction_sgn", "minimize", "project_direction_bounds"]

METHODS = ("sgn", "dgn", "bgn", "cg_gn", "gd", "lbfgs", "lbfgs_sgn")
CSV_HEADER = "iter,f,grad_norm,step_len,dir_time_s,fwd_time_s,elapsed_s,lin_rel_residual"


@dataclass
class OptimizerConfig:
    method: str = "sgn"
    max_iterations: int = 100
    gradient_tolerance: float = 1e-5
    armijo_c1: float = 1e-4
    backtrack_factor: float = 0.5
    max_backtracks: int = 60
    lbfgs_history: int = 10
    cg_eta: float = 1e-3
    stabilization: StabilizationConfig = field(default_factory=StabilizationConfig)
    bound_mode: str = "none"

    def __post_init__(self):
        if self.gradient_tolerance <= 0:
            raise ValueError("gradient tolerance must be positive")
        if not 0.0 < self.backtrack_factor < 1.0:
            raise ValueError("backtrack factor must lie in (0, 1)")


@dataclass
class SearchDirection:
    dp: np.ndarray
    dx: np.ndarray | None = None
    dlam: np.ndarray | None = None
    assemble_s: float = 0.0
    factor_s: float = 0.0
    solve_s: float = 0.0
    relative_residual: float = float("nan")
    extra: dict = field(default_factory=dict)

    @property
    def total_s(self) -> float:
        return self.assemble_s + self.factor_s + self.solve_s


@dataclass
class IterationRecord:
    iteration: int
    f: float
    grad_norm: float
    step_length: float
    direction_time: float
    forward_time: float
    elapsed: float
    lin_rel_residual: float

    def csv_row(self) -> str:
        return (f"{self.iteration},{self.f:.17g},{self.grad_norm:.17g},{self.step_length:.17g},"
                f"{self.direction_time:.6g},{self.forward_time:.6g},{self.elapsed:.6g},"
                f"{self.lin_rel_residual:.6g}")


@dataclass
class OptimizerRun:
    method: str
    records: list
    termination: str
    p: np.ndarray
    x: np.ndarray

    def f_values(self):
        return np.array([r.f for r in self.records])

    def grad_norms(self):
        return np.array([r.grad_norm for r in self.records])

    def write_csv(self, path) -> None:
        with open(path, "w", encoding="ascii") as fh:
            fh.write(CSV_HEADER + "\n")
            for rec in self.records:
                fh.write(rec.csv_row() + "\n")


def project_direction_bounds(dp, p, lower, upper):
    if np.any(p < lower) or np.any(p > upper):
        raise InfeasiblePoint("parameters violate their declared bounds")
    out = dp.copy()
    out[(p >= upper) & (dp > 0)] = 0.0
    out[(p <= lower) & (dp < 0)] = 0.0
    return out


def direction_sgn(prob, x, p, cfg: OptimizerConfig, grad=None) -> SearchDirection:
    """Gauss-Newton step through the sparse saddle point (optimize.py:155-165) on the GPU.

    ``grad`` is ignored, as in the reference (the gradient is recomputed by the adjoint).
    """
    from .engine import sgn_solve_stages
    if _is_device_problem(prob):
        eng = prob.engine
        eng.stab = cfg.stabilization
        prob._load(x, p)
        t = {}
        res, its = eng.direction(t)
        sol = eng.solution_host(0)
    else:
        t0 = time.perf_counter()
        hk, _ = _host_kkt(prob, x, p)
        hk.stab = cfg.stabilization
        t = {}
        hk.torch.cuda.synchronize()
        a_s = time.perf_counter() - t0
        res, its = sgn_solve_stages(hk, t)
        t["assemble_s"] = a_s
        sol = hk.sol[0].cpu().numpy()
    n_x, n_p = prob.n_x, prob.n_p
    return SearchDirection(dp=sol[n_x:n_x + n_p], dx=sol[:n_x], dlam=sol[n_x + n_p:],
                           assemble_s=t.get("assemble_s", 0.0), factor_s=t.get("factor_s", 0.0),
                           solve_s=t.get("solve_s", 0.0), relative_residual=float(res[0]),
                           extra={"refine_iterations": int(its[0])})


def direction_dgn(prob, x, p, cfg: OptimizerConfig, grad=None) -> SearchDirection:
    """Gauss-Newton step through the dense reduced Hessian (reference optimize.py:168-198),
    on the device for device problems:

    * S = -G_x^{-1} G_p: the unshifted G_x factor + one multi-RHS solve with the n_p
      columns of G_p (sensitivity.py:167-178);
    * H = S^T A S + B S + (B S)^T + C, symmetrised (sensitivity.py:232-242): sparse-times-
      dense products from the KKT CSC, S^T (A S) on a DMMA GEMM;
    * dp = -H^{-1} g by the multifrontal LDL^T on the dense pattern; a non-positive pivot
      raises NotPositiveDefinite(pivot_index) like cho_factor (linear_solvers.py:214-240).

    The sensitivity-matrix time and the dense factorization time are reported separately
    (``extra``) as in the reference.
    """
    if not _is_device_problem(prob):
        raise CapabilityMissing("direction_dgn on the device needs a device problem "
                                "(problems.ElasticDesignProblem)")
    import ctypes
    from . import _lib
    from ._lib import check, lib, ptr
    from .device import DeviceFactor, symbolic_for
    eng = prob.engine
    if eng.batch != 1:
        raise CapabilityMissing("direction_dgn: one instance per engine")
    pl = prob.plan
    torch = eng.torch
    st = _lib.stream_handle()
    n_x, n_p, dim = pl.n_x, pl.n_p, pl.dim
    sync = torch.cuda.synchronize
    prob._load(x, p)
    eng.assemble()
    sync()
    t0 = time.perf_counter()
    # S = -G_x^{-1} G_p
    eng.gx_values()
    eng.gfac.numeric(eng.gvals, 0.0, 0.0, st)
    eng.gfac.check(st)
    if not hasattr(eng, "_dgn"):
        T = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.int64, device="cuda")
        E = lambda *shape: torch.empty(shape, dtype=torch.float64, device="cuda")
        dsym = symbolic_for(n_p, np.arange(0, n_p * n_p + 1, n_p, dtype=np.int64),
                            np.tile(np.arange(n_p, dtype=np.int64), n_p))
        eng._dgn = dict(kp=T(pl.K_indptr), ki=T(pl.K_indices), GP=E(n_p, n_x), S=E(n_p, n_x), AS=E(n_p, n_x),
                        STAS=E(n_p, n_p), BS=E(n_p, n_p), C=E(n_p, n_p), H=E(1, n_p * n_p), rhs=E(1, n_p),
                        dp=E(1, n_p), dsym=dsym, dfac=DeviceFactor(dsym, 1))
    d = eng._dgn
    kv = eng.kvals[0]
    check(lib().sgn_csc_block_dense(dim, ptr(d["kp"]), ptr(d["ki"]), ptr(kv), n_x + n_p, n_x, n_x, n_p,
                                    ptr(d["GP"]), st))                      # G_p, column j = RHS j
    eng.gfac.solve_multi(d["GP"], d["S"], st)
    if "neg1" not in d:
        d["neg1"] = torch.full((n_p,), -1.0, dtype=torch.float64, device="cuda")
    check(lib().sgn_axpy(n_x, n_p, ptr(d["neg1"]), ptr(d["S"]), None, ptr(d["S"]), n_x, st))   # S = -G_x^{-1} G_p
    sync()
    t_sens = time.perf_counter() - t0
    # H = S^T A S + B S + (B S)^T + C
    t1 = time.perf_counter()
    check(lib().sgn_csc_spmm(ptr(d["kp"]), ptr(d["ki"]), ptr(kv), 0, n_x, 0, n_x, ptr(d["S"]), n_x,
                             ptr(d["AS"]), n_x, n_p, st))
    check(lib().sgn_gemm_tn(ptr(d["S"]), ptr(d["AS"]), n_p, n_x, ptr(d["STAS"]), st))
    check(lib().sgn_csc_spmm(ptr(d["kp"]), ptr(d["ki"]), ptr(kv), n_x, n_p, 0, n_x, ptr(d["S"]), n_x,
                             ptr(d["BS"]), n_p, n_p, st))
    check(lib().sgn_csc_block_dense(dim, ptr(d["kp"]), ptr(d["ki"]), ptr(kv), n_x, n_p, n_x, n_p,
                                    ptr(d["C"]), st))
    check(lib().sgn_gn_hessian(ptr(d["STAS"]), ptr(d["BS"]), ptr(d["C"]), n_p, ptr(d["H"]), st))
    if grad is None:
        grad = adjoint_gradient(prob, x, p)
    grad = np.asarray(grad, dtype=np.float64)
    sync()
    assemble_s = time.perf_counter() - t1 + t_sens
    # dense factorization + positivity
    t2 = time.perf_counter()
    d["dfac"].numeric(d["H"], 0.0, 0.0, st)
    d["dfac"].check(st)
    mn, pos = ctypes.c_double(), ctypes.c_int64()
    check(lib().sgn_factor_min_pivot(d["dfac"]._h, ctypes.byref(mn), ctypes.byref(pos), st))
    if not mn.value > 0.0:
        raise NotPositiveDefinite(f"dense Gauss-Newton Hessian is not positive definite "
                                  f"(pivot {pos.value}: {mn.value:.3e})", pivot_index=int(pos.value))
    factor_s = time.perf_counter() - t2
    t3 = time.perf_counter()
    d["rhs"][0].copy_(torch.from_numpy(-grad))
    d["dfac"].solve(d["rhs"], d["dp"], False, st)
    dp = d["dp"][0].cpu().numpy()
    solve_s = time.perf_counter() - t3
    h = d["H"][0].cpu().numpy().reshape(n_p, n_p)
    gnorm = np.linalg.norm(grad)
    res = float(np.linalg.norm(h @ dp + grad) / gnorm) if gnorm > 0 else 0.0
    return SearchDirection(dp=dp, assemble_s=assemble_s, factor_s=factor_s, solve_s=solve_s,
                           relative_residual=res, extra={"sens_matrix_s": t_sens, "dense_factor_s": factor_s})


def direction_cg_gn(prob, x, p, cfg: OptimizerConfig, grad=None) -> SearchDirection:
    """Matrix-free CG on the reduced Gauss-Newton operator (reference optimize.py:212-232),
    operator applications on the device (two G_x solves each).  Negative curvature falls
    back to CG's last iterate, or steepest descent if CG has not moved, as in the reference."""
    from .linear_solvers import DeviceReducedOperator, cg_reduced
    from .errors import NegativeCurvature
    if not _is_device_problem(prob):
        raise CapabilityMissing("direction_cg_gn on the device needs a device problem")
    eng = prob.engine
    if eng.batch != 1:
        raise CapabilityMissing("direction_cg_gn: one instance per engine")
    pl = prob.plan
    t0 = time.perf_counter()
    if grad is None:
        grad = adjoint_gradient(prob, x, p)
    prob._load(x, p)
    eng.assemble()
    st = _lib_stream()
    eng.gx_values()
    eng.gfac.numeric(eng.gvals, 0.0, 0.0, st)
    eng.gfac.check(st)
    op = DeviceReducedOperator(eng, pl)
    assemble_s = time.perf_counter() - t0
    try:
        dp, rep = cg_reduced(op, -np.asarray(grad, dtype=np.float64), eta=cfg.cg_eta)
        return SearchDirection(dp=dp, assemble_s=assemble_s, solve_s=rep.solve_time,
                               relative_residual=rep.relative_residual,
                               extra={"cg_iterations": rep.refine_iterations, "operator_applications": op.applications})
    except NegativeCurvature as exc:
        dp = exc.best if exc.best is not None and np.linalg.norm(exc.best) > 0 else -np.asarray(grad)
        return SearchDirection(dp=dp, assemble_s=assemble_s)


def direction_bgn(prob, x, p, cfg: OptimizerConfig, grad=None) -> SearchDirection:
    """Block-substitution Gauss-Newton step (reference optimize.py:201-209): needs B = C = 0
    and a square dc/dp; both factorizations and solves on the device (``solve_block_gn``)."""
    from .sensitivity import solve_block_gn
    t0 = time.perf_counter()
    blocks = gn_blocks(prob, x, p)
    assemble_s = time.perf_counter() - t0
    t1 = time.perf_counter()
    dp = solve_block_gn(prob, x, p, blocks.A)
    return SearchDirection(dp=dp, assemble_s=assemble_s, solve_s=time.perf_counter() - t1)


def direction_gd(prob, x, p, cfg: OptimizerConfig, grad=None) -> SearchDirection:
    """Steepest descent in parameter space (reference optimize.py:235-240); the gradient
    is the device adjoint solve."""
    t0 = time.perf_counter()
    if grad is None:
        grad = adjoint_gradient(prob, x, p)
    return SearchDirection(dp=-np.asarray(grad, dtype=np.float64), assemble_s=time.perf_counter() - t0)


def _lib_stream() -> int:
    from . import _lib
    return _lib.stream_handle()


_DIRECTION_FUNCS = {"sgn": direction_sgn, "dgn": direction_dgn, "bgn": direction_bgn, "cg_gn": direction_cg_gn,
                    "gd": direction_gd}


def direction_lbfgs(history, grad: np.ndarray, apply_h0=None) -> np.ndarray:
    """L-BFGS two-loop recursion, returning -H grad (reference optimize.py:310-335).

    ``history``: (s, y, rho) triples, oldest first; ``apply_h0`` maps a vector through the
    initial inverse Hessian (default gamma I, gamma = s.y / y.y of the newest pair, 1 when
    the history is empty).  n_p-length host vectors: the expensive part of L-BFGS-SGN is
    ``apply_h0`` (a device KKT solve).
    """
    q = np.asarray(grad, dtype=np.float64).copy()
    alphas = []
    for s, y, rho in reversed(history):
        a = rho * (s @ q)
        alphas.append(a)
        q -= a * y
    if apply_h0 is None:
        gamma = 1.0
        if history:
            s, y, _ = history[-1]
            gamma = (s @ y) / (y @ y)
        r = gamma * q
    else:
        r = apply_h0(q)
    for (s, y, rho), a in zip(history, reversed(alphas)):
        b = rho * (y @ r)
        r += s * (a - b)
    return -r


def _direction_lbfgs_sgn(prob, x, p, cfg: OptimizerConfig, g, history) -> SearchDirection:
    """Two-loop recursion whose initial inverse Hessian is the sparse Gauss-Newton solve
    (reference optimize.py:433-457): H0^{-1} q = -(dp slot of K^{-1} (0, -q, 0)).  The KKT is
    assembled and factored once per direction on the device; an empty history reproduces
    ``direction_sgn`` bitwise (reference checks.py:213-226)."""
    from .engine import kkt_inverse_p
    t0 = time.perf_counter()
    if _is_device_problem(prob):
        eng = prob.engine
        eng.stab = cfg.stabilization
        prob._load(x, p)
        eng.assemble()
    else:
        eng, _ = _host_kkt(prob, x, p)
        eng.stab = cfg.stabilization
    eng.torch.cuda.synchronize()
    assemble_s = time.perf_counter() - t0
    reports = []
    n_x, n_p = prob.n_x, prob.n_p

    def apply_h0(q):
        t1 = time.perf_counter()
        sol, res, its = kkt_inverse_p(eng, -np.asarray(q, dtype=np.float64), factor=not reports)
        reports.append((res, its, time.perf_counter() - t1))
        return -sol[n_x:n_x + n_p]

    dp = direction_lbfgs(history, g, apply_h0)
    res, its, solve_s = reports[-1]
    return SearchDirection(dp=dp, assemble_s=assemble_s, solve_s=solve_s, relative_residual=res,
                           extra={"refine_iterations": its})


def _compute_direction(prob, x, p, cfg: OptimizerConfig, g, history) -> SearchDirection:
    """Method dispatch of the outer loop (reference optimize.py:423-430)."""
    if cfg.method == "lbfgs":
        t0 = time.perf_counter()
        dp = direction_lbfgs(history, g)
        return SearchDirection(dp=dp, assemble_s=time.perf_counter() - t0)
    if cfg.method == "lbfgs_sgn":
        return _direction_lbfgs_sgn(prob, x, p, cfg, g, history)
    return _DIRECTION_FUNCS[cfg.method](prob, x, p, cfg, grad=g)


def _push_history(history, s, y, cap):
    """Curvature-guarded history update (reference optimize.py:460-465)."""
    sy = float(s @ y)
    if sy > 1e-12 * np.linalg.norm(s) * np.linalg.norm(y):
        history.append((s, y, 1.0 / sy))
        if len(history) > cap:
            history.pop(0)


def _line_search(prob, p, x, f, g, dp, bounds, cfg):
    """Armijo backtracking over forward solves (optimize.py:468-488)."""
    alpha = 1.0
    fwd_time = 0.0
    for _ in range(cfg.max_backtracks + 1):
        p_try = p + alpha * dp
        if bounds is not None:
            np.clip(p_try, bounds[0], bounds[1], out=p_try)
        slope = float(g @ (p_try - p))
        if slope < 0.0:
            t0 = time.perf_counter()
            try:
                x_try = prob.simulate(p_try, x_init=x)
            except (ForwardSimFailure, NoConvergence, NumericalBlowup):
                x_try = None
            fwd_time += time.perf_counter() - t0
            if x_try is not None:
                f_try = prob.objective(x_try, p_try)
                if np.isfinite(f_try) and f_try <= f + cfg.armijo_c1 * slope:
                    return True, p_try, x_try, f_try, alpha, fwd_time
        alpha *= cfg.backtrack_factor
    return False, None, None, None, 0.0, fwd_time


def minimize(prob, p0, cfg: OptimizerConfig) -> OptimizerRun:
    """Minimize f(x(p), p) with SGN directions and monotone backtracking (optimize.py:353-420)."""
    if cfg.method not in METHODS:
        raise ValueError(f"unknown method {cfg.method!r}; valid: {', '.join(METHODS)}")
    t_start = time.perf_counter()
    p = np.asarray(p0, dtype=np.float64).copy()
    bounds = prob.bounds() if cfg.bound_mode == "project" else None
    if bounds is not None and (np.any(p < bounds[0]) or np.any(p > bounds[1])):
        raise InfeasiblePoint("initial parameters violate bounds")
    t0 = time.perf_counter()
    try:
        x = prob.simulate(p)
    except (NoConvergence, NumericalBlowup) as exc:
        raise ForwardSimFailure(f"initial forward solve failed: {exc}") from exc
    fwd_time = time.perf_counter() - t0
    f = prob.objective(x, p)
    g = adjoint_gradient(prob, x, p)
    records = [IterationRecord(0, f, float(np.linalg.norm(g)), 0.0, 0.0, fwd_time,
                               time.perf_counter() - t_start, float("nan"))]
    history = []
    termination = "max_iterations"
    for it in range(1, cfg.max_iterations + 1):
        if np.linalg.norm(g) <= cfg.gradient_tolerance:
            termination = "gradient_tolerance"
            break
        t0 = time.perf_counter()
        sd = _compute_direction(prob, x, p, cfg, g, history)
        dir_time = time.perf_counter() - t0
        dp = sd.dp
        if bounds is not None:
            dp = project_direction_bounds(dp, p, *bounds)
            if g @ dp >= 0.0:
                dp = project_direction_bounds(-g, p, *bounds)
        if np.linalg.norm(dp) == 0.0:
            termination = "stationary"
            break
        if g @ dp >= 0.0:
            termination = "no_descent"
            break
        accepted, p_new, x_new, f_new, alpha, fwd_time = _line_search(prob, p, x, f, g, dp, bounds, cfg)
        if not accepted:
            termination = "line_search_failure"
            break
        g_new = adjoint_gradient(prob, x_new, p_new)
        if cfg.method in ("lbfgs", "lbfgs_sgn"):
            _push_history(history, p_new - p, g_new - g, cfg.lbfgs_history)
        p, x, f, g = p_new, x_new, f_new, g_new
        records.append(IterationRecord(it, f, float(np.linalg.norm(g)), alpha, dir_time, fwd_time,
                                       time.perf_counter() - t_start, sd.relative_residual))
    return OptimizerRun(method=cfg.method, records=records, termination=termination, p=p, x=x)
