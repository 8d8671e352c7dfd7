"""Drop-in factorization and saddle-point solves, executed on the B200.

Mirrors the reference's solver surface (reference pkg/src/sgnopt/linear_solvers.py):

* ``SolveReport`` / ``StabilizationConfig``            (linear_solvers.py:31-58)
* ``SparseFactorization`` / ``factor_sparse``          (linear_solvers.py:61-102)
  -> multifrontal LDL^T on the device (symmetric input; 1x1 pivots in generic mode);
     unsymmetric square input through its symmetric saddle form [[0, M^T], [M, 0]]
* ``stabilized_matrix``                                 (linear_solvers.py:111-127)
* ``solve_kkt_stabilized``                              (linear_solvers.py:130-175)
  -> factor K + diag(+eps_x, 0, -eps_lambda) with (x_i, lambda_i) 2x2 pivots, then
     left-preconditioned restart-free BiCGSTAB against the UNSHIFTED K on the device
     (linear_solvers.py:178-211).

Dense Cholesky / matrix-free CG (DGN and CG+GN baselines) are outside the hot path.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib
from .device import DeviceFactor, symbolic_for
from .errors import (CapabilityMissing, DimensionMismatch, NegativeCurvature, NoConvergence, SingularMatrix)
from .sparse import CscMatrix

__all__ = ["SolveReport", "StabilizationConfig", "SparseFactorization", "factor_sparse",
           "stabilized_matrix", "solve_kkt_stabilized"]


@dataclass
class SolveReport:
    """Accuracy and timing of one linear solve (linear_solvers.py:31-38)."""

    relative_residual: float
    refine_iterations: int = 0
    factor_time: float = 0.0
    solve_time: float = 0.0


@dataclass
class StabilizationConfig:
    """Signed diagonal shift and refinement settings (linear_solvers.py:41-58)."""

    eps_x: float = 1e-6
    eps_lambda: float = 1e-6
    refine_tolerance: float = 1e-10
    max_refine_iters: int = 50

    def __post_init__(self):
        if self.eps_x < 0 or self.eps_lambda < 0:
            raise ValueError("stabilization shifts must be non-negative")


def _structural_checks(m: CscMatrix) -> None:
    """Empty column / row -> SingularMatrix(pivot_index) (linear_solvers.py:73-85)."""
    if m.rows != m.cols:
        raise DimensionMismatch(f"cannot factor non-square {m.rows}x{m.cols} matrix")
    empty_col = np.flatnonzero(np.diff(m.indptr) == 0)
    if empty_col.size:
        raise SingularMatrix(f"structurally singular: column {empty_col[0]} is empty",
                             pivot_index=int(empty_col[0]))
    present = np.zeros(m.rows, dtype=bool)
    present[m.indices] = True
    if not present.all():
        row = int(np.flatnonzero(~present)[0])
        raise SingularMatrix(f"structurally singular: row {row} is empty", pivot_index=row)


def _symmetric_pattern(m: CscMatrix):
    """Full symmetric pattern (union with the transpose) and the value gather map.

    Returns (indptr, indices, src) where src[k] indexes m.data (or -1 for an entry that is
    structural only in the transpose) and raises for numerically unsymmetric input.
    """
    a = m.to_scipy()
    at = a.T.tocsc()
    at.sort_indices()
    same_pattern = (np.array_equal(a.indptr, at.indptr) and np.array_equal(a.indices, at.indices))
    if same_pattern:
        if not np.array_equal(a.data, at.data):
            diff = np.max(np.abs(a.data - at.data)) if a.nnz else 0.0
            scale = np.max(np.abs(a.data)) if a.nnz else 1.0
            if diff > 1e-14 * max(scale, 1e-300):
                raise CapabilityMissing("unsymmetric factorization (the device LDL^T needs a symmetric matrix)")
        return m.indptr, m.indices, np.arange(m.nnz, dtype=np.int64)
    # structurally unsymmetric but maybe numerically symmetric: take the union
    ones = sp.csc_matrix((np.arange(1, m.nnz + 1, dtype=np.float64), m.indices, m.indptr), shape=m.shape)
    u = (ones + sp.csc_matrix((np.zeros(m.nnz), m.indices, m.indptr), shape=m.shape).T).tocsc()
    u.sort_indices()
    src = u.data.astype(np.int64) - 1
    dense_check = m.to_scipy() - m.to_scipy().T
    if dense_check.nnz and np.max(np.abs(dense_check.data)) > 1e-14 * max(np.max(np.abs(m.data)), 1e-300):
        raise CapabilityMissing("unsymmetric factorization (the device LDL^T needs a symmetric matrix)")
    return u.indptr.astype(np.int64), u.indices.astype(np.int64), src


class _DeviceSystem:
    """Device-resident copy of one symmetric matrix + its factor (shared helper)."""

    def __init__(self, m: CscMatrix, n_x: int = 0, n_p: int = 0, n_c: int = 0):
        torch = _lib.require_cuda()
        indptr, indices, src = _symmetric_pattern(m)
        self.n = m.rows
        self.sym = symbolic_for(m.rows, indptr, indices, n_x, n_p, n_c)
        vals = np.where(src >= 0, m.data[np.maximum(src, 0)], 0.0) if src.size else np.zeros(0)
        self.values = torch.from_numpy(np.ascontiguousarray(vals)).to("cuda").reshape(1, -1)
        self.factor = DeviceFactor(self.sym, 1)
        self.torch = torch

    def factorize(self, eps_x: float = 0.0, eps_lambda: float = 0.0) -> None:
        stream = _lib.stream_handle()
        self.factor.numeric(self.values, eps_x, eps_lambda, stream)
        self.factor.check(stream)

    def solve_host(self, b: np.ndarray) -> np.ndarray:
        torch = self.torch
        b = np.asarray(b, dtype=np.float64)
        cols = b.reshape(self.n, -1)
        out = np.empty_like(cols)
        stream = _lib.stream_handle()
        for j in range(cols.shape[1]):
            db = torch.from_numpy(np.ascontiguousarray(cols[:, j])).to("cuda")
            dx = torch.empty_like(db)
            self.factor.solve(db, dx, False, stream)
            out[:, j] = dx.cpu().numpy()
        return out.reshape(b.shape)


def _is_symmetric(m: CscMatrix) -> bool:
    """Numerically symmetric to 1e-14 relative (pattern union allowed)."""
    a = m.to_scipy()
    d = (a - a.T).tocsc()
    d.eliminate_zeros()
    if d.nnz == 0:
        return True
    return bool(np.max(np.abs(d.data)) <= 1e-14 * max(np.max(np.abs(a.data)) if a.nnz else 0.0, 1e-300))


def _augmented(m: CscMatrix) -> CscMatrix:
    """[[0, M^T], [M, 0]]: the symmetric saddle form of a square unsymmetric M."""
    a = m.to_scipy().tocsc()
    return CscMatrix.from_scipy(sp.bmat([[None, a.T], [a, None]], format="csc"))


class SparseFactorization:
    """Sparse factorization of a square matrix on the device (replaces linear_solvers.py:61-97).

    Symmetric input: multifrontal LDL^T (1x1 pivots in a static order), each solve refined
    by BiCGSTAB against the matrix when its residual exceeds ``refine_tolerance``.
    ``fill_nnz`` counts the equivalent LU entries with the unit diagonal excluded
    (2 * strictly-lower(L) + n), so a factored identity reports exactly n as in the
    reference's SuperLU accounting.  Symmetric indefinite input whose static order meets a
    zero pivot, or whose refinement stalls, is re-factored in the saddle form below (SuperLU's
    partial pivoting succeeds on any nonsingular matrix; so does the saddle form).

    Unsymmetric input (the reference hands it to SuperLU; here dc/dp in the block solve,
    sensitivity.py:284): the device factors the symmetric saddle form [[0, M^T], [M, 0]]
    with the KKT solver's 2x2 pivots on a structural matching of M (no shift), and each
    solve is refined by BiCGSTAB against the exact saddle matrix to ``refine_tolerance``.
    M x = b is the (0, b) right-hand side (x = first half), M^T x = b is (b, 0) (x = second
    half).  ``fill_nnz`` is then nnz of the saddle factor's L minus n.
    """

    __slots__ = ("n", "fill_nnz", "_sys", "_unsym", "_m", "refine_tolerance", "max_refine_iters", "last_report")

    def __init__(self, m: CscMatrix, refine_tolerance: float = 1e-12, max_refine_iters: int = 50):
        _structural_checks(m)
        self.n = m.rows
        self._unsym = not _is_symmetric(m)
        self.refine_tolerance = float(refine_tolerance)
        self.max_refine_iters = int(max_refine_iters)
        self.last_report = None
        self._m = m
        if not self._unsym:
            self._sys = _DeviceSystem(m)
            try:
                self._sys.factorize()
                self.fill_nnz = int(2 * self._sys.sym.stats()["nnz_l"] - self.n)
                return
            except SingularMatrix:
                # a zero pivot in the static symmetric order (symmetric indefinite input, e.g.
                # a zero diagonal): SuperLU would pivot past it, so take the saddle form below
                self._unsym = True
        self._saddle()

    def _saddle(self) -> None:
        self._unsym = True
        self._sys = _DeviceSystem(_augmented(self._m), self.n, 0, self.n)
        self._sys.factorize()
        self.fill_nnz = int(self._sys.sym.stats()["nnz_l"] - self.n)

    def solve(self, b, transpose: bool = False) -> np.ndarray:
        """x = A^{-1} b, or A^{-T} b with ``transpose`` (a no-op for a symmetric factor;
        sensitivity.py:191)."""
        b = np.asarray(b, dtype=np.float64)
        if b.shape[0] != self.n:
            raise DimensionMismatch(f"rhs has {b.shape[0]} rows, expected {self.n}")
        if not self._unsym:
            x = self._solve_symmetric(b)
            if x is not None:
                return x
            self._saddle()        # static pivots too inaccurate for refinement to recover
        return self._solve_saddle(b, transpose)

    def _solve_symmetric(self, b: np.ndarray):
        """Static-order LDL^T solve, refined by BiCGSTAB against the matrix itself when its
        residual exceeds ``refine_tolerance`` (0 iterations for well-conditioned SPD input,
        which is what SuperLU's partial pivoting gives the reference).  None when the
        refinement stalls: the caller switches to the saddle form."""
        torch = self._sys.torch
        cols = b.reshape(self.n, -1)
        out = np.empty_like(cols)
        stream = _lib.stream_handle()
        worst, iters = 0.0, 0
        for j in range(cols.shape[1]):
            if not np.any(cols[:, j]):
                out[:, j] = 0.0
                continue
            d_rhs = torch.from_numpy(np.ascontiguousarray(cols[:, j])).to("cuda")
            d_sol = torch.empty_like(d_rhs)
            rc, res, its = self._sys.factor.solve_refined(self._sys.values, d_rhs, d_sol, self.refine_tolerance,
                                                          self.max_refine_iters, False, stream)
            if rc == _lib.SGN_NO_CONVERGENCE or not np.isfinite(res[0]):
                return None
            out[:, j] = d_sol.cpu().numpy()
            worst, iters = max(worst, float(res[0])), iters + int(its[0])
        self.last_report = SolveReport(worst, iters)
        return out.reshape(b.shape)

    def _solve_saddle(self, b: np.ndarray, transpose: bool) -> np.ndarray:
        torch = self._sys.torch
        n = self.n
        cols = b.reshape(n, -1)
        out = np.empty_like(cols)
        stream = _lib.stream_handle()
        worst, iters = 0.0, 0
        for j in range(cols.shape[1]):
            rhs = np.zeros(2 * n)
            if transpose:
                rhs[:n] = cols[:, j]
            else:
                rhs[n:] = cols[:, j]
            if not np.any(rhs):
                out[:, j] = 0.0
                continue
            d_rhs = torch.from_numpy(rhs).to("cuda")
            d_sol = torch.empty_like(d_rhs)
            rc, res, its = self._sys.factor.solve_refined(self._sys.values, d_rhs, d_sol, self.refine_tolerance,
                                                          self.max_refine_iters, False, stream)
            sol = d_sol.cpu().numpy()
            if rc == _lib.SGN_NO_CONVERGENCE:
                raise NoConvergence(f"unsymmetric solve stalled at relative residual {res[0]:.3e} after "
                                    f"{its[0]} iterations", residual=float(res[0]), iterations=int(its[0]),
                                    best=sol[n:] if transpose else sol[:n])
            out[:, j] = sol[n:] if transpose else sol[:n]
            worst, iters = max(worst, float(res[0])), iters + int(its[0])
        self.last_report = SolveReport(worst, iters)
        return out.reshape(b.shape)


def factor_sparse(m: CscMatrix) -> SparseFactorization:
    """Factor a square sparse matrix on the device (linear_solvers.py:100-102)."""
    return SparseFactorization(m)


def stabilized_matrix(k, cfg: StabilizationConfig) -> CscMatrix:
    """K + diag(+eps_x 1, 0, -eps_lambda 1) as a host CSC (linear_solvers.py:111-127).

    The device path never forms this matrix: the shift is applied inside the front
    assembly of the factorization.
    """
    m: CscMatrix = k.matrix
    if cfg.eps_x == 0.0 and cfg.eps_lambda == 0.0:
        return m
    shift = np.concatenate([np.full(k.n_x, cfg.eps_x), np.zeros(k.n_p), np.full(k.n_c, -cfg.eps_lambda)])
    return CscMatrix.from_scipy(m.to_scipy() + sp.diags(shift, format="csc"))


def solve_kkt_stabilized(k, rhs, cfg: StabilizationConfig | None = None):
    """Accurate saddle-point solve on the device (linear_solvers.py:130-175).

    Factor the stabilized matrix, solve, and -- when the relative residual against the
    unshifted matrix exceeds ``refine_tolerance`` -- run preconditioned BiCGSTAB keeping
    the best iterate.  Returns ``(solution, SolveReport)``; raises ``NoConvergence``
    (with ``best``) past ``max_refine_iters``.
    """
    cfg = cfg or StabilizationConfig()
    m: CscMatrix = k.matrix
    dim = 2 * k.n_x + k.n_p
    rhs = np.asarray(rhs, dtype=np.float64)
    if m.rows != dim or m.cols != dim or rhs.shape != (dim,):
        raise DimensionMismatch(f"system dimension {m.rows} / rhs {rhs.shape} do not match 2*n_x+n_p={dim}")
    _structural_checks(m)
    torch = _lib.require_cuda()
    t0 = time.perf_counter()
    sys_ = _DeviceSystem(m, k.n_x, k.n_p, k.n_c)
    sys_.factorize(cfg.eps_x, cfg.eps_lambda)
    factor_time = time.perf_counter() - t0

    t1 = time.perf_counter()
    if not np.any(rhs):
        return np.zeros(dim), SolveReport(0.0, 0, factor_time, time.perf_counter() - t1)
    d_rhs = torch.from_numpy(rhs.copy()).to("cuda")
    d_sol = torch.empty_like(d_rhs)
    rc, res, its = sys_.factor.solve_refined(sys_.values, d_rhs, d_sol, cfg.refine_tolerance,
                                             cfg.max_refine_iters, False, _lib.stream_handle())
    x = d_sol.cpu().numpy()
    report = SolveReport(float(res[0]), int(its[0]), factor_time, time.perf_counter() - t1)
    if rc == _lib.SGN_NO_CONVERGENCE:
        raise NoConvergence(
            f"BiCGSTAB refinement stalled at relative residual {res[0]:.3e} after {its[0]} iterations",
            residual=float(res[0]), iterations=int(its[0]), best=x)
    return x, report


class DeviceReducedOperator:
    """Matrix-free reduced Gauss-Newton Hessian y -> S^T A S y + B S y + S^T B^T y + C y,
    S = -G_x^{-1} G_p (reference linear_solvers.py:243-268), applied on the device: the
    KKT blocks A, B, C, G_p are read from the engine's KKT CSC (sgn_csc_spmm) and the two
    solves per application use the engine's unshifted G_x factor (symmetric G_x)."""

    def __init__(self, eng, plan):
        from ._lib import check, lib, ptr
        self._check, self._lib, self._ptr = check, lib, ptr
        torch = eng.torch
        self.eng, self.torch = eng, torch
        self.n_x, self.n_p = plan.n_x, plan.n_p
        T = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.int64, device="cuda")
        if not hasattr(eng, "_kpat"):
            eng._kpat = (T(plan.K_indptr), T(plan.K_indices))
        self.kp, self.ki = eng._kpat
        E = lambda n: torch.empty(n, dtype=torch.float64, device="cuda")
        self.y, self.gy, self.t, self.u, self.u2, self.w = E(self.n_p), E(self.n_x), E(self.n_x), E(self.n_x), E(self.n_x), E(self.n_x)
        self.pm1 = torch.tensor([1.0, -1.0], dtype=torch.float64, device="cuda")   # axpy step lengths
        self.r1, self.r2, self.r3 = E(self.n_p), E(self.n_p), E(self.n_p)
        self.applications = 0

    def _spmm(self, r0, nr, c0, nc, x, y, st):
        self._check(self._lib().sgn_csc_spmm(self._ptr(self.kp), self._ptr(self.ki), self._ptr(self.eng.kvals[0]),
                                             r0, nr, c0, nc, self._ptr(x), nc, self._ptr(y), nr, 1, st))

    def apply(self, yv: np.ndarray) -> np.ndarray:
        self.applications += 1
        st = _lib.stream_handle()
        n_x, n_p = self.n_x, self.n_p
        lam0, p0 = n_x + n_p, n_x
        self.y.copy_(self.torch.from_numpy(np.ascontiguousarray(yv, dtype=np.float64)))
        self._spmm(lam0, n_x, p0, n_p, self.y, self.gy, st)                   # G_p y
        self.eng.gfac.solve(self.gy.view(1, -1), self.t.view(1, -1), False, st)
        self._axpy(1, self.t, None, self.t, n_x, st)                          # t = S y = -G_x^{-1} G_p y
        self._spmm(0, n_x, 0, n_x, self.t, self.u, st)                         # A t
        self._spmm(0, n_x, p0, n_p, self.y, self.u2, st)                       # B^T y
        self._axpy(0, self.u2, self.u, self.u, n_x, st)
        self.eng.gfac.solve(self.u.view(1, -1), self.w.view(1, -1), False, st)   # G_x^{-T} u
        self._spmm(p0, n_p, lam0, n_x, self.w, self.r1, st)                    # G_p^T w
        self._spmm(p0, n_p, 0, n_x, self.t, self.r2, st)                       # B t
        self._spmm(p0, n_p, p0, n_p, self.y, self.r3, st)                      # C y
        self._axpy(1, self.r1, self.r2, self.r2, n_p, st)
        self._axpy(0, self.r3, self.r2, self.r2, n_p, st)
        return self.r2.cpu().numpy()

    def _axpy(self, sign, x, y, out, n, st):
        """out = y + (+1 | -1) x on the device (sgn_axpy; sign 0: +1, 1: -1; y None: 0)."""
        self._check(self._lib().sgn_axpy(n, 1, self._ptr(self.pm1[sign:]), self._ptr(x),
                                         self._ptr(y) if y is not None else None, self._ptr(out), n, st))


def cg_reduced(op, rhs: np.ndarray, eta: float = 1e-3, max_iters: int | None = None):
    """CG on the reduced operator to relative residual eta (reference linear_solvers.py:271-323):
    raises NegativeCurvature (last iterate) on non-positive curvature and NoConvergence past
    the cap (default 10 n_p); the recursive residual is confirmed by a true one."""
    rhs = np.asarray(rhs, dtype=np.float64)
    if rhs.shape != (op.n_p,):
        raise DimensionMismatch(f"rhs has length {rhs.size}, expected {op.n_p}")
    if max_iters is None:
        max_iters = 10 * op.n_p
    t0 = time.perf_counter()
    bnorm = float(np.linalg.norm(rhs))
    x = np.zeros_like(rhs)
    if bnorm == 0.0:
        return x, SolveReport(0.0, 0, 0.0, time.perf_counter() - t0)
    r = rhs.copy()
    pdir = r.copy()
    rs = float(r @ r)
    it = 0
    while it < max_iters:
        it += 1
        hp = op.apply(pdir)
        php = float(pdir @ hp)
        if php <= 0.0:
            raise NegativeCurvature(f"non-positive curvature {php:.3e} at CG iteration {it}",
                                    best=x, iterations=it)
        step = rs / php
        x += step * pdir
        r -= step * hp
        if np.linalg.norm(r) <= eta * bnorm:
            true_r = rhs - op.apply(x)
            true_norm = float(np.linalg.norm(true_r))
            if true_norm <= eta * bnorm:
                return x, SolveReport(true_norm / bnorm, it, 0.0, time.perf_counter() - t0)
            r = true_r
        rs_new = float(r @ r)
        pdir = r + (rs_new / rs) * pdir
        rs = rs_new
    res = float(np.linalg.norm(rhs - op.apply(x)) / bnorm)
    raise NoConvergence(f"CG exceeded {max_iters} iterations (relative residual {res:.3e})",
                        residual=res, iterations=it, best=x)
