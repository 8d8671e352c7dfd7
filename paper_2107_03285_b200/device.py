"""Thin Python handles over the native symbolic analysis and device factorization.

``Symbolic`` wraps ``sgn_symbolic_*`` (host, once per sparsity pattern; cached);
``DeviceFactor`` wraps ``sgn_factor_*`` / ``sgn_spmv`` / ``sgn_solve_refined`` on
torch-allocated device buffers.  Nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes
from collections import OrderedDict

import numpy as np

from . import _lib
from ._lib import P_dbl, P_i32, P_i64, SymbolicStats, check, lib, ptr

_CACHE: "OrderedDict[tuple, Symbolic]" = OrderedDict()
_CACHE_MAX = 16


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


# option fields of sgn_symbolic_options and the SGN_* variables that override them (for
# profiling sweeps only; the product path passes options explicitly)
_OPTION_ENV = {"leaf_size": "SGN_LEAF_SIZE", "upd_group": "SGN_UPD_GROUP", "zinline": "SGN_ZINLINE",
               "zquota": "SGN_ZQUOTA", "noz_tiles": "SGN_NOZ_TILES", "fat_tiles": "SGN_FAT_TILES",
               "fat_solve": "SGN_FAT_SOLVE", "generic_pairs": "SGN_GENERIC_PAIRS", "p_order": "SGN_P_ORDER",
               "upd_pair": "SGN_UPD_PAIR", "pair_min_tiles": "SGN_PAIR_MIN_TILES",
               "upd_group_cb": "SGN_UPD_GROUP_CB", "defer_groups": "SGN_DEFER_GROUPS", "zdist": "SGN_ZDIST"}


def symbolic_options(**kw) -> "_lib.SymbolicOptions":
    """Defaults (sgn_symbolic_options_default), then SGN_* environment overrides
    (experiments), then the keyword arguments."""
    import os
    o = _lib.SymbolicOptions()
    lib().sgn_symbolic_options_default(ctypes.byref(o))
    for f, env in _OPTION_ENV.items():
        if os.environ.get(env):
            setattr(o, f, int(os.environ[env]))
    for f, v in kw.items():
        if v is not None:
            setattr(o, f, int(v))
    return o


class Symbolic:
    """Ordering + assembly tree + maps for one pattern (sgn_symbolic_create_ex)."""

    def __init__(self, n: int, indptr, indices, n_x: int = 0, n_p: int = 0, n_c: int = 0,
                 leaf_size: int = 0, **options):
        self.n, self.n_x, self.n_p, self.n_c = int(n), int(n_x), int(n_p), int(n_c)
        self.indptr = _i64(indptr)
        self.indices = _i64(indices)
        h = ctypes.c_void_p()
        piv = ctypes.c_int64(-1)
        self.options = symbolic_options(leaf_size=leaf_size or None, **options)
        rc = lib().sgn_symbolic_create_ex(
            self.n, self.indptr.ctypes.data_as(P_i64), self.indices.ctypes.data_as(P_i64),
            self.n_x, self.n_p, self.n_c, ctypes.byref(self.options), ctypes.byref(h), ctypes.byref(piv))
        check(rc, piv.value, "symbolic analysis")
        self._h = h

    @property
    def handle(self):
        return self._h

    def stats(self) -> dict:
        st = SymbolicStats()
        check(lib().sgn_symbolic_get_stats(self._h, ctypes.byref(st)))
        return {f: getattr(st, f) for f, _ in SymbolicStats._fields_}

    def perm(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.int64)
        check(lib().sgn_symbolic_get_perm(self._h, out.ctypes.data_as(P_i64)))
        return out

    def fronts(self) -> dict:
        nf = self.stats()["n_fronts"]
        first, npiv, nrow, parent = (np.empty(nf, np.int64) for _ in range(4))
        rows_ptr = np.empty(nf + 1, np.int64)
        check(lib().sgn_symbolic_get_fronts(self._h, first.ctypes.data_as(P_i64),
                                            npiv.ctypes.data_as(P_i64), nrow.ctypes.data_as(P_i64),
                                            parent.ctypes.data_as(P_i64),
                                            rows_ptr.ctypes.data_as(P_i64), None))
        rows = np.empty(int(rows_ptr[-1]), np.int64)
        check(lib().sgn_symbolic_get_fronts(self._h, None, None, None, None,
                                            rows_ptr.ctypes.data_as(P_i64), rows.ctypes.data_as(P_i64)))
        return dict(first=first, npiv=npiv, nrow=nrow, parent=parent, rows_ptr=rows_ptr, rows=rows)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._LIB is not None:
            _lib._LIB.sgn_symbolic_destroy(h)
            self._h = None


def symbolic_for(n: int, indptr, indices, n_x: int = 0, n_p: int = 0, n_c: int = 0, **options) -> Symbolic:
    """Cached symbolic analysis (the pattern is analysed once, SURVEY §8(b) sgn_symbolic)."""
    indptr, indices = _i64(indptr), _i64(indices)
    o = symbolic_options(**options)
    key = (int(n), int(n_x), int(n_p), int(n_c), indptr.tobytes().__hash__(),
           indices.tobytes().__hash__(), int(indices.size), bytes(o))
    sym = _CACHE.get(key)
    if sym is None:
        sym = Symbolic(n, indptr, indices, n_x, n_p, n_c, **options)
        _CACHE[key] = sym
        while len(_CACHE) > _CACHE_MAX:
            _CACHE.popitem(last=False)
    else:
        _CACHE.move_to_end(key)
    return sym


class DeviceFactor:
    """Device LDL^T factor storage for `batch` instances sharing one Symbolic."""

    def __init__(self, sym: Symbolic, batch: int = 1):
        self.sym = sym
        self.batch = int(batch)
        h = ctypes.c_void_p()
        check(lib().sgn_factor_create(sym.handle, self.batch, ctypes.byref(h)), what="factor create")
        self._h = h

    def numeric(self, values, eps_x: float = 0.0, eps_lambda: float = 0.0, stream: int = 0):
        """values: torch float64 CUDA tensor (batch, nnz) in the Symbolic's CSC order."""
        stride = values.stride(0) if values.dim() == 2 else 0
        check(lib().sgn_factor_numeric(self._h, ptr(values), stride, float(eps_x),
                                       float(eps_lambda), stream), what="numeric factorization")

    def numeric_v(self, values, eps_x_dev, eps_lambda_dev=None, stream: int = 0):
        """Per-instance shifts (device float64 arrays of length batch)."""
        stride = values.stride(0) if values.dim() == 2 else 0
        check(lib().sgn_factor_numeric_v(self._h, ptr(values), stride, ptr(eps_x_dev),
                                         ptr(eps_lambda_dev), stream), what="numeric factorization")

    def status(self, stream: int = 0) -> np.ndarray:
        """First zero pivot per instance (-1 = none); synchronizes."""
        out = np.empty(self.batch, dtype=np.int64)
        check(lib().sgn_factor_status(self._h, stream, out.ctypes.data_as(P_i64)), what="factor status")
        return out

    def check(self, stream: int = 0) -> None:
        piv = ctypes.c_int64(-1)
        rc = lib().sgn_factor_check(self._h, stream, ctypes.byref(piv))
        check(rc, piv.value, "factorization")

    def solve(self, b, x, leading: bool = False, stream: int = 0) -> None:
        flags = _lib.SGN_SOLVE_LEADING if leading else 0
        check(lib().sgn_factor_solve(self._h, ptr(b), ptr(x), flags, stream), what="solve")

    def set_grid(self, ctas: int) -> int:
        """Persistent factorization grid of ``ctas`` CTAs (<= 0: the occupancy limit, all
        SMs); returns the grid in effect."""
        out = ctypes.c_int32()
        check(lib().sgn_factor_set_grid(self._h, int(ctas), ctypes.byref(out)), what="factor grid")
        return out.value

    def set_retire(self, keep_ctas: int, max_level_fronts: int) -> int:
        """CTAs >= keep_ctas leave the persistent factorization at the first top level of <=
        max_level_fronts fronts (sgn_factor_set_retire); returns the hand-over task index (-1: off)."""
        out = ctypes.c_int64()
        check(lib().sgn_factor_set_retire(self._h, int(keep_ctas), int(max_level_fronts), ctypes.byref(out)),
              what="factor retire")
        return out.value

    def solve_multi(self, B, X, stream: int = 0) -> None:
        """X[j] = A^{-1} B[j] for the rows j of a (nrhs, n) float64 CUDA tensor (batch-1 factor)."""
        check(lib().sgn_factor_solve_multi(self._h, ptr(B), ptr(X), int(B.shape[0]), stream), what="multi solve")

    def spmv(self, values, x, y, leading: bool = False, stream: int = 0) -> None:
        stride = values.stride(0) if values.dim() == 2 else 0
        flags = _lib.SGN_SOLVE_LEADING if leading else 0
        check(lib().sgn_spmv(self._h, ptr(values), stride, ptr(x), ptr(y), flags, stream), what="spmv")

    def solve_ir(self, values, rhs, sol, steps: int, stream: int = 0, sol_lo=None, report: bool = True):
        """Extra-precise iterative refinement (sgn_solve_ir); returns (rel_res[batch],
        corr[batch]) -- exact residuals of the final iterate and the last correction -- or
        (None, None) with report=False (no host synchronisation)."""
        stride = values.stride(0) if values.dim() == 2 else 0
        res = np.zeros(self.batch) if report else None
        corr = np.zeros(self.batch) if report else None
        check(lib().sgn_solve_ir(self._h, ptr(values), stride, ptr(rhs), ptr(sol),
                                 ptr(sol_lo) if sol_lo is not None else None, int(steps),
                                 res.ctypes.data_as(P_dbl) if report else None,
                                 corr.ctypes.data_as(P_dbl) if report else None, stream), what="refinement")
        return res, corr

    def residual_dd(self, values, x, x_lo, b, r, stream: int = 0) -> None:
        """r = b - K (x + x_lo), double-double evaluation (sgn_residual_dd)."""
        stride = values.stride(0) if values.dim() == 2 else 0
        check(lib().sgn_residual_dd(self._h, ptr(values), stride, ptr(x),
                                    ptr(x_lo) if x_lo is not None else None, ptr(b), ptr(r), stream), what="residual")

    def solve_refined(self, values, rhs, sol, tol: float, max_iters: int, leading: bool = False,
                      stream: int = 0):
        """Returns (rc, rel_res[batch], iters[batch]); rc == SGN_NO_CONVERGENCE keeps best in sol."""
        stride = values.stride(0) if values.dim() == 2 else 0
        res = np.zeros(self.batch)
        its = np.zeros(self.batch, dtype=np.int32)
        flags = _lib.SGN_SOLVE_LEADING if leading else 0
        rc = lib().sgn_solve_refined(self._h, ptr(values), stride, ptr(rhs), ptr(sol), float(tol),
                                     int(max_iters), flags, res.ctypes.data_as(P_dbl),
                                     its.ctypes.data_as(P_i32), stream)
        if rc not in (_lib.SGN_OK, _lib.SGN_NO_CONVERGENCE):
            check(rc, what="refined solve")
        return rc, res, its

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._LIB is not None:
            _lib._LIB.sgn_factor_destroy(h)
            self._h = None
