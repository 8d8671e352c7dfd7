"""ctypes binding of the native library ``_sgnb200.so`` (C ABI in include/sgn_b200.h).

The product path has no CPU fallback: if the shared library is missing, or no CUDA
device is present when a device call is made, the call raises.  Device buffers are
torch CUDA tensors (used only for allocation/streams, never for the math).
"""
from __future__ import annotations

import ctypes
import pathlib

from .errors import DeviceError, DimensionMismatch, NoConvergence, SingularMatrix, ToolkitError

LIB_PATH = pathlib.Path(__file__).with_name("_sgnb200.so")

SGN_OK, SGN_SINGULAR, SGN_NO_CONVERGENCE, SGN_DIMENSION, SGN_CUDA_ERROR, SGN_INVALID = range(6)
SGN_SOLVE_LEADING = 1
SGN_ELEM_SPRING, SGN_ELEM_NH_TRI, SGN_ELEM_NH_TET, SGN_ELEM_SHELL_MEMBRANE, SGN_ELEM_HINGE = 1, 2, 3, 4, 5

c_i32, c_i64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
P_i64 = ctypes.POINTER(c_i64)
P_i32 = ctypes.POINTER(c_i32)
P_dbl = ctypes.POINTER(c_dbl)


class SymbolicStats(ctypes.Structure):
    _fields_ = [("n", c_i64), ("n_fronts", c_i64), ("n_levels", c_i64), ("nnz_l", c_i64),
                ("front_doubles", c_i64), ("max_front", c_i64), ("max_piv", c_i64),
                ("launches", c_i64), ("flops", c_dbl), ("pair_mode", c_i64)]


class SymbolicOptions(ctypes.Structure):
    """sgn_symbolic_options (include/sgn_b200.h)."""
    _fields_ = [("leaf_size", c_i32), ("p_order", c_i32), ("upd_group", c_i32), ("zinline", c_i32),
                ("zquota", c_i32), ("noz_tiles", c_i32), ("fat_tiles", c_i32), ("fat_solve", c_i32),
                ("generic_pairs", c_i32), ("upd_pair", c_i32), ("pair_min_tiles", c_i32),
                ("upd_group_cb", c_i32), ("defer_groups", c_i32), ("zdist", c_i32), ("reserved", c_i32 * 2)]


class LsqArgs(ctypes.Structure):
    """sgn_lsq_args (include/sgn_b200.h)."""
    _fields_ = [("n_x", c_i64), ("n_p", c_i64), ("n_t", c_i64), ("tdofs", c_vp), ("tvals", c_vp),
                ("tstride", c_i64), ("w_t", c_dbl), ("w_reg", c_dbl), ("x_scale", c_dbl),
                ("rptr", c_vp), ("ridx", c_vp), ("rcoef", c_vp), ("rtptr", c_vp), ("rtidx", c_vp),
                ("rtcoef", c_vp), ("rscr", c_vp), ("part", c_vp), ("tickets", c_vp)]


# name -> (restype, argtypes); every symbol include/sgn_b200.h declares
SIGNATURES = {
    "sgn_last_error": (ctypes.c_char_p, []),
    "sgn_version": (ctypes.c_int, []),
    "sgn_launch_count": (c_i64, []),
    "sgn_device_sync": (ctypes.c_int, [c_vp]),
    "sgn_symbolic_create": (ctypes.c_int, [c_i64, P_i64, P_i64, c_i64, c_i64, c_i64, c_i32,
                                           ctypes.POINTER(c_vp), P_i64]),
    "sgn_symbolic_options_default": (None, [ctypes.POINTER(SymbolicOptions)]),
    "sgn_symbolic_create_ex": (ctypes.c_int, [c_i64, P_i64, P_i64, c_i64, c_i64, c_i64,
                                              ctypes.POINTER(SymbolicOptions), ctypes.POINTER(c_vp), P_i64]),
    "sgn_symbolic_get_stats": (ctypes.c_int, [c_vp, ctypes.POINTER(SymbolicStats)]),
    "sgn_symbolic_get_perm": (ctypes.c_int, [c_vp, P_i64]),
    "sgn_symbolic_get_fronts": (ctypes.c_int, [c_vp, P_i64, P_i64, P_i64, P_i64, P_i64, P_i64]),
    "sgn_symbolic_destroy": (None, [c_vp]),
    "sgn_factor_create": (ctypes.c_int, [c_vp, c_i32, ctypes.POINTER(c_vp)]),
    "sgn_factor_numeric": (ctypes.c_int, [c_vp, c_vp, c_i64, c_dbl, c_dbl, c_vp]),
    "sgn_factor_numeric_v": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "sgn_factor_check": (ctypes.c_int, [c_vp, c_vp, P_i64]),
    "sgn_factor_status": (ctypes.c_int, [c_vp, c_vp, P_i64]),
    "sgn_masked_copy": (ctypes.c_int, [c_i64, c_i32, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "sgn_fingerprint": (ctypes.c_int, [c_i64, c_i32, c_vp, c_i64, c_vp, c_vp]),
    "sgn_factor_solve": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_vp]),
    "sgn_factor_solve_multi": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_vp]),
    "sgn_factor_set_grid": (ctypes.c_int, [c_vp, c_i32, ctypes.POINTER(ctypes.c_int32)]),
    "sgn_factor_set_retire": (ctypes.c_int, [c_vp, c_i32, c_i32, ctypes.POINTER(ctypes.c_int64)]),
    "sgn_factor_min_pivot": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "sgn_csc_block_dense": (ctypes.c_int, [c_i64, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "sgn_csc_spmm": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64,
                                    c_i64, c_vp]),
    "sgn_gemm_tn": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "sgn_gn_hessian": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "sgn_debug_solve_trace": (ctypes.c_int, [c_vp, c_vp, ctypes.c_int64, c_vp, c_vp]),
    "sgn_debug_factor_trace": (ctypes.c_int, [c_vp, c_vp, ctypes.c_int64, c_vp, c_vp]),
    "sgn_debug_factor_buffer": (ctypes.c_int, [c_vp, c_i32, c_vp, ctypes.c_int64, c_vp]),
    "sgn_debug_poison": (ctypes.c_int, [c_vp, c_dbl]),
    "sgn_factor_destroy": (None, [c_vp]),
    "sgn_solve_ir": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i32, P_dbl, P_dbl, c_vp]),
    "sgn_residual_dd": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "sgn_spmv": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_i32, c_vp]),
    "sgn_solve_refined": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_dbl, c_i32, c_i32,
                                         P_dbl, P_i32, c_vp]),
    "sgn_element_derivs": (ctypes.c_int, [c_i32, c_i64, c_i32, c_vp, c_vp, c_vp, c_i64, c_vp,
                                          c_i64, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "sgn_element_derivs_ex": (ctypes.c_int, [c_i32, c_i64, c_i32, c_vp, c_vp, c_vp, c_i64, c_vp,
                                             c_i64, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp]),
    "sgn_element_energy_grad": (ctypes.c_int, [c_i32, c_i64, c_i32, c_vp, c_vp, c_vp, c_i64,
                                               c_vp, c_i64, c_vp, c_vp, c_i64, c_vp]),
    "sgn_gather_values": (ctypes.c_int, [c_i64, c_i32, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp,
                                         c_i64, c_vp, c_i64, c_vp]),
    "sgn_vertex_assemble": (ctypes.c_int, [c_i32, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                           c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64,
                                           c_vp]),
    "sgn_element_mixed": (ctypes.c_int, [c_i32, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp,
                                         c_i64, c_vp]),
    "sgn_gather_to": (ctypes.c_int, [c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64,
                                     c_vp]),
    "sgn_reduce": (ctypes.c_int, [c_i32, c_i64, c_i32, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "sgn_axpy": (ctypes.c_int, [c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "sgn_fp64_peak": (ctypes.c_int, [c_i32, c_i32, P_dbl, c_vp]),
    "sgn_lsq_eval": (ctypes.c_int, [c_i32, ctypes.c_void_p, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "sgn_restlen_blocks": (ctypes.c_int, [c_i64, c_i32, c_vp, c_vp, c_i64, c_vp, c_dbl, c_vp, c_i64, c_vp]),
    "sgn_adjoint_step": (ctypes.c_int, [c_i32, c_i32, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
}

_LIB = None


def lib() -> ctypes.CDLL:
    """Load the native library (once); raises if it has not been built."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise ToolkitError(
                f"native library {LIB_PATH} is missing; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
        so = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(so, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = so
    return _LIB


def last_error() -> str:
    msg = lib().sgn_last_error()
    return msg.decode() if msg else ""


def check(rc: int, pivot: int = -1, what: str = "") -> None:
    """Map a C-ABI status onto the reference's exception types."""
    if rc == SGN_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == SGN_SINGULAR:
        raise SingularMatrix(msg, pivot_index=int(pivot))
    if rc == SGN_DIMENSION:
        raise DimensionMismatch(msg)
    if rc == SGN_NO_CONVERGENCE:
        raise NoConvergence(msg)
    if rc == SGN_CUDA_ERROR:
        raise DeviceError(msg)
    raise ToolkitError(msg)


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return 0 if t is None else int(t.data_ptr())


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the SGN path runs only on the GPU (no CPU fallback)")
    return torch


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
