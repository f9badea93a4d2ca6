"""ctypes binding of libtrals.so (the C-ABI declared in include/trals.h).

The library is built in-tree by `paper_2210_11362_b200.build.build()` (or
`__graft_entry__.build()`).  There is no fallback: if the shared object is
missing or the CUDA runtime cannot be reached, `lib()` raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtrals.so")

LAYOUT_C, LAYOUT_SLICE, LAYOUT_ZT, LAYOUT_TT = 0, 1, 2, 3
INFO_CHOL, INFO_ASYM, INFO_DEGEN, INFO_FALLBACKS, INFO_ILLCOND, INFO_REFINE, INFO_SLOTS = 0, 1, 2, 3, 4, 5, 6

_dp = c_void_p  # device pointers travel as void*
_lib = None

# name -> (restype, argtypes)
_SIGNATURES = {
    "trals_strerror": (ctypes.c_char_p, [c_int]),
    "trals_version": (c_int, []),
    "trals_launch_count": (ctypes.c_longlong, []),
    "trals_gemm_ws_elems": (c_int64, [c_int64, c_int64, c_int64, c_int64]),
    "trals_gemm_f64": (c_int, [_dp, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64,
                               _dp, c_int64, _dp, POINTER(c_int64), c_int, _dp, c_int64, c_void_p]),
    "trals_core_relayout_f64": (c_int, [_dp, c_int, c_int, c_int64, c_int, _dp, c_int, c_void_p]),
    "trals_half_chain_tmp_elems": (c_int64, [c_int, POINTER(c_int64), POINTER(c_int32)]),
    "trals_half_chain_f64": (c_int, [c_int, POINTER(c_int64), POINTER(c_int32), _dp, POINTER(c_void_p),
                                     _dp, _dp, _dp, c_int64, c_int, c_void_p]),
    "trals_env_f64": (c_int, [_dp, c_int64, c_int64, c_int, _dp, c_int, c_int, _dp, c_int, _dp, c_int64,
                              c_void_p]),
    "trals_absorb_right_f64": (c_int, [_dp, c_int, c_int64, c_int64, c_int, c_int, _dp, _dp, c_int, _dp,
                                       c_int64, c_void_p]),
    "trals_absorb_left_f64": (c_int, [_dp, c_int, c_int64, c_int64, c_int, c_int, _dp, _dp, c_int, _dp,
                                      c_int64, c_void_p]),
    "trals_core_gram_f64": (c_int, [_dp, c_int, c_int64, c_int, _dp, _dp, c_int64, c_void_p]),
    "trals_core_qr_ws_elems": (c_int64, [c_int, c_int]),
    "trals_core_qr_f64": (c_int, [_dp, c_int, c_int, _dp, _dp, c_int64, c_void_p]),
    "trals_gram_chain_f64": (c_int, [c_int, c_int, POINTER(c_int32), POINTER(c_void_p), _dp, _dp, _dp,
                                     c_int64, c_void_p]),
    "trals_gram_chain_part_f64": (c_int, [c_int, c_int, POINTER(c_int32), POINTER(c_void_p), _dp, _dp, _dp,
                                     c_int64, c_int, c_void_p]),
    "trals_cholesky_aux_elems": (c_int64, [c_int]),
    "trals_cholesky_f64": (c_int, [_dp, c_int, _dp, _dp, _dp, c_int, _dp, c_void_p]),
    "trals_chol_solve_ws_elems": (c_int64, [c_int64, c_int]),
    "trals_chol_solve_f64": (c_int, [_dp, _dp, _dp, c_int, _dp, c_int64, _dp, _dp, c_int64, c_void_p]),
    "trals_solve_refine_f64": (c_int, [_dp, _dp, _dp, c_int, _dp, c_int64, _dp, _dp, c_void_p]),
    "trals_spd_fallback_ws_elems": (c_int64, [c_int64, c_int]),
    "trals_spd_fallback_f64": (c_int, [_dp, c_int, _dp, c_int64, _dp, _dp, c_int, c_double, _dp, c_int64, c_void_p]),
    "trals_tri_fallback_f64": (c_int, [_dp, c_int, c_int, _dp, c_int64, _dp, _dp, c_int, c_double, _dp, c_int64,
                                       c_void_p]),
    "trals_oz_range_ws_elems": (c_int64, [c_int64, c_int64, c_int]),
    "trals_oz_range_f64": (c_int, [_dp, c_int64, c_int64, c_int, _dp, _dp, c_int64, c_void_p]),
    "trals_dd_transfer_f64": (c_int, [_dp, c_int, c_int, c_int, _dp, _dp, c_void_p]),
    "trals_dd_r0_ws_elems": (c_int64, [c_int, POINTER(c_int32)]),
    "trals_dd_r0_f64": (c_int, [c_int, c_int, POINTER(c_int32), POINTER(c_void_p), POINTER(c_void_p), _dp, _dp, _dp,
                                c_int64, c_void_p]),
    "trals_tri_prepare_f64": (c_int, [_dp, c_int, _dp, _dp, c_int, _dp, c_void_p]),
    "trals_reverse_axes_f64": (c_int, [_dp, c_int, POINTER(c_int64), _dp, c_void_p]),
    "trals_sumsq_ws_elems": (c_int64, []),
    "trals_sumsq_f64": (c_int, [_dp, c_int64, _dp, _dp, c_void_p]),
    "trals_sumsq_f32": (c_int, [_dp, c_int64, _dp, _dp, c_void_p]),
    "trals_oz_digits_bytes": (c_int64, [c_int64, c_int64]),
    "trals_oz_split_ws_elems": (c_int64, [c_int64, c_int64, c_int]),
    "trals_oz_split_f32": (c_int, [_dp, c_int64, c_int64, c_int, _dp, _dp, _dp, c_int64, c_void_p]),
    "trals_env_oz_ws_elems": (c_int64, [c_int64, c_int64, c_int, c_int, c_int]),
    "trals_env_oz": (c_int, [_dp, _dp, c_int64, c_int64, c_int, _dp, c_int, c_int, _dp, c_int, _dp, c_int64,
                             c_void_p]),
    "trals_oz64_digits_bytes": (c_int64, [c_int64, c_int64]),
    "trals_oz64_split_f64": (c_int, [_dp, c_int64, c_int64, c_int, _dp, _dp, _dp, c_int64, c_void_p]),
    "trals_env_oz64_ws_elems": (c_int64, [c_int64, c_int64, c_int, c_int, c_int]),
    "trals_env_oz64": (c_int, [_dp, _dp, c_int64, c_int64, c_int, _dp, c_int, c_int, _dp, c_int, _dp, c_int64,
                               c_void_p]),
    "trals_error_ws_elems": (c_int64, [c_int64, c_int]),
    "trals_error_terms_f64": (c_int, [_dp, _dp, _dp, c_int64, c_int, _dp, _dp, _dp, c_int64, c_void_p]),
    "trals_residual_ws_elems": (c_int64, [c_int64, c_int64]),
    "trals_residual_f64": (c_int, [_dp, c_int64, c_int64, _dp, _dp, c_int64, _dp, _dp, _dp, c_int64, c_void_p]),
    "trals_crt_supported": (c_int, [c_int64, c_int64, c_int64]),
    "trals_crt_moduli": (c_int, []),
    "trals_crt_row_bits": (c_int, [c_int]),
    "trals_crt_planes_bytes": (c_int64, [c_int64, c_int64]),
    "trals_crt_split_ws_elems": (c_int64, [c_int64, c_int64, c_int]),
    "trals_crt_split_f64": (c_int, [_dp, c_int64, c_int64, c_int, _dp, _dp, _dp, c_int64, c_void_p]),
    "trals_env_crt_ws_elems": (c_int64, [c_int64, c_int64, c_int, c_int, c_int]),
    "trals_env_crt": (c_int, [_dp, _dp, c_int64, c_int64, c_int, _dp, c_int, c_int, _dp, c_int, _dp, c_int64,
                              c_void_p]),
    "trals_env_crt_stage": (c_int, [_dp, _dp, c_int64, c_int64, c_int, _dp, c_int, c_int, _dp, c_int, _dp, c_int64,
                                    c_int, c_void_p]),
    "trals_residual_oz64_ws_elems": (c_int64, [c_int64, c_int64, c_int64]),
    "trals_residual_oz64": (c_int, [_dp, c_int64, c_int64, _dp, _dp, c_int64, _dp, _dp, _dp, c_int64, c_void_p]),
    "trals_mttsp_ws_elems": (c_int64, [c_int, POINTER(c_int64), POINTER(c_int32), c_int]),
    "trals_mttsp_f64": (c_int, [_dp, c_int, POINTER(c_int64), POINTER(c_int32), c_int, POINTER(c_void_p),
                                POINTER(c_void_p), POINTER(c_void_p), _dp, _dp, c_int64, c_void_p]),
}

EXPORTED = tuple(_SIGNATURES)


class TralsError(RuntimeError):
    """A libtrals entry point returned a non-zero status."""


def load(path: str = LIB_PATH):
    """Load the shared object and bind every declared symbol (no GPU needed)."""
    if not os.path.exists(path):
        raise ImportError(
            f"libtrals.so not found at {path}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'`")
    handle = ctypes.CDLL(path)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    return handle


def lib():
    global _lib
    if _lib is None:
        _lib = load()
    return _lib


def check(status: int, what: str) -> None:
    if status != 0:
        msg = lib().trals_strerror(status).decode()
        raise TralsError(f"{what} failed: {msg} (status {status})")


def i64_array(vals):
    arr = (c_int64 * len(vals))(*[int(v) for v in vals])
    return arr


def i32_array(vals):
    return (c_int32 * len(vals))(*[int(v) for v in vals])


def ptr_array(ptrs):
    return (c_void_p * len(ptrs))(*[int(p) for p in ptrs])


__all__ = ["lib", "load", "check", "TralsError", "EXPORTED", "i64_array", "i32_array", "ptr_array",
           "LAYOUT_C", "LAYOUT_SLICE", "LAYOUT_ZT", "LAYOUT_TT", "INFO_CHOL", "INFO_ASYM", "INFO_DEGEN",
           "INFO_FALLBACKS", "INFO_ILLCOND", "INFO_REFINE", "INFO_SLOTS",
           "c_double"]
