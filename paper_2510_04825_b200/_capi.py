"""ctypes binding of libsas.so (include/sas.h).

This is the only place Python touches the C ABI.  It fails loudly: if the
library is missing or no CUDA device is usable, every call raises
BackendError — there is no CPU fallback for the online path.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .errors import BackendError

HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("SAS_LIBRARY", HERE / "libsas.so"))

SAS_OK, SAS_ERR_ARG, SAS_ERR_CUDA, SAS_ERR_NCCL, SAS_ERR_NUMERICAL = 0, 1, 2, 3, 4
SAS_ST_OK, SAS_ST_RANK_DEFICIENT, SAS_ST_NONFINITE = 0, 1, 2
SAS_F64, SAS_C128 = 0, 1
SAS_OP_AFFINE, SAS_OP_STENCIL, SAS_OP_GAUSS = 0, 1, 2
SAS_COEF_CONST, SAS_COEF_LINEAR, SAS_COEF_EXP, SAS_COEF_TABLE = 0, 1, 2, 3
SAS_FLAG_INPUT_DEVICE = 1

#: every symbol declared in include/sas.h (checked by tests/test_capi_symbols.py)
EXPORTS = (
    "sas_plan_create", "sas_solve", "sas_solve_host", "sas_lift", "sas_residual",
    "sas_plan_set_operator", "sas_plan_info", "sas_last_launch_count",
    "sas_plan_destroy", "sas_last_error", "sas_version", "sas_plan_set_timing", "sas_stage_times",
    "sas_tsqr_r", "sas_cg_stencil", "sas_range_rows", "sas_bicgstab_csr",
)
SAS_STAGE_LSQ, SAS_STAGE_GAUSS_ROWS, SAS_STAGE_STENCIL_ROWS = 1, 2, 3
#: test-only symbols (include/sas_debug.h)
DEBUG_EXPORTS = ("sas_debug_exp64_host", "sas_debug_exp64")


class SasDesc(C.Structure):
    _fields_ = [
        ("op_kind", C.c_int32),
        ("dtype", C.c_int32),
        ("param_dim", C.c_int32),
        ("param_complex", C.c_int32),
        ("n_terms", C.c_int32),
        ("term_kind", C.POINTER(C.c_int32)),
        ("term_scale", C.POINTER(C.c_double)),
        ("term_rate", C.POINTER(C.c_double)),
        ("blocks", C.c_void_p),
        ("n_edges", C.c_int32),
        ("edge_nbr", C.POINTER(C.c_int64)),
        ("edge_phi", C.POINTER(C.c_double)),
        ("edge_div", C.c_double),
        ("points", C.POINTER(C.c_double)),
        ("point_dim", C.c_int32),
        ("ridge", C.c_double),
    ]


_lib = None
_lock = threading.Lock()


def _declare(lib):
    vp, i32, i64, u32, dp = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.POINTER(C.c_double)
    lib.sas_plan_create.argtypes = [C.POINTER(SasDesc), vp, i64, i32, C.POINTER(C.c_int64), dp, i32,
                                    vp, vp, i32, u32, C.POINTER(vp)]
    lib.sas_plan_create.restype = C.c_int
    lib.sas_solve.argtypes = [vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp]
    lib.sas_solve.restype = C.c_int
    lib.sas_solve_host.argtypes = [vp, vp, i64, vp, vp, vp, vp, vp, vp, vp]
    lib.sas_solve_host.restype = C.c_int
    lib.sas_lift.argtypes = [vp, vp, i64, vp, vp]
    lib.sas_lift.restype = C.c_int
    lib.sas_residual.argtypes = [vp, vp, vp, i64, vp, vp, vp, vp, vp]
    lib.sas_residual.restype = C.c_int
    lib.sas_plan_set_operator.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), vp, vp, vp]
    lib.sas_plan_set_operator.restype = C.c_int
    lib.sas_plan_info.argtypes = [vp, C.POINTER(i64), C.POINTER(i32), C.POINTER(i32), C.POINTER(i32),
                                  C.POINTER(i32), C.POINTER(i32)]
    lib.sas_plan_info.restype = C.c_int
    lib.sas_last_launch_count.argtypes = [vp]
    lib.sas_last_launch_count.restype = C.c_int32
    lib.sas_plan_set_timing.argtypes = [vp, i32]
    lib.sas_plan_set_timing.restype = C.c_int
    lib.sas_stage_times.argtypes = [vp, C.POINTER(C.c_float), C.POINTER(i32), i32]
    lib.sas_stage_times.restype = C.c_int32
    lib.sas_plan_destroy.argtypes = [vp]
    lib.sas_plan_destroy.restype = None
    lib.sas_last_error.argtypes = []
    lib.sas_last_error.restype = C.c_char_p
    lib.sas_version.argtypes = []
    lib.sas_version.restype = C.c_char_p
    lib.sas_debug_exp64_host.argtypes = [C.c_double]
    lib.sas_debug_exp64_host.restype = C.c_double
    lib.sas_debug_exp64.argtypes = [vp, vp, i64, vp]
    lib.sas_debug_exp64.restype = C.c_int
    lib.sas_tsqr_r.argtypes = [vp, i64, i32, i32, vp, i32, vp]
    lib.sas_tsqr_r.restype = C.c_int
    lib.sas_range_rows.argtypes = [vp, i64, i32, vp, i32, i32, vp, vp, i32, vp]
    lib.sas_range_rows.restype = C.c_int
    lib.sas_bicgstab_csr.argtypes = [i64, vp, vp, vp, vp, vp, vp, i32, C.c_double, C.c_double, i32, i32, i32, vp,
                                     C.POINTER(i32), dp, dp]
    lib.sas_bicgstab_csr.restype = C.c_int
    lib.sas_cg_stencil.argtypes = [i64, i32, vp, vp, vp, vp, vp, C.c_double, C.c_double, i32, i32, i32, vp,
                                   C.POINTER(i32), dp, dp]
    lib.sas_cg_stencil.restype = C.c_int
    return lib


def load(build_if_missing: bool = True):
    """Load libsas.so (building it with nvcc first if it is missing)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists() and build_if_missing:
            from . import build as _build
            _build.build()
        if not LIB_PATH.exists():
            raise BackendError(f"{LIB_PATH} not found; run `python -m paper_2510_04825_b200.build`")
        try:
            _lib = _declare(C.CDLL(str(LIB_PATH)))
        except OSError as exc:
            raise BackendError(f"cannot load {LIB_PATH}: {exc}") from exc
        return _lib


def last_error() -> str:
    msg = load().sas_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str):
    if rc != SAS_OK:
        msg = last_error()
        if rc == SAS_ERR_ARG:
            raise ValueError(f"{what}: {msg}")
        raise BackendError(f"{what} failed (code {rc}): {msg}")


def ptr(a) -> C.c_void_p:
    """Raw data pointer of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return C.c_void_p(0)
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return C.c_void_p(a.ctypes.data)
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return C.c_void_p(a.data_ptr())
    raise TypeError(f"cannot take a pointer of {type(a)!r}")


def dptr(a):
    return C.cast(ptr(a), C.POINTER(C.c_double))
