"""ctypes binding of libmehdg_b200.so (include/mehdg_b200.h).

The product path has no CPU fallback: if the library is missing this module
raises ImportError, and every entry point that needs a GPU raises when none
is visible.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
# MEHDG_LIB_VARIANT=x loads libmehdg_b200.x.so instead (A/B builds of a kernel
# design point measured on the same box; tools/ only)
_VARIANT = os.environ.get("MEHDG_LIB_VARIANT")
LIB_PATH = _PKG / (f"libmehdg_b200.{_VARIANT}.so" if _VARIANT else "libmehdg_b200.so")

MH_OK = 0
MH_E_ARG = -1
MH_E_CUDA = -2
MH_E_NOMEM = -3
MH_E_SINGULAR_LOCAL = -4
MH_E_SINGULAR_FACE = -5
MH_E_STATE = -6
MH_E_UNSUPPORTED = -7
MH_E_CALLBACK = -8

FACE_KIND_NAMES = {0: "chol-neg", 1: "chol-pos", 2: "lu", -1: "singular"}

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is not built; run `python -m paper_2302_10917_b200._build` "
        "(there is no CPU fallback for the Schur-operator path)")

lib = C.CDLL(str(LIB_PATH))

_p = C.c_void_p
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_i8p = C.POINTER(C.c_int8)
_dp = C.c_void_p  # double* (host or device) passed as an address
_ip = C.POINTER(C.c_int)
_fp = C.POINTER(C.c_float)

OP_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)

# name -> argtypes (every symbol declared in include/mehdg_b200.h)
SIGNATURES = {
    "mh_last_error": [],
    "mh_version": [],
    "mh_device_count": [_ip],
    "mh_skeleton_sizes": [C.c_int, C.c_int, _i64p, _i64p, _i64p],
    "mh_build_skeleton": [C.c_int, C.c_int, _p, _p, _p, _p, _p, _p, _p],
    "mh_condense_tables": [C.c_int, C.c_int64, C.c_int64, _p, _p, _p, _p, _p, _p, _p, _p, _i64p],
    "mh_slab_partition": [C.c_int64, C.c_int64, C.c_int, _p],
    "mh_create": [C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int64, C.POINTER(_p)],
    "mh_destroy": [_p],
    "mh_set_stream": [_p, _p],
    "mh_upload_connectivity": [_p, _p, _p, _p],
    "mh_upload_blocks": [_p, _dp, _dp, _dp, _dp, _dp, _dp],
    "mh_upload_blocks_device": [_p, _dp, _dp, _dp, _dp, _dp, _dp],
    "mh_factorize": [_p, _i32p, _i32p, _p, _fp],
    "mh_refactorize_local": [_p, _fp],
    "mh_get_local_factors": [_p, C.c_int64, C.c_int64, _dp, _p],
    "mh_rhs": [_p, _dp],
    "mh_apply": [_p, _dp, _dp],
    "mh_precond": [_p, _dp, _dp],
    "mh_apply_precond": [_p, _dp, _dp],
    "mh_reconstruct": [_p, _dp, _dp],
    "mh_apply_host": [_p, _dp, _dp],
    "mh_apply_host_many": [_p, C.c_int64, _dp, C.c_int64, _dp, C.c_int64],
    "mh_assemble_macros_2d": [_p, C.c_int64, C.c_int, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p,
                              _p, _p],
    "mh_assemble_faces_2d": [_p, C.c_int64, _p, _p, _p, _p, _p],
    "mh_precond_host": [_p, _dp, _dp],
    "mh_rhs_host": [_p, _dp],
    "mh_reconstruct_host": [_p, _dp, _dp],
    "mh_form_element_schur": [_p],
    "mh_apply_mb": [_p, _dp, _dp],
    "mh_get_element_schur": [_p, C.c_int64, C.c_int64, _dp],
    "mh_get_face_inverse": [_p, C.c_int64, _p, _dp],
    "mh_set_face_inverse": [_p, C.c_int64, _p, _dp],
    "mh_profile": [_p, C.c_int],
    "mh_profile_read": [_p, C.POINTER(C.c_double), _i64p, C.POINTER(C.c_double), _i64p],
    "mh_gmres": [_p, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, _ip, _ip, _dp,
                 C.c_int, _ip],
    "mh_gmres_op": [C.c_int, _p, C.c_int64, OP_FN, _p, OP_FN, _p, C.c_double, C.c_int, C.c_int,
                    _dp, _dp, _ip, _ip, _dp, C.c_int, _ip],
    "mh_dot": [_p, C.c_int64, _dp, _dp, C.POINTER(C.c_double)],
    "mh_set_halo": [_p, C.c_int, C.c_int, _p, _p, _p, _p, _p, _p],
    "mh_group_apply": [C.POINTER(_p), C.c_int, C.POINTER(_p), C.POINTER(_p)],
    "mh_comm_unique_id": [_p],
    "mh_comm_init": [_p, _p, C.c_int, C.c_int],
}

for _name, _args in SIGNATURES.items():
    _fn = getattr(lib, _name)
    _fn.argtypes = _args
    _fn.restype = C.c_char_p if _name == "mh_last_error" else C.c_int


class MehdgError(RuntimeError):
    """Failure reported by libmehdg_b200 (status code in ``.code``)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def last_error() -> str:
    return (lib.mh_last_error() or b"").decode()


def check(status: int, what: str = "") -> None:
    if status == MH_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == MH_E_ARG:
        raise ValueError(msg)
    raise MehdgError(status, msg)


def ptr(a) -> int:
    """Address of a numpy array / torch tensor (or None -> 0)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    raise TypeError(f"cannot take the address of {type(a)!r}")


def device_count() -> int:
    c = C.c_int(0)
    check(lib.mh_device_count(C.byref(c)))
    return int(c.value)


def require_gpu() -> None:
    if device_count() < 1:
        raise RuntimeError("libmehdg_b200: no CUDA device visible (there is no CPU fallback)")


def exported_symbols() -> list:
    return sorted(SIGNATURES)


if os.environ.get("MEHDG_DEBUG_LIB"):
    print(f"loaded {LIB_PATH}")
