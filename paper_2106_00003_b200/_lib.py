"""ctypes binding of libgivens.so (include/givens.h). Argument marshalling only.

The library is the product path: if it is missing or fails to load, every op raises --
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgivens.so")

OK, EINVAL, ECUDA, EUNSUPPORTED, ENOMEM = 0, -1, -2, -3, -4
OP_APPLY, OP_BUILD_U, OP_BACKWARD = 0, 1, 2
OP_U_APPLY, OP_U_BUILD_U, OP_U_BACKWARD = 3, 4, 5
FLAG_RECOMPUTE, FLAG_REUSE_TABLES = 1, 2

EXPORTS = [
    "givens_last_error", "givens_version", "givens_num_angles", "givens_supported",
    "givens_schedule", "givens_mask_from_dims", "givens_workspace_bytes", "givens_apply",
    "givens_build_U", "givens_backward", "givens_index_trace", "givens_u_supported", "givens_u_apply",
    "givens_u_build_U", "givens_u_backward", "givens_check_perm", "givens_schedule_ex", "givens_mask_from_dims_ex",
    "givens_apply_ex", "givens_build_U_ex", "givens_backward_ex", "givens_u_apply_ex", "givens_u_build_U_ex",
    "givens_u_backward_ex", "givens_gemm_workspace_bytes", "givens_gemm_apply", "givens_gemm_backward",
    "givens_workspace_reset", "givens_fast_apply", "givens_fast_build_U",
]


class GivensError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"givens error {code}: {msg}")
        self.code = code


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2106_00003_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        C = ctypes.c_int
        L.givens_last_error.restype = ctypes.c_char_p
        L.givens_version.restype = ctypes.c_char_p
        L.givens_num_angles.restype = I64
        L.givens_num_angles.argtypes = [I32]
        L.givens_supported.restype = C
        L.givens_supported.argtypes = [I32]
        L.givens_schedule.restype = C
        L.givens_schedule.argtypes = [I32, P, P]
        L.givens_mask_from_dims.restype = C
        L.givens_mask_from_dims.argtypes = [I32, P, P]
        L.givens_fast_apply.restype = C
        L.givens_fast_apply.argtypes = [I32, I64, P, P, P, I64, P, I64, P, SZ, P]
        L.givens_fast_build_U.restype = C
        L.givens_fast_build_U.argtypes = [I32, P, P, P, I64, P, SZ, P]
        L.givens_workspace_reset.restype = None
        L.givens_workspace_reset.argtypes = [P]
        L.givens_workspace_bytes.restype = SZ
        L.givens_workspace_bytes.argtypes = [C, I32, I64]
        L.givens_apply.restype = C
        L.givens_apply.argtypes = [I32, I64, P, P, P, I64, P, I64, C, P, SZ, P]
        L.givens_build_U.restype = C
        L.givens_build_U.argtypes = [I32, P, P, P, I64, P, SZ, P]
        L.givens_backward.restype = C
        L.givens_backward.argtypes = [I32, I64, P, P, P, I64, P, I64, P, I64, P, C, P, SZ, P]
        L.givens_index_trace.restype = C
        L.givens_index_trace.argtypes = [I32, C, P, P]
        L.givens_u_supported.restype = C
        L.givens_u_supported.argtypes = [I32]
        L.givens_u_apply.restype = C
        L.givens_u_apply.argtypes = [I32, I64, P, P, P, P, I64, P, I64, C, P, SZ, P]
        L.givens_u_build_U.restype = C
        L.givens_u_build_U.argtypes = [I32, P, P, P, P, I64, P, SZ, P]
        L.givens_u_backward.restype = C
        L.givens_u_backward.argtypes = [I32, I64, P, P, P, P, I64, P, I64, P, I64, P, P, C, P, SZ, P]
        L.givens_gemm_workspace_bytes.restype = SZ
        L.givens_gemm_workspace_bytes.argtypes = [I32, I64]
        L.givens_gemm_apply.restype = C
        L.givens_gemm_apply.argtypes = [I32, I64, P, P, P, I64, P, I64, C, P, I32, P, SZ, P]
        L.givens_gemm_backward.restype = C
        L.givens_gemm_backward.argtypes = [I32, I64, P, P, P, I64, P, I64, P, I64, P, C, P, I32, P, SZ, P]
        L.givens_check_perm.restype = C
        L.givens_check_perm.argtypes = [I32, P]
        L.givens_schedule_ex.restype = C
        L.givens_schedule_ex.argtypes = [I32, P, P, P]
        L.givens_mask_from_dims_ex.restype = C
        L.givens_mask_from_dims_ex.argtypes = [I32, P, P, P]
        L.givens_apply_ex.restype = C
        L.givens_apply_ex.argtypes = [I32, I64, P, P, P, I64, P, I64, C, P, I32, P, SZ, P]
        L.givens_build_U_ex.restype = C
        L.givens_build_U_ex.argtypes = [I32, P, P, P, I64, P, I32, P, SZ, P]
        L.givens_backward_ex.restype = C
        L.givens_backward_ex.argtypes = [I32, I64, P, P, P, I64, P, I64, P, I64, P, C, P, I32, P, SZ, P]
        L.givens_u_apply_ex.restype = C
        L.givens_u_apply_ex.argtypes = [I32, I64, P, P, P, P, I64, P, I64, C, P, I32, P, SZ, P]
        L.givens_u_build_U_ex.restype = C
        L.givens_u_build_U_ex.argtypes = [I32, P, P, P, P, I64, P, I32, P, SZ, P]
        L.givens_u_backward_ex.restype = C
        L.givens_u_backward_ex.argtypes = [I32, I64, P, P, P, P, I64, P, I64, P, I64, P, P, C, P, I32, P, SZ, P]
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != OK:
        raise GivensError(rc, lib().givens_last_error().decode())
