"""ctypes binding of the C ABI declared in include/tc_abi.h (and tc_plan.h).

This is the reference-side binding a Python host would add for the B200
backend: plain pointers and sizes, no torch types cross the ABI.  torch is
only used by callers for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libtcb200.so")

TC_OK = 0
STATUS_NAMES = {
    0: "TC_OK", 1: "TC_SHAPE_FAULT", 2: "TC_POOL_EXHAUSTED", 3: "TC_INVALID_ARG", 4: "TC_CUDA_ERROR",
    5: "TC_NCCL_ERROR", 6: "TC_IO_ERROR", 7: "TC_FORMAT_ERROR", 8: "TC_INTERNAL", 9: "TC_COMPILE_ERROR",
}
TC_LAYOUT_K, TC_LAYOUT_MN = 0, 1
TC_DTYPE_BF16, TC_DTYPE_F32 = 0, 1


class TcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class GemmArgs(C.Structure):
    _fields_ = [
        ("M", C.c_int), ("N", C.c_int), ("K", C.c_int),
        ("a_layout", C.c_int), ("b_layout", C.c_int),
        ("A", C.c_void_p), ("lda", C.c_longlong),
        ("B", C.c_void_p), ("ldb", C.c_longlong),
        ("D", C.c_void_p), ("ldd", C.c_longlong),
        ("d_dtype", C.c_int),
        ("bias", C.c_void_p), ("relu", C.c_int),
        ("alpha", C.c_float), ("beta", C.c_float),
        ("splits", C.c_int),
        ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
    ]


class ConvDesc(C.Structure):
    _fields_ = [
        ("N", C.c_int), ("C", C.c_int), ("H", C.c_int), ("W", C.c_int),
        ("K", C.c_int), ("R", C.c_int), ("S", C.c_int),
        ("stride", C.c_int), ("pad", C.c_int),
        ("Ho", C.c_int), ("Wo", C.c_int),
        ("cs", C.c_int), ("ks", C.c_int),
    ]


_lib = None


def lib() -> C.CDLL:
    """Load the product library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"B200 backend library missing: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        L.tc_last_error.restype = C.c_char_p
        L.tc_build_info.restype = C.c_char_p
        L.tc_kernel_launch_count.restype = C.c_ulonglong
        L.tc_gemm_bf16.argtypes = [C.POINTER(GemmArgs), C.c_void_p]
        L.tc_gemm_workspace_bytes.argtypes = [C.POINTER(GemmArgs)]
        L.tc_gemm_workspace_bytes.restype = C.c_size_t
        L.tc_conv2d_fwd.argtypes = [C.POINTER(ConvDesc), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                    C.c_void_p, C.c_size_t, C.c_void_p]
        L.tc_conv2d_bwd_data.argtypes = [C.POINTER(ConvDesc), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_size_t, C.c_void_p]
        L.tc_conv2d_bwd_filter.argtypes = [C.POINTER(ConvDesc), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_size_t, C.c_void_p]
        L.tc_conv2d_workspace_bytes.argtypes = [C.POINTER(ConvDesc), C.c_int]
        L.tc_conv2d_workspace_bytes.restype = C.c_size_t
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != TC_OK:
        raise TcError(status, lib().tc_last_error().decode())


def last_error() -> str:
    return lib().tc_last_error().decode()
