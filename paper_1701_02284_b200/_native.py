"""ctypes binding of the C ABI declared in include/tc_abi.h (and tc_plan.h).

This is the reference-side binding a Python host would add for the B200
backend: plain pointers and sizes, no torch types cross the ABI.  torch is
only used by callers for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# TCB_LIB_VARIANT=<name> loads _lib/libtcb200_<name>.so (kernel A/B experiments)
LIB_PATH = os.path.join(_HERE, "_lib", "libtcb200" + (f"_{os.environ['TCB_LIB_VARIANT']}" if os.environ.get(
    "TCB_LIB_VARIANT") else "") + ".so")

TC_OK = 0
(TC_SHAPE_FAULT, TC_POOL_EXHAUSTED, TC_INVALID_ARG, TC_CUDA_ERROR, TC_NCCL_ERROR, TC_IO_ERROR,
 TC_FORMAT_ERROR, TC_INTERNAL, TC_COMPILE_ERROR) = range(1, 10)
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
        ("bias_n", C.c_int), ("b_rows", C.c_int), ("relu_mask", C.c_void_p), ("mask_ld", C.c_longlong),
    ]


class ConvDesc(C.Structure):
    _fields_ = [
        ("N", C.c_int), ("C", C.c_int), ("H", C.c_int), ("W", C.c_int),
        ("K", C.c_int), ("R", C.c_int), ("S", C.c_int),
        ("stride", C.c_int), ("pad", C.c_int),
        ("Ho", C.c_int), ("Wo", C.c_int),
        ("cs", C.c_int), ("ks", C.c_int), ("wld", C.c_int),
    ]


TC_MAX_IN = 8
TC_STMT_LET, TC_STMT_DEALLOC, TC_STMT_UPDATE, TC_STMT_PRINT = 0, 1, 2, 3
TC_REF_NONE, TC_REF_VAR, TC_REF_PARAM = 0, 1, 2
TC_MODE_REUSE, TC_MODE_DEALLOC = 0, 1
OP_NAMES = [
    "NONE", "LOAD_X", "LOAD_Y", "CONV_FWD", "CONV_BWD_DATA", "CONV_BWD_FILTER", "CONV_BWD_BIAS", "POOL_FWD",
    "POOL_BWD", "RELU_FWD", "RELU_BWD", "SOFTMAX_FWD", "SOFTMAX_BWD", "LRN_FWD", "LRN_BWD", "DROPOUT_MASK", "MUL",
    "ADD", "MATMUL_FWD", "MATMUL_BWD_DATA", "MATMUL_BWD_W", "BIAS_ADD", "BIAS_GRAD", "LOG", "RECIP", "SCALE",
    "CONCAT", "CONCAT_BWD", "BN_FWD", "BN_BWD_DATA", "BN_BWD_GAMMA", "BN_BWD_BETA", "PRINT_LOSS",
]


class Ref(C.Structure):
    _fields_ = [("kind", C.c_int), ("index", C.c_int)]


class Stmt(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("op", C.c_int), ("var", C.c_int), ("storage", C.c_int), ("inplace", C.c_int),
        ("param", C.c_int), ("nin", C.c_int), ("inp", Ref * TC_MAX_IN), ("rank", C.c_int),
        ("dims", C.c_int64 * 4), ("bytes", C.c_int64),
        ("k", C.c_int), ("stride", C.c_int), ("pad", C.c_int), ("max_pool", C.c_int), ("has_bias", C.c_int),
        ("lrn_size", C.c_int), ("slot", C.c_int),
        ("alpha", C.c_double), ("beta", C.c_double), ("lrn_k", C.c_double), ("rate", C.c_double),
        ("scale", C.c_double), ("eps", C.c_double), ("offset", C.c_int64), ("extent", C.c_int64),
        ("lr_alpha", C.c_double), ("momentum", C.c_double), ("decay", C.c_double),
        ("nterms", C.c_int), ("coef", C.c_double * 4),
    ]


class ParamDesc(C.Structure):
    _fields_ = [
        ("name", C.c_char * 64), ("rank", C.c_int), ("dims", C.c_int64 * 4), ("init_kind", C.c_int),
        ("init_value", C.c_double), ("sigma", C.c_double), ("lr_mult", C.c_double), ("decay_mult", C.c_double),
        ("fan_in", C.c_int64), ("fan_out", C.c_int64),
    ]


class VarDesc(C.Structure):
    _fields_ = [("id", C.c_int), ("rank", C.c_int), ("dims", C.c_int64 * 4)]


class Plan(C.Structure):
    _fields_ = [
        ("name", C.c_char_p), ("batch", C.c_int64), ("classes", C.c_int64), ("input_dims", C.c_int64 * 4),
        ("nparams", C.c_int), ("params", C.POINTER(ParamDesc)),
        ("nstmts", C.c_int), ("stmts", C.POINTER(Stmt)),
        ("ntest", C.c_int), ("test_stmts", C.POINTER(Stmt)), ("logits_var", C.c_int),
        ("nvars", C.c_int), ("vars", C.POINTER(VarDesc)), ("max_var", C.c_int),
        ("lr", C.c_double), ("momentum", C.c_double), ("decay", C.c_double), ("clip", C.c_double),
        ("mode", C.c_int),
    ]


class MemSummary(C.Structure):
    _fields_ = [
        ("peak_dealloc_mb", C.c_double), ("peak_reuse_mb", C.c_double), ("param_mb", C.c_double),
        ("workspace_mb", C.c_double), ("peak_dealloc_bytes", C.c_int64), ("peak_reuse_bytes", C.c_int64),
        ("param_bytes", C.c_int64), ("workspace_bytes", C.c_int64),
    ]


class CompileOpts(C.Structure):
    _fields_ = [
        ("lr", C.c_double), ("momentum", C.c_double), ("decay", C.c_double), ("clip", C.c_double),
        ("mode", C.c_int), ("workspace_cap_mb", C.c_double), ("greedy_schedule", C.c_int),
        ("global_batch", C.c_int64), ("no_cse", C.c_int),
    ]


class CtxDesc(C.Structure):
    _fields_ = [("device", C.c_int), ("rank", C.c_int), ("world", C.c_int), ("nccl_id", C.c_void_p),
                ("seed", C.c_uint64), ("use_graph", C.c_int), ("keep", C.c_int), ("precision", C.c_int)]


TC_PREC_BF16, TC_PREC_F32 = 0, 1


class RtMemory(C.Structure):
    _fields_ = [("arena_bytes", C.c_int64), ("arena_keep_bytes", C.c_int64), ("param_bytes", C.c_int64),
                ("workspace_bytes", C.c_int64), ("input_bytes", C.c_int64), ("device_used_bytes", C.c_int64)]


_lib = None


def _bind_runtime(L: C.CDLL) -> None:
    vp, ci = C.c_void_p, C.c_int
    L.tc_ctx_create.argtypes = [vp, C.POINTER(CtxDesc), C.POINTER(vp)]
    L.tc_ctx_destroy.argtypes = [vp]
    L.tc_ctx_destroy.restype = None
    L.tc_ctx_stream.argtypes = [vp]
    L.tc_ctx_stream.restype = vp
    for fn in ("tc_param_upload", "tc_param_download", "tc_velocity_download", "tc_grad_download"):
        getattr(L, fn).argtypes = [vp, ci, vp]
    L.tc_init_params.argtypes = [vp]
    L.tc_stage_batch.argtypes = [vp, vp, vp]
    L.tc_stage_bytes.argtypes = [vp]
    L.tc_stage_bytes.restype = C.c_int64
    L.tc_stage_synthetic.argtypes = [vp, ci, ci]
    L.tc_step.argtypes = [vp, ci, ci, ci]
    L.tc_exec_stmt.argtypes = [vp, ci, ci, ci]
    L.tc_loss.argtypes = [vp, C.POINTER(C.c_double)]
    L.tc_loss_prev.argtypes = [vp, C.POINTER(C.c_double)]
    L.tc_var_download.argtypes = [vp, ci, vp, C.c_int64]
    L.tc_pool_indices_download.argtypes = [vp, ci, vp, C.c_int64]
    L.tc_sync.argtypes = [vp]
    L.tc_memory.argtypes = [vp, C.POINTER(RtMemory)]
    L.tc_launches_per_step.argtypes = [vp]
    L.tc_nccl_unique_id.argtypes = [vp]
    L.tc_profile_step.argtypes = [vp, ci, ci, ci, vp, ci]
    L.tc_profile_launches.argtypes = [vp, vp, ci]
    L.tc_profile_updates.argtypes = [vp, vp, ci]
    L.tc_test.argtypes = [vp, ci, ci, C.POINTER(C.c_double)]
    L.tc_velocity_upload.argtypes = [vp, ci, vp]
    L.tc_ctx_plan.argtypes = [vp]
    L.tc_ctx_plan.restype = vp
    L.tc_snapshot_save.argtypes = [vp, C.c_char_p]
    L.tc_snapshot_load.argtypes = [vp, C.c_char_p, C.POINTER(ci), C.POINTER(ci)]


def _bind_plan(L: C.CDLL) -> None:
    L.tc_net_compile.argtypes = [C.c_char_p, C.c_int64, C.POINTER(CompileOpts), C.POINTER(C.c_void_p)]
    L.tc_net_compile_spec.argtypes = [C.c_char_p, C.c_int64, C.POINTER(CompileOpts), C.POINTER(C.c_void_p)]
    L.tc_net_spec_info.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.tc_plan_save.argtypes = [C.POINTER(Plan), C.c_char_p]
    L.tc_net_codegen.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int64]
    L.tc_net_codegen.restype = C.c_char_p
    L.tc_net_destroy.argtypes = [C.c_void_p]
    L.tc_net_destroy.restype = None
    L.tc_net_plan.argtypes = [C.c_void_p]
    L.tc_net_plan.restype = C.POINTER(Plan)
    for fn in ("tc_net_ir_text", "tc_net_verify"):
        getattr(L, fn).argtypes = [C.c_void_p]
        getattr(L, fn).restype = C.c_char_p
    L.tc_net_memory_table.argtypes = [C.c_void_p, C.c_int]
    L.tc_net_memory_table.restype = C.c_char_p
    L.tc_net_stmt_text.argtypes = [C.c_void_p, C.c_int]
    L.tc_net_stmt_text.restype = C.c_char_p
    L.tc_net_memory_summary.argtypes = [C.c_void_p, C.POINTER(MemSummary)]


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
        _bind_plan(L)
        _bind_runtime(L)
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != TC_OK:
        raise TcError(status, lib().tc_last_error().decode())


def last_error() -> str:
    return lib().tc_last_error().decode()
