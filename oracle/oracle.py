"""ctypes binding of the CPU ORACLE (oracle/tc_oracle.h).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py (cpu_baseline / --impl reference), never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libtc_oracle.so")
_lib = None

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


class PoolStats(C.Structure):
    _fields_ = [("allocs_from_os", C.c_int64), ("reuses", C.c_int64), ("releases", C.c_int64),
                ("live_bytes", C.c_int64), ("peak_bytes", C.c_int64), ("os_bytes", C.c_int64)]


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"oracle library missing: {LIB_PATH} (make -C oracle)")
        L = C.CDLL(LIB_PATH)
        for sfx, P in (("f32", _f32p), ("f64", _f64p)):
            ci = C.c_int
            getattr(L, f"orc_conv_fwd_{sfx}").argtypes = [P, P, C.c_void_p, P] + [ci] * 10
            getattr(L, f"orc_conv_bwd_data_{sfx}").argtypes = [P, P, P] + [ci] * 9
            getattr(L, f"orc_conv_bwd_filter_{sfx}").argtypes = [P, P, P] + [ci] * 9
            getattr(L, f"orc_conv_bwd_bias_{sfx}").argtypes = [P, P, ci, ci, ci]
            getattr(L, f"orc_pool_fwd_{sfx}").argtypes = [P, P, C.c_void_p] + [ci] * 8
            getattr(L, f"orc_pool_bwd_{sfx}").argtypes = [P, P, P] + [ci] * 8
            getattr(L, f"orc_lrn_fwd_{sfx}").argtypes = [P, P, ci, ci, ci, ci, C.c_double, C.c_double, C.c_double]
            getattr(L, f"orc_lrn_bwd_{sfx}").argtypes = [P, P, P, P, ci, ci, ci, ci, C.c_double, C.c_double,
                                                         C.c_double]
            getattr(L, f"orc_softmax_fwd_{sfx}").argtypes = [P, P, ci, ci]
            getattr(L, f"orc_softmax_bwd_{sfx}").argtypes = [P, P, P, ci, ci]
            getattr(L, f"orc_bn_fwd_{sfx}").argtypes = [P, P, P, P, ci, ci, ci, C.c_double]
            getattr(L, f"orc_bn_bwd_{sfx}").argtypes = [P, P, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, ci,
                                                        ci, ci, C.c_double]
            getattr(L, f"orc_matmul_{sfx}").argtypes = [P, P, P, ci, ci, ci, ci, ci]
        L.orc_create.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_int]
        L.orc_create.restype = C.c_void_p
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_init_params.argtypes = [C.c_void_p]
        L.orc_param_get.argtypes = [C.c_void_p, C.c_int, _f32p]
        L.orc_param_set.argtypes = [C.c_void_p, C.c_int, _f32p]
        L.orc_param_get_f64.argtypes = [C.c_void_p, C.c_int, _f64p]
        L.orc_param_set_f64.argtypes = [C.c_void_p, C.c_int, _f64p]
        L.orc_velocity_get.argtypes = [C.c_void_p, C.c_int, _f32p]
        L.orc_synth_batch.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_int, _f32p, _i32p]
        L.orc_set_batch.argtypes = [C.c_void_p, _f32p, _i32p]
        L.orc_step.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]
        L.orc_step.restype = C.c_double
        L.orc_test.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.orc_test.restype = C.c_double
        L.orc_var_get.argtypes = [C.c_void_p, C.c_int, _f32p, C.c_int64]
        L.orc_grad_get.argtypes = [C.c_void_p, C.c_int, _f64p, C.c_int64]
        L.orc_pool_stats_get.argtypes = [C.c_void_p, C.POINTER(PoolStats)]
        L.orc_live_trace.argtypes = [C.c_void_p, np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS"), C.c_int]
        L.orc_set_workspace_cap.argtypes = [C.c_void_p, C.c_double]
        L.orc_set_bf16_storage.argtypes = [C.c_void_p, C.c_int]
        L.orc_plan_load.argtypes = [C.c_char_p]
        L.orc_plan_load.restype = C.c_void_p
        L.orc_plan_free.argtypes = [C.c_void_p]
        L.orc_plan_param_dims.argtypes = [C.c_void_p, C.c_int, np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")]
        L.orc_plan_input_dims.argtypes = [C.c_void_p, np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")]
        _lib = L
    return _lib


def _plan_addr(net) -> int:
    return net.plan_address if isinstance(net, PlanFile) else C.addressof(net.plan)


class _Shape:
    def __init__(self, dims):
        self.dims = tuple(int(d) for d in dims)


class PlanFile:
    """A plan serialized by the product's tc_plan_save, loaded by the oracle alone (bench.py's
    reference arm times the CPU path without loading the product library)."""

    def __init__(self, path: str):
        L = lib()
        self.plan_address = L.orc_plan_load(path.encode())
        if not self.plan_address:
            raise IOError(f"cannot load plan file {path}")
        d = np.zeros(4, np.int64)
        L.orc_plan_input_dims(self.plan_address, d)
        self.input_dims = tuple(int(v) for v in d)
        self.batch = self.input_dims[0]
        self.params = []
        i = 0
        while True:
            r = L.orc_plan_param_dims(self.plan_address, i, d)
            if r < 0:
                break
            self.params.append(_Shape(d[:r]))
            i += 1

    def __del__(self):
        if getattr(self, "plan_address", None) and _lib is not None:
            _lib.orc_plan_free(self.plan_address)
            self.plan_address = None


def synth_batch(net, seed: int, it: int, n0: int = 0):
    """Synthetic (x, labels) of iteration `it` for global samples [n0, n0+batch) (tc_philox.h)."""
    dims = net.input_dims
    x = np.empty(dims, np.float32)
    y = np.empty(dims[0], np.int32)
    lib().orc_synth_batch(_plan_addr(net), seed, it, n0, x, y)
    return x, y


class Oracle:
    """Reference CPU runtime executing a CompiledNetwork's plan (NCHW, fp32 or fp64)."""

    def __init__(self, net, seed: int = 42, f64: bool = False, threads: int = 0):
        self.net = net
        self.f64 = f64
        self._c = lib().orc_create(_plan_addr(net), seed, int(f64), threads)
        self.params = net.params

    def __del__(self):
        c = getattr(self, "_c", None)
        if c and _lib is not None:
            _lib.orc_destroy(c)
            self._c = None

    def init_params(self):
        lib().orc_init_params(self._c)

    def get_param(self, i: int) -> np.ndarray:
        p = self.params[i]
        out = np.empty(p.dims, np.float64 if self.f64 else np.float32)
        (lib().orc_param_get_f64 if self.f64 else lib().orc_param_get)(self._c, i, out)
        return out

    def set_param(self, i: int, a) -> None:
        if self.f64:
            lib().orc_param_set_f64(self._c, i, np.ascontiguousarray(a, np.float64))
        else:
            lib().orc_param_set(self._c, i, np.ascontiguousarray(a, np.float32))

    def velocity(self, i: int) -> np.ndarray:
        out = np.empty(self.params[i].dims, np.float32)
        lib().orc_velocity_get(self._c, i, out)
        return out

    def set_batch(self, x, y) -> None:
        lib().orc_set_batch(self._c, np.ascontiguousarray(x, np.float32), np.ascontiguousarray(y, np.int32))

    def step(self, it: int = 0, n0: int = 0, update: bool = True, keep: bool = False) -> float:
        return lib().orc_step(self._c, it, n0, int(update), int(keep))

    def test(self, it: int = 0, n0: int = 0) -> float:
        return lib().orc_test(self._c, it, n0)

    def var(self, v: int) -> np.ndarray:
        dims = self.net.var_dims(v)
        out = np.empty(dims, np.float32)
        r = lib().orc_var_get(self._c, v, out, out.size)
        if r < 0:
            raise KeyError(f"X{v} not live in the oracle ({r})")
        return out

    def grad(self, i: int) -> np.ndarray:
        out = np.empty(self.params[i].dims, np.float64)
        lib().orc_grad_get(self._c, i, out, out.size)
        return out

    def pool_stats(self) -> PoolStats:
        s = PoolStats()
        lib().orc_pool_stats_get(self._c, C.byref(s))
        return s

    def live_trace(self) -> np.ndarray:
        out = np.zeros(self.net.plan.nstmts, np.int64)
        n = lib().orc_live_trace(self._c, out, out.size)
        return out[:n]

    def set_workspace_cap(self, mb: float) -> None:
        lib().orc_set_workspace_cap(self._c, mb)

    def set_bf16_storage(self, on: bool = True) -> None:
        """Emulate the device's bf16 activation storage / bf16 weight operands."""
        lib().orc_set_bf16_storage(self._c, int(on))
