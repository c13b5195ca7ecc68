"""Python mirror of the runtime interface (tc_runtime.h): the reference's
`train(p, data) -> loss trace` driver over the sm_100a
executor.  No CPU fallback: constructing a Trainer without a CUDA device or
without the built library raises.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from .network import CompiledNetwork


class Trainer:
    def __init__(self, net: CompiledNetwork, device: int = 0, seed: int = 42, use_graph: bool = True,
                 keep: bool = False, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 precision: str = "bf16"):
        L = nat.lib()
        self.net = net
        self._id_buf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        d = nat.CtxDesc(device=device, rank=rank, world=world,
                        nccl_id=C.cast(self._id_buf, C.c_void_p) if self._id_buf else None, seed=seed,
                        use_graph=int(use_graph), keep=int(keep),
                        precision=nat.TC_PREC_F32 if precision == "f32" else nat.TC_PREC_BF16)
        h = C.c_void_p()
        nat.check(L.tc_ctx_create(net.plan_ptr, C.byref(d), C.byref(h)))
        self._h = h
        self.params = net.params

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value and nat._lib is not None:
            nat._lib.tc_ctx_destroy(self._h)
        self._h = None

    def __del__(self):
        self.close()

    @property
    def stream(self) -> int:
        return nat.lib().tc_ctx_stream(self._h)

    # ---- parameters (reference layout, fp32)
    def init_params(self):
        nat.check(nat.lib().tc_init_params(self._h))

    def set_param(self, i: int, a):
        a = np.ascontiguousarray(a, np.float32)
        nat.check(nat.lib().tc_param_upload(self._h, i, a.ctypes.data))

    def _down(self, fn, i):
        out = np.empty(self.params[i].dims, np.float32)
        nat.check(getattr(nat.lib(), fn)(self._h, i, out.ctypes.data))
        return out

    def set_velocity(self, i: int, a):
        a = np.ascontiguousarray(a, np.float32)
        nat.check(nat.lib().tc_velocity_upload(self._h, i, a.ctypes.data))

    def get_param(self, i):
        return self._down("tc_param_download", i)

    def velocity(self, i):
        return self._down("tc_velocity_download", i)

    def grad(self, i):
        return self._down("tc_grad_download", i)

    # ---- data + step
    def stage_batch(self, x, y):
        x = np.ascontiguousarray(x, np.float32)
        y = np.ascontiguousarray(y, np.int32)
        # host buffers stay alive while their async copy may be in flight (two staging slots)
        self._staged = (getattr(self, "_staged", (None,))[-1], (x, y))
        nat.check(nat.lib().tc_stage_batch(self._h, x.ctypes.data, y.ctypes.data))

    @property
    def stage_bytes(self) -> int:
        """Bytes one stage_batch moves host -> device (bf16 images when rounded on the host)."""
        return int(nat.lib().tc_stage_bytes(self._h))

    def stage_synthetic(self, it: int, n0: int = 0):
        nat.check(nat.lib().tc_stage_synthetic(self._h, it, n0))

    def step(self, it: int = 0, n0: int = 0, update: bool = True):
        nat.check(nat.lib().tc_step(self._h, it, n0, int(update)))

    def exec_stmt(self, index: int, it: int = 0, n0: int = 0):
        nat.check(nat.lib().tc_exec_stmt(self._h, index, it, n0))

    def test(self, it: int = 0, n0: int = 0, data=None) -> float:
        """SPEC.md:497 test(p, data) -> precision over one batch: data = (x, y) host batch, or None
        for the on-device synthetic batch of iteration `it`."""
        if data is None:
            self.stage_synthetic(it, n0)
        else:
            self.stage_batch(*data)
        v = C.c_double()
        nat.check(nat.lib().tc_test(self._h, it, n0, C.byref(v)))
        return v.value

    def snapshot_save(self, directory: str) -> None:
        """`<dir>/<param>.ddt` (+ `.velocity.ddt`), SPEC.md:529 format."""
        nat.check(nat.lib().tc_snapshot_save(self._h, directory.encode()))

    def snapshot_load(self, directory: str) -> tuple[int, int]:
        """Resume / fine-tune: returns (loaded, missing) parameter counts."""
        a, b = C.c_int(), C.c_int()
        nat.check(nat.lib().tc_snapshot_load(self._h, directory.encode(), C.byref(a), C.byref(b)))
        return a.value, b.value

    def loss(self) -> float:
        v = C.c_double()
        nat.check(nat.lib().tc_loss(self._h, C.byref(v)))
        return v.value

    def loss_prev(self) -> float:
        """Loss of the step before the last one enqueued (waits for that step only)."""
        v = C.c_double()
        nat.check(nat.lib().tc_loss_prev(self._h, C.byref(v)))
        return v.value

    def sync(self):
        nat.check(nat.lib().tc_sync(self._h))

    def var(self, v: int) -> np.ndarray:
        dims = self.net.var_dims(v)
        out = np.empty(dims, np.float32)
        nat.check(nat.lib().tc_var_download(self._h, v, out.ctypes.data, out.size))
        return out

    def pool_indices(self, v: int) -> np.ndarray:
        dims = self.net.var_dims(v)
        out = np.empty(dims, np.int32)
        nat.check(nat.lib().tc_pool_indices_download(self._h, v, out.ctypes.data, out.size))
        return out

    def memory(self) -> dict:
        m = nat.RtMemory()
        nat.check(nat.lib().tc_memory(self._h, C.byref(m)))
        return {k: getattr(m, k) for k, _ in m._fields_}

    def profile_step(self, it: int = 0, n0: int = 0, update: bool = True) -> np.ndarray:
        """Per-statement device milliseconds of one eager step (CUDA events)."""
        out = np.zeros(self.net.plan.nstmts, np.float32)
        nat.check(nat.lib().tc_profile_step(self._h, it, n0, int(update), out.ctypes.data, out.size))
        return out

    def profile_launches(self) -> np.ndarray:
        """Kernels each statement launched in the last profile_step (0 = folded into its producer)."""
        out = np.zeros(self.net.plan.nstmts, np.int32)
        nat.lib().tc_profile_launches(self._h, out.ctypes.data, out.size)
        return out

    def profile_updates(self) -> np.ndarray:
        """Per-statement ms of the bucket all-reduce + momentum update it completed (last profile_step)."""
        out = np.zeros(self.net.plan.nstmts, np.float32)
        nat.lib().tc_profile_updates(self._h, out.ctypes.data, out.size)
        return out

    @property
    def launches_per_step(self) -> int:
        return nat.lib().tc_launches_per_step(self._h)

    def train(self, iters: int, data=None, start: int = 0) -> list[float]:
        """SPEC.md:497 train(p, data) -> loss trace.  data(it) -> (x, y) host batch,
        or None for the on-device synthetic generator."""
        trace = []
        for it in range(start, start + iters):
            if data is None:
                self.stage_synthetic(it)
            else:
                self.stage_batch(*data(it))
            self.step(it)
            trace.append(self.loss())
        return trace


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    nat.check(nat.lib().tc_nccl_unique_id(buf))
    return buf.raw
