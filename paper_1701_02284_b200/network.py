"""Python mirror of the plan-producer interface (tc_plan.h).

The reference's host interface is C++ (expr.hpp builders + the SPEC.md
compiler stages); this module only wraps the C ABI of this repo's own C++
implementation of it so tests and bench.py can drive it:

    net = compile_network("lenet", 500)      # elaborate + grad + IR + memplan
    print(net.ir_text())                      # --dump-ir
    print(net.memory_table())                 # analyze
    net.memory_summary().peak_dealloc_mb      # 59.167999 for Fig. 2
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _native as nat


@dataclass
class ParamInfo:
    index: int
    name: str
    dims: tuple
    init_kind: int
    init_value: float
    lr_mult: float
    decay_mult: float
    fan_in: int
    fan_out: int

    @property
    def count(self) -> int:
        n = 1
        for d in self.dims:
            n *= d
        return n


class CompiledNetwork:
    """A compiled network: IrProgram + memory report (owner of the tc_net handle)."""

    def __init__(self, name: str, batch: int, *, lr: float = 0.01, momentum: float = 0.9, decay: float = 0.0005,
                 clip: float = 0.0, mode: str = "dealloc", workspace_cap_mb: float = -1.0, greedy: bool = False,
                 global_batch: int = 0, spec: str | None = None, solver_from_spec: bool = False, cse: bool = True):
        L = nat.lib()
        opts = nat.CompileOpts(lr=lr, momentum=momentum, decay=decay, clip=clip,
                               mode=nat.TC_MODE_REUSE if mode == "reuse" else nat.TC_MODE_DEALLOC,
                               workspace_cap_mb=workspace_cap_mb, greedy_schedule=int(greedy),
                               global_batch=global_batch, no_cse=0 if cse else 1)
        h = C.c_void_p()
        if spec is None:
            nat.check(L.tc_net_compile(name.encode(), batch, C.byref(opts), C.byref(h)))
        else:
            nat.check(L.tc_net_compile_spec(spec.encode(), batch, None if solver_from_spec else C.byref(opts),
                                            C.byref(h)))
        self._h = h
        self.plan_ptr = L.tc_net_plan(h)
        self.plan = self.plan_ptr.contents
        self.name = self.plan.name.decode() if spec is not None else name
        self.batch = self.plan.batch

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and nat._lib is not None:
            nat._lib.tc_net_destroy(h)
            self._h = None

    # ---- reports
    def ir_text(self) -> str:
        return nat.lib().tc_net_ir_text(self._h).decode()

    def memory_table(self, csv: bool = False) -> str:
        return nat.lib().tc_net_memory_table(self._h, int(csv)).decode()

    def memory_summary(self) -> nat.MemSummary:
        s = nat.MemSummary()
        nat.check(nat.lib().tc_net_memory_summary(self._h, C.byref(s)))
        return s

    def verify(self) -> str:
        return nat.lib().tc_net_verify(self._h).decode()

    def stmt_text(self, i: int) -> str:
        return nat.lib().tc_net_stmt_text(self._h, i).decode()

    # ---- plan views
    @property
    def stmts(self):
        p = self.plan
        return [p.stmts[i] for i in range(p.nstmts)]

    @property
    def params(self) -> list[ParamInfo]:
        p = self.plan
        out = []
        for i in range(p.nparams):
            d = p.params[i]
            out.append(ParamInfo(i, d.name.decode(), tuple(d.dims[j] for j in range(d.rank)), d.init_kind,
                                 d.init_value, d.lr_mult, d.decay_mult, d.fan_in, d.fan_out))
        return out

    def var_dims(self, var: int) -> tuple:
        p = self.plan
        for i in range(p.nvars):
            v = p.vars[i]
            if v.id == var:
                return tuple(v.dims[j] for j in range(v.rank))
        raise KeyError(var)

    @property
    def input_dims(self) -> tuple:
        return tuple(self.plan.input_dims[i] for i in range(4))


    def codegen(self, mode: str = "dealloc", iters: int = 0, test_iters: int = -1) -> str:
        """Standalone C++ training program over the runtime library."""
        m = nat.TC_MODE_REUSE if mode == "reuse" else nat.TC_MODE_DEALLOC
        return nat.lib().tc_net_codegen(self._h, m, iters, test_iters).decode()

    def spec_info(self) -> dict:
        """Data-source seed and solver iteration counts of a spec-compiled network."""
        seed, it, ti = C.c_uint64(), C.c_int64(), C.c_int64()
        nat.check(nat.lib().tc_net_spec_info(self._h, C.byref(seed), C.byref(it), C.byref(ti)))
        return {"seed": seed.value, "iters": it.value, "test_iters": ti.value}


def compile_network(name: str, batch: int, **kw) -> CompiledNetwork:
    return CompiledNetwork(name, batch, **kw)


def compile_spec(text: str, batch: int = 0, **kw) -> CompiledNetwork:
    """parse_netspec + elaborate + compile: a user network from its text description.
    With no solver keyword the spec's own solver section is used."""
    solver_keys = {"lr", "momentum", "decay", "clip"}
    return CompiledNetwork("", batch, spec=text, solver_from_spec=not (solver_keys & kw.keys()), **kw)


def load_spec(path: str, batch: int = 0, **kw) -> CompiledNetwork:
    with open(path) as f:
        return compile_spec(f.read(), batch, **kw)
