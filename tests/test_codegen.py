"""Codegen: the emitted standalone training program is deterministic, carries
every IR statement as a comment above its one runtime call, has a one-line mode flag, snapshot
calls and a test procedure, and compiles + links against the runtime library alone."""
import os
import subprocess
import tempfile

import pytest

from paper_1701_02284_b200 import _native as nat
from paper_1701_02284_b200.network import compile_network

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_program(src: str, out: str) -> None:
    libdir = os.path.dirname(nat.LIB_PATH)
    with tempfile.NamedTemporaryFile("w", suffix=".cpp", delete=False) as f:
        f.write(src)
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), f.name,
                    "-L", libdir, "-ltcb200", f"-Wl,-rpath,{libdir}", "-o", out], check=True)
    os.unlink(f.name)


def test_codegen_structure_and_determinism():
    net = compile_network("lenet", 500)
    a = net.codegen()
    b = compile_network("lenet", 500).codegen()
    assert a == b  # byte-identical for an identical IrProgram
    lines = a.splitlines()
    n = net.plan.nstmts
    calls = [i for i, line in enumerate(lines) if "tc_exec_stmt(ctx, " in line]
    assert len(calls) == n  # one runtime call per IrStmt
    for k, i in enumerate(calls):  # each preceded by its Fig. 2 statement as a comment
        assert lines[i - 1].strip() == "// " + net.stmt_text(k)
    assert "// val X9 = Pooling(2,2,0,true)(X8)" in a  # SPEC.md:432 example
    assert sum("static const int kMode = TC_MODE_DEALLOC;" in line for line in lines) == 1
    assert "TC_MODE_REUSE;" in compile_network("lenet", 500).codegen(mode="reuse")
    assert "tc_snapshot_load" in a and "tc_snapshot_save" in a and "tc_test(" in a
    assert "tc_net_compile" not in a  # no dependency on the compiler


def test_codegen_program_compiles_and_links():
    net = compile_network("alexnet", 4)
    with tempfile.TemporaryDirectory() as d:
        build_program(net.codegen(iters=3), os.path.join(d, "alexnet_gen"))
        assert os.path.getsize(os.path.join(d, "alexnet_gen")) > 0
