"""SURVEY.md §8(f) rows on the device: the test body (precision), snapshot / resume (.ddt), and
the generated standalone program (codegen) against the in-process interpreter."""
import os
import struct
import subprocess
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as orc  # noqa: E402
from paper_1701_02284_b200 import _native as nat  # noqa: E402
from paper_1701_02284_b200.network import compile_network  # noqa: E402
from paper_1701_02284_b200.runtime import Trainer  # noqa: E402

from test_codegen import build_program  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,batch,precision", [("lenet", 64, "f32"), ("alexnet", 16, "f32"), ("lenet", 64, "bf16")])
def test_precision_matches_oracle(name, batch, precision):
    """test(p, data) -> precision (test-mode dropout = identity): after some
    training, the device's argmax-match fraction equals the oracle's on the same parameters."""
    net = compile_network(name, batch)
    tr = Trainer(net, keep=False, use_graph=True, seed=42, precision=precision)
    tr.init_params()
    for it in range(15):
        tr.stage_synthetic(it)
        tr.step(it)
    o = orc.Oracle(net, seed=42)
    for i in range(len(net.params)):
        o.set_param(i, tr.get_param(i))
    precs = []
    for it in range(100, 104):
        x, y = orc.synth_batch(net, 42, it)
        pd = tr.test(it, data=(x, y))
        o.set_batch(x, y)
        po = o.test(it)
        precs.append((pd, po))
    print(name, precision, "precision device/oracle", precs)
    tol = 0.0 if precision == "f32" else 2.0 / batch
    assert all(abs(a - b) <= tol + 1e-12 for a, b in precs), precs
    # training continues unaffected after a test pass (graph replay still valid)
    tr.stage_synthetic(200)
    tr.step(200)
    assert np.isfinite(tr.loss())


def test_precision_on_perfect_predictions():
    """SPEC.md:500 example: predictions = labels -> 1.0.  A trained LeNet separates the
    synthetic blobs (K Gaussian blobs, sigma 0.1) on held-out batches."""
    net = compile_network("lenet", 64)
    tr = Trainer(net, seed=42)
    tr.init_params()
    tr.train(100)
    precs = [tr.test(500 + k) for k in range(4)]
    print("lenet precision after 100 steps", precs)
    assert min(precs) >= 0.95 and max(precs) == 1.0


def test_snapshot_roundtrip_and_resume(tmp_path):
    net = compile_network("alexnet", 8)
    a = Trainer(net, use_graph=True, seed=3)
    a.init_params()
    for it in range(3):
        a.stage_synthetic(it)
        a.step(it)
    snap = str(tmp_path / "snap")
    a.snapshot_save(snap)
    cont = []
    for it in range(3, 6):
        a.stage_synthetic(it)
        a.step(it)
        cont.append(a.loss())
    # file format: DDSL | u32 1 | u32 rank | u32 dims | f32 LE
    raw = open(os.path.join(snap, "cv1_W.ddt"), "rb").read()
    assert raw[:4] == b"DDSL" and struct.unpack("<II", raw[4:12]) == (1, 4)
    assert struct.unpack("<4I", raw[12:28]) == (96, 3, 11, 11) and len(raw) == 28 + 4 * 96 * 3 * 11 * 11
    b = Trainer(net, use_graph=True, seed=3)  # same data / dropout seed; state comes from the snapshot
    b.init_params()
    for i, p in enumerate(net.params):  # clobber, so everything that matters must come from the files
        b.set_param(i, np.full(p.dims, 0.5, np.float32))
    assert b.snapshot_load(snap) == (len(net.params), 0)
    for i, p in enumerate(net.params):  # bit-exact roundtrip of the saved state
        w = np.fromfile(os.path.join(snap, p.name + ".ddt"), dtype="<f4", offset=12 + 4 * len(p.dims))
        np.testing.assert_array_equal(b.get_param(i).ravel(), w)
    res = []
    for it in range(3, 6):
        b.stage_synthetic(it)
        b.step(it)
        res.append(b.loss())
    assert res == cont  # resumed training continues bit-exactly (params + momentum state)


def test_snapshot_partial_and_corrupt(tmp_path):
    net = compile_network("lenet", 16)
    a = Trainer(net, seed=3)
    a.init_params()
    snap = str(tmp_path / "s")
    a.snapshot_save(snap)
    os.remove(os.path.join(snap, "fc2_W.ddt"))
    os.remove(os.path.join(snap, "fc2_B.ddt"))
    open(os.path.join(snap, "extra.ddt"), "wb").write(b"DDSL")  # extras are ignored
    b = Trainer(net, seed=77)
    b.init_params()
    fresh = b.get_param(6)
    assert b.snapshot_load(snap) == (len(net.params) - 2, 2)  # fc2 keeps its fresh init
    np.testing.assert_array_equal(b.get_param(6), fresh)
    np.testing.assert_array_equal(b.get_param(0), a.get_param(0))
    with open(os.path.join(snap, "cv1_W.ddt"), "r+b") as f:
        f.write(b"XXXX")
    with pytest.raises(nat.TcError) as e:
        b.snapshot_load(snap)
    assert e.value.status == nat.TC_FORMAT_ERROR and "cv1_W.ddt" in str(e.value)


def test_generated_program_matches_interpreter(tmp_path):
    """the generated program, 5 iterations with a fixed seed, prints the losses of the
    in-process interpreter (per-statement tc_exec_stmt) and of the whole-step path (1e-5)."""
    net = compile_network("alexnet", 8)
    exe = str(tmp_path / "gen")
    build_program(net.codegen(iters=5, test_iters=1), exe)
    out = subprocess.run([exe, "5"], capture_output=True, text=True, check=True, env=dict(os.environ, TENSORC_SEED="42"))
    gen = [float(line.split(",")[1]) for line in out.stdout.splitlines() if "," in line]
    assert len(gen) == 5
    interp = Trainer(net, use_graph=False, seed=42)
    interp.init_params()
    step = Trainer(net, use_graph=True, seed=42)
    step.init_params()
    li, ls = [], []
    for it in range(5):
        interp.stage_synthetic(it)
        for k in range(net.plan.nstmts):
            interp.exec_stmt(k, it)
        li.append(interp.loss())
        step.stage_synthetic(it)
        step.step(it)
        ls.append(step.loss())
    print("generated", gen, "interpreter", li, "whole step", ls)
    np.testing.assert_allclose(gen, li, rtol=1e-6)
    np.testing.assert_allclose(gen, ls, rtol=1e-5)
    assert "precision" in out.stdout
