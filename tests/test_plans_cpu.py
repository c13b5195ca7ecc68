"""Serialized plans (tc_plan_save -> orc_plan_load): the committed files that bench.py's reference
arm executes on the CPU oracle are the plans the product compiles today (not stale), and a loaded
plan runs exactly like the in-memory one."""
import os
import tempfile

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1701_02284_b200 import _native as nat
from paper_1701_02284_b200.network import compile_network

import sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
from make_plans import PLANS, plan_path, write_plan  # noqa: E402


@pytest.mark.parametrize("name,batch,sample", PLANS)
def test_committed_plan_is_current(name, batch, sample):
    with tempfile.TemporaryDirectory() as d:
        fresh = os.path.join(d, "p.tcplan")
        write_plan(name, batch, sample, fresh)
        with open(fresh, "rb") as a, open(plan_path(name, sample), "rb") as b:
            assert a.read() == b.read(), f"{plan_path(name, sample)} is stale: run tools/make_plans.py"


def test_loaded_plan_runs_like_compiled():
    net = compile_network("lenet", 64, global_batch=64)
    pf = orc.PlanFile(plan_path("lenet", 64))
    assert pf.input_dims == net.input_dims
    assert [p.dims for p in pf.params] == [p.dims for p in net.params]
    a, b = orc.Oracle(net, seed=5), orc.Oracle(pf, seed=5)
    a.init_params()
    b.init_params()
    la = [a.step(it) for it in range(3)]
    lb = [b.step(it) for it in range(3)]
    assert la == lb
    x1, y1 = orc.synth_batch(net, 5, 2)
    x2, y2 = orc.synth_batch(pf, 5, 2)
    np.testing.assert_array_equal(x1, x2)
    np.testing.assert_array_equal(y1, y2)


def test_bad_plan_file_rejected():
    with tempfile.NamedTemporaryFile(suffix=".tcplan") as f:
        f.write(b"not a plan")
        f.flush()
        with pytest.raises(IOError):
            orc.PlanFile(f.name)
