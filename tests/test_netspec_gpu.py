"""A user network from its text description (nets/smallnet.net, not one of the built-in names)
through tc_net_compile_spec -> tc_ctx_create -> tc_step, against the oracle on the same plan:
per-op parity on identical inputs (bf16 tensor-core / storage ops within 1e-2, max-pool values
bit-exact), pool indices bit-exact, and a 40-step training trajectory in the fp32 mode."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as orc  # noqa: E402
from paper_1701_02284_b200 import _native as nat  # noqa: E402
from paper_1701_02284_b200.network import load_spec  # noqa: E402
from paper_1701_02284_b200.runtime import Trainer  # noqa: E402

from test_bench_config_gpu import per_op_check  # noqa: E402

pytestmark = pytest.mark.gpu
SPEC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "nets", "smallnet.net")


def test_user_network_per_op_parity():
    net = load_spec(SPEC)
    tr = Trainer(net, keep=True, use_graph=False, seed=3)
    tr.init_params()
    x, y = orc.synth_batch(net, 3, 0)
    tr.stage_batch(x, y)
    tr.step(0, update=False)
    ops = {"CONV_FWD", "CONV_BWD_DATA", "CONV_BWD_FILTER", "POOL_FWD", "POOL_BWD", "LRN_FWD", "LRN_BWD",
           "MATMUL_BWD_DATA", "MATMUL_BWD_W", "CONV_BWD_BIAS", "BIAS_GRAD", "SOFTMAX_FWD", "SOFTMAX_BWD"}
    checked, failures = per_op_check(net, tr, ops)
    print("smallnet per-op checked", checked)
    assert not failures, failures
    assert checked.get("CONV_FWD", 0) == 2 and checked.get("LRN_BWD", 0) == 1
    L = orc.lib()
    for s in net.stmts:
        if s.kind == nat.TC_STMT_LET and nat.OP_NAMES[s.op] == "POOL_FWD" and s.max_pool:
            xin = np.ascontiguousarray(tr.var(s.inp[0].index))
            ref_y = np.empty(net.var_dims(s.var), np.float32)
            ref_i = np.empty(net.var_dims(s.var), np.int32)
            L.orc_pool_fwd_f32(xin, ref_y, ref_i.ctypes.data, *xin.shape, s.k, s.stride, s.pad, 1)
            np.testing.assert_array_equal(tr.pool_indices(s.var), ref_i)


def test_user_network_trajectory_f32():
    """40 fp32-mode steps of the user network vs the oracle, judged like the BASELINE networks'
    trajectories (test_trajectory_gpu.py): within max(1e-3, 3 x) the oracle's own deviation from
    its 1e-4-perturbed twin at every step."""
    from test_trajectory_gpu import trajectory
    net = load_spec(SPEC)
    lg, lo, lp = trajectory("smallnet", 0, 40, seed=net.spec_info()["seed"], net=net)
    d = np.maximum.accumulate(np.abs(lg - lo))
    e = np.maximum.accumulate(np.abs(lo - lp))
    print(f"smallnet f32 40 steps: max|device - oracle| = {d[-1]:.2e}, envelope {e[-1]:.2e}, "
          f"loss {lo[0]:.4f} -> {lo[-1]:.4f}")
    assert abs(lg[0] - lo[0]) <= 1e-5 * abs(lo[0])
    assert all(d[k] <= max(1e-3, 3 * e[k]) for k in range(40)), list(zip(d, e))
