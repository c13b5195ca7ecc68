"""Parity at the BENCHMARKED configuration (BASELINE.json configs; bench.py's plan).

bench.py runs the shared arena (keep=False), CUDA-graph replay, every default
producer fold, and the tile / split-K / CTA-pair choices the cost model makes at
the BASELINE batch sizes (AlexNet b128, VGG-16 b64, GoogLeNet b128, ResNet-50
b64).  These tests check exactly that configuration against the CPU oracle:

  * whole step, shared arena + graph replay + default folds, vs the oracle on the
    same parameters and batch: loss and every parameter gradient, judged against
    the bf16 rounding envelope of the step (sensitivity(): the same oracle with
    the device's bf16 storage emulated);
  * eager step == captured step == replayed step, bit for bit;
  * shared arena (keep=False, bench) == private ranges (keep=True, parity mode),
    bit for bit, at the BASELINE batch of every network;
  * per-op parity on identical inputs at the BASELINE shapes (AlexNet b128
    conv / data-gradient / filter-gradient / pool / LRN, VGG-16 b64 block 1):
    tensor-core ops within 1e-2 (north star), max-pool values bit-exact;
  * max-pool argmax indices bit-exact for the overlapping 3x3/2 and 3x3/1
    windows in both precisions.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as orc  # noqa: E402
from paper_1701_02284_b200 import _native as nat  # noqa: E402
from paper_1701_02284_b200.network import compile_network  # noqa: E402
from paper_1701_02284_b200.runtime import Trainer  # noqa: E402

from test_ops_gpu import final_alias, maxrel, oracle_op  # noqa: E402
from test_step_gpu import rel, sensitivity  # noqa: E402

pytestmark = pytest.mark.gpu
BASELINE_BATCH = {"alexnet": 128, "vgg16": 64, "googlenet": 128, "resnet50": 64}


def bench_trainer(net, seed):
    """The bench.py configuration: shared arena, graph replay, default folds."""
    tr = Trainer(net, keep=False, use_graph=True, seed=seed)
    tr.init_params()
    return tr


@pytest.mark.parametrize("name,batch", [("alexnet", 128), ("vgg16", 16), ("googlenet", 16), ("resnet50", 8)])
def test_bench_config_step_parity(name, batch):
    """One step of the bench plan (third launch = graph replay) vs the oracle."""
    seed = 11
    net = compile_network(name, batch)
    tr = bench_trainer(net, seed)
    x, y = orc.synth_batch(net, seed, 0)
    runs = []
    for _ in range(3):  # eager, capture + launch, replay
        tr.stage_batch(x, y)
        tr.step(0, update=False)
        runs.append((tr.loss(), [tr.grad(i) for i in range(len(net.params))]))
    for k in (1, 2):
        assert runs[k][0] == runs[0][0]
        for a, b in zip(runs[k][1], runs[0][1]):
            np.testing.assert_array_equal(a, b)
    lg, grads = runs[2]
    o = orc.Oracle(net, seed=seed)
    o.init_params()
    o.set_batch(x, y)
    lo = o.step(0, update=False)
    env, loss_env = sensitivity(net, x, y, seed=seed, with_loss=True)
    print(f"{name} b{batch}: loss device {lg:.6f} oracle {lo:.6f} (bf16 envelope {loss_env:.2e})")
    assert abs(lg - lo) <= max(1e-2 * abs(lo), 3 * loss_env), (lg, lo, loss_env)
    errs = [(rel(grads[i], o.grad(i)), env[i], p.name) for i, p in enumerate(net.params)]
    bad = [e for e in errs if e[0] > 3 * e[1] + 2e-2]
    print(name, "worst grad rel err", max(errs), "median", float(np.median([e[0] for e in errs])))
    assert not bad, bad[:5]


@pytest.mark.parametrize("name", ["alexnet", "vgg16", "googlenet", "resnet50"])
def test_shared_arena_bit_identical_to_keep(name):
    """Lifetime-shared arena offsets (bench) vs one private range per storage (parity mode):
    two update steps at the BASELINE batch give bit-identical losses, parameters, velocities."""
    batch = BASELINE_BATCH[name]
    net = compile_network(name, batch)
    outs = []
    for keep in (False, True):
        tr = Trainer(net, keep=keep, use_graph=True, seed=21)
        tr.init_params()
        losses = []
        for it in range(3):
            tr.stage_synthetic(it, 0)
            tr.step(it)
            losses.append(tr.loss())
        mem = tr.memory()
        outs.append((losses, [tr.get_param(i) for i in range(len(net.params))],
                     [tr.velocity(i) for i in range(len(net.params))], mem))
        tr.close()
    assert outs[0][3]["arena_bytes"] < outs[1][3]["arena_bytes"]  # the sharing is real
    assert outs[0][0] == outs[1][0], (outs[0][0], outs[1][0])
    for a, b in zip(outs[0][1] + outs[0][2], outs[1][1] + outs[1][2]):
        np.testing.assert_array_equal(a, b)


def per_op_check(net, tr, ops, limit_vars=None):
    """Oracle kernel on the device's own inputs for every statement of `ops`.  A result that a
    folded in-place ReLU (forward, or backward with its mask) overwrote is compared through that
    ReLU: the device value is the final alias, the reference gets the same ReLU applied."""
    final = final_alias(net)
    overwritten = {s.inp[0].index for s in net.stmts if s.kind == nat.TC_STMT_LET and s.inplace}
    succ = {s.inp[0].index: s for s in net.stmts if s.kind == nat.TC_STMT_LET and s.inplace}
    checked, failures = {}, []
    for s in net.stmts:
        if s.kind not in (nat.TC_STMT_LET, nat.TC_STMT_UPDATE):
            continue
        op = nat.OP_NAMES[s.op]
        if op not in ops:
            continue
        post = None
        if s.kind == nat.TC_STMT_LET and s.var not in final:
            t = succ.get(s.var)
            if t is None or t.var not in final or nat.OP_NAMES[t.op] not in ("RELU_FWD", "RELU_BWD"):
                continue
            post = t
        if any(s.inp[i].kind == nat.TC_REF_VAR and s.inp[i].index in overwritten and s.inp[i].index not in final
               for i in range(s.nin)):
            continue
        if limit_vars is not None and not limit_vars(s):
            continue
        ref = oracle_op(net, tr, s)
        if ref is None:
            continue
        if post is None:
            dev = tr.var(s.var) if s.kind == nat.TC_STMT_LET else tr.grad(s.param)
        elif nat.OP_NAMES[post.op] == "RELU_FWD":
            dev, ref = tr.var(post.var), np.maximum(ref, 0)
        else:
            dev, ref = tr.var(post.var), np.where(tr.var(post.inp[1].index) > 0, ref, 0)
        err = maxrel(dev, ref)
        checked[op] = checked.get(op, 0) + 1
        exact = op == "POOL_FWD" and s.max_pool
        if (exact and not np.array_equal(dev, ref)) or (not exact and err > 1e-2):
            failures.append((op, s.var, s.param, err))
    return checked, failures


def test_per_op_alexnet_b128():
    """Identical inputs at the headline shape: conv1-5 fwd / dgrad / wgrad (M = 86,528 for conv2,
    split-K and CTA-pair tiles as the cost model picks them at b128), pools, LRNs, FC grads."""
    net = compile_network("alexnet", 128)
    tr = Trainer(net, keep=True, use_graph=False, seed=5)
    tr.init_params()
    x, y = orc.synth_batch(net, 5, 0)
    tr.stage_batch(x, y)
    tr.step(0, update=False)
    ops = {"CONV_FWD", "CONV_BWD_DATA", "CONV_BWD_FILTER", "POOL_FWD", "POOL_BWD", "LRN_FWD", "LRN_BWD",
           "MATMUL_BWD_DATA", "MATMUL_BWD_W", "CONV_BWD_BIAS", "BIAS_GRAD"}
    checked, failures = per_op_check(net, tr, ops)
    print("alexnet b128 per-op checked", checked)
    assert not failures, failures
    assert checked.get("CONV_FWD", 0) >= 4 and checked.get("CONV_BWD_DATA", 0) >= 3
    assert checked.get("CONV_BWD_FILTER", 0) == 5 and checked.get("POOL_FWD", 0) == 3


def test_per_op_vgg16_b64_block1():
    """VGG-16 at its BASELINE batch: conv1_1 / conv1_2 (M = 3.2M pixels) fwd, dgrad, wgrad, pool1."""
    net = compile_network("vgg16", 64)
    tr = Trainer(net, keep=True, use_graph=False, seed=5)
    tr.init_params()
    x, y = orc.synth_batch(net, 5, 0)
    tr.stage_batch(x, y)
    tr.step(0, update=False)
    block1 = {0, 1, 2, 3}  # conv1_1 W/B, conv1_2 W/B

    def first_block(s):
        dims = tuple(s.dims[i] for i in range(s.rank)) if s.kind == nat.TC_STMT_LET else net.params[s.param].dims
        if s.kind == nat.TC_STMT_UPDATE:
            return s.param in block1
        if nat.OP_NAMES[s.op] == "POOL_FWD":
            return dims[2] == 112
        return len(dims) == 4 and dims[2] == 224  # 224x224 activations / their gradients

    checked, failures = per_op_check(net, tr, {"CONV_FWD", "CONV_BWD_DATA", "CONV_BWD_FILTER", "POOL_FWD",
                                               "CONV_BWD_BIAS"}, first_block)
    print("vgg16 b64 block-1 per-op checked", checked)
    assert not failures, failures
    assert checked.get("CONV_FWD", 0) == 2 and checked.get("CONV_BWD_FILTER", 0) == 2
    assert checked.get("CONV_BWD_DATA", 0) >= 1 and checked.get("POOL_FWD", 0) == 1


@pytest.mark.parametrize("precision", ["bf16", "f32"])
@pytest.mark.parametrize("name,batch", [("alexnet", 4), ("googlenet", 2)])
def test_pool_indices_bit_exact_overlapping(name, batch, precision):
    """Argmax indices of the overlapping windows (AlexNet 3x3/2; GoogLeNet 3x3/2 pad 0/1 and the
    inception 3x3/1 pad 1 pool branch) bit-exact against the oracle on the device's own input,
    in both storage precisions.  First maximum in row-major window order wins (ties: ReLU zeros)."""
    net = compile_network(name, batch)
    tr = Trainer(net, keep=True, use_graph=False, seed=11, precision=precision)
    tr.init_params()
    x, y = orc.synth_batch(net, 11, 0)
    tr.stage_batch(x, y)
    tr.step(0, update=False)
    L = orc.lib()
    windows = set()
    for s in net.stmts:
        if s.kind != nat.TC_STMT_LET or nat.OP_NAMES[s.op] != "POOL_FWD" or not s.max_pool:
            continue
        xin = np.ascontiguousarray(tr.var(s.inp[0].index))
        n, c, h, w = xin.shape
        ho, wo = net.var_dims(s.var)[2:]
        ref_y = np.empty((n, c, ho, wo), np.float32)
        ref_i = np.empty((n, c, ho, wo), np.int32)
        L.orc_pool_fwd_f32(xin, ref_y, ref_i.ctypes.data, n, c, h, w, s.k, s.stride, s.pad, 1)
        dev_i = tr.pool_indices(s.var)
        assert np.array_equal(dev_i, ref_i), (s.var, s.k, s.stride, s.pad, int((dev_i != ref_i).sum()))
        np.testing.assert_array_equal(tr.var(s.var), ref_y)
        ties = float(np.mean(ref_y == 0))
        windows.add((s.k, s.stride, s.pad))
        print(f"{name} {precision} pool X{s.var} {s.k}x{s.k}/{s.stride} pad {s.pad}: indices exact, "
              f"{ties:.1%} all-zero windows")
    assert (3, 2, 0) in windows or (3, 2, 1) in windows
    if name == "googlenet":
        assert (3, 1, 1) in windows


def test_nccl_one_rank_matches_no_comm():
    """The data-parallel path on one GPU: a 1-rank NCCL communicator runs the per-bucket gradient
    all-reduce and the loss all-reduce inside the captured graph; bit-identical to no comm."""
    from paper_1701_02284_b200.runtime import nccl_unique_id
    net = compile_network("alexnet", 16)
    outs = []
    for nid in (None, nccl_unique_id()):
        tr = Trainer(net, use_graph=True, seed=4, world=1, nccl_id=nid)
        tr.init_params()
        losses = []
        for it in range(4):
            tr.stage_synthetic(it, 0)
            tr.step(it)
            losses.append(tr.loss())
        outs.append((losses, [tr.get_param(i) for i in range(len(net.params))]))
        tr.close()
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1], outs[1][1]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_global_clip_matches_oracle(precision):
    """Solver clip > 0: global L2-norm scaling of g + decay p over the whole
    gradient, device vs oracle over 5 steps; the clip engages (it changes the trajectory)."""
    traj = {}
    for clip in (0.0, 0.05):
        net = compile_network("lenet", 16, clip=clip)
        tr = Trainer(net, keep=False, use_graph=True, seed=42, precision=precision)
        tr.init_params()
        o = orc.Oracle(net, seed=42)
        o.init_params()
        lg, lo = [], []
        for it in range(5):
            x, y = orc.synth_batch(net, 42, it)
            tr.stage_batch(x, y)
            tr.step(it)
            lg.append(tr.loss())
            o.set_batch(x, y)
            lo.append(o.step(it))
        traj[clip] = (np.array(lg), np.array(lo))
        p_dev, p_orc = tr.get_param(0), o.get_param(0)
        tol = 1e-4 if precision == "f32" else 2e-2
        assert rel(p_dev, p_orc) < tol, (clip, rel(p_dev, p_orc))
        assert np.max(np.abs(traj[clip][0] - traj[clip][1])) < (1e-4 if precision == "f32" else 2e-2)
    assert np.max(np.abs(traj[0.05][1] - traj[0.0][1])) > 1e-3  # clipping engaged
