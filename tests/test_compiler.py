"""Plan producers: shape rules, gradient derivation shape
(SPEC.md:206), IR verifier (acceptance 4), update formation
 and the flattened plan crossing the C ABI."""
import numpy as np
import pytest

from paper_1701_02284_b200 import _native as nat
from paper_1701_02284_b200.network import compile_network

NETS = [("lenet", 64), ("alexnet", 8), ("vgg16", 2), ("googlenet", 2), ("resnet50", 2), ("inception", 4)]


@pytest.mark.parametrize("name,batch", NETS)
def test_ir_verifier(name, batch):
    net = compile_network(name, batch)
    assert net.verify() == ""


@pytest.mark.parametrize("name,batch", [("lenet", 64), ("alexnet", 4), ("inception", 4)])
def test_greedy_schedule_is_valid(name, batch):
    net = compile_network(name, batch, greedy=True)
    assert net.verify() == ""


def test_shape_examples():
    net = compile_network("lenet", 500)
    ir = net.ir_text()
    # conv k5 on 28 -> 24, pool -> 12, conv -> 8, pool -> 4, flatten -> 800
    assert "val X8 = Convolv(1,0)(X7,cv1_W,cv1_B)    # 500 20 24 24" in ir
    assert "val X9 = Pooling(2,2,0,true)(X8)    # 500 20 12 12" in ir
    assert "val X10 = Convolv(1,0)(X9,cv2_W,cv2_B)    # 500 50 8 8" in ir
    assert net.params[4].dims == (500, 800)  # fc1_W (500, 50*4*4)


def test_alexnet_shapes():
    net = compile_network("alexnet", 128)
    dims = {p.name: p.dims for p in net.params}
    assert dims["cv1_W"] == (96, 3, 11, 11)
    assert dims["fc6_W"] == (4096, 6400)  # pool5 256 x 5 x 5 at 224 input, floor pooling
    total = sum(p.count for p in net.params)
    assert 50.8e6 < total < 50.9e6  # 50.84 M


def test_param_counts():
    counts = {n: sum(p.count for p in compile_network(n, 2).params) for n in ("vgg16", "googlenet", "resnet50")}
    assert 138.3e6 < counts["vgg16"] < 138.4e6
    assert 13.3e6 < counts["googlenet"] < 13.5e6
    assert 25.5e6 < counts["resnet50"] < 25.6e6


def test_every_param_updated_once():
    # every parameter appears in exactly one Update
    for name, batch in NETS:
        net = compile_network(name, batch)
        ups = [s.param for s in net.stmts if s.kind == nat.TC_STMT_UPDATE]
        assert sorted(ups) == list(range(len(net.params))), name


def test_update_form():
    net = compile_network("lenet", 64, lr=0.01, momentum=0.9, decay=0.0005)
    ups = {s.param: s for s in net.stmts if s.kind == nat.TC_STMT_UPDATE}
    u = ups[0]
    assert u.lr_alpha == pytest.approx(-0.01) and u.momentum == pytest.approx(0.9) and u.decay == pytest.approx(0.0005)


def test_googlenet_multipliers_and_loss_heads():
    net = compile_network("googlenet", 2)
    p = {q.name: q for q in net.params}
    assert p["cv11_B"].lr_mult == 2.0 and p["cv11_B"].decay_mult == 0.0  # Param.const(0.2f, 2, 0)
    assert p["cv11_B"].init_value == pytest.approx(0.2)
    pr = [s for s in net.stmts if s.kind == nat.TC_STMT_PRINT][0]
    assert pr.nterms == 3
    assert sorted(round(pr.coef[i] * 2, 6) for i in range(3)) == [-1.0, -0.3, -0.3]


def test_dataflow_order_conv_data_grad_before_weight_update():
    # X72 reads cv2_W before cv2_W <~~ updates it in place.
    net = compile_network("alexnet", 2)
    seen_update = set()
    for s in net.stmts:
        if s.kind == nat.TC_STMT_UPDATE:
            seen_update.add(s.param)
        elif s.kind == nat.TC_STMT_LET:
            for i in range(s.nin):
                if s.inp[i].kind == nat.TC_REF_PARAM:
                    assert s.inp[i].index not in seen_update


def test_compile_error_unknown_network():
    with pytest.raises(nat.TcError) as e:
        compile_network("nosuchnet", 2)
    assert "UnboundName" in str(e.value)


def test_cse_merges_duplicate_subexpressions():
    """SPEC.md:313-319 cse: the same full layer applied twice to the same activations compiles to
    one MatMul / BiasAdd Let pair (statement-count oracle), the built-in networks (no duplicates)
    are unchanged, `.copy` operands are never merged (both Log S.copy and 1/(S.copy) remain), and
    the merged program computes the same loss and gradients (value oracle, CPU)."""
    from oracle import oracle as orc

    with_cse = compile_network("csedemo", 4)
    without = compile_network("csedemo", 4, cse=False)

    def lets(net, op):
        return sum(1 for s in net.stmts if s.kind == nat.TC_STMT_LET and nat.OP_NAMES[s.op] == op)

    assert lets(without, "MATMUL_FWD") == 3 and lets(with_cse, "MATMUL_FWD") == 2
    assert lets(without, "BIAS_ADD") == 3 and lets(with_cse, "BIAS_ADD") == 2
    texts = [with_cse.stmt_text(i) for i in range(len(with_cse.stmts))]
    assert any("Log X" in t and ".copy" in t for t in texts) and any("1/(X" in t and ".copy" in t for t in texts)
    for name in ("lenet", "alexnet"):
        assert len(compile_network(name, 2).stmts) == len(compile_network(name, 2, cse=False).stmts)
    results = []
    for net in (with_cse, without):
        o = orc.Oracle(net, seed=5)
        o.init_params()
        x, y = orc.synth_batch(net, 5, 0)
        o.set_batch(x, y)
        results.append((o.step(0, update=False), [o.grad(i) for i in range(len(net.params))]))
    assert abs(results[0][0] - results[1][0]) <= 1e-6 * abs(results[1][0])
    for a, b in zip(results[0][1], results[1][1]):
        np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-7)
