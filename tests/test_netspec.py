"""Text network description (the reference's netspec-frontend) through the C ABI
(tc_net_compile_spec): user networks reach the compiler, the oracle and the runtime without C++.

  * nets/lenet.net compiles to exactly the built-in LeNet IrProgram: Fig. 2's statement text,
    numbering and memory table;
  * the SPEC's parser examples and error kinds (SyntaxError with position, DuplicateName,
    UnknownLayerKind, UnboundName);
  * a network outside the built-in list (nets/smallnet.net: conv -> relu -> pool -> LRN -> conv,
    a shared-prefix auxiliary head with a weighted loss, dropout, gaussian init) compiles, verifies,
    and trains on the CPU oracle.
"""
import os

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1701_02284_b200 import _native as nat
from paper_1701_02284_b200.network import compile_network, compile_spec, load_spec

NETS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "nets")


def test_lenet_spec_is_fig1_network():
    a = compile_network("lenet", 500)
    b = load_spec(os.path.join(NETS, "lenet.net"))
    assert b.name == "lenet" and b.batch == 500
    assert a.ir_text() == b.ir_text()
    assert a.memory_table() == b.memory_table()
    s = b.memory_summary()
    assert f"{s.peak_dealloc_mb:.6f}" == "59.167999" and f"{s.peak_reuse_mb:.6f}" == "77.248001"
    assert [p.name for p in b.params] == ["cv1_W", "cv1_B", "cv2_W", "cv2_B", "fc1_W", "fc1_B", "fc2_W", "fc2_B"]
    assert b.spec_info() == {"seed": 42, "iters": 1000, "test_iters": 10}
    assert b.plan.lr == pytest.approx(0.01) and b.plan.momentum == pytest.approx(0.9)


def test_batch_override_and_solver_override():
    b = load_spec(os.path.join(NETS, "lenet.net"), 64)
    assert b.batch == 64 and b.input_dims == (64, 1, 28, 28)
    c = load_spec(os.path.join(NETS, "lenet.net"), 64, lr=0.05, momentum=0.5, decay=0.0, clip=1.0)
    assert c.plan.lr == pytest.approx(0.05) and c.plan.clip == pytest.approx(1.0)


def test_conv_declaration_example():
    # `cv1 = conv(k=5, out=20)` -> kind conv, kernel 5, 20 output channels
    text = """data { batch = 2 shape = (1, 12, 12) classes = 3 }
              net t { cv1 = conv(k=5, out=20)  n = full(K) . flatten(4, 1) . cv1  loss = logloss(n) }"""
    net = compile_spec(text)
    assert net.params[0].name == "cv1_W" and net.params[0].dims == (20, 1, 5, 5)
    assert net.params[2].dims == (3, 20 * 8 * 8)


@pytest.mark.parametrize("text,kind,where", [
    ("data { batch = 2 shape = (1, 8, 8) classes = 3 } net t { }", "SyntaxError", None),
    ("data { batch = 2 shape = (1, 8, 8) classes = 3 } net t { n = }", "SyntaxError", "1:62"),
    ("data { batch = 2 shape = (1, 8, 8) classes = 3 }\nnet t { a = conv(3, 4)\n a = relu(4) }", "DuplicateName", "3:2"),
    ("data { batch = 2 shape = (1, 8, 8) classes = 3 }\nnet t { a = frobnicate(3)  loss = logloss(a) }",
     "UnknownLayerKind", "2:13"),
    ("data { batch = 2 shape = (1, 8, 8) classes = 3 }\nnet t { n = full(K) . nope  loss = logloss(n) }",
     "UnboundName", "2:23"),
    ("data { batch = 2 shape = (1, 8, 8) classes = 3 } net t { n = full(K) . flatten(4, 1) loss = logloss(n) } "
     "solver { lr = 0 }", "SyntaxError", None),
])
def test_spec_errors(text, kind, where):
    with pytest.raises(nat.TcError) as e:
        compile_spec(text)
    assert e.value.status == nat.TC_COMPILE_ERROR
    assert kind in str(e.value), str(e.value)
    if where:
        assert f"at {where}:" in str(e.value), str(e.value)


def test_shape_mismatch_is_reported():
    # full(10) fed a 4-D tensor without flatten: shape inference rejects it (SPEC.md:546 analogue)
    text = "data { batch = 2 shape = (1, 8, 8) classes = 3 } net t { n = full(K) . conv(3, 4) loss = logloss(n) }"
    with pytest.raises(nat.TcError):
        compile_spec(text)


def test_user_network_compiles_and_trains_on_the_oracle():
    net = load_spec(os.path.join(NETS, "smallnet.net"))
    assert net.name == "smallnet" and net.batch == 16
    assert net.verify() == ""
    ops = {nat.OP_NAMES[s.op] for s in net.stmts if s.kind == nat.TC_STMT_LET}
    assert {"CONV_FWD", "POOL_FWD", "LRN_FWD", "LRN_BWD", "DROPOUT_MASK", "ADD", "MATMUL_FWD"} <= ops
    info = net.spec_info()
    o = orc.Oracle(net, seed=info["seed"])
    o.init_params()
    losses = [o.step(it) for it in range(60)]
    # two log-loss heads (weights 1 and 0.3) at chance: ~1.3 ln 10
    assert abs(losses[0] - 1.3 * np.log(10)) < 0.3, losses[0]
    assert np.mean(losses[-5:]) < 0.6 * losses[0], losses
