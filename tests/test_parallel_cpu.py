"""Data-parallel host logic on CPU with world size 2 (gloo), no GPU needed:
the G-shard emulation of SURVEY.md §4(i).  Two ranks each run the oracle on
their shard of the global batch with the per-rank plan (loss / |G*B|), the
gradients are all-reduced with gloo, and the result must equal the
single-process gradient of the global batch (dropout masks keyed by the global
sample index)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, per_gpu, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    from paper_1701_02284_b200.parallel import compile_shard, shard_offset

    net = compile_shard(name, per_gpu, world)
    o = orc.Oracle(net, seed=21, threads=2)
    o.init_params()
    o.step(3, shard_offset(rank, per_gpu), update=False)
    grads = []
    for i in range(len(net.params)):
        g = torch.from_numpy(o.grad(i).copy())
        dist.all_reduce(g)
        grads.append(g.numpy())
    loss = torch.tensor([o.step(3, shard_offset(rank, per_gpu), update=False)], dtype=torch.float64)
    dist.all_reduce(loss)
    if rank == 0:
        out_q.put((loss.item(), [g.tolist() for g in grads]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,per_gpu", [("lenet", 4), ("alexnet", 1)])
def test_two_rank_gradient_equals_global_batch(name, per_gpu):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, per_gpu, q)) for r in range(world)]
    for p in procs:
        p.start()
    loss_dp, grads_dp = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0

    from oracle import oracle as orc
    from paper_1701_02284_b200.network import compile_network

    net = compile_network(name, world * per_gpu)
    o = orc.Oracle(net, seed=21)
    o.init_params()
    loss = o.step(3, 0, update=False)
    assert abs(loss - loss_dp) <= 1e-5 * abs(loss)
    for i in range(len(net.params)):
        g = o.grad(i)
        gd = np.array(grads_dp[i]).reshape(g.shape)
        assert np.max(np.abs(g - gd)) <= 1e-4 * max(1e-6, np.max(np.abs(g))), net.params[i].name


def test_reference_arm_under_torchrun_world2():
    """The driver launches `bench.py --impl reference` with torchrun for N > 1: rank 0 alone
    times the reference CPU path and prints one JSON line; the other rank exits 0 silently."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--impl", "reference", "--gpus", "2",
           "--steps", "1", "--warmup", "1"]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["e2e"]["h2d_bytes_per_step"] == 0
