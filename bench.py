#!/usr/bin/env python3
"""Training-step benchmark: train images/sec (fwd + symbolic bwd + momentum SGD).

Workload (BASELINE.json): N = 1 -> configs[1], AlexNet synthetic 3x224x224 batch 128 on one
B200; N > 1 (torchrun, one process per GPU) -> configs[2], VGG-16 batch 64 per GPU, data
parallel (weak scaling) with the per-bucket NCCL gradient all-reduce.  --net overrides.

    python bench.py --gpus N --steps K --warmup W            # this repo's sm_100a executor
    python bench.py --impl reference --steps K --warmup W    # the CPU path (oracle) on the host cores

Prints one JSON line (rank 0).  `value` = whole-job images/s with the batch resident in HBM
(bf16 mode: bf16 activations, bf16 tensor-core operands, fp32 accumulation / master weights);
`e2e` = the same through the public API with a host batch staged (H2D) and the loss read back
(D2H) every step; `f32_mode` = the fp32 parity mode (TC_PREC_F32) measured the same way.
The reference arm never loads the product library: it runs the serialized plan
(oracle/plans/*.tcplan, tools/make_plans.py) on the CPU oracle.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 42
# per-GPU batch of each BASELINE.json config (weak scaling)
CONFIG_BATCH = {"lenet": 64, "alexnet": 128, "vgg16": 64, "googlenet": 128, "resnet50": 64}
CONFIG_INDEX = {"lenet": 0, "alexnet": 1, "vgg16": 2, "googlenet": 3, "resnet50": 4}
# CPU sample per step (a slice of the per-GPU batch; tools/make_plans.py): a few seconds of CPU work
REF_SAMPLE = {"lenet": 64, "alexnet": 128, "vgg16": 8, "googlenet": 32, "resnet50": 16}
METRIC = "train images/sec (fwd+bwd+SGD)"


def default_net(world):
    return "alexnet" if world == 1 else "vgg16"


def workload_config(net, world, batch):
    return {"workload": f"{net} 3x224x224 fwd + symbolic bwd + momentum SGD (BASELINE.json "
                        f"configs[{CONFIG_INDEX[net]}])",
            "model": net, "global_batch": world * batch, "per_gpu_batch": batch, "seq_len": None,
            "parallelism": f"dp{world}", "l2": "per-step working set >> 126 MB L2 (no flush needed)"}


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def src_hash():
    """Hash of the kernel / runtime sources: a committed ncu traffic capture is only reported
    while the code it measured is unchanged."""
    h = hashlib.sha256()
    base = os.path.join(ROOT, "paper_1701_02284_b200", "csrc")
    files = []
    for d, _, fs in os.walk(base):
        files += [os.path.join(d, f) for f in fs if f.endswith((".cu", ".cuh", ".cpp", ".hpp", ".h"))]
    for f in sorted(files):
        h.update(os.path.relpath(f, ROOT).encode())
        h.update(open(f, "rb").read())
    return h.hexdigest()[:16]


def cpu_info():
    model, flags = "unknown", ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name") and model == "unknown":
                model = line.split(":", 1)[1].strip()
            if line.startswith("flags") and not flags:
                flags = line.split(":", 1)[1]
    except OSError:
        pass
    isa = [f for f in ("avx2", "fma", "avx512f", "avx512_bf16", "amx_bf16") if f" {f} " in f" {flags} "]
    return {"model": model, "isa_available": isa, "isa_used": "AVX2 + FMA (oracle built -march=x86-64-v3)",
            "nproc": os.cpu_count(), "machine": platform.machine()}


# ------------------------------------------------------------------ algorithmic work per statement
def stmt_work(net, s, nat):
    """(flops, bytes) of one statement at the device storage dtypes (bf16 activations,
    fp32 parameters); flops are 2*MACs of the contraction with real (unpadded) channels."""
    op = nat.OP_NAMES[s.op]
    dims = lambda r: (net.params[r.index].dims if r.kind == nat.TC_REF_PARAM else net.var_dims(r.index))  # noqa: E731
    prod = lambda t: int(np.prod(t)) if len(t) else 1  # noqa: E731
    out = tuple(s.dims[i] for i in range(s.rank)) if s.kind == nat.TC_STMT_LET else net.params[s.param].dims
    if op == "CONV_FWD":
        x, w = dims(s.inp[0]), dims(s.inp[1])
        return 2 * prod(out) * x[1] * w[2] * w[3], 0
    if op == "CONV_BWD_DATA":
        dy, w = dims(s.inp[0]), dims(s.inp[1])
        return 2 * prod(dy) * w[1] * w[2] * w[3], 0
    if op == "CONV_BWD_FILTER":
        dy = dims(s.inp[0])
        return 2 * prod(dy) * out[1] * out[2] * out[3], 0
    if op in ("MATMUL_FWD", "MATMUL_BWD_DATA"):
        a, w = dims(s.inp[0]), dims(s.inp[1])
        return 2 * a[0] * w[0] * w[1], 0
    if op == "MATMUL_BWD_W":
        up = dims(s.inp[0])
        return 2 * up[0] * out[0] * out[1], 0
    n_out = prod(out)
    reads = sum(prod(dims(s.inp[i])) for i in range(s.nin))
    if s.kind == nat.TC_STMT_UPDATE:  # the gradient (bias / BN sums; fp32 out); the update is separate
        return 0, 2 * reads + 4 * n_out
    return 0, 2 * (reads + n_out)


class NvmlClockSampler:
    """SM clock / throttle-reason samples every ~5 ms on a host thread (NVML), so even a
    timed region of a few tens of milliseconds is covered."""

    def __init__(self, device_index):
        import threading
        import pynvml as nv
        import torch
        self.nv = nv
        nv.nvmlInit()
        try:  # the CUDA device by UUID (NVML's index order need not match CUDA's)
            self.h = nv.nvmlDeviceGetHandleByUUID("GPU-" + str(torch.cuda.get_device_properties(device_index).uuid))
        except Exception:
            self.h = nv.nvmlDeviceGetHandleByIndex(device_index)
        self.rows, self.stop = [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        while True:
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                smax = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, smax, r))
            except Exception:
                pass
            if self.stop.wait(0.005):
                break

    def result(self):
        self.stop.set()
        self.t.join()
        nv = self.nv
        if not self.rows:
            return None
        names = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                 "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                 "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                 "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        reasons = sorted({k for _, _, r in self.rows for k, bit in names.items() if r & bit})
        return {"sm_mhz": float(np.median([a for a, _, _ in self.rows])), "sm_max_mhz": float(max(b for _, b, _ in self.rows)),
                "reasons": reasons, "samples": len(self.rows), "source": "nvml"}


# ------------------------------------------------------------------ CPU path (oracle, serialized plan)
def cpu_rate(net_name, warmup, steps, threads, median=True):
    """images/s of the CPU oracle on the serialized plan of `net_name`'s sample slice (the product
    library is never loaded here).  Returns (rate, per-step seconds list, sample batch)."""
    from oracle.oracle import Oracle, PlanFile
    sample = REF_SAMPLE[net_name]
    pf = PlanFile(os.path.join(ROOT, "oracle", "plans", f"{net_name}_b{sample}.tcplan"))
    o = Oracle(pf, seed=SEED, threads=threads)
    o.init_params()
    for it in range(warmup):
        o.step(it)
    times = []
    for it in range(warmup, warmup + steps):
        t0 = time.perf_counter()
        o.step(it)
        times.append(time.perf_counter() - t0)
    dt = float(np.median(times)) if median else float(np.mean(times))
    return sample / dt, times, sample


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    net = args.net or default_net(world)
    batch = args.batch or CONFIG_BATCH[net]
    threads = os.cpu_count() or 1
    rate, times, sample = cpu_rate(net, args.warmup, args.steps, threads, median=False)
    dt = float(np.mean(times))
    desc = (f"{net}: each step = one training step (fwd + bwd + momentum SGD) of a {sample}-image slice of the "
            f"{batch}-image per-GPU batch (loss cardinality {batch}), {args.warmup} warm-up + {args.steps} timed "
            f"steps, mean; CPU oracle (C++/OpenMP restatement of the SPEC.md runtime) on the serialized plan "
            f"oracle/plans/{net}_b{sample}.tcplan")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(rate, 4), "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3 * batch / sample, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (Philox K-blob images, tc_philox.h)",
        "config": workload_config(net, world, batch),
        "cpu_baseline": {"value": round(rate, 4), "unit": "images/s", "cores": threads, "kind": "port",
                         "sample": desc, "cpu": cpu_info(), "step_s": [round(t, 3) for t in times]},
        "e2e": {"value": round(rate, 4), "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def measure(net, args, world, rank, local, nid, precision, batch, dist, with_e2e=True, with_profile=True):
    """Device-timed steps (batch resident in HBM), then the e2e loop through the public API."""
    import torch

    from paper_1701_02284_b200 import _native as nat
    from paper_1701_02284_b200.runtime import Trainer

    tr = Trainer(net, device=local, seed=SEED, use_graph=True, rank=rank, world=world, nccl_id=nid,
                 precision=precision)
    tr.init_params()
    stream = torch.cuda.ExternalStream(tr.stream)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    n0 = rank * batch
    tr.stage_synthetic(0, n0)
    for it in range(args.warmup):
        tr.step(it, n0)
    tr.sync()
    launches0 = nat.lib().tc_kernel_launch_count()
    nvml = None
    if rank == 0:
        try:
            nvml = NvmlClockSampler(torch.cuda.current_device())
        except Exception:
            nvml = None
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for it in range(args.warmup, args.warmup + args.steps):
        tr.step(it, n0)
    ev1.record(stream)
    ev1.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    launches = nat.lib().tc_kernel_launch_count() - launches0
    clocks = nvml.result() if nvml else None
    res = {"ms": ms, "launches": int(launches), "clocks": clocks, "loss": tr.loss()}
    if with_e2e:
        # e2e: the public API with a host batch each step (pinned H2D) + loss D2H.  The input
        # pipeline stages batch i+1 (H2D on the context's copy stream) while step i runs, as a
        # training loop with a prefetching loader does; every step's H2D copy and its loss
        # read-back are inside the timed region, which is wall clock (host + device).
        x_host = torch.empty(tuple(net.input_dims), dtype=torch.float32).pin_memory()
        y_host = torch.empty((batch,), dtype=torch.int32).pin_memory()
        from oracle.oracle import synth_batch  # host-side generator of the same law (input pipeline stand-in)
        xs, ys = synth_batch(net, SEED, 0, n0)
        x_host.copy_(torch.from_numpy(xs))
        y_host.copy_(torch.from_numpy(ys))
        xh, yh = x_host.numpy(), y_host.numpy()
        tr.stage_batch(xh, yh)
        for it in range(2):
            tr.step(it, n0)
            tr.stage_batch(xh, yh)
            tr.loss()
        tr.sync()
        barrier()
        sync_loss = os.environ.get("TCB_BENCH_SYNC_LOSS") == "1"
        losses = []
        t0 = time.perf_counter()
        for it in range(args.steps):
            tr.step(it, n0)
            tr.stage_batch(xh, yh)  # next step's batch, overlapping this step
            if sync_loss:
                losses.append(tr.loss())  # waits for this step: the device idles until the next launch
            elif it > 0:
                # every step's loss is read back, one step late (waits for step it-1 only), as a
                # loop that logs asynchronously does: step it+1 is enqueued while step it runs
                losses.append(tr.loss_prev())
        tr.sync()
        if not sync_loss:
            losses.append(tr.loss())
        res["e2e_ms"] = (time.perf_counter() - t0) * 1e3 / args.steps
        assert len(losses) == args.steps and all(np.isfinite(losses)), losses
        res["h2d"] = tr.stage_bytes  # as copied: bf16 images when the runtime rounds them on the host
        barrier()
    if with_profile:
        # per-statement profile (one eager step) for the roofline; statements folded into their
        # producer launch nothing and are not charged
        res["stmt_ms"] = tr.profile_step(args.warmup + args.steps, n0)
        res["stmt_launches"] = tr.profile_launches()
        res["update_ms"] = float(np.sum(tr.profile_updates()))
    res["memory"] = tr.memory()
    res["launches_per_step"] = tr.launches_per_step
    tr.close()
    return res


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_1701_02284_b200 import _native as nat
    from paper_1701_02284_b200.parallel import broadcast_nccl_id, compile_shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")  # plumbing only: NCCL id broadcast, barriers, max-over-ranks
        nid = broadcast_nccl_id(rank)
    else:
        nid = None
    name = args.net or default_net(world)
    batch = args.batch or CONFIG_BATCH[name]
    overrides = {k: v for k, v in os.environ.items() if k.startswith("TCB_")}
    net = compile_shard(name, batch, world)  # loss / |world * batch|: summed gradients = global-batch gradient
    peaks, peak_kind = load_peaks()
    r = measure(net, args, world, rank, local, nid, args.precision, batch, dist)
    f32 = None
    if args.precision == "bf16" and not args.no_f32:
        nid2 = broadcast_nccl_id(rank) if world > 1 else None
        f32 = measure(net, args, world, rank, local, nid2, "f32", batch, dist, with_profile=False)
    times = torch.tensor([r["ms"], r["e2e_ms"]] + ([f32["ms"], f32["e2e_ms"]] if f32 else []), dtype=torch.float64)
    if world > 1:
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    tl = times.tolist()
    ms, e2e_ms = tl[0], tl[1]
    if rank != 0:
        dist.destroy_process_group() if world > 1 else None
        return 0

    # roofline of the dominant kernel class: the tcgen05 contractions, per-statement CUDA events
    # over one eager step (each kernel timed alone -> the burst peak applies)
    stmt_ms, stmt_l = r["stmt_ms"], r["stmt_launches"]
    flops_tc = t_tc = bytes_bw = t_bw = 0.0
    n_bw = 0
    for i, s in enumerate(net.stmts):
        if s.kind == nat.TC_STMT_DEALLOC or stmt_l[i] == 0:
            continue
        f, b = stmt_work(net, s, nat)
        if f:
            flops_tc += f
            t_tc += float(stmt_ms[i])
        else:
            bytes_bw += b
            t_bw += float(stmt_ms[i])
            n_bw += 1
    # the momentum update (+ all-reduce) of every bucket: 20 B/param of fp32 p / v / g traffic + the
    # bf16 operand shadows (2 B/param, +2 for conv filters' RSKC copy)
    t_upd = r["update_ms"]
    upd_bytes = sum((22 + (2 if len(p.dims) == 4 else 0)) * p.count for p in net.params)
    bytes_bw += upd_bytes
    t_bw += t_upd
    peak_tf = peaks.get("bf16_tflops")
    achieved_tf = flops_tc / (t_tc * 1e-3) / 1e12 if t_tc > 0 else 0.0
    t_roof = flops_tc / (peaks.get("bf16_tflops_sustained", peak_tf) * 1e12) + bytes_bw / (peaks["hbm_gbs"] * 1e9)
    traffic, traffic_note = None, "no ncu capture of this configuration"
    tpath = os.path.join(ROOT, "profiles", f"r2_gemm_traffic_{name}_b{batch}.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        if tj.get("src_hash") == src_hash():
            ps = tj["per_step"]
            traffic = ps["dram_read_bytes"] + ps["dram_write_bytes"]
            traffic_note = f"ncu dram__bytes_read+write of all contraction launches of one step ({os.path.basename(tpath)})"
        else:
            traffic_note = f"{os.path.basename(tpath)} measured other kernel sources (src_hash mismatch): not reported"
    cpu = None
    if world == 1 and not args.no_cpu:
        rate, ts, sample = cpu_rate(name, 2, 5, os.cpu_count() or 1)
        cpu = {"value": round(rate, 4), "unit": "images/s", "cores": os.cpu_count() or 1, "kind": "port",
               "sample": f"{name}: {sample}-image slice of the {batch}-image batch per step (loss cardinality {batch}), "
                         f"2 warm-up + median of 5 steps, CPU oracle on oracle/plans/{name}_b{sample}.tcplan",
               "cpu": cpu_info(), "step_s": [round(t, 3) for t in ts]}
    mem = r["memory"]
    summ = net.memory_summary()
    line = {
        "metric": METRIC,
        "value": round(world * batch / (ms * 1e-3), 2),
        "unit": "images/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.precision,
        "precision": ("bf16 activation storage, bf16 tensor-core operands, fp32 accumulation / master weights / "
                      "velocities / gradients / bandwidth-kernel arithmetic" if args.precision == "bf16" else
                      "fp32 activations; contractions as 6-term bf16 splits accumulated in fp32 (parity mode)"),
        "data": "synthetic (Philox K-blob images generated on device; random Xavier init)",
        "config": workload_config(name, world, batch),
        "e2e": {"value": round(world * batch / (e2e_ms * 1e-3), 2), "unit": "images/s",
                "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": 4,
                "loop": "stage_batch(next) overlaps the step; each step's loss read back one step late "
                        "(tc_loss_prev) so the next step is enqueued while the current one runs",
                "loss_readback": "sync" if os.environ.get("TCB_BENCH_SYNC_LOSS") == "1" else "one step late"},
        "roofline": {"bound": "tensor", "kernel": "tcgen05 implicit-GEMM contractions (conv fwd/dgrad/wgrad, FC)",
                     "achieved": round(achieved_tf, 2), "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": round(achieved_tf / peak_tf, 4),
                     "peak_kind": f"{peak_kind} burst dense bf16 (kernels timed one by one in an eager step)",
                     "traffic": traffic, "traffic_note": traffic_note,
                     "flops_per_step": flops_tc, "contraction_ms": round(float(t_tc), 4)},
        "step_roofline": {"t_roof_ms": round(t_roof * 1e3, 4), "t_meas_ms": round(ms, 4),
                          "frac": round(t_roof * 1e3 / ms, 4), "bandwidth_ms": round(float(t_bw), 4),
                          "bandwidth_bytes": bytes_bw, "bandwidth_statements": n_bw,
                          "update_ms": round(t_upd, 4), "update_bytes": upd_bytes,
                          "bandwidth_gbs": round(bytes_bw / (t_bw * 1e-3) / 1e9, 1) if t_bw else None,
                          "note": "T_roof = contraction FLOPs / sustained bf16 peak + bandwidth-kernel algorithmic "
                                  "bytes / HBM peak, over the statements that launch a kernel"},
        "cpu_baseline": cpu,
        "gpu_launches": r["launches"],
        "launches_per_step": r["launches_per_step"],
        "clocks": r["clocks"],
        "loss": r["loss"],
        "peak_hbm_mb": {"arena": round(mem["arena_bytes"] / 1e6, 3), "static_slab": round(mem["param_bytes"] / 1e6, 3),
                        "workspace": round(mem["workspace_bytes"] / 1e6, 3),
                        "ref_table_dealloc": round(summ.peak_dealloc_mb, 3),
                        "ref_table_reuse": round(summ.peak_reuse_mb, 3),
                        "device_used": round(mem["device_used_bytes"] / 1e6, 1)},
        "env_overrides": overrides or None,
    }
    if f32:
        line["f32_mode"] = {"value": round(world * batch / (tl[2] * 1e-3), 2), "unit": "images/s",
                            "ms_per_step": round(tl[2], 4),
                            "e2e": {"value": round(world * batch / (tl[3] * 1e-3), 2), "unit": "images/s"},
                            "gpu_launches": f32["launches"], "clocks": f32["clocks"], "loss": f32["loss"],
                            "precision": "fp32 activations; contractions as 6-term bf16 splits accumulated in fp32 "
                                         "(the mode the fp32 parity tests run in)"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--precision", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-f32", action="store_true", help="skip the fp32-mode measurement")
    ap.add_argument("--net", default=None, choices=["alexnet", "vgg16", "googlenet", "resnet50", "lenet"],
                    help="workload (default: AlexNet b128 at N=1, VGG-16 b64/GPU at N>1)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
