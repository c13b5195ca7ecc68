#!/usr/bin/env python3
"""Serialize the plans bench.py's reference arm executes on the CPU oracle.

The reference arm (bench.py --impl reference) must not load the product library, so the plan the
runtime executes for each BASELINE.json configuration is compiled here by the plan producers
(tc_net_compile) and written with tc_plan_save; the oracle loads it with orc_plan_load.  The CPU
sample of a configuration is a slice of its per-GPU batch whose step takes a few seconds on the
GPU box's 16 host cores (bench.py REF_SAMPLE); the loss cardinality stays the configuration's
batch, so the slice's gradients are its share of the full-batch gradient.
tests/test_plans_cpu.py checks the committed files against fresh compiles.

    python tools/make_plans.py        # rewrites oracle/plans/*.tcplan
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (network, per-GPU batch of the BASELINE config, CPU sample batch)
PLANS = [("alexnet", 128, 128), ("vgg16", 64, 8), ("googlenet", 128, 32), ("resnet50", 64, 16), ("lenet", 64, 64)]


def plan_path(name, sample):
    return os.path.join(ROOT, "oracle", "plans", f"{name}_b{sample}.tcplan")


def write_plan(name, batch, sample, path):
    from paper_1701_02284_b200 import _native as nat
    from paper_1701_02284_b200.network import compile_network
    net = compile_network(name, sample, global_batch=batch)
    nat.check(nat.lib().tc_plan_save(net.plan_ptr, path.encode()))


def main():
    os.makedirs(os.path.join(ROOT, "oracle", "plans"), exist_ok=True)
    for name, batch, sample in PLANS:
        p = plan_path(name, sample)
        write_plan(name, batch, sample, p)
        print(p, os.path.getsize(p))


if __name__ == "__main__":
    main()
