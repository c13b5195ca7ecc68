#!/usr/bin/env python3
"""Per-statement device time of one eager training step (CUDA events per IrStmt),
with algorithmic TFLOP/s (contractions) or GB/s (bandwidth statements).

    python tools/stmt_profile.py --net alexnet --batch 128 [--top 40]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="alexnet")
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--top", type=int, default=60)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import bench
    from paper_1701_02284_b200 import _native as nat
    from paper_1701_02284_b200.network import compile_network
    from paper_1701_02284_b200.runtime import Trainer

    net = compile_network(args.net, args.batch)
    tr = Trainer(net, device=0, seed=42, use_graph=False)
    tr.init_params()
    tr.stage_synthetic(0, 0)
    for it in range(3):
        tr.step(it)
    tr.sync()
    ms = np.median(np.stack([tr.profile_step(3 + r) for r in range(args.reps)]), axis=0)
    rows = []
    for i, s in enumerate(net.stmts):
        if s.kind == nat.TC_STMT_DEALLOC:
            continue
        f, b = bench.stmt_work(net, s, nat)
        t = float(ms[i])
        rows.append((t, i, nat.OP_NAMES[s.op], net.stmt_text(i), f / (t * 1e-3) / 1e12 if t > 0 else 0,
                     b / (t * 1e-3) / 1e9 if t > 0 else 0))
    total = sum(r[0] for r in rows)
    print(f"{args.net} b{args.batch}: total {total:.3f} ms over {len(rows)} statements (eager, per-stmt CUDA events)")
    for t, i, op, txt, tf, gb in sorted(rows, reverse=True)[: args.top]:
        print(f"{t:.3f} ms  #{i:<4d} {op:16s} {txt[:70]:70s} {tf:7.1f} TF/s {gb:8.1f} GB/s")


if __name__ == "__main__":
    main()
