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
    ap.add_argument("--shapes", action="store_true", help="append operand shapes of contractions")
    ap.add_argument("--only", default="", help="comma-separated op kinds to list (e.g. CONV_FWD,CONV_BWD_DATA)")
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
        op = nat.OP_NAMES[s.op]
        txt = net.stmt_text(i)[:70]
        if args.shapes and f > 0:
            dims = lambda r: tuple(net.params[r.index].dims if r.kind == nat.TC_REF_PARAM else net.var_dims(r.index))  # noqa: E731
            out = tuple(s.dims[k] for k in range(s.rank)) if s.kind == nat.TC_STMT_LET else tuple(net.params[s.param].dims)
            txt = f"{op[:4]} {dims(s.inp[0])} x {dims(s.inp[1]) if s.nin > 1 else ''} -> {out}"
        rows.append((t, i, op, txt, f / (t * 1e-3) / 1e12 if t > 0 else 0,
                     b / (t * 1e-3) / 1e9 if t > 0 else 0))
    total = sum(r[0] for r in rows)
    print(f"{args.net} b{args.batch}: total {total:.3f} ms over {len(rows)} statements (eager, per-stmt CUDA events)")
    by_op = {}
    for r in rows:
        by_op[r[2]] = by_op.get(r[2], 0.0) + r[0]
    print("  by op: " + ", ".join(f"{k} {v:.3f}" for k, v in sorted(by_op.items(), key=lambda kv: -kv[1]) if v > 0.005))
    only = set(args.only.split(",")) if args.only else None
    for t, i, op, txt, tf, gb in [r for r in sorted(rows, reverse=True) if only is None or r[2] in only][: args.top]:
        print(f"{t:.3f} ms  #{i:<4d} {op:16s} {txt[:70]:70s} {tf:7.1f} TF/s {gb:8.1f} GB/s")


if __name__ == "__main__":
    main()
