#!/usr/bin/env python3
"""DRAM traffic of the contraction launches of one training step, from an ncu CSV capture:

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        --clock-control none -c 300 --csv --log-file t.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-f32
    python tools/gemm_traffic.py t.csv profiles/r2_gemm_traffic_alexnet_b128.json

Picks the launches between the last two k_set_iter markers (one whole step), sums time and
DRAM bytes of the tcgen05 contraction kernels (implicit-GEMM conv fprop / dgrad / wgrad, FC
GEMMs) and stamps the result with bench.src_hash(), so bench.py reports it only while the
kernel sources it measured are unchanged.
"""
import csv
import io
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONTRACTION = re.compile(r"tc_gemm_kernel|tc_conv_halo_kernel|tc_wgrad_halo|tc_conv_c4")


def main(path, out):
    import bench

    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    launches = {}
    for r in rows:
        k = launches.setdefault(r["ID"], {"name": r["Kernel Name"].split("(")[0].replace("void ", ""), "m": {}})
        v = r["Metric Value"].replace(",", "")
        k["m"][r["Metric Name"]] = float(v) if v else 0.0
    order = [launches[i] for i in sorted(launches, key=int)]
    marks = [i for i, k in enumerate(order) if "k_set_iter" in k["name"]]
    a, b = marks[-2], marks[-1]
    step = order[a:b]
    sel = [k for k in step if CONTRACTION.search(k["name"])]
    per = {"launches": len(sel), "time_ns": sum(k["m"].get("gpu__time_duration.sum", 0) for k in sel),
           "dram_read_bytes": sum(k["m"].get("dram__bytes_read.sum", 0) for k in sel),
           "dram_write_bytes": sum(k["m"].get("dram__bytes_write.sum", 0) for k in sel)}
    res = {"src_hash": bench.src_hash(), "source": os.path.basename(path),
           "note": "one whole step (between k_set_iter markers), contraction kernels only; ncu replays "
                   "each kernel alone (cold caches), so bytes are an upper bound on the in-graph traffic",
           "per_step": per,
           "launches": [{"kernel": k["name"], "time_us": round(k["m"].get("gpu__time_duration.sum", 0) / 1e3, 2),
                         "dram_read_mb": round(k["m"].get("dram__bytes_read.sum", 0) / 1e6, 2),
                         "dram_write_mb": round(k["m"].get("dram__bytes_write.sum", 0) / 1e6, 2)} for k in sel]}
    json.dump(res, open(out, "w"), indent=1)
    print(f"{len(sel)} contraction launches, {per['time_ns'] / 1e3:.1f} us, read {per['dram_read_bytes'] / 1e9:.3f} GB, "
          f"write {per['dram_write_bytes'] / 1e9:.3f} GB -> {out}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
