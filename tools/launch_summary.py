#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel launches, total ns, share."""
import collections
import csv
import io
import sys


def main(path, title=""):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
        tot[k] += float(r["Metric Value"])
        cnt[k] += 1
    T = sum(tot.values())
    print(title)
    print(f"total {T:.1f} ns over {sum(cnt.values())} launches")
    print("kernel, launches, total_ns, share")
    for k, v in tot.most_common():
        print(f"{k}, {cnt[k]}, {v:.1f}, {100 * v / T:.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
