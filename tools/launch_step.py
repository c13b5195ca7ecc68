#!/usr/bin/env python3
"""Print the launches of one step (between two k_set_iter launches) of an ncu
`--metrics gpu__time_duration.sum --csv` launch list, in launch order, with the step total."""
import csv
import io
import sys


def main(path, which=-2):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = [r for r in csv.DictReader(io.StringIO("".join(lines))) if r.get("Metric Name") == "gpu__time_duration.sum"]
    ks = [(r["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "").replace("void ", ""),
           float(r["Metric Value"]), r.get("Grid Size", "")) for r in rows]
    starts = [i for i, k in enumerate(ks) if "k_set_iter" in k[0]]
    a, b = starts[which - 1], starts[which]
    tot = 0.0
    for i in range(a, b):
        print(f"{i - a:3d} {ks[i][1] / 1e3:8.1f} us  {ks[i][0]}  {ks[i][2]}")
        tot += ks[i][1]
    print(f"step total {tot / 1e3:.1f} us over {b - a} launches")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else -1)
