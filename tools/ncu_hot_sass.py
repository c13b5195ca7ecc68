#!/usr/bin/env python3
"""Top SASS lines by warp-stall samples from `ncu -i REP --page source --csv --print-source sass`."""
import csv
import subprocess
import sys


def main(rep, n=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out[1:]))
    h = rows[0]
    ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[1:] if len(r) == len(h)]
    tot = sum(int(r[iss] or 0) for r in body)
    order = sorted(range(len(body)), key=lambda i: -int(body[i][iss] or 0))
    print(f"total stall samples {tot}")
    for i in order[:n]:
        r = body[i]
        print(f"{int(r[iss]):7d} {100 * int(r[iss]) / tot:5.1f}%  #{i:5d} {r[ia][-5:]}  {r[isrc].strip()}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
