#!/usr/bin/env python3
"""One line per profiled launch from an `ncu --set full` report: duration, DRAM traffic,
tensor-pipe activity, SM throughput, registers, achieved occupancy.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [title]
"""
import csv
import io
import subprocess
import sys

COLS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "rd_MB"),
    ("dram__bytes_write.sum", "wr_MB"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor%"),
    ("TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg", "tc_active_cyc"),
    ("sm__cycles_elapsed.avg", "sm_cyc"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def main(path, title=""):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    idx = {c: h.index(c) for c, _ in COLS if c in h}
    print(title)
    print("id, kernel, " + ", ".join(n for c, n in COLS if c in idx))
    for r in rows[2:]:
        vals = []
        for c, n in COLS:
            if c not in idx:
                continue
            v = r[idx[c]]
            u = units[idx[c]]
            try:
                f = float(v.replace(",", ""))
                if u == "Gbyte":
                    f *= 1e3
                elif u == "Kbyte":
                    f *= 1e-3
                elif u == "byte":
                    f *= 1e-6
                elif u == "ms":
                    f *= 1e3
                elif u == "ns":
                    f *= 1e-3
                vals.append(f"{f:.1f}")
            except ValueError:
                vals.append(v)
        print(f"{r[0]}, {r[h.index('Kernel Name')].split('(')[0]}, " + ", ".join(vals))


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
