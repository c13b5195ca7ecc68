"""Extract the Fig. 2 memory table into tests/golden/fig2_lenet_b500.json.

Runs only in the build container (reads /root/reference); the JSON it writes is
committed so the tests never touch /root/reference at run time.
"""
import json
import os
import re

SRC = "/root/reference/PAPER.md"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fig2_lenet_b500.json")

lines = open(SRC).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith("IR expression"))
rows = []
pending = None
for l in lines[start + 2:]:
    if l.startswith("\\end{lstlisting}"):
        break
    if not l.strip() or l.startswith("...."):
        if l.startswith("...."):
            rows.append({"omitted": True})
        continue
    m = re.match(r"^(.*?)\s+((?:\d+ )*\d+)?\s*(-?\d+\.\d{6})\s+(\d+\.\d{6})\s+(\d+\.\d{6})\s*$", l)
    if m is None:  # statement wrapped onto the next line (X74)
        pending = l.strip()
        continue
    text = (pending + " " if pending else "") + m.group(1).strip()
    pending = None
    rows.append({"stmt": text, "dims": (m.group(2) or "").strip(), "delta": m.group(3), "total": m.group(4),
                 "reuse": m.group(5)})
json.dump({"source": "PAPER.md:270-303 (Fig. 2)", "rows": rows}, open(OUT, "w"), indent=1)
print(f"wrote {len(rows)} rows to {OUT}")
