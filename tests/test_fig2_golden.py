"""Acceptance criteria 1-2: the compiled LeNet (batch 500)
reproduces Fig. 2 of the paper — every shown row's
statement, dimensions and the three memory columns to the printed 6 decimals.

Backward SSA numbers are not pinned (the omitted lines' naming is
unknown), so backward rows are compared with Xn renamed positionally.
"""
import csv
import io
import json
import os
import re

import pytest

from paper_1701_02284_b200.network import compile_network

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig2_lenet_b500.json")))["rows"]


@pytest.fixture(scope="module")
def lenet500():
    return compile_network("lenet", 500)


def my_rows(net):
    rdr = csv.reader(io.StringIO(net.memory_table(csv=True)))
    next(rdr)
    return [{"stmt": r[0], "dims": r[1], "delta": r[2], "total": r[3], "reuse": r[4]} for r in rdr]


def norm(s):
    return re.sub(r"X\d+", "X#", s.strip())


def test_forward_rows_exact(lenet500):
    mine = my_rows(lenet500)
    fwd = GOLD[: next(i for i, r in enumerate(GOLD) if r.get("omitted"))]
    assert len(fwd) == 16
    for i, g in enumerate(fwd):
        m = mine[i]
        for key in ("dims", "delta", "total", "reuse"):
            assert m[key] == g[key], (i, key, m, g)
        if g["stmt"].startswith("val X52"):  # SSA number of the Log-gradient reciprocal is unpinned
            assert norm(m["stmt"]) == norm(g["stmt"])
        else:
            assert m["stmt"] == g["stmt"], (i, m["stmt"], g["stmt"])


def test_backward_rows_exact(lenet500):
    mine = my_rows(lenet500)
    bwd = GOLD[next(i for i, r in enumerate(GOLD) if r.get("omitted")) + 1:]
    start = next(i for i, r in enumerate(mine) if r["stmt"].startswith("cv2_B <~~"))
    for j, g in enumerate(bwd):
        m = mine[start + j]
        assert norm(m["stmt"]) == norm(g["stmt"]), (j, m["stmt"], g["stmt"])
        for key in ("dims", "delta", "total", "reuse"):
            assert m[key] == g[key], (j, key, m, g)
    assert len(mine) == start + len(bwd)


def test_peaks_and_static_memory(lenet500):
    s = lenet500.memory_summary()
    assert f"{s.peak_dealloc_mb:.6f}" == "59.167999"  # "about 59 MB"
    assert f"{s.peak_reuse_mb:.6f}" == "77.248001"    # "about 77 MB"
    assert 55 <= s.peak_dealloc_mb <= 62 and 70 <= s.peak_reuse_mb <= 85  # SPEC.md:566 bounds
    assert f"{s.param_mb:.6f}" == "3.448640"          # 431,080 params + velocities
    assert f"{s.workspace_mb:.6f}" == "64.000000"     # max(cv1 28.8, cv2 64.0)


def test_workspace_cap_zero():
    s = compile_network("lenet", 500, workspace_cap_mb=0).memory_summary()
    assert s.workspace_mb == 0.0


def test_param_order(lenet500):
    # SPEC.md:58
    assert [p.name for p in lenet500.params] == ["cv1_W", "cv1_B", "cv2_W", "cv2_B", "fc1_W", "fc1_B", "fc2_W",
                                                 "fc2_B"]
    assert sum(p.count for p in lenet500.params) == 431080


def test_dealloc_column_returns_to_zero(lenet500):
    rows = my_rows(lenet500)
    assert rows[-1]["total"] == "0.000000"
    reuse = [float(r["reuse"]) for r in rows]
    assert all(b >= a for a, b in zip(reuse, reuse[1:]))  # SPEC.md:407 monotone
