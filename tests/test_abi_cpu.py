"""The C-ABI library loads without a GPU and exports every entry point that
include/*.h declares; the oracle library exports everything tc_oracle.h
declares.  No compute calls (no device here)."""
import ctypes as C
import glob
import os
import re

from paper_1701_02284_b200 import _native as nat

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(pattern, files):
    names = set()
    for f in files:
        src = open(f).read()
        names |= set(re.findall(pattern, src))
    return names


def test_product_exports_all_declared_symbols():
    names = declared(r"TC_API\s+[\w\s\*]*?\b(tc_\w+)\s*\(", glob.glob(os.path.join(ROOT, "include", "*.h")))
    assert len(names) > 30
    lib = nat.lib()
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing


def test_oracle_exports_all_declared_symbols():
    from oracle import oracle as orc

    names = declared(r"ORC_API\s+[\w\s\*]*?\b(orc_\w+)\s*\(", [os.path.join(ROOT, "oracle", "tc_oracle.h")])
    for t in ("f32", "f64"):  # macro-generated per-op entries
        names |= {f"orc_{op}_{t}" for op in ("conv_fwd", "conv_bwd_data", "conv_bwd_filter", "conv_bwd_bias",
                                             "pool_fwd", "pool_bwd", "lrn_fwd", "lrn_bwd", "softmax_fwd",
                                             "softmax_bwd", "bn_fwd", "bn_bwd", "matmul")}
    lib = orc.lib()
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing


def test_product_does_not_link_the_oracle():
    # the product path never routes through the CPU oracle (no symbol, no dependency)
    lib = C.CDLL(nat.LIB_PATH)
    assert not hasattr(lib, "orc_step")
    deps = os.popen(f"ldd {nat.LIB_PATH}").read()
    assert "tc_oracle" not in deps


def test_status_text_on_bad_args():
    lib = nat.lib()
    assert lib.tc_gemm_bf16(None, None) == 3  # TC_INVALID_ARG without touching a device
    assert b"bad shape" in lib.tc_last_error()
