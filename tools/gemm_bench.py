#!/usr/bin/env python3
"""Kernel-level timing of the tcgen05 GEMM / implicit-GEMM conv entry points (CUDA events,
median of reps, inputs resident).  Shapes: plain GEMMs and the conv layers of the configs.

    python tools/gemm_bench.py [--which gemm,conv] [--net alexnet]
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1701_02284_b200 import _native as nat  # noqa: E402

CONVS = {  # (N, C, H, W, K, R, S, stride, pad)
    "alexnet": [(128, 3, 224, 224, 96, 11, 11, 4, 0), (128, 96, 26, 26, 256, 5, 5, 1, 2),
                (128, 256, 12, 12, 384, 3, 3, 1, 1), (128, 384, 12, 12, 384, 3, 3, 1, 1),
                (128, 384, 12, 12, 256, 3, 3, 1, 1)],
    "vgg16": [(64, 3, 224, 224, 64, 3, 3, 1, 1), (64, 64, 224, 224, 64, 3, 3, 1, 1), (64, 128, 112, 112, 128, 3, 3, 1, 1),
              (64, 256, 56, 56, 256, 3, 3, 1, 1), (64, 512, 28, 28, 512, 3, 3, 1, 1),
              (64, 512, 14, 14, 512, 3, 3, 1, 1)],
    "resnet50": [(64, 64, 56, 56, 64, 3, 3, 1, 1), (64, 64, 56, 56, 256, 1, 1, 1, 0),
                 (64, 256, 56, 56, 64, 1, 1, 1, 0), (64, 256, 14, 14, 256, 3, 3, 1, 1),
                 (64, 1024, 14, 14, 256, 1, 1, 1, 0), (64, 512, 7, 7, 512, 3, 3, 1, 1)],
}


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def gemm_case(M, N, K):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    args = nat.GemmArgs(M=M, N=N, K=K, a_layout=0, b_layout=0, A=A.data_ptr(), lda=K, B=B.data_ptr(), ldb=K,
                        D=D.data_ptr(), ldd=N, d_dtype=nat.TC_DTYPE_BF16, alpha=1.0, beta=0.0, splits=1)
    ms = timeit(lambda: nat.check(nat.lib().tc_gemm_bf16(C.byref(args), None)))
    return ms, 2.0 * M * N * K / (ms * 1e-3) / 1e12


def fc_case(M, N, K, a_mn, b_mn, f32_out):
    """FC-layer GEMMs of the step: wgrad is M=out, N=in, K=batch with both operands MN-major
    (activations stored [batch][features]) and an fp32 gradient; fwd / dgrad are K-major."""
    A = torch.randn(K, M, device="cuda").to(torch.bfloat16) if a_mn else torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(K, N, device="cuda").to(torch.bfloat16) if b_mn else torch.randn(N, K, device="cuda").to(torch.bfloat16)
    D = torch.empty(M, N, device="cuda", dtype=torch.float32 if f32_out else torch.bfloat16)
    ws = torch.empty(256 << 20, device="cuda", dtype=torch.uint8)
    args = nat.GemmArgs(workspace=ws.data_ptr(), workspace_bytes=ws.numel(), M=M, N=N, K=K, a_layout=nat.TC_LAYOUT_MN if a_mn else nat.TC_LAYOUT_K, A=A.data_ptr(),
                        lda=M if a_mn else K, b_layout=nat.TC_LAYOUT_MN if b_mn else nat.TC_LAYOUT_K, B=B.data_ptr(),
                        ldb=N if b_mn else K, D=D.data_ptr(), ldd=N,
                        d_dtype=nat.TC_DTYPE_F32 if f32_out else nat.TC_DTYPE_BF16, alpha=1.0, beta=0.0, splits=0)
    ms = timeit(lambda: nat.check(nat.lib().tc_gemm_bf16(C.byref(args), None)))
    byts = 2 * (M * K + N * K) + D.element_size() * M * N
    return ms, 2.0 * M * N * K / (ms * 1e-3) / 1e12, byts / (ms * 1e-3) / 1e9


def ceil8(v):
    return (v + 7) // 8 * 8


def conv_case(n, c, h, w, k, r, s, st, pad):
    L = nat.lib()
    ho, wo = (h + 2 * pad - r) // st + 1, (w + 2 * pad - s) // st + 1
    cs = 4 if c <= 4 else ceil8(c)
    ks = ceil8(k)
    d = nat.ConvDesc(N=n, C=c, H=h, W=w, K=k, R=r, S=s, stride=st, pad=pad, Ho=ho, Wo=wo, cs=cs, ks=ks,
                     wld=ceil8(r * s * cs))
    x = torch.randn(n, h, w, cs, device="cuda").to(torch.bfloat16)
    y = torch.randn(n, ho, wo, ks, device="cuda").to(torch.bfloat16)
    wt = torch.randn(k, d.wld, device="cuda").to(torch.bfloat16)
    wr = torch.randn(r * s * ks * max(cs, 8), device="cuda").to(torch.bfloat16)
    dw = torch.empty(k, d.wld, device="cuda")
    out = {}
    flops = 2.0 * n * ho * wo * k * c * r * s
    for which in range(3):
        wsb = L.tc_conv2d_workspace_bytes(C.byref(d), which)
        ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
        if which == 0:
            fn = lambda: nat.check(L.tc_conv2d_fwd(C.byref(d), x.data_ptr(), wt.data_ptr(), None, 0, y.data_ptr(),  # noqa
                                                   ws.data_ptr(), wsb, None))
        elif which == 1:
            if cs % 8:
                continue
            fn = lambda: nat.check(L.tc_conv2d_bwd_data(C.byref(d), y.data_ptr(), wr.data_ptr(), x.data_ptr(),  # noqa
                                                        ws.data_ptr(), wsb, None))
        else:
            fn = lambda: nat.check(L.tc_conv2d_bwd_filter(C.byref(d), y.data_ptr(), x.data_ptr(), dw.data_ptr(),  # noqa
                                                          ws.data_ptr(), wsb, None))
        ms = timeit(fn)
        out[["fwd", "dgrad", "wgrad"][which]] = (ms, flops / (ms * 1e-3) / 1e12)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="gemm,conv")
    ap.add_argument("--net", default="alexnet,vgg16,resnet50")
    ap.add_argument("--shapes", default="", help="explicit GEMM shapes MxNxK,MxNxK (bf16 out, K-major)")
    ap.add_argument("--fc", action="store_true", help="AlexNet FC GEMMs (fwd, dgrad, fp32 wgrad)")
    ap.add_argument("--small-k", action="store_true", help="GEMM shapes of 1x1 convs (epilogue-paced)")
    ap.add_argument("--conv-as-gemm", action="store_true", help="AlexNet conv GEMM views with dense operands")
    ap.add_argument("--only", default="", help="run only conv cases whose tuple text contains this")
    args = ap.parse_args()
    print(f"TCB_FORCE_BN={os.environ.get('TCB_FORCE_BN', '')} TCB_IM2COL={os.environ.get('TCB_IM2COL', '')}")
    if args.fc:
        for name, M, N, K, amn, bmn, f32 in [("fc6 fwd", 128, 4096, 9216, 0, 0, 0), ("fc6 dgrad", 128, 9216, 4096, 0, 1, 0),
                                             ("fc6 wgrad", 4096, 9216, 128, 1, 1, 1), ("fc7 fwd", 128, 4096, 4096, 0, 0, 0),
                                             ("fc7 wgrad", 4096, 4096, 128, 1, 1, 1)]:
            ms, tf, gbs = fc_case(M, N, K, amn, bmn, f32)
            print(f"{name:10s} M={M} N={N} K={K}: {ms*1e3:8.1f} us  {tf:7.1f} TF/s  {gbs:7.0f} GB/s")
        return
    if "gemm" in args.which:
        shapes = [(8192, 8192, 8192), (16384, 256, 4096), (16384, 128, 4096), (16384, 64, 4096), (4096, 4096, 4096)]
        if args.small_k:
            shapes = [(200704, 256, k) for k in (64, 128, 256, 512, 1024)] + [(200704, 64, 256), (50176, 1024, 256)]
        if args.shapes:
            shapes = [tuple(int(v) for v in t.split("x")) for t in args.shapes.split(",")]
        if args.conv_as_gemm:  # the GEMM views of im2col convs with dense operands (im2col cost excluded)
            shapes = [(86528, 96, 6400), (373248, 96, 576), (86528, 256, 2400), (18432, 384, 2304), (18432, 256, 3456)]
        for M, N, K in shapes:
            ms, tf = gemm_case(M, N, K)
            print(f"gemm {M}x{N}x{K}: {ms:.3f} ms {tf:.0f} TF/s")
    if "conv" in args.which:
        for net in args.net.split(","):
            for cv in CONVS[net]:
                if args.only and args.only not in str(cv):
                    continue
                r = conv_case(*cv)
                print(f"{net} conv {cv}: " + "  ".join(f"{k} {v[0]:.3f} ms {v[1]:.0f} TF/s" for k, v in r.items()))


if __name__ == "__main__":
    main()
