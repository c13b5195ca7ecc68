"""tcgen05 GEMM / implicit-GEMM conv kernels vs a plain PyTorch fp32 reference.

Tolerance: bf16 operands with fp32 accumulation, per-op relative error
(max |err| / max |ref|) <= 1e-2 (BASELINE.json north_star, tensor-core ops).
"""
import ctypes as C

import pytest

torch = pytest.importorskip("torch")

from paper_1701_02284_b200 import _native as nat  # noqa: E402

TOL = 1e-2
pytestmark = pytest.mark.gpu


def rel_err(out, ref):
    return ((out.float() - ref.float()).abs().max() / ref.float().abs().max().clamp_min(1e-6)).item()


def run_gemm(M, N, K, a_layout, b_layout, d_dtype, bias=False, relu=False, splits=0, alpha=1.0):
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16).cuda()
    B = torch.randn(N, K, generator=g).to(torch.bfloat16).cuda()
    bvec = torch.randn(N, generator=g).cuda() if bias else None
    Ast = A if a_layout == nat.TC_LAYOUT_K else A.t().contiguous()
    Bst = B if b_layout == nat.TC_LAYOUT_K else B.t().contiguous()
    dt = torch.bfloat16 if d_dtype == nat.TC_DTYPE_BF16 else torch.float32
    D = torch.zeros(M, N, dtype=dt, device="cuda")
    args = nat.GemmArgs(M=M, N=N, K=K, a_layout=a_layout, b_layout=b_layout, A=Ast.data_ptr(),
                        lda=Ast.shape[1], B=Bst.data_ptr(), ldb=Bst.shape[1], D=D.data_ptr(), ldd=N,
                        d_dtype=d_dtype, bias=bvec.data_ptr() if bias else None, relu=int(relu), alpha=alpha,
                        beta=0.0, splits=splits)
    ws_bytes = nat.lib().tc_gemm_workspace_bytes(C.byref(args))
    ws = torch.empty(max(ws_bytes, 4), dtype=torch.uint8, device="cuda")
    args.workspace = ws.data_ptr()
    args.workspace_bytes = ws_bytes
    nat.check(nat.lib().tc_gemm_bf16(C.byref(args), None))
    torch.cuda.synchronize()
    ref = alpha * (A.float() @ B.float().t())
    if bias:
        ref = ref + bvec
    if relu:
        ref = ref.clamp_min(0)
    return D, ref


@pytest.mark.parametrize("M,N,K,al,bl", [
    (256, 256, 512, 0, 0),
    (128, 128, 64, 0, 0),
    (200, 96, 368, 0, 0),
    (384, 384, 2304, 0, 0),
    (128, 4096, 6400, 0, 0),
    (256, 192, 256, 1, 0),
    (256, 192, 256, 0, 1),
    (256, 320, 512, 1, 1),
])
def test_gemm_layouts_bf16(M, N, K, al, bl):
    D, ref = run_gemm(M, N, K, al, bl, nat.TC_DTYPE_BF16)
    assert rel_err(D, ref) < TOL


def test_gemm_bias_relu():
    D, ref = run_gemm(300, 200, 320, 0, 0, nat.TC_DTYPE_BF16, bias=True, relu=True)
    assert rel_err(D, ref) < TOL


@pytest.mark.parametrize("splits", [1, 4, 0])
def test_gemm_splitk_f32(splits):
    D, ref = run_gemm(96, 4096, 4096, 1, 1, nat.TC_DTYPE_F32, splits=splits)
    assert rel_err(D, ref) < TOL


@pytest.mark.parametrize("b_layout", [0, 1])
def test_gemm_padded_columns_never_read_past_b(b_layout):
    """D has N = ceil8(out) columns but B has only `out` rows: the rows after B
    (here NaN poison) must never be read, and padded columns come out 0."""
    M, out, N, K = 64, 10, 16, 504
    g = torch.Generator(device="cpu").manual_seed(3)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16).cuda()
    Breal = torch.randn(out, K, generator=g).to(torch.bfloat16)
    if b_layout == 0:
        buf = torch.full((N, K), float("nan"), dtype=torch.bfloat16)
        buf[:out] = Breal
        ldb = K
    else:
        buf = torch.full((K, N), float("nan"), dtype=torch.bfloat16)
        buf[:, :out] = Breal.t()
        ldb = N
    buf = buf.cuda()
    D = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda")
    bias = torch.randn(out, generator=g).cuda()
    args = nat.GemmArgs(M=M, N=N, K=K, a_layout=0, b_layout=b_layout, A=A.data_ptr(), lda=K, B=buf.data_ptr(),
                        ldb=ldb, D=D.data_ptr(), ldd=N, d_dtype=nat.TC_DTYPE_BF16, bias=bias.data_ptr(), relu=1,
                        alpha=1.0, bias_n=out, b_rows=out)
    ws_bytes = nat.lib().tc_gemm_workspace_bytes(C.byref(args))
    ws = torch.empty(max(ws_bytes, 4), dtype=torch.uint8, device="cuda")
    args.workspace, args.workspace_bytes = ws.data_ptr(), ws_bytes
    nat.check(nat.lib().tc_gemm_bf16(C.byref(args), None))
    torch.cuda.synchronize()
    ref = (A.float() @ Breal.float().cuda().t() + bias).clamp_min(0)
    assert torch.isfinite(D.float()).all()
    assert torch.all(D[:, out:] == 0)
    assert rel_err(D[:, :out], ref) < TOL


def nhwc_pad(x_nchw, cs):
    n, c, h, w = x_nchw.shape
    out = torch.zeros(n, h, w, cs, dtype=torch.bfloat16, device=x_nchw.device)
    out[..., :c] = x_nchw.permute(0, 2, 3, 1).to(torch.bfloat16)
    return out


def conv_case(N, C_, H, W, K, R, stride, pad, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = torch.randn(N, C_, H, W, generator=g).to(torch.bfloat16).float().cuda()
    w = (torch.randn(K, C_, R, R, generator=g) * 0.1).to(torch.bfloat16).float().cuda()
    b = torch.randn(K, generator=g).cuda()
    Ho = (H + 2 * pad - R) // stride + 1
    Wo = (W + 2 * pad - R) // stride + 1
    cs = (C_ + 7) // 8 * 8
    ks = (K + 7) // 8 * 8
    d = nat.ConvDesc(N=N, C=C_, H=H, W=W, K=K, R=R, S=R, stride=stride, pad=pad, Ho=Ho, Wo=Wo, cs=cs, ks=ks)
    return x, w, b, d


def w_krsc(w, cs):
    K, C_, R, S = w.shape
    out = torch.zeros(K, R, S, cs, dtype=torch.bfloat16, device=w.device)
    out[..., :C_] = w.permute(0, 2, 3, 1).to(torch.bfloat16)
    return out


def w_rskc(w, cs, ks):
    K, C_, R, S = w.shape
    out = torch.zeros(R, S, ks, cs, dtype=torch.bfloat16, device=w.device)
    out[:, :, :K, :C_] = w.permute(2, 3, 0, 1).to(torch.bfloat16)
    return out


CONV_CASES = [
    (2, 8, 13, 13, 64, 3, 1, 1),
    (2, 3, 35, 35, 96, 11, 4, 0),
    (2, 20, 12, 12, 50, 5, 1, 0),
    (2, 64, 14, 14, 128, 1, 1, 0),
    (2, 96, 27, 27, 256, 5, 1, 2),
    (2, 64, 16, 16, 128, 1, 2, 0),
    (2, 32, 15, 15, 48, 3, 2, 1),
]

# channel strides that are whole 64-channel blocks take the TMA im2col operand path
# (fprop A, bwd-data A for stride 1, bwd-filter B); odd extents, pad 0/1/2, strides 1/2
IM2COL_CASES = [
    (2, 64, 13, 13, 128, 3, 1, 1),
    (2, 128, 15, 15, 64, 3, 2, 1),
    (3, 64, 9, 11, 192, 5, 1, 2),
    (5, 64, 7, 7, 64, 3, 1, 0),
    (1, 256, 13, 13, 384, 3, 1, 1),
    # 32-channel blocks (SWIZZLE_64B boxes): channel strides 96 / 160 / 32, dgrad ks 96 / 160
    (2, 160, 9, 9, 96, 3, 1, 1),
    (3, 96, 13, 13, 160, 3, 1, 1),
    (2, 32, 14, 14, 96, 5, 1, 2),
    (1, 96, 12, 11, 192, 3, 2, 0),
    (2, 96, 26, 26, 256, 5, 1, 2),
    # Cout <= 64: the filter gradient runs swapped (im2col(x)^T dy, transposed reduce)
    (3, 64, 9, 9, 16, 3, 1, 1),
    (2, 128, 10, 10, 32, 1, 1, 0),
    (2, 64, 11, 11, 48, 3, 2, 1),
]


# stride-1 convs over 64-multiple channel strides whose tiles keep >= 80% valid pixels take the
# halo-tile path (tc_conv_halo.cuh): tile row stride wr = 16 / 32 / 64 / 128, several x / y tiles,
# pad 0 / 1 / 2, 3x3 and 5x5, several channel blocks and column tiles (N = 96 / 128 / 384)
HALO_CASES = [
    (2, 64, 56, 56, 128, 3, 1, 1),    # wr 32, 2 x-tiles, 14 y-tiles
    (2, 64, 27, 27, 128, 5, 1, 2),    # wr 32, one x-tile (27 <= 28 valid columns), 5x5
    (2, 64, 56, 56, 96, 3, 1, 0),     # pad 0 (space-to-depth first layer shape), N = 96
    (2, 64, 16, 14, 64, 3, 1, 1),     # wr 16 (two output rows per 32-row chunk)
    (1, 64, 6, 62, 128, 3, 1, 1),     # wr 64
    (1, 64, 3, 126, 64, 3, 1, 1),     # wr 128
    (2, 128, 28, 28, 384, 3, 1, 1),   # 2 channel blocks, 256-wide column tiles
    (1, 256, 30, 30, 256, 3, 1, 1),   # 4 channel blocks
    (2, 64, 20, 20, 32, 5, 1, 2),     # filter gradient with K <= 64: the tap-pair (swapped) form, 5x5
    (2, 128, 14, 14, 48, 3, 1, 1),    # K = 48, two channel blocks
    (2, 64, 30, 30, 96, 3, 1, 0),     # K = 96: tap pairs against two 64-channel dy atoms (N = 96)
    (2, 16, 28, 28, 32, 5, 1, 2),     # 16 channels: one zero-filled partial block, one 16-channel MMA step
    (2, 24, 14, 14, 64, 5, 1, 2),     # 24 channels (two MMA steps), 14 x 14 under 5 x 5: 38% valid rows
    (2, 48, 7, 7, 128, 5, 1, 2),      # 7 x 7 image, one tile per image
    (2, 96, 14, 14, 208, 3, 1, 1),    # K = 208: bwd-data reduces over 3 full + 1 partial dy block
    (2, 384, 7, 7, 192, 3, 1, 1),     # 7 x 7 under 3 x 3 with wide N (6 channel blocks)
    (2, 144, 14, 14, 160, 3, 1, 1),   # 144 channels: a 16-column partial chunk in the padded workspace, K = 160
    (2, 112, 14, 14, 224, 3, 1, 1),   # 112 channels (two blocks, the second 48 wide), K = 224
    (2, 96, 27, 27, 256, 5, 1, 2),    # AlexNet conv2: filter gradient with MMA N = 96, 5 taps per group
    (2, 32, 14, 14, 128, 3, 1, 1),    # filter gradient N = 32 (two tap groups of 5 + 4)
]


# the last three take the first-layer fprop kernel (tc_conv_c4.cuh): 64 outputs, whole 128-pixel
# tiles, 3x3/1 (VGG conv1_1), 7x7/2 pad 3 (GoogLeNet / ResNet conv1), tiles spanning 3-4 rows
@pytest.mark.parametrize("case", [(2, 3, 35, 35, 96, 11, 4, 0), (2, 3, 32, 32, 64, 7, 2, 3), (2, 1, 28, 28, 20, 5, 1, 0),
                                  (2, 3, 64, 64, 64, 3, 1, 1), (2, 3, 128, 128, 64, 7, 2, 3), (1, 3, 96, 96, 64, 7, 2, 3)])
def test_conv_channel_stride4_fwd_and_filter(case):
    """First-layer convs: input staged with channel stride 4 (8-byte tap gathers),
    filter rows padded to a multiple of 8 (wld)."""
    x, w, b, d = conv_case(*case)
    d.cs = 4
    d.wld = (d.R * d.S * 4 + 7) // 8 * 8
    xs = nhwc_pad(x, 4)
    wk = torch.zeros(d.K, d.wld, dtype=torch.bfloat16, device="cuda")
    wk[:, :d.R * d.S * 4] = w_krsc(w, 4).reshape(d.K, -1)
    y = torch.full((d.N, d.Ho, d.Wo, d.ks), float("nan"), dtype=torch.bfloat16, device="cuda")
    nat.check(nat.lib().tc_conv2d_fwd(C.byref(d), xs.data_ptr(), wk.data_ptr(), b.data_ptr(), 0, y.data_ptr(),
                                      None, 0, None))
    ref = torch.nn.functional.conv2d(x, w, b, stride=d.stride, padding=d.pad).permute(0, 2, 3, 1)
    torch.cuda.synchronize()
    assert rel_err(y[..., :d.K], ref) < TOL
    g = torch.Generator(device="cpu").manual_seed(6)
    dy = torch.randn(d.N, d.K, d.Ho, d.Wo, generator=g).to(torch.bfloat16).float().cuda()
    dw = torch.full((d.K, d.wld), float("nan"), dtype=torch.float32, device="cuda")
    wsb = nat.lib().tc_conv2d_workspace_bytes(C.byref(d), 2)
    wsp = torch.empty(max(wsb, 4), dtype=torch.uint8, device="cuda")
    nat.check(nat.lib().tc_conv2d_bwd_filter(C.byref(d), nhwc_pad(dy, d.ks).data_ptr(), xs.data_ptr(), dw.data_ptr(),
                                             wsp.data_ptr(), wsb, None))
    torch.cuda.synchronize()
    refw = torch.nn.grad.conv2d_weight(x, w.shape, dy, stride=d.stride, padding=d.pad).permute(0, 2, 3, 1)
    got = dw[:, :d.R * d.S * 4].reshape(d.K, d.R, d.S, 4)[..., :d.C]
    assert rel_err(got, refw) < TOL


@pytest.mark.parametrize("case", CONV_CASES + IM2COL_CASES + HALO_CASES)
def test_conv_fwd(case):
    x, w, b, d = conv_case(*case)
    xs = nhwc_pad(x, d.cs)
    ws = w_krsc(w, d.cs)
    y = torch.full((d.N, d.Ho, d.Wo, d.ks), float("nan"), dtype=torch.bfloat16, device="cuda")
    nat.check(nat.lib().tc_conv2d_fwd(C.byref(d), xs.data_ptr(), ws.data_ptr(), b.data_ptr(), 0, y.data_ptr(),
                                      None, 0, None))
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x, w, b, stride=d.stride, padding=d.pad).permute(0, 2, 3, 1)
    assert rel_err(y[..., :d.K], ref) < TOL
    assert torch.all(y[..., d.K:] == 0)


@pytest.mark.parametrize("case", CONV_CASES[2:] + [(2, 8, 13, 13, 64, 3, 1, 1)] + IM2COL_CASES + HALO_CASES)
def test_conv_bwd_data(case):
    x, w, b, d = conv_case(*case, seed=1)
    g = torch.Generator(device="cpu").manual_seed(5)
    dy = torch.randn(d.N, d.K, d.Ho, d.Wo, generator=g).to(torch.bfloat16).float().cuda()
    dys = nhwc_pad(dy, d.ks)
    wr = w_rskc(w, d.cs, d.ks)
    dx = torch.full((d.N, d.H, d.W, d.cs), float("nan"), dtype=torch.bfloat16, device="cuda")
    nat.check(nat.lib().tc_conv2d_bwd_data(C.byref(d), dys.data_ptr(), wr.data_ptr(), dx.data_ptr(), None, 0, None))
    torch.cuda.synchronize()
    ref = torch.nn.grad.conv2d_input(x.shape, w, dy, stride=d.stride, padding=d.pad).permute(0, 2, 3, 1)
    assert rel_err(dx[..., :d.C], ref) < TOL


@pytest.mark.parametrize("case", CONV_CASES + IM2COL_CASES + HALO_CASES)
def test_conv_bwd_filter(case):
    x, w, b, d = conv_case(*case, seed=2)
    g = torch.Generator(device="cpu").manual_seed(6)
    dy = torch.randn(d.N, d.K, d.Ho, d.Wo, generator=g).to(torch.bfloat16).float().cuda()
    xs = nhwc_pad(x, d.cs)
    dys = nhwc_pad(dy, d.ks)
    dw = torch.full((d.K, d.R, d.S, d.cs), float("nan"), dtype=torch.float32, device="cuda")
    wsb = nat.lib().tc_conv2d_workspace_bytes(C.byref(d), 2)
    wsp = torch.empty(max(wsb, 4), dtype=torch.uint8, device="cuda")
    nat.check(nat.lib().tc_conv2d_bwd_filter(C.byref(d), dys.data_ptr(), xs.data_ptr(), dw.data_ptr(),
                                             wsp.data_ptr(), wsb, None))
    torch.cuda.synchronize()
    ref = torch.nn.grad.conv2d_weight(x, w.shape, dy, stride=d.stride, padding=d.pad).permute(0, 2, 3, 1)
    assert rel_err(dw[..., :d.C], ref) < TOL


@pytest.mark.parametrize("case", HALO_CASES + [(2, 64, 56, 56, 192, 3, 1, 1), (2, 128, 28, 28, 192, 3, 1, 1)])
def test_conv_fwd_deterministic(case):
    """Bit-identical output across repeated launches and output-buffer contents (bias + ReLU
    epilogue): every output element is written exactly once from a fixed summation order."""
    x, w, b, d = conv_case(*case)
    xs = nhwc_pad(x, d.cs)
    ws = w_krsc(w, d.cs)
    outs = []
    for fill in (float("nan"), 0.0, 7.0):
        y = torch.full((d.N, d.Ho, d.Wo, d.ks), fill, dtype=torch.bfloat16, device="cuda")
        nat.check(nat.lib().tc_conv2d_fwd(C.byref(d), xs.data_ptr(), ws.data_ptr(), b.data_ptr(), 1, y.data_ptr(),
                                          None, 0, None))
        torch.cuda.synchronize()
        outs.append(y.clone())
    for o in outs[1:]:
        assert torch.equal(o.view(torch.int16), outs[0].view(torch.int16))


@pytest.mark.parametrize("case", [(16, 512, 14, 14, 512, 3, 1, 1), (16, 128, 28, 28, 128, 3, 1, 1),
                                  (8, 64, 28, 28, 96, 3, 1, 1), (8, 64, 30, 30, 64, 3, 1, 1),
                                  (16, 256, 14, 14, 512, 1, 1, 0), (16, 256, 14, 14, 128, 1, 1, 0),
                                  (16, 256, 14, 14, 32, 1, 1, 0), (8, 192, 7, 7, 384, 3, 1, 1),
                                  (4, 3, 64, 64, 64, 3, 1, 1)])
def test_wgrad_bias_fold_under_concurrent_load(case):
    """The folded bias gradient (halo / first-layer filter-gradient epilogue warps or the generic
    GEMM's warps 2-3 summing the staged dy tiles; 1x1 cases cover the plain, CTA-pair and swapped
    forms) equals the fp64 pixel sum of dy to fp32 rounding and is bit-identical across repeated
    runs while another stream keeps the SMs busy (the stage-release ordering the sums depend on)."""
    L = nat.lib()
    L.tcb_test_conv2d_bwd_filter_bias.argtypes = [C.POINTER(nat.ConvDesc)] + [C.c_void_p] * 5 + [C.c_size_t, C.c_void_p]
    x, w, b, d = conv_case(*case, seed=2)
    g = torch.Generator(device="cpu").manual_seed(6)
    dy = torch.randn(d.N, d.K, d.Ho, d.Wo, generator=g).to(torch.bfloat16).float().cuda()
    xs, dys = nhwc_pad(x, d.cs), nhwc_pad(dy, d.ks)
    ref = dys.double().sum(dim=(0, 1, 2))[: d.K]
    wsb = L.tc_conv2d_workspace_bytes(C.byref(d), 2)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    dw = torch.empty(d.K, d.R, d.S, d.cs, dtype=torch.float32, device="cuda")
    s_main, s_noise = torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=0)
    big = torch.randn(32 << 20, device="cuda")
    outs = []
    for trial in range(12):
        db = torch.full((d.K,), float("nan"), device="cuda")
        torch.cuda.synchronize()
        if trial % 2:
            with torch.cuda.stream(s_noise):
                for _ in range(10):
                    big.mul_(1.0000001)
        nat.check(L.tcb_test_conv2d_bwd_filter_bias(C.byref(d), dys.data_ptr(), xs.data_ptr(), dw.data_ptr(),
                                                    db.data_ptr(), ws.data_ptr(), wsb, C.c_void_p(s_main.cuda_stream)))
        torch.cuda.synchronize()
        outs.append(db.clone())
    assert float((outs[0].double() - ref).abs().max() / ref.abs().max()) < 1e-5
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
