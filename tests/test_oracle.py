"""Pins the CPU oracle before it is trusted as the parity checker:
SPEC `examples:` lines, f64 finite differences for every primitive
(acceptance 3), the hand-stepped solver (acceptance 5,
SPEC.md:569), pool mode semantics (acceptance 8), the workspace
dual path (acceptance 11) and LeNet end to end (acceptance 6)."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_1701_02284_b200.network import compile_network

L = orc.lib()
rng = np.random.default_rng(0)


# ---------------------------------------------------------------- SPEC examples
def test_conv_all_fours():
    x = np.ones((1, 1, 3, 3), np.float32)
    w = np.ones((1, 1, 2, 2), np.float32)
    y = np.empty((1, 1, 2, 2), np.float32)
    L.orc_conv_fwd_f32(x, w, None, y, 1, 1, 3, 3, 1, 2, 2, 1, 0, 0)
    assert np.all(y == 4.0)


def test_softmax_zero_row():
    x = np.zeros((1, 10), np.float32)
    y = np.empty_like(x)
    L.orc_softmax_fwd_f32(x, y, 1, 10)
    assert np.allclose(y, 0.1, atol=1e-7)


def test_softmax_rows_sum_to_one():
    x = rng.standard_normal((7, 13)).astype(np.float32) * 5
    y = np.empty_like(x)
    L.orc_softmax_fwd_f32(x, y, 7, 13)
    assert np.allclose(y.sum(1), 1.0, atol=1e-6) and np.all(y > 0) and np.all(y < 1)


def test_im2col_equals_direct():
    for (N, C, H, K, R, s, p) in [(2, 3, 9, 4, 3, 1, 1), (1, 5, 11, 6, 5, 2, 2), (2, 2, 8, 3, 1, 1, 0)]:
        x = rng.standard_normal((N, C, H, H)).astype(np.float32)
        w = rng.standard_normal((K, C, R, R)).astype(np.float32)
        b = rng.standard_normal(K).astype(np.float32)
        Ho = (H + 2 * p - R) // s + 1
        y1 = np.empty((N, K, Ho, Ho), np.float32)
        y2 = np.empty_like(y1)
        L.orc_conv_fwd_f32(x, w, b.ctypes.data, y1, N, C, H, H, K, R, R, s, p, 0)
        L.orc_conv_fwd_f32(x, w, b.ctypes.data, y2, N, C, H, H, K, R, R, s, p, 1)
        assert np.max(np.abs(y1 - y2) / (np.abs(y2) + 1e-3)) < 1e-5


def test_maxpool_bwd_bruteforce():
    x = np.array([[1, 3, 2, 2], [0, 3, 1, 5], [4, 4, 0, 0], [1, 2, 0, 0]], np.float64).reshape(1, 1, 4, 4)
    dy = np.array([10.0, 20.0, 30.0, 40.0]).reshape(1, 1, 2, 2)
    dx = np.empty_like(x)
    L.orc_pool_bwd_f64(dy, x, dx, 1, 1, 4, 4, 2, 2, 0, 1)
    want = np.zeros((4, 4))
    want[0, 1] = 10  # first max (3 at (0,1) before (1,1))
    want[1, 3] = 20
    want[2, 0] = 30  # tie 4,4 -> first
    want[2, 2] = 40  # all zeros -> first element of the window
    assert np.array_equal(dx[0, 0], want)
    y = np.empty((1, 1, 2, 2))
    idx = np.empty((1, 1, 2, 2), np.int32)
    L.orc_pool_fwd_f64(x, y, idx.ctypes.data, 1, 1, 4, 4, 2, 2, 0, 1)
    assert idx.ravel().tolist() == [1, 7, 8, 10]


# ---------------------------------------------------------------- finite differences (f64, rel <= 1e-6)
def fd_check(f, x, grad, n=12, tol=1e-6):
    """Central differences (f64).  ReLU / max-pool make the loss piecewise
    smooth, so a point may sit within h of a kink; the check passes when any
    step h in {1e-5, 1e-6, 1e-7} agrees to the relative tolerance."""
    flat = x.reshape(-1)
    g = grad.reshape(-1)
    idxs = rng.choice(flat.size, size=min(n, flat.size), replace=False)
    for i in idxs:
        errs = []
        for h in (1e-5, 1e-6, 1e-7):
            old = flat[i]
            flat[i] = old + h
            fp = f()
            flat[i] = old - h
            fm = f()
            flat[i] = old
            num = (fp - fm) / (2 * h)
            errs.append(abs(num - g[i]) / max(1.0, abs(num), abs(g[i])))
            if errs[-1] <= tol:
                break
        assert min(errs) <= tol, (i, g[i], errs)


def test_fd_conv():
    N, C, H, K, R, s, p = 2, 3, 6, 4, 3, 2, 1
    Ho = (H + 2 * p - R) // s + 1
    x = rng.standard_normal((N, C, H, H))
    w = rng.standard_normal((K, C, R, R))
    b = rng.standard_normal(K)
    cw = rng.standard_normal((N, K, Ho, Ho))

    def f():
        y = np.empty((N, K, Ho, Ho))
        L.orc_conv_fwd_f64(x, w, b.ctypes.data, y, N, C, H, H, K, R, R, s, p, 0)
        return float((y * cw).sum())

    dx = np.empty_like(x)
    dw = np.empty_like(w)
    db = np.empty_like(b)
    L.orc_conv_bwd_data_f64(cw, w, dx, N, C, H, H, K, R, R, s, p)
    L.orc_conv_bwd_filter_f64(cw, x, dw, N, C, H, H, K, R, R, s, p)
    L.orc_conv_bwd_bias_f64(cw, db, N, K, Ho * Ho)
    fd_check(f, x, dx)
    fd_check(f, w, dw)
    fd_check(f, b, db)


@pytest.mark.parametrize("is_max,k,s,p", [(1, 2, 2, 0), (1, 3, 2, 1), (0, 3, 1, 1), (0, 2, 2, 0)])
def test_fd_pool(is_max, k, s, p):
    N, C, H = 2, 3, 7
    Ho = (H + 2 * p - k) // s + 1
    x = rng.standard_normal((N, C, H, H))
    cw = rng.standard_normal((N, C, Ho, Ho))

    def f():
        y = np.empty((N, C, Ho, Ho))
        L.orc_pool_fwd_f64(x, y, None, N, C, H, H, k, s, p, is_max)
        return float((y * cw).sum())

    dx = np.empty_like(x)
    L.orc_pool_bwd_f64(cw, x, dx, N, C, H, H, k, s, p, is_max)
    fd_check(f, x, dx)


def test_fd_lrn():
    N, C, HW = 2, 7, 5
    x = rng.standard_normal((N, C, HW))
    cw = rng.standard_normal((N, C, HW))
    args = (5, 1e-1, 0.75, 1.0)

    def f():
        y = np.empty_like(x)
        L.orc_lrn_fwd_f64(x, y, N, C, HW, *args)
        return float((y * cw).sum())

    y = np.empty_like(x)
    L.orc_lrn_fwd_f64(x, y, N, C, HW, *args)
    dx = np.empty_like(x)
    L.orc_lrn_bwd_f64(cw, x, y, dx, N, C, HW, *args)
    fd_check(f, x, dx)


def test_fd_softmax():
    x = rng.standard_normal((3, 6))
    cw = rng.standard_normal((3, 6))

    def f():
        y = np.empty_like(x)
        L.orc_softmax_fwd_f64(x, y, 3, 6)
        return float((y * cw).sum())

    y = np.empty_like(x)
    L.orc_softmax_fwd_f64(x, y, 3, 6)
    dx = np.empty_like(x)
    L.orc_softmax_bwd_f64(cw, y, dx, 3, 6)
    fd_check(f, x, dx)


def test_fd_batchnorm():
    N, C, HW = 3, 4, 5
    x = rng.standard_normal((N, C, HW))
    g = rng.standard_normal(C)
    b = rng.standard_normal(C)
    cw = rng.standard_normal((N, C, HW))

    def f():
        y = np.empty_like(x)
        L.orc_bn_fwd_f64(x, g, b, y, N, C, HW, 1e-5)
        return float((y * cw).sum())

    dx, dg, db = np.empty_like(x), np.empty_like(g), np.empty_like(b)
    L.orc_bn_bwd_f64(cw, x, g.ctypes.data, dx.ctypes.data, dg.ctypes.data, db.ctypes.data, N, C, HW, 1e-5)
    fd_check(f, x, dx)
    fd_check(f, g, dg)
    fd_check(f, b, db)


@pytest.mark.parametrize("name", ["lenet", "inception"])
def test_fd_full_network_loss(name):
    """Full LeNet / inception-block loss at batch 2, f64."""
    net = compile_network(name, 2)
    o = orc.Oracle(net, seed=7, f64=True)
    o.init_params()
    x, y = orc.synth_batch(net, 7, 0)

    def loss():
        o.set_batch(x, y)
        return o.step(0, 0, update=False)

    loss()
    for i, p in enumerate(net.params):
        w = o.get_param(i)
        g = o.grad(i)

        def f():
            o.set_param(i, w)
            return loss()

        fd_check(f, w, g, n=4)
        o.set_param(i, w)


# ---------------------------------------------------------------- solver (acceptance 5)
def test_update_hand_stepped_three_iterations():
    net = compile_network("lenet", 4, lr=0.01, momentum=0.9, decay=0.0005)
    o = orc.Oracle(net, seed=3, f64=True)
    o.init_params()
    pi = 7  # fc2_B: lr_mult 1, decay_mult 1
    p = o.get_param(pi).astype(np.float64)
    v = np.zeros_like(p)
    for it in range(3):
        o.step(it, 0, update=True)
        g = o.grad(pi)
        v = 0.9 * v - 0.01 * (g + 0.0005 * p)
        p = p + v
        assert np.allclose(o.get_param(pi), p, rtol=0, atol=1e-7)


def test_update_example():  # Update([1,2],[10,10],-0.01,1) -> [0.9, 1.9]
    p = np.array([1.0, 2.0])
    p = 1.0 * p + -0.01 * np.array([10.0, 10.0])
    assert np.allclose(p, [0.9, 1.9])


# ---------------------------------------------------------------- pool modes (acceptance 8)
def test_reuse_mode_no_fresh_allocations_after_first_iteration():
    net = compile_network("lenet", 16, mode="reuse")
    o = orc.Oracle(net)
    o.init_params()
    o.step(0)
    a1 = o.pool_stats().allocs_from_os
    for it in range(1, 5):
        o.step(it)
    st = o.pool_stats()
    assert st.allocs_from_os == a1 and st.reuses > 0


def test_dealloc_mode_trace_matches_memplan():
    net = compile_network("lenet", 16, mode="dealloc")
    o = orc.Oracle(net)
    o.init_params()
    o.step(0)
    trace = o.live_trace()
    import csv
    import io
    rows = list(csv.reader(io.StringIO(net.memory_table(csv=True))))[1:]
    want = [round(float(r[3]) * 1e6) for r in rows]
    got = [int(t) for t in trace]
    assert len(got) == len(want)
    assert all(abs(a - b) <= 4 for a, b in zip(got, want))


def test_reuse_peak_below_static_bound():
    net = compile_network("lenet", 16, mode="reuse")
    o = orc.Oracle(net)
    o.init_params()
    o.step(0)
    assert o.pool_stats().os_bytes <= net.memory_summary().peak_reuse_bytes


# ---------------------------------------------------------------- workspace dual path (acceptance 11)
def test_workspace_cap_zero_direct_equals_im2col():
    net = compile_network("lenet", 8)
    a, b = orc.Oracle(net, seed=5), orc.Oracle(net, seed=5)
    a.init_params()
    b.init_params()
    b.set_workspace_cap(0.0)
    la, lb = a.step(0, update=False), b.step(0, update=False)
    assert abs(la - lb) <= 1e-5 * abs(la)
    for i in range(len(net.params)):
        ga, gb = a.grad(i), b.grad(i)
        assert np.max(np.abs(ga - gb)) <= 1e-5 * max(1e-3, np.max(np.abs(ga)))


# ---------------------------------------------------------------- data
def test_synth_deterministic():
    net = compile_network("lenet", 8)
    x1, y1 = orc.synth_batch(net, 7, 3)
    x2, y2 = orc.synth_batch(net, 7, 3)
    assert np.array_equal(x1, x2) and np.array_equal(y1, y2)
    x3, _ = orc.synth_batch(net, 7, 4)
    assert not np.array_equal(x1, x3)
    assert y1.min() >= 0 and y1.max() < 10


# ---------------------------------------------------------------- end to end (acceptance 6)
def test_lenet_end_to_end():
    net = compile_network("lenet", 64)
    o = orc.Oracle(net, seed=42)
    o.init_params()
    losses = [o.step(it) for it in range(200)]
    assert abs(losses[0] - np.log(10)) < 0.1
    assert np.mean(losses[-20:]) < 1.0
    assert o.test(10_000) > 0.85
