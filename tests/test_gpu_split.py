"""Two-kernel fast forward (gf_joint_coeffs + gf_joint_apply, the path
gf_joint_fwd takes on large images): parity with the oracle, agreement with
the one-kernel tile forward, guard bands, status semantics and bitwise row
bands.

gf_joint_coeffs restates gf/guided.py:136-149 + :170-173 (window moments,
slope, intercept of every low-res cell); gf_joint_apply gf/guided.py:174-178
(bilinear resize of both + affine combine).  Bars: fp32 outputs <= 1e-4 on
[0,1] images (north_star); coefficients compared relative to their range.
"""

import ctypes

import numpy as np
import pytest
import torch

import workloads
from oracle import gf_oracle as O
from paper_1803_05619_b200.sharding import joint_band_backward, joint_band_forward, row_bands

pytestmark = pytest.mark.gpu

GUARD = 4096
SENTINEL = 1.2345e-30


@pytest.fixture(scope="module")
def lib():
    from paper_1803_05619_b200 import _lib

    assert torch.cuda.is_available(), "gpu tests need CUDA"
    return _lib.load()


@pytest.fixture(scope="module")
def gfb():
    import paper_1803_05619_b200 as m

    return m


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ok(lib, rc):
    assert rc == 0, lib.gf_last_error().decode(errors="replace")


def oracle_coeffs(lr_x, lr_y, r, eps):
    """slope, intercept per plane (float64) from the oracle's window moments."""
    X, Y = lr_x.double().cpu().numpy(), lr_y.double().cpu().numpy()
    A = np.empty_like(X)
    Bc = np.empty_like(X)
    for b in range(X.shape[0]):
        g = np.ascontiguousarray(np.transpose(X[b], (1, 2, 0)))
        s = np.ascontiguousarray(np.transpose(Y[b], (1, 2, 0)))
        m = O.window_moments(g, s, r, eps)
        A[b] = np.transpose(m[4], (2, 0, 1))
        Bc[b] = np.transpose(m[5], (2, 0, 1))
    return A, Bc


def coeffs(lib, lr_x, lr_y, r, eps):
    B, C, h, w = lr_x.shape
    A, Bc = torch.empty_like(lr_x), torch.empty_like(lr_x)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    ok(lib, lib.gf_joint_coeffs(0, lr_x.data_ptr(), lr_y.data_ptr(), A.data_ptr(), Bc.data_ptr(),
                                B, C, h, w, r, eps, st.data_ptr(), stream()))
    torch.cuda.synchronize()
    return A, Bc, int(st.item())


def apply(lib, A, Bc, hr_x):
    B, C, h, w = A.shape
    H, W = hr_x.shape[2:]
    out = torch.empty_like(hr_x)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    ok(lib, lib.gf_joint_apply(0, A.data_ptr(), Bc.data_ptr(), hr_x.data_ptr(), out.data_ptr(), B,
                               C, h, w, H, W, st.data_ptr(), stream()))
    torch.cuda.synchronize()
    return out, int(st.item())


# widths: multiples of 4 (segment walk; 4 or 8 columns per lane), one strip and
# several, a ragged last strip; 125 / 30 (w % 4 != 0: the tile kernel)
SHAPES = [(37, 44), (64, 256), (130, 132), (16, 512), (50, 125), (9, 30), (2, 4), (300, 768),
          # heights around the 16-row pieces and below the window, widths around the strips
          (2, 8), (3, 4), (17, 12), (15, 124), (16, 128), (33, 252), (5, 248)]


@pytest.mark.parametrize("r", [0, 1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("h,w", SHAPES)
def test_coeffs_and_apply_vs_oracle(lib, h, w, r):
    eps = 1e-4
    lr_x, lr_y, hr_x = workloads.joint_inputs(2, 3, 4 * h, 4 * w, seed=h + 7 * w + r,
                                              device="cuda")
    A, Bc, st = coeffs(lib, lr_x, lr_y, r, eps)
    assert st == 0
    Ao, Bo = oracle_coeffs(lr_x, lr_y, r, eps)
    # the slope is cov / (var + eps) with var ~ 1e-3: fp32 rounding of the
    # moments (~1e-7) shows as ~1e-3 of the slope range at the smallest
    # variances; the OUTPUT bar below is the north-star one
    sa = max(float(np.abs(Ao).max()), 1.0)
    assert float(np.abs(A.double().cpu().numpy() - Ao).max()) <= 2e-3 * sa
    assert float(np.abs(Bc.double().cpu().numpy() - Bo).max()) <= 2e-3 * sa
    out, st = apply(lib, A, Bc, hr_x)
    assert st == 0
    ref = O.joint_forward_nchw(lr_x.double().cpu().numpy(), lr_y.double().cpu().numpy(),
                               hr_x.double().cpu().numpy(), r, eps)
    assert float(np.abs(out.double().cpu().numpy() - ref).max()) <= 1e-4


@pytest.mark.parametrize("h,w,r", [(37, 44, 2), (130, 132, 1), (64, 256, 8), (50, 125, 3),
                                   (300, 768, 4)])
def test_split_forward_matches_tile_forward(lib, gfb, h, w, r):
    """gf_joint_fwd in mode 2 (two kernels) agrees with mode 1 (one kernel) to
    fp32 rounding of the halo coefficients, and the tape is the same slopes."""
    eps = 1e-4
    lr_x, lr_y, hr_x = workloads.joint_inputs(2, 3, 4 * h, 4 * w, seed=3 * h + w, device="cuda")
    p = gfb.GuidedFilterParams(r, eps)
    outs, slopes = [], []
    for mode in (1, 2):
        old = lib.gf_joint_fwd_mode(mode)
        try:
            o, tape = gfb.forward_joint(lr_x, hr_x, lr_y, p)
        finally:
            assert lib.gf_joint_fwd_mode(old) == mode
        outs.append(o)
        slopes.append(tape._slope_lo)
    assert float((outs[0] - outs[1]).abs().max()) <= 2e-5
    s = max(float(slopes[0].abs().max()), 1.0)
    assert float((slopes[0] - slopes[1]).abs().max()) <= 1e-4 * s
    A, _, _ = coeffs(lib, lr_x, lr_y, r, eps)
    assert torch.equal(A, slopes[1])  # the split forward's tape IS gf_joint_coeffs' slope


def test_split_backward_on_split_tape_vs_oracle(lib, gfb):
    h, w, r, eps = 96, 160, 2, 1e-4
    lr_x, lr_y, hr_x = workloads.joint_inputs(2, 3, 4 * h, 4 * w, seed=11, device="cuda")
    p = gfb.GuidedFilterParams(r, eps)
    old = lib.gf_joint_fwd_mode(2)
    try:
        out, tape = gfb.forward_joint(lr_x, hr_x, lr_y, p)
    finally:
        lib.gf_joint_fwd_mode(old)
    d = torch.randn(out.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    g = gfb.backward(tape, d)
    ref = O.joint_backward_nchw(*(t.double().cpu().numpy() for t in (lr_x, lr_y, hr_x, d)), r, eps)
    for got, want in zip((g.d_guide_lo, g.d_src, g.d_guide_hi), ref):
        err = float(np.abs(got.double().cpu().numpy() - want).max())
        assert err <= 1e-3 * float(np.abs(want).max())


def test_status_semantics(lib):
    """eps = 0 on a constant guide flags DEGENERATE from the coefficient
    kernel; non-finite coefficients flag NONFINITE_OUTPUT from the apply pass
    (gf/guided.py:146-147, :179-180)."""
    h, w = 32, 64
    lr_x = torch.full((1, 3, h, w), 0.5, device="cuda")
    lr_y = torch.rand(1, 3, h, w, device="cuda")
    _, _, st = coeffs(lib, lr_x, lr_y, 2, 0.0)
    assert st & 4  # GF_STATUS_DEGENERATE
    A = torch.rand(1, 3, h, w, device="cuda")
    Bc = torch.rand(1, 3, h, w, device="cuda")
    A[0, 1, 5, 7] = float("inf")
    _, st = apply(lib, A, Bc, torch.rand(1, 3, 4 * h, 4 * w, device="cuda"))
    assert st & 2  # GF_STATUS_NONFINITE_OUTPUT


class Guarded:
    def __init__(self, shape, fill, data=None):
        n = int(np.prod(shape))
        self.n = n
        self.buf = torch.full((n + 2 * GUARD,), fill, dtype=torch.float32, device="cuda")
        self.view = self.buf[GUARD:GUARD + n].view(*shape)
        if data is not None:
            self.view.copy_(data)
        self.fill = fill

    def intact(self):
        g = torch.cat([self.buf[:GUARD], self.buf[GUARD + self.n:]])
        return bool(torch.isnan(g).all()) if self.fill != self.fill else bool((g == self.fill).all())


@pytest.mark.parametrize("h,w,r", [(37, 44, 0), (33, 16, 5), (21, 72, 8), (2, 4, 1),
                                   (130, 68, 3), (16, 32, 2), (19, 30, 2), (40, 260, 4)])
def test_guard_bands(lib, h, w, r):
    """Inputs inside NaN bands, outputs inside sentinel bands: no out-of-bounds
    read reaches the arithmetic, no write leaves the tensors, results equal the
    unguarded call bit for bit."""
    g = torch.Generator(device="cuda").manual_seed(h * 100 + w + r)
    mk = lambda *s: torch.rand(*s, generator=g, device="cuda")  # noqa: E731
    lr_x, lr_y, hr_x = mk(2, 3, h, w), mk(2, 3, h, w), mk(2, 3, 4 * h, 4 * w)
    nan = float("nan")
    gi = [Guarded(t.shape, nan, t) for t in (lr_x, lr_y, hr_x)]
    gA, gB = Guarded(lr_x.shape, SENTINEL), Guarded(lr_x.shape, SENTINEL)
    go = Guarded(hr_x.shape, SENTINEL)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    ok(lib, lib.gf_joint_coeffs(0, gi[0].view.data_ptr(), gi[1].view.data_ptr(),
                                gA.view.data_ptr(), gB.view.data_ptr(), 2, 3, h, w, r, 1e-3,
                                st.data_ptr(), stream()))
    ok(lib, lib.gf_joint_apply(0, gA.view.data_ptr(), gB.view.data_ptr(), gi[2].view.data_ptr(),
                               go.view.data_ptr(), 2, 3, h, w, 4 * h, 4 * w, st.data_ptr(),
                               stream()))
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    for x in gi + [gA, gB, go]:
        assert x.intact()
    A, Bc, _ = coeffs(lib, lr_x, lr_y, r, 1e-3)
    out, _ = apply(lib, A, Bc, hr_x)
    assert torch.equal(A, gA.view) and torch.equal(Bc, gB.view) and torch.equal(out, go.view)


@pytest.mark.parametrize("r", [1, 2, 4])
@pytest.mark.parametrize("world,h", [(2, 256), (3, 300), (5, 517)])
def test_row_bands_bitwise_split(lib, gfb, r, world, h):
    """Row bands under the two-kernel forward are bitwise the whole image's
    (16-row pieces of the coefficient walk on full-image rows)."""
    w, eps, F = 192, 1e-4, 4
    lr_x, lr_y, hr_x = workloads.joint_inputs(2, 3, F * h, F * w, F, seed=200 + r, device="cuda")
    p = gfb.GuidedFilterParams(r, eps)

    def fwd(gl, gh, sl, pp, *, row_origin=0):  # no full_rows: the thread's mode decides
        return gfb.forward_joint(gl, gh, sl, pp, row_origin=row_origin)

    old = lib.gf_joint_fwd_mode(2)
    try:
        out, tape = fwd(lr_x, hr_x, lr_y, p)
        d_out = torch.randn(out.shape, device="cuda",
                            generator=torch.Generator("cuda").manual_seed(r))
        full = gfb.backward(tape, d_out)
        for band in row_bands(h, world, r, F, backward=True):
            o, dlx, dly, dhx = joint_band_backward(fwd, gfb.backward, p, lr_x, lr_y, hr_x, d_out,
                                                   band)
            A, B = band.hr_owned
            for name, got, ref in (("out", o, out[:, :, A:B]),
                                   ("d_lr_x", dlx, full.d_guide_lo[:, :, band.a:band.b]),
                                   ("d_lr_y", dly, full.d_src[:, :, band.a:band.b]),
                                   ("d_hr_x", dhx, full.d_guide_hi[:, :, A:B])):
                assert torch.equal(got, ref), (name, band.a, float((got - ref).abs().max()))
        for band in row_bands(h, world, r, F, backward=False):
            o = joint_band_forward(fwd, p, lr_x, lr_y, hr_x, band)
            A, B = band.hr_owned
            assert torch.equal(o, out[:, :, A:B]), ("fwd", band.a)
    finally:
        lib.gf_joint_fwd_mode(old)


def test_full_rows_selects_the_full_images_path(lib, gfb):
    """A band passes its full image's height; the band then takes the path the
    whole image takes (here: both below the threshold -> one kernel), so the
    default entry stays bitwise across bands."""
    h, w, r, F = 256, 192, 2, 4
    lr_x, lr_y, hr_x = workloads.joint_inputs(1, 3, F * h, F * w, F, seed=9, device="cuda")
    p = gfb.GuidedFilterParams(r, 1e-4)
    out, _ = gfb.forward_joint(lr_x, hr_x, lr_y, p)
    for band in row_bands(h, 2, r, F, backward=False):
        o = joint_band_forward(gfb.forward_joint, p, lr_x, lr_y, hr_x, band)
        A, B = band.hr_owned
        assert torch.equal(o, out[:, :, A:B])
    assert lib.gf_joint_fwd_mode(0) == 0  # the call restored the thread's mode
    with pytest.raises(ValueError):
        gfb.forward_joint(lr_x, hr_x, lr_y, p, full_rows=h - 1)


@pytest.mark.parametrize("h,w,r", [(64, 256, 1), (130, 132, 2), (37, 44, 3), (300, 768, 4)])
def test_ring_walk_is_bitwise_the_register_walk(lib, h, w, r):
    """r <= 4: the coefficient walk's cp.async ring (the default) and its
    register walk (variant hook 24) run the same arithmetic in the same order."""
    lr_x, lr_y, _ = workloads.joint_inputs(2, 3, 4 * h, 4 * w, seed=5 * h + w + r, device="cuda")
    A0, B0, _ = coeffs(lib, lr_x, lr_y, r, 1e-4)
    old = lib.gf_joint_fwd_variant(24)
    try:
        A1, B1, _ = coeffs(lib, lr_x, lr_y, r, 1e-4)
    finally:
        lib.gf_joint_fwd_variant(old)
    assert torch.equal(A0, A1) and torch.equal(B0, B1)


@pytest.mark.parametrize("h,w,r", [(37, 44, 2), (130, 132, 1), (64, 256, 4), (21, 72, 8)])
def test_hr_pass_tile_height_is_bitwise(lib, gfb, h, w, r):
    """The tape backward's hr pass on 32-row tiles (hook gf_joint_bwd_hr_tile(8),
    4 CTAs of 128 threads per SM; measured slower, kept as a variant) gives
    bitwise the 64-row tiles' gradients: products, row partials and column sums
    do not depend on the tile height."""
    lr_x, lr_y, hr_x = workloads.joint_inputs(2, 3, 4 * h, 4 * w, seed=h + w + r, device="cuda")
    p = gfb.GuidedFilterParams(r, 1e-4)
    out, tape = gfb.forward_joint(lr_x, hr_x, lr_y, p)
    d = torch.randn(out.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    g0 = gfb.backward(tape, d)
    old = lib.gf_joint_bwd_hr_tile(8)
    try:
        g1 = gfb.backward(tape, d)
    finally:
        assert lib.gf_joint_bwd_hr_tile(old) == 8
    for a, b in ((g0.d_src, g1.d_src), (g0.d_guide_lo, g1.d_guide_lo),
                 (g0.d_guide_hi, g1.d_guide_hi)):
        assert torch.equal(a, b)


def test_default_path_selection_by_size_and_workspace(lib):
    """gf_joint_fwd at the threshold (3 x 4096^2 = 48 Mi high-res elements): with
    a workspace it is the two-kernel forward (bitwise mode 2), without one the
    one-kernel forward (bitwise mode 1); just below the threshold always the
    one-kernel forward."""
    def fwd(lr_x, lr_y, hr_x, r, ws, mode):
        B, C, h, w = lr_x.shape
        out = torch.empty_like(hr_x)
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        old = lib.gf_joint_fwd_mode(mode)
        try:
            ok(lib, lib.gf_joint_fwd(0, lr_x.data_ptr(), lr_y.data_ptr(), hr_x.data_ptr(),
                                     out.data_ptr(), B, C, h, w, 4 * h, 4 * w, r, 1e-4,
                                     ws.data_ptr() if ws is not None else 0,
                                     ws.numel() if ws is not None else 0, st.data_ptr(), stream()))
        finally:
            lib.gf_joint_fwd_mode(old)
        torch.cuda.synchronize()
        assert int(st.item()) == 0
        return out

    assert lib.gf_joint_split_threshold() == 48 << 20
    for H, split in ((4096, True), (4092, False)):
        lr_x, lr_y, hr_x = workloads.joint_inputs(1, 3, H, H, seed=H, device="cuda")
        h = H // 4
        ws = torch.empty(lib.gf_joint_workspace_bytes(0, 1, 3, h, h, H, H, 2), dtype=torch.uint8,
                         device="cuda")
        auto = fwd(lr_x, lr_y, hr_x, 2, ws, 0)
        assert torch.equal(auto, fwd(lr_x, lr_y, hr_x, 2, ws, 2 if split else 1))
        one = fwd(lr_x, lr_y, hr_x, 2, None, 0)
        assert torch.equal(one, fwd(lr_x, lr_y, hr_x, 2, ws, 1))
        assert float((auto - one).abs().max()) <= 2e-5


def test_cuda_graph_capture_of_forward_and_backward(lib):
    """The two-kernel forward (TMA tensor maps passed by value, cp.async ring)
    and the tape backward capture into a CUDA graph; replays are bitwise the
    eager results (launch-bound loops can run as graphs)."""
    B, C, H, r, eps = 2, 3, 512, 2, 1e-4
    h = H // 4
    lx, ly, hx = workloads.joint_inputs(B, C, H, H, seed=3, device="cuda")
    d = torch.randn_like(hx)
    out, A = torch.empty_like(hx), torch.empty_like(lx)
    g = [torch.empty_like(lx), torch.empty_like(lx), torch.empty_like(hx)]
    ws = torch.empty(lib.gf_joint_workspace_bytes(0, B, C, h, h, H, H, r), dtype=torch.uint8,
                     device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    p = lambda t: t.data_ptr()  # noqa: E731

    def run(sp):
        ok(lib, lib.gf_joint_fwd_tape(0, p(lx), p(ly), p(hx), p(out), p(A), B, C, h, h, H, H, r,
                                      eps, p(ws), ws.numel(), p(st), sp))
        ok(lib, lib.gf_joint_bwd_tape(0, p(lx), p(ly), p(hx), p(A), p(d), p(g[0]), p(g[1]),
                                      p(g[2]), B, C, h, h, H, H, r, eps, 0, p(ws), ws.numel(),
                                      p(st), sp))

    old = lib.gf_joint_fwd_mode(2)
    try:
        run(torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        ref = [out.clone()] + [t.clone() for t in g]
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            run(s.cuda_stream)  # the per-device launch setup happens outside the capture
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            run(torch.cuda.current_stream().cuda_stream)
        for t in [out] + g:
            t.zero_()
        graph.replay()
        graph.replay()
        torch.cuda.synchronize()
    finally:
        lib.gf_joint_fwd_mode(old)
    assert int(st.item()) == 0
    for a, b in zip(ref, [out] + g):
        assert torch.equal(a, b)
