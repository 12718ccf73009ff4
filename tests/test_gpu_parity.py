"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the pinned CPU oracle.

Bars (north_star / SURVEY 8c):
  * fp64 instantiation vs reference golden values: the reference's own 1e-10
    (outputs) and 1e-9 relative (gradients) bars;
  * fp32 path: outputs max abs error <= 1e-4 on [0,1] images; gradients
    max|g - g_ref| / max|g_ref| <= 1e-3 per tensor.
"""

import numpy as np
import pytest
import torch

from oracle import gf_oracle as O

pytestmark = pytest.mark.gpu

OUT_TOL32 = 1e-4
GRAD_TOL32 = 1e-3


@pytest.fixture(scope="module")
def gfb():
    import paper_1803_05619_b200 as m

    assert torch.cuda.is_available(), "gpu tests need CUDA"
    return m


def rel_max(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max()) / max(float(np.abs(b).max()), 1e-30)


def abs_max(a, b):
    return float(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)).max())


def t32(a):
    return torch.from_numpy(np.ascontiguousarray(a)).float().cuda()


def npy(t):
    return t.detach().double().cpu().numpy()


# ---------------------------------------------------------------------------
# primitives
# ---------------------------------------------------------------------------

def test_filters_fp64_match_reference(gfb, golden):
    for name, c in golden.items():
        if name.startswith("mean"):
            r = int(c["r"])
            assert abs_max(gfb.mean_filter(c["x"], r), c["mean"]) <= 1e-12
            assert abs_max(gfb.mean_filter_adjoint(c["g"], r), c["adj"]) <= 1e-12
        elif name.startswith("bil"):
            oh, ow = c["out"].shape[:2]
            h, w = c["x"].shape[:2]
            assert abs_max(gfb.bilinear_resize(c["x"], oh, ow), c["out"]) <= 1e-14
            assert abs_max(gfb.bilinear_resize_adjoint(c["g"], h, w), c["adj"]) <= 1e-13


def test_filters_known_answers(gfb, golden):
    m = gfb.mean_filter(golden["ka_box"]["x"], 1)
    assert m[0, 0, 0] == pytest.approx(3.0, abs=1e-12)
    assert m[1, 1, 0] == pytest.approx(5.0, abs=1e-12)
    out = gfb.bilinear_resize(golden["ka_bilinear"]["x"], 1, 4)
    assert out.ravel().tolist() == [0.0, 0.5, 1.5, 2.0]
    g = np.random.default_rng(7).standard_normal((5, 4, 2))
    assert np.array_equal(gfb.bilinear_resize_adjoint(g, 5, 4), g)


def test_adjoint_identities(gfb):
    rng = np.random.default_rng(50)
    for _ in range(20):
        h, w, c = int(rng.integers(4, 20)), int(rng.integers(4, 20)), int(rng.integers(1, 4))
        r = int(rng.integers(0, 6))
        u = rng.standard_normal((h, w, c))
        v = rng.standard_normal((h, w, c))
        lhs = float(np.vdot(u, gfb.mean_filter(v, r)))
        rhs = float(np.vdot(gfb.mean_filter_adjoint(u, r), v))
        assert abs(lhs - rhs) <= 1e-9 * (abs(lhs) + 1.0)
        oh, ow = int(rng.integers(1, 24)), int(rng.integers(1, 24))
        g = rng.standard_normal((oh, ow, c))
        lhs = float(np.vdot(g, gfb.bilinear_resize(v, oh, ow)))
        rhs = float(np.vdot(gfb.bilinear_resize_adjoint(g, h, w), v))
        assert abs(lhs - rhs) <= 1e-9 * (abs(lhs) + 1.0)


# ---------------------------------------------------------------------------
# joint layer vs reference golden vectors
# ---------------------------------------------------------------------------

def _joint_cases(golden):
    return [(k, c) for k, c in sorted(golden.items()) if k.startswith("joint")]


def test_joint_fp64_matches_reference(gfb, golden):
    for name, c in _joint_cases(golden):
        p = gfb.GuidedFilterParams(int(c["r"]), float(c["eps"]))
        out, tape = gfb.forward_joint(c["guide_lo"], c["guide_hi"], c["src_lo"], p)
        assert isinstance(out, np.ndarray) and out.dtype == np.float64
        assert abs_max(out, c["out"]) <= 1e-10, name
        g = gfb.backward(tape, c["d_out"])
        for f in ("d_src", "d_guide_lo", "d_guide_hi"):
            assert rel_max(getattr(g, f), c[f]) <= 1e-9, (name, f)
        assert abs_max(tape.slope, c["slope"]) <= 1e-10


def test_joint_fp32_matches_reference(gfb, golden):
    for name, c in _joint_cases(golden):
        p = gfb.GuidedFilterParams(int(c["r"]), float(c["eps"]))
        gl, gh, sl = t32(c["guide_lo"]), t32(c["guide_hi"]), t32(c["src_lo"])
        out, tape = gfb.forward_joint(gl, gh, sl, p)
        assert out.dtype == torch.float32 and out.shape == gh.shape
        assert abs_max(npy(out), c["out"]) <= OUT_TOL32, name
        g = gfb.backward(tape, t32(c["d_out"]))
        for f in ("d_src", "d_guide_lo", "d_guide_hi"):
            assert rel_max(npy(getattr(g, f)), c[f]) <= GRAD_TOL32, (name, f)


def test_joint_fp32_generic_path_matches_reference(gfb, golden):
    from paper_1803_05619_b200 import _lib

    lib = _lib.load()
    old = lib.gf_force_generic(1)
    try:
        test_joint_fp32_matches_reference(gfb, golden)
    finally:
        lib.gf_force_generic(old)


# ---------------------------------------------------------------------------
# highres layer vs reference golden vectors
# ---------------------------------------------------------------------------

def test_highres_fp64_matches_reference(gfb, golden):
    for name, c in sorted(golden.items()):
        if not name.startswith("hr"):
            continue
        p = gfb.GuidedFilterParams(int(c["r"]), float(c["eps"]))
        if name.startswith("hrb"):  # 1-channel guide broadcast (NCHW extension)
            g = torch.from_numpy(c["guide"].transpose(2, 0, 1)[None].copy()).cuda()
            s = torch.from_numpy(c["src"].transpose(2, 0, 1)[None].copy()).cuda()
            d = torch.from_numpy(c["d_out"].transpose(2, 0, 1)[None].copy()).cuda()
            out, tape = gfb.forward_highres(g, s, p)
            gr = gfb.backward(tape, d)
            assert abs_max(npy(out)[0].transpose(1, 2, 0), c["out"]) <= 1e-10, name
            assert rel_max(npy(gr.d_src)[0].transpose(1, 2, 0), c["d_src"]) <= 1e-9
            assert rel_max(npy(gr.d_guide_hi)[0].transpose(1, 2, 0), c["d_guide"]) <= 1e-9
            continue
        out, tape = gfb.forward_highres(c["guide"], c["src"], p)
        assert abs_max(out, c["out"]) <= 1e-10, name
        gr = gfb.backward(tape, c["d_out"])
        assert gr.d_guide_lo is None
        assert rel_max(gr.d_src, c["d_src"]) <= 1e-9, name
        assert rel_max(gr.d_guide_hi, c["d_guide"]) <= 1e-9, name


def test_highres_fp32_matches_reference(gfb, golden):
    for name, c in sorted(golden.items()):
        if not name.startswith("hr"):
            continue
        p = gfb.GuidedFilterParams(int(c["r"]), float(c["eps"]))
        g = t32(c["guide"].transpose(2, 0, 1)[None])
        s = t32(c["src"].transpose(2, 0, 1)[None])
        out, tape = gfb.forward_highres(g, s, p)
        assert abs_max(npy(out)[0].transpose(1, 2, 0), c["out"]) <= OUT_TOL32, name
        gr = gfb.backward(tape, t32(c["d_out"].transpose(2, 0, 1)[None]))
        assert rel_max(npy(gr.d_src)[0].transpose(1, 2, 0), c["d_src"]) <= GRAD_TOL32, name
        assert rel_max(npy(gr.d_guide_hi)[0].transpose(1, 2, 0), c["d_guide"]) <= GRAD_TOL32


# ---------------------------------------------------------------------------
# guidance net + training step vs reference golden vectors
# ---------------------------------------------------------------------------

def test_guidance_net_matches_reference(gfb, golden):
    for name, c in sorted(golden.items()):
        if not name.startswith("gn"):
            continue
        params = {k[2:]: v for k, v in c.items() if k.startswith("p:")}
        cout, hidden, cin = params["conv2.weight"].shape[0], params["conv1.weight"].shape[0], \
            params["conv1.weight"].shape[1]
        net = gfb.GuidanceNet(cin, cout, hidden=hidden)
        net.load_parameters(params)
        y, tape = net.forward(c["x"])                    # float64 drop-in path
        assert abs_max(y, c["y"]) <= 1e-10, name
        dx, grads = net.backward(tape, c["dy"])
        assert rel_max(dx, c["dx"]) <= 1e-9, name
        for k, v in grads.items():
            assert rel_max(v, c["g:" + k]) <= 1e-9, (name, k)
        # fp32 path
        y32, tape32 = net.forward(t32(c["x"]))
        assert abs_max(npy(y32), c["y"]) <= 1e-5, name
        dx32, g32 = net.backward(tape32, t32(c["dy"]))
        assert rel_max(npy(dx32), c["dx"]) <= GRAD_TOL32, name
        for k, v in g32.items():
            assert rel_max(npy(v), c["g:" + k]) <= GRAD_TOL32, (name, k)


def test_guidance_net_seeded_init_matches_reference_draws(gfb):
    rng_a = np.random.default_rng(123)
    net = gfb.GuidanceNet(3, 3, hidden=15, kernel=1, rng=rng_a)
    want = O.guidance_init(3, 3, 15, np.random.default_rng(123))
    for k, v in net.parameters().items():
        assert np.array_equal(v.cpu().numpy(), want[k]), k


def test_train_step_matches_reference(gfb, golden):
    c = golden["train0"]
    params = {k[2:]: v for k, v in c.items() if k.startswith("p:")}
    net = gfb.GuidanceNet(3, 3, hidden=15)
    net.load_parameters(params)
    p = gfb.GuidedFilterParams(int(c["r"]), float(c["eps"]))
    nchw = lambda a: t32(a.transpose(0, 3, 1, 2))  # noqa: E731
    # default: the fused filter + MSE + backward (no output); return_out: the
    # forward -> mse_loss -> backward chain
    for return_out in (False, True):
        res = gfb.train_step(net, nchw(c["lr_x"]), nchw(c["hr_x"]), nchw(c["lr_y"]),
                             nchw(c["target"]), p, return_out=return_out)
        assert abs(float(res.loss) - float(c["loss"])) <= 1e-6 * max(1.0, float(c["loss"]))
        if return_out:
            assert abs_max(npy(res.out).transpose(0, 2, 3, 1), c["out"]) <= OUT_TOL32
        else:
            assert res.out is None
        assert rel_max(npy(res.d_lr_y).transpose(0, 2, 3, 1), c["d_lr_y"]) <= GRAD_TOL32
        assert rel_max(npy(res.d_lr_x).transpose(0, 2, 3, 1), c["d_lr_x"]) <= GRAD_TOL32
        assert rel_max(npy(res.d_hr_x).transpose(0, 2, 3, 1), c["d_hr_x"]) <= GRAD_TOL32
        grads = net.unpack(res.dparams)
        # conv2.bias's exact gradient is ~0 here (1e-16): judge every parameter
        # gradient against the largest one (relative-to-gradient-norm bar)
        scale = max(float(np.abs(c["g:" + k]).max()) for k in grads)
        for k, v in grads.items():
            assert abs_max(npy(v), c["g:" + k]) <= GRAD_TOL32 * scale, k


@pytest.mark.parametrize("B,C,h,w,r,eps", [
    (2, 3, 16, 32, 1, 1e-8),     # one tile per plane
    (1, 3, 37, 45, 2, 1e-4),     # ragged tiles on both axes
    (2, 1, 50, 70, 0, 1e-3),     # r = 0
    (1, 3, 40, 66, 5, 1e-2),     # r > 4 (no static column taps)
    (1, 2, 33, 97, 8, 1e-4),     # r = 8, ragged
    (1, 1, 2, 2, 1, 1e-2),       # smallest fused shape
])
def test_joint_mse_backward_matches_oracle(gfb, B, C, h, w, r, eps):
    """Fused filter + MSE + backward vs the oracle's forward_joint -> mse_loss ->
    backward chain (batch mean, gf/training.py:93-101, 230-235)."""
    rng = np.random.default_rng(1000 + 7 * h + w + r)
    H, W = 4 * h, 4 * w
    gl = rng.uniform(0, 1, (B, h, w, C))
    sl = np.clip(0.7 * gl + 0.1 + rng.normal(0, 0.05, gl.shape), 0, 1)
    gh = rng.uniform(0, 1, (B, H, W, C))
    tg = rng.uniform(0, 1, (B, H, W, C))
    g = lambda a: t32(a.transpose(0, 3, 1, 2))  # noqa: E731
    assert gfb._lib.load().gf_joint_is_fused(0, B, C, h, w, H, W, r)
    loss, grads, status = gfb.joint_mse_backward(g(gl), g(gh), g(sl), g(tg),
                                                 gfb.GuidedFilterParams(r, eps))
    assert status.bits() == 0
    want_loss = 0.0
    for n in range(B):
        out, tp = O.forward_joint(gl[n], gh[n], sl[n], r, eps)
        ln, d = O.mse_loss(out, tg[n])
        want_loss += ln / B
        want = O.backward(tp, d / B)  # d_src, d_guide_lo, d_guide_hi
        got = [npy(t[n]).transpose(1, 2, 0)
               for t in (grads.d_src, grads.d_guide_lo, grads.d_guide_hi)]
        # per tensor against its own largest entry, floored by the step's
        # largest gradient (at r = 0 the exact d_guide_lo is identically 0)
        floor = max(float(np.abs(x).max()) for x in want)
        for a, b in zip(got, want):
            assert abs_max(a, b) <= GRAD_TOL32 * max(float(np.abs(b).max()), floor)
    assert abs(float(loss) - want_loss) <= 1e-6 * max(want_loss, 1e-12)


def test_joint_mse_backward_matches_unfused_chain_config2_size(gfb):
    """At BASELINE config-2 plane size (2048^2 hr, r = 1, eps = 1e-8): the fused
    step against forward_joint -> mse_loss -> backward on the same GPU."""
    import workloads

    lr_x, lr_y, hr_x = (t.cuda() for t in workloads.joint_inputs(2, 3, 2048, 2048, seed=11))
    tg = workloads.affine_target(hr_x).contiguous()
    p = gfb.GuidedFilterParams(1, 1e-8)
    loss, grads, status = gfb.joint_mse_backward(lr_x, hr_x, lr_y, tg, p)
    out, tape = gfb.forward_joint(lr_x, hr_x, lr_y, p)
    from paper_1803_05619_b200.training import mse_loss_device
    want, d_out = mse_loss_device(out, tg)
    ref = gfb.backward(tape, d_out)
    assert status.bits() == 0
    assert abs(float(loss) - float(want)) <= 1e-6 * float(want)
    for a, b in ((grads.d_src, ref.d_src), (grads.d_guide_lo, ref.d_guide_lo),
                 (grads.d_guide_hi, ref.d_guide_hi)):
        assert rel_max(npy(a), npy(b)) <= 1e-4


def test_joint_mse_backward_nonfused_shapes(gfb):
    """Shapes the fused kernel does not cover (ratio 2, float64) take the
    forward -> MSE -> backward entries inside the same C call."""
    rng = np.random.default_rng(3)
    for dt, (h, w, H, W) in ((torch.float32, (9, 11, 18, 22)), (torch.float64, (8, 10, 32, 40))):
        gl = rng.uniform(0, 1, (1, h, w, 3))
        sl = rng.uniform(0, 1, (1, h, w, 3))
        gh = rng.uniform(0, 1, (1, H, W, 3))
        tg = rng.uniform(0, 1, (1, H, W, 3))
        g = lambda a: torch.from_numpy(a.transpose(0, 3, 1, 2).copy()).to(dt).cuda()  # noqa: E731
        loss, grads, _ = gfb.joint_mse_backward(g(gl), g(gh), g(sl), g(tg),
                                                gfb.GuidedFilterParams(1, 1e-4))
        out, tp = O.forward_joint(gl[0], gh[0], sl[0], 1, 1e-4)
        want, d = O.mse_loss(out, tg[0])
        d_src, d_glo, d_ghi = O.backward(tp, d)
        tol = GRAD_TOL32 if dt == torch.float32 else 1e-9
        assert abs(float(loss) - want) <= tol * want
        assert rel_max(npy(grads.d_src[0]).transpose(1, 2, 0), d_src) <= tol
        assert rel_max(npy(grads.d_guide_lo[0]).transpose(1, 2, 0), d_glo) <= tol
        assert rel_max(npy(grads.d_guide_hi[0]).transpose(1, 2, 0), d_ghi) <= tol


# ---------------------------------------------------------------------------
# error semantics (gf/guided.py:156-180)
# ---------------------------------------------------------------------------

def test_error_semantics(gfb):
    rng = np.random.default_rng(5)
    gl, gh, sl = rng.uniform(0, 1, (6, 8, 2)), rng.uniform(0, 1, (12, 16, 2)), \
        rng.uniform(0, 1, (6, 8, 2))
    p = gfb.GuidedFilterParams(1, 1e-2)
    with pytest.raises(ValueError):
        gfb.forward_joint(gl, gh, sl[:, :-1], p)
    with pytest.raises(ValueError):
        gfb.forward_joint(gl, gh[:, :, :1], sl, p)
    with pytest.raises(ValueError):
        gfb.forward_joint(gh, gl, gh, p)
    bad = sl.copy()
    bad[0, 0, 0] = np.nan
    with pytest.raises(ValueError):
        gfb.forward_joint(gl, gh, bad, p)
    bad_hi = gh.copy()
    bad_hi[3, 3, 1] = np.inf
    with pytest.raises(ValueError):
        gfb.forward_joint(gl, bad_hi, sl, p)
    with pytest.raises(gfb.DegenerateWindowError):
        gfb.forward_joint(np.full_like(gl, 0.25), gh, sl, gfb.GuidedFilterParams(1, 0.0))
    for dt in (torch.float32,):
        with pytest.raises(gfb.DegenerateWindowError):
            gfb.forward_joint(torch.full((1, 2, 6, 8), 0.25, dtype=dt, device="cuda"),
                              torch.rand(1, 2, 12, 16, dtype=dt, device="cuda"),
                              torch.rand(1, 2, 6, 8, dtype=dt, device="cuda"),
                              gfb.GuidedFilterParams(1, 0.0))
    out, tape = gfb.forward_joint(gl, gh, sl, p)
    with pytest.raises(ValueError):
        gfb.backward(tape, np.zeros_like(sl))
    g = gfb.backward(tape, np.zeros_like(out))
    assert not g.d_src.any() and not g.d_guide_lo.any() and not g.d_guide_hi.any()
    with pytest.raises(ValueError):
        gfb.forward_highres(rng.uniform(0, 1, (8, 8, 1)), rng.uniform(0, 1, (8, 7, 1)), p)


# ---------------------------------------------------------------------------
# semantic properties (pkg/tests/test_guided.py analogues) in fp64
# ---------------------------------------------------------------------------

def test_semantic_properties_fp64(gfb):
    rng = np.random.default_rng(1)
    gl, gh = rng.uniform(0, 1, (6, 8, 2)), rng.uniform(0, 1, (12, 16, 2))
    out, _ = gfb.forward_joint(gl, gh, np.full_like(gl, 5.0), gfb.GuidedFilterParams(1, 1e-8))
    assert np.abs(out - 5.0).max() <= 1e-10
    out, _ = gfb.forward_joint(gl, gh, 2.0 * gl + 3.0, gfb.GuidedFilterParams(1, 0.0))
    assert np.abs(out - (2.0 * gh + 3.0)).max() <= 1e-8
    g = rng.uniform(0, 1, (16, 14, 2))
    out, _ = gfb.forward_highres(g, 0.7 * g - 0.2, gfb.GuidedFilterParams(1, 0.0))
    assert np.abs(out - (0.7 * g - 0.2)).max() <= 1e-8
    out, _ = gfb.forward_highres(g, np.full_like(g, 0.3), gfb.GuidedFilterParams(2, 1e-2))
    assert np.abs(out - 0.3).max() <= 1e-10
    # linearity of the backward in d_out
    sl = rng.uniform(0, 1, (6, 8, 2))
    _, tape = gfb.forward_joint(gl, gh, sl, gfb.GuidedFilterParams(1, 1e-2))
    u, v = rng.standard_normal((12, 16, 2)), rng.standard_normal((12, 16, 2))
    combo = gfb.backward(tape, 0.37 * u - 1.21 * v)
    gu, gv = gfb.backward(tape, u), gfb.backward(tape, v)
    for f in ("d_src", "d_guide_lo", "d_guide_hi"):
        mixed = 0.37 * getattr(gu, f) - 1.21 * getattr(gv, f)
        assert np.abs(getattr(combo, f) - mixed).max() <= 1e-10
    # tape fields re-derive slope/intercept (pkg/tests/test_guided.py:91-98)
    _, tape = gfb.forward_joint(gl, gh, sl, gfb.GuidedFilterParams(2, 1e-2))
    slope = tape.cov_guide_src / (tape.var_guide + tape.params.eps)
    assert np.abs(slope - tape.slope).max() <= 1e-12
    assert tape.variant == "joint"


# ---------------------------------------------------------------------------
# BASELINE-config inputs (seeded synthetic) vs the oracle
# ---------------------------------------------------------------------------

def test_cfg0_full_size_vs_oracle(gfb):
    import workloads

    lr_x, lr_y, hr_x = workloads.joint_inputs(1, 3, 1024, 1024, 4, seed=0)
    p = gfb.GuidedFilterParams(1, 1e-8)
    out, tape = gfb.forward_joint(lr_x.cuda(), hr_x.cuda(), lr_y.cuda(), p)
    want = O.joint_forward_nchw(lr_x.double().numpy(), lr_y.double().numpy(),
                                hr_x.double().numpy(), 1, 1e-8)
    assert abs_max(npy(out), want) <= OUT_TOL32
    d = torch.randn(out.shape, generator=torch.Generator().manual_seed(3))
    g = gfb.backward(tape, d.cuda())
    dlx, dly, dhx = O.joint_backward_nchw(lr_x.double().numpy(), lr_y.double().numpy(),
                                          hr_x.double().numpy(), d.double().numpy(), 1, 1e-8)
    assert rel_max(npy(g.d_guide_lo), dlx) <= GRAD_TOL32
    assert rel_max(npy(g.d_src), dly) <= GRAD_TOL32
    assert rel_max(npy(g.d_guide_hi), dhx) <= GRAD_TOL32


@pytest.mark.parametrize("r", [1, 2, 4, 8])
def test_cfg3_radius_sweep_vs_oracle(gfb, r):
    import workloads

    lr_x, lr_y, hr_x = workloads.joint_inputs(2, 3, 512, 512, 4, seed=10 + r)
    p = gfb.GuidedFilterParams(r, 1e-4)
    out, _ = gfb.forward_joint(lr_x.cuda(), hr_x.cuda(), lr_y.cuda(), p)
    want = O.joint_forward_nchw(lr_x.double().numpy(), lr_y.double().numpy(),
                                hr_x.double().numpy(), r, 1e-4)
    assert abs_max(npy(out), want) <= OUT_TOL32


def test_cfg1_highres_vs_oracle(gfb):
    import workloads

    guide, src = workloads.highres_inputs(2, 3, 512, 512, seed=1)
    p = gfb.GuidedFilterParams(8, 1e-2)
    out, tape = gfb.forward_highres(guide.cuda(), src.cuda(), p)
    want = O.highres_forward_nchw(guide.double().numpy(), src.double().numpy(), 8, 1e-2)
    assert abs_max(npy(out), want) <= OUT_TOL32
    d = torch.randn(out.shape, generator=torch.Generator().manual_seed(4))
    gr = gfb.backward(tape, d.cuda())
    dg, ds = O.highres_backward_nchw(guide.double().numpy(), src.double().numpy(),
                                     d.double().numpy(), 8, 1e-2)
    assert rel_max(npy(gr.d_src), ds) <= GRAD_TOL32
    assert rel_max(npy(gr.d_guide_hi), dg) <= GRAD_TOL32


def test_cfg1_full_size_forward_vs_oracle(gfb):
    import workloads

    guide, src = workloads.highres_inputs(4, 3, 2048, 2048, seed=0)
    p = gfb.GuidedFilterParams(8, 1e-2)
    out, _ = gfb.forward_highres(guide.cuda(), src.cuda(), p)
    o = npy(out)
    for n in range(4):  # oracle per image keeps memory bounded
        want = O.highres_forward_nchw(guide[n:n + 1].double().numpy(),
                                      src[n:n + 1].double().numpy(), 8, 1e-2)
        assert abs_max(o[n:n + 1], want) <= OUT_TOL32, n


def test_determinism_bitwise(gfb):
    import workloads

    lr_x, lr_y, hr_x = [t.cuda() for t in workloads.joint_inputs(2, 3, 256, 320, 4, seed=5)]
    p = gfb.GuidedFilterParams(2, 1e-4)
    a, ta = gfb.forward_joint(lr_x, hr_x, lr_y, p)
    b, _ = gfb.forward_joint(lr_x, hr_x, lr_y, p)
    assert torch.equal(a, b)
    d = torch.randn(a.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    g1, g2 = gfb.backward(ta, d), gfb.backward(ta, d)
    for f in ("d_src", "d_guide_lo", "d_guide_hi"):
        assert torch.equal(getattr(g1, f), getattr(g2, f))


def test_autograd_module(gfb):
    import workloads

    lr_x, lr_y, hr_x = [t.cuda().requires_grad_() for t in
                        workloads.joint_inputs(1, 3, 128, 128, 4, seed=6)]
    m = gfb.FastGuidedFilter(1, 1e-4)
    out = m(lr_x, lr_y, hr_x)
    d = torch.randn_like(out)
    out.backward(d)
    assert m.last_status.bits() == 0
    want = O.joint_backward_nchw(lr_x.detach().double().cpu().numpy(),
                                 lr_y.detach().double().cpu().numpy(),
                                 hr_x.detach().double().cpu().numpy(),
                                 d.double().cpu().numpy(), 1, 1e-4)
    assert rel_max(npy(lr_x.grad), want[0]) <= GRAD_TOL32
    assert rel_max(npy(lr_y.grad), want[1]) <= GRAD_TOL32
    assert rel_max(npy(hr_x.grad), want[2]) <= GRAD_TOL32


# ---------------------------------------------------------------------------
# fused kernels: ragged shapes / radii vs the oracle, and the dispatch
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("h,w,r", [(37, 45, 0), (37, 45, 1), (16, 32, 2), (33, 17, 5),
                                   (64, 96, 8), (21, 70, 12), (2, 3, 1), (130, 66, 3)])
def test_fused_joint_ragged_vs_oracle(gfb, h, w, r):
    from paper_1803_05619_b200 import _lib

    lib = _lib.load()
    assert lib.gf_joint_is_fused(0, 2, 3, h, w, 4 * h, 4 * w, r) == 1
    rng = np.random.default_rng(h * 1000 + w + r)
    lr_x = rng.uniform(0, 1, (2, 3, h, w)).astype(np.float32)
    lr_y = rng.uniform(0, 1, (2, 3, h, w)).astype(np.float32)
    hr_x = rng.uniform(0, 1, (2, 3, 4 * h, 4 * w)).astype(np.float32)
    d = rng.standard_normal((2, 3, 4 * h, 4 * w)).astype(np.float32)
    eps = 1e-3
    p = gfb.GuidedFilterParams(r, eps)
    out, tape = gfb.forward_joint(t32(lr_x), t32(hr_x), t32(lr_y), p)
    want = O.joint_forward_nchw(lr_x, lr_y, hr_x, r, eps)
    assert abs_max(npy(out), want) <= OUT_TOL32
    g = gfb.backward(tape, t32(d))
    dlx, dly, dhx = O.joint_backward_nchw(lr_x, lr_y, hr_x, d, r, eps)
    # at r=0 the exact d_lr_x is 0 (its terms cancel); judge it on the scale of
    # the low-res gradients
    scale = max(float(np.abs(dlx).max()), float(np.abs(dly).max()))
    assert abs_max(npy(g.d_guide_lo), dlx) <= GRAD_TOL32 * scale
    assert rel_max(npy(g.d_src), dly) <= GRAD_TOL32
    # at r=0, A = cov/(var+eps) = 0 exactly, so d_hr_x = d_out*Up(A) is 0
    scale_hr = max(float(np.abs(dhx).max()), float(np.abs(d).max()))
    assert abs_max(npy(g.d_guide_hi), dhx) <= GRAD_TOL32 * scale_hr


@pytest.mark.parametrize("H,W,r,cg", [(77, 132, 1, 1), (77, 132, 3, 3), (300, 260, 8, 1),
                                      (40, 36, 16, 3), (5, 8, 2, 1), (513, 520, 8, 3)])
def test_fused_highres_ragged_vs_oracle(gfb, H, W, r, cg):
    from paper_1803_05619_b200 import _lib

    lib = _lib.load()
    assert lib.gf_highres_fwd_is_fused(0, 2, cg, 3, H, W, r) == 1
    rng = np.random.default_rng(H * 7 + W + r)
    guide = rng.uniform(0, 1, (2, cg, H, W)).astype(np.float32)
    src = rng.uniform(0, 1, (2, 3, H, W)).astype(np.float32)
    p = gfb.GuidedFilterParams(r, 1e-2)
    out, _ = gfb.forward_highres(t32(guide), t32(src), p)
    want = O.highres_forward_nchw(guide, src, r, 1e-2)
    assert abs_max(npy(out), want) <= OUT_TOL32


def test_fused_highres_nonfinite_input_is_input_error(gfb):
    g = torch.rand(1, 1, 64, 64, device="cuda")
    s = torch.rand(1, 3, 64, 64, device="cuda")
    s[0, 1, 10, 20] = float("nan")
    with pytest.raises(ValueError, match="input"):
        gfb.forward_highres(g, s, gfb.GuidedFilterParams(2, 1e-2))
    g2 = torch.rand(1, 1, 64, 64, device="cuda")
    with pytest.raises(gfb.DegenerateWindowError):
        gfb.forward_highres(torch.full_like(g2, 0.5), s.nan_to_num(0.3),
                            gfb.GuidedFilterParams(2, 0.0))


@pytest.mark.parametrize("h,w,r", [(37, 132, 2), (5, 8, 1), (1, 4, 0), (70, 256, 4),
                                   (33, 120, 3), (200, 244, 2), (9, 500, 1), (64, 128, 4),
                                   (300, 12, 2), (40, 36, 6)])
def test_joint_bwd_lr_variants_vs_oracle(gfb, h, w, r):
    """Both low-res backward tails (tile kernel, register-segment walk) against
    the oracle: strips not dividing w, w < one strip, h = 1, pieces spanning
    strips; r = 6 takes the tile kernel under both settings."""
    from paper_1803_05619_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(h * 31 + w + r)
    lr_x = rng.uniform(0, 1, (2, 3, h, w)).astype(np.float32)
    lr_y = rng.uniform(0, 1, (2, 3, h, w)).astype(np.float32)
    hr_x = rng.uniform(0, 1, (2, 3, 4 * h, 4 * w)).astype(np.float32)
    d = rng.standard_normal((2, 3, 4 * h, 4 * w)).astype(np.float32)
    eps = 1e-3
    p = gfb.GuidedFilterParams(r, eps)
    dlx, dly, _ = O.joint_backward_nchw(lr_x, lr_y, hr_x, d, r, eps)
    scale = max(float(np.abs(dlx).max()), float(np.abs(dly).max()))
    for v in (1, 2):
        old = lib.gf_joint_bwd_lr_variant(v)
        try:
            _, tape = gfb.forward_joint(t32(lr_x), t32(hr_x), t32(lr_y), p)
            g = gfb.backward(tape, t32(d))
        finally:
            lib.gf_joint_bwd_lr_variant(old)
        assert abs_max(npy(g.d_guide_lo), dlx) <= GRAD_TOL32 * scale, v
        assert abs_max(npy(g.d_src), dly) <= GRAD_TOL32 * scale, v


def test_fused_joint_nonfinite_input_is_input_error(gfb):
    lr_x = torch.rand(1, 3, 16, 16, device="cuda")
    lr_y = torch.rand(1, 3, 16, 16, device="cuda")
    hr_x = torch.rand(1, 3, 64, 64, device="cuda")
    hr_x[0, 2, 5, 5] = float("inf")
    with pytest.raises(ValueError, match="input"):
        gfb.forward_joint(lr_x, hr_x, lr_y, gfb.GuidedFilterParams(1, 1e-4))


def test_guidance_backward_reuses_forward_statistics(gfb):
    """gn_backward_reuse (the tape's forward workspace) is bitwise the full
    recomputation; a parameter edit after the forward drops the reuse."""
    from paper_1803_05619_b200 import _lib

    lib = _lib.load()
    assert lib.gn_is_fused(0, 3, 3, 15, 48, 64) == 1
    rng = np.random.default_rng(7)
    net = gfb.GuidanceNet(3, 3, hidden=15, rng=rng)
    net.parameters()["norm.norm_gain"][:] = 0.4
    x = t32(rng.uniform(0, 1, (2, 3, 48, 64)).astype(np.float32))
    dy = t32(rng.standard_normal((2, 3, 48, 64)).astype(np.float32))
    _, tape = net.forward(x)
    assert tape.ws is not None
    dx1, g1 = net.backward(tape, dy)
    tape_fresh = gfb.guidance.GuidanceTape(x=tape.x)
    dx2, g2 = net.backward(tape_fresh, dy)
    assert torch.equal(dx1, dx2)
    for k in g1:
        assert torch.equal(g1[k], g2[k]), k
    # parameters edited after the forward: the stale statistics are not used
    net.parameters()["norm.norm_gain"][:] = 0.9
    dx3, _ = net.backward(tape, dy)
    dx4, _ = net.backward(gfb.guidance.GuidanceTape(x=tape.x), dy)
    assert torch.equal(dx3, dx4)
    assert not torch.equal(dx3, dx1)


@pytest.mark.parametrize("hidden", [4, 8, 15, 16])
def test_fused_guidance_net_vs_oracle(gfb, hidden):
    from paper_1803_05619_b200 import _lib

    rng = np.random.default_rng(hidden)
    params = O.guidance_init(3, 3, hidden, rng)
    params["norm.norm_gain"] = np.array([0.6])
    params["norm.gain"] = np.array([0.9])
    params["conv2.bias"] = rng.uniform(-0.1, 0.1, 3)
    params = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in params.items()}
    B, H, W = 2, 48, 64
    x = rng.uniform(0, 1, (B, 3, H, W)).astype(np.float32)
    dy = rng.standard_normal((B, 3, H, W)).astype(np.float32)
    net = gfb.GuidanceNet(3, 3, hidden=hidden)
    net.load_parameters(params)
    y, tape = net.forward(t32(x))
    dx, grads = net.backward(tape, t32(dy))
    want_y, want_dx = [], []
    want_g = {k: 0.0 for k in params}
    for n in range(B):
        xh = x[n].transpose(1, 2, 0).astype(np.float64)
        yy, tp = O.guidance_forward(params, xh)
        dxx, gg = O.guidance_backward(params, tp, dy[n].transpose(1, 2, 0).astype(np.float64))
        want_y.append(yy.transpose(2, 0, 1))
        want_dx.append(dxx.transpose(2, 0, 1))
        for k in gg:
            want_g[k] = want_g[k] + gg[k]
    assert abs_max(npy(y), np.stack(want_y)) <= 1e-5
    assert rel_max(npy(dx), np.stack(want_dx)) <= GRAD_TOL32
    scale = max(float(np.abs(v).max()) for v in want_g.values())
    for k, v in grads.items():
        assert abs_max(npy(v), want_g[k]) <= GRAD_TOL32 * scale, k
    # the general kernels agree with the fused ones
    lib = _lib.load()
    old = lib.gf_force_generic(1)
    try:
        y2, tape2 = net.forward(t32(x))
        dx2, _ = net.backward(tape2, t32(dy))
    finally:
        lib.gf_force_generic(old)
    assert abs_max(npy(y2), npy(y)) <= 1e-5
    assert rel_max(npy(dx2), npy(dx)) <= GRAD_TOL32


@pytest.mark.parametrize("H,W,r,cg", [(77, 132, 1, 1), (77, 132, 3, 3), (300, 260, 8, 1),
                                      (40, 36, 16, 3), (5, 8, 2, 1), (90, 70, 20, 1),
                                      (513, 520, 8, 3)])
def test_fused_highres_backward_vs_oracle(gfb, H, W, r, cg):
    """fp32 streaming backward (gf_fused_highres_bwd.cu) against the oracle and
    against the general float64-intermediate kernels."""
    from paper_1803_05619_b200 import _lib

    rng = np.random.default_rng(H + 3 * W + r)
    guide = rng.uniform(0, 1, (2, cg, H, W)).astype(np.float32)
    src = rng.uniform(0, 1, (2, 3, H, W)).astype(np.float32)
    d = rng.standard_normal((2, 3, H, W)).astype(np.float32)
    p = gfb.GuidedFilterParams(r, 1e-2)
    out, tape = gfb.forward_highres(t32(guide), t32(src), p)
    g = gfb.backward(tape, t32(d))
    dg_want, ds_want = O.highres_backward_nchw(guide, src, d, r, 1e-2)
    assert rel_max(npy(g.d_src), ds_want) <= GRAD_TOL32
    assert rel_max(npy(g.d_guide_hi), dg_want) <= GRAD_TOL32
    lib = _lib.load()
    old = lib.gf_force_generic(1)
    try:
        out2, tape2 = gfb.forward_highres(t32(guide), t32(src), p)
        g2 = gfb.backward(tape2, t32(d))
    finally:
        lib.gf_force_generic(old)
    assert rel_max(npy(g.d_src), npy(g2.d_src)) <= GRAD_TOL32
    assert rel_max(npy(g.d_guide_hi), npy(g2.d_guide_hi)) <= GRAD_TOL32


@pytest.mark.parametrize("H,W,r,cg", [(77, 132, 1, 1), (77, 132, 3, 3), (300, 260, 8, 1),
                                      (5, 8, 2, 1), (513, 520, 8, 3), (64, 4, 1, 1),
                                      (9, 12, 7, 3), (1, 8, 2, 1), (40, 1000, 5, 1),
                                      (1500, 64, 8, 1), (33, 236, 4, 3), (70, 492, 6, 1),
                                      (50, 300, 4, 1), (20, 700, 8, 3), (33, 1000, 8, 1),
                                      (70, 2048, 8, 3), (37, 964, 4, 1), (300, 484, 8, 1),
                                      (2, 12, 8, 1), (45, 512, 8, 3), (19, 496, 4, 3)])
def test_highres_kernel_variants_vs_oracle(gfb, H, W, r, cg):
    """Every fp32 full-res forward kernel (batch/TMA, register-segment with 4
    and 8 columns per lane, 4 per lane register-capped) against the oracle on ragged shapes: strips not
    dividing W, W = 4, H = 1, pieces spanning two strips."""
    from paper_1803_05619_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(H * 11 + W + r)
    guide = rng.uniform(0, 1, (2, cg, H, W)).astype(np.float32)
    src = rng.uniform(0, 1, (2, 3, H, W)).astype(np.float32)
    p = gfb.GuidedFilterParams(r, 1e-2)
    want = O.highres_forward_nchw(guide, src, r, 1e-2)
    outs = []
    for v in (1, 2, 3, 4):
        old = lib.gf_highres_variant(v)
        try:
            out, _ = gfb.forward_highres(t32(guide), t32(src), p)
        finally:
            lib.gf_highres_variant(old)
        assert abs_max(npy(out), want) <= OUT_TOL32, v
        outs.append(npy(out))


@pytest.mark.parametrize("variant,r", [(1, 2), (2, 2), (3, 2), (2, 4), (2, 8), (3, 8), (4, 8)])
def test_highres_kernel_variants_status(gfb, variant, r):
    from paper_1803_05619_b200 import _lib

    lib = _lib.load()
    old = lib.gf_highres_variant(variant)
    try:
        g = torch.rand(1, 1, 64, 64, device="cuda")
        s = torch.rand(1, 3, 64, 64, device="cuda")
        s[0, 1, 10, 20] = float("nan")
        with pytest.raises(ValueError, match="input"):
            gfb.forward_highres(g, s, gfb.GuidedFilterParams(r, 1e-2))
        with pytest.raises(gfb.DegenerateWindowError):
            gfb.forward_highres(torch.full_like(g, 0.5), s.nan_to_num(0.3),
                                gfb.GuidedFilterParams(r, 0.0))
        # eps = 0 with non-degenerate windows is fine
        gfb.forward_highres(g, s.nan_to_num(0.3), gfb.GuidedFilterParams(r, 0.0))
    finally:
        lib.gf_highres_variant(old)


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
def test_fused_guidance_backward_variants_vs_oracle(gfb, variant):
    """The one-heavy-pass backward (variant 0, dx = D + K + L x, dW1 from the
    x moments, two lanes per pixel group; 2: four lanes per group, the
    round-1 kernel; 3: variant 0 capped at 3 CTAs per SM) and the two-pass
    kernels (1) against the oracle at a
    config-2-like image (smooth [0,1] input, small upstream gradient); every
    parameter gradient against its own largest entry."""
    import workloads
    from paper_1803_05619_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(21)
    params = O.guidance_init(3, 3, 15, rng)
    params["norm.norm_gain"] = np.array([0.5])
    params = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in params.items()}
    _, _, x = workloads.joint_inputs(2, 3, 256, 320, seed=4)
    x = x.numpy()
    dy = (1e-5 * rng.standard_normal(x.shape)).astype(np.float32)
    net = gfb.GuidanceNet(3, 3, hidden=15)
    net.load_parameters(params)
    old = lib.gf_gn_bwd_variant(variant)
    try:
        _, tape = net.forward(t32(x))
        dx, grads = net.backward(tape, t32(dy))
    finally:
        lib.gf_gn_bwd_variant(old)
    want_dx, want_g = [], {k: 0.0 for k in params}
    for n in range(x.shape[0]):
        _, tp = O.guidance_forward(params, x[n].transpose(1, 2, 0).astype(np.float64))
        dxx, gg = O.guidance_backward(params, tp, dy[n].transpose(1, 2, 0).astype(np.float64))
        want_dx.append(dxx.transpose(2, 0, 1))
        for k in gg:
            want_g[k] = want_g[k] + gg[k]
    assert rel_max(npy(dx), np.stack(want_dx)) <= GRAD_TOL32
    scale = max(float(np.abs(v).max()) for v in want_g.values())
    for k, v in grads.items():
        own = float(np.abs(want_g[k]).max())
        assert abs_max(npy(v), want_g[k]) <= GRAD_TOL32 * max(own, 1e-2 * scale), k


@pytest.mark.parametrize("r", [0, 1, 2, 4, 8, 12])
def test_joint_fwd_tma_variant_bitwise(gfb, r):
    """The persistent TMA joint forward (variant hook 10: cp.async.bulk.tensor
    ring, tiles two ahead) is bitwise equal to the tile kernel, ragged shapes
    and image borders included (TMA zero-fills outside the image)."""
    from paper_1803_05619_b200 import _lib

    lib = _lib.load()
    for (B, C, h, w) in [(2, 3, 37, 44), (1, 1, 100, 300), (3, 2, 8, 4)]:
        g = torch.Generator(device="cuda").manual_seed(r + h)
        lx = torch.rand(B, C, h, w, device="cuda", generator=g)
        ly = torch.rand(B, C, h, w, device="cuda", generator=g)
        hx = torch.rand(B, C, 4 * h, 4 * w, device="cuda", generator=g)
        p = gfb.GuidedFilterParams(r, 1e-4)
        ref, _ = gfb.forward_joint(lx, hx, ly, p)
        old = lib.gf_joint_fwd_variant(10)
        try:
            got, _ = gfb.forward_joint(lx, hx, ly, p)
        finally:
            lib.gf_joint_fwd_variant(old)
        assert torch.equal(got, ref), (B, C, h, w)


def test_mean_filter_cost_is_radius_independent(gfb):
    """The reference's performance-shape criterion (SPEC.md:541,
    pkg/tests/test_filters.py:206-220): mean_filter at r = 32 costs at most
    1.5x r = 1 on a 1024^2 image -- on the GPU general path (float64), and
    the large-radius result matches the float64 oracle."""
    import time

    x = torch.rand(1, 3, 1024, 1024, dtype=torch.float64, device="cuda")

    def t(r):
        for _ in range(2):
            gfb.mean_filter(x, r)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            t0 = time.perf_counter()
            gfb.mean_filter(x, r)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    t1, t32 = t(1), t(32)
    assert t32 <= 1.5 * t1 + 2e-4, (t1, t32)
    small = x[:, :, :160, :200].contiguous()
    hwc = npy(small)[0].transpose(1, 2, 0)
    for r in (0, 3, 32, 300):
        got = npy(gfb.mean_filter(small, r))[0].transpose(1, 2, 0)
        assert np.abs(got - O.mean_filter(hwc, r)).max() <= 1e-12, r
        got = npy(gfb.mean_filter_adjoint(small, r))[0].transpose(1, 2, 0)
        assert np.abs(got - O.mean_filter_adjoint(hwc, r)).max() <= 1e-12, r


def test_tma_staged_tile_kernels_bitwise(gfb):
    """Variant hook 11: the joint forward, backward hr pass and fused step
    with TMA-staged low-res halo blocks equal the defaults bit for bit."""
    from paper_1803_05619_b200 import _lib

    lib = _lib.load()
    for (B, C, h, w, r) in [(2, 3, 37, 44, 2), (1, 1, 100, 300, 8), (3, 2, 8, 4, 0), (1, 3, 20, 36, 12)]:
        g = torch.Generator(device="cuda").manual_seed(r + h)
        lx, ly = (torch.rand(B, C, h, w, device="cuda", generator=g) for _ in range(2))
        hx, tg = (torch.rand(B, C, 4 * h, 4 * w, device="cuda", generator=g) for _ in range(2))
        d = torch.randn(B, C, 4 * h, 4 * w, device="cuda", generator=g)
        p = gfb.GuidedFilterParams(r, 1e-4)

        def run():
            o, t = gfb.forward_joint(lx, hx, ly, p)
            gr = gfb.backward(t, d)
            loss, g2, _ = gfb.joint_mse_backward(lx, hx, ly, tg, p)
            # the plain forward entry (forward_joint takes the slope-tape one)
            o2 = torch.empty_like(hx)
            st = torch.zeros(1, dtype=torch.int32, device="cuda")
            assert lib.gf_joint_fwd(0, lx.data_ptr(), ly.data_ptr(), hx.data_ptr(), o2.data_ptr(),
                                    B, C, h, w, 4 * h, 4 * w, r, 1e-4, 0, 0, st.data_ptr(),
                                    torch.cuda.current_stream().cuda_stream) == 0
            return [o, gr.d_guide_lo, gr.d_src, gr.d_guide_hi, g2.d_guide_lo, g2.d_src,
                    g2.d_guide_hi, loss, o2]

        ref = run()
        old = (lib.gf_joint_fwd_variant(11), lib.gf_joint_bwd_hr_variant(11),
               lib.gf_joint_mse_variant(11))
        try:
            got = run()
        finally:
            lib.gf_joint_fwd_variant(old[0])
            lib.gf_joint_bwd_hr_variant(old[1])
            lib.gf_joint_mse_variant(old[2])
        # the default backward runs on the forward's slope tape; variant 11
        # recomputes the moments: d_hr (index 3) agrees to fp32 rounding
        for i, (a, b) in enumerate(zip(got, ref)):
            if i == 3:
                tol = 1e-5 * float(b.abs().max()) + 1e-4 * float(d.abs().max())
                assert float((a - b).abs().max()) <= tol, (B, C, h, w, r)
            else:
                assert torch.equal(a, b), (i, B, C, h, w, r)


@pytest.mark.parametrize("B,C,h,w,r", [(2, 3, 37, 44, 1), (1, 3, 64, 128, 2), (1, 2, 20, 36, 8),
                                       (2, 1, 5, 8, 0)])
def test_fused_step_coefficient_tape_matches_recompute(gfb, B, C, h, w, r):
    """The fused training step on a coefficient tape (variant 15:
    k_joint_coeffs writes A and b of every low-res cell, the hr pass reads them
    and gets its gather window of hr_x and the target by TMA) against the
    default moments-recomputing kernel: the loss and the gradients agree to
    fp32 rounding."""
    from paper_1803_05619_b200 import _lib

    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(B * 7 + h + r)
    lx, ly = (torch.rand(B, C, h, w, device="cuda", generator=g) for _ in range(2))
    hx, tg = (torch.rand(B, C, 4 * h, 4 * w, device="cuda", generator=g) for _ in range(2))
    p = gfb.GuidedFilterParams(r, 1e-3)
    l1, g1, _ = gfb.joint_mse_backward(lx, hx, ly, tg, p)
    old = lib.gf_joint_mse_variant(15)
    try:
        l0, g0, _ = gfb.joint_mse_backward(lx, hx, ly, tg, p)
    finally:
        lib.gf_joint_mse_variant(old)
    assert abs(float(l0) - float(l1)) <= 1e-6 * float(l1)
    for a, b in ((g0.d_src, g1.d_src), (g0.d_guide_lo, g1.d_guide_lo),
                 (g0.d_guide_hi, g1.d_guide_hi)):
        # r = 0: the exact slope is 0, so d_guide_hi = d_out * Up(A) is the
        # rounding noise of cov / (var + eps) (~1e-7) in both kernels
        assert abs_max(npy(a), npy(b)) <= 1e-4 * float(b.abs().max()) + 1e-6
