"""GPU parity at BASELINE config 4's FULL sizes (SURVEY 8c "crop parity", 8e).

The float64 oracle cannot run a 16384^2 image (or a batch of 64 3072^2
images) in test time, so the full-size GPU results are checked on aligned
crops: for owned low-res cells [a, b) x [c, d) the oracle runs on the crop
[a-R, b+R) x [c-R, d+R) (clamped to the image; high-res crop exactly 4x that
range) with R = max(2r, r+1), and the owned part of every output and
gradient must match the full-image GPU result (sharding.py's halo argument,
applied to both axes).  The sharded path (sharding.row_bands) is run band by
band on one GPU and compared with the 1-GPU result on every owned row.

Bars as in test_gpu_parity: outputs max abs <= 1e-4, gradients
max|g - g_ref| / max|g_ref| <= 1e-3 per tensor.
"""

import numpy as np
import pytest
import torch

from oracle import gf_oracle as O
from paper_1803_05619_b200.sharding import (halo, joint_band_backward, joint_band_forward,
                                             row_bands)

pytestmark = pytest.mark.gpu

OUT_TOL32 = 1e-4
GRAD_TOL32 = 1e-3
F = 4  # upsampling factor of every BASELINE config


@pytest.fixture(scope="module")
def gfb():
    import paper_1803_05619_b200 as m

    assert torch.cuda.is_available(), "gpu tests need CUDA"
    return m


def rel_max(a, b):
    return float(np.abs(a - b).max()) / max(float(np.abs(b).max()), 1e-30)


def npy(t):
    return t.detach().double().cpu().numpy()


def _crop_check(lr_x, lr_y, hr_x, d_out, out, grads, n, a, b, c, d, r, eps):
    """Oracle on the aligned crop around owned lr cells [a,b) x [c,d) of image n."""
    h, w = lr_x.shape[2], lr_x.shape[3]
    R = halo(r, True)
    y0, y1 = max(a - R, 0), min(b + R, h)
    x0, x1 = max(c - R, 0), min(d + R, w)
    lr = lambda t: npy(t[n:n + 1, :, y0:y1, x0:x1])
    hr = lambda t: npy(t[n:n + 1, :, F * y0:F * y1, F * x0:F * x1])
    lx, ly, hx, dd = lr(lr_x), lr(lr_y), hr(hr_x), hr(d_out)
    want_out = O.joint_forward_nchw(lx, ly, hx, r, eps)
    want = O.joint_backward_nchw(lx, ly, hx, dd, r, eps)
    # owned windows: local (in the crop) and global
    la, lb, lc, ld = a - y0, b - y0, c - x0, d - x0
    got_out = npy(out[n:n + 1, :, F * a:F * b, F * c:F * d])
    err = float(np.abs(got_out - want_out[:, :, F * la:F * lb, F * lc:F * ld]).max())
    assert err <= OUT_TOL32, ("out", n, a, c, err)
    for k, (g, lo_res) in enumerate(((grads.d_guide_lo, True), (grads.d_src, True),
                                     (grads.d_guide_hi, False))):
        s = 1 if lo_res else F
        got = npy(g[n:n + 1, :, s * a:s * b, s * c:s * d])
        ref = want[k][:, :, s * la:s * lb, s * lc:s * ld]
        e = rel_max(got, ref)
        assert e <= GRAD_TOL32, (("d_lr_x", "d_lr_y", "d_hr_x")[k], n, a, c, e)


def _windows(h, w, size, rng, extra=2):
    """Owned lr windows: the four corners, the centre and random interior ones."""
    wins = [(0, 0), (0, w - size), (h - size, 0), (h - size, w - size),
            ((h - size) // 2, (w - size) // 2)]
    for _ in range(extra):
        wins.append((int(rng.integers(0, h - size)), int(rng.integers(0, w - size))))
    return [(a, a + size, c, c + size) for a, c in wins]


def test_cfg4b_full_size_crop_parity(gfb):
    """Config 4b at full size: one 3x16384^2 image, lr 3x4096^2, r=2, eps=1e-4."""
    import workloads

    r, eps = 2, 1e-4
    lr_x, lr_y, hr_x = workloads.joint_inputs(1, 3, 16384, 16384, F, seed=41, device="cuda")
    p = gfb.GuidedFilterParams(r, eps)
    out, tape = gfb.forward_joint(lr_x, hr_x, lr_y, p)
    d_out = torch.randn(out.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    d_out.mul_(1e-3)
    grads = gfb.backward(tape, d_out)
    torch.cuda.synchronize()
    rng = np.random.default_rng(4)
    for (a, b, c, d) in _windows(4096, 4096, 12, rng):
        _crop_check(lr_x, lr_y, hr_x, d_out, out, grads, 0, a, b, c, d, r, eps)


def test_cfg4a_full_size_crop_parity(gfb):
    """Config 4a at full size: batch 64 of 3x3072^2 (lr 3x768^2), r=2, eps=1e-4."""
    import workloads

    r, eps = 2, 1e-4
    lr_x, lr_y, hr_x = workloads.joint_inputs(64, 3, 3072, 3072, F, seed=43, device="cuda")
    p = gfb.GuidedFilterParams(r, eps)
    out, tape = gfb.forward_joint(lr_x, hr_x, lr_y, p)
    d_out = torch.randn(out.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    d_out.mul_(1e-3)
    grads = gfb.backward(tape, d_out)
    torch.cuda.synchronize()
    rng = np.random.default_rng(6)
    for n in (0, 17, 63):
        for (a, b, c, d) in _windows(768, 768, 10, rng, extra=1):
            _crop_check(lr_x, lr_y, hr_x, d_out, out, grads, n, a, b, c, d, r, eps)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_cfg4b_row_bands_match_one_gpu(gfb, world):
    """The row-band decomposition of config 4b (sharding.row_bands, the N-GPU
    path of bench.py), run band by band, against the 1-GPU full-image result:
    forward with the r+1 halo, backward with the max(2r, r+1) halo.  BITWISE
    (SURVEY 8e): crops start on the kernels' 16-row tiles and pass their
    full-image row (row_origin), so tiles, row pieces and shift constants --
    hence every rounding -- are the full image's.  world 3 gives ragged bands."""
    import workloads

    r, eps = 2, 1e-4
    lr_x, lr_y, hr_x = workloads.joint_inputs(1, 3, 16384, 16384, F, seed=47, device="cuda")
    p = gfb.GuidedFilterParams(r, eps)
    out, tape = gfb.forward_joint(lr_x, hr_x, lr_y, p)
    d_out = torch.randn(out.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(7))
    d_out.mul_(1e-3)
    full = gfb.backward(tape, d_out)
    del tape
    for band in row_bands(4096, world, r, F, backward=False):
        o = joint_band_forward(gfb.forward_joint, p, lr_x, lr_y, hr_x, band)
        A, B = band.hr_owned
        assert torch.equal(o, out[:, :, A:B]), ("fwd band", band.a, float((o - out[:, :, A:B]).abs().max()))
    for band in row_bands(4096, world, r, F, backward=True):
        o, dlx, dly, dhx = joint_band_backward(gfb.forward_joint, gfb.backward, p, lr_x, lr_y,
                                               hr_x, d_out, band)
        A, B = band.hr_owned
        for name, got, ref in (("out", o, out[:, :, A:B]),
                               ("d_lr_x", dlx, full.d_guide_lo[:, :, band.a:band.b]),
                               ("d_lr_y", dly, full.d_src[:, :, band.a:band.b]),
                               ("d_hr_x", dhx, full.d_guide_hi[:, :, A:B])):
            assert torch.equal(got, ref), (name, band.a, float((got - ref).abs().max()))


@pytest.mark.parametrize("r", [1, 2, 4, 8])
def test_cfg3_full_size_crop_parity(gfb, r):
    """Config 3 at its largest stated size: batch 16 of 3 x 4096^2 (lr 1024^2),
    eps = 1e-4, forward, checked against the oracle on aligned crops (halo
    r + 1) at the corners, the centre and random windows of three images."""
    import workloads

    eps = 1e-4
    lr_x, lr_y, hr_x = workloads.joint_inputs(16, 3, 4096, 4096, F, seed=60 + r, device="cuda")
    out, _ = gfb.forward_joint(lr_x, hr_x, lr_y, gfb.GuidedFilterParams(r, eps))
    torch.cuda.synchronize()
    rng = np.random.default_rng(r)
    R = halo(r, False)
    h = w = 1024
    for n in (0, 7, 15):
        for (a, b, c, d) in _windows(h, w, 12, rng, extra=2):
            y0, y1, x0, x1 = max(a - R, 0), min(b + R, h), max(c - R, 0), min(d + R, w)
            lr = lambda t: npy(t[n:n + 1, :, y0:y1, x0:x1])  # noqa: E731
            hx = npy(hr_x[n:n + 1, :, F * y0:F * y1, F * x0:F * x1])
            want = O.joint_forward_nchw(lr(lr_x), lr(lr_y), hx, r, eps)
            got = npy(out[n:n + 1, :, F * a:F * b, F * c:F * d])
            ref = want[:, :, F * (a - y0):F * (b - y0), F * (c - x0):F * (d - x0)]
            err = float(np.abs(got - ref).max())
            assert err <= OUT_TOL32, (n, a, c, err)


@pytest.mark.parametrize("norm_gain", [0.0, 0.7])
def test_cfg2_full_size_step_vs_oracle(gfb, norm_gain):
    """Config 2's training step at full image size (hr 2048^2, lr 512^2, r=1,
    eps=1e-8, GuidanceNet 3 -> 15 -> 3) with B = 2 so the batch-mean loss is
    exercised, against the float64 oracle (gf/training.py:143-183): the loss,
    d_lr_x, d_lr_y, d_hr_x and all 95 guidance-net gradients.  norm_gain != 0
    turns on AdaptiveNorm's per-image statistics over 4.2 M pixels
    (gf/guidance.py:152-173) -- where fp32 accumulation could drift."""
    import workloads

    r, eps, B = 1, 1e-8, 2
    lr_x, lr_y, hr_x = (t.cuda() for t in workloads.joint_inputs(B, 3, 2048, 2048, F, seed=21))
    target = workloads.affine_target(hr_x).contiguous()
    net = gfb.GuidanceNet(3, 3, hidden=15, kernel=1, rng=np.random.default_rng(5))
    net.norm.norm_gain[:] = norm_gain
    res = gfb.train_step(net, lr_x, hr_x, lr_y, target, gfb.GuidedFilterParams(r, eps))
    torch.cuda.synchronize()
    params = {k: v.cpu().numpy().copy() for k, v in net.parameters().items()}
    hwc = lambda t: [x.transpose(1, 2, 0) for x in npy(t)]  # noqa: E731
    loss, _, dlx, dly, dhx, grads = O.train_step(params, hwc(lr_x), hwc(hr_x), hwc(lr_y),
                                                 hwc(target), r, eps)
    assert abs(float(res.loss) - loss) <= 1e-5 * loss, (float(res.loss), loss)

    # The leaky ReLU's derivative jumps at h2 = 0 (gf/guidance.py:36-43): at a
    # pixel whose pre-activation is within fp32 rounding of 0 (|h2| ~ 1e-7 was
    # measured for the worst pixel), fp32 and float64 can take different sides
    # and d2 there differs by 0.8 d3 -- a discontinuity of the gradient, not an
    # accuracy loss.  Those pixels (|h2| < 1e-4 for some hidden unit: 0.2 % of
    # the low-res image, < 0.1 % of the high-res one) are excluded from the per-pixel input-gradient bars; the
    # parameter gradients below sum over every pixel.
    def ambiguous(xs):
        out = []
        for x in xs:
            _, tape = O.guidance_forward(params, x)
            h2 = params["norm.gain"][0] * tape["h1"] + params["norm.norm_gain"][0] * tape["xhat"]
            out.append((np.abs(h2) < 1e-4).any(axis=2))
        return np.stack(out)[:, None]  # (B, 1, h, w)

    amb = {"d_lr_x": ambiguous(hwc(lr_x)), "d_hr_x": ambiguous(hwc(hr_x)),
           "d_lr_y": np.zeros((B, 1) + tuple(lr_y.shape[2:]), dtype=bool)}
    for name, got, want in (("d_lr_x", res.d_lr_x, dlx), ("d_lr_y", res.d_lr_y, dly),
                            ("d_hr_x", res.d_hr_x, dhx)):
        want = np.stack([x.transpose(2, 0, 1) for x in want])
        keep = ~np.broadcast_to(amb[name], want.shape)
        assert amb[name].mean() < 1e-2, (name, amb[name].mean())
        err = float(np.abs(npy(got) - want)[keep].max()) / float(np.abs(want).max())
        assert err <= GRAD_TOL32, (name, err)
    got = net.unpack(res.dparams)
    scale = max(float(np.abs(v).max()) for v in grads.values())
    n = 0
    for k, v in grads.items():
        n += v.size
        assert float(np.abs(npy(got[k]) - v).max()) <= GRAD_TOL32 * scale, k
    assert n == 95
