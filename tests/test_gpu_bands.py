"""Row-band sharding is BITWISE equal to the 1-GPU image.

config 4b's full-size check lives in test_gpu_fullsize.py; these cases
cover the other radii of the register-segment backward tail (r <= 4), ragged
band counts and heights that are not multiples of the 16-row tile, and every
output of forward + backward.  Each band runs on its aligned crop with its
full-image row passed as ``row_origin`` (sharding.joint_band_backward).
"""

import pytest
import torch

from paper_1803_05619_b200.sharding import (ALIGN, joint_band_backward, joint_band_forward,
                                             row_bands)

pytestmark = pytest.mark.gpu

F = 4


@pytest.fixture(scope="module")
def gfb():
    import paper_1803_05619_b200 as m

    assert torch.cuda.is_available(), "gpu tests need CUDA"
    return m


@pytest.mark.parametrize("r", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("world,h", [(2, 256), (3, 300), (5, 517), (8, 1000)])
def test_row_bands_bitwise(gfb, r, world, h):
    import workloads

    w = 192
    eps = 1e-4
    lr_x, lr_y, hr_x = workloads.joint_inputs(2, 3, F * h, F * w, F, seed=100 + r, device="cuda")
    p = gfb.GuidedFilterParams(r, eps)
    out, tape = gfb.forward_joint(lr_x, hr_x, lr_y, p)
    d_out = torch.randn(out.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(r))
    full = gfb.backward(tape, d_out)
    bands = row_bands(h, world, r, F, backward=True)
    assert bands[0].a == 0 and bands[-1].b == h
    for band in bands:
        assert band.crop_lo % ALIGN == 0
        o, dlx, dly, dhx = joint_band_backward(gfb.forward_joint, gfb.backward, p, lr_x, lr_y,
                                               hr_x, d_out, band)
        A, B = band.hr_owned
        for name, got, ref in (("out", o, out[:, :, A:B]),
                               ("d_lr_x", dlx, full.d_guide_lo[:, :, band.a:band.b]),
                               ("d_lr_y", dly, full.d_src[:, :, band.a:band.b]),
                               ("d_hr_x", dhx, full.d_guide_hi[:, :, A:B])):
            assert torch.equal(got, ref), (name, band.a, float((got - ref).abs().max()))
    for band in row_bands(h, world, r, F, backward=False):
        o = joint_band_forward(gfb.forward_joint, p, lr_x, lr_y, hr_x, band)
        A, B = band.hr_owned
        assert torch.equal(o, out[:, :, A:B]), ("fwd", band.a)


def test_unaligned_origin_still_within_tolerance(gfb):
    """A crop NOT on a tile row (row_origin odd) is not bitwise but stays
    within the oracle bars of the owned rows (the anchoring is a rounding
    choice, never a correctness one)."""
    import workloads

    r, eps, h, w = 2, 1e-4, 200, 128
    lr_x, lr_y, hr_x = workloads.joint_inputs(1, 3, F * h, F * w, F, seed=5, device="cuda")
    p = gfb.GuidedFilterParams(r, eps)
    out, tape = gfb.forward_joint(lr_x, hr_x, lr_y, p)
    d_out = torch.randn(out.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(2))
    full = gfb.backward(tape, d_out)
    a, b, R = 101, 161, 4
    lo, hi = a - R, b + R
    o, t = gfb.forward_joint(lr_x[:, :, lo:hi].contiguous(), hr_x[:, :, F * lo:F * hi].contiguous(),
                             lr_y[:, :, lo:hi].contiguous(), p, row_origin=lo)
    g = gfb.backward(t, d_out[:, :, F * lo:F * hi].contiguous())
    ref = full.d_guide_lo[:, :, a:b]
    got = g.d_guide_lo[:, :, a - lo:b - lo]
    assert float((got - ref).abs().max()) / float(ref.abs().max()) < 1e-4
    assert float((o[:, :, F * (a - lo):F * (b - lo)] - out[:, :, F * a:F * b]).abs().max()) < 1e-5
