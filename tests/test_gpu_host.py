"""Host-image entry points (gf_*_fwd_host): the pipelined copy-in / kernel /
copy-out over host buffers gives exactly the device entry's bytes, for
batches longer than the two device slots, pinned and pageable buffers, both
dtypes and the reference's HWC numpy call shape."""

import numpy as np
import pytest
import torch

from oracle import gf_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gfb():
    import paper_1803_05619_b200 as m

    assert torch.cuda.is_available(), "gpu tests need CUDA"
    return m


@pytest.mark.parametrize("B,Cg,pinned", [(5, 1, True), (3, 3, False), (1, 1, True)])
def test_highres_host_matches_device(gfb, B, Cg, pinned):
    g = torch.Generator().manual_seed(B * 10 + Cg)
    guide = torch.rand(B, Cg, 96, 132, generator=g)
    src = torch.rand(B, 3, 96, 132, generator=g)
    if pinned:
        guide, src = guide.pin_memory(), src.pin_memory()
    p = gfb.GuidedFilterParams(5, 1e-2)
    host = gfb.forward_highres_host(guide, src, p)
    dev, _ = gfb.forward_highres(guide.cuda(), src.cuda(), p)
    assert torch.equal(host, dev.cpu())


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_joint_host_matches_device(gfb, dtype):
    g = torch.Generator().manual_seed(3)
    lx = torch.rand(4, 3, 20, 28, generator=g, dtype=dtype).pin_memory()
    ly = torch.rand(4, 3, 20, 28, generator=g, dtype=dtype).pin_memory()
    hx = torch.rand(4, 3, 80, 112, generator=g, dtype=dtype).pin_memory()
    p = gfb.GuidedFilterParams(2, 1e-3)
    out = torch.empty(4, 3, 80, 112, dtype=dtype).pin_memory()
    res = gfb.forward_joint_host(lx, hx, ly, p, out=out)
    assert res.data_ptr() == out.data_ptr()
    dev, _ = gfb.forward_joint(lx.cuda(), hx.cuda(), ly.cuda(), p)
    assert torch.equal(out, dev.cpu())


def test_reference_call_shape_numpy_hwc(gfb):
    rng = np.random.default_rng(0)
    gl, sl = rng.uniform(0, 1, (12, 10, 3)), rng.uniform(0, 1, (12, 10, 3))
    gh = rng.uniform(0, 1, (48, 40, 3))
    p = gfb.GuidedFilterParams(2, 1e-3)
    out = gfb.forward_joint_host(gl, gh, sl, p)
    assert isinstance(out, np.ndarray) and out.shape == (48, 40, 3)
    want, _ = O.forward_joint(gl, gh, sl, 2, 1e-3)
    assert float(np.abs(out - want).max()) <= 1e-10
    full = gfb.forward_highres_host(gh, gh[..., ::-1].copy(), p)
    want_h, _ = O.forward_highres(gh, gh[..., ::-1].copy(), 2, 1e-3)
    assert float(np.abs(full - want_h).max()) <= 1e-10


def test_host_error_semantics(gfb):
    g = torch.rand(2, 1, 32, 32)
    s = torch.rand(2, 3, 32, 32)
    s[1, 2, 5, 5] = float("nan")
    with pytest.raises(ValueError, match="input"):
        gfb.forward_highres_host(g, s, gfb.GuidedFilterParams(2, 1e-2))
    with pytest.raises(gfb.DegenerateWindowError):
        gfb.forward_highres_host(torch.full_like(g, 0.5), s.nan_to_num(0.3),
                                 gfb.GuidedFilterParams(2, 0.0))
    with pytest.raises(ValueError):
        gfb.forward_highres_host(g.cuda(), s, gfb.GuidedFilterParams(2, 1e-2))
    with pytest.raises(ValueError):
        gfb.forward_highres_host(torch.rand(2, 2, 32, 32), s, gfb.GuidedFilterParams(2, 1e-2))


@pytest.mark.parametrize("dtype,B,pinned", [(torch.float32, 5, True), (torch.float64, 2, False)])
def test_joint_fwd_bwd_host_matches_device(gfb, dtype, B, pinned):
    """gf_joint_fwd_bwd_host: every output equals the device entries' bytes."""
    g = torch.Generator().manual_seed(B)
    lx = torch.rand(B, 3, 24, 36, generator=g, dtype=dtype)
    ly = torch.rand(B, 3, 24, 36, generator=g, dtype=dtype)
    hx = torch.rand(B, 3, 96, 144, generator=g, dtype=dtype)
    d = torch.randn(B, 3, 96, 144, generator=g, dtype=dtype)
    if pinned:
        lx, ly, hx, d = (t.pin_memory() for t in (lx, ly, hx, d))
    p = gfb.GuidedFilterParams(2, 1e-4)
    out, gr = gfb.forward_backward_joint_host(lx, hx, ly, d, p)
    o_dev, tape = gfb.forward_joint(lx.cuda(), hx.cuda(), ly.cuda(), p)
    g_dev = gfb.backward(tape, d.cuda())
    assert torch.equal(out, o_dev.cpu())
    assert torch.equal(gr.d_guide_lo, g_dev.d_guide_lo.cpu())
    assert torch.equal(gr.d_src, g_dev.d_src.cpu())
    assert torch.equal(gr.d_guide_hi, g_dev.d_guide_hi.cpu())


def test_joint_fwd_bwd_host_reference_hwc(gfb):
    """The reference's HWC float64 numpy call shape, against the oracle."""
    rng = np.random.default_rng(4)
    lx, ly = rng.uniform(0, 1, (2, 10, 14, 3))
    hx = rng.uniform(0, 1, (40, 56, 3))
    d = rng.standard_normal((40, 56, 3))
    p = gfb.GuidedFilterParams(1, 1e-3)
    out, gr = gfb.forward_backward_joint_host(lx, hx, ly, d, p)
    want, tape = O.forward_joint(lx, hx, ly, 1, 1e-3)
    g = O.backward(tape, d)
    assert isinstance(out, np.ndarray) and out.shape == hx.shape
    assert np.abs(out - want).max() <= 1e-10
    assert np.abs(gr.d_guide_lo - g[1]).max() <= 1e-9 * max(1.0, np.abs(g[1]).max())
