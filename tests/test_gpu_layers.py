"""Standalone guidance layers on the GPU: ConvLayer and AdaptiveNorm
(gf/guidance.py:52-173) against the REAL reference's golden vectors
(tests/golden/golden_layers.npz), and GuidanceNet's conv1 / norm / conv2
views over its packed parameters (gf/guidance.py:191-194) -- the reference
caller's ``net.norm.norm_gain[:] = g`` edits the net."""

import os

import numpy as np
import pytest
import torch

from oracle import gf_oracle as O

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_layers.npz"))
CASES = sorted({k.split("/")[0] for k in GOLD.files})


@pytest.fixture(scope="module")
def gfb():
    import paper_1803_05619_b200 as m

    assert torch.cuda.is_available(), "gpu tests need CUDA"
    return m


def g(c, f):
    return GOLD[f"{c}/{f}"]


@pytest.mark.parametrize("case", [c for c in CASES if c.startswith("conv")])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_conv_layer_matches_reference(gfb, case, dtype):
    ci, co, k, d, bias = (int(v) for v in g(case, "meta"))
    layer = gfb.ConvLayer(ci, co, kernel=k, dilation=d, bias=bool(bias))
    params = {"weight": g(case, "weight")}
    if bias:
        params["bias"] = g(case, "bias")
    layer.load_parameters(params)
    x, dy = g(case, "x"), g(case, "dy")
    if dtype == "f64":  # the reference call shape: HWC float64 numpy
        y, tape = layer.forward(x)
        dx, grads = layer.backward(tape, dy)
        tol = 1e-12
    else:  # NCHW fp32 CUDA tensors
        xt = torch.from_numpy(x).permute(2, 0, 1)[None].float().cuda()
        dyt = torch.from_numpy(dy).permute(2, 0, 1)[None].float().cuda()
        yt, tape = layer.forward(xt)
        dxt, gt = layer.backward(tape, dyt)
        y = yt[0].permute(1, 2, 0).double().cpu().numpy()
        dx = dxt[0].permute(1, 2, 0).double().cpu().numpy()
        grads = {kk: v.double().cpu().numpy() for kk, v in gt.items()}
        tol = 1e-5
    scale = lambda a: max(1.0, float(np.abs(a).max()))  # noqa: E731
    assert np.abs(y - g(case, "y")).max() <= tol * scale(g(case, "y"))
    assert np.abs(dx - g(case, "dx")).max() <= tol * scale(g(case, "dx"))
    assert np.abs(grads["weight"] - g(case, "d_weight")).max() <= tol * scale(g(case, "d_weight"))
    if bias:
        assert np.abs(grads["bias"] - g(case, "d_bias")).max() <= tol * scale(g(case, "d_bias"))


@pytest.mark.parametrize("case", [c for c in CASES if c.startswith("norm")])
def test_adaptive_norm_matches_reference(gfb, case):
    gain, ng = g(case, "gains")
    layer = gfb.AdaptiveNorm(gain=gain, norm_gain=ng)
    y, tape = layer.forward(g(case, "x"))
    dx, grads = layer.backward(tape, g(case, "dy"))
    assert np.abs(y - g(case, "y")).max() <= 1e-12
    assert np.abs(dx - g(case, "dx")).max() <= 1e-10 * max(1.0, np.abs(g(case, "dx")).max())
    for k in ("gain", "norm_gain"):
        ref = g(case, f"d_{k}")
        assert np.abs(grads[k] - ref).max() <= 1e-10 * max(1.0, np.abs(ref).max())


def test_batched_layers_sum_parameter_grads(gfb):
    """A batch of B images = B reference calls: per-image outputs, summed
    parameter gradients."""
    rng = np.random.default_rng(9)
    layer = gfb.ConvLayer(3, 4, kernel=3, dilation=2, bias=True, rng=rng)
    norm = gfb.AdaptiveNorm(gain=0.8, norm_gain=1.2)
    x = torch.rand(3, 3, 17, 19, dtype=torch.float64, device="cuda")
    dy = torch.randn(3, 4, 17, 19, dtype=torch.float64, device="cuda")
    y, t = layer.forward(x)
    dx, gr = layer.backward(t, dy)
    z, tn = norm.forward(y)
    dz, gn = norm.backward(tn, dy)
    dw = np.zeros((4, 3, 3, 3))
    for b in range(3):
        xb = x[b].permute(1, 2, 0).cpu().numpy()
        yb, tb = layer.forward(xb)
        assert np.abs(yb - y[b].permute(1, 2, 0).cpu().numpy()).max() <= 1e-12
        _, gb = layer.backward(tb, dy[b].permute(1, 2, 0).cpu().numpy())
        dw += gb["weight"]
        zb, tnb = O.adaptive_norm_forward(yb, 0.8, 1.2)
        assert np.abs(zb - z[b].permute(1, 2, 0).cpu().numpy()).max() <= 1e-12
    assert np.abs(gr["weight"].cpu().numpy() - dw).max() <= 1e-10


def test_guidance_net_layer_views(gfb):
    """net.conv1 / net.norm / net.conv2 are views of the packed parameters:
    chaining them reproduces net.forward, and editing them edits the net."""
    rng = np.random.default_rng(3)
    net = gfb.GuidanceNet(3, 3, hidden=15, kernel=1, rng=rng)
    x = np.random.default_rng(4).uniform(0, 1, (12, 10, 3))
    net.norm.norm_gain[:] = 0.6  # the reference caller's in-place edit
    net.conv2.bias[:] = torch.tensor([0.1, -0.2, 0.3], dtype=torch.float64)
    y, _ = net.forward(x)
    params = {k: v.cpu().numpy().copy() for k, v in net.parameters().items()}
    assert params["norm.norm_gain"][0] == 0.6 and params["conv2.bias"][1] == -0.2
    want, _ = O.guidance_forward(params, x)
    assert np.abs(y - want).max() <= 1e-12
    h1, _ = net.conv1.forward(x)
    h2, _ = net.norm.forward(h1)
    h3 = np.where(h2 >= 0, h2, 0.2 * h2)
    y2, _ = net.conv2.forward(h3)
    assert np.abs(y2 - y).max() <= 1e-12
    # load_parameters on a view writes through to the net
    net.conv1.load_parameters({"weight": np.zeros((15, 3, 1, 1))})
    assert float(net.parameters()["conv1.weight"].abs().max()) == 0.0
    assert net.conv1.weight.data_ptr() == net.parameters()["conv1.weight"].data_ptr()


def test_layers_reject_bad_input(gfb):
    layer = gfb.ConvLayer(3, 2, kernel=3)
    x = np.zeros((5, 5, 3))
    x[2, 2, 1] = np.nan
    with pytest.raises(ValueError):
        layer.forward(x)
    with pytest.raises(ValueError):
        gfb.ConvLayer(3, 2, kernel=2)
    with pytest.raises(ValueError):
        layer.forward(np.zeros((5, 5, 4)))


@pytest.mark.parametrize("task", ["affine", "smooth", "gamma"])
def test_make_dataset_matches_reference(gfb, task):
    """make_dataset (gf/training.py:287-307): the GPU bilinear resample and
    window mean reproduce the reference's seeded dataset."""
    ds = gfb.make_dataset(task, count=2, height=30, width=22, channels=3, seed=7)
    for n, (img, tgt) in enumerate(ds):
        assert np.abs(img - g(f"data_{task}", f"img{n}")).max() <= 1e-14
        # the reference sums windows from a float64 SAT, the GPU directly: 1e-12
        assert np.abs(tgt - g(f"data_{task}", f"tgt{n}")).max() <= 1e-12
