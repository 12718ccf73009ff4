"""Pin oracle/upsampler_oracle.py against golden vectors of the real reference
(tests/golden/golden_upsampler.npz): k x k guidance net, fixed mean guidance,
GuidedUpsampler forward / backward, adam_step and train()."""

import os

import numpy as np
import pytest

from oracle import upsampler_oracle as U

GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden_upsampler.npz")


@pytest.fixture(scope="module")
def gold():
    data = np.load(GOLD)
    cases: dict[str, dict[str, np.ndarray]] = {}
    for key in data.files:
        case, field = key.split("/", 1)
        cases.setdefault(case, {})[field] = data[key]
    return cases


def sub(c, prefix):
    return {k[len(prefix):]: v for k, v in c.items() if k.startswith(prefix)}


def close(a, b, tol):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    scale = max(float(np.abs(b).max()), 1.0)
    return float(np.abs(a - b).max()) <= tol * scale


def test_guidance_k(gold):
    for name, c in gold.items():
        if not name.startswith("gk"):
            continue
        params = sub(c, "p.")
        y, tape = U.guidance_k_forward(params, c["x"], int(c["dilation"]))
        assert close(y, c["y"], 1e-12), name
        dx, g = U.guidance_k_backward(params, tape, c["dy"])
        assert close(dx, c["dx"], 1e-12), name
        for k, v in sub(c, "g.").items():
            assert close(g[k], v, 1e-12), (name, k)


def test_fixed_mean(gold):
    c = gold["fixed"]
    assert close(U.fixed_mean_forward(c["x"], 3), c["y"], 1e-15)
    assert close(U.fixed_mean_backward(c["dy"], 3), c["dx"], 1e-15)


def test_upsampler(gold):
    for name, c in gold.items():
        if not name.startswith("up"):
            continue
        core, guide = U.split(sub(c, "p."))
        learned = bool(c["learned"])
        out, tape = U.upsampler_forward(core, guide, c["image"], int(c["radius"]),
                                        float(c["eps"]), int(c["side"]), learned)
        assert tuple(U.low_dims(*c["image"].shape[:2], int(c["side"]))) == tuple(c["low"])
        assert close(out, c["out"], 1e-10), name
        d_image, grads = U.upsampler_backward(core, guide, tape, c["d_out"], learned)
        assert close(d_image, c["d_image"], 1e-9), name
        want = sub(c, "g.")
        assert set(grads) == set(want), name
        for k, v in want.items():
            assert close(grads[k], v, 1e-9), (name, k)


def test_adam(gold):
    c = gold["adam"]
    p, g, m, v = sub(c, "p."), sub(c, "g."), sub(c, "m."), sub(c, "v.")
    np_, nm, nv, t = U.adam_step(p, g, m, v, int(c["step"]), float(c["lr"]))
    assert t == int(c["step"]) + 1
    for k in p:
        assert close(np_[k], c[f"np.{k}"], 1e-15)
        assert close(nm[k], c[f"nm.{k}"], 1e-15)
        assert close(nv[k], c[f"nv.{k}"], 1e-15)


def test_train(gold):
    for name, c in gold.items():
        if not name.startswith("train"):
            continue
        data = [(c[f"x{j}"], c[f"t{j}"]) for j in range(int(c["n"]))]
        params, hist = U.train(sub(c, "p0."), data, int(c["steps"]), float(c["lr"]), 1, 1e-4, 8,
                               learned=bool(c["learned"]), through_filter=bool(c["through"]))
        assert np.allclose(hist, c["history"], rtol=1e-9, atol=0), name
        # parameters whose gradient is pure rounding noise (e.g. the guide's
        # conv2 bias) move by Adam-normalised noise: judge on the unit scale
        for k, v in sub(c, "p1.").items():
            assert close(params[k], v, 1e-8), (name, k)


def test_oracle_layers_match_reference_golden():
    """Oracle ConvLayer / AdaptiveNorm vs the real reference's standalone
    layers (tests/golden/golden_layers.npz, make_golden_layers.py)."""
    import os

    from oracle import gf_oracle as O
    from oracle import upsampler_oracle as U

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_layers.npz"))
    cases = sorted({k.split("/")[0] for k in z.files})
    for c in cases:
        if c.startswith("data"):
            continue
        if c.startswith("conv"):
            ci, co, k, d, bias = z[f"{c}/meta"]
            w = z[f"{c}/weight"]
            y, padded = U.conv_forward(z[f"{c}/x"], w, int(d))
            if bias:
                y = y + z[f"{c}/bias"]
            assert np.abs(y - z[f"{c}/y"]).max() <= 1e-12, c
            dx, dw = U.conv_backward(padded, w, int(d), z[f"{c}/dy"])
            assert np.abs(dx - z[f"{c}/dx"]).max() <= 1e-12, c
            assert np.abs(dw - z[f"{c}/d_weight"]).max() <= 1e-12, c
            if bias:
                assert np.abs(z[f"{c}/dy"].sum(axis=(0, 1)) - z[f"{c}/d_bias"]).max() <= 1e-12
        else:
            gain, ng = z[f"{c}/gains"]
            y, tape = O.adaptive_norm_forward(z[f"{c}/x"], gain, ng)
            assert np.abs(y - z[f"{c}/y"]).max() <= 1e-12, c
            dx, dg, dn = O.adaptive_norm_backward(tape, z[f"{c}/dy"], gain, ng)
            assert np.abs(dx - z[f"{c}/dx"]).max() <= 1e-10, c
            assert abs(dg - z[f"{c}/d_gain"][0]) <= 1e-10 * max(1, abs(dg)), c
            assert abs(dn - z[f"{c}/d_norm_gain"][0]) <= 1e-10 * max(1, abs(dn)), c
