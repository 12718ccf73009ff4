"""Pin the CPU oracle against golden vectors produced by the real reference.

No GPU needed.  Tolerances follow the reference's own tests (1e-12 for
operators, 1e-10 for the layer, per ``pkg/tests/test_guided.py``); the oracle
restates the same float64 algorithm so agreement is near-bitwise.
"""

import numpy as np
import pytest

from oracle import gf_oracle as O


def close(a, b, tol):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    scale = max(1.0, float(np.abs(b).max()) if b.size else 1.0)
    err = float(np.abs(a - b).max()) if a.size else 0.0
    assert err <= tol * scale, f"max abs err {err:.3e} > {tol:.1e} * {scale:.2e}"


def test_known_answers(golden):
    ka = golden["ka_box"]
    box = O.box_sum(ka["x"], 1)
    assert box[1, 1, 0] == 45.0 and box[0, 0, 0] == 12.0
    np.testing.assert_array_equal(box, ka["box"])
    m = O.mean_filter(ka["x"], 1)
    assert m[0, 0, 0] == pytest.approx(3.0, abs=1e-12)
    assert m[1, 1, 0] == pytest.approx(5.0, abs=1e-12)
    out = O.bilinear_resize(golden["ka_bilinear"]["x"], 1, 4)
    assert out.ravel().tolist() == [0.0, 0.5, 1.5, 2.0]
    # mse hand value (pkg/tests/test_training.py:44-49)
    loss, grad = O.mse_loss(np.array([1.0, 2.0]).reshape(1, 2, 1), np.zeros((1, 2, 1)))
    assert loss == 2.5 and grad.ravel().tolist() == [1.0, 2.0]


def test_filters_match_reference(golden):
    n = 0
    for name, c in golden.items():
        if name.startswith("mean"):
            r = int(c["r"])
            close(O.box_sum(c["x"], r), c["box"], 1e-12)
            close(O.mean_filter(c["x"], r), c["mean"], 1e-12)
            close(O.mean_filter_adjoint(c["g"], r), c["adj"], 1e-12)
            close(O.naive_box_sum(c["x"], r), c["box"], 1e-12)
            n += 1
        elif name.startswith("bil"):
            oh, ow = c["out"].shape[:2]
            h, w = c["x"].shape[:2]
            close(O.bilinear_resize(c["x"], oh, ow), c["out"], 1e-14)
            close(O.bilinear_resize_adjoint(c["g"], h, w), c["adj"], 1e-13)
            n += 1
    assert n >= 10


def test_joint_matches_reference(golden):
    cases = [c for k, c in golden.items() if k.startswith("joint")]
    assert len(cases) >= 10
    for c in cases:
        r, eps = int(c["r"]), float(c["eps"])
        out, tape = O.forward_joint(c["guide_lo"], c["guide_hi"], c["src_lo"], r, eps)
        close(out, c["out"], 1e-10)
        close(tape["slope"], c["slope"], 1e-10)
        close(tape["intercept"], c["intercept"], 1e-10)
        d_src, d_glo, d_ghi = O.backward(tape, c["d_out"])
        close(d_src, c["d_src"], 1e-10)
        close(d_glo, c["d_guide_lo"], 1e-10)
        close(d_ghi, c["d_guide_hi"], 1e-10)


def test_highres_matches_reference(golden):
    cases = [(k, c) for k, c in golden.items() if k.startswith("hr")]
    assert len(cases) >= 8
    for k, c in cases:
        r, eps = int(c["r"]), float(c["eps"])
        g4 = c["guide"].transpose(2, 0, 1)[None]
        s4 = c["src"].transpose(2, 0, 1)[None]
        d4 = c["d_out"].transpose(2, 0, 1)[None]
        out = O.highres_forward_nchw(g4, s4, r, eps)[0].transpose(1, 2, 0)
        close(out, c["out"], 1e-10)
        dg, ds = O.highres_backward_nchw(g4, s4, d4, r, eps)
        close(ds[0].transpose(1, 2, 0), c["d_src"], 1e-10)
        close(dg[0].transpose(1, 2, 0), c["d_guide"], 1e-10)


def test_guidance_matches_reference(golden):
    cases = [c for k, c in golden.items() if k.startswith("gn")]
    assert len(cases) >= 4
    for c in cases:
        params = {k[2:]: v for k, v in c.items() if k.startswith("p:")}
        y, tape = O.guidance_forward(params, c["x"])
        close(y, c["y"], 1e-12)
        dx, grads = O.guidance_backward(params, tape, c["dy"])
        close(dx, c["dx"], 1e-11)
        for k, v in grads.items():
            close(v, c["g:" + k], 1e-10)


def test_train_step_matches_reference(golden):
    c = golden["train0"]
    params = {k[2:]: v for k, v in c.items() if k.startswith("p:")}
    loss, outs, dlx, dly, dhx, grads = O.train_step(
        params, list(c["lr_x"]), list(c["hr_x"]), list(c["lr_y"]), list(c["target"]),
        int(c["r"]), float(c["eps"]))
    assert abs(loss - float(c["loss"])) <= 1e-12
    close(np.stack(outs), c["out"], 1e-10)
    close(np.stack(dlx), c["d_lr_x"], 1e-9)
    close(np.stack(dly), c["d_lr_y"], 1e-9)
    close(np.stack(dhx), c["d_hr_x"], 1e-9)
    for k, v in grads.items():
        close(v, c["g:" + k], 1e-9)


def test_error_semantics():
    rng = np.random.default_rng(0)
    gl, gh, sl = rng.uniform(0, 1, (6, 8, 2)), rng.uniform(0, 1, (12, 16, 2)), rng.uniform(0, 1, (6, 8, 2))
    with pytest.raises(ValueError):
        O.forward_joint(gl, gh, sl[:, :-1], 1, 1e-2)
    with pytest.raises(ValueError):
        O.forward_joint(gh, gl, gh, 1, 1e-2)
    bad = sl.copy()
    bad[0, 0, 0] = np.nan
    with pytest.raises(ValueError):
        O.forward_joint(gl, gh, bad, 1, 1e-2)
    with pytest.raises(O.DegenerateWindowError):
        O.forward_joint(np.full_like(gl, 0.25), gh, sl, 1, 0.0)
