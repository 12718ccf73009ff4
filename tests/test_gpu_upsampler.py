"""GPU parity of the guided-filter path's callers: the k x k
guidance / core net (gnk_*), FixedChannelMeanGuidance, GuidedUpsampler,
Adam and train() -- fp64 against the reference's golden vectors at its own
bars, fp32 against the pinned oracle at the north_star tolerances."""

import os

import numpy as np
import pytest
import torch

from oracle import upsampler_oracle as U

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden_upsampler.npz")


@pytest.fixture(scope="module")
def gfb():
    import paper_1803_05619_b200 as m

    assert torch.cuda.is_available(), "gpu tests need CUDA"
    return m


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


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max()) / max(float(np.abs(b).max()), 1e-300)


def test_guidance_k_fp64_matches_reference(gfb, gold):
    for name, c in gold.items():
        if not name.startswith("gk"):
            continue
        net = gfb.GuidanceNet(3, 3, hidden=int(c["hidden"]), kernel=int(c["kernel"]),
                              dilation=int(c["dilation"]))
        net.load_parameters(sub(c, "p."))
        y, tape = net.forward(c["x"])
        assert rel(y, c["y"]) <= 1e-12, name
        dx, grads = net.backward(tape, c["dy"])
        assert rel(dx, c["dx"]) <= 1e-10, name
        for k, v in sub(c, "g.").items():
            assert rel(grads[k], v) <= 1e-9, (name, k)


def test_guidance_k_fp32_vs_oracle(gfb):
    rng = np.random.default_rng(5)
    params = U.guidance_k_init(3, 3, 24, 3, rng)
    params["norm.norm_gain"] = np.array([0.5])
    params = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in params.items()}
    x = rng.uniform(0, 1, (2, 3, 40, 52)).astype(np.float32)
    dy = rng.standard_normal((2, 3, 40, 52)).astype(np.float32)
    net = gfb.GuidanceNet(3, 3, hidden=24, kernel=3, dilation=2)
    net.load_parameters(params)
    y, tape = net.forward(torch.from_numpy(x).cuda())
    dx, grads = net.backward(tape, torch.from_numpy(dy).cuda())
    want_g = None
    for n in range(2):
        xh = x[n].transpose(1, 2, 0).astype(np.float64)
        yy, tp = U.guidance_k_forward(params, xh, 2)
        dxx, gg = U.guidance_k_backward(params, tp, dy[n].transpose(1, 2, 0).astype(np.float64))
        assert float(np.abs(y[n].cpu().numpy().transpose(1, 2, 0) - yy).max()) <= 1e-4
        assert rel(dx[n].cpu().numpy().transpose(1, 2, 0), dxx) <= 1e-3
        want_g = gg if want_g is None else {k: want_g[k] + gg[k] for k in gg}
    for k, v in want_g.items():
        assert rel(grads[k].double().cpu().numpy(), v) <= 1e-3, k


def test_fixed_mean_matches_reference(gfb, gold):
    c = gold["fixed"]
    fm = gfb.FixedChannelMeanGuidance(3, 3)
    y, tape = fm.forward(c["x"])
    assert float(np.abs(y - c["y"]).max()) <= 1e-15
    dx, g = fm.backward(tape, c["dy"])
    assert float(np.abs(dx - c["dx"]).max()) <= 1e-15 and g == {}
    with pytest.raises(ValueError):
        fm.load_parameters({"w": np.zeros(1)})


def _model_from(gfb, c):
    learned = bool(c["learned"])
    p = sub(c, "p.")
    core_hidden = p["core.conv1.weight"].shape[0]
    guide_hidden = p["guide.conv1.weight"].shape[0] if learned else 4
    model = gfb.build_model(seed=0, core_hidden=core_hidden, guide_hidden=guide_hidden,
                            radius=int(c["radius"]), eps=float(c["eps"]),
                            low_res_side=int(c["side"]), learned_guidance=learned)
    model.load_parameters(p)
    return model


def test_upsampler_fp64_matches_reference(gfb, gold):
    for name, c in gold.items():
        if not name.startswith("up"):
            continue
        model = _model_from(gfb, c)
        out, tape = model.forward(c["image"])
        assert tuple(tape.low_dims) == tuple(c["low"]), name
        assert float(np.abs(out - c["out"]).max()) <= 1e-10, name
        d_image, grads = model.backward(tape, c["d_out"])
        assert rel(d_image, c["d_image"]) <= 1e-9, name
        want = sub(c, "g.")
        assert set(grads) == set(want), name
        for k, v in want.items():
            assert rel(grads[k], v) <= 1e-9 or float(np.abs(grads[k] - v).max()) <= 1e-12, (name, k)


def test_adam_matches_reference(gfb, gold):
    c = gold["adam"]
    p, g, m, v = sub(c, "p."), sub(c, "g."), sub(c, "m."), sub(c, "v.")
    state = gfb.AdamState(m={k: torch.from_numpy(a).cuda() for k, a in m.items()},
                          v={k: torch.from_numpy(a).cuda() for k, a in v.items()},
                          step=int(c["step"]))
    new_p, new_s = gfb.adam_step(p, g, state, gfb.TrainConfig(learning_rate=float(c["lr"])))
    assert new_s.step == int(c["step"]) + 1
    for k in p:
        assert rel(new_p[k], c[f"np.{k}"]) <= 1e-14, k
        assert rel(new_s.m[k].cpu().numpy(), c[f"nm.{k}"]) <= 1e-14
        assert rel(new_s.v[k].cpu().numpy(), c[f"nv.{k}"]) <= 1e-14
    bad = {k: np.full_like(a, np.nan) for k, a in g.items()}
    with pytest.raises(gfb.TrainingError):
        gfb.adam_step(p, bad, gfb.AdamState.init(p), gfb.TrainConfig())


def test_train_fp64_matches_reference(gfb, gold):
    for name, c in gold.items():
        if not name.startswith("train"):
            continue
        learned = bool(c["learned"])
        p0 = sub(c, "p0.")
        model = gfb.build_model(seed=0, core_hidden=p0["core.conv1.weight"].shape[0],
                                guide_hidden=p0["guide.conv1.weight"].shape[0] if learned else 4,
                                radius=1, eps=1e-4, low_res_side=8, learned_guidance=learned)
        model.load_parameters(p0)
        data = [(c[f"x{j}"], c[f"t{j}"]) for j in range(int(c["n"]))]
        cfg = gfb.TrainConfig(learning_rate=float(c["lr"]), steps=int(c["steps"]))
        model, hist = gfb.train(model, data, cfg, through_filter=bool(c["through"]))
        assert np.allclose(hist, c["history"], rtol=1e-9, atol=0), (name, hist, c["history"])
        params = {k: v.double().cpu().numpy() for k, v in model.parameters().items()}
        for k, v in sub(c, "p1.").items():
            assert float(np.abs(params[k] - v).max()) <= 1e-8 * max(1.0, float(np.abs(v).max())), (
                name, k)


def test_train_fp32_decreases_loss(gfb):
    from oracle import gf_oracle as O

    rng = np.random.default_rng(1)
    data = []
    for _ in range(2):
        img = rng.uniform(0, 1, (48, 40, 3))
        data.append((img, O.affine_target(img)))
    model = gfb.build_model(seed=3, core_hidden=8, guide_hidden=15, low_res_side=16, eps=1e-4)
    model, hist = gfb.train(model, data, gfb.TrainConfig(learning_rate=1e-2, steps=30),
                            dtype=torch.float32)
    assert len(hist) == 31 and all(np.isfinite(hist))
    assert hist[-1] < 0.8 * hist[0]


def test_guidance_k_argument_errors(gfb):
    with pytest.raises(ValueError):
        gfb.GuidanceNet(3, 3, hidden=4, kernel=2)
    with pytest.raises(ValueError):
        gfb.GuidanceNet(3, 3, hidden=4, kernel=3, dilation=0)
    with pytest.raises(ValueError):
        gfb.TrainConfig(batch_size=2)
    with pytest.raises(ValueError):
        gfb.train(gfb.build_model(core_hidden=4, guide_hidden=4), [], gfb.TrainConfig(steps=1))


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_training_is_bitwise_deterministic(gfb, dtype):
    """Run-to-run bitwise determinism of train() (the reference's
    pkg/tests/test_training.py:227-234): identical loss histories and trained
    parameters -- every reduction on the path (guidance-net gradients, the
    MSE loss, Adam) is a fixed-order one, no floating-point atomics."""

    def run():
        model = gfb.build_model(seed=12, core_hidden=4, guide_hidden=4, low_res_side=8)
        dataset = gfb.make_dataset("affine", count=3, height=24, width=24, seed=12)
        model, history = gfb.train(model, dataset, gfb.TrainConfig(steps=25, seed=12),
                                   dtype=dtype)
        return history, {k: v.clone() for k, v in model.parameters().items()}

    h1, p1 = run()
    h2, p2 = run()
    assert h1 == h2
    for k in p1:
        assert torch.equal(p1[k], p2[k]), k
