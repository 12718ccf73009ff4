"""Golden vectors for the callers of the guided-filter path:
the k x k guidance / core net, FixedChannelMeanGuidance, GuidedUpsampler
forward / backward, adam_step and a few train() steps -- from the REAL
reference package.  Build container only:

    NUMBA_CACHE_DIR=/tmp/numba PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_upsampler.py

Writes tests/golden/golden_upsampler.npz (keys ``<case>/<field>``).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_golden")
sys.path.insert(0, REF)

from guidedfilter import guidance, training  # noqa: E402
from guidedfilter.guided import GuidedFilterParams  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_upsampler.npz")


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def put(store, case, **fields):
    for k, v in fields.items():
        store[f"{case}/{k}"] = np.asarray(v)


def flat_params(d):
    return {k: np.asarray(v, dtype=np.float64) for k, v in d.items()}


def main():
    store = {}
    rng = np.random.default_rng(20260)

    # ---- k x k guidance / core net: forward + backward -------------------
    for i, (h, w, hid, k, dil) in enumerate([(13, 11, 5, 3, 1), (17, 15, 4, 3, 2),
                                             (9, 12, 6, 5, 1), (10, 10, 3, 1, 1)]):
        net = guidance.GuidanceNet(3, 3, hidden=hid, kernel=k, dilation=dil,
                                   rng=np.random.default_rng(100 + i))
        params = flat_params(net.parameters())
        params["norm.norm_gain"] = np.array([0.7])
        params["norm.gain"] = np.array([0.8])
        params["conv2.bias"] = f32(rng.uniform(-0.2, 0.2, 3))
        params = {kk: f32(v) for kk, v in params.items()}
        net.load_parameters(params)
        x = f32(rng.uniform(0, 1, (h, w, 3)))
        dy = f32(rng.standard_normal((h, w, 3)))
        y, tape = net.forward(x)
        dx, grads = net.backward(tape, dy)
        put(store, f"gk{i}", x=x, dy=dy, y=y, dx=dx, kernel=k, dilation=dil, hidden=hid,
            **{f"p.{kk}": v for kk, v in params.items()},
            **{f"g.{kk}": v for kk, v in grads.items()})

    # ---- FixedChannelMeanGuidance ------------------------------------------
    fm = guidance.FixedChannelMeanGuidance(3, 3)
    x = f32(rng.uniform(0, 1, (7, 9, 3)))
    dy = f32(rng.standard_normal((7, 9, 3)))
    y, tape = fm.forward(x)
    dx, _ = fm.backward(tape, dy)
    put(store, "fixed", x=x, dy=dy, y=y, dx=dx)

    # ---- GuidedUpsampler forward / backward --------------------------------
    for i, (learned, h, w, side, r) in enumerate([(True, 30, 26, 12, 1), (False, 28, 36, 9, 2),
                                                  (True, 41, 33, 16, 1)]):
        model = training.build_model(seed=7 + i, core_hidden=6, guide_hidden=5, radius=r,
                                     eps=1e-4, low_res_side=side, learned_guidance=learned)
        params = {kk: f32(v) for kk, v in model.parameters().items()}
        if learned:
            params["guide.norm.norm_gain"] = np.array([0.5])
        params["core.norm.norm_gain"] = np.array([0.6])
        model.load_parameters(params)
        image = f32(rng.uniform(0, 1, (h, w, 3)))
        d_out = f32(rng.standard_normal((h, w, 3)))
        out, tape = model.forward(image)
        d_image, grads = model.backward(tape, d_out)
        put(store, f"up{i}", image=image, d_out=d_out, out=out, d_image=d_image,
            learned=int(learned), side=side, radius=r, eps=1e-4,
            low=np.array(tape.low_dims),
            **{f"p.{kk}": v for kk, v in params.items()},
            **{f"g.{kk}": v for kk, v in grads.items()})

    # ---- adam_step -----------------------------------------------------------
    params = {"a": f32(rng.standard_normal((3, 4))), "b": f32(rng.standard_normal(5))}
    grads = {k: f32(rng.standard_normal(v.shape)) for k, v in params.items()}
    state = training.AdamState.init(params)
    state.m = {k: f32(rng.standard_normal(v.shape)) * 0.1 for k, v in params.items()}
    state.v = {k: f32(rng.uniform(0, 1, v.shape)) * 0.1 for k, v in params.items()}
    state.step = 4
    cfg = training.TrainConfig(learning_rate=3e-3)
    new_p, new_s = training.adam_step(params, grads, state, cfg)
    put(store, "adam", step=4, lr=3e-3,
        **{f"p.{k}": v for k, v in params.items()}, **{f"g.{k}": v for k, v in grads.items()},
        **{f"m.{k}": v for k, v in state.m.items()}, **{f"v.{k}": v for k, v in state.v.items()},
        **{f"np.{k}": v for k, v in new_p.items()}, **{f"nm.{k}": v for k, v in new_s.m.items()},
        **{f"nv.{k}": v for k, v in new_s.v.items()})

    # ---- train(): a few Adam steps through the filter (and the low-res mode) --
    for i, (through, learned) in enumerate([(True, True), (False, True), (True, False)]):
        model = training.build_model(seed=11 + i, core_hidden=4, guide_hidden=4, radius=1,
                                     eps=1e-4, low_res_side=8, learned_guidance=learned)
        params0 = {kk: f32(v) for kk, v in model.parameters().items()}
        model.load_parameters(params0)
        data = training.make_dataset("affine", count=2, height=20, width=18, seed=3 + i)
        data = [(f32(a), f32(b)) for a, b in data]
        cfg = training.TrainConfig(learning_rate=1e-2, steps=3)
        model, hist = training.train(model, data, cfg, through_filter=through)
        fields = {f"p0.{kk}": v for kk, v in params0.items()}
        fields.update({f"p1.{kk}": np.asarray(v) for kk, v in model.parameters().items()})
        for j, (a, b) in enumerate(data):
            fields[f"x{j}"] = a
            fields[f"t{j}"] = b
        put(store, f"train{i}", through=int(through), learned=int(learned), steps=3, lr=1e-2,
            history=np.array(hist), n=len(data), **fields)

    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT}: {len(store)} arrays")


if __name__ == "__main__":
    main()
