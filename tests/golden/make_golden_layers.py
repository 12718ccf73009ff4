"""Golden vectors of the reference's standalone guidance layers.

Run in the build container only (``/root/reference`` does not exist on the GPU
box):

    NUMBA_CACHE_DIR=/tmp/numba PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_layers.py

Imports ``guidedfilter`` from ``/root/reference/pkg/src`` and writes
``tests/golden/golden_layers.npz``: ConvLayer (gf/guidance.py:52-124) forward
and backward for kernels 1, 3, 5, dilations 1..3, with and without bias, and
AdaptiveNorm (gf/guidance.py:134-173) forward and backward for several
(gain, norm_gain), including a constant channel (the variance floor), and
make_dataset (gf/training.py:287-307) for the three synthetic tasks.  Keys
are ``<case>/<field>``; inputs are float32-representable float64.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_golden")
sys.path.insert(0, REF)

from guidedfilter import guidance, training  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_layers.npz")


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def main():
    out = {}
    conv_cases = [  # name, in, out, k, dilation, bias, h, w
        ("conv_k1", 3, 15, 1, 1, False, 9, 13),
        ("conv_k1_bias", 15, 3, 1, 1, True, 7, 11),
        ("conv_k3", 3, 8, 3, 1, True, 10, 12),
        ("conv_k3_d2", 4, 5, 3, 2, False, 11, 9),
        ("conv_k5_d3", 2, 3, 5, 3, True, 12, 14),
        ("conv_k3_tiny", 3, 4, 3, 2, True, 2, 3),
    ]
    for i, (name, ci, co, k, d, bias, h, w) in enumerate(conv_cases):
        rng = np.random.default_rng(100 + i)
        layer = guidance.ConvLayer(ci, co, kernel=k, dilation=d, bias=bias, rng=rng)
        layer.load_parameters({kk: f32(v) for kk, v in layer.parameters().items()})
        if bias:
            layer.bias = f32(rng.uniform(-0.5, 0.5, co))
        x = f32(rng.uniform(-1, 1, (h, w, ci)))
        y, tape = layer.forward(x)
        dy = f32(rng.standard_normal(y.shape))
        dx, grads = layer.backward(tape, dy)
        out[f"{name}/meta"] = np.array([ci, co, k, d, int(bias)])
        out[f"{name}/weight"] = layer.weight
        if bias:
            out[f"{name}/bias"] = layer.bias
        out[f"{name}/x"] = x
        out[f"{name}/y"] = y
        out[f"{name}/dy"] = dy
        out[f"{name}/dx"] = dx
        for kk, v in grads.items():
            out[f"{name}/d_{kk}"] = v
    norm_cases = [("norm_default", 1.0, 0.0, 8, 10, 5, False),
                  ("norm_mixed", 0.7, 1.3, 9, 7, 15, False),
                  ("norm_only", 0.0, 2.0, 6, 6, 3, False),
                  ("norm_const_channel", 1.1, 0.9, 5, 8, 4, True)]
    for i, (name, gain, ng, h, w, c, const) in enumerate(norm_cases):
        rng = np.random.default_rng(200 + i)
        layer = guidance.AdaptiveNorm(gain=gain, norm_gain=ng)
        x = f32(rng.uniform(-2, 2, (h, w, c)))
        if const:
            x[:, :, 1] = 0.25
        y, tape = layer.forward(x)
        dy = f32(rng.standard_normal(y.shape))
        dx, grads = layer.backward(tape, dy)
        out[f"{name}/gains"] = np.array([gain, ng])
        out[f"{name}/x"] = x
        out[f"{name}/y"] = y
        out[f"{name}/dy"] = dy
        out[f"{name}/dx"] = dx
        out[f"{name}/d_gain"] = grads["gain"]
        out[f"{name}/d_norm_gain"] = grads["norm_gain"]
    # synthetic datasets (gf/training.py:287-307): the bilinear resample and
    # window-mean targets the tests recompute on the GPU
    for task in ("affine", "smooth", "gamma"):
        ds = training.make_dataset(task, count=2, height=30, width=22, channels=3, seed=7)
        for n, (img, tgt) in enumerate(ds):
            out[f"data_{task}/img{n}"] = img
            out[f"data_{task}/tgt{n}"] = tgt
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(out)} arrays")


if __name__ == "__main__":
    main()
