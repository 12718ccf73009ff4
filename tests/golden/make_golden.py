"""Generate golden vectors from the REAL reference package.

Run in the build container only (``/root/reference`` does not exist on the GPU
box):

    NUMBA_CACHE_DIR=/tmp/numba PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It imports ``guidedfilter`` from ``/root/reference/pkg/src`` and writes
``tests/golden/golden.npz``: inputs (float32-representable float64, so both
the fp32 and fp64 GPU instantiations can consume them unchanged) and the
reference's outputs / gradients / tape fields.  Keys are ``<case>/<field>``.
The tests pin ``oracle/gf_oracle.py`` against this file and check the CUDA
path against both.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_golden")
sys.path.insert(0, REF)

from guidedfilter import filters as flt  # noqa: E402
from guidedfilter import guidance, guided, training  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def uni(rng, *shape, lo=0.0, hi=1.0):
    return f32(rng.uniform(lo, hi, shape))


def main():
    store: dict[str, np.ndarray] = {}

    def put(case, **kw):
        for k, v in kw.items():
            store[f"{case}/{k}"] = np.asarray(v)

    # ---- known answers (reference hand values) ---------------------------
    grid = np.arange(1.0, 10.0).reshape(3, 3, 1)
    put("ka_box", x=grid, r=1, box=flt.box_sum(grid, 1), mean=flt.mean_filter(grid, 1))
    row = np.array([0.0, 2.0]).reshape(1, 2, 1)
    put("ka_bilinear", x=row, out=flt.bilinear_resize(row, 1, 4))

    # ---- filters: mean / adjoint / bilinear / adjoint --------------------
    rng = np.random.default_rng(1000)
    for i, (h, w, c, r) in enumerate([(7, 5, 2, 1), (16, 11, 3, 3), (33, 32, 1, 9),
                                      (5, 4, 2, 7), (1, 1, 1, 2), (64, 64, 3, 17)]):
        t = uni(rng, h, w, c, lo=-2, hi=2)
        g = uni(rng, h, w, c, lo=-1, hi=1)
        put(f"mean{i}", x=t, g=g, r=r, mean=flt.mean_filter(t, r),
            adj=flt.mean_filter_adjoint(g, r), box=flt.box_sum(t, r))
    for i, ((h, w), (oh, ow)) in enumerate([((7, 9), (14, 18)), ((16, 16), (5, 11)),
                                           ((4, 4), (4, 4)), ((5, 9), (13, 4)),
                                           ((8, 8), (32, 32)), ((3, 5), (8, 7)),
                                           ((1, 1), (3, 4))]):
        t = uni(rng, h, w, 2, lo=-1, hi=1)
        g = uni(rng, oh, ow, 2, lo=-1, hi=1)
        put(f"bil{i}", x=t, g=g, out=flt.bilinear_resize(t, oh, ow),
            adj=flt.bilinear_resize_adjoint(g, h, w))

    # ---- joint forward + backward ----------------------------------------
    joint_cases = [
        ((6, 8, 2), (12, 16), 0, 1e-2), ((6, 8, 2), (12, 16), 1, 1e-2),
        ((6, 8, 2), (12, 16), 2, 1e-4), ((5, 6, 1), (10, 12), 1, 1e-2),
        ((8, 9, 2), (17, 18), 2, 1e-3), ((7, 9, 2), (14, 18), 1, 1e-4),
        ((16, 16, 3), (64, 64), 1, 1e-8), ((16, 12, 3), (64, 48), 2, 1e-4),
        ((12, 20, 3), (48, 80), 3, 1e-4), ((10, 10, 3), (40, 40), 8, 1e-4),
        ((16, 16, 3), (32, 32), 1, 1e-2), ((9, 7, 1), (9, 7), 1, 1e-2),
        ((20, 24, 3), (80, 96), 1, 1e-8), ((3, 2, 2), (13, 9), 4, 1e-2),
    ]
    for i, (lo, hi, r, eps) in enumerate(joint_cases):
        rng = np.random.default_rng(2000 + i)
        gl = uni(rng, *lo)
        gh = uni(rng, *hi, lo[2])
        sl = uni(rng, *lo)
        d = f32(rng.standard_normal((*hi, lo[2])))
        p = guided.GuidedFilterParams(r, eps)
        out, tape = guided.forward_joint(gl, gh, sl, p)
        g = guided.backward(tape, d)
        put(f"joint{i}", guide_lo=gl, guide_hi=gh, src_lo=sl, d_out=d, r=r, eps=eps,
            out=out, d_src=g.d_src, d_guide_lo=g.d_guide_lo, d_guide_hi=g.d_guide_hi,
            mean_guide=tape.mean_guide, var_guide=tape.var_guide, slope=tape.slope,
            intercept=tape.intercept)

    # ---- highres forward + backward --------------------------------------
    hr_cases = [((9, 8, 2), 1, 1e-2), ((9, 8, 2), 2, 1e-2), ((9, 8, 2), 4, 1e-2),
                ((14, 13, 3), 3, 1e-2), ((32, 32, 3), 4, 1e-2), ((40, 36, 3), 8, 1e-2),
                ((12, 10, 2), 2, 1e-4), ((5, 7, 1), 9, 1e-2)]
    for i, (shape, r, eps) in enumerate(hr_cases):
        rng = np.random.default_rng(3000 + i)
        gd = uni(rng, *shape)
        sr = uni(rng, *shape)
        d = f32(rng.standard_normal(shape))
        p = guided.GuidedFilterParams(r, eps)
        out, tape = guided.forward_highres(gd, sr, p)
        g = guided.backward(tape, d)
        put(f"hr{i}", guide=gd, src=sr, d_out=d, r=r, eps=eps, out=out, d_src=g.d_src,
            d_guide=g.d_guide_hi)
    # 1-channel guide broadcast over 3 channels (config 1 semantics)
    for i, (shape, r) in enumerate([((24, 20), 2), ((48, 40), 8)]):
        rng = np.random.default_rng(3500 + i)
        g1 = uni(rng, *shape, 1)
        sr = uni(rng, *shape, 3)
        d = f32(rng.standard_normal((*shape, 3)))
        p = guided.GuidedFilterParams(r, 1e-2)
        out, tape = guided.forward_highres(np.repeat(g1, 3, axis=2), sr, p)
        g = guided.backward(tape, d)
        put(f"hrb{i}", guide=g1, src=sr, d_out=d, r=r, eps=1e-2, out=out, d_src=g.d_src,
            d_guide=g.d_guide_hi.sum(axis=2, keepdims=True))

    # ---- guidance net (1x1) ----------------------------------------------
    for i, (cin, cout, hidden, ng, shape) in enumerate([
            (3, 3, 15, 0.0, (9, 11)), (3, 3, 15, 0.7, (16, 12)),
            (2, 2, 4, -0.4, (5, 6)), (3, 3, 64, 0.3, (8, 8)), (3, 2, 8, 1.5, (7, 13))]):
        rng = np.random.default_rng(4000 + i)
        net = guidance.GuidanceNet(cin, cout, hidden=hidden, kernel=1, rng=rng)
        net.norm.norm_gain[:] = ng
        net.norm.gain[:] = 1.0 if i % 2 == 0 else 0.8
        net.conv2.bias[:] = f32(rng.uniform(-0.1, 0.1, cout))
        net.conv1.weight[:] = f32(net.conv1.weight)
        net.conv2.weight[:] = f32(net.conv2.weight)
        x = uni(rng, *shape, cin)
        dy = f32(rng.standard_normal((*shape, cout)))
        y, tape = net.forward(x)
        dx, grads = net.backward(tape, dy)
        kw = {f"p:{k}": v for k, v in net.parameters().items()}
        kw.update({f"g:{k}": v for k, v in grads.items()})
        put(f"gn{i}", x=x, dy=dy, y=y, dx=dx, **kw)

    # ---- config-2 style training step (batch 2, small) -------------------
    rng = np.random.default_rng(5000)
    net = guidance.GuidanceNet(3, 3, hidden=15, kernel=1, rng=rng)
    net.norm.norm_gain[:] = 0.5
    net.conv1.weight[:] = f32(net.conv1.weight)
    net.conv2.weight[:] = f32(net.conv2.weight)
    bsz, lo, hi = 2, (8, 10), (32, 40)
    hr_x = [uni(rng, *hi, 3) for _ in range(bsz)]
    lr_x = [flt.bilinear_resize(h, *lo) for h in hr_x]
    lr_x = [f32(v) for v in lr_x]
    lr_y = [uni(rng, *lo, 3) for _ in range(bsz)]
    tgt = [training.affine_target(h) for h in hr_x]
    p = guided.GuidedFilterParams(1, 1e-8)
    loss_total = 0.0
    gsum = None
    outs, dlx, dly, dhx = [], [], [], []
    for n in range(bsz):
        gl, tl = net.forward(lr_x[n])
        gh, th = net.forward(hr_x[n])
        out, tp = guided.forward_joint(gl, gh, lr_y[n], p)
        loss, d = training.mse_loss(out, tgt[n])
        loss_total += loss / bsz
        d = d / bsz
        gg = guided.backward(tp, d)
        dxl, g_lo = net.backward(tl, gg.d_guide_lo)
        dxh, g_hi = net.backward(th, gg.d_guide_hi)
        tot = {k: g_lo[k] + g_hi[k] for k in g_lo}
        gsum = tot if gsum is None else {k: gsum[k] + tot[k] for k in gsum}
        outs.append(out)
        dlx.append(dxl)
        dly.append(gg.d_src)
        dhx.append(dxh)
    kw = {f"p:{k}": v for k, v in net.parameters().items()}
    kw.update({f"g:{k}": v for k, v in gsum.items()})
    put("train0", lr_x=np.stack(lr_x), hr_x=np.stack(hr_x), lr_y=np.stack(lr_y),
        target=np.stack(tgt), r=1, eps=1e-8, loss=loss_total, out=np.stack(outs),
        d_lr_x=np.stack(dlx), d_lr_y=np.stack(dly), d_hr_x=np.stack(dhx), **kw)

    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT}: {len(store)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
