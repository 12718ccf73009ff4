"""CPU oracle: a float64 numpy restatement of the reference guided-filter path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module, and only as the checker (or the timed CPU baseline), never as the
product path.  The product (``paper_1803_05619_b200``) never imports it.

Parity is PINNED, not assumed: ``tests/test_oracle.py`` checks every function
here against golden vectors produced by the real reference package
(``tests/golden/make_golden.py`` imports ``/root/reference/pkg/src`` in the
build container and writes ``tests/golden/*.npz``), plus the reference's own
hand-valued known-answer tests.

Conventions follow the reference exactly: images are float64 HWC
``(h, w, c)`` arrays (``gf/tensor.py:1-11``), box windows are clamped to the
image and normalised by the true pixel count (``gf/filters.py:82-103``),
resampling uses half-pixel centres with edge clamping (``gf/filters.py:119-156``).
``gf/`` below means ``/root/reference/pkg/src/guidedfilter/``.
"""

from __future__ import annotations

import numpy as np

LEAKY_SLOPE = 0.2          # gf/guidance.py:25
NORM_VAR_FLOOR = 1e-5      # gf/guidance.py:26


class DegenerateWindowError(ArithmeticError):
    """gf/guided.py:38-39."""


# --------------------------------------------------------------------------
# linear operators (gf/filters.py)
# --------------------------------------------------------------------------

def box_sum(t: np.ndarray, r: int) -> np.ndarray:
    """Clamped-window sum via a float64 summed-area table.

    Follows gf/filters.py:32-65 (SAT = cumsum rows then cols, four lookups in
    the order ``((s11 - s01) - s10) + s00``).
    """
    if r == 0:
        return t.copy()
    h, w, c = t.shape
    sat = np.zeros((h + 1, w + 1, c), dtype=np.float64)
    sat[1:, 1:] = t.cumsum(axis=0).cumsum(axis=1)
    ys, xs = np.arange(h), np.arange(w)
    y0 = np.maximum(ys - r, 0)
    y1 = np.minimum(ys + r, h - 1) + 1
    x0 = np.maximum(xs - r, 0)
    x1 = np.minimum(xs + r, w - 1) + 1
    out = sat[y1[:, None], x1[None, :]]
    out -= sat[y0[:, None], x1[None, :]]
    out -= sat[y1[:, None], x0[None, :]]
    out += sat[y0[:, None], x0[None, :]]
    return out


def naive_box_sum(t: np.ndarray, r: int) -> np.ndarray:
    """Direct window summation (gf/filters.py:68-79); small cases only."""
    h, w, _ = t.shape
    out = np.empty_like(t)
    for y in range(h):
        ya, yb = max(0, y - r), min(h, y + r + 1)
        for x in range(w):
            xa, xb = max(0, x - r), min(w, x + r + 1)
            out[y, x] = t[ya:yb, xa:xb].sum(axis=(0, 1))
    return out


def window_counts(h: int, w: int, r: int) -> np.ndarray:
    """N(y, x) = ny(y) * nx(x) (gf/filters.py:82-93), shape (h, w, 1)."""
    ys, xs = np.arange(h), np.arange(w)
    ny = np.minimum(ys + r, h - 1) - np.maximum(ys - r, 0) + 1
    nx = np.minimum(xs + r, w - 1) - np.maximum(xs - r, 0) + 1
    return (ny[:, None] * nx[None, :]).astype(np.float64)[:, :, None]


def mean_filter(t: np.ndarray, r: int) -> np.ndarray:
    """gf/filters.py:96-103."""
    h, w, _ = t.shape
    return box_sum(t, r) / window_counts(h, w, r)


def mean_filter_adjoint(g: np.ndarray, r: int) -> np.ndarray:
    """M^T g = box_sum(g / N) (gf/filters.py:106-116)."""
    h, w, _ = g.shape
    return box_sum(g / window_counts(h, w, r), r)


def axis_map(n_in: int, n_out: int):
    """Half-pixel source index/weight per output coordinate (gf/filters.py:119-131)."""
    s = (np.arange(n_out, dtype=np.float64) + 0.5) * (n_in / n_out) - 0.5
    np.clip(s, 0.0, n_in - 1.0, out=s)
    lo = np.minimum(np.floor(s).astype(np.intp), n_in - 1)
    frac = s - lo
    hi = np.minimum(lo + 1, n_in - 1)
    return lo, hi, frac


def bilinear_resize(t: np.ndarray, out_h: int, out_w: int) -> np.ndarray:
    """Rows then columns, lerp as lo + f*(hi - lo) (gf/filters.py:134-156)."""
    h, w, _ = t.shape
    ylo, yhi, fy = axis_map(h, out_h)
    xlo, xhi, fx = axis_map(w, out_w)
    rows = t[ylo]
    tmp = t[yhi] - rows
    tmp *= fy[:, None, None]
    tmp += rows
    lo = tmp[:, xlo]
    out = tmp[:, xhi] - lo
    out *= fx[None, :, None]
    out += lo
    return out


def _segment_rows(vals: np.ndarray, idx: np.ndarray, n: int) -> np.ndarray:
    out = np.zeros((n, vals.shape[1]), dtype=np.float64)
    np.add.at(out, idx, vals)
    return out


def bilinear_resize_adjoint(g: np.ndarray, in_h: int, in_w: int) -> np.ndarray:
    """Exact transpose of bilinear_resize (gf/filters.py:159-188): scatter
    with weights (1-f) to lo and f to hi, rows first, then columns."""
    out_h, out_w, c = g.shape
    ylo, yhi, fy = axis_map(in_h, out_h)
    xlo, xhi, fx = axis_map(in_w, out_w)
    g2 = g.reshape(out_h, out_w * c)
    rows = _segment_rows(g2 * (1.0 - fy)[:, None], ylo, in_h)
    rows += _segment_rows(g2 * fy[:, None], yhi, in_h)
    cols_in = rows.reshape(in_h, out_w, c).transpose(1, 0, 2).reshape(out_w, in_h * c)
    cols = _segment_rows(cols_in * (1.0 - fx)[:, None], xlo, in_w)
    cols += _segment_rows(cols_in * fx[:, None], xhi, in_w)
    return np.ascontiguousarray(cols.reshape(in_w, in_h, c).transpose(1, 0, 2))


# --------------------------------------------------------------------------
# the layer (gf/guided.py)
# --------------------------------------------------------------------------

def window_moments(guide, src, r: int, eps: float):
    """gf/guided.py:136-149."""
    mean_guide = mean_filter(guide, r)
    mean_src = mean_filter(src, r)
    var_guide = mean_filter(guide * guide, r) - mean_guide * mean_guide
    cov = mean_filter(guide * src, r) - mean_guide * mean_src
    if eps == 0.0 and np.any(var_guide <= 0.0):
        raise DegenerateWindowError("eps=0 requires positive guidance variance")
    slope = cov / (var_guide + eps)
    intercept = mean_src - slope * mean_guide
    return mean_guide, mean_src, var_guide, cov, slope, intercept


def _check_finite(*arrs):
    for a in arrs:
        if not np.isfinite(a).all():
            raise ValueError("non-finite input")


def forward_joint(guide_lo, guide_hi, src_lo, r: int, eps: float):
    """Fast (joint-upsampling) forward, gf/guided.py:152-195.  NO A/b smoothing."""
    _check_finite(guide_lo, guide_hi, src_lo)
    if guide_lo.shape != src_lo.shape:
        raise ValueError("guide_lo/src_lo shape mismatch")
    if guide_hi.shape[2] != guide_lo.shape[2]:
        raise ValueError("channel mismatch")
    if guide_hi.shape[0] < guide_lo.shape[0] or guide_hi.shape[1] < guide_lo.shape[1]:
        raise ValueError("guide_hi smaller than guide_lo")
    mg, ms, var, cov, slope, intercept = window_moments(guide_lo, src_lo, r, eps)
    hh, hw = guide_hi.shape[:2]
    slope_hi = bilinear_resize(slope, hh, hw)
    intercept_hi = bilinear_resize(intercept, hh, hw)
    out = intercept_hi + slope_hi * guide_hi
    if not np.isfinite(out).all():
        raise ValueError("guided filter produced non-finite output; increase eps")
    tape = dict(variant="joint", r=r, eps=eps, guide=guide_lo, src=src_lo,
                mean_guide=mg, mean_src=ms, var_guide=var, cov=cov, slope=slope,
                intercept=intercept, guide_hi=guide_hi, slope_hi=slope_hi)
    return out, tape


def forward_highres(guide, src, r: int, eps: float):
    """Full-resolution forward, gf/guided.py:198-233 (A, b re-smoothed)."""
    _check_finite(guide, src)
    if guide.shape != src.shape:
        raise ValueError("guide/src shape mismatch")
    mg, ms, var, cov, slope, intercept = window_moments(guide, src, r, eps)
    slope_hi = mean_filter(slope, r)
    intercept_hi = mean_filter(intercept, r)
    out = intercept_hi + slope_hi * guide
    if not np.isfinite(out).all():
        raise ValueError("guided filter produced non-finite output; increase eps")
    tape = dict(variant="highres", r=r, eps=eps, guide=guide, src=src,
                mean_guide=mg, mean_src=ms, var_guide=var, cov=cov, slope=slope,
                intercept=intercept, guide_hi=guide, slope_hi=slope_hi)
    return out, tape


def _moment_backward(t, d_slope, d_intercept):
    """gf/guided.py:236-264 (all signs +1: no mutation)."""
    r, eps = t["r"], t["eps"]
    denom = t["var_guide"] + eps
    d_cov = d_slope / denom
    d_var = -d_slope * t["cov"] / (denom * denom)
    d_mean_src = d_intercept + (-d_cov * t["mean_guide"])
    d_mean_guide = (-d_intercept * t["slope"]) + (-d_cov * t["mean_src"]) + (
        -2.0 * d_var * t["mean_guide"])
    back_cov = mean_filter_adjoint(d_cov, r)
    d_src = back_cov * t["guide"] + mean_filter_adjoint(d_mean_src, r)
    d_guide = (back_cov * t["src"] + 2.0 * mean_filter_adjoint(d_var, r) * t["guide"]
               + mean_filter_adjoint(d_mean_guide, r))
    return d_src, d_guide


def backward(t, d_out):
    """gf/guided.py:267-297.  Returns (d_src, d_guide_lo or None, d_guide_hi)."""
    if d_out.shape != t["guide_hi"].shape:
        raise ValueError("d_out shape mismatch")
    if t["variant"] == "joint":
        lh, lw = t["guide"].shape[:2]
        d_intercept = bilinear_resize_adjoint(d_out, lh, lw)
        d_slope = bilinear_resize_adjoint(d_out * t["guide_hi"], lh, lw) + (
            -d_intercept * t["mean_guide"])
        d_guide_hi = d_out * t["slope_hi"]
        d_src, d_guide_lo = _moment_backward(t, d_slope, d_intercept)
        return d_src, d_guide_lo, d_guide_hi
    r = t["r"]
    d_intercept = mean_filter_adjoint(d_out, r)
    d_slope = mean_filter_adjoint(d_out * t["guide_hi"], r) + (-d_intercept * t["mean_guide"])
    d_direct = d_out * t["slope_hi"]
    d_src, d_mom = _moment_backward(t, d_slope, d_intercept)
    return d_src, None, d_direct + d_mom


# --------------------------------------------------------------------------
# 1x1 guidance net (gf/guidance.py) and loss (gf/training.py)
# --------------------------------------------------------------------------

def xavier_uniform(rng, out_ch, in_ch, kernel):
    """gf/guidance.py:29-33."""
    fan_in = in_ch * kernel * kernel
    fan_out = out_ch * kernel * kernel
    limit = np.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-limit, limit, (out_ch, in_ch, kernel, kernel))


def guidance_init(in_ch, out_ch, hidden, rng):
    """GuidanceNet(in, out, hidden, kernel=1, rng) parameter draw order
    (gf/guidance.py:187-194, :71-74): conv1 weight, then conv2 weight."""
    w1 = xavier_uniform(rng, hidden, in_ch, 1)
    w2 = xavier_uniform(rng, out_ch, hidden, 1)
    return {
        "conv1.weight": w1,
        "norm.gain": np.array([1.0]),
        "norm.norm_gain": np.array([0.0]),
        "conv2.weight": w2,
        "conv2.bias": np.zeros(out_ch),
    }


def adaptive_norm_forward(x, gain, norm_gain):
    """AdaptiveNorm.forward (gf/guidance.py:152-159): per-channel spatial
    mean / population variance, inv_std = 1/sqrt(var + 1e-5)."""
    mean = x.mean(axis=(0, 1), keepdims=True)
    var = x.var(axis=(0, 1), keepdims=True)
    inv_std = 1.0 / np.sqrt(var + NORM_VAR_FLOOR)
    xhat = (x - mean) * inv_std
    return gain * x + norm_gain * xhat, dict(x=x, xhat=xhat, inv_std=inv_std)


def adaptive_norm_backward(tape, dy, gain, norm_gain):
    """AdaptiveNorm.backward (gf/guidance.py:161-173)."""
    d_gain = float(np.vdot(dy, tape["x"]))
    d_ng = float(np.vdot(dy, tape["xhat"]))
    g = norm_gain * dy
    g_mean = g.mean(axis=(0, 1), keepdims=True)
    g_proj = (g * tape["xhat"]).mean(axis=(0, 1), keepdims=True)
    dx = gain * dy + (g - g_mean - tape["xhat"] * g_proj) * tape["inv_std"]
    return dx, d_gain, d_ng


def guidance_forward(params, x):
    """conv1 (1x1, no bias) -> AdaptiveNorm -> leaky ReLU -> conv2 (1x1 + bias).
    gf/guidance.py:87-104 (conv), :152-159 (norm), :36-39 (lrelu), :209-214."""
    w1 = params["conv1.weight"][:, :, 0, 0]
    w2 = params["conv2.weight"][:, :, 0, 0]
    gain = float(params["norm.gain"][0])
    ng = float(params["norm.norm_gain"][0])
    h1 = x @ w1.T
    mean = h1.mean(axis=(0, 1), keepdims=True)
    var = h1.var(axis=(0, 1), keepdims=True)
    inv_std = 1.0 / np.sqrt(var + NORM_VAR_FLOOR)
    xhat = (h1 - mean) * inv_std
    h2 = gain * h1 + ng * xhat
    mask = h2 >= 0.0
    h3 = np.where(mask, h2, LEAKY_SLOPE * h2)
    y = h3 @ w2.T + params["conv2.bias"]
    return y, dict(x=x, h1=h1, xhat=xhat, inv_std=inv_std, mask=mask, h3=h3)


def guidance_backward(params, tape, dy):
    """gf/guidance.py:216-224 with ConvLayer.backward (:106-124),
    leaky_relu_backward (:42-43), AdaptiveNorm.backward (:161-173)."""
    w1 = params["conv1.weight"][:, :, 0, 0]
    w2 = params["conv2.weight"][:, :, 0, 0]
    gain = float(params["norm.gain"][0])
    ng = float(params["norm.norm_gain"][0])
    d_w2 = np.tensordot(dy, tape["h3"], axes=((0, 1), (0, 1)))
    d_b2 = dy.sum(axis=(0, 1))
    d3 = dy @ w2
    d2 = np.where(tape["mask"], d3, LEAKY_SLOPE * d3)
    d_gain = float(np.vdot(d2, tape["h1"]))
    d_ng = float(np.vdot(d2, tape["xhat"]))
    g = ng * d2
    g_mean = g.mean(axis=(0, 1), keepdims=True)
    g_proj = (g * tape["xhat"]).mean(axis=(0, 1), keepdims=True)
    d1 = gain * d2 + (g - g_mean - tape["xhat"] * g_proj) * tape["inv_std"]
    d_w1 = np.tensordot(d1, tape["x"], axes=((0, 1), (0, 1)))
    dx = d1 @ w1
    grads = {
        "conv1.weight": d_w1[:, :, None, None],
        "norm.gain": np.array([d_gain]),
        "norm.norm_gain": np.array([d_ng]),
        "conv2.weight": d_w2[:, :, None, None],
        "conv2.bias": d_b2,
    }
    return dx, grads


def mse_loss(out, target):
    """gf/training.py:93-101."""
    diff = out - target
    return float(np.mean(diff * diff)), 2.0 * diff / diff.size


def affine_target(image):
    """gf/training.py:265-267."""
    return np.clip(1.5 * image - 0.25, 0.0, 1.0)


def train_step(params, lr_x, hr_x, lr_y, target, r, eps):
    """One config-2 step over a batch (lists of HWC images), batch-mean loss.

    Follows GuidedUpsampler.forward/backward (gf/training.py:143-183) with the
    core net replaced by the given ``lr_y`` (config 2 feeds lr_y directly):
    F on lo then hi, joint GF, mse, GF backward, F backward lo first then hi.
    Returns (loss, out list, d_lr_x list, d_lr_y list, d_hr_x list, grads).
    """
    bsz = len(hr_x)
    grads = {k: np.zeros_like(v) for k, v in params.items()}
    loss_total = 0.0
    outs, dlx, dly, dhx = [], [], [], []
    for n in range(bsz):
        gl, tl = guidance_forward(params, lr_x[n])
        gh, th = guidance_forward(params, hr_x[n])
        out, tp = forward_joint(gl, gh, lr_y[n], r, eps)
        loss, d = mse_loss(out, target[n])
        loss_total += loss / bsz
        d = d / bsz
        d_src, d_glo, d_ghi = backward(tp, d)
        dx_lo, g_lo = guidance_backward(params, tl, d_glo)
        dx_hi, g_hi = guidance_backward(params, th, d_ghi)
        for k in grads:
            grads[k] = grads[k] + (g_lo[k] + g_hi[k])
        outs.append(out)
        dlx.append(dx_lo)
        dly.append(d_src)
        dhx.append(dx_hi)
    return loss_total, outs, dlx, dly, dhx, grads


# --------------------------------------------------------------------------
# NCHW batch helpers (float64); the GPU side is NCHW
# --------------------------------------------------------------------------

def nchw_to_hwc_list(a: np.ndarray):
    return [np.ascontiguousarray(a[n].transpose(1, 2, 0), dtype=np.float64) for n in range(a.shape[0])]


def hwc_list_to_nchw(lst):
    return np.stack([x.transpose(2, 0, 1) for x in lst], axis=0)


def joint_forward_nchw(lr_x, lr_y, hr_x, r, eps):
    """Batched forward_joint on NCHW float arrays; returns NCHW float64 out."""
    outs = []
    for gl, sl, gh in zip(nchw_to_hwc_list(lr_x), nchw_to_hwc_list(lr_y), nchw_to_hwc_list(hr_x)):
        outs.append(forward_joint(gl, gh, sl, r, eps)[0])
    return hwc_list_to_nchw(outs)


def joint_backward_nchw(lr_x, lr_y, hr_x, d_out, r, eps):
    """Returns (d_lr_x, d_lr_y, d_hr_x) NCHW float64."""
    dlx, dly, dhx = [], [], []
    for gl, sl, gh, d in zip(nchw_to_hwc_list(lr_x), nchw_to_hwc_list(lr_y),
                             nchw_to_hwc_list(hr_x), nchw_to_hwc_list(d_out)):
        _, tape = forward_joint(gl, gh, sl, r, eps)
        d_src, d_glo, d_ghi = backward(tape, d)
        dlx.append(d_glo)
        dly.append(d_src)
        dhx.append(d_ghi)
    return hwc_list_to_nchw(dlx), hwc_list_to_nchw(dly), hwc_list_to_nchw(dhx)


def highres_forward_nchw(guide, src, r, eps):
    """guide (B, Cg, H, W) with Cg in {1, C} is replicated over C."""
    c = src.shape[1]
    outs = []
    for g, s in zip(nchw_to_hwc_list(guide), nchw_to_hwc_list(src)):
        if g.shape[2] != c:
            g = np.repeat(g, c, axis=2)
        outs.append(forward_highres(g, s, r, eps)[0])
    return hwc_list_to_nchw(outs)


def highres_backward_nchw(guide, src, d_out, r, eps):
    """Returns (d_guide (B, Cg, H, W), d_src).  A 1-channel guide's gradient is
    the sum over its replicated copies."""
    c = src.shape[1]
    cg = guide.shape[1]
    dgs, dss = [], []
    for g, s, d in zip(nchw_to_hwc_list(guide), nchw_to_hwc_list(src), nchw_to_hwc_list(d_out)):
        if cg != c:
            g = np.repeat(g, c, axis=2)
        _, tape = forward_highres(g, s, r, eps)
        d_src, _, d_g = backward(tape, d)
        if cg != c:
            d_g = d_g.sum(axis=2, keepdims=True)
        dgs.append(d_g)
        dss.append(d_src)
    return hwc_list_to_nchw(dgs), hwc_list_to_nchw(dss)
