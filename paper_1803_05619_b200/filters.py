"""Linear operators of the layer on the GPU -- mirror of gf/filters.py.

``mean_filter`` / ``mean_filter_adjoint`` (gf/filters.py:96-116) and
``bilinear_resize`` / ``bilinear_resize_adjoint`` (gf/filters.py:134-188),
same names, arguments and exceptions, computed by the sm_100a kernels behind
the C ABI.  Inputs follow the conventions of ``_tensors`` (numpy HWC float64,
torch HWC, or torch NCHW on CUDA).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._tensors import as_img, dtype_code, ptr, restore, stream_ptr


def _check_radius(r) -> int:
    if isinstance(r, bool) or not isinstance(r, (int, np.integer)) or r < 0:
        raise ValueError(f"radius must be a non-negative integer, got {r!r}")
    return int(r)


def window_counts(height: int, width: int, r: int) -> np.ndarray:
    """Pixel count of each clamped window (gf/filters.py:82-93); host-side
    integer bookkeeping, shape (height, width, 1)."""
    r = _check_radius(r)
    ys, xs = np.arange(height), np.arange(width)
    ny = np.minimum(ys + r, height - 1) - np.maximum(ys - r, 0) + 1
    nx = np.minimum(xs + r, width - 1) - np.maximum(xs - r, 0) + 1
    return (ny[:, None] * nx[None, :]).astype(np.float64)[:, :, None]


def _mean_nchw(t: torch.Tensor, r: int, adjoint: bool = False) -> torch.Tensor:
    t = t.contiguous()
    B, C, h, w = t.shape
    out = torch.empty_like(t)
    lib = _lib.load()
    fn = lib.gf_mean_filter_adjoint if adjoint else lib.gf_mean_filter
    rc = fn(dtype_code(t), ptr(t), ptr(out), B * C, h, w, int(r), stream_ptr(t.device))
    _lib.check(rc, "mean_filter_adjoint" if adjoint else "mean_filter")
    return out


def _resize_nchw(t: torch.Tensor, out_h: int, out_w: int) -> torch.Tensor:
    t = t.contiguous()
    B, C, h, w = t.shape
    out = torch.empty((B, C, out_h, out_w), dtype=t.dtype, device=t.device)
    rc = _lib.load().gf_bilinear_resize(dtype_code(t), ptr(t), ptr(out), B * C, h, w, out_h,
                                        out_w, stream_ptr(t.device))
    _lib.check(rc, "bilinear_resize")
    return out


def mean_filter(t, r: int):
    """True mean over the clamped radius-r window around each pixel."""
    r = _check_radius(r)
    im = as_img(t, "tensor")
    return restore(_mean_nchw(im.t, r), im)


def mean_filter_adjoint(g, r: int):
    """Transpose of mean_filter: box_sum(g / N)."""
    r = _check_radius(r)
    im = as_img(g, "tensor")
    return restore(_mean_nchw(im.t, r, adjoint=True), im)


def bilinear_resize(t, out_h: int, out_w: int):
    """Resample to (out_h, out_w) with half-pixel centers, axis by axis."""
    if out_h < 1 or out_w < 1:
        raise ValueError(f"output dims must be >= 1, got ({out_h}, {out_w})")
    im = as_img(t, "tensor")
    return restore(_resize_nchw(im.t, int(out_h), int(out_w)), im)


def bilinear_resize_adjoint(g, in_h: int, in_w: int):
    """Exact transpose of bilinear_resize(., g_h, g_w) from (in_h, in_w)."""
    if in_h < 1 or in_w < 1:
        raise ValueError(f"input dims must be >= 1, got ({in_h}, {in_w})")
    im = as_img(g, "tensor")
    t = im.t
    B, C, gh, gw = t.shape
    out = torch.empty((B, C, int(in_h), int(in_w)), dtype=t.dtype, device=t.device)
    rc = _lib.load().gf_bilinear_resize_adjoint(dtype_code(t), ptr(t), ptr(out), B * C, gh, gw,
                                                int(in_h), int(in_w), stream_ptr(t.device))
    _lib.check(rc, "bilinear_resize_adjoint")
    return restore(out, im)
