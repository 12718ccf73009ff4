"""Differentiable guided filtering layer on B200 -- mirror of gf/guided.py.

Same names, argument order, meaning and exceptions as the reference
(``/root/reference/pkg/src/guidedfilter/guided.py``):

* ``forward_joint(guide_lo, guide_hi, src_lo, p) -> (out, tape)``
  (gf/guided.py:152-195): window statistics at low resolution, slope and
  intercept bilinearly upsampled (NOT re-smoothed) and applied to guide_hi.
* ``forward_highres(guide_hi, src_hi, p) -> (out, tape)``
  (gf/guided.py:198-233): statistics at full resolution, slope/intercept
  re-smoothed.  Extension: a 1-channel guide may drive a C-channel source
  (BASELINE config 1); its gradient is the sum over the C broadcast copies.
* ``backward(tape, d_out) -> GuidedFilterGrads`` (gf/guided.py:267-297).

All arithmetic runs in the sm_100a kernels of ``libgf_b200.so`` through the
C ABI (include/gf_b200.h); this module only validates, converts layouts and
maps status bits to exceptions.  Image arguments may be reference-style
float64 numpy HWC arrays, torch HWC CUDA tensors, or batched NCHW CUDA tensors
(see ``_tensors``).  By default every call reads the device status word back
(one 4-byte copy) so errors raise synchronously exactly like the reference;
pass ``check=False`` to keep the call fully asynchronous and inspect
``tape.status`` later.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._tensors import Img, Status, as_img, dtype_code, ptr, restore, stream_ptr, workspace

VARIANT_JOINT = "joint"
VARIANT_HIGHRES = "highres"


class DegenerateWindowError(ArithmeticError):
    """eps=0 requested but some window has no guidance variance (gf/guided.py:38-39)."""


@dataclass(frozen=True)
class GuidedFilterParams:
    """Window radius (moment-resolution pixels) and regularizer (gf/guided.py:42-53)."""

    radius: int = 1
    eps: float = 1e-8

    def __post_init__(self) -> None:
        if isinstance(self.radius, bool) or not isinstance(self.radius, (int, np.integer)) \
                or self.radius < 0:
            raise ValueError(f"radius must be a non-negative integer, got {self.radius!r}")
        if not np.isfinite(self.eps) or self.eps < 0.0:
            raise ValueError(f"eps must be finite and >= 0, got {self.eps!r}")


@dataclass(frozen=True)
class GuidedFilterGrads:
    """Gradients of dot(d_out, out) (gf/guided.py:82-92)."""

    d_src: object
    d_guide_lo: object
    d_guide_hi: object


@dataclass(eq=False)
class GuidedFilterTape:
    """Forward record (gf/guided.py:56-79).

    Keeps references to the inputs only; the moment fields the reference
    stores (mean_guide, mean_src, var_guide, cov_guide_src, slope, intercept,
    slope_hi) are recomputed on the GPU on first access, in the caller's
    convention, so the tape is O(inputs) in memory.
    """

    variant: str
    params: GuidedFilterParams
    _guide: Img
    _src: Img
    _guide_hi: Img
    _out_like: Img
    status: Status
    _cache: dict = field(default_factory=dict)
    _versions: tuple = ()
    row_origin: int = 0  # full-image low-res row of row 0 (row bands, sharding.py)
    # fast fp32 path: the low-res slope A of every cell, written by the forward
    # (gf_joint_fwd_tape) so the backward's high-res pass needs no window
    # moments -- the reference's tape keeps the slope too (gf/guided.py:181-194)
    _slope_lo: object = None

    def __post_init__(self) -> None:
        # autograd-style saved-tensor check: backward recomputes the moments
        # from the inputs (the reference freezes them in the tape), so an
        # in-place edit between forward and backward must not go unnoticed
        self._versions = self._input_versions()

    def _input_versions(self) -> tuple:
        return tuple(im.t._version for im in (self._guide, self._src, self._guide_hi))

    def check_unmodified(self) -> None:
        if self._input_versions() != self._versions:
            raise RuntimeError(
                "an input of the forward pass was modified in place after the forward; "
                "backward would use the new values (clone the input, or run forward again)")

    # reference field names ------------------------------------------------
    @property
    def guide(self):
        return restore(self._guide.t, self._guide)

    @property
    def src(self):
        return restore(self._src.t, self._src)

    @property
    def guide_hi(self):
        return restore(self._guide_hi.t, self._guide_hi)

    def _moments(self):
        self.check_unmodified()
        if "m" not in self._cache:
            self._cache["m"] = _tape_moments(self)
        return self._cache["m"]

    def _field(self, name):
        return restore(self._moments()[name], self._src)

    mean_guide = property(lambda self: self._field("mean_guide"))
    mean_src = property(lambda self: self._field("mean_src"))
    var_guide = property(lambda self: self._field("var_guide"))
    cov_guide_src = property(lambda self: self._field("cov_guide_src"))
    slope = property(lambda self: self._field("slope"))
    intercept = property(lambda self: self._field("intercept"))

    @property
    def slope_hi(self):
        return restore(self._moments()["slope_hi"], self._out_like)


def _stream(img: Img):
    return stream_ptr(img.t.device)


def _same_dtype(*imgs: Img):
    dt = imgs[0].t.dtype
    for im in imgs[1:]:
        if im.t.dtype != dt:
            raise ValueError(f"dtype mismatch: {dt} vs {im.t.dtype}")
    return dt


def forward_joint(guide_lo, guide_hi, src_lo, p: GuidedFilterParams, *, check: bool = True,
                  row_origin: int = 0, full_rows: int | None = None):
    """Joint upsampling: regress src on guide at low res, apply at high res.

    ``row_origin`` (extension, multi-GPU row bands): the full image's low-res
    row index of the inputs' first row.  It changes no value the reference
    defines; it makes the backward cut its row pieces at full-image rows so a
    band's gradients are bitwise those of the whole image (sharding.py).
    ``full_rows`` (with it): the full image's low-res height, so the band takes
    the kernel path (one- or two-kernel forward) the whole image would.
    """
    if isinstance(row_origin, bool) or not isinstance(row_origin, (int, np.integer)) \
            or row_origin < 0:
        raise ValueError(f"row_origin must be a non-negative integer, got {row_origin!r}")
    if not isinstance(p, GuidedFilterParams):
        raise ValueError(f"expected GuidedFilterParams, got {type(p).__name__}")
    gl = as_img(guide_lo, "guide_lo")
    gh = as_img(guide_hi, "guide_hi", device=gl.t.device)
    sl = as_img(src_lo, "src_lo", device=gl.t.device)
    _same_dtype(gl, gh, sl)
    # gf/guided.py:159-168
    if gl.shape != sl.shape:
        raise ValueError(f"guide_lo/src_lo shape mismatch: {gl.shape} vs {sl.shape}")
    if gh.shape[1] != gl.shape[1] or gh.shape[0] != gl.shape[0]:
        raise ValueError(f"channel mismatch: guide_hi has {gh.shape[:2]}, guide_lo has "
                         f"{gl.shape[:2]}")
    if gh.shape[2] < gl.shape[2] or gh.shape[3] < gl.shape[3]:
        raise ValueError(f"guide_hi dims {gh.shape[2:]} smaller than guide_lo {gl.shape[2:]}")
    B, C, h, w = gl.shape
    H, W = gh.shape[2:]
    lib = _lib.load()
    dev = gl.t.device
    dt = dtype_code(gl.t)
    out = torch.empty_like(gh.t)
    status = Status(dev)
    slope = None
    mode = 0
    if full_rows is not None:
        if isinstance(full_rows, bool) or not isinstance(full_rows, (int, np.integer)) \
                or full_rows < h:
            raise ValueError(f"full_rows must be an integer >= the band's rows, got {full_rows!r}")
        full_elems = B * C * (int(full_rows) * H // h) * W
        mode = 2 if full_elems >= lib.gf_joint_split_threshold() else 1
    mode_old = lib.gf_joint_fwd_mode(mode) if mode else 0
    try:
        if lib.gf_joint_is_fused(dt, B, C, h, w, H, W, p.radius) and not any(
                t.data_ptr() % 16 for t in (gl.t, sl.t, gh.t, out)):
            slope = torch.empty_like(gl.t)
            ws = workspace(lib.gf_joint_workspace_bytes(dt, B, C, h, w, H, W, p.radius), dev)
            rc = lib.gf_joint_fwd_tape(dt, ptr(gl.t), ptr(sl.t), ptr(gh.t), ptr(out), ptr(slope), B,
                                       C, h, w, H, W, int(p.radius), float(p.eps), ptr(ws),
                                       ws.numel(), status.ptr, _stream(gl))
        else:
            nbytes = lib.gf_joint_workspace_bytes(dt, B, C, h, w, H, W, p.radius)
            ws = workspace(nbytes, dev)
            rc = lib.gf_joint_fwd(dt, ptr(gl.t), ptr(sl.t), ptr(gh.t), ptr(out), B, C, h, w, H, W,
                                  int(p.radius), float(p.eps), ptr(ws), ws.numel(), status.ptr,
                                  _stream(gl))
    finally:
        if mode:
            lib.gf_joint_fwd_mode(mode_old)
    _lib.check(rc, "forward_joint")
    if check:
        status.raise_if_set("forward_joint", (gl.t, gh.t, sl.t))
    tape = GuidedFilterTape(VARIANT_JOINT, p, gl, sl, gh, gh, status, row_origin=int(row_origin),
                            _slope_lo=slope)
    return restore(out, gh), tape


def forward_highres(guide_hi, src_hi, p: GuidedFilterParams, *, check: bool = True):
    """Full-resolution refinement: moments at full res, coefficients re-smoothed."""
    if not isinstance(p, GuidedFilterParams):
        raise ValueError(f"expected GuidedFilterParams, got {type(p).__name__}")
    g = as_img(guide_hi, "guide_hi")
    s = as_img(src_hi, "src_hi", device=g.t.device)
    _same_dtype(g, s)
    if g.shape != s.shape and not (g.shape[1] == 1 and g.shape[0] == s.shape[0]
                                   and g.shape[2:] == s.shape[2:]):
        raise ValueError(f"guide/src shape mismatch: {g.shape} vs {s.shape}")
    B, Cg, H, W = g.shape
    C = s.shape[1]
    lib = _lib.load()
    dev = g.t.device
    dt = dtype_code(g.t)
    out = torch.empty_like(s.t)
    status = Status(dev)
    # the fused forward needs no workspace; the general kernels do
    fused = lib.gf_highres_fwd_is_fused(dt, B, Cg, C, H, W, p.radius) and not any(
        t.data_ptr() % 16 for t in (g.t, s.t, out))
    nbytes = 0 if fused else lib.gf_highres_workspace_bytes(dt, B, Cg, C, H, W, p.radius)
    ws = workspace(nbytes, dev)
    rc = lib.gf_highres_fwd(dt, ptr(g.t), ptr(s.t), ptr(out), B, Cg, C, H, W, int(p.radius),
                            float(p.eps), ptr(ws), ws.numel(), status.ptr, _stream(g))
    _lib.check(rc, "forward_highres")
    if check:
        status.raise_if_set("forward_highres", (g.t, s.t))
    tape = GuidedFilterTape(VARIANT_HIGHRES, p, g, s, g, s, status)
    return restore(out, s), tape


def backward(tape: GuidedFilterTape, d_out, *, check: bool = True) -> GuidedFilterGrads:
    """Gradients of dot(d_out, out) w.r.t. the forward inputs (gf/guided.py:267-297)."""
    like = tape._out_like
    tape.check_unmodified()
    d = as_img(d_out, "d_out", device=like.t.device)
    if d.shape != like.shape:
        raise ValueError(f"d_out shape {d.shape} does not match output shape {like.shape}")
    if d.t.dtype != like.t.dtype:
        raise ValueError(f"d_out dtype {d.t.dtype} does not match {like.t.dtype}")
    lib = _lib.load()
    p = tape.params
    dev = like.t.device
    dt = dtype_code(like.t)
    status = Status(dev)
    if tape.variant == VARIANT_JOINT:
        gl, sl, gh = tape._guide, tape._src, tape._guide_hi
        B, C, h, w = gl.shape
        H, W = gh.shape[2:]
        d_lr_x = torch.empty_like(gl.t)
        d_lr_y = torch.empty_like(sl.t)
        d_hr_x = torch.empty_like(gh.t)
        ws = workspace(lib.gf_joint_workspace_bytes(dt, B, C, h, w, H, W, p.radius), dev)
        if tape._slope_lo is not None and not any(
                t.data_ptr() % 16 for t in (d.t, d_lr_x, d_lr_y, d_hr_x)):
            rc = lib.gf_joint_bwd_tape(dt, ptr(gl.t), ptr(sl.t), ptr(gh.t), ptr(tape._slope_lo),
                                       ptr(d.t), ptr(d_lr_x), ptr(d_lr_y), ptr(d_hr_x), B, C, h,
                                       w, H, W, int(p.radius), float(p.eps), tape.row_origin,
                                       ptr(ws), ws.numel(), status.ptr, _stream(gl))
        else:
            rc = lib.gf_joint_bwd_band(dt, ptr(gl.t), ptr(sl.t), ptr(gh.t), ptr(d.t),
                                       ptr(d_lr_x), ptr(d_lr_y), ptr(d_hr_x), B, C, h, w, H, W,
                                       int(p.radius), float(p.eps), tape.row_origin, ptr(ws),
                                       ws.numel(), status.ptr, _stream(gl))
        _lib.check(rc, "backward")
        if check:
            status.raise_if_set("backward")
        return GuidedFilterGrads(d_src=restore(d_lr_y, sl), d_guide_lo=restore(d_lr_x, gl),
                                 d_guide_hi=restore(d_hr_x, gh))
    if tape.variant == VARIANT_HIGHRES:
        g, s = tape._guide, tape._src
        B, Cg, H, W = g.shape
        C = s.shape[1]
        d_g = torch.empty_like(g.t)
        d_s = torch.empty_like(s.t)
        ws = workspace(lib.gf_highres_workspace_bytes(dt, B, Cg, C, H, W, p.radius), dev)
        rc = lib.gf_highres_bwd(dt, ptr(g.t), ptr(s.t), ptr(d.t), ptr(d_g), ptr(d_s), B, Cg, C,
                                H, W, int(p.radius), float(p.eps), ptr(ws), ws.numel(),
                                status.ptr, _stream(g))
        _lib.check(rc, "backward")
        if check:
            status.raise_if_set("backward")
        return GuidedFilterGrads(d_src=restore(d_s, s), d_guide_lo=None,
                                 d_guide_hi=restore(d_g, g))
    raise ValueError(f"unknown tape variant {tape.variant!r}")


def _tape_moments(tape: GuidedFilterTape) -> dict:
    """Reference tape fields (gf/guided.py:136-149, :172, :210) on demand."""
    from .filters import _mean_nchw, _resize_nchw

    r, eps = tape.params.radius, tape.params.eps
    g, s = tape._guide.t, tape._src.t
    if g.shape[1] != s.shape[1]:
        g = g.expand(-1, s.shape[1], -1, -1).contiguous()
    mg = _mean_nchw(g, r)
    ms = _mean_nchw(s, r)
    var = _mean_nchw(g * g, r) - mg * mg
    cov = _mean_nchw(g * s, r) - mg * ms
    slope = cov / (var + eps)
    intercept = ms - slope * mg
    if tape.variant == VARIANT_JOINT:
        H, W = tape._guide_hi.shape[2:]
        slope_hi = _resize_nchw(slope, H, W)
    else:
        slope_hi = _mean_nchw(slope, r)
    return dict(mean_guide=mg, mean_src=ms, var_guide=var, cov_guide_src=cov, slope=slope,
                intercept=intercept, slope_hi=slope_hi)
