"""Host-image entry points: the reference's call shape (host arrays in, host
array out -- gf/guided.py:152 forward_joint, :198 forward_highres) over the
C ABI's pipelined host entries (gf_highres_fwd_host / gf_joint_fwd_host).

The batch streams through the GPU image by image: the copy-in of image b+1,
the kernel of image b and the copy-out of image b-1 overlap, so with
page-locked (pinned) host tensors a call costs about the PCIe time of the
whole batch in one direction, not copy-in + kernel + copy-out.

Inputs: CPU torch tensors or numpy arrays, NCHW (B, C, H, W) or one
reference-style HWC image (H, W, C); float32 or float64 (float32 is the
production path).  The result has the input's layout and container; pass
``out=`` (a CPU tensor of the output shape, ideally pinned) to reuse a buffer.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

from . import _lib
from .guided import DegenerateWindowError, GuidedFilterParams

_WS: dict = {}  # (host thread, device) -> cached device workspace (grown on demand)


def _workspace(nbytes: int, device) -> torch.Tensor:
    """One device workspace per (host thread, device).

    The C pipeline runs on its own per-thread streams and releases the GIL,
    so two threads must never share a buffer.  The block comes from torch's
    caching allocator on torch's current stream, which the library's streams
    do not wait on: synchronise that stream once when the block is
    (re)allocated, so no earlier torch work can still be using it.  The
    cached block stays referenced here, so it is never handed out again.
    """
    key = (threading.get_ident(), str(device))
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        torch.cuda.current_stream(device).synchronize()
        _WS[key] = ws
    return ws


def _host_nchw(x, what: str):
    """-> (contiguous CPU NCHW tensor, restore(out_tensor) -> user layout)."""
    is_np = isinstance(x, np.ndarray)
    t = torch.from_numpy(x) if is_np else x
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{what}: expected a numpy array or a CPU tensor")
    if t.device.type != "cpu":
        raise ValueError(f"{what}: host entry points take host (CPU) images")
    if t.dtype not in (torch.float32, torch.float64):
        raise ValueError(f"{what}: expected float32 or float64, got {t.dtype}")
    if t.dim() == 3:  # reference HWC image
        t4 = t.permute(2, 0, 1).unsqueeze(0).contiguous()

        def restore(o):
            o = o[0].permute(1, 2, 0).contiguous()
            return o.numpy() if is_np else o
    elif t.dim() == 4:
        t4 = t.contiguous()

        def restore(o):
            return o.numpy() if is_np else o
    else:
        raise ValueError(f"{what}: expected (H, W, C) or (B, C, H, W), got {tuple(t.shape)}")
    if min(t4.shape) < 1:
        raise ValueError(f"{what}: empty dimension in {tuple(t4.shape)}")
    return t4, restore


def _raise(bits: int, what: str, inputs) -> None:
    if not bits:
        return
    if not all(bool(torch.isfinite(t).all()) for t in inputs):
        raise ValueError(f"{what}: input contains non-finite values")
    if bits & _lib.STATUS_DEGENERATE:
        raise DegenerateWindowError(f"{what}: zero-variance window with eps == 0")
    raise ValueError(f"{what}: output contains non-finite values")


def _out_buffer(out, shape, like: torch.Tensor) -> torch.Tensor:
    if out is None:
        return torch.empty(shape, dtype=like.dtype, pin_memory=like.is_pinned())
    if not isinstance(out, torch.Tensor) or out.device.type != "cpu":
        raise ValueError("out: expected a CPU tensor")
    if tuple(out.shape) != tuple(shape) or out.dtype != like.dtype or not out.is_contiguous():
        raise ValueError(f"out: expected contiguous {like.dtype} {tuple(shape)}")
    return out


def forward_highres_host(guide, src, p: GuidedFilterParams, *, out=None, device=None,
                         check: bool = True):
    """Full-resolution filter of host images (gf/guided.py:198-233 semantics;
    a 1-channel guide is broadcast over the source channels)."""
    if not isinstance(p, GuidedFilterParams):
        raise ValueError(f"expected GuidedFilterParams, got {type(p).__name__}")
    g, _ = _host_nchw(guide, "guide")
    s, restore = _host_nchw(src, "src")
    if g.dtype != s.dtype:
        raise ValueError(f"dtype mismatch: {g.dtype} vs {s.dtype}")
    B, Cg, H, W = g.shape
    C = s.shape[1]
    if s.shape[0] != B or s.shape[2:] != g.shape[2:] or Cg not in (1, C):
        raise ValueError(f"guide/src shape mismatch: {tuple(g.shape)} vs {tuple(s.shape)}")
    device = torch.device(device) if device is not None else torch.device("cuda")
    lib = _lib.load()
    dt = _lib.GF_F32 if s.dtype == torch.float32 else _lib.GF_F64
    o = _out_buffer(out, s.shape, s)
    ws = _workspace(lib.gf_highres_host_workspace_bytes(dt, Cg, C, H, W, int(p.radius)), device)
    st = ctypes.c_uint32(0)
    with torch.cuda.device(device):
        rc = lib.gf_highres_fwd_host(dt, g.data_ptr(), s.data_ptr(), o.data_ptr(), B, Cg, C, H,
                                     W, int(p.radius), float(p.eps), ws.data_ptr(), ws.numel(),
                                     ctypes.addressof(st))
    _lib.check(rc, "forward_highres_host")
    if check:
        _raise(st.value, "forward_highres_host", (g, s))
    return restore(o)


def forward_joint_host(guide_lo, guide_hi, src_lo, p: GuidedFilterParams, *, out=None,
                       device=None, check: bool = True):
    """Fast joint-upsampling filter of host images (gf/guided.py:152-195)."""
    if not isinstance(p, GuidedFilterParams):
        raise ValueError(f"expected GuidedFilterParams, got {type(p).__name__}")
    lx, _ = _host_nchw(guide_lo, "guide_lo")
    hx, restore = _host_nchw(guide_hi, "guide_hi")
    ly, _ = _host_nchw(src_lo, "src_lo")
    if not (lx.dtype == hx.dtype == ly.dtype):
        raise ValueError("guide_lo, guide_hi and src_lo must share a dtype")
    if lx.shape != ly.shape:
        raise ValueError(f"guide_lo/src_lo shape mismatch: {tuple(lx.shape)} vs {tuple(ly.shape)}")
    B, C, h, w = lx.shape
    if hx.shape[0] != B or hx.shape[1] != C:
        raise ValueError(f"guide_hi shape {tuple(hx.shape)} does not match {tuple(lx.shape)}")
    H, W = hx.shape[2:]
    device = torch.device(device) if device is not None else torch.device("cuda")
    lib = _lib.load()
    dt = _lib.GF_F32 if lx.dtype == torch.float32 else _lib.GF_F64
    o = _out_buffer(out, hx.shape, hx)
    ws = _workspace(lib.gf_joint_host_workspace_bytes(dt, C, h, w, H, W, int(p.radius)), device)
    st = ctypes.c_uint32(0)
    with torch.cuda.device(device):
        rc = lib.gf_joint_fwd_host(dt, lx.data_ptr(), ly.data_ptr(), hx.data_ptr(), o.data_ptr(),
                                   B, C, h, w, H, W, int(p.radius), float(p.eps), ws.data_ptr(),
                                   ws.numel(), ctypes.addressof(st))
    _lib.check(rc, "forward_joint_host")
    if check:
        _raise(st.value, "forward_joint_host", (lx, hx, ly))
    return restore(o)


def forward_backward_joint_host(guide_lo, guide_hi, src_lo, d_out, p: GuidedFilterParams, *,
                                outs=None, device=None, check: bool = True):
    """Forward AND backward of the fast layer on host images: the values of
    ``out, tape = forward_joint(...)`` (gf/guided.py:152-195) and
    ``backward(tape, d_out)`` (gf/guided.py:267-283) in one pipelined pass
    (gf_joint_fwd_bwd_host).  Returns ``(out, GuidedFilterGrads)`` with host
    arrays in the inputs' layout.  ``outs`` = optional preallocated CPU
    tensors ``(out, d_lr_x, d_lr_y, d_hr_x)`` (NCHW, ideally pinned)."""
    from .guided import GuidedFilterGrads

    if not isinstance(p, GuidedFilterParams):
        raise ValueError(f"expected GuidedFilterParams, got {type(p).__name__}")
    lx, restore_lo = _host_nchw(guide_lo, "guide_lo")
    hx, restore = _host_nchw(guide_hi, "guide_hi")
    ly, _ = _host_nchw(src_lo, "src_lo")
    d, _ = _host_nchw(d_out, "d_out")
    if not (lx.dtype == hx.dtype == ly.dtype == d.dtype):
        raise ValueError("guide_lo, guide_hi, src_lo and d_out must share a dtype")
    if lx.shape != ly.shape:
        raise ValueError(f"guide_lo/src_lo shape mismatch: {tuple(lx.shape)} vs {tuple(ly.shape)}")
    B, C, h, w = lx.shape
    if hx.shape[0] != B or hx.shape[1] != C:
        raise ValueError(f"guide_hi shape {tuple(hx.shape)} does not match {tuple(lx.shape)}")
    if d.shape != hx.shape:
        raise ValueError(f"d_out shape {tuple(d.shape)} does not match {tuple(hx.shape)}")
    H, W = hx.shape[2:]
    device = torch.device(device) if device is not None else torch.device("cuda")
    lib = _lib.load()
    dt = _lib.GF_F32 if lx.dtype == torch.float32 else _lib.GF_F64
    if outs is None:
        outs = (None, None, None, None)
    o = _out_buffer(outs[0], hx.shape, hx)
    dlx = _out_buffer(outs[1], lx.shape, lx)
    dly = _out_buffer(outs[2], ly.shape, ly)
    dhx = _out_buffer(outs[3], hx.shape, hx)
    ws = _workspace(lib.gf_joint_fwd_bwd_host_workspace_bytes(dt, C, h, w, H, W, int(p.radius)),
                    device)
    st = ctypes.c_uint32(0)
    with torch.cuda.device(device):
        rc = lib.gf_joint_fwd_bwd_host(dt, lx.data_ptr(), ly.data_ptr(), hx.data_ptr(),
                                       d.data_ptr(), o.data_ptr(), dlx.data_ptr(), dly.data_ptr(),
                                       dhx.data_ptr(), B, C, h, w, H, W, int(p.radius),
                                       float(p.eps), ws.data_ptr(), ws.numel(),
                                       ctypes.addressof(st))
    _lib.check(rc, "forward_backward_joint_host")
    if check:
        _raise(st.value, "forward_backward_joint_host", (lx, hx, ly, d))
    grads = GuidedFilterGrads(d_src=restore_lo(dly), d_guide_lo=restore_lo(dlx),
                              d_guide_hi=restore(dhx))
    return restore(o), grads
