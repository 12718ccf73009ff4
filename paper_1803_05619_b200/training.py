"""Config-2 training step on B200: guidance net on both resolutions, joint
guided filter, MSE, and the full backward -- the caller side of the layer in
gf/training.py:143-183 (GuidedUpsampler) with ``lr_y`` standing in for the
low-res core net output, exactly as BASELINE config 2 specifies.

``mse_loss`` mirrors gf/training.py:93-101 (for a batch it is the mean of
the per-image losses, and d_out carries the extra 1/B).  ``train_step``
returns the loss as a device tensor so a training loop never synchronises;
parameter gradients are accumulated into one packed buffer in the
reference's order (low-res call site first, then high-res,
gf/training.py:168-177), which is what the data-parallel allreduce sums.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from ._tensors import Status, as_img, dtype_code, ptr, restore, stream_ptr, workspace
from .guidance import GuidanceNet
from .guided import GuidedFilterGrads, GuidedFilterParams, backward, forward_joint


def affine_target(image):
    """Clipped affine tone curve, gf/training.py:265-267 (target generator)."""
    return (1.5 * image - 0.25).clamp(0.0, 1.0)


def mse_loss_device(out: torch.Tensor, target: torch.Tensor):
    """(loss as a 0-d float64 device tensor, d_out) for NCHW CUDA tensors."""
    if out.shape != target.shape:
        raise ValueError(f"shape mismatch: {tuple(out.shape)} vs {tuple(target.shape)}")
    if out.dtype != target.dtype:
        raise ValueError(f"dtype mismatch: {out.dtype} vs {target.dtype}")
    out = out.contiguous()
    target = target.contiguous()
    B, C, H, W = out.shape
    lib = _lib.load()
    d = torch.empty_like(out)
    loss = torch.empty((), dtype=torch.float64, device=out.device)
    ws = workspace(lib.gf_mse_workspace_bytes(B, C, H, W), out.device)
    rc = lib.gf_mse_loss(dtype_code(out), ptr(out), ptr(target), ptr(d), ptr(loss), B, C, H, W,
                         ptr(ws), ws.numel(), stream_ptr(out.device))
    _lib.check(rc, "mse_loss")
    return loss, d


def mse_loss(out, target):
    """Mean squared error and its gradient w.r.t. ``out`` (gf/training.py:93-101)."""
    o = as_img(out, "out")
    t = as_img(target, "target", device=o.t.device)
    if o.shape != t.shape:
        raise ValueError(f"shape mismatch: {o.shape} vs {t.shape}")
    loss, d = mse_loss_device(o.t, t.t.to(o.t.dtype))
    return float(loss.item()), restore(d, o)


def joint_mse_backward(lr_x: torch.Tensor, hr_x: torch.Tensor, lr_y: torch.Tensor,
                       target: torch.Tensor, p: GuidedFilterParams, *, check: bool = True):
    """Loss and gradients of ``mse_loss(forward_joint(lr_x, hr_x, lr_y, p), target)``.

    What gf/training.py:230-235 (``eval_and_grads``) takes from the forward,
    ``mse_loss`` and ``backward``, in one high-res pass for the fused shapes
    (``gf_joint_mse_bwd``): the output and d_out never reach HBM.  NCHW CUDA
    tensors; returns (loss as a 0-d float64 device tensor, GuidedFilterGrads,
    Status).  Raises like ``forward_joint`` when ``check``.
    """
    for name, t in (("lr_x", lr_x), ("hr_x", hr_x), ("lr_y", lr_y), ("target", target)):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dim() == 4):
            raise ValueError(f"{name}: expected a 4-d CUDA tensor")
    if lr_x.shape != lr_y.shape:
        raise ValueError(f"guide_lo/src_lo shape mismatch: {tuple(lr_x.shape)} vs "
                         f"{tuple(lr_y.shape)}")
    if target.shape != hr_x.shape:
        raise ValueError(f"shape mismatch: {tuple(hr_x.shape)} vs {tuple(target.shape)}")
    if hr_x.shape[:2] != lr_x.shape[:2]:
        raise ValueError(f"channel mismatch: guide_hi has {tuple(hr_x.shape[:2])}, guide_lo "
                         f"has {tuple(lr_x.shape[:2])}")
    if len({t.dtype for t in (lr_x, hr_x, lr_y, target)}) != 1:
        raise ValueError("dtype mismatch between the inputs")
    lr_x, hr_x, lr_y, target = (t.contiguous() for t in (lr_x, hr_x, lr_y, target))
    B, C, h, w = lr_x.shape
    H, W = hr_x.shape[2:]
    lib = _lib.load()
    dev = lr_x.device
    dt = dtype_code(lr_x)
    d_lr_x = torch.empty_like(lr_x)
    d_lr_y = torch.empty_like(lr_y)
    d_hr_x = torch.empty_like(hr_x)
    loss = torch.empty((), dtype=torch.float64, device=dev)
    status = Status(dev)
    ws = workspace(lib.gf_joint_mse_workspace_bytes(dt, B, C, h, w, H, W, p.radius), dev)
    rc = lib.gf_joint_mse_bwd(dt, ptr(lr_x), ptr(lr_y), ptr(hr_x), ptr(target), ptr(loss),
                              ptr(d_lr_x), ptr(d_lr_y), ptr(d_hr_x), B, C, h, w, H, W,
                              int(p.radius), float(p.eps), ptr(ws), ws.numel(), status.ptr,
                              stream_ptr(dev))
    _lib.check(rc, "joint_mse_backward")
    if check:
        status.raise_if_set("joint_mse_backward", (lr_x, hr_x, lr_y))
    return loss, GuidedFilterGrads(d_src=d_lr_y, d_guide_lo=d_lr_x, d_guide_hi=d_hr_x), status


@dataclass
class StepResult:
    loss: torch.Tensor        # 0-d float64 device tensor
    out: torch.Tensor         # (B, C, H, W), or None (fused step, return_out=False)
    dparams: torch.Tensor     # packed guidance-net gradient (summed over the batch)
    d_lr_x: torch.Tensor
    d_lr_y: torch.Tensor
    d_hr_x: torch.Tensor
    status_bits: list


def train_step(net: GuidanceNet, lr_x: torch.Tensor, hr_x: torch.Tensor, lr_y: torch.Tensor,
               target: torch.Tensor, p: GuidedFilterParams, *,
               return_out: bool = False) -> StepResult:
    """One forward + backward of config 2 on NCHW CUDA tensors (no syncs).

    A training step needs the loss and the gradients only (gf/training.py:
    230-235), so by default the filter, the loss and the filter backward run
    fused (``joint_mse_backward``) and ``out`` is None; ``return_out=True``
    runs forward_joint -> mse_loss -> backward and keeps the output.
    """
    g_lo, t_lo = net.forward(lr_x, check=False)
    g_hi, t_hi = net.forward(hr_x, check=False)
    if return_out:
        out, tape = forward_joint(g_lo, g_hi, lr_y, p, check=False)
        loss, d_out = mse_loss_device(out, target)
        grads = backward(tape, d_out, check=False)
        status = tape.status
    else:
        out = None
        loss, grads, status = joint_mse_backward(g_lo, g_hi, lr_y, target, p, check=False)
    dparams = torch.empty(net.param_count(), dtype=hr_x.dtype, device=hr_x.device)
    d_lr_x, _ = net.backward(t_lo, grads.d_guide_lo, dparams=dparams, accumulate=False,
                             check=False)
    d_hr_x, _ = net.backward(t_hi, grads.d_guide_hi, dparams=dparams, accumulate=True,
                             check=False)
    return StepResult(loss, out, dparams, d_lr_x, grads.d_src, d_hr_x, [status])
