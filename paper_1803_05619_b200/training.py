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
from ._tensors import as_img, dtype_code, ptr, restore, stream_ptr, workspace
from .guidance import GuidanceNet
from .guided import GuidedFilterParams, backward, forward_joint


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


@dataclass
class StepResult:
    loss: torch.Tensor        # 0-d float64 device tensor
    out: torch.Tensor         # (B, C, H, W)
    dparams: torch.Tensor     # packed guidance-net gradient (summed over the batch)
    d_lr_x: torch.Tensor
    d_lr_y: torch.Tensor
    d_hr_x: torch.Tensor
    status_bits: list


def train_step(net: GuidanceNet, lr_x: torch.Tensor, hr_x: torch.Tensor, lr_y: torch.Tensor,
               target: torch.Tensor, p: GuidedFilterParams) -> StepResult:
    """One forward + backward of config 2 on NCHW CUDA tensors (no syncs)."""
    g_lo, t_lo = net.forward(lr_x, check=False)
    g_hi, t_hi = net.forward(hr_x, check=False)
    out, tape = forward_joint(g_lo, g_hi, lr_y, p, check=False)
    loss, d_out = mse_loss_device(out, target)
    grads = backward(tape, d_out, check=False)
    dparams = torch.empty(net.param_count(), dtype=hr_x.dtype, device=hr_x.device)
    d_lr_x, _ = net.backward(t_lo, grads.d_guide_lo, dparams=dparams, accumulate=False,
                             check=False)
    d_hr_x, _ = net.backward(t_hi, grads.d_guide_hi, dparams=dparams, accumulate=True,
                             check=False)
    return StepResult(loss, out, dparams, d_lr_x, grads.d_src, d_hr_x, [tape.status])
