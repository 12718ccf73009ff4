"""Boundary plumbing: validation and layout conversion for the Python mirror.

The reference passes one float64 HWC numpy image per call (gf/tensor.py:1-41).
This package accepts, for every image argument:

* a numpy ``(h, w, c)`` float64 array (reference convention): it is uploaded
  to the current CUDA device, computed in float64, and results come back as
  numpy float64 HWC arrays -- a literal drop-in for reference callers;
* a torch ``(h, w, c)`` CUDA tensor (float32 or float64): same convention on
  device;
* a torch ``(B, C, H, W)`` CUDA tensor (float32 or float64): the native
  batched layout of the kernels, no copies.

Arithmetic never happens here: tensors are only checked, permuted and handed
to the C ABI.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


@dataclass
class Img:
    t: torch.Tensor       # contiguous NCHW on CUDA
    kind: str             # "np_hwc" | "torch_hwc" | "torch_nchw"

    @property
    def shape(self):
        return tuple(self.t.shape)


def _cuda_device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1803_05619_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def as_img(t, name: str = "tensor", dtype=None, device=None) -> Img:
    """Validate (gf/tensor.py:27-41 semantics) and convert to NCHW CUDA."""
    if isinstance(t, np.ndarray):
        if t.ndim != 3:
            raise ValueError(f"{name}: expected a 3-d (h, w, c) array, got {t!r}")
        if min(t.shape) < 1:
            raise ValueError(f"{name}: all dimensions must be >= 1, got shape {t.shape}")
        if t.dtype != np.float64:
            raise ValueError(f"{name}: expected float64 data, got {t.dtype}")
        dev = device or _cuda_device()
        x = torch.from_numpy(np.ascontiguousarray(t)).to(dev, non_blocking=False)
        return Img(x.permute(2, 0, 1).unsqueeze(0).contiguous(), "np_hwc")
    if isinstance(t, torch.Tensor):
        if t.dim() not in (3, 4):
            raise ValueError(f"{name}: expected a 3-d (h, w, c) or 4-d (B, C, H, W) tensor, "
                             f"got shape {tuple(t.shape)}")
        if min(t.shape) < 1:
            raise ValueError(f"{name}: all dimensions must be >= 1, got shape {tuple(t.shape)}")
        if t.dtype not in (torch.float32, torch.float64):
            raise ValueError(f"{name}: expected float32 or float64 data, got {t.dtype}")
        if not t.is_cuda:
            raise ValueError(f"{name}: expected a CUDA tensor (no CPU fallback), got {t.device}")
        if t.dim() == 3:
            return Img(t.permute(2, 0, 1).unsqueeze(0).contiguous(), "torch_hwc")
        x = t.contiguous()
        if x.data_ptr() % 16:
            # e.g. a batch slice lr[1:] with odd C*h*w: the fused kernels use
            # 128-bit accesses, so hand them an aligned copy (the C ABI would
            # otherwise take the general kernels, which need a larger workspace)
            x = x.clone(memory_format=torch.contiguous_format)
        return Img(x, "torch_nchw")
    raise ValueError(f"{name}: expected a numpy array or torch tensor, got {type(t).__name__}")


def restore(x: torch.Tensor, like: Img):
    """NCHW result -> the caller's convention (mirrors ``like``)."""
    if like.kind == "torch_nchw":
        return x
    hwc = x[0].permute(1, 2, 0).contiguous()
    if like.kind == "torch_hwc":
        return hwc
    return hwc.cpu().numpy()


def dtype_code(t: torch.Tensor) -> int:
    return _lib.GF_F32 if t.dtype == torch.float32 else _lib.GF_F64


def ptr(t) -> int:
    return t.data_ptr() if t is not None else 0


def stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)


class Status:
    """Device status word (GF_STATUS_* bits) of one or more launches."""

    def __init__(self, device):
        self.buf = torch.zeros(1, dtype=torch.int32, device=device)

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()

    def bits(self) -> int:
        return int(self.buf.item()) & 0xFFFFFFFF

    def raise_if_set(self, what: str = "guided filter", inputs=()) -> None:
        """Reference exception order: input check, degenerate window, output.

        The fused kernels do not test inputs element by element; when a
        DEGENERATE or OUTPUT bit is set, the inputs are scanned on the device
        (gf_check_finite) so a non-finite input is reported as such, exactly
        as the reference's up-front validate() would (gf/guided.py:156-158).
        """
        from .guided import DegenerateWindowError

        b = self.bits()
        if b and not (b & _lib.STATUS_NONFINITE_INPUT) and inputs:
            lib = _lib.load()
            for t in inputs:
                rc = lib.gf_check_finite(dtype_code(t), t.data_ptr(), t.numel(), self.ptr,
                                         stream_ptr(t.device))
                _lib.check(rc, "check_finite")
            b = self.bits()
        if b & _lib.STATUS_NONFINITE_INPUT:
            raise ValueError(f"{what}: input contains non-finite values")
        if b & _lib.STATUS_DEGENERATE:
            raise DegenerateWindowError(
                "eps=0 requires positive guidance variance in every window")
        if b & _lib.STATUS_NONFINITE_OUTPUT:
            raise ValueError("guided filter produced non-finite output; increase eps")
