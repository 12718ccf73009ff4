"""Trainable 1x1 guidance transform F on B200 -- mirror of gf/guidance.py.

``GuidanceNet(in_ch, out_ch, hidden, kernel=1, rng=...)`` with the
reference's parameter names, shapes, initialisation draw order
(gf/guidance.py:29-33, :71-74, :191-194: conv1 weight then conv2 weight,
xavier-uniform; AdaptiveNorm gain=1, norm_gain=0; conv2 bias 0), forward
(gf/guidance.py:209-214) and backward (gf/guidance.py:216-224).  The whole
net runs in the sm_100a kernels behind ``gn_forward`` / ``gn_backward``.

The 1x1 net (BASELINE config 2: 3 -> 15 -> 3) runs the gn_* kernels (a
fused fp32 path for the small hidden widths); ``kernel > 1`` (odd, with
``dilation``, the reference's low-res core net C_l, gf/training.py:186-207)
runs the gnk_* kernels.  ``FixedChannelMeanGuidance`` mirrors
gf/guidance.py:227-255.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._tensors import Img, Status, as_img, dtype_code, ptr, restore, stream_ptr, workspace

LEAKY_SLOPE = 0.2
NORM_VAR_FLOOR = 1e-5


def xavier_uniform(rng: np.random.Generator, out_ch: int, in_ch: int, kernel: int) -> np.ndarray:
    """Same draw as gf/guidance.py:29-33 (so seeded nets match the reference)."""
    fan_in = in_ch * kernel * kernel
    fan_out = out_ch * kernel * kernel
    limit = np.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-limit, limit, (out_ch, in_ch, kernel, kernel))


@dataclass
class GuidanceTape:
    x: Img
    # the forward's workspace (per-image statistics and folded AdaptiveNorm
    # constants) when the fused fp32 kernels ran, and the parameter version
    # it was computed with; backward reuses it while the parameters are
    # unchanged
    ws: torch.Tensor | None = None
    ws_key: tuple | None = None


class GuidanceNet:
    """conv(1x1, no bias) -> adaptive norm -> leaky ReLU -> 1x1 conv with bias."""

    def __init__(self, in_ch: int, out_ch: int, hidden: int = 64, kernel: int = 1,
                 dilation: int = 1, rng: np.random.Generator | None = None, *, device=None):
        if kernel < 1 or kernel % 2 == 0:
            raise ValueError(f"kernel must be odd and >= 1, got {kernel}")
        if dilation < 1:
            raise ValueError(f"dilation must be >= 1, got {dilation}")
        self.in_ch, self.out_ch, self.hidden = int(in_ch), int(out_ch), int(hidden)
        self.kernel, self.dilation = int(kernel), int(dilation)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        if rng is None:
            w1 = np.zeros((hidden, in_ch, kernel, kernel))
            w2 = np.zeros((out_ch, hidden, 1, 1))
        else:
            w1 = xavier_uniform(rng, hidden, in_ch, kernel)
            w2 = xavier_uniform(rng, out_ch, hidden, 1)
        self.flat = torch.zeros(self.param_count(), dtype=torch.float64, device=self.device)
        self.load_parameters({
            "conv1.weight": w1, "norm.gain": np.array([1.0]), "norm.norm_gain": np.array([0.0]),
            "conv2.weight": w2, "conv2.bias": np.zeros(out_ch)})

    # packed layout (include/gf_b200.h): w1, gain, norm_gain, w2, b2
    def param_count(self) -> int:
        k2 = self.kernel * self.kernel
        return self.hidden * self.in_ch * k2 + 2 + self.out_ch * self.hidden + self.out_ch

    def _slices(self):
        k = self.kernel
        a = self.hidden * self.in_ch * k * k
        b = a + 2 + self.out_ch * self.hidden
        return {
            "conv1.weight": (slice(0, a), (self.hidden, self.in_ch, k, k)),
            "norm.gain": (slice(a, a + 1), (1,)),
            "norm.norm_gain": (slice(a + 1, a + 2), (1,)),
            "conv2.weight": (slice(a + 2, b), (self.out_ch, self.hidden, 1, 1)),
            "conv2.bias": (slice(b, b + self.out_ch), (self.out_ch,)),
        }

    def unpack(self, flat) -> dict:
        out = {}
        for k, (sl, shape) in self._slices().items():
            v = flat[sl].reshape(shape)
            out[k] = v
        return out

    def parameters(self) -> dict:
        """name -> float64 device tensor view (reference names and shapes)."""
        return self.unpack(self.flat)

    def load_parameters(self, params: dict) -> None:
        for k, (sl, shape) in self._slices().items():
            v = params[k]
            v = torch.as_tensor(np.asarray(v) if not isinstance(v, torch.Tensor) else v)
            self.flat[sl] = v.to(self.device, torch.float64).reshape(-1)
        self._cast = {}

    def _params_as(self, dtype):
        """Packed parameters in the compute dtype, cast once per load."""
        if dtype == torch.float64:
            return self.flat
        cache = self.__dict__.setdefault("_cast", {})
        key = (dtype, self.flat._version)  # in-place edits of parameters() bump it
        if key not in cache:
            cache.clear()
            cache[key] = self.flat.to(dtype)
        return cache[key]

    def _check_x(self, im: Img, n_ch: int, what: str):
        if im.shape[1] != n_ch:
            raise ValueError(f"expected {n_ch} {what} channels, got {im.shape[1]}")

    def forward(self, x, *, check: bool = True):
        im = as_img(x, "x", device=self.device)
        self._check_x(im, self.in_ch, "input")
        B, _, H, W = im.shape
        lib = _lib.load()
        dt = dtype_code(im.t)
        params = self._params_as(im.t.dtype)
        y = torch.empty((B, self.out_ch, H, W), dtype=im.t.dtype, device=self.device)
        status = Status(self.device)
        tape = GuidanceTape(x=im)
        if self.kernel == 1:
            ws = workspace(lib.gn_workspace_bytes(dt, B, self.in_ch, self.out_ch, self.hidden, H,
                                                  W), self.device)
            rc = lib.gn_forward(dt, ptr(im.t), ptr(y), ptr(params), B, self.in_ch, self.out_ch,
                                self.hidden, H, W, ptr(ws), ws.numel(), status.ptr,
                                stream_ptr(self.device))
            if (lib.gn_is_fused(dt, self.in_ch, self.out_ch, self.hidden, H, W)
                    and ptr(im.t) % 16 == 0 and ptr(y) % 16 == 0):
                tape.ws, tape.ws_key = ws, self._ws_key(im.t)
        else:
            ws = workspace(lib.gnk_workspace_bytes(dt, B, self.in_ch, self.out_ch, self.hidden,
                                                   self.kernel, H, W), self.device)
            rc = lib.gnk_forward(dt, ptr(im.t), ptr(y), ptr(params), B, self.in_ch, self.out_ch,
                                 self.hidden, self.kernel, self.dilation, H, W, ptr(ws),
                                 ws.numel(), status.ptr, stream_ptr(self.device))
        _lib.check(rc, "GuidanceNet.forward")
        if check:
            status.raise_if_set("GuidanceNet.forward")
        return restore(y, im), tape

    def _ws_key(self, x: torch.Tensor):
        return (self.flat._version, x.data_ptr(), x._version, tuple(x.shape), x.dtype)

    def backward(self, tape: GuidanceTape, dy, *, dparams: torch.Tensor | None = None,
                 accumulate: bool = False, check: bool = True):
        """Returns (dx, grads).  With ``dparams`` (a packed tensor of the
        input dtype) the parameter gradient is written / accumulated there
        and ``grads`` are views into it."""
        im = tape.x
        d = as_img(dy, "dy", device=self.device)
        B, _, H, W = im.shape
        if d.shape != (B, self.out_ch, H, W):
            raise ValueError(f"dy shape {d.shape} does not match output {(B, self.out_ch, H, W)}")
        lib = _lib.load()
        dt = dtype_code(im.t)
        params = self._params_as(im.t.dtype)
        dx = torch.empty_like(im.t)
        if dparams is None:
            dparams = torch.zeros(self.param_count(), dtype=im.t.dtype, device=self.device)
        status = Status(self.device)
        if self.kernel == 1:
            # the forward's statistics are reused while x and the parameters
            # are unchanged (gn_backward_reuse), else recomputed
            reuse = tape.ws is not None and tape.ws_key == self._ws_key(im.t)
            ws = tape.ws if reuse else workspace(
                lib.gn_workspace_bytes(dt, B, self.in_ch, self.out_ch, self.hidden, H, W),
                self.device)
            fn = lib.gn_backward_reuse if reuse else lib.gn_backward
            rc = fn(dt, ptr(im.t), ptr(d.t), ptr(dx), ptr(dparams), int(accumulate),
                    ptr(params), B, self.in_ch, self.out_ch, self.hidden, H, W,
                    ptr(ws), ws.numel(), status.ptr, stream_ptr(self.device))
        else:
            ws = workspace(lib.gnk_workspace_bytes(dt, B, self.in_ch, self.out_ch, self.hidden,
                                                   self.kernel, H, W), self.device)
            rc = lib.gnk_backward(dt, ptr(im.t), ptr(d.t), ptr(dx), ptr(dparams),
                                  int(accumulate), ptr(params), B, self.in_ch, self.out_ch,
                                  self.hidden, self.kernel, self.dilation, H, W, ptr(ws),
                                  ws.numel(), status.ptr, stream_ptr(self.device))
        _lib.check(rc, "GuidanceNet.backward")
        if check:
            status.raise_if_set("GuidanceNet.backward")
        grads = self.unpack(dparams)
        if im.kind == "np_hwc":
            grads = {k: v.double().cpu().numpy() for k, v in grads.items()}
        return restore(dx, im), grads


class FixedChannelMeanGuidance:
    """Parameter-free guidance: channel mean of the input, replicated
    (gf/guidance.py:227-255).  Same forward/backward surface as GuidanceNet."""

    def __init__(self, in_ch: int, out_ch: int, *, device=None):
        self.in_ch, self.out_ch = int(in_ch), int(out_ch)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)

    def param_count(self) -> int:
        return 0

    def parameters(self) -> dict:
        return {}

    def load_parameters(self, params: dict) -> None:
        if params:
            raise ValueError("fixed guidance has no parameters")

    def forward(self, x, *, check: bool = True):
        im = as_img(x, "x", device=self.device)
        if im.shape[1] != self.in_ch:
            raise ValueError(f"expected {self.in_ch} input channels, got {im.shape[1]}")
        B, _, H, W = im.shape
        y = torch.empty((B, self.out_ch, H, W), dtype=im.t.dtype, device=self.device)
        lib = _lib.load()
        rc = lib.gf_channel_mean(dtype_code(im.t), ptr(im.t), ptr(y), B, self.in_ch, self.out_ch,
                                 H, W, stream_ptr(self.device))
        _lib.check(rc, "FixedChannelMeanGuidance.forward")
        return restore(y, im), GuidanceTape(x=im)

    def backward(self, tape: GuidanceTape, dy, *, dparams=None, accumulate: bool = False,
                 check: bool = True):
        d = as_img(dy, "dy", device=self.device)
        B, _, H, W = tape.x.shape
        if d.shape != (B, self.out_ch, H, W):
            raise ValueError(f"dy shape {d.shape} does not match output {(B, self.out_ch, H, W)}")
        dx = torch.empty_like(tape.x.t)
        lib = _lib.load()
        rc = lib.gf_channel_mean_adjoint(dtype_code(d.t), ptr(d.t), ptr(dx), B, self.in_ch,
                                         self.out_ch, H, W, stream_ptr(self.device))
        _lib.check(rc, "FixedChannelMeanGuidance.backward")
        return restore(dx, tape.x), {}

