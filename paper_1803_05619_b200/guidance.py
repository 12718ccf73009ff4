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


def _f64(v, device) -> torch.Tensor:
    return torch.as_tensor(np.asarray(v) if not isinstance(v, torch.Tensor) else v).to(
        device, torch.float64)


@dataclass
class LayerTape:
    """Input record of a standalone layer (ConvLayer / AdaptiveNorm): the
    backward recomputes what the reference's ConvTape / NormTape freeze."""

    x: Img


class ConvLayer:
    """2-d cross-correlation with dilation and same-size zero padding
    (gf/guidance.py:52-124) on the GPU (gf_conv2d_fwd / gf_conv2d_bwd).

    ``weight`` (out_ch, in_ch, k, k) and ``bias`` (out_ch) are float64
    device tensors -- for ``GuidanceNet.conv1`` / ``.conv2`` they are views
    into the net's packed parameter vector, so editing them in place (or
    ``load_parameters``) edits the net.  Same initialisation draw as the
    reference (xavier-uniform weight, zero bias)."""

    def __init__(self, in_ch: int, out_ch: int, kernel: int = 1, dilation: int = 1,
                 bias: bool = True, rng: np.random.Generator | None = None, *, device=None,
                 _weight: torch.Tensor | None = None, _bias: torch.Tensor | None = None):
        if kernel < 1 or kernel % 2 == 0:
            raise ValueError(f"kernel must be odd and >= 1, got {kernel}")
        if dilation < 1:
            raise ValueError(f"dilation must be >= 1, got {dilation}")
        self.in_ch, self.out_ch = int(in_ch), int(out_ch)
        self.kernel, self.dilation = int(kernel), int(dilation)
        self.pad = (kernel - 1) * dilation // 2
        if _weight is not None:
            self.device = _weight.device
            self.weight, self.bias = _weight, _bias
            return
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        w = (np.zeros((out_ch, in_ch, kernel, kernel)) if rng is None
             else xavier_uniform(rng, out_ch, in_ch, kernel))
        self.weight = _f64(w, self.device)
        self.bias = torch.zeros(out_ch, dtype=torch.float64, device=self.device) if bias else None

    def parameters(self) -> dict:
        out = {"weight": self.weight}
        if self.bias is not None:
            out["bias"] = self.bias
        return out

    def load_parameters(self, params: dict) -> None:
        """In place (views into a GuidanceNet stay views)."""
        self.weight.copy_(_f64(params["weight"], self.device).reshape(self.weight.shape))
        if self.bias is not None:
            self.bias.copy_(_f64(params["bias"], self.device).reshape(self.bias.shape))

    def forward(self, x, *, check: bool = True):
        im = as_img(x, "x", device=self.device)
        if im.shape[1] != self.in_ch:
            raise ValueError(f"expected {self.in_ch} input channels, got {im.shape[1]}")
        B, _, H, W = im.shape
        lib = _lib.load()
        dt = dtype_code(im.t)
        if check:
            _check_input(lib, im, "x")
        w = self.weight.to(im.t.dtype)
        b = self.bias.to(im.t.dtype) if self.bias is not None else None
        y = torch.empty((B, self.out_ch, H, W), dtype=im.t.dtype, device=self.device)
        rc = lib.gf_conv2d_fwd(dt, ptr(im.t), ptr(w), ptr(b) if b is not None else None, ptr(y),
                               B, self.in_ch, self.out_ch, H, W, self.kernel, self.dilation,
                               stream_ptr(self.device))
        _lib.check(rc, "ConvLayer.forward")
        return restore(y, im), LayerTape(im)

    def backward(self, tape: LayerTape, dy, *, check: bool = True):
        im = tape.x
        B, _, H, W = im.shape
        d = as_img(dy, "dy", device=self.device)
        if d.shape != (B, self.out_ch, H, W):
            raise ValueError(f"dy shape {d.shape} does not match output {(B, self.out_ch, H, W)}")
        lib = _lib.load()
        dt = dtype_code(im.t)
        if check:
            _check_input(lib, d, "dy")
        w = self.weight.to(im.t.dtype)
        dx = torch.empty_like(im.t)
        dw = torch.empty_like(w)
        db = (torch.empty(self.out_ch, dtype=im.t.dtype, device=self.device)
              if self.bias is not None else None)
        rc = lib.gf_conv2d_bwd(dt, ptr(im.t), ptr(w), ptr(d.t), ptr(dx), ptr(dw),
                               ptr(db) if db is not None else None, B, self.in_ch, self.out_ch,
                               H, W, self.kernel, self.dilation, stream_ptr(self.device))
        _lib.check(rc, "ConvLayer.backward")
        grads = {"weight": dw}
        if db is not None:
            grads["bias"] = db
        return restore(dx, im), _grads_like(grads, im)


class AdaptiveNorm:
    """gain * x + norm_gain * standardize(x), statistics per image and channel
    over space, variance floor 1e-5 (gf/guidance.py:134-173), on the GPU
    (gf_adaptive_norm_fwd / _bwd).  ``gain`` / ``norm_gain`` are (1,) float64
    device tensors (views into the packed parameters for GuidanceNet.norm)."""

    def __init__(self, gain: float = 1.0, norm_gain: float = 0.0, *, device=None,
                 _gain: torch.Tensor | None = None, _norm_gain: torch.Tensor | None = None):
        if _gain is not None:
            self.gain, self.norm_gain = _gain, _norm_gain
            self.device = _gain.device
            return
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        self.gain = torch.tensor([float(gain)], dtype=torch.float64, device=self.device)
        self.norm_gain = torch.tensor([float(norm_gain)], dtype=torch.float64,
                                      device=self.device)

    def parameters(self) -> dict:
        return {"gain": self.gain, "norm_gain": self.norm_gain}

    def load_parameters(self, params: dict) -> None:
        self.gain.copy_(_f64(params["gain"], self.device).reshape(1))
        self.norm_gain.copy_(_f64(params["norm_gain"], self.device).reshape(1))

    def forward(self, x, *, check: bool = True):
        im = as_img(x, "x", device=self.device)
        B, C, H, W = im.shape
        lib = _lib.load()
        dt = dtype_code(im.t)
        if check:
            _check_input(lib, im, "x")
        ga, ng = self.gain.to(im.t.dtype), self.norm_gain.to(im.t.dtype)
        y = torch.empty_like(im.t)
        ws = workspace(lib.gf_adaptive_norm_workspace_bytes(B, C), self.device)
        rc = lib.gf_adaptive_norm_fwd(dt, ptr(im.t), ptr(y), ptr(ga), ptr(ng), B, C, H, W,
                                      ptr(ws), ws.numel(), stream_ptr(self.device))
        _lib.check(rc, "AdaptiveNorm.forward")
        return restore(y, im), LayerTape(im)

    def backward(self, tape: LayerTape, dy, *, check: bool = True):
        im = tape.x
        B, C, H, W = im.shape
        d = as_img(dy, "dy", device=self.device)
        if d.shape != im.shape:
            raise ValueError(f"dy shape {d.shape} does not match input {im.shape}")
        lib = _lib.load()
        dt = dtype_code(im.t)
        if check:
            _check_input(lib, d, "dy")
        ga, ng = self.gain.to(im.t.dtype), self.norm_gain.to(im.t.dtype)
        dx = torch.empty_like(im.t)
        dg = torch.empty(1, dtype=im.t.dtype, device=self.device)
        dn = torch.empty(1, dtype=im.t.dtype, device=self.device)
        ws = workspace(lib.gf_adaptive_norm_workspace_bytes(B, C), self.device)
        rc = lib.gf_adaptive_norm_bwd(dt, ptr(im.t), ptr(d.t), ptr(dx), ptr(dg), ptr(dn), ptr(ga),
                                      ptr(ng), B, C, H, W, ptr(ws), ws.numel(),
                                      stream_ptr(self.device))
        _lib.check(rc, "AdaptiveNorm.backward")
        return restore(dx, im), _grads_like({"gain": dg, "norm_gain": dn}, im)


def _check_input(lib, im: Img, what: str) -> None:
    """validate(x, finite=True) (gf/tensor.py:39-40) -> ValueError."""
    st = Status(im.t.device)
    rc = lib.gf_check_finite(dtype_code(im.t), ptr(im.t), im.t.numel(), st.ptr,
                             stream_ptr(im.t.device))
    _lib.check(rc, "validate")
    if st.bits():
        raise ValueError(f"{what} contains non-finite values")


def _grads_like(grads: dict, im: Img) -> dict:
    if im.kind == "np_hwc":
        return {k: v.double().cpu().numpy() for k, v in grads.items()}
    return grads


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
        # the reference's layer objects (gf/guidance.py:191-194), as views
        # into the packed parameters: net.norm.norm_gain[:] = g edits the net
        v = self.parameters()
        self.conv1 = ConvLayer(in_ch, hidden, kernel=kernel, dilation=dilation, bias=False,
                               _weight=v["conv1.weight"])
        self.norm = AdaptiveNorm(_gain=v["norm.gain"], _norm_gain=v["norm.norm_gain"])
        self.conv2 = ConvLayer(hidden, out_ch, kernel=1, bias=True, _weight=v["conv2.weight"],
                               _bias=v["conv2.bias"])

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

