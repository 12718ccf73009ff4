"""torch.autograd / nn.Module front-ends with the (lr_x, lr_y, hr_x) order.

``FastGuidedFilter(r, eps)(lr_x, lr_y, hr_x)`` is the call north_star names:
it maps to ``forward_joint(guide_lo=lr_x, guide_hi=hr_x, src_lo=lr_y)``
(the argument order differs from the reference function).
``FullResGuidedFilter(r, eps)(guide, src)`` maps to ``forward_highres``.
Both are thin: forward and backward are single C-ABI calls, launched
asynchronously on the current stream (status words are checked lazily via
``.last_status``).
"""

from __future__ import annotations

import torch

from .guided import GuidedFilterParams, backward, forward_highres, forward_joint


class _JointFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, lr_x, lr_y, hr_x, params, holder):
        out, tape = forward_joint(lr_x, hr_x, lr_y, params, check=False)
        ctx.tape = tape
        holder.last_status = tape.status
        return out

    @staticmethod
    def backward(ctx, d_out):
        g = backward(ctx.tape, d_out.contiguous(), check=False)
        return g.d_guide_lo, g.d_src, g.d_guide_hi, None, None


class _HighresFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, guide, src, params, holder):
        out, tape = forward_highres(guide, src, params, check=False)
        ctx.tape = tape
        holder.last_status = tape.status
        return out

    @staticmethod
    def backward(ctx, d_out):
        g = backward(ctx.tape, d_out.contiguous(), check=False)
        return g.d_guide_hi, g.d_src, None, None


class FastGuidedFilter(torch.nn.Module):
    def __init__(self, r: int = 1, eps: float = 1e-8):
        super().__init__()
        self.params = GuidedFilterParams(r, eps)
        self.last_status = None

    def forward(self, lr_x, lr_y, hr_x):
        return _JointFn.apply(lr_x, lr_y, hr_x, self.params, self)


class FullResGuidedFilter(torch.nn.Module):
    def __init__(self, r: int = 1, eps: float = 1e-8):
        super().__init__()
        self.params = GuidedFilterParams(r, eps)
        self.last_status = None

    def forward(self, guide, src):
        return _HighresFn.apply(guide, src, self.params, self)
