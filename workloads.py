"""Seeded synthetic inputs for the BASELINE.json configurations.

Test / bench infrastructure (not product code).  The paper's datasets are not
available offline, so every configuration is driven by seeded synthetic data
with the shapes, sizes and value distributions BASELINE.json states.  All
generators use a ``torch.Generator`` seeded explicitly and build NCHW float32
tensors on the requested device; tests feed the same tensors (as float64
numpy) to the CPU oracle.

Ambiguities in BASELINE.json are resolved here and restated in DESIGN.md:
  * the 5x5 Gaussian uses sigma = 1.0 with replicate borders;
  * lr_y's noise is N(0, 0.01) (sigma = 0.01);
  * the per-image 3x3 colour matrix is 0.6*I + 0.4*U[0,1]^(CxC), rows
    normalised to sum 1;
  * config 1's per-channel signal is a_c*guide + b_c, a_c ~ U[0.5, 1.5],
    b_c ~ U[-0.2, 0.2], plus N(0, 0.1) noise, clipped to [0, 1].
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F


def _gen(seed: int, device="cpu") -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def _gauss5(x: torch.Tensor, sigma: float = 1.0) -> torch.Tensor:
    k = torch.tensor([math.exp(-(i * i) / (2 * sigma * sigma)) for i in range(-2, 3)],
                     dtype=x.dtype, device=x.device)
    k = k / k.sum()
    b, c, h, w = x.shape
    y = x.reshape(b * c, 1, h, w)
    y = F.pad(y, (2, 2, 0, 0), mode="replicate")
    y = F.conv2d(y, k.view(1, 1, 1, 5))
    y = F.pad(y, (0, 0, 2, 2), mode="replicate")
    y = F.conv2d(y, k.view(1, 1, 5, 1))
    return y.reshape(b, c, h, w)


def smooth_image(batch, channels, height, width, seed, device="cpu"):
    """hr_x of config 0: U[0,1] -> 5x5 Gaussian -> + U[-0.05, 0.05] -> clip."""
    g = _gen(seed, device)
    x = torch.rand(batch, channels, height, width, generator=g, device=device)
    x = _gauss5(x)
    x = x + (torch.rand(x.shape, generator=g, device=device) - 0.5) * 0.1
    return x.clamp_(0.0, 1.0).contiguous()


def joint_inputs(batch, channels, hr_h, hr_w, factor=4, seed=0, device="cpu"):
    """Config 0/2/3/4 inputs: (lr_x, lr_y, hr_x), float32 NCHW.

    lr_x is the factor x factor box-downsample of hr_x; lr_y is a per-image
    colour matrix applied to lr_x, gamma 0.7, plus N(0, 0.01), clipped.
    """
    hr_x = smooth_image(batch, channels, hr_h, hr_w, seed, device)
    lr_x = F.avg_pool2d(hr_x, factor, factor)
    g = _gen(seed + 7919, device)
    eye = torch.eye(channels, device=device)
    m = 0.6 * eye + 0.4 * torch.rand(batch, channels, channels, generator=g, device=device)
    m = m / m.sum(dim=2, keepdim=True)
    y = torch.einsum("bij,bjhw->bihw", m, lr_x).clamp(0.0, 1.0).pow(0.7)
    y = y + 0.01 * torch.randn(y.shape, generator=g, device=device)
    lr_y = y.clamp_(0.0, 1.0).contiguous()
    return lr_x.contiguous(), lr_y, hr_x


def voronoi_guide(batch, height, width, seeds=64, seed=0, device="cpu"):
    """Config 1 guide: piecewise-constant Voronoi cells (U[0,1] values) plus
    N(0, 0.02), clipped; shape (B, 1, H, W)."""
    g = _gen(seed, device)
    out = torch.empty(batch, 1, height, width, device=device)
    ys = torch.arange(height, device=device, dtype=torch.float32).view(height, 1)
    xs = torch.arange(width, device=device, dtype=torch.float32).view(1, width)
    for n in range(batch):
        py = torch.rand(seeds, generator=g, device=device) * height
        px = torch.rand(seeds, generator=g, device=device) * width
        val = torch.rand(seeds, generator=g, device=device)
        best = torch.full((height, width), float("inf"), device=device)
        lab = torch.zeros((height, width), device=device)
        for s in range(seeds):
            d = (ys - py[s]) ** 2 + (xs - px[s]) ** 2
            closer = d < best
            best = torch.where(closer, d, best)
            lab = torch.where(closer, val[s], lab)
        out[n, 0] = lab
    out = out + 0.02 * torch.randn(out.shape, generator=g, device=device)
    return out.clamp_(0.0, 1.0).contiguous()


def highres_inputs(batch, channels, height, width, seed=0, device="cpu", guide_channels=1):
    """Config 1 inputs: (guide (B, Cg, H, W), src (B, C, H, W)), float32."""
    guide = voronoi_guide(batch, height, width, seed=seed, device=device)
    if guide_channels != 1:
        guide = guide.repeat(1, guide_channels, 1, 1).contiguous()
    g = _gen(seed + 104729, device)
    a = 0.5 + torch.rand(batch, channels, 1, 1, generator=g, device=device)
    b = (torch.rand(batch, channels, 1, 1, generator=g, device=device) - 0.5) * 0.4
    base = guide[:, :1] if guide_channels == 1 else guide
    src = a * base + b + 0.1 * torch.randn(batch, channels, height, width, generator=g,
                                           device=device)
    return guide, src.clamp_(0.0, 1.0).contiguous()


def affine_target(image: torch.Tensor) -> torch.Tensor:
    """gf/training.py:265-267: clip(1.5*x - 0.25, 0, 1)."""
    return (1.5 * image - 0.25).clamp(0.0, 1.0)


# BASELINE.json configs (full sizes); bench and the large parity tests use these.
CONFIGS = {
    "cfg0": dict(kind="joint_fwd", batch=1, channels=3, hr=1024, factor=4, r=1, eps=1e-8),
    "cfg1": dict(kind="highres_fwd", batch=4, channels=3, hr=2048, r=8, eps=1e-2),
    "cfg2": dict(kind="train_step", batch=8, channels=3, hr=2048, factor=4, r=1, eps=1e-8,
                 hidden=15),
    "cfg3": dict(kind="joint_fwd", batch=16, channels=3, hr=4096, factor=4, r=8, eps=1e-4),
    "cfg4a": dict(kind="joint_fwd_bwd", batch=64, channels=3, hr=3072, factor=4, r=2,
                  eps=1e-4, shard="batch"),
    "cfg4b": dict(kind="joint_fwd_bwd", batch=1, channels=3, hr=16384, factor=4, r=2,
                  eps=1e-4, shard="rows"),
}
