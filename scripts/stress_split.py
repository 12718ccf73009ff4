"""Randomised agreement of the two-kernel forward (+ the backward on its tape)
with the one-kernel forward over ragged shapes, radii 0..12 and eps 1e-2..1e-6
(GPU box): d_lr_x / d_lr_y bitwise, outputs to fp32 rounding of the halo
coefficients.  At r = 0 the exact slope is 0, so d_hr_x is rounding noise in
both paths and is not compared relatively."""
import sys, random
import torch
sys.path.insert(0, ".")
import workloads
import paper_1803_05619_b200 as gfb
from paper_1803_05619_b200 import _lib
L = _lib.load()
random.seed(1)
worst = 0.0
n = 0
for it in range(160):
    h = random.choice([2, 3, 5, 9, 15, 16, 17, 31, 32, 33, 47, 64, 65, 100, 130, 257])
    w = random.choice([4, 8, 12, 20, 36, 60, 64, 100, 116, 120, 124, 128, 132, 236, 240, 244, 248, 252, 256, 260, 384, 500, 501, 502])
    r = random.choice([0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 12])
    B, C = random.choice([(1, 1), (1, 3), (2, 3), (3, 2)])
    eps = random.choice([1e-2, 1e-4, 1e-6])
    lr_x, lr_y, hr_x = workloads.joint_inputs(B, C, 4 * h, 4 * w, seed=it, device="cuda")
    p = gfb.GuidedFilterParams(r, eps)
    outs = []
    grads = []
    for mode in (1, 2):
        old = L.gf_joint_fwd_mode(mode)
        try:
            o, tape = gfb.forward_joint(lr_x, hr_x, lr_y, p)
        finally:
            L.gf_joint_fwd_mode(old)
        d = torch.randn(o.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(it))
        g = gfb.backward(tape, d)
        outs.append(o)
        grads.append(g)
    e = float((outs[0] - outs[1]).abs().max())
    ghi = float((grads[0].d_guide_hi - grads[1].d_guide_hi).abs().max()) / max(float(grads[0].d_guide_hi.abs().max()), 1e-30)
    assert torch.equal(grads[0].d_src, grads[1].d_src) and torch.equal(grads[0].d_guide_lo, grads[1].d_guide_lo), (h, w, r)
    assert torch.isfinite(outs[1]).all()
    # slopes scale like 1/eps at the smallest variances: compare outputs relative to eps-driven rounding
    tol = 2e-5 if eps >= 1e-4 else 2e-3
    if e > tol or (eps >= 1e-4 and r > 0 and ghi > 1e-3):
        print("MISMATCH", (B, C, h, w, r, eps), e, ghi)
    worst = max(worst, e if eps >= 1e-4 else 0.0)
    n += 1
print("cases", n, "worst |out diff| (eps >= 1e-4)", worst)
