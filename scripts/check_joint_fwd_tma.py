"""Quick GPU check: the persistent TMA joint forward vs the tile kernel
(variant 9) -- bitwise -- over radii and ragged shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1803_05619_b200 as gfb
lib = gfb._lib.load()
bad = 0
for (B, C, h, w) in [(1, 3, 16, 32), (2, 3, 37, 44), (1, 1, 256, 256), (1, 3, 100, 300), (3, 2, 8, 4)]:
    for r in (0, 1, 2, 3, 4, 8, 12):
        g = torch.Generator(device="cuda").manual_seed(r + h)
        lx = torch.rand(B, C, h, w, device="cuda", generator=g)
        ly = torch.rand(B, C, h, w, device="cuda", generator=g)
        hx = torch.rand(B, C, 4 * h, 4 * w, device="cuda", generator=g)
        p = gfb.GuidedFilterParams(r, 1e-4)
        b, _ = gfb.forward_joint(lx, hx, ly, p)
        old = lib.gf_joint_fwd_variant(10)
        a, _ = gfb.forward_joint(lx, hx, ly, p)
        lib.gf_joint_fwd_variant(old)
        torch.cuda.synchronize()
        eq = torch.equal(a, b)
        bad += not eq
        print(B, C, h, w, r, "equal" if eq else f"DIFF {float((a - b).abs().max())}", flush=True)
print("bad", bad)
