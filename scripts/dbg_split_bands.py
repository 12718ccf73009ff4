import sys
import torch
sys.path.insert(0, ".")
import workloads
import paper_1803_05619_b200 as gfb
from paper_1803_05619_b200 import _lib
from paper_1803_05619_b200.sharding import row_bands, joint_band_forward
L = _lib.load()
h, w, r = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
world = int(sys.argv[4])
lr_x, lr_y, hr_x = workloads.joint_inputs(1, 3, 4 * h, 4 * w, 4, seed=47, device="cuda")
p = gfb.GuidedFilterParams(r, 1e-4)
L.gf_joint_fwd_mode(2)
out, tape = gfb.forward_joint(lr_x, hr_x, lr_y, p)
A = tape._slope_lo
for band in row_bands(h, world, r, 4, backward=False):
    lo, hi = band.crop_lo, band.crop_hi
    o, t = gfb.forward_joint(lr_x[:, :, lo:hi].contiguous(), hr_x[:, :, 4 * lo:4 * hi].contiguous(), lr_y[:, :, lo:hi].contiguous(), p)
    Ab = t._slope_lo
    dA = (Ab != A[:, :, lo:hi])
    rows = dA.any(dim=3).any(dim=1)[0].nonzero().flatten().tolist()
    cols = dA.any(dim=2).any(dim=1)[0].nonzero().flatten().tolist()
    print("band", band.a, band.b, "crop", lo, hi, "A rows differing (crop coords)", rows[:10], "...", rows[-5:], "n", len(rows), "cols", cols[:8], len(cols))
    do = (o != out[:, :, 4 * lo:4 * hi])
    rows = do.any(dim=3).any(dim=1)[0].nonzero().flatten().tolist()
    y0, y1 = band.hr_local
    bad = [y for y in rows if y0 <= y < y1]
    print("   out rows differing", len(rows), "owned-bad", bad[:10], len(bad))
