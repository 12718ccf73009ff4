"""Debug helper: run the fused full-res forward on a grid of shapes/radii,
one subprocess per case so a sticky CUDA error does not hide the rest."""
import subprocess
import sys

CASE = r'''
import sys, torch, numpy as np
import paper_1803_05619_b200 as m
from oracle import gf_oracle as O
B, Cg, C, H, W, r = map(int, sys.argv[1:7])
g = torch.rand(B, Cg, H, W, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
s = torch.rand(B, C, H, W, device="cuda", generator=torch.Generator("cuda").manual_seed(2))
out, _ = m.forward_highres(g, s, m.GuidedFilterParams(r, 1e-2))
torch.cuda.synchronize()
want = O.highres_forward_nchw(g.double().cpu().numpy(), s.double().cpu().numpy(), r, 1e-2)
err = float(np.abs(out.double().cpu().numpy() - want).max())
print("ok" if err < 1e-4 else "BAD", err)
'''

cases = [tuple(map(int, a.split(","))) for a in sys.argv[1:]] or [
    (1, 2, 2, 9, 8, 1), (1, 1, 1, 9, 8, 1), (1, 1, 1, 64, 64, 1), (1, 1, 1, 64, 64, 2),
    (1, 1, 1, 64, 64, 8), (1, 1, 1, 300, 512, 8), (1, 1, 3, 300, 512, 8), (1, 1, 1, 40, 36, 8),
    (1, 1, 1, 64, 64, 9), (1, 1, 1, 64, 64, 16)]
for c in cases:
    p = subprocess.run([sys.executable, "-c", CASE, *map(str, c)], capture_output=True, text=True,
                       env={**__import__("os").environ, "CUDA_LAUNCH_BLOCKING": "1"})
    tail = (p.stdout + p.stderr).strip().splitlines()
    print(c, p.returncode, tail[-1] if tail else "")
