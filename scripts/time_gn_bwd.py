"""Time the fused guidance-net backward variants (0: one heavy pass + dx
fix-up, two lanes per pixel group; 1: two heavy passes; 2: the one-pass
kernel with four lanes per group; 3: 0 capped at 3 CTAs per SM) at BASELINE config-2 shape (8 x 3 x 2048^2, hidden 15) and compare
their outputs with the first one named (GPU box).  Usage: time_gn_bwd.py
[variant ...] (default 1 0)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1803_05619_b200 as gfb  # noqa: E402
import workloads  # noqa: E402
from paper_1803_05619_b200 import _lib  # noqa: E402

lib = _lib.load()
_, _, x = workloads.joint_inputs(8, 3, 2048, 2048, seed=9)
x = x.cuda()
net = gfb.GuidanceNet(3, 3, hidden=15, kernel=1, rng=np.random.default_rng(4), device="cuda")
y, tape = net.forward(x, check=False)
dy = torch.randn(y.shape, generator=torch.Generator().manual_seed(2)).cuda() * 1e-6
vs = [int(a) for a in sys.argv[1:]] or [1, 0]
res = {}
for v in vs:
    lib.gf_gn_bwd_variant(v)
    f = lambda: net.backward(tape, dy, check=False)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        f()
    b.record()
    torch.cuda.synchronize()
    res[v] = f()
    print(f"variant {v}: {a.elapsed_time(b) / 10 * 1e3:.1f} us")
lib.gf_gn_bwd_variant(0)
dx1, dp1 = res[vs[0]]
for v in vs[1:]:
    dx0, dp0 = res[v]
    print(f"variant {v} vs {vs[0]}: dx rel", float((dx0 - dx1).abs().max() / dx1.abs().max()))
    for k in dp1:
        a, b = dp0[k].double(), dp1[k].double()
        print("  ", k, "rel-to-max", float((a - b).abs().max() / max(float(b.abs().max()), 1e-30)))
