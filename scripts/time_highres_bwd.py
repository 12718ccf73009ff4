"""Time the full-res backward (general kernels) at config-1 size."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1803_05619_b200 as gfb  # noqa: E402
from workloads import CONFIGS, highres_inputs  # noqa: E402

c = CONFIGS["cfg1"]
g, s = highres_inputs(4, 3, 2048, 2048, seed=0, device="cuda")
p = gfb.GuidedFilterParams(c["r"], c["eps"])
out, tape = gfb.forward_highres(g, s, p)
d = torch.rand_like(out)
for _ in range(2):
    gfb.backward(tape, d)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    gfb.backward(tape, d)
e1.record()
torch.cuda.synchronize()
print("highres bwd ms/step", e0.elapsed_time(e1) / 5)
e0.record()
for _ in range(5):
    gfb.forward_highres(g, s, p, check=False)
e1.record()
torch.cuda.synchronize()
print("highres fwd ms/step", e0.elapsed_time(e1) / 5)
