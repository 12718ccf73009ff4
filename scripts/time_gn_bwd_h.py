"""Guidance-net backward at config 2's high-res site (8 x 3 x 2048^2, hidden 15),
device time of net.backward (GPU box)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_1803_05619_b200 as gfb
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand(8, 3, 2048, 2048, device="cuda", generator=g)
dy = torch.randn(8, 3, 2048, 2048, device="cuda", generator=g) * 1e-7
net = gfb.GuidanceNet(3, 3, hidden=15, kernel=1, rng=np.random.default_rng(1))
net.norm.norm_gain[:] = 0.5
y, t = net.forward(x)
dp = torch.empty(net.param_count(), device="cuda")
f = lambda: net.backward(t, dy, dparams=dp, check=False)
for _ in range(3): f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): f()
b.record(); torch.cuda.synchronize()
dx, g = f()
print("backward", round(a.elapsed_time(b) / 10 * 1e3, 1), "us; checksum", float(dx.double().abs().sum()), float(dp.double().abs().sum()))
