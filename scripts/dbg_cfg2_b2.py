"""config-2 step with B=2, norm_gain != 0: which image / stage drifts (GPU box)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1803_05619_b200 as gfb, workloads
from oracle import gf_oracle as O

ng = float(sys.argv[1]) if len(sys.argv) > 1 else 0.7
B = int(sys.argv[2]) if len(sys.argv) > 2 else 2
H = 2048
lr_x, lr_y, hr_x = (t.cuda() for t in workloads.joint_inputs(B, 3, H, H, 4, seed=21))
tg = workloads.affine_target(hr_x).contiguous()
net = gfb.GuidanceNet(3, 3, hidden=15, kernel=1, rng=np.random.default_rng(5))
net.norm.norm_gain[:] = ng
p = gfb.GuidedFilterParams(1, 1e-8)
params = {k: v.cpu().numpy().copy() for k, v in net.parameters().items()}
hwc = lambda t, n: t[n].permute(1, 2, 0).double().cpu().numpy()
rel = lambda a, b: float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))
res = gfb.train_step(net, lr_x, hr_x, lr_y, tg, p)
loss, _, dlx, dly, dhx, grads = O.train_step(params, [hwc(lr_x, n) for n in range(B)],
                                             [hwc(hr_x, n) for n in range(B)],
                                             [hwc(lr_y, n) for n in range(B)],
                                             [hwc(tg, n) for n in range(B)], 1, 1e-8)
print("loss", float(res.loss), loss)
for n in range(B):
    print("img", n, "d_lr_x", rel(hwc(res.d_lr_x, n), dlx[n]), "d_lr_y", rel(hwc(res.d_lr_y, n), dly[n]),
          "d_hr_x", rel(hwc(res.d_hr_x, n), dhx[n]))
g_lo, t_lo = net.forward(lr_x)
for n in range(B):
    Gl, tl = O.guidance_forward(params, hwc(lr_x, n))
    print("img", n, "G_lo", rel(hwc(g_lo, n), Gl))
# per image alone
for n in range(B):
    r1 = gfb.train_step(net, lr_x[n:n+1].contiguous(), hr_x[n:n+1].contiguous(), lr_y[n:n+1].contiguous(), tg[n:n+1].contiguous(), p)
    print("alone img", n, "d_lr_x vs batched", rel(r1.d_lr_x[0].permute(1,2,0).double().cpu().numpy(), hwc(res.d_lr_x, n)) ,
          "alone vs oracle(B-scaled)", rel(r1.d_lr_x[0].permute(1,2,0).double().cpu().numpy() / B, dlx[n]))
# kink analysis: errors at pixels whose hidden pre-activation h2 is near 0
n = 0
for site, xin, dref in (("lo", lr_x, dlx), ("hi", hr_x, dhx)):
    G, tape = O.guidance_forward(params, hwc(xin, n))
    h2 = params["norm.gain"][0] * tape["h1"] + params["norm.norm_gain"][0] * tape["xhat"]
    amb = (np.abs(h2) < 1e-4).any(axis=2)
    got = hwc(res.d_lr_x if site == "lo" else res.d_hr_x, n)
    err = np.abs(got - dref[n]).max(axis=2)
    i = np.unravel_index(np.argmax(err), err.shape)
    print(site, "worst px", i, "err/max", err[i] / np.abs(dref[n]).max(), "min|h2| there",
          np.abs(h2[i]).min(), "ambiguous px", int(amb.sum()),
          "err/max excl. ambiguous", err[~amb].max() / np.abs(dref[n]).max())
