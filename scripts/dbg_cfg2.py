"""Localise the fp32 error of the config-2 step with norm_gain != 0 (GPU box)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1803_05619_b200 as gfb, workloads
from oracle import gf_oracle as O

ng = float(sys.argv[1]) if len(sys.argv) > 1 else 0.7
H = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
lr_x, lr_y, hr_x = (t.cuda() for t in workloads.joint_inputs(1, 3, H, H, 4, seed=21))
tg = workloads.affine_target(hr_x).contiguous()
net = gfb.GuidanceNet(3, 3, hidden=15, kernel=1, rng=np.random.default_rng(5))
net.norm.norm_gain[:] = ng
p = gfb.GuidedFilterParams(1, 1e-8)
params = {k: v.cpu().numpy().copy() for k, v in net.parameters().items()}
hwc = lambda t: t[0].permute(1, 2, 0).double().cpu().numpy()
nchw = lambda a: torch.from_numpy(np.ascontiguousarray(a.transpose(2, 0, 1)))[None]
rel = lambda a, b: float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))
Gl, tl = O.guidance_forward(params, hwc(lr_x))
Gh, th = O.guidance_forward(params, hwc(hr_x))
out, tp = O.forward_joint(Gl, Gh, hwc(lr_y), 1, 1e-8)
loss, d = O.mse_loss(out, hwc(tg))
gs = O.backward(tp, d)
dlx_ref, grads_lo = O.guidance_backward(params, tl, gs[1])
g_lo, t_lo = net.forward(lr_x)
g_hi, t_hi = net.forward(hr_x)
print("G_lo rel", rel(hwc(g_lo), Gl), "G_hi rel", rel(hwc(g_hi), Gh))
l2, grads, st = gfb.joint_mse_backward(g_lo, g_hi, lr_y, tg, p)
print("loss", float(l2), loss)
print("d_guide_lo rel", rel(hwc(grads.d_guide_lo), gs[1]), "d_src", rel(hwc(grads.d_src), gs[0]),
      "d_guide_hi", rel(hwc(grads.d_guide_hi), gs[2]))
# guidance backward alone, fed the oracle's exact d_guide_lo (fp32)
dl = nchw(gs[1]).float().cuda()
dx, gr = net.backward(t_lo, dl)
print("gn bwd (exact dy, fp32) dx rel", rel(hwc(dx), dlx_ref))
for k in grads_lo:
    print("   ", k, rel(gr[k].double().cpu().numpy(), grads_lo[k]))
for v in (0, 1):
    lib = gfb._lib.load()
    old = lib.gf_gn_bwd_variant(v)
    dx, gr = net.backward(t_lo, dl)
    lib.gf_gn_bwd_variant(old)
    print("variant", v, "dx rel", rel(hwc(dx), dlx_ref))
# fp64 guidance backward
xt = lr_x.double()
g64, t64 = net.forward(xt)
dx64, _ = net.backward(t64, dl.double())
print("gn bwd fp64 dx rel", rel(hwc(dx64), dlx_ref))
