"""Time the fused training-step filter (gf_joint_mse_bwd) against the unfused
forward -> MSE -> backward chain at BASELINE config-2 shape, per kernel
variant (GPU box).  python scripts/time_joint_mse.py [variants...]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1803_05619_b200 as gfb  # noqa: E402
import workloads  # noqa: E402
from paper_1803_05619_b200 import _lib  # noqa: E402
from paper_1803_05619_b200.training import mse_loss_device  # noqa: E402


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


lr_x, lr_y, hr_x = (t.cuda() for t in workloads.joint_inputs(8, 3, 2048, 2048, seed=3))
tg = workloads.affine_target(hr_x).contiguous()
p = gfb.GuidedFilterParams(1, 1e-8)
lib = _lib.load()


def chain():
    out, tape = gfb.forward_joint(lr_x, hr_x, lr_y, p, check=False)
    _, d = mse_loss_device(out, tg)
    gfb.backward(tape, d, check=False)


print(f"unfused chain: {timeit(chain):.1f} us")
ref = gfb.joint_mse_backward(lr_x, hr_x, lr_y, tg, p)
for v in [int(x) for x in sys.argv[1:]] or [0, 3, 4]:
    lib.gf_joint_mse_variant(v)
    t = timeit(lambda: gfb.joint_mse_backward(lr_x, hr_x, lr_y, tg, p, check=False))
    got = gfb.joint_mse_backward(lr_x, hr_x, lr_y, tg, p)
    dmax = max(float((a - b).abs().max()) for a, b in
               zip((got[1].d_src, got[1].d_guide_lo, got[1].d_guide_hi),
                   (ref[1].d_src, ref[1].d_guide_lo, ref[1].d_guide_hi)))
    print(f"variant {v}: {t:.1f} us  loss {float(got[0]):.9e}  max|diff| vs variant 0 {dmax:.2e}")
lib.gf_joint_mse_variant(0)
