"""Fused training-step filter pass (gf_joint_mse_bwd) at config 2's size:
default (coefficient tape + TMA gather window) vs the moments-recomputing
kernel (variant 3), CUDA events (GPU box)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1803_05619_b200 as gfb, workloads
lib = gfb._lib.load()
lx, ly, hx = workloads.joint_inputs(8, 3, 2048, 2048, 4, seed=1, device="cuda")
tg = workloads.affine_target(hx).contiguous()
p = gfb.GuidedFilterParams(1, 1e-8)
for v in (0, 16, 0, 16):
    old = lib.gf_joint_mse_variant(v)
    f = lambda: gfb.joint_mse_backward(lx, hx, ly, tg, p, check=False)
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): f()
    b.record(); torch.cuda.synchronize()
    lib.gf_joint_mse_variant(old)
    print("variant", v, round(a.elapsed_time(b) / 20 * 1e3, 1), "us", flush=True)
