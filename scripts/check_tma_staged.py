"""TMA-staged tile kernels (variant hooks 11) vs the __ldg-staged defaults:
bitwise equality of the joint forward (variant 9 = tile kernel), backward hr
pass (4) and fused training step (3), then device times at
config 4a (forward + backward) and config 2's fused step (GPU box)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1803_05619_b200 as gfb, workloads
lib = gfb._lib.load()


def with_variants(fwd, bwd, mse, fn):
    o = (lib.gf_joint_fwd_variant(fwd), lib.gf_joint_bwd_hr_variant(bwd), lib.gf_joint_mse_variant(mse))
    try:
        return fn()
    finally:
        lib.gf_joint_fwd_variant(o[0]); lib.gf_joint_bwd_hr_variant(o[1]); lib.gf_joint_mse_variant(o[2])


bad = 0
for (B, C, h, w) in [(1, 3, 16, 32), (2, 3, 37, 44), (1, 1, 256, 256), (1, 3, 100, 300), (3, 2, 8, 4)]:
    for r in (0, 1, 2, 3, 4, 8, 12):
        g = torch.Generator(device="cuda").manual_seed(r + h)
        lx = torch.rand(B, C, h, w, device="cuda", generator=g)
        ly = torch.rand(B, C, h, w, device="cuda", generator=g)
        hx = torch.rand(B, C, 4 * h, 4 * w, device="cuda", generator=g)
        d = torch.randn(B, C, 4 * h, 4 * w, device="cuda", generator=g)
        tg = torch.rand(B, C, 4 * h, 4 * w, device="cuda", generator=g)
        p = gfb.GuidedFilterParams(r, 1e-4)

        def run():
            o, t = gfb.forward_joint(lx, hx, ly, p)
            gr = gfb.backward(t, d)
            loss, g2, _ = gfb.joint_mse_backward(lx, hx, ly, tg, p)
            return [o, gr.d_guide_lo, gr.d_src, gr.d_guide_hi, g2.d_guide_lo, g2.d_src, g2.d_guide_hi, loss]
        a = with_variants(11, 11, 11, run)
        b = with_variants(9, 4, 3, run)
        torch.cuda.synchronize()
        eq = all(torch.equal(x, y) for x, y in zip(a, b))
        bad += not eq
        if not eq:
            print(B, C, h, w, r, "DIFF", [float((x - y).abs().max()) for x, y in zip(a, b)], flush=True)
print("bitwise mismatches:", bad, flush=True)

def timeit(f, n=10):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n

lr_x, lr_y, hr_x = workloads.joint_inputs(64, 3, 3072, 3072, 4, seed=1, device="cuda")
d = torch.randn_like(hr_x)
p = gfb.GuidedFilterParams(2, 1e-4)
out = torch.empty_like(hr_x)
for v in ((0, 0, 0), (11, 11, 11)):
    tf = with_variants(*v, lambda: timeit(lambda: gfb.forward_joint(lr_x, hr_x, lr_y, p, check=False)))
    o, t = gfb.forward_joint(lr_x, hr_x, lr_y, p, check=False)
    tb = with_variants(*v, lambda: timeit(lambda: gfb.backward(t, d, check=False)))
    print(f"cfg4a variants {v}: fwd {tf:.3f} ms  bwd {tb:.3f} ms  step {tf + tb:.3f} ms", flush=True)
del lr_x, lr_y, hr_x, d, o, t
torch.cuda.empty_cache()
lr_x, lr_y, hr_x = workloads.joint_inputs(8, 3, 2048, 2048, 4, seed=1, device="cuda")
tg = workloads.affine_target(hr_x).contiguous()
p = gfb.GuidedFilterParams(1, 1e-8)
for v in ((0, 0, 0), (11, 11, 11)):
    tm = with_variants(*v, lambda: timeit(lambda: gfb.joint_mse_backward(lr_x, hr_x, lr_y, tg, p, check=False)))
    print(f"cfg2 fused filter step variants {v}: {tm:.3f} ms", flush=True)
