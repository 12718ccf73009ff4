"""Time the joint backward's hr-pass variants (1: two-read tile kernel,
0: single gather pass at 4 CTAs/SM, 3: single pass at 3 CTAs/SM) on
config-4 / config-2 shaped batches and compare them (GPU box)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1803_05619_b200 as gfb  # noqa: E402
import workloads  # noqa: E402
from paper_1803_05619_b200 import _lib  # noqa: E402

lib = _lib.load()
for B, H, r in ((8, 3072, 2), (8, 2048, 1)):
    lr_x, lr_y, hr_x = (t.cuda() for t in workloads.joint_inputs(B, 3, H, H, seed=1))
    p = gfb.GuidedFilterParams(r, 1e-4)
    out, tape = gfb.forward_joint(lr_x, hr_x, lr_y, p)
    d_out = torch.randn(out.shape, generator=torch.Generator().manual_seed(0)).cuda()
    res = {}
    for v in (1, 0, 3):
        lib.gf_joint_bwd_hr_variant(v)
        f = lambda: gfb.backward(tape, d_out, check=False)  # noqa: E731
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
        d = max(float((x - y).abs().max() / y.abs().max()) for x, y in
                zip((res[v].d_src, res[v].d_guide_lo, res[v].d_guide_hi),
                    (res[1].d_src, res[1].d_guide_lo, res[1].d_guide_hi)))
        print(f"B={B} H={H} r={r} variant {v}: {a.elapsed_time(b) / 10 * 1e3:.1f} us  rel diff {d:.2e}")
    lib.gf_joint_bwd_hr_variant(0)
    del lr_x, lr_y, hr_x, out, tape, d_out, res
    torch.cuda.empty_cache()
