"""Persistent TMA joint forward (variant 10) vs the tile kernel (variant 0):
device time per call (CUDA events) and fraction of the measured HBM copy
peak at config 3 (16 x 3 x 4096^2) for each radius, config 4a's forward
(64 x 3 x 3072^2, r=2) and config 0 (1 x 3 x 1024^2, r=1, L2 flushed)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1803_05619_b200 as gfb  # noqa: E402
import workloads  # noqa: E402
from paper_1803_05619_b200 import _lib  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
lib = _lib.load()
flush = torch.ones(64 * 1024 * 1024, device="cuda")
cases = [(16, 4096, r) for r in (1, 2, 4, 8)] + [(64, 3072, 2), (1, 1024, 1), (1, 2048, 8)]
for B, H, r in cases:
    lr_x, lr_y, hr_x = workloads.joint_inputs(B, 3, H, H, 4, seed=5, device="cuda")
    p = gfb.GuidedFilterParams(r, 1e-4)
    byts = 4 * B * 3 * (2 * H * H + 2 * (H // 4) ** 2)
    small = byts < 300e6
    res = {}
    for v in (0, 10):
        lib.gf_joint_fwd_variant(v)
        f = lambda: gfb.forward_joint(lr_x, hr_x, lr_y, p, check=False)  # noqa: E731
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            if small:
                flush.sum()
                torch.cuda._sleep(200000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out, _ = f()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = sum(ts) / len(ts)
        res[v] = (ms, out)
        print(f"B={B} H={H} r={r} variant {v}: {ms * 1e3:.1f} us  {byts / ms / 1e6:.0f} GB/s  "
              f"frac {byts / ms / 1e6 / peak:.3f}", flush=True)
    print("   bitwise equal:", torch.equal(res[0][1], res[10][1]), flush=True)
    del lr_x, lr_y, hr_x
    torch.cuda.empty_cache()
lib.gf_joint_fwd_variant(0)
