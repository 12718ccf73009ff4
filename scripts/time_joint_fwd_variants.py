"""Time the joint forward's coefficient-chunking variants at BASELINE config 3
(16 x 3 x 4096^2, r = 8) and check them bitwise against the default (GPU box).
python scripts/time_joint_fwd_variants.py [radius] [variants...]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1803_05619_b200 as gfb  # noqa: E402
import workloads  # noqa: E402
from paper_1803_05619_b200 import _lib  # noqa: E402

r = int(sys.argv[1]) if len(sys.argv) > 1 else 8
variants = [int(x) for x in sys.argv[2:]] or [0, 1, 2, 3]
lr_x, lr_y, hr_x = (t.cuda() for t in workloads.joint_inputs(16, 3, 4096, 4096, seed=5))
p = gfb.GuidedFilterParams(r, 1e-4)
lib = _lib.load()
ref, _ = gfb.forward_joint(lr_x, hr_x, lr_y, p)
for v in variants:
    lib.gf_joint_fwd_variant(v)
    f = lambda: gfb.forward_joint(lr_x, hr_x, lr_y, p, check=False)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        f()
    b.record()
    torch.cuda.synchronize()
    out, _ = f()
    print(f"r={r} variant {v}: {a.elapsed_time(b) / 10 * 1e3:.1f} us  "
          f"max|diff| {float((out - ref).abs().max()):.2e}")
lib.gf_joint_fwd_variant(0)
