"""CUDA-event time of the fp32 full-res forward kernels (variant 1 = batch/TMA,
2 = register segment) at config-1 shape (4 x {1,3} x 2048^2, r=8) and a few
radii; inputs > L2, so no flush needed."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1803_05619_b200 as gfb  # noqa: E402
from paper_1803_05619_b200 import _lib  # noqa: E402
import workloads  # noqa: E402

lib = _lib.load()
guide, src = [t.cuda() for t in workloads.highres_inputs(4, 3, 2048, 2048, seed=0)]
out = torch.empty_like(src)
st = torch.zeros(1, dtype=torch.int32, device="cuda")


def run(r, eps):
    rc = lib.gf_highres_fwd(0, guide.data_ptr(), src.data_ptr(), out.data_ptr(), 4, 1, 3, 2048,
                            2048, r, eps, 0, 0, st.data_ptr(),
                            torch.cuda.current_stream().cuda_stream)
    assert rc == 0, lib.gf_last_error()


for r in [int(x) for x in (sys.argv[1:] or ["8"])]:
    res = {}
    for v in (1, 2, 3, 4):
        old = lib.gf_highres_variant(v)
        for _ in range(3):
            run(r, 1e-2)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record()
            run(r, 1e-2)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        lib.gf_highres_variant(old)
        res[v] = sorted(ts)[len(ts) // 2]
        o = out.clone()
        if v == 1:
            ref = o
        print(f"  variant {v}: max|diff vs 1| {float((o - ref).abs().max()):.2e}")
    print(f"r={r}: batch/TMA {res[1]*1e3:.1f} us  segment {res[2]*1e3:.1f} us  "
          f"segment(8/lane) {res[3]*1e3:.1f} us  "
          f"max|diff| {float((o - ref).abs().max()):.2e}")
