"""Experiment: chunks of planes, the coefficient kernel of chunk i+1 on a
high-priority stream while the apply kernel of chunk i streams (GPU box).
python scripts/time_joint_overlap.py B side r nchunks..."""
import sys

import torch

sys.path.insert(0, ".")
import workloads  # noqa: E402
from paper_1803_05619_b200 import _lib  # noqa: E402

B = int(sys.argv[1]); H = int(sys.argv[2]); r = int(sys.argv[3])
chunks = [int(x) for x in sys.argv[4:]] or [1, 2, 4, 8]
eps, C, h = 1e-4, 3, H // 4
L = _lib.load()
lx, ly, hx = (t.cuda() for t in workloads.joint_inputs(B, C, H, H, seed=5))
out = torch.empty_like(hx)
A = torch.empty_like(lx); Bc = torch.empty_like(lx)
st = torch.zeros(1, dtype=torch.int32, device="cuda")
main = torch.cuda.current_stream()
lo, hi = -1, 0
try:
    hp = torch.cuda.Stream(priority=-5)
except Exception:
    hp = torch.cuda.Stream(priority=-1)
P = lambda t: t.data_ptr()  # noqa: E731

def run(n):
    # planes split in n chunks of whole images
    per = (B + n - 1) // n
    evs = []
    e0 = torch.cuda.Event(); e0.record(main)
    hp.wait_event(e0)
    for i in range(0, B, per):
        b = min(per, B - i)
        rc = L.gf_joint_coeffs(0, P(lx[i:]), P(ly[i:]), P(A[i:]), P(Bc[i:]), b, C, h, h, r, eps, P(st), hp.cuda_stream)
        assert rc == 0, L.gf_last_error()
        ev = torch.cuda.Event(); ev.record(hp); evs.append(ev)
    k = 0
    for i in range(0, B, per):
        b = min(per, B - i)
        main.wait_event(evs[k]); k += 1
        rc = L.gf_joint_apply(0, P(A[i:]), P(Bc[i:]), P(hx[i:]), P(out[i:]), b, C, h, h, H, H, P(st), main.cuda_stream)
        assert rc == 0, L.gf_last_error()

ref = None
for n in chunks:
    out.zero_()
    for _ in range(3):
        run(n)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for _ in range(10):
        run(n)
    b.record(main)
    torch.cuda.synchronize()
    if ref is None:
        ref = out.clone()
    print(f"B={B} H={H} r={r} chunks {n}: {a.elapsed_time(b) / 10 * 1e3:.1f} us  max|diff| {float((out - ref).abs().max()):.2e}")
