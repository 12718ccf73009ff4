"""Two-kernel joint forward (k_joint_coeffs + k_joint_apply) vs the one-kernel
tile forward through gf_joint_fwd (GPU box).
python scripts/time_joint_split.py B side r [variants...]"""
import sys

import torch

sys.path.insert(0, ".")
import workloads  # noqa: E402
from paper_1803_05619_b200 import _lib  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
H = int(sys.argv[2]) if len(sys.argv) > 2 else 3072
r = int(sys.argv[3]) if len(sys.argv) > 3 else 2
variants = [int(x) for x in sys.argv[4:]] or [0, 20, 23, 25]
eps = 1e-4
C, h = 3, H // 4
L = _lib.load()
lx, ly, hx = (t.cuda() for t in workloads.joint_inputs(B, C, H, H, seed=5))
out = torch.empty_like(hx)
ws = torch.empty(L.gf_joint_workspace_bytes(0, B, C, h, h, H, H, r), dtype=torch.uint8, device="cuda")
st = torch.zeros(1, dtype=torch.int32, device="cuda")
P = lambda t: t.data_ptr()  # noqa: E731
sp = torch.cuda.current_stream().cuda_stream
ref = None
for v in variants:
    L.gf_joint_fwd_variant(v)
    f = lambda: L.gf_joint_fwd(0, P(lx), P(ly), P(hx), P(out), B, C, h, h, H, H, r, eps, P(ws), ws.numel(), P(st), sp)  # noqa: E731
    out.zero_()
    for _ in range(3):
        assert f() == 0, L.gf_last_error()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        f()
    b.record()
    torch.cuda.synchronize()
    if ref is None:
        ref = out.clone()
    gb = (2 * hx.numel() + 2 * lx.numel()) * 4 / 1e9
    ms = a.elapsed_time(b) / 10
    print(f"B={B} H={H} r={r} variant {v}: {ms * 1e3:.1f} us  {gb / ms:.0f} GB/s(alg)  "
          f"max|diff vs first| {float((out - ref).abs().max()):.2e} status {int(st.item())}")
L.gf_joint_fwd_variant(0)
