"""Joint backward variants at config 4a (tape entries): default (hr_x and
d_out windows by TMA, 2 CTAs/SM) vs 12 (tape, global loads) and 0-with-
recompute (plain gf_joint_bwd); bitwise check between the tape variants
(GPU box)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, workloads
from paper_1803_05619_b200 import _lib
L = _lib.load()
B, H, C, r, eps = 64, 3072, 3, 2, 1e-4
h = H // 4
lx, ly, hx = workloads.joint_inputs(B, C, H, H, 4, seed=3, device="cuda")
d = torch.randn_like(hx)
sp = torch.cuda.current_stream().cuda_stream
st = torch.zeros(1, dtype=torch.int32, device="cuda")
ws = torch.empty(L.gf_joint_workspace_bytes(0, B, C, h, h, H, H, r), dtype=torch.uint8, device="cuda")
out = torch.empty_like(hx); A = torch.empty_like(lx)
P = lambda t: t.data_ptr()
assert L.gf_joint_fwd_tape(0, P(lx), P(ly), P(hx), P(out), P(A), B, C, h, h, H, H, r, eps, P(ws), ws.numel(), P(st), sp) == 0
res = {}
for v in (0, 12, 0, 8, 8):  # 8: the default hr pass on 32-row tiles
    g = [torch.empty_like(lx), torch.empty_like(ly), torch.empty_like(hx)]
    old = L.gf_joint_bwd_hr_variant(0 if v == 8 else v)
    oldt = L.gf_joint_bwd_hr_tile(8 if v == 8 else 16)
    f = lambda: L.gf_joint_bwd_tape(0, P(lx), P(ly), P(hx), P(A), P(d), P(g[0]), P(g[1]), P(g[2]), B, C, h, h, H, H, r, eps, 0, P(ws), ws.numel(), P(st), sp)
    for _ in range(3): assert f() == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    L.gf_joint_bwd_hr_variant(old)
    L.gf_joint_bwd_hr_tile(oldt)
    res.setdefault(v, g)
    print("variant", v, round(e0.elapsed_time(e1) / 10, 3), "ms  bitwise vs default:",
          all(torch.equal(a, b) for a, b in zip(g, res[0])), flush=True)
