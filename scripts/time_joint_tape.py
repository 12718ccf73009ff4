"""Tape variant of the joint layer (gf_joint_fwd_tape + gf_joint_bwd_tape: the
backward's hr pass reads the forward's low-res slopes) vs gf_joint_fwd +
gf_joint_bwd: agreement and CUDA-event times at config 4a (GPU box)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, workloads
from paper_1803_05619_b200 import _lib
L = _lib.load()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
H = 3072; h = H // 4; C = 3; r = 2; eps = 1e-4
lx, ly, hx = workloads.joint_inputs(B, C, H, H, 4, seed=3, device="cuda")
d = torch.randn_like(hx)
sp = torch.cuda.current_stream().cuda_stream
st = torch.zeros(1, dtype=torch.int32, device="cuda")
ws = torch.empty(L.gf_joint_workspace_bytes(0, B, C, h, h, H, H, r), dtype=torch.uint8, device="cuda")
out = torch.empty_like(hx); out2 = torch.empty_like(hx)
A = torch.empty_like(lx)
g1 = [torch.empty_like(lx), torch.empty_like(ly), torch.empty_like(hx)]
g2 = [torch.empty_like(lx), torch.empty_like(ly), torch.empty_like(hx)]
P = lambda t: t.data_ptr()
def plain():
    assert L.gf_joint_fwd(0, P(lx), P(ly), P(hx), P(out), B, C, h, h, H, H, r, eps, P(ws), ws.numel(), P(st), sp) == 0
    assert L.gf_joint_bwd(0, P(lx), P(ly), P(hx), P(d), P(g1[0]), P(g1[1]), P(g1[2]), B, C, h, h, H, H, r, eps, P(ws), ws.numel(), P(st), sp) == 0
def tape():
    assert L.gf_joint_fwd_tape(0, P(lx), P(ly), P(hx), P(out2), P(A), B, C, h, h, H, H, r, eps, P(ws), ws.numel(), P(st), sp) == 0, L.gf_last_error()
    assert L.gf_joint_bwd_tape(0, P(lx), P(ly), P(hx), P(A), P(d), P(g2[0]), P(g2[1]), P(g2[2]), B, C, h, h, H, H, r, eps, 0, P(ws), ws.numel(), P(st), sp) == 0, L.gf_last_error()
plain(); tape(); torch.cuda.synchronize()
print("out bitwise:", torch.equal(out, out2))
for a, b, n in zip(g1, g2, ("d_lr_x", "d_lr_y", "d_hr_x")):
    print(n, "max rel diff", float((a - b).abs().max() / b.abs().max()))
def t(f, n=10):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
print(f"plain step {t(plain):.3f} ms   tape step {t(tape):.3f} ms")
# tape via global loads (variant 12) vs tape + TMA gather window (default): bitwise
g3 = [torch.empty_like(lx), torch.empty_like(ly), torch.empty_like(hx)]
old = L.gf_joint_bwd_hr_variant(12)
assert L.gf_joint_bwd_tape(0, P(lx), P(ly), P(hx), P(A), P(d), P(g3[0]), P(g3[1]), P(g3[2]), B, C, h, h, H, H, r, eps, 0, P(ws), ws.numel(), P(st), sp) == 0
L.gf_joint_bwd_hr_variant(old)
torch.cuda.synchronize()
for a, b, n in zip(g2, g3, ("d_lr_x", "d_lr_y", "d_hr_x")):
    dd = (a - b).abs()
    print(n, "tile vs global-load tape: equal", torch.equal(a, b), "max", float(dd.max()),
          "where", [int(v) for v in torch.nonzero(dd == dd.max())[0]] if float(dd.max()) > 0 else None)
