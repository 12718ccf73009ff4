import sys, torch
sys.path.insert(0, ".")
import workloads
from paper_1803_05619_b200 import _lib
L = _lib.load()
B, C, H, r, eps = 2, 3, 1024, 2, 1e-4
h = H // 4
lx, ly, hx = workloads.joint_inputs(B, C, H, H, seed=3, device="cuda")
d = torch.randn_like(hx)
out = torch.empty_like(hx); A = torch.empty_like(lx)
g = [torch.empty_like(lx), torch.empty_like(lx), torch.empty_like(hx)]
ws = torch.empty(L.gf_joint_workspace_bytes(0, B, C, h, h, H, H, r), dtype=torch.uint8, device="cuda")
st = torch.zeros(1, dtype=torch.int32, device="cuda")
P = lambda t: t.data_ptr()
def run(sp):
    assert L.gf_joint_fwd_tape(0, P(lx), P(ly), P(hx), P(out), P(A), B, C, h, h, H, H, r, eps, P(ws), ws.numel(), P(st), sp) == 0, L.gf_last_error()
    assert L.gf_joint_bwd_tape(0, P(lx), P(ly), P(hx), P(A), P(d), P(g[0]), P(g[1]), P(g[2]), B, C, h, h, H, H, r, eps, 0, P(ws), ws.numel(), P(st), sp) == 0, L.gf_last_error()
L.gf_joint_fwd_mode(2)
run(torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
ref = [out.clone()] + [t.clone() for t in g]
for t in [out] + g: t.zero_()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    run(s.cuda_stream)  # warm-up on the side stream (occupancy / attribute calls happen here)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=s):
    run(torch.cuda.current_stream().cuda_stream)
for t in [out] + g: t.zero_()
graph.replay(); graph.replay()
torch.cuda.synchronize()
print("graph replay equals eager:", all(torch.equal(a, b) for a, b in zip(ref, [out] + g)), "status", int(st.item()))
