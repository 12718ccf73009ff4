"""PCIe ceiling for the e2e legs: pinned H2D / D2H alone and overlapped, at
the cfg1 per-step byte counts (CUDA events, best of 5)."""
import torch

def t(fn, n=5):
    best = 1e9
    for _ in range(n):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize(); a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best

hi = 268435456 // 4; lo = 201326592 // 4
hin = torch.empty(hi).pin_memory(); din = torch.empty(hi, device="cuda")
dout = torch.empty(lo, device="cuda"); hout = torch.empty(lo).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2d = t(lambda: din.copy_(hin, non_blocking=True))
d2h = t(lambda: hout.copy_(dout, non_blocking=True))
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): din.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2): hout.copy_(dout, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
bo = t(both)
def chunked(nb=16):
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    with torch.cuda.stream(s1):
        for i in range(nb):
            din[i*hi//nb:(i+1)*hi//nb].copy_(hin[i*hi//nb:(i+1)*hi//nb], non_blocking=True)
    cur.wait_stream(s1)
ch = t(chunked)
print(f"h2d {h2d:.3f} ms ({hi*4/h2d/1e6:.1f} GB/s)  d2h {d2h:.3f} ms ({lo*4/d2h/1e6:.1f} GB/s)  "
      f"overlapped {bo:.3f} ms  h2d in 16 chunks {ch:.3f} ms")
