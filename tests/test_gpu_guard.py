"""Out-of-bounds guards for every kernel family (compute-sanitizer is not
available on the GPU pool, so the bounds checks are our own).

Each input lives inside a buffer whose guard bands are NaN (an out-of-bounds
read that reaches the arithmetic poisons the result), each output and the
workspace inside a buffer whose guard bands hold a sentinel pattern (an
out-of-bounds write changes it).  The guarded call must leave every guard
band bit-identical and produce exactly the bytes of an unguarded call.
Shapes are ragged (not multiples of the tile sizes) and the radii cover the
template range edges.
"""

import ctypes

import pytest
import torch

pytestmark = pytest.mark.gpu

GUARD = 4096  # elements on each side; keeps 16-byte alignment for the fused paths
SENTINEL = 1.2345e-30


@pytest.fixture(scope="module")
def lib():
    from paper_1803_05619_b200 import _lib

    assert torch.cuda.is_available(), "gpu tests need CUDA"
    return _lib.load()


class Guarded:
    def __init__(self, shape, dtype, fill, data=None):
        n = 1
        for s in shape:
            n *= int(s)
        self.n = n
        self.buf = torch.full((n + 2 * GUARD,), fill, dtype=dtype, device="cuda")
        self.view = self.buf[GUARD:GUARD + n].view(*shape)
        if data is not None:
            self.view.copy_(data)
        self.fill = fill

    @property
    def ptr(self):
        return self.view.data_ptr()

    def guards_intact(self):
        g = torch.cat([self.buf[:GUARD], self.buf[GUARD + self.n:]])
        if self.fill != self.fill:  # NaN guard
            return bool(torch.isnan(g).all())
        return bool((g == self.fill).all())


def gin(t):
    return Guarded(t.shape, t.dtype, float("nan"), t)


def gout(shape, dtype):
    return Guarded(shape, dtype, SENTINEL)


def gws(nbytes):
    nf = (max(int(nbytes), 16) + 7) // 8
    return Guarded((nf,), torch.float64, SENTINEL)


def status():
    return torch.zeros(1, dtype=torch.int32, device="cuda")


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def rc_ok(lib, rc):
    assert rc == 0, lib.gf_last_error().decode(errors="replace")


def dt_code(dtype):
    return 0 if dtype == torch.float32 else 1


def run_joint(lib, lr_x, lr_y, hr_x, d, r, eps, guarded):
    B, C, h, w = lr_x.shape
    H, W = hr_x.shape[2:]
    dt = dt_code(lr_x.dtype)
    wsb = lib.gf_joint_workspace_bytes(dt, B, C, h, w, H, W, r)
    if guarded:
        ins = [gin(t) for t in (lr_x, lr_y, hr_x, d)]
        outs = [gout(hr_x.shape, lr_x.dtype), gout(lr_x.shape, lr_x.dtype),
                gout(lr_x.shape, lr_x.dtype), gout(hr_x.shape, lr_x.dtype)]
        ws = gws(wsb)
        p = lambda g: g.ptr  # noqa: E731
    else:
        ins = [lr_x, lr_y, hr_x, d]
        outs = [torch.empty_like(hr_x), torch.empty_like(lr_x), torch.empty_like(lr_x),
                torch.empty_like(hr_x)]
        ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
        p = lambda t: t.data_ptr()  # noqa: E731
    st = status()
    rc_ok(lib, lib.gf_joint_fwd(dt, p(ins[0]), p(ins[1]), p(ins[2]), p(outs[0]), B, C, h, w,
                                H, W, r, eps, p(ws), wsb, st.data_ptr(), stream()))
    rc_ok(lib, lib.gf_joint_bwd(dt, p(ins[0]), p(ins[1]), p(ins[2]), p(ins[3]), p(outs[1]),
                                p(outs[2]), p(outs[3]), B, C, h, w, H, W, r, eps, p(ws), wsb,
                                st.data_ptr(), stream()))
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    if guarded:
        for g in ins + outs + [ws]:
            assert g.guards_intact()
        return [o.view.clone() for o in outs]
    return outs


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("h,w,r", [(37, 45, 0), (33, 17, 5), (21, 70, 12), (2, 3, 1),
                                   (130, 66, 3)])
def test_joint_guarded(lib, dtype, h, w, r):
    g = torch.Generator(device="cuda").manual_seed(h * 100 + w + r)
    mk = lambda *s: torch.rand(*s, generator=g, device="cuda", dtype=dtype)  # noqa: E731
    lr_x, lr_y = mk(2, 3, h, w), mk(2, 3, h, w)
    hr_x, d = mk(2, 3, 4 * h, 4 * w), mk(2, 3, 4 * h, 4 * w) - 0.5
    a = run_joint(lib, lr_x, lr_y, hr_x, d, r, 1e-3, guarded=True)
    b = run_joint(lib, lr_x, lr_y, hr_x, d, r, 1e-3, guarded=False)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


def test_joint_guarded_generic_ratio(lib):
    """Non-integer ratio: the general kernels."""
    g = torch.Generator(device="cuda").manual_seed(7)
    mk = lambda *s: torch.rand(*s, generator=g, device="cuda")  # noqa: E731
    lr_x, lr_y = mk(1, 3, 24, 19), mk(1, 3, 24, 19)
    hr_x, d = mk(1, 3, 51, 40), mk(1, 3, 51, 40)
    a = run_joint(lib, lr_x, lr_y, hr_x, d, 2, 1e-3, guarded=True)
    b = run_joint(lib, lr_x, lr_y, hr_x, d, 2, 1e-3, guarded=False)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


def run_highres(lib, guide, src, d, r, eps, guarded):
    B, Cg, H, W = guide.shape
    C = src.shape[1]
    dt = dt_code(src.dtype)
    wsb = lib.gf_highres_workspace_bytes(dt, B, Cg, C, H, W, r)
    if guarded:
        ins = [gin(t) for t in (guide, src, d)]
        outs = [gout(src.shape, src.dtype), gout(guide.shape, src.dtype),
                gout(src.shape, src.dtype)]
        ws = gws(wsb)
        p = lambda g: g.ptr  # noqa: E731
    else:
        ins = [guide, src, d]
        outs = [torch.empty_like(src), torch.empty_like(guide), torch.empty_like(src)]
        ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
        p = lambda t: t.data_ptr()  # noqa: E731
    st = status()
    rc_ok(lib, lib.gf_highres_fwd(dt, p(ins[0]), p(ins[1]), p(outs[0]), B, Cg, C, H, W, r, eps,
                                  p(ws), wsb, st.data_ptr(), stream()))
    rc_ok(lib, lib.gf_highres_bwd(dt, p(ins[0]), p(ins[1]), p(ins[2]), p(outs[1]), p(outs[2]),
                                  B, Cg, C, H, W, r, eps, p(ws), wsb, st.data_ptr(), stream()))
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    if guarded:
        for g in ins + outs + [ws]:
            assert g.guards_intact()
        return [o.view.clone() for o in outs]
    return outs


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("H,W,r,cg", [(77, 132, 1, 1), (40, 36, 16, 3), (5, 8, 2, 1),
                                      (300, 260, 8, 3), (9, 1030, 4, 1)])
def test_highres_guarded(lib, dtype, H, W, r, cg):
    g = torch.Generator(device="cuda").manual_seed(H * 10 + W + r)
    mk = lambda *s: torch.rand(*s, generator=g, device="cuda", dtype=dtype)  # noqa: E731
    guide, src, d = mk(2, cg, H, W), mk(2, 3, H, W), mk(2, 3, H, W) - 0.5
    a = run_highres(lib, guide, src, d, r, 1e-2, guarded=True)
    b = run_highres(lib, guide, src, d, r, 1e-2, guarded=False)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


@pytest.mark.parametrize("hidden", [4, 15, 16, 7])
def test_guidance_and_mse_guarded(lib, hidden):
    g = torch.Generator(device="cuda").manual_seed(hidden)
    B, H, W = 3, 37, 53
    x = torch.rand(B, 3, H, W, generator=g, device="cuda")
    dy = torch.rand(B, 3, H, W, generator=g, device="cuda") - 0.5
    npar = lib.gn_param_count(3, 3, hidden)
    params = torch.rand(npar, generator=g, device="cuda") - 0.5
    wsb = lib.gn_workspace_bytes(0, B, 3, 3, hidden, H, W)

    def once(guarded):
        if guarded:
            gx, gdy, gp = gin(x), gin(dy), gin(params)
            y, dx, dp = gout(x.shape, x.dtype), gout(x.shape, x.dtype), gout((npar,), x.dtype)
            dp.view.zero_()
            ws = gws(wsb)
            p = lambda t: t.ptr  # noqa: E731
        else:
            gx, gdy, gp = x, dy, params
            y, dx = torch.empty_like(x), torch.empty_like(x)
            dp = torch.zeros(npar, device="cuda")
            ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
            p = lambda t: t.data_ptr()  # noqa: E731
        st = status()
        rc_ok(lib, lib.gn_forward(0, p(gx), p(y), p(gp), B, 3, 3, hidden, H, W, p(ws), wsb,
                                  st.data_ptr(), stream()))
        rc_ok(lib, lib.gn_backward(0, p(gx), p(gdy), p(dx), p(dp), 0, p(gp), B, 3, 3, hidden,
                                   H, W, p(ws), wsb, st.data_ptr(), stream()))
        mwsb = lib.gf_mse_workspace_bytes(B, 3, H, W)
        dmse = gout(x.shape, x.dtype) if guarded else torch.empty_like(x)
        mws = gws(mwsb) if guarded else torch.empty(max(mwsb, 16), dtype=torch.uint8,
                                                     device="cuda")
        loss = torch.zeros(1, dtype=torch.float64, device="cuda")
        rc_ok(lib, lib.gf_mse_loss(0, p(y), p(gx), p(dmse), loss.data_ptr(), B, 3, H, W,
                                   p(mws), mwsb, stream()))
        torch.cuda.synchronize()
        assert int(st.item()) == 0
        outs = [y, dx, dp, dmse]
        if guarded:
            for t in [gx, gdy, gp, ws, mws] + outs:
                assert t.guards_intact()
            outs = [o.view.clone() for o in outs]
        return outs + [loss]

    for a, b in zip(once(True), once(False)):
        assert torch.equal(a, b)


def run_joint_mse(lib, lr_x, lr_y, hr_x, tgt, r, eps, guarded):
    B, C, h, w = lr_x.shape
    H, W = hr_x.shape[2:]
    dt = dt_code(lr_x.dtype)
    wsb = lib.gf_joint_mse_workspace_bytes(dt, B, C, h, w, H, W, r)
    if guarded:
        ins = [gin(t) for t in (lr_x, lr_y, hr_x, tgt)]
        outs = [gout((1,), torch.float64), gout(lr_x.shape, lr_x.dtype),
                gout(lr_x.shape, lr_x.dtype), gout(hr_x.shape, lr_x.dtype)]
        ws = gws(wsb)
        p = lambda g: g.ptr  # noqa: E731
    else:
        ins = [lr_x, lr_y, hr_x, tgt]
        outs = [torch.empty(1, dtype=torch.float64, device="cuda"), torch.empty_like(lr_x),
                torch.empty_like(lr_x), torch.empty_like(hr_x)]
        ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
        p = lambda t: t.data_ptr()  # noqa: E731
    st = status()
    rc_ok(lib, lib.gf_joint_mse_bwd(dt, p(ins[0]), p(ins[1]), p(ins[2]), p(ins[3]), p(outs[0]),
                                    p(outs[1]), p(outs[2]), p(outs[3]), B, C, h, w, H, W, r,
                                    eps, p(ws), wsb, st.data_ptr(), stream()))
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    if guarded:
        for g in ins + outs + [ws]:
            assert g.guards_intact()
        return [o.view.clone() for o in outs]
    return outs


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("h,w,r", [(37, 45, 0), (33, 17, 5), (2, 3, 1), (130, 66, 2),
                                   (21, 70, 12)])
def test_joint_mse_guarded(lib, dtype, h, w, r):
    """The fused training-step entry (fused kernel for fp32, the three-entry
    chain for fp64): guard bands intact, bytes equal to an unguarded call."""
    g = torch.Generator(device="cuda").manual_seed(h * 31 + w + r)
    mk = lambda *s: torch.rand(*s, generator=g, device="cuda", dtype=dtype)  # noqa: E731
    lr_x, lr_y = mk(2, 3, h, w), mk(2, 3, h, w)
    hr_x, tgt = mk(2, 3, 4 * h, 4 * w), mk(2, 3, 4 * h, 4 * w)
    a = run_joint_mse(lib, lr_x, lr_y, hr_x, tgt, r, 1e-3, guarded=True)
    b = run_joint_mse(lib, lr_x, lr_y, hr_x, tgt, r, 1e-3, guarded=False)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


def run_joint_tape(lib, lr_x, lr_y, hr_x, d, r, eps, guarded):
    """gf_joint_fwd_tape + gf_joint_bwd_tape (the slope tape and the TMA-staged
    gather window of the backward's hr pass) with every buffer guarded."""
    B, C, h, w = lr_x.shape
    H, W = hr_x.shape[2:]
    wsb = lib.gf_joint_workspace_bytes(0, B, C, h, w, H, W, r)
    if guarded:
        ins = [gin(t) for t in (lr_x, lr_y, hr_x, d)]
        outs = [gout(hr_x.shape, lr_x.dtype), gout(lr_x.shape, lr_x.dtype),
                gout(lr_x.shape, lr_x.dtype), gout(hr_x.shape, lr_x.dtype),
                gout(lr_x.shape, lr_x.dtype)]  # the last: the slope tape
        ws = gws(wsb)
        p = lambda g: g.ptr  # noqa: E731
    else:
        ins = [lr_x, lr_y, hr_x, d]
        outs = [torch.empty_like(hr_x), torch.empty_like(lr_x), torch.empty_like(lr_x),
                torch.empty_like(hr_x), torch.empty_like(lr_x)]
        ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
        p = lambda t: t.data_ptr()  # noqa: E731
    st = status()
    rc_ok(lib, lib.gf_joint_fwd_tape(0, p(ins[0]), p(ins[1]), p(ins[2]), p(outs[0]), p(outs[4]),
                                     B, C, h, w, H, W, r, eps, p(ws), wsb, st.data_ptr(),
                                     stream()))
    rc_ok(lib, lib.gf_joint_bwd_tape(0, p(ins[0]), p(ins[1]), p(ins[2]), p(outs[4]), p(ins[3]),
                                     p(outs[1]), p(outs[2]), p(outs[3]), B, C, h, w, H, W, r, eps,
                                     0, p(ws), wsb, st.data_ptr(), stream()))
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    if guarded:
        for g in ins + outs + [ws]:
            assert g.guards_intact()
        return [o.view.clone() for o in outs]
    return outs


@pytest.mark.parametrize("h,w,r", [(37, 44, 0), (33, 16, 5), (21, 72, 12), (2, 4, 1),
                                   (130, 68, 3), (16, 32, 2)])
def test_joint_tape_guarded(lib, h, w, r):
    g = torch.Generator(device="cuda").manual_seed(h * 100 + w + r)
    mk = lambda *s: torch.rand(*s, generator=g, device="cuda")  # noqa: E731
    lr_x, lr_y = mk(2, 3, h, w), mk(2, 3, h, w)
    hr_x, d = mk(2, 3, 4 * h, 4 * w), mk(2, 3, 4 * h, 4 * w) - 0.5
    a = run_joint_tape(lib, lr_x, lr_y, hr_x, d, r, 1e-3, guarded=True)
    b = run_joint_tape(lib, lr_x, lr_y, hr_x, d, r, 1e-3, guarded=False)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    # against the moments-recomputing backward: out and d_lr bitwise (the low-res
    # tail recomputes), d_hr to fp32 rounding of the slopes (a tile's halo
    # slopes come from the neighbouring tile, computed with its own shift; at
    # r = 0 the exact slope is 0 and both are rounding noise ~ 1e-7 / eps)
    c = run_joint(lib, lr_x, lr_y, hr_x, d, r, 1e-3, guarded=False)
    assert torch.equal(a[0], c[0]) and torch.equal(a[1], c[1]) and torch.equal(a[2], c[2])
    tol = 1e-5 * float(c[3].abs().max()) + 1e-4 * float(d.abs().max())
    assert float((a[3] - c[3]).abs().max()) <= tol
