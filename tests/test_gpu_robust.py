"""Robustness of the boundary:

* unaligned buffers (offset by 4 bytes) on a shape the fused kernels cover:
  the C ABI must either run the general kernels inside the caller's
  workspace or refuse with GF_ERR_WORKSPACE -- never write past it;
* the Python mirror hands unaligned batch slices to the fused kernels as
  aligned copies and still matches the aligned call;
* an in-place edit of a forward input between forward and backward raises;
* two devices / two threads: launches configure each device independently
  (launch_cfg is keyed by device), and host entries on two threads give the
  single-thread result.
"""

import ctypes
import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_1803_05619_b200 import _lib

    assert torch.cuda.is_available(), "gpu tests need CUDA"
    return _lib.load()


def _sp():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _unaligned(t, guard=1024, fill=float("nan")):
    """Copy of t starting 4 bytes past a 16-byte boundary, inside a NaN/sentinel band."""
    n = t.numel()
    buf = torch.full((n + 2 * guard + 1,), fill, dtype=t.dtype, device="cuda")
    v = buf[guard + 1:guard + 1 + n].view(t.shape)
    v.copy_(t)
    assert v.data_ptr() % 16 == 4
    return buf, v


def _joint_inputs(B=2, C=3, h=24, w=36, f=4, seed=0):
    import workloads

    return workloads.joint_inputs(B, C, h * f, w * f, f, seed=seed, device="cuda")


def test_unaligned_joint_bwd_small_workspace_is_refused(lib):
    from paper_1803_05619_b200 import _lib

    lr_x, lr_y, hr_x = _joint_inputs()
    B, C, h, w = lr_x.shape
    H, W = hr_x.shape[2:]
    assert lib.gf_joint_is_fused(0, B, C, h, w, H, W, 1)
    fused_need = lib.gf_joint_workspace_bytes(0, B, C, h, w, H, W, 1)
    SENT = 1.2345e-30
    guard = 4096
    ws_buf = torch.full((fused_need // 4 + 2 * guard,), SENT, device="cuda")
    ws = ws_buf[guard:guard + fused_need // 4]
    _, ulx = _unaligned(lr_x)
    d = torch.randn_like(hr_x)
    outs = [torch.empty_like(lr_x), torch.empty_like(lr_y), torch.empty_like(hr_x)]
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    rc = lib.gf_joint_bwd(0, ulx.data_ptr(), lr_y.data_ptr(), hr_x.data_ptr(), d.data_ptr(),
                          *[o.data_ptr() for o in outs], B, C, h, w, H, W, 1, 1e-8,
                          ws.data_ptr(), fused_need, st.data_ptr(), _sp())
    assert rc == _lib.GF_ERR_WORKSPACE, lib.gf_last_error()
    assert b"general kernels" in lib.gf_last_error()
    torch.cuda.synchronize()
    assert bool((ws_buf[:guard] == SENT).all()) and bool((ws_buf[guard + ws.numel():] == SENT).all())


def test_unaligned_joint_fwd_mse_bwd_refused_or_correct(lib):
    """gf_joint_fwd / gf_joint_mse_bwd / gf_highres_fwd on unaligned pointers:
    with the aligned (fused) workspace size the call is refused; with the
    general size it runs and matches the aligned call."""
    from paper_1803_05619_b200 import _lib

    lr_x, lr_y, hr_x = _joint_inputs(seed=3)
    B, C, h, w = lr_x.shape
    H, W = hr_x.shape[2:]
    _, uhx = _unaligned(hr_x)
    out_buf, uout = _unaligned(torch.zeros_like(hr_x), fill=1.2345e-30)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    rc = lib.gf_joint_fwd(0, lr_x.data_ptr(), lr_y.data_ptr(), uhx.data_ptr(), uout.data_ptr(),
                          B, C, h, w, H, W, 1, 1e-8, 0, 0, st.data_ptr(), _sp())
    assert rc == _lib.GF_ERR_WORKSPACE
    # general workspace: force the general size via the generic hook
    old = lib.gf_force_generic(1)
    try:
        gen = lib.gf_joint_workspace_bytes(0, B, C, h, w, H, W, 1)
        gen_mse = lib.gf_joint_mse_workspace_bytes(0, B, C, h, w, H, W, 1)
    finally:
        lib.gf_force_generic(old)
    ws = torch.empty(gen, dtype=torch.uint8, device="cuda")
    rc = lib.gf_joint_fwd(0, lr_x.data_ptr(), lr_y.data_ptr(), uhx.data_ptr(), uout.data_ptr(),
                          B, C, h, w, H, W, 1, 1e-8, ws.data_ptr(), gen, st.data_ptr(), _sp())
    assert rc == 0, lib.gf_last_error()
    ref = torch.empty_like(hr_x)
    rc = lib.gf_joint_fwd(0, lr_x.data_ptr(), lr_y.data_ptr(), hr_x.data_ptr(), ref.data_ptr(),
                          B, C, h, w, H, W, 1, 1e-8, 0, 0, st.data_ptr(), _sp())
    assert rc == 0
    torch.cuda.synchronize()
    assert float((uout - ref).abs().max()) < 2e-5
    assert bool((out_buf[:1025] == 1.2345e-30).all())
    # the fused training step on an unaligned target
    tgt = (1.5 * hr_x - 0.25).clamp(0, 1)
    _, utgt = _unaligned(tgt)
    fused_mse = lib.gf_joint_mse_workspace_bytes(0, B, C, h, w, H, W, 1)
    ws2 = torch.empty(fused_mse, dtype=torch.uint8, device="cuda")
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    grads = [torch.empty_like(lr_x), torch.empty_like(lr_y), torch.empty_like(hr_x)]
    args = (lr_x.data_ptr(), lr_y.data_ptr(), hr_x.data_ptr(), utgt.data_ptr(), loss.data_ptr(),
            *[g.data_ptr() for g in grads], B, C, h, w, H, W, 1, 1e-8)
    rc = lib.gf_joint_mse_bwd(0, *args, ws2.data_ptr(), fused_mse, st.data_ptr(), _sp())
    assert rc == _lib.GF_ERR_WORKSPACE
    ws3 = torch.empty(gen_mse, dtype=torch.uint8, device="cuda")
    rc = lib.gf_joint_mse_bwd(0, *args, ws3.data_ptr(), gen_mse, st.data_ptr(), _sp())
    assert rc == 0, lib.gf_last_error()
    loss_u = float(loss.item())
    rc = lib.gf_joint_mse_bwd(0, lr_x.data_ptr(), lr_y.data_ptr(), hr_x.data_ptr(),
                              tgt.data_ptr(), loss.data_ptr(), *[g.data_ptr() for g in grads],
                              B, C, h, w, H, W, 1, 1e-8, ws2.data_ptr(), fused_mse,
                              st.data_ptr(), _sp())
    assert rc == 0
    assert abs(loss_u - float(loss.item())) <= 1e-6 * abs(loss_u)


def test_unaligned_highres_fwd_refused_without_workspace(lib):
    from paper_1803_05619_b200 import _lib
    import workloads

    g, s = workloads.highres_inputs(1, 3, 64, 64, seed=1, device="cuda")
    _, us = _unaligned(s)
    out = torch.empty_like(s)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    rc = lib.gf_highres_fwd(0, g.data_ptr(), us.data_ptr(), out.data_ptr(), 1, 1, 3, 64, 64, 8,
                            1e-2, 0, 0, st.data_ptr(), _sp())
    assert rc == _lib.GF_ERR_WORKSPACE


def test_python_mirror_realigns_batch_slices():
    import paper_1803_05619_b200 as gfb

    # odd C*h*w: lr[1:] starts 4 bytes past an aligned boundary
    lr_x, lr_y, hr_x = _joint_inputs(B=3, h=5, w=7, seed=5)
    assert lr_x[1:].data_ptr() % 16 != 0
    p = gfb.GuidedFilterParams(1, 1e-4)
    out_s, tape_s = gfb.forward_joint(lr_x[1:], hr_x[1:], lr_y[1:], p)
    out_c, tape_c = gfb.forward_joint(lr_x[1:].clone(), hr_x[1:].clone(), lr_y[1:].clone(), p)
    assert torch.equal(out_s, out_c)
    d = torch.randn_like(out_s)
    gs, gc = gfb.backward(tape_s, d), gfb.backward(tape_c, d)
    for a, b in zip((gs.d_src, gs.d_guide_lo, gs.d_guide_hi), (gc.d_src, gc.d_guide_lo,
                                                              gc.d_guide_hi)):
        assert torch.equal(a, b)


def test_inplace_edit_between_forward_and_backward_raises():
    import paper_1803_05619_b200 as gfb

    lr_x, lr_y, hr_x = _joint_inputs(B=1, h=16, w=16, seed=2)
    p = gfb.GuidedFilterParams(1, 1e-4)
    out, tape = gfb.forward_joint(lr_x, hr_x, lr_y, p)
    gfb.backward(tape, out)  # unmodified: fine
    hr_x.mul_(0.5)
    with pytest.raises(RuntimeError, match="modified in place"):
        gfb.backward(tape, out)


def test_host_entries_on_two_threads_match_one_thread():
    import paper_1803_05619_b200 as gfb

    lr_x, lr_y, hr_x = [t.cpu() for t in _joint_inputs(B=2, h=64, w=64, seed=7)]
    p = gfb.GuidedFilterParams(2, 1e-4)
    ref = gfb.forward_joint_host(lr_x, hr_x, lr_y, p)
    res = [None] * 4
    errs = []

    def run(k):
        try:
            for _ in range(3):
                res[k] = gfb.forward_joint_host(lr_x, hr_x, lr_y, p)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=run, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for r in res:
        assert torch.equal(r, ref)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_second_device_gets_its_own_launch_config():
    import paper_1803_05619_b200 as gfb
    import workloads

    p = gfb.GuidedFilterParams(8, 1e-2)
    outs = []
    for dev in (0, 1):
        with torch.cuda.device(dev):
            g, s = workloads.highres_inputs(1, 3, 256, 256, seed=0, device=f"cuda:{dev}")
            o, _ = gfb.forward_highres(g, s, p)
            outs.append(o.cpu())
    assert torch.equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[0].numpy(), outs[1].numpy())
