"""Multi-GPU partitioning, checked on CPU with the oracle.

* batch shards cover the batch exactly once;
* row bands with the forward halo (r+1) and the backward halo
  (max(2r, r+1)) reproduce the full-image outputs and gradients exactly
  (to float64 rounding) on the owned rows;
* a world_size-2 gloo job runs the band forward and the data-parallel
  gradient allreduce through torch.distributed, like the NCCL path on GPUs.
"""

import os
import socket

import numpy as np
import pytest
import torch

from oracle import gf_oracle as O
from paper_1803_05619_b200.sharding import Band, allreduce_grads, batch_shard, halo, row_bands


def test_batch_shard_covers_batch():
    for batch in (1, 4, 7, 64):
        for world in (1, 2, 3, 8):
            seen = []
            for k in range(world):
                a, b = batch_shard(batch, world, k)
                assert 0 <= a <= b <= batch
                seen.extend(range(a, b))
            assert seen == list(range(batch))
            sizes = [batch_shard(batch, world, k)[1] - batch_shard(batch, world, k)[0]
                     for k in range(world)]
            assert max(sizes) - min(sizes) <= 1


def test_halo_values():
    assert halo(1, False) == 2 and halo(2, False) == 3
    assert halo(1, True) == 2 and halo(2, True) == 4 and halo(3, True) == 6


def _oracle_joint(lr_x, lr_y, hr_x, r, eps):
    return O.joint_forward_nchw(lr_x, lr_y, hr_x, r, eps)


@pytest.mark.parametrize("r", [1, 2, 3])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_row_bands_forward_exact(r, world):
    rng = np.random.default_rng(10 * r + world)
    h, w, C = 24, 20, 2
    lr_x = rng.uniform(0, 1, (1, C, h, w))
    lr_y = rng.uniform(0, 1, (1, C, h, w))
    hr_x = rng.uniform(0, 1, (1, C, 4 * h, 4 * w))
    full = _oracle_joint(lr_x, lr_y, hr_x, r, 1e-3)
    for band in row_bands(h, world, r, backward=False):
        lo, hi = band.crop_lo, band.crop_hi
        Hlo, Hhi = band.hr_crop
        out = _oracle_joint(lr_x[:, :, lo:hi], lr_y[:, :, lo:hi], hr_x[:, :, Hlo:Hhi], r, 1e-3)
        y0, y1 = band.hr_local
        A, B = band.hr_owned
        assert np.abs(out[:, :, y0:y1] - full[:, :, A:B]).max() <= 1e-12


@pytest.mark.parametrize("r", [1, 2, 3])
def test_row_bands_backward_exact(r):
    rng = np.random.default_rng(100 + r)
    h, w, C = 26, 18, 2
    lr_x = rng.uniform(0, 1, (1, C, h, w))
    lr_y = rng.uniform(0, 1, (1, C, h, w))
    hr_x = rng.uniform(0, 1, (1, C, 4 * h, 4 * w))
    d = rng.standard_normal((1, C, 4 * h, 4 * w))
    full = O.joint_backward_nchw(lr_x, lr_y, hr_x, d, r, 1e-3)
    for band in row_bands(h, 3, r, backward=True):
        lo, hi = band.crop_lo, band.crop_hi
        Hlo, Hhi = band.hr_crop
        g = O.joint_backward_nchw(lr_x[:, :, lo:hi], lr_y[:, :, lo:hi], hr_x[:, :, Hlo:Hhi],
                                  d[:, :, Hlo:Hhi], r, 1e-3)
        la, lb = band.lr_local
        ya, yb = band.hr_local
        assert np.abs(g[0][:, :, la:lb] - full[0][:, :, band.a:band.b]).max() <= 1e-10
        assert np.abs(g[1][:, :, la:lb] - full[1][:, :, band.a:band.b]).max() <= 1e-10
        A, B = band.hr_owned
        assert np.abs(g[2][:, :, ya:yb] - full[2][:, :, A:B]).max() <= 1e-10


def test_row_bands_forward_halo_is_not_enough_for_backward():
    """The r+1 halo is exact for out / d_hr but not for d_lr at r >= 2."""
    rng = np.random.default_rng(7)
    h, w, C, r = 24, 16, 1, 2
    lr_x, lr_y = rng.uniform(0, 1, (2, 1, C, h, w))
    hr_x = rng.uniform(0, 1, (1, C, 4 * h, 4 * w))
    d = rng.standard_normal((1, C, 4 * h, 4 * w))
    full = O.joint_backward_nchw(lr_x, lr_y, hr_x, d, r, 1e-3)
    worst = 0.0
    for band in row_bands(h, 2, r, backward=False):
        lo, hi = band.crop_lo, band.crop_hi
        Hlo, Hhi = band.hr_crop
        g = O.joint_backward_nchw(lr_x[:, :, lo:hi], lr_y[:, :, lo:hi], hr_x[:, :, Hlo:Hhi],
                                  d[:, :, Hlo:Hhi], r, 1e-3)
        la, lb = band.lr_local
        worst = max(worst, np.abs(g[0][:, :, la:lb] - full[0][:, :, band.a:band.b]).max())
    assert worst > 1e-6


# ---------------------------------------------------------------------------
# world_size-2 gloo job
# ---------------------------------------------------------------------------

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, tmpdir):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    rng = np.random.default_rng(0)  # identical inputs on every rank
    h, w, C, r = 20, 12, 2, 2
    lr_x = rng.uniform(0, 1, (1, C, h, w))
    lr_y = rng.uniform(0, 1, (1, C, h, w))
    hr_x = rng.uniform(0, 1, (1, C, 4 * h, 4 * w))
    band = row_bands(h, world, r, backward=False)[rank]
    lo, hi = band.crop_lo, band.crop_hi
    Hlo, Hhi = band.hr_crop
    out = O.joint_forward_nchw(lr_x[:, :, lo:hi], lr_y[:, :, lo:hi], hr_x[:, :, Hlo:Hhi], r, 1e-3)
    y0, y1 = band.hr_local
    mine = torch.from_numpy(np.ascontiguousarray(out[:, :, y0:y1]))
    gathered = [torch.zeros(1, C, 4 * (row_bands(h, world, r)[k].b - row_bands(h, world, r)[k].a),
                            4 * w, dtype=torch.float64) for k in range(world)]
    dist.all_gather(gathered, mine)
    # data-parallel gradient sum (the 95-float guidance-net gradient of config 2)
    g = torch.full((95,), float(rank + 1), dtype=torch.float64)
    allreduce_grads(g)
    if rank == 0:
        full = O.joint_forward_nchw(lr_x, lr_y, hr_x, r, 1e-3)
        err = float(np.abs(torch.cat(gathered, dim=2).numpy() - full).max())
        ok = err <= 1e-12 and bool(torch.all(g == float(sum(range(1, world + 1)))))
        with open(os.path.join(tmpdir, "result.txt"), "w") as f:
            f.write(f"{ok} {err}")
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_band_forward_and_allreduce(tmp_path):
    import torch.multiprocessing as mp

    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    ok, err = open(tmp_path / "result.txt").read().split()
    assert ok == "True", f"band forward mismatch {err}"


@pytest.mark.parametrize("h,world,r", [(4096, 8, 2), (4096, 3, 2), (1000, 8, 4), (517, 5, 1),
                                       (24, 4, 3), (7, 3, 1)])
def test_row_bands_partition_and_alignment(h, world, r):
    """Owned bands tile [0, h) in order; crops start on 16-row tiles (when the
    halo allows) and cover the backward halo."""
    from paper_1803_05619_b200.sharding import ALIGN, GRAIN

    bands = row_bands(h, world, r, backward=True)
    assert len(bands) == world and bands[0].a == 0 and bands[-1].b == h
    R = halo(r, True)
    for k, bd in enumerate(bands):
        if k:
            assert bd.a == bands[k - 1].b
        assert bd.crop_lo % ALIGN == 0
        assert bd.crop_lo <= max(0, bd.a - R) and bd.crop_hi == min(h, bd.b + R)
        if h >= GRAIN * world and bd.b < h:
            assert bd.b % GRAIN == 0


def test_joint_band_backward_helper_exact_on_oracle():
    """sharding.joint_band_backward with the oracle as the layer (no
    row_origin keyword) reproduces the full image's gradients."""
    from paper_1803_05619_b200.sharding import joint_band_backward

    rng = np.random.default_rng(11)
    h, w, C, r = 40, 12, 1, 2
    lr_x, lr_y = rng.uniform(0, 1, (2, 1, C, h, w))
    hr_x = rng.uniform(0, 1, (1, C, 4 * h, 4 * w))
    d = rng.standard_normal((1, C, 4 * h, 4 * w))
    full = O.joint_backward_nchw(lr_x, lr_y, hr_x, d, r, 1e-3)

    class _G:
        def __init__(self, g):
            self.d_guide_lo, self.d_src, self.d_guide_hi = g

    T = torch.from_numpy
    n = lambda t: t.numpy()  # noqa: E731

    def fwd(lx, hx, ly, p):
        return T(O.joint_forward_nchw(n(lx), n(ly), n(hx), r, 1e-3)), (n(lx), n(ly), n(hx))

    def bwd(tape, dd):
        lx, ly, hx = tape
        return _G([T(g) for g in O.joint_backward_nchw(lx, ly, hx, n(dd), r, 1e-3)])

    for band in row_bands(h, 2, r, backward=True):
        _, dlx, dly, dhx = joint_band_backward(fwd, bwd, None, T(lr_x), T(lr_y), T(hr_x), T(d),
                                               band)
        dlx, dly, dhx = n(dlx), n(dly), n(dhx)
        A, B = band.hr_owned
        assert np.abs(dlx - full[0][:, :, band.a:band.b]).max() <= 1e-10
        assert np.abs(dly - full[1][:, :, band.a:band.b]).max() <= 1e-10
        assert np.abs(dhx - full[2][:, :, A:B]).max() <= 1e-10


# ---------------------------------------------------------------------------
# data-parallel training loop (upsampler.train_loop), gloo world 2
# ---------------------------------------------------------------------------

def _fake_eval(i):
    """Deterministic per-image loss and packed gradients (stand-ins for the
    GPU model; the loop's scheduling and reduction are what is tested)."""
    g1 = torch.arange(5, dtype=torch.float64) * (i + 1)
    g2 = torch.full((3,), float(i * i), dtype=torch.float64)
    return torch.tensor(float(i) + 0.5, dtype=torch.float64), [g1, g2]


def _dp_worker(rank, world, port, tmpdir):
    import torch.distributed as dist

    from paper_1803_05619_b200.upsampler import train_loop

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    seen = []

    def update(step, grads):
        seen.append(torch.cat([g.clone() for g in grads]))

    hist = train_loop(3, 5, _fake_eval, update)
    torch.save({"hist": hist, "seen": seen}, os.path.join(tmpdir, f"r{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def test_train_loop_world1_is_reference_order():
    from paper_1803_05619_b200.upsampler import train_loop

    seen = []
    hist = train_loop(4, 3, _fake_eval, lambda s, g: seen.append(torch.cat(g)))
    # images in order, cycling (gf/training.py:240-262): 0 1 2 0, final 1
    assert hist == [0.5, 1.5, 2.5, 0.5, 1.5]
    assert torch.equal(seen[2], torch.cat(_fake_eval(2)[1]))


def test_gloo_world2_data_parallel_train_loop(tmp_path):
    """Global batch of 2 images per step (rank k: image 2*step + k), gradients
    and loss averaged by one all-reduce; both ranks see identical updates."""
    import torch.multiprocessing as mp

    port = _free_port()
    mp.spawn(_dp_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0, r1 = (torch.load(tmp_path / f"r{k}.pt") for k in (0, 1))
    assert r0["hist"] == r1["hist"]
    for a, b in zip(r0["seen"], r1["seen"]):
        assert torch.equal(a, b)
    n = 5
    for step in range(3):
        i, j = (2 * step) % n, (2 * step + 1) % n
        want = (torch.cat(_fake_eval(i)[1]) + torch.cat(_fake_eval(j)[1])) / 2
        assert torch.allclose(r0["seen"][step], want)
        assert r0["hist"][step] == pytest.approx((i + j + 1.0) / 2)
    assert len(r0["hist"]) == 4
