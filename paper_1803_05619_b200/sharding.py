"""Multi-GPU partitioning of the guided-filter path.

The layer has no parameters and no cross-image coupling, so it shards with
no data-path collective:

* **batch shards** (config 4a): rank k owns images [start, end) of the batch;
* **row bands** (config 4b): rank k owns low-res rows [a, b) of one image
  (high-res rows [4a, 4b) for the factor-4 fast path) and computes the layer
  on an *aligned crop* with a low-res halo:
    - forward: halo r + 1 (r for the box window, 1 for the bilinear taps);
    - backward: halo R = max(2r, r + 1) so the owned d_lr rows are exact
      (M^T needs the moment gradients at [a-r, b+r), whose moments need the
      inputs at [a-2r, b+2r)).
  The crop's high-res rows are exactly factor x its low-res rows, so every
  owned output row sees the same taps and windows as in the full image.
  Crops are clamped to the image, so window counts stay those of the image.
  Verified exact against the oracle in tests/test_sharding.py.
  Band edges fall on multiples of ``GRAIN`` (64) low-res rows -- the row
  pieces of the fp32 backward tail -- and the crop's first row is rounded
  down to a multiple of ``ALIGN`` (16) -- the row tiling of the fused fp32
  kernels; the crop's full-image row is handed to the layer (``forward_joint(...,
  row_origin=crop_lo)``), so every tile, row piece and shift constant of the
  fp32 kernels sits where it sits for the whole image: a band's owned rows
  are BITWISE equal to the 1-GPU result (tests/test_gpu_fullsize.py).

The only collective on the path is the data-parallel training step
(config 2): the packed 95-float guidance-net gradient is summed across ranks
(``allreduce_grads``; NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


def batch_shard(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [start, end) images of ``rank`` (possibly empty)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


@dataclass(frozen=True)
class Band:
    """Row band of one rank: owned low-res rows [a, b) and the crops."""

    a: int
    b: int
    crop_lo: int      # low-res crop [crop_lo, crop_hi)
    crop_hi: int
    factor: int

    @property
    def hr_owned(self) -> tuple[int, int]:
        return self.a * self.factor, self.b * self.factor

    @property
    def hr_crop(self) -> tuple[int, int]:
        return self.crop_lo * self.factor, self.crop_hi * self.factor

    @property
    def lr_local(self) -> tuple[int, int]:
        """Owned low-res rows inside the crop."""
        return self.a - self.crop_lo, self.b - self.crop_lo

    @property
    def hr_local(self) -> tuple[int, int]:
        """Owned high-res rows inside the high-res crop."""
        return (self.a - self.crop_lo) * self.factor, (self.b - self.crop_lo) * self.factor


ALIGN = 16  # low-res rows per tile row of the fused fp32 kernels (jf::TLY)
GRAIN = 64  # low-res rows per row piece of the backward tail (jls::kPiece)
PIECE = 16  # low-res rows per piece of the forward's coefficient walk (jcs::kPiece)


def halo(radius: int, backward: bool) -> int:
    return max(2 * radius, radius + 1) if backward else radius + 1


def row_bands(h: int, world: int, radius: int, factor: int = 4, backward: bool = True,
              align: int = ALIGN, grain: int = GRAIN):
    """Bands of ``world`` ranks over ``h`` low-res rows, balanced in units of
    ``grain`` rows (the backward's row pieces: owned rows then start where a
    piece of the full image starts) when h >= grain * world, else of single
    rows; every crop starts on a multiple of ``align`` rows (a tile row)."""
    if align < 1 or grain < 1:
        raise ValueError(f"align and grain must be >= 1, got {align}, {grain}")
    out = []
    R = halo(radius, backward)
    g = grain if h >= grain * world else 1
    units = -(-h // g)
    for k in range(world):
        ua, ub = batch_shard(units, world, k)
        a, b = min(h, ua * g), min(h, ub * g)
        # the two-kernel forward's coefficient walk restarts its running sums
        # at rows 16 j - 1: the piece holding row a - 1 (the first coefficient
        # row the band's bilinear taps read) needs its r warm-up rows in the crop
        piece = (a // PIECE) * PIECE - 1
        lo = max(0, min(a - R, piece - radius)) // align * align
        out.append(Band(a, b, lo, min(h, b + R), factor))
    return out


def allreduce_grads(dparams: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the packed guidance-net gradient over the data-parallel ranks."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(dparams, op=dist.ReduceOp.SUM, group=group)
    return dparams


def joint_band_forward(forward_joint, params, lr_x, lr_y, hr_x, band: Band):
    """Run a joint forward on the band's crop; returns the owned output rows.

    ``forward_joint`` is the layer function (the GPU one in production, the
    oracle in the CPU tests); tensors are NCHW with full-image rows.
    """
    lo, hi = band.crop_lo, band.crop_hi
    Hlo, Hhi = band.hr_crop
    out, _ = forward_joint(lr_x[:, :, lo:hi].contiguous(), hr_x[:, :, Hlo:Hhi].contiguous(),
                           lr_y[:, :, lo:hi].contiguous(), params,
                           **_origin(forward_joint, lo, lr_x.shape[2]))
    y0, y1 = band.hr_local
    return out[:, :, y0:y1]


def _origin(fn, lo: int, h_full: int) -> dict:
    """row_origin / full_rows for the GPU layer (the oracle in the CPU tests
    has neither)."""
    import inspect

    try:
        params = inspect.signature(fn).parameters
    except (TypeError, ValueError):
        return {}
    kw = {}
    if "row_origin" in params:
        kw["row_origin"] = lo
    if "full_rows" in params:
        kw["full_rows"] = h_full
    return kw


def joint_band_backward(forward_joint, backward, params, lr_x, lr_y, hr_x, d_out, band: Band):
    """Forward + backward of one band; returns (out, d_lr_x, d_lr_y, d_hr_x)
    restricted to the band's owned rows.  ``d_out`` has full-image rows."""
    lo, hi = band.crop_lo, band.crop_hi
    Hlo, Hhi = band.hr_crop
    out, tape = forward_joint(lr_x[:, :, lo:hi].contiguous(), hr_x[:, :, Hlo:Hhi].contiguous(),
                              lr_y[:, :, lo:hi].contiguous(), params,
                              **_origin(forward_joint, lo, lr_x.shape[2]))
    g = backward(tape, d_out[:, :, Hlo:Hhi].contiguous())
    y0, y1 = band.hr_local
    l0, l1 = band.lr_local
    return (out[:, :, y0:y1], g.d_guide_lo[:, :, l0:l1], g.d_src[:, :, l0:l1],
            g.d_guide_hi[:, :, y0:y1])
