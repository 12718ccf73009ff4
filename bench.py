"""Benchmark driver for the B200 guided-filter layer.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4a] [--impl ours|reference]

Prints ONE JSON line (rank 0) on stdout.  Default workload: BASELINE.json
configs[4](a), the largest single-GPU configuration and the batch-sharded
multi-GPU one: joint (fast) guided filter forward + backward over a batch of
64 images of 3 x 3072^2 (low-res 3 x 768^2), r=2, eps=1e-4, fp32, the batch
split over the N ranks (strong scaling).  Other configs: cfg0 (joint fwd
1024^2), cfg1 (full-res fwd 4 x 2048^2, r=8), cfg2 (training step), cfg3
(joint fwd sweep point, --hr/--batch/--radius), cfg4b (one 16384^2 image in
row bands).  Inputs are seeded synthetic data with the configs' shapes and
value distributions (workloads.py).

* ``--gpus N`` without a torchrun environment re-launches itself under
  ``torch.distributed.run`` with N ranks (one process per GPU, NCCL,
  NCCL_DEBUG=INFO to stderr so the communicator lines show the rank count).
* ``value``: whole-job output Mpix/s with inputs resident in HBM, timed with
  CUDA events on the launching stream over exactly K steps bracketed by a
  barrier + synchronize, max over ranks.  A "step" is one call of the layer
  (forward, or forward + backward) over the rank's share of the batch.
* ``e2e``: the same metric through the public host API with pinned HOST
  buffers, every input copied in and every output copied out inside the
  timed region (forward + backward: ``forward_backward_joint_host``, which
  pipelines copy-in / kernels / copy-out plane by plane).
* ``roofline``: algorithmic bytes per step / the CUDA-event step
  time, against the measured HBM copy peak (MEASURED_PEAKS.json).
* ``cpu_baseline``: the reference's own CPU path (the unmodified
  ``guidedfilter`` package with its numba kernels, baseline/_ref) on all host
  cores, one process per image (cpu_reference.py); rank 0, N=1 only.
* ``--impl reference``: the same CPU reference on the same config, metric and
  unit, bounded per-step samples; rank 0 only under torchrun.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "guided-filter output Mpix/s (fwd, fwd+bwd) and % of HBM roofline"

from paper_1803_05619_b200.sharding import allreduce_grads, batch_shard, row_bands  # noqa: E402


# ---------------------------------------------------------------------------
# workload descriptions
# ---------------------------------------------------------------------------

def workload_spec(args):
    from workloads import CONFIGS

    c = dict(CONFIGS[args.config])
    if args.batch:
        c["batch"] = args.batch
    if args.hr:
        c["hr"] = args.hr
    if args.radius is not None:
        c["r"] = args.radius
    return c


def algorithmic_bytes(c):
    """SURVEY 8(d) compulsory bytes per step, fp32."""
    B, C, H = c["batch"], c["channels"], c["hr"]
    hw = H * H
    if c["kind"] == "highres_fwd":
        return 4 * B * (1 + 2 * C) * hw
    h = H // c["factor"]
    lw = h * h
    if c["kind"] == "joint_fwd":
        return 4 * B * C * (2 * hw + 2 * lw)
    if c["kind"] == "joint_fwd_bwd":
        return 4 * B * C * (2 * hw + 2 * lw) + 4 * B * C * (3 * hw + 4 * lw)
    if c["kind"] == "train_step":
        return 4 * B * C * (4 * hw + 4 * lw)
    raise ValueError(c["kind"])


# ---------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                mx.append(float(s[1]))
            except ValueError:
                continue
            for n, v in zip(names, s[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def ncu_traffic(config_name):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    capture summary (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(config_name)
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
# our implementation
# ---------------------------------------------------------------------------

class OursStep:
    """Device-resident inputs; one step = one C-ABI layer call (plus, for the
    training config, the full pipeline)."""

    def __init__(self, c, device, seed, rank=0, world=1):
        import torch

        import workloads
        from paper_1803_05619_b200 import _lib

        self.c, self.device, self.world = c, device, world
        self.lib = _lib.load()
        self.stream = torch.cuda.current_stream(device)
        self.sp = self.stream.cuda_stream
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        B, C, H = c["batch"], c["channels"], c["hr"]
        self.pixels = B * H * H
        kind = c["kind"]
        self.kind = kind
        g = torch.Generator(device="cpu").manual_seed(seed)
        if kind == "highres_fwd":
            guide, src = workloads.highres_inputs(B, C, H, H, seed=seed, device=device)
            self.inputs = [guide, src]
            self.out = torch.empty_like(src)
            fused = self.lib.gf_highres_fwd_is_fused(0, B, 1, C, H, H, c["r"])
            nb = 16 if fused else self.lib.gf_highres_workspace_bytes(0, B, 1, C, H, H, c["r"])
            self.ws = torch.empty(nb, dtype=torch.uint8, device=device)
            # generic path: products, 4x(box_v, box_h), coeffs, 2 copies, 2x2 box, apply
            self.launches = 1 if fused else 17
        else:
            f = c["factor"]
            self.scaling = c.get("scaling", "weak")
            if c.get("shard") == "batch":  # config 4a: the batch is split over ranks
                b0, b1 = batch_shard(B, world, rank)
                B = b1 - b0
            lr_x, lr_y, hr_x = workloads.joint_inputs(B, C, H, H, f, seed=seed, device=device)
            self.B, self.H, self.W = B, H, H
            self.pixels = B * H * H
            if c.get("shard") == "rows":  # config 4b: row bands with the backward halo
                band = row_bands(H // f, world, c["r"], factor=f, backward=True)[rank]
                lo, hi = band.crop_lo, band.crop_hi
                self.row0 = lo  # full-image row of the crop: bitwise band results
                Hlo, Hhi = band.hr_crop
                lr_x = lr_x[:, :, lo:hi].contiguous()
                lr_y = lr_y[:, :, lo:hi].contiguous()
                hr_x = hr_x[:, :, Hlo:Hhi].contiguous()
                self.H = Hhi - Hlo
                A0, A1 = band.hr_owned
                self.pixels = B * (A1 - A0) * H  # owned output rows only
                torch.cuda.empty_cache()
            self.inputs = [lr_x, lr_y, hr_x]
            self.row0 = getattr(self, "row0", 0)
            self.h, self.w = self.H // f, self.W // f
            self.out = torch.empty_like(hr_x)
            nb = self.lib.gf_joint_workspace_bytes(0, B, C, self.h, self.w, self.H, self.W, c["r"])
            self.ws = torch.empty(max(nb, 16), dtype=torch.uint8, device=device)
            if kind in ("joint_fwd_bwd", "train_step"):
                self.d_out = torch.randn(hr_x.shape, generator=g).to(device)
                self.slope = torch.empty_like(lr_x)  # the tape's low-res slopes
                self.d_lr_x = torch.empty_like(lr_x)
                self.d_lr_y = torch.empty_like(lr_y)
                self.d_hr_x = torch.empty_like(hr_x)
            if kind == "train_step":
                import numpy as np

                import paper_1803_05619_b200 as gfb

                self.net = gfb.GuidanceNet(3, 3, hidden=c["hidden"], kernel=1,
                                           rng=np.random.default_rng(seed), device=device)
                self.target = workloads.affine_target(hr_x).contiguous()
                self.params = gfb.GuidedFilterParams(c["r"], c["eps"])
            fused = self.lib.gf_joint_is_fused(0, B, C, self.h, self.w, self.H, self.W, c["r"])
            # large calls: the two-kernel forward (coefficients, apply pass)
            split = fused and B * C * self.H * self.W >= self.lib.gf_joint_split_threshold()
            fwd = (2 if split else 1) if fused else 12
            bwd = 2 if fused else 26
            # train step: 2 x (stats, norm, fwd) guidance, the fused GF fwd + MSE +
            # bwd (hr pass, loss sum, lr tail; unfused: GF fwd, mse (2), GF bwd),
            # 2 x (bwd1, sum1, dx, dw1, final) guidance backward (the forward's
            # statistics are reused)
            gf_step = (4 if split else 3) if fused else fwd + 2 + bwd
            self.launches = {"joint_fwd": fwd, "joint_fwd_bwd": fwd + bwd,
                             "train_step": 2 * 3 + gf_step + 2 * 5}[kind]

    def step(self):
        c, L = self.c, self.lib
        B, C, H, r, eps = c["batch"], c["channels"], c["hr"], c["r"], c["eps"]
        if self.kind == "highres_fwd":
            g, s = self.inputs
            rc = L.gf_highres_fwd(0, g.data_ptr(), s.data_ptr(), self.out.data_ptr(), B, 1, C, H,
                                  H, r, eps, self.ws.data_ptr(), self.ws.numel(),
                                  self.status.data_ptr(), self.sp)
            assert rc == 0, L.gf_last_error()
        elif self.kind in ("joint_fwd", "joint_fwd_bwd"):
            lx, ly, hx = self.inputs
            B, h, w, Hh, Ww = self.B, self.h, self.w, self.H, self.W
            if self.kind == "joint_fwd":
                rc = L.gf_joint_fwd(0, lx.data_ptr(), ly.data_ptr(), hx.data_ptr(),
                                    self.out.data_ptr(), B, C, h, w, Hh, Ww, r, eps,
                                    self.ws.data_ptr(), self.ws.numel(), self.status.data_ptr(),
                                    self.sp)
                assert rc == 0, L.gf_last_error()
            else:  # forward keeping the tape's slopes, backward on them (forward_joint/backward)
                rc = L.gf_joint_fwd_tape(0, lx.data_ptr(), ly.data_ptr(), hx.data_ptr(),
                                         self.out.data_ptr(), self.slope.data_ptr(), B, C, h, w,
                                         Hh, Ww, r, eps, self.ws.data_ptr(), self.ws.numel(),
                                         self.status.data_ptr(), self.sp)
                assert rc == 0, L.gf_last_error()
                rc = L.gf_joint_bwd_tape(0, lx.data_ptr(), ly.data_ptr(), hx.data_ptr(),
                                         self.slope.data_ptr(), self.d_out.data_ptr(),
                                         self.d_lr_x.data_ptr(), self.d_lr_y.data_ptr(),
                                         self.d_hr_x.data_ptr(), B, C, h, w, Hh, Ww, r, eps,
                                         self.row0, self.ws.data_ptr(), self.ws.numel(),
                                         self.status.data_ptr(), self.sp)
                assert rc == 0, L.gf_last_error()
        else:  # train_step
            import paper_1803_05619_b200 as gfb

            lx, ly, hx = self.inputs
            self.res = gfb.train_step(self.net, lx, hx, ly, self.target, self.params)
            if self.world > 1:  # data-parallel: the 95-float gradient sum (NCCL)
                allreduce_grads(self.res.dparams)

    def e2e(self, steps, warmup):
        """Public API with pinned HOST buffers: every input of the step copied
        in and every output copied out inside the timed region (host wall
        clock around synchronous calls)."""
        import torch

        import paper_1803_05619_b200 as gfb

        c = self.c
        host_in = [t.cpu().pin_memory() for t in self.inputs]
        p = gfb.GuidedFilterParams(c["r"], c["eps"])
        if self.kind == "joint_fwd_bwd":
            host_in.append(self.d_out.cpu().pin_memory())
            lx, ly, hx, dd = host_in
            host_out = [torch.empty_like(hx).pin_memory(), torch.empty_like(lx).pin_memory(),
                        torch.empty_like(ly).pin_memory(), torch.empty_like(hx).pin_memory()]
        elif self.kind == "train_step":
            # the target is a step input too; the step's results are the loss
            # and the packed guidance-net gradient
            host_in.append(self.target.cpu().pin_memory())
            host_out = [torch.empty((), dtype=torch.float64).pin_memory(),
                        torch.empty(self.net.param_count(), dtype=torch.float32).pin_memory()]
        else:
            host_out = [torch.empty(self.out.shape, dtype=self.out.dtype).pin_memory()]

        def one():
            if self.kind == "highres_fwd":
                gfb.forward_highres_host(host_in[0], host_in[1], p, out=host_out[0],
                                         device=self.device, check=False)
            elif self.kind == "joint_fwd":
                gfb.forward_joint_host(host_in[0], host_in[2], host_in[1], p, out=host_out[0],
                                       device=self.device, check=False)
            elif self.kind == "joint_fwd_bwd":
                # forward + backward over host images, pipelined per plane
                gfb.forward_backward_joint_host(lx, hx, ly, dd, p, outs=host_out,
                                                device=self.device, check=False)
            else:
                dev = [t.to(self.device, non_blocking=True) for t in host_in]
                r = gfb.train_step(self.net, dev[0], dev[2], dev[1], dev[3], p)
                host_out[0].copy_(r.loss, non_blocking=True)
                host_out[1].copy_(r.dparams, non_blocking=True)
                torch.cuda.synchronize(self.device)

        for _ in range(warmup):
            one()
        torch.cuda.synchronize(self.device)
        t0 = time.perf_counter()
        for _ in range(steps):
            one()
        torch.cuda.synchronize(self.device)
        ms = (time.perf_counter() - t0) * 1e3 / steps
        h2d = sum(t.numel() * t.element_size() for t in host_in)
        d2h = sum(t.numel() * t.element_size() for t in host_out)
        return ms, h2d, d2h


# ---------------------------------------------------------------------------
# CPU reference legs (cpu_reference.py: the reference package, numba on)
# ---------------------------------------------------------------------------

def run_reference(args, c, rank, world):
    """--impl reference: the reference's CPU path on all host cores, rank 0 only."""
    if rank != 0:
        return
    import cpu_reference

    total = args.steps + args.warmup
    step_s = min(8.0, max(1.0, 150.0 / max(total + 1, 1)))
    res = cpu_reference.run(c, step_seconds=step_s, steps=args.steps, warmup=args.warmup)
    line = {
        "metric": METRIC, "value": round(res["value"], 4), "unit": "Mpix/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(res["ms_per_step"], 3), "higher_is_better": True,
        "scaling": "strong" if c.get("shard") else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded uniform [0,1], HWC float64: the reference's layout)",
        "config": config_block(args, c, world), "impl": "reference",
        "cpu_baseline": {"value": round(res["value"], 4), "unit": "Mpix/s", "cores": res["cores"],
                         "kind": res["kind"], "sample": res["sample"]},
        "e2e": {"value": round(res["value"], 4), "unit": "Mpix/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_block(args, c, world):
    B, C, H = c["batch"], c["channels"], c["hr"]
    par = {"rows": f"row-bands x{world} (lr halo max(2r,r+1), no data-path collective)",
           "batch": f"batch-shard x{world} (no data-path collective)"}.get(
        c.get("shard"), f"replica x{world} (each rank its own batch)")
    if c["kind"] == "train_step" and world > 1:
        par = f"data-parallel x{world} (NCCL allreduce of the 95 guidance-net grads)"
    blk = {"workload": f"{args.config}: {c['kind']}",
           "batch_per_gpu": (B if not c.get("shard") else f"{B} split over {world}"),
           "global_batch": B * (1 if c.get("shard") else world), "channels": C,
           "hr": [H, H], "radius": c["r"], "eps": c["eps"], "parallelism": par}
    if c["kind"] == "highres_fwd":
        blk["guide_channels"] = 1
    else:
        blk["lr"] = [H // c["factor"], H // c["factor"]]
    if c["kind"] == "train_step":
        blk["guidance_hidden"] = c["hidden"]
    bytes_ = algorithmic_bytes(c)
    blk["l2"] = ("inputs+outputs %.0f MB > 126 MB L2 (no flush needed)" % (bytes_ / 1e6)
                 if bytes_ > 2.5 * 126e6 else "L2 flushed between timed steps (256 MB read sweep)")
    return blk


# ---------------------------------------------------------------------------
# main
# ---------------------------------------------------------------------------

def relaunch(n):
    """--gpus N outside torchrun: one process per GPU under torch.distributed.run."""
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd, env=os.environ.copy())


def launch_check(rank, world):
    """Every rank joins one process group and sums a 1: rank 0 prints the
    world it saw (tests/test_bench.py runs this on CPU with gloo)."""
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        n = int(t.item())
        dist.destroy_process_group()
    else:
        n = 1
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": world, "ranks_seen": n}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg4a")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--hr", type=int, default=0)
    ap.add_argument("--radius", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--launch-check", action="store_true",
                    help="test hook: check the N-rank launch (gloo, no GPU work) and exit")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    # communicator lines (rank count, transport) on stderr; stdout stays one JSON line
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(relaunch(args.gpus))

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus if args.impl == "reference" else 1)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    c = workload_spec(args)

    if args.launch_check:
        launch_check(rank, world)
        return
    if args.impl == "reference":
        run_reference(args, c, rank, world)
        return

    import torch

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=device)

    st = OursStep(c, device, seed=args.seed + (0 if c.get("shard") else 1000 * rank), rank=rank,
                  world=world)
    flush = None
    if algorithmic_bytes(c) <= 2.5 * 126e6:
        flush = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=device)  # 256 MB

    for _ in range(args.warmup):
        st.step()
        if flush is not None:
            flush.sum()  # read-only sweep: evicts our data, leaves L2 clean
    torch.cuda.synchronize(device)
    assert int(st.status.item()) == 0, f"status bits {int(st.status.item())}"

    # timed region: K steps, barrier + sync both sides; per-step events so an
    # L2 flush between steps stays outside the measured kernel time
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(device)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    wall0 = time.perf_counter()
    for k in range(args.steps):
        if flush is not None:
            flush.sum()
            # keep the device busy while the host enqueues the step, so the
            # events bracket the step's device time, not the host's launch
            # latency (matters only for the microsecond-scale configs)
            torch.cuda._sleep(800000)  # ~400 us: covers the Python API call
        evs[k][0].record()
        st.step()
        evs[k][1].record()
    torch.cuda.synchronize(device)
    if dist:
        dist.barrier()
    wall = time.perf_counter() - wall0
    clocks = sampler.stop() if sampler else None
    ms_steps = [a.elapsed_time(b) for a, b in evs]
    ms = sum(ms_steps) / len(ms_steps)
    if dist:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    assert int(st.status.item()) == 0, f"status bits {int(st.status.item())}"

    if c.get("shard"):  # strong scaling: the ranks split one fixed workload
        t = torch.tensor([float(st.pixels)], device=device, dtype=torch.float64)
        if dist:
            dist.all_reduce(t)
        px = float(t.item())
    else:
        px = st.pixels * world
    value = px / (ms * 1e-3) / 1e6

    e2e = None
    if not args.no_e2e:
        e_ms, h2d, d2h = st.e2e(steps=max(3, min(args.steps, 5)), warmup=1)
        if dist:
            t = torch.tensor([e_ms], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": round(px / (e_ms * 1e-3) / 1e6, 3), "unit": "Mpix/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": round(e_ms, 4),
               "api": {"joint_fwd_bwd": "forward_backward_joint_host",
                       "joint_fwd": "forward_joint_host", "highres_fwd": "forward_highres_host",
                       "train_step": "train_step (H2D inputs + target, D2H loss + grads)"}[
                           st.kind]}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    peak, peak_kind = measured_peak()
    # the dominant kernels process this rank's share of the workload
    alg = int(algorithmic_bytes(c) * st.pixels / (c["batch"] * c["hr"] * c["hr"]))
    achieved = alg / (ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": ncu_traffic(args.config),
                "traffic_scope": "DRAM bytes of one step, all kernels (profiles/traffic.json)",
                "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": alg,
                "frac_of_8TBps_nominal": round(achieved / 8000.0, 4)}

    cpu = None
    if world == 1 and not args.no_cpu:
        import cpu_reference

        res = cpu_reference.run(c, step_seconds=4.0, steps=2)
        cpu = {"value": round(res["value"], 4), "unit": "Mpix/s", "cores": res["cores"],
               "kind": res["kind"], "sample": res["sample"]}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Mpix/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 5),
        "higher_is_better": True, "scaling": "strong" if c.get("shard") else "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded; BASELINE.json shapes and distributions, workloads.py)",
        "config": config_block(args, c, world),
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": st.launches * args.steps,
        "clocks": clocks, "wall_s_timed_region": round(wall, 4),
        "ms_per_step_min": round(min(ms_steps), 5),
    }
    if dist:
        dist.destroy_process_group()
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
