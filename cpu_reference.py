"""CPU reference timing for bench.py (measurement infrastructure, not product).

Times the REFERENCE's own CPU implementation of the path on the host cores:
the unmodified ``guidedfilter`` package (pkg/src of the reference, numba
kernels on, ``gf/_kernels.py:36-124``) installed into the git-ignored
``baseline/_ref`` by ``__graft_entry__.build()`` (it ships to the GPU box
with the repo snapshot; ``/root/reference`` itself is never read here).  If
that install is absent it falls back to the repo's float64 numpy restatement
``oracle/gf_oracle.py`` and says so (``kind: "port"``).

The reference is single-threaded per call (numba ``@njit`` without
``parallel``), so the host cores are used by a process pool, one image
sample per process: each worker holds a row band of one image of the
workload (full width, ``rows`` high-res rows, the matching low-res rows) as
the reference's HWC float64 arrays and runs the call the config names:

* ``joint_fwd``      ``forward_joint(guide_lo, guide_hi, src_lo, p)``  (gf/guided.py:152)
* ``joint_fwd_bwd``  the same plus ``backward(tape, d_out)``            (gf/guided.py:267)
* ``highres_fwd``    ``forward_highres(guide3, src, p)`` with the 1-channel
                     guide replicated to 3 channels                     (gf/guided.py:198)
* ``train_step``     GuidanceNet on both resolutions, forward_joint,
                     mse_loss, backward, both GuidanceNet backwards     (gf/training.py:143-183)

Throughput = high-res output pixels of all workers / wall time of the step.
Workers are started (``spawn``) and JIT-warmed before any timed step.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

_W = None  # per-worker state


def reference_available() -> bool:
    return os.path.isfile(os.path.join(REF_DIR, "guidedfilter", "guided.py"))


def _setup_env():
    # one BLAS/OpenMP thread per process: the pool provides the parallelism
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS",
              "NUMBA_NUM_THREADS"):
        os.environ[k] = "1"
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gf_numba_cache")
    os.environ.pop("GUIDEDFILTER_PURE_NUMPY", None)


class _Impl:
    """The reference package (kind 'reference') or the oracle port ('port')."""

    def __init__(self, use_ref: bool):
        self.kind = "reference" if use_ref else "port"
        if use_ref:
            if REF_DIR not in sys.path:
                sys.path.insert(0, REF_DIR)
            import guidedfilter as gf
            from guidedfilter import _kernels

            self.gf = gf
            self.numba = bool(_kernels.enabled())
        else:
            if ROOT not in sys.path:
                sys.path.insert(0, ROOT)
            from oracle import gf_oracle as O

            self.O = O
            self.numba = False

    def joint_fwd(self, gl, gh, sl, r, eps):
        if self.kind == "reference":
            return self.gf.forward_joint(gl, gh, sl, self.gf.GuidedFilterParams(r, eps))
        return self.O.forward_joint(gl, gh, sl, r, eps)

    def backward(self, tape, d):
        if self.kind == "reference":
            return self.gf.backward(tape, d)
        return self.O.backward(tape, d)

    def highres_fwd(self, g, s, r, eps):
        if self.kind == "reference":
            return self.gf.forward_highres(g, s, self.gf.GuidedFilterParams(r, eps))
        return self.O.forward_highres(g, s, r, eps)


def _make_sample(spec, rows, seed):
    import numpy as np

    rng = np.random.default_rng(seed)
    kind, C, W, f = spec["kind"], spec["channels"], spec["hr"], spec.get("factor", 4)
    if kind == "highres_fwd":
        g = rng.uniform(0, 1, (rows, W, 1))
        s = np.clip(0.8 * g + 0.1 + 0.1 * rng.standard_normal((rows, W, C)), 0, 1)
        return {"g3": np.repeat(g, C, axis=2), "s": s, "px": rows * W}
    hl = max(1, rows // f)
    w = W // f
    gl = rng.uniform(0, 1, (hl, w, C))
    sl = rng.uniform(0, 1, (hl, w, C))
    gh = rng.uniform(0, 1, (hl * f, W, C))
    out = {"gl": gl, "sl": sl, "gh": gh, "px": hl * f * W}
    if kind == "joint_fwd_bwd":
        out["d"] = rng.standard_normal((hl * f, W, C))
    if kind == "train_step":
        out["T"] = np.clip(1.5 * gh - 0.25, 0.0, 1.0)
    return out


def _run_once(impl, spec, smp):
    r, eps, kind = spec["r"], spec["eps"], spec["kind"]
    if kind == "highres_fwd":
        impl.highres_fwd(smp["g3"], smp["s"], r, eps)
    elif kind == "joint_fwd":
        impl.joint_fwd(smp["gl"], smp["gh"], smp["sl"], r, eps)
    elif kind == "joint_fwd_bwd":
        _, tape = impl.joint_fwd(smp["gl"], smp["gh"], smp["sl"], r, eps)
        impl.backward(tape, smp["d"])
    elif kind == "train_step":
        _train_step(impl, spec, smp)
    else:
        raise ValueError(kind)


def _train_step(impl, spec, smp):
    """gf/training.py:143-183 (GuidedUpsampler forward/backward minus the
    core net) on one image: F(lr), F(hr), forward_joint, mse_loss, backward,
    F backward at both sites (low-res first)."""
    import numpy as np

    r, eps = spec["r"], spec["eps"]
    if impl.kind == "reference":
        gf = impl.gf
        if "net" not in smp:
            smp["net"] = gf.GuidanceNet(3, 3, hidden=spec.get("hidden", 15), kernel=1,
                                        rng=np.random.default_rng(0))
        net = smp["net"]
        Gl, tl = net.forward(smp["gl"])
        Gh, th = net.forward(smp["gh"])
        out, tp = gf.forward_joint(Gl, Gh, smp["sl"], gf.GuidedFilterParams(r, eps))
        _, d = gf.mse_loss(out, smp["T"])
        g = gf.backward(tp, d)
        net.backward(tl, g.d_guide_lo)
        net.backward(th, g.d_guide_hi)
    else:
        O = impl.O
        if "params" not in smp:
            smp["params"] = O.guidance_init(3, 3, spec.get("hidden", 15),
                                            np.random.default_rng(0))
        O.train_step(smp["params"], [smp["gl"]], [smp["gh"]], [smp["sl"]], [smp["T"]], r, eps)


def _init(spec, rows, use_ref, seed):
    global _W
    _setup_env()
    impl = _Impl(use_ref)
    smp = _make_sample(spec, rows, seed)
    _run_once(impl, spec, smp)  # JIT compile / warm caches, untimed
    _W = (impl, spec, smp)


def _step(_):
    impl, spec, smp = _W
    t0 = time.perf_counter()
    _run_once(impl, spec, smp)
    return time.perf_counter() - t0, smp["px"]


def probe_seconds_per_row(spec, use_ref, rows=32):
    """Single-process time per high-res row of the sample (after a warm call)."""
    _setup_env()
    impl = _Impl(use_ref)
    smp = _make_sample(spec, rows, 0)
    _run_once(impl, spec, smp)
    t0 = time.perf_counter()
    _run_once(impl, spec, smp)
    return (time.perf_counter() - t0) / rows, impl


def run(spec, step_seconds, steps, warmup=0, procs=None, use_ref=None):
    """Time ``steps`` steps of ``procs`` parallel samples, each sized to take
    about ``step_seconds``.  Returns a dict (value Mpix/s, per-step times,
    kind, cores, sample text)."""
    if use_ref is None:
        use_ref = reference_available()
    procs = procs or len(os.sched_getaffinity(0))
    per_row, impl = probe_seconds_per_row(spec, use_ref)
    f = spec.get("factor", 4)
    # whole images when one fits the step budget (the reference's per-pixel
    # cost grows with the image -- its numpy passes leave the caches -- so a
    # band sample would flatter it); otherwise a full-width row band
    if per_row * spec["hr"] <= 2.0 * step_seconds:
        rows = spec["hr"]
    else:
        rows = int(step_seconds / max(per_row, 1e-9))
        rows = max(f * 4, min(spec["hr"], rows // (4 * f) * (4 * f)))
    ctx = mp.get_context("spawn")
    times = []
    px_total = 0
    with ctx.Pool(procs, initializer=_init, initargs=(spec, rows, use_ref, 1)) as pool:
        pool.map(_step, range(procs), chunksize=1)  # every worker initialised
        for _ in range(warmup):
            pool.map(_step, range(procs), chunksize=1)
        for _ in range(steps):
            t0 = time.perf_counter()
            res = pool.map(_step, range(procs), chunksize=1)
            times.append(time.perf_counter() - t0)
            px_total += sum(p for _, p in res)
    wall = sum(times)
    what = ("reference guidedfilter (baseline/_ref, numba %s)" % ("on" if impl.numba else "OFF")
            if impl.kind == "reference" else "float64 numpy oracle port (baseline/_ref absent)")
    band = "whole" if rows == spec["hr"] else f"{rows}x{spec['hr']} hr-row band of a"
    sample = (f"{procs} processes x one {band} {spec['kind']} image "
              f"(C={spec['channels']}, r={spec['r']}) per step, {what}, HWC float64")
    return {"value": px_total / wall / 1e6, "ms_per_step": 1e3 * wall / max(steps, 1),
            "kind": impl.kind, "cores": procs, "sample": sample, "rows": rows,
            "numba": impl.numba}
