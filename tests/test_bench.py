"""bench.py plumbing on CPU: the --gpus N self-launch (one process per rank
under torch.distributed.run), the reference arm's JSON line, and the byte
accounting of the roofline."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=300):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, res.stdout  # exactly one JSON line on stdout
    return json.loads(lines[0])


def test_gpus2_relaunches_two_ranks():
    line = _run(["--gpus", "2", "--launch-check"])
    assert line == {"launch_check": True, "n_gpus": 2, "ranks_seen": 2}


def test_single_process_launch_check():
    assert _run(["--launch-check"])["n_gpus"] == 1


def test_reference_arm_line_small_config():
    line = _run(["--impl", "reference", "--config", "cfg0", "--steps", "1", "--warmup", "3"])
    assert line["impl"] == "reference" and line["unit"] == "Mpix/s" and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["cores"] >= 1 and cb["kind"] in ("reference", "port")
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["workload"].startswith("cfg0")


def test_algorithmic_bytes_match_survey():
    sys.path.insert(0, ROOT)
    import bench
    from workloads import CONFIGS

    # cfg4a fwd 15.40 GB + bwd 23.56 GB; cfg1 469.8 MB; cfg2 1711.3 MB
    assert bench.algorithmic_bytes(CONFIGS["cfg4a"]) == pytest.approx(38.96e9, rel=2e-3)
    assert bench.algorithmic_bytes(CONFIGS["cfg1"]) == 469762048
    assert bench.algorithmic_bytes(CONFIGS["cfg2"]) == pytest.approx(1711.3e6, rel=1e-3)
