"""bench.py contract: the JSON line's keys and the argument checks (CPU), and one
short device run of the small-grid (round-robin, inputs > L2) timing path (GPU)."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, timeout=300):
    return subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                          timeout=timeout)


def test_reference_arm_line():
    """--impl reference: the reference CPU path (oracle/_ref when built, else the port) on the
    engine arm's metric / config, with cpu_baseline and a zero-copy e2e."""
    res = _bench("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["e2e"]["value"] == line["value"]


def test_steps_must_be_a_multiple_of_fuse():
    res = _bench("--steps", "5", "--fuse", "2")
    assert res.returncode == 2 and "multiple of --fuse" in res.stderr


@pytest.mark.gpu
def test_small_grid_line(gpu):
    """Heat-2D 4096^2 (ping-pong pair < L2): timed over round-robin copies, the flushed
    single launch reported beside it, one launch per step, roofline and clocks present."""
    res = _bench("--config", "heat2d", "--steps", "20", "--warmup", "3", "--no-cpu", "--no-e2e")
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["gpu_launches"] == 20
    assert "round-robin" in line["config"]["l2"]
    roof = line["roofline"]
    assert roof["bound"] == "hbm" and 0.2 < roof["frac"] < 1.3
    assert roof["l2_flushed_single_launch"]["ms_per_launch"] > 0
    assert "sm_mhz" in line["clocks"]
