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
    res = _bench("--config", "heat2d", "--steps", "20", "--warmup", "3", "--no-cpu", "--no-e2e", "--no-sweep")
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    # 5 grids x 4 steps as ONE launch per step (grouped batch run) + one ring conversion per grid
    assert line["gpu_launches"] == 20 // 5 + 5
    assert "stepped together" in line["config"]["l2"]
    roof = line["roofline"]
    assert roof["bound"] == "hbm" and 0.2 < roof["frac"] < 1.3
    assert roof["l2_flushed_single_launch"]["ms_per_launch"] > 0
    assert "sm_mhz" in line["clocks"]


def test_default_config_per_world_size():
    """N = 1 runs BASELINE configs[1] (Box-2D9P 8192^2); N > 1 the north-star scaling
    config (Box-3D27P 1024^3 strong-scaled, P2P halos) unless --weak."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    assert b.CONFIGS["box2d"][:2] == ("Box-2D9P", (8192, 8192))
    assert b.CONFIGS["box3d1024"][:2] == ("Box-3D27P", (1024, 1024, 1024))
    for n in (2, 4, 8):  # strong scaling: whole planes per rank, >= 2 halo widths each
        assert 1024 % n == 0 and 1024 // n >= 2


@pytest.mark.gpu
def test_two_rank_strong_scaling_line_shared_gpu():
    """torchrun, 2 ranks sharing the one GPU (gloo control plane, IPC P2P halos):
    the strong-scaling line with its own N = 1 reference (functional, not a timing)."""
    res = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2",
                          "--share-gpu", "--config", "box3d", "--steps", "4", "--warmup", "3"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    line = json.loads([x for x in res.stdout.strip().splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["global_grid"] == [512, 512, 512] and line["config"]["grid_per_gpu"] == [256, 512, 512]
    assert line["n1_same_grid"]["value"] > 0 and line["gpu_launches"] == 4 + 1  # + the ring conversion
    assert "p2p" in line["config"]["parallelism"]


@pytest.mark.gpu
def test_default_line_times_every_other_config(gpu):
    """The default line also times the other BASELINE configs (other_configs), each with
    the engine model's prediction beside it."""
    res = _bench("--steps", "6", "--warmup", "3", "--no-cpu", "--no-e2e", timeout=900)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    oc = line["other_configs"]
    assert sorted(oc) == ["box3d", "box3d1024", "heat2d", "heat3d", "star2d"]
    for name, v in oc.items():
        assert "error" not in v, (name, v)
        assert v["value"] > 0 and 0.05 < v["hbm_frac"] < 1.3
        assert v["model"]["predicted_ms_per_step"] > 0
    assert line["roofline"]["model"]["bound"] in ("hbm", "smem", "tensor")
