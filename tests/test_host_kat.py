"""Known-answer tests of the C++ host compile library (tests/cpp/host_kat.cpp):
the reference unit-test fixtures restated against our stensor:: API, plus a CPU
emulation of the kernel's operand images (A smem image, TMEM metadata words,
koff) that must reproduce a brute-force sweep exactly."""
from __future__ import annotations

import json
import subprocess

import pytest

from conftest import GOLDEN, REPO

SRC = REPO / "paper_2506_22969_b200" / "csrc" / "host"
BIN = REPO / "tests" / "cpp" / "build" / "host_kat"


@pytest.fixture(scope="module")
def kat():
    srcs = [REPO / "tests" / "cpp" / "host_kat.cpp"] + [
        SRC / f"{n}.cpp" for n in ("spec", "morph", "sparsify", "s24", "hwmodel", "device_image")]
    BIN.parent.mkdir(parents=True, exist_ok=True)
    if not BIN.exists() or any(s.stat().st_mtime > BIN.stat().st_mtime for s in srcs + list(
            (SRC / "stensor").glob("*.hpp"))):
        subprocess.run(["g++", "-std=c++20", "-O2", f"-I{SRC}", f"-I{REPO / 'include'}",
                        *map(str, srcs), "-o", str(BIN)], check=True)
    return BIN


def test_reference_known_answers(kat):
    res = subprocess.run([str(kat)], capture_output=True, text=True)
    assert res.returncode == 0, res.stdout[-4000:]
    assert "0 failures" in res.stdout


def test_device_image_emulation(kat):
    res = subprocess.run([str(kat), "image"], capture_output=True, text=True)
    assert res.returncode == 0, res.stdout[-4000:]


def test_perf_model_matches_reference(kat):
    """estimate() of the reference (tests/golden/perf_fixture.json) bit-for-bit."""
    for case in json.loads((GOLDEN / "perf_fixture.json").read_text()):
        args = [str(kat), "perf", case["hw"], str(case["k"]), str(case["r1"]), str(case["r2"]),
                *map(str, case["grid"])]
        got = json.loads(subprocess.run(args, capture_output=True, text=True, check=True).stdout)
        for key in ("t_compute", "t_memory", "t_total", "n_prime", "n_mma"):
            assert got[key] == case[key], (case, key, got[key])
