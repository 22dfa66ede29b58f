"""C++ drop-in: the reference's own StencilSpec / Grid / presets / random_grid /
direct_apply (oracle/_ref, compiled from the unmodified reference) against
sst::sparse_apply (include/sparstencil.hpp) in one program (tests/cpp/dropin_test.cpp,
built by oracle/Makefile when the reference sources are present)."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

from conftest import gpu_available

BIN = Path(__file__).parent / "cpp" / "build" / "dropin_test"
needs_bin = pytest.mark.skipif(not BIN.exists(), reason="dropin_test not built (needs the reference sources)")


@needs_bin
@pytest.mark.skipif(gpu_available(), reason="checks the no-device behaviour")
def test_no_device_throws_not_falls_back():
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "runtime_error" in r.stderr


@needs_bin
@pytest.mark.gpu
def test_reference_caller_switches_to_sparse_apply(gpu):
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("0 failures")
