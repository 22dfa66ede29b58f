"""Shared fixtures. `-m "not gpu"` runs here (CPU only); `-m gpu` on a B200."""
from __future__ import annotations

import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
GOLDEN = REPO / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")


@pytest.fixture(scope="session", autouse=True)
def built():
    """Build the engine library and the checkers if they are missing/stale."""
    from paper_2506_22969_b200 import build as b

    b.build()
    import oracle

    oracle.build()
    yield


def gpu_available() -> bool:
    try:
        from paper_2506_22969_b200._capi import lib

        return lib().sst_device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not gpu_available():
        pytest.fail("GPU test collected on a host without a CUDA device "
                    "(run with -m 'not gpu' on CPU hosts)")
    import torch

    torch.cuda.init()
    return 0
