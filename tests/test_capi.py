"""The C-ABI library: loads on a CPU-only host, exports every symbol
include/sparstencil.h declares, maps errors to the reference exception types,
and refuses (loudly) to run without a device — there is no CPU fallback."""
from __future__ import annotations

import ctypes as C
import re

import numpy as np
import pytest

from conftest import REPO, gpu_available
from paper_2506_22969_b200 import Compiled, SparseStencil, _capi
from paper_2506_22969_b200._capi import lib

HEADER = (REPO / "include" / "sparstencil.h").read_text()
DECLARED = sorted(set(re.findall(r"SST_API\s+[\w\s\*]+?\b(sst_\w+)\s*\(", HEADER)))


def test_header_declares_the_abi():
    assert len(DECLARED) >= 20
    assert sorted(_capi.EXPORTED) == DECLARED


def test_library_exports_every_declared_symbol():
    L = lib()
    for name in DECLARED:
        assert hasattr(L, name), name
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", str(_capi.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (sst_\w+)", out))
    assert set(DECLARED) <= exported
    assert lib().sst_version().startswith(b"sparstencil-b200")


def test_compile_info_and_desc():
    c = Compiled("Box-3D27P", [32, 48, 64], 16, 8)
    i = c.info
    assert (i["dims"], i["k"], i["m_prime"], i["window_w"], i["window_h"], i["window_d"]) == \
        (3, 3, 128, 18, 10, 3)
    assert i["cols"] == 540 and i["p"] == 0 and i["align_cols"] == 0
    d = c.plan_desc()
    assert d.rows == 128 and d.cols == 540 and d.window_d == 3
    assert list(d.grid_dims) == [32, 48, 64]
    vals = np.ctypeslib.as_array(d.a_values, shape=(128 * 270,))
    assert np.count_nonzero(vals) == 128 * 27  # every output row uses all 27 weights


def test_error_status_and_message():
    h = C.c_void_p()
    dims = (C.c_uint64 * 2)(64, 64)
    st = lib().sst_compile(b"nope", dims, 2, 16, 8, 1, C.byref(h))
    assert st == 1 and b"unknown stencil preset" in lib().sst_last_error()
    with pytest.raises(_capi.InvalidArgument):
        _capi.check(st)


@pytest.mark.skipif(gpu_available(), reason="checks the no-device behaviour")
def test_no_device_means_error_not_fallback():
    with pytest.raises(_capi.CudaFailure):
        SparseStencil("Box-2D9P", [64, 64])


def test_device_path_rejects_illegal_layouts():
    c = Compiled("Box-2D9P", [64, 64], 8, 8)  # m' = 64 is not the device layout
    d = c.plan_desc()
    h = C.c_void_p()
    st = lib().sst_plan_create(C.byref(d), 0, C.byref(h))
    assert st in (1, 5, 6)  # invalid argument (or no device on CPU hosts)
    if st == 1:
        assert b"(16, 8)" in lib().sst_last_error()


def test_random_grid_matches_oracle():
    import oracle

    out = np.empty((37, 41), np.float32)
    dims = (C.c_uint64 * 2)(37, 41)
    _capi.check(lib().sst_random_grid(2, dims, 7, out.ctypes.data_as(C.c_void_p)))
    assert np.array_equal(out.astype(np.float64), oracle.random_grid([37, 41], 7))
