"""B200 hardware descriptor and the engine's execution model.

* presets/b200-sparse.hw is in the reference's .hw format (docs/formats.md:32-47):
  the reference's own parser + estimate (perf.cpp:39-134, built into oracle/_ref)
  and the engine's restatement agree on it, and it equals hw_preset("b200-sparse").
* estimate_device (hwmodel.hpp) predicts the measured per-launch time of every
  BASELINE config (profiles/round2/bench_*.json, measured on B200) within 25 %.
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2506_22969_b200 import estimate_device, explore

REPO = Path(__file__).resolve().parents[1]
HW = (REPO / "presets" / "b200-sparse.hw").read_text()


def test_hw_file_equals_builtin_preset():
    for name, dims in (("Box-2D9P", (8192, 8192)), ("Box-3D27P", (512, 512, 512)), ("Heat-1D", (1 << 20,))):
        a = explore(name, dims, hw=HW)
        b = explore(name, dims, hw="b200-sparse")
        assert a == b


@pytest.mark.skipif(not oracle.ref_available(), reason="reference build (oracle/_ref) missing")
def test_hw_file_through_reference_parser_and_model():
    L = oracle.ref()
    import ctypes as C
    for name, dims in (("Box-2D9P", (8192, 8192)), ("Star-2D13P", (16384, 16384)), ("Box-3D27P", (1024,) * 3)):
        k = {"Box-2D9P": 3, "Star-2D13P": 7, "Box-3D27P": 3}[name]
        rows = {(r["r1"], r["r2"]): r for r in explore(name, dims, hw=HW)}
        d = np.asarray(dims, dtype=np.uint64)
        for (r1, r2) in ((16, 8), (8, 16), (8, 8), (1, 2), (16, 16)):
            out = np.zeros(4)
            nm = C.c_uint64()
            assert L.ref_estimate_hw_text(HW.encode(), len(dims), d.ctypes.data, k, r1, r2, out.ctypes.data,
                                          C.byref(nm)) == 0, L.ref_last_error()
            mine = rows[(r1, r2)]
            assert (mine["t_compute"], mine["t_memory"], mine["t_total"], mine["n_mma"]) == \
                (out[0], out[1], out[2], nm.value)


CONFIGS = [("box2d", "Box-2D9P", (8192, 8192)), ("star2d", "Star-2D13P", (16384, 16384)),
           ("heat2d", "Heat-2D", (4096, 4096)), ("box3d", "Box-3D27P", (512,) * 3),
           ("heat3d", "Heat-3D", (512,) * 3), ("box3d1024", "Box-3D27P", (1024,) * 3)]


@pytest.mark.parametrize("cfg,name,dims", CONFIGS)
def test_device_model_matches_measured(cfg, name, dims):
    line = json.loads((REPO / "profiles" / "round2" / f"bench_{cfg}.json").read_text().strip().splitlines()[-1])
    storage = 2 if line["roofline"].get("h16_launches") else 4
    e = estimate_device(name, dims, storage=storage)
    measured_s = line["ms_per_step"] * 1e-3
    assert abs(e["t_total"] / measured_s - 1) <= 0.25, (e, measured_s)


def test_device_model_terms():
    e2 = estimate_device("Box-2D9P", (8192, 8192), storage=4)
    assert e2["bound"] == "hbm"
    assert e2["hbm_bytes"] == pytest.approx(8 * 8190 ** 2)
    h = estimate_device("Box-2D9P", (8192, 8192), storage=2)
    assert h["hbm_bytes"] == pytest.approx(4 * 8190 ** 2) and h["bound"] == "smem"
    assert h["k_pad"] == 192  # (16, 8): window 18 x 10 = 180 columns -> 192
    e3 = estimate_device("Box-3D27P", (512,) * 3)
    assert e3["mma_issues"] == pytest.approx(e3["batches"] * 3 * 6)  # kz = 3 slices x 6 K steps
    # fusion: more work per HBM byte, the smem pipe binds from t = 3 (measured 2D: t = 2 at
    # the launch time of t = 1, then gather-bound)
    f = [estimate_device("Box-2D9P", (8192, 8192), fuse=t, storage=4) for t in (1, 2, 3, 4)]
    assert [x["bound"] for x in f] == ["hbm", "hbm", "smem", "smem"]
    assert f[1]["gstencil"] > 1.8 * f[0]["gstencil"]
    with pytest.raises(ValueError):
        estimate_device("Box-2D9P", (8192, 8192), storage=3)
