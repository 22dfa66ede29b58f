"""run_compile drop-in (reference pipeline.cpp:52-198, codegen.cpp:19-59, 203-242):
report.json, a2.s24 and lut.bin against the reference's own artefacts, produced
by oracle/_ref/ref_compile from the unmodified reference sources
(oracle/make_golden_compile.py -> tests/golden/compile/).

CPU: everything that does not need the device — the report byte-for-byte except
the verification block and issued_mma (run without verification), the
conversion-failed and unverified-scale reports in full, and the artefact hashes.
GPU: the full report, byte-for-byte, with the desk-scale verification run on the
B200 (direct_apply and the LUT-driven 2:4 product as CUDA kernels, bit-identical
to the reference's CPU loops, so max_abs_err / max_rel_err match exactly).
"""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import pytest

from paper_2506_22969_b200 import InvalidArgument, explore, run_compile

GOLD = Path(__file__).parent / "golden" / "compile"
CASES = json.loads((GOLD / "cases.json").read_text())


def _run(case, tmp_path, verify):
    return run_compile(case["stencil"], case["grid"], hw=case["hw"], r1=case["r1"], r2=case["r2"],
                       fuse=case["fuse"], precision=case["precision"], seed=case["seed"],
                       out_dir=str(tmp_path), verify=verify, corrupt_permutation=bool(case["corrupt"]))


def _strip(report: str) -> list[str]:
    """Report lines without the device-dependent parts (issued_mma, verification block)."""
    lines = report.splitlines()
    cut = next(i for i, line in enumerate(lines) if line.startswith('  "verification"'))
    return [line for line in lines[:cut] if not line.startswith('  "issued_mma"')]


@pytest.mark.parametrize("name", sorted(CASES))
def test_report_and_artifacts_match_reference(name, tmp_path):
    case = CASES[name]
    res = _run(case, tmp_path, verify=False)
    want = case["report"]
    if case["corrupt"] or '"unverified-scale"' in want:
        assert res["report"] == want  # no device work in these reports: byte-identical
    else:
        assert _strip(res["report"]) == _strip(want)
        assert '"status": "unverified-skipped"' in res["report"]
    assert (tmp_path / "report.json").read_text() == res["report"]
    for art in ("a2.s24", "lut.bin"):
        if art in case:
            data = (tmp_path / art).read_bytes()
            assert len(data) == case[art]["size"], art
            assert hashlib.sha256(data).hexdigest() == case[art]["sha256"], art
    lut = GOLD / "lut" / f"{name}.bin"
    if lut.exists():
        assert res["lut"] == lut.read_bytes()


def test_explore_matches_reported_choice():
    # the explorer's best layout is the one run_compile used (a100-sparse model)
    case = CASES["Heat-2D_64x64_a100-sparse_r0x0_f1_exact64_s1"]
    best = explore("Heat-2D", [64, 64])[0]
    rep = json.loads(case["report"])
    assert (best["r1"], best["r2"]) == (rep["r1"], rep["r2"])
    assert best["t_total"] == rep["t_total"]


def test_bad_requests_raise_reference_exceptions():
    with pytest.raises(InvalidArgument):
        run_compile("Heat-2D", [64, 64, 64], verify=False)  # dims mismatch
    with pytest.raises(InvalidArgument):
        run_compile("Heat-2D", [64, 64], precision="fp8", verify=False)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_full_report_with_device_verification(gpu, name, tmp_path):
    case = CASES[name]
    res = _run(case, tmp_path, verify=True)
    assert res["report"] == case["report"]
    assert res["ok"] == (json.loads(case["report"])["verification"]["status"] in ("verified", "unverified-scale"))
