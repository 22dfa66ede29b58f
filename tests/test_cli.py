"""The `sstensor` CLI (reference proj/tools/main.cpp:75-193): same subcommands,
options, output lines and exit codes (0 ok, 1 verification failure, 2 error)."""
from __future__ import annotations

import json
import subprocess
from pathlib import Path

import pytest

CLI = Path(__file__).resolve().parents[1] / "paper_2506_22969_b200" / "bin" / "sstensor"
GOLD = json.loads((Path(__file__).parent / "golden" / "compile" / "cases.json").read_text())


def sst(*args):
    return subprocess.run([str(CLI), *args], capture_output=True, text=True, timeout=300)


def test_presets_lists_stencils_and_hardware():
    r = sst("presets")
    assert r.returncode == 0
    assert "Box-2D9P     dims=2 k=3 points=9 box" in r.stdout
    assert "hw: a100-sparse" in r.stdout and "hw: b200-sparse" in r.stdout


def test_compile_writes_reference_artifacts(tmp_path):
    r = sst("compile", "--stencil", "Box-2D9P", "--grid", "37x41", "--r1", "16", "--r2", "8", "--no-verify",
            "--out", str(tmp_path))
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("r1=16 r2=8 p=0 ")
    want = GOLD["Box-2D9P_37x41_a100-sparse_r16x8_f1_exact64_s1"]
    got = (tmp_path / "report.json").read_text()
    cut = want["report"].index('  "verification"')
    strip = lambda t: [line for line in t[:cut].splitlines() if '"issued_mma"' not in line]  # noqa: E731
    assert strip(got) == strip(want["report"])
    import hashlib
    assert hashlib.sha256((tmp_path / "a2.s24").read_bytes()).hexdigest() == want["a2.s24"]["sha256"]


def test_corrupt_permutation_exits_1(tmp_path):
    r = sst("compile", "--stencil", "Heat-2D", "--grid", "64x64", "--corrupt-permutation", "--out", str(tmp_path))
    assert r.returncode == 1 and "status=conversion-failed" in r.stdout
    assert (tmp_path / "report.json").read_text() == \
        GOLD["Heat-2D_64x64_a100-sparse_r0x0_f1_exact64_s1_corrupt"]["report"]


def test_explore_table_and_csv(tmp_path):
    csv = tmp_path / "c.csv"
    r = sst("explore", "--stencil", "Heat-2D", "--grid", "64x64", "--csv", str(csv))
    assert r.returncode == 0
    assert r.stdout.splitlines()[0].split() == ["r1", "r2", "t_compute", "t_memory", "t_total", "n_mma"]
    rows = csv.read_text().splitlines()
    assert rows[0] == "r1,r2,t_compute,t_memory,t_total,n_mma,m_prime,k_prime,n_prime" and len(rows) > 100


@pytest.mark.parametrize("argv", [[], ["frob"], ["compile", "--grid", "64x64"], ["compile", "--bogus", "1"],
                                  ["compile", "--stencil", "Heat-2D", "--grid", "1x2x3x4", "--no-verify"],
                                  ["compile", "--stencil", "Heat-2D", "--grid", "64x64", "--precision", "fp8"]])
def test_usage_and_input_errors_exit_2(argv):
    assert sst(*argv).returncode == 2


@pytest.mark.gpu
def test_compile_verifies_on_device(gpu, tmp_path):
    r = sst("compile", "--stencil", "Heat-2D", "--grid", "64x64", "--out", str(tmp_path))
    assert r.returncode == 0, r.stderr
    assert (tmp_path / "report.json").read_text() == GOLD["Heat-2D_64x64_a100-sparse_r0x0_f1_exact64_s1"]["report"]


@pytest.mark.gpu
def test_verify_all_presets(gpu):
    r = sst("verify")
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("verified") == 8


@pytest.mark.gpu
@pytest.mark.parametrize("stencil,grid", [("Box-2D9P", "2048x2048"), ("Heat-1D", "1000000"),
                                          ("Heat-3D", "64x64x64")])
def test_run_time_loop(gpu, stencil, grid):
    r = sst("run", "--stencil", stencil, "--grid", grid, "--steps", "50")
    assert r.returncode == 0, r.stderr
    assert "GStencil/s" in r.stdout and "launches" in r.stdout


def test_model_subcommand():
    r = sst("model", "--stencil", "Box-2D9P", "--grid", "8192x8192", "--storage", "f32")
    assert r.returncode == 0, r.stderr
    assert "bound: hbm" in r.stdout and "predicted" in r.stdout
    r = sst("model", "--stencil", "Box-2D9P", "--grid", "8192x8192", "--storage", "f64")
    assert r.returncode == 2
