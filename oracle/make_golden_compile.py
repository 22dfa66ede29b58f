"""Golden run_compile artefacts from the reference itself (oracle/_ref/ref_compile,
built from the unmodified /root/reference sources). TEST INFRASTRUCTURE ONLY.

    python oracle/make_golden_compile.py

Writes tests/golden/compile/cases.json: per request the reference's report.json
text, and the sha256 / size of its a2.s24 and lut.bin artefacts (lut.bin bytes
themselves for the smallest cases under tests/golden/compile/lut/).
"""
from __future__ import annotations

import hashlib
import json
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
GOLD = REPO / "tests" / "golden" / "compile"
DRIVER = REPO / "oracle" / "_ref" / "ref_compile"

PRESETS = {1: ["Heat-1D", "1D5P"], 2: ["Heat-2D", "Box-2D9P", "Star-2D13P", "Box-2D49P"],
           3: ["Heat-3D", "Box-3D27P"]}
DESK = {1: ["256", "301"], 2: ["64x64", "37x41"], 3: ["24x24x24", "17x19x23"]}


def cases():
    out = []

    def add(stencil, grid, hw="a100-sparse", r1=0, r2=0, fuse=1, prec="exact64", seed=1, corrupt=0):
        name = f"{stencil}_{grid}_{hw}_r{r1}x{r2}_f{fuse}_{prec}_s{seed}" + ("_corrupt" if corrupt else "")
        out.append((name, stencil, grid, hw, r1, r2, fuse, prec, seed, corrupt))

    for d, names in PRESETS.items():
        for n in names:
            for g in DESK[d]:
                add(n, g)
            add(n, DESK[d][0], prec="round16", seed=3)
            if d > 1:
                add(n, DESK[d][1], r1=16, r2=8)
                add(n, DESK[d][1], r1=8, r2=8, prec="round16")
    for n, g in (("Heat-2D", "64x64"), ("Box-2D9P", "37x41"), ("Heat-3D", "24x24x24"), ("Heat-1D", "256")):
        add(n, g, fuse=2)
    for n, g in (("Heat-2D", "64x64"), ("Box-3D27P", "17x19x23"), ("1D5P", "301")):
        add(n, g, hw="a100-dense")
    add("Heat-2D", "64x64", corrupt=1)
    add("Box-2D9P", "37x41", corrupt=1)
    add("Heat-2D", "300x260")          # above the 256 desk cap: unverified-scale
    add("Heat-3D", "260x20x20")
    return out


def sha(p: Path) -> str:
    return hashlib.sha256(p.read_bytes()).hexdigest()


def main():
    subprocess.run(["make", "-s", "-C", str(REPO / "oracle"), "ref"], check=True)
    GOLD.mkdir(parents=True, exist_ok=True)
    lutdir = GOLD / "lut"
    shutil.rmtree(lutdir, ignore_errors=True)
    lutdir.mkdir()
    cs = cases()
    with tempfile.TemporaryDirectory() as tmp:
        lines = []
        for c in cs:
            name, stencil, grid, hw, r1, r2, fuse, prec, seed, corrupt = c
            lines.append(f"{tmp}/{name} {stencil} {grid} {hw} {r1} {r2} {fuse} {prec} {seed} {corrupt}")
        r = subprocess.run([str(DRIVER)], input="\n".join(lines) + "\n", capture_output=True, text=True)
        print(r.stdout[-2000:], r.stderr[-2000:])
        table = {}
        for c in cs:
            name, stencil, grid, hw, r1, r2, fuse, prec, seed, corrupt = c
            d = Path(tmp) / name
            entry = {"stencil": stencil, "grid": [int(x) for x in grid.split("x")], "hw": hw, "r1": r1,
                     "r2": r2, "fuse": fuse, "precision": prec, "seed": seed, "corrupt": corrupt,
                     "report": (d / "report.json").read_text()}
            for art in ("a2.s24", "lut.bin"):
                f = d / art
                if f.exists():
                    entry[art] = {"sha256": sha(f), "size": f.stat().st_size}
            lut = d / "lut.bin"
            if lut.exists() and lut.stat().st_size <= 64 << 10:
                shutil.copy(lut, lutdir / f"{name}.bin")
            table[name] = entry
    (GOLD / "cases.json").write_text(json.dumps(table, indent=1, sort_keys=True) + "\n")
    print(f"{len(table)} cases -> {GOLD / 'cases.json'}")


if __name__ == "__main__":
    sys.exit(main())
