"""Shared-memory wavefronts per SASS instruction of an ncu report (source page,
sass view): the instructions with the most L1 shared wavefronts and their excess
over the ideal (bank conflicts). Usage: python tools/ncu_smem.py report.ncu-rep [top=25]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
iw, ii, ix, isrc, ie = (h.index(c) for c in ("L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal",
                                             "L1 Wavefronts Shared Excessive", "Source", "Instructions Executed"))
f = lambda r, i: float(r[i] or 0)
tw = sum(f(r, iw) for r in data)
tx = sum(f(r, ix) for r in data)
print(f"shared wavefronts {tw:.0f}, excessive {tx:.0f} ({tx / max(tw, 1) * 100:.1f}%)")
for k in sorted(range(len(data)), key=lambda k: -f(data[k], iw))[:top]:
    r = data[k]
    print(f"{k:5d} wf {f(r, iw):10.0f} ({f(r, iw) / tw * 100:4.1f}%) ideal {f(r, ii):10.0f} excess {f(r, ix):10.0f} "
          f"inst {f(r, ie):9.0f}  {r[isrc][:70]}")
