"""Aggregate an ncu report's warp-stall samples by CUDA source line (needs a
-lineinfo build and --import-source on): where the kernel's warps wait, per role.
Usage: python tools/ncu_lines.py report.ncu-rep [top=40]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# the csv holds one block per source file: a "File" marker row, then a header
data, cur_file, hdr = [], None, None
for r in rows:
    if not r:
        continue
    if r[0].startswith("File") or (len(r) == 1 and r[0].endswith((".cuh", ".cu", ".h"))):
        cur_file = r[-1]
        hdr = None
        continue
    if "Source" in r and "Warp Stall Sampling (All Samples)" in r:
        hdr = r
        continue
    if hdr is None:
        continue
    d = dict(zip(hdr, r))
    try:
        samp = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    stalls = {k[6:]: float(v or 0) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k
              and v not in ("", None)}
    data.append((samp, cur_file, d.get("#", d.get("Line", "?")), d.get("Source", "")[:90], stalls))
T = sum(x[0] for x in data) or 1
print(f"total samples {T:.0f}")
for samp, f, ln, src, st in sorted(data, key=lambda x: -x[0])[:top]:
    main = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{samp / T * 100:5.1f}%  {str(f).split('/')[-1]}:{ln:<5} {src.strip()[:70]:70s} "
          + " ".join(f"{k}:{v / max(samp, 1) * 100:.0f}%" for k, v in main))
