"""Where a single L2-cold launch spends its time (profiling aid, not a bench).
Events around one operator application after bench.py's L2 flush, against variants:
a no-op torch kernel between the flush and the launch, back-to-back launches, and
the in-kernel span from the CTA trace. Usage: python tools/launch_gap.py Heat-2D 4096x4096
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_22969_b200 import SparseStencil, lib  # noqa: E402
from paper_2506_22969_b200._capi import check  # noqa: E402
from paper_2506_22969_b200.multigpu import SlabStencil  # noqa: E402

name = sys.argv[1]
dims = [int(x) for x in sys.argv[2].split("x")]
reps = 20
src = SlabStencil(name, dims).make_local_input(seed=1)
eng = SparseStencil(name, dims)
eng.bind_torch()
eng.upload(src, 0)
eng.run(4)
stream = torch.cuda.current_stream()
big = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.zeros(64 << 20, dtype=torch.int32, device="cuda")
tiny = torch.zeros(1, device="cuda")
ctas = eng.stats()["ctas"]
trace = torch.zeros(4 * ctas, dtype=torch.int64, device="cuda")


def timed(label, pre, nlaunch=1, use_trace=False):
    evs = []
    spans = []
    for i in range(reps):
        pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for j in range(nlaunch):
            eng.run(1, src=(i + j) & 1)
        b.record(stream)
        evs.append((a, b))
        if use_trace:
            torch.cuda.synchronize()
            t = trace.view(ctas, 4).cpu()
            spans.append(float((t[:, 3].max() - t[:, 1].min())) / 1e3)
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) * 1e3 / nlaunch for a, b in evs)
    extra = f"  in-kernel span median {sorted(spans)[len(spans) // 2]:.1f} us" if spans else ""
    print(f"{label:58s} per launch: median {ms[len(ms) // 2]:.1f} us  min {ms[0]:.1f}{extra}")


def flush():
    big.add_(1)
    rd.sum()


def flush_tiny():
    flush()
    tiny.add_(1)


timed("flush; ev; launch; ev (bench.py)", flush)
timed("flush; tiny torch kernel; ev; launch; ev", flush_tiny)
timed("no flush; ev; launch; ev", lambda: None)
timed("flush; ev; 4 launches; ev (per launch)", flush, 4)
timed("flush; ev; 16 launches; ev (per launch)", flush, 16)
check(lib().sst_plan_set_trace(eng._h, C.c_void_p(trace.data_ptr())))
timed("flush; ev; launch; ev  [traced]", flush, 1, True)
check(lib().sst_plan_set_trace(eng._h, None))
eng.close()
