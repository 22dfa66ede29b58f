"""Per-CTA timeline of one launch (profiling aid, not a bench): SM id, prologue,
main-loop and end timestamps from %globaltimer, summarised as spread statistics.
Usage: [FLUSH=1] python tools/trace_ctas.py Box-3D27P 512x512x512 [variant] [launches=5]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_22969_b200 import SparseStencil, lib  # noqa: E402
from paper_2506_22969_b200._capi import check  # noqa: E402
from paper_2506_22969_b200.multigpu import SlabStencil  # noqa: E402
import ctypes as C  # noqa: E402

name = sys.argv[1]
dims = [int(x) for x in sys.argv[2].split("x")]
if len(sys.argv) > 3 and int(sys.argv[3]) >= 0:
    os.environ["SST_VARIANT"] = sys.argv[3]
launches = int(sys.argv[4]) if len(sys.argv) > 4 else 5
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 1  # time steps per launch (multi-step kernel)
src = SlabStencil(name, dims).make_local_input(seed=1)
eng = SparseStencil(name, dims)
eng.bind_torch()
eng.upload(src, 0)
ctas = eng.stats()["ctas"]
buf = torch.zeros(4 * ctas, dtype=torch.int64, device="cuda")
eng.run(3)
torch.cuda.synchronize()
check(lib().sst_plan_set_trace(eng._h, C.c_void_p(buf.data_ptr())))
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda") if os.environ.get("FLUSH") else None
for i in range(launches):
    if flush is not None:  # bench.py's L2 flush: write then read 256 MB
        flush.fill_(i)
        flush.sum()
        torch.cuda.synchronize()
    eng.run(steps, src=(i * steps) & 1)
    torch.cuda.synchronize()
    t = buf.view(ctas, 4).cpu()
    spins = (t[:, 0] >> 32)
    t[:, 0] &= 0xffffffff
    t0 = int(t[:, 1].min())
    start = (t[:, 1] - t0).double() / 1e3
    main = (t[:, 2] - t0).double() / 1e3
    end = (t[:, 3] - t0).double() / 1e3
    work = end - main
    print(f"launch {i}: span {float(end.max()):.1f} us  start max {float(start.max()):.1f}  "
          f"prologue mean {float((main - start).mean()):.2f} max {float((main - start).max()):.2f}  "
          f"work min {float(work.min()):.1f} mean {float(work.mean()):.1f} max {float(work.max()):.1f}  "
          f"dep polls behind: total {int(spins.sum())} max {int(spins.max())}")
    if i == launches - 1:
        order = torch.argsort(work, descending=True)
        print("slowest CTAs (cta, sm, work us):",
              [(int(c), int(t[c, 0]), round(float(work[c]), 1)) for c in order[:12]])
        print("fastest CTAs (cta, sm, work us):",
              [(int(c), int(t[c, 0]), round(float(work[c]), 1)) for c in order[-6:]])
        byx = {}
        nbx = 4
        for c in range(ctas):
            byx.setdefault(c % nbx, []).append(float(work[c]))
        print("mean work by blockIdx % 4:", {k: round(sum(v) / len(v), 1) for k, v in byx.items()})
check(lib().sst_plan_set_trace(eng._h, None))
eng.close()
