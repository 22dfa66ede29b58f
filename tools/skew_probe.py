"""Does the relative placement of the two ping-pong buffers matter? (profiling aid)
Binds the pair at a chosen byte skew (buffer 1 = one allocation + skew) and times
launches. Usage: python tools/skew_probe.py Box-3D27P 512x512x512 [skews_kib=0,4,...]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_22969_b200 import SparseStencil  # noqa: E402
from paper_2506_22969_b200.multigpu import SlabStencil  # noqa: E402

name = sys.argv[1]
dims = [int(x) for x in sys.argv[2].split("x")]
skews = [int(s) for s in (sys.argv[3] if len(sys.argv) > 3 else "0,1,4,16,64,256,1024,1028,2048,2052").split(",")]
steps = 30
src = SlabStencil(name, dims).make_local_input(seed=1)
eng = SparseStencil(name, dims)
nbytes = int(eng.storage["bytes"])
b0 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
for kib in skews:
    raw = torch.empty(nbytes + kib * 1024 + 4096, dtype=torch.uint8, device="cuda")
    b1 = raw[kib * 1024:]
    eng.bind(b0.data_ptr(), b1.data_ptr(), keepalive=[b0, raw])
    eng.upload(src, 0)
    eng.run(4)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.run(steps)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / steps
    print(f"skew {kib:6d} KiB  (b1 - b0) mod 2 MiB = {(b1.data_ptr() - b0.data_ptr()) % (2 << 20):8d}: "
          f"{us:8.2f} us/launch", flush=True)
    del raw, b1
eng.close()
