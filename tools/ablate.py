"""Kernel ablation timing (profiling aid, not a bench; needs the profiling build:
`SST_ABLATION=1 python -m paper_2506_22969_b200.build`): for each config, variant and
debug mode (1 no stores, 2 no gather, 4 no MMA), time `steps` launches with CUDA
events and print microseconds per launch. Usage:
    python tools/ablate.py Box-3D27P 512x512x512 [variants=-1,5,6] [modes=0,1,2,4,7] [steps=50]
"""
import os
import sys

# the ablation bits are compiled only into the profiling build of the library
# (SST_ABLATION=1 python -m paper_2506_22969_b200.build -> libsparstencil_ablation.so);
# modes other than 0 need it, mode 0 alone also runs on the production library
os.environ.setdefault("SST_LIB", "ablation")

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_22969_b200 import SparseStencil  # noqa: E402
from paper_2506_22969_b200.multigpu import SlabStencil  # noqa: E402

name = sys.argv[1]
dims = [int(x) for x in sys.argv[2].split("x")]
variants = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "-1").split(",")]
modes = [int(m) for m in (sys.argv[4] if len(sys.argv) > 4 else "0,1,2,4").split(",")]
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 50
fuse = int(os.environ.get("FUSE", "1"))

flush = (torch.empty(256 << 20, dtype=torch.uint8, device="cuda"),
         torch.zeros(64 << 20, dtype=torch.int32, device="cuda")) if os.environ.get("FLUSH") else None
src = SlabStencil(name, dims, fuse=fuse).make_local_input(seed=1)
for v in variants:
    for m in modes:
        if v >= 0:
            os.environ["SST_VARIANT"] = str(v)
        else:
            os.environ.pop("SST_VARIANT", None)
        os.environ["SST_DEBUG_MODE"] = str(m)
        try:
            eng = SparseStencil(name, dims, fuse=fuse)
        except Exception as e:  # variant does not fit this stencil
            print(f"variant {v:2d} mode {m} : {e}", flush=True)
            continue
        eng.bind_torch()
        eng.upload(src, 0)
        eng.run(3 * fuse)
        torch.cuda.synchronize()
        if flush is None:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            eng.run(steps * fuse)
            b.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(b) * 1e3 / steps
        else:  # L2 flushed before every launch (as bench.py does for small grids)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(steps)]
            cur = 0
            for a, b in evs:
                flush[0].add_(1)
                if os.environ.get("FLUSH") == "2":
                    flush[1].sum()
                a.record()
                cur = eng.run(fuse, src=cur)
                b.record()
            torch.cuda.synchronize()
            us = sum(a.elapsed_time(b) for a, b in evs) * 1e3 / steps
        st = eng.stats()
        cells = 1
        for d in dims:
            cells *= d
        print(f"variant {v:2d} mode {m} : {us:8.2f} us/launch  {cells * fuse / us / 1e3:7.1f} GSt/s  "
              f"patch {st['patch_w']}x{st['patch_h']}x{st['patch_planes']} stages {st['patch_stages']} "
              f"ctas {st['ctas']} smem {st['smem_bytes']} h16 {st['h16_patch_stages']}", flush=True)
        eng.close()
