"""Compute-side cost of the slab schedules on one GPU (profiling aid): a middle
rank's slab (owned slices + r halo slices each side) stepped as the P2P mode does
(one full-interior launch per step) and as the NCCL mode does (interior window,
then the two boundary windows: 3 launches per step, or in 2D one two-window launch),
without the exchange itself.
Usage: python tools/slab_overhead.py Box-3D27P 1024x1024x1024 [world=8] [steps=20]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_22969_b200 import SparseStencil  # noqa: E402
from paper_2506_22969_b200.multigpu import SlabLayout  # noqa: E402

name = sys.argv[1]
dims = [int(x) for x in sys.argv[2].split("x")]
world = int(sys.argv[3]) if len(sys.argv) > 3 else 8
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
probe = SparseStencil(name, [16] * len(dims))
r = probe.r
probe.close()
lay = SlabLayout(owned=dims[0], world=world, rank=world // 2, r=r)
local = [lay.local_slices, *dims[1:]]
eng = SparseStencil(name, local)
eng.bind_torch()
g = torch.rand(local, device="cuda")
eng.upload(g, 0)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def timed(fn):
    fn(3)
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    fn(steps)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / steps


def p2p_shape(n):
    eng.set_row_window(0, 0)
    cur = 0
    for _ in range(n):
        cur = eng.run(1, src=cur)


def nccl_shape(n, merged=False):
    cur = 0
    for _ in range(n):
        a, b = lay.interior_window()
        eng.set_row_window(a - r, b - r)
        eng.run(1, src=cur)
        bw = lay.boundary_windows()
        if merged:  # both boundary windows in one launch (what SlabStencil does in 2D)
            eng.set_row_windows(bw[0][0] - r, bw[0][1] - r, bw[1][0] - r, bw[1][1] - r)
            eng.run(1, src=cur)
        else:
            for a, b in bw:
                eng.set_row_window(a - r, b - r)
                eng.run(1, src=cur)
        cur ^= 1
    eng.set_row_window(0, 0)


t1, t3 = timed(p2p_shape), timed(nccl_shape)
t2 = timed(lambda n: nccl_shape(n, True)) if len(dims) == 2 else None
cells = 1
for d in dims:
    cells *= d
print(f"{name} {'x'.join(map(str, dims))} per GPU, slab of {lay.local_slices} slices (world {world}): "
      f"one launch {t1:.1f} us/step ({cells / t1 / 1e3:.1f} GSt/s owned), "
      f"interior + 2 boundary windows {t3:.1f} us/step ({cells / t3 / 1e3:.1f} GSt/s), x{t3 / t1:.3f}"
      + (f"; interior + one two-window launch {t2:.1f} us/step, x{t2 / t1:.3f}" if t2 else ""))
eng.close()
