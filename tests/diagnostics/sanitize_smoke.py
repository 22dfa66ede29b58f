"""Small device runs for compute-sanitizer (memcheck / synccheck): every kernel
family on tiny ragged grids. Usage: compute-sanitizer --tool memcheck python tests/diagnostics/sanitize_smoke.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402
from paper_2506_22969_b200 import SparseStencil, valid_core  # noqa: E402

cases = [("Box-2D9P", (97, 301), "f16", 3), ("Star-2D13P", (70, 140), "f16x2", 2),
         ("Box-3D27P", (12, 23, 131), "f16", 3), ("Heat-3D", (9, 20, 40), "f16x2", 2),
         ("Heat-1D", (1001,), "f16", 4), ("Box-2D49P", (300, 517), "f16", 1)]
for name, dims, prec, steps in cases:
    g = oracle.random_grid(dims, seed=1)
    eng = SparseStencil(name, list(dims), precision=prec)
    out = valid_core(eng.apply_host(g.astype(np.float32), steps), steps, eng.r)
    eng.close()
    want = oracle.direct_apply(name, g, steps)
    print(name, dims, prec, steps, "max err %.3g" % np.abs(out - want).max(), flush=True)
# temporally fused 3D (KZ = 5 z-streaming kernel)
g = oracle.random_grid((14, 24, 60), seed=3)
eng = SparseStencil("Box-3D27P", [14, 24, 60], fuse=2)
out = valid_core(eng.apply_host(g.astype(np.float32), 2), 2, eng.r)
eng.close()
print("Box-3D27P fuse 2 max err %.3g" % np.abs(out - oracle.direct_apply("Box-3D27P", g, 2)).max(), flush=True)
# dynamic batch scheduling on a small grid
os.environ["SST_DYN"] = "1"
eng = SparseStencil("Box-2D9P", [150, 301])
eng.apply_host(oracle.random_grid((150, 301), seed=4).astype(np.float32), 3)
eng.close()
del os.environ["SST_DYN"]
# slab P2P halo stores (2D dynamic-peer and 3D PEER instantiations): three slab
# plans in one process whose peers are each other's buffers
import ctypes as C  # noqa: E402
from paper_2506_22969_b200 import lib  # noqa: E402
from paper_2506_22969_b200._capi import check  # noqa: E402
from paper_2506_22969_b200.multigpu import SlabLayout  # noqa: E402
for name, owned, rest in (("Box-2D9P", 40, (203,)), ("Box-3D27P", 10, (30, 70))):
    world, dims = 3, None
    engs, lays = [], []
    for k in range(world):
        lay = SlabLayout(owned=owned, world=world, rank=k, r=1)
        e = SparseStencil(name, [lay.local_slices, *rest])
        e.bind()
        e.upload(oracle.random_grid((lay.local_slices, *rest), seed=k).astype(np.float32), 0)
        engs.append(e)
        lays.append(lay)
    bufs = []
    for e in engs:
        b0, b1 = C.c_void_p(), C.c_void_p()
        check(lib().sst_plan_buffers(e._h, C.byref(b0), C.byref(b1)))
        bufs.append((b0, b1))
    for k, e in enumerate(engs):
        for which, nb in ((0, k - 1), (1, k + 1)):
            if 0 <= nb < world:
                check(lib().sst_plan_set_peer(e._h, which, bufs[nb][0], bufs[nb][1], lays[nb].local_slices))
    cur = 0
    for _ in range(2):
        for e in engs:
            e.run(1, src=cur)
        cur ^= 1
    for e in engs:
        e.download(cur)
        e.close()
    print(name, "p2p slabs done", flush=True)
# batched binary16 runs (sst_run_steps_batch), 2D + 3D interleaved, ragged edges
import torch  # noqa: E402
from paper_2506_22969_b200 import run_batch  # noqa: E402
bs = [SparseStencil("Heat-2D", [70, 203]), SparseStencil("Heat-3D", [11, 19, 77])]
for e, d in zip(bs, ([70, 203], [11, 19, 77])):
    e.bind()
    e.upload(torch.from_numpy(oracle.random_grid(d, seed=5).astype(np.float32)).cuda(), 0)
run_batch(bs, 3)
torch.cuda.synchronize()
for e in bs:
    e.close()
print("batch done", flush=True)
os.environ["SST_MULTISTEP"] = "1"
eng = SparseStencil("Box-2D9P", [200, 300])
eng.apply_host(oracle.random_grid((200, 300), seed=2).astype(np.float32), 5)
eng.close()
print("sanitize smoke done")
