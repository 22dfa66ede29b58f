"""The slab-decomposed multi-GPU schedule (multigpu.SlabStencil) executed for real
on the device: two ranks over gloo sharing the one B200 of this environment
(NCCL refuses two ranks per GPU, so halos are host-staged here; on a node the
same code exchanges them with NCCL). Each rank runs the interior window while
halos fly, then the boundary windows. The assembled result must equal a
single-domain sweep of the global grid bitwise: every cell is computed with the
same A'' row and the same tensor-core accumulation order wherever its tile is."""
from __future__ import annotations

import os

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _rank(rank, world, port, name, owned, rest, steps, fuse, q):
    import torch
    import torch.distributed as dist

    from paper_2506_22969_b200.multigpu import SlabStencil

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        glob = np.load(os.environ["SST_TEST_GRID"])
        eng = SlabStencil(name, [owned, *rest], rank=rank, world=world, device=0, fuse=fuse)
        lay = eng.layout
        eng.load(torch.from_numpy(glob[lay.lo:lay.hi].copy()).cuda())
        eng.step(steps)
        torch.cuda.synchronize()
        out = eng.result()
        a, b = lay.computed()
        q.put((rank, lay.lo + a, out[a:b], eng.launches()))
        eng.close()
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,owned,rest,steps,fuse", [
    ("Box-2D9P", 200, (333,), 6, 1),
    ("Star-2D13P", 120, (260,), 4, 1),
    ("Box-3D27P", 24, (40, 150), 5, 1),
    ("Box-2D9P", 160, (300,), 6, 2),
])
def test_two_ranks_equal_single_domain(gpu, tmp_path, name, owned, rest, steps, fuse):
    from paper_2506_22969_b200 import SparseStencil
    from paper_2506_22969_b200._capi import check, lib
    import ctypes as C

    world = 2
    dims = [owned * world, *rest]
    glob = np.empty(dims, dtype=np.float32)
    cd = (C.c_uint64 * len(dims))(*dims)
    check(lib().sst_random_grid(len(dims), cd, 21, glob.ctypes.data_as(C.c_void_p)))
    path = tmp_path / "grid.npy"
    np.save(path, glob)
    os.environ["SST_TEST_GRID"] = str(path)

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + (abs(hash((name, fuse))) % 500)
    procs = [ctx.Process(target=_rank, args=(k, world, port, name, owned, rest, steps, fuse, q))
             for k in range(world)]
    for p in procs:
        p.start()
    parts = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0

    ref = SparseStencil(name, dims, fuse=fuse)
    full = ref.apply_host(glob, steps)
    ref.close()
    for rank, g0, rows, launches in parts:
        assert np.array_equal(rows, full[g0:g0 + len(rows)]), (rank, np.abs(rows - full[g0:g0 + len(rows)]).max())
        assert launches == (steps // fuse) * 2  # interior window + one boundary window per step
