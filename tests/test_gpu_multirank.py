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


def _rank(rank, world, port, name, owned, rest, steps, fuse, q, halo="nccl"):
    import torch
    import torch.distributed as dist

    from paper_2506_22969_b200.multigpu import SlabStencil

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        glob = np.load(os.environ["SST_TEST_GRID"])
        eng = SlabStencil(name, [owned, *rest], rank=rank, world=world, device=0, fuse=fuse, halo=halo)
        lay = eng.layout
        eng.load(torch.from_numpy(glob[lay.lo:lay.hi].copy()).cuda())
        eng.step(steps)
        torch.cuda.synchronize()
        out = eng.result()
        a, b = lay.computed()
        q.put((rank, lay.lo + a, out[a:b], eng.launches(), int(eng.eng.stats()["h16_launches"])))
        eng.close()
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,owned,rest,steps,fuse,halo", [
    ("Box-2D9P", 200, (333,), 6, 1, "nccl"),
    ("Star-2D13P", 120, (260,), 4, 1, "nccl"),
    ("Box-3D27P", 24, (40, 150), 5, 1, "nccl"),
    ("Box-2D9P", 160, (300,), 6, 2, "nccl"),
    # fused halo exchange: each step's epilogue stores the boundary slices straight
    # into the neighbour's buffer (CUDA IPC mapping; NVLink on a node), stream flags
    ("Box-2D9P", 200, (333,), 6, 1, "p2p"),
    ("Star-2D13P", 120, (261,), 5, 1, "p2p"),
    ("Box-3D27P", 24, (40, 150), 5, 1, "p2p"),
    ("Heat-3D", 20, (33, 129), 4, 1, "p2p"),
])
def test_two_ranks_equal_single_domain(gpu, tmp_path, name, owned, rest, steps, fuse, halo):
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
    port = 29700 + (abs(hash((name, fuse, halo))) % 500)
    procs = [ctx.Process(target=_rank, args=(k, world, port, name, owned, rest, steps, fuse, q, halo))
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
    for rank, g0, rows, launches, h16 in parts:
        assert np.array_equal(rows, full[g0:g0 + len(rows)]), (rank, np.abs(rows - full[g0:g0 + len(rows)]).max())
        # nccl: interior window + one boundary window per step; p2p: one launch per step
        assert launches == (steps // fuse) * (2 if halo == "nccl" else 1)
        # p2p slabs keep binary16 between steps, halos included (IPC-mapped binary16 pairs)
        assert h16 == (steps // fuse if halo == "p2p" else 0)


@pytest.mark.parametrize("name,owned,rest,steps", [("Box-2D9P", 100, (203,), 5), ("Box-3D27P", 16, (30, 70), 4),
                                                   ("Star-2D13P", 64, (150,), 3)])
def test_p2p_halo_stores_single_process(gpu, name, owned, rest, steps):
    """The fused halo data path without IPC: three slab plans in one process whose
    peers are each other's buffers, stepped in rank order on one stream."""
    from paper_2506_22969_b200 import SparseStencil, lib
    from paper_2506_22969_b200._capi import check
    from paper_2506_22969_b200.multigpu import SlabLayout
    import ctypes as C

    world = 3
    dims = [owned * world, *rest]
    glob = np.empty(dims, dtype=np.float32)
    cd = (C.c_uint64 * len(dims))(*dims)
    check(lib().sst_random_grid(len(dims), cd, 5, glob.ctypes.data_as(C.c_void_p)))
    engs, lays = [], []
    for k in range(world):
        probe = SparseStencil(name, dims)
        r = probe.r
        probe.close()
        lay = SlabLayout(owned=owned, world=world, rank=k, r=r)
        e = SparseStencil(name, [lay.local_slices, *rest])
        e.bind()
        e.upload(np.ascontiguousarray(glob[lay.lo:lay.hi]), 0)
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
    for _ in range(steps):
        for e in engs:
            e.run(1, src=cur)
        cur ^= 1
    ref = SparseStencil(name, dims)
    full = ref.apply_host(glob, steps)
    ref.close()
    for e, lay in zip(engs, lays):
        out = e.download(cur)
        a, b = lay.computed()
        assert np.array_equal(out[a:b], full[lay.lo + a:lay.lo + b])
        e.close()
