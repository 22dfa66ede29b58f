"""Multi-slab driver in one process (sst_multi_* / sst_run_steps_multi, the
SURVEY.md §8(b) entry): a global grid cut along its slowest axis into slabs,
halos fused into each slab's epilogue (P2P stores), neighbours ordered by stream
flags. Several slabs share device 0 here (this environment has one GPU); the
schedule and the stores are the same on a multi-GPU node, where neighbours sit on
peer GPUs. The result must equal the single-domain sweep BITWISE over the whole
grid (same per-cell arithmetic, same order)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2506_22969_b200 import InvalidArgument, MultiSlabStencil, SparseStencil, run_steps_multi

pytestmark = pytest.mark.gpu


def single(name, g, steps, fuse=1):
    eng = SparseStencil(name, list(g.shape), fuse=fuse)
    try:
        return eng.apply_host(g, steps)
    finally:
        eng.close()


@pytest.mark.parametrize("name,dims", [("Box-2D9P", (257, 300)), ("Heat-2D", (130, 129)),
                                       ("Star-2D13P", (160, 133)), ("Box-3D27P", (40, 36, 70)),
                                       ("Heat-3D", (33, 17, 129))])
@pytest.mark.parametrize("nslabs", [2, 3, 4])
@pytest.mark.parametrize("steps", [1, 6])
def test_run_steps_multi_bitwise_single_domain(gpu, name, dims, nslabs, steps):
    g = oracle.random_grid(dims, seed=21).astype(np.float32)
    want = single(name, g, steps)
    got = run_steps_multi(name, g, steps, [0] * nslabs)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_multi_repeated_runs_and_reload(gpu):
    """Flag epochs continue across runs; a re-upload restarts from a new grid."""
    g = oracle.random_grid((200, 150), seed=22).astype(np.float32)
    h = oracle.random_grid((200, 150), seed=23).astype(np.float32)
    m = MultiSlabStencil("Box-2D9P", [200, 150], [0, 0, 0])
    try:
        m.upload(g)
        m.run(3)
        m.run(4)
        a = m.download()
        m.upload(h)
        m.run(5)
        b = m.download()
        launches = [m.slab(i)["launches"] for i in range(3)]
        owned = [m.slab(i)["owned"] for i in range(3)]
    finally:
        m.close()
    assert np.array_equal(a, single("Box-2D9P", g, 7))
    assert np.array_equal(b, single("Box-2D9P", h, 5))
    assert launches == [12, 12, 12]  # one launch per slab and step
    assert owned == [(0, 67), (67, 134), (134, 200)]


def test_multi_fused_operator(gpu):
    g = oracle.random_grid((48, 40, 66), seed=24).astype(np.float32)
    m = MultiSlabStencil("Box-3D27P", [48, 40, 66], [0, 0], fuse=2)
    try:
        got = m.apply_host(g, 6)
    finally:
        m.close()
    assert np.array_equal(got, single("Box-3D27P", g, 6, fuse=2))


def test_multi_large_3d(gpu):
    """The north-star stencil at 256^3 over 4 slabs: bitwise the single-domain sweep."""
    g = oracle.random_grid((256, 256, 256), seed=25).astype(np.float32)
    got = run_steps_multi("Box-3D27P", g, 10, [0, 0, 0, 0])
    assert np.array_equal(got, single("Box-3D27P", g, 10))


def test_multi_rejects_thin_slabs(gpu):
    g = oracle.random_grid((10, 64), seed=26).astype(np.float32)
    with pytest.raises(InvalidArgument):
        run_steps_multi("Star-2D13P", g, 1, [0, 0, 0])


@pytest.mark.parametrize("name,dims", [("Box-2D9P", [8000, 40]), ("Box-3D27P", [8000, 40, 20])])
def test_explorer_choice_runs_on_the_device(gpu, name, dims):
    """sst_compile(r1 = r2 = 0) explores the tcgen05-legal layouts and must choose
    one sst_plan_create runs (tall-narrow grids used to get (8, 16))."""
    from paper_2506_22969_b200 import Compiled

    c = Compiled(name, dims, 0, 0)
    assert (c.info["r1"], c.info["r2"]) == (16, 8)
    eng = SparseStencil(c)
    try:
        g = oracle.random_grid(dims, seed=27).astype(np.float32)
        out = eng.apply_host(g, 1)
    finally:
        eng.close()
    assert np.array_equal(out[(slice(1, -1),) * len(dims)].astype(np.float64),
                          oracle.direct_apply(name, g.astype(np.float64), 1))


@pytest.mark.parametrize("name,dims,nslabs", [("Box-3D27P", (40, 36, 70), 3), ("Heat-3D", (33, 17, 129), 2),
                                              ("Box-3D27P", (24, 40, 133), 4), ("Box-2D9P", (257, 300), 3),
                                              ("Star-2D13P", (160, 133), 2), ("Heat-2D", (130, 517), 4)])
def test_multi_binary16_halos(gpu, name, dims, nslabs):
    """Slabs keep binary16 between steps, halos included (the neighbours' binary16
    pairs registered with sst_plan_set_peer_h): bitwise the single-domain sweep, every
    launch a binary16 one, across repeated runs."""
    g = oracle.random_grid(dims, seed=31).astype(np.float32)
    m = MultiSlabStencil(name, list(dims), [0] * nslabs)
    try:
        m.upload(g)
        m.run(5)
        m.run(3)
        got = m.download()
        st = [m.slab(i) for i in range(nslabs)]
    finally:
        m.close()
    assert np.array_equal(got.view(np.uint32), single(name, g, 8).view(np.uint32))
    assert all(s["launches"] == 8 and s["h16_launches"] == 8 for s in st), st
