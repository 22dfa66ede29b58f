"""Binary16 inter-step storage (SST_PREC_F16 runs of T >= 2 steps).

Steps 1 .. T-1 are stored as binary16 (RNE in the producing epilogue) and the
last step as fp32. The only consumer of an intermediate grid is the next step's
gather, which rounds its operand to binary16 RNE (the reference round16
semantics, fp16.hpp:13-59), so the result must be BITWISE the fp32-storage
result — over the whole grid, boundary ring included. SST_H16=0 selects the
fp32-storage path for the comparison (read per call).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
from paper_2506_22969_b200 import SparseStencil, valid_core

pytestmark = pytest.mark.gpu


def run_both(name, grid, steps, fuse=1):
    eng = SparseStencil(name, list(grid.shape), fuse=fuse)
    try:
        assert eng.stats()["h16_capable"] == 1
        os.environ["SST_H16"] = "0"
        ref = eng.apply_host(grid, steps)
        s0 = eng.stats()
        os.environ["SST_H16"] = "1"
        got = eng.apply_host(grid, steps)
        s1 = eng.stats()
    finally:
        os.environ.pop("SST_H16", None)
        eng.close()
    launches = steps // fuse
    assert s0["h16_launches"] == 0
    assert s1["h16_launches"] == (launches if launches > 1 else 0)
    assert s1["launches"] - s0["launches"] == launches
    return ref, got, eng


@pytest.mark.parametrize("name", ["Heat-2D", "Box-2D9P", "Star-2D13P", "Box-2D49P"])
@pytest.mark.parametrize("dims", [(97, 301), (130, 129), (21, 23), (70, 10), (300, 517), (9, 9)])
@pytest.mark.parametrize("steps", [2, 3, 6])
def test_h16_storage_bitwise_equals_f32_storage(gpu, name, dims, steps):
    g = oracle.random_grid(dims, seed=11).astype(np.float32)
    ref, got, _ = run_both(name, g, steps)
    assert np.array_equal(ref.view(np.uint32), got.view(np.uint32))


@pytest.mark.parametrize("name,dims,steps", [("Heat-2D", (256, 384), 10), ("Box-2D9P", (333, 290), 25),
                                             ("Star-2D13P", (300, 260), 8)])
def test_h16_storage_matches_round16_oracle(gpu, name, dims, steps):
    g = oracle.random_grid(dims, seed=3)
    ref, got, eng = run_both(name, g.astype(np.float32), steps)
    core = valid_core(got, steps, eng.r).astype(np.float64)
    assert np.array_equal(core, oracle.direct_apply_mt(name, g, steps, round16=True))


def test_h16_wide_range_values(gpu):
    """Values outside binary16's normal range (overflow to inf, subnormals, signs):
    the epilogue's RNE and the gather's RNE see the same f32 value."""
    rng = np.random.default_rng(5)
    g = (rng.standard_normal((200, 333)) * np.exp2(rng.integers(-30, 18, (200, 333)))).astype(np.float32)
    ref, got, _ = run_both("Box-2D9P", g, 4)
    assert np.array_equal(ref.view(np.uint32), got.view(np.uint32))


@pytest.mark.parametrize("fuse", [2, 4])
def test_h16_fused_operator(gpu, fuse):
    g = oracle.random_grid((257, 300), seed=12).astype(np.float32)
    ref, got, _ = run_both("Box-2D9P", g, 4 * fuse, fuse=fuse)
    assert np.array_equal(ref.view(np.uint32), got.view(np.uint32))


def test_h16_full_size_box2d(gpu):
    """BASELINE configs[1] grid: 8192^2, 20 steps, whole grid bitwise."""
    g = oracle.random_grid((8192, 8192), seed=1).astype(np.float32)
    ref, got, _ = run_both("Box-2D9P", g, 20)
    assert np.array_equal(ref.view(np.uint32), got.view(np.uint32))


def test_h16_run_steps_device_buffers(gpu):
    """sst_run_steps on device buffers: the result lands in the buffer plain
    ping-pong ends on ((src + T) & 1), both parities, and the other buffer's
    ring is untouched."""
    import torch

    g = oracle.random_grid((150, 260), seed=13).astype(np.float32)
    want = {}
    for h16 in ("0", "1"):
        os.environ["SST_H16"] = h16
        eng = SparseStencil("Star-2D13P", [150, 260])
        try:
            eng.bind()
            for src in (0, 1):
                for steps in (2, 5):
                    eng.upload(torch.from_numpy(g).cuda(), src)
                    torch.cuda.synchronize()
                    dst = eng.run(steps, src)
                    assert dst == (src + steps) & 1
                    out = eng.download(dst)
                    key = (src, steps)
                    if h16 == "0":
                        want[key] = out
                    else:
                        assert np.array_equal(out.view(np.uint32), want[key].view(np.uint32))
        finally:
            os.environ.pop("SST_H16", None)
            eng.close()


# ---------------------------------------------------------------- 3D z-streaming kernel
@pytest.mark.parametrize("name", ["Heat-3D", "Box-3D27P"])
@pytest.mark.parametrize("dims", [(20, 24, 40), (9, 9, 9), (13, 70, 131), (34, 33, 262), (11, 40, 517)])
@pytest.mark.parametrize("steps", [2, 5])
def test_h16_3d_bitwise_equals_f32_storage(gpu, name, dims, steps):
    """Ragged right edges of every residue mod 8 (the binary16 store map's last
    16-byte chunk carries ring / pad cells staged from the ring cache)."""
    g = oracle.random_grid(dims, seed=21).astype(np.float32)
    ref, got, _ = run_both(name, g, steps)
    assert np.array_equal(ref.view(np.uint32), got.view(np.uint32))


@pytest.mark.parametrize("gx", [37, 38, 39, 40, 41, 42, 43, 44])
def test_h16_3d_every_edge_residue(gpu, gx):
    g = oracle.random_grid((12, 19, gx), seed=gx).astype(np.float32)
    ref, got, _ = run_both("Box-3D27P", g, 3)
    assert np.array_equal(ref.view(np.uint32), got.view(np.uint32))


def test_h16_3d_matches_round16_oracle(gpu):
    g = oracle.random_grid((40, 48, 70), seed=4)
    ref, got, eng = run_both("Box-3D27P", g.astype(np.float32), 6)
    core = valid_core(got, 6, eng.r).astype(np.float64)
    assert np.array_equal(core, oracle.direct_apply_mt("Box-3D27P", g, 6, round16=True))


def test_h16_3d_full_size_box3d(gpu):
    """BASELINE configs[3] grid: Box-3D27P 512^3, 6 steps, whole grid bitwise."""
    g = oracle.random_grid((512, 512, 512), seed=1).astype(np.float32)
    ref, got, _ = run_both("Box-3D27P", g, 6)
    assert np.array_equal(ref.view(np.uint32), got.view(np.uint32))


def test_h16_3d_run_steps_device_buffers(gpu):
    import torch

    g = oracle.random_grid((18, 30, 77), seed=17).astype(np.float32)
    want = {}
    for h16 in ("0", "1"):
        os.environ["SST_H16"] = h16
        eng = SparseStencil("Heat-3D", [18, 30, 77])
        try:
            eng.bind()
            for src in (0, 1):
                for steps in (2, 3):
                    eng.upload(torch.from_numpy(g).cuda(), src)
                    torch.cuda.synchronize()
                    dst = eng.run(steps, src)
                    assert dst == (src + steps) & 1
                    out = eng.download(dst)
                    if h16 == "0":
                        want[(src, steps)] = out
                    else:
                        assert np.array_equal(out.view(np.uint32), want[(src, steps)].view(np.uint32))
        finally:
            os.environ.pop("SST_H16", None)
            eng.close()


# ---------------------------------------------------------------- batched runs
def test_run_batch_equals_individual_runs(gpu):
    """sst_run_steps_batch: several independent grids (different stencils, 2D and 3D)
    stepped together, launches interleaved, each bitwise its own sst_run_steps."""
    import torch

    from paper_2506_22969_b200 import run_batch

    cases = [("Heat-2D", (130, 300)), ("Box-2D9P", (97, 301)), ("Box-3D27P", (20, 24, 70)), ("Heat-2D", (64, 64))]
    engs, grids = [], []
    try:
        for name, dims in cases:
            e = SparseStencil(name, list(dims))
            e.bind()
            engs.append(e)
            grids.append(torch.from_numpy(oracle.random_grid(dims, seed=len(engs)).astype(np.float32)).cuda())
        for steps in (1, 2, 7):
            want = []
            for e, g in zip(engs, grids):
                e.upload(g, 0)
                want.append(e.download(e.run(steps, 0)))
            for e, g, src in zip(engs, grids, (0, 1, 0, 1)):
                e.upload(g, src)
            h0 = [e.stats()["h16_launches"] for e in engs]
            dst = run_batch(engs, steps, [0, 1, 0, 1])
            assert dst == [steps & 1, (1 + steps) & 1, steps & 1, (1 + steps) & 1]
            for e, d, w, h in zip(engs, dst, want, h0):
                assert np.array_equal(e.download(d).view(np.uint32), w.view(np.uint32))
                assert e.stats()["h16_launches"] - h == (steps if steps > 1 else 0)
    finally:
        for e in engs:
            e.close()


def test_run_batch_rejects_bad_batches(gpu):
    from paper_2506_22969_b200 import InvalidArgument, run_batch

    e = SparseStencil("Heat-2D", [64, 64])
    try:
        e.bind()
        with pytest.raises(InvalidArgument):
            run_batch([e, e], 2)
        f = SparseStencil("Box-2D9P", [64, 64], fuse=2)
        try:
            f.bind()
            with pytest.raises(InvalidArgument):
                run_batch([e, f], 2)
        finally:
            f.close()
    finally:
        e.close()


@pytest.mark.parametrize("name,dims,steps", [("Box-2D9P", (8192, 8192), 1000), ("Box-3D27P", (512, 512, 512), 100),
                                             ("Star-2D13P", (16384, 16384), 100)])
def test_h16_baseline_configs_whole_grid_at_stated_T(gpu, name, dims, steps):
    """The BASELINE configs at their stated T, whole grid: binary16 inter-step storage
    is bitwise the fp32-storage sweep (so the per-config parity of the fp32 path,
    test_gpu_baseline_parity.py, carries over cell for cell)."""
    g = oracle.random_grid(dims, seed=1).astype(np.float32)
    ref, got, _ = run_both(name, g, steps)
    assert np.array_equal(ref.view(np.uint32), got.view(np.uint32))


@pytest.mark.parametrize("dims,n", [((130, 300), 4), ((64, 64), 2), ((257, 517), 3)])
def test_run_batch_grouped_identical_grids(gpu, dims, n):
    """Identical 2D grids in a batch run as ONE launch per step for the whole group
    (kModeGroup: per-grid tensor maps in global memory): bitwise each grid's own run,
    from mixed source buffers, and the same as the interleaved schedule (SST_GROUP=0)."""
    import torch

    from paper_2506_22969_b200 import run_batch

    engs = []
    try:
        grids = [torch.from_numpy(oracle.random_grid(dims, seed=40 + i).astype(np.float32)).cuda() for i in range(n)]
        for _ in range(n):
            e = SparseStencil("Box-2D9P", list(dims))
            e.bind()
            engs.append(e)
        srcs = [i & 1 for i in range(n)]
        for steps in (2, 5):
            want = []
            for e, g in zip(engs, grids):
                e.upload(g, 0)
                want.append(e.download(e.run(steps, 0)))
            for mode in ("1", "0"):
                os.environ["SST_GROUP"] = mode
                for e, g, s in zip(engs, grids, srcs):
                    e.upload(g, s)
                l0 = [e.stats()["launches"] for e in engs]
                dst = run_batch(engs, steps, srcs)
                for e, d, w, l in zip(engs, dst, want, l0):
                    assert np.array_equal(e.download(d).view(np.uint32), w.view(np.uint32)), mode
                    assert e.stats()["launches"] - l == steps
    finally:
        os.environ.pop("SST_GROUP", None)
        for e in engs:
            e.close()
