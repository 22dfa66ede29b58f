"""GPU parity: the sm_100a tcgen05.mma.sp path against the CPU oracle (pinned to
the reference's direct_apply), through the C ABI.

Tolerances (f16 operands, f32 accumulation, f32 storage; inputs are the
reference's dyadic random_grid values):
  * 1 step: BIT-EXACT. Inputs k/256 and the dyadic preset weights are exact in
    f16, every product and partial sum is a multiple of 2^-14 below 2, so the
    f32 accumulation is exact and equals the fp64 oracle.
  * T steps, exact semantics: every step rounds the B operand to f16 (RNE —
    the reference's round16 rounding, fp16.hpp:13-59) and accumulates in f32.
    The GPU result equals the oracle iterated with exactly that rounding
    (f16 operands, fp64-exact sum, f32 storage) BITWISE (the 1-step argument
    above holds for every step's f16 inputs).
  * T steps vs the fp64 oracle: the provable worst case (each step's operand
    rounding is <= 2^-12 on [0, 1) data, the presets are averaging operators
    with positive weights summing to 1, so nothing amplifies it):
        max |gpu - oracle| <= T * 2^-12
    The measured errors, and bounds derived from them, are per BASELINE config
    in tests/test_gpu_baseline_parity.py (profiles/parity_r02.json).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2506_22969_b200 import SparseStencil, sparse_apply, valid_core

pytestmark = pytest.mark.gpu

PRESETS_2D = ["Heat-2D", "Box-2D9P", "Star-2D13P", "Box-2D49P"]
PRESETS_3D = ["Heat-3D", "Box-3D27P"]


def tol_abs(steps: int) -> float:
    return steps * 2.0 ** -12


def run(name, grid, steps):
    eng = SparseStencil(name, list(grid.shape))
    try:
        full = eng.apply_host(grid.astype(np.float32), steps)
        return valid_core(full, steps, eng.r).astype(np.float64), eng.stats()
    finally:
        eng.close()


@pytest.mark.parametrize("name", PRESETS_2D)
@pytest.mark.parametrize("dims", [(97, 301), (130, 129), (64, 128), (300, 517), (21, 23),
                                  (9, 9), (70, 10), (33, 134)])
def test_one_step_bit_exact_2d(gpu, name, dims):
    g = oracle.random_grid(dims, seed=1)
    got, _ = run(name, g, 1)
    assert np.array_equal(got, oracle.direct_apply(name, g, 1))


@pytest.mark.parametrize("name", PRESETS_3D)
@pytest.mark.parametrize("dims", [(9, 21, 150), (5, 6, 7), (20, 24, 40), (33, 17, 129)])
def test_one_step_bit_exact_3d(gpu, name, dims):
    g = oracle.random_grid(dims, seed=2)
    got, _ = run(name, g, 1)
    assert np.array_equal(got, oracle.direct_apply(name, g, 1))


@pytest.mark.parametrize("name,dims,steps", [
    ("Heat-2D", (256, 384), 10), ("Box-2D9P", (333, 290), 25), ("Star-2D13P", (300, 260), 8),
    ("Box-2D49P", (200, 200), 6), ("Heat-3D", (40, 44, 48), 6), ("Box-3D27P", (36, 40, 70), 10),
    ("Heat-2D", (512, 512), 100),
])
def test_multi_step_within_tolerance(gpu, name, dims, steps):
    g = oracle.random_grid(dims, seed=3)
    got, _ = run(name, g, steps)
    want = oracle.direct_apply(name, g, steps)
    err = np.abs(got - want)
    assert err.max() <= tol_abs(steps), (err.max(), tol_abs(steps))
    # exact round16 semantics per step: f16 operands, exact sum, f32 storage
    assert np.array_equal(got, oracle.direct_apply_mt(name, g, steps, round16=True))


def test_sparse_apply_is_a_drop_in_for_direct_apply(gpu):
    g = oracle.random_grid((77, 123), seed=4)
    out = sparse_apply("Box-2D9P", g, 1)
    want = oracle.direct_apply("Box-2D9P", g, 1)
    assert out.shape == want.shape == (75, 121) and out.dtype == np.float64
    assert np.array_equal(out, want)
    three = sparse_apply("Heat-3D", oracle.random_grid((12, 13, 14), 5), 3)
    assert three.shape == (6, 7, 8)
    from paper_2506_22969_b200 import InvalidArgument
    with pytest.raises(InvalidArgument):
        sparse_apply("Box-2D9P", g, 0)
    with pytest.raises(InvalidArgument):
        sparse_apply("Star-2D13P", np.zeros((8, 40)), 2)


def test_constant_field_is_a_fixed_point(gpu):
    for name, dims in (("Box-2D9P", (200, 300)), ("Box-3D27P", (20, 30, 40))):
        c = np.full(dims, 0.375, dtype=np.float32)
        eng = SparseStencil(name, list(dims))
        out = eng.apply_host(c, 50)
        eng.close()
        assert np.array_equal(out, c)


def test_linearity(gpu):
    a = oracle.random_grid((256, 256), 6).astype(np.float32)
    b = oracle.random_grid((256, 256), 7).astype(np.float32)
    eng = SparseStencil("Star-2D13P", [256, 256])
    fa, fb, fab = eng.apply_host(a, 1), eng.apply_host(b, 1), eng.apply_host(a * 0.5 + b * 0.25, 1)
    eng.close()
    core = (slice(3, -3), slice(3, -3))
    assert np.array_equal(fab[core], (0.5 * fa + 0.25 * fb)[core])  # exact: dyadic scalings


def test_row_window_split_equals_full_step(gpu):
    """The multi-GPU schedule (interior window + boundary windows) reproduces
    a full-interior step bitwise."""
    import torch

    for name, dims in (("Box-2D9P", (200, 333)), ("Box-3D27P", (24, 40, 150))):
        g = torch.from_numpy(oracle.random_grid(dims, 8).astype(np.float32)).cuda()
        eng = SparseStencil(name, list(dims))
        eng.bind_torch()
        eng.upload(g, 0)
        dst = eng.run(1, src=0)
        full = eng.download(dst)
        r = eng.r
        n = dims[0]
        eng.upload(g, 0)
        for a, b in ((2 * r, n - 2 * r), (r, 2 * r), (n - 2 * r, n - r)):
            eng.set_row_window(a - r, b - r)
            eng.run(1, src=0)
        eng.set_row_window(0, 0)
        split = eng.download(1)
        eng.close()
        assert np.array_equal(full, split)


def test_torch_device_buffers_and_launch_count(gpu):
    import torch

    dims = (130, 260)
    g = oracle.random_grid(dims, 9)
    eng = SparseStencil("Heat-2D", list(dims))
    bufs = eng.bind_torch()
    assert all(b.is_cuda for b in bufs)
    src = torch.from_numpy(g.astype(np.float32)).cuda()
    eng.upload(src, 0)
    before = eng.stats()["launches"]
    dst = eng.run(7, src=0)
    # one launch per time step (dynamic batch scheduling, PDL between steps); the
    # result lands in the other buffer after an odd count
    assert eng.stats()["launches"] - before == 7 and dst == 1
    out = torch.empty(dims, dtype=torch.float32, device="cuda")
    eng.download(dst, out)
    torch.cuda.synchronize()
    host = eng.apply_host(g.astype(np.float32), 7)
    eng.close()
    assert np.array_equal(out.cpu().numpy(), host)


@pytest.mark.parametrize("name,dims", [("Box-2D9P", (8192, 8192)), ("Box-3D27P", (256, 256, 256))])
def test_full_size_one_step_exact(gpu, name, dims):
    """BASELINE.json grid sizes (3D at 256^3 to bound host RAM for the fp64 oracle)."""
    g = oracle.random_grid(dims, 1)
    got, st = run(name, g, 1)
    want = oracle.direct_apply(name, g, 1)
    assert np.array_equal(got, want)
    assert st["batches"] > st["ctas"]  # persistent CTAs stride over many batches


def test_full_size_multi_step_windows(gpu):
    """Box-2D9P 8192^2 x 40 steps: the valid core of any window depends only on
    the window plus a T*r halo, so the oracle checks windows of the full run."""
    name, n, steps, r = "Box-2D9P", 8192, 40, 1
    g = oracle.random_grid((n, n), 1)
    eng = SparseStencil(name, [n, n])
    full = eng.apply_host(g.astype(np.float32), steps)
    eng.close()
    h = steps * r
    for y0, x0 in ((h, h), (4000, 5000), (n - h - 192, n - h - 192), (h, n - h - 192)):
        sub = g[y0 - h:y0 + 192 + h, x0 - h:x0 + 192 + h]
        want = oracle.direct_apply(name, sub, steps)
        got = full[y0:y0 + 192, x0:x0 + 192].astype(np.float64)
        assert np.abs(got - want).max() <= tol_abs(steps)


@pytest.mark.parametrize("name,dims,edge", [("Box-3D27P", (1024, 1024, 1024), 48),
                                            ("Star-2D13P", (16384, 16384), 160)])
def test_full_size_one_step_windows(gpu, name, dims, edge):
    """The remaining BASELINE.json grids at full size (fp32 input from the engine's
    generator, no fp64 copy of the whole grid): one step, bit-exact against the oracle
    on corner, edge and interior windows (one step's output depends only on the window
    plus an r halo)."""
    import ctypes as C

    from paper_2506_22969_b200 import lib
    from paper_2506_22969_b200._capi import check

    g = np.empty(dims, dtype=np.float32)
    cd = (C.c_uint64 * len(dims))(*dims)
    check(lib().sst_random_grid(len(dims), cd, 9, g.ctypes.data_as(C.c_void_p)))
    eng = SparseStencil(name, list(dims))
    try:
        r = eng.r
        out = eng.apply_host(g, 1)
    finally:
        eng.close()
    n = dims[0]
    for o in (r, n // 2 - edge // 2, n - r - edge):  # same offset on every axis
        lo = [o] * len(dims)
        sub = g[tuple(slice(a - r, a + edge + r) for a in lo)].astype(np.float64)
        want = oracle.direct_apply(name, sub, 1)
        got = out[tuple(slice(a, a + edge) for a in lo)].astype(np.float64)
        assert np.array_equal(got, want), (name, o)
    del out, g


@pytest.mark.parametrize("name,fuse", [("Box-2D9P", 2), ("Heat-2D", 3), ("Box-2D9P", 4), ("Box-3D27P", 2),
                                       ("Heat-3D", 2)])
def test_temporal_fusion(gpu, name, fuse):
    """fuse_time_steps (stencil.cpp:272-347) on the device: the fused operator's
    dyadic weights are exact in f16, so one fused launch on dyadic data equals
    `fuse` reference steps exactly; longer runs stay within the f16 tolerance.
    3D: the fused k = 5 operator runs on the KZ = 5 z-streaming kernels."""
    dims = (26, 40, 150) if "3D" in name else (140, 300)
    g = oracle.random_grid(dims, 12)
    eng = SparseStencil(name, list(dims), fuse=fuse)
    one = valid_core(eng.apply_host(g.astype(np.float32), fuse), fuse, eng.r).astype(np.float64)
    assert eng.stats()["launches"] == 1
    assert np.array_equal(one, oracle.direct_apply(name, g, fuse))
    t = 6 * fuse
    many = valid_core(eng.apply_host(g.astype(np.float32), t), t, eng.r).astype(np.float64)
    from paper_2506_22969_b200 import InvalidArgument
    with pytest.raises(InvalidArgument):
        eng.apply_host(g.astype(np.float32), fuse + 1)
    eng.close()
    want = oracle.direct_apply(name, g, t)
    assert np.abs(many - want).max() <= tol_abs(t)
    out = sparse_apply(name, g, t, fuse=fuse)
    assert np.array_equal(out, many)


# Every compiled kernel variant (A'' in TMEM or in smem, batch shape, ring depths,
# 3D streaming and whole-window kernels) forced through SST_VARIANT: 1 step bit-exact.
VARIANTS_2D = list(range(0, 10)) + list(range(28, 32))
VARIANTS_3D = range(10, 28)


@pytest.mark.parametrize("variant", list(VARIANTS_2D) + list(VARIANTS_3D))
def test_every_variant_bit_exact(gpu, monkeypatch, variant):
    monkeypatch.setenv("SST_VARIANT", str(variant))
    cases = ([("Box-2D9P", (150, 301)), ("Star-2D13P", (90, 140))] if variant in VARIANTS_2D
             else [("Box-3D27P", (14, 37, 150)), ("Heat-3D", (9, 20, 40))])
    for name, dims in cases:
        g = oracle.random_grid(dims, seed=11)
        try:
            eng = SparseStencil(name, list(dims))
        except ValueError:  # this variant does not fit the stencil (smem / TMEM budget)
            continue
        try:
            got = valid_core(eng.apply_host(g.astype(np.float32), 2), 2, eng.r).astype(np.float64)
        finally:
            eng.close()
        cur = oracle.direct_apply(name, g, 1)
        want = oracle.direct_apply(name, cur.astype(np.float16).astype(np.float64), 1)
        want = want.astype(np.float32).astype(np.float64)
        ulp = np.spacing(np.abs(want).astype(np.float32)).astype(np.float64)
        assert np.all(np.abs(got - want) <= ulp), (name, variant, np.abs(got - want).max())


# Deep 3D pipelines over long z runs (the right-edge ring cache is refilled by the
# producer, which runs NP + NB + NACC planes ahead of the epilogue: too few ring
# slots once deadlocked variant 17 on 512^3). 512 x 34 x 1200 gives every CTA a
# run of ~32 planes; every stream variant must finish (child process, timeout) and
# equal the default variant bitwise.
_LONG_RUN = """
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import oracle
from paper_2506_22969_b200 import SparseStencil
dims = (512, 34, 1200)
g = oracle.random_grid(dims, seed=5).astype(np.float32)
outs = []
for v in sys.argv[1:]:
    os.environ["SST_VARIANT"] = v
    try:
        eng = SparseStencil("Box-3D27P", list(dims))
    except ValueError:
        continue
    outs.append(eng.apply_host(g, 3))
    eng.close()
assert all(np.array_equal(o, outs[0]) for o in outs), "variants differ"
print("ok", len(outs))
"""


def test_stream_variants_long_runs(gpu):
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", _LONG_RUN, *map(str, VARIANTS_3D[:15])], cwd=root,
                         capture_output=True, text=True, timeout=240)
    assert res.returncode == 0 and res.stdout.startswith("ok"), res.stderr[-2000:]
    assert int(res.stdout.split()[1]) >= 10  # variants that fit the stencil all ran


# The multi-step dataflow launches (SST_MULTISTEP=1: one launch, T steps, cross-CTA
# progress counters; =2: dynamic batch ownership, per-batch flags) must equal T
# single-step launches bitwise: same arithmetic per step, so any
# ordering bug (a batch loading a neighbour's halo before it was stored) shows up
# as a mismatch. Shapes cover grids with fewer batches than SMs, a single batch
# row or column, ragged edges, and many steps.
@pytest.mark.parametrize("name,dims,steps", [
    ("Box-2D9P", (1030, 2050), 40), ("Heat-2D", (64, 4000), 31), ("Star-2D13P", (700, 300), 12),
    ("Box-2D9P", (4000, 150), 33), ("Heat-2D", (40, 40), 9), ("Box-2D49P", (517, 1031), 10),
    ("Box-2D9P", (2048, 2048), 200),
])
def test_multistep_launch_equals_single_steps(gpu, monkeypatch, name, dims, steps):
    g = oracle.random_grid(dims, seed=21).astype(np.float32)

    def go(multistep, dynamic=True):
        monkeypatch.setenv("SST_MULTISTEP", str(int(multistep)))
        monkeypatch.setenv("SST_DYN", "1" if dynamic else "0")
        eng = SparseStencil(name, list(dims))
        try:
            before = eng.stats()["launches"]
            out = eng.apply_host(g, steps)
            return out, eng.stats()["launches"] - before
        finally:
            eng.close()

    multi, n_multi = go(1)                    # static batch ownership, per-CTA counters
    mdyn, n_mdyn = go(2)                      # dynamic ownership, per-batch flags
    single, n_single = go(0)                  # default: dynamic batch scheduling
    static, _ = go(0, dynamic=False)          # static batch striding
    assert n_multi == 1 and n_mdyn == 1 and n_single == steps
    assert np.array_equal(multi, single)
    assert np.array_equal(mdyn, single)
    assert np.array_equal(static, single)


# ---- split-operand precision (SST_PREC_F16X2): B'' = B_hi + B_lo, ~fp32 steps
@pytest.mark.parametrize("name,dims", [("Box-2D9P", (300, 517)), ("Star-2D13P", (130, 129)),
                                       ("Box-3D27P", (33, 17, 129)), ("Heat-3D", (20, 24, 40)),
                                       ("1D5P", (100003,))])
def test_f16x2_one_step_bit_exact(gpu, name, dims):
    g = oracle.random_grid(dims, seed=4)
    eng = SparseStencil(name, list(dims), precision="f16x2")
    try:
        got = valid_core(eng.apply_host(g.astype(np.float32), 1), 1, eng.r).astype(np.float64)
    finally:
        eng.close()
    assert np.array_equal(got, oracle.direct_apply(name, g, 1))


@pytest.mark.parametrize("name,dims,steps", [("Heat-2D", (512, 512), 100), ("Box-2D9P", (333, 290), 25),
                                             ("Box-3D27P", (36, 40, 70), 10)])
def test_f16x2_multi_step_accuracy(gpu, name, dims, steps):
    """Tolerance: f32 accumulation of <= 49 exact products per step, values < 1:
    max |err| <= 2^-20 (1 + T), and at least 100x below the f16 mode's error."""
    g = oracle.random_grid(dims, seed=6)
    want = oracle.direct_apply(name, g, steps)
    errs = {}
    for prec in ("f16", "f16x2"):
        eng = SparseStencil(name, list(dims), precision=prec)
        try:
            got = valid_core(eng.apply_host(g.astype(np.float32), steps), steps, eng.r).astype(np.float64)
        finally:
            eng.close()
        errs[prec] = np.abs(got - want).max()
    assert errs["f16x2"] <= 2.0 ** -20 * (1 + steps), errs
    assert errs["f16x2"] * 100 < errs["f16"], errs


def test_f16x2_rejects_weights_not_exact_in_binary16(gpu):
    doc = "name = tenth\ndims = 2\nshape = star\nk = 3\npoint = 0 0 : 0.1\npoint = 0 1 : 0.9\n"
    with pytest.raises(ValueError):
        SparseStencil(doc, [64, 64], precision="f16x2")
    SparseStencil(doc, [64, 64], precision="f16").close()  # f16 rounds A'' and is accepted


# ---- 1D presets: the 1D grid folded into a 2D view (rows of W cells overlapping by
# the halo, stencil embedded as a 2D star stencil along the rows; sst_compile)
PRESETS_1D = ["Heat-1D", "1D5P"]


@pytest.mark.parametrize("name", PRESETS_1D)
@pytest.mark.parametrize("n", [5, 9, 129, 301, 8192 + 2, 100003, (1 << 20) + 7])
def test_1d_one_step_bit_exact(gpu, name, n):
    g = oracle.random_grid((n,), seed=8)
    got, _ = run(name, g, 1)
    assert np.array_equal(got, oracle.direct_apply(name, g, 1))


@pytest.mark.parametrize("name,n,steps", [("Heat-1D", 70001, 40), ("1D5P", 20000, 25), ("Heat-1D", 9000, 100)])
def test_1d_multi_step(gpu, name, n, steps):
    g = oracle.random_grid((n,), seed=9)
    got, _ = run(name, g, steps)
    want = oracle.direct_apply(name, g, steps)
    assert np.abs(got - want).max() <= tol_abs(steps)
    # exact round16 semantics per step, as for 2D/3D
    assert np.array_equal(got, oracle.direct_apply_mt(name, g, steps, round16=True))


def test_1d_ring_kept_and_sparse_apply(gpu):
    n, steps = 5000, 7
    g = oracle.random_grid((n,), seed=10).astype(np.float32)
    eng = SparseStencil("1D5P", [n])
    try:
        full = eng.apply_host(g, steps)
    finally:
        eng.close()
    assert np.array_equal(full[:2], g[:2]) and np.array_equal(full[-2:], g[-2:])  # the ring keeps the input
    out = sparse_apply("Heat-1D", g.astype(np.float64), 3)
    assert out.shape == (n - 6,)


@pytest.mark.parametrize("name,n", [("Heat-1D", 8192 * 3 + 2 + 5), ("1D5P", 70001), ("1D5P", 8192 + 4)])
def test_1d_run_t_equals_t_single_steps(gpu, name, n):
    # the ring is fixed after EVERY step (sparstencil.h contract), so the whole
    # fixed-size grid after T steps equals T one-step runs, ring included
    g = oracle.random_grid((n,), seed=11).astype(np.float32)
    eng = SparseStencil(name, [n])
    try:
        many = eng.apply_host(g, 6)
        cur = g
        for _ in range(6):
            cur = eng.apply_host(cur, 1)
            assert np.array_equal(cur[-eng.r:], g[-eng.r:]) and np.array_equal(cur[:eng.r], g[:eng.r])
    finally:
        eng.close()
    assert np.array_equal(many, cur)


# Two row windows in one launch (the NCCL slab mode's boundary windows): after the
# interior window has run, one launch over [r, 2r) and [n - 2r, n - r) must leave the
# buffer exactly as one full step does (rows between the windows are rewritten with
# the values the interior launch produced). Small slabs make the first window's
# batches run over the second window.
@pytest.mark.parametrize("name,dims", [("Box-2D9P", (300, 517)), ("Star-2D13P", (90, 140)),
                                       ("Heat-2D", (40, 1000)), ("Box-2D49P", (200, 300))])
def test_two_window_launch_equals_full_step(gpu, name, dims):
    from paper_2506_22969_b200 import InvalidArgument

    g = oracle.random_grid(dims, seed=8).astype(np.float32)
    eng = SparseStencil(name, list(dims))
    try:
        eng.bind()
        r, n = eng.r, dims[0] - 2 * eng.r
        eng.upload(g, 0)
        eng.set_row_window(0, 0)
        eng.run(1, src=0)
        full = eng.download(1)
        eng.upload(g, 0)
        eng.set_row_window(r, n - r)
        eng.run(1, src=0)
        eng.set_row_windows(0, r, n - r, n)
        launches = eng.stats()["launches"]
        eng.run(1, src=0)
        assert eng.stats()["launches"] == launches + 1
        eng.set_row_window(0, 0)
        split = eng.download(1)
        with pytest.raises(InvalidArgument):
            eng.set_row_windows(5, 3, 7, 9)
    finally:
        eng.close()
    assert np.array_equal(split, full)


def test_live_plans_with_different_smem(gpu):
    # the dynamic-smem attribute is per kernel instantiation: creating a plan of a
    # narrower stencil (less smem, same variant) must not break a live wider plan
    wide_g = oracle.random_grid((200, 300), seed=12)
    narrow_g = oracle.random_grid((100, 130), seed=13)
    wide = SparseStencil("Star-2D13P", [200, 300])
    narrow = SparseStencil("Heat-2D", [100, 130])
    try:
        assert wide.stats()["smem_bytes"] > narrow.stats()["smem_bytes"]
        a = valid_core(narrow.apply_host(narrow_g.astype(np.float32), 1), 1, narrow.r)
        b = valid_core(wide.apply_host(wide_g.astype(np.float32), 1), 1, wide.r)
    finally:
        wide.close()
        narrow.close()
    assert np.array_equal(a, oracle.direct_apply("Heat-2D", narrow_g, 1))
    assert np.array_equal(b, oracle.direct_apply("Star-2D13P", wide_g, 1))
