"""The CPU oracle (oracle/oracle.c, the checker every GPU parity test uses) is
pinned against the reference's own direct_apply and random_grid
(tests/golden/direct_apply.npz, written by oracle/make_golden.py from the
reference build), and against the reference live when it is present."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import GOLDEN

GOLD = np.load(GOLDEN / "direct_apply.npz")


@pytest.mark.parametrize("name", oracle.PRESETS)
def test_oracle_matches_reference_golden(name):
    g = GOLD[f"{name}/input"]
    assert np.array_equal(oracle.random_grid(list(g.shape), seed=5), g)
    for steps in (1, 2, 3):
        want = GOLD[f"{name}/steps{steps}"]
        got = oracle.direct_apply(name, g, steps)
        assert got.shape == want.shape
        assert np.array_equal(got, want), (name, steps)  # bit-exact fp64


def test_oracle_preset_points():
    # point counts, lexicographic order, weights summing to 1 (test_stencil.cpp:57-82)
    for name, n in (("Heat-1D", 3), ("1D5P", 5), ("Heat-2D", 5), ("Box-2D9P", 9),
                    ("Star-2D13P", 13), ("Box-2D49P", 49), ("Heat-3D", 7), ("Box-3D27P", 27)):
        _, _, offs, w = oracle.preset(name)
        assert len(w) == n and w.sum() == 1.0
        assert [tuple(o) for o in offs] == sorted(tuple(o) for o in offs)


def test_oracle_properties():
    g = oracle.random_grid([40, 44], seed=2)
    h = oracle.random_grid([40, 44], seed=3)
    # linearity (test_stencil.cpp:176-188)
    a = oracle.direct_apply("Box-2D9P", 0.5 * g + 0.25 * h, 2)
    b = 0.5 * oracle.direct_apply("Box-2D9P", g, 2) + 0.25 * oracle.direct_apply("Box-2D9P", h, 2)
    assert np.allclose(a, b, rtol=0, atol=1e-15)
    # constant field is a fixed point (weights sum to 1)
    c = np.full((20, 21, 22), 0.375)
    assert np.array_equal(oracle.direct_apply("Box-3D27P", c, 3), np.full((14, 15, 16), 0.375))
    with pytest.raises(ValueError):
        oracle.direct_apply("Box-2D9P", np.zeros((2, 9)), 1)


@pytest.mark.skipif(not oracle.ref_available(), reason="reference build not present")
def test_oracle_matches_reference_live():
    for name, dims in (("Heat-2D", [61, 70]), ("Star-2D13P", [50, 47]), ("Heat-3D", [13, 15, 17])):
        g = oracle.random_grid(dims, seed=11)
        assert np.array_equal(oracle.direct_apply(name, g, 2), oracle.ref_direct_apply(name, g, 2))
        assert np.array_equal(oracle.ref_direct_apply_slabs(name, g, 3),
                              oracle.ref_direct_apply(name, g, 1))


@pytest.mark.parametrize("name,dims,steps", [("Heat-2D", (61, 70), 5), ("Box-3D27P", (13, 15, 17), 3),
                                             ("Star-2D13P", (50, 47), 2), ("1D5P", (300,), 7)])
def test_threaded_oracle_equals_serial(name, dims, steps):
    g = oracle.random_grid(dims, seed=11)
    want = oracle.direct_apply(name, g, steps)
    for threads in (1, 3, 8):
        assert np.array_equal(oracle.direct_apply_mt(name, g, steps, threads), want)


@pytest.mark.parametrize("name,dims,steps", [("Heat-2D", (40, 50), 6), ("Box-3D27P", (12, 13, 14), 3)])
def test_round16_oracle_equals_numpy_iteration(name, dims, steps):
    # round16 semantics of the device path: binary16 RNE operands, exact sum, fp32 storage
    g = oracle.random_grid(dims, seed=12)
    cur = g
    for _ in range(steps):
        cur = oracle.direct_apply(name, cur.astype(np.float16).astype(np.float64), 1)
        cur = cur.astype(np.float32).astype(np.float64)
    assert np.array_equal(oracle.direct_apply_mt(name, g, steps, 4, round16=True), cur)


def test_round16_ties_to_even():
    # binary16 RNE at the halfway points (the oracle's rounding is numpy's / the device's)
    vals = np.array([1 + 2.0 ** -11, 1 + 3 * 2.0 ** -11, 0.5 + 2.0 ** -12, 2.0 ** -14 * 1.5,
                     0.99951171875 + 2.0 ** -12], dtype=np.float64)
    g = np.zeros((1, 3 + len(vals) + 2))
    g[0, 3:3 + len(vals)] = vals
    g = np.repeat(g, 3, axis=0)
    got = oracle.direct_apply_mt("Heat-2D", g, 1, 2, round16=True)
    want = oracle.direct_apply("Heat-2D", g.astype(np.float16).astype(np.float64), 1)
    assert np.array_equal(got, want.astype(np.float32).astype(np.float64))


def test_round16_bits_match_numpy():
    # Heat-1D over isolated values: out = 0.5 * round16(v) exactly, so the oracle's
    # bit-level binary16 RNE is checked against numpy's on normals, subnormals,
    # halfway cases and overflow
    rng = np.random.default_rng(0)
    v = (rng.random(30000) * 2.0 ** rng.integers(-26, 17, 30000)).astype(np.float32).astype(np.float64)
    v = np.concatenate([v, [65504.0, 65519.99, 65520.0, 70000.0, 2.0 ** -25, 3 * 2.0 ** -25,
                            1.5 * 2.0 ** -24, 1 + 2.0 ** -11, 1 + 3 * 2.0 ** -11]])
    g = np.zeros(3 * len(v) + 2)
    g[1::3][:len(v)] = v
    out = oracle.direct_apply_mt("Heat-1D", g, 1, 2, round16=True)  # out[i] centred on g[i + 1]
    got = 2.0 * out[0::3][:len(v)]
    want = v.astype(np.float16).astype(np.float64)
    assert np.array_equal(got, want)
