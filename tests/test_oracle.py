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
