"""Bit-exactness of the host compile step (Adaptive Layout Morphing + Structured
Sparsity Conversion + compress_24) against the reference: the .s24 artifact
(values AND 2:4 metadata), the PIT column map, p / alignment / Blossom flags,
for every preset x (r1, r2) in [1,16]^2 — fixtures from oracle/make_golden.py."""
from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

import oracle
from conftest import GOLDEN
from paper_2506_22969_b200 import Compiled, InvalidArgument

DIGESTS = json.loads((GOLDEN / "s24_digests.json").read_text())


@pytest.mark.parametrize("name", sorted(DIGESTS))
def test_s24_all_layouts(name):
    entry = DIGESTS[name]
    bad = []
    for key, want in entry["layouts"].items():
        r1, r2 = map(int, key.split("x"))
        c = Compiled(name, entry["grid"], r1, r2)
        b = c.s24(0)
        co = c.col_origin()
        got = {"sha256": hashlib.sha256(b).hexdigest(), "len": len(b),
               "col_origin_sha256": hashlib.sha256(co.astype("<u8").tobytes()).hexdigest(),
               "p": c.info["p"], "align_cols": c.info["align_cols"],
               "used_blossom": c.info["used_blossom"], "refined": c.info["refined"],
               "cols": c.info["cols"]}
        c.close()
        if got != want:
            bad.append((key, got, want))
    assert not bad, bad[:3]


@pytest.mark.parametrize("path", sorted((GOLDEN / "s24").glob("*.s24")), ids=lambda p: p.stem)
def test_s24_full_bytes_device_layouts(path):
    name, lay = path.stem.rsplit("_", 1)
    r1, r2 = map(int, lay.split("x"))
    nd = {"Heat-3D": 3, "Box-3D27P": 3}.get(name, 2)
    dims = DIGESTS[name]["grid"]
    assert len(dims) == nd
    c = Compiled(name, dims, r1, r2)
    assert c.s24(1) == path.read_bytes()


def test_s24_layout_grid_size_independent():
    """A'' values and metadata do not depend on the grid extent."""
    a = Compiled("Box-2D9P", [64, 64], 16, 8).s24(0)
    b = Compiled("Box-2D9P", [8192, 8192], 16, 8).s24(0)
    assert a == b


def test_metadata_nibbles_and_pairs():
    """Every A'' pair (2t, 2t+1) holds <= 1 nonzero at the device layouts, the
    nibbles are valid 2:4 selectors."""
    for name in ("Heat-2D", "Box-2D9P", "Star-2D13P", "Box-2D49P", "Heat-3D", "Box-3D27P"):
        nd = 3 if "3D" in name else 2
        c = Compiled(name, [40] * nd, 16, 8)
        a = c.matrix()
        assert a.shape[1] % 4 == 0
        nz = (a != 0).reshape(a.shape[0], -1, 2).sum(axis=2)
        assert nz.max() <= 1, name
        b = c.s24(0)
        m, k = int.from_bytes(b[4:12], "little"), int.from_bytes(b[12:20], "little")
        meta = np.frombuffer(b[24 + 8 * m * k // 2:], dtype=np.uint8)
        assert set(np.unique(meta)) <= {4, 8, 9, 12, 13, 14}


@pytest.mark.skipif(not oracle.ref_available(), reason="reference build not present")
def test_live_against_reference_custom_specs():
    """Spec documents (docs/formats.md) compiled by both sides on random layouts."""
    rng = np.random.default_rng(3)
    specs = [
        "name = a\ndims = 2\nshape = box\nk = 5\n" + "".join(
            f"point = {i} {j} : {w}\n" for (i, j), w in
            {(-2, 0): 0.25, (0, 0): 0.5, (1, 1): 0.125, (2, -2): 0.125}.items()),
        "name = b\ndims = 3\nshape = star\nk = 3\npoint = 0 0 0 : 0.5\npoint = 1 0 0 : 0.25\n"
        "point = 0 0 -1 : 0.25\n",
        "name = c\ndims = 1\nshape = star\nk = 7\npoint = -3 : 0.5\npoint = 2 : 0.5\n",
    ]
    for text in specs:
        nd = int(text.split("dims = ")[1][0])
        dims = [33] * nd
        for _ in range(12):
            r1 = int(rng.integers(1, 17))
            r2 = 1 if nd == 1 else int(rng.integers(1, 17))
            want, info, co = oracle.ref_compile(text, dims, r1, r2)
            c = Compiled(text, dims, r1, r2)
            assert c.s24(0) == want
            assert np.array_equal(c.col_origin(), co)
            assert c.info["p"] == info["p"] and c.info["used_blossom"] == info["used_blossom"]


def test_compile_errors_mirror_reference_types():
    with pytest.raises(InvalidArgument):
        Compiled("NoSuchPreset", [64, 64], 16, 8)
    with pytest.raises(InvalidArgument):
        Compiled("Box-2D9P", [64, 64, 64], 16, 8)
    with pytest.raises(InvalidArgument):
        Compiled("Box-2D9P", [2, 64], 16, 8)  # grid smaller than kernel
    with pytest.raises(InvalidArgument):
        Compiled("Box-2D9P", [64, 64], 17, 8)  # merge factor above the fragment bound
    with pytest.raises(InvalidArgument):
        Compiled("name = x\ndims = 2\nshape = star\nk = 3\npoint = 1 1 : 1\n", [9, 9], 2, 2)


def test_explorer_default_is_tcgen05_legal():
    c = Compiled("Box-2D9P", [8192, 8192])
    assert (c.info["r1"], c.info["r2"]) == (16, 8)
    assert c.info["m_prime"] == 128
