"""Regenerate tests/golden/ from the reference itself (oracle/_ref, compiled from
the unmodified /root/reference sources). TEST INFRASTRUCTURE ONLY.

    python oracle/make_golden.py

Writes
  direct_apply.npz   reference direct_apply outputs (all 8 presets, 1-3 steps,
                     ragged desk grids) + the random_grid inputs they came from
  s24_digests.json   sha256 / length / p / align / blossom / refined / cols of the
                     .s24 artifact for every preset x (r1, r2) in [1,16]^2 (1D: r2=1)
                     on the acceptance-gate grids (acceptance_main.cpp:85-90)
  s24/<preset>_r1xr2.s24   full bytes for the device layouts (16,8) and (8,8)
  hier_match.json    hierarchical_match pair traces for m, g <= 6, k <= g
  perf_fixture.json  reference estimate() values (A100 model) for fixed layouts
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
import oracle  # noqa: E402

GOLD = REPO / "tests" / "golden"
ACCEPT_DIMS = {1: [65536], 2: [96, 96], 3: [40, 40, 40]}
DESK_DIMS = {1: [301], 2: [37, 41], 3: [17, 19, 23]}


def main():
    oracle.build()
    assert oracle.ref_available(), "reference not built (make -C oracle ref)"
    GOLD.mkdir(parents=True, exist_ok=True)
    (GOLD / "s24").mkdir(exist_ok=True)

    # -- direct_apply vectors
    arrays = {}
    for name in oracle.PRESETS:
        nd, k, _, _ = oracle.preset(name)
        dims = DESK_DIMS[nd]
        d = np.array(dims, dtype=np.uint64)
        g = np.empty(dims, dtype=np.float64)
        oracle.ref().ref_random_grid(nd, d.ctypes.data, 5, g.ctypes.data)
        arrays[f"{name}/input"] = g
        for steps in (1, 2, 3):
            arrays[f"{name}/steps{steps}"] = oracle.ref_direct_apply(name, g, steps)
    np.savez_compressed(GOLD / "direct_apply.npz", **arrays)

    # -- .s24 digests over all layouts
    dig = {}
    for name in oracle.PRESETS:
        nd, _, _, _ = oracle.preset(name)
        dims = ACCEPT_DIMS[nd]
        entry = {"grid": dims, "layouts": {}}
        for r1 in range(1, 17):
            for r2 in range(1, 17):
                if nd == 1 and r2 != 1:
                    continue
                b, info, co = oracle.ref_compile(name, dims, r1, r2)
                entry["layouts"][f"{r1}x{r2}"] = {
                    "sha256": hashlib.sha256(b).hexdigest(), "len": len(b),
                    "col_origin_sha256": hashlib.sha256(co.astype("<u8").tobytes()).hexdigest(),
                    **{k: info[k] for k in ("p", "align_cols", "used_blossom", "refined", "cols")}}
        dig[name] = entry
        # explorer choice of the reference (a100-sparse, r_max 16) on the BASELINE grids
    (GOLD / "s24_digests.json").write_text(json.dumps(dig, indent=1, sort_keys=True))

    for name in oracle.PRESETS:
        nd, _, _, _ = oracle.preset(name)
        if nd == 1:
            continue
        for r1, r2 in ((16, 8), (8, 8)):
            b, _, _ = oracle.ref_compile(name, ACCEPT_DIMS[nd], r1, r2, tag=1)
            (GOLD / "s24" / f"{name}_{r1}x{r2}.s24").write_bytes(b)

    # -- hierarchical match traces
    hm = {}
    L = oracle.ref()
    import ctypes as C
    for m in range(1, 7):
        for g in range(1, 7):
            for k in range(1, g + 1):
                buf = np.zeros(2 * 64, dtype=np.uint64)
                n = C.c_size_t()
                p = C.c_uint64()
                ref = C.c_int()
                assert L.ref_hier_match(m, g, k, buf.ctypes.data, len(buf), C.byref(n), C.byref(p),
                                        C.byref(ref)) == 0
                hm[f"{m},{g},{k}"] = {"pairs": buf[:2 * n.value].tolist(), "p": p.value,
                                      "refined": ref.value}
    (GOLD / "hier_match.json").write_text(json.dumps(hm, sort_keys=True))

    # -- performance model fixture (reference estimate)
    pf = []
    for hw in ("a100-sparse", "a100-dense"):
        for dims, k, r1, r2 in (([10240, 10240], 3, 2, 2), ([4096, 4096], 3, 1, 2),
                                ([512, 512, 512], 3, 2, 2), ([16384, 16384], 7, 2, 3),
                                ([8192, 8192], 3, 16, 8)):
            d = np.array(dims, dtype=np.uint64)
            out = np.zeros(4)
            nm = C.c_uint64()
            assert L.ref_estimate(hw.encode(), len(dims), d.ctypes.data, k, r1, r2,
                                  out.ctypes.data, C.byref(nm)) == 0
            pf.append({"hw": hw, "grid": dims, "k": k, "r1": r1, "r2": r2,
                       "t_compute": out[0], "t_memory": out[1], "t_total": out[2],
                       "n_prime": int(out[3]), "n_mma": nm.value})
    (GOLD / "perf_fixture.json").write_text(json.dumps(pf, indent=1))
    print("golden fixtures written to", GOLD)


if __name__ == "__main__":
    main()
