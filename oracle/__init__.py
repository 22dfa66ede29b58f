"""TEST INFRASTRUCTURE ONLY — the parity checker, never the product.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this package. It wraps
  * oracle/liboracle.so             — plain-C restatement of the reference CPU
                                      sweep (oracle.c), pinned to the reference
                                      by tests/golden/direct_apply.npz;
  * oracle/_ref/libstensor_ref.so   — the unmodified reference core compiled
                                      from /root/reference by oracle/Makefile
                                      (present wherever it was built; it travels
                                      to the GPU box with the repo snapshot).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libstensor_ref.so"
REF_SRC = Path("/root/reference/proj")

_orc = None
_ref = None


def build(force: bool = False) -> None:
    """Build liboracle.so, and the reference .so when the sources are present."""
    targets = ["all"]
    if REF_SRC.exists():
        targets.append("ref")
    if force:
        subprocess.run(["make", "-C", str(HERE), "clean"], check=True, capture_output=True)
    subprocess.run(["make", "-C", str(HERE), *targets], check=True, capture_output=True)


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not ORACLE_SO.exists():
            build()
        L = C.CDLL(str(ORACLE_SO))
        P, u64, i32 = C.c_void_p, C.c_uint64, C.c_int
        L.or_random_grid.argtypes = [i32, P, u64, P]
        L.or_random_grid_f32.argtypes = [i32, P, u64, P]
        L.or_preset.argtypes = [C.c_char_p, P, P, P, P]
        L.or_preset.restype = i32
        L.or_direct_apply.argtypes = [i32, P, i32, i32, P, P, P, u64, P]
        L.or_direct_apply.restype = i32
        L.or_direct_apply_mt.argtypes = [i32, P, i32, i32, P, P, P, u64, P, i32, i32]
        L.or_direct_apply_mt.restype = i32
        _orc = L
    return _orc


def ref_available() -> bool:
    return REF_SO.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref)")
        L = C.CDLL(str(REF_SO))
        P, u64, i32, sz = C.c_void_p, C.c_uint64, C.c_int, C.c_size_t
        L.ref_last_error.restype = C.c_char_p
        L.ref_random_grid.argtypes = [i32, P, u64, P]
        L.ref_direct_apply.argtypes = [C.c_char_p, i32, P, P, u64, P]
        L.ref_direct_apply_slabs.argtypes = [C.c_char_p, i32, P, P, P, i32]
        L.ref_compile.argtypes = [C.c_char_p, i32, P, i32, i32, i32, C.c_uint32, P, sz,
                                  C.POINTER(sz), P, P, sz]
        L.ref_hier_match.argtypes = [u64, u64, i32, P, sz, C.POINTER(sz), C.POINTER(u64),
                                     C.POINTER(C.c_int)]
        L.ref_estimate.argtypes = [C.c_char_p, i32, P, i32, i32, i32, P, C.POINTER(u64)]
        L.ref_estimate_hw_text.argtypes = [C.c_char_p, i32, P, i32, i32, i32, P, C.POINTER(u64)]
        _ref = L
    return _ref


def _dims(dims):
    return np.ascontiguousarray(dims, dtype=np.uint64)


def random_grid(dims, seed: int = 1, dtype=np.float64) -> np.ndarray:
    d = _dims(dims)
    out = np.empty(tuple(int(x) for x in dims), dtype=dtype)
    fn = orc().or_random_grid if dtype == np.float64 else orc().or_random_grid_f32
    fn(len(d), d.ctypes.data, seed, out.ctypes.data)
    return out


def preset(name: str):
    offs = np.zeros((64, 3), dtype=np.int32)
    w = np.zeros(64, dtype=np.float64)
    dims = C.c_int()
    k = C.c_int()
    n = orc().or_preset(name.encode(), C.byref(dims), C.byref(k), offs.ctypes.data, w.ctypes.data)
    if n < 0:
        raise ValueError(f"unknown preset {name}")
    return dims.value, k.value, offs[:n].copy(), w[:n].copy()


def direct_apply(name: str, grid: np.ndarray, steps: int) -> np.ndarray:
    """C restatement of stensor::direct_apply (valid region, fp64)."""
    ndims, k, offs, w = preset(name)
    g = np.ascontiguousarray(grid, dtype=np.float64)
    if g.ndim != ndims:
        raise ValueError("grid dimensionality does not match stencil")
    shape = tuple(n - steps * (k - 1) for n in g.shape)
    if steps < 1 or any(s < 1 for s in shape):
        raise ValueError("grid smaller than kernel")
    out = np.empty(shape, dtype=np.float64)
    d = _dims(g.shape)
    offs = np.ascontiguousarray(offs)
    rc = orc().or_direct_apply(ndims, d.ctypes.data, k, len(w), offs.ctypes.data, w.ctypes.data,
                               g.ctypes.data, steps, out.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"or_direct_apply failed ({rc})")
    return out


def direct_apply_mt(name: str, grid: np.ndarray, steps: int, threads: int | None = None,
                    round16: bool = False) -> np.ndarray:
    """direct_apply with its output rows split over host threads (bitwise equal to
    direct_apply). round16=True: the device path's SST_PREC_F16 semantics — every
    step rounds its inputs to binary16 (RNE), sums exactly (fp64) and stores fp32."""
    ndims, k, offs, w = preset(name)
    g = np.ascontiguousarray(grid, dtype=np.float64)
    if g.ndim != ndims:
        raise ValueError("grid dimensionality does not match stencil")
    shape = tuple(n - steps * (k - 1) for n in g.shape)
    if steps < 1 or any(s < 1 for s in shape):
        raise ValueError("grid smaller than kernel")
    out = np.empty(shape, dtype=np.float64)
    d = _dims(g.shape)
    offs = np.ascontiguousarray(offs)
    nt = int(threads or os.cpu_count() or 1)
    rc = orc().or_direct_apply_mt(ndims, d.ctypes.data, k, len(w), offs.ctypes.data, w.ctypes.data,
                                  g.ctypes.data, steps, out.ctypes.data, nt, 1 if round16 else 0)
    if rc != 0:
        raise RuntimeError(f"or_direct_apply_mt failed ({rc})")
    return out


def ref_direct_apply(name: str, grid: np.ndarray, steps: int) -> np.ndarray:
    """The reference's own direct_apply (oracle/_ref)."""
    ndims, k, _, _ = preset(name) if name in PRESETS else (grid.ndim, None, None, None)
    g = np.ascontiguousarray(grid, dtype=np.float64)
    kk = k if k is not None else 3
    shape = tuple(n - steps * (kk - 1) for n in g.shape)
    out = np.empty(shape, dtype=np.float64)
    d = _dims(g.shape)
    if ref().ref_direct_apply(name.encode(), g.ndim, d.ctypes.data, g.ctypes.data, steps,
                              out.ctypes.data) != 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return out


def ref_direct_apply_slabs(name: str, grid: np.ndarray, nthreads: int) -> np.ndarray:
    _, k, _, _ = preset(name)
    g = np.ascontiguousarray(grid, dtype=np.float64)
    out = np.empty(tuple(n - (k - 1) for n in g.shape), dtype=np.float64)
    d = _dims(g.shape)
    if ref().ref_direct_apply_slabs(name.encode(), g.ndim, d.ctypes.data, g.ctypes.data,
                                    out.ctypes.data, nthreads) != 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return out


def ref_compile(name: str, dims, r1: int = 0, r2: int = 0, r_max: int = 16, tag: int = 0):
    """(.s24 bytes, info dict, col_origin) from the reference compile chain."""
    d = _dims(dims)
    n = C.c_size_t()
    info = np.zeros(8, dtype=np.uint64)
    L = ref()
    if L.ref_compile(name.encode(), len(d), d.ctypes.data, r1, r2, r_max, tag, None, 0,
                     C.byref(n), info.ctypes.data, None, 0) != 0:
        raise RuntimeError(L.ref_last_error().decode())
    buf = np.empty(n.value, dtype=np.uint8)
    co = np.empty(int(info[4]), dtype=np.uint64)
    if L.ref_compile(name.encode(), len(d), d.ctypes.data, r1, r2, r_max, tag, buf.ctypes.data,
                     n.value, C.byref(n), info.ctypes.data, co.ctypes.data, len(co)) != 0:
        raise RuntimeError(L.ref_last_error().decode())
    keys = ["p", "align_cols", "used_blossom", "refined", "cols", "k_prime", "r1", "r2"]
    return buf.tobytes(), {k: int(v) for k, v in zip(keys, info)}, co


PRESETS = ["Heat-1D", "1D5P", "Heat-2D", "Box-2D9P", "Star-2D13P", "Box-2D49P", "Heat-3D",
           "Box-3D27P"]
