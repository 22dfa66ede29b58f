"""Python host mirror of the reference's stencil API over the engine's C ABI.

Reference call (proj/core/include/stensor/stencil.hpp:72):
    Grid direct_apply(const StencilSpec&, const Grid&, uint64_t steps)
Engine call (same argument meaning, same valid-region result, same error types):
    sparse_apply(stencil, grid, steps) -> np.ndarray

`stencil` is a preset name (stencil.cpp:135-159) or a spec document
(docs/formats.md:3-30). The compile step (flatten -> crush -> convert_layout ->
compress_24) runs in the C++ host library; every time step runs on the B200
through tcgen05.mma.sp. There is no CPU execution path.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _capi
from ._capi import check, lib

PRESETS = ["Heat-1D", "1D5P", "Heat-2D", "Box-2D9P", "Star-2D13P", "Box-2D49P", "Heat-3D",
           "Box-3D27P"]


PRECISIONS = {"f16": _capi.SST_PREC_F16, "f16x2": _capi.SST_PREC_F16X2}


def preset_names() -> list[str]:
    return list(PRESETS)


class Compiled:
    """Host compile products (reference: flatten/crush/convert_layout/compress_24)."""

    def __init__(self, stencil: str, grid_dims: Sequence[int], r1: int = 0, r2: int = 0,
                 fuse: int = 1):
        L = lib()
        self.grid_dims = [int(d) for d in grid_dims]
        dims = (C.c_uint64 * len(self.grid_dims))(*self.grid_dims)
        h = C.c_void_p()
        check(L.sst_compile(stencil.encode(), dims, len(self.grid_dims), int(r1), int(r2),
                            int(fuse), C.byref(h)))
        self._h = h
        info = _capi.CompileInfo()
        check(L.sst_compiled_info(self._h, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in _capi.CompileInfo._fields_ if f != "grid_dims"}
        self.stencil = stencil

    def _fetch(self, fn, ctype, dtype):
        n = C.c_size_t()
        check(fn(self._h, None, 0, C.byref(n)))
        out = np.empty(n.value, dtype=dtype)
        check(fn(self._h, out.ctypes.data_as(C.c_void_p), n.value, C.byref(n)))
        return out

    def s24(self, tag: int = 0) -> bytes:
        L = lib()
        n = C.c_size_t()
        check(L.sst_compiled_s24(self._h, tag, None, 0, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        check(L.sst_compiled_s24(self._h, tag, buf, n.value, C.byref(n)))
        return bytes(buf)

    def perm(self) -> np.ndarray:
        return self._fetch(lib().sst_compiled_perm, C.c_uint64, np.uint64)

    def col_origin(self) -> np.ndarray:
        return self._fetch(lib().sst_compiled_col_origin, C.c_uint64, np.uint64)

    def matrix(self) -> np.ndarray:
        a = self._fetch(lib().sst_compiled_matrix, C.c_double, np.float64)
        return a.reshape(int(self.info["m_prime"]), int(self.info["cols"]))

    def plan_desc(self) -> _capi.PlanDesc:
        d = _capi.PlanDesc()
        check(lib().sst_compiled_plan_desc(self._h, C.byref(d)))
        return d

    def close(self):
        if getattr(self, "_h", None):
            lib().sst_compiled_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SparseStencil:
    """A compiled stencil resident on one B200 (the device-side KernelPlan)."""

    def __init__(self, stencil: str | Compiled, grid_dims: Optional[Sequence[int]] = None,
                 device: int = 0, r1: int = 16, r2: int = 8, fuse: int = 1, precision: str = "f16"):
        """precision: "f16" (B'' rounded to binary16, the reference's round16 operand
        semantics) or "f16x2" (B'' split into hi + lo binary16 terms: ~fp32 steps)."""
        if precision not in PRECISIONS:
            raise _capi.InvalidArgument(f"precision must be one of {sorted(PRECISIONS)}")
        self.compiled = stencil if isinstance(stencil, Compiled) else Compiled(
            stencil, grid_dims, r1, r2, fuse)
        self.grid_dims = self.compiled.grid_dims
        desc = self.compiled.plan_desc()
        # the fusion factor the operator was compiled with (a pre-compiled Compiled
        # carries its own; the plan advances that many time steps per launch)
        self.fuse = max(1, int(desc.fuse))
        self.k = int(self.compiled.info["k"])       # of the (possibly fused) operator
        self.r = (self.k - 1) // 2 // self.fuse     # radius of one original time step
        desc.precision = PRECISIONS[precision]
        self.precision = precision
        h = C.c_void_p()
        check(lib().sst_plan_create(C.byref(desc), int(device), C.byref(h)))
        self._h = h
        self.device = device
        st = _capi.Storage()
        check(lib().sst_plan_storage(self._h, C.byref(st)))
        self.storage = {f: getattr(st, f) for f, _ in _capi.Storage._fields_}
        self._bufs = None  # keeps caller-provided buffers alive

    # -- buffers -----------------------------------------------------------
    def bind(self, buf0: int = 0, buf1: int = 0, keepalive=None):
        """Bind two device buffers (raw pointers) or let the plan allocate (0, 0)."""
        check(lib().sst_plan_bind(self._h, C.c_void_p(buf0 or None), C.c_void_p(buf1 or None)))
        self._bufs = keepalive

    def bind_torch(self):
        """Allocate the ping-pong pair with torch (device memory plumbing only)."""
        import torch
        nbytes = int(self.storage["bytes"])
        dev = torch.device("cuda", self.device)
        bufs = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(2)]
        self.bind(bufs[0].data_ptr(), bufs[1].data_ptr(), keepalive=bufs)
        return bufs

    def upload(self, grid, which: int = 0, stream: int = 0):
        """Dense fp32 grid (numpy host array or torch CUDA tensor) -> buffer `which`."""
        on_dev, ptr, keep = _pointer(grid)
        check(lib().sst_upload(self._h, which, C.c_void_p(ptr), int(on_dev), C.c_void_p(stream or None)))
        return keep

    def download(self, which: int, out=None, stream: int = 0):
        if out is None:
            out = np.empty(self.grid_dims, dtype=np.float32)
        on_dev, ptr, _ = _pointer(out)
        check(lib().sst_download(self._h, which, C.c_void_p(ptr), int(on_dev), C.c_void_p(stream or None)))
        return out

    def run(self, steps: int, src: int = 0, stream: int = 0) -> int:
        dst = C.c_int()
        check(lib().sst_run_steps(self._h, src, int(steps), C.c_void_p(stream or None), C.byref(dst)))
        return dst.value

    def set_row_window(self, y0: int, y1: int):
        check(lib().sst_set_row_window(self._h, int(y0), int(y1)))

    def set_row_windows(self, y0: int, y1: int, y2: int, y3: int):
        """Two row windows [y0, y1) and [y2, y3) in one launch (2D)."""
        check(lib().sst_set_row_windows(self._h, int(y0), int(y1), int(y2), int(y3)))

    def apply_host(self, grid: np.ndarray, steps: int, out: Optional[np.ndarray] = None) -> np.ndarray:
        """Host buffers in, full-size host buffer out (H2D + steps + D2H). Pass
        page-locked arrays (e.g. views of pinned torch tensors) for full PCIe speed."""
        g = np.ascontiguousarray(grid, dtype=np.float32)
        if list(g.shape) != list(self.grid_dims):
            raise _capi.InvalidArgument("grid shape does not match the compiled grid")
        if out is None:
            out = np.empty_like(g)
        elif out.shape != g.shape or out.dtype != np.float32 or not out.flags["C_CONTIGUOUS"]:
            raise _capi.InvalidArgument("out must be a C-contiguous float32 array of the grid shape")
        check(lib().sst_apply_host(self._h, g.ctypes.data_as(C.c_void_p),
                                   out.ctypes.data_as(C.c_void_p), int(steps)))
        return out

    def stats(self) -> dict:
        s = _capi.PlanStats()
        check(lib().sst_plan_stats_get(self._h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in _capi.PlanStats._fields_}

    def close(self):
        if getattr(self, "_h", None):
            lib().sst_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MultiSlabStencil:
    """A compiled stencil slab-decomposed over several slabs in one process
    (sst_multi_*): slab i on device devices[i] (several may share a GPU), halos
    fused into each slab's epilogue (P2P stores), neighbours ordered by stream flags."""

    def __init__(self, stencil: str, grid_dims: Sequence[int], devices: Sequence[int], fuse: int = 1,
                 precision: str = "f16"):
        if precision not in PRECISIONS:
            raise _capi.InvalidArgument(f"precision must be one of {sorted(PRECISIONS)}")
        self.compiled = Compiled(stencil, grid_dims, 16, 8, fuse)
        self.grid_dims = self.compiled.grid_dims
        desc = self.compiled.plan_desc()
        desc.precision = PRECISIONS[precision]
        self.fuse = max(1, int(desc.fuse))
        self.r = (int(self.compiled.info["k"]) - 1) // 2 // self.fuse
        self.devices = [int(d) for d in devices]
        devs = (C.c_int * len(self.devices))(*self.devices)
        h = C.c_void_p()
        check(lib().sst_multi_create(C.byref(desc), len(self.devices), devs, C.byref(h)))
        self._h = h

    def slab(self, i: int) -> dict:
        plan, stream = C.c_void_p(), C.c_void_p()
        owned = (C.c_uint64 * 2)()
        check(lib().sst_multi_slab(self._h, int(i), C.byref(plan), C.byref(stream), owned))
        s = _capi.PlanStats()
        check(lib().sst_plan_stats_get(plan, C.byref(s)))
        return {"owned": (owned[0], owned[1]), "stream": stream.value, "plan": plan.value,
                "launches": int(s.launches), "h16_launches": int(s.h16_launches)}

    def upload(self, grid):
        on_dev, ptr, keep = _pointer(grid)
        check(lib().sst_multi_upload(self._h, C.c_void_p(ptr), int(on_dev)))
        return keep

    def run(self, steps: int):
        check(lib().sst_multi_run(self._h, int(steps)))

    def sync(self):
        check(lib().sst_multi_sync(self._h))

    def download(self, out=None):
        if out is None:
            out = np.empty(self.grid_dims, dtype=np.float32)
        on_dev, ptr, _ = _pointer(out)
        check(lib().sst_multi_download(self._h, C.c_void_p(ptr), int(on_dev)))
        return out

    def apply_host(self, grid: np.ndarray, steps: int) -> np.ndarray:
        self.upload(np.ascontiguousarray(grid, dtype=np.float32))
        self.run(steps)
        return self.download()

    def close(self):
        if getattr(self, "_h", None):
            lib().sst_multi_destroy(self._h)
            self._h = None
        if getattr(self, "compiled", None) is not None:
            self.compiled.close()
            self.compiled = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_steps_multi(stencil: str, grid: np.ndarray, steps: int, devices: Sequence[int],
                    precision: str = "f16") -> np.ndarray:
    """sst_run_steps_multi: one call, full-size result (like SparseStencil.apply_host)."""
    g = np.ascontiguousarray(grid, dtype=np.float32)
    comp = Compiled(stencil, list(g.shape), 16, 8, 1)
    try:
        desc = comp.plan_desc()
        desc.precision = PRECISIONS[precision]
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        out = np.empty_like(g)
        check(lib().sst_run_steps_multi(C.byref(desc), len(devices), devs, g.ctypes.data_as(C.c_void_p),
                                        out.ctypes.data_as(C.c_void_p), int(steps)))
        return out
    finally:
        comp.close()


def _pointer(arr):
    """(on_device, address, keepalive) for numpy arrays and torch tensors."""
    if isinstance(arr, np.ndarray):
        if arr.dtype != np.float32 or not arr.flags["C_CONTIGUOUS"]:
            raise _capi.InvalidArgument("expected a C-contiguous float32 array")
        return False, arr.ctypes.data, arr
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(arr, torch.Tensor):
        if arr.dtype != torch.float32 or not arr.is_contiguous():
            raise _capi.InvalidArgument("expected a contiguous float32 tensor")
        return arr.is_cuda, arr.data_ptr(), arr
    raise _capi.InvalidArgument(f"unsupported buffer type {type(arr)!r}")


def valid_core(full: np.ndarray, steps: int, r: int) -> np.ndarray:
    """Crop a fixed-size result to the reference's valid region after `steps`."""
    c = steps * r
    sl = tuple(slice(c, n - c) for n in full.shape)
    return full[sl]


def sparse_apply(stencil: str, grid: np.ndarray, steps: int, device: int = 0,
                 fuse: int = 1, precision: str = "f16") -> np.ndarray:
    """Drop-in for stensor::direct_apply (stencil.hpp:72): valid-region result
    (extent N - steps*(k-1) per axis) computed on the B200. `fuse` > 1 applies
    the reference's temporal fusion (fuse_time_steps, stencil.cpp:272-347): one
    launch advances `fuse` time steps (used when it divides `steps`)."""
    if steps < 1:
        raise _capi.InvalidArgument("steps must be >= 1")
    g = np.asarray(grid)
    f = fuse if fuse > 1 and steps % fuse == 0 else 1
    eng = SparseStencil(stencil, list(g.shape), device=device, fuse=f, precision=precision)
    try:
        k1 = 2 * eng.r + 1
        for n in g.shape:
            if n < k1 + (steps - 1) * (k1 - 1):
                raise _capi.InvalidArgument("grid smaller than kernel")
        full = eng.apply_host(g.astype(np.float32), steps)
        return valid_core(full, steps, eng.r).astype(np.float64)
    finally:
        eng.close()


def run_compile(stencil: str, grid_dims: Sequence[int], hw: str = "a100-sparse", r1: int = 0, r2: int = 0,
                r_max: int = 16, fuse: int = 1, precision: str = "exact64", seed: int = 1,
                out_dir: Optional[str] = None, verify: bool = True, device: int = 0,
                corrupt_permutation: bool = False) -> dict:
    """Mirror of stensor::run_compile (pipeline.hpp:14-46). Returns the summary,
    the report.json text and the lut.bin bytes; writes report.json / a2.s24 /
    lut.bin to `out_dir` when given. The desk-scale verification (<= 256 per
    axis) runs on the GPU (`verify=False` skips it: status "unverified-skipped")."""
    if precision not in ("exact64", "round16"):
        raise _capi.InvalidArgument("precision must be exact64 or round16")
    L = lib()
    dims = (C.c_uint64 * len(grid_dims))(*[int(d) for d in grid_dims])
    q = _capi.CompileRequest(stencil.encode(), dims, len(grid_dims), hw.encode() if hw else None, int(r1),
                             int(r2), int(r_max), int(fuse), 1 if precision == "round16" else 0, int(seed),
                             out_dir.encode() if out_dir else None, 1 if verify else 0, int(device),
                             1 if corrupt_permutation else 0)
    h = C.c_void_p()
    check(L.sst_run_compile(C.byref(q), C.byref(h)))
    try:
        sm = _capi.CompileSummary()
        check(L.sst_compile_result_summary(h, C.byref(sm)))
        out = {f: getattr(sm, f) for f, _ in _capi.CompileSummary._fields_}
        out["status"] = sm.status.decode()
        out["ok"] = bool(sm.ok)
        n = C.c_size_t()
        check(L.sst_compile_result_report(h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(L.sst_compile_result_report(h, buf, n.value, C.byref(n)))
        out["report"] = buf.raw[:n.value].decode()
        check(L.sst_compile_result_lut(h, None, 0, C.byref(n)))
        lb = (C.c_uint8 * n.value)()
        check(L.sst_compile_result_lut(h, lb, n.value, C.byref(n)))
        out["lut"] = bytes(lb)
        return out
    finally:
        L.sst_compile_result_destroy(h)


def explore(stencil: str, grid_dims: Sequence[int], hw: str = "a100-sparse", fuse: int = 1,
            r_max: int = 16) -> list[dict]:
    """Mirror of stensor::explore_layouts (perf.hpp:45-51): ranked (r1, r2) candidates."""
    L = lib()
    dims = (C.c_uint64 * len(grid_dims))(*[int(d) for d in grid_dims])
    n = C.c_size_t()
    check(L.sst_explore(stencil.encode(), dims, len(grid_dims), hw.encode(), int(fuse), int(r_max), None, 0,
                        C.byref(n)))
    buf = np.empty(n.value, dtype=np.float64)
    check(L.sst_explore(stencil.encode(), dims, len(grid_dims), hw.encode(), int(fuse), int(r_max),
                        buf.ctypes.data_as(C.c_void_p), n.value, C.byref(n)))
    keys = ["r1", "r2", "t_compute", "t_memory", "t_total", "n_mma", "m_prime", "k_prime", "n_prime"]
    rows = buf.reshape(-1, 9)
    return [{k: (int(v) if k in ("r1", "r2", "n_mma", "m_prime", "k_prime", "n_prime") else float(v))
             for k, v in zip(keys, r)} for r in rows]


def estimate_device(stencil: str, grid_dims: Sequence[int], fuse: int = 1, storage: int = 2,
                    tyb: int = 0) -> dict:
    """The engine's execution model of one launch (stensor::estimate_device,
    hwmodel.hpp): HBM, shared-memory pipe and tensor-pipe times on B200, the binding
    one, and the predicted GStencil/s. storage: 2 binary16 between steps, 4 fp32."""
    L = lib()
    dims = (C.c_uint64 * len(grid_dims))(*[int(d) for d in grid_dims])
    out = (C.c_double * 12)()
    check(L.sst_estimate_device(stencil.encode(), dims, len(grid_dims), int(fuse), int(storage), int(tyb), out))
    keys = ["updates", "batches", "hbm_bytes", "smem_wavefronts", "mma_issues", "t_hbm", "t_smem", "t_mma",
            "t_total", "gstencil", "bound", "k_pad"]
    d = dict(zip(keys, list(out)))
    d["bound"] = ("hbm", "smem", "tensor")[int(d["bound"])]
    return d


def run_batch(engines: Sequence["SparseStencil"], steps: int, srcs: Optional[Sequence[int]] = None,
              stream: int = 0) -> list[int]:
    """sst_run_steps_batch: `steps` time steps of several independent grids (one bound
    SparseStencil each), launches interleaved step by step; returns each result buffer."""
    n = len(engines)
    plans = (C.c_void_p * n)(*[e._h for e in engines])
    src = (C.c_int * n)(*(srcs if srcs is not None else [0] * n))
    dst = (C.c_int * n)()
    check(lib().sst_run_steps_batch(plans, n, src, int(steps), C.c_void_p(stream or None), dst))
    return list(dst)
