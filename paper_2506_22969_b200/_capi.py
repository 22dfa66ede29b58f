"""ctypes binding of include/sparstencil.h (the engine's C ABI).

This is exactly the stub a reference-side Python user would add (see
INTEGRATION.md). The library is built in-tree by paper_2506_22969_b200/build.py;
if it is missing we raise — there is no CPU fallback path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / (
    "libsparstencil_ablation.so" if os.environ.get("SST_LIB") == "ablation" else "libsparstencil.so")

SST_OK = 0
SST_PREC_F16 = 1
SST_PREC_F16X2 = 2

# every symbol include/sparstencil.h declares (checked by tests/test_capi.py)
EXPORTED = [
    "sst_compile", "sst_compiled_destroy", "sst_compiled_info", "sst_compiled_s24",
    "sst_compiled_perm", "sst_compiled_col_origin", "sst_compiled_matrix",
    "sst_compiled_plan_desc", "sst_plan_create", "sst_plan_destroy", "sst_plan_storage",
    "sst_plan_stats_get", "sst_plan_bind", "sst_upload", "sst_download", "sst_run_steps",
    "sst_set_row_window", "sst_set_row_windows", "sst_plan_set_trace", "sst_apply_host", "sst_random_grid", "sst_last_error",
    "sst_device_count", "sst_version", "sst_run_compile", "sst_compile_result_destroy",
    "sst_compile_result_summary", "sst_compile_result_report", "sst_compile_result_lut", "sst_explore",
    "sst_plan_set_peer", "sst_plan_buffers", "sst_device_alloc", "sst_device_free", "sst_ipc_handle",
    "sst_ipc_open", "sst_ipc_close", "sst_stream_write_u32", "sst_stream_wait_geq_u32",
    "sst_run_steps_peer", "sst_download_slices", "sst_multi_create", "sst_multi_destroy", "sst_multi_upload",
    "sst_multi_run", "sst_multi_sync", "sst_multi_download", "sst_multi_slab", "sst_run_steps_multi",
    "sst_estimate_device", "sst_run_steps_batch", "sst_plan_buffers_h", "sst_plan_set_peer_h", "sst_launch_count",
]


class SparStencilError(RuntimeError):
    """Base class; subclasses mirror the reference's exception types."""


class InvalidArgument(SparStencilError, ValueError):
    pass  # std::invalid_argument


class LogicError(SparStencilError):
    pass  # std::logic_error


class OutOfRange(SparStencilError, IndexError):
    pass  # std::out_of_range


class CudaFailure(SparStencilError):
    pass


class NoDevice(CudaFailure):
    pass


_STATUS_EXC = {1: InvalidArgument, 2: LogicError, 3: OutOfRange, 4: SparStencilError,
               5: CudaFailure, 6: NoDevice}


class CompileInfo(C.Structure):
    _fields_ = [("dims", C.c_int32), ("k", C.c_int32), ("r1", C.c_int32), ("r2", C.c_int32),
                ("m_prime", C.c_uint64), ("k_prime", C.c_uint64), ("n_prime", C.c_uint64),
                ("cols", C.c_uint64), ("p", C.c_uint64), ("align_cols", C.c_uint64),
                ("used_blossom", C.c_int32), ("refined", C.c_int32),
                ("window_w", C.c_uint64), ("window_h", C.c_uint64), ("window_d", C.c_uint64),
                ("grid_dims", C.c_uint64 * 3), ("fold_n", C.c_uint64), ("fold_w", C.c_uint64)]


class PlanDesc(C.Structure):
    _fields_ = [("dims", C.c_int32), ("k", C.c_int32), ("r1", C.c_int32), ("r2", C.c_int32),
                ("grid_dims", C.c_uint64 * 3), ("rows", C.c_uint64), ("cols", C.c_uint64),
                ("a_values", C.POINTER(C.c_double)), ("a_meta", C.POINTER(C.c_uint8)),
                ("col_origin", C.POINTER(C.c_uint64)),
                ("window_w", C.c_uint64), ("window_h", C.c_uint64), ("window_d", C.c_uint64),
                ("precision", C.c_int32), ("fuse", C.c_uint32), ("fold_n", C.c_uint64),
                ("fold_w", C.c_uint64)]


class Storage(C.Structure):
    _fields_ = [("row_pitch", C.c_uint64), ("plane_pitch", C.c_uint64),
                ("left_pad", C.c_uint64), ("bytes", C.c_uint64)]


class PlanStats(C.Structure):
    _fields_ = [("k_pad", C.c_int32), ("k_steps", C.c_int32), ("tiles_x", C.c_int32),
                ("tiles_y", C.c_int32), ("patch_w", C.c_int32), ("patch_h", C.c_int32),
                ("patch_planes", C.c_int32), ("worst_bank_conflict", C.c_int32),
                ("patch_stages", C.c_int32),
                ("smem_bytes", C.c_int32), ("ctas", C.c_int32), ("batches", C.c_int32),
                ("launches", C.c_uint64), ("h16_launches", C.c_uint64), ("h16_capable", C.c_int32),
                ("h16_patch_stages", C.c_int32)]


class CompileRequest(C.Structure):
    _fields_ = [("stencil", C.c_char_p), ("grid_dims", C.POINTER(C.c_uint64)), ("ndims", C.c_int32),
                ("hw", C.c_char_p), ("r1", C.c_int32), ("r2", C.c_int32), ("r_max", C.c_int32),
                ("fuse", C.c_uint64), ("precision", C.c_int32), ("seed", C.c_uint64),
                ("out_dir", C.c_char_p), ("verify", C.c_int32), ("device", C.c_int32),
                ("corrupt_permutation", C.c_int32)]


class CompileSummary(C.Structure):
    _fields_ = [("ok", C.c_int32), ("r1", C.c_int32), ("r2", C.c_int32), ("used_blossom", C.c_int32),
                ("p", C.c_uint64), ("align_cols", C.c_uint64), ("n_mma", C.c_uint64),
                ("issued_mma", C.c_uint64), ("m_prime", C.c_uint64), ("k_prime", C.c_uint64),
                ("n_prime", C.c_uint64), ("t_compute", C.c_double), ("t_memory", C.c_double),
                ("t_total", C.c_double), ("model_gstencil", C.c_double), ("max_abs_err", C.c_double),
                ("max_rel_err", C.c_double), ("verify_seconds", C.c_double), ("status", C.c_char * 32)]


_lib = None


def lib() -> C.CDLL:
    """Load libsparstencil.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2506_22969_b200.build` "
                          "(no CPU fallback exists)")
    L = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    P, u64, i32, sz = C.c_void_p, C.c_uint64, C.c_int, C.c_size_t
    sig = {
        "sst_compile": (i32, [C.c_char_p, C.POINTER(u64), i32, i32, i32, u64, C.POINTER(P)]),
        "sst_compiled_destroy": (None, [P]),
        "sst_compiled_info": (i32, [P, C.POINTER(CompileInfo)]),
        "sst_compiled_s24": (i32, [P, C.c_uint32, P, sz, C.POINTER(sz)]),
        "sst_compiled_perm": (i32, [P, P, sz, C.POINTER(sz)]),
        "sst_compiled_col_origin": (i32, [P, P, sz, C.POINTER(sz)]),
        "sst_compiled_matrix": (i32, [P, P, sz, C.POINTER(sz)]),
        "sst_compiled_plan_desc": (i32, [P, C.POINTER(PlanDesc)]),
        "sst_plan_create": (i32, [C.POINTER(PlanDesc), i32, C.POINTER(P)]),
        "sst_plan_destroy": (None, [P]),
        "sst_plan_storage": (i32, [P, C.POINTER(Storage)]),
        "sst_plan_stats_get": (i32, [P, C.POINTER(PlanStats)]),
        "sst_plan_bind": (i32, [P, P, P]),
        "sst_upload": (i32, [P, i32, P, i32, P]),
        "sst_download": (i32, [P, i32, P, i32, P]),
        "sst_run_steps": (i32, [P, i32, u64, P, C.POINTER(i32)]),
        "sst_set_row_window": (i32, [P, u64, u64]),
        "sst_set_row_windows": (i32, [P, u64, u64, u64, u64]),
        "sst_plan_set_trace": (i32, [P, P]),
        "sst_apply_host": (i32, [P, P, P, u64]),
        "sst_random_grid": (i32, [i32, C.POINTER(u64), u64, P]),
        "sst_last_error": (C.c_char_p, []),
        "sst_device_count": (i32, []),
        "sst_launch_count": (C.c_ulonglong, []),
        "sst_version": (C.c_char_p, []),
        "sst_run_compile": (i32, [C.POINTER(CompileRequest), C.POINTER(P)]),
        "sst_compile_result_destroy": (None, [P]),
        "sst_compile_result_summary": (i32, [P, C.POINTER(CompileSummary)]),
        "sst_compile_result_report": (i32, [P, P, sz, C.POINTER(sz)]),
        "sst_compile_result_lut": (i32, [P, P, sz, C.POINTER(sz)]),
        "sst_explore": (i32, [C.c_char_p, C.POINTER(u64), i32, C.c_char_p, u64, i32, P, sz, C.POINTER(sz)]),
        "sst_estimate_device": (i32, [C.c_char_p, C.POINTER(u64), i32, u64, i32, i32, P]),
        "sst_run_steps_batch": (i32, [C.POINTER(P), i32, C.POINTER(i32), u64, P, C.POINTER(i32)]),
        "sst_plan_set_peer": (i32, [P, i32, P, P, u64]),
        "sst_plan_buffers": (i32, [P, C.POINTER(P), C.POINTER(P)]),
        "sst_plan_buffers_h": (i32, [P, C.POINTER(P), C.POINTER(P)]),
        "sst_plan_set_peer_h": (i32, [P, i32, P, P]),
        "sst_device_alloc": (i32, [i32, sz, C.POINTER(P)]),
        "sst_device_free": (i32, [P]),
        "sst_ipc_handle": (i32, [P, C.POINTER(C.c_uint8)]),
        "sst_ipc_open": (i32, [i32, C.POINTER(C.c_uint8), C.POINTER(P)]),
        "sst_ipc_close": (i32, [P]),
        "sst_stream_write_u32": (i32, [P, P, C.c_uint32]),
        "sst_stream_wait_geq_u32": (i32, [P, P, C.c_uint32]),
        "sst_run_steps_peer": (i32, [P, i32, u64, P, P, P, P, C.c_uint32, C.POINTER(i32)]),
        "sst_download_slices": (i32, [P, i32, u64, u64, P, i32, P]),
        "sst_multi_create": (i32, [C.POINTER(PlanDesc), i32, C.POINTER(i32), C.POINTER(P)]),
        "sst_multi_destroy": (None, [P]),
        "sst_multi_upload": (i32, [P, P, i32]),
        "sst_multi_run": (i32, [P, u64]),
        "sst_multi_sync": (i32, [P]),
        "sst_multi_download": (i32, [P, P, i32]),
        "sst_multi_slab": (i32, [P, i32, C.POINTER(P), C.POINTER(P), C.POINTER(u64)]),
        "sst_run_steps_multi": (i32, [C.POINTER(PlanDesc), i32, C.POINTER(i32), P, P, u64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(status: int) -> None:
    if status != SST_OK:
        msg = lib().sst_last_error().decode(errors="replace")
        raise _STATUS_EXC.get(status, SparStencilError)(msg)
