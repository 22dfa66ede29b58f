"""B200-native SparStencil engine (arXiv 2506.22969): compiled 2:4-sparse stencil
operators executed with tcgen05.mma.sp on sm_100a, behind the C ABI in
include/sparstencil.h. See DESIGN.md."""
from ._capi import (CudaFailure, InvalidArgument, LogicError, NoDevice, OutOfRange,
                    SparStencilError, lib)
from .engine import (Compiled, MultiSlabStencil, SparseStencil, estimate_device, explore, preset_names, run_batch, run_compile,
                     run_steps_multi, sparse_apply, valid_core)

__all__ = ["Compiled", "SparseStencil", "MultiSlabStencil", "run_steps_multi", "run_batch", "sparse_apply", "run_compile", "explore", "estimate_device", "preset_names",
           "valid_core", "lib",
           "SparStencilError", "InvalidArgument", "LogicError", "OutOfRange", "CudaFailure",
           "NoDevice"]
