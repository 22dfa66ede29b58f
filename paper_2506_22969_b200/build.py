"""In-tree build of libsparstencil.so (host C++20 compile library + sm_100a
CUDA runtime/kernels behind the C ABI in include/sparstencil.h).

    python -m paper_2506_22969_b200.build        # or build() from __graft_entry__

Incremental by mtime; objects under paper_2506_22969_b200/build/ (git-ignored),
the shared library next to this file (and the `sstensor` CLI under bin/) so
they travel to the GPU box with the repo snapshot. cudart is linked statically and the driver API is resolved at
run time (cudaGetDriverEntryPoint), so the library loads on a CPU-only host.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "build"
LIB = PKG / "libsparstencil.so"
CLI = PKG / "bin" / "sstensor"

NVCC = os.environ.get("NVCC", "nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INCLUDES = [f"-I{REPO / 'include'}", f"-I{CSRC / 'host'}", f"-I{CSRC / 'device'}"]
CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-fvisibility=hidden"]
NVFLAGS = ["-std=c++20", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-fvisibility=hidden",
           "--expt-relaxed-constexpr"]
# SST_ABLATION=1: compile the kernels' ablation bits in (tools/ablate.py, profiling only;
# objects go to build_ablation/ and the library to libsparstencil_ablation.so, which
# SST_LIB=ablation selects at load time)
ABLATION = os.environ.get("SST_ABLATION") == "1"
if ABLATION:
    NVFLAGS += ["-DSST_ABLATION=1"]
    OBJ = PKG / "build_ablation"
    LIB = PKG / "libsparstencil_ablation.so"

HOST_SRCS = sorted((CSRC / "host").glob("*.cpp"))
DEVICE_SRCS = sorted((CSRC / "device").glob("*.cu"))
HEADERS = sorted((CSRC).rglob("*.h*")) + sorted((REPO / "include").glob("*.h")) + sorted(
    (CSRC / "device").glob("*.cuh"))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(str(c) for c in cmd), flush=True)
    subprocess.run([str(c) for c in cmd], check=True)


def build(verbose: bool = False, force: bool = False) -> Path:
    from concurrent.futures import ThreadPoolExecutor

    OBJ.mkdir(exist_ok=True)
    objs, jobs = [], []
    for src in HOST_SRCS:
        o = OBJ / (src.stem + ".o")
        objs.append(o)
        if force or _stale(o, [src, *HEADERS, __file__]):
            jobs.append([CXX, *CXXFLAGS, *INCLUDES, "-c", src, "-o", o])
    for src in DEVICE_SRCS:
        o = OBJ / (src.stem + ".cu.o")
        objs.append(o)
        if force or _stale(o, [src, *HEADERS, __file__]):
            jobs.append([NVCC, *NVFLAGS, *INCLUDES, "-c", src, "-o", o])
    # the translation units compile independently (the kernel instantiations dominate)
    jobs.sort(key=lambda c: c[0] != NVCC)  # longest first
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(_run, c, verbose) for c in jobs]:
            f.result()
    if force or _stale(LIB, objs):
        _run([NVCC, "-shared", *ARCH, "-cudart", "static", "-o", LIB, *objs], verbose)
    if ABLATION:  # (the CLI is built from the production objects only)
        return LIB
    # the CLI (reference tools/main.cpp) links the same objects statically
    cli_src = CSRC / "cli" / "sstensor.cpp"
    cli_obj = OBJ / "sstensor.o"
    if force or _stale(cli_obj, [cli_src, *HEADERS, __file__]):
        _run([CXX, *CXXFLAGS, *INCLUDES, "-I/usr/local/cuda/include", "-c", cli_src, "-o", cli_obj], verbose)
    CLI.parent.mkdir(exist_ok=True)
    if force or _stale(CLI, [*objs, cli_obj]):
        _run([NVCC, *ARCH, "-cudart", "static", "-o", CLI, cli_obj, *objs], verbose)
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
