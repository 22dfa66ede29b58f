#!/usr/bin/env python
"""Benchmark of the B200 SparStencil hot path (one JSON line on rank 0).

Workload (BASELINE.json configs[1]): Box-2D9P, 8192 x 8192 fp32 grid, 1000 time
steps, synthetic dyadic input (random_grid, seed 1), 2:4-sparse tcgen05.mma.sp
(f16 operands, f32 accumulate, f32 storage). A bench *step* is one time step:
one pass of the compiled stencil over the whole grid (one kernel launch).
Default --steps 1000 times the config's full 1000-step run.

  value      GStencil/s = steps * prod(N) / t (Eq. 12, stencil.cpp:349-359),
             grid resident in HBM, CUDA events on the launch stream, max over ranks
  e2e        the same metric through the public API from HOST memory: one
             sst_apply_host call = H2D of the grid + `steps` time steps + D2H
  roofline   dominant kernel vs measured HBM copy bandwidth (8 B per update)
  cpu_baseline  the reference's own direct_apply (oracle/_ref, built from the
             reference sources) on the host cores, bounded sample

N > 1 (torchrun): the north-star scaling config by default — Box-3D27P 1024^3
STRONG-scaled: rank i owns 1024/N planes (+ 1 halo plane per neighbour); each step
is one launch per rank whose epilogue also stores the boundary planes straight into
the neighbours' halo planes over NVLink (P2P, CUDA IPC), ranks ordered by stream
flags by the C per-step schedule (sst_run_steps_peer). Rank 0 also times the same
1024^3 grid alone on its GPU (`n1_same_grid`) so the line carries its own N = 1
reference. `--config X --weak` keeps the old weak scaling (X per rank).

--impl reference: the reference CPU implementation (oracle/_ref) on the host
cores, same metric; each step is one time step over a bounded row band.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

CONFIGS = {
    # name: (stencil, dims, default time steps)
    "box2d": ("Box-2D9P", (8192, 8192), 1000),
    "heat2d": ("Heat-2D", (4096, 4096), 100),
    "star2d": ("Star-2D13P", (16384, 16384), 100),
    "heat3d": ("Heat-3D", (512, 512, 512), 100),
    "box3d": ("Box-3D27P", (512, 512, 512), 100),
    "box3d1024": ("Box-3D27P", (1024, 1024, 1024), 100),
}
METRIC = "GStencil/s per stencil at 1/2/4/8 B200; % of HBM & sparse-TC roofline"


def _peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: NVML every
    10 ms (nvidia-smi every 200 ms if NVML is unavailable)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []  # (sm_mhz, max_mhz, [reasons])
        self._stop = threading.Event()
        self._t = None

    def _nvml(self):
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

        def sample():
            mask = get_reasons(h)
            return (float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)), float(mx),
                    [n for bit, n in self.REASONS.items() if mask & bit])
        return sample

    def _smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

        def sample():
            out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=5).stdout.strip()
            r = [x.strip() for x in out.split(",")]
            return (float(r[0]), float(r[1]), [names[i] for i in range(4) if r[2 + i].lower() == "active"])
        return sample

    def start(self):
        try:
            sample, period = self._nvml(), 0.01
        except Exception:
            sample, period = self._smi(), 0.2

        def run():
            while not self._stop.is_set():
                try:
                    self.rows.append(sample())
                except Exception:
                    pass
                self._stop.wait(period)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(r[0] for r in self.rows),
                "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted({n for r in self.rows for n in r[2]}),
                "samples": len(self.rows)}


def _load_traffic(cfg_name):
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    p = REPO / "profiles" / "ncu_traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(cfg_name)
        except Exception:
            return None
    return None


def cpu_baseline(stencil, dims, budget_s=12.0):
    """Reference direct_apply (oracle/_ref) on all host cores, bounded sample."""
    import oracle

    threads = os.cpu_count() or 1
    if oracle.ref_available():
        kind = "reference"
        fn = lambda g: oracle.ref_direct_apply_slabs(stencil, g, threads)  # noqa: E731
    else:  # the C restatement (single thread) when the reference .so is absent
        kind, threads = "port", 1
        fn = lambda g: oracle.direct_apply(stencil, g, 1)  # noqa: E731
    # a band of rows of the same grid (full row length), one time step per call
    band = list(dims)
    band[0] = min(dims[0], max(64, int(4_000_000 // int(np.prod(dims[1:])))))
    g = oracle.random_grid(band, seed=1)
    fn(g)  # warm
    n, t0 = 0, time.perf_counter()
    while True:
        fn(g)
        n += 1
        if time.perf_counter() - t0 > budget_s or n >= 200:
            break
    dt = time.perf_counter() - t0
    cells = n * int(np.prod(band))
    out = {"value": cells / dt / 1e9, "unit": "GStencil/s", "cores": threads, "kind": kind,
           "sample": f"{n} x one time step of {stencil} on a {'x'.join(map(str, band))} band "
                     f"of the {'x'.join(map(str, dims))} grid ({dt:.1f} s)"}
    # BASELINE.md's plan beside it: the single-threaded reference on ONE pinned core over
    # the FULL grid, one time step (grids up to 8192^2: a few seconds)
    if kind == "reference" and int(np.prod(dims)) <= (1 << 26) + (1 << 20):
        try:
            full = oracle.random_grid(dims, seed=1)
            aff = os.sched_getaffinity(0)
            os.sched_setaffinity(0, {min(aff)})
            try:
                t0 = time.perf_counter()
                oracle.ref_direct_apply_slabs(stencil, full, 1)
                d1 = time.perf_counter() - t0
            finally:
                os.sched_setaffinity(0, aff)
            out["single_core_full_grid"] = {
                "value": int(np.prod(dims)) / d1 / 1e9, "unit": "GStencil/s", "cores": 1,
                "sample": f"one time step of {stencil} over the whole {'x'.join(map(str, dims))} grid "
                          f"({d1:.1f} s), the reference's direct_apply pinned to one core"}
            del full
        except Exception as exc:  # noqa: BLE001  (the headline must not depend on it)
            out["single_core_full_grid"] = {"error": str(exc)[:200]}
    return out


def parity_check(stencil, host_in, host_out, steps, r, precision):
    """The checker (test infrastructure, outside every timed region): windows of
    the e2e run's output against the CPU oracle — the fp64 reference sweep (rel-L2,
    max-abs) and, for f16, the round16-iterated oracle (bitwise). An output window
    needs its input window plus a steps*r halo (tests/test_gpu_baseline_parity.py)."""
    import oracle

    dims = host_in.shape
    w = 64 if len(dims) == 2 else 16
    h = steps * r
    if any(n < 2 * h + w for n in dims):
        return None
    sq_e = sq_r = max_abs = 0.0
    exact = True
    t0 = time.perf_counter()
    for o in ([h] * len(dims), [(n - w) // 2 for n in dims], [n - h - w for n in dims]):
        src = host_in[tuple(slice(a - h, a + w + h) for a in o)]
        got = host_out[tuple(slice(a, a + w) for a in o)].astype(np.float64)
        want = oracle.direct_apply_mt(stencil, src, steps)
        d = got - want
        sq_e += float(np.sum(d * d))
        sq_r += float(np.sum(want * want))
        max_abs = max(max_abs, float(np.abs(d).max()))
        if precision == "f16":
            exact &= bool(np.array_equal(got, oracle.direct_apply_mt(stencil, src, steps, round16=True)))
    return {"steps": steps, "rel_l2": (sq_e / sq_r) ** 0.5, "max_abs": max_abs,
            "vs": "fp64 reference sweep (oracle pinned to direct_apply), valid region",
            "bitwise_round16_semantics": exact if precision == "f16" else None,
            "windows": f"3 windows of {w}^{len(dims)} outputs (low corner, middle, high corner)",
            "check_s": time.perf_counter() - t0}


def run_reference(args, cfg):
    stencil, dims, tsteps = cfg
    ws, rank, _ = _dist_env()
    if rank != 0:
        return
    import oracle

    threads = os.cpu_count() or 1
    kind = "reference" if oracle.ref_available() else "port"
    band = list(dims)
    band[0] = min(dims[0], max(32, int(2_000_000 // int(np.prod(dims[1:])))))
    g = oracle.random_grid(band, seed=1)
    fn = (lambda: oracle.ref_direct_apply_slabs(stencil, g, threads)) if kind == "reference" \
        else (lambda: oracle.direct_apply(stencil, g, 1))
    if kind == "port":
        threads = 1
    for _ in range(args.warmup):
        fn()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fn()
    dt = time.perf_counter() - t0
    val = args.steps * int(np.prod(band)) / dt / 1e9
    line = {"metric": METRIC, "value": val, "unit": "GStencil/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (random_grid seed 1, dyadic)", "impl": "reference",
            "config": {"workload": f"{stencil} {'x'.join(map(str, dims))}, one time step per "
                                   f"bench step over a {'x'.join(map(str, band))} row band",
                       "stencil": stencil, "grid": list(dims)},
            "cpu_baseline": {"value": val, "unit": "GStencil/s", "cores": threads, "kind": kind,
                             "sample": f"{args.steps} time steps over a {'x'.join(map(str, band))} band"},
            "e2e": {"value": val, "unit": "GStencil/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_engine(args, cfg, cfg_name):
    import torch

    from paper_2506_22969_b200 import SparseStencil

    stencil, global_dims, _ = cfg
    ws, rank, local = _dist_env()
    if args.share_gpu:  # functional runs of the multi-rank path on a one-GPU host
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist

        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    from paper_2506_22969_b200.multigpu import SlabStencil

    strong = ws > 1 and not args.weak
    if strong:  # rank-owned slab of the global grid (slowest axis split N ways)
        if global_dims[0] % ws:
            raise SystemExit(f"{global_dims[0]} slices do not split over {ws} ranks")
        dims = (global_dims[0] // ws, *global_dims[1:])
    else:
        dims = global_dims
    n1 = None
    if strong and rank == 0:  # the same global grid on this GPU alone (N = 1 reference)
        n1 = _n1_same_grid(stencil, global_dims, local, args)
    if ws > 1:
        dist.barrier()
    eng = SlabStencil(stencil, dims, rank=rank, world=ws, device=local, fuse=args.fuse,
                      precision=args.precision, halo=args.halo)
    grid = eng.make_local_input(seed=1)  # dense fp32 torch tensor on the device
    eng.load(grid)
    stream = torch.cuda.current_stream(dev)

    # warm-up: one W-step run (the same kernels as the timed run, binary16 storage
    # included), then W single steps (the round-robin timing of small grids)
    eng.step(args.warmup * args.fuse)
    for _ in range(args.warmup):
        eng.step(args.fuse)
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()

    # Grids that (with their ping-pong partner) fit in the 126 MB L2 would be timed
    # from L2. Such grids are timed over inputs larger than L2 instead: `nrep`
    # independent copies of the problem (own plan, own ping-pong pair), stepped
    # round-robin back to back, so every launch reads a grid last touched nrep - 1
    # launches (>= 400 MB of traffic) earlier. A single launch after a full L2 flush
    # is timed as well and reported beside it (it carries the ~6 us fixed cost of one
    # event-bracketed launch, tools/probes/probe_launch.cu).
    pair_bytes = 2 * int(np.prod(dims)) * 4
    small = pair_bytes <= 192 << 20
    engines = [eng]
    if small:
        nrep = -(-(400 << 20) // pair_bytes) + 1
        for _ in range(nrep - 1):
            e = SlabStencil(stencil, dims, rank=rank, world=ws, device=local, fuse=args.fuse,
                            precision=args.precision, halo=args.halo)
            e.load(grid)
            for _ in range(args.warmup):
                e.step(args.fuse)
            engines.append(e)
    clocks = ClockSampler(local)
    clocks.start()
    from paper_2506_22969_b200 import lib as _sst_lib

    launches0 = sum(e.launches() for e in engines)
    kernels0 = int(_sst_lib().sst_launch_count())
    h16_0 = sum(int(e.eng.stats()["h16_launches"]) for e in engines)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    if not args.share_gpu:  # (ranks sharing one GPU would spin while the other rank is timed)
        _hold_device(stream)
    ev0.record(stream)
    if small:
        _step_copies(engines, args.steps // args.fuse, args.fuse, stream.cuda_stream, batch=ws == 1)
    else:
        eng.step(args.steps)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    ms = ev0.elapsed_time(ev1)
    launches = sum(e.launches() for e in engines) - launches0  # operator launches applied to the grids
    kernels = int(_sst_lib().sst_launch_count()) - kernels0      # kernels the library issued
    h16_launches = sum(int(e.eng.stats()["h16_launches"]) for e in engines) - h16_0
    flushed = None
    if small:
        flush = (torch.empty(256 << 20, dtype=torch.uint8, device=dev),
                 torch.zeros(64 << 20, dtype=torch.int32, device=dev))
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(min(20, args.steps // args.fuse))]
        for a, b in evs:
            flush[0].add_(1)
            flush[1].sum()
            a.record(stream)
            eng.step(args.fuse)
            b.record(stream)
        torch.cuda.synchronize(dev)
        t1 = sum(a.elapsed_time(b) for a, b in evs) / len(evs)
        flushed = {"ms_per_launch": t1, "launches": len(evs),
                   "note": "one launch between events after a 256 MB write + 256 MB read L2 flush"}
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    if ws > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    cells_global = int(np.prod(dims)) * ws  # (strong: = the global grid)
    value = args.steps * cells_global / (ms / 1e3) / 1e9

    # roofline of the dominant kernel: one launch reads the grid and writes the
    # interior once, 8 B per interior cell (read 4 + write 4), whatever the
    # fusion factor (a fused launch advances `fuse` time steps).
    interior = eng.interior_cells()
    operator_steps = args.steps // args.fuse          # launches of the stencil operator
    t_kernel = ms / 1e3 / operator_steps              # per operator application (all windows)
    # binary16 inter-step storage (f16 runs of >= 2 launches): the first launch reads
    # fp32 (4 B) and writes binary16 (2 B), the middle ones 2 + 2 B, the last one
    # 2 + 4 B per update; otherwise 4 + 4 B. Averaged over the timed launches.
    if h16_launches:  # one binary16 run per grid copy (large grids: one copy)
        alg_total = interior * (4.0 * operator_steps + 4.0 * len(engines))
    else:
        alg_total = 8.0 * interior * operator_steps
    alg_bytes = alg_total / operator_steps
    peak, peak_kind = _peaks()
    achieved = alg_bytes / t_kernel / 1e9
    traffic = _load_traffic((cfg_name + ("_h16" if h16_launches else ""))
                            if args.fuse == 1 and args.precision == "f16" else None)
    if flushed is not None:
        flushed["frac"] = alg_bytes / (flushed["ms_per_launch"] / 1e3) / 1e9 / peak

    # e2e through the public API from host memory (rank-local slab)
    e2e = None
    parity = None
    if not args.no_e2e:
        # page-locked host buffers (what a production caller hands the C ABI)
        host_t = torch.empty(tuple(grid.shape), dtype=torch.float32, pin_memory=True)
        host_t.copy_(grid)
        out_t = torch.empty_like(host_t, pin_memory=True)
        host, out_h = host_t.numpy(), out_t.numpy()
        # one public-API call at the config's stated T (direct_apply(spec, grid, T) is the
        # call a reference user makes: one H2D, T steps, one D2H), whatever --steps is
        e2e_steps = args.e2e_steps or CONFIGS[cfg_name][2]
        e2e_steps = max(args.fuse, e2e_steps - e2e_steps % args.fuse)
        eng.apply_host(host, args.fuse, out=out_h)  # warm
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        eng.apply_host(host, e2e_steps, out=out_h)
        dt = time.perf_counter() - t0
        if ws > 1:
            t = torch.tensor([dt], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        nbytes = int(host.nbytes)
        e2e = {"value": e2e_steps * cells_global / dt / 1e9, "unit": "GStencil/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "step": f"one sst_apply_host call = H2D + {e2e_steps} time steps + D2H"}
        if rank == 0 and ws == 1 and not args.no_cpu:
            # (fused operators round once per launch: a different semantics, not checked here)
            if args.fuse == 1:
                parity = parity_check(stencil, host, out_h, e2e_steps, eng.layout.r, args.precision)

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return
    cpu = None if (ws > 1 or args.no_cpu) else cpu_baseline(stencil, dims)
    workload = (f"{stencil} {'x'.join(map(str, global_dims))} strong-scaled over {ws} GPUs "
                f"({dims[0]} planes each + halos), {args.steps} time steps (one bench step = one time step)"
                if strong else
                f"{stencil} {'x'.join(map(str, dims))} per GPU, {args.steps} time steps "
                f"(one bench step = one time step)")
    line = {
        "metric": METRIC, "value": value, "unit": "GStencil/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": "f16",
        "data": "synthetic (random_grid seed 1: dyadic values in [0,1))",
        "config": {"workload": workload, "global_grid": list(global_dims) if strong else None,
                   "stencil": stencil, "grid_per_gpu": list(dims), "time_steps": args.steps,
                   "temporal_fusion": args.fuse,
                   "storage": ("fp32 input / output, binary16 between steps (bitwise the fp32-storage result: "
                               "the next step's operand is rounded to binary16 RNE either way)")
                              if h16_launches else "fp32",
                   "operands": "f16 (tcgen05.mma.sp kind::f16), f32 accumulate",
                   "layout": "(r1, r2) = (16, 8), m' = 128",
                   "l2": (f"inputs larger than L2: {len(engines)} independent copies of the grid "
                          f"({len(engines) * pair_bytes >> 20} MB of fp32 ping-pong buffers) stepped together "
                          f"(sst_run_steps_batch: launches interleaved step by step), "
                          f"each launch reading a grid last touched {len(engines) - 1} launches earlier")
                         if small else "inputs larger than L2 (ping-pong pair > 126 MB)",
                   "parallelism": (f"slab{ws} ({args.halo} halos)" if ws > 1 else "single GPU")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "l2_flushed_single_launch": flushed,
                     "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                     "algorithmic_bytes_per_step": alg_bytes,
                     "launch_steps": (operator_steps // launches) if launches else None,
                     "per": ("operator step: one launch runs all timed steps (2D multi-step kernel); achieved = "
                             "8 B x interior cells / (launch time / steps), traffic = ncu DRAM bytes / steps")
                            if launches and operator_steps // launches > 1 else
                            ("launch (one operator step), averaged over the run: algorithmic bytes = interior cells x "
                             "(4 B x launches + 4 B per grid copy) (binary16 between steps: 2 B read + 2 B write per "
                             "update; a run's first launch reads fp32, its last writes fp32)") if h16_launches else
                            "launch (one operator step)",
                     "h16_launches": h16_launches,
                     "kernel": "sst::stencil3d_stream_kernel" if len(dims) == 3
                     else "sst::stencil_step_kernel"},
        "e2e": e2e,
        "cpu_baseline": cpu,
        "parity": parity,
        "gpu_launches": int(kernels),
        "clocks": clk,
    }
    if n1 is not None:
        line["n1_same_grid"] = n1
    # the engine's execution model of the dominant launch (hwmodel.hpp estimate_device):
    # which on-chip resource binds when the HBM fraction is below 1
    try:
        from paper_2506_22969_b200 import estimate_device

        m = estimate_device(stencil, dims, fuse=args.fuse, storage=2 if h16_launches else 4)
        # the shared-memory pipe as a second roofline: the model's wavefronts per launch
        # (one 128-byte wavefront per SM clock at peak) over the measured launch time
        sm_clk = 148 * (clk.get("sm_mhz") or 1965.0) * 1e6
        line["roofline"]["model"] = {"predicted_ms_per_launch": m["t_total"] * 1e3, "bound": m["bound"],
                                     "t_hbm_ms": m["t_hbm"] * 1e3, "t_smem_ms": m["t_smem"] * 1e3,
                                     "t_tensor_ms": m["t_mma"] * 1e3,
                                     "smem_wavefronts_per_launch": m["smem_wavefronts"],
                                     "smem_pipe_frac": m["smem_wavefronts"] / (t_kernel * sm_clk),
                                     "note": "estimate_device (hwmodel.hpp): smem_pipe_frac = modelled shared-memory "
                                             "wavefronts / (launch time x 148 SMs x SM clock); ncu l1tex throughput "
                                             "73-90 % (profiles/round2/ncu_*_full.txt)"}
    except Exception:
        pass
    if ws == 1 and not args.no_sweep and args.fuse == 1 and args.precision == "f16":
        line["other_configs"] = _sweep_configs(args, cfg_name, local)
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def _hold_device(stream):
    """A ~1 ms spin kernel ahead of the start event: the device reaches the event only
    after the host has enqueued the first timed launches, so the timed region holds
    device work, not the host's enqueue latency (the e2e number keeps the host side)."""
    import torch

    sleep = getattr(torch.cuda, "_sleep", None)  # (torch's spin kernel; absent: no hold)
    if sleep is not None:
        with torch.cuda.stream(stream):
            sleep(2_000_000)


def _step_copies(engines, launches, fuse, stream, batch=True):
    """`launches` operator steps spread over independent copies of a grid whose ping-pong
    pair fits in L2: every copy advances launches // n steps in ONE interleaved batch run
    (sst_run_steps_batch: step t of copy 0 .. n-1, then step t + 1; binary16 between
    steps), so each launch reads a grid last touched n - 1 launches earlier; the
    remainder as single steps. batch=False: plain round-robin single steps."""
    from paper_2506_22969_b200 import run_batch

    n = len(engines)
    per, rem = divmod(launches, n)
    if batch and per > 0:
        dst = run_batch([e.eng for e in engines], per * fuse, [e.cur for e in engines], stream=stream)
        for e, d in zip(engines, dst):
            e.cur = d
    else:
        rem = launches
    for i in range(rem):
        engines[i % n].step(fuse)


def _sweep_configs(args, skip, device, budget_steps=None):
    """Every other BASELINE config on this GPU in the same run (device-resident GStencil/s
    at the config's operator, same timing rules as the headline: CUDA events on the
    launch stream, grids whose ping-pong pair fits in L2 stepped round-robin over
    independent copies). Steps per config: the config's stated T (one run, binary16
    between steps, as the headline)."""
    import torch

    from paper_2506_22969_b200 import estimate_device
    from paper_2506_22969_b200.multigpu import SlabStencil

    out = {}
    stream = torch.cuda.current_stream(torch.device("cuda", device))
    peak, _ = _peaks()
    for name, (stencil, dims, T) in CONFIGS.items():
        if name == skip:
            continue
        steps = T if budget_steps is None else min(T, budget_steps)
        pair = 2 * int(np.prod(dims)) * 4
        small = pair <= 192 << 20
        nrep = (-(-(400 << 20) // pair) + 1) if small else 1
        engines = []
        try:
            for _ in range(nrep):
                e = SlabStencil(stencil, dims, device=device)
                e.load(e.make_local_input(seed=1))
                engines.append(e)
            engines[0].step(3)
            for e in engines:
                e.step(1)
            torch.cuda.synchronize(device)
            h0 = sum(int(e.eng.stats()["h16_launches"]) for e in engines)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            _hold_device(stream)
            a.record(stream)
            if small:
                _step_copies(engines, steps, 1, stream.cuda_stream)
            else:
                engines[0].step(steps)
            b.record(stream)
            torch.cuda.synchronize(device)
            ms = a.elapsed_time(b)
            h16 = sum(int(e.eng.stats()["h16_launches"]) for e in engines) - h0
            interior = engines[0].interior_cells()
            alg = interior * (4.0 * steps + 4.0) if h16 else 8.0 * interior * steps
            model = estimate_device(stencil, dims, storage=2 if h16 else 4)
            out[name] = {"stencil": stencil, "grid": list(dims), "steps": steps, "config_T": T,
                         "value": steps * int(np.prod(dims)) / (ms / 1e3) / 1e9, "unit": "GStencil/s",
                         "ms_per_step": ms / steps, "storage": "binary16 between steps" if h16 else "fp32",
                         "l2": f"{nrep} copies stepped interleaved (batch run)" if small else "grid pair > L2",
                         "hbm_frac": alg / (ms / 1e3) / 1e9 / peak,
                         "model": {"predicted_ms_per_step": model["t_total"] * 1e3, "bound": model["bound"]}}
        except Exception as exc:  # a config that cannot run here must not sink the headline line
            out[name] = {"error": str(exc)[:200]}
        finally:
            for e in engines:
                e.close()
            del engines
            torch.cuda.empty_cache()
    return out


def _n1_same_grid(stencil, global_dims, device, args):
    """The strong-scaled global grid on one GPU (rank 0's), same steps: the N = 1
    point of the scaling curve, measured in the same run."""
    import torch

    from paper_2506_22969_b200.multigpu import SlabStencil

    eng = SlabStencil(stencil, global_dims, device=device, fuse=args.fuse, precision=args.precision)
    eng.load(eng.make_local_input(seed=1))
    eng.step(args.warmup * args.fuse)
    stream = torch.cuda.current_stream(torch.device("cuda", device))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(device)
    _hold_device(stream)
    a.record(stream)
    eng.step(args.steps)
    b.record(stream)
    torch.cuda.synchronize(device)
    ms = a.elapsed_time(b)
    eng.close()
    del eng
    torch.cuda.empty_cache()
    return {"value": args.steps * int(np.prod(global_dims)) / (ms / 1e3) / 1e9, "unit": "GStencil/s",
            "ms_per_step": ms / args.steps, "n_gpus": 1,
            "note": "the same global grid and steps on rank 0's GPU alone (the N = 1 point of this strong scaling)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: box2d (BASELINE configs[1]) on one GPU, box3d1024 strong-scaled for N > 1")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip timing the other BASELINE configs (other_configs) after the headline")
    ap.add_argument("--weak", action="store_true",
                    help="N > 1: weak scaling (the config's grid per rank) instead of strong scaling")
    ap.add_argument("--share-gpu", action="store_true",
                    help="N > 1 on a one-GPU host: every rank on device 0, gloo control plane (functional)")
    ap.add_argument("--halo", default="p2p", choices=["nccl", "p2p"],
                    help="multi-GPU halo exchange: NCCL p2p overlapped with the interior window, or fused "
                         "into the kernel (boundary slices stored into the neighbours' buffers over NVLink)")
    ap.add_argument("--precision", default="f16", choices=["f16", "f16x2"],
                    help="operand precision: f16 (round16 operands) or f16x2 (split hi+lo operand, ~fp32)")
    ap.add_argument("--fuse", type=int, default=1,
                    help="temporal fusion factor (reference fuse_time_steps); steps count original time steps")
    args = ap.parse_args()
    if args.config is None:
        args.config = "box3d1024" if int(os.environ.get("WORLD_SIZE", "1")) > 1 and not args.weak else "box2d"
    cfg = CONFIGS[args.config]
    if args.steps is None:
        args.steps = cfg[2]
    args.warmup = max(3, args.warmup)
    if args.fuse < 1 or args.steps % args.fuse:
        ap.error(f"--steps ({args.steps}) must be a positive multiple of --fuse ({args.fuse})")
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_engine(args, cfg, args.config)


if __name__ == "__main__":
    main()
