"""Slab decomposition of a stencil sweep over the GPUs of one node.

Each rank owns H consecutive slices of the slowest axis (rows in 2D, planes in
3D) of a global grid of H*world slices and keeps r halo slices on every side
that has a neighbour. One time step is

    isend/irecv halos (NCCL, torch.distributed)   ||   interior slices [2r, n-2r)
    wait for the halos
    boundary slices [r, 2r) and [n-2r, n-r)

so the exchange overlaps the bulk of the compute. The
compute is the engine's sm_100a kernel restricted to a slice window
(sst_set_row_window); the exchange is pure plumbing on views of the plan's
ping-pong buffers. With world == 1 a step is a single full-interior launch.

halo="p2p" fuses the exchange into the compute instead: the ranks map each
other's buffers (CUDA IPC; NVLink peer memory on a node) and every step's
epilogue stores the first / last r interior slices into the neighbours' halo
slices as part of its own TMA stores (sst_plan_set_peer). One launch per step,
no exchange step; neighbours are ordered on the streams by flag words
(cuStreamWriteValue32 after a step, cuStreamWaitValue32 before the next).

The index bookkeeping (which slices a rank owns, sends and receives) lives in
`SlabLayout` so it is testable without a GPU (tests/test_multigpu.py runs it
over gloo with world_size 2).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np


@dataclass(frozen=True)
class SlabLayout:
    """Slices of the slowest axis held by one rank (all in global coordinates)."""

    owned: int   # H: slices owned per rank
    world: int
    rank: int
    r: int       # stencil radius = halo width

    @property
    def global_slices(self) -> int:
        return self.owned * self.world

    @property
    def lo(self) -> int:  # first global slice stored locally
        return max(0, self.rank * self.owned - self.r)

    @property
    def hi(self) -> int:  # one past the last global slice stored locally
        return min(self.global_slices, (self.rank + 1) * self.owned + self.r)

    @property
    def local_slices(self) -> int:
        return self.hi - self.lo

    @property
    def has_up(self) -> bool:
        return self.rank > 0

    @property
    def has_down(self) -> bool:
        return self.rank + 1 < self.world

    # local slice ranges [a, b)
    def send_up(self):  # my first r owned slices -> upper neighbour's bottom halo
        return (self.r, 2 * self.r) if self.has_up else None

    def recv_up(self):  # my top halo <- upper neighbour's last r owned slices
        return (0, self.r) if self.has_up else None

    def send_down(self):
        n = self.local_slices
        return (n - 2 * self.r, n - self.r) if self.has_down else None

    def recv_down(self):
        n = self.local_slices
        return (n - self.r, n) if self.has_down else None

    def computed(self):
        """Local interior window the kernel updates: [r, n - r)."""
        return (self.r, self.local_slices - self.r)

    def interior_window(self):
        """Slices whose stencil inputs are all local before the exchange."""
        a, b = self.computed()
        if self.has_up:
            a += self.r
        if self.has_down:
            b -= self.r
        return (a, b)

    def boundary_windows(self):
        out = []
        a, b = self.computed()
        if self.has_up:
            out.append((a, a + self.r))
        if self.has_down:
            out.append((b - self.r, b))
        return out


def exchange_halos(layout: SlabLayout, slab, pitch: int, group=None):
    """Post the halo exchange on a flat view of the current buffer.

    `slab` is a 1-D tensor over the storage buffer (elements), slice i spanning
    [i*pitch, (i+1)*pitch). Returns the list of pending works (wait() them)."""
    import torch.distributed as dist

    ops = []

    def view(rng):
        a, b = rng
        return slab[a * pitch:b * pitch]

    if layout.has_up:
        ops.append(dist.P2POp(dist.isend, view(layout.send_up()), layout.rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, view(layout.recv_up()), layout.rank - 1, group))
    if layout.has_down:
        ops.append(dist.P2POp(dist.isend, view(layout.send_down()), layout.rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, view(layout.recv_down()), layout.rank + 1, group))
    if not ops:
        return []
    if slab.is_cuda and dist.get_backend(group) != "nccl":
        return _staged_exchange(ops, group)
    return dist.batch_isend_irecv(ops)


class _Done:
    def wait(self):
        return True


def _staged_exchange(ops, group):
    """Host-staged exchange for CPU-side backends (gloo) with device buffers:
    used to run the multi-rank schedule with several ranks sharing one GPU
    (NCCL refuses two ranks per device). Synchronous: no overlap."""
    import torch
    import torch.distributed as dist

    torch.cuda.current_stream().synchronize()
    host = [(op, op.tensor.cpu()) for op in ops]
    works = dist.batch_isend_irecv([dist.P2POp(op.op, h, op.peer, group) for op, h in host])
    for w in works:
        w.wait()
    for op, h in host:
        if op.op is dist.irecv:
            op.tensor.copy_(h)
    return [_Done()]


class SlabStencil:
    """A rank's share of a slab-decomposed stencil sweep on its B200."""

    def __init__(self, stencil: str, dims_per_rank: Sequence[int], rank: int = 0, world: int = 1,
                 device: int = 0, group=None, fuse: int = 1, precision: str = "f16", halo: str = "nccl"):
        if halo not in ("nccl", "p2p"):
            raise ValueError("halo must be 'nccl' or 'p2p'")
        self.halo = halo
        self.precision = precision
        import torch

        from .engine import Compiled, SparseStencil

        self.stencil = stencil
        self.fuse = max(1, int(fuse))
        probe = Compiled(stencil, list(dims_per_rank), 16, 8, self.fuse)
        r = (int(probe.info["k"]) - 1) // 2  # halo width of one (fused) launch
        probe.close()
        self.layout = SlabLayout(owned=int(dims_per_rank[0]), world=world, rank=rank, r=r)
        self.local_dims = [self.layout.local_slices, *[int(d) for d in dims_per_rank[1:]]]
        self.owned_dims = list(dims_per_rank)
        self.device = device
        self.group = group
        self.eng = SparseStencil(stencil, self.local_dims, device=device, fuse=self.fuse, precision=precision)
        self._peers_open = []
        self._flags = None
        if halo == "p2p" and world > 1:
            self.eng.bind()  # plan-owned allocations: IPC-exportable as a whole
            self._setup_p2p()
            self.bufs = None
            self.flat = None
        else:
            self.bufs = self.eng.bind_torch()
            self.flat = [b.view(torch.float32) for b in self.bufs]
        st = self.eng.storage
        self.pitch = int(st["plane_pitch"] if len(self.local_dims) == 3 else st["row_pitch"])
        self.cur = 0

    # -- P2P halos ---------------------------------------------------------
    def _setup_p2p(self):
        """Exchange IPC handles of both ping-pong buffers and a flag pair per rank;
        map the neighbours' and register them as the plan's peers."""
        import ctypes as C

        import torch.distributed as dist

        from ._capi import check, lib

        L = lib()
        b0, b1 = C.c_void_p(), C.c_void_p()
        check(L.sst_plan_buffers(self.eng._h, C.byref(b0), C.byref(b1)))
        flags = C.c_void_p()  # uint32 [from_up, from_down]: launches the neighbour finished
        check(L.sst_device_alloc(int(self.device), 8, C.byref(flags)))
        self._flags = flags.value

        def handle(ptr):
            h = (C.c_uint8 * 64)()
            check(L.sst_ipc_handle(C.c_void_p(ptr), h))
            return bytes(h)

        # f16 plans also export their binary16 pair: runs then keep binary16 between
        # steps, halos included (sst_plan_set_peer_h)
        hbufs = None
        if self.precision == "f16":
            h0, h1 = C.c_void_p(), C.c_void_p()
            if L.sst_plan_buffers_h(self.eng._h, C.byref(h0), C.byref(h1)) == 0:
                hbufs = [handle(h0.value), handle(h1.value)]
        mine = {"bufs": [handle(b0.value), handle(b1.value)], "flags": handle(flags.value),
                "slices": self.layout.local_slices, "device": int(self.device), "hbufs": hbufs}
        table = [None] * self.layout.world
        dist.all_gather_object(table, mine, group=self.group)

        def open_(h):
            p = C.c_void_p()
            check(L.sst_ipc_open(int(self.device), (C.c_uint8 * 64).from_buffer_copy(h), C.byref(p)))
            self._peers_open.append(p.value)
            return p.value

        self._peer_flag = {}
        for which, nb in ((0, self.layout.rank - 1), (1, self.layout.rank + 1)):
            if not 0 <= nb < self.layout.world:
                continue
            e = table[nb]
            # the kernel's TMA stores and the stream flag writes go straight into the
            # neighbour's memory: its GPU must be peer-accessible (NVLink / NVSwitch)
            import torch

            if e["device"] != int(self.device) and not torch.cuda.can_device_access_peer(int(self.device),
                                                                                       e["device"]):
                raise RuntimeError(f"halo='p2p': GPU {self.device} cannot access peer GPU {e['device']} "
                                   "(use halo='nccl')")
            pb = [open_(e["bufs"][0]), open_(e["bufs"][1])]
            check(L.sst_plan_set_peer(self.eng._h, which, C.c_void_p(pb[0]), C.c_void_p(pb[1]),
                                      int(e["slices"])))
            if hbufs is not None and e.get("hbufs"):
                ph = [open_(e["hbufs"][0]), open_(e["hbufs"][1])]
                check(L.sst_plan_set_peer_h(self.eng._h, which, C.c_void_p(ph[0]), C.c_void_p(ph[1])))
            # my step count goes into the neighbour's slot that names me: I am the
            # lower neighbour (from_down, +4) of my upper one and vice versa
            self._peer_flag[which] = open_(e["flags"]) + (4 if which == 0 else 0)
        self._launch = 0
        dist.barrier(group=self.group)

    def _p2p_fence(self):
        """P2P halos: neighbours write into this rank's buffers from their first
        step on, so every rank must have finished (re)loading before any steps."""
        if self.halo == "p2p" and self.layout.world > 1:
            import torch
            import torch.distributed as dist

            torch.cuda.synchronize(torch.device("cuda", self.device))
            dist.barrier(group=self.group)

    def _steps_p2p(self, steps, stream):
        """The per-step schedule in C (sst_run_steps_peer): for each launch u, wait
        until both neighbours finished launch u - 1 (flag words in this rank's memory),
        launch, then write u + 1 into the neighbours' flag words."""
        import ctypes as C

        from ._capi import check, lib

        dst = C.c_int()
        up = self._peer_flag.get(0)
        down = self._peer_flag.get(1)
        check(lib().sst_run_steps_peer(self.eng._h, self.cur, int(steps), C.c_void_p(stream or None),
                                       C.c_void_p(self._flags), C.c_void_p(up), C.c_void_p(down),
                                       self._launch, C.byref(dst)))
        self.cur = dst.value
        self._launch += steps // self.fuse

    # -- data --------------------------------------------------------------
    def make_local_input(self, seed: int = 1):
        """Synthetic dyadic input for this rank's local slices (device tensor)."""
        import torch

        from ._capi import lib
        import ctypes as C

        n = int(np.prod(self.local_dims))
        host = np.empty(self.local_dims, dtype=np.float32)
        dims = (C.c_uint64 * len(self.local_dims))(*self.local_dims)
        from ._capi import check
        check(lib().sst_random_grid(len(self.local_dims), dims, int(seed) + self.layout.rank,
                                    host.ctypes.data_as(C.c_void_p)))
        assert host.size == n
        return torch.from_numpy(host).to(torch.device("cuda", self.device))

    def load(self, grid):
        # P2P: a neighbour's last launch may still TMA-store halo slices into this
        # rank's buffers; every rank's device must be idle before the upload too
        self._p2p_fence()
        self.eng.upload(grid, which=0)
        self._p2p_fence()
        self.cur = 0

    def result(self):
        return self.eng.download(self.cur)

    # -- stepping ----------------------------------------------------------
    def kernels_per_step(self) -> int:
        return 1 + len(self.layout.boundary_windows())

    def launches(self) -> int:
        return int(self.eng.stats()["launches"])

    def interior_cells(self) -> int:
        r = self.layout.r
        cells = 1
        a, b = self.layout.computed()
        cells *= (b - a)
        for d in self.local_dims[1:]:
            cells *= d - 2 * r
        return cells

    def _window(self, a: int, b: int):
        # kernel windows are in interior coordinates of the local grid (slice - r)
        r = self.layout.r
        self.eng.set_row_window(a - r, b - r)

    def step(self, steps: int = 1):
        import torch

        stream = torch.cuda.current_stream(torch.device("cuda", self.device)).cuda_stream
        if self.layout.world == 1:
            self.eng.set_row_window(0, 0)
            self.cur = self.eng.run(steps, src=self.cur, stream=stream)
            return
        if steps % self.fuse:
            raise ValueError("steps must be a multiple of the fusion factor")
        if self.halo == "p2p":
            self.eng.set_row_window(0, 0)
            self._steps_p2p(steps, stream)
            return
        for _ in range(steps // self.fuse):
            works = exchange_halos(self.layout, self.flat[self.cur], self.pitch, self.group)
            a, b = self.layout.interior_window()
            self._window(a, b)
            self.eng.run(self.fuse, src=self.cur, stream=stream)
            for w in works:
                w.wait()
            bw = self.layout.boundary_windows()
            if len(bw) == 2 and len(self.local_dims) == 2:  # both boundary windows, one launch
                r = self.layout.r
                self.eng.set_row_windows(bw[0][0] - r, bw[0][1] - r, bw[1][0] - r, bw[1][1] - r)
                self.eng.run(self.fuse, src=self.cur, stream=stream)
            else:
                for a, b in bw:
                    self._window(a, b)
                    self.eng.run(self.fuse, src=self.cur, stream=stream)
            self.cur ^= 1
        self.eng.set_row_window(0, 0)

    def apply_host(self, host: np.ndarray, steps: int, out: Optional[np.ndarray] = None) -> np.ndarray:
        """End to end from host memory through the public API."""
        if self.layout.world == 1:
            return self.eng.apply_host(host, steps, out=out)
        import torch

        self._p2p_fence()  # neighbours' late halo stores land before the upload
        self.eng.upload(np.ascontiguousarray(host, dtype=np.float32), which=0)
        self._p2p_fence()
        self.cur = 0
        self.step(steps)
        if out is None:
            out = np.empty(self.local_dims, dtype=np.float32)
        self.eng.download(self.cur, out)
        torch.cuda.synchronize(torch.device("cuda", self.device))
        return out

    def close(self):
        """Release the plan (P2P halos: collective over the slab's ranks)."""
        import ctypes as C

        from ._capi import lib

        if self._peers_open or self._flags:
            import torch
            import torch.distributed as dist

            from ._capi import check

            # P2P: neighbours store into this rank's buffers until their last step;
            # wait for them (stream flags), then for every rank (collective close)
            if self.halo == "p2p" and getattr(self, "_peer_flag", None):
                for which in self._peer_flag:
                    check(lib().sst_stream_wait_geq_u32(None, C.c_void_p(self._flags + 4 * which), self._launch))
            torch.cuda.synchronize(torch.device("cuda", self.device))
            if self.halo == "p2p" and dist.is_initialized():
                dist.barrier(group=self.group)
        for p in self._peers_open:
            lib().sst_ipc_close(C.c_void_p(p))
        self._peers_open = []
        if self._flags:
            lib().sst_device_free(C.c_void_p(self._flags))
            self._flags = None
        self.eng.close()
