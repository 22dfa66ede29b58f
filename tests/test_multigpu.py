"""Host logic of the slab-decomposed multi-GPU sweep (paper_2506_22969_b200/
multigpu.py) on CPU: index bookkeeping, and a world_size-2 gloo run of the
exact exchange/compute schedule the NCCL path uses (halo isend/irecv ||
interior window, then boundary windows), with the oracle as the per-rank
compute. The distributed result must equal the single-domain sweep bitwise."""
from __future__ import annotations

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2506_22969_b200.multigpu import SlabLayout, exchange_halos


def test_slab_layout_bookkeeping():
    H, r, W = 10, 1, 3
    lays = [SlabLayout(owned=H, world=W, rank=k, r=r) for k in range(W)]
    assert [(l.lo, l.hi) for l in lays] == [(0, 11), (9, 21), (19, 30)]
    assert lays[0].recv_up() is None and lays[0].recv_down() == (10, 11)
    assert lays[1].send_up() == (1, 2) and lays[1].send_down() == (10, 11)
    assert lays[1].interior_window() == (2, 10) and lays[1].boundary_windows() == [(1, 2), (10, 11)]
    # computed windows tile the global interior exactly once
    rows = []
    for l in lays:
        a, b = l.computed()
        rows += list(range(l.lo + a, l.lo + b))
    assert rows == list(range(r, H * W - r))
    # what a rank sends lands exactly where its neighbour receives
    for up, down in zip(lays, lays[1:]):
        sa, sb = down.send_up()
        ra, rb = up.recv_down()
        assert list(range(down.lo + sa, down.lo + sb)) == list(range(up.lo + ra, up.lo + rb))
    l3 = SlabLayout(owned=8, world=2, rank=0, r=3)
    assert l3.local_slices == 11 and l3.send_down() == (5, 8) and l3.recv_down() == (8, 11)


def _fixed_step(name, buf, r, window):
    """One fixed-size step of the oracle on slices [a, b) (all other cells keep)."""
    a, b = window
    out = buf.copy()
    if b > a:
        sub = buf[a - r:b + r]
        res = oracle.direct_apply(name, sub, 1)
        idx = (slice(a, b),) + tuple(slice(r, n - r) for n in buf.shape[1:])
        out[idx] = res
    return out


def _rank_main(rank, world, port, name, owned, rest, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nd, k, _, _ = oracle.preset(name)
    r = (k - 1) // 2
    lay = SlabLayout(owned=owned, world=world, rank=rank, r=r)
    glob = oracle.random_grid([owned * world, *rest], seed=7)
    buf = glob[lay.lo:lay.hi].copy()
    pitch = int(np.prod(rest))
    for _ in range(steps):
        flat = torch.from_numpy(buf.reshape(-1))  # shares memory with buf
        works = exchange_halos(lay, flat, pitch)
        nxt = _fixed_step(name, buf, r, lay.interior_window())
        for w in works:
            w.wait()
        for win in lay.boundary_windows():
            part = _fixed_step(name, buf, r, win)
            nxt[win[0]:win[1]] = part[win[0]:win[1]]
        buf = nxt
    a, b = lay.computed()
    q.put((rank, lay.lo + a, buf[a:b]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,owned,rest", [("Box-2D9P", 12, (30,)), ("Star-2D13P", 9, (26,)),
                                              ("Heat-3D", 6, (9, 10))])
def test_gloo_two_rank_sweep_equals_single_domain(name, owned, rest):
    world, steps = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (abs(hash(name)) % 1000)
    procs = [ctx.Process(target=_rank_main, args=(k, world, port, name, owned, rest, steps, q))
             for k in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single domain, same fixed-size semantics
    nd, k, _, _ = oracle.preset(name)
    r = (k - 1) // 2
    glob = oracle.random_grid([owned * world, *rest], seed=7)
    ref = glob.copy()
    for _ in range(steps):
        ref = _fixed_step(name, ref, r, (r, owned * world - r))
    for _, g0, rows in sorted(parts, key=lambda t: t[0]):
        assert np.array_equal(rows, ref[g0:g0 + len(rows)])
