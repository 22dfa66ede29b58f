"""Experiment: does the relative placement of the two ping-pong buffers matter?
Binds both buffers inside one allocation, B at A + bytes + extra, for several extras."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_22969_b200 import SparseStencil
from paper_2506_22969_b200.multigpu import SlabStencil

name = sys.argv[1]
dims = [int(x) for x in sys.argv[2].split("x")]
src = SlabStencil(name, dims).make_local_input(seed=1)
for extra in [0, 4096, 65536, 1 << 20, (1 << 20) + 8192, 3 << 20, 17 << 20]:
    eng = SparseStencil(name, dims)
    nb = int(eng.storage["bytes"])
    big = torch.empty(2 * nb + extra + 4096, dtype=torch.uint8, device="cuda")
    base = (big.data_ptr() + 1023) // 1024 * 1024
    eng.bind(base, base + nb + extra, keepalive=big)
    eng.upload(src, 0)
    eng.run(4)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); eng.run(40); b.record(); torch.cuda.synchronize()
    print(f"extra {extra:>10d}: {a.elapsed_time(b) * 1e3 / 40:7.2f} us/step", flush=True)
    eng.close()
