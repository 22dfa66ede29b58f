import sys, numpy as np
import oracle
from paper_2506_22969_b200 import SparseStencil, valid_core
name = sys.argv[1] if len(sys.argv) > 1 else "Box-2D9P"
dims = [int(x) for x in (sys.argv[2].split("x") if len(sys.argv) > 2 else ["96", "160"])]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
g = oracle.random_grid(dims, 1)
eng = SparseStencil(name, dims)
print(eng.stats())
out = eng.apply_host(g.astype(np.float32), steps)
core = valid_core(out, steps, eng.r)
want = oracle.direct_apply(name, g, steps)
d = np.abs(core - want)
print("max abs", d.max(), "mismatches", int((d > 0).sum()), "of", d.size)
if d.max() > 0:
    idx = np.argwhere(d > 0)[:10]
    print(idx, core[tuple(idx[0])], want[tuple(idx[0])])
