"""Small device runs for compute-sanitizer (memcheck / synccheck): every kernel
family on tiny ragged grids. Usage: compute-sanitizer --tool memcheck python tools/sanitize_smoke.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2506_22969_b200 import SparseStencil, valid_core  # noqa: E402

cases = [("Box-2D9P", (97, 301), "f16", 3), ("Star-2D13P", (70, 140), "f16x2", 2),
         ("Box-3D27P", (12, 23, 131), "f16", 3), ("Heat-3D", (9, 20, 40), "f16x2", 2),
         ("Heat-1D", (1001,), "f16", 4), ("Box-2D49P", (300, 517), "f16", 1)]
for name, dims, prec, steps in cases:
    g = oracle.random_grid(dims, seed=1)
    eng = SparseStencil(name, list(dims), precision=prec)
    out = valid_core(eng.apply_host(g.astype(np.float32), steps), steps, eng.r)
    eng.close()
    want = oracle.direct_apply(name, g, steps)
    print(name, dims, prec, steps, "max err %.3g" % np.abs(out - want).max(), flush=True)
os.environ["SST_MULTISTEP"] = "1"
eng = SparseStencil("Box-2D9P", [200, 300])
eng.apply_host(oracle.random_grid((200, 300), seed=2).astype(np.float32), 5)
eng.close()
print("sanitize smoke done")
