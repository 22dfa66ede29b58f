import numpy as np, sys
from paper_2506_22969_b200 import SparseStencil
for name, dims, steps in (("Box-2D9P", (200, 300), 1), ("Box-2D9P", (200, 300), 50), ("Box-3D27P", (20, 30, 40), 1), ("Box-3D27P", (20, 30, 40), 5)):
    c = np.full(dims, 0.375, dtype=np.float32)
    eng = SparseStencil(name, list(dims))
    out = eng.apply_host(c, steps)
    eng.close()
    bad = np.argwhere(out != c)
    print(name, dims, steps, "bad", len(bad), bad[:5].tolist(), out[tuple(bad[0])] if len(bad) else "")
