"""Diagnose the per-step numerics of the f16 sparse tensor-core path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, oracle
from paper_2506_22969_b200 import SparseStencil, valid_core
rng = np.random.default_rng(0)
for name in ("Heat-2D", "Box-2D9P", "Box-3D27P"):
    dims = (96, 160) if "2D" in name else (12, 20, 140)
    x = rng.random(dims).astype(np.float32)
    eng = SparseStencil(name, list(dims))
    got = valid_core(eng.apply_host(x, 1), 1, eng.r).astype(np.float64)
    eng.close()
    x16 = x.astype(np.float16).astype(np.float64)
    exact16 = oracle.direct_apply(name, x16, 1)          # operands rounded, exact sum
    exact = oracle.direct_apply(name, x.astype(np.float64), 1)
    d16 = got - exact16
    print(f"{name}: |gpu-oracle(f16 in)| max {np.abs(d16).max():.3e} mean {d16.mean():+.3e}; "
          f"|gpu-oracle(f32 in)| max {np.abs(got-exact).max():.3e} mean {(got-exact).mean():+.3e}; "
          f"f32-rounded exact16 diff max {np.abs(exact16.astype(np.float32)-exact16).max():.3e}")
# multi-step drift
name, dims, T = "Heat-2D", (512, 512), 100
g = oracle.random_grid(dims, 3)
eng = SparseStencil(name, list(dims))
got = valid_core(eng.apply_host(g.astype(np.float32), T), T, eng.r).astype(np.float64)
eng.close()
want = oracle.direct_apply(name, g, T)
# emulate f16 operand rounding per step on CPU in fp64
cur = g.copy()
for t in range(T):
    cur = oracle.direct_apply(name, cur.astype(np.float16).astype(np.float64), 1)
print("T=100: gpu-oracle mean %+.3e rms %.3e | emulated f16-per-step - oracle mean %+.3e rms %.3e | gpu-emulated max %.3e" % (
    (got-want).mean(), np.sqrt(((got-want)**2).mean()), (cur-want).mean(), np.sqrt(((cur-want)**2).mean()), np.abs(got-cur).max()))
