"""Preconditioner setup only (for ncu launch lists / per-level timing).

python scripts/prof_setup.py L [W] [seed]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_math_0508111_b200 import binding  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 150
W = float(sys.argv[2]) if len(sys.argv) > 2 else 16.5
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 4
eps = torch.empty(L ** 3, dtype=torch.float64, device="cuda")
binding.anderson_build(eps, L, W, seed)
torch.cuda.synchronize()
t0 = time.perf_counter()
K = binding.Precond(eps, L, -1.0, 0.0)
torch.cuda.synchronize()
info = K.info()
print(f"setup L={L} W={W}: {time.perf_counter() - t0:.3f} s levels {info['levels']} coarse {info['coarse_n']} "
      f"nnzL/site {info['nnz_L'] / L ** 3:.2f} setup_ms {info['setup_ms']:.1f}", flush=True)
K.free()
