"""Repeated jd_solve of one BASELINE config (variance / outlier check): per-solve device time,
setup / solve split, iteration counts.

python scripts/rep_solve.py <config> <reps>
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from inputs import CONFIGS  # noqa: E402
from paper_math_0508111_b200 import binding  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = CONFIGS[c]
L = cfg["L"]
eps = torch.empty(L ** 3, dtype=torch.float64, device="cuda")
binding.anderson_build(eps, L, cfg["W"], cfg["seed"])
pp = binding.default_precond_params()
if "AJ_TD" in os.environ:
    pp.tau_drop = float(os.environ["AJ_TD"])
if "AJ_NCOARSE" in os.environ:
    pp.n_coarse_max = int(os.environ["AJ_NCOARSE"])
st = torch.cuda.current_stream()
for i in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    lam, X, res, s = binding.jd_solve(cfg["k"], cfg["sigma"], cfg["tol"], eps, L, cfg["hop"], pparams=pp)
    e1.record(st)
    e1.synchronize()
    print(json.dumps(dict(i=i, ms=e0.elapsed_time(e1), wall_ms=(time.perf_counter() - t0) * 1e3,
                          setup_ms=s["setup_ms"], solve_ms=s["solve_ms"], outer=s["outer"], inner=s["inner_total"],
                          levels=s["precond"]["levels"], coarse=s["precond"]["coarse_n"])),
          flush=True)
