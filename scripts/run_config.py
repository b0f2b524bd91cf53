"""Run jd_solve on a BASELINE config through the C ABI and print timings/stats.

python scripts/run_config.py <config index> [W override] [seed override]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs import CONFIGS  # noqa: E402
from paper_math_0508111_b200 import binding  # noqa: E402


def main():
    c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    cfg = dict(CONFIGS[c])
    if len(sys.argv) > 2:
        cfg["W"] = float(sys.argv[2])
    if len(sys.argv) > 3:
        cfg["seed"] = int(sys.argv[3])
    if len(sys.argv) > 4:
        cfg["L"] = int(sys.argv[4])
    L = cfg["L"]
    eps = torch.empty(L ** 3, dtype=torch.float64, device="cuda")
    binding.anderson_build(eps, L, cfg["W"], cfg["seed"])
    jp = binding.default_jd_params(verbose=1, max_outer=int(os.environ.get("AJ_MAX_OUTER", "600")))
    if "AJ_INNER_MAX" in os.environ:
        jp.inner_max = int(os.environ["AJ_INNER_MAX"])
    if "AJ_INNER_TOL" in os.environ:
        jp.inner_tol = float(os.environ["AJ_INNER_TOL"])
    pp = binding.default_precond_params()
    for key, env in (("tau_drop", "AJ_TD"), ("tau_strong", "AJ_TS"), ("tau_virtual", "AJ_TV"), ("tau_inv", "AJ_TINV"),
                     ("kappa", "AJ_KAPPA")):
        if env in os.environ:
            setattr(pp, key, float(os.environ[env]))
    if "AJ_F32" in os.environ:
        pp.factor_fp32 = int(os.environ["AJ_F32"])
    if "AJ_DENSE_CAP" in os.environ:
        pp.dense_cap = int(os.environ["AJ_DENSE_CAP"])
    if "AJ_NCOARSE" in os.environ:
        pp.n_coarse_max = int(os.environ["AJ_NCOARSE"])
    t0 = time.perf_counter()
    try:
        lam, X, res, st = binding.jd_solve(cfg["k"], cfg["sigma"], cfg["tol"], eps, L, cfg["hop"], pparams=pp,
                                           jparams=jp)
    except Exception as ex:  # report the failure as a JSON line too
        print(json.dumps(dict(config=c, L=L, W=cfg["W"], seed=cfg["seed"], error=str(ex)[:300],
                              wall_s=time.perf_counter() - t0, env={k: v for k, v in os.environ.items()
                                                                    if k.startswith("AJ_")})), flush=True)
        return
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    normA = 6 * abs(cfg["hop"]) + float(eps.abs().max())
    G = (X.T @ X).cpu().numpy()
    out = dict(config=c, L=L, W=cfg["W"], seed=cfg["seed"], wall_s=dt,
               env={k: v for k, v in os.environ.items() if k.startswith("AJ_")}, setup_ms=st["setup_ms"],
               solve_ms=st["solve_ms"], outer=st["outer"], inner=st["inner_total"],
               levels=st["precond"]["levels"], coarse=st["precond"]["coarse_n"],
               tau_drop=st["precond"]["tau_drop"], tau_strong=st["precond"]["tau_strong"],
               tau_virtual=st["precond"]["tau_virtual"], nnz_V=st["precond"]["nnz_V"],
               tau_inv=st["precond"]["tau_inv"], nnz_L_dropped_inv=st["precond"]["nnz_L_dropped_inv"],
               nnzL_per_site=st["precond"]["nnz_L"] / L ** 3, eigenvalues=[float(v) for v in lam],
               resid_rel=[float(v) / normA for v in res], orth_err=float(np.abs(G - np.eye(len(lam))).max()))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
