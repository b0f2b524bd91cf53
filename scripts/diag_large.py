"""Diagnostics for larger lattices: preconditioned SQMR iteration counts and a
verbose JD run. Writes incrementally to stdout (flush)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_math_0508111_b200 import binding  # noqa: E402


def sqmr_its(L, W=16.5, seed=2, tol=1e-8, **pk):
    n = L ** 3
    eps = torch.empty(n, dtype=torch.float64, device="cuda")
    binding.anderson_build(eps, L, W, seed)
    p = binding.default_precond_params(**pk)
    t0 = time.perf_counter()
    K = binding.Precond(eps, L, -1.0, 0.0, p)
    torch.cuda.synchronize()
    ts = time.perf_counter() - t0
    b = torch.randn(n, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    x, it, rel, brk = binding.sqmr_solve(K, x, b, eps, L, -1.0, 0.0, tol=tol, maxit=2000)
    r = torch.empty_like(b)
    binding.spmv(r, x, eps, L, -1.0, 0.0)
    true = float(torch.linalg.norm(r - b) / torch.linalg.norm(b))
    info = K.info()
    K.free()
    # apply time
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    print(f"L={L} {pk} setup {ts:.2f}s levels {info['levels']} coarse {info['coarse_n']} "
          f"nnzL/site {info['nnz_L'] / n:.1f} sqmr its {it} rel {rel:.2e} true {true:.2e} brk {brk}", flush=True)


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "sqmr"
    if mode == "grid":
        L = int(sys.argv[2])
        for td, ts in [(2e-3, 5e-3), (1e-3, 5e-3), (1e-3, 2e-3), (5e-4, 2e-3), (5e-4, 5e-3), (2.5e-4, 1e-3),
                       (2.5e-4, 2.5e-3)]:
            sqmr_its(L, tau_drop=td, tau_strong=ts, factor_fp32=0)
        return
    if mode == "grid2":
        L = int(sys.argv[2])
        for td, ts in [(5e-4, 1e-2), (5e-4, 2e-2), (2.5e-4, 1e-2), (2.5e-4, 2e-2), (1e-3, 2e-2)]:
            try:
                sqmr_its(L, tau_drop=td, tau_strong=ts, factor_fp32=0)
            except Exception as ex:
                print(L, td, ts, "failed", ex, flush=True)
        return
    if mode == "sqmr":
        for L in [50, 64, 80, 100]:
            sqmr_its(L)
        for td in [1e-3, 5e-4]:
            sqmr_its(100, tau_drop=td, tau_strong=10 * td)
        sqmr_its(100, factor_fp32=0)
    else:
        L = int(sys.argv[2])
        eps = torch.empty(L ** 3, dtype=torch.float64, device="cuda")
        binding.anderson_build(eps, L, 16.5, 2)
        jp = binding.default_jd_params(verbose=1, max_outer=int(sys.argv[3]) if len(sys.argv) > 3 else 200)
        try:
            lam, X, res, st = binding.jd_solve(5, 0.0, 1e-10, eps, L, -1.0, jparams=jp)
            print("JD ok", lam, st["outer"], st["inner_total"], flush=True)
        except Exception as ex:
            print("JD failed", ex, flush=True)


if __name__ == "__main__":
    main()
