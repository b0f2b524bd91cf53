"""Kernel-level driver for ncu / timing: disorder, stencil SpMV and one
preconditioner setup + applies at lattice size L (default 250).

python scripts/prof_kernels.py [L] [reps] [what] [seed]   what in {spmv, precond, all}
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_math_0508111_b200 import binding  # noqa: E402


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 250
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    what = sys.argv[3] if len(sys.argv) > 3 else "all"
    seed = int(sys.argv[4]) if len(sys.argv) > 4 else 4
    n = L ** 3
    eps = torch.empty(n, dtype=torch.float64, device="cuda")
    binding.anderson_build(eps, L, 16.5, seed)
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if what in ("spmv", "all"):
        for path in ("bal", "grid", "tma"):   # AJ_SPMV_PATH: the kernel variants (aj_stencil.cu)
            os.environ["AJ_SPMV_PATH"] = path
            binding.spmv(y, x, eps, L, -1.0, 0.0)
            e0.record(st)
            for _ in range(reps):
                binding.spmv(y, x, eps, L, -1.0, 0.0)
            e1.record(st)
            e1.synchronize()
            ms = e0.elapsed_time(e1) / reps
            print(f"spmv[{path}] L={L}: {ms:.4f} ms  {24 * n / ms / 1e6:.1f} GB/s", flush=True)
        os.environ.pop("AJ_SPMV_PATH", None)
    if what in ("precond", "all", "precond2"):
      for mode in (("register", "staged") if what == "precond2" else ("default",)):
        if mode == "staged":
            os.environ["AJ_APPLY_STAGED"] = "1"
        print(f"-- apply kernels: {mode}", flush=True)
        t0 = time.perf_counter()
        K = binding.Precond(eps, L, -1.0, 0.0)
        torch.cuda.synchronize()
        info = K.info()
        print(f"precond setup L={L}: {time.perf_counter() - t0:.2f} s levels {info['levels']} coarse {info['coarse_n']} "
              f"nnzL/site {info['nnz_L'] / n:.2f}", flush=True)
        K.apply(y, x)
        binding.prof_enable(True)
        e0.record(st)
        for _ in range(reps):
            K.apply(y, x)
        e1.record(st)
        e1.synchronize()
        p = binding.prof_get()["precond_apply"]
        binding.prof_enable(False)
        ms = e0.elapsed_time(e1) / reps
        by = p["bytes"] / max(1, p["calls"])
        print(f"precond apply L={L}: {ms:.4f} ms  {by / ms / 1e6:.1f} GB/s (bytes/apply {by:.3e})", flush=True)
        K.free()


if __name__ == "__main__":
    main()
