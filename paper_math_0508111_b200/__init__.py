"""B200-native hot path of arxiv math/0508111 (Schenk, Bollhoefer, Roemer):
preconditioned shift-and-invert Jacobi-Davidson for interior eigenpairs of the
3D Anderson Hamiltonian.  The compute lives in libanderson_jd.so (CUDA,
sm_100a); `binding` is the thin ctypes layer with the C-ABI names.
"""
from . import binding  # noqa: F401
from .binding import (anderson_build, jd_solve, jd_solve_host, multi_dot, ortho_cgs2,  # noqa: F401
                      precond_apply, precond_setup, spmv, sqmr_solve)

__all__ = ["binding", "anderson_build", "spmv", "precond_setup", "precond_apply", "sqmr_solve", "multi_dot",
           "ortho_cgs2", "jd_solve", "jd_solve_host"]
