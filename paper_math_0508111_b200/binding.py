"""Thin ctypes binding of libanderson_jd.so (include/anderson_jd.h).

Argument marshalling only: every step of the hot path runs in the CUDA
library.  Tensors are torch CUDA tensors (fp64, contiguous); the current torch
stream is passed through.  There is no CPU fallback: if the shared library or
a CUDA device is missing, every call raises.
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AJ_LIB") or os.path.join(HERE, "libanderson_jd.so")  # AJ_LIB: experiments only

AJ_OK, AJ_ERR_ARG, AJ_ERR_CUDA, AJ_ERR_BREAKDOWN, AJ_ERR_NOCONV, AJ_ERR_CAPACITY = range(6)

# every symbol include/anderson_jd.h declares (checked by tests/test_abi.py)
EXPORTS = ["aj_last_error", "aj_version", "anderson_build", "spmv", "anderson_build_slab", "spmv_slab",
           "aj_precond_default_params",
           "precond_setup", "precond_apply", "precond_info", "precond_free", "sqmr_solve", "multi_dot",
           "ortho_cgs2", "aj_jd_default_params", "jd_solve", "jd_solve_host", "aj_launch_count",
           "aj_prof_enable", "aj_prof_get", "aj_nccl_unique_id", "aj_comm_nccl_create", "aj_comm_nccl_free",
           "spmv_sharded", "precond_setup_slab", "jd_solve_sharded"]

PROF_CATS = ["spmv", "precond_apply", "precond_setup", "sqmr_update", "jd_subspace"]


class AJError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class PrecondParams(ctypes.Structure):
    _fields_ = [("kappa", ctypes.c_double), ("tau_drop", ctypes.c_double), ("tau_strong", ctypes.c_double),
                ("n_coarse_max", ctypes.c_int32), ("max_levels", ctypes.c_int32), ("stall_frac", ctypes.c_double),
                ("dense_cap", ctypes.c_int32), ("cand_cap", ctypes.c_int32), ("factor_fp32", ctypes.c_int32),
                ("compensate", ctypes.c_int32), ("tau_virtual", ctypes.c_double), ("tau_inv", ctypes.c_double),
                ("shard_precond", ctypes.c_int32)]


class PrecondInfo(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int32), ("coarse_n", ctypes.c_int32), ("nnz_L", ctypes.c_int64),
                ("nnz_A", ctypes.c_int64), ("level_n", ctypes.c_int32 * 1024), ("level_nF", ctypes.c_int32 * 1024),
                ("level_pairs", ctypes.c_int32 * 1024), ("level_nnzS", ctypes.c_int64 * 1024),
                ("setup_ms", ctypes.c_double), ("tau_drop", ctypes.c_double), ("tau_strong", ctypes.c_double),
                ("tau_virtual", ctypes.c_double), ("nnz_V", ctypes.c_int64), ("setup_products", ctypes.c_int64),
                ("setup_bytes", ctypes.c_double), ("tau_inv", ctypes.c_double), ("nnz_L_dropped_inv", ctypes.c_int64)]

    def as_dict(self):
        nl = self.levels
        return dict(levels=nl, coarse_n=self.coarse_n, nnz_L=self.nnz_L, nnz_A=self.nnz_A,
                    tau_drop=self.tau_drop, tau_strong=self.tau_strong, tau_virtual=self.tau_virtual,
                    nnz_V=self.nnz_V, setup_products=self.setup_products, setup_bytes=self.setup_bytes,
                    tau_inv=self.tau_inv, nnz_L_dropped_inv=self.nnz_L_dropped_inv,
                    level_n=list(self.level_n[:nl]), level_nF=list(self.level_nF[:nl]),
                    level_pairs=list(self.level_pairs[:nl]), level_nnzS=list(self.level_nnzS[:nl]),
                    setup_ms=self.setup_ms)


class JdParams(ctypes.Structure):
    _fields_ = [("jmin", ctypes.c_int32), ("jmax", ctypes.c_int32), ("max_outer", ctypes.c_int32),
                ("inner_max", ctypes.c_int32), ("inner_tol", ctypes.c_double), ("switch_tol", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("verbose", ctypes.c_int32)]


class JdStats(ctypes.Structure):
    _fields_ = [("outer", ctypes.c_int32), ("inner_total", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("restarts", ctypes.c_int32), ("setup_ms", ctypes.c_double), ("solve_ms", ctypes.c_double),
                ("total_ms", ctypes.c_double), ("precond", PrecondInfo)]

    def as_dict(self):
        return dict(outer=self.outer, inner_total=self.inner_total, converged=self.converged,
                    restarts=self.restarts, setup_ms=self.setup_ms, solve_ms=self.solve_ms,
                    total_ms=self.total_ms, precond=self.precond.as_dict())


class Prof(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 8), ("bytes", ctypes.c_double * 8), ("calls", ctypes.c_int64 * 8)]

    def as_dict(self):
        return {name: dict(ms=self.ms[i], bytes=self.bytes[i], calls=self.calls[i])
                for i, name in enumerate(PROF_CATS)}


_lib = None


def lib():
    """Load the CUDA library (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing -- run __graft_entry__.build(); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        vp, d, i32, i64, u64 = ctypes.c_void_p, ctypes.c_double, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        dp = ctypes.POINTER(ctypes.c_double)
        sig = {
            "aj_last_error": ([], ctypes.c_char_p), "aj_version": ([], ctypes.c_char_p),
            "anderson_build": ([vp, i32, d, u64, vp], ctypes.c_int),
            "spmv": ([vp, vp, vp, i32, d, d, vp], ctypes.c_int),
            "anderson_build_slab": ([vp, i32, i32, i32, d, u64, vp], ctypes.c_int),
            "spmv_slab": ([vp, vp, vp, i32, i32, d, d, vp], ctypes.c_int),
            "aj_precond_default_params": ([ctypes.POINTER(PrecondParams)], None),
            "precond_setup": ([ctypes.POINTER(vp), vp, i32, d, d, ctypes.POINTER(PrecondParams), vp], ctypes.c_int),
            "precond_apply": ([vp, vp, vp, vp], ctypes.c_int),
            "precond_info": ([vp, ctypes.POINTER(PrecondInfo)], ctypes.c_int),
            "precond_free": ([vp, vp], ctypes.c_int),
            "sqmr_solve": ([vp, vp, vp, vp, i32, d, d, d, i32, ctypes.POINTER(i32), dp, vp], ctypes.c_int),
            "multi_dot": ([dp, vp, i32, vp, i64, vp], ctypes.c_int),
            "ortho_cgs2": ([vp, vp, i32, i64, dp, vp], ctypes.c_int),
            "aj_jd_default_params": ([ctypes.POINTER(JdParams)], None),
            "jd_solve": ([i32, d, d, vp, i32, d, ctypes.POINTER(PrecondParams), ctypes.POINTER(JdParams), dp, vp, dp,
                          ctypes.POINTER(JdStats), vp], ctypes.c_int),
            "jd_solve_host": ([i32, d, d, dp, i32, d, ctypes.POINTER(PrecondParams), ctypes.POINTER(JdParams), dp,
                               dp, dp, ctypes.POINTER(JdStats), vp], ctypes.c_int),
            "aj_launch_count": ([i32], i64),
            "aj_prof_enable": ([i32], ctypes.c_int),
            "aj_prof_get": ([ctypes.POINTER(Prof)], ctypes.c_int),
            "aj_nccl_unique_id": ([ctypes.c_char_p, vp], ctypes.c_int),
            "aj_comm_nccl_create": ([vp, ctypes.c_char_p, vp, i32, i32], ctypes.c_int),
            "aj_comm_nccl_free": ([vp], ctypes.c_int),
            "spmv_sharded": ([vp, vp, vp, i32, i32, i32, d, d, vp, vp], ctypes.c_int),
            "precond_setup_slab": ([ctypes.POINTER(vp), vp, i32, i32, i32, i32, d, d, ctypes.POINTER(PrecondParams),
                                    vp], ctypes.c_int),
            "jd_solve_sharded": ([i32, d, d, vp, i32, i32, i32, d, ctypes.POINTER(PrecondParams),
                                  ctypes.POINTER(JdParams), dp, vp, dp, ctypes.POINTER(JdStats), vp, vp], ctypes.c_int),
        }
        for name, (argt, rest) in sig.items():
            f = getattr(L, name)
            f.argtypes = argt
            f.restype = rest
        _lib = L
    return _lib


def _check(rc):
    if rc != AJ_OK:
        raise AJError(rc, lib().aj_last_error().decode())


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    import torch
    assert isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous(), \
        "expected a contiguous fp64 CUDA tensor"
    return ctypes.c_void_p(t.data_ptr())


def version():
    return lib().aj_version().decode()


def default_precond_params(**kw):
    p = PrecondParams()
    lib().aj_precond_default_params(ctypes.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def default_jd_params(**kw):
    p = JdParams()
    lib().aj_jd_default_params(ctypes.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def anderson_build(eps, L, W, seed):
    _check(lib().anderson_build(_ptr(eps), L, W, seed, _stream()))
    return eps


def spmv(y, x, eps, L, hop, sigma=0.0):
    _check(lib().spmv(_ptr(y), _ptr(x), _ptr(eps), L, hop, sigma, _stream()))
    return y


def anderson_build_slab(eps, L, z0, nz, W, seed):
    """eps of planes [z0, z0 + nz) (z-slab shard), bit-identical to the full lattice's slice."""
    _check(lib().anderson_build_slab(_ptr(eps), L, z0, nz, W, seed, _stream()))
    return eps


def spmv_slab(y, x_ext, eps, L, nz, hop, sigma=0.0):
    """y = (A - sigma I) x on a slab; x_ext = [halo below | nz planes | halo above]."""
    _check(lib().spmv_slab(_ptr(y), _ptr(x_ext), _ptr(eps), L, nz, hop, sigma, _stream()))
    return y


class Precond:
    """Multilevel ILDL handle: precond_setup / precond_apply / precond_free.  With
    slab=(z0, nz, world): precond_setup_slab (the slab's diagonal block, DESIGN.md sect. 6)."""

    def __init__(self, eps, L, hop, sigma=0.0, params=None, slab=None):
        self.h = ctypes.c_void_p()
        p = params or default_precond_params()
        if slab is None:
            _check(lib().precond_setup(ctypes.byref(self.h), _ptr(eps), L, hop, sigma, ctypes.byref(p), _stream()))
            self.n = L ** 3
        else:
            z0, nz, world = slab
            _check(lib().precond_setup_slab(ctypes.byref(self.h), _ptr(eps), L, z0, nz, world, hop, sigma,
                                            ctypes.byref(p), _stream()))
            self.n = L * L * nz

    def apply(self, z, r):
        _check(lib().precond_apply(self.h, _ptr(z), _ptr(r), _stream()))
        return z

    def info(self):
        i = PrecondInfo()
        _check(lib().precond_info(self.h, ctypes.byref(i)))
        return i.as_dict()

    def free(self):
        if self.h:
            _check(lib().precond_free(self.h, _stream()))
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def precond_setup(eps, L, hop, sigma=0.0, params=None):
    return Precond(eps, L, hop, sigma, params)


def precond_apply(handle, z, r):
    return handle.apply(z, r)


def sqmr_solve(precond, x, b, eps, L, hop, sigma, tol=1e-10, maxit=1000):
    it = ctypes.c_int32()
    rr = ctypes.c_double()
    h = precond.h if precond is not None else None
    rc = lib().sqmr_solve(h, _ptr(x), _ptr(b), _ptr(eps), L, hop, sigma, tol, maxit, ctypes.byref(it),
                          ctypes.byref(rr), _stream())
    if rc not in (AJ_OK, AJ_ERR_BREAKDOWN):
        _check(rc)
    return x, it.value, rr.value, rc == AJ_ERR_BREAKDOWN


def multi_dot(V, m, x):
    import numpy as np
    out = np.zeros(m)
    _check(lib().multi_dot(out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _ptr(V), m, _ptr(x), x.numel(),
                           _stream()))
    return out


def ortho_cgs2(x, V, m):
    nrm = ctypes.c_double()
    vp = _ptr(V) if m > 0 else None
    _check(lib().ortho_cgs2(_ptr(x), vp, m, x.numel(), ctypes.byref(nrm), _stream()))
    return x, nrm.value


def jd_solve(k, sigma, tol, eps, L, hop, pparams=None, jparams=None, want_vectors=True):
    """k eigenpairs nearest sigma. Returns (lambda[k] np, X (n,k) torch or None, resid[k] np, stats dict)."""
    import numpy as np
    import torch
    lam = np.zeros(k)
    res = np.zeros(k)
    X = torch.empty((k, L ** 3), dtype=torch.float64, device=eps.device) if want_vectors else None
    st = JdStats()
    pp = pparams or default_precond_params()
    jp = jparams or default_jd_params()
    rc = lib().jd_solve(k, sigma, tol, _ptr(eps), L, hop, ctypes.byref(pp), ctypes.byref(jp),
                        lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _ptr(X) if X is not None else None,
                        res.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(st), _stream())
    _check(rc)
    return lam, (X.T if X is not None else None), res, st.as_dict()


def jd_solve_host(k, sigma, tol, eps_host, L, hop, pparams=None, jparams=None, X_host=None):
    """End-to-end call from host buffers (numpy fp64): eps in, eigenpairs out."""
    import numpy as np
    assert eps_host.dtype == np.float64 and eps_host.flags.c_contiguous
    lam = np.zeros(k)
    res = np.zeros(k)
    st = JdStats()
    pp = pparams or default_precond_params()
    jp = jparams or default_jd_params()
    dpt = ctypes.POINTER(ctypes.c_double)
    xp = X_host.ctypes.data_as(dpt) if X_host is not None else None
    rc = lib().jd_solve_host(k, sigma, tol, eps_host.ctypes.data_as(dpt), L, hop, ctypes.byref(pp),
                             ctypes.byref(jp), lam.ctypes.data_as(dpt), xp, res.ctypes.data_as(dpt),
                             ctypes.byref(st), _stream())
    _check(rc)
    return lam, res, st.as_dict()


def _comm_ptr(comm):
    return ctypes.cast(comm.ptr(), ctypes.c_void_p) if comm is not None else None


def spmv_sharded(y, x, eps, L, z0, nz, hop, sigma, comm):
    """y = (A - sigma I) x on this rank's z-slab, halos exchanged through `comm` (slab.py)."""
    _check(lib().spmv_sharded(_ptr(y), _ptr(x), _ptr(eps), L, z0, nz, hop, sigma, _comm_ptr(comm), _stream()))
    return y


def jd_solve_sharded(k, sigma, tol, eps, L, z0, nz, hop, comm, pparams=None, jparams=None, want_vectors=True):
    """jd_solve on a lattice sharded in z over the ranks of `comm` (slab.TorchComm / slab.NcclComm);
    eps and the returned X (nz L^2, k) are this rank's slab.  Collective."""
    import numpy as np
    import torch
    lam = np.zeros(k)
    res = np.zeros(k)
    X = torch.empty((k, L * L * nz), dtype=torch.float64, device=eps.device) if want_vectors else None
    st = JdStats()
    pp = pparams or default_precond_params()
    jp = jparams or default_jd_params()
    rc = lib().jd_solve_sharded(k, sigma, tol, _ptr(eps), L, z0, nz, hop, ctypes.byref(pp), ctypes.byref(jp),
                                lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _ptr(X) if X is not None else None,
                                res.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(st), _comm_ptr(comm),
                                _stream())
    _check(rc)
    return lam, (X.T if X is not None else None), res, st.as_dict()


def launch_count(reset=False):
    return lib().aj_launch_count(1 if reset else 0)


def prof_enable(on=True, categories=None):
    """Start/stop live per-phase timing; `categories` restricts it to the named
    phases (cheaper: the JD/SQMR vector kernels are thousands of tiny calls)."""
    if on and categories:
        mask = 0
        for c in categories:
            mask |= 1 << PROF_CATS.index(c)
        _check(lib().aj_prof_enable(ctypes.c_int32(-0x80000000 | mask).value))
    else:
        _check(lib().aj_prof_enable(1 if on else 0))


def prof_get():
    p = Prof()
    _check(lib().aj_prof_get(ctypes.byref(p)))
    return p.as_dict()
