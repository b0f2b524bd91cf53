"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Tolerances (DESIGN.md sect. 5):
  disorder      bit-exact (integer hash -> exact double arithmetic)
  spmv          max|y - y_ref| <= 1e-14 * max|y_ref|          (BASELINE north_star)
  precond       same level structure; ||z - z_ref|| <= 1e-12 ||z_ref|| (APPLY_TOL)
  sqmr          converged to tol, true residual <= 10 tol
  multi_dot     <= 1e-13 relative
  jd_solve      |lambda - lambda_ref| <= 1e-10 ||A||, ||Ax - lambda x|| <= 1e-8 ||A||,
                subspace angles <= 1e-7 where Davis-Kahan allows it
"""
import json
import os

import numpy as np
import pytest

from inputs import CONFIGS, rand_vec
from oracle import anderson as an
from oracle import eigs, mlildl
from oracle.sqmr import sqmr as oracle_sqmr

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# preconditioner apply parity, relative 2-norm; the factor is the oracle's entry for entry,
# so the difference is the summation order of the gathers (DESIGN.md sect. 5).  Observed on
# the B200 (round 2, AJ_PARITY_LOG): median 1.3e-14, max 9.5e-14 over every case except the
# uncompensated W=21 L=11 factor (1.36e-12, a more ill-conditioned coarse inverse) -> ~10x.
APPLY_TOL = 1e-12
APPLY_TOL_ILLCOND = 1e-11


def _log_parity(name, case, err):
    """Observed errors, appended to $AJ_PARITY_LOG (JSON lines) when set."""
    path = os.environ.get("AJ_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"test": name, "case": str(case), "err": float(err)}) + "\n")


def T(x):
    import torch
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")


def N(t):
    import torch
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def gpu_eps(b, L, W, seed):
    import torch
    e = torch.empty(L ** 3, dtype=torch.float64, device="cuda")
    b.anderson_build(e, L, W, seed)
    return e


# ---------------------------------------------------------------- disorder
@pytest.mark.parametrize("L,W,seed", [(3, 16.5, 0), (10, 16.5, 0), (17, 12.0, 5), (50, 16.5, 1), (250, 21.0, 6)])
def test_disorder_bit_exact(gpu_lib, L, W, seed):
    e = N(gpu_eps(gpu_lib, L, W, seed))
    ref = an.disorder(L, W, seed)
    assert np.array_equal(e.view(np.uint64), ref.view(np.uint64))


# ---------------------------------------------------------------- spmv
@pytest.mark.parametrize("L", [3, 4, 10, 17, 33, 50, 64, 66, 98, 200, 250])
@pytest.mark.parametrize("hop,sigma", [(-1.0, 0.0), (1.0, 0.37)])
def test_spmv_parity(gpu_lib, L, hop, sigma):
    import torch
    eps = gpu_eps(gpu_lib, L, 16.5, 3)
    x = rand_vec(L ** 3, 11)
    y = torch.empty(L ** 3, dtype=torch.float64, device="cuda")
    gpu_lib.spmv(y, T(x), eps, L, hop, sigma)
    ref = an.stencil_apply(L, an.disorder(L, 16.5, 3), x, hop=hop, sigma=sigma)
    err = np.abs(N(y) - ref).max()
    assert err <= 1e-14 * np.abs(ref).max()


@pytest.mark.parametrize("L", [64, 66, 100, 250])
def test_spmv_kernel_variants_agree(gpu_lib, monkeypatch, L):
    # the balanced one-wave launch runs the same z-march as the tiled grid (bit for bit); the
    # TMA-staged kernel (bands of rows, ragged band heights, plane chunks) computes the same
    # sums in the same order, up to the compiler's fused multiply-adds
    import torch
    eps = gpu_eps(gpu_lib, L, 16.5, 2)
    x = T(rand_vec(L ** 3, 5))
    ys = {}
    for path in ("bal", "grid", "tma"):
        monkeypatch.setenv("AJ_SPMV_PATH", path)
        ys[path] = torch.empty_like(x)
        gpu_lib.spmv(ys[path], x, eps, L, -1.0, 0.11)
    assert torch.equal(ys["bal"], ys["grid"])
    assert torch.linalg.norm(ys["tma"] - ys["grid"]) <= 1e-15 * torch.linalg.norm(ys["grid"])


@pytest.mark.parametrize("L,world", [(12, 3), (17, 4), (64, 8)])
def test_slab_shards_match_full_lattice(gpu_lib, L, world):
    # row (e) building blocks in one process: each z-slab's disorder is the slice of the
    # full lattice bit for bit, and the slab stencil with its two halo planes (taken here
    # from the neighbours' planes, as the NCCL exchange delivers them) reproduces the
    # full SpMV on its planes
    import torch
    from paper_math_0508111_b200 import slab
    W, seed, hop, sigma = 16.5, 3, -1.0, 0.25
    P = L * L
    eps = gpu_eps(gpu_lib, L, W, seed)
    x = T(rand_vec(L ** 3, 4))
    y = torch.empty_like(x)
    gpu_lib.spmv(y, x, eps, L, hop, sigma)
    for r in range(world):
        z0, nz = slab.slab_bounds(L, r, world)
        es = torch.empty(nz * P, dtype=torch.float64, device="cuda")
        gpu_lib.anderson_build_slab(es, L, z0, nz, W, seed)
        assert torch.equal(es, eps[z0 * P:(z0 + nz) * P])
        planes = [(z0 - 1) % L] + list(range(z0, z0 + nz)) + [(z0 + nz) % L]
        xe = torch.cat([x[k * P:(k + 1) * P] for k in planes])
        ys = torch.empty(nz * P, dtype=torch.float64, device="cuda")
        gpu_lib.spmv_slab(ys, xe, es, L, nz, hop, sigma)
        ref = y[z0 * P:(z0 + nz) * P]
        assert torch.linalg.norm(ys - ref) <= 1e-14 * torch.linalg.norm(ref)


def test_spmv_sharded_single_rank(gpu_lib):
    # one rank: the halo exchange wraps periodically and spmv_sharded equals spmv
    import torch
    from paper_math_0508111_b200 import slab
    L = 10
    P = L * L
    eps = gpu_eps(gpu_lib, L, 16.5, 1)
    x = T(rand_vec(L ** 3, 2))
    y = torch.empty_like(x)
    gpu_lib.spmv(y, x, eps, L, -1.0, 0.0)
    xe = torch.zeros((L + 2) * P, dtype=torch.float64, device="cuda")
    xe[P:(L + 1) * P] = x
    ys = torch.empty_like(x)
    slab.spmv_sharded_ext(ys, xe, eps, L, L, -1.0, 0.0)
    assert torch.linalg.norm(ys - y) <= 1e-14 * torch.linalg.norm(y)


def test_spmv_plane_wave_gpu(gpu_lib):
    # closed form independent of the oracle: plane wave eigenfunction of the clean stencil
    import torch
    L = 12
    eps = torch.zeros(L ** 3, dtype=torch.float64, device="cuda")
    s = np.arange(L ** 3)
    i, j, k = s % L, (s // L) % L, s // (L * L)
    kv = 2 * np.pi * np.array([1, 3, 5]) / L
    x = np.cos(kv[0] * i + kv[1] * j + kv[2] * k + 0.2)
    y = torch.empty_like(eps)
    gpu_lib.spmv(y, T(x), eps, L, -1.0, 0.0)
    lam = -2 * np.cos(kv).sum()
    assert np.abs(N(y) - lam * x).max() < 1e-13


# ---------------------------------------------------------------- preconditioner
def resolved(p, L):
    """DESIGN.md R12 auto rule for negative drop parameters: the paper's eps/kappa,
    eps = 1/sqrt(N)."""
    td = p.tau_drop if p.tau_drop >= 0 else 1.0 / (p.kappa * np.sqrt(float(L) ** 3))
    if p.tau_strong >= 0:
        ts = p.tau_strong
    else:
        ts = min(0.05, 40 * td) if p.compensate else 10 * td
    return td, ts


def _oracle_precond(L, eps, hop, sigma, p):
    A = an.matrix(L, eps, hop=hop, sigma=sigma)
    td, ts = resolved(p, L)
    return mlildl.MultilevelILDL(A, lattice_L=L, kappa=p.kappa, tau_drop=td, tau_strong=ts,
                                 n_coarse_max=p.n_coarse_max, max_levels=p.max_levels, stall_frac=p.stall_frac,
                                 dense_cap=p.dense_cap, factor_fp32=bool(p.factor_fp32),
                                 compensate=bool(p.compensate), tau_inv=p.tau_inv)


@pytest.mark.parametrize("fp32,comp", [(0, 1), (1, 1), (0, 0)])
@pytest.mark.parametrize("L,W,seed,hop,sigma", [(8, 16.5, 1, -1.0, 0.0), (12, 16.5, 2, -1.0, 0.0),
                                                (16, 12.0, 3, 1.0, 0.25), (11, 21.0, 4, -1.0, 0.0),
                                                (20, 16.5, 5, -1.0, 0.0), (24, 16.5, 6, -1.0, 0.0)])
def test_precond_parity(gpu_lib, L, W, seed, hop, sigma, fp32, comp):
    import torch
    p = gpu_lib.default_precond_params(n_coarse_max=200, factor_fp32=fp32, compensate=comp)
    eps_g = gpu_eps(gpu_lib, L, W, seed)
    K = gpu_lib.Precond(eps_g, L, hop, sigma, p)
    info = K.info()
    assert (info["tau_drop"], info["tau_strong"]) == resolved(p, L)
    eps = an.disorder(L, W, seed)
    M = _oracle_precond(L, eps, hop, sigma, p)
    # identical multilevel structure (decisions taken on the same fp64 values)
    assert info["levels"] == len(M.levels)
    assert info["level_n"] == [lv.n for lv in M.levels]
    assert info["level_nF"] == [len(lv.F) for lv in M.levels]
    assert info["level_pairs"] == [lv.npairs for lv in M.levels]
    assert info["coarse_n"] == M.coarse_n
    assert info["level_nnzS"] == [lv.S.nnz for lv in M.levels]
    assert info["nnz_L"] == sum(lv.L.nnz for lv in M.levels)
    assert info["nnz_V"] == sum(lv.nvirtual for lv in M.levels)
    assert info["tau_virtual"] == (5.0 * info["tau_drop"] if comp else 0.0)
    for s in (21, 22):
        r = rand_vec(L ** 3, s)
        z = torch.empty(L ** 3, dtype=torch.float64, device="cuda")
        K.apply(z, T(r))
        zr = M.apply(r)
        err = np.linalg.norm(N(z) - zr) / np.linalg.norm(zr)
        _log_parity("precond", (L, W, seed, fp32, comp), err)
        assert err <= (APPLY_TOL_ILLCOND if (W, comp) == (21.0, 0) else APPLY_TOL), err
    K.free()


@pytest.mark.parametrize("tau_inv", [0.1, 0.5])
@pytest.mark.parametrize("L,W,seed", [(12, 16.5, 2), (20, 16.5, 5), (16, 12.0, 3)])
def test_precond_inverse_dropping_parity(gpu_lib, L, W, seed, tau_inv):
    # inverse-based dropping a posteriori (reading R18): the same entries
    # removed as by the oracle (its nu estimates summed in the same order), apply parity
    import torch
    p = gpu_lib.default_precond_params(n_coarse_max=200, tau_inv=tau_inv)
    eps_g = gpu_eps(gpu_lib, L, W, seed)
    K = gpu_lib.Precond(eps_g, L, -1.0, 0.0, p)
    info = K.info()
    M = _oracle_precond(L, an.disorder(L, W, seed), -1.0, 0.0, p)
    assert info["levels"] == len(M.levels)
    assert info["nnz_L"] == sum(lv.L.nnz for lv in M.levels)
    assert info["nnz_L_dropped_inv"] == sum(lv.ndrop_inv for lv in M.levels) > 0
    for s_ in (21, 22):
        r = rand_vec(L ** 3, s_)
        z = torch.empty(L ** 3, dtype=torch.float64, device="cuda")
        K.apply(z, T(r))
        zr = M.apply(r)
        err = np.linalg.norm(N(z) - zr) / np.linalg.norm(zr)
        _log_parity("precond_inv", (L, W, seed, tau_inv), err)
        assert err <= APPLY_TOL, err
    K.free()


@pytest.fixture(scope="module")
def oracle_l48(gpu_lib):
    """The oracle factor of configs[1]'s workload at L=48 (n = 110,592) with the production
    (auto, size-scaled) parameters, built once (~2 min of CPU) for the variant tests."""
    L, W, seed = 48, 16.5, 1
    p = gpu_lib.default_precond_params()
    M = _oracle_precond(L, an.disorder(L, W, seed), -1.0, 0.0, p)
    rs = [rand_vec(L ** 3, s) for s in (31, 32)]
    return dict(L=L, W=W, seed=seed, p=p, M=M, rs=rs, zs=[M.apply(r) for r in rs])


@pytest.mark.parametrize("variant", [{}, {"AJ_PER_LANE": "8"}, {"AJ_PER_LANE": "2"}, {"AJ_SCHUR_TIER": "2"},
                                     {"AJ_SCHUR_TIER": "3"}, {"AJ_SCHUR_TIER": "4"}, {"AJ_SCHUR_TIER": "5"},
                                     {"AJ_FORCE_GB": "64"}, {"AJ_FORCE_GB": "256"}, {"AJ_GJ_STEPS": "1"},
                                     {"AJ_GJ_UNBLOCKED": "1"},
                                     {"AJ_APPLY_STAGED": "1"}, {"AJ_APPLY_STAGED": "1", "AJ_FORCE_GB": "128"},
                                     {"AJ_APPLY_RING": "1", "AJ_RING_MIN": "1"},
                                     {"AJ_APPLY_RING": "1", "AJ_RING_MIN": "100000", "AJ_APPLY_RING_BWD": "0"}])
def test_precond_parity_production_l48(gpu_lib, monkeypatch, oracle_l48, variant):
    # GPU vs ORACLE at a size spanning many tiles (24 levels, coarse ~900) with the production
    # parameters, once with the routed default and once with each kernel variant forced
    # (row-group lanes, every Schur tier, CTA-per-row backward, the swap-based coarse inverse,
    # the bulk-copy staged substitution kernels, the opt-in persistent ring kernels on every
    # level / forward only on the larger levels)
    import torch
    o = oracle_l48
    for k, v in variant.items():
        monkeypatch.setenv(k, v)
    L, M = o["L"], o["M"]
    K = gpu_lib.Precond(gpu_eps(gpu_lib, L, o["W"], o["seed"]), L, -1.0, 0.0, o["p"])
    info = K.info()
    assert info["levels"] == len(M.levels) and info["levels"] > 10
    assert info["level_n"] == [lv.n for lv in M.levels]
    assert info["level_nF"] == [len(lv.F) for lv in M.levels]
    assert info["level_pairs"] == [lv.npairs for lv in M.levels]
    assert info["level_nnzS"] == [lv.S.nnz for lv in M.levels]
    assert info["nnz_L"] == sum(lv.L.nnz for lv in M.levels)
    assert info["nnz_V"] == sum(lv.nvirtual for lv in M.levels)
    assert info["coarse_n"] == M.coarse_n
    for r, zr in zip(o["rs"], o["zs"]):
        z = torch.empty(L ** 3, dtype=torch.float64, device="cuda")
        K.apply(z, T(r))
        err = np.linalg.norm(N(z) - zr) / np.linalg.norm(zr)
        _log_parity("precond_l48", variant, err)
        assert err <= APPLY_TOL, err
    K.free()


@pytest.mark.parametrize("tier", [1, 2, 3, 4, 5])
def test_precond_schur_tiers_agree(gpu_lib, monkeypatch, tier):
    # every Schur tier (1: warp / 2048 table, 2: 64 threads / 4096, 3: 128 / 8192, 4: CTA / 16384,
    # 5: CTA / global-memory table) computes the same level structure and the same factor,
    # bit for bit, as the routed default
    import torch
    L = 16
    p = gpu_lib.default_precond_params(n_coarse_max=200)
    eps_g = gpu_eps(gpu_lib, L, 16.5, 5)
    r = T(rand_vec(L ** 3, 4))
    K1 = gpu_lib.Precond(eps_g, L, -1.0, 0.0, p)
    z1 = torch.empty_like(r)
    K1.apply(z1, r)
    i1 = K1.info()
    K1.free()
    monkeypatch.setenv("AJ_SCHUR_TIER", str(tier))
    K2 = gpu_lib.Precond(eps_g, L, -1.0, 0.0, p)
    z2 = torch.empty_like(r)
    K2.apply(z2, r)
    i2 = K2.info()
    K2.free()
    for key in ("levels", "level_n", "level_nF", "level_pairs", "level_nnzS", "nnz_L", "nnz_V", "coarse_n"):
        assert i1[key] == i2[key], key
    assert torch.equal(z1, z2)


def test_precond_backward_group_sizes_agree(gpu_lib, monkeypatch):
    # the backward kernel's row-group size (1 lane ... a whole CTA per L^T row) only
    # changes the summation order
    import torch
    L = 16
    eps_g = gpu_eps(gpu_lib, L, 16.5, 7)
    r = T(rand_vec(L ** 3, 6))
    zs = {}
    for gb in (None, 1, 32, 64, 128, 256):
        if gb is None:
            monkeypatch.delenv("AJ_FORCE_GB", raising=False)
        else:
            monkeypatch.setenv("AJ_FORCE_GB", str(gb))
        K = gpu_lib.Precond(eps_g, L, -1.0, 0.0, gpu_lib.default_precond_params(n_coarse_max=200))
        z = torch.empty_like(r)
        K.apply(z, r)
        K.free()
        zs[gb] = z
    for gb, z in zs.items():
        assert torch.linalg.norm(z - zs[None]) <= 1e-13 * torch.linalg.norm(zs[None]), gb


@pytest.mark.parametrize("L,ncmax", [(14, 600), (16, 1500)])
def test_coarse_inverse_paths_agree(gpu_lib, monkeypatch, L, ncmax):
    # the coarse inverse three ways: blocked Gauss-Jordan (default, panels of 32 columns,
    # rank-32 updates), one launch per column with implicit pivoting (AJ_GJ_UNBLOCKED) and
    # the swap-based two-launch reference (AJ_GJ_STEPS).  The last two run the same
    # per-element arithmetic (bit for bit); the blocked one sums each panel's updates in a
    # different order (agreement to rounding; ragged last panel when coarse_n % 32 != 0)
    import torch
    eps_g = gpu_eps(gpu_lib, L, 16.5, 3)
    r = T(rand_vec(L ** 3, 8))
    zs = {}
    for mode in ("blocked", "unblocked", "steps"):
        monkeypatch.delenv("AJ_GJ_UNBLOCKED", raising=False)
        monkeypatch.delenv("AJ_GJ_STEPS", raising=False)
        if mode == "unblocked":
            monkeypatch.setenv("AJ_GJ_UNBLOCKED", "1")
        if mode == "steps":
            monkeypatch.setenv("AJ_GJ_STEPS", "1")
        K = gpu_lib.Precond(eps_g, L, -1.0, 0.0, gpu_lib.default_precond_params(n_coarse_max=ncmax))
        assert K.info()["coarse_n"] > 100
        z = torch.empty_like(r)
        K.apply(z, r)
        K.free()
        zs[mode] = z
    assert torch.equal(zs["unblocked"], zs["steps"])
    assert torch.linalg.norm(zs["blocked"] - zs["steps"]) <= 1e-12 * torch.linalg.norm(zs["steps"])


def test_coarse_inverse_blocked_vs_numpy(gpu_lib):
    # the blocked dense inverse against numpy on the oracle's own coarse Schur complement:
    # the GPU apply of a level-free preconditioner (n_coarse_max >= n: the whole matrix is
    # the coarse block) is (A - sigma I)^{-1} r
    import torch
    L = 10
    eps = an.disorder(L, 16.5, 5)
    p = gpu_lib.default_precond_params(n_coarse_max=L ** 3, dense_cap=L ** 3)
    K = gpu_lib.Precond(gpu_eps(gpu_lib, L, 16.5, 5), L, -1.0, 0.3, p)
    assert K.info()["levels"] == 0 and K.info()["coarse_n"] == L ** 3
    r = rand_vec(L ** 3, 9)
    z = torch.empty(L ** 3, dtype=torch.float64, device="cuda")
    K.apply(z, T(r))
    K.free()
    A = an.matrix(L, eps, hop=-1.0, sigma=0.3).toarray()
    zr = np.linalg.solve(A, r)
    assert np.linalg.norm(N(z) - zr) <= 1e-10 * np.linalg.norm(zr)


def test_precond_exactness_limit_gpu(gpu_lib):
    # no dropping, no kappa bound, true independent sets -> K^{-1} = (A - sigma I)^{-1}
    import torch
    L = 6
    p = gpu_lib.default_precond_params(kappa=1e300, tau_drop=0.0, tau_strong=0.0, n_coarse_max=10, stall_frac=0.0,
                                       factor_fp32=0)
    eps = gpu_eps(gpu_lib, L, 16.5, 1)
    K = gpu_lib.Precond(eps, L, -1.0, 0.0, p)
    x = T(rand_vec(L ** 3, 3))
    ax = torch.empty_like(x)
    gpu_lib.spmv(ax, x, eps, L, -1.0, 0.0)
    z = torch.empty_like(x)
    K.apply(z, ax)
    assert torch.linalg.norm(z - x) <= 1e-10 * torch.linalg.norm(x)
    K.free()


@pytest.mark.parametrize("L", [20, 100])
def test_precond_symmetric_gpu(gpu_lib, L):
    # K^{-1} is symmetric at any size (L=100: production parameters, 66 levels, the
    # Schur tiers 2a/2b in use) -- a property the oracle cannot check at that size
    import torch
    eps = gpu_eps(gpu_lib, L, 16.5, 9)
    K = gpu_lib.Precond(eps, L, -1.0, 0.0)
    r1, r2 = T(rand_vec(L ** 3, 1)), T(rand_vec(L ** 3, 2))
    z1, z2 = torch.empty_like(r1), torch.empty_like(r1)
    K.apply(z1, r1)
    K.apply(z2, r2)
    a, b = float(r2 @ z1), float(r1 @ z2)
    scale = float(torch.linalg.norm(r1)) * max(float(torch.linalg.norm(z1)), float(torch.linalg.norm(z2)))
    assert abs(a - b) <= 1e-10 * max(abs(a), abs(b)) or abs(a - b) <= 1e-13 * scale
    K.free()


# ---------------------------------------------------------------- SQMR
@pytest.mark.parametrize("L,sigma", [(10, 0.0), (14, 0.5)])
def test_sqmr_parity(gpu_lib, L, sigma):
    import torch
    hop = -1.0
    p = gpu_lib.default_precond_params(n_coarse_max=200)
    eps_g = gpu_eps(gpu_lib, L, 16.5, 1)
    K = gpu_lib.Precond(eps_g, L, hop, sigma, p)
    b = rand_vec(L ** 3, 5)
    x = torch.empty(L ** 3, dtype=torch.float64, device="cuda")
    x, it, rel, brk = gpu_lib.sqmr_solve(K, x, T(b), eps_g, L, hop, sigma, tol=1e-10, maxit=300)
    assert not brk and rel <= 1e-10
    eps = an.disorder(L, 16.5, 1)
    A = an.matrix(L, eps, hop=hop, sigma=sigma)
    xr = N(x)
    assert np.linalg.norm(A @ xr - b) <= 1e-9 * np.linalg.norm(b)
    M = _oracle_precond(L, eps, hop, sigma, p)
    xo, ito, relo, _ = oracle_sqmr(lambda v: A @ v, M.apply, b, tol=1e-10, maxit=300)
    assert abs(it - ito) <= 2
    assert np.linalg.norm(xr - xo) <= 1e-8 * np.linalg.norm(xo)
    K.free()


def test_sqmr_unpreconditioned_gpu(gpu_lib):
    import torch
    L, hop, sigma = 6, -1.0, 3.0
    eps_g = gpu_eps(gpu_lib, L, 2.0, 1)
    b = rand_vec(L ** 3, 5)
    x = torch.empty(L ** 3, dtype=torch.float64, device="cuda")
    x, it, rel, brk = gpu_lib.sqmr_solve(None, x, T(b), eps_g, L, hop, sigma, tol=1e-12, maxit=500)
    A = an.matrix(L, an.disorder(L, 2.0, 1), hop=hop, sigma=sigma)
    ref = np.linalg.solve(A.toarray(), b)
    assert np.linalg.norm(N(x) - ref) <= 1e-9 * np.linalg.norm(ref)


# ---------------------------------------------------------------- tall-skinny
def test_multi_dot_and_ortho(gpu_lib):
    import torch
    n, m = 100_003, 19
    Vh = np.random.default_rng(1).standard_normal((m, n))
    xh = rand_vec(n, 2)
    V = T(Vh)
    x = T(xh)
    out = gpu_lib.multi_dot(V, m, x)
    ref = Vh @ xh
    assert np.abs(out - ref).max() <= 1e-13 * np.abs(ref).max() * np.sqrt(n)
    Q, _ = np.linalg.qr(Vh.T)
    Qg = T(Q.T)
    x2, nrm = gpu_lib.ortho_cgs2(x.clone(), Qg, m)
    xr = N(x2)
    assert np.abs(Q.T @ xr).max() <= 1e-13
    assert abs(np.linalg.norm(xr) - 1.0) <= 1e-13
    proj = xh - Q @ (Q.T @ xh)
    assert abs(nrm - np.linalg.norm(proj)) <= 1e-12 * np.linalg.norm(proj)


# ---------------------------------------------------------------- Jacobi-Davidson
def _check_eigs(L, W, seed, hop, lam, X, res, lam_ref, X_ref, normA, angle_tol=None, gap=None):
    assert np.all(np.abs(np.sort(lam) - np.sort(lam_ref)) <= 1e-10 * normA), (lam, lam_ref)
    assert np.all(res <= 1e-8 * normA)
    # recompute residuals with the oracle stencil
    eps = an.disorder(L, W, seed)
    for i in range(len(lam)):
        r = an.stencil_apply(L, eps, X[:, i], hop=hop) - lam[i] * X[:, i]
        assert np.linalg.norm(r) <= 1e-8 * normA
    G = X.T @ X
    assert np.abs(G - np.eye(len(lam))).max() <= 1e-8
    if angle_tol is not None:
        oi = np.argsort(lam)
        orf = np.argsort(lam_ref)
        for a, b in zip(oi, orf):
            c = abs(X[:, a] @ X_ref[:, b])
            ang = np.arccos(min(1.0, c))
            assert ang <= angle_tol, ang


def test_jd_config0(gpu_lib):
    cfg = CONFIGS[0]
    L, W, seed, hop, k = cfg["L"], cfg["W"], cfg["seed"], cfg["hop"], cfg["k"]
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "eigs_config0.json")))
    eps = gpu_eps(gpu_lib, L, W, seed)
    # tol 1e-12 so that Davis-Kahan (angle <= ||r|| / gap) certifies 1e-7 angles
    lam, X, res, st = gpu_lib.jd_solve(k, 0.0, 1e-12, eps, L, hop)
    A = an.matrix(L, an.disorder(L, W, seed), hop=hop)
    lr, Xr = eigs.dense_nearest(A, k, 0.0)
    assert np.allclose(lr, gold["eigenvalues"], rtol=0, atol=1e-13)
    normA = 6 + np.abs(an.disorder(L, W, seed)).max()
    _check_eigs(L, W, seed, hop, lam, N(X), res, lr, Xr, normA, angle_tol=1e-7)
    assert st["converged"] == k


@pytest.mark.parametrize("L,W,seed,hop,sigma,k", [(8, 16.5, 1, 1.0, 0.0, 5), (11, 12.0, 2, -1.0, 0.5, 3),
                                                  (12, 21.0, 3, -1.0, -1.0, 1), (6, 16.5, 4, -1.0, 0.0, 4)])
def test_jd_variants(gpu_lib, L, W, seed, hop, sigma, k):
    eps = gpu_eps(gpu_lib, L, W, seed)
    lam, X, res, st = gpu_lib.jd_solve(k, sigma, 1e-11, eps, L, hop)
    A = an.matrix(L, an.disorder(L, W, seed), hop=hop)
    lr, Xr = eigs.dense_nearest(A, k, sigma)
    normA = 6 + np.abs(an.disorder(L, W, seed)).max()
    _check_eigs(L, W, seed, hop, lam, N(X), res, lr, Xr, normA)


def test_jd_config1_l50(gpu_lib):
    path = os.path.join(ROOT, "tests", "golden", "eigs_config1.json")
    if not os.path.exists(path):
        pytest.fail("golden file for config 1 missing (scripts/make_golden.py 1)")
    gold = json.load(open(path))
    cfg = CONFIGS[1]
    L, W, seed, hop, k = cfg["L"], cfg["W"], cfg["seed"], cfg["hop"], cfg["k"]
    eps = gpu_eps(gpu_lib, L, W, seed)
    lam, X, res, st = gpu_lib.jd_solve(k, 0.0, cfg["tol"], eps, L, hop)
    normA = 6 + np.abs(an.disorder(L, W, seed)).max()
    lr = np.array(gold["eigenvalues"][:k])
    assert np.all(np.abs(np.sort(lam) - np.sort(lr)) <= 1e-10 * normA), (lam, lr)
    assert np.all(res <= 1e-8 * normA)
    Xh = N(X)
    e = an.disorder(L, W, seed)
    for i in range(k):
        r = an.stencil_apply(L, e, Xh[:, i], hop=hop) - lam[i] * Xh[:, i]
        assert np.linalg.norm(r) <= 1e-8 * normA


def test_jd_config1_l50_subspace_angles(gpu_lib):
    # configs[1] eigenVECTORS against the oracle golden (tests/golden/eigvecs_config1.npz,
    # plain SI-Lanczos, residuals ~1e-14): the north star's angle bound 1e-7.  Davis-Kahan:
    # angle_i <= ||r_i|| / gap_i; with gaps ~4e-5 near E=0 at L=50 the solve runs to
    # tol 2e-13 (||r|| <= 2.9e-12) so that the bound certifies 1e-7.
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "eigs_config1.json")))
    Xg = np.load(os.path.join(ROOT, "tests", "golden", gold["eigenvectors"]))["X"]   # (k, n)
    cfg = CONFIGS[1]
    L, W, seed, hop, k = cfg["L"], cfg["W"], cfg["seed"], cfg["hop"], cfg["k"]
    eps = gpu_eps(gpu_lib, L, W, seed)
    lam, X, res, st = gpu_lib.jd_solve(k, 0.0, 2e-13, eps, L, hop)
    Xh = N(X)
    lg = np.array(gold["eigenvalues"])          # the k + 3 nearest sigma = 0, ascending |lambda|
    normA = 6 + np.abs(an.disorder(L, W, seed)).max()
    assert np.all(np.abs(np.sort(lam) - np.sort(lg[:k])) <= 1e-10 * normA)
    for i in range(k):
        j = int(np.argmin(np.abs(lg[:k] - lam[i])))
        gap = np.min(np.abs(np.delete(lg, j) - lg[j]))
        # angle via the chordal distance 2 sin(angle/2) of the unit vectors (arccos of the
        # cosine loses all digits below ~1e-8)
        sgn = 1.0 if float(Xh[:, i] @ Xg[j]) >= 0 else -1.0
        ang = 2 * np.arcsin(min(1.0, np.linalg.norm(Xh[:, i] / np.linalg.norm(Xh[:, i]) - sgn * Xg[j]) / 2))
        bound = res[i] / gap
        assert bound <= 1e-7, (i, bound)            # the certificate itself
        assert ang <= 1e-7, (i, ang, bound)
        assert ang <= 2 * bound + 1e-9, (i, ang, bound)


def test_jd_host_e2e(gpu_lib):
    L, W, seed, hop = 10, 16.5, 0, -1.0
    eps = an.disorder(L, W, seed)
    Xh = np.zeros((5, L ** 3))
    lam, res, st = gpu_lib.jd_solve_host(5, 0.0, 1e-10, eps, L, hop, X_host=Xh)
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "eigs_config0.json")))
    normA = 6 + np.abs(eps).max()
    assert np.all(np.abs(np.sort(lam) - np.sort(gold["eigenvalues"])) <= 1e-10 * normA)
    for i in range(5):
        r = an.stencil_apply(L, eps, Xh[i], hop=hop) - lam[i] * Xh[i]
        assert np.linalg.norm(r) <= 1e-8 * normA


def test_jd_config2_l100_properties(gpu_lib):
    # BASELINE configs[2] at full size (n = 10^6): properties that hold at any size --
    # residuals recomputed with the oracle stencil, orthonormality, Rayleigh quotients,
    # and the same 5 eigenvalues from two independent start vectors.
    cfg = CONFIGS[2]
    L, W, seed, hop, k = cfg["L"], cfg["W"], cfg["seed"], cfg["hop"], cfg["k"]
    eps = gpu_eps(gpu_lib, L, W, seed)
    e = an.disorder(L, W, seed)
    normA = 6 + np.abs(e).max()
    lam1, X1, res1, st1 = gpu_lib.jd_solve(k, 0.0, cfg["tol"], eps, L, hop)
    Xh = N(X1)
    for i in range(k):
        ax = an.stencil_apply(L, e, Xh[:, i], hop=hop)
        assert np.linalg.norm(ax - lam1[i] * Xh[:, i]) <= 1e-8 * normA
        assert abs(Xh[:, i] @ ax - lam1[i]) <= 1e-10 * normA
    assert np.abs(Xh.T @ Xh - np.eye(k)).max() <= 1e-8
    jp = gpu_lib.default_jd_params(seed=12345)
    lam2, X2, res2, st2 = gpu_lib.jd_solve(k, 0.0, cfg["tol"], eps, L, hop, jparams=jp)
    assert np.allclose(np.sort(lam1), np.sort(lam2), atol=1e-10 * normA)


def test_jd_config4_l250_properties(gpu_lib):
    # BASELINE configs[4] at full size (n = 15,625,000, W = 16.5, seed 4) on one GPU, the
    # north star's target lattice: residuals recomputed with the oracle stencil, Rayleigh
    # quotients, orthonormality, interior eigenvalues (~1 min of GPU time)
    cfg = CONFIGS[4]
    L, W, seed, hop, k = cfg["L"], 16.5, 4, cfg["hop"], cfg["k"]
    assert L == 250
    eps = gpu_eps(gpu_lib, L, W, seed)
    e = an.disorder(L, W, seed)
    normA = 6 + np.abs(e).max()
    lam, X, res, st = gpu_lib.jd_solve(k, 0.0, cfg["tol"], eps, L, hop)
    Xh = N(X)
    for i in range(k):
        ax = an.stencil_apply(L, e, Xh[:, i], hop=hop)
        assert np.linalg.norm(ax - lam[i] * Xh[:, i]) <= 1e-8 * normA
        assert abs(Xh[:, i] @ ax - lam[i]) <= 1e-10 * normA
        assert res[i] <= 1e-8 * normA
    assert np.abs(Xh.T @ Xh - np.eye(k)).max() <= 1e-8
    assert np.abs(lam).max() < 1e-4   # interior: the level spacing near 0 at n = 1.6e7 is ~5e-7


def test_jd_config4_w12_l100_properties(gpu_lib):
    # BASELINE configs[4]'s hardest disorder, W = 12 (seed 4), at L = 100 (Table 4,
    # l.1235-1237: JD + ILUPACK at W=12 up to M=130): the independent-set levels densify and
    # stall on a coarse block of ~12.7k unknowns, inverted densely (blocked Gauss-Jordan) under
    # the default dense_cap.  Size-independent properties against the oracle stencil.
    cfg = CONFIGS[4]
    L, W, seed, hop, k = 100, 12.0, 4, cfg["hop"], cfg["k"]
    eps = gpu_eps(gpu_lib, L, W, seed)
    e = an.disorder(L, W, seed)
    normA = 6 + np.abs(e).max()
    lam, X, res, st = gpu_lib.jd_solve(k, 0.0, cfg["tol"], eps, L, hop)
    assert st["precond"]["coarse_n"] > 4096   # the stalled, densely inverted coarse block
    Xh = N(X)
    for i in range(k):
        ax = an.stencil_apply(L, e, Xh[:, i], hop=hop)
        assert np.linalg.norm(ax - lam[i] * Xh[:, i]) <= 1e-8 * normA
        assert abs(Xh[:, i] @ ax - lam[i]) <= 1e-10 * normA
        assert res[i] <= 1e-8 * normA
    assert np.abs(Xh.T @ Xh - np.eye(k)).max() <= 1e-8
    assert np.abs(lam).max() < 1e-3


def test_jd_config3_l200_properties(gpu_lib):
    # BASELINE configs[3] at full size (n = 8*10^6) on one GPU: residuals recomputed with
    # the oracle stencil (north-star bounds: ||Ax - lambda x|| <= 1e-8 ||A||), Rayleigh
    # quotients, orthonormality, eigenvalues inside the Gershgorin interval near sigma
    cfg = CONFIGS[3]
    L, W, seed, hop, k = cfg["L"], cfg["W"], cfg["seed"], cfg["hop"], cfg["k"]
    eps = gpu_eps(gpu_lib, L, W, seed)
    e = an.disorder(L, W, seed)
    normA = 6 + np.abs(e).max()
    lam, X, res, st = gpu_lib.jd_solve(k, 0.0, cfg["tol"], eps, L, hop)
    Xh = N(X)
    for i in range(k):
        ax = an.stencil_apply(L, e, Xh[:, i], hop=hop)
        assert np.linalg.norm(ax - lam[i] * Xh[:, i]) <= 1e-8 * normA
        assert abs(Xh[:, i] @ ax - lam[i]) <= 1e-10 * normA
        assert res[i] <= 1e-8 * normA
    assert np.abs(Xh.T @ Xh - np.eye(k)).max() <= 1e-8
    assert np.abs(lam).max() < 1e-3   # interior: the level spacing near 0 at n = 8e6 is ~1e-6


def test_sqmr_graph_path_agrees(gpu_lib, monkeypatch):
    # the optional captured SQMR step (AJ_SQMR_GRAPH=1) runs the same arithmetic
    import torch
    L, hop, sigma = 12, -1.0, 0.0
    eps = gpu_eps(gpu_lib, L, 16.5, 3)
    K = gpu_lib.Precond(eps, L, hop, sigma)
    b = T(rand_vec(L ** 3, 6))
    x1 = torch.empty_like(b)
    _, it1, rel1, _ = gpu_lib.sqmr_solve(K, x1, b, eps, L, hop, sigma, tol=1e-10, maxit=200)
    monkeypatch.setenv("AJ_SQMR_GRAPH", "1")
    x2 = torch.empty_like(b)
    _, it2, rel2, _ = gpu_lib.sqmr_solve(K, x2, b, eps, L, hop, sigma, tol=1e-10, maxit=200)
    assert it1 == it2 and rel2 <= 1e-10
    assert torch.linalg.norm(x1 - x2) <= 1e-13 * torch.linalg.norm(x1)
    K.free()
