"""Pins for oracle/mlildl.py (sect. 7, l.790-973).

Pins: hand-computed d1/d2 and Schur complement on a 4x4 example (the
formulas of l.866-874, l.857, l.900-908 evaluated by hand), exactness limit
(no dropping, no kappa bound -> exact block LDL^T inverse), 2x2 pivot on the
swap matrix, identity, operator symmetry, the inverse-based bound
||L^{-1}||_inf <= kappa per level (l.884-896), and effectiveness.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import anderson as an
from oracle import mlildl
from oracle.sqmr import sqmr

# 4x4 example with unit row maxima (so the level scaling D is the identity)
A4 = np.array([[0.1, 1.0, 0.5, 0.0],
               [1.0, 0.2, 0.0, 0.5],
               [0.5, 0.0, 1.0, 0.2],
               [0.0, 0.5, 0.2, 1.0]])


def test_pivot_quality_by_hand():
    D, Ah = mlildl._scaled(sp.csr_matrix(A4))
    assert np.array_equal(D, np.ones(4))
    dg, lmax1, d1, p = mlildl._pivot_quality(Ah)
    # d1_f = sum_{j != f} |a_jf| / |a_ff|
    assert np.allclose(d1, [15.0, 7.5, 0.7, 0.7])
    assert np.allclose(lmax1, [10.0, 5.0, 0.5, 0.5])
    assert list(p) == [1, 0, 0, 1]


def test_pair_d2_by_hand():
    D, Ah = mlildl._scaled(sp.csr_matrix(A4))
    dg, lmax1, d1, p = mlildl._pivot_quality(Ah)
    pairs = mlildl._pair_candidates(Ah, dg, lmax1, d1, p, kappa=5.0)
    assert len(pairs) == 1
    i, j, B11, B12, B22, lm2 = pairs[0]
    assert (i, j) == (0, 1)
    det = 0.1 * 0.2 - 1.0
    assert np.isclose(B11, 0.2 / det) and np.isclose(B12, -1.0 / det) and np.isclose(B22, 0.1 / det)
    # rows c=2: (0.5, 0) B^{-1}; c=3: (0, 0.5) B^{-1}
    # d2 = (0.5*0.2 + 0.5*1 + 0.5*1 + 0.5*0.1)/0.98, lmax2 = 0.6/0.98
    assert np.isclose(lm2, 0.6 / 0.98)


def test_level_schur_by_hand():
    # blocks {0,1} (key 0.612), {2} (0.5), {3} (0.5): MIS on the strong graph picks {2};
    # S = A_CC - a_C2 a_2C / a_22 on C = {0, 1, 3}
    Lv = mlildl.factor_level(sp.csr_matrix(A4), kappa=5.0, tau_drop=0.0, tau_strong=0.02)
    assert list(Lv.F) == [2] and list(Lv.C) == [0, 1, 3]
    S_ref = np.array([[0.1 - 0.25, 1.0, -0.1],
                      [1.0, 0.2, 0.5],
                      [-0.1, 0.5, 1.0 - 0.04]])
    assert np.allclose(Lv.S.toarray(), S_ref, atol=1e-15)
    assert np.allclose(Lv.L.toarray()[:, 2], [0.5, 0.0, 0.2])


def test_swap_matrix_2x2_pivot():
    A = sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 0.0]]))
    M = mlildl.MultilevelILDL(A, n_coarse_max=0, stall_frac=0.0)
    assert len(M.levels) == 1 and M.levels[0].npairs == 1 and M.coarse_n == 0
    r = np.array([0.3, -2.0])
    assert np.allclose(M.apply(r), [-2.0, 0.3])


def test_identity():
    A = sp.identity(50, format="csr")
    M = mlildl.MultilevelILDL(A, n_coarse_max=0, stall_frac=0.0)
    r = np.arange(50.0)
    assert np.allclose(M.apply(r), r)


def _rand_sym_indef(n, density, seed):
    rng = np.random.default_rng(seed)
    B = sp.random(n, n, density=density, random_state=seed, data_rvs=lambda k: rng.uniform(-1, 1, k))
    A = B + B.T + sp.diags(rng.uniform(-2, 2, n))
    return sp.csr_matrix(A)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_exactness_limit_random(seed):
    # tau_drop = 0, tau_strong = 0 (true independent sets), kappa = inf:
    # the multilevel block LDL^T is exact, so M^{-1} A = I.
    A = _rand_sym_indef(150, 0.03, seed)
    M = mlildl.MultilevelILDL(A, kappa=np.inf, tau_drop=0.0, tau_strong=0.0,
                              n_coarse_max=5, stall_frac=0.0)
    x = np.random.default_rng(seed + 10).standard_normal(150)
    assert np.linalg.norm(M.apply(A @ x) - x) <= 1e-9 * np.linalg.norm(x)


def test_exactness_limit_anderson():
    L = 6
    A = an.matrix(L, an.disorder(L, 16.5, 1), hop=-1.0)
    M = mlildl.MultilevelILDL(A, lattice_L=L, kappa=np.inf, tau_drop=0.0, tau_strong=0.0,
                              n_coarse_max=10, stall_frac=0.0)
    x = np.random.default_rng(3).standard_normal(L ** 3)
    assert np.linalg.norm(M.apply(A @ x) - x) <= 1e-10 * np.linalg.norm(x)


def test_operator_symmetric_and_linear():
    L = 10
    A = an.matrix(L, an.disorder(L, 16.5, 2), hop=-1.0)
    M = mlildl.MultilevelILDL(A, lattice_L=L, n_coarse_max=200)
    rng = np.random.default_rng(4)
    r1, r2 = rng.standard_normal((2, L ** 3))
    z1, z2 = M.apply(r1), M.apply(r2)
    assert np.isclose(r2 @ z1, r1 @ z2, rtol=1e-10)
    assert np.allclose(M.apply(2.0 * r1 - 3.0 * r2), 2.0 * z1 - 3.0 * z2, rtol=1e-10, atol=1e-10)


@pytest.mark.parametrize("kappa", [3.0, 5.0, 10.0])
def test_inverse_bound_per_level(kappa):
    # ||L^{-1}||_inf = 1 + max_c sum_f |L_cf| <= kappa for every level (l.884-896)
    L = 10
    A = an.matrix(L, an.disorder(L, 16.5, 3), hop=-1.0)
    M = mlildl.MultilevelILDL(A, lattice_L=L, kappa=kappa, n_coarse_max=100)
    assert len(M.levels) >= 2
    for Lv in M.levels:
        Ld = abs(Lv.L)
        if Ld.nnz:
            assert 1.0 + Ld.sum(axis=1).max() <= kappa + 1e-12
        # F is an independent set in the strong graph; levels shrink
        assert len(Lv.F) > 0 and len(Lv.C) < Lv.n


def test_level0_is_red_set():
    L = 8
    A = an.matrix(L, an.disorder(L, 16.5, 4), hop=-1.0)
    M = mlildl.MultilevelILDL(A, lattice_L=L, n_coarse_max=50)
    red = an.red_sites(L)
    assert np.all(red[M.levels[0].F])
    assert M.levels[0].npairs == 0


def test_preconditioner_effectiveness():
    # SQMR on (A - 0 I) x = b, L = 12, W = 16.5: preconditioned converges fast,
    # unpreconditioned does not within the same budget (sect. 8, Table 2-3 trend)
    L = 12
    A = an.matrix(L, an.disorder(L, 16.5, 1), hop=-1.0)
    M = mlildl.MultilevelILDL(A, lattice_L=L, n_coarse_max=300)
    b = np.random.default_rng(5).standard_normal(L ** 3)
    x, it, res, _ = sqmr(lambda v: A @ v, M.apply, b, tol=1e-10, maxit=150)
    assert res <= 1e-10 and it <= 60
    assert np.linalg.norm(A @ x - b) <= 1e-9 * np.linalg.norm(b)
    x0, it0, res0, _ = sqmr(lambda v: A @ v, lambda v: v, b, tol=1e-10, maxit=150)
    assert res0 > 1e-6


def test_fp32_factor_storage_close_to_fp64():
    # reading R16: rounding the stored factor to binary32 perturbs the operator
    # by ~1e-7 relative and leaves the preconditioner effective
    L = 10
    A = an.matrix(L, an.disorder(L, 16.5, 2), hop=-1.0)
    M64 = mlildl.MultilevelILDL(A, lattice_L=L, n_coarse_max=200)
    M32 = mlildl.MultilevelILDL(A, lattice_L=L, n_coarse_max=200, factor_fp32=True)
    r = np.random.default_rng(1).standard_normal(L ** 3)
    z64, z32 = M64.apply(r), M32.apply(r)
    assert np.linalg.norm(z32 - z64) <= 1e-5 * np.linalg.norm(z64)
    assert np.linalg.norm(z32 - z64) > 0.0
    b = np.random.default_rng(5).standard_normal(L ** 3)
    x, it, res, _ = sqmr(lambda v: A @ v, M32.apply, b, tol=1e-10, maxit=150)
    assert res <= 1e-10


def test_weak_coupling_compensation_by_hand():
    # reading R17: pivots 0 and 1 are weakly coupled (e < tau_strong) and both
    # strongly coupled to node 2.  B = [[1, e], [e, 1]] is replaced by its first-order
    # inverse I - E, so S = 1 - (a^2 + b^2 - 2 a b e) and L = (a - b e, b - a e);
    # without compensation the e terms are lost.
    a, b, e = 0.5, 0.6, 0.01
    A = sp.csr_matrix(np.array([[1.0, e, a], [e, 1.0, b], [a, b, 1.0]]))
    Lv = mlildl.factor_level(A, kappa=5.0, tau_drop=0.0, tau_strong=0.02)
    assert list(Lv.F) == [0, 1] and Lv.nvirtual == 1
    assert np.isclose(Lv.S.toarray()[0, 0], 1.0 - (a * a + b * b - 2 * a * b * e), rtol=0, atol=1e-15)
    assert np.allclose(Lv.L.toarray()[0, :2], [a - b * e, b - a * e], rtol=0, atol=1e-15)
    exact = 1.0 - np.array([a, b]) @ np.linalg.solve(np.array([[1.0, e], [e, 1.0]]), np.array([a, b]))
    assert abs(Lv.S.toarray()[0, 0] - exact) < 2 * e * e
    L0 = mlildl.factor_level(A, kappa=5.0, tau_drop=0.0, tau_strong=0.02, compensate=False)
    assert L0.nvirtual == 0
    assert np.isclose(L0.S.toarray()[0, 0], 1.0 - (a * a + b * b), atol=1e-15)


def test_compensation_improves_preconditioner():
    # at a coarse strong threshold the compensated factor needs fewer SQMR steps
    L = 16
    A = an.matrix(L, an.disorder(L, 16.5, 2), hop=-1.0)
    b = np.random.default_rng(5).standard_normal(L ** 3)
    its = {}
    for comp in (False, True):
        M = mlildl.MultilevelILDL(A, lattice_L=L, tau_drop=2e-3, tau_strong=0.05, n_coarse_max=300,
                                  compensate=comp)
        x, it, res, _ = sqmr(lambda v: A @ v, M.apply, b, tol=1e-8, maxit=500)
        assert res <= 1e-8
        its[comp] = it
    assert its[True] < its[False]


def test_compensation_threshold_tau_virtual():
    # reading R17: only couplings |a^_uv| >= tau_virtual become virtual blocks; below it
    # the coupling is dropped as without compensation (same 3x3 case as above)
    a, b, e = 0.5, 0.6, 0.01
    A = sp.csr_matrix(np.array([[1.0, e, a], [e, 1.0, b], [a, b, 1.0]]))
    above = mlildl.factor_level(A, kappa=5.0, tau_drop=0.0, tau_strong=0.02, tau_virtual=0.005)
    below = mlildl.factor_level(A, kappa=5.0, tau_drop=0.0, tau_strong=0.02, tau_virtual=0.02)
    assert above.nvirtual == 1 and below.nvirtual == 0
    assert np.isclose(above.S.toarray()[0, 0], 1.0 - (a * a + b * b - 2 * a * b * e), rtol=0, atol=1e-15)
    assert np.isclose(below.S.toarray()[0, 0], 1.0 - (a * a + b * b), rtol=0, atol=1e-15)


def test_compensation_adds_no_schur_fill():
    # reading R17: the virtual terms update only the pattern of A_CC and the real blocks.
    # Chain c0 - u - v - c1 (u = 0, v = 1 win the independent set on index ties; u - v is
    # weak): the compensated S has no (c0, c1) entry -- it would be fill -- while L carries
    # the first-order coupling l_{c0 v} = a_{c0 u} b'_{uv}, b'_{uv} = -(a_uv B_uu B_vv)
    e = 0.01
    A = np.eye(4)
    A[0, 2] = A[2, 0] = 0.5      # u - c0
    A[0, 1] = A[1, 0] = e        # u - v (weak)
    A[1, 3] = A[3, 1] = 0.6      # v - c1
    Lv = mlildl.factor_level(sp.csr_matrix(A), kappa=5.0, tau_drop=0.0, tau_strong=0.02, tau_virtual=0.0)
    assert sorted(Lv.F) == [0, 1] and Lv.nvirtual == 1
    S = Lv.S.toarray()
    assert S[0, 1] == 0.0 and S[1, 0] == 0.0
    Ld = Lv.L.toarray()
    assert np.isclose(Ld[0, 0], 0.5, rtol=0, atol=1e-15)
    assert np.isclose(Ld[0, 1], 0.5 * -(e * (1.0 * 1.0)), rtol=0, atol=1e-15)
    assert np.isclose(Ld[1, 0], 0.6 * -(e * (1.0 * 1.0)), rtol=0, atol=1e-15)
