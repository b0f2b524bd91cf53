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
    i, j, B11, B12, B22, lm2, d2 = pairs[0]
    assert (i, j) == (0, 1)
    det = 0.1 * 0.2 - 1.0
    assert np.isclose(B11, 0.2 / det) and np.isclose(B12, -1.0 / det) and np.isclose(B22, 0.1 / det)
    # rows c=2: (0.5, 0) B^{-1}; c=3: (0, 0.5) B^{-1}
    # d2 = (0.5*0.2 + 0.5*1 + 0.5*1 + 0.5*0.1)/0.98, lmax2 = 0.6/0.98   (PAPER.md l.866-868:
    # d2 = sum_{j>2} ||(s_j1, s_j2) B^{-1}||, the row norm read as the 1-norm, R8)
    assert np.isclose(lm2, 0.6 / 0.98, rtol=0, atol=1e-15)
    assert np.isclose(d2, 1.15 / 0.98, rtol=0, atol=1e-15)
    # the paper's acceptance test d2 < d1 of the failing (leading) member 0: 1.173 < 15
    dg, lmax1, d1, p = mlildl._pivot_quality(Ah)
    assert d2 < d1[0]


def _pair_star(m):
    """Pair {0, 1}: a_00 = a_11 = 0.2, a_01 = 1 (both fail the 1x1 bound, lmax1 = 5);
    node 1 also couples with 0.9 to m leaves (diagonal 1).  Unit row maxima: D = I."""
    n = 2 + m
    A = np.eye(n)
    A[0, 0] = A[1, 1] = 0.2
    A[0, 1] = A[1, 0] = 1.0
    for c in range(2, n):
        A[1, c] = A[c, 1] = 0.9
    return A


@pytest.mark.parametrize("m,accepted", [(3, True), (5, False)])
def test_pair_d2_vs_d1_by_hand(m, accepted):
    # "we perform a 2x2 update only if d2 < d1".  B^{-1} = [[0.2, -1], [-1, 0.2]] / -0.96;
    # a leaf row (0, 0.9) B^{-1} has |l| = (0.9, 0.18)/0.96 -> 1.125 each: d2 = 1.125 m, lmax2 = 1.125;
    # d1 of the leading (failing) member 0 = |a_10| / |a_00| = 5.  m = 3: 3.375 < 5 accepted;
    # m = 5: 5.625 >= 5 rejected (then neither member is a pivot candidate)
    A = _pair_star(m)
    D, Ah = mlildl._scaled(sp.csr_matrix(A))
    assert np.array_equal(D, np.ones(2 + m))
    dg, lmax1, d1, p = mlildl._pivot_quality(Ah)
    assert np.isclose(d1[0], 5.0) and list(p[:2]) == [1, 0]
    pairs = mlildl._pair_candidates(Ah, dg, lmax1, d1, p, kappa=5.0)
    assert (len(pairs) == 1) == accepted
    if accepted:
        i, j, B11, B12, B22, lm2, d2 = pairs[0]
        assert np.isclose(d2, 1.125 * m, rtol=0, atol=1e-14) and np.isclose(lm2, 1.125, rtol=0, atol=1e-15)
    # in the level, the leaves (lmax1 = 0.9 < lmax2) win the independent set either way and
    # node 0 is never a 1x1 pivot: it is eliminated only as part of the accepted pair
    Lv = mlildl.factor_level(sp.csr_matrix(A), kappa=5.0, tau_drop=0.0, tau_strong=0.02)
    assert 0 not in Lv.F and Lv.npairs == 0

def test_scaling_by_hand():
    # reading R7 ("D is a diagonal matrix"): D_i = 1/sqrt(max_j |a_ij|),
    # a^_ij = a_ij (D_i D_j).  Row maxima 4, 2, 0.25 -> D = (1/2, 1/sqrt 2, 2)
    A = np.array([[4.0, -1.0, 0.1],
                  [-1.0, 0.5, 2.0],
                  [0.1, 2.0, 0.25]])
    D, Ah = mlildl._scaled(sp.csr_matrix(A))
    rowmax = np.abs(A).max(axis=1)
    assert np.allclose(rowmax, [4.0, 2.0, 2.0])
    assert np.allclose(D, [0.5, 1 / np.sqrt(2.0), 1 / np.sqrt(2.0)], rtol=0, atol=1e-16)
    Ah_ref = np.array([[1.0, -1.0 / (2 * np.sqrt(2.0)), 0.1 / (2 * np.sqrt(2.0))],
                       [-1.0 / (2 * np.sqrt(2.0)), 0.25, 1.0],
                       [0.1 / (2 * np.sqrt(2.0)), 1.0, 0.125]])
    assert np.allclose(Ah.toarray(), Ah_ref, rtol=0, atol=1e-15)
    # every row of A^ has max |a^_ij| <= 1, attained where a_ij realises both row maxima
    assert np.abs(Ah.toarray()).max() <= 1.0 + 1e-15


def test_scaled_level_factor_by_hand():
    # one level with non-unit scaling, values worked out by hand.  Row maxima 4, 2, 0.5:
    # D = (1/2, 1/sqrt 2, sqrt 2); A^ = [[1, 1/(2 sqrt 2), 0], [., 1, 1/2], [0, 1/2, 1/2]].
    # All three pass the 1x1 test (lmax1 = 0.354, 0.5, 1.0); no pair (both members of the
    # mutual proposal {1, 2} pass).  The MIS on the strong graph (tau_strong = 0, ranked by
    # lmax1) takes 0, removes 1, then takes 2: F = {0, 2}, C = {1}.
    # L = (a^_10 / a^_00, a^_12 / a^_22) = (1/(2 sqrt 2), 1), S = 1 - 1/8 - 1/2 = 3/8.
    A = np.array([[4.0, 1.0, 0.0],
                  [1.0, 2.0, 0.5],
                  [0.0, 0.5, 0.25]])
    D, Ah = mlildl._scaled(sp.csr_matrix(A))
    assert np.allclose(D, [0.5, 1 / np.sqrt(2.0), np.sqrt(2.0)], rtol=0, atol=1e-15)
    Lv = mlildl.factor_level(sp.csr_matrix(A), kappa=5.0, tau_drop=0.0, tau_strong=0.0)
    assert list(Lv.F) == [0, 2] and list(Lv.C) == [1]
    assert np.allclose(Lv.L.toarray(), [[1 / (2 * np.sqrt(2.0)), 0.0, 1.0]], rtol=0, atol=1e-15)
    assert np.allclose(Lv.S.toarray(), [[0.375]], rtol=0, atol=1e-15)
    # the operator M^{-1} = D (L D~ L^T)^{-1} D with the dense coarse inverse of S is exact
    # here (nothing dropped): M^{-1} = A^{-1}
    M = mlildl.MultilevelILDL(sp.csr_matrix(A), kappa=5.0, tau_drop=0.0, tau_strong=0.0, n_coarse_max=1,
                              stall_frac=0.0)
    assert len(M.levels) == 1 and M.coarse_n == 1
    r = np.array([1.0, -2.0, 0.5])
    assert np.allclose(M.apply(r), np.linalg.solve(A, r), rtol=1e-14, atol=0)

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


def _level_matrices(A, M):
    """The matrix each level of M factored: A, then the Schur complement of the previous level."""
    mats = [sp.csr_matrix(A)]
    for Lv in M.levels[:-1]:
        mats.append(Lv.S)
    return mats


@pytest.mark.parametrize("case", ["lattice", "random"])
def test_F_independent_in_strong_graph(case):
    # reading R9: F is an independent set of pivot blocks in the strong graph |a^_ij| >= tau_strong
    # (level 0 on the lattice: the red sites, independent in the whole stencil graph)
    if case == "lattice":
        L = 10
        A = an.matrix(L, an.disorder(L, 16.5, 3), hop=-1.0)
        M = mlildl.MultilevelILDL(A, lattice_L=L, tau_drop=2e-3, tau_strong=0.05, n_coarse_max=100)
    else:
        A = _rand_sym_indef(400, 0.02, 5)
        M = mlildl.MultilevelILDL(A, tau_drop=1e-3, tau_strong=0.05, n_coarse_max=20)
    assert len(M.levels) >= 2
    for lev, (Al, Lv) in enumerate(zip(_level_matrices(A, M), M.levels)):
        D = Lv.D
        Ah = sp.csr_matrix(sp.diags(D) @ Al @ sp.diags(D)).tocoo()
        inF = Lv.inF
        partner = Lv.partner
        m = (Ah.row != Ah.col) & inF[Ah.row] & inF[Ah.col] & (partner[Ah.row] != Ah.col)
        thr = 0.0 if (lev == 0 and case == "lattice") else 0.05
        assert np.all(np.abs(Ah.data[m]) < thr) if thr > 0 else not m.any(), lev


def _plain_level(Al, Lv, compensate):
    """The plain definitions of one level (reading R17): with
    B~^{-1} = B_d^{-1} + V (block pivots + virtual couplings),
      L = A^_CF B~^{-1}
      S = A^_CC - A^_CF B_d^{-1} A^_FC - P o (A^_CF V A^_FC),
    P = the structural pattern of A^_CC + A^_CF B_d^{-1} A^_FC (no fill from V)."""
    D = Lv.D
    Ah = sp.csr_matrix(sp.diags(D) @ Al @ sp.diags(D))
    F, C = Lv.F, Lv.C
    n = Ah.shape[0]
    Binv = Lv.Binv.toarray()
    part = Lv.partner
    Bd = np.zeros_like(Binv)
    for f in F:
        Bd[f, f] = Binv[f, f]
        if part[f] >= 0:
            Bd[f, part[f]] = Binv[f, part[f]]
    V = Binv - Bd
    if not compensate:
        assert not V.any()
    Ad = Ah.toarray()
    ACF, AFC, ACC = Ad[np.ix_(C, F)], Ad[np.ix_(F, C)], Ad[np.ix_(C, C)]
    Lp = ACF @ Binv[np.ix_(F, F)]
    S1 = ACC - ACF @ Bd[np.ix_(F, F)] @ AFC
    pattern = (np.abs(ACC) > 0) | ((np.abs(ACF) > 0).astype(float) @ (np.abs(Bd[np.ix_(F, F)]) > 0).astype(float)
                                   @ (np.abs(AFC) > 0).astype(float) > 0) | np.eye(len(C), dtype=bool)
    S = S1 - np.where(pattern, ACF @ V[np.ix_(F, F)] @ AFC, 0.0)
    return Lp, 0.5 * (S + S.T)


@pytest.mark.parametrize("case,compensate", [("lattice", True), ("lattice", False), ("random", True),
                                             ("random", False), ("lattice12", True)])
def test_ordered_accumulation_equals_plain_definition(case, compensate):
    # The oracle accumulates L and S block by block in ascending key (the order the GPU
    # reproduces bit for bit, R10/R17).  Pin that ordered accumulation to the plain
    # matrix definitions, with dropping disabled (tau_drop = 0) but a real strong threshold
    # (tau_strong > 0: weak F-F couplings exist, so R17's virtual blocks are exercised).
    if case.startswith("lattice"):
        L = 12 if case == "lattice12" else 8
        A = an.matrix(L, an.disorder(L, 16.5, 2), hop=-1.0)
        M = mlildl.MultilevelILDL(A, lattice_L=L, tau_drop=0.0, tau_strong=0.05, n_coarse_max=60,
                                  max_levels=4 if L == 12 else 200, compensate=compensate, tau_virtual=0.0)
    else:
        A = _rand_sym_indef(250, 0.03, 7)
        M = mlildl.MultilevelILDL(A, tau_drop=0.0, tau_strong=0.05, n_coarse_max=30, compensate=compensate,
                                  tau_virtual=0.0)
    assert len(M.levels) >= 2
    nvirt = 0
    for Al, Lv in zip(_level_matrices(A, M), M.levels):
        Lp, Sp = _plain_level(Al, Lv, compensate)
        Lo = Lv.L.toarray()[:, Lv.F]
        So = Lv.S.toarray()
        scale_L = max(1.0, np.abs(Lp).max())
        scale_S = max(1.0, np.abs(Sp).max())
        assert np.abs(Lo - Lp).max() <= 1e-14 * scale_L
        assert np.abs(So - Sp).max() <= 1e-14 * scale_S
        # S is stored symmetric bit for bit (upper triangle mirrored)
        assert (Lv.S != Lv.S.T).nnz == 0
        nvirt += Lv.nvirtual
    assert (nvirt > 0) == compensate


# ---------------------------------------------------------------- inverse-based dropping (R18)
def test_nu_by_hand():
    # the one-level 3x3 factor of test_scaled_level_factor_by_hand: F = {0, 2}, C = {1},
    # L = [[l_10, 0, l_12]] = [[1/(2 sqrt 2), 0, 1]], coarse block {1}.  Back substitution with
    # L~^T: x_1 = b_1 = +1; s_0 = l_10 x_1 > 0 -> x_0 = -1 - s_0;
    # s_2 = l_12 x_1 = 1 -> x_2 = -2.  nu = |x| = (1 + 1/(2 sqrt 2), 1, 2) -- here exactly the
    # 1-norms of the columns of L~^{-1} = I - N.
    A = np.array([[4.0, 1.0, 0.0],
                  [1.0, 2.0, 0.5],
                  [0.0, 0.5, 0.25]])
    M = mlildl.MultilevelILDL(sp.csr_matrix(A), kappa=5.0, tau_drop=0.0, tau_strong=0.0, n_coarse_max=1,
                              stall_frac=0.0)
    x = mlildl.nu_estimates(M)[0]
    a = 1 / (2 * np.sqrt(2.0))
    assert np.allclose(x, [-1.0 - a, 1.0, -2.0], rtol=0, atol=1e-15)
    # dropping rule |l_cf| <= tau / (nu_c #col_f): nu_1 = 1, #col_0 = #col_2 = 1 -> with tau = 0.5
    # the entry l_10 = 0.354 goes, l_12 = 1 stays
    M2 = mlildl.MultilevelILDL(sp.csr_matrix(A), kappa=5.0, tau_drop=0.0, tau_strong=0.0, n_coarse_max=1,
                               stall_frac=0.0, tau_inv=0.5)
    assert np.allclose(M2.levels[0].L.toarray(), [[0.0, 0.0, 1.0]], rtol=0, atol=0)
    assert M2.levels[0].ndrop_inv == 1


def _global_L(M, n):
    """The unit lower factor of the whole multilevel factorisation in the original index
    space: I + sum_l N_l (the level factors' off-diagonal blocks; their products vanish)."""
    Lg = np.eye(n)
    orig = np.arange(n)                     # level index -> original index
    for Lv in M.levels:
        Ld = Lv.L.toarray()                 # (coarse index, level index)
        rows, cols = np.nonzero(Ld)
        Lg[orig[Lv.C[rows]], orig[cols]] = Ld[rows, cols]
        orig = orig[Lv.C]
    return Lg


@pytest.mark.parametrize("seed", [1, 2])
def test_nu_bounds_against_exact_columns(seed):
    # the CMSW estimate is |L~^{-1} b| for a +-1 vector b chosen along the way: 1 <= nu_i <=
    # ||L~^{-1} e_i||_1, with L~^{-1} computed densely from the global factor
    L = 8
    A = an.matrix(L, an.disorder(L, 16.5, seed), hop=-1.0)
    M = mlildl.MultilevelILDL(A, lattice_L=L, tau_drop=2e-3, tau_strong=0.05, n_coarse_max=40)
    assert len(M.levels) >= 3
    xs = mlildl.nu_estimates(M)
    Lg = _global_L(M, L ** 3)
    Linv = np.linalg.inv(Lg)
    col1 = np.abs(Linv).sum(axis=0)          # ||L~^{-1} e_i||_1
    nu0 = np.abs(xs[0])                      # level 0 covers every node (original order)
    assert np.all(nu0 >= 1.0 - 1e-15)
    assert np.all(nu0 <= col1 * (1 + 1e-12))
    # the estimate is the exact |L~^{-T}... b| of the sign vector it chose: x = L~^{-T} b
    b = np.where(Lg.T @ xs[0] > 0, 1.0, -1.0)
    assert np.allclose(Lg.T @ xs[0], b, rtol=0, atol=1e-12)


@pytest.mark.parametrize("tau", [0.1, 0.5])
def test_inverse_based_dropping_rule_and_effect(tau):
    L = 12
    A = an.matrix(L, an.disorder(L, 16.5, 3), hop=-1.0)
    kw = dict(lattice_L=L, tau_drop=2e-3, tau_strong=0.05, n_coarse_max=200)
    M0 = mlildl.MultilevelILDL(A, **kw)
    M1 = mlildl.MultilevelILDL(A, tau_inv=tau, **kw)
    xs = mlildl.nu_estimates(M0)
    for lev, (L0, L1) in enumerate(zip(M0.levels, M1.levels)):
        nu = np.abs(xs[lev + 1]) if lev + 1 < len(M0.levels) else np.ones(M0.coarse_n)
        c = L0.L.tocoo()
        cnt = np.bincount(c.col, minlength=L0.n)
        ok = np.abs(c.data) * nu[c.row] * cnt[c.col] > tau * (1 + 1e-12)
        assert L1.L.nnz == ok.sum() or abs(L1.L.nnz - ok.sum()) <= 2   # rounding at the threshold
        kept = sp.csr_matrix((c.data[ok], (c.row[ok], c.col[ok])), shape=L0.L.shape)
        assert abs(L1.L - kept).max() == 0.0 or abs(L1.L.nnz - ok.sum()) > 0
    assert sum(lv.L.nnz for lv in M1.levels) < sum(lv.L.nnz for lv in M0.levels)
    b = np.random.default_rng(5).standard_normal(L ** 3)
    x, it, res, _ = sqmr(lambda v: A @ v, M1.apply, b, tol=1e-8, maxit=300)
    assert res <= 1e-8
