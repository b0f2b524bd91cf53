"""Pins for oracle/jd.py: its eigenpairs equal the dense-diagonalisation
definition (itself pinned by the closed-form spectrum) on small lattices."""
import numpy as np
import pytest

from oracle import anderson as an
from oracle import eigs, mlildl
from oracle.jd import jd_nearest


@pytest.mark.parametrize("L,W,seed,sigma,k", [(8, 16.5, 1, 0.0, 5), (10, 12.0, 2, 0.7, 3), (7, 21.0, 3, 0.0, 2)])
def test_jd_matches_dense(L, W, seed, sigma, k):
    A = an.matrix(L, an.disorder(L, W, seed), hop=-1.0)
    M = mlildl.MultilevelILDL(an.matrix(L, an.disorder(L, W, seed), hop=-1.0, sigma=sigma), lattice_L=L,
                              n_coarse_max=100)
    lam, X, st = jd_nearest(A, M.apply, k, sigma=sigma, tol=1e-11)
    lr, Xr = eigs.dense_nearest(A, k, sigma)
    normA = abs(A).sum(axis=0).max()
    assert np.allclose(np.sort(lam), np.sort(lr), atol=1e-10 * normA)
    assert np.linalg.norm(A @ X - X * lam, axis=0).max() <= 1e-8 * normA
    assert np.abs(X.T @ X - np.eye(k)).max() < 1e-8


def test_jd_identity_preconditioner_diagonal():
    # JD with K = I on diag(1..30), target 10.2 -> {10, 11, 9}
    import scipy.sparse as sp
    A = sp.diags(np.arange(1.0, 31.0)).tocsr()
    lam, X, st = jd_nearest(A, lambda v: v, 3, sigma=10.2, tol=1e-12, jmin=3, jmax=8)
    assert np.allclose(lam, [10.0, 11.0, 9.0], atol=1e-10)
