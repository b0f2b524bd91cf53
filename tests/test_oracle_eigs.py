"""Pins for oracle/eigs.py: dense diagonalisation and plain shift-and-invert
Lanczos (sect. 4.1 l.335-378) against closed forms / each other."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import anderson as an
from oracle import eigs


def test_si_lanczos_diagonal():
    # SPEC example: diag(1..6), sigma = 3.1, want 2 -> {3, 4}
    A = sp.diags(np.arange(1.0, 7.0)).tocsr()
    lam, X, res = eigs.si_lanczos_nearest(A, 2, sigma=3.1)
    assert np.allclose(lam, [3.0, 4.0], atol=1e-12)


def test_si_lanczos_clean_lattice_closed_form():
    # W = 0, L = 6, tiny disorder breaks degeneracy; eigenvalues near 1.0 from the
    # closed form 2*hop*sum cos within perturbation size
    L = 6
    eps = an.disorder(L, 1e-6, 1)
    A = an.matrix(L, eps, hop=-1.0)
    lam, X, res = eigs.si_lanczos_nearest(A, 3, sigma=-0.9)
    c = np.cos(2 * np.pi * np.arange(L) / L)
    ref = np.sort((-2 * (c[:, None, None] + c[None, :, None] + c[None, None, :])).ravel())
    for v in lam:
        assert np.min(np.abs(ref - v)) < 2e-6


@pytest.mark.parametrize("L,seed,sigma", [(8, 1, 0.0), (10, 0, 0.0), (10, 2, 1.5)])
def test_si_lanczos_matches_dense(L, seed, sigma):
    eps = an.disorder(L, 16.5, seed)
    A = an.matrix(L, eps, hop=-1.0)
    ld, Xd = eigs.dense_nearest(A, 5, sigma)
    ll, Xl, res = eigs.si_lanczos_nearest(A, 5, sigma)
    normA = abs(A).sum(axis=0).max()
    assert np.allclose(ll, ld, atol=1e-12 * normA)
    assert np.all(res <= 1e-12 * normA)
    # subspace angle
    for i in range(5):
        assert abs(abs(Xd[:, i] @ Xl[:, i]) - 1.0) < 1e-12


def test_dense_residuals():
    L = 6
    A = an.matrix(L, an.disorder(L, 16.5, 3), hop=-1.0)
    lam, X = eigs.dense_nearest(A, 5, 0.0)
    assert np.all(np.abs(lam[:-1]) <= np.abs(lam[1:]) + 1e-15)
    assert np.linalg.norm(A @ X - X * lam) < 1e-12


def test_si_lanczos_iterative_inner_matches_dense():
    # the iterative full-accuracy inner solver (reading R14) gives the dense answer
    L = 10
    A = an.matrix(L, an.disorder(L, 16.5, 0), hop=-1.0)
    solve = eigs.iterative_solver(A, 0.0, L=L, tol=1e-14)
    ll, Xl, res = eigs.si_lanczos_nearest(A, 5, 0.0, tol=1e-12, solve=solve)
    ld, Xd = eigs.dense_nearest(A, 5, 0.0)
    normA = abs(A).sum(axis=0).max()
    assert np.allclose(ll, ld, atol=1e-12 * normA)
    assert np.all(res <= 1e-12 * normA)
