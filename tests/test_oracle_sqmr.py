"""Pins for oracle/sqmr.py (simplified QMR)."""
import numpy as np

from oracle.sqmr import sqmr


def test_identity_one_step():
    b = np.arange(1.0, 6.0)
    x, it, res, _ = sqmr(lambda v: v, lambda v: v, b)
    assert it == 1 and np.allclose(x, b)


def test_diag_indefinite_exact_in_n_steps():
    # Krylov method on a 2x2 system terminates in <= 2 steps (exact arithmetic)
    A = np.diag([2.0, -1.0])
    x, it, res, _ = sqmr(lambda v: A @ v, lambda v: v, np.array([1.0, 1.0]))
    assert it <= 2 and np.allclose(x, [0.5, -1.0])


def test_breakdown_reported():
    # diag(1,-1), b = (1,1): q^T A q = 0 at the first step -- a genuine SQMR
    # (Lanczos) breakdown; it must be reported (residual not converged), not hidden.
    A = np.diag([1.0, -1.0])
    x, it, res, _ = sqmr(lambda v: A @ v, lambda v: v, np.array([1.0, 1.0]))
    assert res > 1e-10


def test_matches_dense_solve_indefinite():
    rng = np.random.default_rng(1)
    n = 40
    B = rng.standard_normal((n, n))
    A = B + B.T + np.diag(rng.uniform(-3, 3, n))
    b = rng.standard_normal(n)
    x, it, res, _ = sqmr(lambda v: A @ v, lambda v: v, b, tol=1e-12, maxit=400)
    assert np.allclose(x, np.linalg.solve(A, b), rtol=1e-8, atol=1e-8)
    # recursive QMR residual equals the true residual
    assert abs(np.linalg.norm(b - A @ x) / np.linalg.norm(b) - res) < 1e-10


def test_exact_preconditioner_converges_immediately():
    rng = np.random.default_rng(2)
    n = 60
    B = rng.standard_normal((n, n))
    A = B + B.T
    Ainv = np.linalg.inv(A)
    b = rng.standard_normal(n)
    x, it, res, _ = sqmr(lambda v: A @ v, lambda v: Ainv @ v, b, tol=1e-10)
    assert it <= 2 and np.allclose(A @ x, b, atol=1e-9)


def test_symmetric_indefinite_preconditioner():
    # a symmetric indefinite M^{-1} close to A^{-1} still converges (SQMR's point)
    rng = np.random.default_rng(3)
    n = 80
    B = rng.standard_normal((n, n))
    A = B + B.T + np.diag(rng.uniform(-5, 5, n))
    P = np.linalg.inv(A + 0.05 * np.diag(rng.standard_normal(n)))
    P = 0.5 * (P + P.T)
    b = rng.standard_normal(n)
    x, it, res, _ = sqmr(lambda v: A @ v, lambda v: P @ v, b, tol=1e-10, maxit=200)
    assert res <= 1e-10 and it < 60
