"""Eigenpairs nearest a shift (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

What jd_solve computes has a plain definition: the k eigenpairs of the
symmetric matrix A closest to sigma ("the computation
of 5 eigenvalues of the Anderson matrix A near lambda=0").  The oracle is that
definition:

* `dense_nearest` -- full dense diagonalisation (numpy.linalg.eigh, a library
  primitive) for tiny L (n <= ~4000).
* `si_lanczos_nearest` -- plain shift-and-invert Lanczos of PAPER.md sect. 4.1
  (l.338-362): orthonormal v_1..v_m with (A - sigma I)^{-1} V_m = V_{m+1} T_m,
  full reorthogonalisation, no restart; the inner solve (A - sigma I) y = v is
  done "to full accuracy" (l.324-326) with a sparse direct LU (scipy splu, a
  library primitive; no preconditioner).  Ritz values mu of T_m map back as
  lambda = sigma + 1/mu.
"""
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spl


def order_nearest(lam, sigma):
    """Indices sorting eigenvalues by |lambda - sigma|, ties -> smaller lambda."""
    lam = np.asarray(lam)
    return np.lexsort((lam, np.abs(lam - sigma)))


def dense_nearest(A, k, sigma=0.0):
    """k eigenpairs of dense/sparse symmetric A nearest sigma, by full eigh.
    Returns (lam[k], X[n,k]) ordered by distance to sigma."""
    M = A.toarray() if sp.issparse(A) else np.asarray(A, dtype=np.float64)
    lam, X = np.linalg.eigh(M)
    idx = order_nearest(lam, sigma)[:k]
    return lam[idx], X[:, idx]


def si_lanczos_nearest(A, k, sigma=0.0, tol=1e-12, m0=None, mmax=600, seed=12345, solve=None):
    """k eigenpairs of sparse symmetric A nearest sigma via plain
    shift-and-invert Lanczos (sect. 4.1) with full reorthogonalisation.

    Grows the Krylov dimension m (no implicit restart) until the k wanted
    Ritz pairs satisfy ||A x - lambda x|| <= tol * ||A||_1.
    solve: callable v -> (A - sigma I)^{-1} v to full accuracy; default a sparse
    direct LU (fine up to L ~ 20; SuperLU fill explodes on 3-D lattices beyond,
    see `iterative_solver`).
    Returns (lam[k], X[n,k], resid[k])."""
    A = sp.csr_matrix(A)
    n = A.shape[0]
    normA = abs(A).sum(axis=0).max()
    if solve is None:
        lu = spl.splu(sp.csc_matrix(A - sigma * sp.identity(n)))
        solve = lu.solve
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(n)
    V = [v / np.linalg.norm(v)]
    alpha, beta = [], []
    m = min(n, m0 or max(3 * k + 20, 40))
    mmax = min(mmax, n)
    scale = 0.0
    while True:
        while len(alpha) < m:
            w = solve(V[-1])
            a = V[-1] @ w
            w = w - a * V[-1] - (beta[-1] * V[-2] if beta else 0.0)
            Vm = np.array(V)
            for _ in range(2):                       # full reorthogonalisation
                w = w - Vm.T @ (Vm @ w)
            b = np.linalg.norm(w)
            scale = max(scale, abs(a), b)
            alpha.append(a)
            if b <= 1e-13 * scale:          # invariant subspace found
                beta.append(0.0)
                break
            beta.append(b)
            V.append(w / b)
        T = np.diag(alpha) + np.diag(beta[:-1], 1) + np.diag(beta[:-1], -1)
        mu, S = np.linalg.eigh(T)
        Vm = np.array(V[:len(alpha)]).T
        sel = np.argsort(-np.abs(mu))[: 3 * k]
        lam = sigma + 1.0 / mu[sel]
        X = Vm @ S[:, sel]
        X /= np.linalg.norm(X, axis=0)
        res = np.linalg.norm(A @ X - X * lam, axis=0)
        idx = order_nearest(lam, sigma)[:k]
        if np.all(res[idx] <= tol * normA) or len(alpha) >= mmax or beta[-1] == 0.0:
            return lam[idx], X[:, idx], res[idx]
        m = min(mmax, int(m * 1.5))


def iterative_solver(A, sigma, L=None, tol=1e-14, maxit=2000):
    """(A - sigma I)^{-1} v "to full accuracy" by oracle SQMR
    preconditioned with the oracle multilevel ILDL (reading R14), for lattices
    where a sparse direct LU is out of reach.  Raises if an inner solve stalls
    above 100*tol."""
    from .mlildl import MultilevelILDL
    from .sqmr import sqmr
    As = sp.csr_matrix(A - sigma * sp.identity(A.shape[0]))
    M = MultilevelILDL(As, lattice_L=L, n_coarse_max=1024)
    stats = {"solves": 0, "iters": 0}

    def solve(v):
        x, it, res, _ = sqmr(lambda q: As @ q, M.apply, v, tol=tol, maxit=maxit)
        if not res <= 100 * tol:
            raise RuntimeError(f"inner solve stalled at {res:.2e}")
        stats["solves"] += 1
        stats["iters"] += it
        return x

    solve.stats = stats
    return solve
