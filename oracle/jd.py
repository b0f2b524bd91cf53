"""Symmetric Jacobi-Davidson in plain numpy (TEST INFRASTRUCTURE ONLY -- see
oracle/__init__.py).  Used as the CPU baseline of bench.py (`cpu_baseline`,
`--impl reference`) and as a cross-check of the GPU driver's outer/inner
counts; eigenpair PARITY is always judged against oracle/eigs.py (the plain
definition), which is what pins this module (tests/test_oracle_jd.py).

PAPER.md sect. 4.2 (l.380-421), step by step:
  * search space V (orthonormal, V ^ Q), Ritz pairs of V^T (A - sigma I) V,
    the Ritz value nearest sigma selected ("Ritz approximation [V_k, z]^T A [V_k, z]", l.397-398);
  * residual r = A u - theta u (l.395); converged pairs are locked into Q so that
    "the new approximate eigenpair is orthogonal to those that have already been
    computed" (l.399-402);
  * correction equation (I - Q~Q~^T)(A - theta I)(I - Q~Q~^T) z = -r, Q~ = [Q, u]
    (l.390-393, l.399-401), solved approximately by SQMR with the projected
    preconditioner (I - Y H^{-1} Q~^T) K^{-1}, Y = K^{-1} Q~, H = Q~^T Y (the block
    form of (I - u w^T/w^T u) K^{-1}, l.414-416); the shift is sigma until
    ||r|| < switch_tol ||A|| ("accuracy ... uncritical until the approximate
    eigenpair converges", l.417-419), theta afterwards;
  * expansion "by reorthogonalizing z with respect to [v_1..v_k]" (l.396-397),
    thick restart to jmin Ritz vectors at jmax.
"""
import numpy as np

from .sqmr import sqmr


def jd_nearest(A, K, k, sigma=0.0, tol=1e-10, jmin=10, jmax=25, inner_tol=0.1, inner_max=60,
               switch_tol=1e-3, max_outer=2000, v0=None, seed=7):
    """k eigenpairs of sparse symmetric A nearest sigma.  K: callable r -> K^{-1} r
    (preconditioner for A - sigma I).  Returns (lam, X, stats)."""
    n = A.shape[0]
    normA = abs(A).sum(axis=0).max()
    tol_abs = tol * normA
    rng = np.random.default_rng(seed)
    z = rng.uniform(-0.5, 0.5, n) if v0 is None else np.array(v0, dtype=np.float64)
    Q = np.zeros((n, 0))
    KQ = np.zeros((n, 0))
    lam = []
    V = np.zeros((n, 0))
    AV = np.zeros((n, 0))
    outer = inner = 0
    op_s = lambda v: A @ v - sigma * v  # noqa: E731
    while True:
        for _ in range(2):                                    # CGS2 against [Q, V]
            z = z - Q @ (Q.T @ z)
            z = z - V @ (V.T @ z)
        nz = np.linalg.norm(z)
        if nz == 0.0:
            z = rng.uniform(-0.5, 0.5, n)
            continue
        z = z / nz
        V = np.column_stack([V, z])
        AV = np.column_stack([AV, op_s(z)])
        while True:
            M = V.T @ AV
            M = 0.5 * (M + M.T)
            th, S = np.linalg.eigh(M)
            o = np.lexsort((th, np.abs(th)))
            th, S = th[o], S[:, o]
            u = V @ S[:, 0]
            r = AV @ S[:, 0] - th[0] * u
            rn = np.linalg.norm(r)
            if rn > tol_abs:
                break
            Q = np.column_stack([Q, u])
            KQ = np.column_stack([KQ, K(u)])
            lam.append(sigma + th[0])
            if len(lam) == k:
                return np.array(lam), Q, dict(outer=outer, inner=inner)
            V, AV = V @ S[:, 1:], AV @ S[:, 1:]
            if V.shape[1] == 0:
                break
        if V.shape[1] == 0:
            z = rng.uniform(-0.5, 0.5, n)
            continue
        if outer >= max_outer:
            raise RuntimeError("jd_nearest: max_outer reached")
        if V.shape[1] >= jmax:
            V, AV = V @ S[:, :jmin], AV @ S[:, :jmin]
        Qt = np.column_stack([Q, u])
        Y = np.column_stack([KQ, K(u)])
        Hi = np.linalg.inv(0.5 * ((Qt.T @ Y) + (Qt.T @ Y).T))
        shift = th[0] if rn < switch_tol * normA else 0.0

        def op(q, s=sigma + shift):
            t = A @ q - s * q
            return t - Qt @ (Qt.T @ t)

        def prec(rr):
            w = K(rr)
            return w - Y @ (Hi @ (Qt.T @ w))

        b = -(r - Qt @ (Qt.T @ r))
        z, it, _, _ = sqmr(op, prec, b, tol=inner_tol, maxit=inner_max)
        inner += it
        outer += 1
