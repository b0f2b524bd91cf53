"""Simplified QMR (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

PAPER.md sect. 4.2 l.412-416 ("the simplified QMR method [FreN95, FreJ97]
using the preconditioner ...") and sect. 7.4 l.986-987.  The paper cites but
does not print the recurrences; this is the symmetric QMR of Freund & Jarre
(1997) with a symmetric (indefinite) preconditioner M^{-1}: one product with
the operator and one with M^{-1} per step, coupled two-term recurrences,
plus the recursively updated QMR residual r_x = b - A x (reading R13) used for
the stopping test ||b - A x|| <= tol ||b||.
"""
import numpy as np


def sqmr(op, prec, b, tol=1e-10, maxit=1000, x0=None):
    """Solve op(x) = b.  op, prec: callables (symmetric linear operators).
    Returns (x, iterations, relative recursive residual, history)."""
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return np.zeros_like(b), 0, 0.0, []
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
    r = b - op(x) if x0 is not None else b.copy()
    rx = r.copy()
    tau = np.linalg.norm(r)
    q = prec(r)
    rho = r @ q
    theta = 0.0
    d = np.zeros_like(b)
    s = np.zeros_like(b)
    hist = []
    res = np.linalg.norm(rx) / nb
    for j in range(1, maxit + 1):
        t = op(q)
        sig = q @ t
        if sig == 0.0 or rho == 0.0:
            break                                   # breakdown (reported via res)
        alpha = rho / sig
        r = r - alpha * t
        th = np.linalg.norm(r) / tau
        c2 = 1.0 / (1.0 + th * th)
        tau = tau * th * np.sqrt(c2)
        d = (c2 * theta * theta) * d + (c2 * alpha) * q
        s = (c2 * theta * theta) * s + (c2 * alpha) * t
        theta = th
        x = x + d
        rx = rx - s
        res = np.linalg.norm(rx) / nb
        hist.append(res)
        if res <= tol:
            return x, j, res, hist
        u = prec(r)
        rho_new = r @ u
        beta = rho_new / rho
        rho = rho_new
        q = u + beta * q
    return x, j, res, hist
