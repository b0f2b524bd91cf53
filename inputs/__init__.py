"""Seeded synthetic inputs shared by the oracle-side and GPU-side tests.

Holds NONE of the method's arithmetic: only seeded random vectors / shapes.
(The Anderson disorder itself is not generated here -- both the oracle and
the CUDA path implement the same SplitMix64 counter stream, R3.)
"""
import numpy as np


def rand_vec(n, seed, kind="normal"):
    rng = np.random.default_rng(seed)
    if kind == "normal":
        return rng.standard_normal(n)
    if kind == "uniform":
        return rng.uniform(-0.5, 0.5, n)
    raise ValueError(kind)


def rand_block(n, m, seed):
    """n x m column block (column-major contiguous columns)."""
    rng = np.random.default_rng(seed)
    return np.asfortranarray(rng.standard_normal((n, m)))


# BASELINE.json configs: (L, W, seed, hop, k, sigma, tol)
CONFIGS = {
    0: dict(L=10, W=16.5, seed=0, hop=-1.0, k=5, sigma=0.0, tol=1e-10),
    1: dict(L=50, W=16.5, seed=1, hop=-1.0, k=5, sigma=0.0, tol=1e-10),
    2: dict(L=100, W=16.5, seed=2, hop=-1.0, k=5, sigma=0.0, tol=1e-10),
    3: dict(L=200, W=16.5, seed=3, hop=-1.0, k=5, sigma=0.0, tol=1e-10),
    4: dict(L=250, W=16.5, seed=4, hop=-1.0, k=5, sigma=0.0, tol=1e-10),
}
