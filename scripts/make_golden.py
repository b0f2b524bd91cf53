"""Write tests/golden/*.json from the ORACLE ONLY (never from the CUDA path).

Usage: python scripts/make_golden.py [config ...]
  config 0: L=10 dense diagonalisation (BASELINE.json configs[0])
  config 1: L=50 plain shift-and-invert Lanczos, direct inner solve (configs[1])
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from inputs import CONFIGS  # noqa: E402
from oracle import anderson as an  # noqa: E402
from oracle import eigs  # noqa: E402


def main(which):
    for c in which:
        cfg = CONFIGS[c]
        L, W, seed, hop, k, sigma = (cfg[x] for x in ("L", "W", "seed", "hop", "k", "sigma"))
        eps = an.disorder(L, W, seed)
        A = an.matrix(L, eps, hop=hop)
        t0 = time.time()
        if L <= 14:
            lam, X = eigs.dense_nearest(A, k, sigma)
            res = np.linalg.norm(A @ X - X * lam, axis=0)
            method = "dense numpy.linalg.eigh"
        else:
            solve = eigs.iterative_solver(A, sigma, L=L, tol=1e-14)
            lam, X, res = eigs.si_lanczos_nearest(A, k + 3, sigma, tol=1e-12, solve=solve)
            method = ("plain shift-and-invert Lanczos (full reorth.), inner solves by oracle SQMR + oracle "
                      f"multilevel ILDL to 1e-14: {solve.stats}")
        dt = time.time() - t0
        normA = float(abs(A).sum(axis=0).max())
        out = dict(config=c, L=L, W=W, seed=seed, hop=hop, sigma=sigma, k=k,
                   eigenvalues=[float(v) for v in lam], residuals=[float(v) for v in res],
                   normA_1=normA, method=method, oracle_seconds=dt,
                   source="scripts/make_golden.py -> oracle/ only")
        path = os.path.join(ROOT, "tests", "golden", f"eigs_config{c}.json")
        if L > 14:
            # eigenvectors of the k nearest pairs for the subspace-angle test (fp64, one column each)
            vpath = os.path.join(ROOT, "tests", "golden", f"eigvecs_config{c}.npz")
            np.savez_compressed(vpath, X=np.ascontiguousarray(X[:, :k].T))
            out["eigenvectors"] = os.path.basename(vpath)
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
        print(path, lam, dt)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [0])
