"""Reading R8 against the paper's pivoting: the locally dominant (mutual strongest-neighbour)
matching used for the 2x2 pivots versus a true maximum-weight bipartite matching (PAPER.md
l.577-587, l.623-677: maximise prod |a_{i,pi(i)}|, then split the cycles of pi into 1x1 / 2x2
blocks).  CPU experiment on the oracle's level matrices (scipy's min_weight_full_bipartite_matching
on the costs log(max|a|) - log|a_ij| + 1); prints, per level, the cycle structure of the
maximum-weight permutation, the mutual-proposal pairs, their overlap, and log prod |a_{i,pi(i)}| of
both.  python scripts/matching_compare.py [L] [W] [seed] [levels]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402
from scipy.sparse.csgraph import min_weight_full_bipartite_matching  # noqa: E402

from oracle import anderson as an, mlildl  # noqa: E402


def analyse(A):
    D, Ah = mlildl._scaled(A)
    n = Ah.shape[0]
    dg, lmax1, d1, p = mlildl._pivot_quality(Ah)
    idx = np.arange(n)
    has = p >= 0
    mutual = has.copy()
    mutual[has] = p[p[has]] == idx[has]
    coo = Ah.tocoo()
    absv = np.abs(coo.data)
    keep = absv > 0
    cost = sp.csr_matrix((np.log(absv[keep].max()) - np.log(absv[keep]) + 1.0, (coo.row[keep], coo.col[keep])),
                         shape=(n, n))
    rows, cols = min_weight_full_bipartite_matching(cost)
    pi = np.empty(n, dtype=np.int64)
    pi[rows] = cols
    fixed = pi == idx
    two = (pi[pi] == idx) & ~fixed
    # cycle lengths
    seen = np.zeros(n, bool)
    longer = 0
    for s in np.where(~fixed & ~two)[0]:
        if seen[s]:
            continue
        j, ln = s, 0
        while not seen[j]:
            seen[j] = True
            j = pi[j]
            ln += 1
        longer += ln
    absA = abs(Ah).tocsr()
    lw_match = float(np.sum(np.log(np.asarray(absA[idx, pi]).ravel())))
    # the permutation our rule implies: mutual pairs in which a member fails the 1x1 bound, else identity
    kappa = 5.0
    ok1 = (lmax1 <= kappa - 1) & (dg != 0)
    cand = mutual & ~(ok1 & ok1[np.maximum(p, 0)])
    ours = idx.copy()
    ours[cand] = p[cand]
    with np.errstate(divide="ignore"):
        lw_ours = float(np.sum(np.log(np.asarray(absA[idx, ours]).ravel())))
    both = two & cand & (pi == p)
    return dict(n=int(n), nnz_per_row=float(Ah.nnz / n), mwm_fixed=float(fixed.mean()), mwm_two_cycles=float(two.mean()),
                mwm_longer=float(longer / n), mutual_pairs_all=float(mutual.mean()), ours_pairs=float(cand.mean()),
                ours_in_mwm_two=float(both.sum() / max(1, cand.sum())),
                mwm_two_in_ours=float(both.sum() / max(1, two.sum())), fail_1x1=float((~ok1).mean()),
                fail_1x1_unpaired_ours=float((~ok1 & ~cand).mean()), fail_1x1_unpaired_mwm=float((~ok1 & fixed).mean()),
                logprod_mwm=lw_match, logprod_ours=lw_ours)


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 14
    W = float(sys.argv[2]) if len(sys.argv) > 2 else 16.5
    seed = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    nlev = int(sys.argv[4]) if len(sys.argv) > 4 else 6
    eps = an.disorder(L, W, seed)
    A = an.matrix(L, eps, hop=-1.0, sigma=0.0)
    td = (1.0 / np.sqrt(L ** 3)) / 5.0
    M = mlildl.MultilevelILDL(A, lattice_L=L, kappa=5.0, tau_drop=td, tau_strong=40 * td, n_coarse_max=256,
                              max_levels=nlev, stall_frac=0.005, dense_cap=1 << 20)
    mats = [sp.csr_matrix(A)] + [lv.S for lv in M.levels[:-1]]
    for l, (Al, lv) in enumerate(zip(mats, M.levels)):
        out = analyse(Al)
        out.update(level=l, L=L, W=W, seed=seed, accepted_pairs=int(lv.npairs), nF=int(len(lv.F)))
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
