"""Multilevel incomplete LDL^T preconditioner (TEST INFRASTRUCTURE ONLY -- see
oracle/__init__.py).

Follows PAPER.md sect. 7 (l.790-973) step by step, in the independent-set
reading fixed in DESIGN.md sect. 3.3 (readings R6-R12).  Per level l, with the
level matrix A_l (symmetric, explicit diagonal):

 (i)  Reordering/scaling, sect. 7.1 (l.800-819): D_i = 1/sqrt(max_j |a_ij|),
      A^ = D A D computed as a_ij * (D_i * D_j).
 (ii) Pivot selection, sect. 7.2 (l.821-915):
      - 1x1 quality: lmax1_f = max_{j!=f}|a^_jf| / |a^_ff|,
        d1_f = sum_{j!=f}|a^_jf| / |a^_ff|                      (paper's d_1, l.866)
      - 2x2 pivots from a symmetric matching, sect. 6.2 (l.623-677): every node
        proposes its strongest neighbour p(i) = argmax_{j!=i}|a^_ij|; mutual
        proposals {i, p(i)} in which at least one member fails the 1x1 bound
        become 2x2 candidates B = [[a^_ii, a^_ij],[a^_ij, a^_jj]]; accepted iff
        det B != 0, d2 < d1_lead (the paper's "2x2 update only if d2 < d1",
        l.874) and lmax2 <= kappa-1.
      - inverse-based bound (l.884-896): the new block column of L may not push
        ||L^{-1}||_inf above kappa: each single column entry |l_cf| <= kappa-1
        (candidate test) and every row sum of |L| <= kappa-1 (budget repair);
        violators are postponed to the next level (l.895-897).
      - level 0 on the lattice: the red sites of the bipartite split
        (reading R6); levels > 0: a maximal independent set of candidate
        blocks in the strong graph |a^_ij| >= tau_strong, lowest (quality,
        leader) first, synchronous rounds (reading R9).
 (iii) Factor: L = A^_CF B^{-1} (entries < tau_drop dropped, the paper's
      "drop these entries whenever their absolute value is less than
      eps/kappa", l.909-911), S = A^_CC - A^_CF B^{-1} A^_FC symmetrised and
      off-diagonals < tau_drop dropped (reading R10).  F-F couplings (all weak
      by construction of the independent set) are dropped, or, with
      compensate=True (reading R17), those >= tau_virtual enter B^{-1} to first
      order as virtual 2x2 blocks (in L with fill, in S on the pattern only).
 (iv) Recursion on S (sect. 7.3, l.917-945) until n <= n_coarse_max, the level
      cap, or a level eliminates < stall_frac*n nodes; the last Schur
      complement is inverted densely.
Application (sect. 7.4 l.975-987 / reading R11): z = M^{-1} r with the block
forward / backward substitution, L_21 applied from its stored (dropped) entries.
"""
import numpy as np
import scipy.sparse as sp

from .anderson import red_sites


class Level:
    pass


def _unique_inverse(keys):
    """np.unique(keys, return_inverse=True) by sorting (numpy's hash-based
    unique is pathologically slow on large int64 keys)."""
    keys = np.asarray(keys)
    order = np.argsort(keys, kind="stable")
    ks = keys[order]
    first = np.ones(len(ks), bool)
    first[1:] = ks[1:] != ks[:-1]
    uniq = ks[first]
    inv = np.empty(len(keys), dtype=np.int64)
    inv[order] = np.cumsum(first) - 1
    return uniq, inv


def _unique(keys):
    return _unique_inverse(keys)[0]


def _scaled(A):
    A = sp.csr_matrix(A)
    A.sort_indices()
    n = A.shape[0]
    coo = A.tocoo()
    r, c, v = coo.row, coo.col, coo.data
    rowmax = np.zeros(n)
    np.maximum.at(rowmax, r, np.abs(v))
    D = np.where(rowmax > 0, 1.0 / np.sqrt(np.where(rowmax > 0, rowmax, 1.0)), 1.0)
    ah = v * (D[r] * D[c])
    Ah = sp.csr_matrix((ah, (r, c)), shape=(n, n))
    Ah.sort_indices()
    return D, Ah


def _pivot_quality(Ah):
    n = Ah.shape[0]
    coo = Ah.tocoo()
    r, c, v = coo.row, coo.col, coo.data
    off = r != c
    dg = Ah.diagonal()
    cm = np.zeros(n)
    np.maximum.at(cm, r[off], np.abs(v[off]))
    osum = np.zeros(n)
    np.add.at(osum, r[off], np.abs(v[off]))
    adg = np.abs(dg)
    with np.errstate(divide="ignore", invalid="ignore"):
        lmax1 = np.where(adg > 0, cm / np.where(adg > 0, adg, 1.0), np.inf)
        d1 = np.where(adg > 0, osum / np.where(adg > 0, adg, 1.0), np.inf)
    # strongest neighbour proposal p(i) (ties -> smallest j)
    p = np.full(n, -1, dtype=np.int64)
    ro, co, vo = r[off], c[off], np.abs(v[off])
    order = np.lexsort((co, -vo, ro))
    ro, co = ro[order], co[order]
    first = np.ones(len(ro), bool)
    first[1:] = ro[1:] != ro[:-1]
    p[ro[first]] = co[first]
    return dg, lmax1, d1, p


def _pair_candidates(Ah, dg, lmax1, d1, p, kappa):
    """2x2 pivots from mutual strongest-neighbour proposals (sect. 6.2 / 7.2)."""
    n = Ah.shape[0]
    ok1 = (lmax1 <= kappa - 1) & (dg != 0)
    pairs = []
    idx = np.arange(n)
    has = p >= 0
    mutual = has.copy()
    mutual[has] = p[p[has]] == idx[has]
    cand = np.where(mutual & (idx < p) & ~(ok1 & ok1[np.maximum(p, 0)]))[0]
    ip, ix, dv = Ah.indptr, Ah.indices, Ah.data
    for i in cand:
        j = int(p[i])
        ci, vi = ix[ip[i]:ip[i + 1]], dv[ip[i]:ip[i + 1]]
        cj, vj = ix[ip[j]:ip[j + 1]], dv[ip[j]:ip[j + 1]]
        aii, ajj = dg[i], dg[j]
        aij = vi[np.searchsorted(ci, j)]
        det = aii * ajj - aij * aij
        if det == 0.0:
            continue
        B11, B12, B22 = ajj / det, -aij / det, aii / det
        # union of the neighbours of i and j except i, j, ascending
        nbrs = np.union1d(ci, cj)
        nbrs = nbrs[(nbrs != i) & (nbrs != j)]
        ai = np.zeros(len(nbrs))
        aj = np.zeros(len(nbrs))
        mi = np.isin(nbrs, ci)
        mj = np.isin(nbrs, cj)
        ai[mi] = vi[np.searchsorted(ci, nbrs[mi])]
        aj[mj] = vj[np.searchsorted(cj, nbrs[mj])]
        w = np.abs(ai * B11 + aj * B12) + np.abs(ai * B12 + aj * B22)
        lm2 = float(w.max()) if len(w) else 0.0
        d2 = 0.0
        for x in w:                      # sequential sum in ascending column order
            d2 += x
        lead = i if not ok1[i] else j
        if d2 < d1[lead] and lm2 <= kappa - 1:
            pairs.append((i, j, B11, B12, B22, lm2, d2))
    return pairs


def _mis(nb, keyrank, edges_a, edges_b):
    """Synchronous maximal independent set on blocks (reading R9): a block
    wins when its rank is below every undecided neighbour's rank."""
    und = np.ones(nb, bool)
    sel = np.zeros(nb, bool)
    rounds = 0
    while und.any():
        rounds += 1
        ru = np.where(und, keyrank, np.iinfo(np.int64).max)
        nbmin = np.full(nb, np.iinfo(np.int64).max)
        np.minimum.at(nbmin, edges_a, ru[edges_b])
        win = und & (keyrank < nbmin)
        sel |= win
        hit = np.zeros(nb, bool)
        hit[edges_a[win[edges_b]]] = True
        und &= ~win & ~hit
    return sel, rounds


def factor_level(A, kappa, tau_drop, tau_strong, lattice_L=None, stall_frac=0.005, compensate=True,
                 tau_virtual=None, priority="quality", red=None):
    """One level.  Level 0 of a lattice (lattice_L given, or an explicit `red` mask for a
    z-slab block, DESIGN.md sect. 6) takes the red sites as its independent set."""
    n = A.shape[0]
    D, Ah = _scaled(A)
    dg, lmax1, d1, p = _pivot_quality(Ah)
    ok1 = (lmax1 <= kappa - 1) & (dg != 0)

    # ---- blocks: accepted 2x2 pairs and 1x1 singles -------------------------
    partner = np.full(n, -1, dtype=np.int64)
    b11 = np.zeros(n)
    b12 = np.zeros(n)
    lattice = lattice_L is not None or red is not None
    if not lattice:
        pairs = _pair_candidates(Ah, dg, lmax1, d1, p, kappa)
    else:
        pairs = []
    leader = np.full(n, -1, dtype=np.int64)     # block leader of each candidate node
    q = np.full(n, np.inf)                      # block quality (at the leader)
    for (i, j, B11, B12, B22, lm2, _d2) in pairs:
        partner[i], partner[j] = j, i
        b11[i], b12[i] = B11, B12
        b11[j], b12[j] = B22, B12
        leader[i] = leader[j] = i
        q[i] = lm2
    singles = ok1 & (partner < 0)
    leader[singles] = np.where(singles)[0]
    q[singles] = lmax1[singles]
    with np.errstate(divide="ignore"):
        b11[singles] = 1.0 / dg[singles]

    # ---- independent set ------------------------------------------------------
    if lattice:
        inF = singles & (red if red is not None else red_sites(lattice_L))
        rounds = 0
    else:
        blk = np.where(leader == np.arange(n))[0]           # block ids = leaders
        nb = len(blk)
        bid = np.full(n, -1, dtype=np.int64)
        pos = np.full(n, -1, dtype=np.int64)
        pos[blk] = np.arange(nb)
        m = leader >= 0
        bid[m] = pos[leader[m]]
        keyrank = np.empty(nb, dtype=np.int64)
        if priority == "degree":
            rl = np.diff(Ah.indptr)
            deg = rl[blk] + np.where(partner[blk] >= 0, rl[np.maximum(partner[blk], 0)], 0)
            keyrank[np.lexsort((blk, q[blk], deg))] = np.arange(nb)
        else:
            keyrank[np.lexsort((blk, q[blk]))] = np.arange(nb)
        coo = Ah.tocoo()
        r, c, v = coo.row, coo.col, coo.data
        strong = (r != c) & (np.abs(v) >= tau_strong) & (bid[r] >= 0) & (bid[c] >= 0)
        ea, eb = bid[r[strong]], bid[c[strong]]
        keep = ea != eb
        sel, rounds = _mis(nb, keyrank, ea[keep], eb[keep])
        inF = np.zeros(n, bool)
        inF[m] = sel[bid[m]]

    # ---- row-budget repair: rows of L^{-1} bounded by kappa (l.884-897) -------
    coo = Ah.tocoo()
    r, c, v = coo.row, coo.col, coo.data
    off = r != c
    r, c, v = r[off], c[off], v[off]
    repair_rounds = 0
    while True:
        Lfull = _lfull(Ah, inF, partner, b11, b12, dg)
        Lc = Lfull.tocoo()
        rows_c = Lc.row.astype(np.int64)    # level indices of C nodes (int64: n^2 keys)
        lead_of = np.where(partner[Lc.col] >= 0, np.minimum(Lc.col, partner[Lc.col]), Lc.col)
        w = np.abs(Lc.data)
        # aggregate per (c, block)
        key = rows_c * n + lead_of
        uk, inv = _unique_inverse(key)
        wb = np.zeros(len(uk))
        np.add.at(wb, inv, w)
        bc, bl = uk // n, uk % n
        budget = np.zeros(n)
        np.add.at(budget, bc, wb)
        viol = budget > kappa - 1
        if not viol.any():
            break
        repair_rounds += 1
        # nominate the largest contributor per violating row (ties -> smallest leader)
        mv = viol[bc]
        o = np.lexsort((bl[mv], -wb[mv], bc[mv]))
        cc, ll = bc[mv][o], bl[mv][o]
        firstc = np.ones(len(cc), bool)
        firstc[1:] = cc[1:] != cc[:-1]
        rm = ll[firstc]
        inF[rm] = False
        pr = partner[rm]
        inF[pr[pr >= 0]] = False

    nF = int(inF.sum())
    if nF < stall_frac * n:
        return None

    # ---- factor ------------------------------------------------------------------
    Lv = Level()
    Lv.n = n
    Lv.D = D
    Lv.inF = inF
    Lv.F = np.where(inF)[0]
    Lv.C = np.where(~inF)[0]
    Lv.partner = np.where(inF, partner, -1)
    Lv.b11 = np.where(inF, b11, 0.0)
    Lv.b12 = np.where(inF & (partner >= 0), b12, 0.0)
    Lv.npairs = int(((partner >= 0) & inF).sum() // 2)
    Lv.rounds = rounds
    Lv.repair_rounds = repair_rounds
    cmap = np.full(n, -1, dtype=np.int64)
    cmap[Lv.C] = np.arange(len(Lv.C))
    Lv.cmap = cmap
    tv = 5.0 * tau_drop if tau_virtual is None else tau_virtual
    blocks = _blocks(Ah, inF, partner, b11, b12, compensate, tv)
    Lv.nvirtual = int((blocks["kind"] == 2).sum())
    inc = _incidence(Ah, inF, blocks)
    lt = _l_terms(inc, blocks, n)
    Lv.L = _l_rows(lt, n, cmap, len(Lv.C), tau_drop)
    Lv.S = _schur(Ah, inF, lt, Lv.C, cmap, tau_drop)
    Lv.Binv = _binv_blocks(n, blocks)
    return Lv


def _blocks(Ah, inF, partner, b11, b12, compensate, tau_virtual=0.0):
    """Pivot blocks of a level plus, with `compensate` (reading R17), one virtual
    2x2 block per coupling |a^_uv| >= tau_virtual between two pivot singles u < v: B' = [[0, b'],
    [b', 0]], b' = -(a^_uv (B_uu B_vv)) -- the first-order term of
    B^{-1} = (B_d + E)^{-1} ~ B_d^{-1} - B_d^{-1} E B_d^{-1}.  Key = (lmin, lmax)."""
    n = Ah.shape[0]
    F = np.where(inF)[0]
    rows = []
    for f in F:
        g = partner[f]
        if g < 0:
            rows.append((f, f, f, -1, b11[f], 0.0, 0.0, 0))
        elif f < g:
            rows.append((f, g, f, g, b11[f], b12[f], b11[g], 1))
    if compensate:
        coo = Ah.tocoo()
        r, c, v = coo.row.astype(np.int64), coo.col.astype(np.int64), coo.data
        m = (r < c) & inF[r] & inF[c] & (partner[r] < 0) & (partner[c] < 0) & (np.abs(v) >= tau_virtual)
        for u, w, a in zip(r[m], c[m], v[m]):
            rows.append((u, w, u, w, 0.0, -(a * (b11[u] * b11[w])), 0.0, 2))
    a = np.array(rows, dtype=object) if rows else np.zeros((0, 8), dtype=object)
    blk = {}
    blk["kmin"] = np.array([x[0] for x in rows], dtype=np.int64)
    blk["kmax"] = np.array([x[1] for x in rows], dtype=np.int64)
    blk["f"] = np.array([x[2] for x in rows], dtype=np.int64)
    blk["g"] = np.array([x[3] for x in rows], dtype=np.int64)
    blk["Bff"] = np.array([x[4] for x in rows], dtype=np.float64)
    blk["Bfg"] = np.array([x[5] for x in rows], dtype=np.float64)
    blk["Bgg"] = np.array([x[6] for x in rows], dtype=np.float64)
    blk["kind"] = np.array([x[7] for x in rows], dtype=np.int64)
    blk["key"] = blk["kmin"] * n + blk["kmax"]
    del a
    return blk


def _incidence(Ah, inF, blk):
    """Elements (C row c, block b) for every block with a member adjacent to c:
    a_cf, a_cg = a^ from c to the block's first / second member (0 if absent),
    hf, hg = whether that member is adjacent (structurally) to c."""
    n = Ah.shape[0]
    coo = Ah.tocoo()
    r, c, v = coo.row.astype(np.int64), coo.col.astype(np.int64), coo.data
    m = (~inF[r]) & inF[c]
    rc, uc, av = r[m], c[m], v[m]
    nb = len(blk["f"])
    # member -> blocks containing it (as first or second member)
    mem_b = np.concatenate([np.arange(nb), np.arange(nb)[blk["g"] >= 0]])
    mem_x = np.concatenate([blk["f"], blk["g"][blk["g"] >= 0]])
    mem_pos = np.concatenate([np.zeros(nb, np.int64), np.ones(int((blk["g"] >= 0).sum()), np.int64)])
    o = np.argsort(mem_x, kind="stable")
    mem_b, mem_x, mem_pos = mem_b[o], mem_x[o], mem_pos[o]
    start = np.searchsorted(mem_x, uc, side="left")
    stop = np.searchsorted(mem_x, uc, side="right")
    cnt = stop - start
    rep = np.repeat(np.arange(len(uc)), cnt)
    off = np.arange(len(rep)) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    idx = np.repeat(start, cnt) + off
    e_c, e_b, e_pos, e_a = rc[rep], mem_b[idx], mem_pos[idx], av[rep]
    key = e_c * nb + e_b
    uk, inv = _unique_inverse(key)
    acf = np.zeros(len(uk))
    acg = np.zeros(len(uk))
    hf = np.zeros(len(uk), bool)
    hg = np.zeros(len(uk), bool)
    acf[inv[e_pos == 0]] = e_a[e_pos == 0]
    acg[inv[e_pos == 1]] = e_a[e_pos == 1]
    hf[inv[e_pos == 0]] = True
    hg[inv[e_pos == 1]] = True
    return dict(c=uk // nb, b=uk % nb, acf=acf, acg=acg, hf=hf, hg=hg)


def _l_terms(inc, blk, n):
    """Split row factor L = A^_CF B~^{-1} = L^r + L^v (reading R17).
    L^r (real blocks, B_d^{-1}): for every (c, real block b) the members x of b get
      l^r_cf = a_cf B_ff + a_cg B_gf,  l^r_cg = a_cf B_fg + a_cg B_gg   (singles: a_cf B_ff),
    one entry per (c, x) (structural: also when the value is 0).
    L^v (virtual blocks {f, g}, B~^{-1}_fg = b'): for c adjacent to f, x = g gets a_cf b';
    for c adjacent to g, x = f gets a_cg b'; l^v_cx = sum of its terms in ascending block key
    from 0.  Returns the (c, x) entries of both with their values and flags."""
    b = inc["b"]
    c = inc["c"]
    kind = blk["kind"][b]
    f, g = blk["f"][b], blk["g"][b]
    Bff, Bfg, Bgg = blk["Bff"][b], blk["Bfg"][b], blk["Bgg"][b]
    acf, acg, hf, hg = inc["acf"], inc["acg"], inc["hf"], inc["hg"]
    key = blk["key"][b]
    real = kind != 2
    single = g < 0
    pair = real & ~single
    vf = np.where(single, acf * Bff, acf * Bff + acg * Bfg)
    vg = acf * Bfg + acg * Bgg
    rc = np.concatenate([c[real], c[pair]])
    rx = np.concatenate([f[real], g[pair]])
    rv = np.concatenate([vf[real], vg[pair]])
    virt = kind == 2
    m1, m2 = virt & hf, virt & hg
    vc = np.concatenate([c[m1], c[m2]])
    vx = np.concatenate([g[m1], f[m2]])
    vt = np.concatenate([acf[m1] * Bfg[m1], acg[m2] * Bfg[m2]])
    vk = np.concatenate([key[m1], key[m2]])
    o = np.lexsort((vk, vx, vc))                       # per (c, x): ascending block key
    vc, vx, vt = vc[o], vx[o], vt[o]
    vuk, vinv = _unique_inverse(vc * n + vx)
    lv = np.zeros(len(vuk))
    np.add.at(lv, vinv, vt)                            # sequential, in that order
    rk = rc * n + rx
    allk = _unique(np.concatenate([rk, vuk]))
    Lr = np.zeros(len(allk))
    Lvv = np.zeros(len(allk))
    isr = np.zeros(len(allk), bool)
    isv = np.zeros(len(allk), bool)
    pr = np.searchsorted(allk, rk)
    pv = np.searchsorted(allk, vuk)
    Lr[pr] = rv
    isr[pr] = True
    Lvv[pv] = lv
    isv[pv] = True
    return dict(c=allk // n, x=allk % n, lr=Lr, lv=Lvv, real=isr, virt=isv)


def _l_rows(lt, n, cmap, nC, tau_drop):
    """L_cx = l^r_cx + l^v_cx (one rounding), |L| < tau_drop dropped."""
    val = lt["lr"] + lt["lv"]
    keep = np.abs(val) >= tau_drop
    L = sp.csr_matrix((val[keep], (cmap[lt["c"][keep]], lt["x"][keep])), shape=(nC, n))
    L.sort_indices()
    return L


def _schur(Ah, inF, lt, C, cmap, tau_drop):
    """S = A^_CC - L^r A^_FC - P o (L^v A^_FC) (readings R10/R17),
    upper triangle computed, lower triangle its mirror:
    s_cc' starts at a^_cc'; then the real terms l^r_cx a^_c'x are subtracted for x ascending
    (creating fill), then the virtual terms l^v_cx a^_c'x for x ascending, only on the
    pattern P of A^_CC and the real terms; each term is the rounded product.  Off-diagonals
    |s| < tau_drop are dropped.  (Pinned to the plain matrix definition in
    tests/test_oracle_mlildl.py::test_ordered_accumulation_equals_plain_definition.)"""
    n = Ah.shape[0]
    nC = len(C)
    Ah = sp.csr_matrix(Ah)
    coo = Ah.tocoo()
    r, cc, v = coo.row.astype(np.int64), coo.col.astype(np.int64), coo.data
    # FC(x): the coarse neighbours of each pivot x (structural)
    mfc = inF[r] & ~inF[cc]
    fr, fcol, fval = r[mfc], cmap[cc[mfc]], v[mfc]
    o = np.lexsort((fcol, fr))
    fr, fcol, fval = fr[o], fcol[o], fval[o]
    start = np.searchsorted(fr, lt["x"], side="left")
    stop = np.searchsorted(fr, lt["x"], side="right")
    cnt = stop - start
    rep = np.repeat(np.arange(len(lt["x"])), cnt)
    off = np.arange(len(rep)) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    idx = np.repeat(start, cnt) + off
    tc = cmap[lt["c"][rep]]
    tc2 = fcol[idx]
    tx = lt["x"][rep]
    a = fval[idx]
    tk = tc * nC + tc2
    realt = lt["real"][rep]
    virtt = lt["virt"][rep]
    mc = (~inF[r]) & (~inF[cc])
    k0 = cmap[r[mc]] * nC + cmap[cc[mc]]
    keys = _unique(np.concatenate([k0, tk[realt], np.arange(nC) * (nC + 1)]))
    sval = np.zeros(len(keys))
    sval[np.searchsorted(keys, k0)] = v[mc]
    # real terms (all on the pattern by construction), then virtual terms on the pattern
    pos_r = np.searchsorted(keys, tk[realt])
    T_r = lt["lr"][rep][realt] * a[realt]
    pv = np.minimum(np.searchsorted(keys, tk[virtt]), max(len(keys) - 1, 0))
    onp = keys[pv] == tk[virtt] if len(keys) else np.zeros(int(virtt.sum()), bool)
    pos_v = pv[onp]
    T_v = (lt["lv"][rep][virtt] * a[virtt])[onp]
    x_r, x_v = tx[realt], tx[virtt][onp]
    pos = np.concatenate([pos_r, pos_v])
    T = np.concatenate([T_r, T_v])
    ps = np.concatenate([np.zeros(len(pos_r), np.int64), np.ones(len(pos_v), np.int64)])
    xx = np.concatenate([x_r, x_v])
    ot = np.lexsort((xx, ps, pos))                     # per entry: real then virtual, x ascending
    np.subtract.at(sval, pos[ot], T[ot])
    sr, sc = keys // nC, keys % nC
    # S is symmetric: its upper triangle (c <= c') is taken as computed in row c and
    # mirrored, S = triu(S) + triu(S, 1)^T, so S is symmetric bit for bit (the rounded
    # terms l_cx a_c'x are not symmetric in (c, c'))
    keep = (sr == sc) | ((sr < sc) & (np.abs(sval) >= tau_drop))
    ur, uc, uv = sr[keep], sc[keep], sval[keep]
    off = ur != uc
    S = sp.csr_matrix((np.concatenate([uv, uv[off]]), (np.concatenate([ur, uc[off]]), np.concatenate([uc, ur[off]]))),
                      shape=(nC, nC))
    S.sort_indices()
    return S


def _binv_blocks(n, blk):
    """B~^{-1} on the pivot nodes: block inverses plus the virtual couplings."""
    f, g = blk["f"], blk["g"]
    two = g >= 0
    rows = np.concatenate([f, g[two], f[two], g[two]])
    cols = np.concatenate([f, g[two], g[two], f[two]])
    vals = np.concatenate([blk["Bff"], blk["Bgg"][two], blk["Bfg"][two], blk["Bfg"][two]])
    keep = vals != 0.0
    return sp.csr_matrix((vals[keep], (rows[keep], cols[keep])), shape=(n, n))


def _binv(n, inF, partner, b11, b12):
    """Block-diagonal B^{-1} on F nodes (1x1: 1/a^_ff; 2x2: inverse of the pair)."""
    f = np.where(inF)[0]
    rows = [f]
    cols = [f]
    vals = [b11[f]]
    pf = f[partner[f] >= 0]
    rows.append(pf)
    cols.append(partner[pf])
    vals.append(b12[pf])
    rows, cols, vals = map(np.concatenate, (rows, cols, vals))
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))


def _lfull(Ah, inF, partner, b11, b12, dg):
    """L = A^_{C,F} B^{-1}, rows indexed by level index (C rows only)."""
    n = Ah.shape[0]
    Binv = _binv(n, inF, partner, b11, b12)
    PF = sp.diags(inF.astype(float))
    PC = sp.diags((~inF).astype(float))
    Lf = sp.csr_matrix(PC @ Ah @ PF @ Binv)
    Lf.eliminate_zeros()
    return Lf


class MultilevelILDL:
    """M^{-1} ~ (A - sigma I)^{-1}; see module docstring."""

    def __init__(self, A, lattice_L=None, kappa=5.0, tau_drop=2e-3, tau_strong=2e-2,
                 n_coarse_max=2048, max_levels=200, stall_frac=0.005, dense_cap=8192, factor_fp32=False,
                 compensate=True, tau_virtual=None, priority="quality", red=None, tau_inv=0.0):
        """red: level-0 independent set of a lattice block (default red_sites(lattice_L)).
        tau_inv > 0: inverse-based (aggressive) dropping of L a posteriori (PAPER.md
        l.947-973, reading R18), see `inverse_based_drop`.
        factor_fp32 (reading R16): the stored factor values are rounded to
        IEEE binary32 -- forward entries as fl32(l_cf * D_f), backward entries as
        fl32(l_cf) -- and used in fp64 arithmetic, as on the GPU."""
        self.levels = []
        self.factor_fp32 = bool(factor_fp32)
        cur = sp.csr_matrix(A)
        self.nnzA = cur.nnz
        for lev in range(max_levels):
            if cur.shape[0] <= n_coarse_max:
                break
            Lv = factor_level(cur, kappa, tau_drop, tau_strong,
                              lattice_L if lev == 0 else None, stall_frac, compensate, tau_virtual,
                              priority, red if lev == 0 else None)
            if Lv is None:
                break
            if self.factor_fp32:
                Lc = Lv.L.tocoo()
                fw = (Lc.data * Lv.D[Lc.col]).astype(np.float32).astype(np.float64)
                Lv.Lfwd = sp.csr_matrix((fw, (Lc.row, Lc.col)), shape=Lv.L.shape)
                Lv.Lbwd = sp.csr_matrix((Lc.data.astype(np.float32).astype(np.float64), (Lc.row, Lc.col)),
                                        shape=Lv.L.shape)
            self.levels.append(Lv)
            cur = Lv.S
        if cur.shape[0] > dense_cap:
            raise RuntimeError(f"multilevel ILDL breakdown: coarse size {cur.shape[0]} > {dense_cap}")
        self.coarse_n = cur.shape[0]
        if cur.shape[0] > 0:
            G = np.linalg.inv(cur.toarray())
            self.G = 0.5 * (G + G.T)
        else:
            self.G = np.zeros((0, 0))
        self.nu = None
        if tau_inv > 0.0:
            if self.factor_fp32:
                raise ValueError("inverse-based dropping is defined on the fp64 factor")
            self.nu = inverse_based_drop(self, tau_inv)

    def fill(self):
        """nnz(LDL^T)/nnz(A) analogue: stored L entries + pivots + dense coarse triangle."""
        nl = sum(Lv.L.nnz + len(Lv.F) + Lv.npairs for Lv in self.levels)
        nc = self.coarse_n
        return (nl + nc * (nc + 1) // 2) / self.nnzA

    def apply(self, r):
        return self._apply(np.asarray(r, dtype=np.float64), 0)

    def _apply(self, r, lev):
        if lev == len(self.levels):
            return self.G @ r
        Lv = self.levels[lev]
        rh = Lv.D * r
        if self.factor_fp32:
            wC = rh[Lv.C] - Lv.Lfwd @ r
        else:
            wC = rh[Lv.C] - Lv.L @ rh
        yC = self._apply(wC, lev + 1)
        zh = np.empty_like(r)
        zh[Lv.C] = yC
        zF = Lv.Binv @ rh - (Lv.Lbwd if self.factor_fp32 else Lv.L).T @ yC
        zh[Lv.F] = zF[Lv.F]
        return Lv.D * zh


def nu_estimates(M):
    """nu_i ~ ||L~^{-1} e_i|| for every node of every level ("In principle it
    can be computed using L~^T instead of L~"), reading R18.  L~ is the unit lower factor of
    the whole multilevel factorisation in elimination order [F_0, F_1, ..., C_last], each
    level's block in its own scaled coordinates.  Column i of L~^{-1} is row i of U^{-1},
    U = L~^T; the Cline-Moler-Stewart-Wilkinson estimate solves U x = b by back
    substitution, choosing b_i = +-1 against the partial sum:
        s_i = sum_{j later} l_ji x_j,   b_i = -1 if s_i > 0 else +1,   x_i = b_i - s_i,
    so nu_i = |x_i| = 1 + |s_i|.  The final coarse nodes have no L entries (x = +1).  For a
    pivot f of level l the later nodes j with l_jf != 0 are the coarse nodes of level l,
    whose x is level l+1's; s_f sums its L^T row in ascending coarse index, one rounded
    product then one rounded addition per entry.  Returns [x of level l (length n_l)]."""
    xs = [None] * len(M.levels)
    x_next = np.ones(M.coarse_n)
    for lev in reversed(range(len(M.levels))):
        Lv = M.levels[lev]
        Lc = Lv.L.tocoo()                                  # (coarse index, level index f, l)
        o = np.lexsort((Lc.row, Lc.col))                   # per pivot f: ascending coarse index
        f, cp, l = Lc.col[o], Lc.row[o], Lc.data[o]
        s = np.zeros(Lv.n)
        np.add.at(s, f, l * x_next[cp])                    # sequential, in that order
        x = np.empty(Lv.n)
        x[Lv.C] = x_next
        xf = np.where(s[Lv.F] > 0, -1.0, 1.0) - s[Lv.F]
        x[Lv.F] = xf
        xs[lev] = x
        x_next = x
    return xs


def inverse_based_drop(M, tau):
    """Aggressive dropping a posteriori (reading R18): an entry l_cf of
    level l is dropped when |l_cf| <= tau / (nu_c * #col_f), nu_c the estimate of
    ||L~^{-1} e_c|| (nu_estimates, with the factor before this dropping) and #col_f the
    number of stored entries of column f of L.  Evaluated on the stored forward value
    fl(l_cf D_f) as  (|fl(l_cf D_f)| * nu_c) * #col_f <= tau * D_f  (the same inequality, the
    GPU evaluates it identically on both copies of the entry).  Returns the x vectors."""
    xs = nu_estimates(M)
    for lev, Lv in enumerate(M.levels):
        nu_c = np.abs(xs[lev + 1]) if lev + 1 < len(M.levels) else np.ones(M.coarse_n)
        Lc = Lv.L.tocoo()
        cnt = np.bincount(Lc.col, minlength=Lv.n).astype(np.float64)
        lf = Lc.data * Lv.D[Lc.col]
        keep = (np.abs(lf) * nu_c[Lc.row]) * cnt[Lc.col] > tau * Lv.D[Lc.col]
        Lv.L = sp.csr_matrix((Lc.data[keep], (Lc.row[keep], Lc.col[keep])), shape=Lv.L.shape)
        Lv.L.sort_indices()
        Lv.ndrop_inv = int((~keep).sum())
    return xs
