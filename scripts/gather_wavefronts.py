"""Gather locality of the substitution kernels on the oracle's factor (CPU experiment, DESIGN.md
sect. 4): loads served per L1TEX wavefront (distinct 128-byte lines per warp-wide gather
instruction, G lanes per row as the kernels map them) with the node order the factor inherits from
the lattice (x fastest) versus a Morton (Z-curve) order of the pivots and rows.
python scripts/gather_wavefronts.py   (L=28, production drop parameters of L=150; ~2 min)
"""
import sys, numpy as np
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import anderson as an, mlildl
import scipy.sparse as sp
L=28
eps=an.disorder(L,16.5,1)
A=an.matrix(L,eps,hop=-1.0,sigma=0.0)
td=1.0886e-4; ts=40*td
M=mlildl.MultilevelILDL(A,lattice_L=L,kappa=5.0,tau_drop=td,tau_strong=ts,n_coarse_max=1024,max_levels=12,stall_frac=0.005,dense_cap=1<<20)
PREF=8
def pick(avg, per_lane=8, gmax=32):
    g=1
    while g<gmax and g*per_lane<=avg: g*=2
    return g
def morton(ix,iy,iz):
    def spread(v):
        v=v.astype(np.uint64); r=np.zeros_like(v)
        for b in range(10): r|=((v>>np.uint64(b))&np.uint64(1))<<np.uint64(3*b)
        return r
    return spread(ix)|(spread(iy)<<np.uint64(1))|(spread(iz)<<np.uint64(2))
def wf(indptr, cols, G, colmap=None):
    # rows in order; lanes: 32/G rows per warp, G lanes per row; instruction q: entry e0+lane+q*G
    nr=len(indptr)-1; rw=32//G
    tot_wf=0; tot_ld=0
    for w0 in range(0,nr,rw):
        rows=range(w0,min(nr,w0+rw))
        maxlen=max(indptr[r+1]-indptr[r] for r in rows)
        nq=-(-maxlen//G)
        for q in range(nq):
            lines=set(); n=0
            for r in rows:
                a=indptr[r]+q*G; b=min(indptr[r+1],a+G)
                if b>a:
                    c=cols[a:b]
                    if colmap is not None: c=colmap[c]
                    lines.update((c//16).tolist()); n+=b-a
            tot_wf+=len(lines); tot_ld+=n
    return tot_wf, tot_ld
orig=np.arange(L**3)   # original site of each level node
for li,lv in enumerate(M.levels):
    n=lv.n
    F=np.asarray(lv.F); C=np.asarray(lv.C)
    Lm=sp.csr_matrix(lv.L)           # nC x n (cols = level index of F node)
    # forward: rows = coarse nodes (order C), cols -> pivot index f'
    fmap=-np.ones(n,int); fmap[F]=np.arange(len(F))
    Lc=Lm.tocsr(); Lc.sort_indices()
    cols_f=fmap[Lc.indices]
    G=pick(Lc.nnz/max(1,Lc.shape[0]))
    w1,l1=wf(Lc.indptr, cols_f, G)
    # Morton order of the pivots
    site=orig[F]; key=morton(site%L,(site//L)%L,site//(L*L)); perm=np.argsort(key,kind='stable'); newf=np.empty(len(F),int); newf[perm]=np.arange(len(F))
    w2,l2=wf(Lc.indptr, cols_f, G, newf)
    # Morton order of rows too (coarse nodes) with Morton pivots
    siteC=orig[C]; keyC=morton(siteC%L,(siteC//L)%L,siteC//(L*L)); permC=np.argsort(keyC,kind='stable')
    Lp=Lc[permC]; Lp.sort_indices()
    # columns must be re-sorted in new numbering per row
    colsp=newf[fmap[Lp.indices]]
    ip=Lp.indptr; colsp2=colsp.copy()
    for r in range(Lp.shape[0]): colsp2[ip[r]:ip[r+1]]=np.sort(colsp[ip[r]:ip[r+1]])
    w3,l3=wf(ip, colsp2, G)
    # backward: rows = pivots, cols = coarse index
    LT=Lc.T.tocsr(); LT=LT[F]; LT.sort_indices()
    Gb=pick(LT.nnz/max(1,LT.shape[0]), 8, 32)
    b1,bl1=wf(LT.indptr, LT.indices, Gb)
    newc=np.empty(len(C),int); newc[permC]=np.arange(len(C))
    LTp=LT[perm]; cb=newc[LTp.indices]; ipb=LTp.indptr; cb2=cb.copy()
    for r in range(LTp.shape[0]): cb2[ipb[r]:ipb[r+1]]=np.sort(cb[ipb[r]:ipb[r+1]])
    b3,bl3=wf(ipb, cb2, Gb)
    print(f"lev {li} n {n} nF {len(F)} fwd G{G} loads/wf: lattice {l1/w1:.2f} mortonF {l2/w2:.2f} mortonF+rows {l3/w3:.2f} | bwd G{Gb} lattice {bl1/b1:.2f} morton {bl3/b3:.2f}", flush=True)
    orig=orig[C]
