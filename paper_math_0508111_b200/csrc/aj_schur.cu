// Schur complement and L rows of one multilevel-ILDL level on the GPU.
//
// PAPER.md l.857 / l.900-911 (sect. 7.2): with the pivot blocks F (an independent
// set, R9) and B~^{-1} = B_d^{-1} + V (block pivots plus the virtual
// first-order couplings of reading R17),
//     L   = A^_CF B~^{-1} = L^r + L^v,   L^r = A^_CF B_d^{-1},  L^v = A^_CF V,
//     S   = A^_CC - L^r A^_FC - P o (L^v A^_FC),
// P = the pattern of A^_CC and of L^r A^_FC (the compensation creates no fill).
// Per coarse row c, in this order (oracle/mlildl.py::_l_rows / _schur_blocks do the
// same, so decisions taken on the values -- drops, the next level's pivots -- are
// bit-identical):
//   (A) the row of L: l^r_cx for the members x of every real block with a member
//       adjacent to c (one product pair per x, lval_pair), l^v_cx = sum of the
//       virtual terms a^_cu b'_ux in ascending block key; L_cx = l^r_cx + l^v_cx,
//       entries with |L_cx| < tau dropped;
//   (B) s_cc' = a^_cc' on the coarse entries of row c;
//   (C) for x ascending with a real block: s_cc' -= l^r_cx a^_c'x over the coarse
//       neighbours c' of x (inserting fill);
//   (D) for x ascending with virtual terms: s_cc' -= l^v_cx a^_c'x where (c, c') is
//       already in the row (no fill);
//   (E) off-diagonals with |s| < tau dropped, the survivors sorted by column.
// Each product is rounded, then subtracted (no FMA contraction).  Only the upper
// triangle c' >= c is computed; the caller mirrors it (S is symmetric by construction
// and bit for bit, like the oracle's S = triu(S) + triu(S, 1)^T).
//
// GPU mapping: one coarse row per thread group; the row's columns live in an
// open-addressing table (keys + values) in shared memory.  Before the level, the
// coarse neighbours of every pivot x are compacted into FC lists (coarse index,
// a^_c'x), so the hot loop (C)/(D) is a coalesced stream of 12-byte entries into
// table updates -- no merges, binary searches or index translation.  Inside one x
// every c' occurs once, so the threads of a group never share a slot; the group
// synchronises between consecutive x (the per-entry order above).  A routing pass
// bounds each row's table size (|coarse part of row c| + sum |FC(x)|) and its L-row
// length, and sends it to the smallest tier that is guaranteed to hold it:
//   W1  warp, 1024-entry table,  8 rows per CTA, 2 CTAs per SM
//   W2  warp, 2048-entry table,  4 rows per CTA, 2 CTAs per SM
//   C8  CTA of 256, 8192-entry table (96 KB), 2 CTAs per SM
//   C16 CTA of 256, 16384-entry table (192 KB): may overflow (the bound is loose at
//       deep levels) -> the row is retried in
//   G   CTA of 256, 65536-entry table in global memory.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "aj_common.cuh"
#include "aj_kernels.cuh"
#include "aj_mlildl.cuh"
#include "aj_sparse.cuh"

namespace aj {

// -DAJ_SCHUR_PROF (experiments only): per-phase clock64 sums of k_schur_rows, lane 0 of every
// group, accumulated in g_schur_prof[phase] and printed by schur_prof_dump()
#ifdef AJ_SCHUR_PROF
__device__ unsigned long long g_schur_prof[16];
#define SPROF_DECL long long sp_t0 = clock64(), sp_t1
#define SPROF(ph)                                                          \
  do {                                                                     \
    sp_t1 = clock64();                                                     \
    if (tid == 0) atomicAdd(&g_schur_prof[ph], (unsigned long long)(sp_t1 - sp_t0)); \
    sp_t0 = sp_t1;                                                         \
  } while (0)
#else
#define SPROF_DECL
#define SPROF(ph)
#endif

namespace {
constexpr int TBs = 256;

// ---------------------------------------------------------------------------
// FC lists: for pivot fp (level index x = fidx[fp]) the coarse entries of row x
// in column order: (cmap[col], a^_{x,col}) -- a^ is symmetric, so a^_{c'x}.
__global__ void k_fc_count(int nF, const int32_t* __restrict__ fidx, const int64_t* __restrict__ ptr,
                           const int32_t* __restrict__ col, const int32_t* __restrict__ cmap, int64_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  for (int fp = (blockIdx.x * TBs + threadIdx.x) >> 5; fp < nF; fp += (gridDim.x * TBs) >> 5) {
    const int x = fidx[fp];
    int k = 0;
    for (int64_t e = ptr[x] + lane; e < ptr[x + 1]; e += 32) k += (cmap[col[e]] >= 0) ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
    if (lane == 0) cnt[fp] = k;
  }
}
__global__ void k_fc_fill(int nF, const int32_t* __restrict__ fidx, const int64_t* __restrict__ ptr,
                          const int32_t* __restrict__ col, const double* __restrict__ ah,
                          const int32_t* __restrict__ cmap, const int64_t* __restrict__ FCptr,
                          int32_t* __restrict__ FCcol, double* __restrict__ FCval) {
  const int lane = threadIdx.x & 31;
  for (int fp = (blockIdx.x * TBs + threadIdx.x) >> 5; fp < nF; fp += (gridDim.x * TBs) >> 5) {
    const int x = fidx[fp];
    int64_t w = FCptr[fp];
    for (int64_t e0 = ptr[x]; e0 < ptr[x + 1]; e0 += 32) {
      const int64_t e = e0 + lane;
      int32_t cc = -1;
      if (e < ptr[x + 1]) cc = cmap[col[e]];
      const unsigned bal = __ballot_sync(0xffffffffu, cc >= 0);
      if (cc >= 0) {
        const int64_t o = w + __popc(bal & ((1u << lane) - 1u));
        FCcol[o] = cc;
        FCval[o] = ah[e];
      }
      w += __popc(bal);
    }
  }
}

// ---------------------------------------------------------------------------
// tiers
enum { TIER_W1 = 0, TIER_W2, TIER_P4, TIER_C8, TIER_C16, TIER_G, NTIER };
struct TierCap {
  int table_cap;  // guaranteed-fit bound on the row's table (3/4 of the table)
  int bm;         // L-row / virtual-term capacity
};
__host__ __device__ constexpr TierCap tier_cap(int t) {
  return t == TIER_W1 ? TierCap{768, 512}
       : t == TIER_W2 ? TierCap{1536, 1024}
       : t == TIER_P4 ? TierCap{3072, 2048}
       : t == TIER_C8 ? TierCap{6144, 4096}
       : t == TIER_C16 ? TierCap{12288, 4096}
                       : TierCap{49152, 8192};
}

// per coarse row: table bound nb = |coarse part of row c| + sum over the real-block
// members x adjacent (or partnered) to c of |FC(x)|; L-row bound nl + nvt (real
// members + virtual terms); route to the smallest tier that holds it.
__global__ void k_schur_route(int nC, const int32_t* __restrict__ cidx, const int64_t* __restrict__ ptr,
                              const int32_t* __restrict__ col, const int8_t* __restrict__ inF,
                              const int32_t* __restrict__ partner, const int32_t* __restrict__ fmap,
                              const int32_t* __restrict__ cmap, const int64_t* __restrict__ FCptr,
                              const int32_t* __restrict__ FCcol, const int64_t* __restrict__ Vptr,
                              int* __restrict__ counts, int32_t* __restrict__ lists, int* __restrict__ err) {
  constexpr int SGr = 8;
  const int gl = threadIdx.x & (SGr - 1);
  const unsigned m = ((1u << SGr) - 1u) << ((threadIdx.x & 31) & ~(SGr - 1));
  for (int cp = (blockIdx.x * TBs + threadIdx.x) / SGr; cp < nC; cp += gridDim.x * (TBs / SGr)) {
    const int c = cidx[cp];
    long long nb = 0, nl = 0, nvt = 0;
    // entries of FC(x) in the upper triangle (coarse index >= cp): FC lists are sorted
    auto upper_len = [&](int fx) -> long long {
      int64_t a0 = FCptr[fx], b = FCptr[fx + 1];
      const int64_t e1 = b;
      while (a0 < b) {
        const int64_t mid = (a0 + b) >> 1;
        if (FCcol[mid] < cp)
          a0 = mid + 1;
        else
          b = mid;
      }
      return e1 - a0;
    };
    for (int64_t e = ptr[c] + gl; e < ptr[c + 1]; e += SGr) {
      const int32_t u = col[e];
      if (!inF[u]) {
        nb += (cmap[u] >= cp) ? 1 : 0;
        continue;
      }
      nb += upper_len(fmap[u]);
      nl += 1;
      const int32_t p = partner[u];
      if (p >= 0) {
        nb += upper_len(fmap[p]);
        nl += 1;
      } else if (Vptr) {
        nvt += Vptr[u + 1] - Vptr[u];
      }
    }
#pragma unroll
    for (int o = SGr / 2; o > 0; o >>= 1) {
      nb += __shfl_xor_sync(m, nb, o);
      nl += __shfl_xor_sync(m, nl, o);
      nvt += __shfl_xor_sync(m, nvt, o);
    }
    if (gl == 0) {
      const long long lb = nl + nvt;
      int t = TIER_G;
      for (int k = TIER_W1; k <= TIER_C16; ++k) {
        const TierCap cap = tier_cap(k);
        const bool table_ok = (k == TIER_C16) || nb <= cap.table_cap;  // C16 may overflow -> G
        if (table_ok && lb <= cap.bm && lb <= cap.table_cap) {
          t = k;
          break;
        }
      }
      if (t == TIER_G && lb > tier_cap(TIER_G).bm) atomicExch(err, 3);
      const int pos = atomicAdd(&counts[t], 1);
      lists[(size_t)t * nC + pos] = cp;
    }
  }
}

struct SchurArgs {
  const int32_t *cidx, *cmap, *fmap;
  const int64_t* ptr;
  const int32_t* col;
  const double* ah;
  const int8_t* inF;
  const int32_t* partner;
  const double *b11, *b12;
  const int64_t* Vptr;
  const int32_t* Vcol;
  const double* Vval;
  const int64_t* FCptr;
  const int32_t* FCcol;
  const double* FCval;
  double tau;
  int64_t *row_cnt, *row_off;
  int32_t* tmp_col;
  double* tmp_val;
  int64_t cap;
  unsigned long long* cursor;
  int64_t *lrow_cnt, *lrow_off;
  int32_t* ltmp_col;
  double* ltmp_val;
  int64_t lcap;
  unsigned long long* lcursor;
};

// group barrier: a warp, a whole CTA, or a named barrier (id 1 + group) for groups of
// 64 / 128 threads sharing a CTA
template <int G, int GROUPS = 1>
__device__ __forceinline__ void gsync() {
  if constexpr (G == 32) {
    __syncwarp();
  } else if constexpr (GROUPS == 1) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)(threadIdx.x / G)), "r"(G) : "memory");
  }
}

// bitonic sort of (key, perm) pairs, P a power of two, in group scratch
template <int G, int GROUPS, typename K, typename V>
__device__ void group_bitonic(K* k, V* v, int P, int tid) {
  for (int kk = 2; kk <= P; kk <<= 1)
    for (int jj = kk >> 1; jj > 0; jj >>= 1) {
      for (int t = tid; t < P; t += G) {
        const int ixj = t ^ jj;
        if (ixj > t) {
          const K x = k[t], y = k[ixj];
          const bool up = (t & kk) == 0;
          if ((x > y) == up) {
            k[t] = y;
            k[ixj] = x;
            const V tv = v[t];
            v[t] = v[ixj];
            v[ixj] = tv;
          }
        }
      }
      gsync<G, GROUPS>();
    }
}

// rank sort of n <= RANK_MAX distinct keys in group scratch: every element counts the keys below
// it (n independent broadcast loads instead of the log^2 n dependent exchange stages of the
// bitonic network, each a round trip to the scratch in L2) and writes its index to v[rank].
// Same result as group_bitonic on (k, identity): v = the permutation that sorts k; k is left as is.
constexpr int RANK_MAX = 128;
template <int G, int GROUPS, typename K, typename V>
__device__ void group_ranksort(const K* k, V* v, int n, int tid) {
  for (int i = tid; i < n; i += G) {
    const K ki = k[i];
    int r = 0;
    for (int j = 0; j < n; ++j) {
      const K kj = k[j];
      r += (kj < ki || (kj == ki && j < i)) ? 1 : 0;
    }
    v[r] = (V)i;
  }
  gsync<G, GROUPS>();
}

__host__ __device__ constexpr int pow2_at_least(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// per-group scratch (32-bit words): slot list T, compaction keys T, values 2T,
// L row (x, flags, l^r, l^v) 6 BM, virtual terms (x, t) 3 BM, sort keys/perm 3 BM,
// the sorted L row (x, FC range, l^r, l^v, flags) 12 BM [+ table 3T if in global memory]
template <int T, int BM, bool GTAB>
__host__ __device__ constexpr size_t schur_words() {
  return (size_t)4 * T + (size_t)24 * BM + (GTAB ? (size_t)3 * T : 0);
}

template <int G, int GROUPS, int T, int BM, bool GTAB, bool CAN_OVF>
__global__ void __launch_bounds__(G * GROUPS, 1)  // minBlocks 1: no register cap (tables limit the CTAs per SM)
    k_schur_rows(int nrows, const int32_t* __restrict__ rowlist, SchurArgs a, int32_t* __restrict__ scratch_all,
                 int32_t* __restrict__ ovf_list, int* __restrict__ ovf_count, int* __restrict__ err,
                 unsigned long long* __restrict__ products) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_cnt[GROUPS], s_nvt[GROUPS], s_kept[GROUPS], s_full[GROUPS];
  __shared__ unsigned long long s_base[GROUPS];
  const int grp = threadIdx.x / G, tid = threadIdx.x % G;
  int32_t* scr = scratch_all + (size_t)(blockIdx.x * GROUPS + grp) * schur_words<T, BM, GTAB>();
  int32_t* list = scr;
  int32_t* ekey = scr + T;
  double* evals = reinterpret_cast<double*>(scr + 2 * T);
  int32_t* Lx = scr + 4 * T;
  int32_t* Lfl = Lx + BM;
  double* Lr = reinterpret_cast<double*>(Lfl + BM);
  double* Lv = Lr + BM;
  int32_t* VTx = reinterpret_cast<int32_t*>(Lv + BM);
  int32_t* sp = VTx + BM;
  double* VTt = reinterpret_cast<double*>(sp + BM);
  uint64_t* sk = reinterpret_cast<uint64_t*>(VTt + BM);
  int64_t* Xe0 = reinterpret_cast<int64_t*>(sk + BM);
  int64_t* Xe1 = Xe0 + BM;
  double* Xr = reinterpret_cast<double*>(Xe1 + BM);
  double* Xv = Xr + BM;
  int32_t* Xx = reinterpret_cast<int32_t*>(Xv + BM);
  int32_t* Xf = Xx + BM;
  int32_t* tab;
  double* vals;
  if constexpr (GTAB) {
    tab = scr + 4 * T + 24 * BM;
    vals = reinterpret_cast<double*>(tab + T);
  } else {
    vals = reinterpret_cast<double*>(smem_raw) + (size_t)grp * T;
    tab = reinterpret_cast<int32_t*>(smem_raw + (size_t)GROUPS * T * sizeof(double)) + (size_t)grp * T;
  }
  for (int t = tid; t < T; t += G) tab[t] = -1;
  gsync<G, GROUPS>();
  const double tau = a.tau;
  for (int ri = blockIdx.x * GROUPS + grp; ri < nrows; ri += gridDim.x * GROUPS) {
    const int cp = rowlist[ri];
    const int c = a.cidx[cp];
    const int64_t lo = a.ptr[c], hi = a.ptr[c + 1];
    SPROF_DECL;
    if (tid == 0) {
      s_cnt[grp] = 0;
      s_nvt[grp] = 0;
      s_kept[grp] = 0;
      s_full[grp] = 0;
    }
    gsync<G, GROUPS>();
    // ---- (A1) real blocks adjacent to c: l^r for their members; virtual terms listed
    for (int64_t e = lo + tid; e < hi; e += G) {
      const int32_t u = a.col[e];
      if (!a.inF[u]) continue;
      const int32_t p = a.partner[u];
      const double acu = a.ah[e];
      bool fr;
      if (p < 0) {
        const int pos = lslot<T>(tab, vals, u, &s_cnt[grp], list, &fr);
        Lx[pos] = u;
        Lr[pos] = __dmul_rn(acu, a.b11[u]);
        Lv[pos] = 0.0;
        Lfl[pos] = 1;
        if (a.Vptr)
          for (int64_t ev = a.Vptr[u]; ev < a.Vptr[u + 1]; ++ev) {
            const int32_t v = a.Vcol[ev];
            const int q = atomicAdd(&s_nvt[grp], 1);
            sk[q] = ((uint64_t)(uint32_t)v << 32) | (uint32_t)u;  // (target x, source pivot u)
            sp[q] = q;
            VTx[q] = v;
            VTt[q] = __dmul_rn(acu, a.Vval[ev]);
          }
      } else {
        // a pair is handled once, at its smaller member adjacent to c
        const int64_t ep = lookup_idx(a.col, lo, hi, p);
        if (ep >= 0 && p < u) continue;
        const double acp = (ep >= 0) ? a.ah[ep] : 0.0;
        const int32_t f = min(u, p), g = max(u, p);
        const double acf = (f == u) ? acu : acp, acg = (g == u) ? acu : acp;
        const int pf = lslot<T>(tab, vals, f, &s_cnt[grp], list, &fr);
        Lx[pf] = f;
        Lr[pf] = lval_pair(acf, acg, a.b11[f], a.b12[g]);
        Lv[pf] = 0.0;
        Lfl[pf] = 1;
        const int pg = lslot<T>(tab, vals, g, &s_cnt[grp], list, &fr);
        Lx[pg] = g;
        Lr[pg] = lval_pair(acf, acg, a.b12[f], a.b11[g]);
        Lv[pg] = 0.0;
        Lfl[pg] = 1;
      }
    }
    gsync<G, GROUPS>();
    SPROF(0);
    // ---- (A2) virtual terms accumulated into l^v in ascending block key {u, x}: for a fixed
    // target x that is ascending source pivot u, so the terms are sorted by (x, u) and one
    // thread per target sums its run in order (the oracle's order, bitwise)
    const int nvt = s_nvt[grp];
    if (nvt > 0) {
      if (nvt <= RANK_MAX) {
        gsync<G, GROUPS>();
        group_ranksort<G, GROUPS>(sk, sp, nvt, tid);
      } else {
        const int P = pow2_at_least(nvt);
        for (int t = nvt + tid; t < P; t += G) {
          sk[t] = ~0ull;
          sp[t] = t;
        }
        gsync<G, GROUPS>();
        group_bitonic<G, GROUPS>(sk, sp, P, tid);
      }
      for (int i = tid; i < nvt; i += G) {
        const int q = sp[i];
        const int32_t x = VTx[q];
        if (i > 0 && VTx[sp[i - 1]] == x) continue;  // not the head of its run
        double sum = VTt[q];
        for (int j = i + 1; j < nvt; ++j) {
          const int qj = sp[j];
          if (VTx[qj] != x) break;
          sum = __dadd_rn(sum, VTt[qj]);
        }
        bool fr;
        const int pos = lslot<T>(tab, vals, x, &s_cnt[grp], list, &fr);
        if (fr) {
          Lx[pos] = x;
          Lr[pos] = 0.0;
          Lfl[pos] = 2;
        } else {
          Lfl[pos] |= 2;
        }
        Lv[pos] = sum;
      }
      gsync<G, GROUPS>();
    }
    SPROF(1);
    // ---- (A3) empty the table; the L row sorted by x, with the FC range of each x
    const int nl = s_cnt[grp];
    for (int pos = tid; pos < nl; pos += G) {
      tab[list[pos]] = -1;
      sk[pos] = (uint64_t)(uint32_t)Lx[pos];
      sp[pos] = pos;
    }
    if (nl <= RANK_MAX) {
      gsync<G, GROUPS>();
      if (nl > 1) group_ranksort<G, GROUPS>(sk, sp, nl, tid);
    } else {
      const int P = pow2_at_least(nl);
      for (int t = nl + tid; t < P; t += G) {
        sk[t] = ~0ull;
        sp[t] = t;
      }
      gsync<G, GROUPS>();
      group_bitonic<G, GROUPS>(sk, sp, P, tid);
    }
    SPROF(2);
    for (int i = tid; i < nl; i += G) {
      const int pos = sp[i];
      const int32_t x = Lx[pos];
      const int fx = a.fmap[x];
      Xx[i] = x;
      // upper triangle only (c' >= c): FC(x) is sorted by coarse index, start at cp
      const int64_t f1 = a.FCptr[fx + 1];
      int64_t f0 = a.FCptr[fx];
      {
        int64_t b = f1;
        while (f0 < b) {
          const int64_t mid = (f0 + b) >> 1;
          if (a.FCcol[mid] < cp)
            f0 = mid + 1;
          else
            b = mid;
        }
      }
      Xe0[i] = f0;
      Xe1[i] = f1;
      Xr[i] = Lr[pos];
      Xv[i] = Lv[pos];
      Xf[i] = Lfl[pos];
    }
    if (tid == 0) s_cnt[grp] = 0;
    gsync<G, GROUPS>();
    SPROF(3);
    // ---- (B) s_cc' = a^_cc' (upper triangle c' >= c: the lower one is its mirror)
    for (int64_t e = lo + tid; e < hi; e += G) {
      const int32_t cu = a.cmap[a.col[e]];
      if (cu < cp) continue;  // pivots (cu = -1) and the lower triangle
      const int sl = hslot<T>(tab, vals, cu, &s_cnt[grp], list);
      if (CAN_OVF && sl < 0)
        s_full[grp] = 1;
      else
        vals[sl] = a.ah[e];
    }
    gsync<G, GROUPS>();
    SPROF(4);
    // ---- (C) real terms, x ascending; (D) virtual terms on the pattern, x ascending
    // work lists of (C) and (D): the sorted L-row positions with real / virtual terms
    if (tid < 32) {  // the group's first warp: stable compaction, 32 positions per ballot
      int nr = 0, nv2 = 0;
      const unsigned lower = (1u << tid) - 1u;
      for (int i0 = 0; i0 < nl; i0 += 32) {
        const int i = i0 + tid;
        const int fl = (i < nl) ? Xf[i] : 0;
        const unsigned br = __ballot_sync(0xffffffffu, (fl & 1) != 0);
        const unsigned bv = __ballot_sync(0xffffffffu, (fl & 2) != 0);
        if (fl & 1) sp[nr + __popc(br & lower)] = i;
        if (fl & 2) VTx[nv2 + __popc(bv & lower)] = i;
        nr += __popc(br);
        nv2 += __popc(bv);
      }
      if (tid == 0) {
        s_nvt[grp] = nr;   // reused: number of real items
        s_kept[grp] = nv2; // reused: number of virtual items (s_kept is reset below)
      }
    }
    gsync<G, GROUPS>();
    const int nitems[2] = {s_nvt[grp], s_kept[grp]};
    gsync<G, GROUPS>();
    if (tid == 0) s_kept[grp] = 0;
    constexpr int U = 4;
    unsigned long long nprod = 0;  // table updates of this row (the work model, DESIGN.md sect. 4)
    for (int pass = 0; pass < 2; ++pass) {
      const int* items = pass == 0 ? sp : VTx;
      const int ni = nitems[pass];
      if (ni == 0) continue;
      // software pipeline: the first G*U entries of the next item are loaded while the
      // current item's entries go through the table
      int32_t cc[U], nc_[U];
      double av[U], na_[U];
      int64_t e0 = 0, e1 = 0, ne0 = 0, ne1 = 0;
      double l = 0.0, nl_ = 0.0;
      auto load_item = [&](int j, int64_t& f0, int64_t& f1, double& lv, int32_t (&ccv)[U], double (&avv)[U]) {
        const int i = items[j];
        f0 = Xe0[i];
        f1 = Xe1[i];
        lv = pass == 0 ? Xr[i] : Xv[i];
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int64_t e = f0 + tid + (int64_t)k * G;
          ccv[k] = (e < f1) ? a.FCcol[e] : -1;
          avv[k] = (e < f1) ? a.FCval[e] : 0.0;
        }
      };
      auto apply = [&](const int32_t (&ccv)[U], const double (&avv)[U], double lv) {
#pragma unroll
        for (int k = 0; k < U; ++k) {
          if (ccv[k] < 0) continue;
          int sl;
          if (pass == 0) {
            sl = hslot<T>(tab, vals, ccv[k], &s_cnt[grp], list);
            if (CAN_OVF && sl < 0) {
              s_full[grp] = 1;
              continue;
            }
          } else {
            sl = hfind<T>(tab, ccv[k]);
            if (sl < 0) continue;  // outside the pattern (reading R17)
          }
          vals[sl] = __dsub_rn(vals[sl], __dmul_rn(lv, avv[k]));
        }
      };
      load_item(0, e0, e1, l, cc, av);
      for (int j = 0; j < ni; ++j) {
        if (j + 1 < ni) load_item(j + 1, ne0, ne1, nl_, nc_, na_);
        nprod += (unsigned long long)(e1 - e0);
        apply(cc, av, l);
        for (int64_t eb = e0 + tid + (int64_t)G * U; eb < e1; eb += (int64_t)G * U) {
          int32_t c2[U];
          double a2[U];
#pragma unroll
          for (int k = 0; k < U; ++k) {
            const int64_t e = eb + (int64_t)k * G;
            c2[k] = (e < e1) ? a.FCcol[e] : -1;
            a2[k] = (e < e1) ? a.FCval[e] : 0.0;
          }
          apply(c2, a2, l);
        }
        gsync<G, GROUPS>();
        if (CAN_OVF && s_full[grp]) break;
        e0 = ne0;
        e1 = ne1;
        l = nl_;
#pragma unroll
        for (int k = 0; k < U; ++k) {
          cc[k] = nc_[k];
          av[k] = na_[k];
        }
      }
    }
    SPROF(5);
    // ---- (E) collect through the slot list, empty the table, drop
    const bool full = CAN_OVF && (s_full[grp] != 0 || s_cnt[grp] > (T * 3) / 4);
    const int nc = min(s_cnt[grp], T);
    for (int t = tid; t < nc; t += G) {
      const int32_t sl = list[t];
      const int32_t kk = tab[sl];
      const double vv = vals[sl];
      tab[sl] = -1;
      if (!full && ((kk == cp) || (fabs(vv) >= tau))) {
        const int off = atomicAdd(&s_kept[grp], 1);
        ekey[off] = kk;
        evals[off] = vv;
      }
    }
    gsync<G, GROUPS>();
    if (full) {
      if (tid == 0) {
        if (ovf_list)
          ovf_list[atomicAdd(ovf_count, 1)] = cp;
        else
          atomicExch(err, 2);
      }
      continue;  // uniform
    }
    const int kept = s_kept[grp];
    const int P = pow2_at_least(kept);
    for (int t = tid; t < P; t += G) {
      tab[t] = (t < kept) ? ekey[t] : INT32_MAX;
      vals[t] = (t < kept) ? evals[t] : 0.0;
    }
    gsync<G, GROUPS>();
    SPROF(6);
    group_bitonic<G, GROUPS>(tab, vals, P, tid);
    SPROF(7);
    if (tid == 0) {
      atomicAdd(products, nprod);
      const unsigned long long base = atomicAdd(a.cursor, (unsigned long long)kept);
      s_base[grp] = base;
      a.row_cnt[cp] = kept;
      a.row_off[cp] = (int64_t)base;
    }
    gsync<G, GROUPS>();
    {
      const unsigned long long base = s_base[grp];
      if ((int64_t)base + kept <= a.cap)
        for (int t = tid; t < kept; t += G) {
          a.tmp_col[base + t] = tab[t];
          a.tmp_val[base + t] = vals[t];
        }
    }
    gsync<G, GROUPS>();
    for (int t = tid; t < P; t += G) tab[t] = -1;
    SPROF(8);
    // ---- the L row (x ascending), L_cx = l^r + l^v, |L| < tau dropped (first warp)
    if (tid < 32) {
      const int lane = tid;
      int lk = 0;
      for (int i0 = 0; i0 < nl; i0 += 32) {
        const int i = i0 + lane;
        const bool keep = i < nl && fabs(__dadd_rn(Xr[i], Xv[i])) >= tau;
        lk += __popc(__ballot_sync(0xffffffffu, keep));
      }
      unsigned long long lb = 0;
      if (lane == 0) {
        lb = atomicAdd(a.lcursor, (unsigned long long)lk);
        a.lrow_cnt[cp] = lk;
        a.lrow_off[cp] = (int64_t)lb;
      }
      lb = __shfl_sync(0xffffffffu, lb, 0);
      if ((int64_t)lb + lk <= a.lcap) {
        int w = 0;
        for (int i0 = 0; i0 < nl; i0 += 32) {
          const int i = i0 + lane;
          double lv = 0.0;
          bool keep = false;
          if (i < nl) {
            lv = __dadd_rn(Xr[i], Xv[i]);
            keep = fabs(lv) >= tau;
          }
          const unsigned bal = __ballot_sync(0xffffffffu, keep);
          if (keep) {
            const int o = w + __popc(bal & ((1u << lane) - 1u));
            a.ltmp_col[lb + o] = Xx[i];
            a.ltmp_val[lb + o] = lv;
          }
          w += __popc(bal);
        }
      }
    }
    gsync<G, GROUPS>();
    SPROF(9);
  }
}

template <int G, int GROUPS, int T, int BM, bool GTAB, bool CAN_OVF>
struct Tier {
  static constexpr size_t smem() { return GTAB ? 0 : (size_t)GROUPS * T * (sizeof(int32_t) + sizeof(double)); }
  static constexpr size_t words() { return schur_words<T, BM, GTAB>(); }
  static void prepare() {
    if (!GTAB)
      AJ_CUDA(cudaFuncSetAttribute(k_schur_rows<G, GROUPS, T, BM, GTAB, CAN_OVF>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem()));
  }
  static int resident_ctas() {
    int per = 0;
    AJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_schur_rows<G, GROUPS, T, BM, GTAB, CAN_OVF>,
                                                          G * GROUPS, smem()));
    return std::max(1, per) * num_sms();
  }
  static void launch(int nrows, const int32_t* list, const SchurArgs& a, int32_t* scratch, int grid, int32_t* ovf,
                     int* ovf_count, int* err, unsigned long long* products, cudaStream_t st) {
    k_schur_rows<G, GROUPS, T, BM, GTAB, CAN_OVF><<<grid, G * GROUPS, smem(), st>>>(nrows, list, a, scratch, ovf,
                                                                                   ovf_count, err, products);
    AJ_LAUNCHED();
  }
};

using TierW1 = Tier<32, 8, 1024, 512, false, false>;     // 96 KB, 2 CTAs / SM: 16 rows per SM
using TierW2 = Tier<32, 4, 2048, 1024, false, false>;    // 96 KB: 8 rows per SM
using TierP4 = Tier<64, 2, 4096, 2048, false, false>;    // 96 KB: 4 rows per SM, 2 warps each
using TierC8 = Tier<128, 1, 8192, 4096, false, false>;   // 96 KB: 2 rows per SM, 4 warps each
using TierC16 = Tier<256, 1, 16384, 4096, false, true>;  // 192 KB: 1 row per SM, may overflow
using TierG = Tier<256, 1, 65536, 8192, true, true>;     // global-memory table

// Fork / join for the tier kernels: rows of different tiers are independent (disjoint output
// runs through the global cursors), so the tiers run concurrently on side streams -- on the deep
// levels each tier alone fills only a few SMs.  Streams and events are cached per host thread
// and device (a stream belongs to the device that was current when it was created).
struct TierStreams {
  cudaStream_t s[NTIER] = {};
  cudaEvent_t fork = nullptr, done[NTIER] = {};
};
static TierStreams& tier_streams() {
  constexpr int kMaxDev = 64;
  thread_local TierStreams ts[kMaxDev];
  int dev = 0;
  AJ_CUDA(cudaGetDevice(&dev));
  AJ_REQUIRE(dev >= 0 && dev < kMaxDev, AJ_ERR_CUDA, "device ordinal out of range");
  TierStreams& t = ts[dev];
  if (!t.fork) {
    AJ_CUDA(cudaEventCreateWithFlags(&t.fork, cudaEventDisableTiming));
    for (int k = 0; k < NTIER; ++k) {
      AJ_CUDA(cudaStreamCreateWithFlags(&t.s[k], cudaStreamNonBlocking));
      AJ_CUDA(cudaEventCreateWithFlags(&t.done[k], cudaEventDisableTiming));
    }
  }
  return t;
}

template <typename T>
static T read1(const T* d, cudaStream_t st) {
  T h;
  AJ_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, st));
  AJ_CUDA(cudaStreamSynchronize(st));
  return h;
}
}  // namespace

#ifdef AJ_SCHUR_PROF
static void schur_prof_dump(const char* tag, cudaStream_t st) {
  unsigned long long h[16];
  cudaStreamSynchronize(st);
  cudaMemcpyFromSymbol(h, g_schur_prof, sizeof(h));
  static const char* nm[10] = {"A1 L row", "A2 virtual", "A3 sort L", "A3 FC ranges", "B row insert", "C/D products",
                               "E collect", "E sort", "E write S", "L row write"};
  double tot = 0;
  for (int i = 0; i < 10; ++i) tot += (double)h[i];
  fprintf(stderr, "[schur prof] %s:", tag);
  for (int i = 0; i < 10; ++i) fprintf(stderr, " %s %.1f%%", nm[i], 100.0 * h[i] / (tot > 0 ? tot : 1));
  fprintf(stderr, "\n");
  memset(h, 0, sizeof(h));
  cudaMemcpyToSymbol(g_schur_prof, h, sizeof(h));
}
#endif

void schur_level(const SchurIn& in, SchurOut& out, cudaStream_t st) {
  const int nC = in.nC, nF = in.nF;
  // FC lists
  int64_t* fcnt = dalloc<int64_t>(std::max(nF, 1), st);
  const int gw = std::max(1, std::min(ceil_div((int64_t)std::max(nF, 1) * 32, TBs), num_sms() * 16));
  k_fc_count<<<gw, TBs, 0, st>>>(nF, in.fidx, in.ptr, in.col, in.cmap, fcnt);
  AJ_LAUNCHED();
  int64_t* FCptr = dalloc<int64_t>((size_t)nF + 1, st);
  AJ_CUDA(cudaMemsetAsync(FCptr, 0, sizeof(int64_t), st));
  {
    size_t tmp = 0;
    AJ_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, fcnt, FCptr + 1, std::max(nF, 1), st));
    void* t = dalloc<char>(tmp, st);
    AJ_CUDA(cub::DeviceScan::InclusiveSum(t, tmp, fcnt, FCptr + 1, std::max(nF, 1), st));
    dfree(t, st);
  }
  const int64_t nFC = nF > 0 ? read1(FCptr + nF, st) : 0;
  int32_t* FCcol = dalloc<int32_t>(std::max<int64_t>(nFC, 1), st);
  double* FCval = dalloc<double>(std::max<int64_t>(nFC, 1), st);
  k_fc_fill<<<gw, TBs, 0, st>>>(nF, in.fidx, in.ptr, in.col, in.ah, in.cmap, FCptr, FCcol, FCval);
  AJ_LAUNCHED();
  dfree(fcnt, st);
  out.nnz_fc = nFC;

  // routing: ctr[0..NTIER) rows per tier, ctr[NTIER] C16 overflows, ctr[NTIER + 1] error
  int* ctr = dalloc<int>(16, st);
  AJ_CUDA(cudaMemsetAsync(ctr, 0, 16 * sizeof(int), st));
  const size_t nC1 = (size_t)std::max(nC, 1);
  int32_t* lists = dalloc<int32_t>((size_t)(NTIER + 1) * nC1, st);
  int32_t* ovf = lists + (size_t)NTIER * nC1;
  {
    const int g8 = std::max(1, std::min(ceil_div((int64_t)nC1 * 8, TBs), num_sms() * 32));
    k_schur_route<<<g8, TBs, 0, st>>>(nC, in.cidx, in.ptr, in.col, in.inF, in.partner, in.fmap, in.cmap, FCptr,
                                      FCcol, in.Vptr, ctr, lists, ctr + NTIER + 1);
    AJ_LAUNCHED();
  }
  int cnt[16];
  AJ_CUDA(cudaMemcpyAsync(cnt, ctr, sizeof(cnt), cudaMemcpyDeviceToHost, st));
  AJ_CUDA(cudaStreamSynchronize(st));
  AJ_REQUIRE(cnt[NTIER + 1] == 0, AJ_ERR_CAPACITY,
             "Schur complement: more than 8192 L entries in one row (raise tau_drop)");
  // AJ_SCHUR_TIER=t (testing): every row of a smaller tier moves up to tier t (all rows for
  // the global-table tier); the result is the same bit for bit
  if (const char* force = getenv("AJ_SCHUR_TIER")) {
    const int ft = atoi(force);
    AJ_REQUIRE(ft >= 0 && ft < NTIER, AJ_ERR_ARG, "AJ_SCHUR_TIER must be 0..5");
    for (int t = 0; t < NTIER; ++t)
      if (t != ft && cnt[t] > 0 && (t < ft || ft == TIER_G)) {
        AJ_CUDA(cudaMemcpyAsync(lists + (size_t)ft * nC1 + cnt[ft], lists + (size_t)t * nC1, sizeof(int32_t) * cnt[t],
                                cudaMemcpyDeviceToDevice, st));
        cnt[ft] += cnt[t];
        cnt[t] = 0;
      }
  }
  for (int t = 0; t < NTIER; ++t) out.tier_rows[t] = cnt[t];

  SchurArgs a;
  a.cidx = in.cidx;
  a.cmap = in.cmap;
  a.fmap = in.fmap;
  a.ptr = in.ptr;
  a.col = in.col;
  a.ah = in.ah;
  a.inF = in.inF;
  a.partner = in.partner;
  a.b11 = in.b11;
  a.b12 = in.b12;
  a.Vptr = in.Vptr;
  a.Vcol = in.Vcol;
  a.Vval = in.Vval;
  a.FCptr = FCptr;
  a.FCcol = FCcol;
  a.FCval = FCval;
  a.tau = in.tau;
  out.row_cnt = dalloc<int64_t>(nC1, st);
  out.row_off = dalloc<int64_t>(nC1, st);
  out.lrow_cnt = dalloc<int64_t>(nC1, st);
  out.lrow_off = dalloc<int64_t>(nC1, st);
  a.row_cnt = out.row_cnt;
  a.row_off = out.row_off;
  a.lrow_cnt = out.lrow_cnt;
  a.lrow_off = out.lrow_off;
  unsigned long long* cursor = dalloc<unsigned long long>(3, st);  // S, L cursors; products
  a.cursor = cursor;
  a.lcursor = cursor + 1;

  // per tier: resident grid and scratch words (one region of the scratch buffer per tier)
  struct TierRun {
    int groups;
    size_t words;
    int ctas;
  } tr[NTIER];
  TierW1::prepare();
  TierW2::prepare();
  TierP4::prepare();
  TierC8::prepare();
  TierC16::prepare();
  tr[TIER_W1] = {8, TierW1::words(), TierW1::resident_ctas()};
  tr[TIER_W2] = {4, TierW2::words(), TierW2::resident_ctas()};
  tr[TIER_P4] = {2, TierP4::words(), TierP4::resident_ctas()};
  tr[TIER_C8] = {1, TierC8::words(), TierC8::resident_ctas()};
  tr[TIER_C16] = {1, TierC16::words(), TierC16::resident_ctas()};
  tr[TIER_G] = {1, TierG::words(), num_sms()};
  size_t scr_words = 2, scr_off[NTIER] = {};
  int grid[NTIER];
  int nactive = 0;
  for (int t = 0; t < NTIER; ++t) {
    grid[t] = std::max(1, std::min(tr[t].ctas, ceil_div(std::max(cnt[t], 1), tr[t].groups)));
    scr_off[t] = scr_words;
    if (cnt[t] > 0 && t != TIER_G) {
      scr_words += (size_t)grid[t] * tr[t].groups * tr[t].words;
      ++nactive;
    }
  }
  int32_t* scratch = dalloc<int32_t>(scr_words, st);
  // concurrent tiers when more than one has rows and none fills the GPU by itself for long
  // (AJ_SCHUR_SERIAL=1, testing: one stream)
#ifdef AJ_SCHUR_PROF
  const bool fork = false;
#else
  const bool fork = nactive > 1 && !getenv("AJ_SCHUR_SERIAL");
#endif
  TierStreams* tsp = fork ? &tier_streams() : nullptr;
  int32_t* scratchG = nullptr;
  int* err = ctr + NTIER + 1;

  int64_t cap = std::max<int64_t>(in.cap_hint, (int64_t)nC * 16);
  int64_t lcap = std::max<int64_t>((int64_t)nC * 64, 1024);
  for (int attempt = 0; attempt < 2; ++attempt) {
    out.tmp_col = dalloc<int32_t>(cap, st);
    out.tmp_val = dalloc<double>(cap, st);
    out.ltmp_col = dalloc<int32_t>(lcap, st);
    out.ltmp_val = dalloc<double>(lcap, st);
    a.tmp_col = out.tmp_col;
    a.tmp_val = out.tmp_val;
    a.ltmp_col = out.ltmp_col;
    a.ltmp_val = out.ltmp_val;
    a.cap = cap;
    a.lcap = lcap;
    AJ_CUDA(cudaMemsetAsync(cursor, 0, 3 * sizeof(unsigned long long), st));
    AJ_CUDA(cudaMemsetAsync(ctr + NTIER, 0, 2 * sizeof(int), st));
    auto L0 = [&](int t) { return lists + (size_t)t * nC1; };
#ifdef AJ_SCHUR_PROF
#define SDUMP(name, rows)                                                              \
  if ((rows) > 0 && nC >= 200000) {                                                    \
    char tg[64];                                                                       \
    snprintf(tg, sizeof tg, "nC=%d tier %s rows=%d", nC, name, (int)(rows));           \
    schur_prof_dump(tg, st);                                                           \
  }
#else
#define SDUMP(name, rows)
#endif
    if (fork) AJ_CUDA(cudaEventRecord(tsp->fork, st));
    auto TS = [&](int t) -> cudaStream_t {  // the tier's stream, ordered after the work queued on st so far
      if (!fork) return st;
      AJ_CUDA(cudaStreamWaitEvent(tsp->s[t], tsp->fork, 0));
      return tsp->s[t];
    };
    auto SCR = [&](int t) { return scratch + scr_off[t]; };
    // the largest tables first: their few long rows are the tail of the level
    if (cnt[TIER_C16]) TierC16::launch(cnt[TIER_C16], L0(TIER_C16), a, SCR(TIER_C16), grid[TIER_C16], ovf, ctr + NTIER, err, cursor + 2, TS(TIER_C16));
    SDUMP("C16", cnt[TIER_C16]);
    if (cnt[TIER_C8]) TierC8::launch(cnt[TIER_C8], L0(TIER_C8), a, SCR(TIER_C8), grid[TIER_C8], nullptr, nullptr, err, cursor + 2, TS(TIER_C8));
    SDUMP("C8", cnt[TIER_C8]);
    if (cnt[TIER_P4]) TierP4::launch(cnt[TIER_P4], L0(TIER_P4), a, SCR(TIER_P4), grid[TIER_P4], nullptr, nullptr, err, cursor + 2, TS(TIER_P4));
    SDUMP("P4", cnt[TIER_P4]);
    if (cnt[TIER_W2]) TierW2::launch(cnt[TIER_W2], L0(TIER_W2), a, SCR(TIER_W2), grid[TIER_W2], nullptr, nullptr, err, cursor + 2, TS(TIER_W2));
    SDUMP("W2", cnt[TIER_W2]);
    if (cnt[TIER_W1]) TierW1::launch(cnt[TIER_W1], L0(TIER_W1), a, SCR(TIER_W1), grid[TIER_W1], nullptr, nullptr, err, cursor + 2, TS(TIER_W1));
    SDUMP("W1", cnt[TIER_W1]);
    if (fork)
      for (int t = TIER_W1; t <= TIER_C16; ++t)
        if (cnt[t]) {
          AJ_CUDA(cudaEventRecord(tsp->done[t], tsp->s[t]));
          AJ_CUDA(cudaStreamWaitEvent(st, tsp->done[t], 0));
        }
    int nov = 0;
    if (cnt[TIER_C16]) nov = read1(ctr + NTIER, st);
    // tier G: the rows routed there plus the C16 overflows
    int ng = cnt[TIER_G];
    if (nov > 0) {
      AJ_CUDA(cudaMemcpyAsync(L0(TIER_G) + ng, ovf, sizeof(int32_t) * nov, cudaMemcpyDeviceToDevice, st));
      ng += nov;
    }
    out.tier_rows[TIER_G] = ng;
    out.ovf_rows = nov;
    if (ng > 0) {
      const int gg = std::max(1, std::min(ng, num_sms()));
      if (!scratchG) scratchG = dalloc<int32_t>((size_t)num_sms() * TierG::words(), st);
      TierG::launch(ng, L0(TIER_G), a, scratchG, gg, nullptr, nullptr, err, cursor + 2, st);
    }
    unsigned long long used[3];
    int errc = 0;
    AJ_CUDA(cudaMemcpyAsync(used, cursor, sizeof(used), cudaMemcpyDeviceToHost, st));
    AJ_CUDA(cudaMemcpyAsync(&errc, err, sizeof(int), cudaMemcpyDeviceToHost, st));
    AJ_CUDA(cudaStreamSynchronize(st));
    AJ_REQUIRE(errc == 0, AJ_ERR_CAPACITY,
               "Schur complement: more than 49152 candidate columns in one row (raise tau_drop)");
    out.products = (int64_t)used[2];
    out.nnz_tmp = (int64_t)used[0];
    out.nnz_ltmp = (int64_t)used[1];
    if ((int64_t)used[0] <= cap && (int64_t)used[1] <= lcap) break;
    for (void* q : {(void*)out.tmp_col, (void*)out.tmp_val, (void*)out.ltmp_col, (void*)out.ltmp_val}) dfree(q, st);
    cap = std::max<int64_t>(cap, (int64_t)used[0]);  // exact sizes now known: run again
    lcap = std::max<int64_t>(lcap, (int64_t)used[1]);
    AJ_REQUIRE(attempt == 0, AJ_ERR_CAPACITY, "Schur complement: temp capacity");
  }
  for (void* q : {(void*)FCptr, (void*)FCcol, (void*)FCval, (void*)ctr, (void*)lists, (void*)cursor, (void*)scratch,
                  (void*)scratchG})
    dfree(q, st);
}

// ---------------------------------------------------------------------------
// S from its computed upper triangle: S = U + strict(U)^T.  Rows of U come as sorted
// runs (diagonal first); the transpose of the strict part is a stable radix sort of the
// entries by column (input in row order -> every target row receives its entries in
// ascending source row, i.e. sorted), then each full row is written as [lower | upper].
namespace {
__global__ void k_upper_gather(int nC, const int64_t* __restrict__ uptr, const int64_t* __restrict__ row_off,
                               const int32_t* __restrict__ tcol, const double* __restrict__ tval,
                               int32_t* __restrict__ ucol, double* __restrict__ uval, uint32_t* __restrict__ key,
                               int32_t* __restrict__ erow, unsigned long long* __restrict__ lcnt) {
  const int lane = threadIdx.x & 31;
  for (int r = (blockIdx.x * TBs + threadIdx.x) >> 5; r < nC; r += (gridDim.x * TBs) >> 5) {
    const int64_t d0 = uptr[r], cnt = uptr[r + 1] - d0, s0 = row_off[r];
    for (int64_t t = lane; t < cnt; t += 32) {
      const int32_t c2 = tcol[s0 + t];
      ucol[d0 + t] = c2;
      uval[d0 + t] = tval[s0 + t];
      erow[d0 + t] = r;
      if (c2 > r) {
        key[d0 + t] = (uint32_t)c2;
        atomicAdd(&lcnt[c2], 1ull);
      } else {
        key[d0 + t] = (uint32_t)nC;  // the diagonal: sorts behind every row
      }
    }
  }
}
__global__ void k_full_rows(int nC, const int64_t* __restrict__ Sptr, const int64_t* __restrict__ lptr,
                            const int64_t* __restrict__ uptr, const int32_t* __restrict__ sidx,
                            const int32_t* __restrict__ ucol, const double* __restrict__ uval,
                            const int32_t* __restrict__ erow, int32_t* __restrict__ Scol, double* __restrict__ Sval) {
  const int lane = threadIdx.x & 31;
  for (int r = (blockIdx.x * TBs + threadIdx.x) >> 5; r < nC; r += (gridDim.x * TBs) >> 5) {
    const int64_t d0 = Sptr[r], l0 = lptr[r], nlow = lptr[r + 1] - l0, u0 = uptr[r], nup = uptr[r + 1] - u0;
    for (int64_t t = lane; t < nlow; t += 32) {
      const int32_t e = sidx[l0 + t];
      Scol[d0 + t] = erow[e];
      Sval[d0 + t] = uval[e];
    }
    for (int64_t t = lane; t < nup; t += 32) {
      Scol[d0 + nlow + t] = ucol[u0 + t];
      Sval[d0 + nlow + t] = uval[u0 + t];
    }
  }
}
__global__ void k_add_counts(int n, const unsigned long long* __restrict__ a, const int64_t* __restrict__ b,
                             int64_t* __restrict__ out) {
  for (int i = blockIdx.x * TBs + threadIdx.x; i < n; i += gridDim.x * TBs) out[i] = (int64_t)a[i] + b[i];
}
__global__ void k_iota32(int64_t n, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)TBs + threadIdx.x; i < n; i += (int64_t)gridDim.x * TBs) out[i] = (int32_t)i;
}
template <typename T>
int64_t scan_to_ptr(const T* cnt, int64_t*& ptr, int n, cudaStream_t st) {
  ptr = dalloc<int64_t>((size_t)n + 1, st);
  AJ_CUDA(cudaMemsetAsync(ptr, 0, sizeof(int64_t), st));
  if (n == 0) return 0;
  size_t tmp = 0;
  AJ_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt, ptr + 1, n, st));
  void* t = dalloc<char>(tmp, st);
  AJ_CUDA(cub::DeviceScan::InclusiveSum(t, tmp, cnt, ptr + 1, n, st));
  dfree(t, st);
  return read1(ptr + n, st);
}
}  // namespace

void schur_mirror(int nC, const SchurOut& so, Csr& S, cudaStream_t st) {
  S.n = nC;
  int64_t* uptr = nullptr;
  const int64_t nU = scan_to_ptr(so.row_cnt, uptr, nC, st);
  AJ_REQUIRE(nU < (int64_t)INT32_MAX, AJ_ERR_CAPACITY, "Schur complement: more than 2^31 upper entries");
  const int64_t nU1 = std::max<int64_t>(nU, 1);
  int32_t* ucol = dalloc<int32_t>(nU1, st);
  double* uval = dalloc<double>(nU1, st);
  uint32_t* key = dalloc<uint32_t>(nU1, st);
  uint32_t* key2 = dalloc<uint32_t>(nU1, st);
  int32_t* idx = dalloc<int32_t>(nU1, st);
  int32_t* idx2 = dalloc<int32_t>(nU1, st);
  int32_t* erow = dalloc<int32_t>(nU1, st);
  unsigned long long* lcnt = dalloc<unsigned long long>((size_t)nC + 1, st);
  AJ_CUDA(cudaMemsetAsync(lcnt, 0, sizeof(unsigned long long) * ((size_t)nC + 1), st));
  const int gg = std::max(1, std::min(ceil_div((int64_t)std::max(nC, 1) * 32, TBs), num_sms() * 32));
  k_upper_gather<<<gg, TBs, 0, st>>>(nC, uptr, so.row_off, so.tmp_col, so.tmp_val, ucol, uval, key, erow, lcnt);
  AJ_LAUNCHED();
  const int gi = std::max(1, std::min(ceil_div(nU1, TBs), num_sms() * 16));
  k_iota32<<<gi, TBs, 0, st>>>(nU, idx);
  AJ_LAUNCHED();
  int bits = 1;
  while ((1ll << bits) <= (long long)nC) ++bits;
  {
    size_t tmp = 0;
    AJ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, key2, idx, idx2, (int)nU, 0, bits, st));
    void* t = dalloc<char>(tmp, st);
    AJ_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, key, key2, idx, idx2, (int)nU, 0, bits, st));
    dfree(t, st);
  }
  int64_t* lptr = nullptr;
  scan_to_ptr(lcnt, lptr, nC, st);
  int64_t* fcnt = dalloc<int64_t>(std::max(nC, 1), st);
  k_add_counts<<<std::max(1, std::min(ceil_div(std::max(nC, 1), TBs), num_sms() * 16)), TBs, 0, st>>>(nC, lcnt,
                                                                                                     so.row_cnt, fcnt);
  AJ_LAUNCHED();
  S.nnz = scan_to_ptr(fcnt, S.ptr, nC, st);
  S.col = dalloc<int32_t>(std::max<int64_t>(S.nnz, 1), st);
  S.val = dalloc<double>(std::max<int64_t>(S.nnz, 1), st);
  k_full_rows<<<gg, TBs, 0, st>>>(nC, S.ptr, lptr, uptr, idx2, ucol, uval, erow, S.col, S.val);
  AJ_LAUNCHED();
  for (void* q : {(void*)uptr, (void*)ucol, (void*)uval, (void*)key, (void*)key2, (void*)idx, (void*)idx2, (void*)erow,
                  (void*)lcnt, (void*)lptr, (void*)fcnt})
    dfree(q, st);
}

}  // namespace aj
