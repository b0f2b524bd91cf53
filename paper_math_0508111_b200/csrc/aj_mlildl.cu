// Symmetric multilevel incomplete LDL^T preconditioner on the GPU.
//
// PAPER.md sect. 7 (l.790-973): per level (i) symmetric scaling (l.805-807),
// (ii) 1x1 / matched 2x2 pivots with the d1/d2 test (l.864-874) and the
// inverse-based bound ||L^{-1}|| <= kappa with postponement (l.884-897),
// (iii) L = A_CF B^{-1} with dropping |l| < tau_drop (l.909-911), explicit
// Schur complement of the postponed nodes (l.940-945), recursion, dense coarse.
// The levels are realised as INDEPENDENT SETS (DESIGN.md sect. 3.3): level 0
// is the red half of the bipartite lattice, deeper levels maximal independent
// sets of pivot blocks in the strong graph, so every step -- scaling, pivot
// tests, independent-set rounds, budget repair, L/L^T/S construction and the
// forward/backward application -- is a level-parallel kernel over rows.
//
// Data layout (HBM): every level matrix is CSR (int64 row pointers, int32
// sorted column indices, fp64 values, explicit diagonal).  Per level the
// factor keeps L (rows = coarse nodes, cols = level index, values L_cf*D_f)
// and L^T (rows = level nodes, cols = coarse index, values L_cf) so both
// substitutions are pure gathers (no atomics).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "aj_common.cuh"
#include "aj_kernels.cuh"
#include "aj_mlildl.cuh"
#include "aj_sparse.cuh"

namespace aj {

constexpr int TB = 256;
static int grid_for(int64_t n) { return std::max(1, ceil_div(n, TB)); }

// ---- sub-warp row groups: SG lanes per CSR row (coalesced row segments) ------
constexpr int SG = 8;
__device__ __forceinline__ unsigned sg_mask() {
  const int lane = threadIdx.x & 31;
  return ((1u << SG) - 1u) << (lane & ~(SG - 1));
}
__device__ __forceinline__ double sg_max(double v, unsigned m) {
#pragma unroll
  for (int o = SG / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(m, v, o));
  return v;
}
__device__ __forceinline__ double sg_sum(double v, unsigned m) {
#pragma unroll
  for (int o = SG / 2; o > 0; o >>= 1) v += __shfl_xor_sync(m, v, o);
  return v;
}
__device__ __forceinline__ int sg_min_i(int v, unsigned m) {
#pragma unroll
  for (int o = SG / 2; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(m, v, o));
  return v;
}
__device__ __forceinline__ int sg_or_i(int v, unsigned m) {
#pragma unroll
  for (int o = SG / 2; o > 0; o >>= 1) v |= __shfl_xor_sync(m, v, o);
  return v;
}
static int grid_sg(int64_t rows) { return std::max(1, std::min(ceil_div(rows * SG, TB), num_sms() * 32)); }


// ----------------------------------------------------------------------------
// level-0 CSR of A - sigma I on planes [z0, z0 + nz) of the lattice, periodic in x and y;
// in z periodic inside the block (open_z = 0: the whole lattice, nz = L) or with open
// faces (open_z = 1: a slab's diagonal block, couplings across the faces dropped).
// Sorted rows of 7 (interior), 6 (face planes) or 5 (nz = 1) entries.
__global__ void k_lattice_csr(int L, int nz, int open_z, const double* __restrict__ eps, double hop, double sigma,
                              int64_t* __restrict__ ptr, int32_t* __restrict__ col, double* __restrict__ val) {
  const int64_t P = (int64_t)L * L, n = P * nz;
  for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < n; s += (int64_t)gridDim.x * TB) {
    const int i = (int)(s % L), j = (int)((s / L) % L), k = (int)(s / P);
    const bool dn = !open_z || k > 0, up = !open_z || k < nz - 1;
    auto len = [&](int kk) { return 5 + ((!open_z || kk > 0) ? 1 : 0) + ((!open_z || kk < nz - 1) ? 1 : 0); };
    // rows before plane k: plane 0 has len(0) entries per row, the interior planes 7
    const int64_t base = (k == 0) ? 0 : P * (int64_t)len(0) + P * 7 * (int64_t)(k - 1);
    const int64_t p0 = base + (s - (int64_t)k * P) * len(k);
    int32_t c[7];
    int m = 0;
    c[m++] = (int32_t)s;
    c[m++] = (int32_t)(((i + L - 1) % L) + (int64_t)L * (j + (int64_t)L * k));
    c[m++] = (int32_t)(((i + 1) % L) + (int64_t)L * (j + (int64_t)L * k));
    c[m++] = (int32_t)(i + (int64_t)L * (((j + L - 1) % L) + (int64_t)L * k));
    c[m++] = (int32_t)(i + (int64_t)L * (((j + 1) % L) + (int64_t)L * k));
    if (dn) c[m++] = (int32_t)(i + (int64_t)L * (j + (int64_t)L * ((k + nz - 1) % nz)));
    if (up) c[m++] = (int32_t)(i + (int64_t)L * (j + (int64_t)L * ((k + 1) % nz)));
    for (int a = 1; a < m; ++a) {  // insertion sort
      int32_t v = c[a];
      int b = a - 1;
      while (b >= 0 && c[b] > v) {
        c[b + 1] = c[b];
        --b;
      }
      c[b + 1] = v;
    }
    ptr[s] = p0;
    if (s == n - 1) ptr[n] = p0 + m;
    for (int a = 0; a < m; ++a) {
      col[p0 + a] = c[a];
      val[p0 + a] = (c[a] == (int32_t)s) ? (eps[s] - sigma) : hop;
    }
  }
}

// ----------------------------------------------------------------------------
// (i) scaling D_i = 1/sqrt(max_j |a_ij|); scaled values a^_ij = a_ij * (D_i D_j)
__global__ void k_rowmax_scale(int n, const int64_t* __restrict__ ptr, const double* __restrict__ val,
                               double* __restrict__ D) {
  const int gl = threadIdx.x & (SG - 1);
  const unsigned m = sg_mask();
  for (int i = (blockIdx.x * TB + threadIdx.x) / SG; i < n; i += gridDim.x * (TB / SG)) {
    double mx = 0.0;
    for (int64_t e = ptr[i] + gl; e < ptr[i + 1]; e += SG) mx = fmax(mx, fabs(val[e]));
    mx = sg_max(mx, m);
    if (gl == 0) D[i] = (mx > 0.0) ? 1.0 / sqrt(mx) : 1.0;
  }
}

// scaled values + per-row pivot quality:
//   dg = a^_ii, lmax1 = max_{j!=i}|a^_ij| / |a^_ii|, d1 = sum_{j!=i}|a^_ij| / |a^_ii|,
//   p = argmax_{j!=i} |a^_ij| (ties -> smallest j; rows are column sorted)
__global__ void k_scaled_quality(int n, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                 const double* __restrict__ val, const double* __restrict__ D,
                                 double* __restrict__ ah, double* __restrict__ dg,
                                 double* __restrict__ lmax1, double* __restrict__ d1,
                                 int32_t* __restrict__ prop, int8_t* __restrict__ ok1, double kappa) {
  const int gl = threadIdx.x & (SG - 1);
  const unsigned m = sg_mask();
  for (int i = (blockIdx.x * TB + threadIdx.x) / SG; i < n; i += gridDim.x * (TB / SG)) {
    const double Di = D[i];
    double diag = 0.0, cm = 0.0, os = 0.0;
    int32_t p = INT32_MAX;
    for (int64_t e = ptr[i] + gl; e < ptr[i + 1]; e += SG) {
      const int32_t j = col[e];
      const double v = val[e] * (Di * D[j]);
      ah[e] = v;
      if (j == i) {
        diag = v;
      } else {
        const double a = fabs(v);
        os += a;
        if (a > cm) {  // lane-local: first (smallest j) maximum
          cm = a;
          p = j;
        }
      }
    }
    // group reduction: max |a| with the smallest column among ties
#pragma unroll
    for (int o = SG / 2; o > 0; o >>= 1) {
      const double cm2 = __shfl_xor_sync(m, cm, o);
      const int32_t p2 = __shfl_xor_sync(m, p, o);
      if (cm2 > cm || (cm2 == cm && p2 < p)) {
        cm = cm2;
        p = p2;
      }
    }
    os = sg_sum(os, m);
    diag = sg_sum(diag, m);  // exactly one lane holds the diagonal, the others 0
    if (gl == 0) {
      const double ad = fabs(diag);
      dg[i] = diag;
      const double l1 = (ad > 0.0) ? cm / ad : INFINITY;
      lmax1[i] = l1;
      d1[i] = (ad > 0.0) ? os / ad : INFINITY;
      prop[i] = (cm > 0.0 || p != INT32_MAX) ? (p == INT32_MAX ? -1 : p) : -1;
      ok1[i] = (l1 <= kappa - 1.0 && diag != 0.0) ? 1 : 0;
    }
  }
}

// (ii-a) 2x2 candidates: mutual strongest-neighbour proposals (sect. 6.2), d2 < d1_lead
// and lmax2 <= kappa - 1 (sect. 7.2).  Thread i handles the pair {i, p(i)} when i < p(i).
__global__ void k_pairs(int n, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                        const double* __restrict__ ah, const double* __restrict__ dg,
                        const double* __restrict__ d1, const int32_t* __restrict__ prop,
                        const int8_t* __restrict__ ok1, double kappa, int32_t* __restrict__ partner,
                        double* __restrict__ b11, double* __restrict__ b12, double* __restrict__ q,
                        int* __restrict__ npairs) {
  for (int i = blockIdx.x * TB + threadIdx.x; i < n; i += gridDim.x * TB) {
    const int32_t j = prop[i];
    if (j <= i || prop[j] != i) continue;
    if (ok1[i] && ok1[j]) continue;
    const double aii = dg[i], ajj = dg[j];
    const double aij = lookup(col, ah, ptr[i], ptr[i + 1], j);
    const double det = __dsub_rn(__dmul_rn(aii, ajj), __dmul_rn(aij, aij));
    if (det == 0.0) continue;
    const double B11 = ajj / det, B12 = -aij / det, B22 = aii / det;
    // merge rows i and j (both sorted) over neighbours c not in {i, j}
    int64_t ei = ptr[i], ej = ptr[j];
    const int64_t ei1 = ptr[i + 1], ej1 = ptr[j + 1];
    double lm2 = 0.0, d2 = 0.0;
    while (ei < ei1 || ej < ej1) {
      const int32_t ci = (ei < ei1) ? col[ei] : INT32_MAX;
      const int32_t cj = (ej < ej1) ? col[ej] : INT32_MAX;
      const int32_t c = min(ci, cj);
      double aci = 0.0, acj = 0.0;
      if (ci == c) aci = ah[ei++];
      if (cj == c) acj = ah[ej++];
      if (c == i || c == j) continue;
      // (l_ci, l_cj) = (a_ci, a_cj) B^{-1}; i < j
      const double w = fabs(lval_pair(aci, acj, B11, B12)) + fabs(lval_pair(aci, acj, B12, B22));
      lm2 = fmax(lm2, w);
      d2 += w;
    }
    const int lead = ok1[i] ? j : i;
    if (d2 < d1[lead] && lm2 <= kappa - 1.0) {
      partner[i] = j;
      partner[j] = i;
      b11[i] = B11;
      b12[i] = B12;
      b11[j] = B22;
      b12[j] = B12;
      q[i] = lm2;
      atomicAdd(npairs, 1);
    }
  }
}

// (ii-b) blocks: singles (ok1, unpaired) and pair leaders; red-set selection on level 0
__global__ void k_blocks(int n, int L, int z0, const int8_t* __restrict__ ok1, const double* __restrict__ dg,
                         const double* __restrict__ lmax1, const int32_t* __restrict__ partner,
                         int32_t* __restrict__ leader, double* __restrict__ q, double* __restrict__ b11,
                         int8_t* __restrict__ inF) {
  for (int i = blockIdx.x * TB + threadIdx.x; i < n; i += gridDim.x * TB) {
    const int32_t p = partner[i];
    if (p >= 0) {
      leader[i] = min(i, p);
    } else if (ok1[i]) {
      leader[i] = i;
      q[i] = lmax1[i];
      b11[i] = 1.0 / dg[i];
    } else {
      leader[i] = -1;
    }
    if (L > 0) {  // level 0: red sites of the bipartite split (reading R6), global parity
      const int x = i % L, y = (i / L) % L, z = z0 + i / (L * L);
      bool red = ((x + y + z) & 1) == 0;
      if (L & 1) red = red && x < L - 1 && y < L - 1 && z < L - 1;
      inF[i] = (p < 0 && ok1[i] && red) ? 1 : 0;
    }
  }
}

// MIS rank keys: key = bits(q) for block leaders (q >= 0), else max
__global__ void k_rank_keys(int n, const int32_t* __restrict__ leader, const double* __restrict__ q,
                            uint64_t* __restrict__ key, int32_t* __restrict__ idx) {
  for (int i = blockIdx.x * TB + threadIdx.x; i < n; i += gridDim.x * TB) {
    key[i] = (leader[i] == i) ? (uint64_t)__double_as_longlong(q[i]) : ~0ull;
    idx[i] = i;
  }
}
__global__ void k_rank_scatter(int n, const int32_t* __restrict__ sorted_idx, int32_t* __restrict__ rank) {
  for (int t = blockIdx.x * TB + threadIdx.x; t < n; t += gridDim.x * TB) rank[sorted_idx[t]] = t;
}

// status per block (at leader): 0 undecided, 1 selected, 2 removed
__global__ void k_mis_nbmin(int n, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                            const double* __restrict__ ah, double tau_s, const int32_t* __restrict__ leader,
                            const int8_t* __restrict__ status, const int32_t* __restrict__ rank,
                            int32_t* __restrict__ nbmin) {
  const int gl = threadIdx.x & (SG - 1);
  const unsigned msk = sg_mask();
  for (int i = (blockIdx.x * TB + threadIdx.x) / SG; i < n; i += gridDim.x * (TB / SG)) {
    const int32_t l = leader[i];
    if (l < 0 || status[l] != 0) continue;  // uniform inside the group
    int32_t m = INT32_MAX;
    for (int64_t e = ptr[i] + gl; e < ptr[i + 1]; e += SG) {
      const int32_t j = col[e];
      if (j == i || !(fabs(ah[e]) >= tau_s)) continue;
      const int32_t lj = leader[j];
      if (lj < 0 || lj == l || status[lj] != 0) continue;
      m = min(m, rank[lj]);
    }
    m = sg_min_i(m, msk);
    if (gl == 0) nbmin[i] = m;
  }
}
__global__ void k_mis_win(int n, const int32_t* __restrict__ leader, const int32_t* __restrict__ partner,
                          const int8_t* __restrict__ status, const int32_t* __restrict__ rank,
                          const int32_t* __restrict__ nbmin, int8_t* __restrict__ win) {
  for (int i = blockIdx.x * TB + threadIdx.x; i < n; i += gridDim.x * TB) {
    if (leader[i] != i || status[i] != 0) continue;
    int32_t m = nbmin[i];
    if (partner[i] >= 0) m = min(m, nbmin[partner[i]]);
    if (rank[i] < m) win[i] = 1;
  }
}
__global__ void k_mis_remove(int n, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                             const double* __restrict__ ah, double tau_s, const int32_t* __restrict__ leader,
                             const int8_t* __restrict__ status, const int8_t* __restrict__ win,
                             int8_t* __restrict__ rem) {
  const int gl = threadIdx.x & (SG - 1);
  const unsigned msk = sg_mask();
  for (int i = (blockIdx.x * TB + threadIdx.x) / SG; i < n; i += gridDim.x * (TB / SG)) {
    const int32_t l = leader[i];
    if (l < 0 || status[l] != 0 || win[l]) continue;  // uniform inside the group
    int hit = 0;
    for (int64_t e = ptr[i] + gl; e < ptr[i + 1] && !hit; e += SG) {
      const int32_t j = col[e];
      if (j == i || !(fabs(ah[e]) >= tau_s)) continue;
      const int32_t lj = leader[j];
      if (lj >= 0 && lj != l && win[lj]) hit = 1;
    }
    hit = sg_or_i(hit, msk);
    if (hit && gl == 0) rem[l] = 1;
  }
}
__global__ void k_mis_apply(int n, const int32_t* __restrict__ leader, int8_t* __restrict__ status,
                            int8_t* __restrict__ win, int8_t* __restrict__ rem, int* __restrict__ undecided) {
  int cnt = 0;
  for (int i = blockIdx.x * TB + threadIdx.x; i < n; i += gridDim.x * TB) {
    if (leader[i] != i || status[i] != 0) continue;
    if (win[i])
      status[i] = 1;
    else if (rem[i])
      status[i] = 2;
    else
      ++cnt;
    win[i] = 0;
    rem[i] = 0;
  }
  if (cnt) atomicAdd(undecided, cnt);
}
__global__ void k_mis_final(int n, const int32_t* __restrict__ leader, const int8_t* __restrict__ status,
                            int8_t* __restrict__ inF) {
  for (int i = blockIdx.x * TB + threadIdx.x; i < n; i += gridDim.x * TB) {
    const int32_t l = leader[i];
    inF[i] = (l >= 0 && status[l] == 1) ? 1 : 0;
  }
}

// Iterate the F blocks adjacent to row c (c not in F) and call fn(f, g, l_cf, l_cg, lead)
// once per block; g = -1 for singles.  Order: ascending position in row c of the
// first adjacent member.
template <typename Fn>
__device__ __forceinline__ void for_blocks_of_row(int c, const int64_t* __restrict__ ptr,
                                                  const int32_t* __restrict__ col,
                                                  const double* __restrict__ ah,
                                                  const int8_t* __restrict__ inF,
                                                  const int32_t* __restrict__ partner,
                                                  const double* __restrict__ b11,
                                                  const double* __restrict__ b12, Fn fn, int start = 0,
                                                  int stride = 1) {
  const int64_t lo = ptr[c], hi = ptr[c + 1];
  for (int64_t e = lo + start; e < hi; e += stride) {
    const int32_t u = col[e];
    if (u == c || !inF[u]) continue;
    const int32_t p = partner[u];
    if (p < 0) {
      fn(u, -1, __dmul_rn(ah[e], b11[u]), 0.0, u);
    } else {
      // handle the pair once: at the smaller adjacent member
      const int64_t ep = lookup_idx(col, lo, hi, p);
      if (ep >= 0 && p < u) continue;
      const double a_cp = (ep >= 0) ? ah[ep] : 0.0;
      const int32_t f = min(u, p), g = max(u, p);
      const double a_cf = (f == u) ? ah[e] : a_cp;
      const double a_cg = (g == u) ? ah[e] : a_cp;
      // l_cf = a_cf Binv[f,f] + a_cg Binv[g,f]; l_cg = a_cf Binv[f,g] + a_cg Binv[g,g]
      const double lf = lval_pair(a_cf, a_cg, b11[f], b12[g]);
      const double lg = lval_pair(a_cf, a_cg, b12[f], b11[g]);
      fn(f, g, lf, lg, f);
    }
  }
}

// (ii-c) row-budget repair: rows of L^{-1} bounded, sum_b w_cb <= kappa - 1;
// a violating row nominates its largest block (ties -> smallest leader).
__global__ void k_budget(int n, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                         const double* __restrict__ ah, const int8_t* __restrict__ inF,
                         const int32_t* __restrict__ partner, const double* __restrict__ b11,
                         const double* __restrict__ b12, double kappa, int8_t* __restrict__ nominate,
                         int* __restrict__ nviol) {
  const int gl = threadIdx.x & (SG - 1);
  const unsigned msk = sg_mask();
  for (int c = (blockIdx.x * TB + threadIdx.x) / SG; c < n; c += gridDim.x * (TB / SG)) {
    if (inF[c]) continue;  // uniform inside the group
    double budget = 0.0, wbest = -1.0;
    int32_t lbest = INT32_MAX;
    for_blocks_of_row(
        c, ptr, col, ah, inF, partner, b11, b12,
        [&](int32_t f, int32_t g, double lf, double lg, int32_t lead) {
          const double w = fabs(lf) + (g >= 0 ? fabs(lg) : 0.0);
          budget += w;
          if (w > wbest || (w == wbest && lead < lbest)) {
            wbest = w;
            lbest = lead;
          }
        },
        gl, SG);
    budget = sg_sum(budget, msk);
#pragma unroll
    for (int o = SG / 2; o > 0; o >>= 1) {
      const double w2 = __shfl_xor_sync(msk, wbest, o);
      const int32_t l2 = __shfl_xor_sync(msk, lbest, o);
      if (w2 > wbest || (w2 == wbest && l2 < lbest)) {
        wbest = w2;
        lbest = l2;
      }
    }
    if (gl == 0 && budget > kappa - 1.0) {
      nominate[lbest] = 1;
      atomicAdd(nviol, 1);
    }
  }
}
__global__ void k_budget_apply(int n, const int32_t* __restrict__ partner, int8_t* __restrict__ inF,
                               int8_t* __restrict__ nominate) {
  for (int i = blockIdx.x * TB + threadIdx.x; i < n; i += gridDim.x * TB) {
    if (!inF[i]) continue;
    const int32_t p = partner[i];
    const int32_t l = (p >= 0) ? min(i, p) : i;
    if (nominate[l]) inF[i] = 0;
  }
}
__global__ void k_clear_nominate(int n, const int32_t* __restrict__ partner, const int8_t* __restrict__ inF,
                                 int8_t* __restrict__ nominate, int* __restrict__ nF, int* __restrict__ npairsF) {
  int cf = 0, cp = 0;
  for (int i = blockIdx.x * TB + threadIdx.x; i < n; i += gridDim.x * TB) {
    nominate[i] = 0;
    if (inF[i]) {
      ++cf;
      if (partner[i] > i) ++cp;
    }
  }
  if (cf) atomicAdd(nF, cf);
  if (cp) atomicAdd(npairsF, cp);
}

// (iii) compaction helpers
__global__ void k_cflags(int n, const int8_t* __restrict__ inF, int32_t* __restrict__ flag) {
  for (int i = blockIdx.x * TB + threadIdx.x; i < n; i += gridDim.x * TB) flag[i] = inF[i] ? 0 : 1;
}
__global__ void k_cmap(int n, const int8_t* __restrict__ inF, const int32_t* __restrict__ scan,
                       int32_t* __restrict__ cmap, int32_t* __restrict__ cidx, int32_t* __restrict__ fidx,
                       int32_t* __restrict__ fmap,
                       int32_t* __restrict__ partner_out, const int32_t* __restrict__ partner,
                       double* __restrict__ b11, double* __restrict__ b12) {
  for (int i = blockIdx.x * TB + threadIdx.x; i < n; i += gridDim.x * TB) {
    if (inF[i]) {
      cmap[i] = -1;
      fidx[i - scan[i]] = i;  // scan counts the C nodes before i
      fmap[i] = i - scan[i];
      partner_out[i] = partner[i];
    } else {
      cmap[i] = scan[i];
      cidx[scan[i]] = i;
      fmap[i] = -1;
      partner_out[i] = -1;
      b11[i] = 0.0;
      b12[i] = 0.0;
    }
  }
}

// ----------------------------------------------------------------------------
// Schur complement S = A^_CC - A^_CF B^{-1} A^_FC, symmetric by construction,
// off-diagonals with |s| < tau dropped.  One warp per coarse row.
// Virtual 2x2 blocks (reading R17): every stored coupling |a^_uv| >= tau_v between two pivot
// singles u != v (weak by construction of the independent set) gets
// b'_uv = -(a^_uv (B_uu B_vv)) (product ordered by index) -- the first-order term
// of (B_d + E)^{-1}.  Lists per level node (only pivot singles have entries).
template <bool FILL>
__global__ void k_virtual(int n, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                          const double* __restrict__ ah, const int8_t* __restrict__ inF,
                          const int32_t* __restrict__ partner, const double* __restrict__ b11, double tau_v,
                          int64_t* __restrict__ cnt_or_ptr, int32_t* __restrict__ Vcol, double* __restrict__ Vval) {
  for (int u = blockIdx.x * TB + threadIdx.x; u < n; u += gridDim.x * TB) {
    int64_t w = FILL ? cnt_or_ptr[u] : 0;
    if (inF[u] && partner[u] < 0) {
      for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e) {
        const int32_t v = col[e];
        if (v == u || !inF[v] || partner[v] >= 0 || fabs(ah[e]) < tau_v) continue;
        if (FILL) {
          const int32_t lo = min(u, v), hi = max(u, v);
          Vcol[w] = v;
          Vval[w] = -__dmul_rn(ah[e], __dmul_rn(b11[lo], b11[hi]));
        }
        ++w;
      }
    }
    if (!FILL) cnt_or_ptr[u] = w;
  }
}

__global__ void k_iota(int n, int32_t* __restrict__ out) {
  for (int i = blockIdx.x * TB + threadIdx.x; i < n; i += gridDim.x * TB) out[i] = i;
}

// ----------------------------------------------------------------------------
// dense coarse inverse: Gauss-Jordan with partial pivoting on [A | I]
__global__ void k_dense_init(int n, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                             const double* __restrict__ val, double* __restrict__ M) {
  const int64_t w = 2 * (int64_t)n;
  for (int64_t t = blockIdx.x * (int64_t)TB + threadIdx.x; t < (int64_t)n * w; t += (int64_t)gridDim.x * TB) {
    const int64_t i = t / w, j = t % w;
    M[t] = (j == n + i) ? 1.0 : 0.0;
  }
}
__global__ void k_dense_scatter(int n, const int64_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                const double* __restrict__ val, double* __restrict__ M) {
  for (int i = blockIdx.x * TB + threadIdx.x; i < n; i += gridDim.x * TB)
    for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) M[(int64_t)i * 2 * n + col[e]] = val[e];
}
__global__ void k_gj_pivot(int n, int k, double* __restrict__ M, double* __restrict__ fcol,
                           int* __restrict__ singular) {
  // one CTA: find pivot row, swap rows k <-> p, scale row k, save the elimination column
  __shared__ double sv[TB];
  __shared__ int si[TB];
  const int64_t w = 2 * (int64_t)n;
  double best = -1.0;
  int bi = k;
  for (int i = k + threadIdx.x; i < n; i += TB) {
    const double a = fabs(M[(int64_t)i * w + k]);
    if (a > best) {
      best = a;
      bi = i;
    }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = TB / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      if (sv[threadIdx.x + s] > sv[threadIdx.x] ||
          (sv[threadIdx.x + s] == sv[threadIdx.x] && si[threadIdx.x + s] < si[threadIdx.x])) {
        sv[threadIdx.x] = sv[threadIdx.x + s];
        si[threadIdx.x] = si[threadIdx.x + s];
      }
    }
    __syncthreads();
  }
  const int p = si[0];
  if (sv[0] <= 0.0) {
    if (threadIdx.x == 0) *singular = 1;
    return;
  }
  if (p != k)
    for (int64_t j = threadIdx.x; j < w; j += TB) {
      const double t = M[(int64_t)k * w + j];
      M[(int64_t)k * w + j] = M[(int64_t)p * w + j];
      M[(int64_t)p * w + j] = t;
    }
  __syncthreads();
  const double inv = 1.0 / M[(int64_t)k * w + k];
  __syncthreads();
  for (int64_t j = threadIdx.x; j < w; j += TB) M[(int64_t)k * w + j] *= inv;
  for (int i = threadIdx.x; i < n; i += TB) fcol[i] = (i == k) ? 0.0 : M[(int64_t)i * w + k];
}
__global__ void k_gj_elim(int n, int k, double* __restrict__ M, const double* __restrict__ fcol) {
  const int64_t w = 2 * (int64_t)n;
  // rows i != k: M[i, j] -= f_i * M[k, j] for j > k (columns <= k are never read again)
  for (int i = blockIdx.y; i < n; i += gridDim.y) {
    const double f = fcol[i];  // 0 for i == k
    if (f == 0.0) continue;
    double* Mi = M + (int64_t)i * w;
    const double* Mk = M + (int64_t)k * w;
    for (int64_t j = k + 1 + blockIdx.x * (int64_t)TB + threadIdx.x; j < w; j += (int64_t)gridDim.x * TB)
      Mi[j] -= f * Mk[j];
  }
}
// Gauss-Jordan with implicit row pivoting, one launch per column (the default):
// the rows are never swapped; prow holds the scaled pivot row of step k.  Step k
// eliminates column k from every row but the pivot row, records each CTA's best
// candidate for column k+1 among the rows not yet pivoted (largest |a|, smallest
// row on ties -- the rule of k_gj_pivot), and the last CTA to finish picks the next
// pivot row, scales it and stages it in prow for step k+1.  Per element the
// arithmetic is that of k_gj_pivot + k_gj_elim.
struct GjState {
  int* prow_idx;        // pivot row of each step (n)
  int8_t* pivoted;      // row already used as a pivot (n)
  double* prow;         // 2 x 2n staged, scaled pivot rows (double buffer)
  double* pv;           // per-CTA candidate |a|
  int* pi;              // per-CTA candidate row
  unsigned int* count;  // CTAs finished in the current step
  int* singular;
};

__device__ void gj_pick_and_stage(int n, int k1, double* __restrict__ M, GjState S, int nparts) {
  // one CTA (TB threads): reduce the candidates for column k1 (largest |a|, smallest
  // row on ties), scale the pivot row, stage it
  __shared__ double rv[TB];
  __shared__ int ri[TB];
  __shared__ int s_p;
  __shared__ double s_inv;
  const int64_t w = 2 * (int64_t)n;
  double bb = -1.0;
  int bp = n;
  for (int c = threadIdx.x; c < nparts; c += TB) {
    const double v = __ldcg(&S.pv[c]);
    const int ix = __ldcg(&S.pi[c]);
    if (v > bb || (v == bb && ix < bp)) {
      bb = v;
      bp = ix;
    }
  }
  rv[threadIdx.x] = bb;
  ri[threadIdx.x] = bp;
  __syncthreads();
  for (int s2 = TB / 2; s2 > 0; s2 >>= 1) {
    if (threadIdx.x < s2 &&
        (rv[threadIdx.x + s2] > rv[threadIdx.x] || (rv[threadIdx.x + s2] == rv[threadIdx.x] && ri[threadIdx.x + s2] < ri[threadIdx.x]))) {
      rv[threadIdx.x] = rv[threadIdx.x + s2];
      ri[threadIdx.x] = ri[threadIdx.x + s2];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bb = rv[0];
    bp = ri[0];
    if (!(bb > 0.0) || bp >= n) {
      *S.singular = 1;
      bp = -1;
    } else {
      S.prow_idx[k1] = bp;
      S.pivoted[bp] = 1;
      s_inv = 1.0 / __ldcg(&M[(int64_t)bp * w + k1]);
    }
    s_p = bp;
  }
  __syncthreads();
  const int p = s_p;
  if (p < 0) return;
  const double inv = s_inv;
  double* pr = S.prow + (int64_t)(k1 & 1) * w;
  for (int64_t j = k1 + threadIdx.x; j < w; j += blockDim.x) {
    const double v = __ldcg(&M[(int64_t)p * w + j]) * inv;
    M[(int64_t)p * w + j] = v;
    pr[j] = v;
  }
}

__global__ void k_gj_first(int n, double* __restrict__ M, GjState S) {
  // candidates for column 0 over all rows, then pick/stage (single CTA)
  __shared__ double sv[TB];
  __shared__ int si[TB];
  const int64_t w = 2 * (int64_t)n;
  double best = -1.0;
  int bi = n;
  for (int i = threadIdx.x; i < n; i += TB) {
    const double a = fabs(M[(int64_t)i * w]);
    if (a > best) {
      best = a;
      bi = i;
    }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s2 = TB / 2; s2 > 0; s2 >>= 1) {
    if (threadIdx.x < s2 &&
        (sv[threadIdx.x + s2] > sv[threadIdx.x] || (sv[threadIdx.x + s2] == sv[threadIdx.x] && si[threadIdx.x + s2] < si[threadIdx.x]))) {
      sv[threadIdx.x] = sv[threadIdx.x + s2];
      si[threadIdx.x] = si[threadIdx.x + s2];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    S.pv[0] = sv[0];
    S.pi[0] = si[0];
  }
  __threadfence_block();
  __syncthreads();
  gj_pick_and_stage(n, 0, M, S, 1);
}

__global__ void __launch_bounds__(TB) k_gj_step(int n, int k, double* __restrict__ M, GjState S) {
  __shared__ bool s_last;
  if (*(volatile int*)S.singular) return;  // a previous step found no pivot
  const int64_t w = 2 * (int64_t)n;
  const int p = S.prow_idx[k];
  const double* pr = S.prow + (int64_t)(k & 1) * w;
  const bool next = k + 1 < n;
  double best = -1.0;  // this CTA's candidate for column k+1 (kept by thread 0)
  int bi = n;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    double* Mi = M + (int64_t)i * w;
    if (i != p) {
      const double f = Mi[k];
      if (f != 0.0)
        for (int64_t j = k + 1 + threadIdx.x; j < w; j += TB) Mi[j] -= f * pr[j];
    }
    __syncthreads();
    if (threadIdx.x == 0 && next && !S.pivoted[i]) {
      const double a = fabs(Mi[k + 1]);
      if (a > best) {  // rows visited in ascending order: the first maximum wins ties
        best = a;
        bi = i;
      }
    }
  }
  if (!next) return;
  if (threadIdx.x == 0) {
    S.pv[blockIdx.x] = best;
    S.pi[blockIdx.x] = bi;
    __threadfence();
    s_last = atomicAdd(S.count, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  gj_pick_and_stage(n, k + 1, M, S, gridDim.x);
  if (threadIdx.x == 0) *S.count = 0u;
}

// ---- blocked Gauss-Jordan (default for the coarse inverse; DESIGN.md sect. 4) ----------
// Panels of GB columns.  For panel [k0, k0+b): (1) the panel columns of every row are
// copied (Pold, untouched, and Pw, the working copy); (2) b per-column steps on Pw only
// (n x b, L2-resident) choose the pivot rows P exactly like k_gj_step (largest |a| among
// the rows not yet pivoted, smallest row on ties) and eliminate within the panel;
// (3) Binv = Pold[P, :]^{-1} (b x b, one CTA, partial pivoting); W = Binv M[P, c] for the
// columns c >= k0+b still read; (4) the block Gauss-Jordan update of every row:
// M[P_l, c] = W[l, c], M[i, c] -= Pold[i, :] W[:, c] (i not in P) -- one rank-b pass over
// the matrix per panel instead of b passes.  Row P_k of the right half ends as row k of
// the inverse, as with implicit pivoting (k_gj_extract_perm).
constexpr int GB = 32;

__global__ void k_pan_load(int n, const double* __restrict__ M, int k0, int b, double* __restrict__ Pold,
                           double* __restrict__ Pw) {
  const int64_t w = 2 * (int64_t)n;
  for (int64_t t = blockIdx.x * (int64_t)TB + threadIdx.x; t < (int64_t)n * b; t += (int64_t)gridDim.x * TB) {
    const int64_t i = t / b, c = t % b;
    const double v = M[i * w + k0 + c];
    Pold[t] = v;
    Pw[t] = v;
  }
}

// pick the pivot of panel column jj among the CTAs' candidates, scale and stage its row
__device__ void pan_pick(int n, int b, int jj, int k0, double* __restrict__ Pw, GjState S, int nparts) {
  __shared__ double rv[TB];
  __shared__ int ri[TB];
  __shared__ int s_p;
  __shared__ double s_inv;
  double bb = -1.0;
  int bp = n;
  for (int c = threadIdx.x; c < nparts; c += TB) {
    const double v = __ldcg(&S.pv[c]);
    const int ix = __ldcg(&S.pi[c]);
    if (v > bb || (v == bb && ix < bp)) {
      bb = v;
      bp = ix;
    }
  }
  rv[threadIdx.x] = bb;
  ri[threadIdx.x] = bp;
  __syncthreads();
  for (int s2 = TB / 2; s2 > 0; s2 >>= 1) {
    if (threadIdx.x < s2 &&
        (rv[threadIdx.x + s2] > rv[threadIdx.x] || (rv[threadIdx.x + s2] == rv[threadIdx.x] && ri[threadIdx.x + s2] < ri[threadIdx.x]))) {
      rv[threadIdx.x] = rv[threadIdx.x + s2];
      ri[threadIdx.x] = ri[threadIdx.x + s2];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bb = rv[0];
    bp = ri[0];
    if (!(bb > 0.0) || bp >= n) {
      *S.singular = 1;
      bp = -1;
    } else {
      S.prow_idx[k0 + jj] = bp;
      S.pivoted[bp] = 1;
      s_inv = 1.0 / __ldcg(&Pw[(int64_t)bp * b + jj]);
    }
    s_p = bp;
  }
  __syncthreads();
  const int p = s_p;
  if (p < 0) return;
  double* pr = S.prow + (int64_t)(jj & 1) * GB;
  for (int c = jj + threadIdx.x; c < b; c += TB) {
    const double v = __ldcg(&Pw[(int64_t)p * b + c]) * s_inv;
    Pw[(int64_t)p * b + c] = v;
    pr[c] = v;
  }
}

// candidates for panel column 0 (one CTA)
__global__ void k_pan_first(int n, int b, int k0, double* __restrict__ Pw, GjState S) {
  __shared__ double sv[TB];
  __shared__ int si[TB];
  double best = -1.0;
  int bi = n;
  for (int i = threadIdx.x; i < n; i += TB) {
    if (S.pivoted[i]) continue;
    const double a = fabs(Pw[(int64_t)i * b]);
    if (a > best) {
      best = a;
      bi = i;
    }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s2 = TB / 2; s2 > 0; s2 >>= 1) {
    if (threadIdx.x < s2 &&
        (sv[threadIdx.x + s2] > sv[threadIdx.x] || (sv[threadIdx.x + s2] == sv[threadIdx.x] && si[threadIdx.x + s2] < si[threadIdx.x]))) {
      sv[threadIdx.x] = sv[threadIdx.x + s2];
      si[threadIdx.x] = si[threadIdx.x + s2];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    S.pv[0] = sv[0];
    S.pi[0] = si[0];
  }
  __threadfence_block();
  __syncthreads();
  pan_pick(n, b, 0, k0, Pw, S, 1);
}

// step jj of the panel: eliminate panel column jj from every row but its pivot row (panel
// columns > jj only), propose candidates for column jj+1, the last CTA picks
__global__ void __launch_bounds__(TB) k_pan_step(int n, int b, int jj, int k0, double* __restrict__ Pw, GjState S) {
  __shared__ bool s_last;
  if (*(volatile int*)S.singular) return;
  const int p = S.prow_idx[k0 + jj];
  const double* pr = S.prow + (int64_t)(jj & 1) * GB;
  const bool next = jj + 1 < b;
  // one warp per row, lanes over the panel columns
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double best = -1.0;
  int bi = n;
  for (int i = blockIdx.x * (TB / 32) + wid; i < n; i += gridDim.x * (TB / 32)) {
    double* Pi = Pw + (int64_t)i * b;
    if (i != p) {
      const double f = Pi[jj];
      if (f != 0.0)
        for (int c = jj + 1 + lane; c < b; c += 32) Pi[c] -= f * pr[c];
    }
    __syncwarp();
    if (lane == 0 && next && !S.pivoted[i]) {
      const double a = fabs(Pi[jj + 1]);
      if (a > best) {
        best = a;
        bi = i;
      }
    }
  }
  if (!next) return;
  __shared__ double wv[TB / 32];
  __shared__ int wi[TB / 32];
  if (lane == 0) {
    wv[wid] = best;
    wi[wid] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < TB / 32; ++q)
      if (wv[q] > best || (wv[q] == best && wi[q] < bi)) {
        best = wv[q];
        bi = wi[q];
      }
    S.pv[blockIdx.x] = best;
    S.pi[blockIdx.x] = bi;
    __threadfence();
    s_last = atomicAdd(S.count, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  pan_pick(n, b, jj + 1, k0, Pw, S, gridDim.x);
  if (threadIdx.x == 0) *S.count = 0u;
}

// Binv = (Pold[P, :])^{-1} with partial pivoting (one CTA, b <= GB); pos[P_l] = l
__global__ void k_pan_binv(int b, int k0, const double* __restrict__ Pold, const int* __restrict__ prow_idx,
                           double* __restrict__ Binv, int* __restrict__ pos, int* __restrict__ singular) {
  __shared__ double A[GB][2 * GB + 1];
  __shared__ int s_piv;
  for (int t = threadIdx.x; t < b * 2 * b; t += blockDim.x) {
    const int r = t / (2 * b), c = t % (2 * b);
    A[r][c] = (c < b) ? Pold[(int64_t)prow_idx[k0 + r] * b + c] : (c - b == r ? 1.0 : 0.0);
  }
  if (threadIdx.x < b) pos[prow_idx[k0 + threadIdx.x]] = threadIdx.x;
  __syncthreads();
  for (int k = 0; k < b; ++k) {
    if (threadIdx.x == 0) {
      int p = k;
      for (int r = k + 1; r < b; ++r)
        if (fabs(A[r][k]) > fabs(A[p][k])) p = r;
      if (A[p][k] == 0.0) *singular = 1;
      s_piv = p;
    }
    __syncthreads();
    const int p = s_piv;
    if (p != k)
      for (int c = threadIdx.x; c < 2 * b; c += blockDim.x) {
        const double t = A[k][c];
        A[k][c] = A[p][c];
        A[p][c] = t;
      }
    __syncthreads();
    const double inv = 1.0 / A[k][k];
    __syncthreads();
    for (int c = threadIdx.x; c < 2 * b; c += blockDim.x) A[k][c] *= inv;
    __syncthreads();
    for (int t = threadIdx.x; t < b * 2 * b; t += blockDim.x) {
      const int r = t / (2 * b), c = t % (2 * b);
      if (r != k && c != k) A[r][c] -= A[r][k] * A[k][c];
    }
    __syncthreads();
    for (int r = threadIdx.x; r < b; r += blockDim.x)
      if (r != k) A[r][k] = 0.0;
    __syncthreads();
  }
  for (int t = threadIdx.x; t < b * b; t += blockDim.x) Binv[t] = A[t / b][b + t % b];
}

// W[l, c - c0] = sum_m Binv[l, m] M[P_m, c], c in [c0, 2n)
__global__ void k_pan_W(int n, int b, int k0, const double* __restrict__ M, const int* __restrict__ prow_idx,
                        const double* __restrict__ Binv, double* __restrict__ W) {
  __shared__ double Bs[GB * GB];
  __shared__ int Ps[GB];
  for (int t = threadIdx.x; t < b * b; t += TB) Bs[t] = Binv[t];
  if (threadIdx.x < b) Ps[threadIdx.x] = prow_idx[k0 + threadIdx.x];
  __syncthreads();
  const int64_t w = 2 * (int64_t)n;
  const int64_t c0 = k0 + b, R = w - c0;
  for (int64_t c = blockIdx.x * (int64_t)TB + threadIdx.x; c < R; c += (int64_t)gridDim.x * TB) {
    double m[GB];
#pragma unroll
    for (int l = 0; l < GB; ++l) m[l] = (l < b) ? M[(int64_t)Ps[l] * w + c0 + c] : 0.0;
    for (int l = 0; l < b; ++l) {
      double a = 0.0;
#pragma unroll
      for (int q = 0; q < GB; ++q) a += Bs[l * b + (q < b ? q : 0)] * (q < b ? m[q] : 0.0);
      W[(int64_t)l * R + c] = a;
    }
  }
}

// the rank-b block update of rows [blockIdx.y * PR, ...) over the columns c >= k0+b
constexpr int PR = 64;
__global__ void __launch_bounds__(TB) k_pan_update(int n, int b, int k0, double* __restrict__ M,
                                                   const double* __restrict__ Pold, const double* __restrict__ W,
                                                   const int* __restrict__ pos) {
  __shared__ double Ps[PR][GB];
  __shared__ int ps[PR];
  const int r0 = blockIdx.y * PR;
  for (int t = threadIdx.x; t < PR * GB; t += TB) {
    const int r = t / GB, l = t % GB;
    Ps[r][l] = (r0 + r < n && l < b) ? Pold[(int64_t)(r0 + r) * b + l] : 0.0;
  }
  for (int r = threadIdx.x; r < PR; r += TB) ps[r] = (r0 + r < n) ? pos[r0 + r] : -1;
  __syncthreads();
  const int64_t w = 2 * (int64_t)n;
  const int64_t c0 = k0 + b, R = w - c0;
  const int rows = min(PR, n - r0);
  for (int64_t c = blockIdx.x * (int64_t)TB + threadIdx.x; c < R; c += (int64_t)gridDim.x * TB) {
    double wc[GB];
#pragma unroll
    for (int l = 0; l < GB; ++l) wc[l] = (l < b) ? W[(int64_t)l * R + c] : 0.0;
    for (int r = 0; r < rows; ++r) {
      double* m = M + (int64_t)(r0 + r) * w + c0 + c;
      if (ps[r] >= 0) {
        *m = W[(int64_t)ps[r] * R + c];  // a pivot row of this panel: the scaled block row
      } else {
        double a = *m;
#pragma unroll
        for (int l = 0; l < GB; ++l) a -= Ps[r][l] * wc[l];
        *m = a;
      }
    }
  }
}

__global__ void k_pan_clear_pos(int b, int k0, const int* __restrict__ prow_idx, int* __restrict__ pos) {
  if (threadIdx.x < b) pos[prow_idx[k0 + threadIdx.x]] = -1;
}

// A^{-1}[k][:] = R[prow_idx[k]][:] (implicit pivoting), symmetrised
__global__ void k_gj_extract_perm(int n, const double* __restrict__ M, const int* __restrict__ prow_idx,
                                  double* __restrict__ G) {
  const int64_t w = 2 * (int64_t)n;
  for (int64_t t = blockIdx.x * (int64_t)TB + threadIdx.x; t < (int64_t)n * n; t += (int64_t)gridDim.x * TB) {
    const int64_t i = t / n, j = t % n;
    G[t] = 0.5 * (M[(int64_t)prow_idx[i] * w + n + j] + M[(int64_t)prow_idx[j] * w + n + i]);
  }
}

__global__ void k_gj_extract(int n, const double* __restrict__ M, double* __restrict__ G) {
  const int64_t w = 2 * (int64_t)n;
  for (int64_t t = blockIdx.x * (int64_t)TB + threadIdx.x; t < (int64_t)n * n; t += (int64_t)gridDim.x * TB) {
    const int64_t i = t / n, j = t % n;
    G[t] = 0.5 * (M[i * w + n + j] + M[j * w + n + i]);
  }
}

// ----------------------------------------------------------------------------
// application kernels: G threads per row (G | 32), coalesced row segments,
// shuffle reduction inside the group.  One row per group, no grid-stride
// loop so every lane of a warp reaches the shuffles.
// Programmatic dependent launch (PDL): every apply kernel lets its successor
// launch immediately (griddepcontrol.launch_dependents) and loads everything that
// does not depend on its predecessor -- row bounds, indices, factor values -- before
// griddepcontrol.wait; only the gathers of the predecessor's output come after it.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#ifdef AJ_NO_PDL_WAIT  // timing diagnostic only (results are garbage): the levels overlap freely
__device__ __forceinline__ void pdl_wait() {}
#else
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif

#ifndef AJ_PREF
#define AJ_PREF 8
#endif
constexpr int PREF = AJ_PREF;  // factor entries per lane prefetched before the dependency wait

// factor entries are read once per apply: streaming (evict-first) loads, so the stream does not
// push the gather vectors (rF, zn: re-read by many rows) out of L1 / L2
#ifdef AJ_NO_STREAM_LD
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) { return *p; }
#else
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) { return __ldcs(p); }
#endif

// sum_q val[e_q] * src[col[e_q]] over e_q = b + q*G < e1, q < PREF: all index/value loads
// issued before the gathers (memory-level parallelism instead of a dependent chain per entry);
// the order of the additions is q = 0, 1, ... like the prefetched first batch
template <int G, typename TV>
__device__ __forceinline__ double gather_batch(int64_t b, int64_t e1, const int32_t* __restrict__ col,
                                               const TV* __restrict__ val, const double* __restrict__ src) {
  int32_t c[PREF];
  double v[PREF];
#pragma unroll
  for (int q = 0; q < PREF; ++q) {
    const int64_t e = b + (int64_t)q * G;
    c[q] = (e < e1) ? ld_stream(&col[e]) : -1;
    v[q] = (e < e1) ? (double)ld_stream(&val[e]) : 0.0;
  }
  double acc = 0.0;
#pragma unroll
  for (int q = 0; q < PREF; ++q)
    if (c[q] >= 0) acc += v[q] * __ldg(&src[c[q]]);
  return acc;
}

template <int G, typename TV>
__global__ void __launch_bounds__(TB)
    k_apply_fwd(int nC, const int32_t* __restrict__ cidx, const double* __restrict__ D,
                const double* __restrict__ r, const double* __restrict__ gsrc, const int64_t* __restrict__ Lptr,
                const int32_t* __restrict__ Lcol, const TV* __restrict__ Lval, double* __restrict__ rn,
                double* __restrict__ rFn, const int32_t* __restrict__ fmapn) {
  // gsrc: the vector Lcol indexes -- r itself (level 0) or its compact pivot part rF
  // (levels >= 1); rFn/fmapn: the next level's compact pivot part is written too
  pdl_launch_dependents();
  const int gid = blockIdx.x * TB + threadIdx.x;
  const int cp = gid / G, lane = gid % G;
  const bool act = cp < nC;
  int64_t e0 = 0, e1 = 0;
  int c = 0, fn = -1;
  double Dc = 0.0;
  int32_t pc[PREF];
  double pv[PREF];
  if (act) {
    e0 = Lptr[cp] + lane;
    e1 = Lptr[cp + 1];
    c = cidx[cp];
    Dc = D[c];
    if (rFn && lane == 0) fn = fmapn[cp];
#pragma unroll
    for (int q = 0; q < PREF; ++q) {
      const int64_t e = e0 + (int64_t)q * G;
      pc[q] = (e < e1) ? ld_stream(&Lcol[e]) : -1;
      pv[q] = (e < e1) ? (double)ld_stream(&Lval[e]) : 0.0;
    }
  }
  pdl_wait();
  double acc = 0.0;
  if (act) {
#pragma unroll
    for (int q = 0; q < PREF; ++q)
      if (pc[q] >= 0) acc += pv[q] * __ldg(&gsrc[pc[q]]);
    // rows longer than PREF*G: the same batching (PREF independent index/value loads,
    // then PREF independent gathers), two dependent round trips per batch
    for (int64_t b = e0 + (int64_t)PREF * G; b < e1; b += (int64_t)PREF * G) acc += gather_batch<G>(b, e1, Lcol, Lval, gsrc);
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (act && lane == 0) {
    const double v = Dc * r[c] - acc;
    rn[cp] = v;
    if (fn >= 0) rFn[fn] = v;
  }
}

// backward substitution: blocks [0, bF) take the pivot (F) rows with G lanes
// each, blocks [bF, ...) copy the coarse solution back (z_c = D_c zn_c').
template <int G, typename TV>
__global__ void __launch_bounds__(TB)
    k_apply_bwd(int nF, int nC, int bF, const int32_t* __restrict__ fidx, const int32_t* __restrict__ cidx,
                const double* __restrict__ D, const double* __restrict__ r, const int32_t* __restrict__ partner,
                const double* __restrict__ b11, const double* __restrict__ b12, const int64_t* __restrict__ LTptr,
                const int32_t* __restrict__ LTcol, const TV* __restrict__ LTval, const double* __restrict__ zn,
                double* __restrict__ z, const int64_t* __restrict__ Vptr, const int32_t* __restrict__ Vcol,
                const double* __restrict__ Vval, const double* __restrict__ rF) {
  pdl_launch_dependents();
  if ((int)blockIdx.x >= bF) {
    const int cp = (blockIdx.x - bF) * TB + threadIdx.x;
    int i = 0;
    double Di = 0.0;
    if (cp < nC) {
      i = cidx[cp];
      Di = D[i];
    }
    pdl_wait();
    if (cp < nC) z[i] = Di * zn[cp];
    return;
  }
  const int gid = blockIdx.x * TB + threadIdx.x;
  const int fp = gid / G, lane = gid % G;
  const bool act = fp < nF;
  int64_t e0 = 0, e1 = 0;
  int i = 0, p = -1;
  double Di = 0.0, Dp = 0.0, B1 = 0.0, B2 = 0.0;
  int32_t pc[PREF];
  double pv[PREF];
  if (act) {
    e0 = LTptr[fp] + lane;
    e1 = LTptr[fp + 1];
#pragma unroll
    for (int q = 0; q < PREF; ++q) {
      const int64_t e = e0 + (int64_t)q * G;
      pc[q] = (e < e1) ? ld_stream(&LTcol[e]) : -1;
      pv[q] = (e < e1) ? (double)ld_stream(&LTval[e]) : 0.0;
    }
    if (lane == 0) {
      i = fidx[fp];
      Di = D[i];
      B1 = b11[i];
      p = partner[i];
      if (p >= 0) {
        Dp = D[p];
        B2 = b12[i];
      }
    }
  }
  int iv = 0;
  if (act && Vptr) iv = fidx[fp];
  pdl_wait();
  double acc = 0.0;
  if (act) {
#pragma unroll
    for (int q = 0; q < PREF; ++q)
      if (pc[q] >= 0) acc += pv[q] * __ldg(&zn[pc[q]]);
    for (int64_t b = e0 + (int64_t)PREF * G; b < e1; b += (int64_t)PREF * G) acc += gather_batch<G>(b, e1, LTcol, LTval, zn);
    if (Vptr)  // virtual couplings: -(B~^{-1} - B_d^{-1}) r^_F  (reading R17)
      for (int64_t e = Vptr[iv] + lane; e < Vptr[iv + 1]; e += G) {
        const int32_t v = Vcol[e];
        acc -= Vval[e] * (D[v] * r[v]);
      }
  }
#pragma unroll
  for (int o = (G < 32 ? G : 32) / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if constexpr (G > 32) {  // long rows (deep levels): G / 32 warps per row, fixed-order sum
    __shared__ double part[TB / 32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (lane == 0) {
      acc = 0.0;
#pragma unroll
      for (int k = 0; k < G / 32; ++k) acc += part[(threadIdx.x >> 5) + k];
    }
  }
  if (act && lane == 0) {
    double y = B1 * (Di * (rF ? rF[fp] : r[i]));  // rF: the level's input on its pivots, contiguous
    if (p >= 0) y += B2 * (Dp * r[p]);
    z[i] = Di * (y - acc);
  }
}

// ---- staged apply (DESIGN.md sect. 4) -------------------------------------------------
// The rows a CTA owns are consecutive, so their factor entries are ONE contiguous stream
// [ptr[row0], ptr[row1]) of indices and values.  One thread streams it into shared memory
// with 1-D bulk copies (cp.async.bulk, completion on an mbarrier) -- issued before
// griddepcontrol.wait, so they overlap the previous level's tail -- in chunks of SCAP
// entries through a ring of `nst` stages; the threads hold no prefetch registers and only
// issue the gathers of the predecessor's output (PREF per batch).  The bulk copies cover
// the 4-entry-aligned hull of the range (16-byte granules) and never read past the last
// full granule of the array; the few entries beyond it come from global memory.
constexpr int SCAP = 1920;  // entries per stage: 7.5 KB indices + 15 KB fp64 values (2 stages < 48 KB)

template <typename TV>
struct StageBuf {
  int32_t col[SCAP];
  TV val[SCAP];
};

template <typename TV>
__device__ __forceinline__ void stage_issue(StageBuf<TV>* sb, const int32_t* col, const TV* val, int64_t cs,
                                            int64_t ce, uint64_t* bar) {
  const uint32_t n = (uint32_t)(ce - cs);
  mbar_expect_tx(bar, n * (uint32_t)(4 + sizeof(TV)));
  bulk_g2s(sb->col, col + cs, n * 4u, bar);
  bulk_g2s(sb->val, val + cs, n * (uint32_t)sizeof(TV), bar);
}

// sum over this lane's entries e = e0 + lane + m G inside [lo, hi) of val[e] src[col[e]],
// read from the stage holding entries [cs, cs + SCAP), in batches of PREF gathers
template <int G, typename TV>
__device__ __forceinline__ double stage_gather(int64_t e0, int lane, int64_t lo, int64_t hi, const StageBuf<TV>* b,
                                               int64_t cs, const double* __restrict__ src) {
  int64_t e = e0 + lane;
  if (e < lo) e += ((lo - e + G - 1) / G) * G;
  double acc = 0.0;
  for (; e < hi; e += (int64_t)PREF * G) {
    int32_t c[PREF];
    double v[PREF];
#pragma unroll
    for (int q = 0; q < PREF; ++q) {
      const int64_t ee = e + (int64_t)q * G;
      c[q] = (ee < hi) ? b->col[ee - cs] : -1;
      v[q] = (ee < hi) ? (double)b->val[ee - cs] : 0.0;
    }
    double part = 0.0;
#pragma unroll
    for (int q = 0; q < PREF; ++q)
      if (c[q] >= 0) part += v[q] * __ldg(&src[c[q]]);
    acc += part;
  }
  return acc;
}

// The CTA-wide part shared by both substitutions: stream [E0, E1) through the stages and
// return this lane's partial sum of its row [e0, e1) (act: the thread has a row).
// Call with the first min(nch, nst) chunks already issued (issue_first) before pdl_wait.
template <typename TV>
struct StagePlan {
  int64_t SB, SE;
  int nch;
};
template <typename TV>
__device__ __forceinline__ StagePlan<TV> stage_plan(int64_t E0, int64_t E1, int64_t nnz) {
  StagePlan<TV> p;
  p.SB = E0 & ~int64_t(3);
  const int64_t top = nnz & ~int64_t(3);
  p.SE = min((E1 + 3) & ~int64_t(3), top);
  p.nch = p.SE > p.SB ? (int)((p.SE - p.SB + SCAP - 1) / SCAP) : 0;
  return p;
}
template <typename TV>
__device__ __forceinline__ void stage_issue_first(const StagePlan<TV>& p, StageBuf<TV>* sb, uint64_t* bar, int nst,
                                                  const int32_t* col, const TV* val) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int c = 0; c < min(p.nch, nst); ++c)
      stage_issue(sb + c, col, val, p.SB + (int64_t)c * SCAP, min(p.SE, p.SB + (int64_t)(c + 1) * SCAP), &bar[c]);
  }
  __syncthreads();
}
template <int G, typename TV>
__device__ __forceinline__ double stage_consume(const StagePlan<TV>& p, StageBuf<TV>* sb, uint64_t* bar, int nst,
                                                const int32_t* __restrict__ col, const TV* __restrict__ val,
                                                bool act, int64_t e0, int64_t e1, int lane,
                                                const double* __restrict__ src) {
  double acc = 0.0;
  for (int ch = 0; ch < p.nch; ++ch) {
    const int s = ch % nst;
    const int64_t cs = p.SB + (int64_t)ch * SCAP, ce = min(p.SE, cs + SCAP);
    mbar_wait(&bar[s], (uint32_t)((ch / nst) & 1));
    if (act) acc += stage_gather<G, TV>(e0, lane, max(e0, cs), min(e1, ce), sb + s, cs, src);
    if (ch + nst < p.nch) {
      __syncthreads();  // every thread is done with stage s
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        stage_issue(sb + s, col, val, p.SB + (int64_t)(ch + nst) * SCAP,
                    min(p.SE, p.SB + (int64_t)(ch + nst + 1) * SCAP), &bar[s]);
      }
    }
  }
  // entries past the last full 16-byte granule of the array (only the last CTA has them)
  if (act && e1 > p.SE) {
    int64_t e = e0 + lane;
    if (e < p.SE) e += ((p.SE - e + G - 1) / G) * G;
    for (; e < e1; e += G) acc += (double)val[e] * __ldg(&src[col[e]]);
  }
  return acc;
}

template <int G, typename TV>
__global__ void __launch_bounds__(TB, 6)
    k_apply_fwd_s(int nC, int nst, int64_t nnz, const int32_t* __restrict__ cidx, const double* __restrict__ D,
                  const double* __restrict__ r, const double* __restrict__ gsrc, const int64_t* __restrict__ Lptr,
                  const int32_t* __restrict__ Lcol, const TV* __restrict__ Lval, double* __restrict__ rn,
                  double* __restrict__ rFn, const int32_t* __restrict__ fmapn) {
  extern __shared__ __align__(128) unsigned char smraw[];
  StageBuf<TV>* sb = reinterpret_cast<StageBuf<TV>*>(smraw);
  __shared__ __align__(8) uint64_t bar[2];
  pdl_launch_dependents();
  constexpr int R = TB / G;
  const int row0 = blockIdx.x * R, row1 = min(nC, row0 + R);
  const int cp = row0 + threadIdx.x / G, lane = threadIdx.x % G;
  const bool act = cp < nC;
  const StagePlan<TV> pl = stage_plan<TV>(Lptr[row0], Lptr[row1], nnz);
  stage_issue_first(pl, sb, bar, nst, Lcol, Lval);
  int64_t e0 = 0, e1 = 0;
  int c = 0, fn = -1;
  double Dc = 0.0;
  if (act) {
    e0 = Lptr[cp];
    e1 = Lptr[cp + 1];
    c = cidx[cp];
    Dc = D[c];
    if (rFn && lane == 0) fn = fmapn[cp];
  }
  pdl_wait();
  double acc = stage_consume<G, TV>(pl, sb, bar, nst, Lcol, Lval, act, e0, e1, lane, gsrc);
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (act && lane == 0) {
    const double v = Dc * r[c] - acc;
    rn[cp] = v;
    if (fn >= 0) rFn[fn] = v;
  }
}

template <int G, typename TV>
__global__ void __launch_bounds__(TB, 6)
    k_apply_bwd_s(int nF, int nC, int bF, int nst, int64_t nnz, const int32_t* __restrict__ fidx,
                  const int32_t* __restrict__ cidx, const double* __restrict__ D, const double* __restrict__ r,
                  const int32_t* __restrict__ partner, const double* __restrict__ b11, const double* __restrict__ b12,
                  const int64_t* __restrict__ LTptr, const int32_t* __restrict__ LTcol, const TV* __restrict__ LTval,
                  const double* __restrict__ zn, double* __restrict__ z, const int64_t* __restrict__ Vptr,
                  const int32_t* __restrict__ Vcol, const double* __restrict__ Vval, const double* __restrict__ rF) {
  extern __shared__ __align__(128) unsigned char smraw[];
  StageBuf<TV>* sb = reinterpret_cast<StageBuf<TV>*>(smraw);
  __shared__ __align__(8) uint64_t bar[2];
  pdl_launch_dependents();
  if ((int)blockIdx.x >= bF) {  // coarse part: z_c = D_c zn_c'
    const int cp = (blockIdx.x - bF) * TB + threadIdx.x;
    int i = 0;
    double Di = 0.0;
    if (cp < nC) {
      i = cidx[cp];
      Di = D[i];
    }
    pdl_wait();
    if (cp < nC) z[i] = Di * zn[cp];
    return;
  }
  constexpr int R = (TB / G) > 0 ? TB / G : 1;
  const int row0 = blockIdx.x * R, row1 = min(nF, row0 + R);
  const int fp = row0 + threadIdx.x / G, lane = threadIdx.x % G;
  const bool act = fp < nF;
  const StagePlan<TV> pl = stage_plan<TV>(LTptr[row0], LTptr[row1], nnz);
  stage_issue_first(pl, sb, bar, nst, LTcol, LTval);
  int64_t e0 = 0, e1 = 0;
  int i = 0, p = -1, iv = 0;
  double Di = 0.0, Dp = 0.0, B1 = 0.0, B2 = 0.0;
  if (act) {
    e0 = LTptr[fp];
    e1 = LTptr[fp + 1];
    if (Vptr) iv = fidx[fp];
    if (lane == 0) {
      i = fidx[fp];
      Di = D[i];
      B1 = b11[i];
      p = partner[i];
      if (p >= 0) {
        Dp = D[p];
        B2 = b12[i];
      }
    }
  }
  pdl_wait();
  double acc = stage_consume<G, TV>(pl, sb, bar, nst, LTcol, LTval, act, e0, e1, lane, zn);
  if (act && Vptr)  // virtual couplings: -(B~^{-1} - B_d^{-1}) r^_F  (reading R17)
    for (int64_t e = Vptr[iv] + lane; e < Vptr[iv + 1]; e += G) {
      const int32_t v = Vcol[e];
      acc -= Vval[e] * (D[v] * r[v]);
    }
#pragma unroll
  for (int o = (G < 32 ? G : 32) / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if constexpr (G > 32) {  // long rows (deep levels): G / 32 warps per row, fixed-order sum
    __shared__ double part[TB / 32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (lane == 0) {
      acc = 0.0;
#pragma unroll
      for (int k = 0; k < G / 32; ++k) acc += part[(threadIdx.x >> 5) + k];
    }
  }
  if (act && lane == 0) {
    double y = B1 * (Di * (rF ? rF[fp] : r[i]));
    if (p >= 0) y += B2 * (Dp * r[p]);
    z[i] = Di * (y - acc);
  }
}

// ---- persistent ring apply (DESIGN.md sect. 4; opt-in, AJ_APPLY_RING=1) ------------------
// Large levels: one CTA per SM owns a run of consecutive rows holding ~1/grid of the level's
// factor entries (row partition `part`, balanced by entries at setup).  A producer warp streams
// the CTA's contiguous (index, value) range through a ring of RNST shared-memory stages with 1-D
// bulk copies (full/empty mbarrier pair per stage); RNW consumer warps walk the rows in tiles of
// RNW * 32 / G rows, each warp at its own pace: it waits for the stages holding its rows'
// entries, gathers the predecessor's output (PREF independent gathers per batch), reduces over
// the G lanes of a row and writes.  Every warp passes every stage in order (wait full, then
// arrive empty), so a stage is refilled only when all warps are past it.  The factor stream
// never waits behind a row pointer or a gather, and the first RNST stages are issued before
// griddepcontrol.wait.  Row metadata is loaded one tile ahead.
// Measured (profiles/round2_s5_apply_experiments.txt, L=150): 16 warps + 4 x 2048-entry stages
// at one CTA per SM (so that the next level's CTAs are co-resident) 4.61 ms; 2 CTAs per SM with
// 8 x 1024 3.76 ms; 28 warps + 16 x 1024 (192 KB, the defaults below) 3.63 ms -- against 3.67 ms
// of the register-prefetch kernels: the consumers' gather latency, not the factor stream, is the
// bound, so the ring buys nothing and stays opt-in.
#ifndef AJ_RCAP
#define AJ_RCAP 1024
#define AJ_RNST 16
#define AJ_RNW 28
#define AJ_RING_CTAS 1
#endif
#ifndef AJ_RING_MINB
#define AJ_RING_MINB 1
#endif
constexpr int RCAP = AJ_RCAP;  // entries per stage: 4 KB indices + 8 KB fp64 values
constexpr int RNST = AJ_RNST;  // stages (192 KB)
constexpr int RNW = AJ_RNW;    // consumer warps
constexpr int RING_CTAS = AJ_RING_CTAS;  // ring CTAs per SM
constexpr int RTB = RNW * 32 + 32;  // + the producer warp

template <typename TV>
struct RingBuf {
  int32_t col[RCAP];
  TV val[RCAP];
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

struct RingPlan {
  int64_t SB, SE;  // 4-entry-aligned hull of the CTA's entry range that the ring covers
  int nch;
};
__device__ __forceinline__ RingPlan ring_plan(int64_t E0, int64_t E1, int64_t nnz) {
  RingPlan p;
  p.SB = E0 & ~int64_t(3);
  p.SE = min((E1 + 3) & ~int64_t(3), nnz & ~int64_t(3));  // never past the last full 16-byte granule
  p.nch = p.SE > p.SB ? (int)((p.SE - p.SB + RCAP - 1) / RCAP) : 0;
  return p;
}

// producer (one lane): all chunks of the CTA's range in order, a stage refilled once every
// consumer warp has arrived on its empty barrier
template <typename TV>
__device__ __forceinline__ void ring_produce(const RingPlan& p, RingBuf<TV>* sb, uint64_t* full, uint64_t* empty,
                                             const int32_t* col, const TV* val) {
  for (int ch = 0; ch < p.nch; ++ch) {
    const int s = ch % RNST;
    if (ch >= RNST) {
      mbar_wait(&empty[s], (uint32_t)(((ch / RNST) - 1) & 1));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    const int64_t cs = p.SB + (int64_t)ch * RCAP, ce = min(p.SE, cs + RCAP);
    const uint32_t n = (uint32_t)(ce - cs);
    mbar_expect_tx(&full[s], n * (uint32_t)(4 + sizeof(TV)));
    bulk_g2s(sb[s].col, col + cs, n * 4u, &full[s]);
    bulk_g2s(sb[s].val, val + cs, n * (uint32_t)sizeof(TV), &full[s]);
  }
}

// consumer-side state of one warp: `cur` = first chunk it has not released yet
struct RingWarp {
  int cur = 0;
};
template <typename TV>
__device__ __forceinline__ void ring_skip_to(RingWarp& w, int ch, uint64_t* full, uint64_t* empty) {
  for (; w.cur < ch; ++w.cur) {
    mbar_wait(&full[w.cur % RNST], (uint32_t)((w.cur / RNST) & 1));
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[w.cur % RNST]);
  }
}

// this lane's partial sum over its row's entries e = e0 + lane + m G in [e0, e1), read from the
// ring; [w0, w1) is the warp's entry range of the tile (warp-uniform).  Entries >= SE (past the
// last full granule of the array) come from global memory.
template <int G, typename TV>
__device__ __forceinline__ double ring_row_sum(RingWarp& w, const RingPlan& p, RingBuf<TV>* sb, uint64_t* full,
                                               uint64_t* empty, int64_t w0, int64_t w1, bool act, int64_t e0,
                                               int64_t e1, int lane, const int32_t* __restrict__ col,
                                               const TV* __restrict__ val, const double* __restrict__ src) {
  double acc = 0.0;
  const int64_t wh = min(w1, p.SE);
  if (wh > w0) {
    const int chA = (int)((w0 - p.SB) / RCAP), chB = (int)((wh - 1 - p.SB) / RCAP);
    ring_skip_to<TV>(w, chA, full, empty);
    for (int ch = chA; ch <= chB; ++ch) {
      const int s = ch % RNST;
      const int64_t cs = p.SB + (int64_t)ch * RCAP, ce = min(p.SE, cs + RCAP);
      mbar_wait(&full[s], (uint32_t)((ch / RNST) & 1));
      if (act) {
        const int64_t lo = max(e0, cs), hi = min(e1, ce);
        int64_t e = e0 + lane;
        if (e < lo) e += ((lo - e + G - 1) / G) * G;
        const RingBuf<TV>* b = sb + s;
        for (; e < hi; e += (int64_t)PREF * G) {
          int32_t c[PREF];
          double v[PREF];
#pragma unroll
          for (int q = 0; q < PREF; ++q) {
            const int64_t ee = e + (int64_t)q * G;
            c[q] = (ee < hi) ? b->col[ee - cs] : -1;
            v[q] = (ee < hi) ? (double)b->val[ee - cs] : 0.0;
          }
          double part = 0.0;
#pragma unroll
          for (int q = 0; q < PREF; ++q)
            if (c[q] >= 0) part += v[q] * __ldg(&src[c[q]]);
          acc += part;
        }
      }
      if (ch < chB) {  // done with this stage; the last one stays held for the next tile
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
        w.cur = ch + 1;
      }
    }
  }
  if (act && e1 > p.SE) {
    int64_t e = e0 + lane;
    if (e < p.SE) e += ((p.SE - e + G - 1) / G) * G;
    for (; e < e1; e += G) acc += (double)val[e] * __ldg(&src[col[e]]);
  }
  return acc;
}

// The backward ring kernel's per-row right-hand side, computed by extra CTAs of the level's
// FORWARD kernel (it needs only the level's input r): yv_f = B~^{-1}-row of D r on the pivot block
// (1x1 / 2x2 part plus the virtual couplings, reading R17), dF_f = D_f.  The backward epilogue is
// then z_f = dF_f (yv_f - sum), with every operand indexed by the pivot row (coalesced, loaded a
// tile ahead) instead of three dependent gathers per row.
struct PrepArgs {
  int nF, nparts;
  const int32_t* fidx;
  const int32_t* partner;
  const double *b11, *b12;
  const int64_t* Vptr;
  const int32_t* Vcol;
  const double* Vval;
  const double* rF;
  double *yv, *dF;
};
__device__ __forceinline__ void bwd_prep_rows(const PrepArgs& a, const double* __restrict__ D,
                                              const double* __restrict__ r, int first, int stride) {
  for (int fp = first; fp < a.nF; fp += stride) {
    const int i = a.fidx[fp];
    const double Di = D[i];
    double y = a.b11[i] * (Di * (a.rF ? a.rF[fp] : r[i]));
    const int p = a.partner[i];
    if (p >= 0) y += a.b12[i] * (D[p] * r[p]);
    if (a.Vptr)
      for (int64_t e = a.Vptr[i]; e < a.Vptr[i + 1]; ++e) {
        const int32_t v = a.Vcol[e];
        y += a.Vval[e] * (D[v] * r[v]);
      }
    a.yv[fp] = y;
    a.dF[fp] = Di;
  }
}

template <int G, typename TV>
__global__ void __launch_bounds__(RTB, AJ_RING_MINB)
    k_apply_fwd_r(int64_t nnz, const int32_t* __restrict__ part, const int32_t* __restrict__ cidx,
                  const double* __restrict__ D, const double* __restrict__ r, const double* __restrict__ gsrc,
                  const int64_t* __restrict__ Lptr, const int32_t* __restrict__ Lcol, const TV* __restrict__ Lval,
                  double* __restrict__ rn, double* __restrict__ rFn, const int32_t* __restrict__ fmapn,
                  PrepArgs prep) {
  extern __shared__ __align__(128) unsigned char smraw[];
  RingBuf<TV>* sb = reinterpret_cast<RingBuf<TV>*>(smraw);
  __shared__ __align__(8) uint64_t full[RNST], empty[RNST];
  pdl_launch_dependents();
  if ((int)blockIdx.x >= prep.nparts) {  // prep CTAs
    pdl_wait();
    bwd_prep_rows(prep, D, r, ((int)blockIdx.x - prep.nparts) * RTB + (int)threadIdx.x,
                  ((int)gridDim.x - prep.nparts) * RTB);
    return;
  }
  const int row0 = part[blockIdx.x], row1 = part[blockIdx.x + 1];
  const RingPlan pl = ring_plan(Lptr[row0], Lptr[row1], nnz);
  const int warp = threadIdx.x >> 5, l32 = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < RNST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], RNW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == RNW) {
    if (l32 == 0) ring_produce<TV>(pl, sb, full, empty, Lcol, Lval);
    return;
  }
  constexpr int RW = 32 / G, RT = RNW * RW;
  const int sub = l32 / G, lane = l32 % G;
  int wr = row0 + warp * RW;  // the warp's first row of the tile
  int cp = wr + sub;
  bool act = cp < row1;
  int64_t e0 = 0, e1 = 0;
  int c = 0, fn = -1;
  if (act) {
    e0 = Lptr[cp];
    e1 = Lptr[cp + 1];
    c = cidx[cp];
    if (rFn && lane == 0) fn = fmapn[cp];
  }
  pdl_wait();
  RingWarp w;
  for (; wr < row1; wr += RT) {
    // the next tile's row bounds and indices, one tile ahead
    const int cpn = cp + RT;
    const bool actn = cpn < row1;
    int64_t e0n = 0, e1n = 0;
    int cn = 0, fnn = -1;
    if (actn) {
      e0n = Lptr[cpn];
      e1n = Lptr[cpn + 1];
      cn = cidx[cpn];
      if (rFn && lane == 0) fnn = fmapn[cpn];
    }
    double Dc = 0.0, rc = 0.0;
    if (act && lane == 0) {
      Dc = D[c];
      rc = r[c];
    }
    const int last = (min(RW, row1 - wr) - 1) * G;  // a lane of the warp's last active row
    const int64_t w0 = __shfl_sync(0xffffffffu, e0, 0), w1 = __shfl_sync(0xffffffffu, e1, last);
    double acc = ring_row_sum<G, TV>(w, pl, sb, full, empty, w0, w1, act, e0, e1, lane, Lcol, Lval, gsrc);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (act && lane == 0) {
      const double v = Dc * rc - acc;
      rn[cp] = v;
      if (fn >= 0) rFn[fn] = v;
    }
    cp = cpn;
    act = actn;
    e0 = e0n;
    e1 = e1n;
    c = cn;
    fn = fnn;
  }
  ring_skip_to<TV>(w, pl.nch, full, empty);  // pass the remaining stages so the producer can finish
}

// backward: CTAs [0, nparts) take the pivot rows through the ring (source zn, the next level's
// solution), CTAs >= nparts copy the coarse solution back (z_c = D_c zn_c', RCPY nodes each)
constexpr int RCPY = 4;
template <int G, typename TV>
__global__ void __launch_bounds__(RTB, AJ_RING_MINB)
    k_apply_bwd_r(int nC, int nparts, int64_t nnz, const int32_t* __restrict__ part,
                  const int32_t* __restrict__ fidx, const int32_t* __restrict__ cidx, const double* __restrict__ D,
                  const double* __restrict__ yv, const double* __restrict__ dF, const int64_t* __restrict__ LTptr,
                  const int32_t* __restrict__ LTcol, const TV* __restrict__ LTval, const double* __restrict__ zn,
                  double* __restrict__ z) {
  extern __shared__ __align__(128) unsigned char smraw[];
  RingBuf<TV>* sb = reinterpret_cast<RingBuf<TV>*>(smraw);
  __shared__ __align__(8) uint64_t full[RNST], empty[RNST];
  pdl_launch_dependents();
  if ((int)blockIdx.x >= nparts) {  // coarse part
    const int base = ((int)blockIdx.x - nparts) * (RTB * RCPY) + (int)threadIdx.x;
    int i[RCPY];
    double Di[RCPY];
#pragma unroll
    for (int q = 0; q < RCPY; ++q) {
      const int cp = base + q * RTB;
      i[q] = cp < nC ? cidx[cp] : -1;
    }
#pragma unroll
    for (int q = 0; q < RCPY; ++q) Di[q] = i[q] >= 0 ? D[i[q]] : 0.0;
    pdl_wait();
#pragma unroll
    for (int q = 0; q < RCPY; ++q)
      if (i[q] >= 0) z[i[q]] = Di[q] * zn[base + q * RTB];
    return;
  }
  const int row0 = part[blockIdx.x], row1 = part[blockIdx.x + 1];
  const RingPlan pl = ring_plan(LTptr[row0], LTptr[row1], nnz);
  const int warp = threadIdx.x >> 5, l32 = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < RNST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], RNW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == RNW) {
    if (l32 == 0) ring_produce<TV>(pl, sb, full, empty, LTcol, LTval);
    return;
  }
  constexpr int RW = 32 / G, RT = RNW * RW;
  const int sub = l32 / G, lane = l32 % G;
  int wr = row0 + warp * RW;
  int fp = wr + sub;
  bool act = fp < row1;
  int64_t e0 = 0, e1 = 0;
  int i = 0;
  if (act) {
    e0 = LTptr[fp];
    e1 = LTptr[fp + 1];
    if (lane == 0) i = fidx[fp];
  }
  pdl_wait();
  RingWarp w;
  for (; wr < row1; wr += RT) {
    const int fpn = fp + RT;
    const bool actn = fpn < row1;
    int64_t e0n = 0, e1n = 0;
    int in = 0;
    if (actn) {
      e0n = LTptr[fpn];
      e1n = LTptr[fpn + 1];
      if (lane == 0) in = fidx[fpn];
    }
    double y = 0.0, Df = 0.0;
    if (act && lane == 0) {
      y = yv[fp];
      Df = dF[fp];
    }
    const int last = (min(RW, row1 - wr) - 1) * G;
    const int64_t w0 = __shfl_sync(0xffffffffu, e0, 0), w1 = __shfl_sync(0xffffffffu, e1, last);
    double acc = ring_row_sum<G, TV>(w, pl, sb, full, empty, w0, w1, act, e0, e1, lane, LTcol, LTval, zn);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (act && lane == 0) z[i] = Df * (y - acc);
    fp = fpn;
    act = actn;
    e0 = e0n;
    e1 = e1n;
    i = in;
  }
  ring_skip_to<TV>(w, pl.nch, full, empty);
}

// row partition of a CSR-like pointer array into nparts runs of ~equal entry counts
__global__ void k_row_partition(int nrows, const int64_t* __restrict__ ptr, int nparts, int32_t* __restrict__ part) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > nparts) return;
  if (b == nparts) {
    part[b] = nrows;
    return;
  }
  const int64_t nnz = ptr[nrows], target = (nnz / nparts) * b + min((int64_t)b, nnz % nparts);
  int lo = 0, hi = nrows;  // first row with ptr[row] >= target
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (ptr[mid] >= target) hi = mid; else lo = mid + 1;
  }
  part[b] = lo;
}

// G lanes per row such that each lane holds ~per_lane entries: 8 on large levels
// (streaming, more loads in flight per thread), 4 on small L2-resident ones (more
// threads); measured at L = 50..200 (DESIGN.md sect. 4)
static int pick_group(double avg_len, int64_t nnz, int gmax = 32) {
  const char* ev = getenv("AJ_PER_LANE");  // testing: read per setup so a test can force it
  const int per_lane = ev ? atoi(ev) : (nnz > (int64_t(1) << 22) ? 8 : 4);
  int g = 1;
  while (g < gmax && g * per_lane <= avg_len) g <<= 1;  // ~per_lane entries per lane (memory-level parallelism)
  return g;
}

template <typename K, typename... Args>
static void launch_pdl_block(K kernel, int grid, int block, size_t smem, cudaStream_t st, Args... args) {
  if (smem > 48 * 1024) AJ_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  AJ_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
  AJ_LAUNCHED();
}
template <typename K, typename... Args>
static void launch_pdl_smem(K kernel, int grid, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(TB);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  AJ_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
  AJ_LAUNCHED();
}
template <typename K, typename... Args>
static void launch_pdl(K kernel, int grid, cudaStream_t st, Args... args) {
  launch_pdl_smem(kernel, grid, 0, st, args...);
}

// stages of the staged kernels for a level (0: the register-prefetch kernels): one stage
// when the CTAs' streams mostly fit in SCAP entries, else two (chunk c+1 in flight while c is
// gathered).  Opt-in (AJ_APPLY_STAGED=1): measured slower than the register-prefetch kernels
// (apply L=150 3.23 vs 2.83 ms, L=200 8.27 vs 7.43 ms; DESIGN.md sect. 4).
static int pick_stages(int64_t nnz, int64_t rows, int g) {
  if (!getenv("AJ_APPLY_STAGED") || rows <= 0 || nnz <= 0) return 0;
  const double per_cta = (double)nnz / (double)ceil_div(rows, std::max(1, TB / g));
  return per_cta <= 0.75 * SCAP ? 1 : 2;
}

template <int G>
static void fwd_g(const Level& v, const double* r, const double* gsrc, double* rn, double* rFn,
                  const int32_t* fmapn, int grid, cudaStream_t st) {
  if (v.fpart) {  // persistent ring kernel, one CTA per partition run (+ the backward prep CTAs)
    PrepArgs pa{v.nF, v.nfpart, v.fidx, v.partner, v.b11, v.b12, v.Vptr, v.Vcol, v.Vval, v.rF, v.yv, v.dF};
    const int gridr = v.nfpart + (v.bpart ? std::max(1, std::min(num_sms(), ceil_div(v.nF, RTB))) : 0);
    if (v.f32)
      launch_pdl_block(k_apply_fwd_r<G, float>, gridr, RTB, RNST * sizeof(RingBuf<float>), st, v.nnzL,
                       (const int32_t*)v.fpart, (const int32_t*)v.cidx, (const double*)v.D, r, gsrc,
                       (const int64_t*)v.Lptr, (const int32_t*)v.Lcol, (const float*)v.Lval, rn, rFn, fmapn, pa);
    else
      launch_pdl_block(k_apply_fwd_r<G, double>, gridr, RTB, RNST * sizeof(RingBuf<double>), st, v.nnzL,
                       (const int32_t*)v.fpart, (const int32_t*)v.cidx, (const double*)v.D, r, gsrc,
                       (const int64_t*)v.Lptr, (const int32_t*)v.Lcol, (const double*)v.Lval, rn, rFn, fmapn, pa);
    return;
  }
  if (v.nst_f > 0) {
    if (v.f32)
      launch_pdl_smem(k_apply_fwd_s<G, float>, grid, v.nst_f * sizeof(StageBuf<float>), st, v.nC, v.nst_f, v.nnzL,
                      (const int32_t*)v.cidx, (const double*)v.D, r, gsrc, (const int64_t*)v.Lptr,
                      (const int32_t*)v.Lcol, (const float*)v.Lval, rn, rFn, fmapn);
    else
      launch_pdl_smem(k_apply_fwd_s<G, double>, grid, v.nst_f * sizeof(StageBuf<double>), st, v.nC, v.nst_f,
                      v.nnzL, (const int32_t*)v.cidx, (const double*)v.D, r, gsrc, (const int64_t*)v.Lptr,
                      (const int32_t*)v.Lcol, (const double*)v.Lval, rn, rFn, fmapn);
    return;
  }
  if (v.f32)
    launch_pdl(k_apply_fwd<G, float>, grid, st, v.nC, (const int32_t*)v.cidx, (const double*)v.D, r, gsrc,
               (const int64_t*)v.Lptr, (const int32_t*)v.Lcol, (const float*)v.Lval, rn, rFn, fmapn);
  else
    launch_pdl(k_apply_fwd<G, double>, grid, st, v.nC, (const int32_t*)v.cidx, (const double*)v.D, r, gsrc,
               (const int64_t*)v.Lptr, (const int32_t*)v.Lcol, (const double*)v.Lval, rn, rFn, fmapn);
}
template <int G>
static void bwd_g(const Level& v, const double* r, const double* zn, double* z, int bF, int grid, cudaStream_t st) {
  if constexpr (G <= 32) {
    if (v.bpart) {  // persistent ring kernel (yv, dF from the level's forward kernel)
      const int gridr = v.nbpart + ceil_div(v.nC, RTB * RCPY);
      if (v.f32)
        launch_pdl_block(k_apply_bwd_r<G, float>, gridr, RTB, RNST * sizeof(RingBuf<float>), st, v.nC, v.nbpart,
                         v.nnzLT, (const int32_t*)v.bpart, (const int32_t*)v.fidx, (const int32_t*)v.cidx,
                         (const double*)v.D, (const double*)v.yv, (const double*)v.dF, (const int64_t*)v.LTptr,
                         (const int32_t*)v.LTcol, (const float*)v.LTval, zn, z);
      else
        launch_pdl_block(k_apply_bwd_r<G, double>, gridr, RTB, RNST * sizeof(RingBuf<double>), st, v.nC, v.nbpart,
                         v.nnzLT, (const int32_t*)v.bpart, (const int32_t*)v.fidx, (const int32_t*)v.cidx,
                         (const double*)v.D, (const double*)v.yv, (const double*)v.dF, (const int64_t*)v.LTptr,
                         (const int32_t*)v.LTcol, (const double*)v.LTval, zn, z);
      return;
    }
  }
  if (v.nst_b > 0) {
    if (v.f32)
      launch_pdl_smem(k_apply_bwd_s<G, float>, grid, v.nst_b * sizeof(StageBuf<float>), st, v.nF, v.nC, bF, v.nst_b,
                      v.nnzLT, (const int32_t*)v.fidx, (const int32_t*)v.cidx, (const double*)v.D, r,
                      (const int32_t*)v.partner, (const double*)v.b11, (const double*)v.b12,
                      (const int64_t*)v.LTptr, (const int32_t*)v.LTcol, (const float*)v.LTval, zn, z,
                      (const int64_t*)v.Vptr, (const int32_t*)v.Vcol, (const double*)v.Vval, (const double*)v.rF);
    else
      launch_pdl_smem(k_apply_bwd_s<G, double>, grid, v.nst_b * sizeof(StageBuf<double>), st, v.nF, v.nC, bF,
                      v.nst_b, v.nnzLT, (const int32_t*)v.fidx, (const int32_t*)v.cidx, (const double*)v.D, r,
                      (const int32_t*)v.partner, (const double*)v.b11, (const double*)v.b12,
                      (const int64_t*)v.LTptr, (const int32_t*)v.LTcol, (const double*)v.LTval, zn, z,
                      (const int64_t*)v.Vptr, (const int32_t*)v.Vcol, (const double*)v.Vval, (const double*)v.rF);
    return;
  }
  if (v.f32)
    launch_pdl(k_apply_bwd<G, float>, grid, st, v.nF, v.nC, bF, (const int32_t*)v.fidx, (const int32_t*)v.cidx,
               (const double*)v.D, r, (const int32_t*)v.partner, (const double*)v.b11, (const double*)v.b12,
               (const int64_t*)v.LTptr, (const int32_t*)v.LTcol, (const float*)v.LTval, zn, z,
               (const int64_t*)v.Vptr, (const int32_t*)v.Vcol, (const double*)v.Vval, (const double*)v.rF);
  else
    launch_pdl(k_apply_bwd<G, double>, grid, st, v.nF, v.nC, bF, (const int32_t*)v.fidx, (const int32_t*)v.cidx,
               (const double*)v.D, r, (const int32_t*)v.partner, (const double*)v.b11, (const double*)v.b12,
               (const int64_t*)v.LTptr, (const int32_t*)v.LTcol, (const double*)v.LTval, zn, z,
               (const int64_t*)v.Vptr, (const int32_t*)v.Vcol, (const double*)v.Vval, (const double*)v.rF);
}

// kernel choice of a level's two substitutions: lanes per row, staged variants, and on large
// levels the row partition of the persistent ring kernels (AJ_APPLY_RING=0: off;
// AJ_RING_MIN: smallest entry count that takes them)
static void plan_apply(Level& v, cudaStream_t st) {
  v.gf = pick_group(v.nC ? (double)v.nnzL / v.nC : 1.0, v.nnzL);
  // few long L^T rows (deep levels): up to a CTA per row; else at most a warp per row
  v.gb = pick_group(v.nF ? (double)v.nnzLT / v.nF : 1.0, v.nnzLT, v.nF <= 2048 ? TB : 32);
  if (const char* fg = getenv("AJ_FORCE_GB")) v.gb = atoi(fg);  // testing: every backward group size
  v.nst_f = pick_stages(v.nnzL, v.nC, v.gf);
  v.nst_b = pick_stages(v.nnzLT, v.nF, v.gb);
  for (void* q : {(void*)v.fpart, (void*)v.bpart, (void*)v.yv, (void*)v.dF}) dfree(q, st);
  v.fpart = v.bpart = nullptr;
  v.yv = v.dF = nullptr;
  v.nfpart = v.nbpart = 0;
  const char* ring = getenv("AJ_APPLY_RING");
  const char* rmin = getenv("AJ_RING_MIN");
  const int64_t ring_min = rmin ? atoll(rmin) : (int64_t(1) << 22);
  if (ring && atoi(ring) != 0 && v.nst_f == 0 && v.nC > 0 && v.nnzL >= ring_min) {
    v.nfpart = (int)std::min<int64_t>(num_sms() * RING_CTAS, std::max<int64_t>(1, v.nnzL / (2 * RCAP)));
    v.fpart = dalloc<int32_t>(v.nfpart + 1, st);
    k_row_partition<<<ceil_div(v.nfpart + 1, TB), TB, 0, st>>>(v.nC, v.Lptr, v.nfpart, v.fpart);
    AJ_LAUNCHED();
    const char* rb = getenv("AJ_APPLY_RING_BWD");  // testing: 0 keeps the register backward kernels
    if (!(rb && atoi(rb) == 0) && v.nst_b == 0 && v.nF > 0 && v.gb <= 32) {
      v.nbpart = (int)std::min<int64_t>(num_sms() * RING_CTAS, std::max<int64_t>(1, v.nnzLT / (2 * RCAP)));
      v.bpart = dalloc<int32_t>(v.nbpart + 1, st);
      k_row_partition<<<ceil_div(v.nbpart + 1, TB), TB, 0, st>>>(v.nF, v.LTptr, v.nbpart, v.bpart);
      AJ_LAUNCHED();
      v.yv = dalloc<double>(v.nF, st);
      v.dF = dalloc<double>(v.nF, st);
    }
  }
}

// forward step of level v: r -> rn (the next level's input), and, if `nxt` is a sparse
// level, its compact pivot part nxt->rF
static void launch_fwd(const Level& v, const double* r, double* rn, const Level* nxt, cudaStream_t st) {
  if (v.nC == 0) return;
  const int grid = std::max(1, ceil_div((int64_t)v.nC * v.gf, TB));
  const double* gsrc = v.rF ? v.rF : r;  // levels >= 1 index their compact pivot part
  double* rFn = nxt ? nxt->rF : nullptr;
  const int32_t* fmapn = nxt ? nxt->fmap : nullptr;
  switch (v.gf) {
    case 1: fwd_g<1>(v, r, gsrc, rn, rFn, fmapn, grid, st); break;
    case 2: fwd_g<2>(v, r, gsrc, rn, rFn, fmapn, grid, st); break;
    case 4: fwd_g<4>(v, r, gsrc, rn, rFn, fmapn, grid, st); break;
    case 8: fwd_g<8>(v, r, gsrc, rn, rFn, fmapn, grid, st); break;
    case 16: fwd_g<16>(v, r, gsrc, rn, rFn, fmapn, grid, st); break;
    default: fwd_g<32>(v, r, gsrc, rn, rFn, fmapn, grid, st); break;
  }
}
static void launch_bwd(const Level& v, const double* r, const double* zn, double* z, cudaStream_t st) {
  const int bF = ceil_div((int64_t)v.nF * v.gb, TB);
  const int grid = std::max(1, bF + ceil_div(v.nC, TB));
  switch (v.gb) {
    case 1: bwd_g<1>(v, r, zn, z, bF, grid, st); break;
    case 2: bwd_g<2>(v, r, zn, z, bF, grid, st); break;
    case 4: bwd_g<4>(v, r, zn, z, bF, grid, st); break;
    case 8: bwd_g<8>(v, r, zn, z, bF, grid, st); break;
    case 16: bwd_g<16>(v, r, zn, z, bF, grid, st); break;
    case 32: bwd_g<32>(v, r, zn, z, bF, grid, st); break;
    case 64: bwd_g<64>(v, r, zn, z, bF, grid, st); break;
    case 128: bwd_g<128>(v, r, zn, z, bF, grid, st); break;
    default: bwd_g<256>(v, r, zn, z, bF, grid, st); break;
  }
}

// z = G r (dense, warp per row)
__global__ void k_dense_mv(int n, const double* __restrict__ G, const double* __restrict__ r,
                           double* __restrict__ z) {
  pdl_launch_dependents();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * TB + threadIdx.x) >> 5; i < n; i += (gridDim.x * TB) >> 5) {
    // four independent partial sums per lane: loads of four 256-byte row segments in flight
    const double* __restrict__ Gi = G + (int64_t)i * n;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int j = lane;
    for (; j + 96 < n; j += 128) {
      a0 += Gi[j] * r[j];
      a1 += Gi[j + 32] * r[j + 32];
      a2 += Gi[j + 64] * r[j + 64];
      a3 += Gi[j + 96] * r[j + 96];
    }
    for (; j < n; j += 32) a0 += Gi[j] * r[j];
    const double acc = warp_sum((a0 + a1) + (a2 + a3));
    if (lane == 0) z[i] = acc;
  }
}

// L rows: gather the per-row runs (forward values scaled by D of the column)
template <typename TV>
__global__ void k_l_gather(int nC, const int64_t* __restrict__ Lptr, const int64_t* __restrict__ row_off,
                           const int32_t* __restrict__ tcol, const double* __restrict__ tval,
                           const double* __restrict__ D, int32_t* __restrict__ Lcol, TV* __restrict__ Lval,
                           uint64_t* __restrict__ tkey, double* __restrict__ traw, const int32_t* __restrict__ fmap,
                           int compact) {
  const int lane = threadIdx.x & 31;
  for (int cp = (blockIdx.x * TB + threadIdx.x) >> 5; cp < nC; cp += (gridDim.x * TB) >> 5) {
    const int64_t d0 = Lptr[cp], cnt = Lptr[cp + 1] - d0, s0 = row_off[cp];
    for (int64_t t = lane; t < cnt; t += 32) {
      const int32_t f = tcol[s0 + t];
      const double l = tval[s0 + t];
      Lcol[d0 + t] = compact ? fmap[f] : f;
      Lval[d0 + t] = (TV)(l * D[f]);
      tkey[d0 + t] = ((uint64_t)(uint32_t)fmap[f] << 32) | (uint64_t)(uint32_t)cp;  // transpose key
      traw[d0 + t] = l;
    }
  }
}
__global__ void k_lt_count(int64_t nnz, const uint64_t* __restrict__ skey, int64_t* __restrict__ cnt) {
  for (int64_t t = blockIdx.x * (int64_t)TB + threadIdx.x; t < nnz; t += (int64_t)gridDim.x * TB)
    atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[skey[t] >> 32]), 1ull);
}
template <typename TV>
__global__ void k_lt_fill(int64_t nnz, const uint64_t* __restrict__ skey, const double* __restrict__ sval,
                          int32_t* __restrict__ LTcol, TV* __restrict__ LTval) {
  for (int64_t t = blockIdx.x * (int64_t)TB + threadIdx.x; t < nnz; t += (int64_t)gridDim.x * TB) {
    LTcol[t] = (int32_t)(skey[t] & 0xffffffffull);
    LTval[t] = (TV)sval[t];
  }
}

// ============================================================================
// host side
static void exclusive_scan_i32(const int32_t* in, int32_t* out, int n, cudaStream_t st) {
  size_t tmp = 0;
  AJ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, st));
  void* t = dalloc<char>(tmp, st);
  AJ_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, n, st));
  dfree(t, st);
}
template <typename T>
static T read_scalar(const T* d, cudaStream_t st) {
  T h;
  AJ_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, st));
  AJ_CUDA(cudaStreamSynchronize(st));
  return h;
}
// counts (n) -> ptr (n+1) with total (one device->host read); returns total
static int64_t counts_to_ptr(int64_t* cnt, int64_t*& ptr, int n, cudaStream_t st) {
  ptr = dalloc<int64_t>((size_t)n + 1, st);
  AJ_CUDA(cudaMemsetAsync(ptr, 0, sizeof(int64_t), st));
  if (n == 0) return 0;
  size_t tmp = 0;
  AJ_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt, ptr + 1, n, st));
  void* t = dalloc<char>(tmp, st);
  AJ_CUDA(cub::DeviceScan::InclusiveSum(t, tmp, cnt, ptr + 1, n, st));
  dfree(t, st);
  return read_scalar(ptr + n, st);
}

void Csr::release(cudaStream_t st) {
  dfree(ptr, st);
  dfree(col, st);
  dfree(val, st);
  ptr = nullptr;
  col = nullptr;
  val = nullptr;
}

void Level::release(cudaStream_t st) {
  for (void* p : {(void*)D, (void*)cmap, (void*)cidx, (void*)fidx, (void*)fmap, (void*)partner, (void*)b11, (void*)b12,
                  (void*)Lptr, (void*)Lcol, (void*)Lval, (void*)LTptr, (void*)LTcol, (void*)LTval, (void*)Vptr,
                  (void*)Vcol, (void*)Vval, (void*)r, (void*)z, (void*)rF, (void*)fpart, (void*)bpart, (void*)yv, (void*)dF})
    dfree(p, st);
}

// Factor one level.  Returns false on stall (nothing allocated into lv then).
static bool verbose_setup();
static bool factor_level(const Csr& A, int latticeL, int z0, const aj_precond_params& P, Level& lv, Csr& S,
                         cudaStream_t st) {
  const int n = A.n;
  const int g = grid_for(n);
  double* D = dalloc<double>(n, st);
  double* ah = dalloc<double>(A.nnz, st);
  double* dg = dalloc<double>(n, st);
  double* lmax1 = dalloc<double>(n, st);
  double* d1 = dalloc<double>(n, st);
  double* q = dalloc<double>(n, st);
  double* b11 = dalloc<double>(n, st);
  double* b12 = dalloc<double>(n, st);
  int32_t* prop = dalloc<int32_t>(n, st);
  int32_t* partner = dalloc<int32_t>(n, st);
  int32_t* leader = dalloc<int32_t>(n, st);
  int8_t* ok1 = dalloc<int8_t>(n, st);
  int8_t* inF = dalloc<int8_t>(n, st);
  int8_t* nominate = dalloc<int8_t>(n, st);
  int* counters = dalloc<int>(8, st);
  AJ_CUDA(cudaMemsetAsync(counters, 0, 8 * sizeof(int), st));
  AJ_CUDA(cudaMemsetAsync(partner, 0xff, n * sizeof(int32_t), st));
  AJ_CUDA(cudaMemsetAsync(b12, 0, n * sizeof(double), st));
  AJ_CUDA(cudaMemsetAsync(nominate, 0, n, st));

  const int gsg = grid_sg(n);
  k_rowmax_scale<<<gsg, TB, 0, st>>>(n, A.ptr, A.val, D);
  AJ_LAUNCHED();
  k_scaled_quality<<<gsg, TB, 0, st>>>(n, A.ptr, A.col, A.val, D, ah, dg, lmax1, d1, prop, ok1, P.kappa);
  AJ_LAUNCHED();
  if (latticeL == 0) {
    k_pairs<<<g, TB, 0, st>>>(n, A.ptr, A.col, ah, dg, d1, prop, ok1, P.kappa, partner, b11, b12, q,
                              counters + 0);
    AJ_LAUNCHED();
  }
  k_blocks<<<g, TB, 0, st>>>(n, latticeL, z0, ok1, dg, lmax1, partner, leader, q, b11, inF);
  AJ_LAUNCHED();

  int rounds = 0;
  if (latticeL == 0) {
    // maximal independent set of blocks on the strong graph, ranked by (q, leader)
    uint64_t* key = dalloc<uint64_t>(n, st);
    uint64_t* key2 = dalloc<uint64_t>(n, st);
    int32_t* idx = dalloc<int32_t>(n, st);
    int32_t* idx2 = dalloc<int32_t>(n, st);
    int32_t* rank = dalloc<int32_t>(n, st);
    int32_t* nbmin = dalloc<int32_t>(n, st);
    int8_t* status = dalloc<int8_t>(n, st);
    int8_t* win = dalloc<int8_t>(n, st);
    int8_t* rem = dalloc<int8_t>(n, st);
    AJ_CUDA(cudaMemsetAsync(status, 0, n, st));
    AJ_CUDA(cudaMemsetAsync(win, 0, n, st));
    AJ_CUDA(cudaMemsetAsync(rem, 0, n, st));
    k_rank_keys<<<g, TB, 0, st>>>(n, leader, q, key, idx);
    AJ_LAUNCHED();
    size_t tmp = 0;
    AJ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, key2, idx, idx2, n, 0, 64, st));
    void* t = dalloc<char>(tmp, st);
    AJ_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, key, key2, idx, idx2, n, 0, 64, st));
    dfree(t, st);
    k_rank_scatter<<<g, TB, 0, st>>>(n, idx2, rank);
    AJ_LAUNCHED();
    for (;;) {
      ++rounds;
      AJ_CUDA(cudaMemsetAsync(counters + 1, 0, sizeof(int), st));
      k_mis_nbmin<<<gsg, TB, 0, st>>>(n, A.ptr, A.col, ah, P.tau_strong, leader, status, rank, nbmin);
      AJ_LAUNCHED();
      k_mis_win<<<g, TB, 0, st>>>(n, leader, partner, status, rank, nbmin, win);
      AJ_LAUNCHED();
      k_mis_remove<<<gsg, TB, 0, st>>>(n, A.ptr, A.col, ah, P.tau_strong, leader, status, win, rem);
      AJ_LAUNCHED();
      k_mis_apply<<<g, TB, 0, st>>>(n, leader, status, win, rem, counters + 1);
      AJ_LAUNCHED();
      if (read_scalar(counters + 1, st) == 0) break;
      AJ_REQUIRE(rounds < 10000, AJ_ERR_BREAKDOWN, "independent-set rounds did not terminate");
    }
    k_mis_final<<<g, TB, 0, st>>>(n, leader, status, inF);
    AJ_LAUNCHED();
    for (void* p : {(void*)key, (void*)key2, (void*)idx, (void*)idx2, (void*)rank, (void*)nbmin,
                    (void*)status, (void*)win, (void*)rem})
      dfree(p, st);
  }
  // row-budget repair (inverse-based bound on the rows of L^{-1})
  for (int it = 0;; ++it) {
    AJ_CUDA(cudaMemsetAsync(counters + 2, 0, sizeof(int), st));
    k_budget<<<gsg, TB, 0, st>>>(n, A.ptr, A.col, ah, inF, partner, b11, b12, P.kappa, nominate, counters + 2);
    AJ_LAUNCHED();
    if (read_scalar(counters + 2, st) == 0) break;
    k_budget_apply<<<g, TB, 0, st>>>(n, partner, inF, nominate);
    AJ_LAUNCHED();
    AJ_CUDA(cudaMemsetAsync(nominate, 0, n, st));
    AJ_REQUIRE(it < 100000, AJ_ERR_BREAKDOWN, "budget repair did not terminate");
  }
  AJ_CUDA(cudaMemsetAsync(counters + 3, 0, 2 * sizeof(int), st));
  k_clear_nominate<<<g, TB, 0, st>>>(n, partner, inF, nominate, counters + 3, counters + 4);
  AJ_LAUNCHED();
  int hc[8];
  AJ_CUDA(cudaMemcpyAsync(hc, counters, sizeof(hc), cudaMemcpyDeviceToHost, st));
  AJ_CUDA(cudaStreamSynchronize(st));
  const int nF = hc[3], npairsF = hc[4];

  auto free_tmp = [&]() {
    for (void* p : {(void*)ah, (void*)dg, (void*)lmax1, (void*)d1, (void*)q, (void*)prop, (void*)leader,
                    (void*)ok1, (void*)inF, (void*)nominate, (void*)counters})
      dfree(p, st);
  };
  if (nF < P.stall_frac * n || nF == 0) {
    free_tmp();
    for (void* p : {(void*)D, (void*)b11, (void*)b12, (void*)partner}) dfree(p, st);
    return false;
  }
  const int nC = n - nF;
  lv.n = n;
  lv.nF = nF;
  lv.nC = nC;
  lv.npairs = npairsF;
  lv.rounds = rounds;
  lv.D = D;
  lv.b11 = b11;
  lv.b12 = b12;
  lv.cmap = dalloc<int32_t>(n, st);
  lv.cidx = dalloc<int32_t>(std::max(nC, 1), st);
  lv.partner = dalloc<int32_t>(n, st);
  lv.fidx = dalloc<int32_t>(std::max(nF, 1), st);
  lv.fmap = dalloc<int32_t>(n, st);
  {
    int32_t* flag = dalloc<int32_t>(n, st);
    int32_t* scan = dalloc<int32_t>(n, st);
    k_cflags<<<g, TB, 0, st>>>(n, inF, flag);
    AJ_LAUNCHED();
    exclusive_scan_i32(flag, scan, n, st);
    // b11/b12 of C nodes zeroed inside k_cmap (they were block data of non-F nodes)
    k_cmap<<<g, TB, 0, st>>>(n, inF, scan, lv.cmap, lv.cidx, lv.fidx, lv.fmap, lv.partner, partner, b11, b12);
    AJ_LAUNCHED();
    dfree(flag, st);
    dfree(scan, st);
  }
  lv.f32 = P.factor_fp32 != 0;
  // virtual 2x2 blocks of the weak pivot-pivot couplings (reading R17)
  lv.nnzV = 0;
  if (P.compensate && latticeL == 0) {
    int64_t* cnt = dalloc<int64_t>(n, st);
    k_virtual<false><<<g, TB, 0, st>>>(n, A.ptr, A.col, ah, inF, partner, b11, P.tau_virtual, cnt, nullptr, nullptr);
    AJ_LAUNCHED();
    lv.nnzV = counts_to_ptr(cnt, lv.Vptr, n, st);
    if (lv.nnzV > 0) {
      lv.Vcol = dalloc<int32_t>(lv.nnzV, st);
      lv.Vval = dalloc<double>(lv.nnzV, st);
      k_virtual<true><<<g, TB, 0, st>>>(n, A.ptr, A.col, ah, inF, partner, b11, P.tau_virtual, lv.Vptr, lv.Vcol, lv.Vval);
      AJ_LAUNCHED();
    } else {
      dfree(lv.Vptr, st);
      lv.Vptr = nullptr;
    }
    dfree(cnt, st);
  }
  // L rows and the Schur complement on the coarse nodes (aj_schur.cu): the survivors of
  // each row are appended to temp buffers through global cursors, then gathered
  {
    S.n = nC;
    SchurIn si;
    si.n = n;
    si.nC = nC;
    si.nF = nF;
    si.ptr = A.ptr;
    si.col = A.col;
    si.ah = ah;
    si.inF = inF;
    si.partner = partner;
    si.cmap = lv.cmap;
    si.cidx = lv.cidx;
    si.fmap = lv.fmap;
    si.fidx = lv.fidx;
    si.b11 = b11;
    si.b12 = b12;
    si.Vptr = lv.Vptr;
    si.Vcol = lv.Vcol;
    si.Vval = lv.Vval;
    si.tau = P.tau_drop;
    si.cap_hint = std::max<int64_t>(2 * A.nnz, (int64_t)nC * 16);
    SchurOut so;
    schur_level(si, so, st);
    int64_t* row_cnt = so.row_cnt;
    int64_t* row_off = so.row_off;
    int64_t* lrow_cnt = so.lrow_cnt;
    int64_t* lrow_off = so.lrow_off;
    int32_t* tmp_col = so.tmp_col;
    double* tmp_val = so.tmp_val;
    int32_t* ltmp_col = so.ltmp_col;
    double* ltmp_val = so.ltmp_val;
    for (int t = 0; t < 6; ++t) lv.schur_tier_rows[t] = so.tier_rows[t];
    lv.schur_ovf_rows = so.ovf_rows;
    lv.nnzFC = so.nnz_fc;
    lv.schur_products = so.products;
    lv.nnzA = A.nnz;
    // S in CSR order: the computed upper triangle and its mirror
    schur_mirror(nC, so, S, st);
    const int gg = std::max(1, std::min(ceil_div((int64_t)nC * 32, TB), num_sms() * 32));
    // L (forward rows over coarse nodes, values l*D_f) and L^T (rows over pivots, by sort)
    lv.nnzL = counts_to_ptr(lrow_cnt, lv.Lptr, nC, st);
    lv.nnzLT = lv.nnzL;
    const int64_t nL = std::max<int64_t>(lv.nnzL, 1);
    lv.Lcol = dalloc<int32_t>(nL, st);
    lv.Lval = lv.f32 ? (void*)dalloc<float>(nL, st) : (void*)dalloc<double>(nL, st);
    uint64_t* tkey = dalloc<uint64_t>(nL, st);
    uint64_t* tkey2 = dalloc<uint64_t>(nL, st);
    double* traw = dalloc<double>(nL, st);
    double* traw2 = dalloc<double>(nL, st);
    if (lv.f32)
      k_l_gather<float><<<gg, TB, 0, st>>>(nC, lv.Lptr, lrow_off, ltmp_col, ltmp_val, D, lv.Lcol, (float*)lv.Lval,
                                            tkey, traw, lv.fmap, latticeL == 0 ? 1 : 0);
    else
      k_l_gather<double><<<gg, TB, 0, st>>>(nC, lv.Lptr, lrow_off, ltmp_col, ltmp_val, D, lv.Lcol, (double*)lv.Lval,
                                             tkey, traw, lv.fmap, latticeL == 0 ? 1 : 0);
    AJ_LAUNCHED();
    {
      size_t tmpb = 0;
      AJ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmpb, tkey, tkey2, traw, traw2, (int)lv.nnzL, 0, 64, st));
      void* tb = dalloc<char>(tmpb, st);
      AJ_CUDA(cub::DeviceRadixSort::SortPairs(tb, tmpb, tkey, tkey2, traw, traw2, (int)lv.nnzL, 0, 64, st));
      dfree(tb, st);
      int64_t* cntF = dalloc<int64_t>(std::max(nF, 1), st);
      AJ_CUDA(cudaMemsetAsync(cntF, 0, sizeof(int64_t) * std::max(nF, 1), st));
      const int gl = std::max(1, std::min(grid_for(lv.nnzL), num_sms() * 32));
      k_lt_count<<<gl, TB, 0, st>>>(lv.nnzL, tkey2, cntF);
      AJ_LAUNCHED();
      const int64_t chk = counts_to_ptr(cntF, lv.LTptr, nF, st);
      AJ_REQUIRE(chk == lv.nnzL, AJ_ERR_CUDA, "L transpose count mismatch");
      lv.LTcol = dalloc<int32_t>(nL, st);
      lv.LTval = lv.f32 ? (void*)dalloc<float>(nL, st) : (void*)dalloc<double>(nL, st);
      if (lv.f32)
        k_lt_fill<float><<<gl, TB, 0, st>>>(lv.nnzL, tkey2, traw2, lv.LTcol, (float*)lv.LTval);
      else
        k_lt_fill<double><<<gl, TB, 0, st>>>(lv.nnzL, tkey2, traw2, lv.LTcol, (double*)lv.LTval);
      AJ_LAUNCHED();
      dfree(cntF, st);
    }
    for (void* q : {(void*)tkey, (void*)tkey2, (void*)traw, (void*)traw2}) dfree(q, st);
    for (void* q : {(void*)tmp_col, (void*)tmp_val, (void*)ltmp_col, (void*)ltmp_val, (void*)row_off, (void*)lrow_off,
                    (void*)lrow_cnt, (void*)row_cnt})
      dfree(q, st);
    lv.nnzS = S.nnz;
  }
  dfree(partner, st);
  free_tmp();
  return true;
}

static void precond_capture(Precond* K, cudaStream_t st);
static void inverse_based_drop(Precond* K, double tau, cudaStream_t st);

static bool verbose_setup() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("AJ_VERBOSE");
    v = (e && atoi(e) > 0) ? 1 : 0;
  }
  return v == 1;
}
static double wall_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Resolve "auto" (negative) drop parameters: tau_drop = 2e-3 min(1, (50/L)^2),
// tau_strong = min(0.05, 40 tau_drop) with compensation (R17), else 10 tau_drop,
// tau_virtual = 5..10 tau_drop (L = 50..100) (R12; the paper scales its drop tolerance with the size too,
// eps = 1/sqrt(N)).
aj_precond_params resolve_params(const aj_precond_params& in, int L) {
  aj_precond_params P = in;
  // the paper's rule: drop at eps / kappa with
  // eps = 1/sqrt(N), N = L^3 the whole lattice (also for a z-slab shard); R12
  if (P.tau_drop < 0.0) P.tau_drop = 1.0 / (P.kappa * std::sqrt((double)L * L * L));
  if (P.tau_strong < 0.0) P.tau_strong = P.compensate ? std::min(0.05, 40.0 * P.tau_drop) : 10.0 * P.tau_drop;
  if (P.tau_virtual < 0.0)  // 5 tau_drop up to L = 50, 10 tau_drop from L = 100 (measured, R17)
    P.tau_virtual = std::min(10.0, std::max(5.0, 5.0 + 5.0 * (L - 50) / 50.0)) * P.tau_drop;
  if (!P.compensate) P.tau_virtual = 0.0;
  if (P.max_levels > 1023) P.max_levels = 1023;
  return P;
}

Precond* precond_create(const double* eps, int L, double hop, double sigma, const aj_precond_params& Pin,
                        cudaStream_t st) {
  return precond_create_slab(eps, L, 0, L, false, hop, sigma, Pin, st);
}

Precond* precond_create_slab(const double* eps, int L, int z0, int nz, bool open_z, double hop, double sigma,
                             const aj_precond_params& Pin, cudaStream_t st) {
  AJ_REQUIRE(L >= 3, AJ_ERR_ARG, "precond_setup: L must be >= 3");
  const aj_precond_params P = resolve_params(Pin, L);
  (void)num_sms();  // device init: SM count + memory-pool release threshold
  AJ_REQUIRE(P.kappa > 1.0 && P.tau_drop >= 0.0 && P.tau_strong >= 0.0 && P.cand_cap >= 64,
             AJ_ERR_ARG, "precond_setup: invalid parameters");
  AJ_REQUIRE(nz >= 1 && z0 >= 0 && z0 + nz <= L && (open_z || nz == L), AJ_ERR_ARG, "precond_setup: bad slab");
  const int64_t n64 = (int64_t)L * L * nz;
  AJ_REQUIRE(n64 < (int64_t)INT32_MAX, AJ_ERR_ARG, "precond_setup: L^2 nz exceeds int32 indexing");
  cudaEvent_t e0, e1;
  AJ_CUDA(cudaEventCreate(&e0));
  AJ_CUDA(cudaEventCreate(&e1));
  AJ_CUDA(cudaEventRecord(e0, st));
  ProfScope ps(PROF_SETUP, 0.0, st);
  Precond* K = new Precond();
  K->L = L;
  K->n0 = (int)n64;
  K->P = P;
  try {
    Csr A;
    A.n = (int)n64;
    A.nnz = open_z ? (nz == 1 ? 5 * n64 : 7 * n64 - 2 * (int64_t)L * L) : 7 * n64;
    K->nnzA0 = A.nnz;
    A.ptr = dalloc<int64_t>(n64 + 1, st);
    A.col = dalloc<int32_t>(A.nnz, st);
    A.val = dalloc<double>(A.nnz, st);
    k_lattice_csr<<<std::min(grid_for(n64), num_sms() * 16), TB, 0, st>>>(L, nz, open_z ? 1 : 0, eps, hop, sigma, A.ptr, A.col,
                                                                           A.val);
    AJ_LAUNCHED();
    for (int lev = 0; lev < P.max_levels && lev < 1023; ++lev) {
      if (A.n <= P.n_coarse_max) break;
      Level lv;
      Csr S;
      const double t0 = verbose_setup() ? wall_ms() : 0.0;
      if (!factor_level(A, lev == 0 ? L : 0, z0, P, lv, S, st)) break;
      if (verbose_setup()) {
        AJ_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr,
                "[aj setup] level %d n=%d nF=%d pairs=%d virt=%lld mis_rounds=%d nnzA=%lld nnzS=%lld nnzL=%lld "
                "nnzFC=%lld products=%lld tiers=%d/%d/%d/%d/%d/%d (C16->G %d) %.2f ms\n",
                lev, lv.n, lv.nF, lv.npairs, (long long)lv.nnzV / 2, lv.rounds, (long long)A.nnz, (long long)S.nnz,
                (long long)lv.nnzL, (long long)lv.nnzFC, (long long)lv.schur_products, lv.schur_tier_rows[0],
                lv.schur_tier_rows[1], lv.schur_tier_rows[2], lv.schur_tier_rows[3], lv.schur_tier_rows[4],
                lv.schur_tier_rows[5], lv.schur_ovf_rows,
                wall_ms() - t0);
      }
      if (lev > 0) {
        lv.r = dalloc<double>(lv.n, st);
        lv.z = dalloc<double>(lv.n, st);
        lv.rF = dalloc<double>(std::max(lv.nF, 1), st);
      }
      plan_apply(lv, st);
      K->lv.push_back(lv);
      A.release(st);
      A = S;
    }
    AJ_REQUIRE(A.n <= P.dense_cap, AJ_ERR_BREAKDOWN,
               "multilevel ILDL breakdown: coarse system of size " + std::to_string(A.n) +
                   " exceeds dense_cap (increase kappa)");
    const int nc = A.n;
    K->nc = nc;
    K->rc = dalloc<double>(std::max(nc, 1), st);
    K->zc = dalloc<double>(std::max(nc, 1), st);
    K->G = dalloc<double>(std::max<int64_t>((int64_t)nc * nc, 1), st);
    const double tc0 = verbose_setup() ? wall_ms() : 0.0;
    if (nc > 0) {
      double* M = dalloc<double>((int64_t)nc * 2 * nc, st);
      double* fcol = dalloc<double>(nc, st);
      int* sing = dalloc<int>(1, st);
      AJ_CUDA(cudaMemsetAsync(sing, 0, sizeof(int), st));
      const int gd = std::min(grid_for((int64_t)nc * 2 * nc), num_sms() * 16);
      k_dense_init<<<gd, TB, 0, st>>>(nc, A.ptr, A.col, A.val, M);
      AJ_LAUNCHED();
      k_dense_scatter<<<grid_for(nc), TB, 0, st>>>(nc, A.ptr, A.col, A.val, M);
      AJ_LAUNCHED();
      // one (pivot, eliminate) launch pair per column; the elimination touches only the
      // columns j > k that are still read (left part) or returned (right part)
      if (getenv("AJ_GJ_STEPS")) {  // testing: the two-launch-per-column reference path
        const int gy = std::min(nc, 1024);
        for (int k = 0; k < nc; ++k) {
          k_gj_pivot<<<1, TB, 0, st>>>(nc, k, M, fcol, sing);
          AJ_LAUNCHED();
          const int gx = std::max(1, std::min(ceil_div(2 * nc - k - 1, TB), 8));
          k_gj_elim<<<dim3(gx, gy), TB, 0, st>>>(nc, k, M, fcol);
          AJ_LAUNCHED();
        }
        AJ_REQUIRE(read_scalar(sing, st) == 0, AJ_ERR_BREAKDOWN, "coarse Schur complement is singular");
        k_gj_extract<<<std::min(grid_for((int64_t)nc * nc), num_sms() * 16), TB, 0, st>>>(nc, M, K->G);
        AJ_LAUNCHED();
      } else if (!getenv("AJ_GJ_UNBLOCKED")) {  // default: blocked Gauss-Jordan, panels of GB columns
        const int gs = std::min(nc, num_sms() * 4);
        GjState S;
        S.prow_idx = dalloc<int>(nc, st);
        S.pivoted = dalloc<int8_t>(nc, st);
        S.prow = dalloc<double>(2 * GB, st);
        S.pv = dalloc<double>(gs, st);
        S.pi = dalloc<int>(gs, st);
        S.count = dalloc<unsigned int>(1, st);
        S.singular = sing;
        double* Pold = dalloc<double>((int64_t)nc * GB, st);
        double* Pw = dalloc<double>((int64_t)nc * GB, st);
        double* Binv = dalloc<double>(GB * GB, st);
        double* Wb = dalloc<double>((int64_t)GB * 2 * nc, st);
        int* pos = dalloc<int>(nc, st);
        AJ_CUDA(cudaMemsetAsync(S.pivoted, 0, nc, st));
        AJ_CUDA(cudaMemsetAsync(S.count, 0, sizeof(unsigned int), st));
        AJ_CUDA(cudaMemsetAsync(pos, 0xff, (size_t)nc * sizeof(int), st));
        const int rows_ctas = std::max(1, std::min(gs, ceil_div(nc, TB / 32)));
        for (int k0 = 0; k0 < nc; k0 += GB) {
          const int b = std::min(GB, nc - k0);
          k_pan_load<<<std::min(grid_for((int64_t)nc * b), num_sms() * 8), TB, 0, st>>>(nc, M, k0, b, Pold, Pw);
          AJ_LAUNCHED();
          k_pan_first<<<1, TB, 0, st>>>(nc, b, k0, Pw, S);
          AJ_LAUNCHED();
          for (int jj = 0; jj < b; ++jj) {
            k_pan_step<<<rows_ctas, TB, 0, st>>>(nc, b, jj, k0, Pw, S);
            AJ_LAUNCHED();
          }
          k_pan_binv<<<1, 256, 0, st>>>(b, k0, Pold, S.prow_idx, Binv, pos, sing);
          AJ_LAUNCHED();
          const int64_t R = 2 * (int64_t)nc - k0 - b;
          if (R > 0) {
            const int gx = std::max(1, std::min(ceil_div(R, TB), num_sms() * 4));
            k_pan_W<<<gx, TB, 0, st>>>(nc, b, k0, M, S.prow_idx, Binv, Wb);
            AJ_LAUNCHED();
            const int gxu = std::max(1, std::min(ceil_div(R, TB), 64));
            k_pan_update<<<dim3(gxu, ceil_div(nc, PR)), TB, 0, st>>>(nc, b, k0, M, Pold, Wb, pos);
            AJ_LAUNCHED();
          }
          k_pan_clear_pos<<<1, GB, 0, st>>>(b, k0, S.prow_idx, pos);
          AJ_LAUNCHED();
        }
        AJ_REQUIRE(read_scalar(sing, st) == 0, AJ_ERR_BREAKDOWN, "coarse Schur complement is singular");
        k_gj_extract_perm<<<std::min(grid_for((int64_t)nc * nc), num_sms() * 16), TB, 0, st>>>(nc, M, S.prow_idx,
                                                                                               K->G);
        AJ_LAUNCHED();
        for (void* q : {(void*)S.prow_idx, (void*)S.pivoted, (void*)S.prow, (void*)S.pv, (void*)S.pi, (void*)S.count,
                        (void*)Pold, (void*)Pw, (void*)Binv, (void*)Wb, (void*)pos})
          dfree(q, st);
      } else {  // testing (AJ_GJ_UNBLOCKED): one launch per column
        const int gs = std::min(nc, num_sms() * (getenv("AJ_GJ_CTAS") ? atoi(getenv("AJ_GJ_CTAS")) : 4));
        GjState S;
        S.prow_idx = dalloc<int>(nc, st);
        S.pivoted = dalloc<int8_t>(nc, st);
        S.prow = dalloc<double>(4 * (int64_t)nc, st);
        S.pv = dalloc<double>(gs, st);
        S.pi = dalloc<int>(gs, st);
        S.count = dalloc<unsigned int>(1, st);
        S.singular = sing;
        AJ_CUDA(cudaMemsetAsync(S.pivoted, 0, nc, st));
        AJ_CUDA(cudaMemsetAsync(S.count, 0, sizeof(unsigned int), st));
        k_gj_first<<<1, TB, 0, st>>>(nc, M, S);
        AJ_LAUNCHED();
        for (int k = 0; k < nc; ++k) {
          k_gj_step<<<gs, TB, 0, st>>>(nc, k, M, S);
          AJ_LAUNCHED();
        }
        AJ_REQUIRE(read_scalar(sing, st) == 0, AJ_ERR_BREAKDOWN, "coarse Schur complement is singular");
        k_gj_extract_perm<<<std::min(grid_for((int64_t)nc * nc), num_sms() * 16), TB, 0, st>>>(nc, M, S.prow_idx,
                                                                                               K->G);
        AJ_LAUNCHED();
        for (void* q : {(void*)S.prow_idx, (void*)S.pivoted, (void*)S.prow, (void*)S.pv, (void*)S.pi, (void*)S.count})
          dfree(q, st);
      }
      dfree(M, st);
      dfree(fcol, st);
      dfree(sing, st);
    }
    if (verbose_setup()) {
      AJ_CUDA(cudaStreamSynchronize(st));
      fprintf(stderr, "[aj setup] coarse n=%d dense inverse %.2f ms\n", nc, wall_ms() - tc0);
    }
    A.release(st);
    if (P.tau_inv > 0.0) inverse_based_drop(K, P.tau_inv, st);
  } catch (...) {
    precond_destroy(K, st);
    throw;
  }
  AJ_CUDA(cudaEventRecord(e1, st));
  AJ_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  AJ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  // info
  aj_precond_info& I = K->info;
  memset(&I, 0, sizeof(I));
  I.levels = (int)K->lv.size();
  I.coarse_n = K->nc;
  I.nnz_A = K->nnzA0;
  for (size_t l = 0; l < K->lv.size(); ++l) {
    const Level& v = K->lv[l];
    I.setup_products += v.schur_products;
    // compulsory traffic of the level (12 B per (index, value) entry): read the level matrix,
    // write and re-read its FC lists, stream one FC entry per Schur product, write S (temp
    // run + CSR gather) and L (temp run, CSR, transpose)
    I.setup_bytes += 12.0 * ((double)v.nnzA + 2.0 * v.nnzFC + (double)v.schur_products + 3.0 * v.nnzS + 4.0 * v.nnzL);
    I.nnz_L += v.nnzL;
    I.nnz_V += v.nnzV / 2;
    I.level_n[l] = v.n;
    I.level_nF[l] = v.nF;
    I.level_pairs[l] = v.npairs;
    I.level_nnzS[l] = v.nnzS;
  }
  ps.set_bytes(I.setup_bytes);  // live profile of the setup phase: its work model (DESIGN.md sect. 4)
  I.setup_ms = ms;
  I.tau_drop = P.tau_drop;
  I.tau_strong = P.tau_strong;
  I.tau_virtual = P.tau_virtual;
  I.tau_inv = P.tau_inv;
  for (const auto& v : K->lv) I.nnz_L_dropped_inv += v.ndrop_inv;
  K->bytes_per_apply = precond_bytes_per_apply(K);
  precond_capture(K, st);
  return K;
}

void precond_destroy(Precond* K, cudaStream_t st) {
  if (!K) return;
  if (K->exec) cudaGraphExecDestroy(K->exec);
  for (auto& l : K->lv) l.release(st);
  dfree(K->G, st);
  dfree(K->rc, st);
  dfree(K->zc, st);
  delete K;
}

// levels >= 1 and the coarse solve, between internal buffers (captured once
// into a CUDA graph at the end of precond_create)
static void precond_inner(const Precond* K, cudaStream_t st) {
  const int nl = (int)K->lv.size();
  for (int l = 1; l < nl; ++l) {
    const Level& v = K->lv[l];
    launch_fwd(v, v.r, (l + 1 < nl) ? K->lv[l + 1].r : K->rc, (l + 1 < nl) ? &K->lv[l + 1] : nullptr, st);
  }
  if (K->nc > 0) {
    const double* rin = (nl >= 1) ? K->rc : nullptr;
    if (nl >= 1) {
      k_dense_mv<<<std::max(1, ceil_div((int64_t)K->nc * 32, TB)), TB, 0, st>>>(K->nc, K->G, rin, K->zc);
      AJ_LAUNCHED();
    }
  }
  for (int l = nl - 1; l >= 1; --l) {
    const Level& v = K->lv[l];
    launch_bwd(v, v.r, (l + 1 < nl) ? K->lv[l + 1].z : K->zc, v.z, st);
  }
}

// ----------------------------------------------------------------------------
// Inverse-based (aggressive) dropping a posteriori (reading R18,
// oracle/mlildl.py::nu_estimates / inverse_based_drop): the Cline-Moler-Stewart-
// Wilkinson estimate x of the column norms nu_i ~ ||L~^{-1} e_i|| by back substitution
// with L~^T, level by level from the coarse block up (one thread per L^T row, the row
// summed in ascending coarse index: the oracle's order), then every entry with
// (|fl(l D_f)| nu_c) #col_f <= tau D_f is removed from both copies of L.
__global__ void k_nu_pivots(int nF, const int64_t* __restrict__ LTptr, const int32_t* __restrict__ LTcol,
                            const double* __restrict__ LTval, const double* __restrict__ xn,
                            const int32_t* __restrict__ fidx, double* __restrict__ x) {
  for (int fp = blockIdx.x * TB + threadIdx.x; fp < nF; fp += gridDim.x * TB) {
    double s = 0.0;
    for (int64_t e = LTptr[fp]; e < LTptr[fp + 1]; ++e) s = __dadd_rn(s, __dmul_rn(LTval[e], xn[LTcol[e]]));
    x[fidx[fp]] = __dsub_rn(s > 0.0 ? -1.0 : 1.0, s);
  }
}
__global__ void k_nu_coarse(int nC, const int32_t* __restrict__ cidx, const double* __restrict__ xn,
                            double* __restrict__ x) {
  for (int cp = blockIdx.x * TB + threadIdx.x; cp < nC; cp += gridDim.x * TB) x[cidx[cp]] = xn[cp];
}
__device__ __forceinline__ bool inv_keep(double lf, double nu_c, double cnt_f, double tau, double Df) {
  return __dmul_rn(__dmul_rn(fabs(lf), nu_c), cnt_f) > __dmul_rn(tau, Df);
}
// forward rows (over coarse nodes): count / compact the kept entries
template <bool FILL>
__global__ void k_inv_fwd(int nC, const int64_t* __restrict__ Lptr, const int32_t* __restrict__ Lcol,
                          const double* __restrict__ Lval, int compact, const int32_t* __restrict__ fmap,
                          const int32_t* __restrict__ fidx, const double* __restrict__ D,
                          const int64_t* __restrict__ LTptr, const double* __restrict__ xn, double tau,
                          int64_t* __restrict__ cnt_or_ptr, int32_t* __restrict__ Lcol2, double* __restrict__ Lval2) {
  for (int cp = blockIdx.x * TB + threadIdx.x; cp < nC; cp += gridDim.x * TB) {
    const double nu = fabs(xn[cp]);
    int64_t w = FILL ? cnt_or_ptr[cp] : 0;
    for (int64_t e = Lptr[cp]; e < Lptr[cp + 1]; ++e) {
      const int fp = compact ? Lcol[e] : fmap[Lcol[e]];
      const int f = fidx[fp];
      const double cntf = (double)(LTptr[fp + 1] - LTptr[fp]);
      if (!inv_keep(Lval[e], nu, cntf, tau, D[f])) continue;
      if (FILL) {
        Lcol2[w] = Lcol[e];
        Lval2[w] = Lval[e];
      }
      ++w;
    }
    if (!FILL) cnt_or_ptr[cp] = w;
  }
}
// backward rows (over pivots): the same decision, fl(l D_f) recomputed exactly as k_l_gather
template <bool FILL>
__global__ void k_inv_bwd(int nF, const int64_t* __restrict__ LTptr, const int32_t* __restrict__ LTcol,
                          const double* __restrict__ LTval, const int32_t* __restrict__ fidx,
                          const double* __restrict__ D, const double* __restrict__ xn, double tau,
                          int64_t* __restrict__ cnt_or_ptr, int32_t* __restrict__ LTcol2, double* __restrict__ LTval2,
                          int64_t* __restrict__ ndrop) {
  for (int fp = blockIdx.x * TB + threadIdx.x; fp < nF; fp += gridDim.x * TB) {
    const int f = fidx[fp];
    const double Df = D[f];
    const int64_t e0 = LTptr[fp], e1 = LTptr[fp + 1];
    const double cntf = (double)(e1 - e0);
    int64_t w = FILL ? cnt_or_ptr[fp] : 0;
    for (int64_t e = e0; e < e1; ++e) {
      const int cp = LTcol[e];
      const double lf = LTval[e] * Df;
      if (!inv_keep(lf, fabs(xn[cp]), cntf, tau, Df)) continue;
      if (FILL) {
        LTcol2[w] = cp;
        LTval2[w] = LTval[e];
      }
      ++w;
    }
    if (!FILL) {
      cnt_or_ptr[fp] = w;
      atomicAdd(reinterpret_cast<unsigned long long*>(ndrop), (unsigned long long)((e1 - e0) - w));
    }
  }
}

static void inverse_based_drop(Precond* K, double tau, cudaStream_t st) {
  AJ_REQUIRE(!K->P.factor_fp32, AJ_ERR_ARG, "inverse-based dropping needs the fp64 factor (factor_fp32 = 0)");
  const int nl = (int)K->lv.size();
  if (nl == 0) return;
  std::vector<double*> x(nl + 1, nullptr);
  x[nl] = dalloc<double>(std::max(K->nc, 1), st);
  launch_fill(x[nl], 1.0, std::max(K->nc, 1), st);  // coarse block: no L entries, x = b = +1
  for (int l = nl - 1; l >= 0; --l) {
    const Level& v = K->lv[l];
    x[l] = dalloc<double>(std::max(v.n, 1), st);
    const int gf = std::max(1, std::min(grid_for(std::max(v.nF, 1)), num_sms() * 8));
    k_nu_pivots<<<gf, TB, 0, st>>>(v.nF, v.LTptr, v.LTcol, (const double*)v.LTval, x[l + 1], v.fidx, x[l]);
    AJ_LAUNCHED();
    const int gc = std::max(1, std::min(grid_for(std::max(v.nC, 1)), num_sms() * 8));
    k_nu_coarse<<<gc, TB, 0, st>>>(v.nC, v.cidx, x[l + 1], x[l]);
    AJ_LAUNCHED();
  }
  int64_t* ndrop = dalloc<int64_t>(1, st);
  for (int l = 0; l < nl; ++l) {
    Level& v = K->lv[l];
    const double* xn = x[l + 1];
    AJ_CUDA(cudaMemsetAsync(ndrop, 0, sizeof(int64_t), st));
    const int gc = std::max(1, std::min(grid_for(std::max(v.nC, 1)), num_sms() * 8));
    const int gf = std::max(1, std::min(grid_for(std::max(v.nF, 1)), num_sms() * 8));
    const int compact = v.rF ? 1 : 0;  // levels >= 1 store pivot-local columns
    int64_t* cnt = dalloc<int64_t>(std::max(v.nC, 1), st);
    k_inv_fwd<false><<<gc, TB, 0, st>>>(v.nC, v.Lptr, v.Lcol, (const double*)v.Lval, compact, v.fmap, v.fidx, v.D,
                                        v.LTptr, xn, tau, cnt, nullptr, nullptr);
    AJ_LAUNCHED();
    int64_t* Lptr2 = nullptr;
    const int64_t nL2 = counts_to_ptr(cnt, Lptr2, v.nC, st);
    int32_t* Lcol2 = dalloc<int32_t>(std::max<int64_t>(nL2, 1), st);
    double* Lval2 = dalloc<double>(std::max<int64_t>(nL2, 1), st);
    k_inv_fwd<true><<<gc, TB, 0, st>>>(v.nC, v.Lptr, v.Lcol, (const double*)v.Lval, compact, v.fmap, v.fidx, v.D,
                                       v.LTptr, xn, tau, Lptr2, Lcol2, Lval2);
    AJ_LAUNCHED();
    int64_t* cntF = dalloc<int64_t>(std::max(v.nF, 1), st);
    k_inv_bwd<false><<<gf, TB, 0, st>>>(v.nF, v.LTptr, v.LTcol, (const double*)v.LTval, v.fidx, v.D, xn, tau, cntF,
                                        nullptr, nullptr, ndrop);
    AJ_LAUNCHED();
    int64_t* LTptr2 = nullptr;
    const int64_t nLT2 = counts_to_ptr(cntF, LTptr2, v.nF, st);
    AJ_REQUIRE(nLT2 == nL2, AJ_ERR_CUDA, "inverse-based dropping: L and L^T disagree");
    int32_t* LTcol2 = dalloc<int32_t>(std::max<int64_t>(nL2, 1), st);
    double* LTval2 = dalloc<double>(std::max<int64_t>(nL2, 1), st);
    k_inv_bwd<true><<<gf, TB, 0, st>>>(v.nF, v.LTptr, v.LTcol, (const double*)v.LTval, v.fidx, v.D, xn, tau, LTptr2,
                                       LTcol2, LTval2, ndrop);
    AJ_LAUNCHED();
    v.ndrop_inv = v.nnzL - nL2;
    for (void* q : {(void*)v.Lptr, (void*)v.Lcol, v.Lval, (void*)v.LTptr, (void*)v.LTcol, v.LTval, (void*)cnt,
                    (void*)cntF})
      dfree(q, st);
    v.Lptr = Lptr2;
    v.Lcol = Lcol2;
    v.Lval = Lval2;
    v.LTptr = LTptr2;
    v.LTcol = LTcol2;
    v.LTval = LTval2;
    v.nnzL = v.nnzLT = nL2;
    plan_apply(v, st);
  }
  dfree(ndrop, st);
  for (double* p : x) dfree(p, st);
}

static void precond_capture(Precond* K, cudaStream_t st) {
  if (K->lv.size() < 1) return;
  cudaStream_t cs = capture_stream();
  AJ_CUDA(cudaStreamSynchronize(st));
  const int64_t before = g_launches;
  AJ_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  precond_inner(K, cs);
  cudaGraph_t g;
  AJ_CUDA(cudaStreamEndCapture(cs, &g));
  K->graph_nodes = g_launches - before;
  g_launches = before;
  AJ_CUDA(cudaGraphInstantiate(&K->exec, g, 0));
  AJ_CUDA(cudaGraphDestroy(g));
}

// z = K^{-1} r
void precond_run(const Precond* K, double* z, const double* r, cudaStream_t st) {
  ProfScope ps(PROF_PREC, (double)K->bytes_per_apply, st);
  const int nl = (int)K->lv.size();
  if (nl == 0) {
    k_dense_mv<<<std::max(1, ceil_div((int64_t)K->nc * 32, TB)), TB, 0, st>>>(K->nc, K->G, r, z);
    AJ_LAUNCHED();
    return;
  }
  const Level& v0 = K->lv[0];
  launch_fwd(v0, r, (nl > 1) ? K->lv[1].r : K->rc, (nl > 1) ? &K->lv[1] : nullptr, st);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  AJ_CUDA(cudaStreamIsCapturing(st, &cs));
  if (K->exec && cs != cudaStreamCaptureStatusActive) {
    AJ_CUDA(cudaGraphLaunch(K->exec, st));
    g_launches += K->graph_nodes;
  } else {
    precond_inner(K, st);
  }
  launch_bwd(v0, r, (nl > 1) ? K->lv[1].z : K->zc, z, st);
}

int64_t precond_bytes_per_apply(const Precond* K) {
  // algorithmic HBM bytes of one application: every stored factor entry read once
  // (8 B value + 4 B index) plus per-level vectors (r read twice, D, z/rn writes)
  int64_t b = 0;
  for (const auto& v : K->lv) {
    b += (v.nnzL + v.nnzLT) * (v.f32 ? 8 : 12) + v.nnzV * 12;
    b += (int64_t)v.n * (8 /*D*/ + 8 /*r*/ + 8 /*z*/ + 4 /*cmap*/ + 8 * 2 /*b11,b12 for F*/ + 4 /*partner*/);
    b += (int64_t)v.nC * (4 + 8 + 8 + 8);  // cidx, D_c r_c, rn write, L ptr
    if (v.rF) b += (int64_t)v.nF * (8 + 4);  // compact pivot part written by the previous step (+ fmap)
  }
  b += (int64_t)K->nc * K->nc * 8;
  return b;
}

}  // namespace aj
