// Correction-equation SQMR and the symmetric Jacobi-Davidson driver.
//
// PAPER.md sect. 4.2 (l.380-421): JD expands V with corrections from
//   (I - Q~Q~^T)(A - theta I)(I - Q~Q~^T) z = -r,   Q~ = [Q, u],
// solved approximately by the simplified QMR method (l.412-416, l.986) with the
// projected preconditioner (I - Y H^{-1} Q~^T) K^{-1}, Y = K^{-1} Q~, H = Q~^T Y
// -- the block form of (I - u w^T / w^T u) K^{-1}, K w = u (l.414-415).
// K is the multilevel ILDL of A - sigma I (aj_mlildl.cu), built once per solve.
//
// Device residency: every SQMR scalar (rho, tau, theta, alpha, ...) lives in
// device memory and is updated by the "last block" of the fused reduction
// kernels, so one SQMR step is: fused stencil+dots, two fused update kernels,
// the preconditioner sweep, two tall-skinny dot kernels and one update kernel;
// the host only reads the residual norm for the stopping test.
#include <algorithm>
#include <climits>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "aj_common.cuh"
#include "aj_kernels.cuh"
#include "aj_mlildl.cuh"
#include "aj_solver.cuh"

namespace aj {

constexpr int TB = 256;
static int sgrid(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, TB), (int64_t)num_sms() * 8));
}

// scalar slots
enum { S_TAU = 0, S_THETA, S_A1, S_A2, S_RX2, S_BRK, S_RHO0, S_RHO1, S_NB, S_COUNT = 16 };

// the SQMR scalar recurrences of one step from ||r||^2 = rr, sigma_q = sig, alpha
__device__ __forceinline__ void sqmr_B_scalars(double* sc, double rr, double sig, double alpha) {
  const double tau = sc[S_TAU], th_old = sc[S_THETA];
  const double th = sqrt(rr) / tau;
  const double c2 = 1.0 / (1.0 + th * th);
  sc[S_A1] = c2 * th_old * th_old;
  sc[S_A2] = c2 * alpha;
  sc[S_THETA] = th;
  sc[S_TAU] = tau * th * sqrt(c2);
  if (sig == 0.0 || !isfinite(alpha)) sc[S_BRK] = 1.0;
}

// t' = t - Qt c ;  alpha = rho/sigma_q ; r -= alpha t' ; ||r||^2 -> theta, tau, coefficients
// (sharded: the last block leaves the local ||r||^2 in rb.out and k_sqmr_B_scalars runs
// after the all-reduce)
__global__ void __launch_bounds__(TB)
    k_sqmr_B(int64_t n, int m, const double* __restrict__ Qt, double* __restrict__ t, double* __restrict__ r,
             const double* __restrict__ dotsA, const double* __restrict__ rho_cur, double* __restrict__ sc,
             RedBuf rb, int dist) {
  __shared__ double sc_c[32];
  if (threadIdx.x < m) sc_c[threadIdx.x] = dotsA[threadIdx.x];
  __syncthreads();
  const double sig = dotsA[m];
  const double alpha = (*rho_cur) / sig;
  double acc[1] = {0.0};
  for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < n; s += (int64_t)gridDim.x * TB) {
    double tv = t[s];
    for (int c = 0; c < m; ++c) tv -= __ldg(&Qt[(int64_t)c * n + s]) * sc_c[c];
    t[s] = tv;
    const double rv = r[s] - alpha * tv;
    r[s] = rv;
    acc[0] += rv * rv;
  }
  if (block_reduce_finalize<1, TB>(acc, rb, blockIdx.x, gridDim.x) && threadIdx.x == 0 && !dist)
    sqmr_B_scalars(sc, rb.out[0], sig, alpha);
}
__global__ void k_sqmr_B_scalars(int m, const double* __restrict__ rr, const double* __restrict__ dotsA,
                                 const double* __restrict__ rho_cur, double* __restrict__ sc) {
  const double sig = dotsA[m];
  sqmr_B_scalars(sc, rr[0], sig, (*rho_cur) / sig);
}

// d = a1 d + a2 q ; x += d ; s = a1 s + a2 t' ; rx -= s ; ||rx||^2
__global__ void __launch_bounds__(TB)
    k_sqmr_C(int64_t n, const double* __restrict__ q, const double* __restrict__ t, double* __restrict__ d,
             double* __restrict__ x, double* __restrict__ sv, double* __restrict__ rx, double* __restrict__ sc,
             RedBuf rb) {
  const double a1 = sc[S_A1], a2 = sc[S_A2];
  double acc[1] = {0.0};
  for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < n; s += (int64_t)gridDim.x * TB) {
    const double dv = a1 * d[s] + a2 * q[s];
    d[s] = dv;
    x[s] += dv;
    const double svv = a1 * sv[s] + a2 * t[s];
    sv[s] = svv;
    const double rxv = rx[s] - svv;
    rx[s] = rxv;
    acc[0] += rxv * rxv;
  }
  if (block_reduce_finalize<1, TB>(acc, rb, blockIdx.x, gridDim.x) && threadIdx.x == 0) sc[S_RX2] = rb.out[0];
}

// g = Hinv (Q~^T w); rho_new = w^T r - (Y^T r) . g; q = (w - Y g) + beta q
__global__ void __launch_bounds__(TB)
    k_sqmr_F(int64_t n, int m, const double* __restrict__ Y, const double* __restrict__ w,
             double* __restrict__ q, const double* __restrict__ dQw, const double* __restrict__ dYr,
             const double* __restrict__ Hinv, const double* __restrict__ rho_prev, double* __restrict__ rho_out,
             int first, double* __restrict__ sc) {
  __shared__ double g[32];
  __shared__ double s_beta;
  if (threadIdx.x < m) {
    double a = 0.0;
    for (int b = 0; b < m; ++b) a += Hinv[threadIdx.x + b * m] * dQw[b];
    g[threadIdx.x] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double rho = dYr[m];
    for (int c = 0; c < m; ++c) rho -= dYr[c] * g[c];
    const double beta = first ? 0.0 : rho / (*rho_prev);
    s_beta = beta;
    if (blockIdx.x == 0) {
      *rho_out = rho;
      if (rho == 0.0 || !isfinite(beta)) sc[S_BRK] = 1.0;
    }
  }
  __syncthreads();
  const double beta = s_beta;
  for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < n; s += (int64_t)gridDim.x * TB) {
    double u = w[s];
    for (int c = 0; c < m; ++c) u -= __ldg(&Y[(int64_t)c * n + s]) * g[c];
    q[s] = u + (first ? 0.0 : beta * q[s]);
  }
}

__global__ void k_sqmr_init_scalars(double* sc, const double* nb2) {
  const double nb = sqrt(*nb2);
  for (int i = 0; i < S_COUNT; ++i) sc[i] = 0.0;
  sc[S_TAU] = nb;
  sc[S_NB] = nb;
  sc[S_RX2] = *nb2;
  sc[S_RHO0] = 1.0;
  sc[S_RHO1] = 1.0;
}

// ----------------------------------------------------------------------------
// small dense kernels (one CTA): symmetric eigen (parallel cyclic Jacobi,
// round-robin pairing), sorted by |theta| then theta; H^{-1} by Gauss-Jordan.
constexpr int EIG_MAX = 48;
__global__ void __launch_bounds__(256) k_small_eig(int j, int ldm, const double* __restrict__ Min,
                                                   double* __restrict__ theta, double* __restrict__ S) {
  __shared__ double A[EIG_MAX][EIG_MAX + 1];
  __shared__ double Vv[EIG_MAX][EIG_MAX + 1];
  __shared__ double cs[EIG_MAX / 2], sn[EIG_MAX / 2];
  __shared__ int pp[EIG_MAX / 2], qq[EIG_MAX / 2];
  __shared__ double s_off, s_tot;
  __shared__ int order[EIG_MAX];
  const int tid = threadIdx.x;
  for (int t = tid; t < j * j; t += blockDim.x) {
    const int a = t % j, b = t / j;
    A[a][b] = 0.5 * (Min[a + b * ldm] + Min[b + a * ldm]);
    Vv[a][b] = (a == b) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int J2 = (j + 1) & ~1;  // even number of players (dummy = j if odd)
  const int npair = J2 / 2;
  for (int sweep = 0; sweep < 40 && j > 1; ++sweep) {
    if (tid == 0) {
      double off = 0.0, tot = 0.0;
      for (int a = 0; a < j; ++a)
        for (int b = 0; b < j; ++b) {
          const double v = A[a][b] * A[a][b];
          tot += v;
          if (a != b) off += v;
        }
      s_off = off;
      s_tot = tot;
    }
    __syncthreads();
    if (s_off <= 1e-32 * s_tot || s_off == 0.0) break;
    for (int rd = 0; rd < J2 - 1; ++rd) {
      if (tid < npair) {
        int p, q;
        if (tid == 0) {
          p = rd;
          q = J2 - 1;
        } else {
          p = (rd + tid) % (J2 - 1);
          q = (rd - tid + (J2 - 1)) % (J2 - 1);
        }
        if (p > q) {
          const int tmp = p;
          p = q;
          q = tmp;
        }
        double c = 1.0, s = 0.0;
        if (q < j) {
          const double apq = A[p][q];
          if (apq != 0.0) {
            const double tau = (A[q][q] - A[p][p]) / (2.0 * apq);
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
          }
        }
        pp[tid] = p;
        qq[tid] = q;
        cs[tid] = c;
        sn[tid] = s;
      }
      __syncthreads();
      // rows: A <- J^T A
      for (int t = tid; t < npair * j; t += blockDim.x) {
        const int pi = t / j, k = t % j;
        const int p = pp[pi], q = qq[pi];
        if (q >= j) continue;
        const double c = cs[pi], s = sn[pi];
        const double ap = A[p][k], aq = A[q][k];
        A[p][k] = c * ap - s * aq;
        A[q][k] = s * ap + c * aq;
      }
      __syncthreads();
      // columns: A <- A J ; V <- V J
      for (int t = tid; t < npair * j; t += blockDim.x) {
        const int pi = t / j, k = t % j;
        const int p = pp[pi], q = qq[pi];
        if (q >= j) continue;
        const double c = cs[pi], s = sn[pi];
        const double ap = A[k][p], aq = A[k][q];
        A[k][p] = c * ap - s * aq;
        A[k][q] = s * ap + c * aq;
        const double vp = Vv[k][p], vq = Vv[k][q];
        Vv[k][p] = c * vp - s * vq;
        Vv[k][q] = s * vp + c * vq;
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    for (int a = 0; a < j; ++a) order[a] = a;
    for (int a = 1; a < j; ++a) {  // sort by (|theta|, theta)
      const int v = order[a];
      const double tv = A[v][v];
      int b = a - 1;
      while (b >= 0) {
        const double tb = A[order[b]][order[b]];
        const bool greater = (fabs(tb) > fabs(tv)) || (fabs(tb) == fabs(tv) && tb > tv);
        if (!greater) break;
        order[b + 1] = order[b];
        --b;
      }
      order[b + 1] = v;
    }
  }
  __syncthreads();
  for (int t = tid; t < j * j; t += blockDim.x) {
    const int a = t % j, b = t / j;
    S[a + b * j] = Vv[a][order[b]];
  }
  for (int t = tid; t < j; t += blockDim.x) theta[t] = A[order[t]][order[t]];
}

// Hinv = H^{-1} for the symmetrised m x m H (ld ldh), m <= 17, by Gauss-Jordan with
// partial pivoting in one CTA: per column, warp 0 picks the pivot row (largest |a|,
// smallest row on ties), then all threads swap, scale and eliminate.  A pivot with
// |a| <= 1e-13 max|H| is a breakdown: *status = 1 and Hinv is not written (the caller
// reads the status before using Hinv).
constexpr int INV_MAX = 17;
__global__ void __launch_bounds__(256)
    k_small_inv(int m, const double* __restrict__ H, int ldh, double* __restrict__ Hinv, int* __restrict__ status) {
  __shared__ double A[INV_MAX][2 * INV_MAX + 1];
  __shared__ int s_piv;
  __shared__ double s_thr;
  const int tid = threadIdx.x, w = 2 * m;
  for (int t = tid; t < m * w; t += blockDim.x) {
    const int a = t / w, b = t % w;
    A[a][b] = (b < m) ? 0.5 * (H[a + b * ldh] + H[b + a * ldh]) : (b - m == a ? 1.0 : 0.0);
  }
  __syncthreads();
  if (tid < 32) {
    double mx = 0.0;
    for (int t = tid; t < m * m; t += 32) mx = fmax(mx, fabs(A[t / m][t % m]));
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (tid == 0) s_thr = 1e-13 * mx;
  }
  for (int k = 0; k < m; ++k) {
    __syncthreads();
    if (tid < 32) {
      const int a = k + tid;
      double v = (a < m) ? fabs(A[a][k]) : -1.0;
      int ix = (a < m) ? a : INT_MAX;
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, ix, o);
        if (v2 > v || (v2 == v && i2 < ix)) {
          v = v2;
          ix = i2;
        }
      }
      if (tid == 0) s_piv = (v > s_thr) ? ix : -1;
    }
    __syncthreads();
    const int p = s_piv;
    if (p < 0) {
      if (tid == 0) *status = 1;
      return;  // uniform
    }
    if (p != k)
      for (int b = tid; b < w; b += blockDim.x) {
        const double t = A[k][b];
        A[k][b] = A[p][b];
        A[p][b] = t;
      }
    __syncthreads();
    const double inv = 1.0 / A[k][k];
    __syncthreads();
    for (int b = tid; b < w; b += blockDim.x) A[k][b] *= inv;
    __syncthreads();
    // eliminate column k from the other rows; column k itself is read from a copy
    double fa = 0.0;
    if (tid < m) fa = A[tid][k];
    __syncthreads();
    __shared__ double fcol[INV_MAX];
    if (tid < m) fcol[tid] = (tid == k) ? 0.0 : fa;
    __syncthreads();
    for (int t = tid; t < m * w; t += blockDim.x) {
      const int a = t / w, b = t % w;
      if (a != k && fcol[a] != 0.0) A[a][b] -= fcol[a] * A[k][b];
    }
  }
  __syncthreads();
  for (int t = tid; t < m * m; t += blockDim.x) {
    const int a = t % m, b = t / m;
    Hinv[a + b * m] = A[a][m + b];
  }
  if (tid == 0) *status = 0;
}

// M[:, j] and M[j, :] <- dots (j+1 values)
__global__ void k_set_mcol(double* M, int ldm, int j, const double* __restrict__ dots) {
  const int a = threadIdx.x;
  if (a <= j) {
    M[a + j * ldm] = dots[a];
    M[j + a * ldm] = dots[a];
  }
}
// M <- diag(theta[off .. off+cnt))
__global__ void k_set_mdiag(double* M, int ldm, int cnt, const double* __restrict__ theta, int off) {
  for (int t = threadIdx.x; t < cnt * cnt; t += blockDim.x) {
    const int a = t % cnt, b = t / cnt;
    M[a + b * ldm] = (a == b) ? theta[off + a] : 0.0;
  }
}
// y = a*x + b*y with (a, b) = (1, -theta[0]) style device scalar: r = Au - theta u
__global__ void k_resid(int64_t n, const double* __restrict__ Au, const double* __restrict__ u,
                        const double* __restrict__ theta, double* __restrict__ r, RedBuf rb) {
  const double th = theta[0];
  double acc[1] = {0.0};
  for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < n; s += (int64_t)gridDim.x * TB) {
    const double v = Au[s] - th * u[s];
    r[s] = v;
    acc[0] += v * v;
  }
  block_reduce_finalize<1, TB>(acc, rb, blockIdx.x, gridDim.x);
}
// start vector: uniform(-0.5, 0.5) from the counter stream `key`
// (s0: global index of the first local site, so a sharded start vector is the slice of the full one)
__global__ void k_start(int64_t n, uint64_t key, double* __restrict__ v, int64_t s0) {
  for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < n; s += (int64_t)gridDim.x * TB)
    v[s] = uniform01(key, (uint64_t)(s0 + s)) - 0.5;
}
// max |eps|
__global__ void k_absmax(int64_t n, const double* __restrict__ x, unsigned long long* out) {
  double m = 0.0;
  for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < n; s += (int64_t)gridDim.x * TB)
    m = fmax(m, fabs(x[s]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}
__global__ void k_negate_proj(int64_t n, double* __restrict__ b, const double* __restrict__ r,
                              const double* __restrict__ Qt, int m, const double* __restrict__ c) {
  __shared__ double sc_c[32];
  if (threadIdx.x < m) sc_c[threadIdx.x] = c[threadIdx.x];
  __syncthreads();
  for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < n; s += (int64_t)gridDim.x * TB) {
    double v = r[s];
    for (int a = 0; a < m; ++a) v -= __ldg(&Qt[(int64_t)a * n + s]) * sc_c[a];
    b[s] = -v;
  }
}

// ============================================================================
Workspace::Workspace(int64_t n_, cudaStream_t st) : n(n_) {
  rs.init(st);
  hpin = pinned_scalars();       // per host thread, reused across solves
  cap_stream = capture_stream();
  // opt-in (AJ_SQMR_GRAPH=1): capturing two graphs per correction equation costs more
  // than it saves at ~20 SQMR steps per solve (L=50 step 361 vs 337 ms)
  const char* e = getenv("AJ_SQMR_GRAPH");
  use_graphs = (e && atoi(e) == 1);
  sc = dalloc<double>(S_COUNT, st);
  small = dalloc<double>(8192, st);
  for (int i = 0; i < 9; ++i) vec[i] = dalloc<double>(n, st);
}
void Workspace::release(cudaStream_t st) {
  rs.release(st);
  hpin = nullptr;       // owned per host thread (pinned_scalars / capture_stream)
  cap_stream = nullptr;
  dfree(sc, st);
  dfree(small, st);
  for (int i = 0; i < 9; ++i) dfree(vec[i], st);
}

void dom_precond(const Domain& dom, const Precond* K, double* z, const double* r, cudaStream_t st) {
  if (!dom.sharded() || !dom.rfull) {
    precond_run(K, z, r, st);
    return;
  }
  dom_gather_full(dom, dom.rfull, r, st);
  precond_run(K, dom.zfull, dom.rfull, st);
  AJ_CUDA(cudaMemcpyAsync(z, dom.zfull + dom.site0(), (size_t)dom.n * sizeof(double), cudaMemcpyDeviceToDevice, st));
}

// SQMR on the projected operator.  Qt/Y: n x (m+1); column m of Qt holds q, column m of Y holds w.
// b: right-hand side (already orthogonal to Q~); x: solution out.
SqmrResult sqmr_run(const Precond* K, const double* eps, const Domain& dom, double hop, double shift, const double* Qt,
                    const double* Y, int m, const double* Hinv, const double* b, double* x, double tol,
                    int maxit, Workspace& ws, cudaStream_t st) {
  const int64_t n = ws.n;
  double* Qtm = const_cast<double*>(Qt);
  double* Ym = const_cast<double*>(Y);
  double* q = Qtm + (int64_t)m * n;
  double* w = Ym + (int64_t)m * n;
  double *r = ws.vec[0], *t = ws.vec[1], *d = ws.vec[2], *sv = ws.vec[3], *rx = ws.vec[4];
  double* sc = ws.sc;
  double* dA = ws.small;          // m+1  (padded 32)
  double* dQw = ws.small + 64;    // m    (padded)
  double* dYr = ws.small + 128;   // m+1  (padded)
  double* nb2 = ws.small + 192;   // 1
  double* red = ws.small + 200;   // scratch outs
  SqmrResult res;
  launch_copy(r, b, n, st);
  launch_copy(rx, b, n, st);
  launch_fill(x, 0.0, n, st);
  launch_fill(d, 0.0, n, st);
  launch_fill(sv, 0.0, n, st);
  launch_dot(nb2, b, b, n, ws.rs, st);
  dom_allreduce(dom, nb2, 1, 0, st);
  k_sqmr_init_scalars<<<1, 1, 0, st>>>(sc, nb2);
  AJ_LAUNCHED();
  double hs[S_COUNT];
  AJ_CUDA(cudaMemcpyAsync(hs, sc, sizeof(hs), cudaMemcpyDeviceToHost, st));
  AJ_CUDA(cudaStreamSynchronize(st));
  const double nb = hs[S_NB];
  if (nb == 0.0) {
    res.iters = 0;
    res.relres = 0.0;
    return res;
  }
  const double sig_total = shift;  // operator A - (sigma + shift) I; caller folds sigma in
  auto precond_proj = [&](int step, cudaStream_t s2) {
    // w = K^{-1} r ; q = (w - Y Hinv Q~^T w) + beta q ; rho
    if (K)
      dom_precond(dom, K, w, r, s2);
    else
      launch_copy(w, r, n, s2);
    if (m > 0) {
      launch_multi_dot(dQw, Qt, m, n, w, n, ws.rs, s2);
      dom_allreduce(dom, dQw, m, 0, s2);
    }
    launch_multi_dot(dYr, Y, m + 1, n, r, n, ws.rs, s2);
    dom_allreduce(dom, dYr, m + 1, 0, s2);
    double* rho_out = sc + ((step & 1) ? S_RHO1 : S_RHO0);
    const double* rho_prev = sc + ((step & 1) ? S_RHO0 : S_RHO1);
    ProfScope ps(PROF_SQMR, 8.0 * n * (m + 3), s2);
    k_sqmr_F<<<sgrid(n), TB, 0, s2>>>(n, m, Y, w, q, dQw, dYr, Hinv, rho_prev, rho_out, step == 0 ? 1 : 0, sc);
    AJ_LAUNCHED();
  };
  precond_proj(0, st);
  int it = 0;
  double relres = 1.0;
  // One SQMR step (fused stencil + dots, the two update kernels, the residual
  // readback and the next projected preconditioning) is captured into a CUDA
  // graph per parity of the step (the rho slots alternate); the host launches one
  // graph and reads the pinned residual per step.
  auto body = [&](int p, cudaStream_t s2) {
    dom_spmv_dots(dom, t, q, eps, hop, sig_total, Qt, n, m + 1, ws.rs.buf(dA, 0), s2);
    const double* rho_cur = sc + ((p ^ 1) ? S_RHO1 : S_RHO0);
    {
      ProfScope ps(PROF_SQMR, 8.0 * n * (m + 4 + 10), s2);
      const int dist = dom.sharded() ? 1 : 0;
      k_sqmr_B<<<sgrid(n), TB, 0, s2>>>(n, m, Qt, t, r, dA, rho_cur, sc, ws.rs.buf(red, 1), dist);
      AJ_LAUNCHED();
      if (dist) {
        dom_allreduce(dom, red, 1, 0, s2);
        k_sqmr_B_scalars<<<1, 1, 0, s2>>>(m, red, dA, rho_cur, sc);
        AJ_LAUNCHED();
      }
      k_sqmr_C<<<sgrid(n), TB, 0, s2>>>(n, q, t, d, x, sv, rx, sc, ws.rs.buf(red + 8, 2));
      AJ_LAUNCHED();
      dom_allreduce(dom, sc + S_RX2, 1, 0, s2);
    }
    AJ_CUDA(cudaMemcpyAsync(ws.hpin, sc, S_COUNT * sizeof(double), cudaMemcpyDeviceToHost, s2));
  };
  const bool use_graph = ws.use_graphs && maxit >= 4 && !dom.sharded();  // callbacks are not captured
  cudaGraphExec_t gx[2] = {nullptr, nullptr};
  std::vector<ProfRec> gprof[2];
  int64_t gnodes[2] = {0, 0};
  auto cleanup_graphs = [&]() {
    for (int p = 0; p < 2; ++p) {
      if (gx[p]) cudaGraphExecDestroy(gx[p]);
      gx[p] = nullptr;
      prof_release(gprof[p]);
    }
  };
  try {
    if (use_graph) {
      for (int p = 0; p < 2; ++p) {
        const int64_t before = g_launches;
        // capture on the workspace's private stream (the caller's stream may be the
        // legacy default stream, which cannot be captured); launches go to `st`
        const cudaStream_t cs = ws.cap_stream;
        prof_set_capture_sink(&gprof[p]);
        AJ_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        body(p, cs);
        precond_proj(p == 0 ? 2 : 1, cs);  // any step of that parity (step > 0)
        cudaGraph_t g;
        const cudaError_t ec = cudaStreamEndCapture(cs, &g);
        prof_set_capture_sink(nullptr);
        AJ_CUDA(ec);
        AJ_CUDA(cudaGraphInstantiate(&gx[p], g, 0));
        AJ_CUDA(cudaGraphDestroy(g));
        gnodes[p] = g_launches - before;
        g_launches = before;
      }
    }
    for (it = 1; it <= maxit; ++it) {
      const int p = it & 1;
      if (use_graph) {
        AJ_CUDA(cudaGraphLaunch(gx[p], st));
        g_launches += gnodes[p];
        AJ_CUDA(cudaStreamSynchronize(st));
        prof_accumulate(gprof[p]);
      } else {
        body(p, st);
        AJ_CUDA(cudaStreamSynchronize(st));
      }
      const double* hs2 = ws.hpin;
      relres = sqrt(hs2[S_RX2]) / nb;
      if (hs2[S_BRK] != 0.0) {
        res.breakdown = true;
        break;
      }
      if (relres <= tol || it == maxit) break;
      if (!use_graph) precond_proj(it, st);
    }
  } catch (...) {
    prof_set_capture_sink(nullptr);
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(ws.cap_stream, &cst) == cudaSuccess && cst == cudaStreamCaptureStatusActive) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(ws.cap_stream, &g);
      if (g) cudaGraphDestroy(g);
    }
    cleanup_graphs();
    throw;
  }
  cleanup_graphs();
  res.iters = std::min(it, maxit);
  res.relres = relres;
  return res;
}

}  // namespace aj
