// Symmetric Jacobi-Davidson driver (sect. 4.2, l.380-421; jdbsym
// l.1018-1024).  Host code orchestrating device kernels; the host only reads
// a handful of scalars per outer iteration (theta_1, ||r||) for control flow.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "aj_common.cuh"
#include "aj_kernels.cuh"
#include "aj_mlildl.cuh"
#include "aj_solver.cuh"

namespace aj {

// kernels defined in aj_solver.cu
__global__ void k_small_eig(int j, int ldm, const double* Min, double* theta, double* S);
__global__ void k_small_inv(int m, const double* H, int ldh, double* Hinv, int* status);
__global__ void k_set_mcol(double* M, int ldm, int j, const double* dots);
__global__ void k_set_mdiag(double* M, int ldm, int cnt, const double* theta, int off);
__global__ void k_resid(int64_t n, const double* Au, const double* u, const double* theta, double* r, RedBuf rb);
__global__ void k_start(int64_t n, uint64_t key, double* v, int64_t s0);
__global__ void k_absmax(int64_t n, const double* x, unsigned long long* out);
__global__ void k_negate_proj(int64_t n, double* b, const double* r, const double* Qt, int m, const double* c);

static int sg(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), (int64_t)num_sms() * 8)); }

template <typename T>
static void rd(T* h, const T* d, size_t cnt, cudaStream_t st) {
  AJ_CUDA(cudaMemcpyAsync(h, d, cnt * sizeof(T), cudaMemcpyDeviceToHost, st));
  AJ_CUDA(cudaStreamSynchronize(st));
}

JdResult jd_run(int k, double sigma, double tol, const double* eps, const Domain& dom_in, double hop,
                const aj_precond_params& pp, const aj_jd_params& jp, double* h_lambda, double* d_X,
                double* h_resid, aj_precond_info* pinfo, cudaStream_t st) {
  Domain dom = dom_in;  // + the whole-lattice buffers of the replicated sharded preconditioner
  const int L = dom.L;
  AJ_REQUIRE(L >= 3, AJ_ERR_ARG, "jd_solve: L must be >= 3");
  AJ_REQUIRE(k >= 1 && k <= 16, AJ_ERR_ARG, "jd_solve: 1 <= k <= 16");  // m = k + 1 <= 17 (k_small_inv)
  AJ_REQUIRE(jp.jmax <= 48 && jp.jmin >= 1 && jp.jmin < jp.jmax && jp.jmax >= 2, AJ_ERR_ARG,
             "jd_solve: need 1 <= jmin < jmax <= 48");
  AJ_REQUIRE(tol > 0.0 && h_lambda, AJ_ERR_ARG, "jd_solve: tol > 0 and h_lambda required");
  const int64_t n = dom.n;
  AJ_REQUIRE((int64_t)k + 2 <= n && jp.jmax < n, AJ_ERR_ARG, "jd_solve: lattice too small for k / jmax");
  JdResult R;
  cudaEvent_t e0, e1, e2;
  AJ_CUDA(cudaEventCreate(&e0));
  AJ_CUDA(cudaEventCreate(&e1));
  AJ_CUDA(cudaEventCreate(&e2));
  AJ_CUDA(cudaEventRecord(e0, st));

  // sharded (DESIGN.md sect. 6): shard_precond 0 = every rank factors the whole lattice
  // (eps all-gathered once) and applies it to the all-gathered residual -- the single-GPU
  // preconditioner; 1 = block Jacobi over the z-slabs (each rank its slab's diagonal block)
  Precond* K = nullptr;
  if (dom.sharded() && pp.shard_precond == 0) {
    const int64_t N = (int64_t)L * L * L;
    dom.rfull = dalloc<double>(N, st);
    dom.zfull = dalloc<double>(N, st);
    try {
      dom_gather_full(dom, dom.zfull, eps, st);  // the whole disorder (zfull as scratch)
      K = precond_create(dom.zfull, L, hop, sigma, pp, st);
    } catch (...) {
      dfree(dom.rfull, st);
      dfree(dom.zfull, st);
      throw;
    }
  } else {
    K = dom.sharded() ? precond_create_slab(eps, L, dom.z0, dom.nz, true, hop, sigma, pp, st)
                      : precond_create(eps, L, hop, sigma, pp, st);
  }
  if (pinfo) *pinfo = K->info;
  AJ_CUDA(cudaEventRecord(e1, st));
  Workspace ws(n, st);
  const int jmax = jp.jmax, jmin = jp.jmin;
  double* V = dalloc<double>(n * jmax, st);
  double* AV = dalloc<double>(n * jmax, st);
  double* Vt = dalloc<double>(n * jmax, st);
  double* AVt = dalloc<double>(n * jmax, st);
  // missed-eigenvalue safeguard (R15): after the k-th pair is locked, a Ritz value of the
  // remaining search space nearer to sigma than the farthest of the k locked pairs keeps JD going
  // for up to `extra` more pairs; the k nearest of all locked pairs are returned
  // (AJ_JD_EXTRA, testing: 0 = stop at the k-th pair as round 1 did)
  const char* exenv = getenv("AJ_JD_EXTRA");
  const int extra = std::max(0, std::min(exenv ? atoi(exenv) : 2, 17 - k));  // m = nq + 1 <= 17 (k_small_inv)
  double* QT = dalloc<double>(n * (k + extra + 2), st);
  double* Y = dalloc<double>(n * (k + extra + 2), st);
  double* u = dalloc<double>(n, st);
  double* Au = dalloc<double>(n, st);
  double* r = dalloc<double>(n, st);
  double* z = dalloc<double>(n, st);
  double* b = dalloc<double>(n, st);
  double* sm = dalloc<double>(16384, st);
  unsigned long long* amax = dalloc<unsigned long long>(1, st);
  int* hstat = dalloc<int>(1, st);
  double* M = sm;            // jmax x jmax (ld jmax)
  double* S = sm + 4096;     // j x j
  double* theta = sm + 8192; // j
  double* Hb = sm + 8256;    // m x mpad
  double* Hinv = sm + 8768;  // m x m
  double* cq = sm + 9088;
  double* cv = sm + 9216;
  double* mcol = sm + 9344;
  double* nrm = sm + 9472;
  double* rn2 = sm + 9480;
  std::vector<double> lam;
  int status = AJ_OK;
  auto cleanup = [&]() {
    for (void* p : {(void*)V, (void*)AV, (void*)Vt, (void*)AVt, (void*)QT, (void*)Y, (void*)u, (void*)Au, (void*)r,
                    (void*)z, (void*)b, (void*)sm, (void*)amax, (void*)hstat})
      dfree(p, st);
    ws.release(st);
    precond_destroy(K, st);
    dfree(dom.rfull, st);
    dfree(dom.zfull, st);
  };
  try {
    AJ_CUDA(cudaMemsetAsync(amax, 0, sizeof(unsigned long long), st));
    k_absmax<<<sg(n), 256, 0, st>>>(n, eps, amax);
    AJ_LAUNCHED();
    dom_allreduce(dom, reinterpret_cast<double*>(amax), 1, 1, st);  // max |eps| (bit patterns of doubles >= 0)
    unsigned long long hm;
    rd(&hm, amax, 1, st);
    double emax;
    memcpy(&emax, &hm, sizeof(double));
    const double normA = 6.0 * fabs(hop) + emax;  // ||A||_1
    const double tol_abs = tol * normA;
    uint64_t key = mix64(jp.seed ^ 0x4A44535441525431ull);
    k_start<<<sg(n), 256, 0, st>>>(n, key, z, dom.site0());
    AJ_LAUNCHED();
    int j = 0, nq = 0;
    double theta0 = 0.0, rnorm = 0.0;
    bool done = false;
    while (!done) {
      // ---- expand: z orthogonalised against [Q, V] (CGS2) and normalised
      double zn2 = 0.0;
      for (int attempt = 0;; ++attempt) {
        launch_dot(nrm, z, z, n, ws.rs, st);
        dom_allreduce(dom, nrm, 1, 0, st);
        double before;
        rd(&before, nrm, 1, st);
        for (int pass = 0; pass < 2; ++pass) {
          if (nq > 0) {
            launch_multi_dot(cq, QT, nq, n, z, n, ws.rs, st);
            dom_allreduce(dom, cq, nq, 0, st);
            launch_gemv(z, 1.0, -1.0, QT, nq, n, cq, n, st);
          }
          if (j > 0) {
            launch_multi_dot(cv, V, j, n, z, n, ws.rs, st);
            dom_allreduce(dom, cv, j, 0, st);
            launch_gemv(z, 1.0, -1.0, V, j, n, cv, n, st);
          }
        }
        launch_dot(nrm, z, z, n, ws.rs, st);
        dom_allreduce(dom, nrm, 1, 0, st);
        rd(&zn2, nrm, 1, st);
        if (std::isfinite(zn2) && zn2 > 1e-20 * std::max(before, 1e-300)) break;
        AJ_REQUIRE(attempt < 8, AJ_ERR_BREAKDOWN, "jd_solve: cannot extend the search space");
        key = mix64(key + 0x9E3779B97F4A7C15ull);
        k_start<<<sg(n), 256, 0, st>>>(n, key, z, dom.site0());  // correction in span: random restart vector
        AJ_LAUNCHED();
      }
      double* vj = V + (int64_t)j * n;
      launch_copy(vj, z, n, st);
      launch_normalize(vj, nrm, n, st);
      dom_spmv(dom, AV + (int64_t)j * n, vj, eps, hop, sigma, st);
      launch_multi_dot(mcol, V, j + 1, n, AV + (int64_t)j * n, n, ws.rs, st);
      dom_allreduce(dom, mcol, j + 1, 0, st);
      k_set_mcol<<<1, 64, 0, st>>>(M, jmax, j, mcol);
      AJ_LAUNCHED();
      ++j;
      // ---- Rayleigh-Ritz, locking and deflation
      bool need_new_start = false;
      for (;;) {
        k_small_eig<<<1, 256, 0, st>>>(j, jmax, M, theta, S);
        AJ_LAUNCHED();
        launch_gemv(u, 0.0, 1.0, V, j, n, S, n, st);
        launch_gemv(Au, 0.0, 1.0, AV, j, n, S, n, st);
        k_resid<<<sg(n), 256, 0, st>>>(n, Au, u, theta, r, ws.rs.buf(rn2));
        AJ_LAUNCHED();
        dom_allreduce(dom, rn2, 1, 0, st);
        double h2[2];
        AJ_CUDA(cudaMemcpyAsync(&h2[0], theta, sizeof(double), cudaMemcpyDeviceToHost, st));
        AJ_CUDA(cudaMemcpyAsync(&h2[1], rn2, sizeof(double), cudaMemcpyDeviceToHost, st));
        AJ_CUDA(cudaStreamSynchronize(st));
        theta0 = h2[0];
        rnorm = sqrt(std::max(h2[1], 0.0));
        if (rnorm > tol_abs) break;
        // lock the converged Ritz pair
        launch_copy(QT + (int64_t)nq * n, u, n, st);
        dom_precond(dom, K, Y + (int64_t)nq * n, u, st);
        lam.push_back(sigma + theta0);
        ++nq;
        if (jp.verbose)
          fprintf(stderr, "[jd] converged %d: lambda=%.15g |r|=%.3e outer=%d inner=%d\n", nq, sigma + theta0,
                  rnorm, R.outer, R.inner_total);
        if (nq >= k) {
          bool more = false;
          if (nq < k + extra && j >= 2) {
            std::vector<double> dist;
            for (double l : lam) dist.push_back(fabs(l - sigma));
            std::nth_element(dist.begin(), dist.begin() + (k - 1), dist.end());
            double th1;
            rd(&th1, theta + 1, 1, st);  // the nearest Ritz value of the space without the locked vector
            more = fabs(th1) < dist[k - 1];
            if (more && jp.verbose)
              fprintf(stderr, "[jd] %d pairs locked, but a Ritz value at distance %.6e < %.6e remains: continuing\n",
                      nq, fabs(th1), dist[k - 1]);
          }
          if (!more) {
            done = true;
            break;
          }
        }
        if (j == 1) {
          j = 0;
          need_new_start = true;
          break;
        }
        launch_gemm_ts(Vt, n, V, j, n, S + j, j - 1, n, st);
        launch_gemm_ts(AVt, n, AV, j, n, S + j, j - 1, n, st);
        std::swap(V, Vt);
        std::swap(AV, AVt);
        k_set_mdiag<<<1, 256, 0, st>>>(M, jmax, j - 1, theta, 1);
        AJ_LAUNCHED();
        --j;
      }
      if (done) break;
      if (need_new_start) {
        key = mix64(key + 0x9E3779B97F4A7C15ull);
        k_start<<<sg(n), 256, 0, st>>>(n, key, z, dom.site0());
        AJ_LAUNCHED();
        continue;
      }
      if (R.outer >= jp.max_outer) {
        status = AJ_ERR_NOCONV;
        break;
      }
      if (j >= jmax) {  // thick restart with the jmin Ritz vectors nearest sigma
        launch_gemm_ts(Vt, n, V, j, n, S, jmin, n, st);
        launch_gemm_ts(AVt, n, AV, j, n, S, jmin, n, st);
        std::swap(V, Vt);
        std::swap(AV, AVt);
        k_set_mdiag<<<1, 256, 0, st>>>(M, jmax, jmin, theta, 0);
        AJ_LAUNCHED();
        j = jmin;
        ++R.restarts;
      }
      // ---- correction equation with Q~ = [Q, u]
      const int m = nq + 1;
      const int mpad = (m + 7) & ~7;
      launch_copy(QT + (int64_t)nq * n, u, n, st);
      dom_precond(dom, K, Y + (int64_t)nq * n, u, st);
      for (int c = 0; c < m; ++c) launch_multi_dot(Hb + c * mpad, QT, m, n, Y + (int64_t)c * n, n, ws.rs, st);
      dom_allreduce(dom, Hb, m * mpad, 0, st);
      // Hinv = H^{-1} (H column c at Hb + c * mpad); a singular H (K^{-1} Q~ losing rank)
      // is reported, never silently replaced by the previous outer iteration's Hinv
      k_small_inv<<<1, 256, 0, st>>>(m, Hb, mpad, Hinv, hstat);
      AJ_LAUNCHED();
      {
        int hs = 0;
        rd(&hs, hstat, 1, st);
        AJ_REQUIRE(hs == 0, AJ_ERR_BREAKDOWN,
                   "jd_solve: H = Q~^T K^{-1} Q~ of the projected preconditioner is singular (outer " +
                       std::to_string(R.outer) + ")");
      }
      const double shift = (rnorm < jp.switch_tol * normA) ? theta0 : 0.0;
      launch_multi_dot(cq, QT, m, n, r, n, ws.rs, st);
      dom_allreduce(dom, cq, m, 0, st);
      k_negate_proj<<<sg(n), 256, 0, st>>>(n, b, r, QT, m, cq);
      AJ_LAUNCHED();
      SqmrResult sr = sqmr_run(K, eps, dom, hop, sigma + shift, QT, Y, m, Hinv, b, z, jp.inner_tol, jp.inner_max,
                               ws, st);
      R.inner_total += sr.iters;
      ++R.outer;
      if (jp.verbose && (R.outer % 10 == 0))
        fprintf(stderr, "[jd] outer %d j=%d theta=%.6e |r|=%.3e inner=%d relres=%.2e%s\n", R.outer, j, theta0,
                rnorm, sr.iters, sr.relres, sr.breakdown ? " (breakdown)" : "");
    }
    // results: eigenvalues, recomputed residuals, eigenvectors -- of more than k locked pairs
    // (safeguard above) the k nearest sigma, in the order they converged
    if (nq > k) {
      std::vector<int> idx(nq);
      for (int i = 0; i < nq; ++i) idx[i] = i;
      std::stable_sort(idx.begin(), idx.end(),
                       [&](int a, int c) { return fabs(lam[a] - sigma) < fabs(lam[c] - sigma); });
      idx.resize(k);
      std::sort(idx.begin(), idx.end());
      for (int i = 0; i < k; ++i) {
        if (idx[i] != i) launch_copy(QT + (int64_t)i * n, QT + (int64_t)idx[i] * n, n, st);
        lam[i] = lam[idx[i]];
      }
      lam.resize(k);
      nq = k;
    }
    R.converged = nq;
    for (int i = 0; i < nq; ++i) h_lambda[i] = lam[i];
    if (h_resid) {
      for (int i = 0; i < nq; ++i) {
        dom_spmv(dom, Au, QT + (int64_t)i * n, eps, hop, lam[i], st);
        launch_dot(nrm, Au, Au, n, ws.rs, st);
        dom_allreduce(dom, nrm, 1, 0, st);
        double v;
        rd(&v, nrm, 1, st);
        h_resid[i] = sqrt(v);
      }
    }
    if (d_X && nq > 0)
      AJ_CUDA(cudaMemcpyAsync(d_X, QT, sizeof(double) * n * nq, cudaMemcpyDeviceToDevice, st));
    AJ_CUDA(cudaEventRecord(e2, st));
    AJ_CUDA(cudaEventSynchronize(e2));
    float ms1 = 0, ms2 = 0;
    AJ_CUDA(cudaEventElapsedTime(&ms1, e0, e1));
    AJ_CUDA(cudaEventElapsedTime(&ms2, e1, e2));
    R.setup_ms = ms1;
    R.solve_ms = ms2;
  } catch (...) {
    cleanup();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    throw;
  }
  cleanup();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  R.status = status;
  return R;
}

}  // namespace aj
