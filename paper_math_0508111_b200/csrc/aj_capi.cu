// extern "C" boundary of the library (declared in include/anderson_jd.h).
// Argument checking + translation of aj::Error into return codes.
#include <cstring>
#include <string>

#include "aj_common.cuh"
#include "aj_kernels.cuh"
#include "aj_mlildl.cuh"
#include "aj_solver.cuh"

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

template <typename F>
int guarded(const char* name, F&& f) {
  try {
    int dev_count = 0;
    cudaError_t e = cudaGetDeviceCount(&dev_count);
    if (e != cudaSuccess || dev_count == 0)
      return fail(AJ_ERR_CUDA, std::string(name) + ": no CUDA device available (no CPU fallback exists)");
    return f();
  } catch (const aj::Error& e) {
    return fail(e.code, std::string(name) + ": " + e.what());
  } catch (const std::exception& e) {
    return fail(AJ_ERR_CUDA, std::string(name) + ": " + e.what());
  }
}

inline cudaStream_t S(void* s) { return (cudaStream_t)s; }
}  // namespace

extern "C" {

const char* aj_last_error(void) { return g_err.c_str(); }

const char* aj_version(void) { return "anderson_jd 0.1 sm_100a"; }

int64_t aj_launch_count(int32_t reset) {
  const int64_t v = aj::g_launches;
  if (reset) aj::g_launches = 0;
  return v;
}

int aj_prof_enable(int32_t on) {
  return guarded("aj_prof_enable", [&] {
    // on: 1 = all categories, or a category bit mask (bit c = category c) with bit 31 set
    const unsigned mask = (on & 0x80000000) ? (unsigned)on & 0x7fffffffu : 0u;
    aj::prof_enable(on != 0, mask);
    return AJ_OK;
  });
}

int aj_prof_get(aj_prof* out) {
  if (!out) return fail(AJ_ERR_ARG, "aj_prof_get: NULL");
  return guarded("aj_prof_get", [&] {
    aj::prof_get(out);
    return AJ_OK;
  });
}

int anderson_build(double* d_eps, int32_t L, double W, uint64_t seed, void* stream) {
  if (!d_eps || L < 3 || !(W >= 0.0)) return fail(AJ_ERR_ARG, "anderson_build: need d_eps, L >= 3, W >= 0");
  return guarded("anderson_build", [&] {
    aj::launch_disorder(d_eps, L, W, seed, S(stream));
    return AJ_OK;
  });
}

int spmv(double* d_y, const double* d_x, const double* d_eps, int32_t L, double hop, double sigma,
         void* stream) {
  if (!d_y || !d_x || !d_eps || L < 3 || d_y == d_x) return fail(AJ_ERR_ARG, "spmv: bad arguments");
  return guarded("spmv", [&] {
    aj::launch_spmv(d_y, d_x, d_eps, L, hop, sigma, S(stream));
    return AJ_OK;
  });
}

int anderson_build_slab(double* d_eps, int32_t L, int32_t z0, int32_t nz, double W, uint64_t seed, void* stream) {
  if (!d_eps || L < 3 || z0 < 0 || nz < 1 || z0 + nz > L || !(W >= 0.0))
    return fail(AJ_ERR_ARG, "anderson_build_slab: need d_eps, L >= 3, 0 <= z0, 1 <= nz, z0 + nz <= L, W >= 0");
  return guarded("anderson_build_slab", [&] {
    aj::launch_disorder_slab(d_eps, L, z0, nz, W, seed, S(stream));
    return AJ_OK;
  });
}

int spmv_slab(double* d_y, const double* d_x_ext, const double* d_eps, int32_t L, int32_t nz, double hop,
              double sigma, void* stream) {
  if (!d_y || !d_x_ext || !d_eps || L < 3 || nz < 1 || nz > L) return fail(AJ_ERR_ARG, "spmv_slab: bad arguments");
  return guarded("spmv_slab", [&] {
    aj::launch_spmv_slab(d_y, d_x_ext, d_eps, L, nz, hop, sigma, S(stream));
    return AJ_OK;
  });
}

void aj_precond_default_params(aj_precond_params* p) {
  if (!p) return;
  p->kappa = 5.0;
  p->tau_drop = -1.0;      // auto: 1/(kappa sqrt(L^3)), the paper's eps/kappa (R12)
  p->tau_strong = -1.0;    // auto: min(0.05, 40 tau_drop) (R17), 10 tau_drop without compensation
  p->n_coarse_max = 2048;  // 6-7 % less time per SQMR step than 1024 at equal setup time (DESIGN.md sect. 4)
  p->max_levels = 1023;
  p->stall_frac = 0.005;
  p->dense_cap = 40960;    // W=12 stalls on a coarse block of 12 686 (L=100) / 34 648 (L=130): 13 GB inverse + 27 GB workspace
  p->cand_cap = 2048;
  p->factor_fp32 = 0;      // DESIGN.md R16: fp32 storage is opt-in (hurts at large L)
  p->compensate = 1;       // DESIGN.md R17
  p->tau_virtual = -1.0;   // auto: 5..10 tau_drop for L = 50..100 (R17)
  p->tau_inv = 0.0;        // inverse-based dropping off (R18: measured, see sect. 7a)
  p->shard_precond = 0;    // sharded solve: replicated whole-lattice preconditioner (DESIGN.md sect. 6)
}

int precond_setup(void** handle, const double* d_eps, int32_t L, double hop, double sigma,
                  const aj_precond_params* params, void* stream) {
  if (!handle || !d_eps || L < 3) return fail(AJ_ERR_ARG, "precond_setup: bad arguments");
  return guarded("precond_setup", [&] {
    aj_precond_params p;
    if (params)
      p = *params;
    else
      aj_precond_default_params(&p);
    *handle = aj::precond_create(d_eps, L, hop, sigma, p, S(stream));
    return AJ_OK;
  });
}

int precond_apply(void* handle, double* d_z, const double* d_r, void* stream) {
  if (!handle || !d_z || !d_r || d_z == d_r) return fail(AJ_ERR_ARG, "precond_apply: bad arguments");
  return guarded("precond_apply", [&] {
    aj::precond_run((aj::Precond*)handle, d_z, d_r, S(stream));
    return AJ_OK;
  });
}

int precond_info(void* handle, aj_precond_info* info) {
  if (!handle || !info) return fail(AJ_ERR_ARG, "precond_info: bad arguments");
  *info = ((aj::Precond*)handle)->info;
  return AJ_OK;
}

int precond_free(void* handle, void* stream) {
  if (!handle) return AJ_OK;
  return guarded("precond_free", [&] {
    // the frees are stream-ordered on `stream` (after every apply enqueued on it);
    // the device-wide synchronisation first also orders them after applies the
    // caller enqueued on other streams, so no pool block is reused under a kernel
    AJ_CUDA(cudaDeviceSynchronize());
    cudaStream_t st = S(stream);
    aj::precond_destroy((aj::Precond*)handle, st);
    AJ_CUDA(cudaStreamSynchronize(st));
    return AJ_OK;
  });
}

int sqmr_solve(void* handle, double* d_x, const double* d_b, const double* d_eps, int32_t L, double hop,
               double sigma, double tol, int32_t maxit, int32_t* h_iters, double* h_relres, void* stream) {
  if (!d_x || !d_b || !d_eps || L < 3 || maxit < 1) return fail(AJ_ERR_ARG, "sqmr_solve: bad arguments");
  return guarded("sqmr_solve", [&] {
    const int64_t n = (int64_t)L * L * L;
    cudaStream_t st = S(stream);
    aj::Workspace ws(n, st);
    double* Qt = aj::dalloc<double>(n, st);  // holds q (m = 0)
    double* Y = aj::dalloc<double>(n, st);   // holds w
    aj::SqmrResult r;
    try {
      r = aj::sqmr_run((aj::Precond*)handle, d_eps, aj::domain_full(L), hop, sigma, Qt, Y, 0, nullptr, d_b, d_x, tol,
                       maxit, ws, st);
    } catch (...) {
      aj::dfree(Qt, st);
      aj::dfree(Y, st);
      ws.release(st);
      throw;
    }
    aj::dfree(Qt, st);
    aj::dfree(Y, st);
    ws.release(st);
    AJ_CUDA(cudaStreamSynchronize(st));
    if (h_iters) *h_iters = r.iters;
    if (h_relres) *h_relres = r.relres;
    if (r.breakdown) return fail(AJ_ERR_BREAKDOWN, "sqmr_solve: Lanczos breakdown");
    return AJ_OK;
  });
}

int multi_dot(double* h_out, const double* d_V, int32_t m, const double* d_x, int64_t n, void* stream) {
  if (!h_out || !d_V || !d_x || m < 1 || m > 512 || n < 1) return fail(AJ_ERR_ARG, "multi_dot: bad arguments");
  return guarded("multi_dot", [&] {
    cudaStream_t st = S(stream);
    aj::RedScratch rs;
    rs.init(st);
    const int pad = (m + 7) & ~7;
    double* out = aj::dalloc<double>(pad, st);
    aj::launch_multi_dot(out, d_V, m, n, d_x, n, rs, st);
    AJ_CUDA(cudaMemcpyAsync(h_out, out, m * sizeof(double), cudaMemcpyDeviceToHost, st));
    AJ_CUDA(cudaStreamSynchronize(st));
    aj::dfree(out, st);
    rs.release(st);
    return AJ_OK;
  });
}

int ortho_cgs2(double* d_x, const double* d_V, int32_t m, int64_t n, double* h_norm, void* stream) {
  if (!d_x || (!d_V && m > 0) || m < 0 || m > 64 || n < 1) return fail(AJ_ERR_ARG, "ortho_cgs2: bad arguments");
  return guarded("ortho_cgs2", [&] {
    cudaStream_t st = S(stream);
    aj::RedScratch rs;
    rs.init(st);
    double* c = aj::dalloc<double>(72, st);
    double* nrm = aj::dalloc<double>(8, st);
    for (int pass = 0; pass < 2 && m > 0; ++pass) {
      aj::launch_multi_dot(c, d_V, m, n, d_x, n, rs, st);
      aj::launch_gemv(d_x, 1.0, -1.0, d_V, m, n, c, n, st);
    }
    aj::launch_dot(nrm, d_x, d_x, n, rs, st);
    double h;
    AJ_CUDA(cudaMemcpyAsync(&h, nrm, sizeof(double), cudaMemcpyDeviceToHost, st));
    AJ_CUDA(cudaStreamSynchronize(st));
    if (h > 0.0) aj::launch_normalize(d_x, nrm, n, st);
    if (h_norm) *h_norm = sqrt(h);
    AJ_CUDA(cudaStreamSynchronize(st));
    aj::dfree(c, st);
    aj::dfree(nrm, st);
    rs.release(st);
    return AJ_OK;
  });
}

void aj_jd_default_params(aj_jd_params* p) {
  if (!p) return;
  p->jmin = 10;
  p->jmax = 25;
  p->max_outer = 2000;
  p->inner_max = 150;   // DESIGN.md R15: measured vs 60 at L=50..250, W=16.5 and 21
  p->inner_tol = 3e-3;
  p->switch_tol = 1e-3;
  p->seed = 7;
  p->verbose = 0;
}

static int jd_common(int32_t k, double sigma, double tol, const double* d_eps, const aj::Domain& dom, double hop,
                     const aj_precond_params* pparams, const aj_jd_params* jparams, double* h_lambda, double* d_X,
                     double* h_resid, aj_jd_stats* stats, cudaStream_t st) {
  aj_precond_params pp;
  aj_jd_params jp;
  if (pparams)
    pp = *pparams;
  else
    aj_precond_default_params(&pp);
  if (jparams)
    jp = *jparams;
  else
    aj_jd_default_params(&jp);
  aj_precond_info pinfo;
  memset(&pinfo, 0, sizeof(pinfo));
  aj::JdResult R = aj::jd_run(k, sigma, tol, d_eps, dom, hop, pp, jp, h_lambda, d_X, h_resid, &pinfo, st);
  if (stats) {
    stats->outer = R.outer;
    stats->inner_total = R.inner_total;
    stats->converged = R.converged;
    stats->restarts = R.restarts;
    stats->setup_ms = R.setup_ms;
    stats->solve_ms = R.solve_ms;
    stats->total_ms = R.setup_ms + R.solve_ms;
    stats->precond = pinfo;
  }
  if (R.status == AJ_ERR_NOCONV)
    return fail(AJ_ERR_NOCONV, "jd_solve: max_outer reached with " + std::to_string(R.converged) + " of " +
                                   std::to_string(k) + " pairs converged");
  return R.status;
}

int jd_solve(int32_t k, double sigma, double tol, const double* d_eps, int32_t L, double hop,
             const aj_precond_params* pparams, const aj_jd_params* jparams, double* h_lambda, double* d_X,
             double* h_resid, aj_jd_stats* stats, void* stream) {
  if (!d_eps || !h_lambda || L < 3 || k < 1) return fail(AJ_ERR_ARG, "jd_solve: bad arguments");
  return guarded("jd_solve", [&] {
    return jd_common(k, sigma, tol, d_eps, aj::domain_full(L), hop, pparams, jparams, h_lambda, d_X, h_resid, stats,
                     S(stream));
  });
}

int jd_solve_host(int32_t k, double sigma, double tol, const double* h_eps, int32_t L, double hop,
                  const aj_precond_params* pparams, const aj_jd_params* jparams, double* h_lambda, double* h_X,
                  double* h_resid, aj_jd_stats* stats, void* stream) {
  if (!h_eps || !h_lambda || L < 3 || k < 1) return fail(AJ_ERR_ARG, "jd_solve_host: bad arguments");
  return guarded("jd_solve_host", [&] {
    cudaStream_t st = S(stream);
    const int64_t n = (int64_t)L * L * L;
    double* d_eps = aj::dalloc<double>(n, st);
    double* d_X = h_X ? aj::dalloc<double>(n * k, st) : nullptr;
    int rc;
    try {
      AJ_CUDA(cudaMemcpyAsync(d_eps, h_eps, n * sizeof(double), cudaMemcpyHostToDevice, st));
      rc = jd_common(k, sigma, tol, d_eps, aj::domain_full(L), hop, pparams, jparams, h_lambda, d_X, h_resid, stats,
                     st);
      if (h_X && (rc == AJ_OK || rc == AJ_ERR_NOCONV))
        AJ_CUDA(cudaMemcpyAsync(h_X, d_X, n * k * sizeof(double), cudaMemcpyDeviceToHost, st));
      AJ_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
      aj::dfree(d_eps, st);
      aj::dfree(d_X, st);
      throw;
    }
    aj::dfree(d_eps, st);
    aj::dfree(d_X, st);
    return rc;
  });
}

// ---- z-slab sharded solve (include/anderson_jd.h, DESIGN.md sect. 6) ----------------
static bool slab_ok(int32_t L, int32_t z0, int32_t nz, const aj_comm* comm) {
  if (L < 3 || z0 < 0 || nz < 1 || z0 + nz > L) return false;
  if (comm && (comm->world < 1 || comm->rank < 0 || comm->rank >= comm->world)) return false;
  if (comm && comm->world > 1 && (!comm->allreduce || !comm->halo_start || !comm->halo_wait || nz >= L)) return false;
  if (!(comm && comm->world > 1) && (z0 != 0 || nz != L)) return false;  // one process owns the whole lattice
  return true;
}

int spmv_sharded(double* d_y, const double* d_x, const double* d_eps, int32_t L, int32_t z0, int32_t nz, double hop,
                 double sigma, const aj_comm* comm, void* stream) {
  if (!d_y || !d_x || !d_eps || d_y == d_x || !slab_ok(L, z0, nz, comm))
    return fail(AJ_ERR_ARG, "spmv_sharded: bad arguments");
  return guarded("spmv_sharded", [&] {
    cudaStream_t st = S(stream);
    aj::Domain dom = aj::domain_slab(L, z0, nz, comm, st);
    try {
      aj::dom_spmv(dom, d_y, d_x, d_eps, hop, sigma, st);
    } catch (...) {
      aj::domain_release(dom, st);
      throw;
    }
    aj::domain_release(dom, st);
    return AJ_OK;
  });
}

int precond_setup_slab(void** handle, const double* d_eps, int32_t L, int32_t z0, int32_t nz, int32_t world,
                       double hop, double sigma, const aj_precond_params* params, void* stream) {
  if (!handle || !d_eps || L < 3 || z0 < 0 || nz < 1 || z0 + nz > L || world < 1 || (world == 1 && nz != L) ||
      (world > 1 && nz >= L))
    return fail(AJ_ERR_ARG, "precond_setup_slab: bad arguments");
  return guarded("precond_setup_slab", [&] {
    aj_precond_params p;
    if (params)
      p = *params;
    else
      aj_precond_default_params(&p);
    *handle = aj::precond_create_slab(d_eps, L, z0, nz, world > 1, hop, sigma, p, S(stream));
    return AJ_OK;
  });
}

int jd_solve_sharded(int32_t k, double sigma, double tol, const double* d_eps, int32_t L, int32_t z0, int32_t nz,
                     double hop, const aj_precond_params* pparams, const aj_jd_params* jparams, double* h_lambda,
                     double* d_X, double* h_resid, aj_jd_stats* stats, const aj_comm* comm, void* stream) {
  if (!d_eps || !h_lambda || k < 1 || !slab_ok(L, z0, nz, comm)) return fail(AJ_ERR_ARG, "jd_solve_sharded: bad arguments");
  return guarded("jd_solve_sharded", [&] {
    cudaStream_t st = S(stream);
    aj::Domain dom = aj::domain_slab(L, z0, nz, comm, st);
    int rc;
    try {
      rc = jd_common(k, sigma, tol, d_eps, dom, hop, pparams, jparams, h_lambda, d_X, h_resid, stats, st);
    } catch (...) {
      aj::domain_release(dom, st);
      throw;
    }
    aj::domain_release(dom, st);
    return rc;
  });
}

}  // extern "C"
