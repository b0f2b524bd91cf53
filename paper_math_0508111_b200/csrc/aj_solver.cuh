// SQMR / JD internal interfaces.
#pragma once
#include "aj_common.cuh"
#include "aj_kernels.cuh"
#include "aj_mlildl.cuh"

namespace aj {

struct Workspace {
  int64_t n;
  RedScratch rs;
  double* sc = nullptr;     // SQMR scalars
  double* small = nullptr;  // dot outputs / small matrices
  double* vec[9] = {};      // n-vectors: r, t, d, s, rx + spare
  double* hpin = nullptr;   // pinned host copy of the SQMR scalars
  bool use_graphs = false;  // SQMR step as a CUDA graph (opt-in: AJ_SQMR_GRAPH=1)
  cudaStream_t cap_stream = nullptr;  // private stream used only for graph capture
  Workspace(int64_t n_, cudaStream_t st);
  void release(cudaStream_t st);
};

struct SqmrResult {
  int iters = 0;
  double relres = 1.0;
  bool breakdown = false;
};

// z = K^{-1} r on this rank's part: the local apply, or (sharded, replicated
// preconditioner: dom.rfull set) all-gather r, apply the whole-lattice K, keep the slab
void dom_precond(const Domain& dom, const Precond* K, double* z, const double* r, cudaStream_t st);

SqmrResult sqmr_run(const Precond* K, const double* eps, const Domain& dom, double hop, double shift, const double* Qt,
                    const double* Y, int m, const double* Hinv, const double* b, double* x, double tol,
                    int maxit, Workspace& ws, cudaStream_t st);

struct JdResult {
  int status = AJ_OK;
  int converged = 0, outer = 0, inner_total = 0, restarts = 0;
  double setup_ms = 0, solve_ms = 0;
};

JdResult jd_run(int k, double sigma, double tol, const double* eps, const Domain& dom, double hop,
                const aj_precond_params& pp, const aj_jd_params& jp, double* h_lambda, double* d_X,
                double* h_resid, aj_precond_info* pinfo, cudaStream_t st);

}  // namespace aj
