// Internal launch interfaces of the Anderson JD library.
#pragma once
#include <vector>

#include "aj_common.cuh"

namespace aj {

// Reduction scratch shared by the fused-reduction kernels of one solve.
// partials: kMaxPartials doubles; tickets: kMaxTickets zero-initialised counters.
constexpr int kMaxPartials = 148 * 64 * 80;
constexpr int kMaxTickets = 64;
struct RedScratch {
  double* partials = nullptr;
  unsigned* tickets = nullptr;
  void init(cudaStream_t s);
  void release(cudaStream_t s);
  RedBuf buf(double* out, int ticket = 0) const { return RedBuf{partials, tickets + ticket, out}; }
};

// --- per-host-thread resources, created once (aj_blas.cu): stream-capture stream and a
//     small pinned host buffer; creating/freeing them per solve costs host time in the path
cudaStream_t capture_stream();
double* pinned_scalars();  // 64 doubles

// --- lattice (aj_stencil.cu) ---
void launch_disorder(double* eps, int L, double W, uint64_t seed, cudaStream_t st);
void launch_spmv(double* y, const double* x, const double* eps, int L, double hop, double sig,
                 cudaStream_t st);
// y = (A - sig I) x and out[c] = <y, W_c>, c < nv (nv <= 10) via rb (fused reduction)
void launch_spmv_dots(double* y, const double* x, const double* eps, int L, double hop, double sig,
                      const double* W, int64_t ld, int nv, const RedBuf& rb, cudaStream_t st);
int spmv_grid_blocks(int L);
// z-slab shard: planes [z0, z0 + nz) of the disorder; SpMV with halo planes (x_ext: nz + 2 planes)
void launch_disorder_slab(double* eps, int L, int z0, int nz, double W, uint64_t seed, cudaStream_t st);
void launch_spmv_slab(double* y, const double* x_ext, const double* eps, int L, int nz, double hop, double sig,
                      cudaStream_t st);

// --- the lattice a process works on (aj_stencil.cu): the whole periodic lattice, or
//     one z-slab of a lattice sharded over comm->world processes (DESIGN.md sect. 6)
struct Domain {
  int L = 0, z0 = 0, nz = 0;
  int64_t n = 0;                  // local sites L^2 nz
  const aj_comm* comm = nullptr;  // null (or world == 1): this process owns the periodic lattice
  double* halo = nullptr;         // sharded: 2 L^2 receive planes [below | above] (device)
  double* rfull = nullptr;        // sharded, replicated preconditioner: whole-lattice r and z
  double* zfull = nullptr;        //   (L^3 each, jd_run allocates them)
  bool sharded() const { return comm != nullptr && comm->world > 1; }
  int64_t site0() const { return (int64_t)z0 * L * L; }
};
Domain domain_full(int L);
// sharded domain; allocates the halo planes (release with domain_release)
Domain domain_slab(int L, int z0, int nz, const aj_comm* comm, cudaStream_t st);
void domain_release(Domain& d, cudaStream_t st);
// in-place reduction over the ranks (op 0 sum, 1 max); no-op unless sharded
void dom_allreduce(const Domain& d, double* buf, int count, int op, cudaStream_t st);
// sharded: the whole lattice vector on every rank from the ranks' slabs (zero-padded
// all-reduce sum: every site has exactly one nonzero contribution, so the result is exact)
void dom_gather_full(const Domain& d, double* full, const double* part, cudaStream_t st);
// y = (A - sig I) x on the domain (halo exchange overlapped with the interior planes)
void dom_spmv(const Domain& d, double* y, const double* x, const double* eps, double hop, double sig,
              cudaStream_t st);
// ... and out[c] = <y, W_c> (c < nv) over all ranks, via rb (rb.out: >= 2 nv doubles when sharded)
void dom_spmv_dots(const Domain& d, double* y, const double* x, const double* eps, double hop, double sig,
                   const double* W, int64_t ld, int nv, const RedBuf& rb, cudaStream_t st);

// --- tall skinny (aj_blas.cu) ---
// out[0..m) = V^T x   (out device, padded to a multiple of 8)
void launch_multi_dot(double* out, const double* V, int m, int64_t ld, const double* x, int64_t n,
                      const RedScratch& rs, cudaStream_t st);
// y = beta*y + alpha * V c      (c device, m <= 64; y may not alias V)
void launch_gemv(double* y, double beta, double alpha, const double* V, int m, int64_t ld,
                 const double* c, int64_t n, cudaStream_t st);
// O[:, 0..q) = V[:, 0..p) S   (S device col-major p x q, lds = p; O may not alias V)
void launch_gemm_ts(double* O, int64_t ldo, const double* V, int p, int64_t ldv, const double* S,
                    int q, int64_t n, cudaStream_t st);
// out[0] = <x, y>
void launch_dot(double* out, const double* x, const double* y, int64_t n, const RedScratch& rs,
                cudaStream_t st);
// y = a*x + b*y
void launch_axpby(double* y, double a, const double* x, double b, int64_t n, cudaStream_t st);
// x *= 1/sqrt(*nrm2)  (nrm2 device scalar holding ||x||^2)
void launch_normalize(double* x, const double* nrm2, int64_t n, cudaStream_t st);
void launch_copy(double* y, const double* x, int64_t n, cudaStream_t st);
void launch_fill(double* y, double v, int64_t n, cudaStream_t st);

void prof_enable(bool on, unsigned mask = 0);
void prof_get(aj_prof* out);
struct ProfRec {
  cudaEvent_t a, b;
  int cat;
  double bytes;
};
void prof_set_capture_sink(std::vector<ProfRec>* sink);
void prof_accumulate(const std::vector<ProfRec>& recs);
void prof_release(std::vector<ProfRec>& recs);
bool prof_enabled();

}  // namespace aj
