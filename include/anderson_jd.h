/*
 * anderson_jd.h -- C ABI of the B200-native Anderson / Jacobi-Davidson hot path.
 *
 * Paper: O. Schenk, M. Bollhoefer, R. A. Roemer, "On large scale diagonalization
 * techniques for the Anderson model of localization" (arxiv math/0508111),
 * referenced below as PAPER.md with line numbers.
 *
 * Conventions (all entry points):
 *   - Plain pointers. A `d_` prefix means a device (HBM) pointer, `h_` a host
 *     pointer.  Caller owns every buffer it passes; the library owns only the
 *     opaque handles it returns (freed with the matching *_free call).
 *   - Vectors of the lattice are fp64, length n = L^3, site s = i + L*(j + L*k)
 *     (x fastest), periodic boundaries.
 *   - Blocks of vectors are column-major with leading dimension n.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Work is enqueued on it; functions that return host results synchronise it.
 *   - Return value: AJ_OK (0) or an AJ_ERR_* code; aj_last_error() returns a
 *     thread-local human-readable message for the last failure.  No entry point
 *     falls back to the CPU: without a usable sm_100a device they fail with
 *     AJ_ERR_CUDA.
 */
#ifndef ANDERSON_JD_H
#define ANDERSON_JD_H

#include <stdint.h>

#if defined(__GNUC__)
#define AJ_API __attribute__((visibility("default")))
#else
#define AJ_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define AJ_OK 0
#define AJ_ERR_ARG 1        /* invalid argument (sizes, NULL pointers, L < 3) */
#define AJ_ERR_CUDA 2       /* CUDA runtime / launch failure, no device      */
#define AJ_ERR_BREAKDOWN 3  /* preconditioner or Krylov breakdown            */
#define AJ_ERR_NOCONV 4     /* eigensolver hit max_outer before k pairs      */
#define AJ_ERR_CAPACITY 5   /* internal capacity exceeded (see message)      */

AJ_API const char* aj_last_error(void);
/* Library version string, e.g. "anderson_jd 0.1 sm_100a". */
AJ_API const char* aj_version(void);

/* ------------------------------------------------------------------------- *
 * anderson_build -- the disorder potential eps of Eq. (eigenequation)
 * (PAPER.md l.182-193): eps_s ~ U[-W/2, W/2), s in [0, L^3).
 * Generator (R3): SplitMix64 counter stream keyed by `seed`,
 *   h_s = mix64(seed + (s+1)*0x9E3779B97F4A7C15), u_s = (h_s >> 11) * 2^-53,
 *   eps_s = (u_s - 0.5) * W        (bit-exact, order independent).
 * d_eps: device, n doubles, written.  Errors: AJ_ERR_ARG if L < 3 or W < 0.
 * ------------------------------------------------------------------------- */
AJ_API int anderson_build(double* d_eps, int32_t L, double W, uint64_t seed, void* stream);

/* ------------------------------------------------------------------------- *
 * spmv -- y = (A - sigma I) x, matrix free (Eq.
 * (eigenequation) l.182-186): (A x)_s = hop * sum_{6 periodic nbrs} x_nb + eps_s x_s.
 * d_y, d_x, d_eps: device, n doubles; d_y must not alias d_x.
 * ------------------------------------------------------------------------- */
AJ_API int spmv(double* d_y, const double* d_x, const double* d_eps, int32_t L, double hop,
         double sigma, void* stream);

/* ------------------------------------------------------------------------- *
 * z-slab shard of the lattice (north star: "the lattice shards naturally into
 * z-slabs ... with one-plane halo exchange"; DESIGN.md sect. 6, row (e)).
 *
 * anderson_build_slab -- eps of the planes z0 <= k < z0 + nz (sites
 * s = z0 L^2 ... (z0 + nz) L^2 - 1 of anderson_build, same generator, so the
 * shard equals the slice of the full lattice bit for bit).
 * d_eps: device, nz L^2 doubles, written.  Errors: AJ_ERR_ARG unless
 * L >= 3, z0 >= 0, nz >= 1, z0 + nz <= L, W >= 0.
 * ------------------------------------------------------------------------- */
AJ_API int anderson_build_slab(double* d_eps, int32_t L, int32_t z0, int32_t nz, double W, uint64_t seed,
                               void* stream);

/* ------------------------------------------------------------------------- *
 * spmv_slab -- y = (A - sigma I) x on a slab of nz planes (same operator as
 * spmv), periodic in x and y.  d_x_ext: device,
 * (nz + 2) L^2 doubles: plane 0 = the plane below the slab (global z0 - 1,
 * periodic), planes 1..nz = the slab, plane nz + 1 = the plane above; the
 * caller fills the two halo planes (binding: slab.halo_exchange over
 * torch.distributed).  d_eps: nz L^2 (anderson_build_slab); d_y: nz L^2,
 * must not alias d_x_ext.  Errors: AJ_ERR_ARG on null pointers, L < 3,
 * nz < 1 or nz > L.
 * ------------------------------------------------------------------------- */
AJ_API int spmv_slab(double* d_y, const double* d_x_ext, const double* d_eps, int32_t L, int32_t nz,
                     double hop, double sigma, void* stream);

/* ------------------------------------------------------------------------- *
 * Symmetric multilevel incomplete LDL^T preconditioner K ~ A - sigma I
 * (sect. 7, l.790-973), independent-set levels (DESIGN.md sect. 3.3):
 * level 0 = red sites of the bipartite lattice, deeper levels = maximal
 * independent sets of 1x1 / matched 2x2 pivots, inverse-based pivot bound
 * ||L^{-1}||_inf <= kappa (l.884-897), dropping |l| < tau_drop (l.909-911),
 * recursion on the Schur complement (l.917-945), dense coarse inverse.
 * ------------------------------------------------------------------------- */
typedef struct {
  double kappa;          /* inverse bound, paper default 5    */
  double tau_drop;       /* drop tolerance for L and S; < 0: auto = the paper's
                            eps/kappa with eps = 1/sqrt(N), N = L^3
                            (R12)           */
  double tau_strong;     /* strong-coupling threshold of the independent sets;
                            < 0: auto, min(0.05, 40 tau_drop) with compensation,
                            else 10 * tau_drop                                    */
  int32_t n_coarse_max;  /* stop recursing at this size, invert densely; default 2048 */
  int32_t max_levels;    /* level cap (<= 1023)                                  */
  double stall_frac;     /* stop when a level eliminates < stall_frac * n        */
  int32_t dense_cap;     /* largest coarse system accepted (else BREAKDOWN); default 40960 */
  int32_t cand_cap;      /* reserved (>= 64)                                     */
  int32_t factor_fp32;   /* 1: store L / L^T values in fp32 (fp64 accumulation)  */
  int32_t compensate;    /* 1: first-order treatment of the dropped weak pivot-pivot
                            couplings, B^{-1} ~ B_d^{-1} - B_d^{-1} E B_d^{-1} (R17) */
  double tau_virtual;    /* only couplings |a^_uv| >= tau_virtual are compensated;
                            < 0: auto, 5 tau_drop (L <= 50) .. 10 tau_drop
                            (L >= 100), linear in between                        */
  double tau_inv;        /* inverse-based (aggressive) dropping a posteriori,
                            PAPER.md l.947-973: drop l_cf when
                            |l_cf| <= tau_inv / (nu_c #col_f), nu_c ~ ||L~^{-1} e_c||
                            (R18); 0 = off; needs factor_fp32 = 0      */
  int32_t shard_precond; /* jd_solve_sharded only (DESIGN.md sect. 6):
                            0 = replicated: every rank factors the WHOLE lattice
                            (eps all-gathered once) and applies it to the
                            all-gathered residual -- the single-GPU preconditioner,
                            identical iteration counts; 1 = block Jacobi over the
                            slabs (precond_setup_slab; measured to stall the inner
                            solves, kept for comparison)                           */
} aj_precond_params;

typedef struct {
  int32_t levels;         /* number of sparse levels                              */
  int32_t coarse_n;       /* size of the dense coarse system                      */
  int64_t nnz_L;          /* stored entries of all L factors                      */
  int64_t nnz_A;          /* 7 n                                                  */
  int32_t level_n[1024];  /* size of each level                                   */
  int32_t level_nF[1024]; /* pivots eliminated at each level                      */
  int32_t level_pairs[1024]; /* 2x2 pivots at each level                          */
  int64_t level_nnzS[1024];  /* nnz of the Schur complement produced by each level */
  double setup_ms;        /* device time of precond_setup                         */
  double tau_drop;        /* resolved drop tolerance                              */
  double tau_strong;      /* resolved strong-coupling threshold                   */
  double tau_virtual;     /* resolved compensation threshold (0 if compensate=0)  */
  int64_t nnz_V;          /* virtual 2x2 blocks over all levels (R17)             */
  int64_t setup_products; /* Schur products l_cx a_c'x over all levels (work model) */
  double setup_bytes;     /* compulsory setup traffic model, bytes (DESIGN.md sect. 4) */
  double tau_inv;         /* resolved inverse-based dropping threshold (0 = off)   */
  int64_t nnz_L_dropped_inv; /* L entries removed by the inverse-based dropping      */
} aj_precond_info;

AJ_API void aj_precond_default_params(aj_precond_params* p);

/* handle: out, opaque; d_eps device n doubles (read during setup only). */
AJ_API int precond_setup(void** handle, const double* d_eps, int32_t L, double hop, double sigma,
                  const aj_precond_params* params, void* stream);
/* z = K^{-1} r.  d_z, d_r: device n doubles, may not alias. Symmetric linear operator. */
AJ_API int precond_apply(void* handle, double* d_z, const double* d_r, void* stream);
AJ_API int precond_info(void* handle, aj_precond_info* info);
/* Releases the handle.  The device is synchronised first (applies enqueued on any
 * stream finish before the factor's memory returns to the pool), then the buffers
 * are freed stream-ordered on `stream` and `stream` is synchronised.  NULL = no-op. */
AJ_API int precond_free(void* handle, void* stream);

/* ------------------------------------------------------------------------- *
 * sqmr_solve -- simplified QMR for
 * (A - sigma I) x = b with the preconditioner `handle` (NULL = identity).
 * Stops when ||b - (A - sigma I) x|| <= tol ||b|| (recursive QMR residual,
 * PAPER.md l.1094-1095) or after maxit steps.  d_x: out (zero start), d_b: in.
 * h_iters / h_relres: out (host).  Returns AJ_ERR_BREAKDOWN on a Lanczos
 * breakdown (q^T A q = 0 or rho = 0).
 * ------------------------------------------------------------------------- */
AJ_API int sqmr_solve(void* handle, double* d_x, const double* d_b, const double* d_eps, int32_t L,
               double hop, double sigma, double tol, int32_t maxit, int32_t* h_iters,
               double* h_relres, void* stream);

/* ------------------------------------------------------------------------- *
 * Tall-skinny building blocks of the JD subspace work (DESIGN.md row 4).
 * d_V: n x m column-major (ld = n).
 * multi_dot:   h_out[m] = V^T x                       (fp64, deterministic order)
 * ortho_cgs2:  x <- (I - V V^T)^2 x / ||.||, h_norm = norm before normalising
 *              (V assumed orthonormal; 2-pass classical Gram-Schmidt).
 * ------------------------------------------------------------------------- */
AJ_API int multi_dot(double* h_out, const double* d_V, int32_t m, const double* d_x, int64_t n,
              void* stream);
AJ_API int ortho_cgs2(double* d_x, const double* d_V, int32_t m, int64_t n, double* h_norm,
               void* stream);

/* ------------------------------------------------------------------------- *
 * jd_solve -- the k eigenpairs of A nearest sigma by symmetric Jacobi-Davidson
 * (sect. 4.2, l.380-421): Ritz extraction on V^T A V, correction
 * equation (I-Q~Q~^T)(A-theta I)(I-Q~Q~^T) z = -r, Q~ = [Q, u], solved by SQMR
 * with the projected preconditioner (I - Y H^{-1} Q~^T) K^{-1}, Y = K^{-1} Q~,
 * H = Q~^T Y (the block form of (I - u w^T / w^T u) K^{-1}, l.414-416), K the
 * multilevel ILDL at sigma; thick restart; deflation of converged pairs.
 * Converged when ||A x - lambda x||_2 <= tol * ||A||_1, ||A||_1 = 6|hop| + max|eps|.
 *
 * JD locks the Ritz pair nearest sigma as it converges, which is usually, not
 * provably, the order of distance from sigma; after the k-th pair a Ritz value
 * of the remaining search space nearer to sigma than the farthest locked pair
 * keeps the iteration going for up to 2 more pairs, and the k nearest of all
 * locked pairs are returned (R15; a heuristic, not a certificate).
 *
 * d_eps: device n doubles.  h_lambda: host k (out, in the order the pairs converged).
 * d_X: device n*k (out, orthonormal eigenvectors, may be NULL).
 * h_resid: host k (out, ||A x - lambda x||_2 recomputed after convergence).
 * Returns AJ_ERR_NOCONV (with the converged prefix filled) if max_outer is hit.
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t jmin, jmax;    /* search space after restart / maximum                 */
  int32_t max_outer;     /* outer iteration cap                                  */
  int32_t inner_max;     /* SQMR steps per correction equation                   */
  double inner_tol;      /* relative SQMR tolerance for the correction equation  */
  double switch_tol;     /* use theta (not sigma) as shift once ||r|| < this*||A|| */
  uint64_t seed;         /* start vector stream key                              */
  int32_t verbose;       /* 1: per-outer log on stderr                           */
} aj_jd_params;

typedef struct {
  int32_t outer, inner_total, converged, restarts;
  double setup_ms, solve_ms, total_ms;
  aj_precond_info precond;
} aj_jd_stats;

AJ_API void aj_jd_default_params(aj_jd_params* p);

AJ_API int jd_solve(int32_t k, double sigma, double tol, const double* d_eps, int32_t L, double hop,
             const aj_precond_params* pparams, const aj_jd_params* jparams, double* h_lambda,
             double* d_X, double* h_resid, aj_jd_stats* stats, void* stream);

/* Same, end to end from HOST buffers: h_eps (n doubles) is copied in, the
 * eigenvectors are copied back into h_X (n*k doubles, may be NULL). */
AJ_API int jd_solve_host(int32_t k, double sigma, double tol, const double* h_eps, int32_t L, double hop,
                  const aj_precond_params* pparams, const aj_jd_params* jparams, double* h_lambda,
                  double* h_X, double* h_resid, aj_jd_stats* stats, void* stream);

/* ------------------------------------------------------------------------- *
 * z-slab sharded solve over `world` processes, one GPU each (row (e); north star:
 * "The lattice shards naturally into z-slabs across 1/2/4/8 GPUs ... with one-plane
 * halo exchange and dot-product allreduce via NCCL"; the paper's motivation is
 * N = 10^6..10^8).  Rank r owns the planes
 * z0 <= k < z0 + nz of the periodic L^3 lattice; its vectors are the nz L^2 sites of
 * those planes (same site order as the full lattice, offset z0 L^2).  Every
 * cross-rank step goes through an aj_comm:
 *   allreduce   in-place sum (op 0) or max (op 1) of `count` doubles over the ranks,
 *               ordered on `stream` (the fused dot products of SQMR/JD, <= 64 values);
 *   halo_start  send this slab's first plane to rank-1 and its last plane to rank+1,
 *               receive rank-1's last plane into d_recv_lo and rank+1's first plane into
 *               d_recv_hi (periodic in z), ordered after prior work on `stream`;
 *   halo_wait   orders `stream` after the receives (the interior planes of the SpMV
 *               run in between).
 * Callbacks return 0 on success.  The library provides an NCCL implementation
 * (aj_comm_nccl_create); the binding provides a torch.distributed one (gloo on CPU
 * tests).  A NULL comm or world == 1 means one process owns the periodic lattice.
 * ------------------------------------------------------------------------- */
typedef struct aj_comm {
  int32_t world;
  int32_t rank;
  void* ctx;
  int (*allreduce)(void* ctx, double* d_buf, int32_t count, int32_t op, void* stream);
  int (*halo_start)(void* ctx, const double* d_send_lo, const double* d_send_hi, double* d_recv_lo,
                    double* d_recv_hi, int64_t count, void* stream);
  int (*halo_wait)(void* ctx, void* stream);
} aj_comm;

/* NCCL communicator of the sharded solve.  libnccl: path of the libnccl.so.2 to
 * dlopen (NULL = the default search; pass the one torch.distributed loaded).
 * aj_nccl_unique_id writes the 128-byte ncclUniqueId (rank 0 creates it, the
 * caller broadcasts it); aj_comm_nccl_create: every rank, collective. */
AJ_API int aj_nccl_unique_id(const char* libnccl, void* h_id);
AJ_API int aj_comm_nccl_create(aj_comm** comm, const char* libnccl, const void* h_id, int32_t world, int32_t rank);
AJ_API int aj_comm_nccl_free(aj_comm* comm);

/* y = (A - sigma I) x on this rank's slab (the operator of spmv), the two halo
 * planes exchanged through `comm` (overlapped with the interior planes).
 * d_y, d_x, d_eps: device, nz L^2 doubles (d_eps from anderson_build_slab).
 * Errors: AJ_ERR_ARG on bad sizes (nz >= 2 when comm->world > 1), AJ_ERR_CUDA if a
 * callback fails. */
AJ_API int spmv_sharded(double* d_y, const double* d_x, const double* d_eps, int32_t L, int32_t z0, int32_t nz,
                        double hop, double sigma, const aj_comm* comm, void* stream);

/* The multilevel ILDL of this rank's diagonal block of A - sigma I: the slab with
 * periodic x, y and (for world > 1) open z faces -- block Jacobi over the slabs at the
 * finest level, every level inside the slab (DESIGN.md sect. 6).  Level 0 is the red
 * set of the GLOBAL lattice parity.  world == 1 reproduces precond_setup. */
AJ_API int precond_setup_slab(void** handle, const double* d_eps, int32_t L, int32_t z0, int32_t nz, int32_t world,
                              double hop, double sigma, const aj_precond_params* params, void* stream);

/* jd_solve on the sharded lattice: same arguments and results as jd_solve, with
 * d_eps (nz L^2, this rank's slab) and d_X (nz L^2 x k, this rank's part of the
 * eigenvectors, may be NULL); h_lambda / h_resid are identical on every rank.  The
 * preconditioner follows pparams->shard_precond: 0 (default) the whole-lattice multilevel
 * ILDL on every rank, applied to the residual all-gathered through comm->allreduce
 * (zero-padded sum of the slabs, exact), 1 precond_setup_slab (block Jacobi over slabs).
 * Collective: every rank calls it with the same k, sigma, tol, params. */
AJ_API int jd_solve_sharded(int32_t k, double sigma, double tol, const double* d_eps, int32_t L, int32_t z0,
                            int32_t nz, double hop, const aj_precond_params* pparams, const aj_jd_params* jparams,
                            double* h_lambda, double* d_X, double* h_resid, aj_jd_stats* stats, const aj_comm* comm,
                            void* stream);

/* Number of kernel launches issued by this thread since the last reset
 * (bench accounting of "gpu_launches"). */
AJ_API int64_t aj_launch_count(int32_t reset);

/* ------------------------------------------------------------------------- *
 * Live per-phase device timing (CUDA events recorded on the launching stream
 * around each phase while enabled; used by bench.py for the roofline).
 * Categories: 0 stencil SpMV (incl. fused dots), 1 preconditioner apply,
 * 2 preconditioner setup, 3 SQMR vector updates, 4 JD subspace kernels.
 * bytes = algorithmic HBM bytes of the recorded calls (DESIGN.md sect. 4).
 * aj_prof_enable(1) resets and starts recording every category, (0) stops;
 * aj_prof_enable(0x80000000 | mask) records only the categories of `mask`
 * (bit c = category c).  aj_prof_get synchronises the device and returns the
 * totals of this thread.
 * ------------------------------------------------------------------------- */
#define AJ_PROF_CATS 8
typedef struct {
  double ms[AJ_PROF_CATS];
  double bytes[AJ_PROF_CATS];
  int64_t calls[AJ_PROF_CATS];
} aj_prof;
AJ_API int aj_prof_enable(int32_t on);
AJ_API int aj_prof_get(aj_prof* out);

#ifdef __cplusplus
}
#endif
#endif /* ANDERSON_JD_H */
