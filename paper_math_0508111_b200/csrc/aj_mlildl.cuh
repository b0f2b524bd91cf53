// Multilevel ILDL data structures (see aj_mlildl.cu).
#pragma once
#include <vector>

#include "aj_common.cuh"

namespace aj {

struct Csr {
  int n = 0;
  int64_t nnz = 0;
  int64_t* ptr = nullptr;  // n+1
  int32_t* col = nullptr;  // nnz, sorted per row
  double* val = nullptr;   // nnz
  void release(cudaStream_t st);
};

struct Level {
  int n = 0, nF = 0, nC = 0, npairs = 0, rounds = 0;
  int schur_tier_rows[6] = {0, 0, 0, 0, 0, 0};  // coarse rows per Schur tier (W1, W2, P4, C8, C16, G)
  int schur_ovf_rows = 0;                     // C16 rows retried in G
  int64_t nnzFC = 0;                          // coarse entries of the pivot rows (Schur work per row = their FC lists)
  int64_t nnzA = 0;                           // entries of the level matrix
  int64_t schur_products = 0;                 // Schur products l_cx a_c'x computed at this level
  int64_t ndrop_inv = 0;                      // L entries removed by the inverse-based dropping
  int64_t nnzL = 0, nnzLT = 0, nnzS = 0;
  double* D = nullptr;          // n   symmetric scaling of this level
  int32_t* cmap = nullptr;      // n   coarse index of C nodes, -1 for F
  int32_t* cidx = nullptr;      // nC  level index of coarse node c'
  int32_t* fidx = nullptr;      // nF  level index of pivot node f'
  int32_t* fmap = nullptr;      // n   pivot index of F nodes, -1 for C
  int32_t* partner = nullptr;   // n   2x2 partner of F nodes, else -1
  double* b11 = nullptr;        // n   B^{-1}[f,f]   (F nodes)
  double* b12 = nullptr;        // n   B^{-1}[f,g]   (F nodes of a pair)
  int64_t* Lptr = nullptr;      // nC+1
  int32_t* Lcol = nullptr;      // F node: level index (level 0), pivot index f' (levels >= 1, gathers rF)
  void* Lval = nullptr;         // L_cf * D_f  (float if f32, else double)
  int64_t* LTptr = nullptr;     // nF+1, rows in F order
  int32_t* LTcol = nullptr;     // coarse index
  void* LTval = nullptr;        // L_cf        (float if f32, else double)
  bool f32 = false;             // factor values stored in fp32 (accumulation stays fp64)
  int64_t* Vptr = nullptr;      // n+1 virtual couplings of pivot singles (reading R17)
  int32_t* Vcol = nullptr;      // level index of the coupled pivot
  double* Vval = nullptr;       // b'_uv
  int64_t nnzV = 0;
  int gf = 1, gb = 1;           // threads per row of the forward / backward kernels
  int nst_f = 0, nst_b = 0;     // shared-memory stages of the staged kernels (0: register prefetch)
  int32_t* fpart = nullptr;     // nfpart+1 row boundaries of the persistent ring forward kernel (large levels)
  int32_t* bpart = nullptr;     // nbpart+1, backward
  int nfpart = 0, nbpart = 0;
  double* yv = nullptr;         // nF  backward right-hand side B~^{-1}(D r)_F, written by the ring forward kernel
  double* dF = nullptr;         // nF  D on the pivots, compact
  double* rF = nullptr;         // nF: r on the pivots, compact (levels >= 1; written by the previous forward step)
  double* r = nullptr;          // level workspace (levels >= 1)
  double* z = nullptr;
  void release(cudaStream_t st);
};

struct Precond {
  int L = 0, n0 = 0;
  int64_t nnzA0 = 0;  // entries of the level-0 matrix
  aj_precond_params P{};
  std::vector<Level> lv;
  int nc = 0;
  double* G = nullptr;   // nc x nc dense symmetric inverse of the coarse Schur complement
  double* rc = nullptr;
  double* zc = nullptr;
  aj_precond_info info{};
  int64_t bytes_per_apply = 0;
  cudaGraphExec_t exec = nullptr;  // levels >= 1 + coarse, captured once
  int64_t graph_nodes = 0;
};

// one level's Schur complement + L rows (aj_schur.cu); outputs per coarse row a run in
// temp buffers (tmp_* for S, ltmp_* for L, row_off/lrow_off = run starts), allocated
// here, freed by the caller
struct SchurIn {
  int n, nC, nF;
  const int64_t* ptr;
  const int32_t* col;
  const double* ah;  // scaled level matrix
  const int8_t* inF;
  const int32_t *partner, *cmap, *cidx, *fmap, *fidx;
  const double *b11, *b12;
  const int64_t* Vptr;  // virtual couplings (reading R17), may be null
  const int32_t* Vcol;
  const double* Vval;
  double tau;
  int64_t cap_hint;  // expected S temp entries
};
struct SchurOut {
  int64_t *row_cnt = nullptr, *row_off = nullptr, *lrow_cnt = nullptr, *lrow_off = nullptr;
  int32_t *tmp_col = nullptr, *ltmp_col = nullptr;
  double *tmp_val = nullptr, *ltmp_val = nullptr;
  int64_t nnz_tmp = 0, nnz_ltmp = 0, nnz_fc = 0;
  int64_t products = 0;  // table updates (Schur products l_cx a_c'x), phases C + D
  int tier_rows[6] = {0, 0, 0, 0, 0, 0};  // W1, W2, P4, C8, C16, G
  int ovf_rows = 0;
};
void schur_level(const SchurIn& in, SchurOut& out, cudaStream_t st);
// S = U + strict(U)^T from the upper-triangle runs of schur_level (S allocated here)
void schur_mirror(int nC, const SchurOut& so, Csr& S, cudaStream_t st);

aj_precond_params resolve_params(const aj_precond_params& in, int L);
Precond* precond_create(const double* eps, int L, double hop, double sigma, const aj_precond_params& P,
                        cudaStream_t st);
// the diagonal block of planes [z0, z0 + nz) (open_z: couplings across the slab faces
// dropped -- block Jacobi over z-slabs, DESIGN.md sect. 6); eps: the slab's nz L^2 values
Precond* precond_create_slab(const double* eps, int L, int z0, int nz, bool open_z, double hop, double sigma,
                             const aj_precond_params& P, cudaStream_t st);
void precond_destroy(Precond* K, cudaStream_t st);
void precond_run(const Precond* K, double* z, const double* r, cudaStream_t st);
int64_t precond_bytes_per_apply(const Precond* K);

}  // namespace aj
