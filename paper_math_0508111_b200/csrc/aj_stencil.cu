// Anderson lattice: disorder generation and the matrix-free fp64 stencil SpMV.
//
// PAPER.md sect. 3, Eq. (eigenequation) l.182-186 and l.282-285 ("the
// underlying matrix-vector multiplication ... only the diagonal needs to be
// stored").  HBM-bound: 24 algorithmic bytes per site (read eps, x; write y).
//
// Kernel design (DESIGN.md sect. 4.1): a 2.5-D sweep.  A CTA owns a
// 32 (x) by 8 (y) column tile and marches along z over a chunk of planes,
// keeping x(k-1), x(k), x(k+1) of its own column in registers; the four
// in-plane neighbours are re-read through L1 (they are the neighbouring
// lanes'/warps' loads of the same plane), so every x element leaves HBM once.
#include "aj_common.cuh"
#include "aj_kernels.cuh"

#include <cstring>
#include <string>

namespace aj {

__global__ void k_disorder(double* __restrict__ eps, int64_t n, double W, uint64_t seed) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    double u = uniform01(seed, (uint64_t)s);
    eps[s] = (u - 0.5) * W;  // one subtraction (exact) then one multiply: bit-exact
  }
}

void launch_disorder(double* eps, int L, double W, uint64_t seed, cudaStream_t st) {
  int64_t n = (int64_t)L * L * L;
  int grid = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)num_sms() * 16);
  k_disorder<<<grid, 256, 0, st>>>(eps, n, W, seed);
  AJ_LAUNCHED();
}

constexpr int SBX = 32, SBY = 8;

// y = (A - sig I) x; optional fused dot products  dots[c] += sum_s y_s * W_c[s]
// for the NV vectors W_c = Wv + c*ld (column block), reduced with the
// last-block epilogue into rb.out[0..NV).
template <int NV>
__global__ void __launch_bounds__(SBX* SBY)
    k_spmv(double* __restrict__ y, const double* __restrict__ x, const double* __restrict__ eps,
           int L, double hop, double sig, int kchunk, const double* __restrict__ Wv, int64_t ld,
           RedBuf rb) {
  const int i = blockIdx.x * SBX + threadIdx.x;
  const int j = blockIdx.y * SBY + threadIdx.y;
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(k0 + kchunk, L);
  double acc[NV > 0 ? NV : 1];
#pragma unroll
  for (int c = 0; c < (NV > 0 ? NV : 1); ++c) acc[c] = 0.0;
  if (i < L && j < L && k0 < L) {
    const int64_t P = (int64_t)L * L;
    const int im = (i == 0) ? L - 1 : i - 1, ip = (i == L - 1) ? 0 : i + 1;
    const int jm = (j == 0) ? L - 1 : j - 1, jp = (j == L - 1) ? 0 : j + 1;
    const int64_t r0 = (int64_t)j * L, rm = (int64_t)jm * L, rp = (int64_t)jp * L;
    const int km = (k0 == 0) ? L - 1 : k0 - 1;
    double xm = __ldg(&x[km * P + r0 + i]);
    double xc = __ldg(&x[k0 * P + r0 + i]);
    for (int k = k0; k < k1; ++k) {
      const int kp = (k == L - 1) ? 0 : k + 1;
      const double xp = __ldg(&x[kp * P + r0 + i]);
      const int64_t b = k * P;
      const double s = (__ldg(&x[b + r0 + im]) + __ldg(&x[b + r0 + ip])) +
                       (__ldg(&x[b + rm + i]) + __ldg(&x[b + rp + i])) + (xm + xp);
      const double v = hop * s + (__ldg(&eps[b + r0 + i]) - sig) * xc;
      y[b + r0 + i] = v;
      if constexpr (NV > 0) {
#pragma unroll
        for (int c = 0; c < NV; ++c) acc[c] += v * __ldg(&Wv[c * ld + b + r0 + i]);
      }
      xm = xc;
      xc = xp;
    }
  }
  if constexpr (NV > 0) block_reduce_finalize<NV, SBX * SBY>(acc, rb, blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z),
                                                       gridDim.x * gridDim.y * gridDim.z);
}

// Even-L variant: every lane owns two consecutive x-sites (16-byte loads and
// stores of x, eps and y); the x-neighbours i-1 / i+2 come from the adjacent
// lanes by warp shuffle, only tile-edge lanes touch memory for them.  z-march of
// the column tile (bx, by) over planes [k0, k1), dots accumulated into acc.
template <int NV>
__device__ __forceinline__ void spmv2_march(double* __restrict__ y, const double* __restrict__ x,
                                            const double* __restrict__ eps, int L, double hop, double sig, int bx,
                                            int by, int k0, int k1, const double* __restrict__ Wv, int64_t ld,
                                            double (&acc)[NV > 0 ? NV : 1]) {
  const int lane = threadIdx.x;
  const int i = (bx * SBX + lane) * 2;
  const int j = by * SBY + threadIdx.y;
  const bool act = (i < L) && (j < L);
  const int64_t P = (int64_t)L * L;
  const int jj = act ? j : 0, ii = act ? i : 0;
  const int jm = (jj == 0) ? L - 1 : jj - 1, jp = (jj == L - 1) ? 0 : jj + 1;
  const int64_t r0 = (int64_t)jj * L, rm = (int64_t)jm * L, rp = (int64_t)jp * L;
  const int im = (ii == 0) ? L - 1 : ii - 1, ip2 = (ii + 2 >= L) ? ii + 2 - L : ii + 2;
  const bool edge_l = (lane == 0), edge_r = (lane == SBX - 1) || (ii + 2 >= L);
  if (k0 < k1) {
    // register queue of planes k-1, k, k+1 and the diagonal of plane k; the
    // loads of plane k+2 and of eps(k+1) are issued one iteration ahead so two
    // independent HBM streams are in flight per thread
    const int km = (k0 == 0) ? L - 1 : k0 - 1;
    const int kp0 = (k0 == L - 1) ? 0 : k0 + 1;
    const double2 z2 = make_double2(0.0, 0.0);
    double2 xm = z2, xc = z2, xp = z2, ec = z2;
    if (act) {
      xm = __ldg(reinterpret_cast<const double2*>(&x[km * P + r0 + ii]));
      xc = __ldg(reinterpret_cast<const double2*>(&x[(int64_t)k0 * P + r0 + ii]));
      xp = __ldg(reinterpret_cast<const double2*>(&x[(int64_t)kp0 * P + r0 + ii]));
      ec = __ldg(reinterpret_cast<const double2*>(&eps[(int64_t)k0 * P + r0 + ii]));
    }
    for (int k = k0; k < k1; ++k) {
      const int64_t b = (int64_t)k * P;
      double2 xpp = z2, en = z2, xr0 = z2, xr1 = z2;
      double left = 0.0, right = 0.0;
      if (act) {
        if (k + 1 < k1) {
          const int kpp = (k + 2 >= L) ? k + 2 - L : k + 2;
          xpp = __ldg(reinterpret_cast<const double2*>(&x[(int64_t)kpp * P + r0 + ii]));
          en = __ldg(reinterpret_cast<const double2*>(&eps[b + P + r0 + ii]));
        }
        xr0 = __ldg(reinterpret_cast<const double2*>(&x[b + rm + ii]));
        xr1 = __ldg(reinterpret_cast<const double2*>(&x[b + rp + ii]));
        if (edge_l) left = __ldg(&x[b + r0 + im]);
        if (edge_r) right = __ldg(&x[b + r0 + ip2]);
      }
      const double sl = __shfl_up_sync(0xffffffffu, xc.y, 1);
      const double sr = __shfl_down_sync(0xffffffffu, xc.x, 1);
      if (!edge_l) left = sl;
      if (!edge_r) right = sr;
      double2 v;
      const double s0 = (left + xc.y) + (xr0.x + xr1.x) + (xm.x + xp.x);
      const double s1 = (xc.x + right) + (xr0.y + xr1.y) + (xm.y + xp.y);
      v.x = hop * s0 + (ec.x - sig) * xc.x;
      v.y = hop * s1 + (ec.y - sig) * xc.y;
      if (act) {
        __stcs(reinterpret_cast<double2*>(&y[b + r0 + ii]), v);
        if constexpr (NV > 0) {
#pragma unroll
          for (int c = 0; c < NV; ++c) {
            const double2 w = __ldg(reinterpret_cast<const double2*>(&Wv[c * ld + b + r0 + ii]));
            acc[c] += v.x * w.x + v.y * w.y;
          }
        }
      }
      xm = xc;
      xc = xp;
      xp = xpp;
      ec = en;
    }
  }
}

template <int NV>
__global__ void __launch_bounds__(SBX* SBY, 4)
    k_spmv2(double* __restrict__ y, const double* __restrict__ x, const double* __restrict__ eps, int L,
            double hop, double sig, int kchunk, const double* __restrict__ Wv, int64_t ld, RedBuf rb) {
  double acc[NV > 0 ? NV : 1];
#pragma unroll
  for (int c = 0; c < (NV > 0 ? NV : 1); ++c) acc[c] = 0.0;
  const int k0 = blockIdx.z * kchunk;
  spmv2_march<NV>(y, x, eps, L, hop, sig, blockIdx.x, blockIdx.y, k0, min(k0 + kchunk, L), Wv, ld, acc);
  if constexpr (NV > 0)
    block_reduce_finalize<NV, SBX * SBY>(acc, rb, blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z),
                                         gridDim.x * gridDim.y * gridDim.z);
}

// Balanced persistent launch of the same z-march: exactly one wave (4 CTAs per SM), the
// tx * ty * L (column tile, plane) units split into equal contiguous ranges in tile-major
// order, so every CTA marches ~units/grid planes of one or two column tiles (no partial
// last wave; the z-halo re-read is 2 planes per range).
template <int NV>
__global__ void __launch_bounds__(SBX* SBY, 4)
    k_spmv2_bal(double* __restrict__ y, const double* __restrict__ x, const double* __restrict__ eps, int L,
                double hop, double sig, int tx, int64_t units, const double* __restrict__ Wv, int64_t ld,
                RedBuf rb) {
  double acc[NV > 0 ? NV : 1];
#pragma unroll
  for (int c = 0; c < (NV > 0 ? NV : 1); ++c) acc[c] = 0.0;
  int64_t u = units * blockIdx.x / gridDim.x;
  const int64_t u1 = units * (blockIdx.x + 1) / gridDim.x;
  while (u < u1) {
    const int t = (int)(u / L), k0 = (int)(u % L);
    const int k1 = (int)(k0 + (u1 - u) < (int64_t)L ? k0 + (u1 - u) : (int64_t)L);
    spmv2_march<NV>(y, x, eps, L, hop, sig, t % tx, t / tx, k0, k1, Wv, ld, acc);
    u += k1 - k0;
  }
  if constexpr (NV > 0) block_reduce_finalize<NV, SBX * SBY>(acc, rb, blockIdx.x, gridDim.x);
}

// ---- TMA-staged variant (even L, 64 <= L <= 512; DESIGN.md sect. 4) ------------------
// A CTA owns a band of ny <= TY_MAX full x-rows [j0, j0 + ny) and a chunk of planes
// [k0, k1).  The bulk-copy engine (cp.async.bulk, completion on an mbarrier) streams, for
// every plane k0-1 .. k1, the band plus its two halo rows (j0-1, j0+ny, periodic) into a
// ring of NS shared-memory stages; the threads only wait on the stage barriers and compute
// from shared memory: x-neighbours (periodic wrap inside the row), y-neighbours (the rows
// above / below in the stage), z-neighbours (the previous / next stage).  eps, the fused
// dot vectors and y go through registers (16-byte loads / streaming stores).  CTAs with
// the same plane chunk and adjacent bands are adjacent in launch order, so the halo rows a
// band re-reads are its neighbour's rows of the same plane, mostly L2 hits.  Same
// summation order as k_spmv2 (x-, y-, z-neighbour pairs), so the result is bit-identical.
constexpr int TMA_NS = 5;       // stages: planes k-1, k, k+1 in use, two in flight
constexpr int TMA_THREADS = 256;
constexpr int TMA_SMEM = 110 * 1024;  // two CTAs per SM
constexpr int TMA_MP = 6;             // pairs per thread and plane: (ty+2) L <= TMA_SMEM / (8 NS)

struct TmaGeom {
  int T, Z, kchunk, ty_max;
};

template <int NV>
__global__ void __launch_bounds__(TMA_THREADS, 2)
    k_spmv_tma(double* __restrict__ y, const double* __restrict__ x, const double* __restrict__ eps, int L,
               double hop, double sig, TmaGeom g, const double* __restrict__ Wv, int64_t ld, RedBuf rb) {
  extern __shared__ __align__(128) double sx[];
  __shared__ __align__(8) uint64_t bar[TMA_NS];
  const int t = blockIdx.x % g.T, zc = blockIdx.x / g.T;
  const int j0 = (int)((int64_t)t * L / g.T), j1 = (int)((int64_t)(t + 1) * L / g.T), ny = j1 - j0;
  const int k0 = zc * g.kchunk, k1 = min(L, k0 + g.kchunk);
  const int64_t P = (int64_t)L * L;
  const int rowlen = L;                       // doubles per row
  const int stage_elems = (g.ty_max + 2) * L;  // doubles per stage
  const int nq = (k1 - k0) + 2;                // planes k0-1 .. k1
  const uint32_t row_bytes = (uint32_t)L * 8u;
  double acc[NV > 0 ? NV : 1];
#pragma unroll
  for (int c = 0; c < (NV > 0 ? NV : 1); ++c) acc[c] = 0.0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TMA_NS; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int q) {  // plane k0 - 1 + q into stage q % NS (thread 0)
    const int kk = (k0 - 1 + q + L) % L;
    double* dst = sx + (size_t)(q % TMA_NS) * stage_elems;
    uint64_t* b = &bar[q % TMA_NS];
    const double* pl = x + (int64_t)kk * P;
    mbar_expect_tx(b, (uint32_t)(ny + 2) * row_bytes);
    bulk_g2s(dst, pl + (int64_t)((j0 - 1 + L) % L) * L, row_bytes, b);
    bulk_g2s(dst + rowlen, pl + (int64_t)j0 * L, (uint32_t)ny * row_bytes, b);
    bulk_g2s(dst + (size_t)(ny + 1) * rowlen, pl + (int64_t)(j1 % L) * L, row_bytes, b);
  };
  if (k0 < k1) {
    if (threadIdx.x == 0)
      for (int q = 0; q < min(TMA_NS, nq); ++q) issue(q);
    const int half = L >> 1;
    const int npairs = ny * half;  // <= TMA_MP * TMA_THREADS (stage budget, tma_geom)
    // per-thread pair offsets, the same on every plane: centre / left / right in the stage,
    // global offset inside the band (no integer division in the plane loop)
    int oc[TMA_MP], ol[TMA_MP], orr[TMA_MP], og[TMA_MP];
#pragma unroll
    for (int m = 0; m < TMA_MP; ++m) {
      const int p = threadIdx.x + m * TMA_THREADS;
      const int r = p < npairs ? p / half : 0;
      const int i = p < npairs ? (p - r * half) * 2 : 0;
      oc[m] = (r + 1) * rowlen + i;
      ol[m] = (r + 1) * rowlen + (i == 0 ? L - 1 : i - 1);
      orr[m] = (r + 1) * rowlen + (i + 2 == L ? 0 : i + 2);
      og[m] = p < npairs ? r * L + i : -1;
    }
    // eps of the next plane is loaded one plane ahead into registers (the stage holds x only)
    double2 en[TMA_MP];
    auto load_eps = [&](int k) {
      const double* eb = eps + (int64_t)k * P + (int64_t)j0 * L;
#pragma unroll
      for (int m = 0; m < TMA_MP; ++m)
        if (og[m] >= 0) en[m] = __ldcs(reinterpret_cast<const double2*>(eb + og[m]));
    };
    load_eps(k0);
    for (int k = k0; k < k1; ++k) {
      const int q = k - k0 + 1;
      double2 ec[TMA_MP];
#pragma unroll
      for (int m = 0; m < TMA_MP; ++m) ec[m] = en[m];
      if (k + 1 < k1) load_eps(k + 1);
      if (k == k0) {
        mbar_wait(&bar[0], 0);
        mbar_wait(&bar[1 % TMA_NS], 0);
      }
      mbar_wait(&bar[(q + 1) % TMA_NS], (uint32_t)(((q + 1) / TMA_NS) & 1));
      const double* sm = sx + (size_t)((q - 1) % TMA_NS) * stage_elems;
      const double* sc = sx + (size_t)(q % TMA_NS) * stage_elems;
      const double* sp = sx + (size_t)((q + 1) % TMA_NS) * stage_elems;
      const int64_t base = (int64_t)k * P + (int64_t)j0 * L;
#pragma unroll
      for (int m = 0; m < TMA_MP; ++m) {
        if (og[m] < 0) break;
        const int o = oc[m];
        const double2 xc = *reinterpret_cast<const double2*>(sc + o);
        const double left = sc[ol[m]];
        const double right = sc[orr[m]];
        const double2 xr0 = *reinterpret_cast<const double2*>(sc + o - rowlen);
        const double2 xr1 = *reinterpret_cast<const double2*>(sc + o + rowlen);
        const double2 xm = *reinterpret_cast<const double2*>(sm + o);
        const double2 xp = *reinterpret_cast<const double2*>(sp + o);
        const int64_t gi = base + og[m];
        const double s0 = (left + xc.y) + (xr0.x + xr1.x) + (xm.x + xp.x);
        const double s1 = (xc.x + right) + (xr0.y + xr1.y) + (xm.y + xp.y);
        double2 v;
        v.x = hop * s0 + (ec[m].x - sig) * xc.x;
        v.y = hop * s1 + (ec[m].y - sig) * xc.y;
        __stcs(reinterpret_cast<double2*>(y + gi), v);
        if constexpr (NV > 0) {
#pragma unroll
          for (int c = 0; c < NV; ++c) {
            const double2 w = __ldg(reinterpret_cast<const double2*>(&Wv[c * ld + gi]));
            acc[c] += v.x * w.x + v.y * w.y;
          }
        }
      }
      __syncthreads();  // every thread is done with stage (q - 1) % NS
      if (threadIdx.x == 0 && q - 1 + TMA_NS < nq) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(q - 1 + TMA_NS);
      }
    }
  }
  if constexpr (NV > 0) block_reduce_finalize<NV, TMA_THREADS>(acc, rb, blockIdx.x, gridDim.x);
}

// Kernel choice for the full-lattice SpMV (measured at L=100..250, DESIGN.md sect. 4):
// the TMA-staged kernel for the plain product (nv = 0) at even 128 <= L <= 512, the tiled
// register z-march otherwise (with fused dots the extra dot-vector streams keep enough
// loads in flight: 5.0 TB/s at L=250).  AJ_SPMV_PATH=tma|bal|grid (testing) forces one
// (tma/bal need even L, tma 64 <= L <= 512).
enum SpmvPath { SP_GRID1, SP_GRID2, SP_BAL, SP_TMA };

static TmaGeom tma_geom(int L) {
  TmaGeom g{0, 0, 0, 0};
  if (L % 2 != 0 || L < 64 || L > 512) return g;
  const int rows = TMA_SMEM / (TMA_NS * 8 * L);  // rows per stage in the budget
  const int ty = std::min(16, rows - 2);
  if (ty < 4) return g;
  g.T = ceil_div(L, ty);
  g.ty_max = ceil_div(L, g.T);
  const int target = num_sms() * 2;  // one wave of two CTAs per SM
  g.Z = std::max(1, target / g.T);
  g.kchunk = ceil_div(L, g.Z);
  g.Z = ceil_div(L, g.kchunk);
  return g;
}

static SpmvPath spmv_path(int L, int nv) {
  if (L % 2 != 0) return SP_GRID1;
  const char* e = getenv("AJ_SPMV_PATH");
  if (e && !strcmp(e, "tma") && tma_geom(L).T > 0) return SP_TMA;
  if (e && !strcmp(e, "grid")) return SP_GRID2;
  if (e && !strcmp(e, "bal")) return SP_BAL;
  return (nv == 0 && L >= 128 && tma_geom(L).T > 0) ? SP_TMA : SP_GRID2;
}

static size_t tma_smem_bytes(const TmaGeom& g, int L) { return (size_t)TMA_NS * (g.ty_max + 2) * L * 8; }

template <int NV>
static void launch_tma(const TmaGeom& g, double* y, const double* x, const double* eps, int L, double hop,
                       double sig, const double* W, int64_t ld, const RedBuf& rb, cudaStream_t st) {
  static int attr_dev[64] = {0};
  int dev = 0;
  AJ_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && !attr_dev[dev]) {
    AJ_CUDA(cudaFuncSetAttribute(k_spmv_tma<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, TMA_SMEM));
    attr_dev[dev] = 1;
  }
  k_spmv_tma<NV><<<g.T * g.Z, TMA_THREADS, tma_smem_bytes(g, L), st>>>(y, x, eps, L, hop, sig, g, W, ld, rb);
}

static dim3 spmv_grid(int L, int& kchunk) {
  const int tx = (L % 2 == 0) ? ceil_div(L, 2 * SBX) : ceil_div(L, SBX);
  int tiles = tx * ceil_div(L, SBY);
  // aim for >= 4 waves of 256-thread CTAs over 148 SMs, chunks of >= 4 planes
  int want = num_sms() * 8;
  int nz = std::max(1, std::min(L, ceil_div(want, tiles)));
  kchunk = std::max(4, ceil_div(L, nz));
  kchunk = std::min(kchunk, L);
  nz = ceil_div(L, kchunk);
  return dim3(tx, ceil_div(L, SBY), nz);
}

int spmv_grid_blocks(int L) {
  int kc;
  dim3 g = spmv_grid(L, kc);
  return (int)(g.x * g.y * g.z);
}

template <int NV>
static void spmv_dispatch(SpmvPath path, double* y, const double* x, const double* eps, int L, double hop,
                          double sig, const double* W, int64_t ld, const RedBuf& rb, cudaStream_t st) {
  const dim3 b(SBX, SBY);
  if (path == SP_TMA) {
    launch_tma<NV>(tma_geom(L), y, x, eps, L, hop, sig, W, ld, rb, st);
  } else if (path == SP_BAL) {
    const int tx = ceil_div(L, 2 * SBX), ty = ceil_div(L, SBY);
    const int64_t units = (int64_t)tx * ty * L;
    const int grid = (int)std::min<int64_t>(units, (int64_t)num_sms() * 4);
    k_spmv2_bal<NV><<<grid, b, 0, st>>>(y, x, eps, L, hop, sig, tx, units, W, ld, rb);
  } else {
    int kc;
    const dim3 g = spmv_grid(L, kc);
    if (path == SP_GRID2)
      k_spmv2<NV><<<g, b, 0, st>>>(y, x, eps, L, hop, sig, kc, W, ld, rb);
    else
      k_spmv<NV><<<g, b, 0, st>>>(y, x, eps, L, hop, sig, kc, W, ld, rb);
  }
  AJ_LAUNCHED();
}

void launch_spmv(double* y, const double* x, const double* eps, int L, double hop, double sig,
                 cudaStream_t st) {
  ProfScope ps(PROF_SPMV, 24.0 * L * L * L, st);
  spmv_dispatch<0>(spmv_path(L, 0), y, x, eps, L, hop, sig, nullptr, 0, RedBuf{}, st);
}

void launch_spmv_dots(double* y, const double* x, const double* eps, int L, double hop, double sig,
                      const double* W, int64_t ld, int nv, const RedBuf& rb, cudaStream_t st) {
  ProfScope ps(PROF_SPMV, (24.0 + 8.0 * nv) * L * L * L, st);
  const SpmvPath path = spmv_path(L, nv);
  switch (nv) {
#define CASE(N)                                                       \
  case N:                                                             \
    spmv_dispatch<N>(path, y, x, eps, L, hop, sig, W, ld, rb, st);    \
    break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
#undef CASE
    default:
      throw Error(AJ_ERR_ARG, "spmv_dots: nv out of range");
  }
}

// ---- z-slab shard (DESIGN.md sect. 6, row (e)) --------------------------------
// Disorder of planes [z0, z0 + nz): the same counter stream as k_disorder, indexed by
// the global site, so the shards of a lattice are bit-identical to its slices.
__global__ void k_disorder_slab(double* __restrict__ eps, int64_t s0, int64_t n, double W, uint64_t seed) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    double u = uniform01(seed, (uint64_t)(s0 + s));
    eps[s] = (u - 0.5) * W;
  }
}

void launch_disorder_slab(double* eps, int L, int z0, int nz, double W, uint64_t seed, cudaStream_t st) {
  const int64_t P = (int64_t)L * L, n = P * nz;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), (int64_t)num_sms() * 16));
  k_disorder_slab<<<grid, 256, 0, st>>>(eps, P * z0, n, W, seed);
  AJ_LAUNCHED();
}

// y = (A - sig I) x on a slab of nz planes: x_ext holds nz + 2 planes, plane 0 the
// halo below (global plane z0 - 1), planes 1..nz the slab, plane nz + 1 the halo above;
// periodic in x and y.  Same z-marching tile and the same summation order as k_spmv.
__global__ void __launch_bounds__(SBX* SBY)
    k_spmv_slab(double* __restrict__ y, const double* __restrict__ xe, const double* __restrict__ eps, int L,
                int nz, double hop, double sig, int kchunk) {
  const int i = blockIdx.x * SBX + threadIdx.x;
  const int j = blockIdx.y * SBY + threadIdx.y;
  const int k0 = blockIdx.z * kchunk;
  const int k1 = min(k0 + kchunk, nz);
  if (i >= L || j >= L || k0 >= nz) return;
  const int64_t P = (int64_t)L * L;
  const int im = (i == 0) ? L - 1 : i - 1, ip = (i == L - 1) ? 0 : i + 1;
  const int jm = (j == 0) ? L - 1 : j - 1, jp = (j == L - 1) ? 0 : j + 1;
  const int64_t r0 = (int64_t)j * L, rm = (int64_t)jm * L, rp = (int64_t)jp * L;
  double xm = __ldg(&xe[(int64_t)k0 * P + r0 + i]);        // global plane z0 + k0 - 1
  double xc = __ldg(&xe[(int64_t)(k0 + 1) * P + r0 + i]);
  for (int k = k0; k < k1; ++k) {
    const double xp = __ldg(&xe[(int64_t)(k + 2) * P + r0 + i]);
    const int64_t b = (int64_t)(k + 1) * P;
    const double s = (__ldg(&xe[b + r0 + im]) + __ldg(&xe[b + r0 + ip])) +
                     (__ldg(&xe[b + rm + i]) + __ldg(&xe[b + rp + i])) + (xm + xp);
    const int64_t o = (int64_t)k * P + r0 + i;
    y[o] = hop * s + (__ldg(&eps[o]) - sig) * xc;
    xm = xc;
    xc = xp;
  }
}

void launch_spmv_slab(double* y, const double* x_ext, const double* eps, int L, int nz, double hop, double sig,
                      cudaStream_t st) {
  const int tiles = ceil_div(L, SBX) * ceil_div(L, SBY);
  int zb = std::max(1, std::min(nz, ceil_div(num_sms() * 8, tiles)));
  int kc = std::max(1, ceil_div(nz, zb));
  zb = ceil_div(nz, kc);
  ProfScope ps(PROF_SPMV, 24.0 * L * L * nz, st);
  k_spmv_slab<<<dim3(ceil_div(L, SBX), ceil_div(L, SBY), zb), dim3(SBX, SBY), 0, st>>>(y, x_ext, eps, L, nz, hop,
                                                                                        sig, kc);
  AJ_LAUNCHED();
}

// ---- the sharded SpMV (DESIGN.md sect. 6): planes of this rank's slab, the z-neighbours of
// its first / last plane taken from the received halo planes.  Two plane ranges per launch
// ([a0, a1) then [b0, b1)), split into chunks of kchunk planes over blockIdx.z; same tile,
// z-march and summation order as k_spmv.  Optional fused dots as in k_spmv.
template <int NV>
__global__ void __launch_bounds__(SBX* SBY)
    k_spmv_halo(double* __restrict__ y, const double* __restrict__ x, const double* __restrict__ xlo,
                const double* __restrict__ xhi, const double* __restrict__ eps, int L, int nz, double hop, double sig,
                int a0, int a1, int b0, int b1, int kchunk, const double* __restrict__ Wv, int64_t ld, RedBuf rb) {
  const int i = blockIdx.x * SBX + threadIdx.x;
  const int j = blockIdx.y * SBY + threadIdx.y;
  const int na = (a1 - a0 + kchunk - 1) / kchunk;
  int k0, k1;
  if ((int)blockIdx.z < na) {
    k0 = a0 + blockIdx.z * kchunk;
    k1 = min(k0 + kchunk, a1);
  } else {
    k0 = b0 + (blockIdx.z - na) * kchunk;
    k1 = min(k0 + kchunk, b1);
  }
  double acc[NV > 0 ? NV : 1];
#pragma unroll
  for (int c = 0; c < (NV > 0 ? NV : 1); ++c) acc[c] = 0.0;
  if (i < L && j < L && k0 < k1) {
    const int64_t P = (int64_t)L * L;
    const int im = (i == 0) ? L - 1 : i - 1, ip = (i == L - 1) ? 0 : i + 1;
    const int jm = (j == 0) ? L - 1 : j - 1, jp = (j == L - 1) ? 0 : j + 1;
    const int64_t r0 = (int64_t)j * L, rm = (int64_t)jm * L, rp = (int64_t)jp * L;
    auto plane = [&](int k) -> const double* { return k < 0 ? xlo : (k >= nz ? xhi : x + (int64_t)k * P); };
    double xm = __ldg(&plane(k0 - 1)[r0 + i]);
    double xc = __ldg(&x[(int64_t)k0 * P + r0 + i]);
    for (int k = k0; k < k1; ++k) {
      const double xp = __ldg(&plane(k + 1)[r0 + i]);
      const int64_t b = (int64_t)k * P;
      const double s = (__ldg(&x[b + r0 + im]) + __ldg(&x[b + r0 + ip])) +
                       (__ldg(&x[b + rm + i]) + __ldg(&x[b + rp + i])) + (xm + xp);
      const double v = hop * s + (__ldg(&eps[b + r0 + i]) - sig) * xc;
      y[b + r0 + i] = v;
      if constexpr (NV > 0) {
#pragma unroll
        for (int c = 0; c < NV; ++c) acc[c] += v * __ldg(&Wv[c * ld + b + r0 + i]);
      }
      xm = xc;
      xc = xp;
    }
  }
  if constexpr (NV > 0)
    block_reduce_finalize<NV, SBX * SBY>(acc, rb, blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z),
                                         gridDim.x * gridDim.y * gridDim.z);
}

__global__ void k_add_into(int n, double* __restrict__ a, const double* __restrict__ b) {
  if (threadIdx.x < n) a[threadIdx.x] += b[threadIdx.x];
}

Domain domain_full(int L) {
  Domain d;
  d.L = L;
  d.z0 = 0;
  d.nz = L;
  d.n = (int64_t)L * L * L;
  return d;
}

Domain domain_slab(int L, int z0, int nz, const aj_comm* comm, cudaStream_t st) {
  Domain d;
  d.L = L;
  d.z0 = z0;
  d.nz = nz;
  d.n = (int64_t)L * L * nz;
  d.comm = comm;
  if (d.sharded()) d.halo = dalloc<double>(2 * (size_t)L * L, st);
  return d;
}

void domain_release(Domain& d, cudaStream_t st) {
  dfree(d.halo, st);
  d.halo = nullptr;
}

void dom_allreduce(const Domain& d, double* buf, int count, int op, cudaStream_t st) {
  if (!d.sharded() || count <= 0) return;
  const int rc = d.comm->allreduce(d.comm->ctx, buf, count, op, (void*)st);
  AJ_REQUIRE(rc == 0, AJ_ERR_CUDA, "comm allreduce failed (code " + std::to_string(rc) + ")");
}

void dom_gather_full(const Domain& d, double* full, const double* part, cudaStream_t st) {
  const int64_t N = (int64_t)d.L * d.L * d.L;
  AJ_REQUIRE(N < (int64_t)INT32_MAX, AJ_ERR_ARG, "dom_gather_full: L^3 exceeds the comm's int32 count");
  AJ_CUDA(cudaMemsetAsync(full, 0, (size_t)N * sizeof(double), st));
  AJ_CUDA(cudaMemcpyAsync(full + d.site0(), part, (size_t)d.n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (d.sharded()) dom_allreduce(d, full, (int)N, 0, st);
}

// interior planes [1, nz-1) while the halo planes travel, then planes 0 and nz-1
static void spmv_halo_launch(const Domain& d, double* y, const double* x, const double* eps, double hop, double sig,
                             const double* W, int64_t ld, int nv, const RedBuf& rb, int a0, int a1, int b0, int b1,
                             cudaStream_t st) {
  const int L = d.L;
  const int np = (a1 - a0) + (b1 - b0);
  if (np <= 0) return;
  const int tiles = ceil_div(L, SBX) * ceil_div(L, SBY);
  int zb = std::max(1, std::min(np, ceil_div(num_sms() * 8, tiles)));
  const int kc = std::max(1, ceil_div(np, zb));
  zb = ceil_div(a1 - a0, kc) + ceil_div(b1 - b0, kc);
  const dim3 g(ceil_div(L, SBX), ceil_div(L, SBY), zb), b(SBX, SBY);
  const double* xlo = d.halo;
  const double* xhi = d.halo + (int64_t)L * L;
  switch (nv) {
#define CASE(N)                                                                                                \
  case N:                                                                                                      \
    k_spmv_halo<N><<<g, b, 0, st>>>(y, x, xlo, xhi, eps, L, d.nz, hop, sig, a0, a1, b0, b1, kc, W, ld, rb); \
    break;
    CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10)
#undef CASE
    default:
      throw Error(AJ_ERR_ARG, "spmv_dots: nv out of range");
  }
  AJ_LAUNCHED();
}

static void spmv_sharded_impl(const Domain& d, double* y, const double* x, const double* eps, double hop, double sig,
                              const double* W, int64_t ld, int nv, const RedBuf& rb, cudaStream_t st) {
  const int64_t P = (int64_t)d.L * d.L;
  const aj_comm* c = d.comm;
  int rc = c->halo_start(c->ctx, x, x + (int64_t)(d.nz - 1) * P, d.halo, d.halo + P, P, (void*)st);
  AJ_REQUIRE(rc == 0, AJ_ERR_CUDA, "comm halo_start failed (code " + std::to_string(rc) + ")");
  ProfScope ps(PROF_SPMV, (24.0 + 8.0 * nv) * (double)d.n, st);
  const bool split = d.nz >= 3;
  RedBuf rb2 = rb;
  rb2.out = rb.out + nv;  // the boundary planes' partial dots
  if (split) spmv_halo_launch(d, y, x, eps, hop, sig, W, ld, nv, rb, 1, d.nz - 1, 0, 0, st);
  rc = c->halo_wait(c->ctx, (void*)st);
  AJ_REQUIRE(rc == 0, AJ_ERR_CUDA, "comm halo_wait failed (code " + std::to_string(rc) + ")");
  const int b0 = d.nz - 1 > 0 ? d.nz - 1 : 1;  // nz == 1: one boundary plane only
  spmv_halo_launch(d, y, x, eps, hop, sig, W, ld, nv, split ? rb2 : rb, 0, 1, b0, d.nz, st);
  if (nv > 0) {
    if (split) {
      k_add_into<<<1, 32, 0, st>>>(nv, rb.out, rb2.out);  // interior + boundary, fixed order
      AJ_LAUNCHED();
    }
    dom_allreduce(d, rb.out, nv, 0, st);
  }
}

void dom_spmv(const Domain& d, double* y, const double* x, const double* eps, double hop, double sig,
              cudaStream_t st) {
  if (!d.sharded()) {
    AJ_REQUIRE(d.nz == d.L, AJ_ERR_ARG, "dom_spmv: a single process needs the whole lattice");
    launch_spmv(y, x, eps, d.L, hop, sig, st);
    return;
  }
  spmv_sharded_impl(d, y, x, eps, hop, sig, nullptr, 0, 0, RedBuf{}, st);
}

void dom_spmv_dots(const Domain& d, double* y, const double* x, const double* eps, double hop, double sig,
                   const double* W, int64_t ld, int nv, const RedBuf& rb, cudaStream_t st) {
  if (!d.sharded()) {
    launch_spmv_dots(y, x, eps, d.L, hop, sig, W, ld, nv, rb, st);
    return;
  }
  spmv_sharded_impl(d, y, x, eps, hop, sig, W, ld, nv, rb, st);
}

}  // namespace aj
