// Tall-skinny fp64 kernels for the JD subspace work (DESIGN.md row 4) and the
// vector updates of the Krylov solver (row 2).  All HBM-bound: no tensor
// cores (fp64 contractions of width <= 64 sit far below the flop/byte
// crossover, and B200's fp64 tensor path is not the bottleneck here).
#include <algorithm>
#include <atomic>
#include <cstring>
#include <vector>

#include "aj_common.cuh"
#include "aj_kernels.cuh"

namespace aj {

// Per-(host thread, device) resources: a stream is bound to the device that was
// current when it was created, so the caches are keyed by the current device.
constexpr int kMaxDev = 64;
static int current_device() {
  int dev = 0;
  AJ_CUDA(cudaGetDevice(&dev));
  AJ_REQUIRE(dev >= 0 && dev < kMaxDev, AJ_ERR_CUDA, "device ordinal out of range");
  return dev;
}

cudaStream_t capture_stream() {
  thread_local cudaStream_t s[kMaxDev] = {};
  const int dev = current_device();
  if (!s[dev]) AJ_CUDA(cudaStreamCreateWithFlags(&s[dev], cudaStreamNonBlocking));
  return s[dev];
}

double* pinned_scalars() {
  thread_local double* p[kMaxDev] = {};
  const int dev = current_device();
  if (!p[dev]) AJ_CUDA(cudaMallocHost(&p[dev], 64 * sizeof(double)));
  return p[dev];
}



thread_local int64_t g_launches = 0;

// ---- live profiling ------------------------------------------------------
static thread_local bool g_prof_on = false;
static thread_local std::vector<ProfRec> g_prof_open;
static thread_local std::vector<cudaEvent_t> g_event_pool;
static thread_local aj_prof g_prof_acc;

static cudaEvent_t pool_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  AJ_CUDA(cudaEventCreate(&e));
  return e;
}

// While a stream is being captured into a CUDA graph, the scope records
// *external* event nodes (they fire on every graph launch) and registers the pair
// with the capturing code (g_prof_capture), which accumulates them per launch.
static thread_local std::vector<ProfRec>* g_prof_capture = nullptr;

static thread_local unsigned g_prof_mask = ~0u;

ProfScope::ProfScope(int c, double by, cudaStream_t s) : cat(c), bytes(by), st(s), rec(nullptr) {
  if (!g_prof_on || !((g_prof_mask >> c) & 1u)) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (g_prof_capture) AJ_CUDA(cudaStreamIsCapturing(s, &cs));  // only capturing code installs a sink
  ProfRec* r = new ProfRec{pool_event(), pool_event(), c, by};
  if (cs == cudaStreamCaptureStatusActive)
    AJ_CUDA(cudaEventRecordWithFlags(r->a, s, cudaEventRecordExternal));
  else
    AJ_CUDA(cudaEventRecord(r->a, s));
  rec = r;
}
void ProfScope::set_bytes(double b) {
  bytes = b;
  if (rec) ((ProfRec*)rec)->bytes = b;
}
ProfScope::~ProfScope() {
  if (!rec) return;
  ProfRec* r = (ProfRec*)rec;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (g_prof_capture) cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive) {
    cudaEventRecordWithFlags(r->b, st, cudaEventRecordExternal);
    g_prof_capture->push_back(*r);
  } else {
    cudaEventRecord(r->b, st);
    g_prof_open.push_back(*r);
  }
  delete r;
}

void prof_set_capture_sink(std::vector<ProfRec>* sink) { g_prof_capture = sink; }
// accumulate the event pairs of one completed graph launch
void prof_accumulate(const std::vector<ProfRec>& recs) {
  if (!g_prof_on) return;
  for (const auto& r : recs) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) continue;
    g_prof_acc.ms[r.cat] += ms;
    g_prof_acc.bytes[r.cat] += r.bytes;
    g_prof_acc.calls[r.cat] += 1;
  }
}
void prof_release(std::vector<ProfRec>& recs) {
  for (auto& r : recs) {
    g_event_pool.push_back(r.a);
    g_event_pool.push_back(r.b);
  }
  recs.clear();
}
bool prof_enabled() { return g_prof_on; }

static void prof_resolve() {
  for (auto& r : g_prof_open) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    g_prof_acc.ms[r.cat] += ms;
    g_prof_acc.bytes[r.cat] += r.bytes;
    g_prof_acc.calls[r.cat] += 1;
    g_event_pool.push_back(r.a);
    g_event_pool.push_back(r.b);
  }
  g_prof_open.clear();
}

void prof_enable(bool on, unsigned mask) {
  if (on) {
    prof_resolve();
    memset(&g_prof_acc, 0, sizeof(g_prof_acc));
    g_prof_mask = mask ? mask : ~0u;
  }
  g_prof_on = on;
}
void prof_get(aj_prof* out) {
  prof_resolve();
  *out = g_prof_acc;
}

int num_sms() {
  static std::atomic<int> cache[kMaxDev];
  const int dev = current_device();
  int sms = cache[dev].load();
  if (sms == 0) {
    AJ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cache[dev].store(sms);
    // keep freed stream-ordered allocations mapped: the factorisation allocates and
    // frees GBs per level, and the default threshold (0) would unmap them at every
    // synchronisation and remap them at the next cudaMallocAsync
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  return sms;
}

void RedScratch::init(cudaStream_t s) {
  partials = dalloc<double>(kMaxPartials, s);
  tickets = dalloc<unsigned>(kMaxTickets, s);
  AJ_CUDA(cudaMemsetAsync(tickets, 0, kMaxTickets * sizeof(unsigned), s));
}
void RedScratch::release(cudaStream_t s) {
  dfree(partials, s);
  dfree(tickets, s);
  partials = nullptr;
  tickets = nullptr;
}

constexpr int TB = 256;
constexpr int MD_NV = 8;

static int stream_grid(int64_t n) {
  int64_t need = ceil_div(n, (int64_t)TB);
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)num_sms() * 8));
}

// out[c0 + c] = sum_s V[(c0+c)*ld + s] * x[s],   c0 = blockIdx.y * MD_NV
__global__ void __launch_bounds__(TB)
    k_multi_dot(const double* __restrict__ V, int m, int64_t ld, const double* __restrict__ x,
                int64_t n, double* partials, unsigned* tickets, double* out) {
  const int c0 = blockIdx.y * MD_NV;
  double acc[MD_NV];
#pragma unroll
  for (int c = 0; c < MD_NV; ++c) acc[c] = 0.0;
  for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < n; s += (int64_t)gridDim.x * TB) {
    const double xs = __ldg(&x[s]);
#pragma unroll
    for (int c = 0; c < MD_NV; ++c)
      if (c0 + c < m) acc[c] += __ldg(&V[(int64_t)(c0 + c) * ld + s]) * xs;
  }
  RedBuf rb{partials + (size_t)blockIdx.y * gridDim.x * MD_NV, tickets + blockIdx.y, out + c0};
  block_reduce_finalize<MD_NV, TB>(acc, rb, blockIdx.x, gridDim.x);
}

void launch_multi_dot(double* out, const double* V, int m, int64_t ld, const double* x, int64_t n,
                      const RedScratch& rs, cudaStream_t st) {
  if (m <= 0) return;
  int gy = ceil_div(m, MD_NV);
  int gx = stream_grid(n);
  AJ_REQUIRE(gy <= kMaxTickets && (int64_t)gx * gy * MD_NV <= kMaxPartials, AJ_ERR_CAPACITY,
             "multi_dot: too many columns");
  ProfScope ps(PROF_JD, 8.0 * n * (m + 1), st);
  k_multi_dot<<<dim3(gx, gy), TB, 0, st>>>(V, m, ld, x, n, rs.partials, rs.tickets, out);
  AJ_LAUNCHED();
}

// y = beta*y + alpha * V c
__global__ void __launch_bounds__(TB) k_gemv(double* __restrict__ y, double beta, double alpha,
                                             const double* __restrict__ V, int m, int64_t ld,
                                             const double* __restrict__ c, int64_t n) {
  __shared__ double sc[64];
  if (threadIdx.x < m) sc[threadIdx.x] = c[threadIdx.x];
  __syncthreads();
  for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < n; s += (int64_t)gridDim.x * TB) {
    double acc = 0.0;
    for (int p = 0; p < m; ++p) acc += __ldg(&V[(int64_t)p * ld + s]) * sc[p];
    y[s] = (beta == 0.0 ? 0.0 : beta * y[s]) + alpha * acc;
  }
}

void launch_gemv(double* y, double beta, double alpha, const double* V, int m, int64_t ld,
                 const double* c, int64_t n, cudaStream_t st) {
  AJ_REQUIRE(m <= 64, AJ_ERR_CAPACITY, "gemv: m > 64");
  ProfScope ps(PROF_JD, 8.0 * n * (m + (beta == 0.0 ? 1 : 2)), st);
  k_gemv<<<stream_grid(n), TB, 0, st>>>(y, beta, alpha, V, m, ld, c, n);
  AJ_LAUNCHED();
}

// O[:, 0..q) = V[:, 0..p) S ; each thread owns one row, p <= 64 values in registers
template <int PMAX>
__global__ void __launch_bounds__(TB) k_gemm_ts(double* __restrict__ O, int64_t ldo,
                                                const double* __restrict__ V, int p, int64_t ldv,
                                                const double* __restrict__ S, int q, int64_t n) {
  extern __shared__ double sS[];  // p*q
  for (int t = threadIdx.x; t < p * q; t += TB) sS[t] = S[t];
  __syncthreads();
  for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < n; s += (int64_t)gridDim.x * TB) {
    double v[PMAX];
#pragma unroll
    for (int a = 0; a < PMAX; ++a) v[a] = (a < p) ? __ldg(&V[(int64_t)a * ldv + s]) : 0.0;
    for (int b = 0; b < q; ++b) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < PMAX; ++a)
        if (a < p) acc += v[a] * sS[b * p + a];
      O[(int64_t)b * ldo + s] = acc;
    }
  }
}

void launch_gemm_ts(double* O, int64_t ldo, const double* V, int p, int64_t ldv, const double* S,
                    int q, int64_t n, cudaStream_t st) {
  if (q <= 0) return;
  AJ_REQUIRE(p <= 64 && q <= 64, AJ_ERR_CAPACITY, "gemm_ts: p or q > 64");
  size_t sm = (size_t)p * q * sizeof(double);
  int g = stream_grid(n);
  ProfScope ps(PROF_JD, 8.0 * n * (p + q), st);
  if (p <= 16)
    k_gemm_ts<16><<<g, TB, sm, st>>>(O, ldo, V, p, ldv, S, q, n);
  else if (p <= 32)
    k_gemm_ts<32><<<g, TB, sm, st>>>(O, ldo, V, p, ldv, S, q, n);
  else
    k_gemm_ts<64><<<g, TB, sm, st>>>(O, ldo, V, p, ldv, S, q, n);
  AJ_LAUNCHED();
}

__global__ void __launch_bounds__(TB) k_dot(const double* __restrict__ x,
                                            const double* __restrict__ y, int64_t n, RedBuf rb) {
  double acc[1] = {0.0};
  for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < n; s += (int64_t)gridDim.x * TB)
    acc[0] += __ldg(&x[s]) * __ldg(&y[s]);
  block_reduce_finalize<1, TB>(acc, rb, blockIdx.x, gridDim.x);
}

void launch_dot(double* out, const double* x, const double* y, int64_t n, const RedScratch& rs,
                cudaStream_t st) {
  k_dot<<<stream_grid(n), TB, 0, st>>>(x, y, n, rs.buf(out));
  AJ_LAUNCHED();
}

__global__ void k_axpby(double* __restrict__ y, double a, const double* __restrict__ x, double b,
                        int64_t n) {
  for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < n; s += (int64_t)gridDim.x * TB)
    y[s] = a * x[s] + (b == 0.0 ? 0.0 : b * y[s]);
}
void launch_axpby(double* y, double a, const double* x, double b, int64_t n, cudaStream_t st) {
  k_axpby<<<stream_grid(n), TB, 0, st>>>(y, a, x, b, n);
  AJ_LAUNCHED();
}

__global__ void k_normalize(double* __restrict__ x, const double* nrm2, int64_t n) {
  const double inv = 1.0 / sqrt(*nrm2);
  for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < n; s += (int64_t)gridDim.x * TB)
    x[s] *= inv;
}
void launch_normalize(double* x, const double* nrm2, int64_t n, cudaStream_t st) {
  k_normalize<<<stream_grid(n), TB, 0, st>>>(x, nrm2, n);
  AJ_LAUNCHED();
}

__global__ void k_copy(double* __restrict__ y, const double* __restrict__ x, int64_t n) {
  for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < n; s += (int64_t)gridDim.x * TB)
    y[s] = x[s];
}
void launch_copy(double* y, const double* x, int64_t n, cudaStream_t st) {
  k_copy<<<stream_grid(n), TB, 0, st>>>(y, x, n);
  AJ_LAUNCHED();
}

__global__ void k_fill(double* __restrict__ y, double v, int64_t n) {
  for (int64_t s = blockIdx.x * (int64_t)TB + threadIdx.x; s < n; s += (int64_t)gridDim.x * TB)
    y[s] = v;
}
void launch_fill(double* y, double v, int64_t n, cudaStream_t st) {
  k_fill<<<stream_grid(n), TB, 0, st>>>(y, v, n);
  AJ_LAUNCHED();
}

}  // namespace aj
