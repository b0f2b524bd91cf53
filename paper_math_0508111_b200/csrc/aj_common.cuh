// Common helpers of the Anderson JD library (sm_100a, fp64 throughout).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/anderson_jd.h"

namespace aj {

// ---------------------------------------------------------------------------
// errors: every internal failure throws aj::Error; the C ABI converts it into
// a return code + thread-local message.
struct Error : public std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define AJ_CUDA(call)                                                               \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      throw ::aj::Error(AJ_ERR_CUDA, std::string(#call " failed: ") +               \
                                         cudaGetErrorString(e_) + " @" + __FILE__ + \
                                         ":" + std::to_string(__LINE__));           \
  } while (0)

#define AJ_REQUIRE(cond, code, msg)                         \
  do {                                                      \
    if (!(cond)) throw ::aj::Error((code), std::string(msg)); \
  } while (0)

// launch accounting (thread local) -- see aj_launch_count()
extern thread_local int64_t g_launches;
#define AJ_LAUNCHED()                        \
  do {                                       \
    ::aj::g_launches++;                      \
    AJ_CUDA(cudaGetLastError());             \
  } while (0)

// live profiling (aj_prof_*): RAII scope recording an event pair on `st`
struct ProfScope {
  int cat;
  double bytes;
  cudaStream_t st;
  void* rec;
  ProfScope(int cat, double bytes, cudaStream_t st);
  ~ProfScope();
  void set_bytes(double b);  // the byte model once it is known (the setup's work model)
};
enum { PROF_SPMV = 0, PROF_PREC = 1, PROF_SETUP = 2, PROF_SQMR = 3, PROF_JD = 4 };

constexpr int kWarp = 32;
constexpr int kReduceThreads = 256;
constexpr int kMaxRed = 64;  // max values reduced by one fused reduction

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// Device memory helpers (stream-ordered pool allocator).
template <typename T>
T* dalloc(size_t count, cudaStream_t s) {
  void* p = nullptr;
  if (count == 0) count = 1;
  AJ_CUDA(cudaMallocAsync(&p, count * sizeof(T), s));
  return (T*)p;
}
inline void dfree(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

// Number of SMs of the current device (cached).
int num_sms();

// ---------------------------------------------------------------------------
// device helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// SplitMix64 finaliser (R3); identical definition in oracle/anderson.py.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ double uniform01(uint64_t key, uint64_t i) {
  uint64_t h = mix64(key + (i + 1ull) * 0x9E3779B97F4A7C15ull);
  return (double)(h >> 11) * 0x1.0p-53;
}

// ---------------------------------------------------------------------------
// Fused deterministic block reduction with "last block finalises" epilogue.
// Each block reduces NV per-thread values, thread 0 stores them to
// partials[bid * NV + k] (bid in [0, nblocks)); the last block to arrive (atomic ticket)
// sums the partials in a fixed order into out[0..NV) and resets the ticket.
// Deterministic for a fixed grid size.  Returns true in the finalising block
// (after out[] is written and visible to that block), false elsewhere.
struct RedBuf {
  double* partials;   // >= gridDim.x * NV
  unsigned* ticket;   // one counter, zero on entry
  double* out;        // NV results
};

template <int NV, int BLOCK>
__device__ __forceinline__ bool block_reduce_finalize(double (&v)[NV], const RedBuf& rb, int bid, int nblocks) {
  __shared__ double sred[NV][BLOCK / kWarp];
  __shared__ bool s_last;
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;  // linear id (2-D CTAs allowed)
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double x = warp_sum(v[k]);
    if (lane == 0) sred[k][wid] = x;
  }
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
      for (int w = 0; w < BLOCK / kWarp; ++w) s += sred[k][w];
      rb.partials[(size_t)bid * NV + k] = s;
    }
    __threadfence();
    unsigned t = atomicAdd(rb.ticket, 1u);
    s_last = (t == (unsigned)nblocks - 1u);
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  // last block: fixed-order reduction of all partials
  const int nb = nblocks;
  for (int k = 0; k < NV; ++k) {
    double s = 0.0;
    for (int b = tid; b < nb; b += BLOCK) s += __ldcg(&rb.partials[(size_t)b * NV + k]);
    s = warp_sum(s);
    if (lane == 0) sred[k][wid] = s;
  }
  __syncthreads();
  if (tid == 0) {
    for (int k = 0; k < NV; ++k) {
      double s = 0.0;
      for (int w = 0; w < BLOCK / kWarp; ++w) s += sred[k][w];
      rb.out[k] = s;
    }
    *rb.ticket = 0u;
    __threadfence();
  }
  __syncthreads();
  return true;
}

// ---- mbarrier + 1-D bulk copy (cp.async.bulk, the TMA engine without a tensor map) ----
// dst / src 16-byte aligned, bytes a multiple of 16; completion is signalled on `bar`
// (armed by mbar_expect_tx with the total bytes of the phase).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

}  // namespace aj
