// Device helpers shared by the multilevel ILDL setup kernels (aj_mlildl.cu,
// aj_schur.cu): sorted-row lookups, the 2x2 block product, and the per-row
// open-addressing hash tables of the Schur-complement kernels.
#pragma once
#include "aj_common.cuh"

namespace aj {

// position of column `key` in the sorted row [lo,hi), or -1
__device__ __forceinline__ int64_t lookup_idx(const int32_t* __restrict__ col, int64_t lo, int64_t hi,
                                              int32_t key) {
  int64_t a = lo, b = hi;
  while (a < b) {
    int64_t mid = (a + b) >> 1;
    if (col[mid] < key)
      a = mid + 1;
    else
      b = mid;
  }
  return (a < hi && col[a] == key) ? a : -1;
}

// returns a^_{row,key} or 0 (sorted row [lo,hi))
__device__ __forceinline__ double lookup(const int32_t* __restrict__ col, const double* __restrict__ ah,
                                         int64_t lo, int64_t hi, int32_t key) {
  const int64_t e = lookup_idx(col, lo, hi, key);
  return e >= 0 ? ah[e] : 0.0;
}

// l_cu for member u of a block {f} or {f, g} (f < g) from the row values
// a_cf, a_cg (0 if absent): l_cu = a_cf * Binv[f,u] + a_cg * Binv[g,u]
// (the order of oracle/mlildl.py::_l_rows; no FMA contraction).
__device__ __forceinline__ double lval_pair(double a_cf, double a_cg, double Bvu_f, double Bvu_g) {
  return __dadd_rn(__dmul_rn(a_cf, Bvu_f), __dmul_rn(a_cg, Bvu_g));
}

constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x >> 1); }

__device__ __forceinline__ uint32_t hash_slot(int32_t key, int bits) {
  return ((uint32_t)key * 2654435761u) >> (32 - bits);
}

// find-or-insert `key` into a table of size T (power of 2); returns the slot, or
// -1 once the table holds 3T/4 keys (the row is then handed to a larger tier; the
// load cap keeps probe chains short).  New keys get value 0 and their slot
// appended to `list`.
template <int T>
__device__ __forceinline__ int hslot(int32_t* tab, double* val, int32_t key, int* cnt, int32_t* list) {
  constexpr int BITS = ilog2c(T);
  static_assert((T & (T - 1)) == 0, "table size");
  uint32_t h = hash_slot(key, BITS);
  for (int probe = 0; probe < T; ++probe) {
    const int32_t prev = atomicCAS(&tab[h], -1, key);
    if (prev == -1) {
      val[h] = 0.0;
      const int pos = atomicAdd(cnt, 1);
      if (pos < T) list[pos] = (int32_t)h;
      return pos < (T * 3) / 4 ? (int)h : -1;
    }
    if (prev == key) return (int)h;
    h = (h + 1) & (T - 1);
  }
  return -1;
}

// slot of `key`, or -1 if absent (no insertion)
template <int T>
__device__ __forceinline__ int hfind(const int32_t* tab, int32_t key) {
  constexpr int BITS = ilog2c(T);
  uint32_t h = hash_slot(key, BITS);
  for (int probe = 0; probe < T; ++probe) {
    const int32_t k = tab[h];
    if (k == key) return (int)h;
    if (k == -1) return -1;
    h = (h + 1) & (T - 1);
  }
  return -1;
}

// find-or-insert returning the key's position in the insertion list (stored in the
// value slot); *fresh = true on insertion.  Concurrent inserts of the SAME key are
// not allowed (callers insert distinct keys in parallel, repeated keys serially).
template <int T>
__device__ __forceinline__ int lslot(int32_t* tab, double* val, int32_t key, int* cnt, int32_t* list, bool* fresh) {
  constexpr int BITS = ilog2c(T);
  uint32_t h = hash_slot(key, BITS);
  for (int probe = 0; probe < T; ++probe) {
    const int32_t prev = atomicCAS(&tab[h], -1, key);
    if (prev == -1) {
      const int pos = atomicAdd(cnt, 1);
      list[pos] = (int32_t)h;
      val[h] = __longlong_as_double((long long)pos);
      *fresh = true;
      return pos;
    }
    if (prev == key) {
      *fresh = false;
      return (int)__double_as_longlong(val[h]);
    }
    h = (h + 1) & (T - 1);
  }
  return -1;
}

}  // namespace aj
