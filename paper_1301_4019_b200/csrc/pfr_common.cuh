// Common device helpers for the resampling kernels (sm_100a).
//
// Everything on this path is HBM/L2 bound integer and scan work: no tensor
// cores.  The helpers here are the memory-access primitives (vector loads with
// cache hints, L2 eviction policies), warp scans with a FIXED association
// order (so floating-point results are run-to-run deterministic), and the
// status-word flags through which data-dependent validation reaches the host.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/pfr.h"

namespace pfr {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// status word (device); host maps bits to the reference's exceptions
__device__ __forceinline__ void status_or(uint32_t* status, uint32_t bits) {
  // read first: informational bits (any-positive) are set by nearly every
  // warp, and a same-address atomic per warp would serialise in L2
  if (bits && status && (*(volatile uint32_t*)status & bits) != bits) atomicOr(status, bits);
}

// warp-aggregated OR: one atomic per warp
__device__ __forceinline__ void status_or_warp(uint32_t* status, uint32_t bits) {
  unsigned m = __activemask();
  uint32_t agg = __reduce_or_sync(m, bits);
  if ((threadIdx.x & 31) == (__ffs(m) - 1)) status_or(status, agg);
}

// check_weights (diagnostics.py:38-51) on bit patterns: three integer maxima
// per element instead of float classification.  Non-finite <=> magnitude
// bits >= the infinity pattern; some x < 0 <=> unsigned max > the -0.0
// pattern; some x > 0 <=> signed max > 0.  Zero padding is neutral.
template <typename T>
struct FlagAcc;
template <>
struct FlagAcc<float> {
  uint32_t mag = 0u, ub = 0u;
  int32_t sb = INT32_MIN;
  __device__ __forceinline__ void add(float x) {
    const uint32_t b = __float_as_uint(x);
    mag = max(mag, b & 0x7FFFFFFFu);
    ub = max(ub, b);
    sb = max(sb, (int32_t)b);
  }
  __device__ __forceinline__ uint32_t flags() const {
    return (mag >= 0x7F800000u ? PFR_ST_NONFINITE : 0u) | (ub > 0x80000000u ? PFR_ST_NEGATIVE : 0u) |
           (sb > 0 ? PFR_ST_POSITIVE : 0u);
  }
};
template <>
struct FlagAcc<double> {
  uint64_t mag = 0u, ub = 0u;
  int64_t sb = INT64_MIN;
  __device__ __forceinline__ void add(double x) {
    const uint64_t b = (uint64_t)__double_as_longlong(x);
    const uint64_t m = b & 0x7FFFFFFFFFFFFFFFull;
    mag = m > mag ? m : mag;
    ub = b > ub ? b : ub;
    sb = (int64_t)b > sb ? (int64_t)b : sb;
  }
  __device__ __forceinline__ uint32_t flags() const {
    return (mag >= 0x7FF0000000000000ull ? PFR_ST_NONFINITE : 0u) |
           (ub > 0x8000000000000000ull ? PFR_ST_NEGATIVE : 0u) | (sb > 0 ? PFR_ST_POSITIVE : 0u);
  }
};

// ---------------------------------------------------------------------------
// L2 cache policies (createpolicy) and hinted loads/stores

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// streaming 16-byte read-only load, no L1 allocation, L2 policy hint.
// Not volatile: the loads are pure, so the compiler may batch them (MLP).
__device__ __forceinline__ uint4 ld_stream16(const void* ptr, uint64_t pol) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(ptr), "l"(pol));
  return r;
}

__device__ __forceinline__ void st_hint16(void* ptr, uint4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(ptr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}

__device__ __forceinline__ void st_hint4(void* ptr, uint32_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(ptr), "r"(v), "l"(pol) : "memory");
}

__device__ __forceinline__ int ld_hint_i32(const int* ptr, uint64_t pol) {
  int r;
  asm volatile("ld.global.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(ptr), "l"(pol));
  return r;
}

// relaxed gpu-scope 64-bit load/store used for the lookback tree cells
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---------------------------------------------------------------------------
// element traits: load 4 consecutive elements as one vector

template <typename T>
struct Vec4;
template <>
struct Vec4<float> {
  static __device__ __forceinline__ void load(const float* p, float (&x)[4], uint64_t pol) {
    uint4 r = ld_stream16(p, pol);
    x[0] = __uint_as_float(r.x);
    x[1] = __uint_as_float(r.y);
    x[2] = __uint_as_float(r.z);
    x[3] = __uint_as_float(r.w);
  }
};
template <>
struct Vec4<double> {
  static __device__ __forceinline__ void load(const double* p, double (&x)[4], uint64_t pol) {
    uint4 a = ld_stream16(p, pol);
    uint4 b = ld_stream16(p + 2, pol);
    x[0] = __hiloint2double(a.y, a.x);
    x[1] = __hiloint2double(a.w, a.z);
    x[2] = __hiloint2double(b.y, b.x);
    x[3] = __hiloint2double(b.w, b.z);
  }
};
template <>
struct Vec4<int32_t> {
  static __device__ __forceinline__ void load(const int32_t* p, int32_t (&x)[4], uint64_t pol) {
    uint4 r = ld_stream16(p, pol);
    x[0] = (int32_t)r.x;
    x[1] = (int32_t)r.y;
    x[2] = (int32_t)r.z;
    x[3] = (int32_t)r.w;
  }
};
template <>
struct Vec4<int64_t> {
  static __device__ __forceinline__ void load(const int64_t* p, int64_t (&x)[4], uint64_t pol) {
    uint4 a = ld_stream16(p, pol);
    uint4 b = ld_stream16(p + 2, pol);
    x[0] = (int64_t)(((uint64_t)a.y << 32) | a.x);
    x[1] = (int64_t)(((uint64_t)a.w << 32) | a.z);
    x[2] = (int64_t)(((uint64_t)b.y << 32) | b.x);
    x[3] = (int64_t)(((uint64_t)b.w << 32) | b.z);
  }
};

// IEEE add without contraction (the accumulators must not be fused into FMAs
// with neighbouring multiplies: association is part of the result)
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ int64_t add_rn(int64_t a, int64_t b) { return a + b; }

// Kogge-Stone inclusive warp scan; lane 31 ends with a balanced binary tree
// sum of the 32 inputs.  Fixed association => deterministic.
template <typename A>
__device__ __forceinline__ A warp_inclusive_scan(A v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    A o = __shfl_up_sync(0xffffffffu, v, off);
    if (lane >= off) v = add_rn(o, v);
  }
  return v;
}

__device__ __forceinline__ int warp_inclusive_scan_int(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int o = __shfl_up_sync(0xffffffffu, v, off);
    if (lane >= off) v += o;
  }
  return v;
}

// ---------------------------------------------------------------------------
// carry cell encoding for the deterministic lookback tree: one 64-bit word
// that is atomically published.  "kEmpty" can never be produced by encode().
template <typename A>
struct Cell;
template <>
struct Cell<double> {
  static constexpr uint64_t kEmpty = 0xFFFFFFFFFFFFFFFFull;
  static __device__ __forceinline__ uint64_t encode(double v) {
    uint64_t b = (uint64_t)__double_as_longlong(v);
    if (v != v) b = 0x7FF8000000000000ull;  // canonical NaN (keeps kEmpty free)
    return b;
  }
  static __device__ __forceinline__ double decode(uint64_t b) { return __longlong_as_double((long long)b); }
};
template <>
struct Cell<float> {
  static constexpr uint64_t kEmpty = 0xFFFFFFFFFFFFFFFFull;
  static __device__ __forceinline__ uint64_t encode(float v) { return (uint64_t)__float_as_uint(v); }
  static __device__ __forceinline__ float decode(uint64_t b) { return __uint_as_float((uint32_t)b); }
};
template <>
struct Cell<int64_t> {
  // integer sums of int32 inputs fit in 63 bits: shift left, bit 0 stays 0,
  // so the all-ones empty pattern can never be produced
  static constexpr uint64_t kEmpty = 0xFFFFFFFFFFFFFFFFull;
  static __device__ __forceinline__ uint64_t encode(int64_t v) { return (uint64_t)v << 1; }
  static __device__ __forceinline__ int64_t decode(uint64_t b) { return (int64_t)b >> 1; }
};

template <typename A>
__device__ __forceinline__ A cell_wait(const uint64_t* cell) {
  uint64_t b;
  while ((b = ld_relaxed_u64(cell)) == Cell<A>::kEmpty) {
    __nanosleep(32);
  }
  return Cell<A>::decode(b);
}

__device__ __forceinline__ int ceil_log2_i64(int64_t x) {
  int l = 0;
  while ((int64_t(1) << l) < x) ++l;
  return l;
}

// order-preserving 64-bit encoding of doubles (atomicMax on a max cell)
__device__ __forceinline__ unsigned long long ordered_bits(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_ordered(unsigned long long o) {
  unsigned long long b = (o & 0x8000000000000000ull) ? (o & 0x7FFFFFFFFFFFFFFFull) : ~o;
  return __longlong_as_double((long long)b);
}

}  // namespace pfr
