// Counter-based generators used on the device.
//
// * Philox4x32-10 -- the GPU's own stream ("philox" rng mode): counters are
//   (element, step, purpose, attempt) and the key is the 64-bit derive_seed of
//   the caller's RngStream (rng.py:39-49), so every draw is a pure function of
//   (seed, ids, element, step): schedule- and launch-geometry independent.
// * Philox4x64-10 -- numpy's bit generator, replayed exactly ("numpy" rng
//   mode): the k-th raw u64 of RngStream(seed, ids).generator() is
//   philox4x64_10(counter = k/4 + 1, key = (derive_seed(seed,0,*ids),
//   derive_seed(seed,1,*ids)))[k % 4] (rng.py:69-74).
//   Generator.random() = (u64 >> 11) * 2^-53; integers(0, N) draws u32s (low
//   half of a u64 first) through Lemire's method (numpy distributions.c).
#pragma once

#include <cstdint>

namespace pfr {

struct Key2x64 {
  uint64_t k0, k1;
};

__host__ __device__ __forceinline__ void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                       uint32_t k0, uint32_t k1, uint32_t (&out)[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
#ifdef __CUDA_ARCH__
    const uint32_t lo0 = 0xD2511F53u * c0;
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2);
#else
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t lo0 = (uint32_t)p0, hi0 = (uint32_t)(p0 >> 32);
    const uint32_t lo1 = (uint32_t)p1, hi1 = (uint32_t)(p1 >> 32);
#endif
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

__host__ __device__ __forceinline__ void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  lo = (uint64_t)p;
  hi = (uint64_t)(p >> 64);
#endif
}

__host__ __device__ __forceinline__ void philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                                       uint64_t k0, uint64_t k1, uint64_t (&out)[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ull, c0, hi0, lo0);
    mulhilo64(0xCA5A826395121157ull, c2, hi1, lo1);
    const uint64_t n0 = hi1 ^ c1 ^ k0;
    const uint64_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// k-th raw u64 of the numpy stream (0-based)
__host__ __device__ __forceinline__ uint64_t numpy_raw64(Key2x64 key, uint64_t k) {
  uint64_t o[4];
  philox4x64_10(k / 4 + 1, 0, 0, 0, key.k0, key.k1, o);
  return o[k & 3];
}

__host__ __device__ __forceinline__ double u64_to_unit(uint64_t x) {
  return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}

// own-stream helpers -------------------------------------------------------

// purpose tags (third counter word) keep different uses of one RngStream apart
enum : uint32_t {
  kTagSystematic = 0x5359u,
  kTagStratified = 0x5354u,
  kTagMetropolis = 0x4D45u,
  kTagRejection = 0x524Au,
  kTagMultinomial = 0x4D55u,
  kTagRedraw = 0x8000u,
};

__host__ __device__ __forceinline__ float u32_to_unit_f(uint32_t x) {
  return (float)(x >> 8) * (1.0f / 16777216.0f);  // 24-bit, [0,1)
}
__host__ __device__ __forceinline__ double u32_to_unit_d(uint32_t x) {
#ifdef __CUDA_ARCH__
  // x * 2^-32 exactly, without the quarter-rate I2F.F64: the double with
  // high word 2^20 and low word x is 2^20 + x * 2^-32; subtracting 2^20 is exact
  return __hiloint2double(0x41300000, (int)x) - 1048576.0;
#else
  return (double)x * (1.0 / 4294967296.0);  // [0,1)
#endif
}

// open-interval variants (0, 1) for the own-stream acceptance tests: the
// midpoint of the cell, so u is never 0 and a zero weight can never be
// accepted (u * w[k] <= w[j] = 0 would hold at u = 0)
__host__ __device__ __forceinline__ float u32_to_unit_f_open(uint32_t x) {
#ifdef __CUDA_ARCH__
  // (1 + m 2^-23) - (1 - 2^-24) = (2m + 1) 2^-24, exact (Sterbenz): shift,
  // or, one FADD instead of shift, or, I2F, FMUL
  return __uint_as_float((x >> 9) | 0x3F800000u) - 0.99999994f;
#else
  return (float)(((x >> 9) << 1) | 1u) * (1.0f / 16777216.0f);  // (2m + 1) 2^-24, m < 2^23
#endif
}
__host__ __device__ __forceinline__ double u32_to_unit_d_open(uint32_t x) {
#ifdef __CUDA_ARCH__
  // (2^20 + x 2^-32) - (2^20 - 2^-33) = (2x + 1) 2^-33, exact (Sterbenz)
  return __hiloint2double(0x41300000, (int)x) - 1048575.9999999999;
#else
  return u32_to_unit_d(x) + 1.1641532182693481e-10;  // (2x + 1) 2^-33, exact
#endif
}

// Lemire bounded integer in [0, n): exact (rejection on the biased sliver;
// a rejected draw is replaced from a dedicated redraw counter so the result
// stays a pure function of the counter).  threshold = 2^32 mod n.
__device__ __forceinline__ uint32_t bounded_u32(uint32_t x, uint32_t n, uint32_t threshold, uint32_t c0,
                                                uint32_t c1, uint32_t tag, uint32_t k0, uint32_t k1) {
  uint64_t m = (uint64_t)x * n;
  uint32_t attempt = 0;
  while ((uint32_t)m < threshold) {  // probability < n / 2^32; never for powers of two
    uint32_t o[4];
    philox4x32_10(c0, c1, tag | kTagRedraw, ++attempt, k0, k1, o);
    m = (uint64_t)o[0] * n;
  }
  return (uint32_t)(m >> 32);
}

}  // namespace pfr
