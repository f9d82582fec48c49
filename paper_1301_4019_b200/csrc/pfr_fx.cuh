// Fixed-point fast path of the systematic/stratified offspring formula
// (shared by the fused delivery and the batched filter).
#pragma once

#include <cstdint>

namespace pfr {

// Fast path in S-bit fixed point, S = min(32, 51 - ceil(log2(N+1))):
// r_fx = round(W * fl(N/total) * 2^S) from ONE fma against 2^52 (the integer
// appears in the low mantissa bits: no float->int conversion), t_fx = r_fx +
// u_fx (exact integer add).  Against the reference's r = fl(fl(W*N)/total) and
// fl(r + u) the fixed-point values differ by at most 2 units of 2^-S
// (3 roundings of 2^-53 relative on r < N, N*2^S < 2^51, plus the
// quantisations), so whenever the fractional parts of r and r+u sit more than
// dr = 4 units from an integer, both floors are the reference's; otherwise
// the exact IEEE sequence runs (probability ~2^-S+4 per element).
struct FxParams {
  double sfx;       // fl(N / total) * 2^S
  double scale;     // 2^S
  long long ufx;    // round(u_sys * 2^S)
  uint32_t mask;    // 2^S - 1
  int S;
};
constexpr uint32_t kFxMargin = 4;

__device__ __forceinline__ long long fx_round(double x, double scale) {
  // round(x * scale) for 0 <= x * scale < 2^51
  return __double_as_longlong(__fma_rn(x, scale, 4503599627370496.0)) - 0x4330000000000000LL;
}

__device__ __forceinline__ bool fx_safe(long long v, uint32_t mask) {
  return (((uint32_t)v + kFxMargin) & mask) > 2 * kFxMargin;
}

// S = min(32, 51 - ceil(log2(N+1))) (host side: fx_bits)
inline int fx_bits(int64_t n) {
  int L = 1;
  while ((int64_t(1) << L) <= n) ++L;  // 2^L > N
  return L >= 19 ? 51 - L : 32;
}

template <typename A>
__device__ __forceinline__ FxParams fx_params(int64_t n, A total, A u_sys, int S) {
  FxParams f;
  f.S = S;
  f.scale = __longlong_as_double((long long)(1023 + S) << 52);  // 2^S
  f.mask = S >= 32 ? 0xFFFFFFFFu : ((1u << S) - 1u);
  f.sfx = __ddiv_rn((double)n, (double)total) * f.scale;
  f.ufx = fx_round((double)u_sys, f.scale);
  return f;
}

}  // namespace pfr
