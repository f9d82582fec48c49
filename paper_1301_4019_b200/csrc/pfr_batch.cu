// Batches of independent filters (SURVEY.md 8(e) "batched independent
// filters", 8(f) N1, BASELINE config 5): no communication between filters.
//
//   k_deliver_batched  systematic delivery of M filters of N particles, one
//                      CTA per filter: permute_parallel(
//                      cumulative_offspring_to_ancestors(
//                      systematic_cumulative_offspring(w_m))) per filter
//                      (resamplers.py:127-153, ancestry.py:69-76, 139-174)
//   pfr_pf_run         the bootstrap particle filter of pf.py:111-204 on the
//                      linear-Gaussian model, M filters at once: ESS-triggered
//                      systematic resampling, the copy step fused with the
//                      propagation (out-of-place gather x'[i] = x[c[i]], which
//                      Eq. 2 makes equivalent to pf_copy_step, pf.py:86-97),
//                      weighting, normalisation, log-likelihood, filtered mean.
//                      Per step (N % 32 == 0): k_pf_expand (one CTA per tile
//                      and filter) -> k_pf_repair (rare) -> K3 of the fused
//                      delivery over the resampled filters -> k_pf_fixup
//                      (rare) -> k_pf_step (one CTA per tile and filter);
//                      other N: k_pf_resample_local -> k_pf_step (DESIGN 3.6).
//
// segment_deliver (one CTA, one filter): pass 1 folds the tile aggregates
// (tile association of pfr_tile.cuh, serial across tiles), pass 2 recomputes
// W per element, O = min(N, floor((W*N)/W_N + u)) with the exact IEEE
// sequence, the running max (resamplers.py:150), and expands the slot words
// (pfr_expand.cuh); pass 3 resolves the in-place ancestry by walking the
// loser chains backwards (as k_dv_inplace).  The tile-parallel PF path uses
// the same associations, so every path gives identical results.
#include <cstdlib>
#include <algorithm>

#include "pfr_expand.cuh"
#include "pfr_fx.cuh"
#include "pfr_internal.h"
#include "pfr_tile.cuh"

namespace pfr {

namespace {

constexpr uint32_t kTagPfInit = 0x5049u;   // "PI"
constexpr uint32_t kTagPfProp = 0x5050u;   // "PP"
constexpr uint32_t kTagPfSys = 0x5053u;    // "PS"
constexpr uint32_t kTagBatchSys = 0x4253u; // "BS"

struct SegSmem {
  uint4 stage[kSlotCap * 4 / 16];  // word staging (32 KB)
  uint32_t heads[kTileThreads];
  double warp_sums[kTileThreads / 32];
  int32_t warp_last[kTileThreads / 32];
  int64_t imax8[kTileThreads / 32];
  double bcast;
  int32_t bcast_i;
};

__device__ __forceinline__ double philox_unit53(uint32_t c0, uint32_t c1, uint32_t tag, uint32_t k0, uint32_t k1) {
  uint32_t o[4];
  philox4x32_10(c0, c1, tag, 0, k0, k1, o);
  return u64_to_unit(((uint64_t)o[0] << 32) | o[1]);
}

// Systematic delivery of one filter of n particles (all threads of the CTA).
// u: the shared offset (already cast to the weight dtype).  Returns the
// longest chain walk in `longest` (per thread).
template <typename T, bool kResolve = true>
__device__ void segment_deliver(const T* __restrict__ w, int64_t n, double u, uint32_t* words, uint32_t* bitmap,
                                int32_t* __restrict__ c, int& longest, SegSmem& S, uint32_t pidx_offset = 0) {
  const int64_t tiles = num_tiles(n);
  // pass 1: total W_N = serial fold of the tile aggregates
  double total = 0.0;
  for (int64_t b = 0; b < tiles; ++b) {
    T x[kTileItems];
    tile_load_any<T>(w, n, b * kTile, x);
    TileScan<double> s;
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) s.loc[j] = (double)x[j];
    tile_scan<double>(s, S.warp_sums);
    if (threadIdx.x == kTileThreads - 1) S.bcast = __dadd_rn(s.thread_excl, s.loc[kTileItems - 1]);
    __syncthreads();
    total = __dadd_rn(total, S.bcast);
    __syncthreads();
  }
  // pass 2: O per element (exact sequence of resamplers.py:143-151), running
  // max, slot words
  double carry = 0.0;
  int64_t run = 0;  // running max of O before this tile
  int32_t o_prev = 0;
  const double nd = (double)n;
  for (int64_t b = 0; b < tiles; ++b) {
    const int64_t base = b * kTile;
    T x[kTileItems];
    tile_load_any<T>(w, n, base, x);
    TileScan<double> s;
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) s.loc[j] = (double)x[j];
    tile_scan<double>(s, S.warp_sums);
    int32_t o[kTileItems];
    int64_t mx = 0;
    const int e0 = threadIdx.x * kTileItems;
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
      const double W = __dadd_rn(carry, __dadd_rn(s.thread_excl, s.loc[j]));
      const double r = __ddiv_rn(__dmul_rn(W, nd), total);
      int64_t ov = (int64_t)floor(__dadd_rn(r, u));
      ov = ov > n ? n : (ov < 0 ? 0 : ov);
      if (base + e0 + j == n - 1) ov = n;  // O[N-1] = N
      if (base + e0 + j >= n) ov = n;      // padding past the filter
      o[j] = (int32_t)ov;
      mx = max(mx, ov);
    }
    int64_t tile_max;
    const int64_t before = block_excl_max<int64_t>(mx, (int64_t)0, S.imax8, tile_max);
    int64_t rr = max(run, before);
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
      rr = max(rr, (int64_t)o[j]);
      o[j] = (int32_t)rr;  // maximum.accumulate (resamplers.py:150)
    }
    tile_expand(o, o_prev, b, n, words, bitmap, reinterpret_cast<uint32_t*>(S.stage), S.heads, S.warp_last,
                pidx_offset);
    if (threadIdx.x == kTileThreads - 1) {
      S.bcast = __dadd_rn(s.thread_excl, s.loc[kTileItems - 1]);
      S.bcast_i = o[kTileItems - 1];
    }
    __syncthreads();
    carry = __dadd_rn(carry, S.bcast);
    o_prev = S.bcast_i;
    run = max(run, tile_max);
    __syncthreads();
  }
  __syncthreads();
  if constexpr (!kResolve) return;  // the caller runs the in-place pass
  // pass 3: in-place ancestry (backward chain walks)
  for (int64_t i = threadIdx.x; i < n; i += kTileThreads) {
    const bool has = (__ldcg(bitmap + (i >> 5)) >> (i & 31)) & 1u;
    if (has) {
      c[i] = (int32_t)i;
      continue;
    }
    uint32_t wd = __ldcg(words + i);
    int st = 0;
    while (wd & kFirst) {
      wd = __ldcg(words + (wd & kParentMask));
      if (++st > n) break;  // cannot happen for a valid ancestry
    }
    c[i] = (int32_t)(wd & kParentMask);
    longest = max(longest, st);
  }
}

template <typename T>
__global__ void __launch_bounds__(kTileThreads) k_deliver_batched(const T* __restrict__ w, int64_t M, int64_t n,
                                                                   const double* offsets, uint32_t k0, uint32_t k1,
                                                                   uint32_t* words, uint32_t* bitmap,
                                                                   int64_t bitmap_stride, int32_t* c,
                                                                   int32_t* max_steps) {
  __shared__ SegSmem S;
  int longest = 0;
  for (int64_t m = blockIdx.x; m < M; m += gridDim.x) {
    const double u0 = offsets ? offsets[m] : philox_unit53((uint32_t)m, (uint32_t)(m >> 32), kTagBatchSys, k0, k1);
    const double u = (double)(T)u0;  // cast to the weight dtype (resamplers.py:135)
    segment_deliver<T>(w + m * n, n, u, words + m * n, bitmap + m * bitmap_stride, c + m * n, longest, S);
    __syncthreads();
  }
  if (max_steps) {
    longest = __reduce_max_sync(0xffffffffu, longest);
    if ((threadIdx.x & 31) == 0 && longest) atomicMax(max_steps, longest);
  }
}

// ---------------------------------------------------------------------------
// batched bootstrap particle filter
struct PfArgs {
  int64_t M, N, T;
  double coeff, trans_std, obs_std, init_mean, init_std, ess_threshold;
  const double* y;      // [M, T]
  double* x0;           // [M, N] particles (ping)
  double* x1;           // [M, N] particles (pong)
  double* w;            // [M, N] unnormalised weights of the last step
  int32_t* c;           // [M, N] in-place ancestry of the current step
  uint32_t* words;      // [M, N] slot words (scratch)
  uint32_t* bitmap;     // [M, bitmap_stride]
  int64_t bitmap_stride;
  uint8_t* need;        // [M] resample at the next step
  DvState* dv;          // K3 state (overflow flag)
  int c_global;          // c holds global particle numbers (global in-place pass)
  int64_t tiles;         // tiles per filter
  int fx_S;              // fixed-point bits of the offspring fast path
  double* agg;          // [M, tiles] tile aggregates of w
  double* excl;         // [M, tiles + 1] exclusive tile prefixes, total
  uint8_t* repair;      // [M] filter needs the running-max repair
  uint32_t* rlist;      // [2, M] filters to resample at the next step (double buffered by step parity)
  uint32_t* rcount;     // [2]
  double* part;         // [M, tiles, 4] tile partials
  unsigned int* slice_done;  // [M] tiles finished (reset by the last)
  double* means;        // [M, T]
  double* loglik;       // [M]
  double* ess;          // [M, T]
  uint8_t* resampled;   // [M, T]
  uint32_t k0, k1;
  uint32_t* status;
};

// two standard normals from one Philox call (Box-Muller in float with the
// SFU log/sin/cos, abs. error ~1e-6: the transition noise of the model,
// pf.py:188-189)
__device__ __forceinline__ float2 normal2(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t tag, uint32_t k0,
                                          uint32_t k1) {
  uint32_t o[4];
  philox4x32_10(c0, c1, c2, tag, k0, k1, o);
  const float u1 = ((float)(o[0] >> 8) + 1.0f) * (1.0f / 16777216.0f);  // (0, 1]
  const float u2 = (float)(o[1] >> 8) * (1.0f / 16777216.0f);
  const float rad = sqrtf(-2.0f * __logf(u1));
  float sn, cs;
  __sincosf(6.283185307179586f * u2, &sn, &cs);
  return make_float2(rad * cs, rad * sn);
}

// four standard normals from one Philox call (all four words: two Box-Muller
// pairs) -- the transition noise of particles 4q .. 4q+3 of a filter
__device__ __forceinline__ float4 normal4(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t tag, uint32_t k0,
                                          uint32_t k1) {
  uint32_t o[4];
  philox4x32_10(c0, c1, c2, tag, k0, k1, o);
  float z[4];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float u1 = ((float)(o[2 * h] >> 8) + 1.0f) * (1.0f / 16777216.0f);  // (0, 1]
    const float u2 = (float)(o[2 * h + 1] >> 8) * (1.0f / 16777216.0f);
    const float rad = sqrtf(-2.0f * __logf(u1));
    float sn, cs;
    __sincosf(6.283185307179586f * u2, &sn, &cs);
    z[2 * h] = rad * cs;
    z[2 * h + 1] = rad * sn;
  }
  return make_float4(z[0], z[1], z[2], z[3]);
}

__global__ void __launch_bounds__(256) k_pf_init(PfArgs a) {
  const int64_t total = a.M * a.N;
  for (int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 2; p < total;
       p += (int64_t)gridDim.x * blockDim.x * 2) {
    const float2 z = normal2((uint32_t)(p >> 1), (uint32_t)(p >> 33), 0, kTagPfInit, a.k0, a.k1);
    a.x0[p] = a.init_mean + a.init_std * (double)z.x;
    if (p + 1 < total) a.x0[p + 1] = a.init_mean + a.init_std * (double)z.y;
  }
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < a.M; m += (int64_t)gridDim.x * blockDim.x) {
    a.need[m] = 0;
    a.loglik[m] = 0.0;
    a.ess[m * a.T] = (double)a.N;  // uniform initial weights
  }
}

// Resampling of the filters whose ESS fell below the threshold (the step
// before left their tile aggregates, exclusive tile prefixes and totals; see
// k_pf_step).  Global in-place path (N % 32 == 0): one CTA per (tile,
// filter) -- offspring of the tile from its prefix (the same association and
// IEEE sequence as segment_deliver), then the slot words with GLOBAL parent
// numbers into a contiguous bitmap; one global in-place pass (K3 of the fused
// delivery, launch_dv_inplace) then resolves every filter's chains at once
// (chains never leave a filter: its slots only name its own parents).  A tile
// whose O decreases (rounding; never observed) flags its filter for
// k_pf_repair, which redoes the filter with segment_deliver's running max.
__global__ void __launch_bounds__(kTileThreads, 4) k_pf_expand(PfArgs a, int64_t t) {
  __shared__ SegSmem S;
  const int64_t m = blockIdx.y, b = blockIdx.x, n = a.N;
  if (b == 0 && m == 0 && threadIdx.x == 0) a.dv->flags = 0;  // K3 overflow flag of the previous step
  const bool go = a.need[m] != 0;
  if (b == 0 && threadIdx.x == 0) a.resampled[m * a.T + t] = go ? 1 : 0;
  if (!go) return;
  const double u = philox_unit53((uint32_t)m, (uint32_t)t, kTagPfSys, a.k0, a.k1);
  const int64_t base = b * kTile;
  double x[kTileItems];
  tile_load_any<double>(a.w + m * n, n, base, x);
  TileScan<double> s;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) s.loc[j] = x[j];
  tile_scan<double>(s, S.warp_sums);
  const double* ex = a.excl + m * (a.tiles + 1);
  const double carry = __ldcg(ex + b), total = __ldcg(ex + a.tiles);
  const double nd = (double)n;
  // fixed-point fast path (pfr_fx.cuh), the exact sequence when fragile
  const FxParams fx = fx_params<double>(n, total, u, a.fx_S);
  auto off = [&](double W) -> int64_t {
    const long long r = fx_round(W, fx.sfx);
    const long long tt = r + fx.ufx;
    if (fx_safe(r, fx.mask) & fx_safe(tt, fx.mask)) return min((int64_t)(tt >> fx.S), n);
    const double rr = __ddiv_rn(__dmul_rn(W, nd), total);
    int64_t ov = (int64_t)floor(__dadd_rn(rr, u));
    return ov > n ? n : (ov < 0 ? (int64_t)0 : ov);
  };
  int32_t o[kTileItems];
  const int64_t e0 = base + threadIdx.x * kTileItems;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) {
    int64_t ov = off(__dadd_rn(carry, __dadd_rn(s.thread_excl, s.loc[j])));
    if (e0 + j >= n - 1) ov = n;  // O[N-1] = N; padding past the filter
    o[j] = (int32_t)ov;
  }
  const int32_t o_prev = b > 0 ? (int32_t)off(carry) : 0;
  const int len = (int)min((int64_t)kTile, n - base);
  if (tile_decreases(o, o_prev, len, S.warp_last)) {
    if (threadIdx.x == 0) a.repair[m] = 1;
    return;
  }
  tile_expand(o, o_prev, b, n, a.words + m * n, a.bitmap + m * (n / 32), reinterpret_cast<uint32_t*>(S.stage),
              S.heads, S.warp_last, (uint32_t)(m * n));
}

// rare: a filter whose O decreased somewhere -- the whole filter again with
// the running max (segment_deliver passes 1-2)
__global__ void __launch_bounds__(kTileThreads) k_pf_repair(PfArgs a, int64_t t) {
  __shared__ SegSmem S;
  for (int64_t m = blockIdx.x; m < a.M; m += gridDim.x) {
    if (!*(volatile uint8_t*)(a.repair + m)) continue;
    const double u = philox_unit53((uint32_t)m, (uint32_t)t, kTagPfSys, a.k0, a.k1);
    int longest = 0;
    segment_deliver<double, false>(a.w + m * a.N, a.N, u, a.words + m * a.N, a.bitmap + m * (a.N / 32), nullptr,
                                   longest, S, (uint32_t)(m * a.N));
    __syncthreads();
    if (threadIdx.x == 0) a.repair[m] = 0;
  }
}

// Other N (or the PFR_PF_PATH=1 knob): one CTA per filter, segment_deliver
// with its own pass 3 (c local to the filter).
__global__ void __launch_bounds__(kTileThreads) k_pf_resample_local(PfArgs a, int64_t t) {
  __shared__ SegSmem S;
  for (int64_t m = blockIdx.x; m < a.M; m += gridDim.x) {
    const bool go = a.need[m] != 0;
    if (threadIdx.x == 0) a.resampled[m * a.T + t] = go ? 1 : 0;
    if (!go) continue;
    const double u = philox_unit53((uint32_t)m, (uint32_t)t, kTagPfSys, a.k0, a.k1);
    int longest = 0;
    segment_deliver<double, true>(a.w + m * a.N, a.N, u, a.words + m * a.N, a.bitmap + m * a.bitmap_stride,
                                  a.c + m * a.N, longest, S);
    __syncthreads();
  }
}

// rare: a chain longer than K3's walk bound -- redo the in-place pass of the
// resampled filters with unbounded per-thread walks (global numbers)
__global__ void __launch_bounds__(kTileThreads) k_pf_fixup(PfArgs a, int64_t t, int force) {
  // the list the next step fills (its previous reader, the in-place pass of
  // step t - 1, has finished)
  if (blockIdx.x == 0 && threadIdx.x == 0) a.rcount[(t + 1) & 1] = 0;
  if (!force && !(*(volatile unsigned*)&a.dv->flags & 2u)) return;
  for (int64_t m = blockIdx.x; m < a.M; m += gridDim.x) {
    if (!a.need[m]) continue;
    const uint32_t* bitmap = a.bitmap + m * (a.N / 32);
    const int64_t base = m * a.N;
    for (int64_t i = threadIdx.x; i < a.N; i += blockDim.x) {
      if ((__ldcg(bitmap + (i >> 5)) >> (i & 31)) & 1u) {
        a.c[base + i] = (int32_t)(base + i);
        continue;
      }
      uint32_t wd = __ldcg(a.words + base + i);
      int64_t st = 0;
      while ((wd & kFirst) && st++ <= a.N) wd = __ldcg(a.words + (wd & kParentMask));
      a.c[base + i] = (int32_t)(wd & kParentMask);
    }
  }
}

// Propagate (through the ancestry when resampled) + weight + per-filter
// reductions, one CTA per (tile, filter).  Compute runs striped (in round r
// thread t owns the 4 particles at (256 r + t) * 4: coalesced 16-byte
// accesses when N % 4 == 0); the new weights are restaged through shared
// memory so that thread t then owns the tile's particles [16t, 16t + 16) and
// each tile publishes the aggregate of its new weights in the association of
// tile_scan (exactly segment_deliver's pass-1 value).  The last tile of a
// filter to finish (per-filter counter) folds the tile partials in tile order
// (deterministic), finishes the filter's step and, when it must resample
// next, the exclusive tile prefixes and the total (serial folds, as
// segment_deliver's pass 1/2 carries).
template <bool kVec>
__global__ void __launch_bounds__(kTileThreads, 4) k_pf_step(PfArgs a, int64_t t) {
  __shared__ double red[4][kTileThreads / 32];
  __shared__ double warp_sums[kTileThreads / 32];
  __shared__ __align__(16) double2 ubuf[kTile / 2];
  __shared__ bool last;
  const int64_t m = blockIdx.y, b = blockIdx.x;
  const int64_t n = a.N;
  const bool res = a.need[m] != 0;
  const double* src = ((t & 1) ? a.x1 : a.x0) + m * n;
  double* dst = ((t & 1) ? a.x0 : a.x1) + m * n;
  double* w = a.w + m * n;
  const int32_t* cm = a.c + m * n;
  const int64_t c_base = a.c_global ? m * n : 0;
  const double y = a.y[m * a.T + t];
  const double inv_obs = 1.0 / a.obs_std;
  const double dens_norm = inv_obs * 0.3989422804014327;  // 1 / (obs_std sqrt(2 pi))
  const int64_t base = b * kTile;
  double su = 0.0, sux = 0.0, suu = 0.0, sw = 0.0;
  constexpr int kRounds = kTile / (4 * kTileThreads);
#pragma unroll 2
  for (int r = 0; r < kRounds; ++r) {
    const int l0 = (r * kTileThreads + threadIdx.x) * 4;  // tile-local index of my first particle
    const int64_t e0 = base + l0;
    const bool full = kVec && e0 + 4 <= n;
    double xo[4], wp[4];
    if (full) {
      if (res) {
        const int4 ci = __ldcs(reinterpret_cast<const int4*>(cm + e0));
        xo[0] = __ldg(src + (ci.x - c_base));
        xo[1] = __ldg(src + (ci.y - c_base));
        xo[2] = __ldg(src + (ci.z - c_base));
        xo[3] = __ldg(src + (ci.w - c_base));
      } else {
        const double2 v0 = __ldcs(reinterpret_cast<const double2*>(src + e0));
        const double2 v1 = __ldcs(reinterpret_cast<const double2*>(src + e0) + 1);
        xo[0] = v0.x, xo[1] = v0.y, xo[2] = v1.x, xo[3] = v1.y;
      }
      if (res || t == 0) {
        wp[0] = wp[1] = wp[2] = wp[3] = 1.0;
      } else {
        const double2 v0 = __ldcs(reinterpret_cast<const double2*>(w + e0));
        const double2 v1 = __ldcs(reinterpret_cast<const double2*>(w + e0) + 1);
        wp[0] = v0.x, wp[1] = v0.y, wp[2] = v1.x, wp[3] = v1.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t k = e0 + j;
        xo[j] = 0.0;
        wp[j] = 0.0;
        if (k < n) {
          xo[j] = res ? src[cm[k] - c_base] : src[k];
          wp[j] = (res || t == 0) ? 1.0 : w[k];
        }
      }
    }
    double un[4];
    // the normals of particles e0 .. e0+3 (e0 % 4 == 0) of the filter
    const float4 z4 = normal4((uint32_t)(e0 >> 2), (uint32_t)m, (uint32_t)t, kTagPfProp, a.k0, a.k1);
    const float zz[4] = {z4.x, z4.y, z4.z, z4.w};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = 2 * q + h;
        const double xn = a.coeff * xo[j] + a.trans_std * (double)zz[j];
        const double e = (y - xn) * inv_obs;
        sw += wp[j];
        double u = wp[j] * (dens_norm * exp(-0.5 * e * e));
        if (!full && e0 + j >= n) u = 0.0;
        xo[j] = xn;
        un[j] = u;
        su += u;
        sux += u * xn;
        suu += u * u;
      }
    }
    if (full) {
      __stcs(reinterpret_cast<double2*>(dst + e0), make_double2(xo[0], xo[1]));
      __stcs(reinterpret_cast<double2*>(dst + e0) + 1, make_double2(xo[2], xo[3]));
      __stcg(reinterpret_cast<double2*>(w + e0), make_double2(un[0], un[1]));
      __stcg(reinterpret_cast<double2*>(w + e0) + 1, make_double2(un[2], un[3]));
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (e0 + j < n) {
          dst[e0 + j] = xo[j];
          w[e0 + j] = un[j];
        }
    }
    ubuf[swz(l0 / 2)] = make_double2(un[0], un[1]);
    ubuf[swz(l0 / 2 + 1)] = make_double2(un[2], un[3]);
  }
  __syncthreads();
  TileScan<double> s;
#pragma unroll
  for (int k = 0; k < kTileItems / 2; ++k) {
    const double2 v = ubuf[swz(threadIdx.x * (kTileItems / 2) + k)];
    s.loc[2 * k] = v.x;
    s.loc[2 * k + 1] = v.y;
  }
  // tile aggregate of the new weights (segment_deliver's association)
  tile_scan<double>(s, warp_sums);
  if (threadIdx.x == kTileThreads - 1) a.agg[m * a.tiles + b] = __dadd_rn(s.thread_excl, s.loc[kTileItems - 1]);
  // block reduction: warp butterfly, then the 8 warps in order
  double v[4] = {su, sux, suu, sw};
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int off = 16; off; off >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], off);
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int q = 0; q < 4; ++q) red[q][threadIdx.x >> 5] = v[q];
  __syncthreads();
  if (threadIdx.x == 0) {
    double* part = a.part + (m * a.tiles + b) * 4;
    for (int q = 0; q < 4; ++q) {
      double r = 0;
      for (int k = 0; k < kTileThreads / 32; ++k) r += red[q][k];
      part[q] = r;
    }
    __threadfence();
    last = atomicAdd(&a.slice_done[m], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  double r[4] = {0, 0, 0, 0};
  for (int64_t sl = 0; sl < a.tiles; ++sl)
    for (int q = 0; q < 4; ++q) r[q] += __ldcg(a.part + (m * a.tiles + sl) * 4 + q);
  a.slice_done[m] = 0;
  const double total = r[0] / r[3];  // sum of normalised weights x density
  if (!(total > 0.0) || !isfinite(total)) {
    status_or(a.status, PFR_ST_NOPROGRESS);  // weight collapse (pf.py:193-198)
  } else {
    a.loglik[m] += log(total);
  }
  a.means[m * a.T + t] = r[1] / r[0];
  const double ess_next = r[0] * r[0] / r[2];
  if (t + 1 < a.T) a.ess[m * a.T + t + 1] = ess_next;
  const bool need = (ess_next / (double)n < a.ess_threshold);
  a.need[m] = need ? 1 : 0;
  if (need && t + 1 < a.T) {
    const int nb = (int)((t + 1) & 1);
    if (a.c_global) a.rlist[nb * a.M + atomicAdd(a.rcount + nb, 1u)] = (uint32_t)m;
    double* ex = a.excl + m * (a.tiles + 1);
    double carry = 0.0;
    for (int64_t sl = 0; sl < a.tiles; ++sl) {
      ex[sl] = carry;
      carry = __dadd_rn(carry, __ldcg(a.agg + m * a.tiles + sl));
    }
    ex[a.tiles] = carry;
  }
}

}  // namespace

size_t pf_workspace_bytes(int64_t M, int64_t N) {
  const int64_t mn = M * N;
  const int64_t bstride = (N + 31) / 32 + 4;
  size_t b = 0;
  auto add = [&](size_t bytes) { b += (bytes + 255) / 256 * 256; };
  add(mn * 8);          // x0
  add(mn * 8);          // x1
  add(mn * 8);          // w
  add(mn * 4);          // c
  add(mn * 4 + 16);     // words
  add(M * bstride * 4); // bitmap
  add(M);               // need
  const int64_t tiles = num_tiles(N);
  add(M * tiles * 8);        // tile aggregates
  add(M * (tiles + 1) * 8);  // tile prefixes
  add(M);                    // repair flags
  add(2 * M * 4 + 8);        // resample lists + counts
  add(M * tiles * 4 * 8);    // tile partials
  add(M * 4);                // tile counters
  add(sizeof(DvState)); // K3 state
  return b;
}

size_t batched_workspace_bytes(int64_t M, int64_t N) {
  size_t b = 0;
  auto add = [&](size_t bytes) { b += (bytes + 255) / 256 * 256; };
  add(M * N * 4 + 16);
  add(M * ((N + 31) / 32 + 4) * 4);
  return b;
}

cudaError_t launch_deliver_batched(const void* w, int64_t M, int64_t n, int dtype, const double* offsets,
                                   const pfr_rng* rng, int32_t* c, int32_t* max_steps, void* ws, cudaStream_t s) {
  char* p = static_cast<char*>(ws);
  uint32_t* words = reinterpret_cast<uint32_t*>(p);
  p += (M * n * 4 + 16 + 255) / 256 * 256;
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(p);
  const int64_t bstride = (n + 31) / 32 + 4;
  if (max_steps) {
    cudaError_t e = cudaMemsetAsync(max_steps, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
  }
  const uint32_t k0 = rng ? (uint32_t)rng->key0 : 0u, k1 = rng ? (uint32_t)(rng->key0 >> 32) : 0u;
  const unsigned grid = (unsigned)std::min<int64_t>(M, (int64_t)num_sms() * 8);
  if (dtype == PFR_F64)
    k_deliver_batched<double><<<grid, kTileThreads, 0, s>>>((const double*)w, M, n, offsets, k0, k1, words, bitmap,
                                                            bstride, c, max_steps);
  else
    k_deliver_batched<float><<<grid, kTileThreads, 0, s>>>((const float*)w, M, n, offsets, k0, k1, words, bitmap,
                                                           bstride, c, max_steps);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_pf_run(const pfr_pf_model* model, const double* y, int64_t M, int64_t N, int64_t T,
                          double ess_threshold, const pfr_rng* rng, double* means, double* loglik, double* ess,
                          uint8_t* resampled, uint32_t* status, void* ws, cudaStream_t s) {
  PfArgs a;
  a.M = M;
  a.N = N;
  a.T = T;
  a.coeff = model->coeff;
  a.trans_std = model->trans_std;
  a.obs_std = model->obs_std;
  a.init_mean = model->initial_mean;
  a.init_std = model->initial_std;
  a.ess_threshold = ess_threshold;
  a.y = y;
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t bytes) {
    char* q = p;
    p += (bytes + 255) / 256 * 256;
    return q;
  };
  const int64_t mn = M * N;
  a.x0 = reinterpret_cast<double*>(take(mn * 8));
  a.x1 = reinterpret_cast<double*>(take(mn * 8));
  a.w = reinterpret_cast<double*>(take(mn * 8));
  a.c = reinterpret_cast<int32_t*>(take(mn * 4));
  a.words = reinterpret_cast<uint32_t*>(take(mn * 4 + 16));
  a.bitmap_stride = (N + 31) / 32 + 4;
  a.bitmap = reinterpret_cast<uint32_t*>(take(M * a.bitmap_stride * 4));
  a.need = reinterpret_cast<uint8_t*>(take(M));
  a.tiles = num_tiles(N);
  a.fx_S = fx_bits(N);
  a.agg = reinterpret_cast<double*>(take(M * a.tiles * 8));
  a.excl = reinterpret_cast<double*>(take(M * (a.tiles + 1) * 8));
  a.repair = reinterpret_cast<uint8_t*>(take(M));
  a.rlist = reinterpret_cast<uint32_t*>(take(2 * M * 4 + 8));
  a.rcount = a.rlist + 2 * M;
  a.part = reinterpret_cast<double*>(take(M * a.tiles * 4 * 8));
  a.slice_done = reinterpret_cast<unsigned int*>(take(M * 4));
  a.dv = reinterpret_cast<DvState*>(take(sizeof(DvState)));
  a.means = means;
  a.loglik = loglik;
  a.ess = ess;
  a.resampled = resampled;
  a.k0 = (uint32_t)rng->key0;
  a.k1 = (uint32_t)(rng->key0 >> 32);
  a.status = status;
  // ESS at t = 0: uniform weights
  cudaError_t e = cudaMemsetAsync(ess, 0, sizeof(double) * M * T, s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(a.slice_done, 0, sizeof(unsigned int) * M, s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(a.dv, 0, sizeof(DvState), s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(a.repair, 0, M, s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(a.rcount, 0, 8, s);
  if (e != cudaSuccess) return e;
  // stale slot words of filters that did not resample stay valid particle
  // numbers for the global in-place pass
  e = cudaMemsetAsync(a.words, 0, (size_t)mn * 4, s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(a.bitmap, 0, (size_t)M * a.bitmap_stride * 4, s);
  if (e != cudaSuccess) return e;
  // PFR_PF_PATH (test knob): 0 global in-place pass (default), 1 per-filter
  // pass 3, 2 global pass followed by the unbounded fixup pass
  int path = 0;
  if (const char* v = getenv("PFR_PF_PATH")) path = atoi(v);
  const bool global_pass = (N % 32) == 0 && path != 1;
  a.c_global = global_pass ? 1 : 0;
  const unsigned g0 = (unsigned)std::min<int64_t>((mn / 2 + 255) / 256 + 1, (int64_t)num_sms() * 16);
  k_pf_init<<<g0, 256, 0, s>>>(a);
  note_launch();
  const unsigned gr = (unsigned)std::min<int64_t>(M, (int64_t)num_sms() * 8);
  for (int64_t t = 0; t < T; ++t) {
    if (t > 0) {
      if (global_pass) {
        k_pf_expand<<<dim3((unsigned)a.tiles, (unsigned)M), kTileThreads, 0, s>>>(a, t);
        note_launch();
        k_pf_repair<<<gr, kTileThreads, 0, s>>>(a, t);
        note_launch();
        e = launch_dv_inplace(a.words, a.bitmap, mn, a.c, a.dv, status, s, a.rlist + (t & 1) * M,
                              a.rcount + (t & 1), N);
        if (e != cudaSuccess) return e;
        k_pf_fixup<<<gr, kTileThreads, 0, s>>>(a, t, path == 2);
        note_launch();
      } else {
        k_pf_resample_local<<<gr, kTileThreads, 0, s>>>(a, t);
        note_launch();
      }
    } else {
      e = cudaMemsetAsync(resampled, 0, M * T, s);
      if (e != cudaSuccess) return e;
    }
    if (N % 4 == 0)
      k_pf_step<true><<<dim3((unsigned)a.tiles, (unsigned)M), kTileThreads, 0, s>>>(a, t);
    else
      k_pf_step<false><<<dim3((unsigned)a.tiles, (unsigned)M), kTileThreads, 0, s>>>(a, t);
    note_launch();
  }
  return cudaGetLastError();
}

}  // namespace pfr
