// Batches of independent filters (SURVEY.md 8(e) "batched independent
// filters", 8(f) N1, BASELINE config 5): no communication, one CTA per filter.
//
//   k_deliver_batched  systematic delivery of M filters of N particles:
//                      permute_parallel(cumulative_offspring_to_ancestors(
//                      systematic_cumulative_offspring(w_m))) per filter
//                      (resamplers.py:127-153, ancestry.py:69-76, 139-174)
//   k_pf_init / k_pf_step / k_pf_resample
//                      the bootstrap particle filter of pf.py:111-204 on the
//                      linear-Gaussian model, M filters at once: ESS-triggered
//                      systematic resampling, the copy step fused with the
//                      propagation (out-of-place gather x'[i] = x[c[i]], which
//                      Eq. 2 makes equivalent to pf_copy_step, pf.py:86-97),
//                      weighting, normalisation, log-likelihood, filtered mean.
//
// The per-filter delivery runs inside one CTA: pass 1 folds the tile
// aggregates (tile association of pfr_tile.cuh, serial across tiles), pass 2
// recomputes W per element, O = min(N, floor((W*N)/W_N + u)) with the exact
// IEEE sequence, the running max (resamplers.py:150), and expands the slot
// words (pfr_expand.cuh); pass 3 resolves the in-place ancestry by walking
// the loser chains backwards (as k_dv_inplace).  Words live in a per-filter
// global scratch (L2-resident for N <= 2^16).
#include <cstdlib>
#include <algorithm>

#include "pfr_expand.cuh"
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
  double* part;         // [M, kPfSlices, 4] slice partials
  unsigned int* slice_done;  // [M] slices finished (reset by the last)
  double* means;        // [M, T]
  double* loglik;       // [M]
  double* ess;          // [M, T]
  uint8_t* resampled;   // [M, T]
  uint32_t k0, k1;
  uint32_t* status;
};

// two standard normals from one Philox call (Box-Muller in float: the
// transition noise of the model, pf.py:188-189)
__device__ __forceinline__ float2 normal2(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t tag, uint32_t k0,
                                          uint32_t k1) {
  uint32_t o[4];
  philox4x32_10(c0, c1, c2, tag, k0, k1, o);
  const float u1 = ((float)(o[0] >> 8) + 1.0f) * (1.0f / 16777216.0f);  // (0, 1]
  const float u2 = (float)(o[1] >> 8) * (1.0f / 16777216.0f);
  const float rad = sqrtf(-2.0f * logf(u1));
  float sn, cs;
  sincospif(2.0f * u2, &sn, &cs);
  return make_float2(rad * cs, rad * sn);
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

// resampling of the filters whose ESS fell below the threshold: passes 1-2
// of the delivery per filter CTA (slot words with GLOBAL parent numbers into a
// contiguous bitmap: N % 32 == 0), then one global in-place pass (K3 of the
// fused delivery, launch_dv_inplace) resolves every filter's chains at once
// (chains never leave a filter: its slots only name its own parents).  Other
// N: the per-CTA pass 3.  c holds global particle numbers.
template <bool kGlobal>
__global__ void __launch_bounds__(kTileThreads) k_pf_resample(PfArgs a, int64_t t) {
  __shared__ SegSmem S;
  if (blockIdx.x == 0 && threadIdx.x == 0) a.dv->flags = 0;  // K3 overflow flag of the previous step
  for (int64_t m = blockIdx.x; m < a.M; m += gridDim.x) {
    const bool go = a.need[m] != 0;
    if (threadIdx.x == 0) a.resampled[m * a.T + t] = go ? 1 : 0;
    if (!go) continue;
    const double u = philox_unit53((uint32_t)m, (uint32_t)t, kTagPfSys, a.k0, a.k1);
    int longest = 0;
    if constexpr (kGlobal) {
      segment_deliver<double, false>(a.w + m * a.N, a.N, u, a.words + m * a.N, a.bitmap + m * (a.N / 32), nullptr,
                                     longest, S, (uint32_t)(m * a.N));
    } else {
      segment_deliver<double, true>(a.w + m * a.N, a.N, u, a.words + m * a.N, a.bitmap + m * a.bitmap_stride,
                                    a.c + m * a.N, longest, S);
    }
    __syncthreads();
  }
}

// rare: a chain longer than K3's walk bound -- redo the in-place pass of the
// resampled filters with unbounded per-thread walks (global numbers)
__global__ void __launch_bounds__(kTileThreads) k_pf_fixup(PfArgs a, int force) {
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

// propagate (through the ancestry when resampled) + weight + per-filter
// reductions.  Grid (slices, M): kPfSlices CTAs per filter each reduce their
// contiguous slice; the last slice to finish (per-filter counter) folds the
// slice partials in slice order (deterministic) and finishes the filter.
constexpr int kPfSlices = 8;

__global__ void __launch_bounds__(256) k_pf_step(PfArgs a, int64_t t) {
  __shared__ double red[4][8];
  __shared__ bool last;
  const int64_t m = blockIdx.y;
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
  // this slice: pairs [p0, p1) of the filter
  const int64_t pairs = (n + 1) / 2;
  const int64_t p0 = pairs * blockIdx.x / gridDim.x, p1 = pairs * (blockIdx.x + 1) / gridDim.x;
  double su = 0.0, sux = 0.0, suu = 0.0, sw = 0.0;
  for (int64_t pp = p0 + threadIdx.x; pp < p1; pp += blockDim.x) {
    const int64_t i = 2 * pp;
    const float2 z = normal2((uint32_t)pp, (uint32_t)m, (uint32_t)t, kTagPfProp, a.k0, a.k1);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t k = i + h;
      if (k >= n) break;
      const double xo = res ? src[cm[k] - c_base] : src[k];
      const double wp = (res || t == 0) ? 1.0 : w[k];
      const double xn = a.coeff * xo + a.trans_std * (double)(h ? z.y : z.x);
      const double e = (y - xn) * inv_obs;
      const double u = wp * (dens_norm * exp(-0.5 * e * e));
      dst[k] = xn;
      w[k] = u;
      su += u;
      sux += u * xn;
      suu += u * u;
      sw += wp;
    }
  }
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
    double* part = a.part + (m * kPfSlices + blockIdx.x) * 4;
    for (int q = 0; q < 4; ++q) {
      double r = 0;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) r += red[q][k];
      part[q] = r;
    }
    __threadfence();
    last = atomicAdd(&a.slice_done[m], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  double r[4] = {0, 0, 0, 0};
  for (int sl = 0; sl < (int)gridDim.x; ++sl)
    for (int q = 0; q < 4; ++q) r[q] += __ldcg(a.part + (m * kPfSlices + sl) * 4 + q);
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
  a.need[m] = (ess_next / (double)n < a.ess_threshold) ? 1 : 0;
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
  add(M * 8 * 4 * 8);   // slice partials
  add(M * 4);           // slice counters
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
  a.part = reinterpret_cast<double*>(take(M * 8 * 4 * 8));
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
        k_pf_resample<true><<<gr, kTileThreads, 0, s>>>(a, t);
        note_launch();
        e = launch_dv_inplace(a.words, a.bitmap, mn, a.c, a.dv, status, s);
        if (e != cudaSuccess) return e;
        k_pf_fixup<<<gr, kTileThreads, 0, s>>>(a, path == 2);
        note_launch();
      } else {
        k_pf_resample<false><<<gr, kTileThreads, 0, s>>>(a, t);
        note_launch();
      }
    } else {
      e = cudaMemsetAsync(resampled, 0, M * T, s);
      if (e != cudaSuccess) return e;
    }
    k_pf_step<<<dim3(kPfSlices, (unsigned)M), 256, 0, s>>>(a, t);
    note_launch();
  }
  return cudaGetLastError();
}

}  // namespace pfr
