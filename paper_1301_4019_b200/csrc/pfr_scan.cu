// Prefix sums, cumulative offspring, weight validation, log-weight adapter.
//
// Reference: primitives.py:34-66 (scans), resamplers.py:105-153 (cumulative
// offspring), diagnostics.py:38-51 (check_weights), 138-155 (log weights).
//
// Kernels (all HBM bound; bytes per element in DESIGN.md):
//   k_tile_sums   -- pass 1 of the offspring path: read w once, validate
//                    (finite / >= 0 / any > 0), publish tile sums into the
//                    deterministic lookback tree; the tile holding w[N-1]
//                    publishes W[N-1] (the normaliser).
//   k_offspring   -- pass 2: re-read w (L2-resident at the sizes that matter),
//                    rebuild W from the tree, O = min(N, floor(N W/W[N-1] + u)),
//                    running-max repair through a second (max) tree, store O.
//   k_scan        -- single-pass inclusive/exclusive scan with the same tree.
#include <cmath>

#include "pfr_internal.h"
#include "pfr_tile.cuh"

namespace pfr {

namespace {

constexpr unsigned kTicketPass1 = 0;
constexpr unsigned kTicketPass2 = 1;
constexpr unsigned kTicketScan = 2;

template <typename T>
__device__ __forceinline__ uint32_t weight_flags(T x) {
  uint32_t f = 0;
  if (!isfinite((double)x)) f |= PFR_ST_NONFINITE;
  if (x < T(0)) f |= PFR_ST_NEGATIVE;
  if (x > T(0)) f |= PFR_ST_POSITIVE;
  return f;
}

template <typename A>
__device__ __forceinline__ A mul_rn(A a, A b);
template <>
__device__ __forceinline__ double mul_rn(double a, double b) {
  return __dmul_rn(a, b);
}
template <>
__device__ __forceinline__ float mul_rn(float a, float b) {
  return __fmul_rn(a, b);
}
template <typename A>
__device__ __forceinline__ A div_rn(A a, A b);
template <>
__device__ __forceinline__ double div_rn(double a, double b) {
  return __ddiv_rn(a, b);
}
template <>
__device__ __forceinline__ float div_rn(float a, float b) {
  return __fdiv_rn(a, b);
}

__device__ __forceinline__ int64_t floor_to_i64(double x) { return (int64_t)floor(x); }
__device__ __forceinline__ int64_t floor_to_i64(float x) { return (int64_t)floorf(x); }

// ---------------------------------------------------------------------------
// pass 1: tile sums + validation + normaliser
template <typename T, typename A>
__global__ void __launch_bounds__(kTileThreads) k_tile_sums(const T* __restrict__ w, int64_t n, Tree tree,
                                                             WsHeader* hdr, uint32_t* status) {
  __shared__ __align__(16) uint4 stage[kTile * sizeof(T) / 16];
  __shared__ A warp_sums[kTileThreads / 32];
  __shared__ int slot;
  const int64_t b = acquire_tile(&hdr->ticket[kTicketPass1], &slot);
  const int64_t base = b * kTile;
  const uint64_t pol = policy_evict_last();  // keep w in L2 for pass 2
  T x[kTileItems];
  tile_load<T>(w, n, base, stage, pol, x);
  TileScan<A> s;
  uint32_t flags = 0;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) {
    const bool valid = base + threadIdx.x * kTileItems + j < n;
    if (valid) flags |= weight_flags(x[j]);
    s.loc[j] = (A)x[j];
  }
  status_or_warp(status, flags);
  tile_scan<A>(s, warp_sums);
  if (threadIdx.x == 0) tree_publish<A, SumOp>(tree, b, s.tile_total);
  // the tile holding w[N-1] computes the normaliser W[N-1]
  if (b == tree.tiles - 1) {
    A prefix = A(0);
    __syncwarp();
    if (threadIdx.x < 32) prefix = tree_prefix<A, SumOp>(tree, b, A(0));
    if (threadIdx.x == 0) warp_sums[0] = prefix;
    __syncthreads();
    prefix = warp_sums[0];
    const int64_t p = (n - 1) - base;
    if (threadIdx.x == p / kTileItems) {
      const A basev = add_rn(prefix, s.thread_excl);
      A wl = s.loc[0];
#pragma unroll
      for (int j = 0; j < kTileItems; ++j)
        if (j == p % kTileItems) wl = s.loc[j];
      const A total = add_rn(basev, wl);
      st_relaxed_u64(&hdr->cell[0], Cell<A>::encode(total));
    }
  }
}

// ---------------------------------------------------------------------------
// pass 2: cumulative offspring
enum UMode { kUSystematic = 0, kUArray = 1, kUNumpy = 2, kUPhilox = 3 };

template <typename T, typename A, int UM>
__device__ __forceinline__ A stratum_offset(int64_t k0based, A u_sys, const double* __restrict__ uniforms,
                                            Key2x64 key) {
  if constexpr (UM == kUSystematic) {
    return u_sys;
  } else if constexpr (UM == kUArray) {
    return (A)(T)uniforms[k0based];  // cast to the weight dtype (resamplers.py:124)
  } else if constexpr (UM == kUNumpy) {
    return (A)(T)u64_to_unit(numpy_raw64(key, (uint64_t)k0based));
  } else {
    uint32_t o[4];
    philox4x32_10((uint32_t)(k0based >> 2), (uint32_t)(k0based >> 34), kTagStratified, 0, (uint32_t)key.k0,
                  (uint32_t)(key.k0 >> 32), o);
    const uint32_t r = o[k0based & 3];
    return (A)(T)u32_to_unit_d(r);
  }
}

template <typename T, typename A, int UM>
__global__ void __launch_bounds__(kTileThreads)
    k_offspring(const T* __restrict__ w, int64_t n, Tree sum_tree, Tree max_tree, WsHeader* hdr, A u_sys,
                const double* __restrict__ uniforms, Key2x64 key, int32_t* __restrict__ O, uint32_t* status) {
  __shared__ __align__(16) uint4 stage[kTile * sizeof(T) / 16 > kTile * 4 / 16 ? kTile * sizeof(T) / 16
                                                                                 : kTile * 4 / 16];
  __shared__ A warp_sums[kTileThreads / 32];
  __shared__ int64_t imax8[kTileThreads / 32];
  __shared__ int slot;
  __shared__ A sh_prefix;
  __shared__ int64_t sh_pmax;
  const int64_t b = acquire_tile(&hdr->ticket[kTicketPass2], &slot);
  const int64_t base = b * kTile;
  T x[kTileItems];
  tile_load<T>(w, n, base, stage, policy_evict_first(), x);
  TileScan<A> s;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) s.loc[j] = (A)x[j];
  tile_scan<A>(s, warp_sums);
  if (threadIdx.x < 32) {
    const A p = tree_prefix<A, SumOp>(sum_tree, b, A(0));
    if (threadIdx.x == 0) sh_prefix = p;
  }
  __syncthreads();
  const A total = Cell<A>::decode(ld_relaxed_u64(&hdr->cell[0]));
  const A nA = (A)n;
  const A basev = add_rn(sh_prefix, s.thread_excl);
  int32_t o[kTileItems];
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) {
    const A W = add_rn(basev, s.loc[j]);
    const A r = div_rn(mul_rn(W, nA), total);
    int64_t k = floor_to_i64(r) + 1;  // 1-based stratum
    if (k > n) k = n;
    if (k < 1) k = 1;
    const A u = stratum_offset<T, A, UM>(k - 1, u_sys, uniforms, key);
    int64_t ov = floor_to_i64(add_rn(r, u));
    if (ov > n) ov = n;
    if (ov < 0) ov = 0;
    o[j] = (int32_t)ov;
  }
  // running-max repair (resamplers.py:150): exact, order independent
  const int64_t my_max = o[kTileItems - 1];
  int64_t tile_max;
  const int64_t before = block_excl_max<int64_t>(my_max, INT64_MIN, imax8, tile_max);
  if (threadIdx.x == 0) tree_publish<int64_t, MaxOp>(max_tree, b, tile_max);
  __syncwarp();
  if (threadIdx.x < 32) {
    const int64_t pm = tree_prefix<int64_t, MaxOp>(max_tree, b, INT64_MIN);
    if (threadIdx.x == 0) sh_pmax = pm;
  }
  __syncthreads();
  const int64_t floor_v = MaxOp::combine(sh_pmax, before);
  uint32_t repaired = 0;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) {
    if (o[j] < floor_v) {
      o[j] = (int32_t)floor_v;
      repaired = PFR_ST_REPAIRED;
    }
    if (base + threadIdx.x * kTileItems + j == n - 1) o[j] = (int32_t)n;  // O[-1] = N
  }
  status_or_warp(status, repaired);
  tile_store<int32_t>(O, n, base, stage, o, policy_evict_last());
}

// ---------------------------------------------------------------------------
// single-pass scan (inclusive or exclusive) with monotone repair for floats
template <typename T, typename A, typename U, bool kFloat>
__global__ void __launch_bounds__(kTileThreads)
    k_scan(const T* __restrict__ in, U* __restrict__ out, int64_t n, Tree sum_tree, Tree max_tree, WsHeader* hdr,
           int exclusive, int repair, void* total_out, int64_t expect_total, uint32_t* status) {
  constexpr size_t kStageIn = kTile * sizeof(T) / 16;
  constexpr size_t kStageOut = kTile * sizeof(U) / 16;
  __shared__ __align__(16) uint4 stage[kStageIn > kStageOut ? kStageIn : kStageOut];
  __shared__ A warp_sums[kTileThreads / 32];
  __shared__ A amax8[kTileThreads / 32];
  __shared__ A wlast[kTileThreads / 32];
  __shared__ int slot;
  __shared__ A sh_prefix, sh_pmax;
  const int64_t b = acquire_tile(&hdr->ticket[kTicketScan], &slot);
  const int64_t base = b * kTile;
  T x[kTileItems];
  tile_load<T>(in, n, base, stage, policy_evict_first(), x);
  TileScan<A> s;
  uint32_t flags = 0;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) {
    const bool valid = base + threadIdx.x * kTileItems + j < n;
    if constexpr (kFloat) {
      if (valid && !isfinite((double)x[j])) flags |= PFR_ST_NONFINITE;
    } else {
      if (valid && x[j] < T(0)) flags |= PFR_ST_NEGCOUNT;
    }
    s.loc[j] = (A)x[j];
  }
  status_or_warp(status, flags);
  tile_scan<A>(s, warp_sums);
  if (threadIdx.x == 0) tree_publish<A, SumOp>(sum_tree, b, s.tile_total);
  __syncwarp();
  if (threadIdx.x < 32) {
    const A p = tree_prefix<A, SumOp>(sum_tree, b, A(0));
    if (threadIdx.x == 0) sh_prefix = p;
  }
  __syncthreads();
  const A basev = add_rn(sh_prefix, s.thread_excl);
  A v[kTileItems];
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) v[j] = add_rn(basev, s.loc[j]);
  A prev_tile_last = A(0);  // W of the element before this tile
  if (kFloat && !repair) {
    // no repair: the exclusive shift needs the raw W at the end of tile b-1,
    // published per tile (depends only on the sum tree: no serial chain)
    if (threadIdx.x == kTileThreads - 1) st_relaxed_u64(&max_tree.cells[b], Cell<A>::encode(v[kTileItems - 1]));
    if (exclusive && threadIdx.x == 0 && b > 0) sh_pmax = cell_wait<A>(&max_tree.cells[b - 1]);
    __syncthreads();
    prev_tile_last = b ? sh_pmax : A(0);
  } else if constexpr (kFloat) {
    // W_raw is monotone inside a thread; repair across threads and tiles with a
    // running max (exact): W = max(prefix max of earlier tiles, earlier threads, own)
    const A ident = -INFINITY;
    A tile_max;
    const A before = block_excl_max<A>(v[kTileItems - 1], ident, amax8, tile_max);
    if (threadIdx.x == 0) tree_publish<A, MaxOp>(max_tree, b, tile_max);
    __syncwarp();
    if (threadIdx.x < 32) {
      const A pm = tree_prefix<A, MaxOp>(max_tree, b, ident);
      if (threadIdx.x == 0) sh_pmax = pm;
    }
    __syncthreads();
    const A fl = MaxOp::combine(sh_pmax, before);
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) v[j] = MaxOp::combine(fl, v[j]);
    prev_tile_last = (b == 0) ? A(0) : sh_pmax;
  } else {
    prev_tile_last = sh_prefix;
  }
  // total = W[N-1]
  {
    const int64_t p = (n - 1) - base;
    if (p >= 0 && p < kTile && threadIdx.x == p / kTileItems) {
      A t = v[0];
#pragma unroll
      for (int j = 0; j < kTileItems; ++j)
        if (j == p % kTileItems) t = v[j];
      if constexpr (kFloat) {
        if (total_out) *reinterpret_cast<double*>(total_out) = (double)t;
      } else {
        if (total_out) *reinterpret_cast<int64_t*>(total_out) = (int64_t)t;
        if (expect_total >= 0 && (int64_t)t != expect_total) status_or(status, PFR_ST_BADSUM);
      }
    }
  }
  U y[kTileItems];
  if (!exclusive) {
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) y[j] = (U)v[j];
  } else {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    A prev = __shfl_up_sync(0xffffffffu, v[kTileItems - 1], 1);
    if (lane == 31) wlast[warp] = v[kTileItems - 1];
    __syncthreads();
    if (lane == 0) prev = (warp == 0) ? prev_tile_last : wlast[warp - 1];
#pragma unroll
    for (int j = kTileItems - 1; j > 0; --j) y[j] = (U)v[j - 1];
    y[0] = (U)prev;
  }
  tile_store<U>(out, n, base, stage, y, policy_evict_first());
}

// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_check_weights(const T* __restrict__ w, int64_t n, uint32_t* status) {
  uint32_t f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    f |= weight_flags(w[i]);
  status_or_warp(status, f);
}

template <typename T, typename U, bool kCumulative>
__global__ void k_adjacent_difference(const T* __restrict__ in, U* __restrict__ out, int64_t n, uint32_t* status) {
  uint32_t f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const T cur = in[i];
    const T prev = i ? in[i - 1] : T(0);
    if constexpr (kCumulative) {
      if (i == 0 && cur < T(0)) f |= PFR_ST_NEGCOUNT;
      if (i > 0 && cur < prev) f |= PFR_ST_NOTMONOTONE;
      if (i == n - 1 && (int64_t)cur != n) f |= PFR_ST_BADEND;
    } else {
      if (!isfinite((double)cur)) f |= PFR_ST_NONFINITE;
    }
    out[i] = (U)(cur - prev);
  }
  status_or_warp(status, f);
}

// log-weights: ordered-integer max (exact) then exp(lw - max)
__device__ __forceinline__ unsigned long long ordered_bits(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_ordered(unsigned long long o) {
  unsigned long long b = (o & 0x8000000000000000ull) ? (o & 0x7FFFFFFFFFFFFFFFull) : ~o;
  return __longlong_as_double((long long)b);
}

template <typename T>
__global__ void k_logw_max(const T* __restrict__ lw, int64_t n, unsigned long long* cell, uint32_t* status) {
  unsigned long long m = 0;  // below every ordered value of a real number
  uint32_t f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = (double)lw[i];
    if (x != x || x == INFINITY) {
      f |= PFR_ST_NONFINITE;
      continue;
    }
    if (x > -INFINITY) f |= PFR_ST_POSITIVE;
    const unsigned long long o = ordered_bits(x);
    m = o > m ? o : m;
  }
  for (int off = 16; off; off >>= 1) {
    unsigned long long o = __shfl_xor_sync(0xffffffffu, m, off);
    m = o > m ? o : m;
  }
  if ((threadIdx.x & 31) == 0 && m) atomicMax(cell, m);
  status_or_warp(status, f);
}

template <typename T>
__global__ void k_logw_exp(const T* __restrict__ lw, T* __restrict__ w, int64_t n,
                           const unsigned long long* cell) {
  const T m = (T)from_ordered(*cell);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if constexpr (sizeof(T) == 8)
      w[i] = exp(lw[i] - m);
    else
      w[i] = expf(lw[i] - m);
  }
}

int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

Tree make_tree(uint64_t* cells, int64_t tiles) {
  Tree t;
  t.cells = cells;
  t.tiles = tiles;
  t.levels = tree_levels(tiles);
  return t;
}

template <typename T, typename A>
cudaError_t offspring_typed(const T* w, int64_t n, int stratified, double offset, const double* uniforms,
                            const pfr_rng* rng, int32_t* O, uint32_t* status, const Workspace& ws, cudaStream_t s) {
  const int64_t tiles = num_tiles(n);
  Tree sum_tree = make_tree(ws.sum_cells, tiles);
  Tree max_tree = make_tree(ws.max_cells, tiles);
  k_tile_sums<T, A><<<(unsigned)tiles, kTileThreads, 0, s>>>(w, n, sum_tree, ws.hdr, status);
  note_launch();
  Key2x64 key{rng ? rng->key0 : 0, rng ? rng->key1 : 0};
  const A u_sys = (A)(T)offset;  // systematic: u cast to the weight dtype (resamplers.py:135)
  if (!stratified) {
    k_offspring<T, A, kUSystematic>
        <<<(unsigned)tiles, kTileThreads, 0, s>>>(w, n, sum_tree, max_tree, ws.hdr, u_sys, nullptr, key, O, status);
  } else if (uniforms) {
    k_offspring<T, A, kUArray>
        <<<(unsigned)tiles, kTileThreads, 0, s>>>(w, n, sum_tree, max_tree, ws.hdr, u_sys, uniforms, key, O, status);
  } else if (rng && rng->mode == PFR_RNG_NUMPY) {
    k_offspring<T, A, kUNumpy>
        <<<(unsigned)tiles, kTileThreads, 0, s>>>(w, n, sum_tree, max_tree, ws.hdr, u_sys, nullptr, key, O, status);
  } else {
    k_offspring<T, A, kUPhilox>
        <<<(unsigned)tiles, kTileThreads, 0, s>>>(w, n, sum_tree, max_tree, ws.hdr, u_sys, nullptr, key, O, status);
  }
  note_launch();
  return cudaGetLastError();
}

template <typename T, typename A, typename U, bool kFloat>
cudaError_t scan_typed(const void* in, void* out, int64_t n, int exclusive, int repair, void* total,
                       int64_t expect_total, uint32_t* status, const Workspace& ws, cudaStream_t s) {
  const int64_t tiles = num_tiles(n);
  Tree sum_tree = make_tree(ws.sum_cells, tiles);
  Tree max_tree = make_tree(ws.max_cells, tiles);
  k_scan<T, A, U, kFloat><<<(unsigned)tiles, kTileThreads, 0, s>>>(
      (const T*)in, (U*)out, n, sum_tree, max_tree, ws.hdr, exclusive, repair, total, expect_total, status);
  note_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_offspring(const void* w, int64_t n, int dtype, int accum, int stratified, double offset,
                             const double* uniforms, const pfr_rng* rng, int32_t* O, uint32_t* status,
                             const Workspace& ws, cudaStream_t s) {
  cudaError_t e = workspace_reset(ws, s);
  if (e != cudaSuccess) return e;
  if (dtype == PFR_F64) return offspring_typed<double, double>((const double*)w, n, stratified, offset, uniforms, rng, O, status, ws, s);
  if (accum == PFR_ACC_NATIVE)
    return offspring_typed<float, float>((const float*)w, n, stratified, offset, uniforms, rng, O, status, ws, s);
  return offspring_typed<float, double>((const float*)w, n, stratified, offset, uniforms, rng, O, status, ws, s);
}

cudaError_t launch_scan(const void* in, void* out, int64_t n, int dtype, int out_dtype, int accum, int exclusive,
                        void* total, int64_t expect_total, uint32_t* status, const Workspace& ws, cudaStream_t s) {
  cudaError_t e = workspace_reset(ws, s);
  if (e != cudaSuccess) return e;
  const int repair = (accum & PFR_SCAN_MONOTONE) ? 1 : 0;
  const bool native = (accum & 0xFF) == PFR_ACC_NATIVE;
#define PFR_SCAN_ARGS in, out, n, exclusive, repair, total, expect_total, status, ws, s
  switch (dtype) {
    case PFR_F64:
      return scan_typed<double, double, double, true>(PFR_SCAN_ARGS);
    case PFR_F32:
      if (out_dtype == PFR_F64) return scan_typed<float, double, double, true>(PFR_SCAN_ARGS);
      if (native) return scan_typed<float, float, float, true>(PFR_SCAN_ARGS);
      return scan_typed<float, double, float, true>(PFR_SCAN_ARGS);
    case PFR_I32:
      if (out_dtype == PFR_I32) return scan_typed<int32_t, int64_t, int32_t, false>(PFR_SCAN_ARGS);
      return scan_typed<int32_t, int64_t, int64_t, false>(PFR_SCAN_ARGS);
    case PFR_I64:
      if (out_dtype == PFR_I32) return scan_typed<int64_t, int64_t, int32_t, false>(PFR_SCAN_ARGS);
      return scan_typed<int64_t, int64_t, int64_t, false>(PFR_SCAN_ARGS);
  }
#undef PFR_SCAN_ARGS
  return cudaErrorInvalidValue;
}

cudaError_t launch_check_weights(const void* w, int64_t n, int dtype, uint32_t* status, cudaStream_t s) {
  const int g = grid_for(n, 256);
  if (dtype == PFR_F64)
    k_check_weights<double><<<g, 256, 0, s>>>((const double*)w, n, status);
  else
    k_check_weights<float><<<g, 256, 0, s>>>((const float*)w, n, status);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_adjacent_difference(const void* in, void* out, int64_t n, int dtype, int out_dtype,
                                       uint32_t* status, cudaStream_t s) {
  const int g = grid_for(n, 256);
  switch (dtype) {
    case PFR_F64:
      k_adjacent_difference<double, double, false><<<g, 256, 0, s>>>((const double*)in, (double*)out, n, status);
      break;
    case PFR_F32:
      k_adjacent_difference<float, float, false><<<g, 256, 0, s>>>((const float*)in, (float*)out, n, status);
      break;
    case PFR_I32:
      if (out_dtype == PFR_I64)
        k_adjacent_difference<int32_t, int64_t, true><<<g, 256, 0, s>>>((const int32_t*)in, (int64_t*)out, n, status);
      else
        k_adjacent_difference<int32_t, int32_t, true><<<g, 256, 0, s>>>((const int32_t*)in, (int32_t*)out, n, status);
      break;
    case PFR_I64:
      if (out_dtype == PFR_I64)
        k_adjacent_difference<int64_t, int64_t, true><<<g, 256, 0, s>>>((const int64_t*)in, (int64_t*)out, n, status);
      else
        k_adjacent_difference<int64_t, int32_t, true><<<g, 256, 0, s>>>((const int64_t*)in, (int32_t*)out, n, status);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_logweights(const void* lw, void* w, int64_t n, int dtype, uint32_t* status, const Workspace& ws,
                              cudaStream_t s) {
  unsigned long long* cell = reinterpret_cast<unsigned long long*>(&ws.hdr->cell[1]);
  cudaError_t e = cudaMemsetAsync(cell, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  const int g = grid_for(n, 256);
  if (dtype == PFR_F64) {
    k_logw_max<double><<<g, 256, 0, s>>>((const double*)lw, n, cell, status);
    k_logw_exp<double><<<g, 256, 0, s>>>((const double*)lw, (double*)w, n, cell);
  } else {
    k_logw_max<float><<<g, 256, 0, s>>>((const float*)lw, n, cell, status);
    k_logw_exp<float><<<g, 256, 0, s>>>((const float*)lw, (float*)w, n, cell);
  }
  note_launch(2);
  return cudaGetLastError();
}

}  // namespace pfr
