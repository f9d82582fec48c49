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

#include <algorithm>

#include <cooperative_groups.h>

#include "pfr_hier.cuh"
#include "pfr_internal.h"
#include "pfr_tile.cuh"

namespace cg = cooperative_groups;

namespace pfr {

namespace {

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

constexpr unsigned kScanRepair = 0x10u;  // DvState.flags: the scan output needs the running-max repair

__device__ __forceinline__ void griddep_wait_scan() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---------------------------------------------------------------------------
// Two-pass scan (inclusive_prefix_sum / exclusive_prefix_sum / vector_sum,
// primitives.py:34-66; offspring_to_cumulative, ancestry.py:85-88).
// S1: one CTA per tile, tile aggregate in the in-tile association of S2,
//     validation flags, hierarchical tile prefixes (pfr_hier.cuh).
// S2: one CTA per tile, re-reads its tile (L2), out = tile prefix + in-tile
//     scan; flags ulp-level decreases (a parallel association is not the
//     reference's serial fold) for the rare-path running-max repair S3.
template <typename T, typename A, bool kFloat>
__global__ void __launch_bounds__(kTileThreads) k_sc_reduce(const T* __restrict__ in, int64_t n, Hier<A> h,
                                                             uint32_t* status, uint32_t fmask) {
  __shared__ A warp_sums[kTileThreads / 32];
  __shared__ uint32_t cta_flags;
  __shared__ int stage;
  const int64_t b = blockIdx.x;
  if (threadIdx.x == 0) cta_flags = 0;
  {
    T x[kTileItems];
    tile_load_any<T>(in, n, b * kTile, x);
    uint32_t f = 0;
    TileScan<A> s;
    if constexpr (kFloat) {
      FlagAcc<T> acc;
#pragma unroll
      for (int j = 0; j < kTileItems; ++j) acc.add(x[j]);
      f = acc.flags() & fmask;  // NONFINITE, plus NEGATIVE | POSITIVE for weights
    } else {
#pragma unroll
      for (int j = 0; j < kTileItems; ++j)
        if (x[j] < T(0)) f |= PFR_ST_NEGCOUNT;
    }
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) s.loc[j] = (A)x[j];
    tile_scan<A>(s, warp_sums);
    if (threadIdx.x == kTileThreads - 1) h.agg[b] = add_rn(s.thread_excl, s.loc[kTileItems - 1]);
    f = __reduce_or_sync(0xffffffffu, f);
    if ((threadIdx.x & 31) == 0 && f) atomicOr(&cta_flags, f);
  }
  hier_tile_done(h, b, &cta_flags, &stage, status);
  if (stage == 2 && threadIdx.x == 0) h.state->flags = 0;
}

template <typename T, typename A, typename U, bool kFloat>
__global__ void __launch_bounds__(kTileThreads)
    k_sc_apply(const T* in, U* out, int64_t n, Hier<A> h, int exclusive, int repair, void* total_out,
               int64_t expect_total, uint32_t* status) {
  constexpr size_t kStageOut = kTile * sizeof(U) / 16;
  __shared__ __align__(16) uint4 stage[kStageOut];
  __shared__ A warp_sums[kTileThreads / 32];
  __shared__ A wlast[kTileThreads / 32];
  griddep_wait_scan();
  const int64_t b = blockIdx.x;
  const int64_t base = b * kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x[kTileItems];
  tile_load_any<T>(in, n, base, x);
  TileScan<A> s;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) s.loc[j] = (A)x[j];
  tile_scan<A>(s, warp_sums);
  const A ex = b ? h.tile_excl(b) : A(0);
  const A prev_tile_end = b ? h.tile_end(b - 1) : A(0);
  A v[kTileItems];
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) v[j] = add_rn(ex, add_rn(s.thread_excl, s.loc[j]));
  // value before this thread's first element
  A prev = __shfl_up_sync(0xffffffffu, v[kTileItems - 1], 1);
  if (lane == 31) wlast[warp] = v[kTileItems - 1];
  __syncthreads();
  if (lane == 0) prev = warp ? wlast[warp - 1] : prev_tile_end;
  const int e0 = threadIdx.x * kTileItems;
  const int64_t len = min((int64_t)kTile, n - base);
  if (kFloat && repair) {
    bool bad = e0 < len && (b > 0 || e0 > 0) && v[0] < prev;
#pragma unroll
    for (int j = 1; j < kTileItems; ++j) bad |= e0 + j < len && v[j] < v[j - 1];
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&h.state->flags, kScanRepair);
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
#pragma unroll
    for (int j = kTileItems - 1; j > 0; --j) y[j] = (U)v[j - 1];
    y[0] = (U)prev;
  }
  tile_store<U>(out, n, base, stage, y, policy_evict_first());
}

// S3 (rare path, cooperative; returns at once unless S2 flagged a decrease):
// out = running max of out (exact), status REPAIRED, total = max.
template <typename U>
__global__ void __launch_bounds__(kTileThreads) k_sc_repair(U* out, int64_t n, int64_t tiles, DvState* state,
                                                             U* tmax, int exclusive, void* total_out,
                                                             uint32_t* status) {
  __shared__ U smax8[kTileThreads / 32];
  griddep_wait_scan();
  if (!(*(volatile unsigned*)&state->flags & kScanRepair)) return;
  cg::grid_group grid = cg::this_grid();
  // A: per-tile maxima
  for (int64_t b = blockIdx.x; b < tiles; b += gridDim.x) {
    U m = -INFINITY;
    for (int64_t i = b * kTile + threadIdx.x; i < min(n, (b + 1) * kTile); i += kTileThreads) m = fmax(m, out[i]);
    U bm;
    block_excl_max<U>(m, (U)-INFINITY, smax8, bm);
    if (threadIdx.x == 0) tmax[b] = bm;
  }
  grid.sync();
  // B: exclusive max over tiles (serial: rare path)
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    U run = -INFINITY;
    for (int64_t b = 0; b < tiles; ++b) {
      const U v = tmax[b];
      tmax[b] = run;
      run = fmax(run, v);
    }
    if (total_out) *reinterpret_cast<double*>(total_out) = fmax(*reinterpret_cast<double*>(total_out), (double)run);
    status_or(status, PFR_ST_REPAIRED);
  }
  grid.sync();
  // C: apply, one thread per tile segment of 16 (serial within, block max-scan across)
  for (int64_t b = blockIdx.x; b < tiles; b += gridDim.x) {
    const int64_t i0 = b * kTile + threadIdx.x * kTileItems;
    U loc[kTileItems];
    U m = -INFINITY;
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
      loc[j] = i0 + j < n ? out[i0 + j] : (U)-INFINITY;
      m = fmax(m, loc[j]);
    }
    U bm;
    const U before = block_excl_max<U>(m, (U)-INFINITY, smax8, bm);
    U run = fmax(before, tmax[b]);
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
      run = fmax(run, loc[j]);
      if (i0 + j < n) out[i0 + j] = run;
    }
  }
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) state->flags &= ~kScanRepair;
}

// ---------------------------------------------------------------------------
// Serial fold (accum = PFR_ACC_SERIAL): np.cumsum bit for bit.  The reference
// scan is a strict left-to-right fold in the input dtype (primitives.py:34-51,
// vector_sum 60-66); floating-point addition does not associate, so the only
// way to reproduce every rounding is to perform the same additions in the
// same order.  One CTA: thread 0 folds a 4096-element chunk staged in shared
// memory (independent shared loads hoisted ahead of the dependent add chain:
// ~4-5 cycles per element), while warps 1..7 store the previous chunk and
// load the next one (three rotating buffers).  Parity mode: ~2.3 ms at 2^20.
constexpr int kSerChunk = 4096;

template <typename T, typename U>
__global__ void __launch_bounds__(256) k_scan_serial(const T* __restrict__ in, U* __restrict__ out, int64_t n,
                                                     int exclusive, double* total_out, uint32_t* status,
                                                     uint32_t fmask, DvState* state) {
  extern __shared__ __align__(16) unsigned char ser_smem[];
  T* buf = reinterpret_cast<T*>(ser_smem);  // [3][kSerChunk]
  const int64_t chunks = (n + kSerChunk - 1) / kSerChunk;
  FlagAcc<T> facc;
  auto load = [&](int64_t c) {
    T* dst = buf + (c % 3) * kSerChunk;
    const int64_t base = c * kSerChunk;
    const int len = (int)min((int64_t)kSerChunk, n - base);
    for (int i = threadIdx.x - 32; i < len; i += blockDim.x - 32) {
      const T v = __ldcs(in + base + i);
      facc.add(v);
      dst[i] = v;
    }
  };
  auto store = [&](int64_t c) {
    const T* src = buf + (c % 3) * kSerChunk;
    const int64_t base = c * kSerChunk;
    const int len = (int)min((int64_t)kSerChunk, n - base);
    for (int i = threadIdx.x - 32; i < len; i += blockDim.x - 32) __stcs(out + base + i, (U)src[i]);
  };
  if (threadIdx.x >= 32) load(0);
  __syncthreads();
  T acc = T(0);
  for (int64_t c = 0; c < chunks; ++c) {
    if (threadIdx.x == 0) {
      T* cur = buf + (c % 3) * kSerChunk;
      const int len = (int)min((int64_t)kSerChunk, n - c * kSerChunk);
      int i = 0;
      for (; i + 8 <= len; i += 8) {
        T v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = cur[i + j];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const T nv = add_rn(acc, v[j]);
          cur[i + j] = exclusive ? acc : nv;
          acc = nv;
        }
      }
      for (; i < len; ++i) {
        const T nv = add_rn(acc, cur[i]);
        cur[i] = exclusive ? acc : nv;
        acc = nv;
      }
    } else if (threadIdx.x >= 32) {
      if (c > 0) store(c - 1);
      if (c + 1 < chunks) load(c + 1);
    }
    __syncthreads();
  }
  if (threadIdx.x >= 32) store(chunks - 1);
  if (threadIdx.x == 0) {
    if (total_out) *total_out = (double)acc;
    if (state) state->flags = 0;  // pipeline flags of a delivery that consumes this scan
  }
  if (threadIdx.x >= 32) status_or_warp(status, facc.flags() & fmask);
}

// ---------------------------------------------------------------------------
// check_weights (diagnostics.py:38-51): 16-byte vector loads, four in flight
// per thread, flags from integer maxima of the bit patterns (FlagAcc)
template <typename T>
__global__ void __launch_bounds__(256) k_check_weights(const T* __restrict__ w, int64_t n, uint32_t* status) {
  constexpr int kPer = 16 / sizeof(T);
  FlagAcc<T> acc;
  const int64_t nvec = ((reinterpret_cast<uintptr_t>(w) & 15) == 0) ? n / kPer : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; v + 3 * stride < nvec; v += 4 * stride) {
    uint4 x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = __ldcs(reinterpret_cast<const uint4*>(w) + v + k * stride);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const T* e = reinterpret_cast<const T*>(&x[k]);
#pragma unroll
      for (int t = 0; t < kPer; ++t) acc.add(e[t]);
    }
  }
  for (; v < nvec; v += stride) {
    const uint4 x = __ldcs(reinterpret_cast<const uint4*>(w) + v);
    const T* e = reinterpret_cast<const T*>(&x);
#pragma unroll
    for (int t = 0; t < kPer; ++t) acc.add(e[t]);
  }
  for (int64_t i = nvec * kPer + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) acc.add(w[i]);
  status_or_warp(status, acc.flags());
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

template <typename K, typename... Args>
cudaError_t launch_ex(K kernel, dim3 grid, dim3 block, cudaStream_t s, bool pdl, bool cooperative, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cooperative) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  note_launch();
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <typename T, typename A, typename U, bool kFloat>
cudaError_t scan_typed(const void* in, void* out, int64_t n, int exclusive, int repair, void* total,
                       int64_t expect_total, uint32_t* status, const Workspace& ws, cudaStream_t s,
                       uint32_t fmask) {
  const int64_t tiles = num_tiles(n);
  A* agg = reinterpret_cast<A*>(ws.sum_cells);
  Hier<A> h{agg, reinterpret_cast<A*>(ws.max_cells), agg + tiles + 8, ws.dv, tiles};
  cudaError_t e = launch_ex(k_sc_reduce<T, A, kFloat>, dim3((unsigned)tiles), dim3(kTileThreads), s, false, false,
                            (const T*)in, n, h, status, fmask);
  if (e != cudaSuccess) return e;
  e = launch_ex(k_sc_apply<T, A, U, kFloat>, dim3((unsigned)tiles), dim3(kTileThreads), s, true, false,
                (const T*)in, (U*)out, n, h, exclusive, repair, total, expect_total, status);
  if (e != cudaSuccess) return e;
  if constexpr (kFloat) {
    if (repair) {
      // tile maxima scratch: the sum-tree region past the aggregates and group totals
      U* tmax = reinterpret_cast<U*>(agg + tiles + 8 + (tiles + kGroupTiles - 1) / kGroupTiles + 8);
      // cooperative, launched every time (exits unless flagged): a small grid
      // co-resides with concurrent work (see rare_grid in pfr_deliver.cu)
      e = launch_ex(k_sc_repair<U>, dim3(16u), dim3(kTileThreads), s, true, true, (U*)out, n, tiles,
                    ws.dv, tmax, exclusive, total, status);
    }
  }
  return e;
}

template <typename T, typename U>
cudaError_t launch_scan_serial(const void* in, void* out, int64_t n, int exclusive, void* total, uint32_t* status,
                               uint32_t fmask, DvState* state, cudaStream_t s) {
  const size_t smem = 3 * kSerChunk * sizeof(T);
  auto kernel = k_scan_serial<T, U>;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kernel<<<1, 256, smem, s>>>((const T*)in, (U*)out, n, exclusive, (double*)total, status, fmask, state);
  note_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_scan(const void* in, void* out, int64_t n, int dtype, int out_dtype, int accum, int exclusive,
                        void* total, int64_t expect_total, uint32_t* status, const Workspace& ws, cudaStream_t s) {
  const int repair = (accum & PFR_SCAN_MONOTONE) ? 1 : 0;
  const bool native = (accum & 0xFF) == PFR_ACC_NATIVE;
  const uint32_t fmask =
      PFR_ST_NONFINITE | ((accum & PFR_SCAN_WEIGHTS) ? (uint32_t)(PFR_ST_NEGATIVE | PFR_ST_POSITIVE) : 0u);
  if ((accum & 0xFF) == PFR_ACC_SERIAL && (dtype == PFR_F32 || dtype == PFR_F64)) {
    // the serial fold runs in the input dtype; the output is converted after
    if (dtype == PFR_F64)
      return launch_scan_serial<double, double>(in, out, n, exclusive, total, status, fmask, nullptr, s);
    if (out_dtype == PFR_F64)
      return launch_scan_serial<float, double>(in, out, n, exclusive, total, status, fmask, nullptr, s);
    return launch_scan_serial<float, float>(in, out, n, exclusive, total, status, fmask, nullptr, s);
  }
#define PFR_SCAN_ARGS in, out, n, exclusive, repair, total, expect_total, status, ws, s, fmask
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

cudaError_t launch_serial_weights_scan(const void* w, void* W, int64_t n, int dtype, uint32_t* status, DvState* state,
                                      cudaStream_t s) {
  const uint32_t fmask = PFR_ST_NONFINITE | PFR_ST_NEGATIVE | PFR_ST_POSITIVE;
  if (dtype == PFR_F64) return launch_scan_serial<double, double>(w, W, n, 0, nullptr, status, fmask, state, s);
  return launch_scan_serial<float, float>(w, W, n, 0, nullptr, status, fmask, state, s);
}

cudaError_t launch_check_weights(const void* w, int64_t n, int dtype, uint32_t* status, cudaStream_t s) {
  const int64_t vecs = n * (dtype == PFR_F64 ? 8 : 4) / 16;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((vecs + 1023) / 1024, (int64_t)num_sms() * 8));
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

// max of the log-weights (ordered bits) into *cell, with the validation flags
cudaError_t launch_logw_max(const void* lw, int64_t n, int dtype, unsigned long long* cell, uint32_t* status,
                            cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(cell, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  const int g = grid_for(n, 256);
  if (dtype == PFR_F64)
    k_logw_max<double><<<g, 256, 0, s>>>((const double*)lw, n, cell, status);
  else
    k_logw_max<float><<<g, 256, 0, s>>>((const float*)lw, n, cell, status);
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
