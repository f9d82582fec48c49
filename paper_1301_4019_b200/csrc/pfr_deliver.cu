// Fused systematic / stratified delivery: weights -> in-place-valid ancestry.
//
// Computes permute_parallel(cumulative_offspring_to_ancestors(O)) with
// O = systematic_cumulative_offspring(w) or stratified_... (ancestry.py:69-76,
// 139-174; resamplers.py:105-153) -- the timed region of the reference's
// bench.py:155-161 for the offspring algorithms -- in three HBM-streaming
// kernels chained with programmatic dependent launch:
//
//   K1 k_dv_reduce   read w once: validation flags and the per-tile
//                    aggregate (the in-tile association of K2); tile prefixes
//                    built hierarchically (pfr_hier.cuh): deterministic, no
//                    single-CTA tail.
//   K2 k_dv_expand   re-read w (L2), W = tile prefix + in-tile scan, O from the
//                    position formula (fixed-point fast path, exact IEEE
//                    sequence near integers), then the sorted ancestry as
//                    32-bit slot words  parent | FIRST(slot is its parent's
//                    first slot)  over the tile's slot range (pfr_expand.cuh),
//                    plus the has-offspring bitmap.  No global atomics.
//   K3 k_dv_inplace  one pass over the indices: c[x] = x if x has offspring;
//                    a hole h walks BACKWARDS: while slot z is a first slot,
//                    z = parent(z); then c[h] = parent(z).  This is the
//                    reference's loser chain read from its end (the chain
//                    L -> d[L] -> ... -> h has d[y] = first slot of y), so
//                    every c[x] is written exactly once (coalesced for the
//                    trivial cases, queued chain walks for the rest).
//
// Rare paths, all inside one cooperative kernel k_dv_rare that returns at once
// when not needed: (a) ulp-level non-monotone O (W is not a strict serial
// fold) -> global running-max repair (resamplers.py:150) and recomputation;
// (b) a chain longer than the walk bound -> pointer jumping (Wyllie) over the
// claim graph.
#include <cooperative_groups.h>

#include <cstdlib>

#include "pfr_expand.cuh"
#include "pfr_fx.cuh"
#include "pfr_hier.cuh"
#include "pfr_inplace.cuh"
#include "pfr_internal.h"
#include "pfr_tile.cuh"

namespace cg = cooperative_groups;

namespace pfr {

namespace {


constexpr uint32_t kNeedsRepair = 1u;
constexpr uint32_t kOverflow = 2u;

__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename A>
struct DvArgs {
  const void* w;
  int64_t n;
  int64_t tiles;
  A* agg;        // [tiles]
  A* excl;       // see K1: in-group tile prefixes, total, group prefixes, tile flags
  A* sum_scratch;  // [groups] group totals
  A u_sys;       // systematic offset (cast to the weight dtype)
  const double* uniforms;
  Key2x64 key;
  uint32_t* words;   // [n]
  uint32_t* bitmap;  // [ceil(n/32)]
  int32_t* c;
  int32_t* O_out;    // optional cumulative offspring output
  int32_t* max_steps;
  DvState* state;
  uint32_t* status;
  int fx_S;          // fixed-point fraction bits of the offspring fast path
  const unsigned long long* logw_max;  // non-null: p.w holds log-weights, w = exp(lw - max) on the fly
  const A* Wser;     // non-null (accum = SERIAL): W = np.cumsum(w) bit for bit, computed by the serial fold
  int expand;        // 1: full delivery; 0: cumulative offspring O_out only
  // rare-path scratch
  int32_t* O;        // [n]
  int64_t* tmax;     // [tiles]
  int32_t *d, *J0, *J1, *R0, *R1;
};

// ---------------------------------------------------------------------------
// stratum offsets (cast to the weight dtype, resamplers.py:124/135)
enum UMode { kUSys = 0, kUArr = 1, kUNp = 2, kUPh = 3 };
constexpr int kULogW = 4;  // OR-ed into UM: the input holds log-weights (tile_weights)

template <typename T, typename A, int UM>
__device__ __forceinline__ A stratum_u(int64_t k0, const DvArgs<A>& p) {
  constexpr int M = UM & 3;
  if constexpr (M == kUSys) {
    return p.u_sys;
  } else if constexpr (M == kUArr) {
    return (A)(T)p.uniforms[k0];
  } else if constexpr (M == kUNp) {
    return (A)(T)u64_to_unit(numpy_raw64(p.key, (uint64_t)k0));
  } else {
    uint32_t o[4];
    philox4x32_10((uint32_t)(k0 >> 2), (uint32_t)(k0 >> 34), kTagStratified, 0, (uint32_t)p.key.k0,
                  (uint32_t)(p.key.k0 >> 32), o);
    return (A)(T)u32_to_unit_d(o[k0 & 3]);
  }
}

// O = min(N, floor(r + u[k-1])), r = (W * N) / total, k = min(N, floor(r) + 1)
// evaluated exactly as the reference's rounding sequence; the float64 fast
// path replaces the division by a multiply with N/total and falls back to
// the exact sequence whenever r or r+u lies within 2^-44 (relative) of an
// integer -- far more than the <= 2^-51 gap between the two r's -- so both
// floors are provably identical.
// the exact IEEE sequence of the reference (rare: kept out of line so its
// register needs do not inflate the streaming path)
template <typename T, typename A, int UM>
__device__ __noinline__ int32_t offspring_exact(A W, A total, int64_t n, const DvArgs<A>& p) {
  A r;
  if constexpr (sizeof(A) == 8)
    r = __ddiv_rn(__dmul_rn(W, (double)n), total);
  else
    r = __fdiv_rn(__fmul_rn(W, (float)n), total);
  int64_t k = (int64_t)floor((double)r) + 1;
  if (k > n) k = n;
  if (k < 1) k = 1;
  const A u = stratum_u<T, A, UM>(k - 1, p);
  int64_t o = (int64_t)floor((double)add_rn(r, u));
  return (int32_t)(o > n ? n : (o < 0 ? 0 : o));
}

template <typename T, typename A, int UM>
__device__ __forceinline__ int32_t offspring_of(A W, A total, const FxParams& f, int64_t n, const DvArgs<A>& p) {
  if constexpr (sizeof(A) == 8) {
    const long long r = fx_round(W, f.sfx);
    bool ok = fx_safe(r, f.mask);
    long long ufx = f.ufx;
    if constexpr ((UM & 3) != kUSys) {
      long long k = (r >> f.S) + 1;
      if (k > n) k = n;
      if (k < 1) k = 1;
      ufx = fx_round((double)stratum_u<T, A, UM>(k - 1, p), f.scale);
    }
    const long long t = r + ufx;
    ok &= fx_safe(t, f.mask);
    if (ok) return min((int32_t)(t >> f.S), (int32_t)n);
  }
  return offspring_exact<T, A, UM>(W, total, n, p);
}

// ---------------------------------------------------------------------------
// K1: one CTA per 4096-element tile: validation flags and the tile aggregate
// (the tile-local inclusive value at its last position, in exactly the
// association K2 uses); tile prefixes built hierarchically (pfr_hier.cuh).
// the tile's weights in registers: loaded, or exp(lw - max lw) computed from
// log-weights exactly as logweights_to_weights does (diagnostics.py:138-155;
// the same expression as k_logw_exp, so both paths see identical weights);
// positions past n stay 0
template <typename T, typename A, bool LW>
__device__ __forceinline__ void tile_weights(const DvArgs<A>& p, int64_t base, T (&x)[kTileItems]) {
  tile_load_any<T>((const T*)p.w, p.n, base, x);
  if constexpr (LW) {
    const T m = (T)from_ordered(__ldcg(p.logw_max));
    const int64_t e0 = base + (int64_t)threadIdx.x * kTileItems;
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
      T v;
      if constexpr (sizeof(T) == 8)
        v = exp(x[j] - m);
      else
        v = expf(x[j] - m);
      // all -inf (max -inf): every weight 0, which K1 reports (no positive weight)
      x[j] = (e0 + j < p.n && m > -INFINITY) ? v : T(0);
    }
  }
}

template <typename A>
__device__ __forceinline__ Hier<A> hier_of(const DvArgs<A>& p) {
  return Hier<A>{p.agg, p.excl, p.sum_scratch, p.state, p.tiles};
}
template <typename A>
__device__ __forceinline__ A tile_excl(const DvArgs<A>& p, int64_t b) {
  return hier_of(p).tile_excl(b);
}

template <typename T, typename A, int kTilesPerCta, bool LW = false>
__global__ void __launch_bounds__(kTileThreads) k_dv_reduce(DvArgs<A> p) {
  __shared__ A warp_sums[kTileThreads / 32];
  __shared__ uint32_t cta_flags;
  __shared__ int stage;
  // kTilesPerCta consecutive tiles per CTA, every load issued before the
  // first reduction (launched with 1: more tiles per CTA, or a persistent
  // double-buffered variant, measured slower)
  const int64_t b0 = (int64_t)blockIdx.x * kTilesPerCta;
  T x[kTilesPerCta][kTileItems];
#pragma unroll
  for (int t = 0; t < kTilesPerCta; ++t)
    if (b0 + t < p.tiles) tile_weights<T, A, LW>(p, (b0 + t) * kTile, x[t]);
#pragma unroll
  for (int t = 0; t < kTilesPerCta; ++t) {
    const int64_t b = b0 + t;
    if (b >= p.tiles) break;  // CTA-uniform
    if (threadIdx.x == 0) cta_flags = 0;
    FlagAcc<T> facc;
    TileScan<A> s;
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
      facc.add(x[t][j]);
      s.loc[j] = (A)x[t][j];
    }
    tile_scan<A>(s, warp_sums);
    if (threadIdx.x == kTileThreads - 1) p.agg[b] = add_rn(s.thread_excl, s.loc[kTileItems - 1]);
    const uint32_t flags = __reduce_or_sync(0xffffffffu, facc.flags());
    if ((threadIdx.x & 31) == 0 && flags) atomicOr(&cta_flags, flags);
    hier_tile_done(hier_of(p), b, &cta_flags, &stage, p.status);
    if (stage == 2 && threadIdx.x == 0) p.state->flags = 0;  // pipeline flags of this delivery
  }
}

// ---------------------------------------------------------------------------
// tile -> O (registers): shared by K2 and the repair path.  Index math is
// 32-bit inside the tile (N < 2^31).
template <typename T, typename A, int UM>
__device__ __forceinline__ void tile_offspring(const DvArgs<A>& p, int64_t b, uint4* stage, A* warp_sums,
                                               int32_t (&o)[kTileItems], int32_t& o_prev) {
  const int64_t base = b * kTile;
  const int last = (p.n - 1 - base < kTile) ? (int)(p.n - 1 - base) : -1;
  const int e0 = threadIdx.x * kTileItems;
  A total;
  if (p.Wser) {
    // accum = SERIAL: the reference's own W (np.cumsum, serial fold) is given;
    // the offspring formula then runs in the weight dtype (A = T), exactly
    // as resamplers.py:139-153
    A Wv[kTileItems];
    tile_load_any<A>(p.Wser, p.n, base, Wv);
    total = __ldg(p.Wser + p.n - 1);
    const FxParams fx = fx_params<A>(p.n, total, p.u_sys, p.fx_S);
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) o[j] = offspring_of<T, A, UM>(Wv[j], total, fx, p.n, p);
  } else {
    T x[kTileItems];
    tile_weights<T, A, (UM & kULogW) != 0>(p, base, x);
    TileScan<A> s;
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) s.loc[j] = (A)x[j];
    tile_scan<A>(s, warp_sums);
    total = hier_of(p).total();
    const FxParams fx = fx_params<A>(p.n, total, p.u_sys, p.fx_S);
    const A ex = tile_excl(p, b);
    const A tex = s.thread_excl;
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
      const A W = add_rn(ex, add_rn(tex, s.loc[j]));
      o[j] = offspring_of<T, A, UM>(W, total, fx, p.n, p);
    }
  }
  if (last >= 0) {  // the final tile: O[N-1] = N, and padding past N stays at N
#pragma unroll
    for (int j = 0; j < kTileItems; ++j)
      if (e0 + j >= last) o[j] = (int32_t)p.n;
  }
  o_prev = 0;
  if (b > 0) {
    const FxParams fx = fx_params<A>(p.n, total, p.u_sys, p.fx_S);
    // W at the last position of tile b-1
    const A Wp = p.Wser ? __ldg(p.Wser + base - 1) : add_rn(tile_excl(p, b - 1), __ldcg(p.agg + b - 1));
    o_prev = offspring_of<T, A, UM>(Wp, total, fx, p.n, p);
  }
}

// ---------------------------------------------------------------------------
// K2
template <typename T, typename A, int UM>
__global__ void __launch_bounds__(kTileThreads, 4) k_dv_expand(DvArgs<A> p) {
  __shared__ __align__(16) uint4 stage[kSlotCap * 4 / 16];  // word staging (32 KB)
  __shared__ uint32_t heads[kTileThreads];
  __shared__ A warp_sums[kTileThreads / 32];
  __shared__ int32_t warp_last[kTileThreads / 32];
  griddep_wait();
  const int64_t b = blockIdx.x;
  const int len = (int)min((int64_t)kTile, p.n - b * kTile);
  int32_t o[kTileItems];
  int32_t o_prev;
  tile_offspring<T, A, UM>(p, b, stage, warp_sums, o, o_prev);
  if (p.O_out) tile_store<int32_t>(p.O_out, p.n, b * kTile, stage, o, policy_evict_last());
  if (tile_decreases(o, o_prev, len, warp_last)) {
    if (threadIdx.x == 0) atomicOr(&p.state->flags, kNeedsRepair);
    return;  // the rare-path kernel recomputes everything
  }
  if (p.expand) tile_expand(o, o_prev, b, p.n, p.words, p.bitmap, reinterpret_cast<uint32_t*>(stage), heads, warp_last);
}

// ---------------------------------------------------------------------------
// K3: persistent; each warp owns a contiguous run of 32-index groups (lane l
// takes index 32k + l: coalesced loads of the slot words, coalesced stores of
// c).  c[x] = x for indices with offspring and the slot's parent for
// non-first holes.  A first-slot hole starts a backward chain (z = parent(z)
// while z is a first slot): chains are appended to a per-warp queue in shared
// memory (ballot compaction) and advanced in STEP PASSES that run only when
// the queue holds >= 8 chains per lane: each pass issues up to 8 independent
// chain loads per lane, resolves, and compacts the survivors in place.  So a
// chain step costs one full-lane slot (no divergence) and its L2 latency is
// shared by 8 loads.  Chain steps reach 10^4+ slots (drift x steps), so they
// are L2 reads of the words written by K2.
// kScanG: 32-index groups scanned per iteration; kThresh: queued chains that
// trigger a step pass
template <int kScanG, int kThresh, int kMinBlocks, bool kSegs = false>
__global__ void __launch_bounds__(kIpThreads, kMinBlocks) k_dv_inplace(const uint32_t* __restrict__ words,
                                                          const uint32_t* __restrict__ bitmap, int64_t n,
                                                          int32_t* __restrict__ c, int32_t* max_steps,
                                                          DvState* state, uint32_t* status, IpSegments segs) {
  __shared__ IpQueue Q;
  griddep_wait();
  if (state->flags & kNeedsRepair) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nn = (uint32_t)n;
  // segment mode: the index space is the listed segments, back to back
  const uint32_t groups = kSegs ? *segs.count * segs.groups : (nn + kGroup - 1) / kGroup;
  auto pg = [&](uint32_t g) -> uint32_t {
    if constexpr (kSegs) return __ldg(segs.list + g / segs.groups) * segs.groups + g % segs.groups;
    return g;
  };
  const uint32_t gw = blockIdx.x * kIpWarps + warp, nw = gridDim.x * kIpWarps;
  const uint32_t g0 = (uint32_t)((uint64_t)groups * gw / nw), g1 = (uint32_t)((uint64_t)groups * (gw + 1) / nw);
  const uint32_t gfull = kSegs ? groups : nn / kGroup;  // groups entirely below n
  int qlen = 0;
  int longest = 0;
  bool overflow = false;
  uint32_t g = g0;
  // steady state: whole iterations, no bounds checks
  for (; g + kScanG <= min(g1, gfull); g += kScanG) {
    if (qlen >= kThresh) qlen = step_pass(Q, warp, lane, qlen, words, c, longest, overflow);
    while (qlen > kQ - 32 * kScanG) qlen = step_pass(Q, warp, lane, qlen, words, c, longest, overflow);
    uint32_t wd[kScanG], bw[kScanG];
#pragma unroll
    for (int q = 0; q < kScanG; ++q) {
      const uint32_t gp = pg(g + q);
      wd[q] = __ldg(words + gp * kGroup + lane);
      bw[q] = __ldg(bitmap + gp);
    }
#pragma unroll
    for (int q = 0; q < kScanG; ++q) scan_group(Q, warp, lane, pg(g + q) * kGroup + lane, true, wd[q], bw[q], qlen, c);
    __syncwarp();
  }
  // tail groups
  for (; g < g1; ++g) {
    if (qlen > kQ - 32) qlen = step_pass(Q, warp, lane, qlen, words, c, longest, overflow);
    const uint32_t gp = pg(g);
    const uint32_t x = gp * kGroup + lane;
    const bool in = kSegs || x < nn;
    const uint32_t wd = in ? __ldg(words + x) : 0u;
    scan_group(Q, warp, lane, x, in, wd, __ldg(bitmap + gp), qlen, c);
    __syncwarp();
  }
  while (qlen) qlen = step_pass(Q, warp, lane, qlen, words, c, longest, overflow);
  if (overflow) {
    atomicOr(&state->flags, kOverflow);
    status_or(status, PFR_ST_OVERFLOW);
  }
  if (max_steps) {
    longest = __reduce_max_sync(0xffffffffu, longest);
    if (lane == 0 && longest) atomicMax(max_steps, longest);
  }
}

// the repair path's in-place pass: a plain (non-persistent) sweep
__device__ void resolve_all(const uint32_t* __restrict__ words, const uint32_t* __restrict__ bitmap, int64_t n,
                            int32_t* __restrict__ c, int& longest, bool& overflow) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t wd = __ldcg(words + i);
    const bool has = (__ldcg(bitmap + (i >> 5)) >> (i & 31)) & 1u;
    if (has) {
      c[i] = (int32_t)i;
      continue;
    }
    uint32_t v = wd;
    int st = 0;
    while (v & kFirst) {
      if (++st > kBackBound) {
        overflow = true;
        break;
      }
      v = __ldcg(words + (v & kParentMask));
    }
    c[i] = (int32_t)(v & kParentMask);
    longest = max(longest, st);
  }
}

// ---------------------------------------------------------------------------
// rare paths (cooperative): repair of non-monotone O, pointer jumping
template <typename T, typename A, int UM>
__global__ void __launch_bounds__(kTileThreads) k_dv_rare(DvArgs<A> p) {
  __shared__ __align__(16) uint4 stage[kSlotCap * 4 / 16];
  __shared__ uint32_t heads[kTileThreads];
  __shared__ A warp_sums[kTileThreads / 32];
  __shared__ int64_t imax8[kTileThreads / 32];
  __shared__ int32_t warp_last[kTileThreads / 32];
  griddep_wait();
  const uint32_t flags0 = *(volatile uint32_t*)&p.state->flags;
  if (!flags0) return;
  cg::grid_group grid = cg::this_grid();
  const int64_t n = p.n;
  if (flags0 & kNeedsRepair) {
    status_or(blockIdx.x == 0 && threadIdx.x == 0 ? p.status : nullptr, PFR_ST_REPAIRED);
    // A: raw O per tile -> global, tile maxima
    for (int64_t b = blockIdx.x; b < p.tiles; b += gridDim.x) {
      int32_t o[kTileItems];
      int32_t o_prev;
      tile_offspring<T, A, UM>(p, b, stage, warp_sums, o, o_prev);
      int64_t mx = INT64_MIN;
#pragma unroll
      for (int j = 0; j < kTileItems; ++j)
        if (b * kTile + threadIdx.x * kTileItems + j < n) mx = max(mx, (int64_t)o[j]);
      int64_t tmx;
      block_excl_max<int64_t>(mx, INT64_MIN, imax8, tmx);
      if (threadIdx.x == 0) p.tmax[b] = tmx;
      tile_store<int32_t>(p.O, n, b * kTile, stage, o, policy_evict_last());
    }
    grid.sync();
    // B: exclusive running max of the tile maxima (serial: rare path)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      int64_t run = INT64_MIN;
      for (int64_t b = 0; b < p.tiles; ++b) {
        const int64_t v = p.tmax[b];
        p.tmax[b] = run;
        run = max(run, v);
      }
    }
    grid.sync();
    // C: repaired O, words, bitmap
    for (int64_t b = blockIdx.x; b < p.tiles; b += gridDim.x) {
      int32_t o[kTileItems];
      tile_load<int32_t>(p.O, n, b * kTile, stage, policy_evict_last(), o);
      const int64_t before_tiles = __ldcg(p.tmax + b);
      int64_t mx = INT64_MIN;
#pragma unroll
      for (int j = 0; j < kTileItems; ++j)
        if (b * kTile + threadIdx.x * kTileItems + j < n) mx = max(mx, (int64_t)o[j]);
      int64_t tmx;
      const int64_t before_threads = block_excl_max<int64_t>(mx, INT64_MIN, imax8, tmx);
      int64_t run = max(before_tiles, before_threads);
#pragma unroll
      for (int j = 0; j < kTileItems; ++j) {
        if (b * kTile + threadIdx.x * kTileItems + j < n) {
          run = max(run, (int64_t)o[j]);
          o[j] = (int32_t)run;
        }
        if (b * kTile + threadIdx.x * kTileItems + j == n - 1) o[j] = (int32_t)n;
      }
      const int32_t o_prev = b ? (int32_t)max(before_tiles, (int64_t)0) : 0;
      if (p.O_out) tile_store<int32_t>(p.O_out, n, b * kTile, stage, o, policy_evict_last());
      if (p.expand)
        tile_expand(o, o_prev, b, n, p.words, p.bitmap, reinterpret_cast<uint32_t*>(stage), heads, warp_last);
    }
    grid.sync();
    if (!p.expand) return;  // cumulative offspring only: done
    // D: in-place indices
    bool overflow = false;
    int longest = 0;
    resolve_all(p.words, p.bitmap, n, p.c, longest, overflow);
    if (overflow) atomicOr(&p.state->flags, kOverflow);
    if (p.max_steps && longest) atomicMax(p.max_steps, longest);
    grid.sync();
  }
  if (!(*(volatile uint32_t*)&p.state->flags & kOverflow)) return;
  status_or(blockIdx.x == 0 && threadIdx.x == 0 ? p.status : nullptr, PFR_ST_OVERFLOW);
  // pointer jumping over the claim graph x -> d[x] (d[x] = first slot of x)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t x = t0; x < n; x += stride) p.d[x] = (int32_t)n;
  grid.sync();
  for (int64_t s = t0; s < n; s += stride) {
    const uint32_t wd = __ldcg(p.words + s);
    if (wd & kFirst) p.d[wd & kParentMask] = (int32_t)s;
  }
  grid.sync();
  for (int64_t x = t0; x < n; x += stride) {
    const int32_t dx = p.d[x];
    p.J0[x] = dx < n ? dx : (int32_t)x;
    p.R0[x] = dx < n ? 1 : 0;
  }
  int rounds = 1;
  while ((int64_t(1) << rounds) < n) ++rounds;
  ++rounds;
  int32_t *J = p.J0, *Jn = p.J1, *R = p.R0, *Rn = p.R1;
  for (int r = 0; r < rounds; ++r) {
    grid.sync();
    for (int64_t x = t0; x < n; x += stride) {
      const int32_t y = J[x];
      Jn[x] = J[y];
      Rn[x] = R[x] + R[y];
    }
    int32_t* t = J;
    J = Jn;
    Jn = t;
    t = R;
    R = Rn;
    Rn = t;
  }
  grid.sync();
  int longest = 0;
  for (int64_t i = t0; i < n; i += stride) {
    const uint32_t wd = __ldcg(p.words + i);
    if (wd & kFirst) continue;  // first slots are not losers
    p.c[J[i]] = (int32_t)(wd & kParentMask);
    longest = max(longest, R[i]);
  }
  if (p.max_steps && longest) atomicMax(p.max_steps, longest);
}

// ---------------------------------------------------------------------------
template <typename K, typename... Args>
cudaError_t launch_pdl_smem(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool cooperative,
                            Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
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

template <typename K, typename... Args>
cudaError_t launch_pdl(K kernel, dim3 grid, dim3 block, cudaStream_t s, bool cooperative, Args... args) {
  return launch_pdl_smem(kernel, grid, block, 0, s, cooperative, args...);
}

template <typename T, typename A, int UM>
cudaError_t deliver_typed(DvArgs<A> p, cudaStream_t s) {
  // PFR_DV_STAGES (profiling aid): launch only the first k kernels
  static const int stages = [] {
    const char* v = getenv("PFR_DV_STAGES");
    return v ? atoi(v) : 4;
  }();
  const unsigned tiles = (unsigned)p.tiles;
  cudaError_t e;
  if (p.Wser) {
    // accum = SERIAL: the serial fold (np.cumsum bit for bit, with
    // check_weights' flags) replaces K1; it also resets the pipeline flags
    e = launch_serial_weights_scan(p.w, const_cast<A*>(p.Wser), p.n, sizeof(T) == 8 ? PFR_F64 : PFR_F32,
                                   p.status, p.state, s);
  } else {
    // one tile per CTA (2 or 4 consecutive tiles per CTA measured 29 -> 37 / 43
    // us at 2^24: the per-tile hierarchy step is serial inside a CTA)
    k_dv_reduce<T, A, 1, (UM & kULogW) != 0><<<(unsigned)p.tiles, kTileThreads, 0, s>>>(p);
    note_launch();
    e = cudaGetLastError();
  }
  if (e != cudaSuccess || stages < 2) return e;
  e = launch_pdl(k_dv_expand<T, A, UM>, dim3(tiles), dim3(kTileThreads), s, false, p);
  if (e != cudaSuccess || stages < 3) return e;
  if (p.expand) {
    // K3 tunables measured on B200 (scan width 2..8 groups, step-pass
    // threshold 32..128, 4 vs 6 CTAs/SM): <4, 64, 4> is best; more CTAs/SM
    // spill and lose 40%
    auto kernel = k_dv_inplace<4, 64, 4>;
    int occ3 = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, kernel, kIpThreads, 0);
    if (e != cudaSuccess) return e;
    if (occ3 < 1) occ3 = 1;
    // >= 8 groups per warp: small problems spread over many warps (the chain
    // walks are latency bound), large ones fill the machine once (persistent)
    const int64_t warps_needed = (p.n + 32 * 8 - 1) / (32 * 8);
    const unsigned grid3 =
        (unsigned)max((int64_t)1, min((int64_t)num_sms() * occ3, (warps_needed + kIpWarps - 1) / kIpWarps));
    e = launch_pdl(kernel, dim3(grid3), dim3(kIpThreads), s, false, (const uint32_t*)p.words,
                   (const uint32_t*)p.bitmap, p.n, p.c, p.max_steps, p.state, p.status, IpSegments{nullptr, nullptr, 0});
    if (e != cudaSuccess || stages < 4) return e;
  }
  static int occ = -1;
  if (occ < 0) {
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dv_rare<T, A, UM>, kTileThreads, 0);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
  }
  // one CTA per SM: the grid only has to be co-resident (grid.sync), and in
  // the common case every CTA returns at once, so a small grid launches fastest
  (void)occ;
  return launch_pdl(k_dv_rare<T, A, UM>, dim3(num_sms()), dim3(kTileThreads), s, true, p);
}

template <typename T, typename A>
cudaError_t deliver_mode(DvArgs<A> p, int stratified, const double* uniforms, const pfr_rng* rng, cudaStream_t s) {
  if (p.logw_max) {  // log-weights: the same pipeline with exp(lw - max) on load
    if (!stratified) return deliver_typed<T, A, kUSys | kULogW>(p, s);
    if (uniforms) return deliver_typed<T, A, kUArr | kULogW>(p, s);
    if (rng && rng->mode == PFR_RNG_NUMPY) return deliver_typed<T, A, kUNp | kULogW>(p, s);
    return deliver_typed<T, A, kUPh | kULogW>(p, s);
  }
  if (!stratified) return deliver_typed<T, A, kUSys>(p, s);
  if (uniforms) return deliver_typed<T, A, kUArr>(p, s);
  if (rng && rng->mode == PFR_RNG_NUMPY) return deliver_typed<T, A, kUNp>(p, s);
  return deliver_typed<T, A, kUPh>(p, s);
}

template <typename T, typename A>
DvArgs<A> make_args(const void* w, int64_t n, double offset, const double* uniforms, const pfr_rng* rng, int32_t* c,
                    int32_t* O_out, int32_t* max_steps, uint32_t* status, const Workspace& ws) {
  DvArgs<A> p;
  p.w = w;
  p.n = n;
  p.tiles = num_tiles(n);
  p.agg = reinterpret_cast<A*>(ws.sum_cells);
  p.sum_scratch = p.agg + p.tiles + 8;  // the sum tree region holds >= 2 * tiles cells
  p.excl = reinterpret_cast<A*>(ws.max_cells);
  p.u_sys = (A)(T)offset;
  p.uniforms = uniforms;
  p.key = Key2x64{rng ? rng->key0 : 0, rng ? rng->key1 : 0};
  p.words = reinterpret_cast<uint32_t*>(ws.a);
  p.bitmap = reinterpret_cast<uint32_t*>(ws.d);
  p.c = c;
  p.O_out = O_out;
  p.max_steps = max_steps;
  p.state = ws.dv;
  p.status = status;
  p.fx_S = fx_bits(n);
  p.logw_max = nullptr;
  p.Wser = nullptr;
  p.expand = c != nullptr;
  p.O = ws.O;
  p.tmax = reinterpret_cast<int64_t*>(ws.j1);  // tiles << n
  p.d = ws.O;  // O is dead once the words exist
  p.J0 = ws.j0;
  p.J1 = ws.j1;
  p.R0 = ws.r0;
  p.R1 = ws.r1;
  return p;
}

}  // namespace

// K3 on its own, for callers that wrote slot words and the has-offspring
// bitmap themselves (the batched filter: global parent numbers, so one pass
// serves every filter).  Sets kOverflow in state->flags when a chain exceeds
// the walk bound (the caller owns the fallback).
cudaError_t launch_dv_inplace(const uint32_t* words, const uint32_t* bitmap, int64_t n, int32_t* c, DvState* state,
                              uint32_t* status, cudaStream_t s, const uint32_t* seg_list, const uint32_t* seg_count,
                              int64_t seg_len) {
  auto kernel = seg_list ? k_dv_inplace<4, 64, 4, true> : k_dv_inplace<4, 64, 4, false>;
  int occ3 = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, kernel, kIpThreads, 0);
  if (e != cudaSuccess) return e;
  if (occ3 < 1) occ3 = 1;
  const int64_t warps_needed = (n + 32 * 8 - 1) / (32 * 8);
  const unsigned grid3 =
      (unsigned)max((int64_t)1, min((int64_t)num_sms() * occ3, (warps_needed + kIpWarps - 1) / kIpWarps));
  return launch_pdl(kernel, dim3(grid3), dim3(kIpThreads), s, false, words, bitmap, n, c, (int32_t*)nullptr, state,
                    status, IpSegments{seg_list, seg_count, (uint32_t)(seg_len / 32)});
}

// systematic_/stratified_cumulative_offspring (resamplers.py:105-153): the
// delivery's K1 + K2 with O stored and no expansion (rare path repairs O)
cudaError_t launch_offspring(const void* w, int64_t n, int dtype, int accum, int stratified, double offset,
                             const double* uniforms, const pfr_rng* rng, int32_t* O, uint32_t* status,
                             const Workspace& ws, cudaStream_t s) {
  return launch_deliver(w, n, dtype, accum, stratified, offset, uniforms, rng, nullptr, O, nullptr, status, ws, s);
}

cudaError_t launch_deliver(const void* w, int64_t n, int dtype, int accum, int stratified, double offset,
                           const double* uniforms, const pfr_rng* rng, int32_t* c, int32_t* O_out,
                           int32_t* max_steps, uint32_t* status, const Workspace& ws, cudaStream_t s, int logw) {
  if (max_steps) {
    cudaError_t e = cudaMemsetAsync(max_steps, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
  }
  if (accum == PFR_ACC_SERIAL) {
    // parity mode: W = np.cumsum(w) by the serial fold into the workspace,
    // offspring in the weight dtype (log-weights: converted first, like
    // logweights_to_weights followed by the delivery)
    if (logw) {
      cudaError_t e = launch_logweights(w, ws.f0, n, dtype, status, ws, s);
      if (e != cudaSuccess) return e;
      w = ws.f0;
    }
    if (dtype == PFR_F64) {
      auto p = make_args<double, double>(w, n, offset, uniforms, rng, c, O_out, max_steps, status, ws);
      p.Wser = reinterpret_cast<const double*>(ws.f1);
      return deliver_mode<double, double>(p, stratified, uniforms, rng, s);
    }
    auto p = make_args<float, float>(w, n, offset, uniforms, rng, c, O_out, max_steps, status, ws);
    p.Wser = reinterpret_cast<const float*>(ws.f1);
    return deliver_mode<float, float>(p, stratified, uniforms, rng, s);
  }
  // log-weights: one max pass (with the log-weight validation flags), then
  // K1/K2 compute exp(lw - max) as they load -- w is never stored
  const unsigned long long* lmax = nullptr;
  if (logw) {
    unsigned long long* cell = reinterpret_cast<unsigned long long*>(&ws.hdr->cell[1]);
    cudaError_t e = launch_logw_max(w, n, dtype, cell, status, s);
    if (e != cudaSuccess) return e;
    lmax = cell;
  }
  auto args = [&](auto a) {
    a.logw_max = lmax;
    return a;
  };
  if (dtype == PFR_F64)
    return deliver_mode<double, double>(
        args(make_args<double, double>(w, n, offset, uniforms, rng, c, O_out, max_steps, status, ws)), stratified,
        uniforms, rng, s);
  if (accum == PFR_ACC_NATIVE)
    return deliver_mode<float, float>(
        args(make_args<float, float>(w, n, offset, uniforms, rng, c, O_out, max_steps, status, ws)), stratified,
        uniforms, rng, s);
  return deliver_mode<float, double>(
      args(make_args<float, double>(w, n, offset, uniforms, rng, c, O_out, max_steps, status, ws)), stratified,
      uniforms, rng, s);
}

}  // namespace pfr
