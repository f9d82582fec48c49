// Fused systematic / stratified delivery: weights -> in-place-valid ancestry.
//
// Computes permute_parallel(cumulative_offspring_to_ancestors(O)) with
// O = systematic_cumulative_offspring(w) or stratified_... (ancestry.py:69-76,
// 139-174; resamplers.py:105-153) -- the timed region of the reference's
// bench.py:155-161 for the offspring algorithms -- in three HBM-streaming
// kernels chained with programmatic dependent launch:
//
//   K1 k_dv_reduce   read w once: validation flags, per-tile inclusive scan
//                    aggregate; the last CTA scans the tile aggregates (fixed
//                    association => deterministic) into excl[] and the total.
//   K2 k_dv_expand   re-read w (L2), W = excl[b] + tile scan, O from the
//                    position formula (division-free fast path, exact IEEE
//                    path within 2^-44 of an integer), then write the sorted
//                    ancestry as 32-bit words  parent | FIRST(slot is its
//                    parent's first slot)  over the tile's slot range, plus a
//                    bitmap  has-offspring(x).  No atomics, no waits.
//   K3 k_dv_inplace  one pass over the indices: c[x] = x if x has offspring;
//                    a hole h walks BACKWARDS: while slot z is a first slot,
//                    z = parent(z); then c[h] = parent(z).  This is the
//                    reference's loser chain read from its end (the chain
//                    L -> d[L] -> ... -> h has d[y] = first slot of y), so
//                    every c[x] is written by its own thread: coalesced.
//
// Rare paths, all inside one cooperative kernel k_dv_rare that returns at once
// when not needed: (a) ulp-level non-monotone O (W is not a strict serial
// fold) -> global running-max repair (resamplers.py:150) and recomputation;
// (b) a chain longer than the walk bound -> pointer jumping (Wyllie) over the
// claim graph.
#include <cooperative_groups.h>

#include "pfr_internal.h"
#include "pfr_tile.cuh"

namespace cg = cooperative_groups;

namespace pfr {

namespace {

constexpr uint32_t kFirst = 0x80000000u;
constexpr uint32_t kParentMask = 0x7FFFFFFFu;
constexpr int kBackBound = 64;

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
  A* excl;       // [tiles + 1]; excl[tiles] = total
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
  // rare-path scratch
  int32_t* O;        // [n]
  int64_t* tmax;     // [tiles]
  int32_t *d, *J0, *J1, *R0, *R1;
};

template <typename T>
__device__ __forceinline__ uint32_t wflags(T x) {
  uint32_t f = 0;
  if (!isfinite((double)x)) f |= PFR_ST_NONFINITE;
  if (x < T(0)) f |= PFR_ST_NEGATIVE;
  if (x > T(0)) f |= PFR_ST_POSITIVE;
  return f;
}

// ---------------------------------------------------------------------------
// stratum offsets (cast to the weight dtype, resamplers.py:124/135)
enum UMode { kUSys = 0, kUArr = 1, kUNp = 2, kUPh = 3 };

template <typename T, typename A, int UM>
__device__ __forceinline__ A stratum_u(int64_t k0, const DvArgs<A>& p) {
  if constexpr (UM == kUSys) {
    return p.u_sys;
  } else if constexpr (UM == kUArr) {
    return (A)(T)p.uniforms[k0];
  } else if constexpr (UM == kUNp) {
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
__device__ __forceinline__ int32_t offspring_of(A W, A total, A scale, int64_t n, const DvArgs<A>& p) {
  if constexpr (sizeof(A) == 8) {
    const double rf = __dmul_rn(W, scale);
    const double tol = fmax(rf, 1.0) * 5.684341886080802e-14;  // 2^-44
    const double fr = floor(rf);
    if ((rf - fr) >= tol && (fr + 1.0 - rf) >= tol) {
      int64_t k = (int64_t)fr + 1;
      if (k > n) k = n;
      const double tf = __dadd_rn(rf, (double)stratum_u<T, A, UM>(k - 1, p));
      const double ft = floor(tf);
      if ((tf - ft) >= tol && (ft + 1.0 - tf) >= tol) {
        const int64_t o = (int64_t)ft;
        return (int32_t)(o > n ? n : (o < 0 ? 0 : o));
      }
    }
  }
  return offspring_exact<T, A, UM>(W, total, n, p);
}

// ---------------------------------------------------------------------------
// K1: validation + tile aggregates; the last CTA scans them.  Per-tile flags
// go to a plain array (no same-address atomics from thousands of CTAs); the
// last CTA ORs them into the caller's status word once.
template <typename A>
__device__ __forceinline__ uint32_t* tile_flags(const DvArgs<A>& p) {
  return reinterpret_cast<uint32_t*>(p.excl + p.tiles + 2);
}

template <typename T, typename A>
__global__ void __launch_bounds__(kTileThreads) k_dv_reduce(DvArgs<A> p) {
  __shared__ __align__(16) uint4 stage[kTile * sizeof(T) / 16];
  __shared__ A warp_sums[kTileThreads / 32];
  __shared__ uint32_t cta_flags;
  __shared__ bool is_last;
  const int b = blockIdx.x;
  const int64_t base = (int64_t)b * kTile;
  const int len = (int)min((int64_t)kTile, p.n - base);
  if (threadIdx.x == 0) cta_flags = 0;
  T x[kTileItems];
  tile_load<T>((const T*)p.w, p.n, base, stage, policy_evict_last(), x);  // keep w in L2 for K2
  TileScan<A> s;
  uint32_t flags = 0;
  const int e0 = threadIdx.x * kTileItems;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) {
    if (e0 + j < len) flags |= wflags(x[j]);
    s.loc[j] = (A)x[j];
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(&cta_flags, flags);
  tile_scan<A>(s, warp_sums);  // (ends with a barrier: cta_flags is complete)
  if (threadIdx.x == kTileThreads - 1) {
    // aggregate := tile-local inclusive value at the tile's last position
    p.agg[b] = add_rn(s.thread_excl, s.loc[kTileItems - 1]);
    tile_flags(p)[b] = cta_flags;
    __threadfence();
    const unsigned t = atomicAdd(&p.state->done, 1u);
    is_last = (t == (unsigned)(p.tiles - 1));
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // exclusive scan over the tile aggregates: serial within a thread's chunk,
  // Kogge-Stone across threads, serial across warps (fixed association)
  const int T_ = (int)p.tiles;
  const int chunk = (T_ + kTileThreads - 1) / kTileThreads;
  const int c0 = threadIdx.x * chunk, c1 = min(c0 + chunk, T_);
  A mine = A(0);
  uint32_t fl = 0;
  for (int i = c0; i < c1; ++i) {
    mine = add_rn(mine, __ldcg(p.agg + i));
    fl |= __ldcg(tile_flags(p) + i);
  }
  fl = __reduce_or_sync(0xffffffffu, fl);
  const A incl = warp_inclusive_scan(mine);
  A excl = __shfl_up_sync(0xffffffffu, incl, 1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) excl = A(0);
  if (lane == 31) warp_sums[warp] = incl;
  if (lane == 0 && fl) atomicOr(&cta_flags, fl);
  __syncthreads();
  A wp = A(0);
  for (int v = 0; v < warp; ++v) wp = add_rn(wp, warp_sums[v]);
  A run = lane ? add_rn(wp, excl) : wp;
  for (int i = c0; i < c1; ++i) {
    p.excl[i] = run;
    run = add_rn(run, __ldcg(p.agg + i));
  }
  if (c0 < T_ && c1 == T_) p.excl[T_] = run;  // the total
  if (threadIdx.x == 0) {
    p.state->done = 0;
    p.state->flags = 0;
    status_or(p.status, cta_flags);
  }
}

// ---------------------------------------------------------------------------
// tile -> O (registers): shared by K2 and the repair path.  Index math is
// 32-bit inside the tile (N < 2^31).
template <typename T, typename A, int UM>
__device__ __forceinline__ void tile_offspring(const DvArgs<A>& p, int64_t b, uint4* stage, A* warp_sums,
                                               int32_t (&o)[kTileItems], int32_t& o_prev) {
  const int64_t base = b * kTile;
  T x[kTileItems];
  tile_load<T>((const T*)p.w, p.n, base, stage, policy_evict_first(), x);
  TileScan<A> s;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) s.loc[j] = (A)x[j];
  tile_scan<A>(s, warp_sums);
  const A total = p.excl[p.tiles];
  const A scale = (A)p.n / total;
  const A ex = p.excl[b];
  const int last = (p.n - 1 - base < kTile) ? (int)(p.n - 1 - base) : -1;
  const int e0 = threadIdx.x * kTileItems;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) {
    const A W = add_rn(ex, add_rn(s.thread_excl, s.loc[j]));
    o[j] = (int32_t)offspring_of<T, A, UM>(W, total, scale, p.n, p);
    if (e0 + j == last) o[j] = (int32_t)p.n;  // O[N-1] = N
  }
  o_prev = 0;
  if (b > 0) {
    const A Wp = add_rn(p.excl[b - 1], p.agg[b - 1]);  // W at the last position of tile b-1
    o_prev = (int32_t)offspring_of<T, A, UM>(Wp, total, scale, p.n, p);
  }
}

// true when o decreases anywhere inside the tile or against the previous
// tile's last O (the caller then defers to the repair path)
__device__ __forceinline__ bool tile_decreases(const int32_t (&o)[kTileItems], int32_t o_prev, int len,
                                               int32_t* warp_last) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e0 = threadIdx.x * kTileItems;
  bool bad = false;
#pragma unroll
  for (int j = 1; j < kTileItems; ++j) bad |= (e0 + j < len) && o[j] < o[j - 1];
  int prev = __shfl_up_sync(0xffffffffu, o[kTileItems - 1], 1);
  if (lane == 31) warp_last[warp] = o[kTileItems - 1];
  __syncthreads();
  if (lane == 0) prev = warp ? warp_last[warp - 1] : o_prev;
  if (e0 < len) bad |= o[0] < prev;
  return __syncthreads_or(bad);
}

// word staging in shared memory: 16-byte slots XOR-swizzled (bank spread
// for the per-thread contiguous writes, conflict-free striped read-out)
__device__ __forceinline__ int sw4(int pos) { return (swz(pos >> 2) << 2) | (pos & 3); }

// smem O table (same swizzle): element x of the tile
__device__ __forceinline__ int os_get(const int32_t* Os, int x) { return Os[sw4(x)]; }

constexpr int kLightCap = 2 * kTile;  // words a light tile may stage (32 KB)
constexpr int kLightMaxO = 64;         // per-parent offspring bound of the light path

// Expand the tile's parents over their slots: words (parent | FIRST) and the
// has-offspring bitmap.  Light path (the common case): every thread writes
// its own 16 parents' slots into shared memory, then the CTA streams the
// tile's slot range out with coalesced stores.  Heavy path (a parent with more
// than kLightMaxO offspring, or a slot range over 8192): balanced chunks of
// 4096 slots, each thread locating its parent by binary search.
__device__ void tile_expand(const int32_t (&o)[kTileItems], int32_t o_prev, int64_t b, int64_t n, uint32_t* words,
                            uint32_t* bitmap, uint32_t* sbuf /* 32 KB */, int32_t* warp_last) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = b * kTile;
  const int len = (int)min((int64_t)kTile, n - base);
  const int e0 = tid * kTileItems;
  const uint32_t pbase = (uint32_t)base + (uint32_t)e0;
  // O of the element before this thread's first parent
  int prev = __shfl_up_sync(0xffffffffu, o[kTileItems - 1], 1);
  if (lane == 31) warp_last[warp] = o[kTileItems - 1];
  __syncthreads();
  if (lane == 0) prev = warp ? warp_last[warp - 1] : o_prev;
  uint32_t bits = 0;
  int maxo = 0;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) {
    const int pv = j ? o[j - 1] : prev;
    if (e0 + j < len) {
      if (o[j] > pv) bits |= 1u << j;
      maxo = max(maxo, o[j] - pv);
    }
  }
  const uint32_t hi = __shfl_down_sync(0xffffffffu, bits, 1);
  if ((tid & 1) == 0 && e0 < len) bitmap[(base >> 5) + (tid >> 1)] = bits | (hi << 16);
  const int S0 = o_prev;
  __shared__ int s_end;  // O of the tile's last element: N for the final tile
  if (tid == kTileThreads - 1) s_end = (len == kTile) ? o[kTileItems - 1] : (int)n;
  const bool heavy = __syncthreads_or(maxo > kLightMaxO);
  const int end = s_end;
  if (!heavy && end - S0 <= kLightCap) {
    // light: own parents -> staged words
    int q = prev - S0;
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
      if (e0 + j < len) {
        const int e = o[j] - S0;
        if (q < e) {
          sbuf[sw4(q)] = (pbase + j) | kFirst;
          for (int r = q + 1; r < e; ++r) sbuf[sw4(r)] = pbase + j;
        }
        q = e;
      }
    }
    __syncthreads();
    const int cnt = end - S0;
    uint32_t* dst = words + S0;
    for (int i = tid; i < cnt; i += kTileThreads) dst[i] = sbuf[sw4(i)];
    __syncthreads();
    return;
  }
  // heavy: O table in the first 16 KB, 4096-slot chunks staged in the second
  int32_t* Os = reinterpret_cast<int32_t*>(sbuf);
  uint32_t* wbuf = sbuf + kTile;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int4 v = make_int4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
    reinterpret_cast<int4*>(Os)[swz(tid * 4 + q)] = v;
  }
  __syncthreads();
  for (int r0 = S0; r0 < end; r0 += kTile) {
    const int sb = r0 + e0;
    const int se = min(sb + kTileItems, end);
    if (sb < se) {
      int lo = 0, hi2 = len - 1;  // parent of slot sb: smallest x with O(x) > sb
      while (lo < hi2) {
        const int mid = (lo + hi2) >> 1;
        if (os_get(Os, mid) > sb)
          hi2 = mid;
        else
          lo = mid + 1;
      }
      int xi = lo;
      int ox = os_get(Os, xi);
      int oex = xi ? os_get(Os, xi - 1) : o_prev;
      for (int s = sb; s < se; ++s) {
        while (ox <= s) {
          ++xi;
          oex = ox;
          ox = os_get(Os, xi);
        }
        wbuf[sw4(s - r0)] = ((uint32_t)base + xi) | (s == oex ? kFirst : 0u);
      }
    }
    __syncthreads();
    const int cnt = min(kTile, end - r0);
    for (int i = tid; i < cnt; i += kTileThreads) words[r0 + i] = wbuf[sw4(i)];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K2
template <typename T, typename A, int UM>
__global__ void __launch_bounds__(kTileThreads, 3) k_dv_expand(DvArgs<A> p) {
  __shared__ __align__(16) uint4 stage[2 * kTile * 4 / 16];  // tile stage, then word staging (32 KB)
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
  tile_expand(o, o_prev, b, p.n, p.words, p.bitmap, reinterpret_cast<uint32_t*>(stage), warp_last);
}

// ---------------------------------------------------------------------------
// K3: 16 indices per thread, striped (index = base + 256 j + t), so the
// coalesced word loads and the clustered chain loads of a warp share sectors;
// all of a thread's pending chains advance together (16 loads in flight).
constexpr int kInplaceItems = 16;

__device__ __forceinline__ void resolve_tile(const uint32_t* __restrict__ words, const uint32_t* __restrict__ bitmap,
                                             int64_t n, int32_t* __restrict__ c, int64_t base, int& longest,
                                             bool& overflow) {
  const int t = threadIdx.x;
  // v[j]: the final output, or for a pending chain the current node
  uint32_t v[kInplaceItems];
  uint32_t active = 0;
#pragma unroll
  for (int j = 0; j < kInplaceItems; ++j) {
    const int64_t i = base + (int64_t)j * kTileThreads + t;
    v[j] = 0;
    if (i < n) {
      const uint32_t wd = __ldcg(words + i);
      const bool has = (__ldcg(bitmap + (i >> 5)) >> (i & 31)) & 1u;
      v[j] = has ? (uint32_t)i : (wd & kParentMask);
      if (!has && (wd & kFirst)) active |= 1u << j;
    }
  }
  int steps = 0;
  while (active) {
    if (++steps > kBackBound) {
      overflow = true;
      break;
    }
    uint32_t wz[kInplaceItems];
#pragma unroll
    for (int j = 0; j < kInplaceItems; ++j)
      if (active & (1u << j)) wz[j] = __ldcg(words + v[j]);
#pragma unroll
    for (int j = 0; j < kInplaceItems; ++j) {
      if (active & (1u << j)) {
        v[j] = wz[j] & kParentMask;
        if (!(wz[j] & kFirst)) active &= ~(1u << j);
      }
    }
  }
  longest = max(longest, overflow ? kBackBound : steps);
#pragma unroll
  for (int j = 0; j < kInplaceItems; ++j) {
    const int64_t i = base + (int64_t)j * kTileThreads + t;
    if (i < n) __stcs(c + i, (int32_t)v[j]);
  }
}

__global__ void __launch_bounds__(kTileThreads, 5) k_dv_inplace(const uint32_t* __restrict__ words,
                                                             const uint32_t* __restrict__ bitmap, int64_t n,
                                                             int32_t* __restrict__ c, int32_t* max_steps,
                                                             DvState* state, uint32_t* status) {
  griddep_wait();
  if (state->flags & kNeedsRepair) return;
  int longest = 0;
  bool overflow = false;
  resolve_tile(words, bitmap, n, c, (int64_t)blockIdx.x * kTileThreads * kInplaceItems, longest, overflow);
  if (overflow) {
    atomicOr(&state->flags, kOverflow);
    status_or(status, PFR_ST_OVERFLOW);
  }
  if (max_steps && longest) atomicMax(max_steps, longest);
  // (no early trigger: dependents launch at grid completion)
}

// ---------------------------------------------------------------------------
// rare paths (cooperative): repair of non-monotone O, pointer jumping
template <typename T, typename A, int UM>
__global__ void __launch_bounds__(kTileThreads) k_dv_rare(DvArgs<A> p) {
  __shared__ __align__(16) uint4 stage[2 * kTile * 4 / 16];
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
      tile_expand(o, o_prev, b, n, p.words, p.bitmap, reinterpret_cast<uint32_t*>(stage), warp_last);
    }
    grid.sync();
    // D: in-place indices
    bool overflow = false;
    int longest = 0;
    const int64_t span = (int64_t)kTileThreads * kInplaceItems;
    for (int64_t t = blockIdx.x; t * span < n; t += gridDim.x)
      resolve_tile(p.words, p.bitmap, n, p.c, t * span, longest, overflow);
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
cudaError_t launch_pdl(K kernel, dim3 grid, dim3 block, cudaStream_t s, bool cooperative, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
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

template <typename T, typename A, int UM>
cudaError_t deliver_typed(DvArgs<A> p, cudaStream_t s) {
  const unsigned tiles = (unsigned)p.tiles;
  k_dv_reduce<T, A><<<tiles, kTileThreads, 0, s>>>(p);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = launch_pdl(k_dv_expand<T, A, UM>, dim3(tiles), dim3(kTileThreads), s, false, p);
  if (e != cudaSuccess) return e;
  const unsigned blocks3 = (unsigned)((p.n + kTile - 1) / kTile);
  e = launch_pdl(k_dv_inplace, dim3(blocks3), dim3(256), s, false, (const uint32_t*)p.words,
                 (const uint32_t*)p.bitmap, p.n, p.c, p.max_steps, p.state, p.status);
  if (e != cudaSuccess) return e;
  static int occ = -1;
  if (occ < 0) {
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dv_rare<T, A, UM>, kTileThreads, 0);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
  }
  return launch_pdl(k_dv_rare<T, A, UM>, dim3(num_sms() * occ), dim3(kTileThreads), s, true, p);
}

template <typename T, typename A>
cudaError_t deliver_mode(DvArgs<A> p, int stratified, const double* uniforms, const pfr_rng* rng, cudaStream_t s) {
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

cudaError_t launch_deliver(const void* w, int64_t n, int dtype, int accum, int stratified, double offset,
                           const double* uniforms, const pfr_rng* rng, int32_t* c, int32_t* O_out,
                           int32_t* max_steps, uint32_t* status, const Workspace& ws, cudaStream_t s) {
  if (max_steps) {
    cudaError_t e = cudaMemsetAsync(max_steps, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
  }
  if (dtype == PFR_F64)
    return deliver_mode<double, double>(
        make_args<double, double>(w, n, offset, uniforms, rng, c, O_out, max_steps, status, ws), stratified,
        uniforms, rng, s);
  if (accum == PFR_ACC_NATIVE)
    return deliver_mode<float, float>(
        make_args<float, float>(w, n, offset, uniforms, rng, c, O_out, max_steps, status, ws), stratified, uniforms,
        rng, s);
  return deliver_mode<float, double>(
      make_args<float, double>(w, n, offset, uniforms, rng, c, O_out, max_steps, status, ws), stratified, uniforms,
      rng, s);
}

}  // namespace pfr
