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

#include <cstdlib>

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

// Fast path in 31-bit fixed point: r_fx = round(W * N/total * 2^31) (one
// multiply + one conversion), t_fx = r_fx + u_fx (exact integer add).  The
// float64 products differ from the reference's r = (W*N)/total by at most
// 2^-51 r, the conversions by one unit, so whenever the fractional parts of
// r and r+u sit more than dr = N/2^13 + 16 units (far above those bounds)
// from an integer, the floors are the reference's; otherwise the exact IEEE
// sequence runs.  All checks are 32-bit on the low word.
template <typename T, typename A, int UM>
__device__ __forceinline__ int32_t offspring_of(A W, A total, A sfx, long long ufx_sys, uint32_t dr, int64_t n,
                                                const DvArgs<A>& p) {
  if constexpr (sizeof(A) == 8) {
    const long long r = __double2ll_rn(__dmul_rn(W, sfx));
    const uint32_t span = 0x7FFFFFFFu - 2u * dr;
    bool ok = ((uint32_t)r & 0x7FFFFFFFu) - dr <= span;
    long long ufx = ufx_sys;
    if constexpr (UM != kUSys) {
      long long k = (r >> 31) + 1;
      if (k > n) k = n;
      if (k < 1) k = 1;
      ufx = __double2ll_rn((double)stratum_u<T, A, UM>(k - 1, p) * 2147483648.0);
    }
    const long long t = r + ufx;
    ok &= ((uint32_t)t & 0x7FFFFFFFu) - dr <= span;
    if (ok) {
      const long long o = t >> 31;
      return (int32_t)(o > n ? n : o);
    }
  }
  return offspring_exact<T, A, UM>(W, total, n, p);
}

// blocked direct loads: thread t gets elements [16t, 16t + 16) of the tile
// (L1-allocating 16-byte loads; the 4-8 loads of a thread hit the same lines)
template <typename T>
__device__ __forceinline__ void tile_load_direct(const T* __restrict__ in, int64_t n, int64_t base,
                                                 T (&x)[kTileItems]) {
  constexpr int kPerVec = 16 / sizeof(T);
  const int64_t e0 = base + (int64_t)threadIdx.x * kTileItems;
  if (e0 + kTileItems <= n) {
    uint4 v[kTileItems / kPerVec];
#pragma unroll
    for (int q = 0; q < kTileItems / kPerVec; ++q) v[q] = __ldg(reinterpret_cast<const uint4*>(in + e0) + q);
#pragma unroll
    for (int q = 0; q < kTileItems / kPerVec; ++q) {
      union {
        uint4 u;
        T e[kPerVec];
      } tmp;
      tmp.u = v[q];
#pragma unroll
      for (int e = 0; e < kPerVec; ++e) x[q * kPerVec + e] = tmp.e[e];
    }
  } else {
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) x[j] = (e0 + j < n) ? in[e0 + j] : T(0);
  }
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
  // persistent: CTA-strided tiles, one fence + one counter bump per CTA
  if (threadIdx.x == 0) cta_flags = 0;
  uint32_t flags = 0;
  for (int64_t b = blockIdx.x; b < p.tiles; b += gridDim.x) {
    const int64_t base = b * kTile;
    const int len = (int)min((int64_t)kTile, p.n - base);
    T x[kTileItems];
    tile_load_direct<T>((const T*)p.w, p.n, base, x);
    TileScan<A> s;
    const int e0 = threadIdx.x * kTileItems;
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
      if (e0 + j < len) flags |= wflags(x[j]);
      s.loc[j] = (A)x[j];
    }
    tile_scan<A>(s, warp_sums);
    // aggregate := tile-local inclusive value at the tile's last position
    if (threadIdx.x == kTileThreads - 1) p.agg[b] = add_rn(s.thread_excl, s.loc[kTileItems - 1]);
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(&cta_flags, flags);
  __syncthreads();
  if (threadIdx.x == 0) {
    tile_flags(p)[blockIdx.x] = cta_flags;
    __threadfence();
    const unsigned t = atomicAdd(&p.state->done, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  if (threadIdx.x == 0) cta_flags = 0;
  __threadfence();
  // exclusive scan over the tile aggregates, 4096 at a time through shared
  // memory (coalesced loads): serial within a thread's 16, Kogge-Stone across
  // threads, serial across warps, serial carry across chunks (fixed
  // association => deterministic)
  A* sagg = reinterpret_cast<A*>(stage);  // >= 4096 * 4 bytes; A=double needs 32 KB -> 2 passes of 2048
  constexpr int kChunk = (kTile * sizeof(T)) / sizeof(A);
  constexpr int kPer = kChunk / kTileThreads;
  const int T_ = (int)p.tiles;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  A carry = A(0);
  uint32_t fl = 0;
  for (int c0 = 0; c0 < T_; c0 += kChunk) {
    const int cn = min(kChunk, T_ - c0);
    for (int i = threadIdx.x; i < cn; i += kTileThreads) sagg[i] = __ldcg(p.agg + c0 + i);
    __syncthreads();
    A v[kPer];
    A mine = A(0);
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int i = threadIdx.x * kPer + k;
      v[k] = i < cn ? sagg[i] : A(0);
      mine = add_rn(mine, v[k]);
    }
    const A incl = warp_inclusive_scan(mine);
    A ex = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) ex = A(0);
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    A wp = carry, tot = carry;
    for (int u = 0; u < kTileThreads / 32; ++u) {
      if (u < warp) wp = add_rn(wp, warp_sums[u]);
      tot = add_rn(tot, warp_sums[u]);
    }
    A run = lane ? add_rn(wp, ex) : wp;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int i = threadIdx.x * kPer + k;
      if (i < cn) sagg[i] = run;
      run = add_rn(run, v[k]);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < cn; i += kTileThreads) p.excl[c0 + i] = sagg[i];
    carry = tot;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < (int)gridDim.x; i += kTileThreads) fl |= __ldcg(tile_flags(p) + i);
  fl = __reduce_or_sync(0xffffffffu, fl);
  if (lane == 0 && fl) atomicOr(&cta_flags, fl);
  __syncthreads();
  if (threadIdx.x == 0) {
    p.excl[T_] = carry;  // the total
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
  tile_load_direct<T>((const T*)p.w, p.n, base, x);
  TileScan<A> s;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) s.loc[j] = (A)x[j];
  tile_scan<A>(s, warp_sums);
  const A total = p.excl[p.tiles];
  const A sfx = sizeof(A) == 8 ? (A)p.n / total * (A)2147483648.0 : A(0);  // N/total * 2^31
  const long long ufx = sizeof(A) == 8 ? __double2ll_rn((double)p.u_sys * 2147483648.0) : 0;
  const uint32_t dr = (uint32_t)(p.n >> 13) + 16u;
  const A ex = p.excl[b];
  const A tex = s.thread_excl;
  const int last = (p.n - 1 - base < kTile) ? (int)(p.n - 1 - base) : -1;
  const int e0 = threadIdx.x * kTileItems;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) {
    const A W = add_rn(ex, add_rn(tex, s.loc[j]));
    o[j] = offspring_of<T, A, UM>(W, total, sfx, ufx, dr, p.n, p);
    if (e0 + j == last) o[j] = (int32_t)p.n;  // O[N-1] = N
  }
  o_prev = 0;
  if (b > 0) {
    const A Wp = add_rn(p.excl[b - 1], p.agg[b - 1]);  // W at the last position of tile b-1
    o_prev = offspring_of<T, A, UM>(Wp, total, sfx, ufx, dr, p.n, p);
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
// K3: persistent, warp-pipelined.  Each warp owns a contiguous run of
// 256-index chunks (index = chunk + 32 k + lane: coalesced).  Per iteration
// it (1) loads a chunk and resolves the trivial indices (has offspring, or a
// loser slot that claims its own hole), (2) appends the holes that are first
// slots -- pending backward chains -- to its shared-memory queue, and (3)
// advances every queued chain by one step.  Chunk loads and chain loads of an
// iteration are independent, so each iteration costs about one L2 round trip
// and the chain latency hides under the streaming; the queue drains at the end.
constexpr int kQCap = 512;        // queue entries per warp
constexpr int kChunkK = 8;        // indices per lane per chunk
constexpr int kChunkSpan = 32 * kChunkK;
constexpr int kInplaceWarps = 8;  // warps per CTA

struct WarpQueue {
  int32_t elem[kQCap];
  uint32_t node[kQCap];
  uint8_t steps[kQCap];
};

// one round over the queue: every entry takes one backward step; finished
// entries write c, the rest are compacted in place (order preserved)
__device__ __forceinline__ int queue_round(WarpQueue& q, int qlen, const uint32_t* __restrict__ words,
                                           int32_t* __restrict__ c, int& longest, bool& overflow) {
  const int lane = threadIdx.x & 31;
  int out = 0;
  for (int g = 0; g < qlen; g += 128) {
    uint32_t wz[4];
    int idx[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      idx[r] = g + 32 * r + lane;
      if (idx[r] < qlen) wz[r] = __ldcg(words + q.node[idx[r]]);
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const bool valid = idx[r] < qlen;
      bool keep = false;
      int32_t e = 0;
      int st = 0;
      if (valid) {
        e = q.elem[idx[r]];
        st = q.steps[idx[r]] + 1;
        if (!(wz[r] & kFirst)) {
          c[e] = (int32_t)(wz[r] & kParentMask);
          longest = max(longest, st);
        } else if (st >= kBackBound) {
          overflow = true;
        } else {
          keep = true;
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      __syncwarp();
      if (keep) {
        const int pos = out + __popc(m & ((1u << lane) - 1));
        q.elem[pos] = e;
        q.node[pos] = wz[r] & kParentMask;
        q.steps[pos] = (uint8_t)st;
      }
      out += __popc(m);
      __syncwarp();
    }
  }
  return out;
}

__global__ void __launch_bounds__(32 * kInplaceWarps) k_dv_inplace(const uint32_t* __restrict__ words,
                                                                  const uint32_t* __restrict__ bitmap, int64_t n,
                                                                  int32_t* __restrict__ c, int32_t* max_steps,
                                                                  DvState* state, uint32_t* status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  griddep_wait();
  if (state->flags & kNeedsRepair) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpQueue& q = reinterpret_cast<WarpQueue*>(smem_raw)[warp];
  const int64_t chunks = (n + kChunkSpan - 1) / kChunkSpan;
  const int64_t gw = (int64_t)blockIdx.x * kInplaceWarps + warp, nw = (int64_t)gridDim.x * kInplaceWarps;
  const int64_t ch0 = chunks * gw / nw, ch1 = chunks * (gw + 1) / nw;
  int qlen = 0;
  int longest = 0;
  bool overflow = false;
  for (int64_t ch = ch0; ch < ch1; ++ch) {
    const int64_t cb = ch * kChunkSpan;
    uint32_t wd[kChunkK], bw[kChunkK];
#pragma unroll
    for (int k = 0; k < kChunkK; ++k) {
      const int64_t i = cb + 32 * k + lane;
      wd[k] = i < n ? __ldcs(words + i) : 0u;
      bw[k] = (cb + 32 * k < n) ? __ldcs(bitmap + ((cb >> 5) + k)) : 0u;
    }
    // advance the pending chains while the chunk loads are in flight
    if (qlen) qlen = queue_round(q, qlen, words, c, longest, overflow);
#pragma unroll
    for (int k = 0; k < kChunkK; ++k) {
      const int64_t i = cb + 32 * k + lane;
      const bool in = i < n;
      const bool has = (bw[k] >> lane) & 1u;
      const bool pend = in && !has && (wd[k] & kFirst);
      if (in) __stcs(c + i, has ? (int32_t)i : (int32_t)(wd[k] & kParentMask));
      const unsigned m = __ballot_sync(0xffffffffu, pend);
      if (pend) {
        const int pos = qlen + __popc(m & ((1u << lane) - 1));
        q.elem[pos] = (int32_t)i;
        q.node[pos] = wd[k] & kParentMask;
        q.steps[pos] = 0;
      }
      qlen += __popc(m);
    }
    __syncwarp();
    // keep room for the next chunk
    while (qlen > kQCap - kChunkSpan) qlen = queue_round(q, qlen, words, c, longest, overflow);
  }
  while (qlen) qlen = queue_round(q, qlen, words, c, longest, overflow);
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
  static int occ1 = -1;
  if (occ1 < 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, k_dv_reduce<T, A>, kTileThreads, 0);
    if (occ1 < 1) occ1 = 1;
  }
  const unsigned grid1 = (unsigned)min((int64_t)num_sms() * occ1, p.tiles);
  k_dv_reduce<T, A><<<grid1, kTileThreads, 0, s>>>(p);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || stages < 2) return e;
  e = launch_pdl(k_dv_expand<T, A, UM>, dim3(tiles), dim3(kTileThreads), s, false, p);
  if (e != cudaSuccess || stages < 3) return e;
  static int occ3 = -1;
  const size_t smem3 = sizeof(WarpQueue) * kInplaceWarps;
  if (occ3 < 0) {
    e = cudaFuncSetAttribute(k_dv_inplace, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, k_dv_inplace, 32 * kInplaceWarps, smem3);
    if (e != cudaSuccess) return e;
    if (occ3 < 1) occ3 = 1;
  }
  e = launch_pdl_smem(k_dv_inplace, dim3(num_sms() * occ3), dim3(32 * kInplaceWarps), smem3, s, false,
                      (const uint32_t*)p.words, (const uint32_t*)p.bitmap, p.n, p.c, p.max_steps, p.state, p.status);
  if (e != cudaSuccess || stages < 4) return e;
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
