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
  A* sub;        // [8 * tiles] subtile (512-element) aggregates, written by K1
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
  // one weight shard of a larger vector (sharded.py protocol v3); the single
  // GPU path has gn = n, gpt = null, gbase = 0, words covering [0, n)
  int64_t gn;        // N of the offspring formula (the global N)
  const double* gpt; // non-null: {weight before this shard, W_N} on the device
  int glast;         // the shard holds the global last particle (O[N-1] = N)
  int gfirst;        // the shard starts at particle 0
  int64_t gbase;     // global index of local element 0 (parents and slots are global)
  int64_t wlo, whi;  // `words` holds slots [wlo, whi) at words[slot - wlo]; outside -> PFR_ST_OVERFLOW
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

// Branch-free fast path for the streaming loops: the fixed-point O and an
// "unsafe" flag (the fractional part within the margin of an integer, or an
// accumulator without the fast path); the caller redoes flagged elements with
// offspring_exact after its loop, so the hot loop has no call and no
// divergent branch.  Systematic: t = round(W * sfx + ufx) from ONE fma
// against 2^52 + ufx (ufx is an integer, so this is round(W * sfx) + ufx up
// to the tie rule, inside the same error bound); only t's fraction matters
// because every stratum has the same offset (resamplers.py:145-153).
template <typename T, typename A, int UM>
__device__ __forceinline__ int32_t offspring_fast(A W, const FxParams& f, double csys, int32_t n, bool& unsafe,
                                                  const DvArgs<A>& p) {
  if constexpr (sizeof(A) == 8) {
    if constexpr ((UM & 3) == kUSys) {
      const double t = __fma_rn(W, f.sfx, csys);
      const uint32_t lo = (uint32_t)__double2loint(t);
      const uint32_t hi = (uint32_t)__double2hiint(t) - 0x43300000u;
      const uint32_t o = f.S >= 32 ? hi : __funnelshift_r(lo, hi, f.S);
      unsafe = ((lo + kFxMargin) & f.mask) <= 2 * kFxMargin;
      return min((int32_t)o, n);
    } else {
      const long long r = fx_round(W, f.sfx);
      long long k = (r >> f.S) + 1;
      if (k > n) k = n;
      if (k < 1) k = 1;
      const long long t = r + fx_round((double)stratum_u<T, A, UM>(k - 1, p), f.scale);
      unsafe = !(fx_safe(r, f.mask) && fx_safe(t, f.mask));
      return min((int32_t)(t >> f.S), n);
    }
  } else {
    unsafe = true;
    return 0;
  }
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
__device__ __forceinline__ void lane_weights(const DvArgs<A>& p, int64_t e0, T (&x)[kTileItems]) {
  constexpr int kPerVec = 16 / sizeof(T);
  const T* in = (const T*)p.w;
  if (e0 + kTileItems <= p.n && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
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
    for (int j = 0; j < kTileItems; ++j) x[j] = (e0 + j < p.n) ? in[e0 + j] : T(0);
  }
  if constexpr (LW) {
    const T m = (T)from_ordered(__ldcg(p.logw_max));
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

// ---------------------------------------------------------------------------
// The association of W (fast path; fixed by indices alone, so deterministic).
// A SUBTILE is 512 elements handled by one warp, 16 consecutive per lane.
//   loc_j   serial inclusive sum of the lane's elements (in A)
//   tex     exclusive Kogge-Stone scan of the lane totals (lane 0: 0)
//   sub(s)  = tex(lane 31) + loc_15(lane 31)            (K1 stores it)
//   Q_q(b)  = serial fold of sub(8b), ..., sub(8b + q - 1)  (Q_0 = 0)
//   agg(b)  = Q_8(b), the tile aggregate the hierarchy scans (pfr_hier.cuh)
//   SP(s)   = tile_excl(b) + Q_q(b)                 for s = 8b + q
//   W       = SP(s) + (tex + loc_j)
// so W at the last element of subtile s is SP(s) + sub(s), which the next
// subtile recomputes from the same stored values for its O(prev): slot ranges
// of neighbouring subtiles always meet exactly.
constexpr int kSub = 32 * kTileItems;  // 512
constexpr int kSubPerTile = kTile / kSub;  // 8

// K1: one CTA per 4096-element tile: validation flags, the 8 subtile
// aggregates and the tile aggregate; tile prefixes built hierarchically.
template <typename T, typename A, int kTilesPerCta, bool LW = false>
__global__ void __launch_bounds__(kTileThreads) k_dv_reduce(DvArgs<A> p) {
  static_assert(kTilesPerCta == 1, "one tile per CTA");
  __shared__ A warp_aggs[kTileThreads / 32];
  __shared__ uint32_t warp_flags[kTileThreads / 32];
  __shared__ uint32_t cta_flags;
  __shared__ int stage;
  const int64_t b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x[kTileItems];
  lane_weights<T, A, LW>(p, b * kTile + (int64_t)threadIdx.x * kTileItems, x);
  FlagAcc<T> facc;
  A loc = (A)x[0];
  facc.add(x[0]);
#pragma unroll
  for (int j = 1; j < kTileItems; ++j) {
    facc.add(x[j]);
    loc = add_rn(loc, (A)x[j]);
  }
  const A incl = warp_inclusive_scan(loc);
  const A tex = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 31) {
    const A sa = add_rn(tex, loc);
    p.sub[b * kSubPerTile + warp] = sa;
    warp_aggs[warp] = sa;
  }
  const uint32_t flags = __reduce_or_sync(0xffffffffu, facc.flags());
  if (lane == 0) warp_flags[warp] = flags;
  __syncthreads();
  if (threadIdx.x == kTileThreads - 1) {
    A t = warp_aggs[0];
    uint32_t f = warp_flags[0];
#pragma unroll
    for (int w = 1; w < kTileThreads / 32; ++w) {
      t = add_rn(t, warp_aggs[w]);
      f |= warp_flags[w];
    }
    p.agg[b] = t;
    cta_flags = f;
  }
  hier_tile_done(hier_of(p), b, &cta_flags, &stage, p.status);
  if (stage == 2 && threadIdx.x == 0) p.state->flags = 0;  // pipeline flags of this delivery
}

// subtile s -> O of the lane's 16 elements, and O(prev) = O at the last
// element of subtile s-1 (0 for s = 0), uniform.  One warp, no block barrier;
// every prefix value is fetched by one lane, all in one round trip with the
// weights.
template <typename T, typename A, int UM, bool kShard = false>
__device__ __forceinline__ void subtile_offspring(const DvArgs<A>& p, int64_t s, int32_t (&o)[kTileItems],
                                                  int32_t& o_prev) {
  const int lane = threadIdx.x & 31;
  const int64_t e0 = s * kSub + (int64_t)lane * kTileItems;
  const int64_t b = s >> 3;
  const int q = (int)(s & 7);
  const Hier<A> h = hier_of(p);
  A v = A(0);
  if (lane < 8) {
    if (lane < q) v = __ldcg(p.sub + b * kSubPerTile + lane);
  } else if (lane < 16) {
    if (q == 0 && b > 0) v = __ldcg(p.sub + (b - 1) * kSubPerTile + (lane - 8));
  } else if (lane == 16) {
    v = __ldcg(h.group_prefix() + b / kGroupTiles);
  } else if (lane == 17) {
    v = __ldcg(h.excl + b);
  } else if (lane == 18) {
    if (b > 0) v = __ldcg(h.group_prefix() + (b - 1) / kGroupTiles);
  } else if (lane == 19) {
    if (b > 0) v = __ldcg(h.excl + b - 1);
  } else if (lane == 20) {
    v = h.total();
  }
  T x[kTileItems];
  lane_weights<T, A, (UM & kULogW) != 0>(p, e0, x);
  // uniform prefix arithmetic (every lane, identical)
  const A te = add_rn(__shfl_sync(0xffffffffu, v, 16), __shfl_sync(0xffffffffu, v, 17));
  A Q = A(0), Qm = A(0);
#pragma unroll
  for (int i = 0; i < 7; ++i) {
    const A a = __shfl_sync(0xffffffffu, v, i);
    if (i < q) {
      Qm = Q;
      Q = add_rn(Q, a);
    }
  }
  const A SP = add_rn(te, Q);
  A wprev;
  if (q > 0) {
    wprev = add_rn(add_rn(te, Qm), __shfl_sync(0xffffffffu, v, q - 1));
  } else {
    const A tep = add_rn(__shfl_sync(0xffffffffu, v, 18), __shfl_sync(0xffffffffu, v, 19));
    A Qp = A(0);
#pragma unroll
    for (int i = 8; i < 15; ++i) Qp = add_rn(Qp, __shfl_sync(0xffffffffu, v, i));
    wprev = add_rn(add_rn(tep, Qp), __shfl_sync(0xffffffffu, v, 15));
  }
  // sharded: W of the global vector = (weight before the shard) + local W
  constexpr bool shard = kShard;
  A gp = A(0), total = __shfl_sync(0xffffffffu, v, 20);
  if constexpr (shard) {
    gp = (A)__ldcg(p.gpt);
    total = (A)__ldcg(p.gpt + 1);
  }
  auto globalW = [&](A wl) {
    if constexpr (shard)
      return add_rn(gp, wl);
    else
      return wl;
  };
  // the lane's serial partials and the Kogge-Stone exclusive offset; when the
  // weights are narrower than the accumulator the partials are recomputed in
  // the second loop (the same sequence) instead of being kept in registers
  A tot = (A)x[0];
#pragma unroll
  for (int j = 1; j < kTileItems; ++j) tot = add_rn(tot, (A)x[j]);
  const A incl = warp_inclusive_scan(tot);
  A tex = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) tex = A(0);
  const int64_t gn = shard ? p.gn : p.n;
  const FxParams fx = fx_params<A>(gn, total, p.u_sys, p.fx_S);
  const double csys = 4503599627370496.0 + (double)fx.ufx;  // 2^52 + ufx (exact)
  const int32_t gN = (int32_t)gn;
  A loc = A(0);
  uint32_t unsafe = 0;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) {
    loc = j ? add_rn(loc, (A)x[j]) : (A)x[0];
    bool u;
    o[j] = offspring_fast<T, A, UM>(globalW(add_rn(SP, add_rn(tex, loc))), fx, csys, gN, u, p);
    unsafe |= (uint32_t)u << j;
  }
  if (__any_sync(0xffffffffu, unsafe)) {  // rare: the reference's exact IEEE sequence
    loc = A(0);
    for (int j = 0; j < kTileItems; ++j) {
      loc = j ? add_rn(loc, (A)x[j]) : (A)x[0];
      if ((unsafe >> j) & 1u)
        o[j] = offspring_exact<T, A, UM>(globalW(add_rn(SP, add_rn(tex, loc))), total, gn, p);
    }
  }
  // the final subtile of the global vector: O[N-1] = N, padding past N stays
  // at N (a shard that is not last needs nothing: its zero padding repeats
  // the last O)
  if ((!shard || p.glast) && e0 + kTileItems > p.n - 1) {
    const int64_t lim = p.n - 1 - e0;
#pragma unroll
    for (int j = 0; j < kTileItems; ++j)
      if (j >= lim) o[j] = gN;
  }
  if (s > 0)
    o_prev = offspring_of<T, A, UM>(globalW(wprev), total, fx, gn, p);
  else  // before the shard W is exactly the weight before it (sharded.py)
    o_prev = (shard && !p.gfirst) ? offspring_of<T, A, UM>(gp, total, fx, gn, p) : 0;
}

// ---------------------------------------------------------------------------
// tile -> O (registers, blocked: thread t owns elements [16t, 16t+16)): shared
// by K2 (cumulative offspring) and the repair path.  Warp w computes subtile
// 8b + w.  Index math is 32-bit inside the tile (N < 2^31).
template <typename T, typename A, int UM>
__device__ __forceinline__ void tile_offspring(const DvArgs<A>& p, int64_t b, uint4* stage, A* warp_sums,
                                               int32_t (&o)[kTileItems], int32_t& o_prev) {
  (void)stage;
  (void)warp_sums;
  const int64_t base = b * kTile;
  if (p.Wser) {
    // accum = SERIAL: the reference's own W (np.cumsum, serial fold) is given;
    // the offspring formula then runs in the weight dtype (A = T), exactly
    // as resamplers.py:139-153
    const int last = (p.n - 1 - base < kTile) ? (int)(p.n - 1 - base) : -1;
    const int e0 = threadIdx.x * kTileItems;
    A Wv[kTileItems];
    tile_load_any<A>(p.Wser, p.n, base, Wv);
    const A total = __ldg(p.Wser + p.n - 1);
    const FxParams fx = fx_params<A>(p.n, total, p.u_sys, p.fx_S);
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) o[j] = offspring_of<T, A, UM>(Wv[j], total, fx, p.n, p);
    if (last >= 0) {
#pragma unroll
      for (int j = 0; j < kTileItems; ++j)
        if (e0 + j >= last) o[j] = (int32_t)p.n;
    }
    o_prev = b > 0 ? offspring_of<T, A, UM>(__ldg(p.Wser + base - 1), total, fx, p.n, p) : 0;
    return;
  }
  __shared__ int32_t s_oprev;
  int32_t op;
  subtile_offspring<T, A, UM>(p, b * kSubPerTile + (threadIdx.x >> 5), o, op);
  if (threadIdx.x == 0) s_oprev = op;
  __syncthreads();
  o_prev = s_oprev;
  __syncthreads();
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

// ---------------------------------------------------------------------------
// K2w / K3w: the systematic / stratified delivery's production and
// resolution as two warp-level kernels.  The unit of work is a 512-element
// SUBTILE owned by one warp (16 consecutive elements per lane): no block
// barrier anywhere, so every warp of the SM hides the others' latency.
constexpr int kFWarps = 8;      // warps per CTA
constexpr int kWBuf = 1024;     // per-warp staging of slot positions (4 KB)

struct __align__(16) WarpSmem {
  uint32_t buf[kWBuf];
};

// Words (parent | FIRST) for the subtile's slot range [o_prev, oend) and its
// has-offspring bitmap, by one warp.  Per 512-slot chunk (16-byte aligned):
// every parent with offspring writes its index at its first slot O[j-1] (a
// plain scattered store: first slots are distinct), all other positions hold
// -1; then a max-scan over the slot positions (lane l owns 16 consecutive
// ones; Kogge-Stone over the lane maxima; a carry across chunks) gives every
// slot its parent, since parents increase with the slot.  No loops over
// offspring counts, no atomics, 16-byte coalesced stores.  Positions are
// XOR-swizzled in 16-byte units so the per-lane vector accesses are
// bank-conflict free.
__device__ __forceinline__ int sw_hd(int v) { return v ^ ((v >> 3) & 3); }  // 16-byte unit swizzle
template <bool kShard = false>
__device__ __forceinline__ bool subtile_expand(const int32_t (&o)[kTileItems], int32_t prev_l, int32_t o_prev,
                                               int32_t oend, int64_t s, int64_t n, uint32_t* __restrict__ words,
                                               uint32_t* __restrict__ bitmap, WarpSmem& W, int64_t gbase = 0,
                                               int64_t wlo = 0, int64_t whi = INT64_MAX) {
  // words[slot - wlo] for slots in [wlo, whi); parents are written as global
  // numbers gbase + local index; returns false when a slot fell outside
  // (a shard whose window overhangs its halo: the caller falls back)
  const int lane = threadIdx.x & 31;
  const int64_t base = s * kSub;
  const int64_t e0 = base + (int64_t)lane * kTileItems;
  bool outside = false;
  uint32_t bits = 0;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) {
    const int pv = j ? o[j - 1] : prev_l;
    if (o[j] > pv) bits |= 1u << j;  // padding past N repeats O = N: never a parent
  }
  const uint32_t hi = __shfl_down_sync(0xffffffffu, bits, 1);
  if ((lane & 1) == 0 && e0 < n) bitmap[(base >> 5) + (lane >> 1)] = bits | (hi << 16);
  if (oend <= o_prev) return true;  // uniform: no slots
  int32_t* hb = reinterpret_cast<int32_t*>(W.buf);
  int4* hb4 = reinterpret_cast<int4*>(W.buf);
  const int pb = (int)(gbase + e0);  // global index of the lane's first parent
  int carry = -1;
  const bool single = oend - (o_prev & ~3) <= kWBuf;
  // chunks of kWBuf = 1024 positions (a typical subtile's ~512 slots fit one
  // chunk whatever their alignment), scanned as up to two rows of 512
  for (int c0 = o_prev & ~3; c0 < oend; c0 += kWBuf) {
    const int rows = oend - c0 > kSub ? 2 : 1;
#pragma unroll
    for (int q = 0; q < 4; ++q) hb4[sw_hd(4 * lane + q)] = make_int4(-1, -1, -1, -1);
    if (rows == 2) {
#pragma unroll
      for (int q = 0; q < 4; ++q) hb4[sw_hd(128 + 4 * lane + q)] = make_int4(-1, -1, -1, -1);
    }
    __syncwarp();
    // head of parent j at its first slot O[j-1] - c0; the swizzle
    // (sw_hd(r >> 2) << 2) | (r & 3) folds to r ^ ((r >> 3) & 12).  In the
    // usual single-chunk case (the whole range fits one chunk) every head
    // lies in [0, oend - c0) within the buffer, so the range test is dropped
    // (uniform branch; later chunks of a long range see heads below c0)
    if (single) {
      int r = prev_l - c0;
#pragma unroll
      for (int j = 0; j < kTileItems; ++j) {
        if ((bits >> j) & 1u) hb[r ^ ((r >> 3) & 12)] = pb + j;
        r = o[j] - c0;
      }
    } else {
      int r = prev_l - c0;
#pragma unroll
      for (int j = 0; j < kTileItems; ++j) {
        if (((bits >> j) & 1u) && (unsigned)r < (unsigned)kWBuf) hb[r ^ ((r >> 3) & 12)] = pb + j;
        r = o[j] - c0;
      }
    }
    __syncwarp();
    for (int row = 0; row < rows; ++row) {
      int4 hv[4];
      int mx = -1;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        hv[q] = hb4[sw_hd(128 * row + 4 * lane + q)];
        mx = max(mx, max(max(hv[q].x, hv[q].y), max(hv[q].z, hv[q].w)));
      }
      int incl = mx;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl = max(incl, t);
      }
      int cur = __shfl_up_sync(0xffffffffu, incl, 1);
      if (lane == 0) cur = -1;
      cur = max(cur, carry);
      carry = max(carry, __shfl_sync(0xffffffffu, incl, 31));
      uint32_t wv[kTileItems];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e[4] = {hv[q].x, hv[q].y, hv[q].z, hv[q].w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          cur = max(cur, e[t]);
          wv[4 * q + t] = (uint32_t)cur | (e[t] >= 0 ? kFirst : 0u);
        }
      }
      const int s0 = c0 + kSub * row + lane * kTileItems;
      if (s0 >= o_prev && s0 + kTileItems <= oend && (!kShard || (s0 >= wlo && s0 + kTileItems <= whi))) {
        uint4* dst = reinterpret_cast<uint4*>(words + (s0 - wlo));
#pragma unroll
        for (int q = 0; q < kTileItems / 4; ++q)
          dst[q] = make_uint4(wv[4 * q], wv[4 * q + 1], wv[4 * q + 2], wv[4 * q + 3]);
      } else if (s0 < oend && s0 + kTileItems > o_prev) {
        // an edge row: whole 16-byte groups as vectors, element stores only
        // in the (at most two) groups the range cuts
#pragma unroll
        for (int q = 0; q < kTileItems / 4; ++q) {
          const int v0 = s0 + 4 * q;
          if (v0 >= o_prev && v0 + 4 <= oend && (!kShard || (v0 >= wlo && v0 + 4 <= whi))) {
            *reinterpret_cast<uint4*>(words + (v0 - wlo)) = make_uint4(wv[4 * q], wv[4 * q + 1], wv[4 * q + 2], wv[4 * q + 3]);
          } else if (v0 < oend && v0 + 4 > o_prev) {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int64_t sl = v0 + t;
              if (sl >= o_prev && sl < oend) {
                if (!kShard || (sl >= wlo && sl < whi))
                  words[sl - wlo] = wv[4 * q + t];
                else
                  outside = true;
              }
            }
          }
        }
      }
    }
    __syncwarp();
  }
  if constexpr (kShard) return !__any_sync(0xffffffffu, outside);
  return true;
}

// K2w: produce every subtile (grid-stride): O from the position formula,
// the slot words of the subtile's slot range and its has-offspring bitmap.
template <typename T, typename A, int UM, bool kShard = false>
__global__ void __launch_bounds__(kFWarps * 32, 3) k_dv_produce(DvArgs<A> p) {
  extern __shared__ __align__(16) unsigned char fused_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpSmem& W = reinterpret_cast<WarpSmem*>(fused_smem)[warp];
  griddep_wait();
  const int64_t n = p.n;
  const int64_t nS = (n + kSub - 1) / kSub;
  for (int64_t k = blockIdx.x * (int64_t)kFWarps + warp; k < nS; k += (int64_t)gridDim.x * kFWarps) {
    int32_t o[kTileItems];
    int32_t o_prev;
    subtile_offspring<T, A, UM, kShard>(p, k, o, o_prev);
    int32_t prev_l = __shfl_up_sync(0xffffffffu, o[kTileItems - 1], 1);
    if (lane == 0) prev_l = o_prev;
    const bool bad = __any_sync(0xffffffffu, o[0] < prev_l);
    const int32_t oend = __shfl_sync(0xffffffffu, o[kTileItems - 1], 31);
    if (!bad) {
      if (!subtile_expand<kShard>(o, prev_l, o_prev, oend, k, n, p.words, p.bitmap, W, p.gbase, p.wlo, p.whi) &&
          lane == 0)
        status_or(p.status, PFR_ST_OVERFLOW);  // a shard's window beyond its halo (sharded.py falls back)
    } else if (lane == 0) {
      atomicOr(&p.state->flags, kNeedsRepair);
      if (kShard) status_or(p.status, PFR_ST_OVERFLOW);  // a shard has no repair path: the host falls back
    }
  }
}

// K3w's chain queue: one per warp, in shared memory.
constexpr int kRQ = 1024;     // entries (>= kRThresh + the 512 chains one subtile can add)
constexpr int kRThresh = 256; // a pass runs once this many chains wait (160-384 measure alike)
struct ResolveQ {
  uint2 xz[kRQ];  // (hole, next slot)
  uint8_t st[kRQ];
};

// One step for every queued chain when every word is written: dense, eight
// loads per lane in flight, survivors compacted to the front.  Entries are
// (local hole, global slot); words are indexed by global slot and exist for
// [wlo, whi) only (a shard's halo: a chain leaving it sets the overflow flag
// and the host falls back).
template <bool kShard = false, bool kTrack = true>
__device__ __forceinline__ int lean_pass(ResolveQ& Q, int lane, int qlen, const uint32_t* __restrict__ words,
                                         int32_t* __restrict__ c, int64_t wlo, int64_t whi, int64_t gbase,
                                         int& longest, bool& overflow) {
  constexpr int K = 8;
  int out = 0;
  for (int b = 0; b < qlen; b += 32 * K) {
    uint2 xz[K];
    uint32_t w[K];
    int st[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int e = b + 32 * i + lane;
      if (e < qlen) {
        xz[i] = Q.xz[e];
        if constexpr (kTrack) st[i] = Q.st[e] + 1;
        const int64_t z = xz[i].y;
        w[i] = (!kShard || (z >= wlo && z < whi)) ? __ldcg(words + z) : 0xFFFFFFFFu;
      }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (b + 32 * i >= qlen) break;  // warp-uniform
      const bool valid = b + 32 * i + lane < qlen;
      bool keep = false;
      if (valid) {
        const uint32_t par = w[i] & kParentMask;
        if (kShard && w[i] == 0xFFFFFFFFu) {
          overflow = true;  // outside the shard's halo (or an unwritten word): the host falls back
        } else if (!(w[i] & kFirst)) {
          c[xz[i].x] = (int32_t)par;
          if constexpr (kTrack) longest = max(longest, st[i]);
        } else if ((kTrack && st[i] >= kBackBound) || (kShard && (int64_t)par >= whi)) {
          overflow = true;  // abandoned: the rare-path kernel resolves every chain
        } else {
          keep = true;
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int pos = out + __popc(m & ((1u << lane) - 1));
        Q.xz[pos] = make_uint2(xz[i].x, w[i] & kParentMask);
        if constexpr (kTrack) Q.st[pos] = (uint8_t)st[i];
      }
      out += __popc(m);
    }
    __syncwarp();
  }
  (void)gbase;
  return out;
}

// K3w: resolve every subtile.  Lane l takes indices 128q + 4l + {0..3} of
// the subtile (q = 0..3): 16-byte coalesced loads of the words (prefetched
// one subtile ahead) and stores of c, the has-offspring bits from 4 bitmap
// words.  Trivial indices are final at once; first-slot holes join the
// warp's chain queue, which advances one step for every queued chain per
// pass, a pass running once enough chains wait -- so a pass costs one L2
// round trip for several subtiles' chains, overlapped with the next
// subtile's prefetched loads.
// kTrack (max_steps requested): per-chain step counts for max_steps and the
// per-chain bound; otherwise the drain is bounded by its pass count (a chain
// left then is resolved by the rare path, as an abandoned one)
template <typename A, bool kShard = false, bool kTrack = true>
__global__ void __launch_bounds__(kFWarps * 32, 2) k_dv_resolve(DvArgs<A> p) {
  extern __shared__ __align__(16) unsigned char fused_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  ResolveQ& Q = reinterpret_cast<ResolveQ*>(fused_smem)[warp];
  griddep_wait();
  if (p.state->flags & kNeedsRepair) return;
  const int64_t n = p.n;
  const uint32_t nn = (uint32_t)n;
  const int64_t nS = (n + kSub - 1) / kSub;
  int qlen = 0, longest = 0;
  bool overflow = false;
  // slot / parent numbers are global (gbase + local index) and words[slot -
  // wlo] covers [wlo, whi): the single-GPU call has gbase = wlo = 0, whi = n
  const int64_t gbase = kShard ? p.gbase : 0, wlo = kShard ? p.wlo : 0, whi = kShard ? p.whi : p.n;
  const uint32_t* __restrict__ wds = p.words - wlo;  // indexed by global slot (only inside [wlo, whi))
  auto pass = [&]() {
    return lean_pass<kShard, kTrack>(Q, lane, qlen, wds, p.c, wlo, whi, gbase, longest, overflow);
  };
  const bool vec_ok = !kShard || ((gbase - wlo) & 3) == 0;  // 16-byte word loads need a 4-aligned offset
  const uint4* __restrict__ words4 = reinterpret_cast<const uint4*>(p.words + (gbase - wlo));
  int4* __restrict__ c4 = reinterpret_cast<int4*>(p.c);
  const int64_t stride = (int64_t)gridDim.x * kFWarps;
  auto load = [&](int64_t rr, uint4 (&wv)[4], uint32_t (&bm)[4]) {
    const uint32_t xb = (uint32_t)rr * kSub;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t x0 = xb + 128 * q + 4 * lane;
      if (xb + kSub <= nn && vec_ok) {
        wv[q] = __ldg(words4 + (x0 >> 2));
      } else {
        const uint32_t* wx = p.words + (gbase - wlo) + x0;
        wv[q].x = x0 < nn ? __ldg(wx) : 0u;
        wv[q].y = x0 + 1 < nn ? __ldg(wx + 1) : 0u;
        wv[q].z = x0 + 2 < nn ? __ldg(wx + 2) : 0u;
        wv[q].w = x0 + 3 < nn ? __ldg(wx + 3) : 0u;
      }
      bm[q] = x0 < nn ? __ldg(p.bitmap + (x0 >> 5)) >> (x0 & 31) : 0u;
    }
  };
  int64_t rr = blockIdx.x * (int64_t)kFWarps + warp;
  uint4 nwv[4];
  uint32_t nbm[4];
  if (rr < nS) load(rr, nwv, nbm);
  for (; rr < nS; rr += stride) {
    const uint32_t xb = (uint32_t)rr * kSub;
    const bool full = xb + kSub <= nn && vec_ok;
    uint4 wv[4];
    uint32_t bm[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      wv[q] = nwv[q];
      bm[q] = nbm[q];
    }
    if (rr + stride < nS) load(rr + stride, nwv, nbm);  // prefetch the next subtile
    uint32_t pend = 0;  // bit 4q + t
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t x0 = xb + 128 * q + 4 * lane;
      const uint32_t e[4] = {wv[q].x, wv[q].y, wv[q].z, wv[q].w};
      int32_t o[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const bool has = (bm[q] >> t) & 1u;
        o[t] = has ? (int32_t)(gbase + x0 + t) : (int32_t)(e[t] & kParentMask);
        if (!has && (e[t] & kFirst) && x0 + t < nn) pend |= 1u << (4 * q + t);
      }
      // pending holes get a placeholder, overwritten when their chain
      // resolves (__syncwarp orders the two stores)
      if (full) {
        __stcs(c4 + (x0 >> 2), make_int4(o[0], o[1], o[2], o[3]));
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (x0 + t < nn) p.c[x0 + t] = o[t];
      }
    }
    const int cnt = __popc(pend);
    int off = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, off, d);
      if (lane >= d) off += t;
    }
    const int total = __shfl_sync(0xffffffffu, off, 31);
    off -= cnt;
    while (qlen + total > kRQ) qlen = pass();
    int pos = qlen + off;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t e[4] = {wv[q].x, wv[q].y, wv[q].z, wv[q].w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if ((pend >> (4 * q + t)) & 1u) {
          Q.xz[pos] = make_uint2(xb + 128 * q + 4 * lane + t, e[t] & kParentMask);  // (local hole, global slot)
          if constexpr (kTrack) Q.st[pos] = 0;
          ++pos;
        }
      }
    }
    qlen += total;
    __syncwarp();
    if (qlen >= kRThresh) qlen = pass();
  }
  for (int drain = 0; qlen; ++drain) {
    if (!kTrack && drain > kBackBound) {
      overflow = true;  // the rare path resolves every chain
      break;
    }
    qlen = pass();
  }
  if (overflow) {
    atomicOr(&p.state->flags, kOverflow);
    status_or(p.status, PFR_ST_OVERFLOW);
  }
  if (kTrack && p.max_steps) {
    longest = __reduce_max_sync(0xffffffffu, longest);
    if (lane == 0 && longest) atomicMax(p.max_steps, longest);
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

// The rare-path kernel is launched after every delivery and exits at once
// unless a flag is set; it is cooperative (grid syncs), and a cooperative
// launch needs all its CTAs resident together -- with a full-machine grid it
// waits for concurrent work on other streams to drain (measured: 4x slower
// concurrent steps when it queued behind the persistent rejection kernels).
// A 16-CTA grid co-resides with anything; the rare work itself (repair,
// pointer jumping) is grid-strided and only slower on adversarial inputs.
// PFR_RARE_GRID overrides (A/B aid).
inline int rare_grid() {
  static const int g = [] {
    const char* v = getenv("PFR_RARE_GRID");
    return v ? std::max(1, atoi(v)) : 16;
  }();
  return g;
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
  // PFR_DV_PIPELINE=legacy (A/B aid): the CTA-tile pipeline K2 + K3
  static const bool legacy = [] {
    const char* v = getenv("PFR_DV_PIPELINE");
    return v && v[0] == 'l';
  }();
  if (p.expand && !p.Wser && !legacy) {
    const int smem = (int)(sizeof(WarpSmem) * kFWarps);
    const int smem3 = (int)(sizeof(ResolveQ) * kFWarps);
    static int occ2 = -1, occ3 = -1;
    if (occ2 < 0) {
      e = cudaFuncSetAttribute(k_dv_produce<T, A, UM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(k_dv_resolve<A, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(k_dv_resolve<A, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
      if (e != cudaSuccess) return e;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_dv_produce<T, A, UM>, kFWarps * 32, smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, k_dv_resolve<A, false, true>, kFWarps * 32, smem3);
      occ2 = max(occ2, 1);
      occ3 = max(occ3, 1);
    }
    const int64_t subs = (p.n + kSub - 1) / kSub;
    const int64_t g2 = max((int64_t)1, min((int64_t)num_sms() * occ2, (subs + kFWarps - 1) / kFWarps));
    const int64_t g3 = max((int64_t)1, min((int64_t)num_sms() * occ3, (subs + kFWarps - 1) / kFWarps));
    e = launch_pdl_smem(k_dv_produce<T, A, UM>, dim3((unsigned)g2), dim3(kFWarps * 32), (size_t)smem, s, false, p);
    if (e != cudaSuccess || stages < 3) return e;
    e = p.max_steps
            ? launch_pdl_smem(k_dv_resolve<A, false, true>, dim3((unsigned)g3), dim3(kFWarps * 32), (size_t)smem3, s,
                              false, p)
            : launch_pdl_smem(k_dv_resolve<A, false, false>, dim3((unsigned)g3), dim3(kFWarps * 32), (size_t)smem3,
                              s, false, p);
    if (e != cudaSuccess || stages < 4) return e;
    return launch_pdl(k_dv_rare<T, A, UM>, dim3(rare_grid()), dim3(kTileThreads), s, true, p);
  }
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
  return launch_pdl(k_dv_rare<T, A, UM>, dim3(rare_grid()), dim3(kTileThreads), s, true, p);
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
  p.sub = reinterpret_cast<A*>(ws.sub_cells);
  p.gn = n;
  p.gpt = nullptr;
  p.glast = 1;
  p.gfirst = 1;
  p.gbase = 0;
  p.wlo = 0;
  p.whi = n;
  return p;
}

}  // namespace

// ---------------------------------------------------------------------------
// Weight-sharded delivery, protocol v3 (sharded.py): the shard's local work
// through the single-GPU kernels.  K1 builds the shard's hierarchy; the
// shard's END value (W at its last element in the subtile association,
// SP(last) + sub(last)) is what the next shard's prefix adds, so the previous
// shard's last O and this shard's O(before) are computed from the same IEEE
// sum.  K2w writes the slot words of the shard's window into the extended
// array words[slot - wlo], K3w resolves the shard's indices from it.

template <typename A>
__global__ void k_shard_end(DvArgs<A> p, double* out) {
  const int64_t nS = (p.n + kSub - 1) / kSub;
  const int64_t s = nS - 1;
  const int64_t b = s >> 3;
  const int q = (int)(s & 7);
  const Hier<A> h = hier_of(p);
  if (threadIdx.x != 0) return;
  A Q = A(0);
  for (int i = 0; i < q; ++i) Q = add_rn(Q, __ldcg(p.sub + b * kSubPerTile + i));
  const A SP = add_rn(h.tile_excl(b), Q);
  *out = (double)add_rn(SP, __ldcg(p.sub + s));
}

namespace {
template <typename T>
cudaError_t shard_local_end_t(const void* w, int64_t n, uint32_t* status, double* end, const Workspace& ws,
                              cudaStream_t s) {
  auto p = make_args<T, double>(w, n, 0.0, nullptr, nullptr, nullptr, nullptr, nullptr, status, ws);
  k_dv_reduce<T, double, 1, false><<<(unsigned)p.tiles, kTileThreads, 0, s>>>(p);
  note_launch();
  k_shard_end<double><<<1, 32, 0, s>>>(p, end);
  note_launch();
  return cudaGetLastError();
}

template <typename T, int UM>
cudaError_t shard_produce_t(DvArgs<double> p, cudaStream_t s) {
  const int smem = (int)(sizeof(WarpSmem) * kFWarps);
  static int occ = -1;
  if (occ < 0) {
    cudaError_t e = cudaFuncSetAttribute(k_dv_produce<T, double, UM, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dv_produce<T, double, UM, true>, kFWarps * 32, smem);
    occ = max(occ, 1);
  }
  const int64_t subs = (p.n + kSub - 1) / kSub;
  const int64_t g = max((int64_t)1, min((int64_t)num_sms() * occ, (subs + kFWarps - 1) / kFWarps));
  k_dv_produce<T, double, UM, true><<<(unsigned)g, kFWarps * 32, smem, s>>>(p);
  note_launch();
  return cudaGetLastError();
}

template <typename T>
cudaError_t shard_resolve_t(DvArgs<double> p, cudaStream_t s) {
  const int smem = (int)(sizeof(ResolveQ) * kFWarps);
  static int occ = -1;
  if (occ < 0) {
    cudaError_t e = cudaFuncSetAttribute(k_dv_resolve<double, true, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dv_resolve<double, true, true>, kFWarps * 32, smem);
    occ = max(occ, 1);
  }
  const int64_t subs = (p.n + kSub - 1) / kSub;
  const int64_t g = max((int64_t)1, min((int64_t)num_sms() * occ, (subs + kFWarps - 1) / kFWarps));
  k_dv_resolve<double, true, true><<<(unsigned)g, kFWarps * 32, smem, s>>>(p);
  note_launch();
  return cudaGetLastError();
}

template <typename T>
DvArgs<double> shard_args(const void* w, int64_t n_loc, int64_t base, int64_t n_global, const double* pt, int first,
                          int last, double offset, const double* uniforms, const pfr_rng* rng, uint32_t* ext,
                          int64_t wlo, int64_t whi, int32_t* c, int32_t* max_steps, uint32_t* status,
                          const Workspace& ws) {
  auto p = make_args<T, double>(w, n_loc, offset, uniforms, rng, c, nullptr, max_steps, status, ws);
  p.gn = n_global;
  p.fx_S = fx_bits(n_global);
  p.gpt = pt;
  p.gfirst = first;
  p.glast = last;
  p.gbase = base;
  p.wlo = wlo;
  p.whi = whi;
  p.words = ext;
  return p;
}
}  // namespace

cudaError_t launch_shard_local_end(const void* w, int64_t n, int dtype, uint32_t* status, double* end,
                                   const Workspace& ws, cudaStream_t s) {
  if (dtype == PFR_F64) return shard_local_end_t<double>(w, n, status, end, ws, s);
  return shard_local_end_t<float>(w, n, status, end, ws, s);
}

cudaError_t launch_shard_produce(const void* w, int64_t n_loc, int dtype, int64_t base, int64_t n_global,
                                 const double* pt, int first, int last, int stratified, double offset,
                                 const double* uniforms, const pfr_rng* rng, uint32_t* ext, int64_t wlo, int64_t whi,
                                 uint32_t* status, const Workspace& ws, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(ext, 0xFF, (size_t)(whi - wlo) * sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const int mode = !stratified ? kUSys : uniforms ? kUArr : (rng && rng->mode == PFR_RNG_NUMPY) ? kUNp : kUPh;
  auto run = [&](auto tag) -> cudaError_t {
    using T = decltype(tag);
    auto p = shard_args<T>(w, n_loc, base, n_global, pt, first, last, offset, uniforms, rng, ext, wlo, whi, nullptr,
                           nullptr, status, ws);
    switch (mode) {
      case kUSys: return shard_produce_t<T, kUSys>(p, s);
      case kUArr: return shard_produce_t<T, kUArr>(p, s);
      case kUNp: return shard_produce_t<T, kUNp>(p, s);
      default: return shard_produce_t<T, kUPh>(p, s);
    }
  };
  return dtype == PFR_F64 ? run(double(0)) : run(float(0));
}

cudaError_t launch_shard_resolve_fast(int64_t n_loc, int dtype, int64_t base, const uint32_t* ext, int64_t wlo,
                                      int64_t whi, int32_t* c, int32_t* max_steps, uint32_t* status,
                                      const Workspace& ws, cudaStream_t s) {
  if (max_steps) {
    cudaError_t e = cudaMemsetAsync(max_steps, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
  }
  // the state flags must not carry a repair request into the resolve (K1 of
  // this shard cleared them; a shard needing repair already reported overflow)
  if (dtype == PFR_F64)
    return shard_resolve_t<double>(shard_args<double>(nullptr, n_loc, base, 0, nullptr, 0, 0, 0.0, nullptr, nullptr,
                                                      const_cast<uint32_t*>(ext), wlo, whi, c, max_steps, status,
                                                      ws),
                                   s);
  return shard_resolve_t<float>(shard_args<float>(nullptr, n_loc, base, 0, nullptr, 0, 0, 0.0, nullptr, nullptr,
                                                   const_cast<uint32_t*>(ext), wlo, whi, c, max_steps, status, ws),
                                s);
}

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
