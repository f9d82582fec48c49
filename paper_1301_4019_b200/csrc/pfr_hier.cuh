// Hierarchical tile prefixes without a single-CTA tail.
//
// Pass 1 of every two-pass scan (the weight scan of the fused delivery and
// pfr_scan) runs one CTA per 4096-element tile and writes the tile
// aggregate.  The last tile to finish in each group of 64 tiles scans the
// group's aggregates with one warp; the last group to finish scans the group
// totals.  Every floating-point association is fixed by tile and group
// indices alone (deterministic and schedule independent).  Counters live in
// the workspace's DvState, are zero at workspace creation and are reset by
// whoever consumes them.
//
// Layout of `excl` (A elements):
//   [0, tiles)              exclusive prefix of the tile inside its group
//   [tiles]                 the total
//   [tiles+1, tiles+2+G)    exclusive prefix of the group totals
// followed by the per-tile validation flags (uint32).  `gsum` holds the G
// group totals.
#pragma once

#include "pfr_internal.h"
#include "pfr_tile.cuh"

namespace pfr {

constexpr int kGroupTiles = 64;

template <typename A>
struct Hier {
  A* agg;        // [tiles]
  A* excl;       // see above
  A* gsum;       // [groups]
  DvState* state;
  int64_t tiles;

  __device__ __forceinline__ int64_t groups() const { return (tiles + kGroupTiles - 1) / kGroupTiles; }
  __device__ __forceinline__ A* group_prefix() const { return excl + tiles + 1; }
  __device__ __forceinline__ uint32_t* tile_flags() const {
    return reinterpret_cast<uint32_t*>(excl + tiles + 2 + groups());
  }
  __device__ __forceinline__ A total() const { return __ldcg(excl + tiles); }
  // exclusive prefix of tile b (the association every consumer uses)
  __device__ __forceinline__ A tile_excl(int64_t b) const {
    return add_rn(__ldcg(group_prefix() + b / kGroupTiles), __ldcg(excl + b));
  }
  // inclusive value at the last element of tile b
  __device__ __forceinline__ A tile_end(int64_t b) const { return add_rn(tile_excl(b), __ldcg(agg + b)); }
};

// exclusive scan of v[0..cnt) (cnt <= 64) by one warp: lane l holds v[2l],
// v[2l+1]; pair sums, Kogge-Stone across lanes.  Writes out[k]; returns the
// total in every lane.
template <typename A>
__device__ __forceinline__ A warp_excl64(const A* v, int cnt, A* out) {
  const int lane = threadIdx.x & 31;
  const A a0 = 2 * lane < cnt ? __ldcg(v + 2 * lane) : A(0);
  const A a1 = 2 * lane + 1 < cnt ? __ldcg(v + 2 * lane + 1) : A(0);
  const A pr = add_rn(a0, a1);
  const A incl = warp_inclusive_scan(pr);
  A ex = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) ex = A(0);
  if (2 * lane < cnt) out[2 * lane] = ex;
  if (2 * lane + 1 < cnt) out[2 * lane + 1] = add_rn(ex, a0);
  return __shfl_sync(0xffffffffu, incl, 31);
}

// Called by every thread of the CTA owning tile b after agg[b] is written and
// the CTA's validation bits are in *cta_flags (shared).  The CTA completing
// the last group publishes the group prefixes, the total and the OR of all
// tile flags into *status, and resets the counters.
template <typename A>
__device__ __forceinline__ void hier_tile_done(const Hier<A>& h, int64_t b, uint32_t* cta_flags, int* stage,
                                               uint32_t* status) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  const int64_t g = b / kGroupTiles;
  const int64_t G = h.groups();
  if (threadIdx.x == blockDim.x - 1) {
    h.tile_flags()[b] = *cta_flags;
    __threadfence();
    const int64_t gsize = min((int64_t)kGroupTiles, h.tiles - g * kGroupTiles);
    const unsigned t = atomicAdd(&h.state->gcnt[g], 1u);
    *stage = (t == (unsigned)gsize - 1) ? 1 : 0;
  }
  __syncthreads();
  if (!*stage) return;  // block-uniform
  __syncthreads();      // every thread has read *stage before warp 0 rewrites it below
  // last tile of group g: scan the group's aggregates
  if (warp == 0) {
    __threadfence();
    const int64_t t0 = g * kGroupTiles;
    const int cnt = (int)min((int64_t)kGroupTiles, h.tiles - t0);
    const A gt = warp_excl64(h.agg + t0, cnt, h.excl + t0);
    if (lane == 0) {
      h.gsum[g] = gt;
      h.state->gcnt[g] = 0;
      __threadfence();
      const unsigned t = atomicAdd(&h.state->done, 1u);
      *stage = (t == (unsigned)G - 1) ? 2 : 0;
    }
  }
  __syncthreads();
  if (*stage != 2) return;
  // last group: exclusive scan of the group totals (64 per warp pass, serial
  // carry across passes), the total, the validation flags
  __threadfence();
  if (warp == 0) {
    A carry = A(0);
    for (int64_t g0 = 0; g0 < G; g0 += 64) {
      const int cnt = (int)min((int64_t)64, G - g0);
      A* out = h.group_prefix() + g0;
      const A tot = warp_excl64(h.gsum + g0, cnt, out);
      __syncwarp();
      if (g0) {  // shift by the carry of the previous passes
        if (2 * lane < cnt) out[2 * lane] = add_rn(carry, out[2 * lane]);
        if (2 * lane + 1 < cnt) out[2 * lane + 1] = add_rn(carry, out[2 * lane + 1]);
      }
      carry = g0 ? add_rn(carry, tot) : tot;
      __syncwarp();
    }
    if (lane == 0) h.excl[h.tiles] = carry;  // the total
  }
  uint32_t fl = 0;
  for (int64_t i = threadIdx.x; i < h.tiles; i += blockDim.x) fl |= __ldcg(h.tile_flags() + i);
  fl = __reduce_or_sync(0xffffffffu, fl);
  if (lane == 0 && fl) atomicOr(cta_flags, fl);
  __syncthreads();
  if (threadIdx.x == 0) {
    h.state->done = 0;
    status_or(status, *cta_flags);
  }
}

}  // namespace pfr
