// Sorted-ancestry expansion of one 4096-parent tile into slot words
// (shared by the fused delivery, its repair path and the batched delivery).
//
// A slot word is  parent | FIRST  (FIRST: the slot is its parent's first
// slot, i.e. the slot prepermute gives the parent, ancestry.py:125-136).
#pragma once

#include "pfr_internal.h"
#include "pfr_tile.cuh"

namespace pfr {

constexpr uint32_t kFirst = 0x80000000u;
constexpr uint32_t kParentMask = 0x7FFFFFFFu;

// word staging in shared memory: 16-byte slots XOR-swizzled (bank spread
// for the per-thread contiguous accesses, conflict-free striped read-out)
__device__ __forceinline__ int sw4(int pos) { return (swz(pos >> 2) << 2) | (pos & 3); }

constexpr int kSlotCap = 2 * kTile;        // staged slot positions per chunk (32 KB of words)
constexpr int kChunkSlots = kSlotCap - 4;  // slots per chunk (room for the 16-byte alignment shift)
constexpr int kSlotsPerThread = kSlotCap / kTileThreads;  // 32

// true when o decreases anywhere inside the tile or against the previous
// tile's last O (the caller then defers to the repair path)
static __device__ __forceinline__ bool tile_decreases(const int32_t (&o)[kTileItems], int32_t o_prev, int len,
                                               int32_t* warp_last) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e0 = threadIdx.x * kTileItems;
  (void)e0;
  (void)len;  // padding past N holds O = N: it never decreases
  bool bad = false;
#pragma unroll
  for (int j = 1; j < kTileItems; ++j) bad |= o[j] < o[j - 1];
  int prev = __shfl_up_sync(0xffffffffu, o[kTileItems - 1], 1);
  if (lane == 31) warp_last[warp] = o[kTileItems - 1];
  __syncthreads();
  if (lane == 0) prev = warp ? warp_last[warp - 1] : o_prev;
  bad |= o[0] < prev;
  return __syncthreads_or(bad);
}

// Expand the tile's parents over their slots: words (parent | FIRST) for the
// tile's slot range [O(base-1), O(base+len-1)), and the has-offspring bitmap.
// Per chunk of <= kChunkSlots slots: every parent whose first slot falls in
// the chunk writes its head word and sets a head bit (no loops over
// offspring counts, so no divergence however skewed the weights are); each
// thread then owns 32 consecutive slot positions and fills the non-head slots
// with the latest head's parent -- a block-wide exclusive max-scan of "last
// head in my range" carries parents across threads (parents increase with
// slot) and a running carry across chunks.  The chunk is written out with
// coalesced 16-byte stores (positions are shifted so that global vectors are
// aligned; partial edge vectors are written element-wise).
// `pidx_offset` is added to every parent index written (a batched filter
// writes global parent numbers so one in-place pass can serve the batch).
static __device__ void tile_expand(const int32_t (&o)[kTileItems], int32_t o_prev, int64_t b, int64_t n, uint32_t* words,
                            uint32_t* bitmap, uint32_t* sbuf /* kSlotCap words */, uint32_t* heads /* 256 */,
                            int32_t* warp_last /* 8 */, uint32_t pidx_offset = 0) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = b * kTile;
  const int len = (int)min((int64_t)kTile, n - base);
  const int e0 = tid * kTileItems;
  const uint32_t pbase = (uint32_t)base + (uint32_t)e0 + pidx_offset;
  // O of the element before this thread's first parent
  int prev = __shfl_up_sync(0xffffffffu, o[kTileItems - 1], 1);
  if (lane == 31) warp_last[warp] = o[kTileItems - 1];
  __syncthreads();
  if (lane == 0) prev = warp ? warp_last[warp - 1] : o_prev;
  uint32_t bits = 0;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) {
    const int pv = j ? o[j - 1] : prev;
    if (o[j] > pv) bits |= 1u << j;  // padding past N repeats O = N: never a parent
  }
  const uint32_t hi = __shfl_down_sync(0xffffffffu, bits, 1);
  if ((tid & 1) == 0 && e0 < len) bitmap[(base >> 5) + (tid >> 1)] = bits | (hi << 16);
  __shared__ int s_end;  // O of the tile's last element: N for the final tile
  if (tid == kTileThreads - 1) s_end = (len == kTile) ? o[kTileItems - 1] : (int)n;
  __syncthreads();
  const int end = s_end;
  int carry = -1;  // parent of the last slot of the previous chunk
  for (int c0 = o_prev; c0 < end; c0 += kChunkSlots) {
    const int cn = min(kChunkSlots, end - c0);
    // position = slot - c0 + sh keeps global vectors 16-byte aligned
    const int sh = (int)((reinterpret_cast<uintptr_t>(words + c0) >> 2) & 3);
    heads[tid] = 0u;
    __syncthreads();
    // heads: parents whose first slot lies in this chunk.  A thread's heads
    // are increasing and usually span one or two head words: their bits are
    // gathered in registers and published with <= 2 shared atomics.
    {
      int q = prev;
      const int wbase = max(prev - c0 + sh, 0) >> 5;
      uint32_t m0 = 0u, m1 = 0u;
#pragma unroll
      for (int j = 0; j < kTileItems; ++j) {
        if (bits & (1u << j)) {
          const int r = q - c0;
          if ((unsigned)r < (unsigned)cn) {
            const int pos = r + sh;
            sbuf[sw4(pos)] = (pbase + j) | kFirst;
            const int d = (pos >> 5) - wbase;
            const uint32_t bit = 1u << (pos & 31);
            if (d == 0)
              m0 |= bit;
            else if (d == 1)
              m1 |= bit;
            else
              atomicOr(&heads[pos >> 5], bit);
          }
        }
        if (e0 + j < len) q = o[j];
      }
      if (m0) atomicOr(&heads[wbase], m0);
      if (m1) atomicOr(&heads[wbase + 1], m1);
    }
    __syncthreads();
    // fill: thread owns positions [32 tid, 32 tid + 32)
    const int p0 = tid * kSlotsPerThread;
    const bool active = p0 < cn + sh;  // warp-uniform for all but one warp
    const uint32_t hb = active ? heads[tid] : 0u;
    int last_head = -1;
    if (hb) last_head = (int)(sbuf[sw4(p0 + 31 - __clz(hb))] & kParentMask);
    int blk_max;
    const int before = block_excl_max<int>(last_head, -1, warp_last, blk_max);
    if (active) {
      uint32_t cur = (uint32_t)max(carry, before);
      uint4* sv = reinterpret_cast<uint4*>(sbuf);
#pragma unroll
      for (int k = 0; k < kSlotsPerThread / 4; ++k) {
        uint4 v = sv[swz(p0 / 4 + k)];
        uint32_t e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (hb & (1u << (4 * k + t)))
            cur = e[t] & kParentMask;
          else
            e[t] = cur;
        }
        sv[swz(p0 / 4 + k)] = make_uint4(e[0], e[1], e[2], e[3]);
      }
    }
    carry = max(carry, blk_max);
    __syncthreads();
    // write out positions [sh, sh + cn) -> words[c0 - sh + pos]
    uint32_t* dst = words + (c0 - sh);
    const int nvec = (cn + sh + 3) >> 2;
    const uint4* sv = reinterpret_cast<const uint4*>(sbuf);
    for (int v = tid; v < nvec; v += kTileThreads) {
      const uint4 x = sv[swz(v)];
      const int p = 4 * v;
      if (p >= sh && p + 4 <= sh + cn) {
        reinterpret_cast<uint4*>(dst)[v] = x;
      } else {
        const uint32_t e[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (p + t >= sh && p + t < sh + cn) dst[p + t] = e[t];
      }
    }
    __syncthreads();
  }
}

}  // namespace pfr
