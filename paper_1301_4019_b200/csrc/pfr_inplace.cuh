// Backward chain walks of the in-place ancestry (K3 of the fused delivery and
// the batched filter's fused step): per-warp chain queues in shared memory.
#pragma once

#include "pfr_expand.cuh"

namespace pfr {

constexpr int kBackBound = 255;  // chain steps walked before the fallback (fits the queue's uint8)

constexpr int kIpThreads = 256;
constexpr int kIpWarps = kIpThreads / 32;
constexpr int kQ = 512;          // queue entries per warp
constexpr int kStepPer = 4;      // chain loads per lane per step batch
constexpr int kGroup = 32;

// optional segment list for K3: only the listed segments of `groups` 32-index
// groups each (the batched filter's resampled filters)
struct IpSegments {
  const uint32_t* list;   // segment numbers (null: the whole index range)
  const uint32_t* count;  // number of listed segments (device)
  uint32_t groups;        // groups per segment
};

struct IpQueue {
  uint32_t x[kIpWarps][kQ];
  uint32_t z[kIpWarps][kQ];
  uint8_t st[kIpWarps][kQ];
};

// one step for every queued chain; survivors compacted to the front
static __device__ __forceinline__ int step_pass(IpQueue& Q, int warp, int lane, int qlen,
                                                const uint32_t* __restrict__ words, int32_t* __restrict__ c,
                                                int& longest, bool& overflow) {
  int out = 0;
  for (int b = 0; b < qlen; b += 32 * kStepPer) {
    uint32_t x[kStepPer], z[kStepPer], w[kStepPer];
    int st[kStepPer];
    bool valid[kStepPer];
#pragma unroll
    for (int i = 0; i < kStepPer; ++i) {
      const int e = b + 32 * i + lane;
      valid[i] = e < qlen;
      if (valid[i]) {
        x[i] = Q.x[warp][e];
        z[i] = Q.z[warp][e];
        st[i] = Q.st[warp][e] + 1;
        w[i] = __ldcg(words + z[i]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < kStepPer; ++i) {
      if (b + 32 * i >= qlen) break;  // warp-uniform
      bool keep = false;
      if (valid[i]) {
        if (!(w[i] & kFirst)) {
          c[x[i]] = (int32_t)(w[i] & kParentMask);
          longest = max(longest, st[i]);
        } else if (st[i] >= kBackBound) {
          overflow = true;  // abandoned: the rare-path kernel resolves every chain
        } else {
          keep = true;
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int pos = out + __popc(m & ((1u << lane) - 1));
        Q.x[warp][pos] = x[i];
        Q.z[warp][pos] = w[i] & kParentMask;
        Q.st[warp][pos] = (uint8_t)st[i];
      }
      out += __popc(m);
    }
    __syncwarp();
  }
  return out;
}

// classify one 32-index group: trivial indices store c, first-slot holes queue
static __device__ __forceinline__ void scan_group(IpQueue& Q, int warp, int lane, uint32_t x, bool in, uint32_t wd,
                                           uint32_t bw, int& qlen, int32_t* __restrict__ c) {
  const bool has = (bw >> lane) & 1u;
  const bool pend = in && !has && (wd & kFirst);
  if (in && !pend) __stcs(c + x, has ? (int32_t)x : (int32_t)(wd & kParentMask));
  const unsigned m = __ballot_sync(0xffffffffu, pend);
  if (pend) {
    const int pos = qlen + __popc(m & ((1u << lane) - 1));
    Q.x[warp][pos] = x;
    Q.z[warp][pos] = wd & kParentMask;
    Q.st[warp][pos] = 0;
  }
  qlen += __popc(m);
}

}  // namespace pfr
