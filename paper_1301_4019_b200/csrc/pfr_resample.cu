// Metropolis, rejection and multinomial resamplers, lower_bound.
//
// Reference: resamplers.py:56-102 (multinomial, serial/sorted variant),
// 204-234 (Metropolis), 237-310 (rejection, capped), primitives.py:91-106
// (lower_bound).
//
// Metropolis and rejection need no collective over the weights: each output
// slot runs its own chain / proposal loop reading w through the read-only
// path (ld.global.nc).  Random draws come from a counter-based generator so
// they are a pure function of (stream, slot, step): no state in memory.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "pfr_internal.h"
#include "pfr_tile.cuh"

namespace pfr {

namespace {

constexpr int kChainsPerThread = 4;

template <typename T>
__device__ __forceinline__ T ldg(const T* p) {
  return __ldg(p);
}

template <typename T>
__device__ __forceinline__ T div_rn_t(T a, T b);
template <>
__device__ __forceinline__ float div_rn_t(float a, float b) {
  return __fdiv_rn(a, b);
}
template <>
__device__ __forceinline__ double div_rn_t(double a, double b) {
  return __ddiv_rn(a, b);
}

// reference acceptance (resamplers.py:228-232): ratio rounded in the weight
// dtype, compared against the float64 uniform; a zero current weight accepts
template <typename T>
__device__ __forceinline__ bool accept_ref(double u, T wk, T wj) {
  if (wk == T(0)) return true;
  const T ratio = div_rn_t(wj, wk);
  return u <= (double)ratio;
}

// ---------------------------------------------------------------------------
// Metropolis, own Philox4x32-10 stream: chain i, step b uses counter
// (i, b/2, tag, 0): words (2*(b&1), 2*(b&1)+1) = (proposal, uniform).
template <typename T>
__global__ void __launch_bounds__(256) k_metropolis_philox(const T* __restrict__ w, int64_t n, int64_t steps,
                                                           uint32_t k0, uint32_t k1, uint32_t threshold,
                                                           int64_t c_begin, int64_t c_count,
                                                           int32_t* __restrict__ a, uint32_t* status,
                                                           int32_t* __restrict__ claim) {
  // chains [c_begin, c_begin + c_count) of the N-chain resampler (a sharded
  // rank runs its slice with global chain numbers: same draws, same result)
  __shared__ uint32_t blk_flags;
  const int64_t local = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * kChainsPerThread;
  const int64_t first = c_begin + local;
  int64_t k[kChainsPerThread];
  T wk[kChainsPerThread];
#pragma unroll
  for (int c = 0; c < kChainsPerThread; ++c) {
    const int64_t i = min(first + c, c_begin + c_count - 1);
    k[c] = i;
    wk[c] = ldg(w + i);
  }
  if (status) {  // launch-uniform
    // check_weights (diagnostics.py:38-51) on the chains' own weights: every
    // w[i] of the launch's slice is read once here, so no separate pass.
    // One global atomic per block, and only for bits not yet set.
    if (threadIdx.x == 0) blk_flags = 0;
    __syncthreads();
    FlagAcc<T> facc;
#pragma unroll
    for (int c = 0; c < kChainsPerThread; ++c)
      if (local + c < c_count) facc.add(wk[c]);
    const uint32_t f = __reduce_or_sync(0xffffffffu, facc.flags());
    if ((threadIdx.x & 31) == 0 && f) atomicOr(&blk_flags, f);
    __syncthreads();
    if (threadIdx.x == 0 && blk_flags && (*(volatile uint32_t*)status & blk_flags) != blk_flags)
      atomicOr(status, blk_flags);
  }
  if (local >= c_count) return;
  const uint32_t nn = (uint32_t)n;
  for (int64_t b = 0; b < steps; b += 2) {
    uint32_t j[kChainsPerThread][2];
    T u[kChainsPerThread][2];
    T wj[kChainsPerThread][2];
#pragma unroll
    for (int c = 0; c < kChainsPerThread; ++c) {
      const uint32_t i = (uint32_t)(first + c);
      uint32_t o[4];
      philox4x32_10(i, (uint32_t)(b >> 1), kTagMetropolis, 0, k0, k1, o);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        j[c][h] = threshold == 0 ? __umulhi(o[2 * h], nn)  // power-of-two N: Lemire never rejects
                                 : bounded_u32(o[2 * h], nn, threshold, i, (uint32_t)(b + h), kTagMetropolis, k0, k1);
        if constexpr (sizeof(T) == 4)
          u[c][h] = u32_to_unit_f_open(o[2 * h + 1]);
        else
          u[c][h] = u32_to_unit_d_open(o[2 * h + 1]);
      }
    }
    // issue every gather of this step pair before consuming any (MLP)
#pragma unroll
    for (int c = 0; c < kChainsPerThread; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h) wj[c][h] = ldg(w + j[c][h]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (b + h >= steps) break;
#pragma unroll
      for (int c = 0; c < kChainsPerThread; ++c) {
        // u <= w[j]/w[k]  <=>  u * w[k] <= w[j]  (w[k] > 0); w[k] == 0 accepts
        const bool acc = (wk[c] == T(0)) || (u[c][h] * wk[c] <= wj[c][h]);
        if (acc) {
          k[c] = j[c][h];
          wk[c] = wj[c][h];
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kChainsPerThread; ++c)
    if (local + c < c_count) {
      a[local + c] = (int32_t)k[c];
      // fused delivery: the permute's claim (prepermute, ancestry.py:125-136)
      if (claim) atomicMin(claim + k[c], (int32_t)(c_begin + local + c));
    }
}

// Metropolis replaying numpy's stream (power-of-two N): per step the
// generator yields N doubles then N integers (one u32 each, low half first).
template <typename T>
__global__ void __launch_bounds__(256) k_metropolis_numpy(const T* __restrict__ w, int64_t n, int64_t steps,
                                                          Key2x64 key, int log2n, int64_t c_begin, int64_t c_count,
                                                          int32_t* __restrict__ a) {
  const int64_t local = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * kChainsPerThread;
  if (local >= c_count) return;
  const int64_t first = c_begin + local;
  int64_t k[kChainsPerThread];
  T wk[kChainsPerThread];
#pragma unroll
  for (int c = 0; c < kChainsPerThread; ++c) {
    const int64_t i = min(first + c, c_begin + c_count - 1);
    k[c] = i;
    wk[c] = ldg(w + i);
  }
  const uint64_t per_step = (uint64_t)n + (uint64_t)n / 2;  // u64 words per step
  for (int64_t b = 0; b < steps; ++b) {
    const uint64_t ubase = (uint64_t)b * per_step;
    const uint64_t jbase = ubase + (uint64_t)n;
    double u[kChainsPerThread];
    int64_t j[kChainsPerThread];
#pragma unroll
    for (int c = 0; c < kChainsPerThread; ++c) {
      const uint64_t i = (uint64_t)(first + c);
      u[c] = u64_to_unit(numpy_raw64(key, ubase + i));
      const uint64_t word = numpy_raw64(key, jbase + i / 2);
      const uint32_t x = (i & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
      j[c] = (int64_t)(((uint64_t)x << log2n) >> 32);
    }
    T wj[kChainsPerThread];
#pragma unroll
    for (int c = 0; c < kChainsPerThread; ++c) wj[c] = ldg(w + j[c]);
#pragma unroll
    for (int c = 0; c < kChainsPerThread; ++c) {
      if (accept_ref<T>(u[c], wk[c], wj[c])) {
        k[c] = j[c];
        wk[c] = wj[c];
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kChainsPerThread; ++c)
    if (local + c < c_count) a[local + c] = (int32_t)k[c];
}

// Metropolis from caller-supplied draws u[b*N + i] (float64), j[b*N + i]
template <typename T, typename I>
__global__ void __launch_bounds__(256) k_metropolis_arrays(const T* __restrict__ w, int64_t n, int64_t steps,
                                                           const double* __restrict__ ud, const I* __restrict__ jd,
                                                           int32_t* __restrict__ a, uint32_t* status) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t k = i;
  T wk = ldg(w + i);
  uint32_t f = 0;
  for (int64_t b = 0; b < steps; ++b) {
    const int64_t j = (int64_t)jd[b * n + i];
    if (j < 0 || j >= n) {
      f |= PFR_ST_RANGE;
      continue;
    }
    const T wj = ldg(w + j);
    if (accept_ref<T>(ud[b * n + i], wk, wj)) {
      k = j;
      wk = wj;
    }
  }
  status_or(status, f);
  a[i] = (int32_t)k;
}

// ---------------------------------------------------------------------------
// Rejection, own stream, warp-cooperative slot queue.  Slot i, trip t uses
// counter (i, t/2, tag, 0), words (2*(t&1), 2*(t&1)+1) = (proposal, uniform);
// trip 0 proposes i itself (resamplers.py:291-294).  Warps grab chunks of 256
// slots with one atomic and refill idle lanes from the chunk via ballot/popc,
// so lanes stay busy although trip counts vary by orders of magnitude.
template <typename T>
struct RejArgs {
  const T* w;
  int64_t n;
  double bound;
  double cap;  // > 0: capped variant, v = min(w, cap), bound = cap
  uint32_t k0, k1, threshold;
  uint32_t max_trips;
  int64_t s0;     // first slot of this launch (global number: RNG counters, trip 0)
  int64_t count;  // slots of this launch; outputs are indexed slot - s0
  int32_t* a;
  int32_t* trips;
  T* out_w;
  unsigned long long* next_chunk;
  uint32_t* status;
  int32_t* claim;  // fused delivery: the permute's claims (atomicMin of the slot at its ancestor)
};

constexpr int kRejChunk = 256;

// Each lane evaluates kRejBatch (default 8) consecutive trips of its slot per iteration:
// the trips' proposals do not depend on earlier outcomes, so their Philox
// words and weight gathers are all issued before the first comparison (4
// gathers in flight per lane instead of one dependent L2 round trip per trip).
// The first accepting trip of the batch wins, so results, trip counts and the
// stream mapping are exactly those of a one-trip-at-a-time loop; the few
// trips evaluated past the acceptance are discarded.
// draws of trips trip .. trip+B-1 of `slot` (trip even): Philox counters
// (slot, trip/2 + q), words (2h, 2h+1) = (proposal, uniform); trip 0
// proposes the slot itself (resamplers.py:291-294)
template <typename T, int B>
struct RejBatch {
  uint32_t j[B];
  uint32_t x[B];  // raw uniform words: u = unit(x) (rej_u), and u > 2^-(k+1) iff x >= 2^(31-k)
};

// the acceptance uniform of a raw word (open interval, cell midpoints)
template <typename T>
__device__ __forceinline__ T rej_u(uint32_t x) {
  if constexpr (sizeof(T) == 4)
    return u32_to_unit_f_open(x);
  else
    return u32_to_unit_d_open(x);
}

template <typename T, int B>
__device__ __forceinline__ void rej_draws(const RejArgs<T>& A, uint32_t slot, uint32_t trip, RejBatch<T, B>& d) {
  const uint32_t nn = (uint32_t)A.n;
#pragma unroll
  for (int q = 0; q < B / 2; ++q) {
    uint32_t o[4];
    philox4x32_10(slot, (trip >> 1) + q, kTagRejection, 0, A.k0, A.k1, o);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      // power-of-two N (threshold 0): Lemire never rejects
      d.j[2 * q + h] = A.threshold == 0 ? __umulhi(o[2 * h], nn)
                                        : bounded_u32(o[2 * h], nn, A.threshold, slot, trip + 2 * q + h,
                                                      kTagRejection, A.k0, A.k1);
      d.x[2 * q + h] = o[2 * h + 1];
    }
  }
  if (trip == 0) d.j[0] = slot;
}

// Certain-reject table.  A trip (j, beta) is rejected when beta * bound >
// v[j]; when v[j] < thr and beta > 2^-(k+1) that is certain without reading
// v[j] (thr = (T)(bound 2^-(k+1)) = (T)bound 2^-(k+1) exactly, so the exact
// product beta * bound exceeds thr and its rounding is >= thr > v[j]; beta >
// 2^-(k+1) is one integer compare on the raw Philox word).  k_rej_table
// writes, for eight thresholds thr_k, one bit per group of g = 2^lg
// consecutive weights (set when the group's largest capped weight is >=
// thr_k) and counts the set bits; the
// rejection kernel picks the k minimising the expected share of trips that
// still need the gather, 2^-(k+1) + set_k / groups, and holds that bitmap
// (<= 2^20 bits, 128 KiB) in shared memory.  The table only skips loads whose
// outcome is already decided, so acceptances, trip counts and the stream
// mapping are exactly those of the plain kernel.
//
// Why: the plain kernel is bound by the L1TEX sector rate of its random
// gathers (ncu: l1tex throughput 91% of peak; one sector per trip), not by
// HBM or L2.  With the table (log-normal sigma = 1, sup = max w: k = 3, ~8%
// of trips gather) L1 drops to ~20% and the kernel becomes issue-bound on
// Philox: 413 -> 349 us at N = 2^20 (float32).
constexpr int kRejTabK = 8;                  // thresholds 2^-1 .. 2^-8 of the bound
constexpr int64_t kRejTabMaxBits = 1 << 20;  // 128 KiB of shared memory
constexpr int kRejTabThreads = 1024;  // one CTA per SM (128 KiB table)

struct RejTab {
  uint32_t* counts;  // [kRejTabK] set groups per threshold
  uint32_t* bits;    // [kRejTabK][words]
  int64_t groups;    // ceil(N / g)
  int64_t words;     // ceil(groups / 32)
  int lg;            // log2 g
};

// v = *p when c (a predicated non-coherent load: no branch around it)
__device__ __forceinline__ void ldg_if(const float* p, bool c, float& v) {
  asm("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q ld.global.nc.f32 %0, [%1];\n}"
      : "+f"(v)
      : "l"(p), "r"((unsigned)c));
}
__device__ __forceinline__ void ldg_if(const double* p, bool c, double& v) {
  asm("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q ld.global.nc.f64 %0, [%1];\n}"
      : "+d"(v)
      : "l"(p), "r"((unsigned)c));
}

template <typename T>
__device__ __forceinline__ T rej_thr(double bound, int k) {
  // in T, like the kernel's product u * (T)bound: rounding is monotone, so
  // u > 2^-(k+1) gives fl(u * (T)bound) >= fl((T)bound * 2^-(k+1)) = thr
  return (T)bound * (T)ldexp(1.0, -(k + 1));
}

// (also check_weights' flags, diagnostics.py:38-51: the table reads every
// weight once, so the rejection needs no separate validation pass)
template <typename T, bool kCapped>
__global__ void __launch_bounds__(256) k_rej_table(const T* __restrict__ w, int64_t n, double bound, double cap,
                                                   RejTab tb, uint32_t* status) {
  constexpr int kW = 4;  // words per warp and pass: four independent loads in flight per lane
  const int lane = threadIdx.x & 31;
  const T capv = (T)cap;
  T thr[kRejTabK];
#pragma unroll
  for (int k = 0; k < kRejTabK; ++k) thr[k] = rej_thr<T>(cap > 0 ? cap : bound, k);
  const int64_t g = (int64_t)1 << tb.lg;
  uint32_t cnt = 0;  // lane k < kRejTabK: set bits of threshold k
  FlagAcc<T> facc;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w0 = (blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5)) * kW; w0 < tb.words;
       w0 += warps * kW) {
    // group maximum of the capped weights; NaN never exceeds a threshold and
    // is skipped (the plain kernel never accepts a NaN proposal either)
    T vmax[kW];
    if (tb.lg == 0) {  // one weight per bit: the four loads first
#pragma unroll
      for (int q = 0; q < kW; ++q) {
        const int64_t e = (w0 + q) * 32 + lane;
        vmax[q] = e < n ? ldg(w + e) : T(0);
        if (e < n) facc.add(vmax[q]);
      }
#pragma unroll
      for (int q = 0; q < kW; ++q) {
        const T v = kCapped ? (vmax[q] < capv ? vmax[q] : capv) : vmax[q];
        vmax[q] = v > T(0) ? v : T(0);  // NaN -> 0
      }
    } else
#pragma unroll
    for (int q = 0; q < kW; ++q) {
      vmax[q] = T(0);
      const int64_t grp = (w0 + q) * 32 + lane;
      if (grp < tb.groups) {
        const int64_t e0 = grp * g, e1 = min(e0 + g, n);
        for (int64_t e = e0; e < e1; ++e) {
          const T wj = ldg(w + e);
          facc.add(wj);
          const T v = kCapped ? (wj < capv ? wj : capv) : wj;
          if (v > vmax[q]) vmax[q] = v;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kW; ++q) {
      uint32_t mine = 0;
#pragma unroll
      for (int k = 0; k < kRejTabK; ++k) {
        const uint32_t bk = __ballot_sync(0xffffffffu, vmax[q] >= thr[k]);
        if (lane == k) mine = bk;
      }
      if (lane < kRejTabK && w0 + q < tb.words) {
        tb.bits[(int64_t)lane * tb.words + w0 + q] = mine;
        cnt += __popc(mine);
      }
    }
  }
  if (lane < kRejTabK && cnt) atomicAdd(tb.counts + lane, cnt);
  status_or_warp(status, facc.flags());
}

// Steady state: every lane owns a slot; the gathers of batch k are issued,
// then the draws of batch k+1 are computed while they are in flight, then
// batch k is resolved (two batch buffers used in turn: no copies).  A lane
// whose slot finishes discards its precomputed batch and takes the next slot
// of the warp's chunk (one atomic per 256 slots); the new slot's first batch
// is drawn in the same (non-divergent) draw call as everyone's next batch.
//
// Tail: once the chunks are exhausted, lanes without a slot HELP the slots
// still running instead of idling -- trip t of a slot depends only on (slot,
// t), so helper h of a slot evaluates trips t + hB .. t + hB + B - 1 in the
// same pass and the first accepting trip over the owner and its helpers wins
// (a shared-memory atomicMin on (trip, proposal)).  Results, trip counts and
// the stream mapping are exactly those of a one-trip-at-a-time loop; the
// geometric tail (a warp's last slot runs ~4x the mean trips) no longer
// leaves 31 lanes idle.
template <typename T, bool kCapped, int kRejBatch, bool kTab = false>
__global__ void __launch_bounds__(kTab ? kRejTabThreads : 256, 1) k_rejection_philox(RejArgs<T> A, RejTab tb) {
  constexpr int B = kRejBatch;
  __shared__ unsigned long long s_best[kTab ? kRejTabThreads / 32 : 8][32];  // per warp, per owner lane
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const T bound = (T)A.bound;
  const T capv = (T)A.cap;
  int64_t chunk_next = 0, chunk_end = 0;  // warp-uniform local queue
  bool exhausted = false;                 // warp-uniform: no chunks left
  int64_t slot = -1;
  uint32_t trip = 0;
  uint32_t flags = 0;
  int iter = 0;
  bool fresh = false;  // the slot was just taken: no batch drawn yet
  // certain-reject table (kTab): trip q needs its gather only when beta *
  // bound <= thr or the proposal's group holds a capped weight above thr
  extern __shared__ uint32_t rej_tab[];
  uint32_t ulim = 0xFFFFFFFFu;  // 2^(31-k) - 1 with a table; no table: every trip gathers
  if constexpr (kTab) {
    __shared__ int s_k;
    if (threadIdx.x == 0) {
      int best = -1;
      double bc = 0.75;  // use a table only when it saves at least a quarter of the gathers
      for (int k = 0; k < kRejTabK; ++k) {
        const double c = ldexp(1.0, -(k + 1)) + (double)tb.counts[k] / (double)tb.groups;
        if (c < bc) {
          bc = c;
          best = k;
        }
      }
      s_k = best;
    }
    __syncthreads();
    const int k = s_k;
    if (k >= 0) {
      const uint4* src = reinterpret_cast<const uint4*>(tb.bits + (int64_t)k * tb.words);
      uint4* dst = reinterpret_cast<uint4*>(rej_tab);
      for (int64_t i = threadIdx.x; i < tb.words / 4; i += blockDim.x) dst[i] = __ldcg(src + i);
      ulim = (1u << (31 - k)) - 1u;
    }
    __syncthreads();
  }
  // gathers of one batch; need[q] false: the trip is a certain reject
  // (branch-free: the bit is read unconditionally -- with no table `big` is
  // 0 and the bit is ignored -- and the gather is a predicated load)
  auto gather = [&](const RejBatch<T, B>& d, T (&wj)[B], bool (&need)[B]) {
#pragma unroll
    for (int q = 0; q < B; ++q) {
      bool nd = true;
      if constexpr (kTab) {
        const uint32_t gq = d.j[q] >> tb.lg;
        const uint32_t bit = rej_tab[gq >> 5] >> (gq & 31);
        // u = (2m+1) 2^-24 (f32, m = x >> 9) or (2x+1) 2^-33 (f64) exceeds
        // 2^-(k+1) exactly when x > 2^(31-k) - 1 (ulim; all ones: no table)
        nd = (d.x[q] <= ulim) | (bit & 1u);
      }
      need[q] = nd;
      wj[q] = T(0);
      ldg_if(A.w + d.j[q], nd, wj[q]);
    }
  };
  RejBatch<T, B> buf0, buf1;

  auto finish = [&](uint32_t jd, T wd, uint32_t ntrips) {
    A.a[slot] = (int32_t)jd;
    if (A.claim) atomicMin(A.claim + jd, (int32_t)(A.s0 + slot));
    if (A.trips) A.trips[slot] = (int32_t)ntrips;
    if (kCapped) {
      const T vd = wd < capv ? wd : capv;
      A.out_w[slot] = (vd == T(0)) ? T(1) : div_rn_t(wd, vd);
    }
    slot = -1;
  };
  auto no_progress = [&]() {
    flags |= PFR_ST_NOPROGRESS;
    A.a[slot] = (int32_t)(A.s0 + slot);
    if (A.claim) atomicMin(A.claim + A.s0 + slot, (int32_t)(A.s0 + slot));
    if (A.trips) A.trips[slot] = (int32_t)A.max_trips;
    if (kCapped) A.out_w[slot] = T(1);
    slot = -1;
  };
  // give up early once any slot reported no progress (reference raises)
  auto give_up = [&]() {
    if (((++iter) & 63) == 0) {
      if (__ballot_sync(0xffffffffu, flags != 0) || (*(volatile uint32_t*)A.status & PFR_ST_NOPROGRESS)) {
        flags |= PFR_ST_NOPROGRESS;
        return true;
      }
    }
    return false;
  };
  // 0: continue, 1: warp done, 2: chunks exhausted with idle lanes (tail)
  auto step = [&](RejBatch<T, B>& cur, RejBatch<T, B>& nxt) -> int {
    unsigned idle = __ballot_sync(0xffffffffu, slot < 0);
    while (idle) {
      if (chunk_next >= chunk_end) {
        if (exhausted) break;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(A.next_chunk, (unsigned long long)kRejChunk);
        base = __shfl_sync(0xffffffffu, base, 0);
        if ((int64_t)base >= A.count) {
          exhausted = true;
          break;
        }
        chunk_next = (int64_t)base;
        chunk_end = min((int64_t)base + kRejChunk, A.count);
      }
      const int rank = __popc(idle & lt_mask);
      const int take = min((int64_t)__popc(idle), chunk_end - chunk_next);
      if (slot < 0 && rank < take) {
        slot = chunk_next + rank;
        trip = 0;
        fresh = true;  // its first batch is drawn below, with everyone's next batch
      }
      chunk_next += take;
      idle = __ballot_sync(0xffffffffu, slot < 0);
    }
    if (idle) return __ballot_sync(0xffffffffu, slot >= 0) ? 2 : 1;
    T wj[B];
    bool need[B];
    if constexpr (kTab) {
      // not pipelined: few trips need a gather, and the table kernel's
      // occupancy (32 warps per SM) hides the rest
      (void)nxt;
      rej_draws<T, B>(A, (uint32_t)(A.s0 + slot), trip, cur);
      fresh = false;
      gather(cur, wj, need);
    } else {
      if (!fresh) gather(cur, wj, need);
      // one non-divergent draw per step: the next batch, or a fresh slot's first
      rej_draws<T, B>(A, (uint32_t)(A.s0 + slot), fresh ? 0u : trip + B, nxt);
      if (fresh) {
        fresh = false;
        return give_up() ? 1 : 0;
      }
    }
    int done = -1;  // batch position of the first accepting trip
    uint32_t jd = 0;
    T wd = T(0);
#pragma unroll
    for (int q = B - 1; q >= 0; --q) {
      const T vj = kCapped ? (wj[q] < capv ? wj[q] : capv) : wj[q];
      // beta <= v[j] / bound  <=>  beta * bound <= v[j]
      if (need[q] && rej_u<T>(cur.x[q]) * bound <= vj) {
        done = q;
        jd = cur.j[q];
        wd = wj[q];
      }
    }
    // round cap: the trips past max_trips do not exist
    if (trip + (uint32_t)B >= A.max_trips && (done < 0 || trip + (uint32_t)done + 1 > A.max_trips))
      no_progress();
    else if (done >= 0)
      finish(jd, wd, trip + done + 1);
    else
      trip += B;
    return give_up() ? 1 : 0;
  };
  int st;
  while (true) {
    if ((st = step(buf0, buf1)) != 0) break;
    if ((st = step(buf1, buf0)) != 0) break;
  }
  if (st == 2) {
    // tail: owners and helpers
    while (true) {
      const unsigned act = __ballot_sync(0xffffffffu, slot >= 0);
      if (!act) break;
      const int na = __popc(act), ni = 32 - na;
      int owner, h;
      if (slot >= 0) {
        owner = lane;
        h = 0;
      } else {
        const int r = __popc(~act & lt_mask);  // rank among the idle lanes
        unsigned m = act;                      // owner = the (r % na)-th owner lane
        for (int i = r % na; i > 0; --i) m &= m - 1u;
        owner = __ffs(m) - 1;
        h = r / na + 1;
      }
      const int k_own = __popc(act & ((1u << owner) - 1u));  // owner's rank among the owners
      const int helpers = ni / na + (k_own < ni % na ? 1 : 0);
      const int64_t oslot = __shfl_sync(0xffffffffu, slot, owner);
      const uint32_t otrip = __shfl_sync(0xffffffffu, trip, owner);
      if (slot >= 0) s_best[warp][lane] = ~0ull;
      __syncwarp();
      const uint32_t t0 = otrip + (uint32_t)(h * B);
      if (t0 < A.max_trips) {
        rej_draws<T, B>(A, (uint32_t)(A.s0 + oslot), t0, buf0);
        T wj[B];
        bool need[B];
        gather(buf0, wj, need);
        unsigned long long key = ~0ull;
#pragma unroll
        for (int q = B - 1; q >= 0; --q) {
          const T vj = kCapped ? (wj[q] < capv ? wj[q] : capv) : wj[q];
          if (need[q] && t0 + (uint32_t)q < A.max_trips && rej_u<T>(buf0.x[q]) * bound <= vj)
            key = ((unsigned long long)(t0 + (uint32_t)q) << 32) | buf0.j[q];
        }
        if (key != ~0ull) atomicMin(&s_best[warp][owner], key);
      }
      __syncwarp();
      if (slot >= 0) {
        const unsigned long long best = s_best[warp][lane];
        if (best != ~0ull) {
          const uint32_t jd = (uint32_t)best;
          finish(jd, kCapped ? ldg(A.w + jd) : T(0), (uint32_t)(best >> 32) + 1);
        } else {
          trip += (uint32_t)((helpers + 1) * B);
          if (trip >= A.max_trips) no_progress();
        }
      }
      __syncwarp();
      if (give_up()) break;
    }
  }
  status_or_warp(A.status, flags);
}

// ---------------------------------------------------------------------------
// lower_bound: smallest j with W[j] >= u (compared in float64), clamped to N-1
template <typename T>
__device__ __forceinline__ int64_t lower_bound_dev(const T* __restrict__ W, int64_t n, double u) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((double)ldg(W + mid) < u)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo < n ? lo : n - 1;
}

template <typename T>
__global__ void k_lower_bound(const T* __restrict__ W, int64_t n, const double* __restrict__ u, int64_t m,
                              int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)lower_bound_dev(W, n, u[i]);
}

// multinomial, numpy stream: u_i = random()_i * float(W[N-1]) (resamplers.py:68-69)
template <typename T>
__global__ void k_multinomial_numpy(const T* __restrict__ W, int64_t n, Key2x64 key, int64_t s0, int64_t count,
                                    int32_t* __restrict__ out) {
  const double total = (double)W[n - 1];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
    const double u = u64_to_unit(numpy_raw64(key, (uint64_t)(s0 + t))) * total;
    out[t] = (int32_t)lower_bound_dev(W, n, u);
  }
}

// ---------------------------------------------------------------------------
// Own-stream multinomial without materialised spacings.  U_k = S_k / S_N *
// W[N-1] with S_k = E_0 + ... + E_k, E_k = -log(u_k) from Philox counter k
// (the k_exponentials draws).  The spacings are never stored: pass 1 sums
// each 4096-element tile of E (regenerated), one CTA scans the tile sums,
// and the merge regenerates its tile's E, scans it with the SAME code as
// pass 1 and adds the tile prefix.  S_k = max(P_t + L_k, S_last(t-1)): the
// clamp keeps U sorted across a tile boundary where the tile-prefix scan
// rounds an ulp below the previous tile's last value (a tile adds ~4096, so
// one clamp never reaches past one boundary).  CTA t then writes a[k] =
// min(N-1, #{j : W[j] < U_k}) for its own U tile: binary searches over W
// staged in shared memory when the tile's W run fits.
constexpr int kMnThreads = 128, kMnPer = 8, kMnWarps = kMnThreads / 32;
constexpr int kMnTile = kMnThreads * kMnPer;  // 1024 spacings per tile: more CTAs in flight

__device__ __forceinline__ double mn_spacing(int64_t k, uint32_t k0, uint32_t k1) {
  uint32_t o[4];
  philox4x32_10((uint32_t)k, (uint32_t)(k >> 32), kTagMultinomial, 0, k0, k1, o);
  const uint64_t x = ((uint64_t)o[0] << 32) | o[1];
  const double u = ((double)(x >> 11) + 1.0) * (1.0 / 9007199254740992.0);  // (0, 1]
  return -log(u);
}

// inclusive scan of one tile's kMnTile spacings e (thread tid holds indices
// kMnPer tid .. kMnPer (tid + 1) - 1; past N: 0), fixed association:
// thread-serial, Kogge-Stone over the warp's thread totals, serial fold of
// the warp totals.  L[i] = inclusive value; returns the tile's last inclusive value.
__device__ double mn_tile_scan(const double (&e)[kMnPer], double (&L)[kMnPer], double* s_warp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double run = 0.0;
#pragma unroll
  for (int i = 0; i < kMnPer; ++i) {
    run += e[i];
    L[i] = run;
  }
  double incl = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  double excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = 0.0;
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  double wex = 0.0, tot = 0.0;
#pragma unroll
  for (int q = 0; q < kMnWarps; ++q) {
    if (q == warp) wex = tot;
    tot += s_warp[q];
  }
  const double base = wex + excl;
#pragma unroll
  for (int i = 0; i < kMnPer; ++i) L[i] = base + L[i];
  __syncthreads();  // s_warp reused below
  if (tid == kMnThreads - 1) s_warp[kMnWarps] = L[kMnPer - 1];
  __syncthreads();
  const double last = s_warp[kMnWarps];
  __syncthreads();
  return last;
}

// pass 1: the spacings E_k (k <= N) into E, and each tile's scan total
__global__ void __launch_bounds__(kMnThreads) k_mn_tilesum(int64_t n, uint32_t k0, uint32_t k1, int64_t tiles,
                                                    double* __restrict__ E, double* __restrict__ tsum) {
  __shared__ double s_warp[kMnWarps + 1];
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t e0 = t * kMnTile + (int64_t)threadIdx.x * kMnPer;
    double e[kMnPer], L[kMnPer];
#pragma unroll
    for (int i = 0; i < kMnPer; ++i) e[i] = e0 + i <= n ? mn_spacing(e0 + i, k0, k1) : 0.0;
    if (e0 + kMnPer <= n + 1) {
      double2* dst = reinterpret_cast<double2*>(E + e0);
#pragma unroll
      for (int i = 0; i < kMnPer / 2; ++i) dst[i] = make_double2(e[2 * i], e[2 * i + 1]);
    } else {
#pragma unroll
      for (int i = 0; i < kMnPer; ++i)
        if (e0 + i <= n) E[e0 + i] = e[i];
    }
    const double tot = mn_tile_scan(e, L, s_warp);
    if (threadIdx.x == 0) tsum[t] = tot;
  }
}

// exclusive prefix of the tile sums, one CTA (1024 threads, fixed
// association): P[t], and P[tiles] = S_N = P[last] + tsum[last]
__global__ void __launch_bounds__(1024) k_mn_tileprefix(const double* __restrict__ tsum, int64_t tiles,
                                                        double* __restrict__ P) {
  __shared__ double s_w[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t per = (tiles + 1023) / 1024;
  const int64_t t0 = (int64_t)tid * per, t1 = min(t0 + per, tiles);
  double run = 0.0;
  for (int64_t t = t0; t < t1; ++t) run += tsum[t];
  double incl = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  double excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = 0.0;
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  double wex = 0.0, tot = 0.0;
  for (int q = 0; q < 32; ++q) {
    if (q == warp) wex = tot;
    tot += s_w[q];
  }
  double acc = wex + excl;
  for (int64_t t = t0; t < t1; ++t) {
    P[t] = acc;
    acc += tsum[t];
  }
  if (t1 == tiles && t0 < t1) P[tiles] = P[tiles - 1] + tsum[tiles - 1];
}

template <typename T>
__device__ __forceinline__ int64_t mn_below_range(const T* __restrict__ W, int64_t lo, int64_t hi, double u) {
  while (lo < hi) {  // first j in [lo, hi) with W[j] >= u
    const int64_t mid = (lo + hi) >> 1;
    if ((double)ldg(W + mid) < u)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// U at a tile's first index (S clamped to the previous tile's last value),
// exactly as k_mn_merge computes it: thread 0's L[0] = (0 + 0) + (0 + e0)
__device__ __forceinline__ double mn_first_u(const double* __restrict__ E, const double* __restrict__ P,
                                             const double* __restrict__ tsum, int64_t t, double scale) {
  const double l0 = (0.0 + 0.0) + (0.0 + E[t * kMnTile]);
  const double sk = P[t] + l0;
  const double prev = t > 0 ? P[t - 1] + tsum[t - 1] : 0.0;
  return (sk > prev ? sk : prev) * scale;
}

// U = S * (W[N-1] / S_N): one multiply per uniform (monotone in S)
template <typename T>
__device__ __forceinline__ double mn_scale(const T* __restrict__ W, int64_t n, const double* __restrict__ P,
                                           int64_t tiles) {
  return (double)ldg(W + n - 1) / P[tiles];
}

constexpr int kMnStage = 2048;  // W run staged in shared memory (a tile's run: ~1024 +- 3 sigma)

// every tile's W run start lo[t - tb] = #{W < U_first(t)}, t in [tb, te]:
// one thread each, all the binary searches in flight together (used when
// the merge CTAs loop over several tiles each)
template <typename T>
__global__ void __launch_bounds__(256) k_mn_search(const T* __restrict__ W, int64_t n, const double* __restrict__ E,
                                                   const double* __restrict__ P, const double* __restrict__ tsum,
                                                   int64_t tiles, int64_t tb, int64_t te, int64_t* __restrict__ lo) {
  const int64_t t = tb + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > te) return;
  lo[t - tb] = t * kMnTile >= n ? n : mn_below_range<T>(W, 0, n, mn_first_u(E, P, tsum, t, mn_scale<T>(W, n, P, tiles)));
}

// lo_t == nullptr: one tile per CTA, which searches its own run bounds
// while its spacings load and scan; else the bounds come from k_mn_search
template <typename T>
__global__ void __launch_bounds__(kMnThreads) k_mn_merge(const T* __restrict__ W, int64_t n, const double* __restrict__ E,
                                                  const double* __restrict__ P, const double* __restrict__ tsum,
                                                  const int64_t* __restrict__ lo_t, int64_t tiles, int64_t s0,
                                                  int64_t s1, int32_t* __restrict__ out, int32_t* __restrict__ claim) {
  __shared__ double s_warp[kMnWarps + 1];
  __shared__ T sw[kMnStage];
  __shared__ int64_t s_lohi[2];
  const double scale = mn_scale<T>(W, n, P, tiles);
  const int64_t tb = s0 / kMnTile, te = (s1 + kMnTile - 1) / kMnTile;  // U tiles covering [s0, s1)
  for (int64_t t = tb + blockIdx.x; t < te; t += gridDim.x) {
    // the tile's W run [lo(t), lo(t+1) + 1) with lo(t) = #{W < U_first(t)}
    // (U_last(t) <= U_first(t+1)): two binary searches, in flight while
    // the spacings load and scan
    if (threadIdx.x < 2) {
      const int64_t tt = t + threadIdx.x;
      s_lohi[threadIdx.x] = lo_t ? lo_t[tt - tb]
                            : tt * kMnTile >= n ? n
                                                : mn_below_range<T>(W, 0, n, mn_first_u(E, P, tsum, tt, scale));
    }
    const int64_t k0i = t * kMnTile + (int64_t)threadIdx.x * kMnPer;  // this thread's first index
    double e[kMnPer], L[kMnPer];
    if (k0i + kMnPer <= n + 1) {
      const double2* src = reinterpret_cast<const double2*>(E + k0i);
#pragma unroll
      for (int i = 0; i < kMnPer / 2; ++i) {
        const double2 v = __ldcs(src + i);
        e[2 * i] = v.x;
        e[2 * i + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < kMnPer; ++i) e[i] = k0i + i <= n ? E[k0i + i] : 0.0;
    }
    mn_tile_scan(e, L, s_warp);
    const double pt = P[t];
    const double prev_last = t > 0 ? P[t - 1] + tsum[t - 1] : 0.0;
    double u[kMnPer];
#pragma unroll
    for (int i = 0; i < kMnPer; ++i) {
      const double sk = pt + L[i];
      u[i] = (sk > prev_last ? sk : prev_last) * scale;
    }
    // the tile's W run [lo(t), lo(t+1) + 1): U_last(t) <= U_first(t+1)
    const int64_t lo = s_lohi[0], hi = max(lo, min(n, s_lohi[1] + 1));  // after mn_tile_scan's barriers
    const bool staged = hi - lo <= kMnStage;  // CTA-uniform
    if (staged) {
      // eight independent loads in flight per thread, then the stores
      for (int64_t j0 = lo + threadIdx.x; j0 < hi; j0 += 8 * (int64_t)blockDim.x) {
        T v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int64_t j = j0 + r * (int64_t)blockDim.x;
          v[r] = j < hi ? ldg(W + j) : T(0);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int64_t j = j0 + r * (int64_t)blockDim.x;
          if (j < hi) sw[j - lo] = v[r];
        }
      }
    }
    __syncthreads();
    if (staged) {
      // 32-bit positions inside the staged run.  Float W: (double)w < u iff
      // w < u rounded up to float (no float lies strictly between), so the
      // compares stay in float
      float uf[kMnPer];
#pragma unroll
      for (int i = 0; i < kMnPer; ++i) uf[i] = __double2float_ru(u[i]);
      auto below = [&](int x, int i) -> bool {
        if constexpr (sizeof(T) == 4)
          return sw[x] < uf[i];
        else
          return sw[x] < u[i];
      };
      const int m = (int)(hi - lo);
      int a = 0, b = m;
      while (a < b) {
        const int mid = (a + b) >> 1;
        if (below(mid, 0))
          a = mid + 1;
        else
          b = mid;
      }
      const int kmax = (int)min((int64_t)kMnPer, n - k0i);
#pragma unroll
      for (int i = 0; i < kMnPer; ++i) {
        if (i >= kmax) break;
        // the walk advances ~1 W per uniform: test four positions at once
        // (independent loads), repeat only when all four are below u
        while (true) {
          int adv = 0;
#pragma unroll
          for (int r = 0; r < 4; ++r) adv += (a + r < m && below(a + r, i)) ? 1 : 0;
          a += adv;
          if (adv < 4) break;
        }
        const int64_t k = k0i + i;
        const int64_t pos = lo + a;
        if (k >= s0 && k < s1) {
          const int32_t v = (int32_t)(pos < n ? pos : n - 1);
          out[k - s0] = v;
          if (claim) atomicMin(claim + v, (int32_t)k);
        }
      }
      __syncthreads();
      continue;
    }
    int64_t pos = mn_below_range<T>(W, lo, hi, u[0]);  // #{W < u[0]}
#pragma unroll
    for (int i = 0; i < kMnPer; ++i) {
      const int64_t k = k0i + i;
      if (k >= n) break;
      while (pos < hi && (double)ldg(W + pos) < u[i]) ++pos;
      if (k >= s0 && k < s1) {
        const int32_t v = (int32_t)(pos < n ? pos : n - 1);
        out[k - s0] = v;
        if (claim) atomicMin(claim + v, (int32_t)k);
      }
    }
    __syncthreads();
  }
}

// Code 4 (multinomial_ancestors_serial) with numpy draws: L_p = ln(d_p)/(N-p)
__global__ void k_serial_logs(int64_t n, Key2x64 key, double* __restrict__ L) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const double d = u64_to_unit(numpy_raw64(key, (uint64_t)p));
    L[p] = (d > 0.0 ? log(d) : -INFINITY) / (double)(n - p);
  }
}

// a[i] = (#{j : Wx[j] <= u}) - 1 with u = total * exp(lnmax_{N-1-i})
template <typename T>
__global__ void k_serial_sweep(const T* __restrict__ Wx, const T* __restrict__ w, int64_t n,
                               const double* __restrict__ lnmax, int32_t* __restrict__ out) {
  const double total = (double)Wx[n - 1] + (double)w[n - 1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double u = total * exp(lnmax[n - 1 - i]);
    int64_t lo = 0, hi = n;  // first j with Wx[j] > u
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((double)ldg(Wx + mid) <= u)
        lo = mid + 1;
      else
        hi = mid;
    }
    out[i] = (int32_t)(lo > 0 ? lo - 1 : 0);
  }
}

int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

uint32_t lemire_threshold(int64_t n) { return (uint32_t)((0x100000000ull - (uint64_t)n) % (uint64_t)n); }

int log2_exact(int64_t n) {
  int l = 0;
  while ((int64_t(1) << l) < n) ++l;
  return (int64_t(1) << l) == n ? l : -1;
}

}  // namespace

cudaError_t launch_lower_bound(const void* W, int64_t n, int dtype, const double* u, int64_t m, int32_t* out,
                               cudaStream_t s) {
  const int g = grid_for(m, 256);
  if (dtype == PFR_F64)
    k_lower_bound<double><<<g, 256, 0, s>>>((const double*)W, n, u, m, out);
  else
    k_lower_bound<float><<<g, 256, 0, s>>>((const float*)W, n, u, m, out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_metropolis(const void* w, int64_t n, int dtype, int64_t steps, const pfr_rng* rng,
                              const double* u_draws, const void* j_draws, int idx_dtype, int32_t* a,
                              uint32_t* status, cudaStream_t s, int64_t c_begin, int64_t c_count, int32_t* claim) {
  const int mode = rng ? rng->mode : PFR_RNG_ARRAYS;
  if (c_count < 0) c_count = n;
  if (mode == PFR_RNG_ARRAYS && (c_begin != 0 || c_count != n)) return cudaErrorNotSupported;
  if (c_count == 0) return cudaSuccess;
  const int64_t threads = (c_count + kChainsPerThread - 1) / kChainsPerThread;
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  if (mode == PFR_RNG_ARRAYS) {
    const unsigned b1 = (unsigned)((n + 255) / 256);
    if (dtype == PFR_F64) {
      if (idx_dtype == PFR_I64)
        k_metropolis_arrays<double, int64_t><<<b1, 256, 0, s>>>((const double*)w, n, steps, u_draws, (const int64_t*)j_draws, a, status);
      else
        k_metropolis_arrays<double, int32_t><<<b1, 256, 0, s>>>((const double*)w, n, steps, u_draws, (const int32_t*)j_draws, a, status);
    } else {
      if (idx_dtype == PFR_I64)
        k_metropolis_arrays<float, int64_t><<<b1, 256, 0, s>>>((const float*)w, n, steps, u_draws, (const int64_t*)j_draws, a, status);
      else
        k_metropolis_arrays<float, int32_t><<<b1, 256, 0, s>>>((const float*)w, n, steps, u_draws, (const int32_t*)j_draws, a, status);
    }
  } else if (mode == PFR_RNG_NUMPY) {
    const int l2 = log2_exact(n);
    if (l2 < 0 || n < 2) return cudaErrorNotSupported;  // numpy replay needs a power-of-two N
    Key2x64 key{rng->key0, rng->key1};
    if (dtype == PFR_F64)
      k_metropolis_numpy<double><<<blocks, 256, 0, s>>>((const double*)w, n, steps, key, l2, c_begin, c_count, a);
    else
      k_metropolis_numpy<float><<<blocks, 256, 0, s>>>((const float*)w, n, steps, key, l2, c_begin, c_count, a);
  } else {
    const uint32_t k0 = (uint32_t)rng->key0, k1 = (uint32_t)(rng->key0 >> 32);
    const uint32_t thr = lemire_threshold(n);
    if (dtype == PFR_F64)
      k_metropolis_philox<double><<<blocks, 256, 0, s>>>((const double*)w, n, steps, k0, k1, thr, c_begin, c_count, a,
                                                          status, claim);
    else
      k_metropolis_philox<float><<<blocks, 256, 0, s>>>((const float*)w, n, steps, k0, k1, thr, c_begin, c_count, a,
                                                         status, claim);
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_rejection(const void* w, int64_t n, int dtype, double bound, double cap, const pfr_rng* rng,
                             int64_t max_rounds, int32_t* a, int32_t* trips, void* out_w, uint32_t* status,
                             const Workspace& ws, cudaStream_t s, int64_t s_begin, int64_t s_count, int32_t* claim) {
  if (s_count < 0) s_count = n - s_begin;
  if (rng && rng->mode == PFR_RNG_NUMPY && s_begin == 0 && s_count == n) {
    cudaError_t e = launch_check_weights(w, n, dtype, status, s);  // check_weights' flags
    if (e != cudaSuccess) return e;
    return launch_rejection_replay(w, n, dtype, bound, cap, rng, max_rounds, a, trips, out_w, status, ws, s);
  }
  if (!rng || rng->mode != PFR_RNG_PHILOX) return cudaErrorNotSupported;
  unsigned long long* next = reinterpret_cast<unsigned long long*>(&ws.hdr->cell[2]);
  cudaError_t e = cudaMemsetAsync(next, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  const uint32_t k0 = (uint32_t)rng->key0, k1 = (uint32_t)(rng->key0 >> 32);
  const uint32_t max_trips = (uint32_t)std::min<int64_t>(max_rounds + 1, 0x7FFFFFFF);
  // persistent: one resident wave fills the machine, chunks hand out the slots
  auto blocks_for = [](auto kernel) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, 256, 0) != cudaSuccess || occ < 1) occ = 1;
    return num_sms() * occ;
  };
  // trips evaluated per lane and iteration (PFR_REJ_BATCH: profiling aid).
  // Packed draws (three trips per Philox call from 42-bit fields) measured
  // slower in round 2 (the 64-bit field extraction costs more issue slots
  // than the saved rounds) and were removed.
  static const int batch = [] {
    const char* v = getenv("PFR_REJ_BATCH");
    return v ? atoi(v) : 0;
  }();

  // certain-reject table: N <= 4 * 2^20 (groups of g <= 4 weights), the
  // workspace's O region as scratch (PFR_OP_REJECTION reserves it)
  static const bool tab_on = [] {
    const char* v = getenv("PFR_REJ_TABLE");
    return !(v && v[0] == '0');
  }();
  RejTab tb{};
  bool use_tab = false;
  if (tab_on && ws.O && n >= 4096 && n <= 4 * kRejTabMaxBits) {
    int lg = 0;
    while (((n + ((int64_t)1 << lg) - 1) >> lg) > kRejTabMaxBits) ++lg;
    tb.lg = lg;
    tb.groups = (n + ((int64_t)1 << lg) - 1) >> lg;
    tb.words = ((tb.groups + 127) / 128) * 4;  // whole uint4 rows
    tb.counts = reinterpret_cast<uint32_t*>(ws.O);
    tb.bits = tb.counts + 64;  // 256-byte aligned
    e = cudaMemsetAsync(tb.counts, 0, kRejTabK * sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    const int tblocks = (int)std::min<int64_t>((tb.words + 31) / 32, (int64_t)num_sms() * 8);
    const double cb = cap > 0 ? cap : bound;
    if (dtype == PFR_F64) {
      if (cap > 0)
        k_rej_table<double, true><<<tblocks, 256, 0, s>>>((const double*)w, n, cb, cap, tb, status);
      else
        k_rej_table<double, false><<<tblocks, 256, 0, s>>>((const double*)w, n, cb, cap, tb, status);
    } else {
      if (cap > 0)
        k_rej_table<float, true><<<tblocks, 256, 0, s>>>((const float*)w, n, cb, cap, tb, status);
      else
        k_rej_table<float, false><<<tblocks, 256, 0, s>>>((const float*)w, n, cb, cap, tb, status);
    }
    note_launch();
    use_tab = true;
  }
  if (!use_tab) {
    // check_weights' flags (the table kernel reports them when it runs)
    e = launch_check_weights(w, n, dtype, status, s);
    if (e != cudaSuccess) return e;
  }
  const size_t tab_smem = use_tab ? (size_t)tb.words * 4 : 0;
  // measured (N=2^20, sigma=1, sup = max w): table kernel 8 trips per lane
  // and batch for both dtypes (349 / 353 us); plain kernel float32 8, float64 4
  const int b_f32 = batch ? batch : 8, b_f64 = batch ? batch : (use_tab ? 8 : 4);
  auto tab_blocks = [&](auto kernel) {
    // every call: the instantiations share one function-pointer type
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kRejTabMaxBits / 8));
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kRejTabThreads, tab_smem) != cudaSuccess ||
        occ < 1)
      occ = 1;
    return num_sms() * occ;
  };
#define PFR_REJ_LAUNCH(T, CAP, B)                                                                             \
  do {                                                                                                        \
    if (use_tab)                                                                                              \
      k_rejection_philox<T, CAP, B, true>                                                                     \
          <<<tab_blocks(k_rejection_philox<T, CAP, B, true>), kRejTabThreads, tab_smem, s>>>(A, tb);          \
    else                                                                                                      \
      k_rejection_philox<T, CAP, B><<<blocks_for(k_rejection_philox<T, CAP, B>), 256, 0, s>>>(A, tb);         \
  } while (0)
#define PFR_REJ_DISPATCH(T, CAP)                \
  do {                                          \
    switch (sizeof(T) == 4 ? b_f32 : b_f64) {   \
      case 2: PFR_REJ_LAUNCH(T, CAP, 2); break; \
      case 4: PFR_REJ_LAUNCH(T, CAP, 4); break; \
      default: PFR_REJ_LAUNCH(T, CAP, 8); break; \
    }                                           \
  } while (0)
  if (dtype == PFR_F64) {
    RejArgs<double> A{(const double*)w, n, cap > 0 ? cap : bound, cap, k0, k1, lemire_threshold(n), max_trips,
                      s_begin, s_count, a, trips, (double*)out_w, next, status, claim};
    if (cap > 0)
      PFR_REJ_DISPATCH(double, true);
    else
      PFR_REJ_DISPATCH(double, false);
  } else {
    RejArgs<float> A{(const float*)w, n, cap > 0 ? cap : bound, cap, k0, k1, lemire_threshold(n), max_trips,
                     s_begin, s_count, a, trips, (float*)out_w, next, status, claim};
    if (cap > 0)
      PFR_REJ_DISPATCH(float, true);
    else
      PFR_REJ_DISPATCH(float, false);
  }
#undef PFR_REJ_DISPATCH
#undef PFR_REJ_LAUNCH
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_multinomial(const void* w, int64_t n, int dtype, int accum, const pfr_rng* rng,
                               const double* uniforms, int sorted_serial, int32_t* a, uint32_t* status,
                               const Workspace& ws, cudaStream_t s, int64_t s_begin, int64_t s_count,
                               int32_t* claim) {
  if (s_count < 0) s_count = n - s_begin;
  const bool full = s_begin == 0 && s_count == n;
  if (sorted_serial && !full) return cudaErrorNotSupported;
  // W = inclusive scan of w (monotone, weights are non-negative) into scratch
  void* W = ws.f1;
  const int scan_flags = accum | PFR_SCAN_MONOTONE;
  const int g = grid_for(n, 256);
  if (sorted_serial) {
    // Code 4: exclusive scan Wx, log spacings scanned in float64
    if (!rng || rng->mode != PFR_RNG_NUMPY) return cudaErrorNotSupported;
    cudaError_t e = launch_scan(w, W, n, dtype, dtype, scan_flags, 1, nullptr, -1, status, ws, s);
    if (e != cudaSuccess) return e;
    Key2x64 key{rng->key0, rng->key1};
    k_serial_logs<<<g, 256, 0, s>>>(n, key, ws.f0);
    note_launch();
    // the log-spacing scan has negative terms: no monotone repair
    e = launch_scan(ws.f0, ws.f0, n, PFR_F64, PFR_F64, PFR_ACC_F64, 0, nullptr, -1, status, ws, s);
    if (e != cudaSuccess) return e;
    if (dtype == PFR_F64)
      k_serial_sweep<double><<<g, 256, 0, s>>>((const double*)W, (const double*)w, n, ws.f0, a);
    else
      k_serial_sweep<float><<<g, 256, 0, s>>>((const float*)W, (const float*)w, n, ws.f0, a);
    note_launch();
    return cudaGetLastError();
  }
  // the weight scan also validates w (check_weights' flags into status)
  cudaError_t e = launch_scan(w, W, n, dtype, dtype, scan_flags | PFR_SCAN_WEIGHTS, 0, nullptr, -1, status, ws, s);
  if (e != cudaSuccess) return e;
  const int mode = uniforms ? PFR_RNG_ARRAYS : (rng ? rng->mode : PFR_RNG_PHILOX);
  if (mode == PFR_RNG_ARRAYS) {
    // the caller's uniforms of these slots
    return launch_lower_bound(W, n, dtype, uniforms + s_begin, s_count, a, s);
  } else if (mode == PFR_RNG_NUMPY) {
    Key2x64 key{rng->key0, rng->key1};
    const int gs = grid_for(s_count, 256);
    if (dtype == PFR_F64)
      k_multinomial_numpy<double><<<gs, 256, 0, s>>>((const double*)W, n, key, s_begin, s_count, a);
    else
      k_multinomial_numpy<float><<<gs, 256, 0, s>>>((const float*)W, n, key, s_begin, s_count, a);
    note_launch();
  } else {
    const uint32_t k0 = (uint32_t)rng->key0, k1 = (uint32_t)(rng->key0 >> 32);
    // the N+1 spacings and their tile sums, the tile prefixes (and S_N),
    // the merge (scratch: f0 = E, O = the tile sums and prefixes)
    if (!ws.O) return cudaErrorNotSupported;
    const int64_t tiles = (n + 1 + kMnTile - 1) / kMnTile;
    double* E = ws.f0;
    double* tsum = reinterpret_cast<double*>(ws.O);
    double* P = tsum + ((tiles + 31) / 32) * 32;
    const int gt = (int)std::min<int64_t>(tiles, (int64_t)num_sms() * 16);
    k_mn_tilesum<<<gt, kMnThreads, 0, s>>>(n, k0, k1, tiles, E, tsum);
    k_mn_tileprefix<<<1, 1024, 0, s>>>(tsum, tiles, P);
    const int64_t s1 = s_begin + s_count;
    const int64_t tb = s_begin / kMnTile, te = (s1 + kMnTile - 1) / kMnTile;
    const int gm = (int)std::min<int64_t>(te - tb, (int64_t)num_sms() * 16);
    static const bool carve = [] {
      cudaFuncSetAttribute(k_mn_merge<double>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
      cudaFuncSetAttribute(k_mn_merge<float>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
      return true;
    }();
    (void)carve;
    // more tiles than CTAs: the bounds first, all searches at once
    int64_t* lo = te - tb > gm ? reinterpret_cast<int64_t*>(P + ((tiles + 1 + 31) / 32) * 32) : nullptr;
    const unsigned gs = (unsigned)((te - tb + 1 + 255) / 256);
    if (dtype == PFR_F64) {
      if (lo) k_mn_search<double><<<gs, 256, 0, s>>>((const double*)W, n, E, P, tsum, tiles, tb, te, lo);
      k_mn_merge<double><<<gm, kMnThreads, 0, s>>>((const double*)W, n, E, P, tsum, lo, tiles, s_begin, s1, a, claim);
    } else {
      if (lo) k_mn_search<float><<<gs, 256, 0, s>>>((const float*)W, n, E, P, tsum, tiles, tb, te, lo);
      k_mn_merge<float><<<gm, kMnThreads, 0, s>>>((const float*)W, n, E, P, tsum, lo, tiles, s_begin, s1, a, claim);
    }
    note_launch(lo ? 4 : 3);
    note_launch();
  }
  return cudaGetLastError();
}

}  // namespace pfr
