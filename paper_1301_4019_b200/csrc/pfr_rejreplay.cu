// Rejection resampling on the reference's own random stream (parity mode).
//
// Reference: _rejection_loop, resamplers.py:282-310 (rejection_ancestors
// 237-255, rejection_ancestors_capped 258-279).  The loop is
// round-synchronous: every slot first proposes itself with one uniform
// (random(N)); then, per round, the still-pending slots -- in ascending slot
// order -- draw integers(0, N, m) followed by random(m) from ONE generator.
// The stream position of a draw therefore depends on the sizes of all
// earlier pending sets, and the replay runs round by round:
//
//   phase 1  every pending position k evaluates its proposal j_k and its
//            uniform beta_k at their stream positions (a pure function of the
//            round's start state and k), keep[k] = !(beta_k <= ratio[j_k]);
//   phase 2  accepted slots write a = j, trips = round + 1; survivors are
//            compacted IN ORDER (block counts -> block prefix -> ordered
//            block-local scan) into the next pending list.
//
// numpy stream model (numpy 2.x distributions.c / philox.h; pinned by the
// golden stream vectors): the k-th raw u64 is Philox4x64-10(counter k/4 +
// 1)[k % 4] (pfr_rng.cuh); random() = (u64 >> 11) 2^-53; integers(0, N)
// takes 32-bit words from next_uint32, which returns the LOW half of a fresh
// u64 and keeps the high half buffered for the next 32-bit request (the
// buffer survives across calls, so it can hold a word from before the
// previous random() call; random() never touches it), mapped by
// Lemire's method: j = (u32 * N) >> 32, redrawn while the low word is below
// (2^32 - N) mod N.  A power-of-two N never redraws; otherwise a redraw
// (probability ~N/2^32 per draw) shifts every later draw of its round, so
// such a round is recomputed by one thread (rare, exact).
//
// One cooperative launch runs the rounds with grid-wide barriers while many
// slots are pending and hands the tail (<= kTailM pending) to one CTA.
#include <cooperative_groups.h>

#include <algorithm>

#include "pfr_common.cuh"
#include "pfr_internal.h"

namespace cg = cooperative_groups;

namespace pfr {

namespace {

constexpr int kRrThreads = 256;
constexpr int64_t kTailM = 16384;

struct StreamPos {
  uint64_t q;   // next fresh u64 index
  uint64_t bq;  // the u64 whose high half is buffered (valid when bf)
  uint32_t bf;  // 1: a high half is buffered for next_uint32
};

// t-th 32-bit request of an integers() call starting at state s
__device__ __forceinline__ uint32_t stream_u32(Key2x64 key, StreamPos s, uint64_t t) {
  if (s.bf) {
    if (t == 0) return (uint32_t)(numpy_raw64(key, s.bq) >> 32);
    t -= 1;
  }
  const uint64_t x = numpy_raw64(key, s.q + t / 2);
  return (t & 1) ? (uint32_t)(x >> 32) : (uint32_t)x;
}

// state after `u32s` 32-bit requests
__device__ __forceinline__ StreamPos stream_after_u32(StreamPos s, uint64_t u32s) {
  if (u32s == 0) return s;
  if (s.bf) {
    s.bf = 0;
    u32s -= 1;
  }
  s.q += (u32s + 1) / 2;
  s.bf = (uint32_t)(u32s & 1);
  s.bq = s.q - 1;  // an odd count leaves the high half of the last fresh word
  return s;
}

template <typename T>
struct RrArgs {
  const T* w;
  int64_t n;
  double bound;  // sup_w, or sup_v for the capped variant
  int capped;
  Key2x64 key;
  uint32_t thr;  // Lemire threshold (2^32 - N) mod N
  int64_t max_rounds;
  int32_t* a;
  int32_t* trips;  // optional
  uint32_t* status;
  int32_t* list0;  // pending lists: slot numbers in ascending order
  int32_t* list1;
  int32_t* jj;     // proposals of the current round, by position
  uint8_t* keep;   // 1: the position stays pending
  int32_t* bcnt;   // per-block survivor counts
  uint32_t* cells; // [0..1] Lemire-redraw flags (round parity), [2..3] u32s a redone round consumed
};

// ratio = v / bound in the weight dtype (resamplers.py:291), widened to
// float64 for the comparison with the float64 uniform (numpy promotion)
template <typename T>
__device__ __forceinline__ double ratio_of(const RrArgs<T>& p, int64_t j) {
  const T bT = (T)p.bound;
  T v = p.w[j];
  if (p.capped) v = v < bT ? v : bT;  // np.minimum(w, sup_v) (w is validated: no NaN)
  if constexpr (sizeof(T) == 8)
    return __ddiv_rn(v, bT);
  else
    return (double)__fdiv_rn(v, bT);
}

__device__ __forceinline__ int64_t part_lo(int64_t m, int G, int b) { return m * b / G; }

// block-wide exclusive scan of 0/1 flags (kRrThreads threads); returns the
// prefix, *total gets the block total
__device__ __forceinline__ int block_flag_scan(bool f, int* warp_cnt, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned m = __ballot_sync(0xffffffffu, f);
  if (lane == 0) warp_cnt[warp] = __popc(m);
  __syncthreads();
  int before = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kRrThreads / 32; ++w) {
    const int c = warp_cnt[w];
    if (w < warp) before += c;
    tot += c;
  }
  __syncthreads();
  *total = tot;
  return before + __popc(m & ((1u << lane) - 1));
}

template <typename T>
__global__ void __launch_bounds__(kRrThreads) k_rej_replay(RrArgs<T> p) {
  __shared__ int warp_cnt[kRrThreads / 32];
  __shared__ int64_t s_red[kRrThreads / 32];
  cg::grid_group grid = cg::this_grid();
  const int64_t n = p.n;
  const int tid = threadIdx.x;
  int G = gridDim.x;
  const int B = blockIdx.x;
  bool multi = true;
  auto sync = [&]() {
    if (multi)
      grid.sync();
    else
      __syncthreads();
  };

  // ---- round 0: slot i proposes itself with random()_i (resamplers.py:293-294)
  {
    uint32_t flags = 0;
    const int64_t lo = part_lo(n, G, B), hi = part_lo(n, G, B + 1);
    int64_t cnt = 0;
    for (int64_t i = lo + tid; i < hi; i += kRrThreads) {
      const double r = ratio_of(p, i);
      if (!(r <= 1.7976931348623157e308)) flags |= PFR_ST_RATIO;  // inf or NaN
      const double beta = u64_to_unit(numpy_raw64(p.key, (uint64_t)i));
      const bool pend = beta > r;
      p.keep[i] = pend;
      p.a[i] = (int32_t)i;
      if (p.trips) p.trips[i] = 1;
      cnt += pend;
    }
    status_or_warp(p.status, flags);
    cnt = __reduce_add_sync(0xffffffffu, (unsigned)cnt);
    if ((tid & 31) == 0) s_red[tid >> 5] = cnt;
    __syncthreads();
    if (tid == 0) {
      int64_t t = 0;
      for (int w = 0; w < kRrThreads / 32; ++w) t += s_red[w];
      p.bcnt[B] = (int32_t)t;
      if (B == 0) {
        p.cells[0] = p.cells[1] = 0u;
      }
    }
    sync();
    if (*(volatile uint32_t*)p.status & PFR_ST_RATIO) return;  // the host raises ValueError
  }

  // ---- ordered compaction of round 0 (positions = slots)
  int64_t m = 0, before = 0;
  for (int b = 0; b < G; ++b) {
    const int64_t c = *(volatile int32_t*)&p.bcnt[b];
    if (b < B) before += c;
    m += c;
  }
  {
    const int64_t lo = part_lo(n, G, B), hi = part_lo(n, G, B + 1);
    int64_t run = before;
    for (int64_t k0 = lo; k0 < hi; k0 += kRrThreads) {
      const int64_t k = k0 + tid;
      const bool f = k < hi && p.keep[k];
      int tot;
      const int pos = block_flag_scan(f, warp_cnt, &tot);
      if (f) p.list0[run + pos] = (int32_t)k;
      run += tot;
    }
  }
  StreamPos st{(uint64_t)n, 0u, 0u};  // random(N) consumed N fresh words
  int32_t* L = p.list0;
  int32_t* Ln = p.list1;
  sync();

  for (int64_t r = 1; m > 0; ++r) {
    if (r > p.max_rounds) {
      if (B == 0 && tid == 0) status_or(p.status, PFR_ST_NOPROGRESS);
      return;
    }
    if (multi && m <= kTailM) {
      // tail: one CTA continues alone
      if (B != 0) return;
      multi = false;
      G = 1;
    }
    uint32_t* bad = p.cells + (r & 1);
    uint32_t* used = p.cells + 2 + (r & 1);
    // ---- phase 1: this block's positions
    const int64_t lo = part_lo(m, G, B), hi = part_lo(m, G, B + 1);
    const StreamPos su = stream_after_u32(st, (uint64_t)m);  // uniforms start after the integers
    {
      int64_t cnt = 0;
      bool redraw = false;
      for (int64_t k = lo + tid; k < hi; k += kRrThreads) {
        const uint32_t u = stream_u32(p.key, st, (uint64_t)k);
        const uint64_t mm = (uint64_t)u * (uint64_t)n;
        redraw |= (uint32_t)mm < p.thr;
        const int32_t j = (int32_t)(mm >> 32);
        const double beta = u64_to_unit(numpy_raw64(p.key, su.q + (uint64_t)k));
        const bool pend = !(beta <= ratio_of(p, j));
        p.jj[k] = j;
        p.keep[k] = pend;
        cnt += pend;
      }
      if (__any_sync(0xffffffffu, redraw) && (tid & 31) == 0) atomicOr(bad, 1u);
      cnt = __reduce_add_sync(0xffffffffu, (unsigned)cnt);
      if ((tid & 31) == 0) s_red[tid >> 5] = cnt;
      __syncthreads();
      if (tid == 0) {
        int64_t t = 0;
        for (int w = 0; w < kRrThreads / 32; ++w) t += s_red[w];
        p.bcnt[B] = (int32_t)t;
      }
    }
    sync();
    uint64_t u32s = (uint64_t)m;
    if (*(volatile uint32_t*)bad) {
      // a Lemire redraw shifted the round: recompute it serially (exact)
      if (B == 0 && tid == 0) {
        uint64_t t = 0;
        for (int64_t k = 0; k < m; ++k) {
          uint64_t mm;
          do {
            mm = (uint64_t)stream_u32(p.key, st, t++) * (uint64_t)n;
          } while ((uint32_t)mm < p.thr);
          p.jj[k] = (int32_t)(mm >> 32);
        }
        const StreamPos s2 = stream_after_u32(st, t);
        for (int b = 0; b < G; ++b) p.bcnt[b] = 0;
        for (int64_t k = 0; k < m; ++k) {
          const double beta = u64_to_unit(numpy_raw64(p.key, s2.q + (uint64_t)k));
          const bool pend = !(beta <= ratio_of(p, p.jj[k]));
          p.keep[k] = pend;
          if (pend) {
            int b = 0;
            while (b + 1 < G && k >= part_lo(m, G, b + 1)) ++b;
            p.bcnt[b] += 1;
          }
        }
        *(volatile uint32_t*)used = (uint32_t)(t - (uint64_t)m);  // extra words beyond m (fits: rare)
        __threadfence();
      }
      sync();
      u32s = (uint64_t)m + *(volatile uint32_t*)used;
    }
    // ---- phase 2: accepted writes, ordered compaction
    int64_t mn = 0;
    before = 0;
    for (int b = 0; b < G; ++b) {
      const int64_t c = *(volatile int32_t*)&p.bcnt[b];
      if (b < B) before += c;
      mn += c;
    }
    {
      int64_t run = before;
      for (int64_t k0 = lo; k0 < hi; k0 += kRrThreads) {
        const int64_t k = k0 + tid;
        const bool in = k < hi;
        const bool f = in && p.keep[k];
        const int32_t slot = in ? L[k] : 0;
        if (in && !f) {
          p.a[slot] = p.jj[k];
          if (p.trips) p.trips[slot] = (int32_t)(r + 1);
        }
        int tot;
        const int pos = block_flag_scan(f, warp_cnt, &tot);
        if (f) Ln[run + pos] = slot;
        run += tot;
      }
    }
    if (B == 0 && tid == 0) p.cells[(r + 1) & 1] = 0u;  // next round's flag (last read in round r-1)
    st = stream_after_u32(st, u32s);
    st.q += (uint64_t)m;  // the uniforms
    int32_t* t = L;
    L = Ln;
    Ln = t;
    m = mn;
    sync();
  }
}

// capped variant: importance weights w[a]/v[a], 1 where v[a] == 0
// (resamplers.py:275-277), in the weight dtype
template <typename T>
__global__ void k_rr_outw(const T* __restrict__ w, int64_t n, double cap, const int32_t* __restrict__ a,
                          T* __restrict__ out_w) {
  const T c = (T)cap;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const T wa = w[a[i]];
    const T va = wa < c ? wa : c;
    T r;
    if constexpr (sizeof(T) == 8)
      r = __ddiv_rn(wa, va);
    else
      r = __fdiv_rn(wa, va);
    out_w[i] = va == T(0) ? T(1) : r;
  }
}

template <typename T>
cudaError_t rej_replay_typed(const T* w, int64_t n, double bound, double cap, const pfr_rng* rng, int64_t max_rounds,
                             int32_t* a, int32_t* trips, T* out_w, uint32_t* status, const Workspace& ws,
                             cudaStream_t s) {
  RrArgs<T> p;
  p.w = w;
  p.n = n;
  p.capped = cap > 0;
  p.bound = cap > 0 ? cap : bound;
  p.key = Key2x64{rng->key0, rng->key1};
  p.thr = (uint32_t)((0x100000000ull - (uint64_t)n) % (uint64_t)n);
  p.max_rounds = max_rounds;
  p.a = a;
  p.trips = trips;
  p.status = status;
  p.list0 = ws.j0;
  p.list1 = ws.j1;
  p.jj = ws.r0;
  p.keep = reinterpret_cast<uint8_t*>(ws.r1);
  p.bcnt = ws.d;
  p.cells = reinterpret_cast<uint32_t*>(ws.O);
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rej_replay<T>, kRrThreads, 0);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorNotSupported;
  const int64_t want = (n + kRrThreads - 1) / kRrThreads;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, num_sms()));
  void* args[] = {&p};
  e = cudaLaunchCooperativeKernel((const void*)k_rej_replay<T>, dim3(grid), dim3(kRrThreads), args, 0, s);
  note_launch();
  if (e != cudaSuccess || !p.capped) return e;
  k_rr_outw<T><<<(unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8), 256, 0, s>>>(w, n, cap, a,
                                                                                                      out_w);
  note_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_rejection_replay(const void* w, int64_t n, int dtype, double bound, double cap,
                                    const pfr_rng* rng, int64_t max_rounds, int32_t* a, int32_t* trips, void* out_w,
                                    uint32_t* status, const Workspace& ws, cudaStream_t s) {
  if (!ws.j0 || !ws.O || !ws.d) return cudaErrorInvalidValue;
  if (dtype == PFR_F64)
    return rej_replay_typed<double>((const double*)w, n, bound, cap, rng, max_rounds, a, trips, (double*)out_w,
                                    status, ws, s);
  return rej_replay_typed<float>((const float*)w, n, bound, cap, rng, max_rounds, a, trips, (float*)out_w, status,
                                 ws, s);
}

}  // namespace pfr
