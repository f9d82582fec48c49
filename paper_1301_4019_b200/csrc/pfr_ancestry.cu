// Ancestry conversions and the in-place permutation.
//
// Reference: ancestry.py (conversions 69-94, predicate 97-101, prepermute
// 125-136, permute_parallel 139-174), pf.py:86-97 (in-place copy).
//
// permute_parallel semantics (restated): d = prepermute(a); a slot i "loses"
// when d[a[i]] != i; it follows x <- d[x] until d[x] is the sentinel and
// claims that slot; c = a[d].  Equivalently c[x] = x for every x with
// offspring, and the hole a losing chain ends in receives a[i].  The
// claim graph x -> d[x] has in-degree <= 1 and losers have in-degree 0, so the
// chains are vertex-disjoint and each ends in its own hole (SURVEY.md finding
// 3): plain stores are race free and the result is schedule independent --
// bit-identical to the reference's serial loop.
//
// Kernels:
//   k_claim / k_walk        -- general ancestry: atomicMin claims, bounded walk
//   k_permute_sorted        -- directly from cumulative offspring O (sorted a):
//                              merge-path over (parent ends, slots) so every CTA
//                              gets 4096 items regardless of the weight skew;
//                              d[x] = O[x-1] needs no atomics
//   k_fallback              -- cooperative pointer jumping (Wyllie list
//                              ranking) for chains longer than the walk bound
//   k_expand                -- cumulative_offspring_to_ancestors, merge-path
#include <cooperative_groups.h>

#include "pfr_internal.h"
#include "pfr_tile.cuh"

namespace cg = cooperative_groups;

namespace pfr {

namespace {

constexpr int kWalkBound = 128;  // steps before a walker defers to the fallback
constexpr int kMergeItems = kTile;  // merge-path items per CTA (4096)
constexpr int kMergePerThread = kTileItems;  // 16

template <typename I>
__device__ __forceinline__ int64_t ld_idx(const I* p, int64_t i) {
  return (int64_t)p[i];
}

// smallest v in [lo, hi) with O[v] >= d - v  (MergePath split, ties: parent end first)
template <typename Get>
__device__ __forceinline__ int64_t merge_split(int64_t d, int64_t lo, int64_t hi, Get O) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (O(mid) >= d - mid)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

__device__ __forceinline__ void mark_overflow(WsHeader* hdr, uint32_t* status) {
  hdr->overflow = 1;
  status_or(status, PFR_ST_OVERFLOW);
}

// ---------------------------------------------------------------------------
// permute from cumulative offspring (sorted ancestry never materialised)
__global__ void __launch_bounds__(kTileThreads)
    k_permute_sorted(const int32_t* __restrict__ O, int64_t n, int32_t* __restrict__ c, int32_t* max_steps,
                     WsHeader* hdr, uint32_t* status) {
  __shared__ int32_t Os[kMergeItems + 2];
  __shared__ int64_t split[2];
  const int64_t d0 = (int64_t)blockIdx.x * kMergeItems;
  const int64_t d1 = min(d0 + kMergeItems, 2 * n);
  if (threadIdx.x < 2) {
    const int64_t d = threadIdx.x ? d1 : d0;
    split[threadIdx.x] = merge_split(d, max((int64_t)0, d - n), min(d, n), [&](int64_t v) { return (int64_t)O[v]; });
  }
  __syncthreads();
  const int64_t v0 = split[0], v1 = split[1];
  // Os[k] = O[v0 - 1 + k] for k in [0, v1 - v0 + 1]; O[-1] = 0
  for (int64_t k = threadIdx.x; k <= v1 - v0 + 1; k += blockDim.x) {
    const int64_t v = v0 - 1 + k;
    Os[k] = (v < 0) ? 0 : ((v < n) ? O[v] : (int32_t)n);
  }
  __syncthreads();
  auto Oat = [&](int64_t v) -> int64_t {  // v in [v0-1, v1]
    if (v < 0) return 0;
    if (v >= n) return n;
    return Os[v - v0 + 1];
  };
  auto Ox = [&](int64_t x) -> int64_t {  // any x in [-1, n)
    if (x >= v0 - 1 && x <= v1) return Oat(x);
    return x < 0 ? 0 : (int64_t)__ldg(O + x);
  };
  // this thread's diagonal
  const int64_t td = d0 + (int64_t)threadIdx.x * kMergePerThread;
  if (td >= d1) return;
  const int64_t tlo = max(v0, td - n), thi = min(v1, td);
  int64_t v = merge_split(td, tlo, max(tlo, thi), [&](int64_t m) { return Oat(m); });
  int64_t s = td - v;
  const int64_t tend = min(td + kMergePerThread, d1);
  int longest = 0;
  uint32_t flags = 0;
  for (int64_t it = td; it < tend; ++it) {
    const int64_t ov = (v < n) ? Oat(v) : (int64_t)1 << 62;
    if (v < n && (s >= n || ov <= s)) {
      // parent v ends: it keeps its own slot when it has offspring
      if (ov > Oat(v - 1)) c[v] = (int32_t)v;
      ++v;
    } else {
      // slot s belongs to parent v; losers are the non-first slots of the block
      if (s != Oat(v - 1)) {
        int64_t x = s;
        int steps = 0;
        while (true) {
          const int64_t hi = Ox(x);
          const int64_t lo = Ox(x - 1);
          if (hi == lo) break;  // x has no offspring: the hole
          x = lo;               // d[x] = first slot of parent x
          if (++steps > kWalkBound) break;
        }
        if (steps > kWalkBound) {
          flags |= PFR_ST_OVERFLOW;
          hdr->overflow = 1;
        } else {
          c[x] = (int32_t)v;
          longest = max(longest, steps);
        }
      }
      ++s;
    }
  }
  status_or(status, flags);
  if (max_steps && longest) atomicMax(max_steps, longest);
}

// ---------------------------------------------------------------------------
// general ancestry: claims then walks
template <typename I>
__global__ void k_claim(const I* __restrict__ a, int64_t n, int32_t* __restrict__ d, int32_t* max_steps,
                        uint32_t* status) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && max_steps) *max_steps = 0;
  uint32_t f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = ld_idx(a, i);
    if (v < 0 || v >= n) {
      f |= PFR_ST_RANGE;
      continue;
    }
    atomicMin(d + v, (int32_t)i);
  }
  status_or_warp(status, f);
}

// Pointer jumping (Wyllie list ranking) over the claim graph x -> d[x] by ONE
// CTA: the rare fallback of the general permute when a walker exceeded the
// walk bound (adversarial ancestries; realistic ones stay far below it).
template <typename I>
__device__ void block_pointer_jump(const I* __restrict__ a, int64_t n, const int32_t* __restrict__ d,
                                   int32_t* __restrict__ c, int32_t* J0, int32_t* J1, int32_t* R0, int32_t* R1,
                                   int32_t* max_steps) {
  const int64_t stride = blockDim.x;
  for (int64_t x = threadIdx.x; x < n; x += stride) {
    const int64_t dx = __ldcg(d + x);
    J0[x] = dx < n ? (int32_t)dx : (int32_t)x;
    R0[x] = dx < n ? 1 : 0;
  }
  int rounds = 1;
  while ((int64_t(1) << rounds) < n) ++rounds;
  ++rounds;
  int32_t *J = J0, *Jn = J1, *R = R0, *Rn = R1;
  for (int r = 0; r < rounds; ++r) {
    __syncthreads();
    for (int64_t x = threadIdx.x; x < n; x += stride) {
      const int32_t y = __ldcg(J + x);
      Jn[x] = __ldcg(J + y);
      Rn[x] = __ldcg(R + x) + __ldcg(R + y);
    }
    int32_t* t = J;
    J = Jn;
    Jn = t;
    t = R;
    R = Rn;
    Rn = t;
  }
  __syncthreads();
  int longest = 0;
  for (int64_t i = threadIdx.x; i < n; i += stride) {
    const int64_t v = ld_idx(a, i);
    if (v < 0 || v >= n || __ldcg(d + v) == i) continue;  // not a loser
    c[__ldcg(J + i)] = (int32_t)v;
    longest = max(longest, __ldcg(R + i));
  }
  if (max_steps && longest) atomicMax(max_steps, longest);
}

template <typename I>
__global__ void k_walk(const I* __restrict__ a, int64_t n, const int32_t* __restrict__ d, int32_t* __restrict__ c,
                       int32_t* max_steps, WsHeader* hdr, unsigned int* done, int32_t* J0, int32_t* J1, int32_t* R0,
                       int32_t* R1, uint32_t* status) {
  __shared__ bool last;
  int longest = 0;
  uint32_t f = 0;
  // 4 consecutive indices per thread per iteration: their claim checks (one
  // random d[a[i]] load each) are issued together
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; i0 < n; i0 += stride) {
    int64_t ai[4], di[4];
    if (sizeof(I) == 4 && i0 + 4 <= n && (reinterpret_cast<uintptr_t>(a) & 15) == 0) {
      const int4 av = __ldcs(reinterpret_cast<const int4*>(a + i0));
      const int4 dv = __ldcs(reinterpret_cast<const int4*>(d + i0));
      ai[0] = av.x, ai[1] = av.y, ai[2] = av.z, ai[3] = av.w;
      di[0] = dv.x, di[1] = dv.y, di[2] = dv.z, di[3] = dv.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool in = i0 + j < n;
        ai[j] = in ? ld_idx(a, i0 + j) : -1;
        di[j] = in ? (int64_t)d[i0 + j] : n;
      }
    }
    int64_t won[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool ok = ai[j] >= 0 && ai[j] < n;
      won[j] = ok ? (int64_t)__ldg(d + ai[j]) : i0 + j;  // out of range or padding: nothing to walk
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t i = i0 + j;
      if (i >= n) break;
      if (di[j] < n) c[i] = (int32_t)i;  // i has offspring: it keeps its slot
      if (ai[j] < 0 || ai[j] >= n) continue;
      if (won[j] == i) continue;  // claim won
      int64_t x = i, nx = di[j];
      int steps = 0;
      while (nx < n && steps <= kWalkBound) {
        x = nx;
        nx = __ldg(d + x);
        ++steps;
      }
      if (nx < n) {
        f |= PFR_ST_OVERFLOW;
        hdr->overflow = 1;
      } else {
        c[x] = (int32_t)ai[j];
        longest = max(longest, steps);
      }
    }
  }
  status_or_warp(status, f);
  if (max_steps && longest) atomicMax(max_steps, longest);
  // the last CTA to finish runs the (rare) fallback: no extra launch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (*(volatile int32_t*)&hdr->overflow == 1) block_pointer_jump<I>(a, n, d, c, J0, J1, R0, R1, max_steps);
  if (threadIdx.x == 0) *done = 0;
}

// ---------------------------------------------------------------------------
// cooperative fallback: pointer jumping over the claim graph.  Runs only when a
// walker overflowed (hdr->overflow set); otherwise every CTA returns at once.
// kSorted: the graph is defined by O (d[x] = O[x-1] when o[x] > 0) and a loser's
// value is its parent, found by binary search; else by (a, d).
struct FallbackArgs {
  const void* a;  // ancestry (general) or O (sorted)
  int idx64;      // general: a is int64
  const int32_t* d;
  int64_t n;
  int32_t* c;
  int32_t *J0, *J1, *R0, *R1;
  int32_t* max_steps;
  WsHeader* hdr;
};

template <bool kSorted>
__device__ __forceinline__ int64_t fb_next(const FallbackArgs& A, int64_t x) {
  if constexpr (kSorted) {
    const int32_t* O = (const int32_t*)A.a;
    const int64_t hi = O[x], lo = x ? O[x - 1] : 0;
    return hi > lo ? lo : -1;
  } else {
    const int64_t dx = A.d[x];
    return dx < A.n ? dx : -1;
  }
}

// parent of slot i for sorted ancestry: smallest p with O[p] > i
__device__ __forceinline__ int64_t sorted_parent(const int32_t* O, int64_t n, int64_t i) {
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (O[mid] > i)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

template <bool kSorted>
__global__ void k_fallback(FallbackArgs A) {
  if (*(volatile int32_t*)&A.hdr->overflow != 1) return;
  cg::grid_group grid = cg::this_grid();
  const int64_t n = A.n;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t x = t0; x < n; x += stride) {
    const int64_t nx = fb_next<kSorted>(A, x);
    A.J0[x] = nx < 0 ? (int32_t)x : (int32_t)nx;
    A.R0[x] = nx < 0 ? 0 : 1;
  }
  int rounds = 1;
  while ((int64_t(1) << rounds) < n) ++rounds;
  ++rounds;
  int32_t *J = A.J0, *Jn = A.J1, *R = A.R0, *Rn = A.R1;
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
    int64_t value;
    bool loser;
    if constexpr (kSorted) {
      const int32_t* O = (const int32_t*)A.a;
      const int64_t p = sorted_parent(O, n, i);
      loser = i != (p ? (int64_t)O[p - 1] : 0);
      value = p;
    } else {
      value = A.idx64 ? ((const int64_t*)A.a)[i] : ((const int32_t*)A.a)[i];
      loser = value >= 0 && value < n && A.d[value] != i;
    }
    if (!loser) continue;
    const int32_t h = J[i];
    A.c[h] = (int32_t)value;
    longest = max(longest, R[i]);
  }
  if (A.max_steps && longest) atomicMax(A.max_steps, longest);
}

// ---------------------------------------------------------------------------
// cumulative offspring -> sorted ancestry (merge-path expand)
template <typename I>
__global__ void __launch_bounds__(kTileThreads)
    k_expand(const I* __restrict__ O, int64_t n, int32_t* __restrict__ a) {
  __shared__ int64_t split[2];
  const int64_t d0 = (int64_t)blockIdx.x * kMergeItems;
  const int64_t d1 = min(d0 + kMergeItems, 2 * n);
  if (threadIdx.x < 2) {
    const int64_t d = threadIdx.x ? d1 : d0;
    split[threadIdx.x] = merge_split(d, max((int64_t)0, d - n), min(d, n), [&](int64_t v) { return ld_idx(O, v); });
  }
  __syncthreads();
  const int64_t v0 = split[0], v1 = split[1];
  const int64_t td = d0 + (int64_t)threadIdx.x * kMergePerThread;
  if (td >= d1) return;
  const int64_t tlo = max(v0, td - n), thi = max(tlo, min(v1, td));
  int64_t v = merge_split(td, tlo, thi, [&](int64_t m) { return ld_idx(O, m); });
  int64_t s = td - v;
  const int64_t tend = min(td + kMergePerThread, d1);
  int64_t ov = v < n ? ld_idx(O, v) : 0;
  for (int64_t it = td; it < tend; ++it) {
    if (v < n && (s >= n || ov <= s)) {
      ++v;
      if (v < n) ov = ld_idx(O, v);
    } else {
      a[s] = (int32_t)v;
      ++s;
    }
  }
}

template <typename I>
__global__ void k_check_cumulative(const I* __restrict__ O, int64_t n, uint32_t* status) {
  uint32_t f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cur = ld_idx(O, i);
    if (i == 0 && cur < 0) f |= PFR_ST_NEGCOUNT;
    if (i > 0 && cur < ld_idx(O, i - 1)) f |= PFR_ST_NOTMONOTONE;
    if (i == n - 1 && cur != n) f |= PFR_ST_BADEND;
  }
  status_or_warp(status, f);
}

template <typename I>
__global__ void k_histogram(const I* __restrict__ a, int64_t n, int32_t* __restrict__ o, uint32_t* status) {
  uint32_t f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = ld_idx(a, i);
    if (v < 0 || v >= n) {
      f |= PFR_ST_RANGE;
      continue;
    }
    atomicAdd(o + v, 1);
  }
  status_or_warp(status, f);
}

__global__ void k_fill_i32(int32_t* __restrict__ d, int64_t n, int32_t value) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = value;
}

template <typename I>
__global__ void k_mark(const I* __restrict__ c, int64_t n, int32_t* __restrict__ used, uint32_t* status) {
  uint32_t f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = ld_idx(c, i);
    if (v < 0 || v >= n) {
      f |= PFR_ST_RANGE;
      continue;
    }
    used[v] = 1;
  }
  status_or_warp(status, f);
}

template <typename I>
__global__ void k_predicate(const I* __restrict__ c, int64_t n, const int32_t* __restrict__ used,
                            int32_t* result) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (used[i] && ld_idx(c, i) != i) bad = true;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *result = 0;
}

__global__ void k_set_i32(int32_t* p, int32_t v) { *p = v; }

__global__ void k_copy_particles(double* __restrict__ x, int64_t n, int64_t width, const int32_t* __restrict__ c) {
  const int64_t total = n * width;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / width, k = e - i * width;
    const int64_t src = c[i];
    if (src != i) x[e] = x[src * width + k];
  }
}

int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

template <bool kSorted>
cudaError_t launch_fallback(const FallbackArgs& args, cudaStream_t s) {
  static int blocks_per_sm = -1;
  if (blocks_per_sm < 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_fallback<kSorted>, 256, 0);
    if (e != cudaSuccess) return e;
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  FallbackArgs a = args;
  void* params[] = {&a};
  // launched every time and exits unless a walker overflowed: a small
  // cooperative grid co-resides with concurrent work (a full-machine grid
  // waits for other streams' kernels to drain; see rare_grid in pfr_deliver.cu)
  dim3 grid((unsigned)std::min(num_sms() * blocks_per_sm, 16)), block(256);
  note_launch();
  return cudaLaunchCooperativeKernel((const void*)k_fallback<kSorted>, grid, block, params, 0, s);
}

}  // namespace

cudaError_t launch_permute_cumulative(const int32_t* O, int64_t n, int32_t* c, int32_t* max_steps, uint32_t* status,
                                      const Workspace& ws, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(&ws.hdr->overflow, 0, sizeof(int32_t), s);
  if (e != cudaSuccess) return e;
  if (max_steps) {
    e = cudaMemsetAsync(max_steps, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
  }
  const unsigned blocks = (unsigned)((2 * n + kMergeItems - 1) / kMergeItems);
  k_permute_sorted<<<blocks, kTileThreads, 0, s>>>(O, n, c, max_steps, ws.hdr, status);
  note_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  FallbackArgs fa{O, 0, nullptr, n, c, ws.j0, ws.j1, ws.r0, ws.r1, max_steps, ws.hdr};
  return launch_fallback<true>(fa, s);
}

cudaError_t launch_permute(const void* a, int64_t n, int idx_dtype, int32_t* c, int32_t* max_steps,
                           uint32_t* status, const Workspace& ws, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(&ws.hdr->overflow, 0, sizeof(int32_t), s);
  if (e != cudaSuccess) return e;
  // d = "sentinel" (0x7F7F7F7F >= N for every supported N)
  e = cudaMemsetAsync(ws.d, 0x7F, (size_t)n * sizeof(int32_t), s);
  if (e != cudaSuccess) return e;
  const int g = grid_for(n, 256);
  const int gw = grid_for((n + 3) / 4, 256);  // k_walk: 4 indices per thread
  unsigned int* done = &ws.dv->pad[0];  // zero at workspace creation; reset by the last CTA
  if (idx_dtype == PFR_I64) {
    k_claim<int64_t><<<g, 256, 0, s>>>((const int64_t*)a, n, ws.d, max_steps, status);
    k_walk<int64_t><<<gw, 256, 0, s>>>((const int64_t*)a, n, ws.d, c, max_steps, ws.hdr, done, ws.j0, ws.j1, ws.r0,
                                      ws.r1, status);
  } else {
    k_claim<int32_t><<<g, 256, 0, s>>>((const int32_t*)a, n, ws.d, max_steps, status);
    k_walk<int32_t><<<gw, 256, 0, s>>>((const int32_t*)a, n, ws.d, c, max_steps, ws.hdr, done, ws.j0, ws.j1, ws.r0,
                                      ws.r1, status);
  }
  note_launch(2);
  return cudaGetLastError();
}

// the general permute in two halves, for producers that claim while they
// write the ancestry (the fused Metropolis delivery): reset d (and the
// overflow marker) before the producer, then the walk
cudaError_t launch_claims_reset(int64_t n, int32_t* max_steps, const Workspace& ws, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(&ws.hdr->overflow, 0, sizeof(int32_t), s);
  if (e != cudaSuccess) return e;
  if (max_steps) {
    e = cudaMemsetAsync(max_steps, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
  }
  return cudaMemsetAsync(ws.d, 0x7F, (size_t)n * sizeof(int32_t), s);
}

// ---------------------------------------------------------------------------
// Partitioned permute (a rank's share of permute_parallel, ancestry.py:139-174,
// over the all-gathered ancestry): c[x] for the indices x of [c_begin,
// c_begin + c_count) only.  With the claims d (prepermute over the FULL a),
// x with offspring keeps c[x] = x; a hole x walks the loser chain BACKWARDS:
// slot z is the first claim of its parent exactly when d[a[z]] == z, and then
// the chain came from a[z]; the first z that is not a first claim is the
// loser, and c[x] = a[z] (the chain's length in hops is the reference's
// steps).  Order free, so the union over ranks is the single-GPU result.  A
// chain longer than kRangeBound sets PFR_ST_OVERFLOW (the caller falls back
// to the full permute).
constexpr int kRangeBound = 4096;
__global__ void k_permute_range(const int32_t* __restrict__ a, int64_t n, const int32_t* __restrict__ d,
                                int64_t c_begin, int64_t c_count, int32_t* __restrict__ c, int32_t* max_steps,
                                uint32_t* status) {
  int longest = 0;
  uint32_t f = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < c_count; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = c_begin + t;
    if (__ldg(d + x) < n) {
      c[t] = (int32_t)x;
      continue;
    }
    int64_t z = x;
    int hops = 0;
    int32_t p = __ldg(a + z);
    while (__ldg(d + p) == z) {
      z = p;
      p = __ldg(a + z);
      if (++hops > kRangeBound) {
        f |= PFR_ST_OVERFLOW;
        break;
      }
    }
    c[t] = p;
    longest = max(longest, hops);
  }
  status_or_warp(status, f);
  if (max_steps) {
    longest = __reduce_max_sync(__activemask(), longest);
    if ((threadIdx.x & 31) == 0 && longest) atomicMax(max_steps, longest);
  }
}

cudaError_t launch_permute_range(const int32_t* a, int64_t n, int64_t c_begin, int64_t c_count, int32_t* c,
                                 int32_t* max_steps, uint32_t* status, const Workspace& ws, cudaStream_t s) {
  cudaError_t e = launch_claims_reset(n, max_steps, ws, s);
  if (e != cudaSuccess) return e;
  k_claim<int32_t><<<grid_for(n, 256), 256, 0, s>>>(a, n, ws.d, nullptr, status);
  note_launch();
  if (c_count > 0) {
    k_permute_range<<<grid_for(c_count, 256), 256, 0, s>>>(a, n, ws.d, c_begin, c_count, c, max_steps, status);
    note_launch();
  }
  return cudaGetLastError();
}

cudaError_t launch_walk(const int32_t* a, int64_t n, int32_t* c, int32_t* max_steps, uint32_t* status,
                        const Workspace& ws, cudaStream_t s) {
  const int gw = grid_for((n + 3) / 4, 256);
  unsigned int* done = &ws.dv->pad[0];
  k_walk<int32_t><<<gw, 256, 0, s>>>(a, n, ws.d, c, max_steps, ws.hdr, done, ws.j0, ws.j1, ws.r0, ws.r1, status);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_prepermute(const void* a, int64_t n, int idx_dtype, int32_t* d, uint32_t* status,
                              cudaStream_t s) {
  const int g = grid_for(n, 256);
  k_fill_i32<<<g, 256, 0, s>>>(d, n, (int32_t)n);
  if (idx_dtype == PFR_I64)
    k_claim<int64_t><<<g, 256, 0, s>>>((const int64_t*)a, n, d, nullptr, status);
  else
    k_claim<int32_t><<<g, 256, 0, s>>>((const int32_t*)a, n, d, nullptr, status);
  note_launch(2);
  return cudaGetLastError();
}

cudaError_t launch_expand(const void* O, int64_t n, int idx_dtype, int32_t* a, uint32_t* status, bool validate,
                          cudaStream_t s) {
  const unsigned blocks = (unsigned)((2 * n + kMergeItems - 1) / kMergeItems);
  const int g = grid_for(n, 256);
  if (idx_dtype == PFR_I64) {
    if (validate) k_check_cumulative<int64_t><<<g, 256, 0, s>>>((const int64_t*)O, n, status);
    k_expand<int64_t><<<blocks, kTileThreads, 0, s>>>((const int64_t*)O, n, a);
  } else {
    if (validate) k_check_cumulative<int32_t><<<g, 256, 0, s>>>((const int32_t*)O, n, status);
    k_expand<int32_t><<<blocks, kTileThreads, 0, s>>>((const int32_t*)O, n, a);
  }
  note_launch(validate ? 2 : 1);
  return cudaGetLastError();
}

cudaError_t launch_histogram(const void* a, int64_t n, int idx_dtype, int32_t* o, uint32_t* status, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(o, 0, (size_t)n * sizeof(int32_t), s);
  if (e != cudaSuccess) return e;
  const int g = grid_for(n, 256);
  if (idx_dtype == PFR_I64)
    k_histogram<int64_t><<<g, 256, 0, s>>>((const int64_t*)a, n, o, status);
  else
    k_histogram<int32_t><<<g, 256, 0, s>>>((const int32_t*)a, n, o, status);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_predicate(const void* c, int64_t n, int idx_dtype, int32_t* result, uint32_t* status,
                             const Workspace& ws, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(ws.d, 0, (size_t)n * sizeof(int32_t), s);
  if (e != cudaSuccess) return e;
  const int g = grid_for(n, 256);
  k_set_i32<<<1, 1, 0, s>>>(result, 1);
  if (idx_dtype == PFR_I64) {
    k_mark<int64_t><<<g, 256, 0, s>>>((const int64_t*)c, n, ws.d, status);
    k_predicate<int64_t><<<g, 256, 0, s>>>((const int64_t*)c, n, ws.d, result);
  } else {
    k_mark<int32_t><<<g, 256, 0, s>>>((const int32_t*)c, n, ws.d, status);
    k_predicate<int32_t><<<g, 256, 0, s>>>((const int32_t*)c, n, ws.d, result);
  }
  note_launch(3);
  return cudaGetLastError();
}

cudaError_t launch_copy_particles(double* x, int64_t n, int64_t width, const int32_t* c, cudaStream_t s) {
  const int g = grid_for(n * width, 256);
  k_copy_particles<<<g, 256, 0, s>>>(x, n, width, c);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pfr
