// Tile machinery shared by the scan, offspring and delivery kernels.
//
// A tile is 4096 consecutive elements handled by one 256-thread CTA, 16
// consecutive elements per thread ("blocked").  Global memory is read and
// written with fully coalesced 16-byte vectors (striped) and transposed
// through an XOR-swizzled shared-memory buffer, so HBM sees one pass of
// 128-byte lines.
//
// Carries between tiles use a DETERMINISTIC lookback tree instead of the
// classic decoupled lookback: every tile publishes its aggregate as leaf
// (0, b); the tile that completes a node (l, m) (its rightmost leaf) combines
// left + right child; tile b's exclusive prefix is the left-to-right sum of the
// maximal aligned nodes covering [0, b).  Every floating-point association is
// fixed by the tile index alone, so results are bit-identical from run to run
// and across launch geometries, while tiles still only wait on earlier tiles
// (single pass, no grid barrier).  A second tree of exact integer/float
// maxima repairs ulp-level non-monotonicity (running max) the same way.
#pragma once

#include "pfr_common.cuh"

namespace pfr {

constexpr int kTileThreads = 256;
constexpr int kTileItems = 16;
constexpr int kTile = kTileThreads * kTileItems;  // 4096

__host__ __device__ __forceinline__ int64_t num_tiles(int64_t n) { return (n + kTile - 1) / kTile; }

// ---------------------------------------------------------------------------
// lookback tree layout: level l holds ceil(T / 2^l) cells.
struct Tree {
  uint64_t* cells;
  int64_t tiles;
  int levels;  // number of levels (>= 1)

  __host__ __device__ static int64_t cells_needed(int64_t tiles) {
    int64_t total = 0, cnt = tiles;
    while (true) {
      total += cnt;
      if (cnt <= 1) break;
      cnt = (cnt + 1) / 2;
    }
    return total;
  }
  __host__ __device__ int64_t offset(int l) const {
    int64_t off = 0, cnt = tiles;
    for (int i = 0; i < l; ++i) {
      off += cnt;
      cnt = (cnt + 1) / 2;
    }
    return off;
  }
  __device__ uint64_t* cell(int l, int64_t m) const { return cells + offset(l) + m; }
};

__host__ __device__ inline int tree_levels(int64_t tiles) {
  int l = 1;
  int64_t cnt = tiles;
  while (cnt > 1) {
    cnt = (cnt + 1) / 2;
    ++l;
  }
  return l;
}

struct SumOp {
  template <typename A>
  __device__ static A combine(A left, A right) {
    return add_rn(left, right);
  }
};
struct MaxOp {
  __device__ static double combine(double a, double b) { return fmax(a, b); }
  __device__ static float combine(float a, float b) { return fmaxf(a, b); }
  __device__ static int64_t combine(int64_t a, int64_t b) { return a > b ? a : b; }
  __device__ static int combine(int a, int b) { return a > b ? a : b; }
};

// Publish leaf (0, b) = v and complete every node whose rightmost leaf is b.
// Called by ONE thread.
template <typename A, typename Op>
__device__ void tree_publish(const Tree& t, int64_t b, A v) {
  st_relaxed_u64(t.cell(0, b), Cell<A>::encode(v));
  int64_t m = b;
  int l = 0;
  while ((m & 1) && l + 1 < t.levels) {
    A left = cell_wait<A>(t.cell(l, m - 1));
    v = Op::combine(left, v);
    ++l;
    m >>= 1;
    st_relaxed_u64(t.cell(l, m), Cell<A>::encode(v));
  }
}

// Exclusive combination of leaves [0, b) in fixed left-to-right node order.
// Executed by one full warp; returns the value in every lane.  `identity` is
// the neutral element (0 for sums, -inf / INT64_MIN for max).
template <typename A, typename Op>
__device__ A tree_prefix(const Tree& t, int64_t b, A identity) {
  const int lane = threadIdx.x & 31;
  // lane l handles level l (levels <= 32 for any n < 2^43)
  A mine = identity;
  bool have = false;
  int64_t start = 0;
  if (lane < t.levels && ((b >> lane) & 1)) {
    // nodes at higher levels come first: start of this node = b with bits < = lane cleared
    start = (b >> (lane + 1)) << (lane + 1);
    mine = cell_wait<A>(t.cell(lane, start >> lane));
    have = true;
  }
  // combine from the highest level down (left to right along the prefix)
  A acc = identity;
  bool first = true;
  for (int l = 31; l >= 0; --l) {
    A v = __shfl_sync(0xffffffffu, mine, l);
    bool h = __shfl_sync(0xffffffffu, have, l);
    if (h) {
      acc = first ? v : Op::combine(acc, v);
      first = false;
    }
  }
  return acc;
}

// ---------------------------------------------------------------------------
// shared-memory staging with an XOR swizzle on 16-byte slots:
// slot(v) = v ^ ((v >> 3) & 7) makes both the striped (consecutive v) and the
// blocked (v = k*t + j, k = 4 or 8) access patterns bank-conflict free.
__device__ __forceinline__ int swz(int v) { return v ^ ((v >> 3) & 7); }

// Load a tile of T into per-thread blocked registers x[16] (zero padded).
template <typename T>
__device__ __forceinline__ void tile_load(const T* __restrict__ in, int64_t n, int64_t base, uint4* smem,
                                          uint64_t pol, T (&x)[kTileItems]) {
  constexpr int kPerVec = 16 / sizeof(T);
  constexpr int kVecs = kTile / kPerVec;
  const int tid = threadIdx.x;
  const int64_t remain = n - base;
  if (remain >= kTile) {
    // issue every load of the tile before the first shared-memory store
    uint4 buf[kVecs / kTileThreads];
#pragma unroll
    for (int k = 0; k < kVecs / kTileThreads; ++k)
      buf[k] = ld_stream16(in + base + (int64_t)(k * kTileThreads + tid) * kPerVec, pol);
#pragma unroll
    for (int k = 0; k < kVecs / kTileThreads; ++k) smem[swz(k * kTileThreads + tid)] = buf[k];
  } else {
#pragma unroll
    for (int k = 0; k < kVecs / kTileThreads; ++k) {
      const int v = k * kTileThreads + tid;
      const int64_t e0 = (int64_t)v * kPerVec;
      if (e0 + kPerVec <= remain) {
        smem[swz(v)] = ld_stream16(in + base + e0, pol);
      } else {
        union {
          uint4 u;
          T e[kPerVec];
        } tmp;
#pragma unroll
        for (int j = 0; j < kPerVec; ++j) tmp.e[j] = (e0 + j < remain) ? in[base + e0 + j] : T(0);
        smem[swz(v)] = tmp.u;
      }
    }
  }
  __syncthreads();
  constexpr int kMyVecs = kTileItems / kPerVec;
#pragma unroll
  for (int j = 0; j < kMyVecs; ++j) {
    union {
      uint4 u;
      T e[kPerVec];
    } tmp;
    tmp.u = smem[swz(tid * kMyVecs + j)];
#pragma unroll
    for (int e = 0; e < kPerVec; ++e) x[j * kPerVec + e] = tmp.e[e];
  }
  __syncthreads();
}

// Blocked direct loads: thread t gets elements [16t, 16t + 16) of the tile
// through L1-allocating 16-byte loads (the 4-8 loads of a thread cover whole
// lines), zero padded past n.  No shared memory, no barrier.
template <typename T>
__device__ __forceinline__ void tile_load_any(const T* __restrict__ in, int64_t n, int64_t base, T (&x)[kTileItems]) {
  constexpr int kPerVec = 16 / sizeof(T);
  const int64_t e0 = base + (int64_t)threadIdx.x * kTileItems;
  if (e0 + kTileItems <= n && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
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

// Store per-thread blocked registers y[16] of U to out[base ...] (clipped at n).
template <typename U>
__device__ __forceinline__ void tile_store(U* __restrict__ out, int64_t n, int64_t base, uint4* smem,
                                           const U (&y)[kTileItems], uint64_t pol) {
  constexpr int kPerVec = 16 / sizeof(U);
  constexpr int kVecs = kTile / kPerVec;
  constexpr int kMyVecs = kTileItems / kPerVec;
  const int tid = threadIdx.x;
#pragma unroll
  for (int j = 0; j < kMyVecs; ++j) {
    union {
      uint4 u;
      U e[kPerVec];
    } tmp;
#pragma unroll
    for (int e = 0; e < kPerVec; ++e) tmp.e[e] = y[j * kPerVec + e];
    smem[swz(tid * kMyVecs + j)] = tmp.u;
  }
  __syncthreads();
  const int64_t remain = n - base;
#pragma unroll
  for (int k = 0; k < kVecs / kTileThreads; ++k) {
    const int v = k * kTileThreads + tid;
    const int64_t e0 = (int64_t)v * kPerVec;
    uint4 val = smem[swz(v)];
    if (e0 + kPerVec <= remain) {
      st_hint16(out + base + e0, val, pol);
    } else if (e0 < remain) {
      union {
        uint4 u;
        U e[kPerVec];
      } tmp;
      tmp.u = val;
      for (int j = 0; j < kPerVec && e0 + j < remain; ++j) out[base + e0 + j] = tmp.e[j];
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// In-tile scan.  Produces, per thread, the serial partials loc[j] (in A) and
// the thread's exclusive offset within the tile, plus the tile aggregate.
//   value(t, j) = (tile_prefix + thread_excl(t)) + loc[j]
// association: thread-serial partials; Kogge-Stone over the 32 thread totals
// of a warp; serial over the 8 warp totals.
template <typename A>
struct TileScan {
  A loc[kTileItems];
  A thread_excl;  // sum of everything before this thread inside the tile
  A tile_total;   // aggregate of the whole tile
};

template <typename A>
__device__ __forceinline__ void tile_scan(TileScan<A>& s, A* warp_sums /* smem [8] */) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 1; j < kTileItems; ++j) s.loc[j] = add_rn(s.loc[j - 1], s.loc[j]);
  const A mine = s.loc[kTileItems - 1];
  const A incl = warp_inclusive_scan(mine);
  A excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = A(0);
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  A wp = A(0);
  A total = A(0);
#pragma unroll
  for (int w = 0; w < kTileThreads / 32; ++w) {
    const A ws = warp_sums[w];
    if (w < warp) wp = add_rn(wp, ws);
    total = add_rn(total, ws);
  }
  s.thread_excl = (lane == 0) ? wp : add_rn(wp, excl);
  s.tile_total = total;
  __syncthreads();
}

// Block-wide exclusive max over per-thread values (exact, order free).
template <typename A>
__device__ __forceinline__ A block_excl_max(A v, A identity, A* smem8, A& block_max) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  A incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    A o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl = MaxOp::combine(incl, o);
  }
  A excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = identity;
  if (lane == 31) smem8[warp] = incl;
  __syncthreads();
  A wp = identity, tot = identity;
#pragma unroll
  for (int w = 0; w < kTileThreads / 32; ++w) {
    const A x = smem8[w];
    if (w < warp) wp = MaxOp::combine(wp, x);
    tot = MaxOp::combine(tot, x);
  }
  __syncthreads();
  block_max = tot;
  return MaxOp::combine(wp, excl);
}

// Ticketed tile index: tiles are processed in increasing order of
// acquisition, so waiting only on smaller tiles can never deadlock.
__device__ __forceinline__ int64_t acquire_tile(unsigned int* ticket, int* smem_slot) {
  // the workspace reset leaves tickets at 0xFFFFFFFF: the first ticket is 0
  if (threadIdx.x == 0) *smem_slot = (int)(atomicAdd(ticket, 1u) + 1u);
  __syncthreads();
  const int64_t b = *smem_slot;
  __syncthreads();
  return b;
}

}  // namespace pfr
