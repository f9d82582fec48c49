// Weight-sharded single filter: the per-rank kernels.
//
// One very large filter is split into contiguous weight shards, one per GPU.
// The host protocol (paper_1301_4019_b200/sharded.py) all-gathers the shard
// totals, so each rank knows the weight before its shard (`prefix`) and the
// global total; every rank then computes the cumulative offspring of its own
// parents with the reference formula (resamplers.py:139-153) in GLOBAL slot
// numbers, expands them into slot words over its slot window, exchanges the
// words with the ranks that own those indices, and resolves the in-place
// ancestry of its indices (ancestry.py:139-174, read backwards from each
// hole as in pfr_deliver.cu).  Loser chains that leave the shard become
// walkers (hole, slot, steps) that the host routes to the owner of `slot`.
//
// All kernels here are simple one-pass streaming kernels; the words window is
// the only per-element intermediate.
#include "pfr_internal.h"
#include "pfr_tile.cuh"

namespace pfr {

namespace {

constexpr uint32_t kFirst = 0x80000000u;
constexpr uint32_t kParentMask = 0x7FFFFFFFu;

struct ShardU {
  int stratified;
  double u_sys;           // systematic offset, already cast to the weight dtype
  const double* uniforms; // stratified, caller-supplied (global stratum index)
  int mode;               // PFR_RNG_*
  Key2x64 key;
  int f32;                // weight dtype float32: per-stratum u cast to float first
};

__device__ __forceinline__ double stratum_u_global(const ShardU& U, int64_t k0) {
  if (!U.stratified) return U.u_sys;
  double u;
  if (U.uniforms) {
    u = U.uniforms[k0];
  } else if (U.mode == PFR_RNG_NUMPY) {
    u = u64_to_unit(numpy_raw64(U.key, (uint64_t)k0));
  } else {
    uint32_t o[4];
    philox4x32_10((uint32_t)(k0 >> 2), (uint32_t)(k0 >> 34), kTagStratified, 0, (uint32_t)U.key.k0,
                  (uint32_t)(U.key.k0 >> 32), o);
    u = u32_to_unit_d(o[k0 & 3]);
  }
  return U.f32 ? (double)__double2float_rn(u) : u;
}

// O[i] = min(N, floor((W*N)/total + u[k-1])), k = min(N, floor(r)+1), with
// W = prefix + W_loc[i] (the IEEE sequence of resamplers.py:143-147)
__global__ void k_shard_offspring(const double* __restrict__ W_loc, int64_t n_loc, double prefix, double total,
                                  int64_t n_global, int last_global, ShardU U, int32_t* __restrict__ O) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_loc; i += stride) {
    const double W = __dadd_rn(prefix, W_loc[i]);
    const double r = __ddiv_rn(__dmul_rn(W, (double)n_global), total);
    int64_t k = (int64_t)floor(r) + 1;
    if (k > n_global) k = n_global;
    if (k < 1) k = 1;
    int64_t o = (int64_t)floor(__dadd_rn(r, stratum_u_global(U, k - 1)));
    if (o > n_global) o = n_global;
    if (o < 0) o = 0;
    if (last_global && i == n_loc - 1) o = n_global;  // O[N-1] = N (resamplers.py:151)
    O[i] = (int32_t)o;
  }
}

// slot words over [o_begin, O[n_loc-1]): parent | FIRST on a parent's first slot
__global__ void k_shard_words(const int32_t* __restrict__ O, int64_t n_loc, int64_t index_base, int32_t o_begin,
                              uint32_t* __restrict__ words, uint8_t* __restrict__ has, uint32_t* status) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  uint32_t f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_loc; i += stride) {
    const int32_t lo = i ? O[i - 1] : o_begin;
    const int32_t hi = O[i];
    if (hi < lo) {
      f |= PFR_ST_NOTMONOTONE;
      if (has) has[i] = 0;
      continue;
    }
    if (has) has[i] = hi > lo;
    const uint32_t p = (uint32_t)(index_base + i);
    for (int32_t s = lo; s < hi; ++s) words[s - o_begin] = p | (s == lo ? kFirst : 0u);
  }
  status_or_warp(status, f);
}

// Backward chain walk from hole h inside the shard; returns true when resolved
// (value in *out), false when the chain leaves [base, base+n) at slot *z.
__device__ __forceinline__ bool walk_local(uint32_t wd, const uint32_t* __restrict__ words, int64_t base, int64_t n,
                                           int32_t* out, int64_t* z, int* steps) {
  int st = *steps;
  while (wd & kFirst) {
    const int64_t y = (int64_t)(wd & kParentMask);
    ++st;
    if (y < base || y >= base + n) {
      *z = y;
      *steps = st;
      return false;
    }
    if (st > n + 1) {  // cannot happen for a valid ancestry
      *z = -1;
      *steps = st;
      return false;
    }
    wd = __ldg(words + (y - base));
  }
  *out = (int32_t)(wd & kParentMask);
  *steps = st;
  return true;
}

__global__ void k_shard_resolve(const uint32_t* __restrict__ words, const uint8_t* __restrict__ has, int64_t n_loc,
                                int64_t index_base, int32_t* __restrict__ c, int32_t* __restrict__ pend,
                                int32_t* pend_count, int32_t* max_steps, uint32_t* status) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int longest = 0;
  uint32_t f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_loc; i += stride) {
    const int64_t x = index_base + i;
    if (has[i]) {
      c[i] = (int32_t)x;
      continue;
    }
    int32_t v;
    int64_t z;
    int st = 0;
    if (walk_local(words[i], words, index_base, n_loc, &v, &z, &st)) {
      c[i] = v;
      longest = max(longest, st);
    } else if (z < 0) {
      f |= PFR_ST_NONTERMINATION;
    } else {
      const int slot = atomicAdd(pend_count, 1);
      pend[3 * slot] = (int32_t)x;
      pend[3 * slot + 1] = (int32_t)z;
      pend[3 * slot + 2] = st;
    }
  }
  status_or_warp(status, f);
  if (max_steps) {
    longest = __reduce_max_sync(__activemask(), longest);
    if ((threadIdx.x & 31) == 0 && longest) atomicMax(max_steps, longest);
  }
}

// routed walkers (hole, slot, steps) with slot in this shard
__global__ void k_shard_advance(const int32_t* __restrict__ walkers, int64_t count, const uint32_t* __restrict__ words,
                                int64_t n_loc, int64_t index_base, int32_t* __restrict__ done, int32_t* done_count,
                                int32_t* __restrict__ fwd, int32_t* fwd_count, int32_t* max_steps, uint32_t* status) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  uint32_t f = 0;
  int longest = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += stride) {
    const int32_t h = walkers[3 * t];
    const int64_t z0 = walkers[3 * t + 1];
    int st = walkers[3 * t + 2];
    if (z0 < index_base || z0 >= index_base + n_loc) {
      f |= PFR_ST_RANGE;
      continue;
    }
    int32_t v;
    int64_t z;
    if (walk_local(__ldg(words + (z0 - index_base)), words, index_base, n_loc, &v, &z, &st)) {
      const int k = atomicAdd(done_count, 1);
      done[2 * k] = h;
      done[2 * k + 1] = v;
      longest = max(longest, st);
    } else if (z < 0) {
      f |= PFR_ST_NONTERMINATION;
    } else {
      const int k = atomicAdd(fwd_count, 1);
      fwd[3 * k] = h;
      fwd[3 * k + 1] = (int32_t)z;
      fwd[3 * k + 2] = st;
    }
  }
  status_or_warp(status, f);
  if (max_steps) {
    longest = __reduce_max_sync(__activemask(), longest);
    if ((threadIdx.x & 31) == 0 && longest) atomicMax(max_steps, longest);
  }
}

__global__ void k_shard_scatter(const int32_t* __restrict__ done, int64_t count, int64_t index_base, int64_t n_loc,
                                int32_t* __restrict__ c, uint32_t* status) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  uint32_t f = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += stride) {
    const int64_t h = done[2 * t] - index_base;
    if (h < 0 || h >= n_loc) {
      f |= PFR_ST_RANGE;
      continue;
    }
    c[h] = done[2 * t + 1];
  }
  status_or_warp(status, f);
}

// ---------------------------------------------------------------------------
// Boundary bands of the sharded protocol (sharded.py): a rank's slot words
// live in an EXTENDED array covering slots [base - H, base + n_loc + H)
// (sentinel 0xFFFFFFFF where no word was written); the neighbours' windows
// reach it through their boundary bands.
constexpr uint32_t kSentinel = 0xFFFFFFFFu;  // FIRST | parent 2^31-1: no word has it (N < 2^31 - 1)

// fill the sentinel positions of ext from the neighbours' boundary bands:
// from_left = the left neighbour's ext[n, n + 2H) (slots [base - H, base + H)),
// from_right = the right neighbour's ext[0, 2H) (slots [base + n - H, base + n + H));
// null at the ends of the rank order
__global__ void k_shard_merge(uint32_t* __restrict__ ext, int64_t n_loc, int64_t H,
                              const uint32_t* __restrict__ from_left, const uint32_t* __restrict__ from_right) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < 2 * H; q += stride) {
    if (from_left) {
      const uint32_t v = from_left[q];
      if (v != kSentinel && ext[q] == kSentinel) ext[q] = v;
    }
    if (from_right) {
      const uint32_t v = from_right[q];
      if (v != kSentinel && ext[n_loc + q] == kSentinel) ext[n_loc + q] = v;
    }
  }
}

int grid_for_n(int64_t n) {
  const int64_t g = (n + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

cudaError_t launch_shard_offspring(const double* W_loc, int64_t n_loc, int dtype, double prefix, double total,
                                   int64_t n_global, int last_global, int stratified, double offset,
                                   const double* uniforms, const pfr_rng* rng, int32_t* O, cudaStream_t s) {
  ShardU U;
  U.stratified = stratified;
  U.f32 = dtype == PFR_F32;
  U.u_sys = U.f32 ? (double)(float)offset : offset;
  U.uniforms = uniforms;
  U.mode = rng ? rng->mode : PFR_RNG_ARRAYS;
  U.key = Key2x64{rng ? rng->key0 : 0, rng ? rng->key1 : 0};
  k_shard_offspring<<<grid_for_n(n_loc), 256, 0, s>>>(W_loc, n_loc, prefix, total, n_global, last_global, U, O);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_shard_words(const int32_t* O, int64_t n_loc, int64_t index_base, int32_t o_begin, uint32_t* words,
                               uint8_t* has, uint32_t* status, cudaStream_t s) {
  k_shard_words<<<grid_for_n(n_loc), 256, 0, s>>>(O, n_loc, index_base, o_begin, words, has, status);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_shard_resolve(const uint32_t* words, const uint8_t* has, int64_t n_loc, int64_t index_base,
                                 int32_t* c, int32_t* pend, int32_t* pend_count, int32_t* max_steps, uint32_t* status,
                                 cudaStream_t s) {
  k_shard_resolve<<<grid_for_n(n_loc), 256, 0, s>>>(words, has, n_loc, index_base, c, pend, pend_count, max_steps,
                                                    status);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_shard_advance(const int32_t* walkers, int64_t count, const uint32_t* words, int64_t n_loc,
                                 int64_t index_base, int32_t* done, int32_t* done_count, int32_t* fwd,
                                 int32_t* fwd_count, int32_t* max_steps, uint32_t* status, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  k_shard_advance<<<grid_for_n(count), 256, 0, s>>>(walkers, count, words, n_loc, index_base, done, done_count, fwd,
                                                    fwd_count, max_steps, status);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_shard_scatter(const int32_t* done, int64_t count, int64_t index_base, int64_t n_loc, int32_t* c,
                                 uint32_t* status, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  k_shard_scatter<<<grid_for_n(count), 256, 0, s>>>(done, count, index_base, n_loc, c, status);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_shard_merge(uint32_t* ext, int64_t n_loc, int64_t H, const uint32_t* from_left,
                               const uint32_t* from_right, cudaStream_t s) {
  k_shard_merge<<<grid_for_n(2 * H), 256, 0, s>>>(ext, n_loc, H, from_left, from_right);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pfr
