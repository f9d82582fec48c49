// Remaining reference functions around the resampling step.
//
//   k_permute_serial   permute_serial (ancestry.py:104-122, PAPER Code 11):
//                      the serial pairwise-swap algorithm, run by ONE device
//                      thread (inherently sequential; kept for API parity --
//                      permute_parallel is the production permutation).
//   k_stable_*         stable_sum (primitives.py:69-88): balanced pairwise
//                      tree over the zero-padded power-of-two vector.  Aligned
//                      power-of-two blocks are exactly the reference's
//                      subtrees, so the result is bit-identical.
//   k_wstats_*         ESS and resampling MSE (diagnostics.py:54-80), the
//                      quantities the filter and the bench harness evaluate
//                      around each resampling step, in one deterministic pass.
#include <algorithm>

#include "pfr_internal.h"
#include "pfr_tile.cuh"

namespace pfr {

namespace {

template <typename I>
__global__ void k_permute_serial(const I* __restrict__ a, int64_t n, int32_t* __restrict__ c, uint32_t* status) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t v = (int64_t)a[i];
    if (v < 0 || v >= n) {
      status_or(status, PFR_ST_RANGE);
      return;
    }
    c[i] = (int32_t)v;
  }
  int64_t i = 0;
  while (i < n) {
    const int32_t ai = c[i];
    if (ai != i && c[ai] != ai) {
      c[i] = c[ai];  // swap c[i], c[ai]; c[ai] becomes ai
      c[ai] = ai;
    } else {
      ++i;
    }
  }
}

// pairwise level-by-level reduction of 2^k values held as 16 per thread
// (blocked) over a 4096-element aligned block: exactly the balanced tree
template <typename T>
__global__ void __launch_bounds__(256) k_stable_block(const T* __restrict__ in, int64_t n, int64_t m,
                                                       T* __restrict__ out) {
  __shared__ T sh[256];
  const int64_t base = (int64_t)blockIdx.x * kTile;
  T x[kTileItems];
  const int64_t e0 = base + (int64_t)threadIdx.x * kTileItems;
#pragma unroll
  for (int j = 0; j < kTileItems; ++j) x[j] = (e0 + j < n) ? in[e0 + j] : T(0);
  // levels 1..4 inside the thread
#pragma unroll
  for (int w = kTileItems / 2; w >= 1; w >>= 1)
#pragma unroll
    for (int j = 0; j < w; ++j) x[j] = x[2 * j] + x[2 * j + 1];
  // levels 5..12 across threads: pairs (2t, 2t+1)
  sh[threadIdx.x] = x[0];
  __syncthreads();
  for (int w = 128; w >= 1; w >>= 1) {
    T v = T(0);
    if (threadIdx.x < w) v = sh[2 * threadIdx.x] + sh[2 * threadIdx.x + 1];
    __syncthreads();
    if (threadIdx.x < w) sh[threadIdx.x] = v;
    __syncthreads();
  }
  if (threadIdx.x == 0 && (int64_t)blockIdx.x < m) out[blockIdx.x] = sh[0];
}

// final levels over the m block sums (m a power of two): ping-pong between
// v[0, m) and v[m, 2m) so that every level reads the previous one intact
template <typename T>
__global__ void __launch_bounds__(1024) k_stable_top(T* __restrict__ v, int64_t m, void* result) {
  T* src = v;
  T* dst = v + m;
  for (int64_t w = m / 2; w >= 1; w >>= 1) {
    for (int64_t i = threadIdx.x; i < w; i += blockDim.x) dst[i] = src[2 * i] + src[2 * i + 1];
    __syncthreads();
    T* t = src;
    src = dst;
    dst = t;
  }
  if (threadIdx.x == 0) *reinterpret_cast<double*>(result) = (double)src[0];
}

// pass 1: per-block partials of sum w and sum w^2 (float64, fixed order)
template <typename T>
__global__ void __launch_bounds__(256) k_wstats_sums(const T* __restrict__ w, int64_t n, double* __restrict__ part) {
  __shared__ double red[2][8];
  double s0 = 0, s1 = 0;
  const int64_t base = (int64_t)blockIdx.x * kTile;
  for (int64_t i = base + threadIdx.x; i < min(n, base + kTile); i += blockDim.x) {
    const double x = (double)w[i];
    s0 += x;
    s1 += x * x;
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, off);
    s1 += __shfl_xor_sync(0xffffffffu, s1, off);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = s0;
    red[1][threadIdx.x >> 5] = s1;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double t = 0;
    for (int k = 0; k < 8; ++k) t += red[threadIdx.x][k];
    part[2 * blockIdx.x + threadIdx.x] = t;
  }
}

// pass 2: per-block partials of sum (o/N - w/S)^2 with S = out[0]
template <typename T, typename I>
__global__ void __launch_bounds__(256) k_wstats_mse(const T* __restrict__ w, const I* __restrict__ o, int64_t n,
                                                     const double* __restrict__ out, double* __restrict__ part) {
  __shared__ double red[8];
  const double S = out[0], nd = (double)n;
  double s = 0;
  const int64_t base = (int64_t)blockIdx.x * kTile;
  for (int64_t i = base + threadIdx.x; i < min(n, base + kTile); i += blockDim.x) {
    const double d = (double)o[i] / nd - (double)w[i] / S;
    s += d * d;
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int k = 0; k < 8; ++k) t += red[k];
    part[blockIdx.x] = t;
  }
}

// in-order folds: out = {sum w, sum w^2, ESS, MSE}
__global__ void k_wstats_final(const double* __restrict__ part, int64_t blocks, int64_t n, int stage,
                               double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  if (stage == 0) {
    double s0 = 0, s1 = 0;
    for (int64_t b = 0; b < blocks; ++b) {
      s0 += part[2 * b];
      s1 += part[2 * b + 1];
    }
    out[0] = s0;
    out[1] = s1;
    out[2] = s0 * s0 / s1;
    out[3] = 0.0;
  } else {
    double t = 0;
    for (int64_t b = 0; b < blocks; ++b) t += part[b];
    out[3] = t / (double)n;
  }
}

}  // namespace

cudaError_t launch_permute_serial(const void* a, int64_t n, int idx_dtype, int32_t* c, uint32_t* status,
                                  cudaStream_t s) {
  if (idx_dtype == PFR_I64)
    k_permute_serial<int64_t><<<1, 1, 0, s>>>((const int64_t*)a, n, c, status);
  else
    k_permute_serial<int32_t><<<1, 1, 0, s>>>((const int32_t*)a, n, c, status);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_stable_sum(const void* w, int64_t n, int dtype, void* result, void* scratch, cudaStream_t s) {
  // padded size 2^k >= n; blocks of 4096 (or the whole padded vector if smaller)
  int64_t size = 1;
  while (size < n) size <<= 1;
  const int64_t blocks = std::max<int64_t>(1, size / kTile);
  if (size <= kTile) {
    // a single (partial) block: the in-block tree with m = 1 covers 4096 >= size, padding zeros only
    if (dtype == PFR_F64)
      k_stable_block<double><<<1, 256, 0, s>>>((const double*)w, n, 1, (double*)scratch);
    else
      k_stable_block<float><<<1, 256, 0, s>>>((const float*)w, n, 1, (float*)scratch);
  } else if (dtype == PFR_F64) {
    k_stable_block<double><<<(unsigned)blocks, 256, 0, s>>>((const double*)w, n, blocks, (double*)scratch);
  } else {
    k_stable_block<float><<<(unsigned)blocks, 256, 0, s>>>((const float*)w, n, blocks, (float*)scratch);
  }
  if (dtype == PFR_F64)
    k_stable_top<double><<<1, 1024, 0, s>>>((double*)scratch, size <= kTile ? 1 : blocks, result);
  else
    k_stable_top<float><<<1, 1024, 0, s>>>((float*)scratch, size <= kTile ? 1 : blocks, result);
  note_launch(2);
  return cudaGetLastError();
}

cudaError_t launch_weight_stats(const void* w, int64_t n, int dtype, const void* o, int idx_dtype, double* out,
                                void* scratch, cudaStream_t s) {
  const int64_t blocks = num_tiles(n);
  double* part = static_cast<double*>(scratch);
  if (dtype == PFR_F64)
    k_wstats_sums<double><<<(unsigned)blocks, 256, 0, s>>>((const double*)w, n, part);
  else
    k_wstats_sums<float><<<(unsigned)blocks, 256, 0, s>>>((const float*)w, n, part);
  k_wstats_final<<<1, 32, 0, s>>>(part, blocks, n, 0, out);
  note_launch(2);
  if (!o) return cudaGetLastError();
#define PFR_WS_MSE(T, I) \
  k_wstats_mse<T, I><<<(unsigned)blocks, 256, 0, s>>>((const T*)w, (const I*)o, n, out, part)
  if (dtype == PFR_F64) {
    if (idx_dtype == PFR_I64) PFR_WS_MSE(double, int64_t); else PFR_WS_MSE(double, int32_t);
  } else {
    if (idx_dtype == PFR_I64) PFR_WS_MSE(float, int64_t); else PFR_WS_MSE(float, int32_t);
  }
#undef PFR_WS_MSE
  k_wstats_final<<<1, 32, 0, s>>>(part, blocks, n, 1, out);
  note_launch(2);
  return cudaGetLastError();
}

// Random-gather probe (measurement only): every thread walks 8 independent
// LCG streams and gathers buf[index] for each (the top log2 n bits of the
// state: uniform over a power-of-two n), XOR-folding the loaded words so the
// loads stay live.  Two integer ops per gather: bound by the memory system
// (L2 sectors when buf is L2 resident, HBM sectors otherwise) -- the floor
// the Metropolis and rejection gathers are compared with.
template <typename U>
__global__ void __launch_bounds__(256) k_probe_gather(const U* __restrict__ buf, int shift, int iters,
                                                      unsigned long long* sink) {
  uint32_t st[8];
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int q = 0; q < 8; ++q) st[q] = (tid * 8u + q) * 0x9E3779B9u ^ 0x85EBCA6Bu;
  U acc = 0;
  for (int it = 0; it < iters; ++it) {
    U v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      st[q] = st[q] * 1664525u + 1013904223u;
      v[q] = __ldg(buf + (shift >= 32 ? 0u : (st[q] >> shift)));
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) acc ^= v[q];
  }
  if (acc == (U)0x5EED5EEDu) atomicAdd(sink, 1ull);
}

cudaError_t launch_probe_gather(const void* buf, int64_t n, int elem_bytes, int64_t gathers, unsigned long long* sink,
                                cudaStream_t s) {
  int L = 0;
  while ((int64_t(1) << L) < n) ++L;
  const unsigned grid = (unsigned)num_sms() * 8;
  const int64_t threads = (int64_t)grid * 256;
  const int iters = (int)std::max<int64_t>(1, gathers / (threads * 8));
  if (elem_bytes == 8)
    k_probe_gather<unsigned long long><<<grid, 256, 0, s>>>((const unsigned long long*)buf, 32 - L, iters, sink);
  else
    k_probe_gather<uint32_t><<<grid, 256, 0, s>>>((const uint32_t*)buf, 32 - L, iters, sink);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pfr
