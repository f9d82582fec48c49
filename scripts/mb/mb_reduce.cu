// Microbenchmark: why is the tile-reduce pass slow?  Variants over 2^24 f32.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1301_4019_b200/csrc/pfr_tile.cuh"
using namespace pfr;

__global__ void v_plain(const float4* __restrict__ w, int64_t nv, double* out) {
  // grid-stride, 4 float4 per thread in flight
  double acc = 0;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i + 3 * stride < nv; i += 4 * stride) {
    float4 a = __ldcs(w + i), b = __ldcs(w + i + stride), c = __ldcs(w + i + 2 * stride), d = __ldcs(w + i + 3 * stride);
    acc += (double)a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w + c.x + c.y + c.z + c.w + d.x + d.y + d.z + d.w;
  }
  for (; i < nv; i += stride) { float4 a = __ldcs(w + i); acc += (double)a.x + a.y + a.z + a.w; }
  if (acc == 12345.678) out[0] = acc;
}

template <int MODE>
__global__ void __launch_bounds__(256) v_tile(const float* __restrict__ w, int64_t n, double* agg, unsigned* done) {
  __shared__ __align__(16) uint4 stage[kTile * 4 / 16];
  __shared__ double warp_sums[8];
  const int64_t b = blockIdx.x;
  float x[16];
  if (MODE == 3) {
    // direct striped loads, no smem
    const float4* p = reinterpret_cast<const float4*>(w + b * kTile);
    float4 v[4];
    for (int k = 0; k < 4; ++k) v[k] = __ldcs(p + k * 256 + threadIdx.x);
    double s = 0;
    for (int k = 0; k < 4; ++k) s += (double)v[k].x + v[k].y + v[k].z + v[k].w;
    s = warp_inclusive_scan(s);
    if ((threadIdx.x & 31) == 31) warp_sums[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) { double t = 0; for (int i = 0; i < 8; ++i) t += warp_sums[i]; agg[b] = t; }
    return;
  }
  tile_load<float>(w, n, b * kTile, stage, policy_evict_last(), x);
  TileScan<double> s;
  for (int j = 0; j < 16; ++j) s.loc[j] = (double)x[j];
  if (MODE >= 1) tile_scan<double>(s, warp_sums);
  if (threadIdx.x == 255) {
    agg[b] = MODE >= 1 ? s.thread_excl + s.loc[15] : s.loc[3];
    if (MODE == 2) { __threadfence(); atomicAdd(done, 1u); }
  }
}

int main() {
  const int64_t n = 1 << 24;
  float* w; double* agg; unsigned* done; void* flush;
  cudaMalloc(&w, n * 4); cudaMalloc(&agg, 1 << 20); cudaMalloc(&done, 4); cudaMalloc(&flush, 512 << 20);
  cudaMemset(w, 0, n * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto fn) {
    float best = 1e9;
    for (int r = 0; r < 8; ++r) {
      cudaMemsetAsync(flush, r, 512 << 20);
      cudaEventRecord(e0); fn(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (r > 1 && ms < best) best = ms;
    }
    printf("%-28s %8.2f us  %7.0f GB/s  (%s)\n", name, best * 1e3, n * 4 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run("plain grid-stride x4", [&] { v_plain<<<sms * 8, 256>>>((const float4*)w, n / 4, agg); });
  run("plain grid-stride x4 2048b", [&] { v_plain<<<2048, 512>>>((const float4*)w, n / 4, agg); });
  run("tile load only", [&] { v_tile<0><<<n / kTile, 256>>>(w, n, agg, done); });
  run("tile load+scan", [&] { v_tile<1><<<n / kTile, 256>>>(w, n, agg, done); });
  run("tile load+scan+fence+atomic", [&] { v_tile<2><<<n / kTile, 256>>>(w, n, agg, done); });
  run("tile direct loads no smem", [&] { v_tile<3><<<n / kTile, 256>>>(w, n, agg, done); });
  run("cudaMemcpy D2D 64MB", [&] { cudaMemcpyAsync(flush, w, n * 4, cudaMemcpyDeviceToDevice); });
  return 0;
}
