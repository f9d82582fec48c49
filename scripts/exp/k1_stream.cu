// Experiment: streaming-read rates for K1-shaped work (N floats, 4096-element
// tiles).  A: one tile per CTA, blocked 16 floats per thread (tile_load_any
// pattern); B: same, striped coalesced float4; C: persistent CTAs with a
// 4-stage cp.async.bulk (TMA 1-D) ring into shared memory.
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) kA(const float* __restrict__ w, int64_t n, float* out) {
  const int64_t e0 = (int64_t)blockIdx.x * 4096 + threadIdx.x * 16;
  float s = 0.f;
  const float4* p = reinterpret_cast<const float4*>(w + e0);
#pragma unroll
  for (int q = 0; q < 4; ++q) { float4 v = __ldg(p + q); s += v.x + v.y + v.z + v.w; }
  if (s == 123.f) out[0] = s;
}
__global__ void __launch_bounds__(256) kB(const float* __restrict__ w, int64_t n, float* out) {
  const float4* p = reinterpret_cast<const float4*>(w + (int64_t)blockIdx.x * 4096);
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q) { float4 v = __ldg(p + q * 256 + threadIdx.x); s += v.x + v.y + v.z + v.w; }
  if (s == 123.f) out[0] = s;
}

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(b))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
          (unsigned)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}

template <int S>
__global__ void __launch_bounds__(256) kC(const float* __restrict__ w, int64_t n, float* out) {
  extern __shared__ __align__(128) float buf[];  // S x 4096
  __shared__ uint64_t full[S];
  const int64_t tiles = n / 4096;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int64_t b = blockIdx.x;
  if (threadIdx.x == 0)
    for (int s = 0; s < S; ++s) {
      const int64_t bb = b + (int64_t)s * gridDim.x;
      if (bb < tiles) { mbar_expect(&full[s], 16384); bulk_g2s(buf + s * 4096, w + bb * 4096, 16384, &full[s]); }
    }
  float acc = 0.f;
  for (int i = 0; b < tiles; ++i, b += gridDim.x) {
    const int s = i % S;
    mbar_wait(&full[s], (i / S) & 1);
    const float4* p = reinterpret_cast<const float4*>(buf + s * 4096) + threadIdx.x * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) { float4 v = p[(q + threadIdx.x) & 3]; acc += v.x + v.y + v.z + v.w; }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t bb = b + (int64_t)S * gridDim.x;
      if (bb < tiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect(&full[s], 16384);
        bulk_g2s(buf + s * 4096, w + bb * 4096, 16384, &full[s]);
      }
    }
  }
  if (acc == 123.f) out[0] = acc;
}

extern "C" int run(int which, const float* w, int64_t n, float* out, int grid_mult, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned tiles = (unsigned)(n / 4096);
  if (which == 0) kA<<<tiles, 256, 0, s>>>(w, n, out);
  else if (which == 1) kB<<<tiles, 256, 0, s>>>(w, n, out);
  else {
    int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = 4 * 16384;
    cudaFuncSetAttribute(kC<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kC<4><<<sms * grid_mult, 256, smem, s>>>(w, n, out);
  }
  return (int)cudaGetLastError();
}
