// Experiment: random 4-byte gather rate by load path (L2-resident 64 MiB f32
// vector): A ld.global.nc (LDG), B ld.global.nc.L1::no_allocate, C texture
// fetch (tex1Dfetch on a linear texture object), D ld.global.cg (L2 only).
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) kg(const float* __restrict__ buf, cudaTextureObject_t tex, int shift,
                                          int iters, float* sink) {
  uint32_t st[8];
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int q = 0; q < 8; ++q) st[q] = (tid * 8u + q) * 0x9E3779B9u ^ 0x85EBCA6Bu;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      st[q] = st[q] * 1664525u + 1013904223u;
      const uint32_t j = st[q] >> shift;
      if (MODE == 0) v[q] = __ldg(buf + j);
      if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v[q]) : "l"(buf + j));
      if (MODE == 2) v[q] = tex1Dfetch<float>(tex, (int)j);
      if (MODE == 3) v[q] = __ldcg(buf + j);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += v[q];
  }
  if (acc == 1234.5f) sink[0] = acc;
}

extern "C" int run(int mode, const float* buf, int log2n, long long gathers, float* sink, int grid_mult,
                   void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int dev;
  cudaGetDevice(&dev);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = sms * grid_mult;
  const long long threads = (long long)grid * 256;
  const int iters = (int)(gathers / (threads * 8));
  static cudaTextureObject_t tex = 0;
  static const float* tex_buf = nullptr;
  if (mode == 2 && tex_buf != buf) {
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = (void*)buf;
    rd.res.linear.desc = cudaCreateChannelDesc<float>();
    rd.res.linear.sizeInBytes = (size_t)4 << log2n;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    if (cudaCreateTextureObject(&tex, &rd, &td, nullptr) != cudaSuccess) return 99;
    tex_buf = buf;
  }
  const int shift = 32 - log2n;
  switch (mode) {
    case 0: kg<0><<<grid, 256, 0, s>>>(buf, tex, shift, iters, sink); break;
    case 1: kg<1><<<grid, 256, 0, s>>>(buf, tex, shift, iters, sink); break;
    case 2: kg<2><<<grid, 256, 0, s>>>(buf, tex, shift, iters, sink); break;
    default: kg<3><<<grid, 256, 0, s>>>(buf, tex, shift, iters, sink); break;
  }
  return (int)cudaGetLastError();
}
