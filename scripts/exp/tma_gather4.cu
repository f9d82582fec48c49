// Experiment: TMA tile::gather4 random-row rate (rows of 16 B = 4 f32) vs the
// LDG sector floor.  Every lane runs its own ring of kS gather4 requests
// (4 random rows each) into shared memory, one mbarrier per slot.
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

constexpr int kWarps = 4, kS = 2;
constexpr int kSlot = 32;  // floats per slot: 128-byte aligned TMA destinations

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
          (unsigned)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, uint64_t* bar, int r0, int r1, int r2,
                                        int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(0), "r"(r0), "r"(r1),
      "r"(r2), "r"(r3)
      : "memory");
}

__global__ void __launch_bounds__(kWarps * 32) kt(const __grid_constant__ CUtensorMap map, int shift, int iters,
                                                  float* sink) {
  __shared__ __align__(128) float buf[kWarps * 32 * kS * kSlot];  // 64 B used per 128-B slot
  __shared__ __align__(8) uint64_t bar[kWarps * 32 * kS];
  const int t = threadIdx.x;
  for (int s = 0; s < kS; ++s) mbar_init(&bar[t * kS + s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  uint32_t st = (blockIdx.x * blockDim.x + t) * 0x9E3779B9u ^ 0x85EBCA6Bu;
  auto rnd = [&]() {
    st = st * 1664525u + 1013904223u;
    return (int)(st >> shift);
  };
  for (int s = 0; s < kS; ++s) {
    mbar_expect(&bar[t * kS + s], 64);
    gather4(&buf[(t * kS + s) * kSlot], &map, &bar[t * kS + s], rnd(), rnd(), rnd(), rnd());
  }
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    for (int s = 0; s < kS; ++s) {
      mbar_wait(&bar[t * kS + s], it & 1);
      acc += buf[(t * kS + s) * kSlot];
      if (it + 1 < iters) {
        mbar_expect(&bar[t * kS + s], 64);
        gather4(&buf[(t * kS + s) * kSlot], &map, &bar[t * kS + s], rnd(), rnd(), rnd(), rnd());
      }
    }
  }
  if (acc == 1234.5f) sink[0] = acc;
}

extern "C" int run(const float* buf, int log2n, long long rows, float* sink, int blocks_per_sm, void* stream) {
  static CUtensorMap map;
  static const float* mb = nullptr;
  if (mb != buf) {
    cuuint64_t dims[2] = {4, (cuuint64_t)1 << (log2n - 2)};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {4, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)buf, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return 1000 + (int)r;
    mb = buf;
  }
  int dev, sms;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = sms * blocks_per_sm;
  const long long per_iter = (long long)grid * kWarps * 32 * kS * 4;  // rows per iteration
  const int iters = (int)(rows / per_iter);
  kt<<<grid, kWarps * 32, 0, (cudaStream_t)stream>>>(map, 32 - (log2n - 2), iters, sink);
  return (int)cudaGetLastError();
}
