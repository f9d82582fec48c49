/* The C ABI from plain C: one fused systematic delivery.
 *   gcc -std=c11 -I include -I /usr/local/cuda/include examples/deliver.c \
 *       -L paper_1301_4019_b200 -lpfr -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,... -o deliver
 *   ./deliver [N]
 * Exit 0 when the ancestry satisfies o[i] > 0 => c[i] = i (ancestry.py:97-101). */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "pfr.h"

#define CK(x)                                                        \
  do {                                                               \
    cudaError_t e_ = (x);                                            \
    if (e_ != cudaSuccess) {                                         \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));       \
      return 2;                                                      \
    }                                                                \
  } while (0)

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : (1 << 20);
  float* w = (float*)malloc(sizeof(float) * n);
  int32_t* c = (int32_t*)malloc(sizeof(int32_t) * n);
  int32_t* o = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  uint64_t s = 88172645463325252ull;
  for (int64_t i = 0; i < n; ++i) { /* xorshift weights in (0, 1] */
    s ^= s << 13, s ^= s >> 7, s ^= s << 17;
    w[i] = (float)((s >> 11) * (1.0 / 9007199254740992.0)) + 1e-6f;
  }
  const size_t ws_bytes = pfr_workspace_bytes(PFR_OP_ANY, n, PFR_F32);
  void *w_dev, *c_dev, *st_dev, *ws_dev;
  CK(cudaMalloc(&w_dev, sizeof(float) * n));
  CK(cudaMalloc(&c_dev, sizeof(int32_t) * n));
  CK(cudaMalloc(&st_dev, 4));
  CK(cudaMalloc(&ws_dev, ws_bytes));
  CK(cudaMemset(ws_dev, 0, ws_bytes)); /* zero-filled once per workspace */
  CK(cudaMemset(st_dev, 0, 4));
  CK(cudaMemcpy(w_dev, w, sizeof(float) * n, cudaMemcpyHostToDevice));
  pfr_rng r = {0x1234u, 0x5678u, PFR_RNG_PHILOX, 0};
  int rc = pfr_deliver_offspring(w_dev, n, PFR_F32, PFR_ACC_F64, /*stratified=*/0, 0.25, NULL, &r, (int32_t*)c_dev,
                                 NULL, NULL, (uint32_t*)st_dev, ws_dev, ws_bytes, NULL);
  if (rc != PFR_OK) {
    fprintf(stderr, "pfr_deliver_offspring: %s\n", pfr_last_error());
    return 1;
  }
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(c, c_dev, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < n; ++i) o[c[i]]++;
  int ok = 1;
  for (int64_t i = 0; i < n; ++i)
    if (o[i] > 0 && c[i] != i) ok = 0;
  printf("N=%lld: in-place predicate %s\n", (long long)n, ok ? "holds" : "FAILS");
  cudaFree(w_dev), cudaFree(c_dev), cudaFree(st_dev), cudaFree(ws_dev);
  free(w), free(c), free(o);
  return ok ? 0 : 1;
}
