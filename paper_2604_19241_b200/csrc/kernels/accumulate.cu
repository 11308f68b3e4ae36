// bf16 accumulation of sub-batch weight gradients for the non-bitwise (NB) split-batch backward
// (PAPER.md:647-651): acc = bf16_rne(float(acc) + float(add)), the per-op
// rounded two-way split of precision.cpp:98-134 (split_batch_experiment) on real gradients.
// HBM-bound: 6 bytes per element (2 B read acc, 2 B read add, 2 B write), 16 B vectors,
// grid-stride over a 148-multiple grid.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "eplab_b200.h"
#include "../host/errors.hpp"

namespace eplab_dev {

__global__ void __launch_bounds__(256) bf16_accumulate_kernel(uint4* __restrict__ acc, const uint4* __restrict__ add,
                                                              size_t n_vec, __nv_bfloat16* __restrict__ acc_tail,
                                                              const __nv_bfloat16* __restrict__ add_tail, int n_tail) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_vec; i += stride) {
    uint4 a = acc[i];
    const uint4 b = __ldg(add + i);
    __nv_bfloat162* pa = reinterpret_cast<__nv_bfloat162*>(&a);
    const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 fa = __bfloat1622float2(pa[j]), fb = __bfloat1622float2(pb[j]);
      pa[j] = __floats2bfloat162_rn(__fadd_rn(fa.x, fb.x), __fadd_rn(fa.y, fb.y));
    }
    acc[i] = a;
  }
  if (blockIdx.x == 0 && (int)threadIdx.x < n_tail)
    acc_tail[threadIdx.x] = __float2bfloat16_rn(__fadd_rn(__bfloat162float(acc_tail[threadIdx.x]),
                                                          __bfloat162float(add_tail[threadIdx.x])));
}

}  // namespace eplab_dev

extern "C" int eplab_bf16_accumulate(void* d_acc, const void* d_add, size_t n, void* stream) {
  using namespace eplab_dev;
  if ((reinterpret_cast<uintptr_t>(d_acc) | reinterpret_cast<uintptr_t>(d_add)) & 15) {
    eplab_host::set_last_error("eplab_bf16_accumulate: pointers must be 16-byte aligned");
    return EPLAB_ERR_VALIDATION;
  }
  if (n == 0) return EPLAB_OK;
  const size_t n_vec = n / 8;
  const int n_tail = (int)(n % 8);
  int dev = 0, n_sm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  const size_t want = (n_vec + 255) / 256;
  const int grid = (int)(want < (size_t)n_sm * 8 ? (want ? want : 1) : (size_t)n_sm * 8);
  bf16_accumulate_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      static_cast<uint4*>(d_acc), static_cast<const uint4*>(d_add), n_vec,
      static_cast<__nv_bfloat16*>(d_acc) + n_vec * 8, static_cast<const __nv_bfloat16*>(d_add) + n_vec * 8, n_tail);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    eplab_host::set_last_error(std::string("eplab_bf16_accumulate: ") + cudaGetErrorString(e));
    return EPLAB_ERR_INTERNAL;
  }
  return EPLAB_OK;
}
