// Host-side construction of TMA tensor maps (cuTensorMapEncodeTiled through the
// runtime's driver entry point, so the library does not link libcuda directly).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace eplab_host {

inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      throw std::runtime_error("cuTensorMapEncodeTiled entry point unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// Row-major bf16 matrix [rows][cols] (cols contiguous, row pitch `ld` elements);
// box = box_cols (inner) x box_rows; 128B swizzle for operand loads (box_cols = 64),
// 64B swizzle for the 32x32 epilogue store tiles.
inline CUtensorMap make_bf16_map(const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                                 uint32_t box_cols, uint32_t box_rows,
                                 CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                    const_cast<void*>(base), dims, strides, box, estr,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r) +
                             " rows=" + std::to_string(rows) + " cols=" + std::to_string(cols));
  return m;
}

}  // namespace eplab_host

namespace eplab_host {
// 32x32 epilogue store tile map (64B swizzle), see gemm_engine.cuh stage_row.
inline CUtensorMap make_store_map(const void* base, uint64_t rows, uint64_t cols) {
  return make_bf16_map(base, rows, cols, cols, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
}
}  // namespace eplab_host
