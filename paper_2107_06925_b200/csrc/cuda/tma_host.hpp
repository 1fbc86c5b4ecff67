// Host-side TMA tensor-map construction (cuTensorMapEncodeTiled via the runtime's
// driver entry point, so the library does not link libcuda directly).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>

#include "capi_util.hpp"

namespace chimera::cuda {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      throw chimera::capi::InternalError("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D bf16 tensor: `inner` contiguous elements per row, `outer` rows `row_stride`
// elements apart; box = {box_inner, box_outer}; 128-byte swizzle (box_inner = 64) unless given.
inline CUtensorMap make_map_2d_bf16(const void* base, uint64_t inner, uint64_t outer,
                                    uint64_t row_stride, uint32_t box_inner, uint32_t box_outer,
                                    CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_stride * 2};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                                 strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw chimera::capi::InternalError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) +
                                       ") inner=" + std::to_string(inner) + " outer=" +
                                       std::to_string(outer) + " stride=" + std::to_string(row_stride));
  return m;
}

// 2-D fp32 tensor, 128-byte swizzle: box_inner * 4 must be <= 128 (box_inner = 32).
inline CUtensorMap make_map_2d_f32(const void* base, uint64_t inner, uint64_t outer, uint64_t row_stride,
                                   uint32_t box_inner, uint32_t box_outer) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_stride * 4};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw chimera::capi::InternalError("cuTensorMapEncodeTiled(f32) failed (" + std::to_string(int(r)) + ")");
  return m;
}

}  // namespace chimera::cuda
