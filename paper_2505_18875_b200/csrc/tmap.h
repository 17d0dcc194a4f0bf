// tmap.h — host-side TMA tensor-map encoding (cuTensorMapEncodeTiled through the runtime's driver entry point,
// so the library needs no -lcuda) for row-major bf16 matrices [rows, d] with 128-byte swizzle.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace svg2 {

inline PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// box = 64 columns (128 bytes, one swizzle span) x box_rows rows; box_rows = 1 for gather4 maps.
inline bool make_tmap_bf16(CUtensorMap* m, const void* ptr, uint64_t rows, int d, uint32_t box_rows) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  cuuint64_t gdim[2] = {cuuint64_t(d), rows};
  cuuint64_t gstr[1] = {cuuint64_t(d) * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), gdim, gstr, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// [B, H, N, d] bf16 with element strides (sB, sH, sN), d contiguous: a 4-D map {d, N, H, B}, box 64 columns x box_rows
// tokens of one head (the same 128-byte-swizzled smem tile as the 2-D map).  Strides must be multiples of 8 elements.
inline bool make_tmap_bf16_4d(CUtensorMap* m, const void* ptr, int d, int N, int H, int B, long long sN, long long sH,
                              long long sB, uint32_t box_rows) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  cuuint64_t gdim[4] = {cuuint64_t(d), cuuint64_t(N), cuuint64_t(H), cuuint64_t(B)};
  cuuint64_t gstr[3] = {cuuint64_t(sN) * 2, cuuint64_t(sH) * 2, cuuint64_t(sB) * 2};
  cuuint32_t box[4] = {64, box_rows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), gdim, gstr, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 8-bit elements (e4m3 V' of the FP8 PV path): rows of d bytes, boxes of d bytes x box_rows (one 128-byte swizzle
// row per token for d = 128)
inline bool make_tmap_u8(CUtensorMap* m, const void* ptr, uint64_t rows, int d, uint32_t box_rows) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  cuuint64_t gdim[2] = {cuuint64_t(d), rows};
  cuuint64_t gstr[1] = {cuuint64_t(d)};
  cuuint32_t box[2] = {uint32_t(d), box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr), gdim, gstr, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace svg2
