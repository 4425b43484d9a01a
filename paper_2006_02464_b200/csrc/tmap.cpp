#include "tmap.h"
#include <cuda_runtime.h>
#include <mutex>

namespace cw {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn g_encode = nullptr;
static std::once_flag g_once;

bool tmap_init() {
  std::call_once(g_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<EncodeTiledFn>(fn);
  });
  return g_encode != nullptr;
}

bool make_tmap_2d(CUtensorMap* out, const void* base, uint64_t k, uint64_t rows,
                  uint32_t box_rows, uint64_t ld) {
  if (!tmap_init()) return false;
  cuuint64_t dims[2] = {k, rows};
  cuuint64_t strides[1] = {(ld ? ld : k) * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return g_encode(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tmap_nhwc(CUtensorMap* out, const void* base, uint64_t n, uint64_t h, uint64_t w,
                    uint64_t c, uint32_t box_w, uint32_t box_h, uint32_t box_n, uint32_t stride,
                    uint64_t ctot) {
  if (!tmap_init()) return false;
  const uint64_t ct = ctot ? ctot : c;
  cuuint64_t dims[4] = {c, w, h, n};
  cuuint64_t strides[3] = {ct * 2, w * ct * 2, h * w * ct * 2};
  cuuint32_t box[4] = {64, box_w * stride, box_h * stride, box_n};
  cuuint32_t estr[4] = {1, stride, stride, 1};
  return g_encode(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tmap_2d_f32(CUtensorMap* out, const void* base, uint64_t cols, uint64_t rows,
                      uint32_t box_rows) {
  if (!tmap_init()) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return g_encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tmap_2d_sw64(CUtensorMap* out, const void* base, uint64_t k, uint64_t rows,
                       uint32_t box_rows) {
  if (!tmap_init()) return false;
  cuuint64_t dims[2] = {k, rows};
  cuuint64_t strides[1] = {k * 2};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return g_encode(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Whole padded NHWC4 rows (stem): dims (8, wp / 2, hp, n) with strides (16 B, row, image).
bool make_tmap_stem_rows(CUtensorMap* out, const void* base, uint64_t n, uint64_t hp, uint64_t wp,
                         uint32_t rows) {
  if (!tmap_init() || wp % 2 || wp / 2 > 256) return false;
  const uint64_t row = wp * 8;
  cuuint64_t dims[4] = {8, wp / 2, hp, n};
  cuuint64_t strides[3] = {16, row, hp * row};
  cuuint32_t box[4] = {8, (cuuint32_t)(wp / 2), rows, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return g_encode(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace cw
