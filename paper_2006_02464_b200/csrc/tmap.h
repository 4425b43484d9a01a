// TMA tensor-map construction (host). The driver entry point is resolved
// through the runtime (cudaGetDriverEntryPoint) so libcw.so does not link
// libcuda and still loads on a machine without a GPU.
#pragma once
#include <cuda.h>
#include <cstdint>

namespace cw {

// Resolve cuTensorMapEncodeTiled; returns false when no driver is present.
bool tmap_init();

// [rows][k] bf16 row-major matrix (row stride ld elements, default k), box = 64 (k) x
// box_rows, 128B swizzle. Columns >= k are out of bounds: zero on loads, clipped on stores
// (a channel slice of a concat buffer: base at the slice, k = its width, ld = the stride).
bool make_tmap_2d(CUtensorMap* out, const void* base, uint64_t k, uint64_t rows, uint32_t box_rows,
                  uint64_t ld = 0);

// NHWC bf16 activation tensor of c channels (pixel stride ctot channels, default c), box =
// 64 channels x (box_w*stride) x (box_h*stride) x box_n with element stride `stride` on W
// and H (loads box_w x box_h x box_n pixels).
bool make_tmap_nhwc(CUtensorMap* out, const void* base, uint64_t n, uint64_t h, uint64_t w,
                    uint64_t c, uint32_t box_w, uint32_t box_h, uint32_t box_n, uint32_t stride,
                    uint64_t ctot = 0);

// [rows][cols] fp32 row-major matrix, box = 32 (cols) x box_rows, 128B swizzle.
bool make_tmap_2d_f32(CUtensorMap* out, const void* base, uint64_t cols, uint64_t rows,
                      uint32_t box_rows);

// [rows][k] bf16 row-major matrix, box = 32 (k) x box_rows, 64B swizzle (stem weights).
bool make_tmap_2d_sw64(CUtensorMap* out, const void* base, uint64_t k, uint64_t rows,
                       uint32_t box_rows);

// Whole padded NHWC4 rows for the 7x7/s2 stem: bf16 [n][hp][wp][4] as a 4D map (8 elements =
// 2 pixels, wp / 2, hp, n), box = kMkStemRows full rows of one image, no swizzle (rows land
// contiguous, wp * 8 bytes apart). Rows outside the image are zero-filled.
bool make_tmap_stem_rows(CUtensorMap* out, const void* base, uint64_t n, uint64_t hp, uint64_t wp,
                         uint32_t rows);

}  // namespace cw
