// Host-side TMA tensor-map construction and caching (cuTensorMapEncodeTiled through the
// runtime's driver entry point, so the library does not link libcuda directly).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace compar {

// Shared-memory swizzle of a TMA box (must match the UMMA descriptor layout type / the
// consumer's address arithmetic).
enum class Swz : int {
    None = CU_TENSOR_MAP_SWIZZLE_NONE,
    B128 = CU_TENSOR_MAP_SWIZZLE_128B,              // 16-byte chunks XOR (row & 7), 1024-byte atom
    B128_32B = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B  // 32-byte chunks within a 128-byte span
};

// 2-D row-major tensor: `rows` x `cols` elements, row pitch `ld` elements of `elem_bytes`.
// Box = box_rows x box_cols elements.  Out-of-bounds box elements are zero-filled by the
// hardware.  Returns false on failure.
bool make_tmap_2d(CUtensorMap *out, const void *base, int elem_bytes, int64_t rows, int64_t cols, int64_t ld,
                  uint32_t box_rows, uint32_t box_cols, Swz swizzle);

// 3-D tensor {cols, rows, planes}: row pitch `ld` elements, plane pitch `plane` elements; box
// box_cols x box_rows x 1.  (World-mode slab-packed B: plane j = slab j, a K x slab_w block.)
bool make_tmap_3d(CUtensorMap *out, const void *base, int elem_bytes, int64_t planes, int64_t rows, int64_t cols,
                  int64_t ld, int64_t plane, uint32_t box_rows, uint32_t box_cols, Swz swizzle);

// Cached wrapper: tensor maps are keyed by (ptr, shape, ld, box, swizzle) so repeated
// submissions on the same buffers skip the host-side encode (SURVEY §7 hard part 4).
bool get_tmap_2d(CUtensorMap *out, const void *ptr, int elem_bytes, int64_t rows, int64_t cols, int64_t ld,
                 uint32_t box_rows, uint32_t box_cols, Swz swizzle);

}  // namespace compar
