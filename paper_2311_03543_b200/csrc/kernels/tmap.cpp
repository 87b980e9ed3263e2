#include "tmap.h"

#include <cudaTypedefs.h>

#include <mutex>
#include <unordered_map>

namespace compar {

namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_once;

void resolve() {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}
}  // namespace

bool make_tmap_2d(CUtensorMap *out, const void *base, int elem_bytes, int64_t rows, int64_t cols, int64_t ld,
                  uint32_t box_rows, uint32_t box_cols, Swz swizzle) {
    std::call_once(g_once, resolve);
    if (!g_encode) return false;
    // FP32 operands of the TF32 variant are moved as raw FP32 bits; the tensor core reads
    // them as TF32 (low mantissa bits ignored, R6).
    const CUtensorMapDataType dt = elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * static_cast<cuuint64_t>(elem_bytes)};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode(out, dt, 2, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          static_cast<CUtensorMapSwizzle>(static_cast<int>(swizzle)),
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_tmap_3d(CUtensorMap *out, const void *base, int elem_bytes, int64_t planes, int64_t rows, int64_t cols,
                  int64_t ld, int64_t plane, uint32_t box_rows, uint32_t box_cols, Swz swizzle) {
    std::call_once(g_once, resolve);
    if (!g_encode) return false;
    const CUtensorMapDataType dt = elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(planes)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * static_cast<cuuint64_t>(elem_bytes),
                             static_cast<cuuint64_t>(plane) * static_cast<cuuint64_t>(elem_bytes)};
    cuuint32_t box[3] = {box_cols, box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = g_encode(out, dt, 3, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          static_cast<CUtensorMapSwizzle>(static_cast<int>(swizzle)),
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

namespace {
struct MapKey {
    const void *ptr;
    int64_t rows, cols, ld;
    uint32_t br, bc;
    int elem, sw;
    bool operator==(const MapKey &o) const {
        return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld && br == o.br && bc == o.bc &&
               elem == o.elem && sw == o.sw;
    }
};
struct MapKeyHash {
    size_t operator()(const MapKey &k) const {
        size_t h = reinterpret_cast<size_t>(k.ptr);
        auto mix = [&](uint64_t v) { h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2); };
        mix(k.rows), mix(k.cols), mix(k.ld), mix(k.br), mix(k.bc), mix(k.elem), mix(k.sw);
        return h;
    }
};
std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;
}  // namespace

bool get_tmap_2d(CUtensorMap *out, const void *ptr, int elem, int64_t rows, int64_t cols, int64_t ld, uint32_t br,
                 uint32_t bc, Swz sw) {
    MapKey key{ptr, rows, cols, ld, br, bc, elem, static_cast<int>(sw)};
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
        *out = it->second;
        return true;
    }
    if (!make_tmap_2d(out, ptr, elem, rows, cols, ld, br, bc, sw)) return false;
    if (g_maps.size() > 1024) g_maps.clear();
    g_maps.emplace(key, *out);
    return true;
}

}  // namespace compar
