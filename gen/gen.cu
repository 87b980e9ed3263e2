// Device twin of gen/inputs.py (see include/compar_gen.h).  No GEMM arithmetic here.
#include <cuda_runtime.h>
#include <stdint.h>

#include "compar_gen.h"

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ float value_f32(uint64_t h, int dist) {
    if (dist == 0) return static_cast<float>(static_cast<int32_t>(h >> 40) - (1 << 23)) * 0x1p-23f;
    if (dist == 1) return static_cast<float>(static_cast<uint32_t>(h >> 40)) * 0x1p-24f;
    return static_cast<float>(static_cast<int32_t>(h % 5ull) - 2);
}

__device__ __forceinline__ uint16_t bf16_rne(float f) {
    const uint32_t u = __float_as_uint(f);
    return static_cast<uint16_t>((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

__global__ void fill_kernel(void *dst, int dtype, int64_t rows, int64_t cols, int64_t ld, int64_t row0, int64_t col0,
                            uint64_t seed, int tag, int dist, int transposed) {
    // storage extents
    const int64_t srows = transposed ? cols : rows, scols = transposed ? rows : cols;
    const int64_t total = srows * scols;
    const uint64_t base = seed ^ (static_cast<uint64_t>(tag) << 56);
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t sr = idx / scols, sc = idx - sr * scols;
        const uint64_t i = static_cast<uint64_t>(row0 + (transposed ? sc : sr));
        const uint64_t j = static_cast<uint64_t>(col0 + (transposed ? sr : sc));
        const float v = value_f32(splitmix64(base ^ (i << 28) ^ j), dist);
        if (dtype == 0)
            static_cast<float *>(dst)[sr * ld + sc] = v;
        else
            static_cast<uint16_t *>(dst)[sr * ld + sc] = bf16_rne(v);
    }
}

}  // namespace

extern "C" int compar_gen_fill(void *dst, int dtype, int64_t rows, int64_t cols, int64_t ld, int64_t row0, int64_t col0,
                               uint64_t seed, int tag, int dist, int transposed, void *stream) {
    if (rows < 0 || cols < 0 || row0 < 0 || col0 < 0 || (dtype != 0 && dtype != 1) || dist < 0 || dist > 2) return 1;
    if (rows == 0 || cols == 0) return 0;
    if (!dst || ld < (transposed ? rows : cols)) return 1;
    int64_t total = rows * cols;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    fill_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        dst, dtype, rows, cols, ld, row0, col0, seed, tag, dist, transposed);
    return static_cast<int>(cudaGetLastError());
}
