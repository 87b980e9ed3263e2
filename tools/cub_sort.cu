// Yardstick for the sort interface (NEXT-3): CUB's DeviceRadixSort::SortKeys (onesweep) on the same
// keys as tools/sort_bench.py (FP32 random bit patterns), CUDA-event time, median of 10.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/cub_sort.cu -o /tmp/cub_sort
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void fill(uint32_t *x, int64_t n, uint64_t seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = seed + 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        x[i] = (uint32_t)(z ^ (z >> 31));
    }
}

int main() {
    for (int lg = 16; lg <= 28; lg += 2) {
        const int64_t n = int64_t(1) << lg;
        float *in, *out;
        cudaMalloc(&in, n * 4);
        cudaMalloc(&out, n * 4);
        fill<<<1184, 256>>>(reinterpret_cast<uint32_t *>(in), n, 7);
        size_t tmp_bytes = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, in, out, (int)n);
        void *tmp;
        cudaMalloc(&tmp, tmp_bytes);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        std::vector<float> ts;
        for (int r = 0; r < 11; ++r) {
            cudaEventRecord(a);
            cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, in, out, (int)n);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r) ts.push_back(ms);
        }
        std::sort(ts.begin(), ts.end());
        const double us = ts[ts.size() / 2] * 1e3;
        std::printf("{\"n\": %lld, \"cub_sortkeys_us\": %.2f, \"gkeys_s\": %.2f}\n", (long long)n, us, n / us / 1e3);
        cudaFree(in);
        cudaFree(out);
        cudaFree(tmp);
    }
    return 0;
}
