// Fixed cost of a launch as the runtime's task events see it: event time of EMPTY kernels with the
// launch configurations of the tcgen05 kernels (148 CTAs, 2-CTA clusters, 352 threads, ~225 KB
// dynamic smem, four 128-byte __grid_constant__ tensor-map parameters) against a minimal launch.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/launch_cost.cu -lcuda -o /tmp/launch_cost
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void tiny() {}
__global__ void big_plain(int *p) { if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1; }
__global__ void __cluster_dims__(2, 1, 1) big_cluster(int *p) { if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1; }
__global__ void __cluster_dims__(2, 1, 1) big_cluster_maps(const __grid_constant__ CUtensorMap a,
                                                           const __grid_constant__ CUtensorMap b,
                                                           const __grid_constant__ CUtensorMap c,
                                                           const __grid_constant__ CUtensorMap d, int *p) {
    if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = (int)reinterpret_cast<const char *>(&a)[0] + (int)reinterpret_cast<const char *>(&d)[0];
}

template <class F>
static void timeit(const char *name, F launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<float> idle, b2b;
    for (int r = 0; r < 30; ++r) {
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 5) idle.push_back(ms * 1e3f);
    }
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 50; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    std::sort(idle.begin(), idle.end());
    std::printf("{\"launch\": \"%s\", \"idle_stream_us\": %.2f, \"back_to_back_us\": %.2f}\n", name, idle[idle.size() / 2],
                ms * 1e3f / 50);
}

int main() {
    int *p;
    cudaMalloc(&p, 4);
    const int smem = 225 * 1024;
    cudaFuncSetAttribute(big_plain, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(big_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(big_cluster_maps, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    CUtensorMap m{};
    timeit("tiny <<<1, 32>>>", [&] { tiny<<<1, 32>>>(); });
    timeit("148 x 352 threads, no smem", [&] { big_plain<<<148, 352>>>(p); });
    timeit("148 x 352 threads, 225 KB smem", [&] { big_plain<<<148, 352, smem>>>(p); });
    timeit("148 x 352, 225 KB, cluster 2", [&] { big_cluster<<<148, 352, smem>>>(p); });
    timeit("148 x 352, 225 KB, cluster 2, 4 tensor maps", [&] { big_cluster_maps<<<148, 352, smem>>>(m, m, m, m, p); });
    timeit("128 x 352, 225 KB, cluster 2, 4 tensor maps", [&] { big_cluster_maps<<<128, 352, smem>>>(m, m, m, m, p); });
    return 0;
}
