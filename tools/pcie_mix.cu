// PCIe direction mix on one B200 (the e2e host pipeline's limit): H2D and D2H
// copy-engine rates alone and concurrently, and H2D beside a device->host copy done by a KERNEL of
// `ctas` CTAs storing into mapped pinned memory (a rate-limited D2H: fewer CTAs, fewer bytes in
// flight).  Question: does a slower, continuous D2H leave the H2D direction its solo rate?
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/pcie_mix.cu -o /tmp/pcie_mix
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

__global__ void d2h_kernel(const float4 *__restrict__ src, float4 *dst, int64_t n4) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

static float ms_between(cudaEvent_t a, cudaEvent_t b) {
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    const size_t h2d_bytes = size_t(4) << 30, d2h_bytes = size_t(2) << 30;
    void *hin, *hout, *din, *dout;
    cudaHostAlloc(&hin, h2d_bytes, cudaHostAllocMapped);
    cudaHostAlloc(&hout, d2h_bytes, cudaHostAllocMapped);
    cudaMalloc(&din, h2d_bytes);
    cudaMalloc(&dout, d2h_bytes);
    cudaMemset(dout, 1, d2h_bytes);
    void *hout_dev;
    cudaHostGetDevicePointer(&hout_dev, hout, 0);
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t a0, a1, b0, b1;
    cudaEventCreate(&a0);
    cudaEventCreate(&a1);
    cudaEventCreate(&b0);
    cudaEventCreate(&b1);
    auto h2d = [&]() {
        cudaEventRecord(a0, s1);
        cudaMemcpyAsync(din, hin, h2d_bytes, cudaMemcpyHostToDevice, s1);
        cudaEventRecord(a1, s1);
    };
    for (int rep = 0; rep < 2; ++rep) {
        h2d();
        cudaDeviceSynchronize();
        std::printf("{\"case\": \"h2d alone\", \"h2d_gbs\": %.1f}\n", h2d_bytes / ms_between(a0, a1) / 1e6);
        cudaEventRecord(b0, s2);
        cudaMemcpyAsync(hout, dout, d2h_bytes, cudaMemcpyDeviceToHost, s2);
        cudaEventRecord(b1, s2);
        cudaDeviceSynchronize();
        std::printf("{\"case\": \"d2h alone (copy engine)\", \"d2h_gbs\": %.1f}\n", d2h_bytes / ms_between(b0, b1) / 1e6);
        h2d();
        cudaEventRecord(b0, s2);
        cudaMemcpyAsync(hout, dout, d2h_bytes, cudaMemcpyDeviceToHost, s2);
        cudaEventRecord(b1, s2);
        cudaDeviceSynchronize();
        std::printf("{\"case\": \"both copy engines\", \"h2d_gbs\": %.1f, \"d2h_gbs\": %.1f}\n",
                    h2d_bytes / ms_between(a0, a1) / 1e6, d2h_bytes / ms_between(b0, b1) / 1e6);
        for (int ctas : {1, 2, 4, 8, 16, 32, 148}) {
            cudaEventRecord(b0, s2);
            d2h_kernel<<<ctas, 512, 0, s2>>>(static_cast<const float4 *>(dout), static_cast<float4 *>(hout_dev),
                                            int64_t(d2h_bytes / 16));
            cudaEventRecord(b1, s2);
            cudaDeviceSynchronize();
            const double solo = d2h_bytes / ms_between(b0, b1) / 1e6;
            h2d();
            cudaEventRecord(b0, s2);
            d2h_kernel<<<ctas, 512, 0, s2>>>(static_cast<const float4 *>(dout), static_cast<float4 *>(hout_dev),
                                            int64_t(d2h_bytes / 16));
            cudaEventRecord(b1, s2);
            cudaDeviceSynchronize();
            std::printf("{\"case\": \"h2d + kernel d2h\", \"ctas\": %d, \"kernel_d2h_alone_gbs\": %.1f, \"h2d_gbs\": %.1f, "
                        "\"d2h_gbs\": %.1f}\n", ctas, solo, h2d_bytes / ms_between(a0, a1) / 1e6,
                        d2h_bytes / ms_between(b0, b1) / 1e6);
        }
    }
    return 0;
}
