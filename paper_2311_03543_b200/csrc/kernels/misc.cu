// Small kernels around the GEMM variants:
//   * scale:  C_out = beta * C_in (beta == 0: zeros, C_in unread) — the BLAS quick path for
//             k == 0 or alpha == 0, where A and B must not be read (R3);
//   * spin:   a one-thread %globaltimer spin of a prescribed duration, the synthetic-cost
//             fixture behind USER test variants.
#include "kernels.h"

namespace compar {

cudaError_t preload_tc_kernels();
cudaError_t preload_tma_kernels();
cudaError_t preload_simt_kernels();
cudaError_t preload_tc2_kernels();
cudaError_t preload_tcw_kernels();
cudaError_t preload_tcm_kernels();
cudaError_t preload_tck_kernels();

namespace {

__global__ void scale_kernel(int64_t m, int64_t n, float beta, const float *__restrict__ cin, int64_t ldin,
                             float *__restrict__ cout, int64_t ldout) {
    const int64_t total = m * n;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = idx / n, c = idx - r * n;
        cout[r * ldout + c] = beta == 0.f ? 0.f : beta * cin[r * ldin + c];
    }
}

__global__ void spin_kernel(int64_t ns) {
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (static_cast<int64_t>(t - t0) < ns);
}

}  // namespace

cudaError_t launch_scale(const GemmLaunch &g) {
    if (g.m == 0 || g.n == 0) return cudaSuccess;
    int64_t blocks = (g.m * g.n + 255) / 256;
    if (blocks > 4L * g.num_sms * 8) blocks = 4L * g.num_sms * 8;
    scale_kernel<<<static_cast<unsigned>(blocks), 256, 0, g.stream>>>(g.m, g.n, g.beta, g.C_in, g.ldc_in, g.C_out,
                                                                      g.ldc_out);
    return cudaGetLastError();
}

cudaError_t launch_spin(cudaStream_t s, int64_t ns) {
    spin_kernel<<<1, 1, 0, s>>>(ns);
    return cudaGetLastError();
}

cudaError_t preload_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, scale_kernel);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, spin_kernel);
    if (e == cudaSuccess) e = preload_tc_kernels();
    if (e == cudaSuccess) e = preload_tma_kernels();
    if (e == cudaSuccess) e = preload_simt_kernels();
    if (e == cudaSuccess) e = preload_tc2_kernels();
    if (e == cudaSuccess) e = preload_tcw_kernels();
    if (e == cudaSuccess) e = preload_tcm_kernels();
    if (e == cudaSuccess) e = preload_tck_kernels();
    return e;
}

}  // namespace compar
