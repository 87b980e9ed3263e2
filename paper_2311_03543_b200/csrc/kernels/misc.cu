// Small kernels around the GEMM variants:
//   * scale:  C_out = beta * C_in (beta == 0: zeros, C_in unread) — the BLAS quick path for
//             k == 0 or alpha == 0, where A and B must not be read (R3);
//   * spin:   a one-thread %globaltimer spin of a prescribed duration, the synthetic-cost
//             fixture behind USER test variants;
//   * rows to host: a device -> mapped-pinned-host copy of a row block by a few CTAs — a rate-limited
//             D2H for the host-memory pipeline.
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

__global__ void __launch_bounds__(512) rows_to_host_kernel(float *dst, int64_t ld_dst, const float *__restrict__ src,
                                                           int64_t ld_src, int64_t rows, int64_t cols, int vec) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (vec) {   // 16-byte rows: float4 per thread
        const int64_t q = cols / 4;
        for (int64_t i = t0; i < rows * q; i += stride) {
            const int64_t r = i / q, c = (i - r * q) * 4;
            *reinterpret_cast<float4 *>(dst + r * ld_dst + c) = __ldcs(reinterpret_cast<const float4 *>(src + r * ld_src + c));
        }
    } else {
        for (int64_t i = t0; i < rows * cols; i += stride) {
            const int64_t r = i / cols, c = i - r * cols;
            dst[r * ld_dst + c] = src[r * ld_src + c];
        }
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

cudaError_t launch_rows_to_host(float *dst, int64_t ld_dst, const float *src, int64_t ld_src, int64_t rows,
                                int64_t cols, int ctas, cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return cudaSuccess;
    const int vec = (cols % 4 == 0) && (ld_dst % 4 == 0) && (ld_src % 4 == 0) &&
                    (reinterpret_cast<uintptr_t>(dst) % 16 == 0) && (reinterpret_cast<uintptr_t>(src) % 16 == 0);
    rows_to_host_kernel<<<ctas, 512, 0, s>>>(dst, ld_dst, src, ld_src, rows, cols, vec);
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
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, rows_to_host_kernel);
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
