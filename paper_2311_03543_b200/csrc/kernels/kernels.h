// Internal launcher interface between the C++ runtime and the sm_100a kernels.
// Not part of the public ABI (include/compar.h).  All pointers are device pointers.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace compar {

// One variant launch over a row panel: C_out = alpha * A * B + beta * C_in
// (PAPER.md P:76-80, P:201-205 read as xGEMM; R1-R3).
struct GemmLaunch {
    int64_t m, n, k;           // panel rows, columns, reduction depth
    float alpha, beta;         // beta == 0: C_in is never read
    const void *A; int64_t lda;        // m x k row-major (FP32 or BF16 bits)
    const void *B; int64_t ldb;        // k x n row-major, or n x k when transB
    int transB;
    const float *C_in; int64_t ldc_in;
    float *C_out; int64_t ldc_out;
    cudaStream_t stream;
    int num_sms;               // SMs of the device (persistent grids)
};

cudaError_t launch_simt_f32(const GemmLaunch &g);            // variant (a)
cudaError_t launch_simt_bf16(const GemmLaunch &g);           // variant (a), BF16 operands

// The sort interface (sort.cu): in-place ascending sort of n 4-byte keys (key_type 0 u32, 1 i32,
// 2 f32 totalOrder).  The radix sort needs sort_radix_scratch_bytes(n) of device scratch.
size_t sort_radix_scratch_bytes(int64_t n);
int64_t sort_bitonic_max();
cudaError_t launch_sort_radix(void *keys, int64_t n, int key_type, void *scratch, cudaStream_t s, int num_sms);
cudaError_t launch_sort_bitonic(void *keys, int64_t n, int key_type, cudaStream_t s);
cudaError_t launch_tma_f32(const GemmLaunch &g);             // variant (b)
cudaError_t launch_tc_gemm(const GemmLaunch &g, bool bf16);  // variant (c): tcgen05 TF32 / BF16
cudaError_t launch_tc_gemm_2sm(const GemmLaunch &g, bool bf16);  // variant (c), CTA-pair (cta_group::2)
cudaError_t launch_tc_gemm_2sm_wide(const GemmLaunch &g, bool bf16);  // variant (c), wide CTA-pair 256x512
// variant (c), CTA-pair kernel with TMA C epilogue (tc_gemm_2sm_mc.cu): `pairs` = 1 (cluster of 2) or
// 2 (cluster of 4, B shared by TMA multicast); needs TMA-compatible C.  Reached through launch_tc_gemm_2sm.
cudaError_t launch_tc_gemm_pairs(const GemmLaunch &g, bool bf16, int pairs);
cudaError_t launch_scale(const GemmLaunch &g);               // k == 0 or alpha == 0: C_out = beta*C_in
cudaError_t launch_spin(cudaStream_t s, int64_t ns);         // synthetic-cost fixture
cudaError_t preload_kernels();                               // force module load (no lazy loading in calibration)
int *sched_workspace(cudaStream_t s);                        // {next, done} tile counters for persistent kernels
struct SkWorkspace {                                         // stream-K partials (tc_gemm_2sm_mc.cu)
    unsigned *flags = nullptr;
    float *partial = nullptr;
    int cap = 0;
    uint32_t epoch = 0;
};
SkWorkspace *sk_workspace(cudaStream_t s, int clusters);
// Split-K partial planes of the tc_*_sk variant (grown on demand, per stream).
struct SplitWorkspace {
    float *part = nullptr;
    unsigned *count = nullptr;
    size_t part_bytes = 0, count_words = 0;
};
SplitWorkspace *split_workspace(cudaStream_t s, size_t part_bytes, size_t count_words);

// tc_*_sk (variant c, split-K form of the TMA-epilogue pair kernel): the number of K splits is a
// function of K alone — ceil(K / BK) k-blocks (BK = 64 BF16 / 32 TF32 elements), at least 32 per
// split, at most 8 splits — so a panel's arithmetic never depends on M (row panels stay bitwise
// equal).  0 = not eligible (fewer than 2 splits, or a partial workspace above 1 GiB).
inline int tc_splitk_splits(int64_t m, int64_t n, int64_t k, bool bf16) {
    const int64_t bk = bf16 ? 64 : 32;
    const int64_t kb = (k + bk - 1) / bk;
    int64_t s = kb / 32;
    if (s > 8) s = 8;
    if (s < 2) return 0;
    const int64_t tiles = ((m + 255) / 256) * ((n + 255) / 256);
    if (tiles * s * 256 * 256 * 4 > (int64_t(1) << 30)) return 0;   // partial planes <= 1 GiB
    return static_cast<int>(s);
}
cudaError_t launch_tc_gemm_splitk(const GemmLaunch &g, bool bf16);

// TMA eligibility (the selector's constraint filter).
inline bool tma_compatible(const void *p, int64_t ld, int elem_bytes) {
    return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && ((ld * elem_bytes) % 16 == 0);
}

}  // namespace compar
