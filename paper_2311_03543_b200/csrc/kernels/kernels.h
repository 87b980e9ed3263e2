// Internal launcher interface between the C++ runtime and the sm_100a kernels.
// Not part of the public ABI (include/compar.h).  All pointers are device pointers.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace compar {

// Launcher tuning knobs, read once per runtime context from the environment (read_knobs) and
// passed with every launch — nothing reads the environment on the launch path.  0 = the launcher's
// own choice.  They only change tile widths / raster order / schedule, never any element's k order.
struct Knobs {
    int tc1_bn = 0;          // COMPAR_TC1_BN: 1-SM tile width 256 / 128 / 64
    int tc1_group = 0;       // COMPAR_TC1_GROUP: 1-SM raster band (row blocks)
    int tc2_bn = 0;          // COMPAR_TC2_BN: pair tile width 256 / 128
    int tc2_group = 0;       // COMPAR_TCM_GROUP: pair raster band (cluster tiles)
    int tc2_rowstore_group = 0;   // COMPAR_TC_GROUP: raster band of the row-store pair kernel
    int tc2_producers = 2;   // COMPAR_TC2_PRODUCERS: TMA producer warps per CTA in the pair kernel (1 or 2)
    int tc2_tmem_cin = 1;    // COMPAR_TC2_TMEM_CIN=0: single-wave pair launches read C_in from shared memory
    int tc2_deep = 1;        // COMPAR_TC2_DEEP=0: no deep-ring (6-stage) pair instantiation for multi-wave grids
    int even_waves = 1;      // COMPAR_EVEN_WAVES=0: the pair kernel on every CTA pair even when its
                             // last wave of tiles is partial
    int tcw_group = 0;       // COMPAR_TCW_GROUP: wide-pair raster band (pair rows)
    int tcw_delay = 24;      // COMPAR_TCW_DELAY: wide-pair epilogue-overlap delay in k-steps
    int tma_tile = 0;        // COMPAR_TMA_TILE: tma_f32 tile 128 / 64
};
Knobs read_knobs();

// World-mode (row panels + broadcast of B) extras of a wide-pair launch (tc_gemm_2sm_wide.cu):
//   * slab wait (flags != nullptr): B arrives as nslab contiguous slabs of slab_w columns (packed:
//     slab j is a K x slab_w row-major block; transB: rows [j slab_w, (j+1) slab_w) of B^T); before
//     loading the B tiles of slab j a producer waits until flags[j] >= seq (written on the comm
//     stream after slab j landed), and tiles are visited column-major so slab j's tiles come first;
//   * split launch (helper_sms > 0): the main launch runs on num_sms - helper_sms SMs (the rest
//     are left to the broadcast's kernels); once `helper_after` (the broadcast's end) has fired, a
//     helper launch on helper_stream adds helper_sms SMs, drawing tiles from the same counter; the
//     launch's stream then waits for `helper_done` (recorded after the helper).
struct WorldLaunch {
    const unsigned *flags = nullptr;
    unsigned seq = 0;
    int slab_w = 0, nslab = 0;
    int helper_sms = 0;
    cudaStream_t helper_stream = nullptr;
    cudaEvent_t helper_after = nullptr, helper_done = nullptr;
    mutable int launches = 0;    // out: kernel launches issued (1, or 2 with the helper)
};

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
    const Knobs *knobs = nullptr;        // nullptr: defaults
    const WorldLaunch *world = nullptr;  // wide-pair kernel only
};

inline const Knobs &knobs_of(const GemmLaunch &g) {
    static const Knobs defaults;
    return g.knobs ? *g.knobs : defaults;
}

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
// variant (c), CTA-pair kernel with TMA C epilogue (tc_gemm_2sm_mc.cu); needs TMA-compatible C.
// Reached through launch_tc_gemm_2sm.
cudaError_t launch_tc_gemm_pairs(const GemmLaunch &g, bool bf16);
cudaError_t launch_scale(const GemmLaunch &g);               // k == 0 or alpha == 0: C_out = beta*C_in
cudaError_t launch_spin(cudaStream_t s, int64_t ns);         // synthetic-cost fixture
// Device rows -> mapped pinned host memory (dst: the host buffer's device alias) by `ctas` CTAs: a
// rate-limited D2H that leaves the H2D direction more of the PCIe link than a copy engine does.
cudaError_t launch_rows_to_host(float *dst, int64_t ld_dst, const float *src, int64_t ld_src, int64_t rows,
                                int64_t cols, int ctas, cudaStream_t s);
cudaError_t preload_kernels();                               // force module load (no lazy loading in calibration)
int *sched_workspace(cudaStream_t s);                        // {next, done} tile counters for persistent kernels
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

// tc_*_ck (variant c, cluster split-K, tc_gemm_ck.cu): the two CTAs of a cluster split a tile's
// ceil(K / BK) k-blocks at h = ceil(kb / 2) — a function of K alone (row panels stay bitwise equal).
// Eligible from 2 k-blocks on, and only where the 128 x 256 tiles of the (panel) shape fit one wave
// of clusters (tiles <= SMs): a single-wave form, not calibrated on multi-wave shapes it cannot win.
inline int tc_clusterk_half(int64_t k, bool bf16) {
    const int64_t bk = bf16 ? 64 : 32;
    const int64_t kb = (k + bk - 1) / bk;
    return static_cast<int>((kb + 1) / 2);
}
inline bool tc_clusterk_ok(int64_t m, int64_t n, int64_t k, bool bf16, int sms) {
    return k > (bf16 ? 64 : 32) && ((m + 127) / 128) * ((n + 255) / 256) <= sms;
}
cudaError_t launch_tc_gemm_ck(const GemmLaunch &g, bool bf16);

// tc_f32x3 (variant c, FP32-accuracy form, tc_f32x3.cu): operands split into TF32 hi + lo in a
// per-stream workspace of tc_f32x3_workspace_bytes(), then one TF32 tcgen05 GEMM over 3K in
// chunks of 1024 original k.  Eligible from K >= tc_f32x3_min_k.
constexpr int64_t tc_f32x3_min_k = 64;
size_t tc_f32x3_workspace_bytes(int64_t m, int64_t n, int64_t k, int transB);
cudaError_t launch_tc_gemm_f32x3(const GemmLaunch &g);
// The per-stream split-K planes and tc_f32x3 operand workspaces (up to GiBs) are released when the
// last runtime context terminates (compar_terminate).
void release_f32x3_workspaces();
void release_split_workspaces();

// TMA eligibility (the selector's constraint filter).
inline bool tma_compatible(const void *p, int64_t ld, int elem_bytes) {
    return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && ((ld * elem_bytes) % 16 == 0);
}

}  // namespace compar
