// Variant (c), FP32-accuracy form "tc_f32x3" (precision class F32_SPLIT; R38) for sm_100a.
//
// The paper's matrix multiply works on FP32 `float` arrays (PAPER.md P:78 [§2.1], P:201-205
// [Table 2, BLAS / CUBLAS SGEMM]).  FP32 FFMA peaks at 74 TFLOP/s on a B200; the TF32 tensor cores
// at ~1.1 PFLOP/s, but one TF32 product keeps only 11 of FP32's 24 significand bits.  Splitting
// every operand into two TF32 numbers, x = x_hi + x_lo + O(2^-22 |x|) (x_hi = RN_tf32(x),
// x_lo = RN_tf32(x - x_hi), the subtraction exact), and dropping only the lo*lo term,
//
//     a*b = a_hi*b_hi + a_hi*b_lo + a_lo*b_hi + O(3 * 2^-22 |a||b|),
//
// gives every product to within 3 * 2^-22 relative — below the c*K*u (u = 2^-24) accumulation
// term of the FP32 dot-product bound from K >= 64 on, which is where the variant is eligible.
//
// Realisation: the three products are ONE TF32 GEMM over a tripled K.  A split pass writes A'
// (m x 3K) and B' (3K x n; transB: n x 3K) so that A' B' = sum of the three products for every k,
// in chunks of kChunkK original k laid out as (a_hi | a_lo | a_hi) against (b_lo | b_hi | b_hi): the
// small cross terms first, hi*hi last (seg_pos below).  The product GEMM is the CTA-pair tcgen05 TF32 kernel
// (tc_gemm_2sm_mc.cu) on the pre-split operands, whose low 13 mantissa bits are zero, so the
// hardware's TF32 reading of the FP32 bits (R6) is exact.  K is taken in chunks of kChunkK
// original k (3 * kChunkK tensor-core k): the tensor core's FP32 accumulator is not round-to-
// nearest (R33: about one truncation per MMA), so each chunk's accumulation stays short and the
// chunks are combined by the kernel's own epilogue, C = alpha * acc + 1 * C (one round-to-nearest
// FMA per chunk and element): chunk 0 applies the caller's beta * C_in, chunks >= 1 accumulate
// into C_out in place.  Chunks depend on K alone, so a row panel's arithmetic never depends on M.
//
// Traffic per launch: split pass reads A, B once (4 B / element) and writes 12 B / element; each
// chunk's GEMM reads its A' / B' column / row block and C, and writes C.  Workspace: 12 (mk + kn)
// bytes (rows padded to 16 B), library-owned per stream.
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>

#include "kernels.h"

namespace compar {
namespace {

constexpr int64_t kChunkK = 1024;   // original k per tensor-core accumulation chunk

// Round-to-nearest-even onto the TF32 grid (10 explicit mantissa bits: the low 13 FP32 bits
// cleared).  Infinities and NaNs pass unchanged; a finite value that would round up to infinity
// is truncated instead (it stays finite: its lo part carries the difference).
__device__ __forceinline__ float tf32_rn(float x) {
    const uint32_t u = __float_as_uint(x);
    if ((u & 0x7f800000u) == 0x7f800000u) return x;
    uint32_t r = (u + 0x0fffu + ((u >> 13) & 1u)) & 0xffffe000u;
    if ((r & 0x7f800000u) == 0x7f800000u) r = u & 0xffffe000u;
    return __uint_as_float(r);
}

__device__ __forceinline__ void split2(float x, float &hi, float &lo) {
    hi = tf32_rn(x);
    lo = isfinite(hi) ? tf32_rn(__fsub_rn(x, hi)) : 0.f;   // x - hi is exact in FP32
}

// Chunked layout of the tripled K (R38).  Original k lies in chunk c = k / kChunkK at offset
// j = k - c kChunkK; the chunk's width kc = min(kChunkK, K - c kChunkK) is padded to kcp = round4(kc)
// (zero entries, which add nothing), and its 3 kcp tensor-core k hold three segments starting at
// 3 c kChunkK: segment 0 at + j, segment 1 at + kcp + j, segment 2 at + 2 kcp + j.  A takes
// (hi, lo, hi) and B (lo, hi, hi), so a chunk sums hi*lo + lo*hi first, while the accumulator is
// still ~2^-11 of the result, and hi*hi last: the truncating accumulator (R33) then loses about one
// ulp of the result per MMA of the hi*hi segment only (kChunkK / 8 of them), not per MMA of all three.
__device__ __forceinline__ void seg_pos(int64_t k, int64_t K, int64_t &p0, int64_t &kcp) {
    const int64_t c = k / kChunkK;
    const int64_t kc = K - c * kChunkK < kChunkK ? K - c * kChunkK : kChunkK;
    kcp = (kc + 3) / 4 * 4;
    p0 = 3 * c * kChunkK + (k - c * kChunkK);
}

// K runs along columns (A, and B when transB): Y[r][segments of k] for X[r][k], k < round4(K)
// (zero beyond K), four k per work item i.  lo_first = 0: (hi, lo, hi) — the A side; 1: (lo, hi,
// hi) — the B side.
__device__ __forceinline__ void split_cols_item(int64_t i, const float *__restrict__ X, int64_t ldx,
                                                float *__restrict__ Y, int64_t ldy, int64_t K, int lo_first) {
    const int64_t q = (K + 3) / 4;
    const int64_t r = i / q, k0 = (i - r * q) * 4;
    const float *x = X + r * ldx + k0;
    float v[4];
    if (k0 + 4 <= K) {
        const float4 t = __ldcs(reinterpret_cast<const float4 *>(x));
        v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
    } else {
        for (int e = 0; e < 4; ++e) v[e] = k0 + e < K ? x[e] : 0.f;
    }
    float h[4], l[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) split2(v[e], h[e], l[e]);
    int64_t p0, kcp;
    seg_pos(k0, K, p0, kcp);
    float *y = Y + r * ldy + p0;
    const float4 hv = make_float4(h[0], h[1], h[2], h[3]), lv = make_float4(l[0], l[1], l[2], l[3]);
    __stcg(reinterpret_cast<float4 *>(y), lo_first ? lv : hv);
    __stcg(reinterpret_cast<float4 *>(y + kcp), lo_first ? hv : lv);
    __stcg(reinterpret_cast<float4 *>(y + 2 * kcp), hv);
}

// K runs along rows (row-major B, K x N): rows of Y at the (lo, hi, hi) segment positions of k,
// for k < round4(K) (zero rows beyond K), four columns per work item i.
__device__ __forceinline__ void split_rows_item(int64_t i, const float *__restrict__ X, int64_t ldx,
                                                float *__restrict__ Y, int64_t ldy, int64_t K, int64_t cols) {
    const int64_t q = (cols + 3) / 4;
    const int64_t k = i / q, c0 = (i - k * q) * 4;
    int64_t p0, kcp;
    seg_pos(k, K, p0, kcp);
    float *y0 = Y + p0 * ldy + c0;
    float *y1 = y0 + kcp * ldy;
    float *y2 = y0 + 2 * kcp * ldy;
    if (c0 + 4 <= cols) {
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < K) t = __ldcs(reinterpret_cast<const float4 *>(X + k * ldx + c0));
        float h[4], l[4];
        split2(t.x, h[0], l[0]);
        split2(t.y, h[1], l[1]);
        split2(t.z, h[2], l[2]);
        split2(t.w, h[3], l[3]);
        const float4 hv = make_float4(h[0], h[1], h[2], h[3]), lv = make_float4(l[0], l[1], l[2], l[3]);
        __stcg(reinterpret_cast<float4 *>(y0), lv);
        __stcg(reinterpret_cast<float4 *>(y1), hv);
        __stcg(reinterpret_cast<float4 *>(y2), hv);
    } else {
        for (int64_t c = c0; c < cols; ++c) {
            float hh, ll;
            split2(k < K ? X[k * ldx + c] : 0.f, hh, ll);
            y0[c - c0] = ll;
            y1[c - c0] = hh;
            y2[c - c0] = hh;
        }
    }
}

// Both operands in ONE launch (a launch is ~4 us of fixed cost at the sizes where this matters):
// work items [0, a_items) split A, the rest split B (columns when transB, rows otherwise).
struct SplitArgs {
    const float *A;
    int64_t lda;
    float *A3;
    int64_t lda3;
    const float *B;
    int64_t ldb;
    float *B3;
    int64_t ldb3;
    int64_t m, n, k;
    int transB;
    int64_t a_items, items;
};

__global__ void __launch_bounds__(256) split_ab_kernel(const SplitArgs a) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < a.items;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i < a.a_items)
            split_cols_item(i, a.A, a.lda, a.A3, a.lda3, a.k, 0);
        else if (a.transB)
            split_cols_item(i - a.a_items, a.B, a.ldb, a.B3, a.ldb3, a.k, 1);
        else
            split_rows_item(i - a.a_items, a.B, a.ldb, a.B3, a.ldb3, a.k, a.n);
    }
}

struct X3Workspace {
    float *buf = nullptr;
    size_t bytes = 0;
};

std::mutex g_x3_mu;
std::map<cudaStream_t, X3Workspace> g_x3;

float *x3_workspace(cudaStream_t s, size_t bytes) {
    std::lock_guard<std::mutex> lk(g_x3_mu);
    auto &slots = g_x3;
    X3Workspace &w = slots[s];
    if (w.bytes < bytes) {
        if (w.buf) {
            cudaStreamSynchronize(s);   // the previous launch on this stream may still read it
            cudaFree(w.buf);
        }
        w.buf = nullptr;
        w.bytes = 0;
        if (cudaMalloc(&w.buf, bytes) != cudaSuccess) return nullptr;
        w.bytes = bytes;
    }
    return w.buf;
}

inline int64_t round4(int64_t x) { return (x + 3) / 4 * 4; }

unsigned grid_for(int64_t work, int num_sms) {
    const int64_t b = (work + 255) / 256;
    const int64_t cap = static_cast<int64_t>(num_sms) * 8;
    return static_cast<unsigned>(b < cap ? (b > 0 ? b : 1) : cap);
}

}  // namespace

void release_f32x3_workspaces() {
    std::lock_guard<std::mutex> lk(g_x3_mu);
    for (auto &kv : g_x3)
        if (kv.second.buf) cudaFree(kv.second.buf);   // (cudaFree waits for the device)
    g_x3.clear();
}

size_t tc_f32x3_workspace_bytes(int64_t m, int64_t n, int64_t k, int transB) {
    const int64_t k3 = 3 * round4(k);
    const int64_t a = m * k3;
    const int64_t b = transB ? n * k3 : k3 * round4(n);
    return static_cast<size_t>(a + b) * 4;
}

cudaError_t launch_tc_gemm_f32x3(const GemmLaunch &g) {
    const int64_t m = g.m, n = g.n, k = g.k;
    const int64_t k3 = 3 * round4(k);
    const int64_t lda3 = k3;
    const int64_t ldb3 = g.transB ? k3 : round4(n);
    float *ws = x3_workspace(g.stream, tc_f32x3_workspace_bytes(m, n, k, g.transB));
    if (!ws) return cudaErrorMemoryAllocation;
    float *A3 = ws;
    float *B3 = ws + m * lda3;
    SplitArgs sa;
    sa.A = static_cast<const float *>(g.A), sa.lda = g.lda, sa.A3 = A3, sa.lda3 = lda3;
    sa.B = static_cast<const float *>(g.B), sa.ldb = g.ldb, sa.B3 = B3, sa.ldb3 = ldb3;
    sa.m = m, sa.n = n, sa.k = k, sa.transB = g.transB;
    sa.a_items = m * ((k + 3) / 4);
    sa.items = sa.a_items + (g.transB ? n * ((k + 3) / 4) : round4(k) * ((n + 3) / 4));
    split_ab_kernel<<<grid_for(sa.items, g.num_sms), 256, 0, g.stream>>>(sa);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // the product GEMM: one launch of a tcgen05 TF32 kernel per chunk of 3 * kChunkK tensor-core
    // k; the first applies the caller's beta * C_in, later ones accumulate into C_out (beta = 1, a
    // round-to-nearest FMA per element).  One kernel over the whole 3K with the chunks switched
    // in-kernel (C kept in L2 between a tile's chunks) measured slower at every size (8192^3 5.15
    // vs 4.77 ms, 16384^3 44.7 vs 39.9 ms: a tile's long A' / B' panels no longer share L2 across the
    // tiles in flight), so the chunks are separate launches.  The tile-width choice keeps every
    // element's k order, so row panels stay bitwise equal.  Only the last chunk can be short
    // (3 * round4(kc) k).
    // Small grids (at most 16 pair tiles) take the 1-SM kernel, the rest the CTA-pair kernel: the
    // un-split tcgen05 forms sum every element's k in the same MMA steps, so their results are bitwise
    // identical (tests/test_gpu_parity.py::test_unsplit_tcgen05_forms_bitwise_identical) and the
    // choice may depend on the panel's M without breaking the row-panel invariance.
    const bool pair = ((m + 255) / 256) * ((n + 255) / 256) > 16;
    for (int64_t c0 = 0; c0 < k; c0 += kChunkK) {
        GemmLaunch gc = g;
        const int64_t kcp = round4(k - c0 < kChunkK ? k - c0 : kChunkK);
        gc.k = 3 * kcp;
        gc.A = A3 + 3 * c0;
        gc.lda = lda3;
        gc.B = g.transB ? B3 + 3 * c0 : B3 + 3 * c0 * ldb3;
        gc.ldb = ldb3;
        if (c0 > 0) {
            gc.beta = 1.f;
            gc.C_in = g.C_out;
            gc.ldc_in = g.ldc_out;
        }
        e = pair ? launch_tc_gemm_2sm(gc, false) : launch_tc_gemm(gc, false);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace compar
