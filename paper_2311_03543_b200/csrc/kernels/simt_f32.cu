// Variant (a) "simt_f32": shared-memory tiled FP32 FFMA GEMM for sm_100a.
//
// Role: the B200 re-design of the paper's hand-written "CUDA" mmul variant
// (PAPER.md P:201-205 [Table 2], P:220 [§3.2]) — strict FP32, no tensor cores.
// C_out = alpha * A * B + beta * C_in (R1-R3).
//
// Design:
//   * CTA tile 128 x 128, K step 8, 256 threads, 8 x 8 register micro-tile per thread split as
//     2 x 2 blocks of 4 x 4 at stride 64 (conflict-free float4 shared loads);
//   * coalesced float4 global loads (vector path when pointers / ld allow), A staged
//     transposed (As[k][m]) so both operands are read as float4 along M / N;
//   * register-prefetch double buffering: tile k+1 is loaded while tile k is multiplied;
//   * any shape: edges are predicated (no padding required), transB supported.
#include <cuda_bf16.h>

#include "kernels.h"

namespace compar {
namespace {

constexpr int BM = 128, BN = 128, BK = 8, THREADS = 256;

__device__ __forceinline__ float to_f32(float x) { return x; }

// Two independent FP32 FMAs in one sm_100 FFMA2 (fma.rn.f32x2): {c0, c1} = a * {b0, b1} + {c0, c1},
// each with one RN rounding exactly as fmaf, so results are bitwise those of scalar FFMA.  The
// broadcast of `a` folds into FFMA2's scalar-operand form (no extra MOV).
__device__ __forceinline__ void ffma2(float &c0, float &c1, float a, float b0, float b1) {
    unsigned long long c, b, aa;
    asm("mov.b64 %0, {%1, %2};" : "=l"(c) : "f"(c0), "f"(c1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(b0), "f"(b1));
    asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(aa), "l"(b));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(c0), "=f"(c1) : "l"(c));
}
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }

// Four consecutive elements of row r starting at column c, widened to FP32 (exact for BF16).
template <bool kVec>
__device__ __forceinline__ float4 load_row4(const float *__restrict__ base, int64_t ld, int64_t r, int64_t c,
                                            int64_t R, int64_t C) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r >= R) return v;
    const float *p = base + r * ld + c;
    if (kVec && c + 3 < C) {
        v = *reinterpret_cast<const float4 *>(p);
    } else {
        if (c + 0 < C) v.x = p[0];
        if (c + 1 < C) v.y = p[1];
        if (c + 2 < C) v.z = p[2];
        if (c + 3 < C) v.w = p[3];
    }
    return v;
}

template <bool kVec>
__device__ __forceinline__ float4 load_row4(const __nv_bfloat16 *__restrict__ base, int64_t ld, int64_t r, int64_t c,
                                            int64_t R, int64_t C) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r >= R) return v;
    const __nv_bfloat16 *p = base + r * ld + c;
    if (kVec && c + 3 < C) {
        const uint2 u = *reinterpret_cast<const uint2 *>(p);   // 4 x BF16 in one 8-byte load
        const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u.x));
        const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u.y));
        v = make_float4(lo.x, lo.y, hi.x, hi.y);
    } else {
        if (c + 0 < C) v.x = to_f32(p[0]);
        if (c + 1 < C) v.y = to_f32(p[1]);
        if (c + 2 < C) v.z = to_f32(p[2]);
        if (c + 3 < C) v.w = to_f32(p[3]);
    }
    return v;
}

// T = float (variant a) or __nv_bfloat16 (simt_bf16: BF16 operands widened exactly to FP32 on load,
// FP32 FFMA accumulation — the any-shape fallback of the BF16 precision class).
template <typename T, bool kVecA, bool kVecB, bool kTransB>
__global__ void __launch_bounds__(THREADS, 2) simt_f32_kernel(GemmLaunch g) {
    __shared__ __align__(16) float As[2][BK][BM + 4];   // +4: the transposed A stores are bank-conflict free
    __shared__ __align__(16) float Bs[2][BK][BN + 4];

    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
    const int64_t n0 = static_cast<int64_t>(blockIdx.x) * BN;
    const T *__restrict__ A = static_cast<const T *>(g.A);
    const T *__restrict__ B = static_cast<const T *>(g.B);

    // Load mapping. A (m x k): thread -> row tid/2, k quad (tid&1)*4.
    const int a_r = tid >> 1, a_k = (tid & 1) * 4;
    // B (k x n): thread -> k row tid/32, n quad (tid&31)*4.  transB (n x k): like A.
    const int b_k = kTransB ? (tid & 1) * 4 : (tid >> 5);
    const int b_n = kTransB ? (tid >> 1) : (tid & 31) * 4;

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    const int64_t nk = (g.k + BK - 1) / BK;
    float4 ra, rb;
    auto gload = [&](int64_t kt) {
        const int64_t k0 = kt * BK;
        ra = load_row4<kVecA>(A, g.lda, m0 + a_r, k0 + a_k, g.m, g.k);
        if (kTransB)
            rb = load_row4<kVecB>(B, g.ldb, n0 + b_n, k0 + b_k, g.n, g.k);
        else
            rb = load_row4<kVecB>(B, g.ldb, k0 + b_k, n0 + b_n, g.k, g.n);
    };
    auto sstore = [&](int buf) {
        As[buf][a_k + 0][a_r] = ra.x;
        As[buf][a_k + 1][a_r] = ra.y;
        As[buf][a_k + 2][a_r] = ra.z;
        As[buf][a_k + 3][a_r] = ra.w;
        if (kTransB) {
            Bs[buf][b_k + 0][b_n] = rb.x;
            Bs[buf][b_k + 1][b_n] = rb.y;
            Bs[buf][b_k + 2][b_n] = rb.z;
            Bs[buf][b_k + 3][b_n] = rb.w;
        } else {
            *reinterpret_cast<float4 *>(&Bs[buf][b_k][b_n]) = rb;
        }
    };

    if (nk > 0) {
        gload(0);
        sstore(0);
    }
    __syncthreads();
    for (int64_t kt = 0; kt < nk; ++kt) {
        const int buf = static_cast<int>(kt & 1);
        if (kt + 1 < nk) gload(kt + 1);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            const float4 a0 = *reinterpret_cast<const float4 *>(&As[buf][kk][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4 *>(&As[buf][kk][64 + ty * 4]);
            const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][64 + tx * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; j += 2) ffma2(acc[i][j], acc[i][j + 1], a[i], b[j], b[j + 1]);
        }
        if (kt + 1 < nk) sstore(buf ^ 1);
        __syncthreads();
    }

    // Epilogue: C_out = alpha*acc + beta*C_in (C_in unread when beta == 0).
    const bool cvec = ((g.ldc_out & 3) == 0) && ((reinterpret_cast<uintptr_t>(g.C_out) & 15) == 0) &&
                      (g.beta == 0.f || (((g.ldc_in & 3) == 0) && ((reinterpret_cast<uintptr_t>(g.C_in) & 15) == 0)));
    // C_in is gathered kRows rows at a time before their stores: C_in may alias C_out, so the
    // compiler cannot hoist a load above an earlier store, and load/store pairs issued in turn
    // would serialise 16 memory round trips (kRows = 2 keeps the epilogue within 128 registers).
    constexpr int kRows = 2;
#pragma unroll
    for (int i0 = 0; i0 < 8; i0 += kRows) {
        float ci[kRows][8];
        if (g.beta != 0.f) {
#pragma unroll
            for (int ii = 0; ii < kRows; ++ii) {
                const int i = i0 + ii;
                const int64_t r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t c = n0 + h * 64 + tx * 4;
                    const float *src = g.C_in + r * g.ldc_in + c;
                    if (r < g.m && cvec && c + 3 < g.n) {
                        const float4 v = *reinterpret_cast<const float4 *>(src);
                        ci[ii][h * 4 + 0] = v.x, ci[ii][h * 4 + 1] = v.y, ci[ii][h * 4 + 2] = v.z, ci[ii][h * 4 + 3] = v.w;
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j) ci[ii][h * 4 + j] = r < g.m && c + j < g.n ? src[j] : 0.f;
                    }
                }
            }
        }
#pragma unroll
        for (int ii = 0; ii < kRows; ++ii) {
            const int i = i0 + ii;
            const int64_t r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
            if (r >= g.m) continue;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t c = n0 + h * 64 + tx * 4;
                float o[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    o[j] = g.alpha * acc[i][h * 4 + j];
                    if (g.beta != 0.f) o[j] = fmaf(g.beta, ci[ii][h * 4 + j], o[j]);
                }
                if (cvec && c + 3 < g.n) {
                    *reinterpret_cast<float4 *>(g.C_out + r * g.ldc_out + c) = make_float4(o[0], o[1], o[2], o[3]);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (c + j < g.n) g.C_out[r * g.ldc_out + c + j] = o[j];
                }
            }
        }
    }
}

template <typename T, bool VA, bool VB, bool TB>
cudaError_t launch_t(const GemmLaunch &g) {
    dim3 grid(static_cast<unsigned>((g.n + BN - 1) / BN), static_cast<unsigned>((g.m + BM - 1) / BM));
    simt_f32_kernel<T, VA, VB, TB><<<grid, THREADS, 0, g.stream>>>(g);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_simt(const GemmLaunch &g) {
    if ((g.m + BM - 1) / BM > 65535) return cudaErrorInvalidValue;
    // 4-element vector loads need ld % 4 == 0 and a 4-element-aligned base (16 B FP32, 8 B BF16)
    const uintptr_t va_mask = 4 * sizeof(T) - 1;
    const bool va = ((g.lda & 3) == 0) && ((reinterpret_cast<uintptr_t>(g.A) & va_mask) == 0);
    const bool vb = ((g.ldb & 3) == 0) && ((reinterpret_cast<uintptr_t>(g.B) & va_mask) == 0);
    if (g.transB) {
        if (va && vb) return launch_t<T, true, true, true>(g);
        if (va) return launch_t<T, true, false, true>(g);
        if (vb) return launch_t<T, false, true, true>(g);
        return launch_t<T, false, false, true>(g);
    }
    if (va && vb) return launch_t<T, true, true, false>(g);
    if (va) return launch_t<T, true, false, false>(g);
    if (vb) return launch_t<T, false, true, false>(g);
    return launch_t<T, false, false, false>(g);
}

}  // namespace

cudaError_t launch_simt_f32(const GemmLaunch &g) { return launch_simt<float>(g); }
cudaError_t launch_simt_bf16(const GemmLaunch &g) { return launch_simt<__nv_bfloat16>(g); }

}  // namespace compar

namespace compar {
cudaError_t preload_simt_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, simt_f32_kernel<float, true, true, false>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, simt_f32_kernel<float, true, true, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, simt_f32_kernel<float, false, false, false>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, simt_f32_kernel<float, false, false, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, simt_f32_kernel<__nv_bfloat16, true, true, false>);
    return e;
}
}  // namespace compar
