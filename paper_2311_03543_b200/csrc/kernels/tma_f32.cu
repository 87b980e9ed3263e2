// Variant (b) "tma_f32": TMA-fed, mbarrier-pipelined FP32 FFMA GEMM for sm_100a.
//
// Role: a second hand-written strict-FP32 "CUDA" mmul variant (PAPER.md P:201-205,
// P:220) whose operand movement is Blackwell-native: cp.async.bulk.tensor (TMA) into a
// multi-stage shared-memory ring, completion tracked by mbarrier transaction counts, one
// producer warp and eight FFMA consumer warps.
// C_out = alpha * A * B + beta * C_in (R1-R3).
//
//   * CTA tile 128 x 128, K step 32 (one 128-byte swizzle row of FP32), 4 stages;
//   * A box 128 x 32, SWIZZLE_128B (K-major); B box 32 x 128 unswizzled (row-major B), or
//     128 x 32 SWIZZLE_128B when transB;
//   * consumer thread (tx, ty) owns rows ty + 16 i and columns {4tx.., 64 + 4tx..}
//     (or tx + 16 j for transB): A read as float4 along K (conflict-free under the
//     swizzle), B read as float4 along N;
//   * TMA zero-fills out-of-bounds boxes; the epilogue predicates.
// Eligibility: 16-byte aligned A/B and lda, ldb multiples of 4 (TMA stride rule).
#include <cuda.h>

#include <cstdlib>
#include <mutex>

#include "kernels.h"
#include "ptx.cuh"
#include "tmap.h"

namespace compar {
namespace {

// {c0, c1} = a * {b0, b1} + {c0, c1} as one sm_100 FFMA2 (fma.rn.f32x2): two RN FMAs, bitwise
// equal to two fmaf calls (see simt_f32.cu).
__device__ __forceinline__ void ffma2(float &c0, float &c1, float a, float b0, float b1) {
    unsigned long long c, b, aa;
    asm("mov.b64 %0, {%1, %2};" : "=l"(c) : "f"(c0), "f"(c1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(b0), "f"(b1));
    asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(aa), "l"(b));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(c0), "=f"(c1) : "l"(c));
}

// Tile TB x TB (128, or 64 for grids that would not fill the GPU: 4x the CTAs of a small problem),
// K-step BK = 32 (one 128-byte swizzle row), 4-stage TMA ring.  Each consumer thread owns an 8-row x
// MJ-column micro-tile: 8 x 8 for TB = 128 (256 threads), 8 x 4 for TB = 64 (128 threads: one warp
// per SM sub-partition even when a small grid leaves one CTA per SM).  Every element accumulates its
// k in the same order with the same FMA, so C is bitwise the same for either tile.
constexpr int BK = 32, STAGES = 4;
template <int TB>
struct TmaCfg {
    static constexpr int MJ4 = TB == 128 ? 2 : 1;            // float4 column groups per thread
    static constexpr int MJ = 4 * MJ4;                       // micro-tile columns
    static constexpr int TY = TB / 8;                        // consumer threads along M
    static constexpr int TX = TB / MJ;                       // consumer threads along N
    static constexpr int kConsumers = TX * TY;
    static constexpr int kThreads = kConsumers + 32;
    static constexpr uint32_t A_BYTES = TB * BK * 4, B_BYTES = BK * TB * 4, STAGE_BYTES = A_BYTES + B_BYTES;
    // transB: transposed B stage [BK][TB]; double-buffered for TB = 128 (one CTA per SM), single for
    // TB = 64 so three CTAs still fit an SM
    static constexpr uint32_t T_BYTES = BK * TB * 4;
    static constexpr int kTBufs = TB == 128 ? 2 : 1;
    static constexpr uint32_t smem(bool transB) {
        return STAGES * STAGE_BYTES + (transB ? kTBufs * T_BYTES : 0) + 1024 + 128;
    }
    static constexpr int kMinBlocks = TB == 128 ? 1 : 3;
};

struct TmaParams {
    int64_t m, n, k;
    float alpha, beta;
    const float *C_in;
    int64_t ldc_in;
    float *C_out;
    int64_t ldc_out;
    int num_kb;
    int cvec;
};

// byte offset of the float4 holding (row, k4*4 .. k4*4+3) in a 128-byte-swizzled [rows][32] FP32 tile
__device__ __forceinline__ uint32_t sw128_off(int row, int k4) { return row * 128 + ((k4 ^ (row & 7)) << 4); }

template <bool kTransB, int TB>
__global__ void __launch_bounds__(TmaCfg<TB>::kThreads, TmaCfg<TB>::kMinBlocks)
    tma_f32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TmaParams p) {
    using Cf = TmaCfg<TB>;
    constexpr int BM = TB, BN = TB, TY = Cf::TY, TX = Cf::TX, MJ = Cf::MJ, MJ4 = Cf::MJ4, kConsumers = Cf::kConsumers;
    constexpr uint32_t A_BYTES = Cf::A_BYTES, STAGE_BYTES = Cf::STAGE_BYTES;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned base as an offset into smem_raw (not a uintptr_t round trip), so the compiler
    // keeps the shared address space and the micro-tile reads are LDS, not generic loads
    uint8_t *smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *tbuf = smem + STAGES * STAGE_BYTES;              // transB: kTBufs x [BK][BN] FP32
    uint64_t *bars = reinterpret_cast<uint64_t *>(tbuf + (kTransB ? Cf::kTBufs * Cf::T_BYTES : 0));
    const uint32_t full0 = ptx::smem_u32(bars), empty0 = full0 + 8 * STAGES;
    const uint32_t smem0 = ptx::smem_u32(smem);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM, n0 = static_cast<int64_t>(blockIdx.x) * BN;

    if (tid == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(full0 + 8 * s, 1);
            ptx::mbar_init(empty0 + 8 * s, kConsumers / 32);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();

    if (warp == kConsumers / 32) {  // ---------------- producer warp
        if (lane == 0) {
            for (int kb = 0; kb < p.num_kb; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                ptx::mbar_wait(empty0 + 8 * s, ph ^ 1);
                const uint32_t sa = smem0 + s * STAGE_BYTES, sb = sa + A_BYTES, fb = full0 + 8 * s;
                ptx::mbar_arrive_expect_tx(fb, STAGE_BYTES);
                ptx::tma_load_2d(sa, &tmA, fb, kb * BK, static_cast<int32_t>(m0));
                if (kTransB)
                    ptx::tma_load_2d(sb, &tmB, fb, kb * BK, static_cast<int32_t>(n0));
                else
                    ptx::tma_load_2d(sb, &tmB, fb, static_cast<int32_t>(n0), kb * BK);
            }
        }
        return;
    }

    // ---------------- consumer warps
    const int tx = tid % TX, ty = tid / TX;
    float acc[8][MJ];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < MJ; ++j) acc[i][j] = 0.f;

    for (int kb = 0; kb < p.num_kb; ++kb) {
        const int s = kb % STAGES;
        ptx::mbar_wait(full0 + 8 * s, (kb / STAGES) & 1);
        const uint8_t *sa = smem + s * STAGE_BYTES;
        const uint8_t *sb = sa + A_BYTES;
        if (kTransB) {
            // B^T arrives as [BN rows of n][32 k] (128-byte swizzle); the consumers transpose it into
            // tbuf[kb % kTBufs] = [32 k][BN] so the inner loop below is the row-major one (B columns
            // paired in adjacent registers for FFMA2, each element's k order unchanged).  Double
            // buffering needs one consumer barrier per stage: a warp rewriting buffer (kb+1)&1 has
            // passed barrier kb, which every warp reaches only after its compute on kb-1; a single
            // buffer also needs one before it is rewritten.
            if (Cf::kTBufs == 1 && kb > 0) asm volatile("bar.sync 1, %0;" ::"r"(kConsumers) : "memory");
            float *t = reinterpret_cast<float *>(tbuf + (kb % Cf::kTBufs) * Cf::T_BYTES);
#pragma unroll
            for (int q = 0; q < BN * (BK / 4) / kConsumers; ++q) {
                const int idx = tid + q * kConsumers, r = idx % BN, c = idx / BN;
                const float4 v = *reinterpret_cast<const float4 *>(sb + sw128_off(r, c));
                t[(4 * c + 0) * BN + r] = v.x;
                t[(4 * c + 1) * BN + r] = v.y;
                t[(4 * c + 2) * BN + r] = v.z;
                t[(4 * c + 3) * BN + r] = v.w;
            }
            asm volatile("bar.sync 1, %0;" ::"r"(kConsumers) : "memory");
            sb = reinterpret_cast<const uint8_t *>(t);
        }
        // Fragments one step ahead (double-buffered registers): the A float4s of k-quad k4 + 1 and
        // the B row of k + 1 are read from shared memory before the FFMA2s of k, so an LDS latency
        // is exposed once per stage, not once per k-quad.  Each element's k order is unchanged.
        auto load_a = [&](float4(&a)[8], int k4) {
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = *reinterpret_cast<const float4 *>(sa + sw128_off(ty + TY * i, k4));
        };
        auto load_b = [&](float(&b)[MJ], int kq) {
            const float *brow = reinterpret_cast<const float *>(sb + kq * (BN * 4));
#pragma unroll
            for (int h = 0; h < MJ4; ++h) {
                const float4 bh = *reinterpret_cast<const float4 *>(brow + h * (BN / MJ4) + tx * 4);
                b[4 * h + 0] = bh.x, b[4 * h + 1] = bh.y, b[4 * h + 2] = bh.z, b[4 * h + 3] = bh.w;
            }
        };
        auto fma_k = [&](const float4(&a)[8], int kk, const float(&b)[MJ]) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float av = kk == 0 ? a[i].x : kk == 1 ? a[i].y : kk == 2 ? a[i].z : a[i].w;
#pragma unroll
                for (int j = 0; j < MJ; j += 2) ffma2(acc[i][j], acc[i][j + 1], av, b[j], b[j + 1]);
            }
        };
        float4 a0[8], a1[8];
        float b0[MJ], b1[MJ];
        load_a(a0, 0);
        load_b(b0, 0);
#pragma unroll 1
        for (int k8 = 0; k8 < BK / 8; ++k8) {
            const int q = 8 * k8;               // first k of this pair of k-quads
            const bool more = k8 + 1 < BK / 8;
            load_a(a1, 2 * k8 + 1);
            load_b(b1, q + 1);
            fma_k(a0, 0, b0);
            load_b(b0, q + 2);
            fma_k(a0, 1, b1);
            load_b(b1, q + 3);
            fma_k(a0, 2, b0);
            load_b(b0, q + 4);
            fma_k(a0, 3, b1);
            if (more) load_a(a0, 2 * k8 + 2);
            load_b(b1, q + 5);
            fma_k(a1, 0, b0);
            load_b(b0, q + 6);
            fma_k(a1, 1, b1);
            load_b(b1, q + 7);
            fma_k(a1, 2, b0);
            if (more) load_b(b0, q + 8);
            fma_k(a1, 3, b1);
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(empty0 + 8 * s);
    }

    // ---------------- epilogue
    // alpha * acc in place, then + beta * C_in (o = alpha * acc, then fmaf(beta, C_in, o)); all of
    // C_in is gathered before the first store: C_in may alias C_out, so the compiler cannot hoist a
    // load above an earlier store, and load / store pairs issued in turn would serialise 8 * MJ4
    // memory round trips.  (In place: 159 registers instead of 166, 1.7-1.9 % faster at 3072^3 -
    // 8192^3.)
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < MJ; ++j) acc[i][j] = p.alpha * acc[i][j];
    if (p.beta != 0.f) {
        float ci[8][MJ];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int64_t r = m0 + ty + TY * i;
            const float *cin = p.C_in + r * p.ldc_in;
#pragma unroll
            for (int h = 0; h < MJ4; ++h) {
                const int64_t c = n0 + h * (BN / MJ4) + tx * 4;
                if (r < p.m && p.cvec && c + 3 < p.n) {
                    const float4 v = *reinterpret_cast<const float4 *>(cin + c);
                    ci[i][h * 4 + 0] = v.x, ci[i][h * 4 + 1] = v.y, ci[i][h * 4 + 2] = v.z, ci[i][h * 4 + 3] = v.w;
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) ci[i][h * 4 + j] = r < p.m && c + j < p.n ? cin[c + j] : 0.f;
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < MJ; ++j) acc[i][j] = fmaf(p.beta, ci[i][j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t r = m0 + ty + TY * i;
        if (r >= p.m) continue;
        float *crow = p.C_out + r * p.ldc_out;
#pragma unroll
        for (int h = 0; h < MJ4; ++h) {
            const int64_t c = n0 + h * (BN / MJ4) + tx * 4;
            float o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) o[j] = acc[i][h * 4 + j];
            if (p.cvec && c + 3 < p.n) {
                *reinterpret_cast<float4 *>(crow + c) = make_float4(o[0], o[1], o[2], o[3]);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (c + j < p.n) crow[c + j] = o[j];
            }
        }
    }
}

template <bool kTransB, int TB>
cudaError_t launch_t(const GemmLaunch &g) {
    using Cf = TmaCfg<TB>;
    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [] {
        attr = cudaFuncSetAttribute(tma_f32_kernel<kTransB, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::smem(kTransB));
    });
    if (attr != cudaSuccess) return attr;
    CUtensorMap ta, tb;
    if (!get_tmap_2d(&ta, g.A, 4, g.m, g.k, g.lda, TB, BK, Swz::B128)) return cudaErrorInvalidValue;
    bool ok = kTransB ? get_tmap_2d(&tb, g.B, 4, g.n, g.k, g.ldb, TB, BK, Swz::B128)
                      : get_tmap_2d(&tb, g.B, 4, g.k, g.n, g.ldb, BK, TB, Swz::None);
    if (!ok) return cudaErrorInvalidValue;
    TmaParams p;
    p.m = g.m, p.n = g.n, p.k = g.k, p.alpha = g.alpha, p.beta = g.beta;
    p.C_in = g.C_in, p.ldc_in = g.ldc_in, p.C_out = g.C_out, p.ldc_out = g.ldc_out;
    p.num_kb = static_cast<int>((g.k + BK - 1) / BK);
    p.cvec = ((g.ldc_out & 3) == 0) && ((reinterpret_cast<uintptr_t>(g.C_out) & 15) == 0) &&
             (g.beta == 0.f || (((g.ldc_in & 3) == 0) && ((reinterpret_cast<uintptr_t>(g.C_in) & 15) == 0)));
    dim3 grid(static_cast<unsigned>((g.n + TB - 1) / TB), static_cast<unsigned>((g.m + TB - 1) / TB));
    tma_f32_kernel<kTransB, TB><<<grid, Cf::kThreads, Cf::smem(kTransB), g.stream>>>(ta, tb, p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_tma_f32(const GemmLaunch &g) {
    if ((g.m + 127) / 128 > 65535) return cudaErrorInvalidValue;
    // 64 x 64 tiles (8 x 4 micro-tiles, 128 consumer threads) when 128 x 128 tiles would fill at
    // most three quarters of the SMs (measured: 768^3 81.5 -> 37.1 us, 1024^3 105 -> 72 us,
    // 1280^3 130 -> 120 us; from 1536^3 (144 tiles) the 128 tile's 8 x 8 micro-tiles win).
    // COMPAR_TMA_TILE=128 / 64 (Knobs) forces one.
    const int64_t tiles128 = ((g.m + 127) / 128) * ((g.n + 127) / 128);
    const int force = knobs_of(g).tma_tile;
    const bool small = force == 64 || (force != 128 && 4 * tiles128 <= 3 * static_cast<int64_t>(g.num_sms));
    if (small) return g.transB ? launch_t<true, 64>(g) : launch_t<false, 64>(g);
    return g.transB ? launch_t<true, 128>(g) : launch_t<false, 128>(g);
}

cudaError_t preload_tma_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, tma_f32_kernel<false, 128>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, tma_f32_kernel<true, 128>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, tma_f32_kernel<false, 64>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, tma_f32_kernel<true, 64>);
    return e;
}

}  // namespace compar
