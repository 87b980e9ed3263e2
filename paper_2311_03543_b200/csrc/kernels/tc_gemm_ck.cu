// Variant (c), cluster split-K form "tc_*_ck": two 1-SM tcgen05 CTAs (a cluster) share one output
// tile and split its K, then reduce through distributed shared memory.  sm_100a.
//
// Same math as tc_gemm.cu (C_out = alpha*A*B + beta*C_in, BF16 / TF32 in, FP32 TMEM accumulation;
// DESIGN.md R1-R6).  Why a variant: on single-wave shapes every tcgen05 form is bound by the MMAs
// one SM issues along K — a K = 16 `tcgen05.mma` costs ~140 cycles even at N = 64
// (profiles/r02_single_wave_trace.md) — so halving each SM's K halves the mainloop, at the price of
// one DSMEM exchange.  Structure (one tile per cluster, non-persistent):
//   CTA r of the cluster computes the 128 x BN tile over k-blocks [r*h, (r+1)*h) (h = ceil(kb/2):
//   the split is a function of K alone, so row panels stay bitwise equal to the unsplit problem);
//   warp 0 TMA producer (the first ring-full of loads issued before the block barrier), warp 1
//   TMEM allocator + MMA issuer, warps 2..5 epilogue (TMEM lane quarter q = warp % 4);
//   cluster barrier 1 (both rings idle) -> each epilogue warp copies its 32 accumulator rows
//   (tcgen05.ld) into the OWNER CTA's receive buffer (rows [0,64) -> CTA 0, [64,128) -> CTA 1;
//   st.shared::cluster, slot = this CTA's rank; the buffer aliases the drained ring) ->
//   cluster barrier 2 -> each CTA reduces its 64 rows in rank order (slot 0 + slot 1: fixed, so the
//   result is deterministic) and writes alpha*sum + beta*C_in with row-coalesced float4 accesses.
#include <cuda.h>

#include <mutex>

#include "kernels.h"
#include "ptx.cuh"
#include "tmap.h"

namespace compar {
namespace {

constexpr int kThreadsK = 192;

#ifdef COMPAR_TRACE
// Development-only phase stamps of CTA 0 (tools/trace_pair.py run2, -DCOMPAR_TRACE build).
__device__ unsigned long long g_trace2[16];
#define TRACE2(i)                                                                             \
    do {                                                                                      \
        if (blockIdx.x == 0) g_trace2[i] = clock64();                                        \
    } while (0)
#define TRACE2_GT(i)                                                                          \
    do {                                                                                      \
        if (blockIdx.x == 0) {                                                                \
            unsigned long long t;                                                             \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));                           \
            g_trace2[i] = t;                                                                  \
        }                                                                                     \
    } while (0)
#else
#define TRACE2(i) ((void)0)
#define TRACE2_GT(i) ((void)0)
#endif

template <bool kBF16, bool kTransB, int kBN>
struct TcKCfg {
    static constexpr int BM = 128, BN = kBN;
    static constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;     // one accumulator
    static constexpr int ELEM = kBF16 ? 2 : 4;
    static constexpr int BK = 128 / ELEM;
    static constexpr int UMMA_K = 32 / ELEM;
    static constexpr int STAGES = 4;
    static constexpr uint32_t A_BYTES = BM * 128;
    static constexpr uint32_t B_BYTES = BN * 128;
    static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int B_ATOM_N = 128 / ELEM;
    static constexpr int B_BOXES = kTransB ? 1 : BN / B_ATOM_N;
    static constexpr uint32_t B_BOX_BYTES = kTransB ? B_BYTES : BK * 128;
    static constexpr bool B_BASE32 = !kBF16 && !kTransB;
    static constexpr uint32_t B_SBO = B_BASE32 ? 512 : 1024;
    static constexpr uint32_t B_LAYOUT = B_BASE32 ? 1 : 2;
    static constexpr uint32_t RING_BYTES = STAGES * STAGE_BYTES;
    static constexpr uint32_t RECV_BYTES = 2u * 64u * BN * 4u;     // [slot][64 rows][BN] FP32
    static constexpr uint32_t DATA_BYTES = RING_BYTES > RECV_BYTES ? RING_BYTES : RECV_BYTES;
    static constexpr uint32_t SMEM = DATA_BYTES + 1024 + 512;
    static constexpr uint32_t IDESC = (1u << 4) | ((kBF16 ? 1u : 2u) << 7) | ((kBF16 ? 1u : 2u) << 10) |
                                      ((kTransB ? 0u : 1u) << 16) | ((uint32_t(BN) >> 3) << 17) |
                                      ((uint32_t(BM) >> 4) << 24);
};

struct TcKParams {
    int64_t m, n, k;
    float alpha, beta;
    const float *C_in;
    int64_t ldc_in;
    float *C_out;
    int64_t ldc_out;
    int m_blocks, n_blocks, num_kb, kb_half;
    int cvec;   // 16-byte C accesses allowed (ld % 4 == 0, 16-byte aligned)
};

// Byte offset of (slot, row, 4-column group g4) in a receive buffer: a row's 32-column chunk c is
// 128 contiguous bytes whose eight 16-byte groups are rotated by the row (g' = (g + row) & 7), so a
// warp writing 32 rows of one chunk spreads over the banks.
template <int BN>
__device__ __forceinline__ uint32_t recv_off(int slot, int row, int g4) {
    const int c = g4 >> 3, g = g4 & 7;
    return static_cast<uint32_t>((((slot * 64 + row) * BN + c * 32) * 4) + (((g + row) & 7) << 4));
}

template <bool kBF16, bool kTransB, int kBN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsK, 1)
    tc_gemm_ck_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcKParams p) {
    using C = TcKCfg<kBF16, kTransB, kBN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t smem0 = ptx::smem_u32(smem);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::DATA_BYTES);
    const uint32_t full0 = ptx::smem_u32(bars);
    const uint32_t empty0 = full0 + 8 * C::STAGES;
    const uint32_t tfull = empty0 + 8 * C::STAGES;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + C::DATA_BYTES + 480);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        TRACE2_GT(10);
        TRACE2(0);
    }
    const uint32_t rank = ptx::cluster_ctarank();
    const int tile = static_cast<int>(blockIdx.x >> 1);
    const int mb = tile / p.n_blocks, nb = tile - (tile / p.n_blocks) * p.n_blocks;
    const int kb0 = rank ? p.kb_half : 0;
    const int kb1 = rank ? p.num_kb : p.kb_half;
    const int nk = kb1 - kb0;

    auto load_stage = [&](int stage, int kb) {
        const uint32_t sa = smem0 + stage * C::STAGE_BYTES;
        const uint32_t sb = sa + C::A_BYTES;
        const uint32_t fb = full0 + 8 * stage;
        ptx::mbar_arrive_expect_tx(fb, C::STAGE_BYTES);
        ptx::tma_load_2d(sa, &tmA, fb, kb * C::BK, mb * C::BM);
        if (kTransB) {
            ptx::tma_load_2d(sb, &tmB, fb, kb * C::BK, nb * C::BN);
        } else {
#pragma unroll
            for (int b = 0; b < C::B_BOXES; ++b)
                ptx::tma_load_2d(sb + b * C::B_BOX_BYTES, &tmB, fb, nb * C::BN + b * C::B_ATOM_N, kb * C::BK);
        }
    };
    int early = 0;
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        for (int s = 0; s < C::STAGES; ++s) {
            ptx::mbar_init(full0 + 8 * s, 1);
            ptx::mbar_init(empty0 + 8 * s, 1);
        }
        ptx::mbar_init(tfull, 1);
        ptx::fence_mbar_init();
        early = nk < C::STAGES ? nk : C::STAGES;     // the ring's first loads, before the block barrier
        for (int i = 0; i < early; ++i) load_stage(i, kb0 + i);
    }
    if (warp == 1) ptx::tmem_alloc<C::TMEM_COLS>(ptx::smem_u32(tmem_slot));
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) TRACE2(1);

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer: this CTA's half of K
            int stage = early % C::STAGES;
            uint32_t phase = early == C::STAGES ? 1u : 0u;
            for (int i = early; i < nk; ++i) {
                ptx::mbar_wait(empty0 + 8 * stage, phase ^ 1);
                load_stage(stage, kb0 + i);
                if (++stage == C::STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {  // ---------------- MMA issuer
        const uint64_t adesc0 = ptx::smem_desc_sw128(smem0, 16, 1024);
        const uint64_t bdesc0 = kTransB ? ptx::smem_desc_sw128(smem0 + C::A_BYTES, 16, 1024)
                                        : ptx::smem_desc(smem0 + C::A_BYTES, C::B_BOX_BYTES, C::B_SBO, C::B_LAYOUT);
        int stage = 0;
        uint32_t phase = 0;
        for (int i = 0; i < nk; ++i) {
            ptx::mbar_wait(full0 + 8 * stage, phase);
            if (i == 0 && lane == 0) TRACE2(2);
            ptx::tc_fence_after();
            if (lane == 0) {
                const uint32_t so = stage * C::STAGE_BYTES;
                const uint64_t as = ptx::desc_adv(adesc0, so), bs = ptx::desc_adv(bdesc0, so);
#pragma unroll
                for (int j = 0; j < C::BK / C::UMMA_K; ++j) {
                    const uint64_t adesc = ptx::desc_adv(as, j * 32);
                    const uint64_t bdesc = ptx::desc_adv(bs, kTransB ? j * 32 : j * C::UMMA_K * 128);
                    if (kBF16)
                        ptx::mma_bf16(tmem_base, adesc, bdesc, C::IDESC, (i | j) != 0);
                    else
                        ptx::mma_tf32(tmem_base, adesc, bdesc, C::IDESC, (i | j) != 0);
                }
                ptx::tc_commit(empty0 + 8 * stage);
            }
            __syncwarp();
            if (++stage == C::STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }
        if (lane == 0) ptx::tc_commit(tfull);
        __syncwarp();
    }
    // epilogue warps: this thread's C_in values (rows ew + 4 i of the CTA's 64, columns lane * 4 +
    // 128 j) are fetched while the mainloop runs — issued together, not one dependent round trip
    // per row in the reduction below
    constexpr int kCj = (C::BN + 127) / 128;
    float4 cin[16][kCj];
    const int ew = warp - 2;
    if (warp >= 2) {
        const bool ldc = p.beta != 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
#pragma unroll
            for (int j = 0; j < kCj; ++j) {
                cin[i][j] = make_float4(0.f, 0.f, 0.f, 0.f);
                const int64_t grow = static_cast<int64_t>(mb) * C::BM + static_cast<int64_t>(rank) * 64 + ew + 4 * i;
                const int col = lane * 4 + 128 * j;
                const int64_t gcol = static_cast<int64_t>(nb) * C::BN + col;
                if (ldc && col < C::BN && grow < p.m && p.cvec && gcol + 4 <= p.n)
                    cin[i][j] = ptx::ldg128_now(p.C_in + grow * p.ldc_in + gcol);
            }
        }
        ptx::mbar_wait(tfull, 0);                    // the accumulator is complete
        ptx::tc_fence_after();
        if (warp == 2 && lane == 0) TRACE2(3);
    }
    // both CTAs' rings are idle (every MMA read its stage; every load landed): the receive buffers
    // (aliasing the rings) may be written from either CTA
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    if (threadIdx.x == 64) TRACE2(4);
    if (warp >= 2) {
        const int q = warp & 3;                      // TMEM lanes / tile rows [32q, 32q + 32)
        const uint32_t owner = static_cast<uint32_t>(q >> 1);
        const int row = (q & 1) * 32 + lane;         // row inside the owner's 64
        const uint32_t dst = ptx::mapa_rank(smem0, owner);
        const uint32_t tq = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
        uint32_t r[32], rn[32];
        ptx::tmem_ld_32x32b_x32(tq, r);
        ptx::tmem_ld_wait();
#pragma unroll 1
        for (int c = 0; c < C::BN / 32; ++c) {
            if (c + 1 < C::BN / 32) ptx::tmem_ld_32x32b_x32(tq + (c + 1) * 32, rn);   // next chunk in flight
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                const uint32_t a = dst + recv_off<C::BN>(static_cast<int>(rank), row, c * 8 + g);
                asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(r[4 * g]),
                             "r"(r[4 * g + 1]), "r"(r[4 * g + 2]), "r"(r[4 * g + 3])
                             : "memory");
            }
            if (c + 1 < C::BN / 32) {
                ptx::tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; ++e) r[e] = rn[e];
            }
        }
    }
    if (threadIdx.x == 64) TRACE2(5);
    ptx::tc_fence_before();
    ptx::cluster_sync();                             // both partials of every owned row have landed
    if (threadIdx.x == 64) TRACE2(6);
    if (warp >= 2) {
        // rows [64 rank, 64 rank + 64) of the tile: 16 per warp, 4 consecutive columns per lane; in
        // groups of kG rows, both partial slots read for the whole group before any store
        const bool ldc = p.beta != 0.f;
        constexpr int kG = 8 / kCj;
#pragma unroll
        for (int i0 = 0; i0 < 16; i0 += kG) {
            float4 s0[kG][kCj], s1[kG][kCj];
#pragma unroll
            for (int i = 0; i < kG; ++i) {
#pragma unroll
                for (int j = 0; j < kCj; ++j) {
                    const int col = lane * 4 + 128 * j;
                    if (col < C::BN) {
                        s0[i][j] = ptx::lds128(smem0 + recv_off<C::BN>(0, ew + 4 * (i0 + i), col >> 2));
                        s1[i][j] = ptx::lds128(smem0 + recv_off<C::BN>(1, ew + 4 * (i0 + i), col >> 2));
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < kG; ++i) {
                const int rr = ew + 4 * (i0 + i);
                const int64_t grow = static_cast<int64_t>(mb) * C::BM + static_cast<int64_t>(rank) * 64 + rr;
                float *cout = p.C_out + grow * p.ldc_out;
#pragma unroll
                for (int j = 0; j < kCj; ++j) {
                    const int col = lane * 4 + 128 * j;
                    const int64_t gcol = static_cast<int64_t>(nb) * C::BN + col;
                    if (col >= C::BN || grow >= p.m || gcol >= p.n) continue;
                    const float4 cij = cin[i0 + i][j];
                    float o[4] = {p.alpha * (s0[i][j].x + s1[i][j].x), p.alpha * (s0[i][j].y + s1[i][j].y),
                                  p.alpha * (s0[i][j].z + s1[i][j].z), p.alpha * (s0[i][j].w + s1[i][j].w)};
                    if (p.cvec && gcol + 4 <= p.n) {
                        if (ldc) {
                            o[0] = fmaf(p.beta, cij.x, o[0]);
                            o[1] = fmaf(p.beta, cij.y, o[1]);
                            o[2] = fmaf(p.beta, cij.z, o[2]);
                            o[3] = fmaf(p.beta, cij.w, o[3]);
                        }
                        *reinterpret_cast<float4 *>(cout + gcol) = make_float4(o[0], o[1], o[2], o[3]);
                    } else {                         // ragged / unaligned edge: scalar
                        const float *cr = p.C_in + grow * p.ldc_in;
                        for (int e = 0; e < 4 && gcol + e < p.n; ++e) {
                            float v = o[e];
                            if (ldc) v = fmaf(p.beta, cr[gcol + e], v);
                            cout[gcol + e] = v;
                        }
                    }
                }
            }
        }
    }
    if (threadIdx.x == 64) TRACE2(7);
    __syncthreads();
    if (threadIdx.x == 0) {
        TRACE2(8);
        TRACE2_GT(11);
    }
    if (warp == 1) ptx::tmem_dealloc<C::TMEM_COLS>(tmem_base);
}

template <bool kBF16, bool kTransB, int kBN>
cudaError_t launch_tck_t(const GemmLaunch &g) {
    using C = TcKCfg<kBF16, kTransB, kBN>;
    static std::once_flag attr_once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once, [] {
        attr_err = cudaFuncSetAttribute(tc_gemm_ck_kernel<kBF16, kTransB, kBN>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    });
    if (attr_err != cudaSuccess) return attr_err;
    CUtensorMap ta, tb;
    if (!get_tmap_2d(&ta, g.A, C::ELEM, g.m, g.k, g.lda, C::BM, C::BK, Swz::B128)) return cudaErrorInvalidValue;
    bool ok = kTransB ? get_tmap_2d(&tb, g.B, C::ELEM, g.n, g.k, g.ldb, C::BN, C::BK, Swz::B128)
                      : get_tmap_2d(&tb, g.B, C::ELEM, g.k, g.n, g.ldb, C::BK, C::B_ATOM_N,
                                    C::B_BASE32 ? Swz::B128_32B : Swz::B128);
    if (!ok) return cudaErrorInvalidValue;
    TcKParams p;
    p.m = g.m, p.n = g.n, p.k = g.k;
    p.alpha = g.alpha, p.beta = g.beta;
    p.C_in = g.C_in, p.ldc_in = g.ldc_in, p.C_out = g.C_out, p.ldc_out = g.ldc_out;
    p.m_blocks = static_cast<int>((g.m + C::BM - 1) / C::BM);
    p.n_blocks = static_cast<int>((g.n + C::BN - 1) / C::BN);
    p.num_kb = static_cast<int>((g.k + C::BK - 1) / C::BK);
    p.kb_half = tc_clusterk_half(g.k, kBF16);
    p.cvec = ((g.ldc_out & 3) == 0) && ((reinterpret_cast<uintptr_t>(g.C_out) & 15) == 0) &&
             (g.beta == 0.f || (((g.ldc_in & 3) == 0) && ((reinterpret_cast<uintptr_t>(g.C_in) & 15) == 0)));
    if (p.num_kb < 2) return cudaErrorInvalidValue;
    const int64_t tiles = static_cast<int64_t>(p.m_blocks) * p.n_blocks;
    if (2 * tiles > INT32_MAX) return cudaErrorInvalidValue;
    tc_gemm_ck_kernel<kBF16, kTransB, kBN><<<static_cast<unsigned>(2 * tiles), kThreadsK, C::SMEM, g.stream>>>(ta, tb, p);
    return cudaGetLastError();
}

}  // namespace

#ifdef COMPAR_TRACE
int trace2_read(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_trace2, sizeof(g_trace2)) == cudaSuccess ? 0 : -1;
}
#endif

cudaError_t launch_tc_gemm_ck(const GemmLaunch &g, bool bf16) {
    // Tile width: the narrowest of 64 / 128 / 256 whose 2 CTAs per tile fit one wave — most SMs
    // busy, since a K = 16 MMA costs about the same at any N (profiles/r02_single_wave_trace.md);
    // 256 when none fits.  Every element's k split and order are the same for any width
    // (bitwise-identical C).
    const int64_t mb = (g.m + 127) / 128;
    int bn = 256;
    for (int w : {64, 128}) {
        if (2 * mb * ((g.n + w - 1) / w) <= g.num_sms) {
            bn = w;
            break;
        }
    }
    if (knobs_of(g).tc1_bn == 256 || knobs_of(g).tc1_bn == 128 || knobs_of(g).tc1_bn == 64) bn = knobs_of(g).tc1_bn;
    if (bn == 64) {
        if (bf16) return g.transB ? launch_tck_t<true, true, 64>(g) : launch_tck_t<true, false, 64>(g);
        return g.transB ? launch_tck_t<false, true, 64>(g) : launch_tck_t<false, false, 64>(g);
    }
    if (bn == 128) {
        if (bf16) return g.transB ? launch_tck_t<true, true, 128>(g) : launch_tck_t<true, false, 128>(g);
        return g.transB ? launch_tck_t<false, true, 128>(g) : launch_tck_t<false, false, 128>(g);
    }
    if (bf16) return g.transB ? launch_tck_t<true, true, 256>(g) : launch_tck_t<true, false, 256>(g);
    return g.transB ? launch_tck_t<false, true, 256>(g) : launch_tck_t<false, false, 256>(g);
}

cudaError_t preload_tck_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaSuccess;
#define COMPAR_PRELOAD_TCK(B, T, N) \
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, tc_gemm_ck_kernel<B, T, N>);
    COMPAR_PRELOAD_TCK(true, false, 256)
    COMPAR_PRELOAD_TCK(true, true, 256)
    COMPAR_PRELOAD_TCK(false, false, 256)
    COMPAR_PRELOAD_TCK(false, true, 256)
    COMPAR_PRELOAD_TCK(true, false, 128)
    COMPAR_PRELOAD_TCK(true, true, 128)
    COMPAR_PRELOAD_TCK(false, false, 128)
    COMPAR_PRELOAD_TCK(false, true, 128)
    COMPAR_PRELOAD_TCK(true, false, 64)
    COMPAR_PRELOAD_TCK(true, true, 64)
    COMPAR_PRELOAD_TCK(false, false, 64)
    COMPAR_PRELOAD_TCK(false, true, 64)
#undef COMPAR_PRELOAD_TCK
    return e;
}

}  // namespace compar

#ifdef COMPAR_TRACE
extern "C" int compar_trace2_read(unsigned long long *out) { return compar::trace2_read(out); }
#endif
