// Variant (c), CTA-pair form "tc_*_2sm": tcgen05.mma.cta_group::2 GEMM for sm_100a.
//
// Same math and epilogue as tc_gemm.cu (C_out = alpha*A*B + beta*C_in, BF16 / TF32 in, FP32
// TMEM accumulation; R1-R6), but two SMs of a TPC cooperate on a 256 x 256 output
// tile: CTA r of the pair loads rows [128 r, 128 r + 128) of the A tile and
// columns [128 r, 128 r + 128) of the B tile; the leader CTA (rank 0) issues one
// tcgen05.mma.cta_group::2 M=256 N=256 per UMMA_K slice, which reads A and B halves from both
// CTAs' shared memory and accumulates each CTA's 128 rows in its own TMEM.  Per SM this halves
// the B traffic (L2 -> SMEM and SMEM -> tensor core) relative to the 1-SM 128 x 256 tile.
//
// Synchronisation (all mbarriers at identical smem offsets in both CTAs):
//   full[s]   leader only; count 1 (leader arrive.expect_tx(both CTAs' bytes)); both CTAs'
//             TMA loads (cta_group::2) complete_tx on it;
//   empty[s]  each CTA; the leader's tcgen05.commit multicasts an arrival to both;
//   tfull[a]  each CTA; leader commit multicast when accumulator a is final;
//   tempty[a] leader only; count 8 = 4 epilogue warps x 2 CTAs (remote arrivals);
//   rfull[r]  each CTA: tile id r of the dynamic schedule published (leader producer writes
//             both CTAs' ring slots through DSMEM and arrives on both);
//   rempty[r] leader only; count 10 = leader MMA + 4 leader epilogue + peer producer + 4 peer
//             epilogue warps.
// Tiles come from a global atomic counter drawn by the leader's producer (see sched.cpp).
#include <cuda.h>

#include <mutex>

#include "kernels.h"
#include "ptx.cuh"
#include "tmap.h"

namespace compar {
namespace {

constexpr int kThreads2 = 192;
constexpr int kGroupM2 = 8;  // default 256-row cluster tiles per raster band (COMPAR_TC_GROUP overrides)
constexpr int kRing2 = 4;

template <bool kBF16, bool kTransB>
struct Tc2Cfg {
    static constexpr int BM = 128;              // A rows per CTA (UMMA_M = 256 per pair)
    static constexpr int BN = 256;              // UMMA_N; each CTA holds BN/2 columns of B
    static constexpr int BN_CTA = BN / 2;
    static constexpr int ELEM = kBF16 ? 2 : 4;
    static constexpr int BK = 128 / ELEM;
    static constexpr int UMMA_K = 32 / ELEM;
    static constexpr int STAGES = 6;
    static constexpr uint32_t A_BYTES = BM * 128;
    static constexpr uint32_t B_BYTES = BN_CTA * 128;
    static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int B_ATOM_N = 128 / ELEM;
    static constexpr int B_BOXES = kTransB ? 1 : BN_CTA / B_ATOM_N;
    static constexpr uint32_t B_BOX_BYTES = kTransB ? B_BYTES : BK * 128;
    static constexpr bool B_BASE32 = !kBF16 && !kTransB;
    static constexpr uint32_t B_SBO = B_BASE32 ? 512 : 1024;
    static constexpr uint32_t B_LAYOUT = B_BASE32 ? 1 : 2;
    static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + 1024 + 512;
    static constexpr uint32_t IDESC = (1u << 4) | ((kBF16 ? 1u : 2u) << 7) | ((kBF16 ? 1u : 2u) << 10) |
                                      ((kTransB ? 0u : 1u) << 16) | ((uint32_t(BN) >> 3) << 17) |
                                      ((uint32_t(2 * BM) >> 4) << 24);
};

struct Tc2Params {
    int64_t m, n, k;
    float alpha, beta;
    const float *C_in;
    int64_t ldc_in;
    float *C_out;
    int64_t ldc_out;
    int m_blocks, n_blocks, num_kb;  // m_blocks in 256-row pair tiles
    int group_m;
    int cvec;
    int *sched;  // {next, done}
};

// group > 0: bands of `group` m-blocks, m fastest inside a band; group < 0: bands of -group
// n-blocks, n fastest (the transposed raster).
__device__ __forceinline__ void tile_coords2(int t, int m_blocks, int n_blocks, int group, int &mb, int &nb) {
    if (group < 0) {
        tile_coords2(t, n_blocks, m_blocks, -group, nb, mb);
        return;
    }
    const int per_group = group * n_blocks;
    const int g = t / per_group;
    const int first_m = g * group;
    const int gm = min(m_blocks - first_m, group);
    const int r = t - g * per_group;
    mb = first_m + r % gm;
    nb = r / gm;
}

__device__ __forceinline__ uint32_t peer_addr(uint32_t local, uint32_t peer_rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(peer_rank));
    return r;
}

template <bool kBF16, bool kTransB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    tc_gemm_2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       Tc2Params p) {
    using C = Tc2Cfg<kBF16, kTransB>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE_BYTES);
    const uint32_t full0 = ptx::smem_u32(bars);
    const uint32_t empty0 = full0 + 8 * C::STAGES;
    const uint32_t tfull0 = empty0 + 8 * C::STAGES;
    const uint32_t tempty0 = tfull0 + 16;
    const uint32_t rfull0 = tempty0 + 16;
    const uint32_t rempty0 = rfull0 + 8 * kRing2;
    const uint32_t ring0 = rempty0 + 8 * kRing2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + C::STAGES * C::STAGE_BYTES + 480);
    const uint32_t smem0 = ptx::smem_u32(smem);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        for (int s = 0; s < C::STAGES; ++s) {
            ptx::mbar_init(full0 + 8 * s, 1);
            ptx::mbar_init(empty0 + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(tfull0 + 8 * a, 1);
            ptx::mbar_init(tempty0 + 8 * a, 8);
        }
        for (int r = 0; r < kRing2; ++r) {
            ptx::mbar_init(rfull0 + 8 * r, 1);
            ptx::mbar_init(rempty0 + 8 * r, 10);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc_2sm<512>(ptx::smem_u32(tmem_slot));
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int num_tiles = p.m_blocks * p.n_blocks;
    const uint32_t rempty_leader = ptx::leader_addr(rempty0);
    // Consumer side of the tile ring (both CTAs): the i-th tile of this pair.
    auto next_tile = [&](int i) -> int {
        const int slot = i % kRing2;
        ptx::mbar_wait_cluster(rfull0 + 8 * slot, (i / kRing2) & 1);
        const int t = static_cast<int>(ptx::ld_shared_u32(ring0 + 4 * slot));
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(rempty_leader + 8 * slot);
        return t;
    };

    if (warp == 0) {
        if (lane == 0) {  // ---------------- scheduler (leader) + TMA producer (both CTAs)
            int stage = 0;
            uint32_t phase = 0;
            for (int i = 0;; ++i) {
                int t;
                if (leader) {
                    const int slot = i % kRing2;
                    ptx::mbar_wait_cluster(rempty0 + 8 * slot, ((i / kRing2) & 1) ^ 1);
                    t = atomicAdd(&p.sched[0], 1);
                    ptx::st_shared_u32(ring0 + 4 * slot, static_cast<uint32_t>(t));
                    ptx::st_shared_cluster_u32(peer_addr(ring0 + 4 * slot, 1), static_cast<uint32_t>(t));
                    ptx::mbar_arrive(rfull0 + 8 * slot);
                    ptx::mbar_arrive_cluster(peer_addr(rfull0 + 8 * slot, 1));
                } else {  // single-lane consumer (no __syncwarp: the other lanes are parked)
                    const int slot = i % kRing2;
                    ptx::mbar_wait_cluster(rfull0 + 8 * slot, (i / kRing2) & 1);
                    t = static_cast<int>(ptx::ld_shared_u32(ring0 + 4 * slot));
                    ptx::mbar_arrive_cluster(rempty_leader + 8 * slot);
                }
                if (t >= num_tiles) break;
                int mb, nb;
                tile_coords2(t, p.m_blocks, p.n_blocks, p.group_m, mb, nb);
                const int32_t arow = mb * 2 * C::BM + static_cast<int32_t>(rank) * C::BM;
                const int32_t bcol = nb * C::BN + static_cast<int32_t>(rank) * C::BN_CTA;
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    ptx::mbar_wait(empty0 + 8 * stage, phase ^ 1);
                    const uint32_t sa = smem0 + stage * C::STAGE_BYTES;
                    const uint32_t sb = sa + C::A_BYTES;
                    const uint32_t fb_local = full0 + 8 * stage;
                    const uint32_t fb = ptx::leader_addr(fb_local);
                    // Only the leader arrives (count 1) and expects both CTAs' bytes; the peer's TMA
                    // bytes can land before that arrive (tx-count transiently negative) but the phase
                    // cannot complete without it, and the peer cannot run a phase ahead because it
                    // waits on its own empty[s], released only after the leader consumed stage s.
                    // (A remote arrive here would need a release.cluster fence = MEMBAR.GPU per k-step.)
                    if (leader) ptx::mbar_arrive_expect_tx(fb_local, 2 * C::STAGE_BYTES);
                    ptx::tma_load_2d_2sm(sa, &tmA, fb, kb * C::BK, arow);
                    if (kTransB) {
                        ptx::tma_load_2d_2sm(sb, &tmB, fb, kb * C::BK, bcol);
                    } else {
#pragma unroll
                        for (int b = 0; b < C::B_BOXES; ++b)
                            ptx::tma_load_2d_2sm(sb + b * C::B_BOX_BYTES, &tmB, fb, bcol + b * C::B_ATOM_N,
                                                 kb * C::BK);
                    }
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
            if (leader) {  // last pair out re-arms the counters for the next launch on this stream
                __threadfence();
                if (atomicAdd(&p.sched[1], 1) == static_cast<int>(gridDim.x >> 1) - 1) {
                    p.sched[0] = 0;
                    p.sched[1] = 0;
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {  // ---------------- MMA issuer (leader CTA only)
            int stage = 0;
            uint32_t phase = 0;
            for (int local = 0;; ++local) {
                const int t = next_tile(local);
                if (t >= num_tiles) break;
                const int acc = local & 1;
                const uint32_t acc_phase = (local >> 1) & 1;
                ptx::mbar_wait_cluster(tempty0 + 8 * acc, acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * C::BN;
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    ptx::mbar_wait(full0 + 8 * stage, phase);
                    ptx::tc_fence_after();
                    if (lane == 0) {
                        const uint32_t so = stage * C::STAGE_BYTES;
                        const uint64_t adesc0 = ptx::smem_desc(smem0, 16, 1024, 2);
                        const uint64_t bdesc0 = kTransB ? ptx::smem_desc(smem0 + C::A_BYTES, 16, 1024, 2)
                                                        : ptx::smem_desc(smem0 + C::A_BYTES, C::B_BOX_BYTES, C::B_SBO,
                                                                         C::B_LAYOUT);
                        const uint64_t as = ptx::desc_adv(adesc0, so), bs = ptx::desc_adv(bdesc0, so);
#pragma unroll
                        for (int j = 0; j < C::BK / C::UMMA_K; ++j) {
                            const uint64_t adesc = ptx::desc_adv(as, j * 32);
                            const uint64_t bdesc = ptx::desc_adv(bs, kTransB ? j * 32 : j * C::UMMA_K * 128);
                            if (kBF16)
                                ptx::mma_bf16_2sm(d_tmem, adesc, bdesc, C::IDESC, (kb | j) != 0);
                            else
                                ptx::mma_tf32_2sm(d_tmem, adesc, bdesc, C::IDESC, (kb | j) != 0);
                        }
                        ptx::tc_commit_2sm_mc(empty0 + 8 * stage, 0x3);
                    }
                    __syncwarp();
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (lane == 0) ptx::tc_commit_2sm_mc(tfull0 + 8 * acc, 0x3);
                __syncwarp();
            }
        }
    } else {  // ---------------- epilogue warps 2..5 (both CTAs, own TMEM rows)
        const int q = warp & 3;
        const uint32_t tempty_leader = ptx::leader_addr(tempty0);
        for (int local = 0;; ++local) {
            const int t = next_tile(local);
            if (t >= num_tiles) break;
            int mb, nb;
            tile_coords2(t, p.m_blocks, p.n_blocks, p.group_m, mb, nb);
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            ptx::mbar_wait(tfull0 + 8 * acc, acc_phase);
            ptx::tc_fence_after();
            const int64_t row = static_cast<int64_t>(mb) * 2 * C::BM + rank * C::BM + q * 32 + lane;
            const bool row_ok = row < p.m;
            float *crow = p.C_out + row * p.ldc_out;
            const float *cin = p.C_in + row * p.ldc_in;
#pragma unroll 1
            for (int c = 0; c < C::BN / 32; ++c) {
                uint32_t r[32];
                ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * C::BN + c * 32, r);
                ptx::tmem_ld_wait();
                const int64_t col0 = static_cast<int64_t>(nb) * C::BN + c * 32;
                if (!row_ok || col0 >= p.n) continue;
                if (p.cvec && col0 + 32 <= p.n) {
#pragma unroll
                    for (int v = 0; v < 8; ++v) {
                        float4 o;
                        o.x = p.alpha * __uint_as_float(r[4 * v + 0]);
                        o.y = p.alpha * __uint_as_float(r[4 * v + 1]);
                        o.z = p.alpha * __uint_as_float(r[4 * v + 2]);
                        o.w = p.alpha * __uint_as_float(r[4 * v + 3]);
                        if (p.beta != 0.f) {
                            const float4 ci = *reinterpret_cast<const float4 *>(cin + col0 + 4 * v);
                            o.x = fmaf(p.beta, ci.x, o.x);
                            o.y = fmaf(p.beta, ci.y, o.y);
                            o.z = fmaf(p.beta, ci.z, o.z);
                            o.w = fmaf(p.beta, ci.w, o.w);
                        }
                        *reinterpret_cast<float4 *>(crow + col0 + 4 * v) = o;
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        if (col0 + e < p.n) {
                            float o = p.alpha * __uint_as_float(r[e]);
                            if (p.beta != 0.f) o = fmaf(p.beta, cin[col0 + e], o);
                            crow[col0 + e] = o;
                        }
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(tempty_leader + 8 * acc);
        }
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_2sm<512>(tmem_base);
    }
}

template <bool kBF16, bool kTransB>
cudaError_t launch_tc2_t(const GemmLaunch &g) {
    using C = Tc2Cfg<kBF16, kTransB>;
    static std::once_flag attr_once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once, [] {
        attr_err = cudaFuncSetAttribute(tc_gemm_2sm_kernel<kBF16, kTransB>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    });
    if (attr_err != cudaSuccess) return attr_err;
    CUtensorMap ta, tb;
    if (!get_tmap_2d(&ta, g.A, C::ELEM, g.m, g.k, g.lda, C::BM, C::BK, Swz::B128)) return cudaErrorInvalidValue;
    bool ok = kTransB ? get_tmap_2d(&tb, g.B, C::ELEM, g.n, g.k, g.ldb, C::BN_CTA, C::BK, Swz::B128)
                      : get_tmap_2d(&tb, g.B, C::ELEM, g.k, g.n, g.ldb, C::BK, C::B_ATOM_N,
                                    C::B_BASE32 ? Swz::B128_32B : Swz::B128);
    if (!ok) return cudaErrorInvalidValue;
    Tc2Params p;
    p.m = g.m, p.n = g.n, p.k = g.k;
    p.alpha = g.alpha, p.beta = g.beta;
    p.C_in = g.C_in, p.ldc_in = g.ldc_in, p.C_out = g.C_out, p.ldc_out = g.ldc_out;
    p.m_blocks = static_cast<int>((g.m + 2 * C::BM - 1) / (2 * C::BM));
    p.n_blocks = static_cast<int>((g.n + C::BN - 1) / C::BN);
    p.num_kb = static_cast<int>((g.k + C::BK - 1) / C::BK);
    p.group_m = knobs_of(g).tc2_rowstore_group != 0 ? knobs_of(g).tc2_rowstore_group : kGroupM2;
    p.cvec = ((g.ldc_out & 3) == 0) && ((reinterpret_cast<uintptr_t>(g.C_out) & 15) == 0) &&
             (g.beta == 0.f || (((g.ldc_in & 3) == 0) && ((reinterpret_cast<uintptr_t>(g.C_in) & 15) == 0)));
    p.sched = sched_workspace(g.stream);
    if (!p.sched) return cudaErrorMemoryAllocation;
    const int tiles = p.m_blocks * p.n_blocks;
    const int max_clusters = g.num_sms / 2;
    const int clusters = tiles < max_clusters ? tiles : max_clusters;
    tc_gemm_2sm_kernel<kBF16, kTransB><<<2 * clusters, kThreads2, C::SMEM, g.stream>>>(ta, tb, p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_tc_gemm_2sm(const GemmLaunch &g, bool bf16) {
    // C movable by TMA (16-byte aligned, ldc * 4 % 16 == 0): the TMA-epilogue form of the same
    // pair tile (tc_gemm_2sm_mc.cu; 134 vs 164 us on config 5a).  Otherwise: row stores.
    if (tma_compatible(g.C_out, g.ldc_out, 4) && (g.beta == 0.f || tma_compatible(g.C_in, g.ldc_in, 4)))
        return launch_tc_gemm_pairs(g, bf16);
    if (bf16) return g.transB ? launch_tc2_t<true, true>(g) : launch_tc2_t<true, false>(g);
    return g.transB ? launch_tc2_t<false, true>(g) : launch_tc2_t<false, false>(g);
}

cudaError_t preload_tc2_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, tc_gemm_2sm_kernel<true, false>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, tc_gemm_2sm_kernel<true, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, tc_gemm_2sm_kernel<false, false>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, tc_gemm_2sm_kernel<false, true>);
    return e;
}

}  // namespace compar
