// Variant (c), wide CTA-pair form "tc_*_2sm_w": tcgen05.mma.cta_group::2 with a 256 x 512 pair tile.
//
// Same math as tc_gemm.cu / tc_gemm_2sm.cu (C_out = alpha*A*B + beta*C_in, BF16 / TF32 in, FP32
// TMEM accumulation; R1-R6).  Each CTA of the pair owns 128 rows x 512 columns of the
// output: per K-step the leader issues TWO M=256 N=256 MMAs (pair columns [0,256) and
// [256,512)) that share the A tile, so per SM the L2 -> SMEM traffic per FLOP is 3/4 of the
// 256 x 256 pair tile and 1/2 of the 1-SM 128 x 256 tile (on a power-capped B200 the
// bytes moved per FLOP set the clock).  The two accumulators fill all 512 TMEM columns, so a
// tile's epilogue is not overlapped with the next tile's MMAs; the producer keeps prefetching the
// next tile's K-blocks meanwhile, and the epilogue itself is asynchronous bulk traffic:
//   per 32 x 32 chunk: TMA load of C_in (issued two chunks ahead) -> tcgen05.ld -> alpha*acc +
//   beta*C_in in registers -> st.shared (SWIZZLE_128B layout) -> TMA store of C_out,
// double-buffered per epilogue warp, so C moves as full 128-byte lines and out-of-range rows /
// columns are clipped by the TMA unit (no predication).
//
// B column split (cta_group::2 takes N/2 columns of B from each CTA, at the same smem offset):
// CTA r holds, per accumulator h, pair columns [256 h + 128 r, +128) as 128/ATOM MN-atoms.
// Synchronisation as in tc_gemm_2sm.cu, with one accumulator set: tfull (leader commit multicast),
// tempty (leader only, count 8 = 4 epilogue warps x 2 CTAs); cbar[w][b]: C_in chunk landed.
// Eligibility adds the TMA rule for C: 16-byte aligned C_in/C_out, ldc * 4 % 16 == 0.
//
// World mode (row panels + broadcast of B; kernels.h WorldLaunch): on a rank that
// receives B slab by slab, the producers wait per tile for the slab's "landed" flag (written on
// the comm stream after the slab's copy) and the tiles are visited column-major, so one
// persistent launch consumes the slabs as they arrive; a slab-packed row-major B is read through
// a 3-D tensor map {column in slab, k, slab}.  A helper launch started after the broadcast (on
// the SMs NCCL used) shares the tile counter with the main launch.
#include <cuda.h>

#include <mutex>

#include "kernels.h"
#include "ptx.cuh"
#include "tmap.h"

namespace compar {
namespace {

constexpr int kEpiWarpsW = 4;
constexpr int kThreadsW = 64 + 32 * kEpiWarpsW;
constexpr int kGroupW = 4;
constexpr int kRingW = 4;
constexpr int kDelayW = 24;  // default epilogue-overlap delay in k-steps (COMPAR_TCW_DELAY overrides)

template <bool kBF16, bool kTransB>
struct TcWCfg {
    static constexpr int BM = 128;               // A rows per CTA (UMMA_M = 256 per pair)
    static constexpr int BN = 512;               // pair tile columns = 2 accumulators of 256
    static constexpr int ELEM = kBF16 ? 2 : 4;
    static constexpr int BK = 128 / ELEM;
    static constexpr int UMMA_K = 32 / ELEM;
    static constexpr int STAGES = 4;
    static constexpr uint32_t A_BYTES = BM * 128;             // 16 KB
    static constexpr uint32_t BH_BYTES = 128 * 128;           // one 128-column half-chunk: 16 KB
    static constexpr uint32_t STAGE_BYTES = A_BYTES + 2 * BH_BYTES;
    static constexpr int B_ATOM_N = 128 / ELEM;
    static constexpr int B_BOXES = kTransB ? 1 : 128 / B_ATOM_N;   // per 128-column chunk
    static constexpr uint32_t B_BOX_BYTES = kTransB ? BH_BYTES : BK * 128;
    static constexpr bool B_BASE32 = !kBF16 && !kTransB;
    static constexpr uint32_t B_SBO = B_BASE32 ? 512 : 1024;
    static constexpr uint32_t B_LAYOUT = B_BASE32 ? 1 : 2;
    static constexpr uint32_t EPI_BYTES = kEpiWarpsW * 2 * 4096;   // 2 x (32 x 32 fp32) per epilogue warp
    static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 512;
    static constexpr uint32_t IDESC = (1u << 4) | ((kBF16 ? 1u : 2u) << 7) | ((kBF16 ? 1u : 2u) << 10) |
                                      ((kTransB ? 0u : 1u) << 16) | ((256u >> 3) << 17) | ((256u >> 4) << 24);
};

struct TcWParams {
    int64_t m, n, k;
    float alpha, beta;
    int m_blocks, n_blocks, num_kb;  // 256-row x 512-column pair tiles
    int group_m;
    int delay;       // k-steps of accumulator half 0 issued before half 1 is needed (epilogue overlap)
    int *sched;
    // world mode (WorldLaunch): slab flags, 3-D slab-packed B, counter shared with a helper launch
    const unsigned *flags;   // nullptr: B is resident
    unsigned seq;
    int slab_w;              // columns per slab (a multiple of 512)
    int b3d;                 // 1: tmB is the 3-D map of the slab-packed row-major B
    int static_first;        // clusters take tile cl first (0: every tile from the counter)
    int counter_base;        // first tile handed out by the counter
    int arm_total;           // clusters of all launches sharing the counter (last one re-arms it)
};

__device__ __forceinline__ void tile_coords_w(int t, int m_blocks, int n_blocks, int group, int &mb, int &nb) {
    const int per_group = group * n_blocks;
    const int g = t / per_group;
    const int first_m = g * group;
    const int gm = min(m_blocks - first_m, group);
    const int r = t - g * per_group;
    mb = first_m + r % gm;
    nb = r / gm;
}

// World mode (B arriving column slab by column slab): tile columns are visited in groups of
// 1, 1, 2, 4, 8, 8, ... columns — the first tiles need only the first slabs — and inside a group in
// bands of `group` pair rows, so a band's A rows are re-read once per group instead of once per
// column (a plain column-major order re-reads the whole A panel for every 512-column strip).
__device__ __forceinline__ void tile_coords_world(int t, int m_blocks, int n_blocks, int group, int &mb, int &nb) {
    int c0 = 0, cw = 1;
    for (int g = 0;; ++g) {
        cw = g < 2 ? 1 : min(8, 1 << (g - 1));
        if (c0 + cw > n_blocks) cw = n_blocks - c0;
        const int cnt = m_blocks * cw;
        if (t < cnt || c0 + cw >= n_blocks) break;
        t -= cnt;
        c0 += cw;
    }
    const int per_band = group * cw;
    const int band = t / per_band;
    const int first_m = band * group;
    const int gm = min(m_blocks - first_m, group);
    const int r = t - band * per_band;
    mb = first_m + r % gm;
    nb = c0 + r / gm;
}

__device__ __forceinline__ uint32_t peer_addr_w(uint32_t local, uint32_t peer_rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(peer_rank));
    return r;
}

template <bool kBF16, bool kTransB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsW, 1)
    tc_gemm_2sm_wide_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                            const __grid_constant__ CUtensorMap tmCo, const __grid_constant__ CUtensorMap tmCi,
                            TcWParams p) {
    using C = TcWCfg<kBF16, kTransB>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t smem0 = ptx::smem_u32(smem);
    const uint32_t epi0 = smem0 + C::STAGES * C::STAGE_BYTES;          // 1024-aligned chunk buffers
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE_BYTES + C::EPI_BYTES);
    const uint32_t full0 = ptx::smem_u32(bars);
    const uint32_t empty0 = full0 + 8 * C::STAGES;
    const uint32_t tfull = empty0 + 8 * C::STAGES;
    const uint32_t tempty = tfull + 8;            // [2]: accumulator half h drained (leader)
    const uint32_t rfull0 = tempty + 16;
    const uint32_t rempty0 = rfull0 + 8 * kRingW;
    const uint32_t cbar0 = rempty0 + 8 * kRingW;                        // 2 per epilogue warp
    const uint32_t ring0 = cbar0 + 16 * kEpiWarpsW;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + C::STAGES * C::STAGE_BYTES + C::EPI_BYTES + 480);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    constexpr int kConsumers = 2 + 2 * kEpiWarpsW;   // leader MMA + peer producer + 2 x epilogue warps
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        ptx::prefetch_tmap(&tmCo);
        ptx::prefetch_tmap(&tmCi);
        for (int s = 0; s < C::STAGES; ++s) {
            ptx::mbar_init(full0 + 8 * s, 1);
            ptx::mbar_init(empty0 + 8 * s, 1);
        }
        ptx::mbar_init(tfull, 1);
        ptx::mbar_init(tempty, 2 * kEpiWarpsW);
        ptx::mbar_init(tempty + 8, 2 * kEpiWarpsW);
        for (int r = 0; r < kRingW; ++r) {
            ptx::mbar_init(rfull0 + 8 * r, 1);
            ptx::mbar_init(rempty0 + 8 * r, kConsumers);
        }
        for (int b = 0; b < 2 * kEpiWarpsW; ++b) ptx::mbar_init(cbar0 + 8 * b, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc_2sm<512>(ptx::smem_u32(tmem_slot));
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int num_tiles = p.m_blocks * p.n_blocks;
    const uint32_t rempty_leader = ptx::leader_addr(rempty0);
    // tile 0 of cluster cl is tile cl (no ring round trip, no atomic before the first loads);
    // tile i >= 1 comes through ring index i - 1 from the global counter, from counter_base on
    // (a helper launch has no static tile: its tile i is ring index i)
    const int cl = static_cast<int>(blockIdx.x >> 1);
    const int sf = p.static_first;
    auto next_tile = [&](int i) -> int {  // whole-warp consumer of the tile ring
        if (i == 0 && sf) return cl;
        const int slot = (i - sf) % kRingW;
        ptx::mbar_wait_cluster(rfull0 + 8 * slot, ((i - sf) / kRingW) & 1);
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
                const int slot = (i - sf) % kRingW;
                if (i == 0 && sf) {
                    t = cl;
                } else if (leader) {
                    ptx::mbar_wait_cluster(rempty0 + 8 * slot, (((i - sf) / kRingW) & 1) ^ 1);
                    t = p.counter_base + atomicAdd(&p.sched[0], 1);
                    ptx::st_shared_u32(ring0 + 4 * slot, static_cast<uint32_t>(t));
                    ptx::st_shared_cluster_u32(peer_addr_w(ring0 + 4 * slot, 1), static_cast<uint32_t>(t));
                    ptx::mbar_arrive(rfull0 + 8 * slot);
                    ptx::mbar_arrive_cluster(peer_addr_w(rfull0 + 8 * slot, 1));
                } else {
                    ptx::mbar_wait_cluster(rfull0 + 8 * slot, ((i - sf) / kRingW) & 1);
                    t = static_cast<int>(ptx::ld_shared_u32(ring0 + 4 * slot));
                    ptx::mbar_arrive_cluster(rempty_leader + 8 * slot);
                }
                if (t >= num_tiles) break;
                int mb, nb;
                if (p.flags)
                    tile_coords_world(t, p.m_blocks, p.n_blocks, p.group_m, mb, nb);
                else
                    tile_coords_w(t, p.m_blocks, p.n_blocks, p.group_m, mb, nb);
                const int32_t arow = mb * 2 * C::BM + static_cast<int32_t>(rank) * C::BM;
                const int32_t bcol0 = nb * C::BN + static_cast<int32_t>(rank) * 128;   // + 256 h
                // world mode: this tile's 512 columns lie in slab nb*512 / slab_w; wait until it landed
                const int slab = p.flags ? (nb * C::BN) / p.slab_w : 0;
                if (p.flags) {
                    ptx::spin_until_geq(p.flags + slab, p.seq);
                    ptx::fence_proxy_async_global();
                }
                const int32_t scol0 = bcol0 - slab * p.slab_w;   // column inside the slab (3-D map)
                // Step order: with delay D > 0 (every tile but the CTA's first), the
                // first D k-steps feed accumulator half 0 only, then the same D k-steps half 1 (A
                // re-loaded), then both halves: half 0 restarts while the epilogue still drains half
                // 1.  Each half still sums its k-steps in increasing order (bitwise = D = 0).
                const int D = i == 0 ? 0 : min(p.delay, p.num_kb);
                for (int st = 0; st < p.num_kb + D; ++st) {
                    const int kb = st < D ? st : st < 2 * D ? st - D : st - D;
                    const int hmask = st < D ? 1 : st < 2 * D ? 2 : 3;
                    ptx::mbar_wait(empty0 + 8 * stage, phase ^ 1);
                    const uint32_t sa = smem0 + stage * C::STAGE_BYTES;
                    const uint32_t fb_local = full0 + 8 * stage;
                    const uint32_t fb = ptx::leader_addr(fb_local);
                    if (leader)
                        ptx::mbar_arrive_expect_tx(fb_local, hmask == 3 ? 2 * C::STAGE_BYTES
                                                                         : 2 * (C::A_BYTES + C::BH_BYTES));
                    ptx::tma_load_2d_2sm(sa, &tmA, fb, kb * C::BK, arow);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (!((hmask >> h) & 1)) continue;
                        const uint32_t sb = sa + C::A_BYTES + h * C::BH_BYTES;
                        if (kTransB) {
                            ptx::tma_load_2d_2sm(sb, &tmB, fb, kb * C::BK, bcol0 + 256 * h);
                        } else if (p.b3d) {
#pragma unroll
                            for (int b = 0; b < C::B_BOXES; ++b)
                                ptx::tma_load_3d_2sm(sb + b * C::B_BOX_BYTES, &tmB, fb,
                                                     scol0 + 256 * h + b * C::B_ATOM_N, kb * C::BK, slab);
                        } else {
#pragma unroll
                            for (int b = 0; b < C::B_BOXES; ++b)
                                ptx::tma_load_2d_2sm(sb + b * C::B_BOX_BYTES, &tmB, fb,
                                                     bcol0 + 256 * h + b * C::B_ATOM_N, kb * C::BK);
                        }
                    }
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
            if (leader) {
                __threadfence();
                if (atomicAdd(&p.sched[1], 1) == p.arm_total - 1) {
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
                const int D = local == 0 ? 0 : min(p.delay, p.num_kb);
                ptx::mbar_wait_cluster(tempty, (local & 1) ^ 1);        // half 0 drained
                if (D == 0) ptx::mbar_wait_cluster(tempty + 8, (local & 1) ^ 1);
                ptx::tc_fence_after();
                for (int st = 0; st < p.num_kb + D; ++st) {
                    const int kb = st < D ? st : st < 2 * D ? st - D : st - D;
                    const int hmask = st < D ? 1 : st < 2 * D ? 2 : 3;
                    if (D > 0 && st == D) {                                  // half 1 drained
                        ptx::mbar_wait_cluster(tempty + 8, (local & 1) ^ 1);
                        ptx::tc_fence_after();
                    }
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
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                if (!((hmask >> h) & 1)) continue;
                                const uint64_t bdesc = ptx::desc_adv(
                                    bs, h * C::BH_BYTES + (kTransB ? j * 32 : j * C::UMMA_K * 128));
                                if (kBF16)
                                    ptx::mma_bf16_2sm(tmem_base + 256 * h, adesc, bdesc, C::IDESC, (kb | j) != 0);
                                else
                                    ptx::mma_tf32_2sm(tmem_base + 256 * h, adesc, bdesc, C::IDESC, (kb | j) != 0);
                            }
                        }
                        ptx::tc_commit_2sm_mc(empty0 + 8 * stage, 0x3);
                    }
                    __syncwarp();
                    if (++stage == C::STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (lane == 0) ptx::tc_commit_2sm_mc(tfull, 0x3);
                __syncwarp();
            }
        }
    } else {  // ---------------- epilogue warps 2..5: TMEM lane quarter q, 16 chunks of 32 x 32
        const int q = warp & 3;
        const int ew = warp - 2;
        // staging chunk b of this warp and its C_in barrier (computed: no local-memory arrays)
        auto buf = [&](int b) -> uint32_t { return epi0 + static_cast<uint32_t>(2 * ew + b) * 4096; };
        auto cbar = [&](int b) -> uint32_t { return cbar0 + 16 * ew + 8 * b; };
        uint32_t loads_odd = 0;                           // bit b: odd number of C_in loads into chunk b
        const uint32_t tempty_leader = ptx::leader_addr(tempty);
        const bool ldc = p.beta != 0.f;
        const uint32_t swz = lane * 128;                  // this thread's row in a chunk buffer
        for (int local = 0;; ++local) {
            const int t = next_tile(local);
            if (t >= num_tiles) break;
            int mb, nb;
            if (p.flags)
                    tile_coords_world(t, p.m_blocks, p.n_blocks, p.group_m, mb, nb);
                else
                    tile_coords_w(t, p.m_blocks, p.n_blocks, p.group_m, mb, nb);
            const int32_t row_base = mb * 2 * C::BM + static_cast<int32_t>(rank) * C::BM + q * 32;
            const int32_t col_base = nb * C::BN;
            auto chunk_col = [&](int idx) { return col_base + 256 * (idx >> 3) + 32 * (idx & 7); };
            if (lane == 0) {
                ptx::bulk_wait_read<0>();                 // previous tile's stores have left smem
                if (ldc) {
                    for (int b = 0; b < 2; ++b) {
                        ptx::mbar_arrive_expect_tx(cbar(b), 4096);
                        ptx::tma_load_2d(buf(b), &tmCi, cbar(b), chunk_col(b), row_base);
                    }
                }
            }
            if (ldc) loads_odd ^= 3u;                     // warp-uniform phase bookkeeping
            __syncwarp();
            ptx::mbar_wait(tfull, local & 1);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int idx = 0; idx < 16; ++idx) {
                const int b = idx & 1;
                uint32_t r[32];
                ptx::tmem_ld_32x32b_x32(
                    tmem_base + (static_cast<uint32_t>(q * 32) << 16) + 256 * (idx >> 3) + 32 * (idx & 7), r);
                ptx::tmem_ld_wait();
                if ((idx & 7) == 7) {                     // half idx>>3 is in registers: release it
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive_cluster(tempty_leader + 8 * (idx >> 3));
                }
                if (ldc) {
                    ptx::mbar_wait(cbar(b), ((loads_odd >> b) & 1) ^ 1);
                } else if (idx >= 2) {
                    if (lane == 0) ptx::bulk_wait_read<1>();   // store idx-2 has left buf[b]
                    __syncwarp();
                }
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    const uint32_t a = buf(b) + swz + ((g ^ (lane & 7)) << 4);
                    float4 o;
                    o.x = p.alpha * __uint_as_float(r[4 * g + 0]);
                    o.y = p.alpha * __uint_as_float(r[4 * g + 1]);
                    o.z = p.alpha * __uint_as_float(r[4 * g + 2]);
                    o.w = p.alpha * __uint_as_float(r[4 * g + 3]);
                    if (ldc) {
                        const float4 ci = ptx::lds128(a);
                        o.x = fmaf(p.beta, ci.x, o.x);
                        o.y = fmaf(p.beta, ci.y, o.y);
                        o.z = fmaf(p.beta, ci.z, o.z);
                        o.w = fmaf(p.beta, ci.w, o.w);
                    }
                    ptx::sts128(a, o);
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    ptx::tma_store_2d(&tmCo, buf(b), chunk_col(idx), row_base);
                    ptx::bulk_commit();
                    if (ldc && idx + 2 < 16) {            // refill buf[b] with chunk idx+2 once it is read
                        ptx::bulk_wait_read<0>();
                        ptx::mbar_arrive_expect_tx(cbar(b), 4096);
                        ptx::tma_load_2d(buf(b), &tmCi, cbar(b), chunk_col(idx + 2), row_base);
                    }
                }
                if (ldc && idx + 2 < 16) loads_odd ^= 1u << b;
                __syncwarp();
            }
        }
        if (lane == 0) ptx::bulk_wait<0>();               // all C stores complete before exit
        __syncwarp();
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_2sm<512>(tmem_base);
    }
}

template <bool kBF16, bool kTransB>
cudaError_t launch_tcw_t(const GemmLaunch &g) {
    using C = TcWCfg<kBF16, kTransB>;
    static std::once_flag attr_once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once, [] {
        attr_err = cudaFuncSetAttribute(tc_gemm_2sm_wide_kernel<kBF16, kTransB>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    });
    if (attr_err != cudaSuccess) return attr_err;
    const WorldLaunch *w = g.world;
    const bool slabs = w && w->flags;
    if (slabs && (w->slab_w <= 0 || w->slab_w % C::BN != 0)) return cudaErrorInvalidValue;
    const bool b3d = slabs && !kTransB && w->nslab > 1;
    CUtensorMap ta, tb, tco, tci;
    if (!get_tmap_2d(&ta, g.A, C::ELEM, g.m, g.k, g.lda, C::BM, C::BK, Swz::B128)) return cudaErrorInvalidValue;
    bool ok;
    if (kTransB)
        ok = get_tmap_2d(&tb, g.B, C::ELEM, g.n, g.k, g.ldb, 128, C::BK, Swz::B128);
    else if (b3d)   // slab-packed: plane j = slab j, a K x slab_w row-major block (not cached: per task)
        ok = make_tmap_3d(&tb, g.B, C::ELEM, w->nslab, g.k, w->slab_w, w->slab_w, g.k * w->slab_w, C::BK, C::B_ATOM_N,
                          C::B_BASE32 ? Swz::B128_32B : Swz::B128);
    else
        ok = get_tmap_2d(&tb, g.B, C::ELEM, g.k, g.n, g.ldb, C::BK, C::B_ATOM_N, C::B_BASE32 ? Swz::B128_32B : Swz::B128);
    if (!ok) return cudaErrorInvalidValue;
    if (!get_tmap_2d(&tco, g.C_out, 4, g.m, g.n, g.ldc_out, 32, 32, Swz::B128)) return cudaErrorInvalidValue;
    if (g.beta != 0.f) {
        if (!get_tmap_2d(&tci, g.C_in, 4, g.m, g.n, g.ldc_in, 32, 32, Swz::B128)) return cudaErrorInvalidValue;
    } else {
        tci = tco;  // unused
    }
    const Knobs &kn = knobs_of(g);
    TcWParams p;
    p.m = g.m, p.n = g.n, p.k = g.k;
    p.alpha = g.alpha, p.beta = g.beta;
    p.m_blocks = static_cast<int>((g.m + 2 * C::BM - 1) / (2 * C::BM));
    p.n_blocks = static_cast<int>((g.n + C::BN - 1) / C::BN);
    p.num_kb = static_cast<int>((g.k + C::BK - 1) / C::BK);
    // raster bands of 4 pair-rows; 8 when K <= 8192, where a band's A rows plus the B columns a
    // wave touches then fit in L2 (8192^3: 741 vs 752 us; 32768^3 keeps 4: 52.3 vs 53.7 ms);
    // (world mode: the same bands inside geometric column groups, tile_coords_world)
    p.group_m = kn.tcw_group > 0 ? kn.tcw_group : (g.k <= 8192 ? 2 * kGroupW : kGroupW);
    p.delay = kn.tcw_delay;
    p.sched = sched_workspace(g.stream);
    if (!p.sched) return cudaErrorMemoryAllocation;
    p.flags = slabs ? w->flags : nullptr;
    p.seq = slabs ? w->seq : 0;
    p.slab_w = slabs ? w->slab_w : C::BN;
    p.b3d = b3d ? 1 : 0;
    const int tiles = p.m_blocks * p.n_blocks;
    const int helper = (w && w->helper_sms >= 2 && w->helper_stream) ? w->helper_sms / 2 : 0;   // clusters
    const int max_clusters = g.num_sms / 2 - helper;
    const int clusters = tiles < max_clusters ? tiles : max_clusters;
    if (clusters < 1) return cudaSuccess;
    const int extra = tiles > clusters ? (helper < tiles - clusters ? helper : tiles - clusters) : 0;
    p.static_first = 1;
    p.counter_base = clusters;
    p.arm_total = clusters + extra;
    if (extra > 0) {   // the helper must not touch the counter before earlier launches on g.stream re-armed it
        cudaEventRecord(w->helper_done, g.stream);
        cudaStreamWaitEvent(w->helper_stream, w->helper_done, 0);
    }
    tc_gemm_2sm_wide_kernel<kBF16, kTransB><<<2 * clusters, kThreadsW, C::SMEM, g.stream>>>(ta, tb, tco, tci, p);
    cudaError_t e = cudaGetLastError();
    if (w) w->launches = 1;
    if (e != cudaSuccess || extra == 0) return e;
    // helper: starts once the broadcast has released its SMs, takes every tile from the counter
    if (w->helper_after) cudaStreamWaitEvent(w->helper_stream, w->helper_after, 0);
    p.static_first = 0;
    tc_gemm_2sm_wide_kernel<kBF16, kTransB><<<2 * extra, kThreadsW, C::SMEM, w->helper_stream>>>(ta, tb, tco, tci, p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    w->launches = 2;
    cudaEventRecord(w->helper_done, w->helper_stream);
    return cudaStreamWaitEvent(g.stream, w->helper_done, 0);
}

}  // namespace

cudaError_t launch_tc_gemm_2sm_wide(const GemmLaunch &g, bool bf16) {
    if (bf16) return g.transB ? launch_tcw_t<true, true>(g) : launch_tcw_t<true, false>(g);
    return g.transB ? launch_tcw_t<false, true>(g) : launch_tcw_t<false, false>(g);
}

cudaError_t preload_tcw_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, tc_gemm_2sm_wide_kernel<true, false>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, tc_gemm_2sm_wide_kernel<true, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, tc_gemm_2sm_wide_kernel<false, false>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, tc_gemm_2sm_wide_kernel<false, true>);
    return e;
}

}  // namespace compar
