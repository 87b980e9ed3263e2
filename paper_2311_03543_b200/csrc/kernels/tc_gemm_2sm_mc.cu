// Variant (c), CTA-pair form "tc_*_2sm" with a TMA epilogue (and its split-K form "tc_*_sk") for
// sm_100a.
//
// Same math as tc_gemm.cu (C_out = alpha*A*B + beta*C_in, BF16 / TF32 in, FP32 TMEM accumulation;
// DESIGN.md R1-R6).  A cluster of two CTAs owns a 256 x BN output tile (BN = 256, or 128 for grids
// that would leave CTA pairs idle): one tcgen05.mma.cta_group::2 M=256 N=BN per UMMA_K slice, each
// CTA holding 128 A rows and BN/2 B columns.  Each CTA's accumulator is 128 x BN (BN TMEM columns),
// so two accumulators alternate and tile i's epilogue overlaps tile i+1's MMAs (the wide kernel's
// 512-column accumulator cannot).  Epilogue as in the wide kernel: TMA load of C_in
// ahead, alpha*acc + beta*C_in in registers, swizzled smem staging, TMA store of C_out.
//
// Synchronisation (mbarriers at identical smem offsets in both CTAs):
//   full[s]   leader; count 1 (leader arrive.expect_tx of both CTAs' bytes);
//   empty[s]  both CTAs; the leader's tcgen05.commit multicast;
//   tfull[a]  both CTAs; the leader's commit multicast;
//   tempty[a] leader; count 8 = 4 epilogue warps x 2 CTAs;
//   rfull/rempty  the tile ring: CTA 0's producer draws tile ids from the global counter
//             (sched.cpp) and publishes them to both CTAs over DSMEM;
//   cbar[w][b] C_in chunk landed (epilogue warp w, buffer b).
// (A cluster-of-4 form sharing B by TMA multicast and a stream-K schedule were measured in round 1,
// not faster — DESIGN.md §5 — and removed.)
#include <cuda.h>

#include <mutex>

#include "kernels.h"
#include "ptx.cuh"
#include "tmap.h"

namespace compar {
namespace {

// Warps: 0 producer + scheduler, 1 MMA, 2..5 and 7..10 epilogue (two per TMEM lane quarter, each
// taking every other 32-column chunk, so a tile's epilogue — exposed on the last tile of every CTA
// pair — takes half the time), 6 second producer.
constexpr int kEpiWarpsM = 8;
constexpr int kThreadsM = 96 + 32 * kEpiWarpsM;
constexpr int kGroupM4 = 4;  // 512-row cluster tiles per raster band (COMPAR_TCM_GROUP overrides)
constexpr int kRingM = 4;

// kDeep (multi-wave launches of 256-wide tiles, where each tile's epilogue overlaps the next tile's
// mainloop): 6 stages and one C staging buffer per epilogue warp instead of 5 and 2 — more A bytes in
// flight per SM for the HBM-bound shapes (config 5a 128.4 -> 126.3 us, 8192^3 742 -> 738 us); the
// single-wave launch keeps the second buffer, whose C_in prefetch its exposed epilogue needs
// (2048^3: 33.3 vs 34.8 us with one).
template <bool kBF16, bool kTransB, int kBN, bool kDeep = false>
struct TcMCfg {
    static constexpr int BM = 128;              // A rows per CTA (UMMA_M = 256 per pair)
    static constexpr int BN = kBN;              // UMMA_N (256, or 128 for grids that leave pairs idle);
                                                // each CTA holds BN/2 columns of B
    static constexpr uint32_t TMEM_COLS = 2 * BN;   // two accumulators
    static constexpr int BN_CTA = BN / 2;
    static constexpr int ELEM = kBF16 ? 2 : 4;
    static constexpr int BK = 128 / ELEM;
    static constexpr int UMMA_K = 32 / ELEM;
    // 256-wide tiles: 5 stages so the 8 epilogue warps' staging (64 KiB) fits beside the ring
    // (kDeep: 6 stages beside 32 KiB)
    static constexpr int STAGES = kBN == 256 && !kDeep ? 5 : 6;
    static constexpr uint32_t A_BYTES = BM * 128;
    static constexpr uint32_t B_BYTES = BN_CTA * 128;
    static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int B_ATOM_N = 128 / ELEM;
    // B boxes of one CTA's BN/2-column slice
    static constexpr int B_BOXES = kTransB ? 2 : BN_CTA / B_ATOM_N;
    static constexpr uint32_t B_BOX_BYTES = B_BYTES / B_BOXES;
    static constexpr bool B_BASE32 = !kBF16 && !kTransB;
    static constexpr uint32_t B_SBO = B_BASE32 ? 512 : 1024;
    static constexpr uint32_t B_LAYOUT = B_BASE32 ? 1 : 2;
    static constexpr uint32_t B_LBO = kTransB ? 16 : BK * 128;   // MN-major: stride between N atoms
    // C_in / C_out staging chunks (32 x 32 FP32) per epilogue warp: a warp handles BN/64 chunks —
    // both of a 128-wide tile are loaded before its accumulator is ready; the 256-wide tile's four
    // cycle through two buffers
    static constexpr int EPI_BUFS = kDeep ? 1 : 2;
    static constexpr uint32_t EPI_BYTES = kEpiWarpsM * EPI_BUFS * 4096;
    static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 1024;
    // chunks per epilogue warp beyond its staging buffers: on a CTA pair's last tile they are staged
    // in the drained ring (LAST_BUFS per warp, one mbarrier each)
    static constexpr int LAST_BUFS = kBN / 64 > EPI_BUFS ? kBN / 64 - EPI_BUFS : 0;
    static constexpr uint32_t IDESC = (1u << 4) | ((kBF16 ? 1u : 2u) << 7) | ((kBF16 ? 1u : 2u) << 10) |
                                      ((kTransB ? 0u : 1u) << 16) | ((uint32_t(BN) >> 3) << 17) |
                                      ((uint32_t(2 * BM) >> 4) << 24);
};

struct TcMParams {
    int64_t m, n, k;
    float alpha, beta;
    int m_blocks, n_blocks, num_kb;  // 256-row x BN-column cluster tiles
    int group_m;
    int *sched;
    int nprod;             // TMA producer warps per CTA (1 or 2)
    // split-K variant (tc_*_sk): every tile's k-blocks are cut into `splits` ranges of
    // ksplit k-blocks; each range is one work item whose raw FP32 partial goes to plane `split` of
    // `spart`; splitk_reduce_kernel then sums the planes in split order (fixed, so the result
    // depends only on (K, splits), never on the schedule) and applies alpha / beta.
    int splits, ksplit;
    float *spart;          // [splits][m padded to 256][n padded to 256] raw FP32 partials
    int64_t spart_ld, spart_plane;
    // single wave (every pair owns at most one tile) with beta != 0: the idle second accumulator's
    // TMEM columns hold the tile's C_in, staged while the mainloop runs
    int tmem_cin;
};

#ifdef COMPAR_TRACE
// Development-only phase stamps (tools/trace_pair.py builds a separate library with -DCOMPAR_TRACE):
// clock64 at fixed points of CTAs 0 and 1, globaltimer at entry / exit.
__device__ unsigned long long g_trace[2][16];
__device__ unsigned long long g_trace_cta[2 * 160];   // globaltimer at entry / exit of CTAs 0..159
// per-item globaltimer stamps of CTAs 0..159, items 0..7: [0] first TMA of the item issued (warp 0),
// [1] accumulator committed (MMA warp, leader), [2] last C_out store issued (epilogue warp 2)
__device__ unsigned long long g_trace_item[160 * 8 * 3];
#define TRACE_ITEM(j, w)                                                                      \
    do {                                                                                      \
        if (blockIdx.x < 160 && (j) < 8) {                                                    \
            unsigned long long t;                                                             \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));                           \
            g_trace_item[(blockIdx.x * 8 + (j)) * 3 + (w)] = t;                               \
        }                                                                                     \
    } while (0)
#define TRACE_CTA(i)                                                                          \
    do {                                                                                      \
        if (blockIdx.x < 160) {                                                               \
            unsigned long long t;                                                             \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));                           \
            g_trace_cta[2 * blockIdx.x + (i)] = t;                                            \
        }                                                                                     \
    } while (0)
#define TRACE(i)                                                                              \
    do {                                                                                      \
        if (blockIdx.x < 2) g_trace[blockIdx.x][i] = clock64();                               \
    } while (0)
#define TRACE_GT(i)                                                                           \
    do {                                                                                      \
        if (blockIdx.x < 2) {                                                                 \
            unsigned long long t;                                                             \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));                           \
            g_trace[blockIdx.x][i] = t;                                                       \
        }                                                                                     \
    } while (0)
#else
#define TRACE(i) ((void)0)
#define TRACE_GT(i) ((void)0)
#define TRACE_CTA(i) ((void)0)
#define TRACE_ITEM(j, w) ((void)0)
#endif

enum { kFull = 0, kSplit = 1 };
struct Item {
    int tile, kb0, kb1, kind;
};

__device__ __forceinline__ void tile_coords_m(int t, int m_blocks, int n_blocks, int group, int &mb, int &nb) {
    const int per_group = group * n_blocks;
    const int g = t / per_group;
    const int first_m = g * group;
    const int gm = min(m_blocks - first_m, group);
    const int r = t - g * per_group;
    mb = first_m + r % gm;
    nb = r / gm;
}

template <bool kBF16, bool kTransB, int kBN, bool kDeep>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsM, 1)
    tc_gemm_2sm_mc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmCo, const __grid_constant__ CUtensorMap tmCi,
                          TcMParams p) {
    using C = TcMCfg<kBF16, kTransB, kBN, kDeep>;
    constexpr int kCluster = 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t smem0 = ptx::smem_u32(smem);
    const uint32_t epi0 = smem0 + C::STAGES * C::STAGE_BYTES;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE_BYTES + C::EPI_BYTES);
    const uint32_t full0 = ptx::smem_u32(bars);
    const uint32_t empty0 = full0 + 8 * C::STAGES;
    const uint32_t tfull0 = empty0 + 8 * C::STAGES;
    const uint32_t tempty0 = tfull0 + 16;
    const uint32_t rfull0 = tempty0 + 16;
    const uint32_t rempty0 = rfull0 + 8 * kRingM;
    const uint32_t cbar0 = rempty0 + 8 * kRingM;
    const uint32_t ring0 = cbar0 + 8 * C::EPI_BUFS * kEpiWarpsM;
    const uint32_t lbar0 = ring0 + 4 * kRingM;   // [warp][LAST_BUFS] C_in chunks of the last tile
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + C::STAGES * C::STAGE_BYTES + C::EPI_BYTES + 1016);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        TRACE_GT(10);
        TRACE(0);
        TRACE_CTA(0);
    }
    const uint32_t rank = ptx::cluster_ctarank();   // 0 (MMA leader) or 1
    const bool leader = rank == 0;
    // consumers of a tile-ring slot: 4 epilogue warps per CTA, the peer's producer, the MMA warp
    // (+ both CTAs' second producer warps when p.nprod == 2)
    const int kConsumers = kCluster * kEpiWarpsM + (kCluster - 1) + 1 + (p.nprod == 2 ? kCluster : 0);
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
        ptx::prefetch_tmap(&tmCo);
        ptx::prefetch_tmap(&tmCi);
        for (int s = 0; s < C::STAGES; ++s) {
            ptx::mbar_init(full0 + 8 * s, 1);
            ptx::mbar_init(empty0 + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(tfull0 + 8 * a, 1);
            ptx::mbar_init(tempty0 + 8 * a, 2 * kEpiWarpsM);
        }
        for (int r = 0; r < kRingM; ++r) {
            ptx::mbar_init(rfull0 + 8 * r, 1);
            ptx::mbar_init(rempty0 + 8 * r, kConsumers);
        }
        for (int b = 0; b < C::EPI_BUFS * kEpiWarpsM; ++b) ptx::mbar_init(cbar0 + 8 * b, 1);
        for (int b = 0; b < C::LAST_BUFS * kEpiWarpsM; ++b) ptx::mbar_init(lbar0 + 8 * b, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc_2sm<C::TMEM_COLS>(ptx::smem_u32(tmem_slot));
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) TRACE(1);

    const int num_tiles = p.m_blocks * p.n_blocks;
    const int num_items = num_tiles * p.splits;                // ring values are work items
    auto dyn_item = [&](int t) -> Item {
        if (p.splits == 1) return Item{t, 0, p.num_kb, kFull};
        const int sidx = t % p.splits;
        const int kb0 = sidx * p.ksplit;
        return Item{t / p.splits, kb0, min(p.num_kb, kb0 + p.ksplit), kSplit};
    };
    const uint32_t rempty_root = ptx::mapa_rank(rempty0, 0);
    const int cl = static_cast<int>(blockIdx.x) / kCluster;   // this cluster's index in the grid
    // Item 0 of cluster cl is item cl (no ring round trip, no atomic on the critical path of the
    // first tile); item j >= 1 comes through ring index j - 1 from the global counter, offset by
    // the number of clusters.
    const int n_cl = static_cast<int>(gridDim.x) / kCluster;
    auto next_item = [&](int j, Item &it) -> bool {  // whole-warp consumer (MMA and epilogue warps)
        if (j == 0) {
            it = dyn_item(cl);
            return true;
        }
        const int slot = (j - 1) % kRingM;
        ptx::mbar_wait_cluster(rfull0 + 8 * slot, ((j - 1) / kRingM) & 1);
        const int t = static_cast<int>(ptx::ld_shared_u32(ring0 + 4 * slot));
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(rempty_root + 8 * slot);
        if (t >= num_items) return false;
        it = dyn_item(t);
        return true;
    };

    if (warp == 0 || warp == 6) {
        // ---------------- scheduler (CTA 0 warp 0) + TMA producers: with p.nprod == 2, warp 0
        // issues the even and warp 6 the odd k-steps (two independent issue streams per SM).
        const int me = warp == 0 ? 0 : 1;
        if (lane == 0 && me < p.nprod) {
            uint32_t kstep = 0;
            for (int i = 0;; ++i) {
                Item it;
                if (i == 0) {
                    it = dyn_item(cl);
                } else {
                    int t;
                    const int slot = (i - 1) % kRingM;
                    if (rank == 0 && me == 0) {
                        ptx::mbar_wait_cluster(rempty0 + 8 * slot, (((i - 1) / kRingM) & 1) ^ 1);
                        t = n_cl + atomicAdd(&p.sched[0], 1);
                        ptx::st_shared_u32(ring0 + 4 * slot, static_cast<uint32_t>(t));
                        ptx::st_shared_cluster_u32(ptx::mapa_rank(ring0 + 4 * slot, 1), static_cast<uint32_t>(t));
                        ptx::mbar_arrive(rfull0 + 8 * slot);
                        ptx::mbar_arrive_cluster(ptx::mapa_rank(rfull0 + 8 * slot, 1));
                    } else {
                        ptx::mbar_wait_cluster(rfull0 + 8 * slot, ((i - 1) / kRingM) & 1);
                        t = static_cast<int>(ptx::ld_shared_u32(ring0 + 4 * slot));
                        ptx::mbar_arrive_cluster(rempty_root + 8 * slot);
                    }
                    if (t >= num_items) break;
                    it = dyn_item(t);
                }
                int mb, nb;
                tile_coords_m(it.tile, p.m_blocks, p.n_blocks, p.group_m, mb, nb);
                const int32_t arow = mb * (kCluster * C::BM) + static_cast<int32_t>(rank) * C::BM;
                const int32_t bcol = nb * C::BN + static_cast<int32_t>(rank) * C::BN_CTA;
                for (int kb = it.kb0; kb < it.kb1; ++kb, ++kstep) {
                    if (p.nprod == 2 && (kstep & 1) != static_cast<uint32_t>(me)) continue;
                    const int stage = static_cast<int>(kstep % C::STAGES);
                    const uint32_t phase = (kstep / C::STAGES) & 1;
                    ptx::mbar_wait_cluster(empty0 + 8 * stage, phase ^ 1);
                    const uint32_t sa = smem0 + stage * C::STAGE_BYTES;
                    const uint32_t sb = sa + C::A_BYTES;
                    const uint32_t fb_local = full0 + 8 * stage;
                    const uint32_t fb = ptx::mapa_rank(fb_local, 0);
                    // The leader arms its barrier with both CTAs' bytes.  Bytes may land before the
                    // arm (transiently negative tx); no CTA runs a phase ahead, because every
                    // producer first waits for empty[s].
                    if (leader) ptx::mbar_arrive_expect_tx(fb_local, 2 * C::STAGE_BYTES);
                    ptx::tma_load_2d_2sm(sa, &tmA, fb, kb * C::BK, arow);
#pragma unroll
                    for (int b = 0; b < C::B_BOXES; ++b) {
                        const int32_t c0 = kTransB ? kb * C::BK : bcol + b * C::B_ATOM_N;
                        const int32_t c1 = kTransB ? bcol + b * (C::BN_CTA / 2) : kb * C::BK;
                        ptx::tma_load_2d_2sm(sb + b * C::B_BOX_BYTES, &tmB, fb, c0, c1);
                    }
                    if (kstep == 0 && me == 0) TRACE(2);
                    if (kb == it.kb0 && me == 0) TRACE_ITEM(i, 0);
                }
            }
            if (rank == 0 && me == 0) {  // last cluster out re-arms the counters for the next launch on this stream
                __threadfence();
                if (atomicAdd(&p.sched[1], 1) == static_cast<int>(gridDim.x / kCluster) - 1) {
                    p.sched[0] = 0;
                    p.sched[1] = 0;
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {  // ---------------- MMA issuer (leader)
            int stage = 0;
            uint32_t phase = 0;
            for (int local = 0;; ++local) {
                Item it;
                if (!next_item(local, it)) break;
                const int acc = local & 1;
                const uint32_t acc_phase = (local >> 1) & 1;
                ptx::mbar_wait_cluster(tempty0 + 8 * acc, acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * C::BN;
                for (int kb = it.kb0; kb < it.kb1; ++kb) {
                    ptx::mbar_wait(full0 + 8 * stage, phase);
                    if (local == 0 && lane == 0) TRACE(3);
                    ptx::tc_fence_after();
                    if (lane == 0) {
                        const uint32_t so = stage * C::STAGE_BYTES;
                        const uint64_t adesc0 = ptx::smem_desc(smem0, 16, 1024, 2);
                        const uint64_t bdesc0 = kTransB ? ptx::smem_desc(smem0 + C::A_BYTES, 16, 1024, 2)
                                                        : ptx::smem_desc(smem0 + C::A_BYTES, C::B_LBO, C::B_SBO,
                                                                         C::B_LAYOUT);
                        const uint64_t as = ptx::desc_adv(adesc0, so), bs = ptx::desc_adv(bdesc0, so);
#pragma unroll
                        for (int j = 0; j < C::BK / C::UMMA_K; ++j) {
                            const uint64_t adesc = ptx::desc_adv(as, j * 32);
                            const uint64_t bdesc = ptx::desc_adv(bs, kTransB ? j * 32 : j * C::UMMA_K * 128);
                            const uint32_t accum = kb != it.kb0 || j != 0;
                            if (kBF16)
                                ptx::mma_bf16_2sm(d_tmem, adesc, bdesc, C::IDESC, accum);
                            else
                                ptx::mma_tf32_2sm(d_tmem, adesc, bdesc, C::IDESC, accum);
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
                if (local == 0 && lane == 0) TRACE(4);
                if (lane == 0) TRACE_ITEM(local, 1);
                __syncwarp();
            }
        }
    } else {  // ---------------- epilogue warps 2..5, 7..10: TMEM lane quarter q, every other 32 x 32 chunk
        const int q = warp & 3;
        const int ew = warp < 6 ? warp - 2 : warp - 3;   // 0..7
        const int half = ew >> 2;                        // this warp's chunks: idx = half + 2 j
        constexpr int NB = C::EPI_BUFS;
        // staging chunk b of this warp and its C_in barrier (computed: no local-memory arrays)
        auto buf = [&](int b) -> uint32_t { return epi0 + static_cast<uint32_t>(NB * ew + b) * 4096; };
        auto cbar = [&](int b) -> uint32_t { return cbar0 + 8 * static_cast<uint32_t>(NB * ew + b); };
        // the last tile's extra C_in chunks: 4 KiB slots of the drained stage ring, and their barriers
        auto lbuf = [&](int x) -> uint32_t { return smem0 + static_cast<uint32_t>(C::LAST_BUFS * ew + x) * 4096; };
        auto lbar = [&](int x) -> uint32_t { return lbar0 + 8 * static_cast<uint32_t>(C::LAST_BUFS * ew + x); };
        uint32_t loads_odd = 0;   // bit b: an odd number of C_in loads issued into chunk b
        const uint32_t tempty_leader = ptx::mapa_rank(tempty0, 0);
        const bool ldc = p.beta != 0.f;
        const uint32_t swz = lane * 128;
        constexpr int kChunks = C::BN / 64;              // per warp
        auto tcol = [&](int j) -> uint32_t { return static_cast<uint32_t>(32 * (half + 2 * j)); };
        for (int local = 0;; ++local) {
            Item it;
            if (!next_item(local, it)) break;
            int mb, nb;
            tile_coords_m(it.tile, p.m_blocks, p.n_blocks, p.group_m, mb, nb);
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            if (it.kind == kSplit) {  // raw partial of k-range `sidx` -> plane sidx of the workspace
                const int sidx = it.kb0 / p.ksplit;
                ptx::mbar_wait(tfull0 + 8 * acc, acc_phase);
                ptx::tc_fence_after();
                const int64_t prow_g = static_cast<int64_t>(mb) * (kCluster * C::BM) + rank * C::BM + q * 32 + lane;
                float *part = p.spart + static_cast<size_t>(sidx) * p.spart_plane + prow_g * p.spart_ld +
                              static_cast<int64_t>(nb) * C::BN;
#pragma unroll 1
                for (int j = 0; j < kChunks; ++j) {
                    uint32_t r[32];
                    ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * C::BN + tcol(j), r);
                    ptx::tmem_ld_wait();
                    if (j == kChunks - 1) {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive_cluster(tempty_leader + 8 * acc);
                    }
#pragma unroll
                    for (int v = 0; v < 8; ++v)
                        __stcg(reinterpret_cast<float4 *>(part + tcol(j)) + v,
                               make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                           __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3])));
                }
                continue;
            }
            const int32_t row_base = mb * (kCluster * C::BM) + static_cast<int32_t>(rank) * C::BM + q * 32;
            const int32_t col_base = nb * C::BN;
            if (lane == 0) {
                ptx::bulk_wait_read<0>();                 // previous tile's stores have left smem
                if (ldc) {
                    for (int b = 0; b < NB && b < kChunks; ++b) {
                        ptx::mbar_arrive_expect_tx(cbar(b), 4096);
                        ptx::tma_load_2d(buf(b), &tmCi, cbar(b), col_base + static_cast<int32_t>(tcol(b)), row_base);
                    }
                }
            }
            if (ldc) loads_odd ^= (1u << NB) - 1;
            __syncwarp();
            // Single wave: this warp's C_in chunks go through its staging buffers into TMEM columns
            // [BN, 2 BN) (the second accumulator, which no later tile uses) before the accumulator is
            // ready — the tile's exposed epilogue then reads C_in from TMEM and only writes C.
            const bool tcin = p.tmem_cin && ldc && local == 0;
            const uint32_t tm_cin = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + C::BN;
            if (tcin) {
#pragma unroll 1
                for (int j = 0; j < kChunks; ++j) {
                    const int b = j % NB;
                    if (j >= NB) {   // buffer b's previous chunk was read by the lanes: reload it
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            ptx::mbar_arrive_expect_tx(cbar(b), 4096);
                            ptx::tma_load_2d(buf(b), &tmCi, cbar(b), col_base + static_cast<int32_t>(tcol(j)), row_base);
                        }
                        loads_odd ^= 1u << b;
                    }
                    ptx::mbar_wait(cbar(b), ((loads_odd >> b) & 1) ^ 1);
                    uint32_t v[32];
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        const float4 c4 = ptx::lds128(buf(b) + swz + ((g ^ (lane & 7)) << 4));
                        v[4 * g + 0] = __float_as_uint(c4.x);
                        v[4 * g + 1] = __float_as_uint(c4.y);
                        v[4 * g + 2] = __float_as_uint(c4.z);
                        v[4 * g + 3] = __float_as_uint(c4.w);
                    }
                    ptx::tmem_st_32x32b_x32(tm_cin + tcol(j), v);
                }
                ptx::tmem_st_wait();
                __syncwarp();
            }
            ptx::mbar_wait(tfull0 + 8 * acc, acc_phase);
            if (local == 0 && warp == 2 && lane == 0) TRACE(5);
            // The pair's last tile: once its accumulator is complete the MMAs have drained the
            // stage ring, and no later item will refill it, so the chunks beyond this warp's staging
            // buffers are all loaded into ring memory now, in parallel (not one after another as
            // staging buffers free up) — the last tile's epilogue is exposed.  "Last" is known when
            // the producer has already published the next ring value as the end marker; a warp
            // that does not see it yet takes the ordinary path (decisions are per warp and safe).
            bool last = false;
            if (C::LAST_BUFS > 0 && ldc && !tcin) {
                if (lane == 0) {
                    const int slot = local % kRingM;
                    if (ptx::mbar_try_wait_cluster(rfull0 + 8 * slot, (local / kRingM) & 1))
                        last = static_cast<int>(ptx::ld_shared_u32(ring0 + 4 * slot)) >= num_items;
                    if (last) {
                        for (int x = 0; x < C::LAST_BUFS; ++x) {
                            ptx::mbar_arrive_expect_tx(lbar(x), 4096);
                            ptx::tma_load_2d(lbuf(x), &tmCi, lbar(x), col_base + static_cast<int32_t>(tcol(NB + x)),
                                             row_base);
                        }
                    }
                }
                last = __shfl_sync(0xffffffffu, last, 0);
            }
            ptx::tc_fence_after();
            const uint32_t tm = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * C::BN;
            // accumulator chunk j+1 is read from TMEM while chunk j is being finished
            uint32_t r[32], rn[32];
            ptx::tmem_ld_32x32b_x32(tm + tcol(0), r);
            ptx::tmem_ld_wait();
#pragma unroll 1
            for (int jj = 0; jj < kChunks; ++jj) {
                const int b = jj % NB;
                if (jj + 1 < kChunks) ptx::tmem_ld_32x32b_x32(tm + tcol(jj + 1), rn);
                const bool tr = local == 0 && warp == 2 && lane == 0 && jj == 1;   // (trace stamps only)
                if (tr) TRACE(12);
                // chunk staged in the drained ring (the last tile's C_in beyond the staging buffers; with
                // tcin — a single wave, so the only tile is the last — the output of those chunks)
                const bool lx = (last || tcin) && jj >= NB && C::LAST_BUFS > 0;
                const uint32_t cb = lx ? lbuf(jj - NB) : buf(b);
                float4 ci[8];
                if (tcin) {                                // C_in from TMEM; buf(b) only stages the output
                    uint32_t cr[32];
                    ptx::tmem_ld_32x32b_x32(tm_cin + tcol(jj), cr);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int g = 0; g < 8; ++g)
                        ci[g] = make_float4(__uint_as_float(cr[4 * g]), __uint_as_float(cr[4 * g + 1]),
                                            __uint_as_float(cr[4 * g + 2]), __uint_as_float(cr[4 * g + 3]));
                } else if (lx) {
                    ptx::mbar_wait(lbar(jj - NB), 0);      // used once per launch: phase 0
                } else if (ldc) {
                    ptx::mbar_wait(cbar(b), ((loads_odd >> b) & 1) ^ 1);
                } else if (jj >= NB) {
                    if (lane == 0) ptx::bulk_wait_read<NB - 1>();
                    __syncwarp();
                }
                if (tr) TRACE(13);
                // all eight C_in vectors first, then the eight results (no load waits behind a store)
                if (ldc && !tcin) {
#pragma unroll
                    for (int g = 0; g < 8; ++g) ci[g] = ptx::lds128(cb + swz + ((g ^ (lane & 7)) << 4));
                }
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    float4 o;
                    o.x = p.alpha * __uint_as_float(r[4 * g + 0]);
                    o.y = p.alpha * __uint_as_float(r[4 * g + 1]);
                    o.z = p.alpha * __uint_as_float(r[4 * g + 2]);
                    o.w = p.alpha * __uint_as_float(r[4 * g + 3]);
                    if (ldc) {
                        o.x = fmaf(p.beta, ci[g].x, o.x);
                        o.y = fmaf(p.beta, ci[g].y, o.y);
                        o.z = fmaf(p.beta, ci[g].z, o.z);
                        o.w = fmaf(p.beta, ci[g].w, o.w);
                    }
                    ptx::sts128(cb + swz + ((g ^ (lane & 7)) << 4), o);
                }
                if (tr) TRACE(9);
                ptx::fence_proxy_async_smem();
                if (tr) TRACE(14);
                __syncwarp();
                if (lane == 0) {
                    ptx::tma_store_2d(&tmCo, cb, col_base + static_cast<int32_t>(tcol(jj)), row_base);
                    ptx::bulk_commit();
                    if (tr) TRACE(15);
                    if (ldc && !last && !tcin && jj + NB < kChunks) {
                        ptx::bulk_wait_read<0>();
                        ptx::mbar_arrive_expect_tx(cbar(b), 4096);
                        ptx::tma_load_2d(buf(b), &tmCi, cbar(b), col_base + static_cast<int32_t>(tcol(jj + NB)), row_base);
                    }
                }
                if (ldc && !last && !tcin && jj + NB < kChunks) loads_odd ^= 1u << b;
                if (jj + 1 < kChunks) {
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 32; ++e) r[e] = rn[e];
                }
                if (jj + 2 == kChunks || kChunks == 1) {   // this warp's last TMEM read has completed:
                    ptx::tc_fence_before();                // free the accumulator for tile + 2
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive_cluster(tempty_leader + 8 * acc);
                }
                __syncwarp();
            }
            if (local == 0 && warp == 2 && lane == 0) TRACE(6);
            if (warp == 2 && lane == 0) TRACE_ITEM(local, 2);
        }
        if (lane == 0) ptx::bulk_wait<0>();
        if (warp == 2 && lane == 0) TRACE(7);
        __syncwarp();
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (threadIdx.x == 0) {
        TRACE(8);
        TRACE_GT(11);
        TRACE_CTA(1);
    }
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_2sm<C::TMEM_COLS>(tmem_base);
    }
}

#ifdef COMPAR_TRACE
int trace_read(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace)) == cudaSuccess ? 0 : -1;
}
int trace_cta_read(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_trace_cta, sizeof(g_trace_cta)) == cudaSuccess ? 0 : -1;
}
int trace_item_read(unsigned long long *out, int clear) {
    if (cudaMemcpyFromSymbol(out, g_trace_item, sizeof(g_trace_item)) != cudaSuccess) return -1;
    if (clear) {
        static unsigned long long z[160 * 8 * 3];
        if (cudaMemcpyToSymbol(g_trace_item, z, sizeof(z)) != cudaSuccess) return -1;
    }
    return 0;
}
#endif

// Split-K epilogue: C_out = alpha * (P_0 + P_1 + ... + P_{S-1}) + beta * C_in, the planes summed in
// split order; 4 consecutive columns per thread (16-byte C accesses: the variant requires TMA-style
// C alignment), grid-stride over rows x column quads.
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float *__restrict__ part, int splits, int64_t ld,
                                                            int64_t plane, int64_t m, int64_t n, float alpha,
                                                            float beta, const float *__restrict__ C_in,
                                                            int64_t ldc_in, float *__restrict__ C_out,
                                                            int64_t ldc_out) {
    const int64_t nq = (n + 3) / 4;
    const int64_t total = m * nq;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t row = i / nq, col = (i - row * nq) * 4;
        const float *pp = part + row * ld + col;
        float4 a = __ldcs(reinterpret_cast<const float4 *>(pp));
        for (int s = 1; s < splits; ++s) {
            const float4 x = __ldcs(reinterpret_cast<const float4 *>(pp + s * plane));
            a.x += x.x, a.y += x.y, a.z += x.z, a.w += x.w;
        }
        float o[4] = {alpha * a.x, alpha * a.y, alpha * a.z, alpha * a.w};
        if (col + 4 <= n) {
            if (beta != 0.f) {
                const float4 ci = *reinterpret_cast<const float4 *>(C_in + row * ldc_in + col);
                o[0] = fmaf(beta, ci.x, o[0]);
                o[1] = fmaf(beta, ci.y, o[1]);
                o[2] = fmaf(beta, ci.z, o[2]);
                o[3] = fmaf(beta, ci.w, o[3]);
            }
            *reinterpret_cast<float4 *>(C_out + row * ldc_out + col) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
            for (int e = 0; e < 4 && col + e < n; ++e) {
                float v = o[e];
                if (beta != 0.f) v = fmaf(beta, C_in[row * ldc_in + col + e], v);
                C_out[row * ldc_out + col + e] = v;
            }
        }
    }
}

template <bool kBF16, bool kTransB, int kBN = 256, bool kDeep = false>
cudaError_t launch_tcm_t(const GemmLaunch &g, int splits = 1) {
    using C = TcMCfg<kBF16, kTransB, kBN, kDeep>;
    constexpr int kCluster = 2;
    static std::once_flag attr_once;
    static cudaError_t attr_err = cudaSuccess;
    static int max_clusters = 0;
    std::call_once(attr_once, [] {
        attr_err = cudaFuncSetAttribute(tc_gemm_2sm_mc_kernel<kBF16, kTransB, kBN, kDeep>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (attr_err != cudaSuccess) return;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at;
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = kCluster, at.val.clusterDim.y = 1, at.val.clusterDim.z = 1;
        cfg.gridDim = dim3(kCluster * 64), cfg.blockDim = dim3(kThreadsM), cfg.dynamicSmemBytes = C::SMEM;
        cfg.attrs = &at, cfg.numAttrs = 1;
        attr_err = cudaOccupancyMaxActiveClusters(&max_clusters, tc_gemm_2sm_mc_kernel<kBF16, kTransB, kBN, kDeep>, &cfg);
    });
    if (attr_err != cudaSuccess) return attr_err;
    if (max_clusters <= 0) return cudaErrorInvalidConfiguration;
    CUtensorMap ta, tb, tco, tci;
    if (!get_tmap_2d(&ta, g.A, C::ELEM, g.m, g.k, g.lda, C::BM, C::BK, Swz::B128)) return cudaErrorInvalidValue;
    bool ok = kTransB ? get_tmap_2d(&tb, g.B, C::ELEM, g.n, g.k, g.ldb, C::BN_CTA / 2, C::BK, Swz::B128)
                      : get_tmap_2d(&tb, g.B, C::ELEM, g.k, g.n, g.ldb, C::BK, C::B_ATOM_N,
                                    C::B_BASE32 ? Swz::B128_32B : Swz::B128);
    if (!ok) return cudaErrorInvalidValue;
    if (!get_tmap_2d(&tco, g.C_out, 4, g.m, g.n, g.ldc_out, 32, 32, Swz::B128)) return cudaErrorInvalidValue;
    if (g.beta != 0.f) {
        if (!get_tmap_2d(&tci, g.C_in, 4, g.m, g.n, g.ldc_in, 32, 32, Swz::B128)) return cudaErrorInvalidValue;
    } else {
        tci = tco;  // unused
    }
    const Knobs &kn = knobs_of(g);
    TcMParams p;
    p.m = g.m, p.n = g.n, p.k = g.k;
    p.alpha = g.alpha, p.beta = g.beta;
    p.m_blocks = static_cast<int>((g.m + kCluster * C::BM - 1) / (kCluster * C::BM));
    p.n_blocks = static_cast<int>((g.n + C::BN - 1) / C::BN);
    p.num_kb = static_cast<int>((g.k + C::BK - 1) / C::BK);
    // bands of 4 cluster tiles; 8 when K <= 8192 (8192^3: 729 vs 743 us; 32768^3 keeps 4)
    p.group_m = kn.tc2_group > 0 ? kn.tc2_group : (g.k <= 8192 ? 2 * kGroupM4 : kGroupM4);
    p.sched = sched_workspace(g.stream);
    if (!p.sched) return cudaErrorMemoryAllocation;
    const int tiles = p.m_blocks * p.n_blocks;
    p.splits = 1, p.ksplit = p.num_kb, p.spart = nullptr, p.spart_ld = 0, p.spart_plane = 0;
    p.tmem_cin = 0;
    if (splits > 1) {
        p.splits = splits;
        p.ksplit = (p.num_kb + splits - 1) / splits;
        p.spart_ld = static_cast<int64_t>(p.n_blocks) * C::BN;
        p.spart_plane = static_cast<int64_t>(p.m_blocks) * kCluster * C::BM * p.spart_ld;
        SplitWorkspace *w = split_workspace(g.stream, static_cast<size_t>(splits) * p.spart_plane * 4, 0);
        if (!w) return cudaErrorMemoryAllocation;
        p.spart = w->part;
    }
    const int items = tiles * p.splits;
    int clusters = g.num_sms / kCluster < max_clusters ? g.num_sms / kCluster : max_clusters;
    if (clusters < 1) clusters = 1;
    if (items < clusters) clusters = items;
    // even waves: the fewest clusters that still need the same number of item waves, so no wave
    // is partial (config 5a: 256 tiles on 64 pairs = 4 full waves instead of 3.46 waves on 74,
    // whose last 0.46 wave ran MMA-bound on 68 SMs while the rest idled); the makespan in tiles
    // per cluster is unchanged and each tile gets more of the HBM / L2 bandwidth
    if (kn.even_waves) {
        const int waves = (items + clusters - 1) / clusters;
        clusters = (items + waves - 1) / waves;
    }
    p.nprod = kn.tc2_producers == 1 ? 1 : 2;
    // single wave of 256-wide tiles with beta != 0: C_in staged in the second accumulator's TMEM
    p.tmem_cin = kn.tc2_tmem_cin && kBN == 256 && p.splits == 1 && g.beta != 0.f && items <= clusters;
    tc_gemm_2sm_mc_kernel<kBF16, kTransB, kBN, kDeep><<<kCluster * clusters, kThreadsM, C::SMEM, g.stream>>>(ta, tb, tco, tci, p);
    if (p.splits > 1) {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        const int64_t quads = g.m * ((g.n + 3) / 4);
        const int64_t blocks = (quads + 255) / 256;
        splitk_reduce_kernel<<<static_cast<unsigned>(blocks < (1 << 30) ? blocks : (1 << 30)), 256, 0, g.stream>>>(
            p.spart, p.splits, p.spart_ld, p.spart_plane, g.m, g.n, g.alpha, g.beta, g.C_in, g.ldc_in, g.C_out,
            g.ldc_out);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_tc_gemm_pairs(const GemmLaunch &g, bool bf16) {
    // 256 x 128 pair tiles (N = 128 MMAs) when 256 x 256 ones would give fewer tiles than half the
    // CTA pairs (e.g. 1536^3: 36 tiles for 74 pairs); same k order per element, bitwise-same C.
    // COMPAR_TC2_BN=256 / 128 (Knobs) forces one.
    const int force = knobs_of(g).tc2_bn;
    const int64_t tiles256 = ((g.m + 255) / 256) * ((g.n + 255) / 256);
    const bool narrow = force == 128 || (force != 256 && 2 * tiles256 < g.num_sms / 2);   // tiles < pairs / 2
    if (narrow) {
        if (bf16) return g.transB ? launch_tcm_t<true, true, 128>(g) : launch_tcm_t<true, false, 128>(g);
        return g.transB ? launch_tcm_t<false, true, 128>(g) : launch_tcm_t<false, false, 128>(g);
    }
    if (knobs_of(g).tc2_deep && 2 * tiles256 > g.num_sms) {   // more 256-wide tiles than pairs: deep ring
        if (bf16) return g.transB ? launch_tcm_t<true, true, 256, true>(g) : launch_tcm_t<true, false, 256, true>(g);
        return g.transB ? launch_tcm_t<false, true, 256, true>(g) : launch_tcm_t<false, false, 256, true>(g);
    }
    if (bf16) return g.transB ? launch_tcm_t<true, true>(g) : launch_tcm_t<true, false>(g);
    return g.transB ? launch_tcm_t<false, true>(g) : launch_tcm_t<false, false>(g);
}

cudaError_t launch_tc_gemm_splitk(const GemmLaunch &g, bool bf16) {
    const int s = tc_splitk_splits(g.m, g.n, g.k, bf16);
    if (s < 2) return cudaErrorInvalidValue;
    if (bf16) return g.transB ? launch_tcm_t<true, true>(g, s) : launch_tcm_t<true, false>(g, s);
    return g.transB ? launch_tcm_t<false, true>(g, s) : launch_tcm_t<false, false>(g, s);
}

cudaError_t preload_tcm_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaSuccess;
#define COMPAR_PRELOAD_TCM(B, T, N) \
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, tc_gemm_2sm_mc_kernel<B, T, N, false>);
    COMPAR_PRELOAD_TCM(true, false, 256)
    COMPAR_PRELOAD_TCM(true, true, 256)
    COMPAR_PRELOAD_TCM(false, false, 256)
    COMPAR_PRELOAD_TCM(false, true, 256)
    COMPAR_PRELOAD_TCM(true, false, 128)
    COMPAR_PRELOAD_TCM(true, true, 128)
    COMPAR_PRELOAD_TCM(false, false, 128)
    COMPAR_PRELOAD_TCM(false, true, 128)
#undef COMPAR_PRELOAD_TCM
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, tc_gemm_2sm_mc_kernel<true, false, 256, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, tc_gemm_2sm_mc_kernel<true, true, 256, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, tc_gemm_2sm_mc_kernel<false, false, 256, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, tc_gemm_2sm_mc_kernel<false, true, 256, true>);
    return e;
}

}  // namespace compar

#ifdef COMPAR_TRACE
extern "C" int compar_trace_read(unsigned long long *out) { return compar::trace_read(out); }
extern "C" int compar_trace_cta_read(unsigned long long *out) { return compar::trace_cta_read(out); }
extern "C" int compar_trace_item_read(unsigned long long *out, int clear) { return compar::trace_item_read(out, clear); }
#endif
