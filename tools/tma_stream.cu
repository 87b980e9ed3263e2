// HBM streaming microbenchmark for the skinny-GEMM A operand (BASELINE config 5a, A = 65536 x 4096
// BF16): how fast can 148 persistent CTAs pull 128-row A blocks through TMA with no compute, and
// does the box shape matter?
//   mode 0: 2-D boxes 128 rows x 64 elements (16 KiB, the GEMM mainloop's A box), S stages
//   mode 1: 3-D boxes (64 elements, 128 rows, G k-atoms) = G x 16 KiB, each row read as G*128 B
//   mode 2: plain coalesced ld.global.v4 streaming read (reference)
//   mode 3: G separate 2-D boxes (128 x 64) issued back to back per stage (same bytes as mode 1)
//   mode 4: the GEMM's load pattern without the MMA: per stage one A box + G B boxes (64 K-rows x
//           64 cols of an L2-resident 4096 x 256 B), i.e. 16 KiB HBM + G x 8 KiB L2
//   mode 5: mode 4 in clusters of 2 CTAs (different A row blocks, same k step): each CTA loads
//           half of the B boxes with TMA multicast to both (cross-CTA empty barriers)
//   mode 6: mode 5's lockstep pair without multicast (each CTA loads all its B boxes)
//   mode 7: mode 4 with two producer warps in one CTA, each owning alternate stages
// usage: tma_stream [M] [K] [stages] [G]
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) {                                                         \
            std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));       \
            std::exit(1);                                                                \
        }                                                                                \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(n));
}
__device__ __forceinline__ void expect_tx(uint32_t b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t ph) {
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(b),
        "r"(ph)
        : "memory");
}
__device__ __forceinline__ void tma2(uint32_t dst, const CUtensorMap *m, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            dst),
        "l"(m), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma3(uint32_t dst, const CUtensorMap *m, uint32_t bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
        "[%2];" ::"r"(dst),
        "l"(m), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// one thread streams: issue up to S boxes ahead, retire in order (no compute)
template <int MODE>
__global__ void __launch_bounds__(32, 1) stream_kernel(const __grid_constant__ CUtensorMap tm,
                                                       const __grid_constant__ CUtensorMap tb, int m_blocks, int kb_n,
                                                       int G, int S, int *counter) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bars[16];
    if (threadIdx.x != 0) return;
    const uint32_t box = MODE == 0 ? 16384 : MODE == 4 ? 16384 + G * 8192 : G * 16384;  // bytes per stage
    for (int s = 0; s < S; ++s) mbar_init(smem_u32(&bars[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    int issued = 0, retired = 0;
    const int steps = (MODE == 0 || MODE == 4) ? kb_n : kb_n / G;  // stages per 128-row tile
    int tile = atomicAdd(counter, 1), it = 0;
    int rtile = tile;  (void)rtile;
    while (true) {
        // issue as far ahead as the ring allows
        while (issued - retired < S && tile < m_blocks) {
            const int s = issued % S;
            const uint32_t b = smem_u32(&bars[s]);
            expect_tx(b, box);
            if (MODE == 0)
                tma2(smem_u32(smem + s * box), &tm, b, it * 64, tile * 128);
            else if (MODE == 4) {
                tma2(smem_u32(smem + s * box), &tm, b, it * 64, tile * 128);
                for (int g = 0; g < G; ++g) tma2(smem_u32(smem + s * box + 16384 + g * 8192), &tb, b, g * 64, it * 64);
            }
            else if (MODE == 1)
                tma3(smem_u32(smem + s * box), &tm, b, 0, tile * 128, it * G);
            else
                for (int g = 0; g < G; ++g) tma2(smem_u32(smem + s * box + g * 16384), &tm, b, (it * G + g) * 64, tile * 128);
            ++issued;
            if (++it == steps) {
                it = 0;
                tile = atomicAdd(counter, 1);
            }
        }
        if (retired == issued) break;
        const int s = retired % S;
        mbar_wait(smem_u32(&bars[s]), (retired / S) & 1);
        ++retired;
    }
}

__device__ __forceinline__ void tma2_mc(uint32_t dst, const CUtensorMap *m, uint32_t bar, int c0, int c1,
                                        uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, "
        "{%3, %4}], [%2], %5;" ::"r"(dst),
        "l"(m), "r"(bar), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32, 1)
    stream_mc_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tb, int m_blocks,
                     int kb_n, int G, int S, int mc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t full[16], empty[16];
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), 2);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x != 0) return;
    const uint32_t box = 16384 + G * 8192;
    const int pairs = m_blocks / 2, npair_ctas = gridDim.x / 2, pid = blockIdx.x / 2;
    const int my_tiles = pid < pairs ? (pairs - pid + npair_ctas - 1) / npair_ctas : 0;
    const long total = long(my_tiles) * kb_n;
    long issued = 0, retired = 0;
    while (retired < total) {
        while (issued < total && issued - retired < S) {
            const int s = int(issued % S);
            if (issued >= S) mbar_wait(smem_u32(&empty[s]), uint32_t(((issued / S) - 1) & 1));
            const long tile_i = issued / kb_n;
            const int it = int(issued % kb_n);
            const int mblk = 2 * (pid + int(tile_i) * npair_ctas) + int(rank);
            const uint32_t b = smem_u32(&full[s]);
            expect_tx(b, box);
            tma2(smem_u32(smem + s * box), &tm, b, it * 64, mblk * 128);
            if (mc) {
                for (int g = int(rank); g < G; g += 2)
                    tma2_mc(smem_u32(smem + s * box + 16384 + g * 8192), &tb, b, g * 64, it * 64, 0x3);
            } else {
                for (int g = 0; g < G; ++g) tma2(smem_u32(smem + s * box + 16384 + g * 8192), &tb, b, g * 64, it * 64);
            }
            ++issued;
        }
        const int s = int(retired % S);
        mbar_wait(smem_u32(&full[s]), uint32_t((retired / S) & 1));
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(mapa(smem_u32(&empty[s]), rank ^ 1u))
                     : "memory");
        ++retired;
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// mode 7: warp w issues and retires the stages with index % 2 == w (two independent rings of S/2)
__global__ void __launch_bounds__(64, 1) stream2_kernel(const __grid_constant__ CUtensorMap tm,
                                                        const __grid_constant__ CUtensorMap tb, int m_blocks, int kb_n,
                                                        int G, int S, int *counter) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bars[16];
    __shared__ int tiles[2];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) != 0) return;
    const uint32_t box = 16384 + G * 8192;
    const int S2 = S / 2;
    for (int s = 0; s < S2; ++s) mbar_init(smem_u32(&bars[w * 8 + s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // each warp streams its own tiles (own counter draws): two independent producers per CTA
    int issued = 0, retired = 0, it = 0;
    int tile = atomicAdd(counter, 1);
    (void)tiles;
    uint8_t *base = smem + w * S2 * box;
    while (true) {
        while (issued - retired < S2 && tile < m_blocks) {
            const int s = issued % S2;
            const uint32_t b = smem_u32(&bars[w * 8 + s]);
            expect_tx(b, box);
            tma2(smem_u32(base + s * box), &tm, b, it * 64, tile * 128);
            for (int g = 0; g < G; ++g) tma2(smem_u32(base + s * box + 16384 + g * 8192), &tb, b, g * 64, it * 64);
            ++issued;
            if (++it == kb_n) {
                it = 0;
                tile = atomicAdd(counter, 1);
            }
        }
        if (retired == issued) break;
        const int s = retired % S2;
        mbar_wait(smem_u32(&bars[w * 8 + s]), (retired / S2) & 1);
        ++retired;
    }
}

__global__ void read_kernel(const uint4 *__restrict__ p, size_t n, unsigned long long *sink) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        uint4 v = __ldcs(p + i);
        acc.x ^= v.x, acc.y ^= v.y, acc.z ^= v.z, acc.w ^= v.w;
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) atomicAdd(sink, 1ull);
}

int main(int argc, char **argv) {
    const long M = argc > 1 ? atol(argv[1]) : 65536, K = argc > 2 ? atol(argv[2]) : 4096;
    const int S = argc > 3 ? atoi(argv[3]) : 4, G = argc > 4 ? atoi(argv[4]) : 4;
    const size_t bytes = size_t(M) * K * 2;
    void *A;
    CK(cudaMalloc(&A, bytes));
    CK(cudaMemset(A, 1, bytes));
    int *counter;
    CK(cudaMalloc(&counter, 4));
    unsigned long long *sink;
    CK(cudaMalloc(&sink, 8));
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    CUtensorMap t2, t3, tB;
    void *Bm;
    CK(cudaMalloc(&Bm, size_t(K) * 256 * 2));
    CK(cudaMemset(Bm, 1, size_t(K) * 256 * 2));
    {
        cuuint64_t d[2] = {256, cuuint64_t(K)};
        cuuint64_t st[1] = {512};
        cuuint32_t bx[2] = {64, 64}, es[2] = {1, 1};
        if (enc(&tB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, Bm, d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
            return 2;
    }
    {
        cuuint64_t d[2] = {cuuint64_t(K), cuuint64_t(M)};
        cuuint64_t st[1] = {cuuint64_t(K) * 2};
        cuuint32_t bx[2] = {64, 128}, es[2] = {1, 1};
        if (enc(&t2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, A, d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
            return 2;
    }
    {
        cuuint64_t d[3] = {64, cuuint64_t(M), cuuint64_t(K / 64)};
        cuuint64_t st[2] = {cuuint64_t(K) * 2, 128};
        cuuint32_t bx[3] = {64, 128, cuuint32_t(G)}, es[3] = {1, 1, 1};
        if (enc(&t3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, A, d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) {
            std::printf("3d encode failed\n");
            return 2;
        }
    }
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto run = [&](int mode, int S_, int ctas_per_sm) {
        const int smem = (mode == 0 || mode == 2 ? 16384 : (mode >= 4) ? 16384 + G * 8192 : G * 16384) * S_;
        if (mode == 0) CK(cudaFuncSetAttribute(stream_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        if (mode == 1) CK(cudaFuncSetAttribute(stream_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        if (mode == 3) CK(cudaFuncSetAttribute(stream_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        if (mode == 4) CK(cudaFuncSetAttribute(stream_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        if (mode == 7) CK(cudaFuncSetAttribute(stream2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        if (mode == 5 || mode == 6) CK(cudaFuncSetAttribute(stream_mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        std::vector<float> ts;
        for (int r = 0; r < 8; ++r) {
            CK(cudaMemset(counter, 0, 4));
            CK(cudaEventRecord(e0));
            if (mode == 0) stream_kernel<0><<<sms * ctas_per_sm, 32, smem>>>(t2, tB, int(M / 128), int(K / 64), G, S_, counter);
            if (mode == 1) stream_kernel<1><<<sms * ctas_per_sm, 32, smem>>>(t3, tB, int(M / 128), int(K / 64), G, S_, counter);
            if (mode == 7) stream2_kernel<<<sms, 64, smem>>>(t2, tB, int(M / 128), int(K / 64), G, S_, counter);
            if (mode == 5 || mode == 6)
                stream_mc_kernel<<<sms, 32, smem>>>(t2, tB, int(M / 128), int(K / 64), G, S_, mode == 5);
            if (mode == 4) stream_kernel<4><<<sms * ctas_per_sm, 32, smem>>>(t2, tB, int(M / 128), int(K / 64), G, S_, counter);
            if (mode == 3) stream_kernel<3><<<sms * ctas_per_sm, 32, smem>>>(t2, tB, int(M / 128), int(K / 64), G, S_, counter);
            if (mode == 2) read_kernel<<<sms * 8, 512>>>(static_cast<const uint4 *>(A), bytes / 16, sink);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            ts.push_back(ms);
        }
        float best = 1e9;
        for (float t : ts) best = t < best ? t : best;
        std::printf("mode %d stages %d G %d ctas/sm %d: %.1f us  %.0f GB/s\n", mode, S_, (mode == 1 || mode == 3 || mode >= 4) ? G : 1,
                    ctas_per_sm, best * 1e3, bytes / (best * 1e-3) / 1e9);
    };
    run(2, 0, 1);
    for (int s : {2, 4, 6, 8, 12}) run(0, s, 1);
    run(0, 4, 2);
    run(0, 6, 2);
    for (int s : {1, 2, 3}) run(1, s, 1);
    run(1, 1, 2);
    for (int s : {1, 2, 3}) run(3, s, 1);
    for (int s : {4, 6}) if ((16384 + G * 8192) * s <= 227 * 1024) run(4, s, 1);
    for (int s : {2, 3}) if ((16384 + G * 8192) * s * 2 <= 227 * 1024) run(4, s, 2);
    for (int s : {4, 6}) if ((16384 + G * 8192) * s <= 227 * 1024) run(7, s, 1);
    for (int s : {4, 6}) if ((16384 + G * 8192) * s <= 227 * 1024) run(5, s, 1);
    for (int s : {4, 6}) if ((16384 + G * 8192) * s <= 227 * 1024) run(6, s, 1);
    (void)S;
    return 0;
}
