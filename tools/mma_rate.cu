// Microbenchmark: cycles per tcgen05.mma (BF16, K = 16) issued back to back by one thread, one CTA
// (or CTA pair) per SM, all SMs busy.  Operands are whatever shared memory holds (the result is not
// read); the accumulator is never reset.  Variants: cta_group::1 (M = 128) / ::2 (M = 256 over a
// pair), N in {64, 128, 256}, B K-major (transB) or MN-major (row-major B, 128-byte swizzle atoms
// of 64 columns x 8 k-rows).  Development tool for the single-wave analysis; built
// and run by `python tools/mma_rate.py`.
#include <cstdio>
#include <cstdlib>

#include "../paper_2311_03543_b200/csrc/kernels/ptx.cuh"

using namespace compar;

// MODE 0: MMAs only; 1: + tcgen05.commit to a stage barrier after every 4 MMAs (never waited);
// 2: the kernels' stage ring without loads: a producer thread waits empty[s] and arrives full[s],
// the MMA thread waits full[s], issues 4 MMAs and commits empty[s]; S stages.  3-5: an already
// satisfied mbarrier wait and/or tcgen05.fence::after_thread_sync before every 4 MMAs (+ commit).
template <int CG, int N, bool BMN, int MODE = 0, int S = 4, int G = 4>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, unsigned long long *out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t s0 = ptx::smem_u32(smem);
    constexpr uint32_t A_BYTES = 128 * 128;                      // 128 rows x 64 bf16 (one k-block)
    constexpr int NB = N / CG;                                   // B columns held by this CTA
    const uint32_t sa = s0, sb = s0 + A_BYTES;
    __shared__ uint64_t bar, full[S], empty[S];
    __shared__ uint32_t tslot[2];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    constexpr uint32_t COLS = N < 32 ? 32 : N;
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar), 1);
        tslot[1] = 0x1234u;
        for (int i = 0; i < S; ++i) ptx::mbar_init(ptx::smem_u32(&full[i]), 1), ptx::mbar_init(ptx::smem_u32(&empty[i]), 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) {
        if (CG == 2)
            ptx::tmem_alloc_2sm<COLS>(ptx::smem_u32(&tslot[0]));
        else
            ptx::tmem_alloc<COLS>(ptx::smem_u32(&tslot[0]));
    }
    ptx::tc_fence_before();
    if (CG == 2)
        ptx::cluster_sync();
    else
        __syncthreads();
    ptx::tc_fence_after();
    const uint32_t d = tslot[0];
    const bool leader = CG == 1 || ptx::cluster_ctarank() == 0;
    // idesc: D F32, A/B BF16, a K-major, b major bit, N>>3, M>>4
    constexpr uint32_t M = 128 * CG;
    constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((BMN ? 1u : 0u) << 16) |
                               ((uint32_t(N) >> 3) << 17) | ((M >> 4) << 24);
    const uint64_t adesc0 = ptx::smem_desc_sw128(sa, 16, 1024);
    // K-major B: rows of 128 B (64 k), SBO 1024 between 8-row groups; MN-major B: atoms of 64
    // columns x 8 k-rows (1 KiB), LBO = the stride between 64-column atoms (one k-block: 8 KiB),
    // SBO 1024 between 8-k-row groups.
    const uint64_t bdesc0 = BMN ? ptx::smem_desc(sb, 64 * 128, 1024, 2) : ptx::smem_desc_sw128(sb, 16, 1024);
    unsigned long long t0 = 0, t1 = 0;
    if (MODE == 9 && warp == 1 && leader) {   // lane 1 does the (satisfied) wait, then __syncwarp
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (lane == 1) ptx::mbar_wait(ptx::smem_u32(&full[0]), 1);
            __syncwarp();
            if (lane == 0) {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    ptx::mma_bf16(d, ptx::desc_adv(adesc0, j * 32), ptx::desc_adv(bdesc0, j * 32), IDESC, 1);
            }
            __syncwarp();
        }
        if (lane == 0) ptx::tc_commit(ptx::smem_u32(&bar));
        __syncwarp();
    } else if (MODE == 10 && warp == 1 && leader) {   // warp 2 waits, named barrier hands over
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            asm volatile("bar.sync 1, 64;" ::: "memory");
            if (lane == 0) {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    ptx::mma_bf16(d, ptx::desc_adv(adesc0, j * 32), ptx::desc_adv(bdesc0, j * 32), IDESC, 1);
            }
            __syncwarp();
        }
        if (lane == 0) ptx::tc_commit(ptx::smem_u32(&bar));
        __syncwarp();
    } else if (MODE == 10 && warp == 2 && leader) {
        for (int it = 0; it < iters; ++it) {
            ptx::mbar_wait(ptx::smem_u32(&full[0]), 1);
            asm volatile("bar.arrive 1, 64;" ::: "memory");
        }
    } else if (warp == 1 && leader) {
        if (lane == 0) {
            t0 = clock64();
            for (int it = 0; it < iters; ++it) {
                if (MODE == 2) {
                    ptx::mbar_wait(ptx::smem_u32(&full[it % S]), (it / S) & 1);
                    ptx::tc_fence_after();
                } else if (MODE == 3) {            // a wait that is already satisfied + the fence
                    ptx::mbar_wait(ptx::smem_u32(&full[0]), 1);
                    ptx::tc_fence_after();
                } else if (MODE == 4) {            // the satisfied wait alone
                    ptx::mbar_wait(ptx::smem_u32(&full[0]), 1);
                } else if (MODE == 5) {            // the fence alone
                    ptx::tc_fence_after();
                } else if (MODE == 6) {            // poll a (set) shared-memory flag
                    uint32_t v;
                    do {
                        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(ptx::smem_u32(&tslot[0]) + 4u) : "memory");
                    } while (v != 0x1234u);
                } else if (MODE == 7) {            // satisfied wait with .relaxed semantics
                    uint32_t ok;
                    do {
                        asm volatile(
                            "{\n\t.reg .pred p;\n\t"
                            "mbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 p, [%1], %2;\n\t"
                            "selp.u32 %0, 1, 0, p;\n\t}"
                            : "=r"(ok) : "r"(ptx::smem_u32(&full[0])), "r"(1u) : "memory");
                    } while (!ok);
                } else if (MODE == 8) {            // satisfied non-blocking test_wait
                    uint32_t ok;
                    do {
                        asm volatile(
                            "{\n\t.reg .pred p;\n\t"
                            "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                            "selp.u32 %0, 1, 0, p;\n\t}"
                            : "=r"(ok) : "r"(ptx::smem_u32(&full[0])), "r"(1u) : "memory");
                    } while (!ok);
                }
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    const uint64_t a = ptx::desc_adv(adesc0, j * 32);
                    const uint64_t b = ptx::desc_adv(bdesc0, BMN ? j * 16 * 128 : j * 32);
                    if (CG == 2)
                        ptx::mma_bf16_2sm(d, a, b, IDESC, 1);
                    else
                        ptx::mma_bf16(d, a, b, IDESC, 1);
                }
                if (MODE >= 1) {
                    if (CG == 2)
                        ptx::tc_commit_2sm_mc(ptx::smem_u32(&empty[it % S]), 0x3);
                    else
                        ptx::tc_commit(ptx::smem_u32(&empty[it % S]));
                }
            }
            if (CG == 2)
                ptx::tc_commit_2sm_mc(ptx::smem_u32(&bar), 0x3);
            else
                ptx::tc_commit(ptx::smem_u32(&bar));
        }
        __syncwarp();
    } else if (MODE == 2 && warp == 0 && lane == 0 && leader) {   // producer without loads
        for (int it = 0; it < iters; ++it) {
            ptx::mbar_wait(ptx::smem_u32(&empty[it % S]), ((it / S) & 1) ^ 1);
            ptx::mbar_arrive(ptx::smem_u32(&full[it % S]));
        }
    }
    ptx::mbar_wait(ptx::smem_u32(&bar), 0);
    if (warp == 1 && leader && lane == 0 && t0) {
        t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    (void)NB;
    ptx::tc_fence_before();
    if (CG == 2)
        ptx::cluster_sync();
    else
        __syncthreads();
    if (warp == 0) {
        if (CG == 2)
            ptx::tmem_dealloc_2sm<COLS>(d);
        else
            ptx::tmem_dealloc<COLS>(d);
    }
}

template <int CG, int N, bool BMN, int MODE = 0, int S = 4, int G = 4>
void run(int iters, int sms) {
    auto k = mma_rate<CG, N, BMN, MODE, S, G>;
    const int smem = 128 * 128 + 256 * 128 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long *out;
    cudaMalloc(&out, sizeof(unsigned long long) * sms);
    cudaMemset(out, 0, sizeof(unsigned long long) * sms);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, k, iters, out);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[256] = {};
    cudaMemcpy(h, out, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
    double s = 0;
    int cnt = 0;
    for (int i = 0; i < sms; ++i)
        if (h[i]) s += h[i], ++cnt;
    const double per = cnt ? s / cnt / (double(G) * iters) : 0;
    printf("{\"group\": %d, \"mode\": %d, \"stages\": %d, \"cta_group\": %d, \"N\": %d, \"b\": \"%s\", \"iters\": %d, \"ctas\": %d, \"cycles_per_mma\": %.2f, "
           "\"floor\": %.1f, \"err\": \"%s\"}\n",
           G, MODE, S, CG, N, BMN ? "mn" : "k", iters, sms, per, 128.0 * N / (256.0 * CG), cudaGetErrorString(e));
    cudaFree(out);
}

int main(int argc, char **argv) {
    const int iters = argc > 1 ? atoi(argv[1]) : 512;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<1, 64, false>(iters, sms);
    run<1, 64, false, 4, 4, 1>(iters, sms), run<1, 64, false, 4, 4, 2>(iters, sms), run<1, 64, false, 4, 4, 4>(iters, sms);
    run<1, 64, false, 4, 4, 8>(iters, sms), run<1, 64, false, 4, 4, 16>(iters, sms);
    run<1, 128, false, 4, 4, 4>(iters, sms), run<1, 128, false, 4, 4, 8>(iters, sms), run<1, 128, false, 4, 4, 16>(iters, sms);
    run<2, 128, false, 4, 4, 4>(iters, sms), run<2, 128, false, 4, 4, 8>(iters, sms);
    run<2, 64, false, 4, 4, 4>(iters, sms), run<2, 64, false, 4, 4, 8>(iters, sms), run<2, 64, false, 0, 4, 4>(iters, sms);
    return 0;
}
