// The `sort` interface: "the sort function, two parameters
// are utilized: an array of floats and a scalar integer" — sort(arr, n) in place, ascending
// (R24; FP32 in IEEE totalOrder, also uint32 / int32).  Two sm_100a variants:
//
//   sort_radix   — LSD radix sort, 4 passes of 8 bits, "onesweep" structure: one histogram pass
//                  over the keys builds all four global digit histograms, then each pass is ONE
//                  kernel: a tile of 4096 keys is ranked in registers / shared memory (warp
//                  match-any multisplit, stable) and sorted by digit in shared memory, its
//                  per-digit tile offsets come from a decoupled look-back over the preceding
//                  tiles' published counts (tile ids are drawn from an atomic counter, so a tile's
//                  predecessors are always resident), and each digit's run is written out with
//                  contiguous stores.  HBM traffic: 4 B/key (histogram) + 8 B/key per pass
//                  = 36 B/key.
//   sort_bitonic — one CTA, bitonic network on (order code, index) pairs in shared memory: for
//                  n <= 16384 a single launch with no global round trips.  The index makes every
//                  pair unique, so the result is the same stable order as the radix sort.
//
// Keys are mapped to an order-preserving uint32 code on load (F32: totalOrder) and back on store.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace compar {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kChunks = 16;                       // 16 keys per lane
constexpr int kTile = kThreads * kChunks;         // 4096 keys per tile
constexpr int kLookback = 4;                      // predecessors read per look-back round trip
constexpr uint32_t kAgg = 1u << 30, kIncl = 2u << 30, kCountMask = (1u << 30) - 1;

template <int KT>
__device__ __forceinline__ uint32_t fwd(uint32_t b) {
    if (KT == 0) return b;                                       // uint32
    if (KT == 1) return b ^ 0x80000000u;                         // int32
    return (b >> 31) ? ~b : (b ^ 0x80000000u);                   // float32 totalOrder
}
template <int KT>
__device__ __forceinline__ uint32_t inv(uint32_t c) {
    if (KT == 0) return c;
    if (KT == 1) return c ^ 0x80000000u;
    return (c >> 31) ? (c ^ 0x80000000u) : ~c;
}

// All four digit histograms in one read of the keys: hist[p][d], p = pass (digit bits 8p..8p+7).
template <int KT>
__global__ void __launch_bounds__(kThreads) radix_hist_kernel(const uint32_t *__restrict__ keys, int64_t n,
                                                             uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[4][256];
    for (int i = threadIdx.x; i < 4 * 256; i += kThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n; i += stride) {
        const uint32_t c = fwd<KT>(__ldcs(keys + i));
#pragma unroll
        for (int p = 0; p < 4; ++p) atomicAdd(&h[p][(c >> (8 * p)) & 255], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * 256; i += kThreads) {
        const uint32_t v = (&h[0][0])[i];
        if (v) atomicAdd(hist + i, v);
    }
}

// Look-back status words are self-contained (flag + count in one 32-bit word), so a relaxed
// GPU-scope load is enough (a volatile access would be a system-scope LDG.STRONG.SYS).
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Block-wide exclusive scan of one value per thread (kThreads threads); `wsum` is kWarps words.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *wsum) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    uint32_t off = incl - v;
    for (int w = 0; w < warp; ++w) off += wsum[w];
    __syncthreads();
    return off;
}

// One LSD pass: in -> out by digit (code >> shift) & 255.  IN_RAW: `in` holds user keys (apply
// the order code); OUT_RAW: store user keys (undo it).
//   1. rank: each warp ranks its 512-key slice (16 chunks of 32, stable) with match-any into a
//      warp-private digit histogram;
//   2. per digit: tile count, warp offsets, tile-local digit offsets (block scan); publish the
//      tile count for the look-back as early as possible;
//   3. local sort: every key goes to its tile-local sorted slot in shared memory;
//   4. look-back: per digit, the sum of the preceding tiles' counts;
//   5. scatter: consecutive threads write consecutive slots of the sorted tile, so each digit's run
//      lands as contiguous (coalesced) stores.
template <int KT, bool IN_RAW, bool OUT_RAW, int CH>
__global__ void __launch_bounds__(kThreads, CH > 16 ? 2 : 3) radix_pass_kernel(const uint32_t *__restrict__ in, uint32_t *__restrict__ out,
                                                             int64_t n, int shift, const uint32_t *__restrict__ hist,
                                                             uint32_t *status, int *tile_ctr) {
    __shared__ uint32_t warp_hist[kWarps][256];
    __shared__ uint32_t sorted[(CH * kThreads)];
    __shared__ uint32_t digit_base[256];   // global position of tile-local slot 0 of each digit
    __shared__ uint32_t wsum[kWarps];
    __shared__ int tile_s;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) tile_s = atomicAdd(tile_ctr, 1);
    for (int d = lane; d < 256; d += 32) warp_hist[warp][d] = 0;
    const uint32_t goff = block_excl_scan(hist[tid], wsum);   // (its barriers publish tile_s too)
    const int tile = tile_s;

    const uint32_t lt = (1u << lane) - 1u;
    const int64_t base = static_cast<int64_t>(tile) * (CH * kThreads) + static_cast<int64_t>(warp) * (CH * 32);
    uint32_t code[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const int64_t i = base + c * 32 + lane;
        const uint32_t k = i < n ? __ldcs(in + i) : 0xffffffffu;
        code[c] = (IN_RAW && i < n) ? fwd<KT>(k) : k;
    }
    // Peers (lanes with the same digit) from 8 ballots — one per digit bit — instead of
    // match.any: the ballots run on the ALU pipes, match.any / ffs on the narrow ADU / XU pipes
    // that bounded the first version (ncu: ADU 68 %, XU saturated).
    // Keys past n (last tile only) were loaded as code 0xffffffff: digit 255 in every pass, so they
    // rank after every real key of the tile and occupy its last sorted slots, which the scatter
    // below never reads (i < valid_n); only their count is taken out of the published digit-255
    // count.  No per-key validity test is needed in the ranking.
    uint16_t rank[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const uint32_t d = (code[c] >> shift) & 255u;
        uint32_t peers = 0xffffffffu;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const uint32_t v = __ballot_sync(0xffffffffu, (d >> b) & 1u);
            peers &= ((d >> b) & 1u) ? v : ~v;
        }
        const uint32_t before = warp_hist[warp][d];
        __syncwarp();
        rank[c] = static_cast<uint16_t>(before + __popc(peers & lt));
        if ((peers & lt) == 0) warp_hist[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t v = warp_hist[w][tid];
        warp_hist[w][tid] = run;
        run += v;
    }
    const int64_t tile0 = static_cast<int64_t>(tile) * (CH * kThreads);
    const int valid_n = static_cast<int>(n - tile0 < (CH * kThreads) ? n - tile0 : (CH * kThreads));
    if (tid == kThreads - 1) run -= static_cast<uint32_t>((CH * kThreads) - valid_n);   // padding keys are not published
    uint32_t *st = status + static_cast<int64_t>(tile) * 256 + tid;
    __stcg(st, (tile == 0 ? kIncl : kAgg) | run);
    const uint32_t local = block_excl_scan(run, wsum);         // tile-local start of digit `tid`
    for (int w = 0; w < kWarps; ++w) warp_hist[w][tid] += local;
    __syncthreads();
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const uint32_t d = (code[c] >> shift) & 255u;
        sorted[warp_hist[warp][d] + rank[c]] = code[c];
    }
    uint32_t prefix = 0;
    if (tile > 0) {
        // Windowed look-back: the status words of kLookback predecessors are loaded together (one
        // round trip instead of kLookback), then consumed in order until an inclusive prefix; a
        // predecessor that has not published yet restarts the window at it after a back-off.
        for (int j = tile - 1;;) {
            uint32_t v[kLookback];
#pragma unroll
            for (int w = 0; w < kLookback; ++w)
                v[w] = j - w >= 0 ? ld_relaxed_gpu(status + static_cast<int64_t>(j - w) * 256 + tid) : kIncl;
            int w = 0;
            bool done = false;
#pragma unroll
            for (; w < kLookback; ++w) {
                const uint32_t flag = v[w] & ~kCountMask;
                if (flag == 0) break;
                prefix += v[w] & kCountMask;
                if (flag == kIncl) {
                    done = true;
                    break;
                }
            }
            if (done) break;
            j -= w;
            if (w < kLookback) __nanosleep(32);   // predecessor still ranking: back off
        }
        __stcg(st, kIncl | (prefix + run));
    }
    digit_base[tid] = goff + prefix - local;
    __syncthreads();
#pragma unroll 4
    for (int i = tid; i < valid_n; i += kThreads) {
        const uint32_t c = sorted[i];
        const uint32_t pos = digit_base[(c >> shift) & 255u] + static_cast<uint32_t>(i);
        out[pos] = OUT_RAW ? inv<KT>(c) : c;
    }
}

constexpr int kBitonicMax = 16384;

template <int KT>
__global__ void __launch_bounds__(1024) bitonic_kernel(uint32_t *__restrict__ keys, int n, int n2) {
    extern __shared__ unsigned long long s[];
    for (int i = threadIdx.x; i < n2; i += blockDim.x)
        s[i] = i < n ? ((static_cast<unsigned long long>(fwd<KT>(keys[i])) << 32) | static_cast<unsigned>(i))
                     : ~0ull;
    __syncthreads();
    // every thread takes whole compare-exchange pairs (i, i + j): pair p -> i = 2p - (p mod j)
    for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int p = threadIdx.x; p < (n2 >> 1); p += blockDim.x) {
                const int i = 2 * p - (p & (j - 1));
                const unsigned long long a = s[i], b = s[i + j];
                if ((a > b) == ((i & k) == 0)) {
                    s[i] = b;
                    s[i + j] = a;
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) keys[i] = inv<KT>(static_cast<uint32_t>(s[i] >> 32));
}

int64_t tiles_of(int64_t n, int ch = kChunks) { return (n + ch * kThreads - 1) / (ch * kThreads); }
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Tile size: kChunks (16) keys per lane = 4096-key tiles up to 16 M keys; 32 per lane = 8192-key
// tiles above, where the look-back and per-tile fixed work amortise over twice the keys (2^28
// keys: 40.1 -> 45.1 Gkeys/s; 2^20 keys: 15.4 -> 13.9, so small sorts keep the smaller tile).
template <int KT, int CH>
cudaError_t radix_t(uint32_t *keys, int64_t n, uint8_t *scratch, cudaStream_t s, int num_sms) {
    const int64_t T = tiles_of(n, CH);
    uint32_t *tmp = reinterpret_cast<uint32_t *>(scratch);
    uint8_t *meta = scratch + align256(static_cast<size_t>(n) * 4);
    uint32_t *hist = reinterpret_cast<uint32_t *>(meta);                 // [4][256]
    int *ctr = reinterpret_cast<int *>(meta + 4 * 256 * 4);               // [4]
    uint32_t *status = reinterpret_cast<uint32_t *>(meta + 4 * 256 * 4 + 256);  // [4][T][256]
    cudaError_t e = cudaMemsetAsync(meta, 0, 4 * 256 * 4 + 256 + static_cast<size_t>(4 * T * 256) * 4, s);
    if (e != cudaSuccess) return e;
    const int64_t hb = (n + kThreads * 16 - 1) / (kThreads * 16);
    const int hist_blocks = static_cast<int>(hb < 4 * num_sms ? (hb > 0 ? hb : 1) : 4 * num_sms);
    radix_hist_kernel<KT><<<hist_blocks, kThreads, 0, s>>>(keys, n, hist);
    const unsigned grid = static_cast<unsigned>(T);
    uint32_t *st = status;
    radix_pass_kernel<KT, true, false, CH><<<grid, kThreads, 0, s>>>(keys, tmp, n, 0, hist, st, ctr);
    radix_pass_kernel<KT, false, false, CH><<<grid, kThreads, 0, s>>>(tmp, keys, n, 8, hist + 256, st + T * 256, ctr + 1);
    radix_pass_kernel<KT, false, false, CH><<<grid, kThreads, 0, s>>>(keys, tmp, n, 16, hist + 512, st + 2 * T * 256,
                                                                  ctr + 2);
    radix_pass_kernel<KT, false, true, CH><<<grid, kThreads, 0, s>>>(tmp, keys, n, 24, hist + 768, st + 3 * T * 256,
                                                                 ctr + 3);
    return cudaGetLastError();
}

template <int KT>
cudaError_t bitonic_t(uint32_t *keys, int64_t n, cudaStream_t s) {
    int n2 = 2;
    while (n2 < n) n2 <<= 1;
    const int smem = n2 * 8;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(bitonic_kernel<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kBitonicMax * 8);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    bitonic_kernel<KT><<<1, 1024, smem, s>>>(keys, static_cast<int>(n), n2);
    return cudaGetLastError();
}

}  // namespace

size_t sort_radix_scratch_bytes(int64_t n) {
    return align256(static_cast<size_t>(n) * 4) + 4 * 256 * 4 + 256 + static_cast<size_t>(4 * tiles_of(n) * 256) * 4;
}

int64_t sort_bitonic_max() { return kBitonicMax; }

cudaError_t launch_sort_radix(void *keys, int64_t n, int key_type, void *scratch, cudaStream_t s, int num_sms) {
    if (n <= 1) return cudaSuccess;
    if (n >= (int64_t(1) << 30)) return cudaErrorInvalidValue;
    uint32_t *k = static_cast<uint32_t *>(keys);
    uint8_t *sc = static_cast<uint8_t *>(scratch);
    if (n >= (int64_t(1) << 24)) {
        if (key_type == 0) return radix_t<0, 32>(k, n, sc, s, num_sms);
        if (key_type == 1) return radix_t<1, 32>(k, n, sc, s, num_sms);
        return radix_t<2, 32>(k, n, sc, s, num_sms);
    }
    if (key_type == 0) return radix_t<0, kChunks>(k, n, sc, s, num_sms);
    if (key_type == 1) return radix_t<1, kChunks>(k, n, sc, s, num_sms);
    return radix_t<2, kChunks>(k, n, sc, s, num_sms);
}

cudaError_t launch_sort_bitonic(void *keys, int64_t n, int key_type, cudaStream_t s) {
    if (n <= 1) return cudaSuccess;
    if (n > kBitonicMax) return cudaErrorInvalidValue;
    uint32_t *k = static_cast<uint32_t *>(keys);
    if (key_type == 0) return bitonic_t<0>(k, n, s);
    if (key_type == 1) return bitonic_t<1>(k, n, s);
    return bitonic_t<2>(k, n, s);
}

}  // namespace compar
