// Per-stream tile-scheduler workspace for the persistent tcgen05 kernels.
//
// Each persistent launch draws output tiles from a global atomic counter, so the set of tiles
// in flight is always a contiguous range in raster order however the CTAs drift relative to
// each other (a static round-robin schedule lets CTAs drift apart by whole tiles over a long
// K, which destroys L2 reuse between CTAs that share A rows / B columns — DESIGN.md §5).
// The counter pair {next, done} is zeroed once and re-zeroed by the last CTA of every launch;
// launches on one stream are ordered, so one pair per stream is enough.
#include <cuda_runtime.h>

#include <map>
#include <mutex>

#include "kernels.h"

namespace compar {

int *sched_workspace(cudaStream_t s) {
    static std::mutex mu;
    static std::map<cudaStream_t, int *> slots;
    std::lock_guard<std::mutex> lk(mu);
    auto it = slots.find(s);
    if (it != slots.end()) return it->second;
    int *p = nullptr;
    if (cudaMalloc(&p, 2 * sizeof(int)) != cudaSuccess) return nullptr;
    if (cudaMemset(p, 0, 2 * sizeof(int)) != cudaSuccess) return nullptr;
    slots.emplace(s, p);
    return p;
}

// Stream-K workspace (tc_gemm_2sm_mc.cu): per cluster one flag word and one 256 x 256 FP32
// partial accumulator; `epoch` counts the stream-K launches on this stream, so flags never need
// resetting (a flag reaches 8 * epoch when that launch's partial is published).
SkWorkspace *sk_workspace(cudaStream_t s, int clusters) {
    static std::mutex mu;
    static std::map<cudaStream_t, SkWorkspace> slots;
    std::lock_guard<std::mutex> lk(mu);
    SkWorkspace &w = slots[s];
    if (w.cap < clusters) {
        if (w.flags) cudaFree(w.flags);
        if (w.partial) cudaFree(w.partial);
        w = SkWorkspace{};
        const int cap = clusters < 128 ? 128 : clusters;
        if (cudaMalloc(&w.flags, cap * sizeof(unsigned)) != cudaSuccess) return nullptr;
        if (cudaMemset(w.flags, 0, cap * sizeof(unsigned)) != cudaSuccess) return nullptr;
        if (cudaMalloc(&w.partial, static_cast<size_t>(cap) * 256 * 256 * sizeof(float)) != cudaSuccess) return nullptr;
        w.cap = cap;
    }
    return &w;
}

SplitWorkspace *split_workspace(cudaStream_t s, size_t part_bytes, size_t count_words) {
    static std::mutex mu;
    static std::map<cudaStream_t, SplitWorkspace> slots;
    std::lock_guard<std::mutex> lk(mu);
    SplitWorkspace &w = slots[s];
    if (w.part_bytes < part_bytes) {
        if (w.part) cudaFree(w.part);
        w.part = nullptr;
        w.part_bytes = 0;
        if (cudaMalloc(&w.part, part_bytes) != cudaSuccess) return nullptr;
        w.part_bytes = part_bytes;
    }
    if (w.count_words < count_words) {
        if (w.count) cudaFree(w.count);
        w.count = nullptr;
        w.count_words = 0;
        if (cudaMalloc(&w.count, count_words * sizeof(unsigned)) != cudaSuccess) return nullptr;
        if (cudaMemset(w.count, 0, count_words * sizeof(unsigned)) != cudaSuccess) return nullptr;
        w.count_words = count_words;
    }
    return &w;
}

}  // namespace compar
