// Per-stream tile-scheduler workspace for the persistent tcgen05 kernels.
//
// Each persistent launch draws output tiles from a global atomic counter, so the set of tiles
// in flight is always a contiguous range in raster order however the CTAs drift relative to
// each other (a static round-robin schedule lets CTAs drift apart by whole tiles over a long
// K, which destroys L2 reuse between CTAs that share A rows / B columns — DESIGN.md §5).
// The counter pair {next, done} is zeroed once and re-zeroed by the last CTA of every launch;
// launches on one stream are ordered, so one pair per stream is enough.
#include <cuda_runtime.h>

#include <cstdlib>
#include <map>
#include <mutex>

#include "kernels.h"

namespace compar {

Knobs read_knobs() {
    auto get = [](const char *name, int dflt) {
        const char *v = std::getenv(name);
        return (v && *v) ? std::atoi(v) : dflt;
    };
    Knobs k;
    k.tc1_bn = get("COMPAR_TC1_BN", 0);
    k.tc1_group = get("COMPAR_TC1_GROUP", 0);
    k.tc2_bn = get("COMPAR_TC2_BN", 0);
    k.tc2_group = get("COMPAR_TCM_GROUP", 0);
    k.tc2_rowstore_group = get("COMPAR_TC_GROUP", 0);
    k.tc2_producers = get("COMPAR_TC2_PRODUCERS", 2) == 1 ? 1 : 2;
    k.even_waves = get("COMPAR_EVEN_WAVES", 1) != 0;
    k.tc2_deep = get("COMPAR_TC2_DEEP", 1) != 0;
    k.tc2_tmem_cin = get("COMPAR_TC2_TMEM_CIN", 1) != 0;
    k.tcw_group = get("COMPAR_TCW_GROUP", 0);
    k.tcw_delay = get("COMPAR_TCW_DELAY", 24);
    if (k.tcw_delay < 0) k.tcw_delay = 0;
    k.tma_tile = get("COMPAR_TMA_TILE", 0);
    return k;
}

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

namespace {
std::mutex g_split_mu;
std::map<cudaStream_t, SplitWorkspace> g_split;
}  // namespace

void release_split_workspaces() {
    std::lock_guard<std::mutex> lk(g_split_mu);
    for (auto &kv : g_split) {
        if (kv.second.part) cudaFree(kv.second.part);
        if (kv.second.count) cudaFree(kv.second.count);
    }
    g_split.clear();
}

SplitWorkspace *split_workspace(cudaStream_t s, size_t part_bytes, size_t count_words) {
    std::lock_guard<std::mutex> lk(g_split_mu);
    auto &slots = g_split;
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
