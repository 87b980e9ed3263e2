#include "history.h"

namespace compar {

int History::intern(const std::string &name) {
    auto it = ids_.find(name);
    if (it != ids_.end()) return it->second;
    const int id = static_cast<int>(names_.size());
    names_.push_back(name);
    ids_.emplace(name, id);
    return id;
}

bool History::calibrating(const std::vector<int> &ids, const Key &k) {
    const int64_t need = static_cast<int64_t>(calib_warmup) + calib_k;
    for (int id : ids)
        if (rec(id, k).seen < need) return true;
    return false;
}

int History::decide(const std::vector<int> &ids, const Key &k, Mode *mode) {
    const int64_t need = static_cast<int64_t>(calib_warmup) + calib_k;
    // Calibration: least-seen eligible variant, first in registry order on ties.
    int best = -1;
    int64_t best_seen = 0;
    for (size_t i = 0; i < ids.size(); ++i) {
        const int64_t s = rec(ids[i], k).seen;
        if (best < 0 || s < best_seen) {
            best = static_cast<int>(i);
            best_seen = s;
        }
    }
    if (best >= 0 && best_seen < need) {
        *mode = best_seen < calib_warmup ? kWarmup : kCalib;
        return best;
    }
    // Model: argmin of sum/count compared as sum_a * count_b < sum_b * count_a (exact).
    best = -1;
    for (size_t i = 0; i < ids.size(); ++i) {
        const Record &r = rec(ids[i], k);
        if (r.count == 0) continue;
        if (best < 0) {
            best = static_cast<int>(i);
            continue;
        }
        const Record &b = rec(ids[best], k);
        // 128-bit products: sums < 2^96 in practice, counts < 2^31.
        if (r.sum_ns * static_cast<unsigned __int128>(b.count) < b.sum_ns * static_cast<unsigned __int128>(r.count))
            best = static_cast<int>(i);
    }
    *mode = kModel;
    return best < 0 ? 0 : best;
}

bool History::commit(int id, const Key &k) {
    Record &r = rec(id, k);
    const bool warm = r.seen < calib_warmup;
    ++r.seen;
    return warm;
}

void History::harvest(int id, const Key &k, int64_t ns) {
    Record &r = rec(id, k);
    if (ns < 0) ns = 0;
    r.min_ns = r.count == 0 ? ns : (ns < r.min_ns ? ns : r.min_ns);
    ++r.count;
    r.sum_ns += static_cast<unsigned __int128>(ns);
    r.sumsq_ns += static_cast<unsigned __int128>(ns) * static_cast<unsigned __int128>(ns);
}

void History::merge(const std::string &variant, const Key &k, const Record &in) {
    Record &r = rec(intern(variant), k);
    if (in.count > 0) r.min_ns = r.count == 0 ? in.min_ns : (in.min_ns < r.min_ns ? in.min_ns : r.min_ns);
    r.seen += in.seen;
    r.count += in.count;
    r.sum_ns += in.sum_ns;
    r.sumsq_ns += in.sumsq_ns;
}

}  // namespace compar
