#include "history.h"

namespace compar {

bool History::calibrating(const std::vector<std::string> &names, const Key &k) {
    const int64_t need = static_cast<int64_t>(calib_warmup) + calib_k;
    for (const auto &n : names)
        if (rec(n, k).seen < need) return true;
    return false;
}

int History::decide(const std::vector<std::string> &names, const Key &k, Mode *mode) {
    const int64_t need = static_cast<int64_t>(calib_warmup) + calib_k;
    // Calibration: least-seen eligible variant, first in registry order on ties.
    int best = -1;
    int64_t best_seen = 0;
    for (size_t i = 0; i < names.size(); ++i) {
        const int64_t s = rec(names[i], k).seen;
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
    for (size_t i = 0; i < names.size(); ++i) {
        const Record &r = rec(names[i], k);
        if (r.count == 0) continue;
        if (best < 0) {
            best = static_cast<int>(i);
            continue;
        }
        const Record &b = rec(names[best], k);
        // 128-bit products: sums < 2^96 in practice, counts < 2^31.
        if (r.sum_ns * static_cast<unsigned __int128>(b.count) < b.sum_ns * static_cast<unsigned __int128>(r.count))
            best = static_cast<int>(i);
    }
    *mode = kModel;
    return best < 0 ? 0 : best;
}

bool History::commit(const std::string &variant, const Key &k) {
    Record &r = rec(variant, k);
    const bool warm = r.seen < calib_warmup;
    ++r.seen;
    return warm;
}

void History::harvest(const std::string &variant, const Key &k, int64_t ns) {
    Record &r = rec(variant, k);
    if (ns < 0) ns = 0;
    r.min_ns = r.count == 0 ? ns : (ns < r.min_ns ? ns : r.min_ns);
    ++r.count;
    r.sum_ns += static_cast<unsigned __int128>(ns);
    r.sumsq_ns += static_cast<unsigned __int128>(ns) * static_cast<unsigned __int128>(ns);
}

void History::merge(const std::string &variant, const Key &k, const Record &in) {
    Record &r = rec(variant, k);
    if (in.count > 0) r.min_ns = r.count == 0 ? in.min_ns : (in.min_ns < r.min_ns ? in.min_ns : r.min_ns);
    r.seen += in.seen;
    r.count += in.count;
    r.sum_ns += in.sum_ns;
    r.sumsq_ns += in.sumsq_ns;
}

}  // namespace compar
