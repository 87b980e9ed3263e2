#include "history.h"

#include <array>
#include <cmath>
#include <utility>

namespace compar {

int History::intern(const std::string &name) {
    auto it = ids_.find(name);
    if (it != ids_.end()) return it->second;
    const int id = static_cast<int>(names_.size());
    names_.push_back(name);
    ids_.emplace(name, id);
    return id;
}

bool History::best_mean(const std::vector<int> &ids, const Key &k, unsigned __int128 *sum, int64_t *count) const {
    bool found = false;
    for (int id : ids) {
        const Record *r = find(id, k);
        if (!r || r->count == 0) continue;
        // r < best  <=>  r.sum * best.count < best.sum * r.count (exact)
        if (!found || r->sum_ns * static_cast<unsigned __int128>(*count) <
                          *sum * static_cast<unsigned __int128>(r->count)) {
            *sum = r->sum_ns;
            *count = r->count;
            found = true;
        }
    }
    return found;
}

namespace {
// The records of one decision's eligible variants, looked up once (the submit path is the paper's
// "decision overhead": one map lookup per variant instead of one per test).
struct KeyView {
    std::vector<Record *> r;
    bool have_best = false;
    unsigned __int128 bs = 0;   // best mean as the exact fraction bs / bc
    int64_t bc = 0;
};

void view(History &h, const std::vector<int> &ids, const Key &k, KeyView &v) {
    v.r.resize(ids.size());
    for (size_t i = 0; i < ids.size(); ++i) v.r[i] = &h.rec(ids[i], k);
    for (const Record *r : v.r) {
        if (r->count == 0) continue;
        if (!v.have_best || r->sum_ns * static_cast<unsigned __int128>(v.bc) <
                                v.bs * static_cast<unsigned __int128>(r->count)) {
            v.bs = r->sum_ns;
            v.bc = r->count;
            v.have_best = true;
        }
    }
}

// R32 on a prepared view.
bool pruned_in(const KeyView &v, int prune_pct, const std::vector<double> *lb, size_t i) {
    if (prune_pct <= 0 || !v.have_best) return false;
    const Record &r = *v.r[i];
    if (r.count > 0 && 100 * r.sum_ns * static_cast<unsigned __int128>(v.bc) >
                           static_cast<unsigned __int128>(prune_pct) * v.bs * static_cast<unsigned __int128>(r.count))
        return true;
    const double l = lb ? (*lb)[i] : 0.0;
    return l > 0.0 && l * 100.0 * static_cast<double>(v.bc) > static_cast<double>(prune_pct) * static_cast<double>(v.bs);
}
}  // namespace

bool History::pruned(const std::vector<int> &ids, const Key &k, const std::vector<double> *lb, size_t i) {
    KeyView v;
    view(*this, ids, k, v);
    return pruned_in(v, prune_pct, lb, i);
}

int History::warm_count(double lb_ns) const {
    if (long_warm_ms <= 0 || lb_ns < 10e6) return calib_warmup;
    const int w = static_cast<int>(std::ceil(static_cast<double>(long_warm_ms) * 1e6 / lb_ns));
    return w > 6 ? 6 : (w < calib_warmup ? calib_warmup : w);
}

bool History::calibrating(const std::vector<int> &ids, const Key &k, const std::vector<double> *lb) {
    KeyView v;
    view(*this, ids, k, v);
    for (size_t i = 0; i < ids.size(); ++i) {
        const int64_t need = static_cast<int64_t>(warm_count(lb ? (*lb)[i] : 0.0)) + calib_k;
        if (v.r[i]->seen < need && !pruned_in(v, prune_pct, lb, i)) return true;
    }
    return false;
}

int History::decide(const std::vector<int> &ids, const Key &k, Mode *mode, const std::vector<double> *lb) {
    KeyView v;
    view(*this, ids, k, v);
    // Calibration.  Interleaved: least-seen eligible variant, first in registry order on ties.
    // Blocked: the variant of smallest lower bound (ties: eligibility order) that has not completed
    // its W + K executions.  Pruned variants (R32) are done calibrating.
    int best = -1;
    int64_t best_seen = 0;
    double best_lb = 0.0;
    for (size_t i = 0; i < ids.size(); ++i) {
        const int64_t s = v.r[i]->seen;
        const double l = lb ? (*lb)[i] : 0.0;
        const int64_t need = static_cast<int64_t>(warm_count(l)) + calib_k;   // W + K (R39: W per variant)
        if (s >= need || pruned_in(v, prune_pct, lb, i)) continue;
        if (calib_blocked) {
            if (best < 0 || l < best_lb) {
                best = static_cast<int>(i);
                best_seen = s;
                best_lb = l;
            }
        } else if (best < 0 || s < best_seen) {
            best = static_cast<int>(i);
            best_seen = s;
        }
    }
    if (best >= 0) {
        *mode = best_seen < warm_count(lb ? (*lb)[best] : 0.0) ? kWarmup : kCalib;
        return best;
    }
    // Model: argmin of sum/count compared as sum_a * count_b < sum_b * count_a (exact).
    best = -1;
    for (size_t i = 0; i < ids.size(); ++i) {
        const Record &r = *v.r[i];
        if (r.count == 0) continue;
        if (best < 0) {
            best = static_cast<int>(i);
            continue;
        }
        const Record &b = *v.r[best];
        // 128-bit products: sums < 2^96 in practice, counts < 2^31.
        if (r.sum_ns * static_cast<unsigned __int128>(b.count) < b.sum_ns * static_cast<unsigned __int128>(r.count))
            best = static_cast<int>(i);
    }
    *mode = kModel;
    return best < 0 ? 0 : best;
}

bool History::commit(int id, const Key &k, int warm_n) {
    Record &r = rec(id, k);
    const bool warm = r.seen < warm_n;
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

void History::features(const Key &k, double *x) {
    const double m = static_cast<double>(k.m), n = static_cast<double>(k.n), kk = static_cast<double>(k.k);
    const double eb = k.dtype == 1 ? 2.0 : 4.0;
    x[0] = 1.0;
    x[1] = 2.0 * m * n * kk * 1e-9;
    x[2] = (eb * (m * kk + kk * n) + 4.0 * m * n * (k.beta0 ? 1.0 : 2.0)) * 1e-6;
}

namespace {
// Solve the s x s system a * w = b (Gaussian elimination, partial pivoting); false if singular.
bool solve(int s, double a[3][3], double b[3], double w[3]) {
    for (int c = 0; c < s; ++c) {
        int p = c;
        for (int r = c + 1; r < s; ++r)
            if (std::fabs(a[r][c]) > std::fabs(a[p][c])) p = r;
        if (std::fabs(a[p][c]) < 1e-300) return false;
        if (p != c) {
            for (int j = 0; j < s; ++j) std::swap(a[p][j], a[c][j]);
            std::swap(b[p], b[c]);
        }
        for (int r = c + 1; r < s; ++r) {
            const double f = a[r][c] / a[c][c];
            for (int j = c; j < s; ++j) a[r][j] -= f * a[c][j];
            b[r] -= f * b[c];
        }
    }
    for (int c = s - 1; c >= 0; --c) {
        double v = b[c];
        for (int j = c + 1; j < s; ++j) v -= a[c][j] * w[j];
        w[c] = v / a[c][c];
    }
    return true;
}
}  // namespace

bool History::predict(int id, const Key &q, double *ns) const {
    // samples of the same family: (x, t) with t = mean ns
    std::vector<std::pair<std::array<double, 3>, double>> pts;
    for (const auto &kv : table_) {
        if (kv.first.first != id || kv.second.count == 0) continue;
        const Key &k = kv.first.second;
        if (k.dtype != q.dtype || k.compute != q.compute || k.transB != q.transB) continue;
        std::array<double, 3> x;
        features(k, x.data());
        pts.push_back({x, static_cast<double>(kv.second.sum_ns) / static_cast<double>(kv.second.count)});
    }
    if (static_cast<int>(pts.size()) < kMinFitKeys) return false;
    double best_res = 0, best_w[3] = {0, 0, 0};
    bool found = false;
    for (int mask = 1; mask < 8; ++mask) {
        int cols[3], s = 0;
        for (int j = 0; j < 3; ++j)
            if (mask >> j & 1) cols[s++] = j;
        double a[3][3] = {}, b[3] = {}, w[3] = {};
        for (const auto &p : pts) {
            const double wt = 1.0 / (p.second * p.second + 1.0);
            for (int r = 0; r < s; ++r) {
                b[r] += wt * p.first[cols[r]] * p.second;
                for (int c2 = 0; c2 < s; ++c2) a[r][c2] += wt * p.first[cols[r]] * p.first[cols[c2]];
            }
        }
        if (!solve(s, a, b, w)) continue;
        bool nonneg = true;
        for (int r = 0; r < s; ++r) nonneg = nonneg && w[r] >= 0.0;
        if (!nonneg) continue;
        double full[3] = {0, 0, 0};
        for (int r = 0; r < s; ++r) full[cols[r]] = w[r];
        double res = 0;
        for (const auto &p : pts) {
            const double pr = full[0] * p.first[0] + full[1] * p.first[1] + full[2] * p.first[2];
            const double e = (pr - p.second) / p.second;
            res += e * e;
        }
        if (!found || res < best_res) {
            found = true;
            best_res = res;
            for (int j = 0; j < 3; ++j) best_w[j] = full[j];
        }
    }
    if (!found) return false;
    double x[3];
    features(q, x);
    *ns = best_w[0] * x[0] + best_w[1] * x[1] + best_w[2] * x[2];
    return true;
}

bool History::estimate(int id, const Key &k, double *est, bool *pred) const {
    const Record *r = find(id, k);
    if (r && r->count > 0) {
        *est = static_cast<double>(r->sum_ns) / static_cast<double>(r->count);
        *pred = false;
        return true;
    }
    *pred = true;
    return predict(id, k, est);
}

int History::decide_predict(const std::vector<int> &ids, const Key &k, Mode *mode, const std::vector<double> *lb) const {
    // best estimate over the variants that have one (for the lower-bound skip of the others)
    double floor_est = 0.0;
    bool have = false;
    std::vector<double> est(ids.size(), 0.0);
    std::vector<char> known(ids.size(), 0), pred(ids.size(), 0);
    for (size_t i = 0; i < ids.size(); ++i) {
        bool p = false;
        if (estimate(ids[i], k, &est[i], &p)) {
            known[i] = 1;
            pred[i] = p ? 1 : 0;
            if (!have || est[i] < floor_est) floor_est = est[i];
            have = true;
        }
    }
    int best = -1;
    for (size_t i = 0; i < ids.size(); ++i) {
        if (!known[i]) {
            const double l = lb ? (*lb)[i] : 0.0;
            if (have && prune_pct > 0 && l > 0.0 && l * 100.0 > static_cast<double>(prune_pct) * floor_est) continue;
            return -1;
        }
        if (best < 0 || est[i] < est[best]) best = static_cast<int>(i);
    }
    if (best < 0) return -1;
    if (!pred[best] && explore_pct > 0) {
        // R37: the best estimate is a measured mean; a variant known only by its prediction,
        // predicted within explore_pct/100 of it, is measured (W + 1 runs) before it is trusted.
        for (size_t i = 0; i < ids.size(); ++i)
            if (known[i] && pred[i] && est[i] * 100.0 <= static_cast<double>(explore_pct) * est[best]) {
                const Record *r = find(ids[i], k);
                *mode = (r ? r->seen : 0) < warm_count(lb ? (*lb)[i] : 0.0) ? kWarmup : kCalib;
                return static_cast<int>(i);
            }
    }
    *mode = pred[best] ? kPredict : kModel;
    return best;
}

std::vector<int> History::unknown_predict(const std::vector<int> &ids, const Key &k, const std::vector<double> *lb) const {
    double floor_est = 0.0;
    bool have = false;
    std::vector<int> unk;
    for (size_t i = 0; i < ids.size(); ++i) {
        double e;
        bool p;
        if (estimate(ids[i], k, &e, &p)) {
            if (!have || e < floor_est) floor_est = e;
            have = true;
        } else {
            unk.push_back(static_cast<int>(i));
        }
    }
    std::vector<int> out;
    for (int i : unk) {
        const double l = lb ? (*lb)[i] : 0.0;
        if (have && prune_pct > 0 && l > 0.0 && l * 100.0 > static_cast<double>(prune_pct) * floor_est) continue;
        out.push_back(i);
    }
    return out;
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
