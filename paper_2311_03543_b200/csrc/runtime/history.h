// History-based variant selector (the StarPU-style performance model of PAPER.md P:118,
// P:224).  Host-only, no CUDA.
//
// Deliberate readings (R9-R13):
//   * key = (m_panel, n, k, dtype, compute, transB, beta==0), not SPEC's log2 footprint bucket;
//   * per (variant, key): seen (assigned executions incl. warm-ups and pending), count,
//     128-bit integer sums of ns and ns^2, min — the mean is order-independent and the
//     argmin comparison exact (cross-multiplication), so decisions are deterministic;
//   * calibration: while some eligible variant has seen < W + K, pick argmin seen
//     (ties -> lowest registry index; "interleaved") or the first variant in eligibility order with
//     seen < W + K ("blocked", R19); the first W executions of a variant are warm-ups (dropped);
//   * model: argmin mean ns over eligible variants with count > 0 (ties -> lowest index).
#pragma once
#include <cstdint>
#include <map>
#include <string>
#include <tuple>
#include <vector>

namespace compar {

struct Key {
    int64_t m, n, k;
    int dtype, compute, transB, beta0;
    bool operator<(const Key &o) const {
        return std::tie(m, n, k, dtype, compute, transB, beta0) <
               std::tie(o.m, o.n, o.k, o.dtype, o.compute, o.transB, o.beta0);
    }
    bool operator==(const Key &o) const {
        return m == o.m && n == o.n && k == o.k && dtype == o.dtype && compute == o.compute && transB == o.transB &&
               beta0 == o.beta0;
    }
};

struct Record {
    int64_t seen = 0;
    int64_t count = 0;
    unsigned __int128 sum_ns = 0;
    unsigned __int128 sumsq_ns = 0;
    int64_t min_ns = 0;
    int64_t warm_ns = 0;  // last discarded warm-up time (sizes the calibration batch, a8 / c13)
};

enum Mode { kWarmup = 0, kCalib = 1, kModel = 2, kEager = 3, kHint = 4, kNoop = 5, kPredict = 6 };

class History {
public:
    int calib_warmup = 1;
    int calib_k = 3;
    bool calib_blocked = true;

    // Records belong to variant NAMES (so a loaded perf model applies to whichever registry index
    // that name gets); names are interned to small ids for the hot path.
    int intern(const std::string &name);
    const std::string &name(int id) const { return names_[id]; }

    Record &rec(int id, const Key &k) { return table_[{id, k}]; }
    const Record *find(int id, const Key &k) const {
        auto it = table_.find({id, k});
        return it == table_.end() ? nullptr : &it->second;
    }
    // True if any eligible variant is still calibrating for this key.
    bool calibrating(const std::vector<int> &ids, const Key &k);
    // Decision over the ordered eligible list: returns the position in `ids`.
    int decide(const std::vector<int> &ids, const Key &k, Mode *mode);
    // Account an assigned execution; returns true if it is a warm-up.
    bool commit(int id, const Key &k);
    void harvest(int id, const Key &k, int64_t ns);

    const std::map<std::pair<int, Key>, Record> &table() const { return table_; }
    void merge(const std::string &variant, const Key &k, const Record &r);

    // ---- performance-model generalisation ("additional
    // training of these models").  For an unseen key, variant v's time is predicted from its own
    // measured keys of the same (dtype, compute, transB) family with
    //     t ~ w0 + w1 * flops + w2 * bytes,     w >= 0,
    // fitted by relative-error least squares (weights 1/t^2) over every non-empty feature subset,
    // keeping the non-negative solution of least weighted residual.  Needs >= kMinFitKeys keys.
    static constexpr int kMinFitKeys = 3;
    static void features(const Key &k, double *x);   // x[0..2] = 1, GFLOP, MB
    bool predict(int id, const Key &k, double *ns) const;
    // Decision of the "predict" scheduler: measured mean where (v, key) has samples, prediction
    // otherwise; returns -1 (caller falls back to calibration) if some variant has neither.
    int decide_predict(const std::vector<int> &ids, const Key &k, Mode *mode) const;
    // Positions (into ids) of the variants with neither a sample for k nor a prediction: the only
    // ones the predict scheduler still has to calibrate for k.
    std::vector<int> unknown_predict(const std::vector<int> &ids, const Key &k) const;

private:
    std::map<std::string, int> ids_;
    std::vector<std::string> names_;
    std::map<std::pair<int, Key>, Record> table_;
};

}  // namespace compar
