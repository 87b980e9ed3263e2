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
//   * model: argmin mean ns over eligible variants with count > 0 (ties -> lowest index);
//   * calibration pruning (R32; VERDICT r1 "bound the calibration cost"): with
//     prune = P percent > 0, a variant stops calibrating for a key as soon as its mean exceeds
//     P/100 x the best mean of the key, or its static lower bound lb (FLOPs at its class's nominal
//     peak, bytes at nominal HBM) exceeds P/100 x that best mean; blocked calibration visits the
//     variants in increasing lb (ties: eligibility order), so the fast classes set the best mean
//     before the slow ones are considered.  lb = 0 (USER variants, other interfaces) never prunes
//     statically and keeps the eligibility order.
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
    int prune_pct = 300;   // 0: no pruning (SPEC S:363-371 behaviour)
    int explore_pct = 150; // predict mode (R37): measure a predicted variant within this % of the measured best
    int long_warm_ms = 200; // R39: variants whose static lower bound is >= 10 ms warm up for ~this long (0: off)

    // R39: warm-up executions of a variant whose static lower bound is lb_ns: W, or for long kernels
    // (lb >= 10 ms) enough to run ~long_warm_ms first (at most 6) — their timed samples then see the
    // power-capped steady state the model-mode runs will see, not the boost of a cool GPU.
    int warm_count(double lb_ns) const;

    // Records belong to variant NAMES (so a loaded perf model applies to whichever registry index
    // that name gets); names are interned to small ids for the hot path.
    int intern(const std::string &name);
    const std::string &name(int id) const { return names_[id]; }

    Record &rec(int id, const Key &k) { return table_[{id, k}]; }
    const Record *find(int id, const Key &k) const {
        auto it = table_.find({id, k});
        return it == table_.end() ? nullptr : &it->second;
    }
    // True if any eligible variant is still calibrating for this key (pruned ones are done).
    // lb: per position of ids, the static lower bound in ns (nullptr or 0 entries: none).
    bool calibrating(const std::vector<int> &ids, const Key &k, const std::vector<double> *lb = nullptr);
    // Decision over the ordered eligible list: returns the position in `ids`.
    int decide(const std::vector<int> &ids, const Key &k, Mode *mode, const std::vector<double> *lb = nullptr);
    // R32: is position i of ids pruned from calibration for k?
    bool pruned(const std::vector<int> &ids, const Key &k, const std::vector<double> *lb, size_t i);
    // Account an assigned execution (warm: its variant's warm_count); returns true if it is a warm-up.
    bool commit(int id, const Key &k, int warm);
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
    // A variant with neither whose lower bound exceeds prune_pct/100 x the best estimate is skipped.
    // R37: when the best estimate is measured, the first variant (eligibility order) known only by
    // a prediction within explore_pct/100 of it is returned instead, as a warm-up / calibration run.
    int decide_predict(const std::vector<int> &ids, const Key &k, Mode *mode,
                       const std::vector<double> *lb = nullptr) const;
    // Positions (into ids) of the variants with neither a sample for k nor a prediction (and not
    // skipped by their lower bound): the only ones the predict scheduler still has to calibrate.
    std::vector<int> unknown_predict(const std::vector<int> &ids, const Key &k,
                                     const std::vector<double> *lb = nullptr) const;

private:
    // best (smallest) mean over ids with samples: as the exact fraction sum / count; false if none
    bool best_mean(const std::vector<int> &ids, const Key &k, unsigned __int128 *sum, int64_t *count) const;
    // predict-mode estimate of position i (measured mean, else prediction); false if neither
    bool estimate(int id, const Key &k, double *est, bool *pred) const;
    std::map<std::string, int> ids_;
    std::vector<std::string> names_;
    std::map<std::pair<int, Key>, Record> table_;
};

}  // namespace compar
