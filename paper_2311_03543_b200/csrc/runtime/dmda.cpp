#include "dmda.h"

#include <algorithm>

namespace compar {

namespace {
bool overlap(const Span &a, const Span &b) { return a.lo < b.hi && b.lo < a.hi && a.lo < a.hi && b.lo < b.hi; }
}  // namespace

void Placer::configure(int nranks, int lanes) {
    nranks_ = nranks < 1 ? 1 : nranks;
    lanes_ = lanes < 1 ? 1 : lanes;
    reset();
}

void Placer::reset() {
    ready_.assign(static_cast<size_t>(nranks_) * lanes_, 0);
    live_.clear();
}

int Placer::place(const Access &a, int64_t exec_ns, int64_t *end, std::vector<uint64_t> *deps) const {
    // Residency: each byte a task reads is valid only on the rank of its latest writer.  Per read
    // span, walk the overlapping writers from the latest back, each claiming the part of the span
    // no later writer covers; every claiming writer's rank must agree (a span whose bytes were
    // last written on two ranks cannot be read anywhere: no inter-rank transfer, R22).
    int pin = -1;
    for (const Span &s : a.reads) {
        std::vector<const Live *> ws;
        for (const Live &l : live_)
            if (l.write && overlap(s, l.s)) ws.push_back(&l);
        std::sort(ws.begin(), ws.end(), [](const Live *x, const Live *y) { return x->task > y->task; });
        std::vector<Span> open{s};          // parts of s no later writer has covered yet
        for (const Live *l : ws) {
            std::vector<Span> rest;
            bool claims = false;
            for (const Span &u : open) {
                if (!overlap(u, l->s)) {
                    rest.push_back(u);
                    continue;
                }
                claims = true;
                if (u.lo < l->s.lo) rest.push_back({u.lo, l->s.lo});
                if (l->s.hi < u.hi) rest.push_back({l->s.hi, u.hi});
            }
            open.swap(rest);
            if (!claims) continue;
            const int r = rank_of(l->w);
            if (pin >= 0 && pin != r) return -1;
            pin = r;
            if (open.empty()) break;
        }
    }
    const int W = workers();
    int best = -1;
    int64_t best_end = 0;
    for (int w = 0; w < W; ++w) {
        if (pin >= 0 && rank_of(w) != pin) continue;
        int64_t est = ready_[w];
        for (const Live &l : live_) {
            if (rank_of(l.w) != rank_of(w)) continue;  // other ranks hold other copies
            bool conflict = false;
            for (const Span &s : a.reads)
                if (l.write && overlap(s, l.s)) conflict = true;  // RAW
            for (const Span &s : a.writes)
                if (overlap(s, l.s)) conflict = true;  // WAW / WAR
            if (conflict) est = std::max(est, l.end);
        }
        const int64_t e = est + exec_ns;
        if (best < 0 || e < best_end) {
            best = w;
            best_end = e;
        }
    }
    if (best < 0) return -1;
    *end = best_end;
    if (deps) {
        deps->clear();
        for (const Live &l : live_) {
            if (rank_of(l.w) != rank_of(best) || l.w == best) continue;  // same lane: stream order
            bool conflict = false;
            for (const Span &s : a.reads)
                if (l.write && overlap(s, l.s)) conflict = true;
            for (const Span &s : a.writes)
                if (overlap(s, l.s)) conflict = true;
            if (conflict && std::find(deps->begin(), deps->end(), l.task) == deps->end()) deps->push_back(l.task);
        }
    }
    return best;
}

void Placer::commit(uint64_t task, int w, int64_t end, const Access &a) {
    ready_[w] = end;
    for (const Span &s : a.reads) live_.push_back({task, w, end, s, false});
    for (const Span &s : a.writes) live_.push_back({task, w, end, s, true});
}

}  // namespace compar
