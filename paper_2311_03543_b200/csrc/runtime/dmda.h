// Task-level placement for the task-parallel world (desc.world = COMPAR_WORLD_TASKS) — SURVEY
// §8(f) NEXT-1: "choose (variant, GPU) by expected completion = device ready time + predicted ns,
// StarPU dmda-style, with multi-stream dependency tracking by buffer" ("mapping,
// scheduling, and data transfers"; SPEC S:326-330 SchedulerDecision, S:366 schedule).  Host-only.
//
// Workers are (rank, lane) pairs, w = rank * lanes + lane: one process per GPU, `lanes` library
// streams per GPU.  Every rank runs this placer on the same submission sequence, so every rank
// computes the same decisions without communicating (the history they read is kept identical by
// the sample exchange in compar.cpp).
//
// Readings (R20-R23):
//   * ready[w] is a virtual clock: the predicted end of the last task placed on w; a full sync
//     (compar_sync(COMPAR_TASK_ALL)) resets it and forgets all accesses;
//   * dependencies are tracked on the byte ranges a task reads (A, B, C_in) and writes (C_out),
//     against the accesses of tasks placed since the last full sync: read-after-write,
//     write-after-read and write-after-write on the same rank order the task after the earlier one
//     (its earliest start is the earlier task's predicted end; lanes wait on its end event);
//   * ranks hold separate copies of every buffer and nothing moves data between ranks, so a task
//     that READS a range last written by a task on rank r can only run on rank r (transfer cost
//     infinite elsewhere); WAR / WAW across ranks touch different copies and need no ordering;
//   * model decision: argmin over allowed workers of est_start(w) + exec (workers are identical
//     GPUs, so the variant argmin is the selector's); ties -> lowest worker.
#pragma once
#include <cstdint>
#include <vector>

namespace compar {

struct Span {
    uintptr_t lo, hi;  // [lo, hi)
};

struct Access {
    std::vector<Span> reads, writes;
};

class Placer {
public:
    void configure(int nranks, int lanes);
    int workers() const { return nranks_ * lanes_; }
    int lanes() const { return lanes_; }
    int rank_of(int w) const { return w / lanes_; }
    // Chooses the worker for a task of predicted duration `exec_ns`.  Returns -1 if no worker may
    // run it (its reads span data last written on two different ranks).  *end = predicted end;
    // deps = tasks on the chosen worker's rank (other lanes included) that must finish first.
    int place(const Access &a, int64_t exec_ns, int64_t *end, std::vector<uint64_t> *deps) const;
    void commit(uint64_t task, int w, int64_t end, const Access &a);
    void reset();
    int64_t ready(int w) const { return ready_[w]; }

private:
    struct Live {
        uint64_t task;
        int w;
        int64_t end;
        Span s;
        bool write;
    };
    int nranks_ = 1, lanes_ = 1;
    std::vector<int64_t> ready_;
    std::vector<Live> live_;
};

}  // namespace compar
