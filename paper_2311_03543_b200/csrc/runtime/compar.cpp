// libcompar runtime: the C ABI of include/compar.h over the sm_100a kernels.
//
// Maps the paper's runtime model onto one B200 per process:
//   * variant registry        <- method_declare interface/target/name and
//                                the StarPU codelet;
//   * task submit / sync      <- "creation and the submission of the task" and the
//                                unregister-after-wait rule;
//   * history selector        <- "the STARPU decision-making process relies on ... models"
//                                (P:224), algorithm in history.{h,cpp};
//   * row panels + NCCL bcast <- BASELINE.json north star (multi-GPU, one process per GPU);
//   * task-parallel world     <- StarPU "mapping, scheduling" across workers, dmda
//                                placement in dmda.{h,cpp}.
#include "compar.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "../kernels/kernels.h"
#include "dmda.h"
#include "history.h"

namespace compar {
namespace {

thread_local std::string t_err;

// NVTX ranges around the runtime's phases (select, bcast, launch, harvest, sync): visible in any
// NVTX-aware profiler, a few ns each when none is attached (header-only nvtx3).
struct Range {
    explicit Range(const char *name) { nvtxRangePushA(name); }
    ~Range() { nvtxRangePop(); }
    Range(const Range &) = delete;
    Range &operator=(const Range &) = delete;
};

compar_status fail(compar_status s, const std::string &msg) {
    t_err = msg;
    return s;
}
compar_status cuda_fail(cudaError_t e, const char *what) {
    return fail(COMPAR_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

enum Iface { kGemm = 0, kSort = 1, kGeneric = 2 };

struct Variant {
    std::string name;
    compar_target target;
    compar_gemm_fn fn;
    void *user;
    int hid;  // interned history id of `name`
    int iface = kGemm;
    compar_sort_fn sfn = nullptr;
    std::string giface;               // generic interface name
    compar_generic_fn gfn = nullptr;
};

thread_local void *t_current_stream = nullptr;   // compar_current_stream() inside a generic variant

struct PanelRun {
    compar_panel p{};
    int batch = 1;  // launches between start and stop (batched calibration timing)
    cudaEvent_t start = nullptr, stop = nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> sub;  // per-chunk kernel spans (host pipeline)
    int64_t virtual_ns = 0;
};

struct Task {
    uint64_t id = 0;
    Key key{};
    int variant = -1;
    int mode = kNoop;
    bool warm = false;
    bool history = false;  // sample goes to the history when harvested
    compar_status status = COMPAR_OK;
    std::vector<PanelRun> panels;
    cudaEvent_t begin = nullptr, end = nullptr, bc0 = nullptr, bc1 = nullptr;
    std::vector<cudaEvent_t> extra;  // per-slab broadcast events (world mode)
    bool world = false;
    // task-parallel world (world = COMPAR_WORLD_TASKS)
    bool tasks = false;
    bool remote = false;   // placed on another rank: no launch here, sample arrives by exchange
    int owner = 0, lane = 0;
    bool have_xns = false;
    int64_t xns = 0;       // exchanged sample (-2: the owner's execution failed)
};

struct Ctx {
    std::mutex mu;
    compar_config cfg{};
    bool virt = false;
    int device = 0, num_sms = 148;
    cudaStream_t stream = nullptr;
    std::vector<cudaEvent_t> pool;
    std::vector<Variant> variants;
    History hist;
    uint64_t next_task = 1;
    std::map<uint64_t, Task> tasks;
    compar_stats stats{};
    std::string perf_path;
    void *staging[4] = {nullptr, nullptr, nullptr, nullptr};
    size_t staging_bytes[4] = {0, 0, 0, 0};
    void *breplica = nullptr;
    size_t breplica_bytes = 0;
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    int64_t *red_buf = nullptr;  // device scalar for the rank-consistent sample all-reduce
    compar_reduce_fn reduce_hook = nullptr;
    void *reduce_user = nullptr;
    // world-mode broadcast pipeline
    cudaStream_t comm_stream = nullptr;
    cudaStream_t aux_stream = nullptr;   // world mode: the GEMM's extra CTAs launched after the broadcast
    uint32_t *slab_flags = nullptr;      // world mode: per-slab "landed" words read by the fused GEMM
    uint32_t slab_seq = 0;               // world broadcasts issued (flag value of the current one)
    void *bpacked = nullptr;  // root: B packed into contiguous N-slabs
    size_t bpacked_bytes = 0;
    int bcast_loopback = 0;       // 1 rank: emulate the broadcast with D2D copies (tests the slab path);
                                  // 2: also leave the NCCL SM reserve (exercises the helper launch)
    int bcast_reserve_sms = 16;   // SMs left free for NCCL while a slab GEMM overlaps a broadcast
    // copy-engine chain broadcast (compar_ce_export / compar_ce_import): no NCCL, no SMs
    bool ce = false;
    void *ce_buf = nullptr;        // own chain buffer (root: packed slabs; others: the replica)
    size_t ce_cap = 0;
    uint32_t *ce_flags = nullptr;  // [0, kCeMax): ready (written by self); [kCeMax, 2 kCeMax): consumed
                                   // (written by the downstream rank after copying a chunk out)
    void *ce_up_buf = nullptr;     // upstream rank's buffer and flags (IPC-mapped; ranks > 0)
    uint32_t *ce_up_flags = nullptr;
    uint32_t ce_seq = 0;           // world broadcasts issued (identical on every rank: SPMD)
    // host-memory pipeline
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
    int host_chunks = 32;   // row chunks of the host-memory pipeline (32768-row bench: 8 -> 32 chunks, e2e 178 -> 170 ms)
    int host_tail_split = 1;   // COMPAR_HOST_TAIL_SPLIT=0: uniform chunks to the end
    int d2h_kernel_ctas = 4;   // COMPAR_D2H_KERNEL_CTAS: CTAs of the mapped-memory D2H copy (0: copy engine)
    // task-parallel world
    Placer placer;
    bool placer_ready = false;
    std::vector<cudaStream_t> lane_streams;
    std::vector<cudaEvent_t> lane_done;
    cudaEvent_t sub_event = nullptr, cal_fence = nullptr;
    bool cal_fence_set = false;
    compar_reduce_n_fn reduce_n_hook = nullptr;
    void *reduce_n_user = nullptr;
    int64_t *xbuf = nullptr;  // device buffer of the NCCL sample exchange
    size_t xbuf_n = 0;
    // sort interface
    void *sort_scratch = nullptr;
    size_t sort_scratch_bytes = 0;
    cudaEvent_t sort_done = nullptr;  // end of the last sort task (sort tasks share the scratch)
    bool sort_done_set = false;
    // batched calibration timing (a8 / c13)
    int64_t batch_below_ns = 100000;
    void *scratch = nullptr;  // C_out of the r - 1 extra launches
    size_t scratch_bytes = 0;
    // reports of tasks the selector harvested implicitly (step 6), kept until compar_sync
    std::map<uint64_t, std::pair<compar_status, compar_report>> done;
    bool in_select = false;   // compar_select: never harvest tasks whose harvest is collective
    // the next task that reuses a shared library buffer waits for the previous user to finish
    cudaEvent_t staging_free = nullptr;   // host-mode staging buffers
    bool staging_free_set = false;
    cudaEvent_t bcast_free = nullptr;     // world-mode packed B / replica / slab flags
    bool bcast_free_set = false;
    // NCCL robustness: bounded waits, sticky failure after an asynchronous error or a timeout
    int64_t sync_timeout_ms = 600000;
    compar_status sticky = COMPAR_OK;
    std::string sticky_msg;
    Knobs knobs;              // launcher tuning knobs, read from the environment once at init
};

std::mutex g_live_mu;
std::set<Ctx *> g_live;

Ctx *as_ctx(void *p) {
    std::lock_guard<std::mutex> lk(g_live_mu);
    Ctx *c = static_cast<Ctx *>(p);
    return g_live.count(c) ? c : nullptr;
}

int env_int(const char *name, int dflt) {
    const char *v = std::getenv(name);
    if (!v || !*v) return dflt;
    char *end = nullptr;
    long x = std::strtol(v, &end, 10);
    return (end && *end == 0) ? static_cast<int>(x) : dflt;
}

int elem_bytes(compar_dtype d) { return d == COMPAR_BF16 ? 2 : 4; }

std::string u128_str(unsigned __int128 v) {
    if (v == 0) return "0";
    char buf[48];
    int i = 47;
    buf[i] = 0;
    while (v > 0) {
        buf[--i] = static_cast<char>('0' + static_cast<int>(v % 10));
        v /= 10;
    }
    return std::string(buf + i);
}
bool parse_u128(const std::string &s, unsigned __int128 *out) {
    if (s.empty()) return false;
    unsigned __int128 v = 0;
    for (char c : s) {
        if (c < '0' || c > '9') return false;
        v = v * 10 + static_cast<unsigned>(c - '0');
    }
    *out = v;
    return true;
}

// ---------------------------------------------------------------- events
cudaEvent_t get_event(Ctx *c) {
    if (!c->pool.empty()) {
        cudaEvent_t e = c->pool.back();
        c->pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    return e;
}
void put_event(Ctx *c, cudaEvent_t &e) {
    if (e) c->pool.push_back(e);
    e = nullptr;
}
void release_task_events(Ctx *c, Task &t) {
    for (auto &p : t.panels) {
        put_event(c, p.start);
        put_event(c, p.stop);
        for (auto &s : p.sub) {
            put_event(c, s.first);
            put_event(c, s.second);
        }
        p.sub.clear();
    }
    put_event(c, t.begin);
    put_event(c, t.end);
    put_event(c, t.bc0);
    put_event(c, t.bc1);
    for (auto &e : t.extra) put_event(c, e);
    t.extra.clear();
}
int64_t elapsed_ns(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    if (!a || !b || cudaEventElapsedTime(&ms, a, b) != cudaSuccess) return 0;
    return static_cast<int64_t>(std::llround(static_cast<double>(ms) * 1e6));
}

// ---------------------------------------------------------------- partition (a4)
void partition(int64_t m, int p, std::vector<int64_t> &offs) {
    offs.assign(static_cast<size_t>(p) + 1, 0);
    const int64_t per = (m + p - 1) / p;
    const int64_t base = ((per + 127) / 128) * 128;
    for (int r = 0; r < p; ++r) offs[r] = std::min(m, static_cast<int64_t>(r) * base);
    offs[p] = m;
}

// ---------------------------------------------------------------- validation
compar_status validate(Ctx *c, const compar_gemm_desc *d) {
    if (!d) return fail(COMPAR_E_INVALID, "desc is NULL");
    if (d->m < 0 || d->n < 0 || d->k < 0) return fail(COMPAR_E_INVALID, "negative dimension");
    if (d->in_dtype != COMPAR_F32 && d->in_dtype != COMPAR_BF16) return fail(COMPAR_E_INVALID, "bad in_dtype");
    if (d->compute < COMPAR_COMPUTE_F32_STRICT || d->compute > COMPAR_COMPUTE_F32_SPLIT)
        return fail(COMPAR_E_INVALID, "bad compute");
    if ((d->in_dtype == COMPAR_BF16) != (d->compute == COMPAR_COMPUTE_BF16))
        return fail(COMPAR_E_INVALID, "BF16 storage requires COMPUTE_BF16 and vice versa");
    if (d->transB != 0 && d->transB != 1) return fail(COMPAR_E_INVALID, "transB must be 0 or 1");
    if (d->mem != COMPAR_MEM_DEVICE && d->mem != COMPAR_MEM_HOST) return fail(COMPAR_E_INVALID, "bad mem");
    if (d->panels < 0 || d->panels > COMPAR_MAX_PANELS) return fail(COMPAR_E_INVALID, "panels out of range");
    if (d->world < COMPAR_WORLD_LOCAL || d->world > COMPAR_WORLD_TASKS) return fail(COMPAR_E_INVALID, "bad world");
    if (d->world && d->panels > 1) return fail(COMPAR_E_INVALID, "world and loopback panels are exclusive");
    if (d->world == COMPAR_WORLD_TASKS && d->mem != COMPAR_MEM_DEVICE)
        return fail(COMPAR_E_INVALID, "the task-parallel world takes device buffers");
    // world = 1 without compar_comm_init is a 1-rank world (plain launch, or the loopback pipeline)
    if (d->variant_hint < -1 || d->variant_hint >= static_cast<int>(c->variants.size()))
        return fail(COMPAR_E_INVALID, "variant_hint out of range");
    if (d->m == 0 || d->n == 0) return COMPAR_OK;
    if (d->k > 0 && d->alpha != 0.f) {
        if (!c->virt && (!d->A || (!d->B && !(d->world == COMPAR_WORLD_PANELS && c->rank != 0))))
            return fail(COMPAR_E_INVALID, "A/B NULL");
        if (d->lda < d->k) return fail(COMPAR_E_INVALID, "lda < k");
        if (d->ldb < (d->transB ? d->k : d->n)) return fail(COMPAR_E_INVALID, "ldb too small");
    }
    if (d->beta != 0.f) {
        if (!c->virt && !d->C_in) return fail(COMPAR_E_INVALID, "C_in NULL with beta != 0");
        if (d->ldc_in < d->n) return fail(COMPAR_E_INVALID, "ldc_in < n");
    }
    if (!c->virt && !d->C_out) return fail(COMPAR_E_INVALID, "C_out NULL");
    if (d->ldc_out < d->n) return fail(COMPAR_E_INVALID, "ldc_out < n");
    return COMPAR_OK;
}

// ---------------------------------------------------------------- eligibility (step 1)
bool admits(compar_target t, compar_dtype dt, compar_compute cp) {
    switch (t) {
        case COMPAR_TGT_USER: return true;
        case COMPAR_TGT_SIMT_F32:
        case COMPAR_TGT_TMA_F32: return dt == COMPAR_F32 && cp != COMPAR_COMPUTE_BF16;
        case COMPAR_TGT_TC_TF32:
        case COMPAR_TGT_TC2_TF32:
        case COMPAR_TGT_TCW_TF32:
        case COMPAR_TGT_TCS_TF32:
        case COMPAR_TGT_TCK_TF32: return dt == COMPAR_F32 && cp == COMPAR_COMPUTE_TF32;
        case COMPAR_TGT_TCX_F32: return dt == COMPAR_F32 && cp == COMPAR_COMPUTE_F32_SPLIT;
        case COMPAR_TGT_TC_BF16:
        case COMPAR_TGT_TC2_BF16:
        case COMPAR_TGT_TCW_BF16:
        case COMPAR_TGT_TCS_BF16:
        case COMPAR_TGT_TCK_BF16:
        case COMPAR_TGT_SIMT_BF16: return dt == COMPAR_BF16 && cp == COMPAR_COMPUTE_BF16;
        case COMPAR_TGT_SORT_RADIX:
        case COMPAR_TGT_SORT_BITONIC: return false;   // the sort interface's variants
    }
    return false;
}

struct Plan {
    Key key{};
    std::vector<compar_panel> panels;
    bool host_staged = false;
};

// Pointers the kernels will read (device or staging) decide TMA eligibility.
bool constraints_ok(const Ctx *c, compar_target t, const compar_gemm_desc *d, const Plan &plan) {
    if (t == COMPAR_TGT_USER) return true;
    const int64_t mrows = plan.key.m;
    const bool simt = t == COMPAR_TGT_SIMT_F32 || t == COMPAR_TGT_SIMT_BF16;
    if ((simt || t == COMPAR_TGT_TMA_F32) && (mrows + 127) / 128 > 65535) return false;
    if (simt) return true;
    const int eb = (t == COMPAR_TGT_TC_BF16 || t == COMPAR_TGT_TC2_BF16 || t == COMPAR_TGT_TCW_BF16 ||
                    t == COMPAR_TGT_TCS_BF16 || t == COMPAR_TGT_TCK_BF16) ? 2 : 4;
    if ((t == COMPAR_TGT_TCS_TF32 || t == COMPAR_TGT_TCS_BF16) &&
        tc_splitk_splits(mrows, d->n, d->k, t == COMPAR_TGT_TCS_BF16) < 2)
        return false;
    if ((t == COMPAR_TGT_TCK_TF32 || t == COMPAR_TGT_TCK_BF16) && !tc_clusterk_ok(mrows, d->n, d->k, t == COMPAR_TGT_TCK_BF16, c->num_sms))
        return false;
    // FP32-accuracy split form (R38): the per-product split error is below the FP32 bound's c*K*u
    // from K >= 64; its workspace holds the launch's operands whole, so not for host-memory tasks
    // (whose row chunks would re-split B every chunk), and at most 32 GiB.  Row-panel (world) tasks
    // launch it once per B slab: each launch re-splits the rank's A panel (HBM-bound, small beside
    // the slab's GEMM) and the slab
    if (t == COMPAR_TGT_TCX_F32 &&
        (d->k < tc_f32x3_min_k || d->mem == COMPAR_MEM_HOST ||
         tc_f32x3_workspace_bytes(mrows, d->n, d->k, d->transB) > (size_t(32) << 30)))
        return false;
    if (d->m > INT32_MAX || d->n > INT32_MAX || d->k > INT32_MAX) return false;
    if ((d->lda * eb) % 16 != 0 || (d->ldb * eb) % 16 != 0) return false;
    // the wide variant moves C with TMA; the split-K variant's final reduction uses 16-byte C accesses
    const bool tma_c = t == COMPAR_TGT_TCW_TF32 || t == COMPAR_TGT_TCW_BF16 || t == COMPAR_TGT_TCS_TF32 ||
                       t == COMPAR_TGT_TCS_BF16;
    if (tma_c && ((d->ldc_out * 4) % 16 != 0 || (d->beta != 0.f && (d->ldc_in * 4) % 16 != 0))) return false;
    if (c->virt) return true;
    for (const auto &p : plan.panels) {
        if (reinterpret_cast<uintptr_t>(p.A) % 16 != 0) return false;
        if (p.B && reinterpret_cast<uintptr_t>(p.B) % 16 != 0) return false;
        if (tma_c && reinterpret_cast<uintptr_t>(p.C_out) % 16 != 0) return false;
        if (tma_c && d->beta != 0.f && reinterpret_cast<uintptr_t>(p.C_in) % 16 != 0) return false;
    }
    return true;
}

void eligible_set(Ctx *c, const compar_gemm_desc *d, const Plan &plan, std::vector<int> &idx,
                  std::vector<int> &hids) {
    idx.clear();
    hids.clear();
    for (size_t v = 0; v < c->variants.size(); ++v) {
        if (v < 63 && (c->cfg.variant_mask >> v) & 1) continue;
        const Variant &var = c->variants[v];
        if (var.iface != kGemm) continue;
        if (!admits(var.target, d->in_dtype, d->compute)) continue;
        if (!constraints_ok(c, var.target, d, plan)) continue;
        idx.push_back(static_cast<int>(v));
        hids.push_back(var.hid);
    }
}

// ---------------------------------------------------------------- staging (host-mode buffers)
compar_status ensure_buffer(void **buf, size_t *have, size_t need) {
    if (need <= *have && *buf) return COMPAR_OK;
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    *have = 0;
    if (need == 0) return COMPAR_OK;
    cudaError_t e = cudaMalloc(buf, need);
    if (e != cudaSuccess) return fail(COMPAR_E_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    *have = need;
    return COMPAR_OK;
}

compar_status build_plan(Ctx *c, const compar_gemm_desc *d, Plan &plan, const void *A, const void *B,
                         const float *Cin, float *Cout) {
    const int eb = elem_bytes(d->in_dtype);
    plan.panels.clear();
    std::vector<int64_t> offs;
    if (d->world == COMPAR_WORLD_PANELS) {
        partition(d->m, c->nranks, offs);
        compar_panel p{};
        p.index = c->rank;
        p.row0 = offs[c->rank];
        p.rows = offs[c->rank + 1] - offs[c->rank];
        p.A = A;
        p.B = B;
        p.C_in = Cin;
        p.C_out = Cout;
        if (p.rows > 0) plan.panels.push_back(p);
        plan.key.m = offs[1] - offs[0];
    } else {
        const int P = d->panels > 1 ? d->panels : 1;
        partition(d->m, P, offs);
        for (int r = 0; r < P; ++r) {
            compar_panel p{};
            p.index = r;
            p.row0 = offs[r];
            p.rows = offs[r + 1] - offs[r];
            if (p.rows == 0) continue;
            p.A = A ? static_cast<const char *>(A) + static_cast<size_t>(p.row0) * d->lda * eb : nullptr;
            p.B = B;
            p.C_in = Cin ? Cin + p.row0 * d->ldc_in : nullptr;
            p.C_out = Cout ? Cout + p.row0 * d->ldc_out : nullptr;
            plan.panels.push_back(p);
        }
        plan.key.m = offs[1] - offs[0];
    }
    plan.key.n = d->n;
    plan.key.k = d->k;
    plan.key.dtype = d->in_dtype;
    plan.key.compute = d->compute;
    plan.key.transB = d->transB;
    plan.key.beta0 = d->beta == 0.f ? 1 : 0;
    return COMPAR_OK;
}

// ---------------------------------------------------------------- bounded waits (NCCL robustness)
// Marks the context's cross-rank path failed: the communicator is aborted (its pending
// collectives end) and every later task that needs a collective fails with E_NCCL.
void make_sticky(Ctx *c, const std::string &msg) {
    if (c->sticky == COMPAR_OK) {
        c->sticky = COMPAR_E_NCCL;
        c->sticky_msg = msg;
    }
    if (c->comm) {
        ncclCommAbort(c->comm);
        c->comm = nullptr;
    }
}

// Waits for `ev`.  For work that involves other ranks (collective = true) the wait polls
// ncclCommGetAsyncError and the sync timeout instead of blocking in the driver: a rank that died,
// or a collective that errored, turns into E_NCCL here instead of a hang.
compar_status wait_event(Ctx *c, cudaEvent_t ev, bool collective, cudaError_t *cuda_err) {
    *cuda_err = cudaSuccess;
    if (!ev) return COMPAR_OK;
    if (!collective || (!c->comm && !c->ce)) {
        *cuda_err = cudaEventSynchronize(ev);
        return COMPAR_OK;
    }
    if (c->sticky != COMPAR_OK) return fail(c->sticky, c->sticky_msg);
    const auto t0 = std::chrono::steady_clock::now();
    for (int spins = 0;; ++spins) {
        const cudaError_t e = cudaEventQuery(ev);
        if (e != cudaErrorNotReady) {
            *cuda_err = e;
            return COMPAR_OK;
        }
        ncclResult_t ar = ncclSuccess;
        if (c->comm) ncclCommGetAsyncError(c->comm, &ar);
        const int64_t ms = std::chrono::duration_cast<std::chrono::milliseconds>(
                               std::chrono::steady_clock::now() - t0).count();
        if (ar != ncclSuccess && ar != ncclInProgress) {
            make_sticky(c, std::string("NCCL asynchronous error: ") + ncclGetErrorString(ar));
            return fail(COMPAR_E_NCCL, c->sticky_msg);
        }
        if (c->sync_timeout_ms > 0 && ms > c->sync_timeout_ms) {
            make_sticky(c, "cross-rank wait timed out after " + std::to_string(ms) + " ms (sync_timeout_ms)");
            return fail(COMPAR_E_NCCL, c->sticky_msg);
        }
        if (spins < 256)
            std::this_thread::yield();
        else
            std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

// ---------------------------------------------------------------- harvest
compar_status finish_task(Ctx *c, Task &t, compar_report *rep);

// Waits for a local task and returns its history sample: max over panels of the kernel span
// (batched calibration: span / r; host pipeline: sum of the chunk kernels).
int64_t measure(Ctx *c, Task &t, compar_report *rep) {
    int64_t sample = 0;
    cudaEvent_t last = t.end ? t.end : (t.panels.empty() ? nullptr : t.panels.back().stop);
    if (!c->virt && last) {
        cudaError_t e = cudaSuccess;
        const compar_status ws = wait_event(c, last, (t.world || t.tasks) && c->nranks > 1, &e);
        if (ws != COMPAR_OK && t.status == COMPAR_OK) {
            t.status = ws;
            return 0;
        }
        if (e != cudaSuccess && t.status == COMPAR_OK) {
            t.status = COMPAR_E_TASK_FAILED;
            t_err = std::string("task execution failed: ") + cudaGetErrorString(e);
        }
    }
    for (size_t i = 0; i < t.panels.size(); ++i) {
        int64_t ns = 0;
        if (c->virt) {
            ns = t.panels[i].virtual_ns;
        } else if (!t.panels[i].sub.empty() && t.panels[i].batch > 1) {  // batched calibration: median launch
            std::vector<int64_t> v;
            for (auto &s : t.panels[i].sub) v.push_back(elapsed_ns(s.first, s.second));
            std::nth_element(v.begin(), v.begin() + v.size() / 2, v.end());
            ns = v[v.size() / 2];
            if (rep) rep->batch = std::max(rep->batch, t.panels[i].batch);
        } else if (!t.panels[i].sub.empty()) {  // host pipeline: sum of the chunk kernels
            for (auto &s : t.panels[i].sub) ns += elapsed_ns(s.first, s.second);
        } else if (t.panels[i].start) {
            const int64_t r = t.panels[i].batch;
            ns = (elapsed_ns(t.panels[i].start, t.panels[i].stop) + r / 2) / r;
            if (rep) rep->batch = std::max(rep->batch, t.panels[i].batch);
        }
        if (rep && i < COMPAR_MAX_PANELS) rep->panel_ns[i] = ns;
        sample = std::max(sample, ns);
    }
    return sample;
}

// Task-parallel world, several ranks: the owner of each task contributes its sample, the others
// -1, and an element-wise max over the ranks gives every rank the same samples (so the replicated
// history and placer stay identical).  Collective: every rank calls it with the same task list.
compar_status exchange_samples(Ctx *c, const std::vector<Task *> &ts) {
    if (ts.empty()) return COMPAR_OK;
    std::vector<int64_t> buf(ts.size(), -1);
    for (size_t i = 0; i < ts.size(); ++i) {
        Task &t = *ts[i];
        if (t.remote) continue;
        const int64_t ns = measure(c, t, nullptr);
        buf[i] = t.status == COMPAR_OK ? ns : -2;
    }
    if (c->nranks > 1) {
        const int n = static_cast<int>(buf.size());
        if (c->reduce_n_hook) {
            c->reduce_n_hook(buf.data(), n, c->reduce_n_user);
        } else if (c->comm) {
            if (c->xbuf_n < buf.size()) {
                if (c->xbuf) cudaFree(c->xbuf);
                c->xbuf = nullptr;
                c->xbuf_n = 0;
                if (cudaMalloc(&c->xbuf, buf.size() * sizeof(int64_t)) != cudaSuccess)
                    return fail(COMPAR_E_OOM, "sample exchange buffer");
                c->xbuf_n = buf.size();
            }
            cudaMemcpyAsync(c->xbuf, buf.data(), buf.size() * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream);
            const ncclResult_t r = ncclAllReduce(c->xbuf, c->xbuf, buf.size(), ncclInt64, ncclMax, c->comm, c->stream);
            cudaMemcpyAsync(buf.data(), c->xbuf, buf.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream);
            if (r != ncclSuccess) {
                make_sticky(c, std::string("sample exchange: ") + ncclGetErrorString(r));
                return fail(COMPAR_E_NCCL, c->sticky_msg);
            }
            cudaEvent_t ev = get_event(c);
            cudaEventRecord(ev, c->stream);
            cudaError_t ce = cudaSuccess;
            const compar_status ws = wait_event(c, ev, true, &ce);
            put_event(c, ev);
            if (ws != COMPAR_OK) return ws;
        } else {
            return fail(COMPAR_E_STATE, "task-parallel world over several ranks needs a communicator or a reduce hook");
        }
    }
    for (size_t i = 0; i < ts.size(); ++i) {
        ts[i]->xns = buf[i];
        ts[i]->have_xns = true;
    }
    return COMPAR_OK;
}

// The task-parallel tasks among `ids` whose samples have not been exchanged yet (id order).
compar_status exchange_ids(Ctx *c, const std::vector<uint64_t> &ids) {
    if (c->nranks <= 1) return COMPAR_OK;
    std::vector<Task *> xs;
    for (uint64_t id : ids) {
        auto it = c->tasks.find(id);
        if (it != c->tasks.end() && it->second.tasks && !it->second.have_xns) xs.push_back(&it->second);
    }
    return exchange_samples(c, xs);
}

// A task whose harvest is a collective (NCCL sample all-reduce or exchange across ranks): only
// harvested where every rank harvests it (submit / sync), never from compar_select.
bool collective_harvest(const Ctx *c, const Task &t) {
    return c->nranks > 1 && (t.world || t.tasks);
}

// Implicit harvest (step 6): the task's report is kept in `done` until compar_sync returns it.
compar_status harvest_ids(Ctx *c, const std::vector<uint64_t> &ids) {
    Range r("compar.harvest");
    compar_status s = exchange_ids(c, ids);
    if (s != COMPAR_OK) return s;
    for (uint64_t id : ids) {
        auto it = c->tasks.find(id);
        compar_report rep;
        const compar_status st = finish_task(c, it->second, &rep);
        c->done[id] = {st, rep};
        c->tasks.erase(it);
    }
    return COMPAR_OK;
}

// Step 6: before a decision, every pending execution of this key is harvested in task-id order
// (std::map iterates in id order).
compar_status harvest_key(Ctx *c, const Key &k) {
    std::vector<uint64_t> ids;
    for (auto &kv : c->tasks)
        if (kv.second.history && kv.second.key == k && !(c->in_select && collective_harvest(c, kv.second)))
            ids.push_back(kv.first);
    return harvest_ids(c, ids);
}

compar_status harvest_all(Ctx *c) {
    std::vector<uint64_t> ids;
    for (auto &kv : c->tasks)
        if (kv.second.history && !(c->in_select && collective_harvest(c, kv.second))) ids.push_back(kv.first);
    return harvest_ids(c, ids);
}

compar_status finish_task(Ctx *c, Task &t, compar_report *rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->task = t.id;
    rep->variant = t.variant;
    rep->mode = t.mode;
    rep->warmup = t.warm ? 1 : 0;
    rep->npanels = static_cast<int>(t.panels.size());
    rep->rank = t.tasks ? t.owner : c->rank;
    rep->lane = t.lane;
    int64_t sample = measure(c, t, rep);
    if (t.tasks && t.have_xns) {  // task-parallel world: the owner's sample, identical on all ranks
        if (t.xns == -2 && t.status == COMPAR_OK) {
            t.status = COMPAR_E_TASK_FAILED;
            t_err = "task failed on its owner rank";
        }
        sample = t.xns > 0 ? t.xns : 0;
        rep->panel_ns[0] = sample;
    } else if (t.tasks && t.remote) {
        t.status = COMPAR_E_STATE;
        t_err = "remote task synced without the collective sample exchange";
    }
    if (!c->virt && !t.remote) {
        rep->total_ns = t.begin ? elapsed_ns(t.begin, t.end)
                                : (t.panels.empty() ? 0 : elapsed_ns(t.panels.front().start, t.panels.back().stop));
        rep->bcast_ns = elapsed_ns(t.bc0, t.bc1);
    } else {
        for (auto &p : t.panels) rep->total_ns += p.virtual_ns;
        if (t.remote) rep->total_ns = sample;
    }
    // SPMD: every rank harvests the same task sequence; the sample is the max over ranks so
    // all ranks keep an identical history (rank-consistent decisions).
    if (t.world && c->nranks > 1 && t.history && c->reduce_hook) {
        c->reduce_hook(&sample, c->reduce_user);
    } else if (t.world && c->comm && (c->nranks > 1 || c->bcast_loopback) && t.history) {
        cudaMemcpyAsync(c->red_buf, &sample, sizeof(int64_t), cudaMemcpyHostToDevice, c->stream);
        ncclResult_t r = ncclAllReduce(c->red_buf, c->red_buf, 1, ncclInt64, ncclMax, c->comm, c->stream);
        cudaMemcpyAsync(&sample, c->red_buf, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream);
        if (r != ncclSuccess) {
            make_sticky(c, std::string("sample all-reduce: ") + ncclGetErrorString(r));
            if (t.status == COMPAR_OK) t.status = COMPAR_E_NCCL;
        } else {
            cudaEvent_t ev = get_event(c);
            cudaEventRecord(ev, c->stream);
            cudaError_t ce = cudaSuccess;
            const compar_status ws = wait_event(c, ev, true, &ce);
            put_event(c, ev);
            if (ws != COMPAR_OK && t.status == COMPAR_OK) t.status = ws;
        }
    }
    rep->ns = sample;
    rep->status = t.status;
    if (t.history && t.status == COMPAR_OK && !t.warm && t.variant >= 0) {
        c->hist.harvest(c->variants[t.variant].hid, t.key, sample);
        c->stats.harvested++;
    }
    if (t.history && t.status == COMPAR_OK && t.warm && t.variant >= 0)
        c->hist.rec(c->variants[t.variant].hid, t.key).warm_ns = std::max<int64_t>(sample, 1);
    if (rep->batch == 0) rep->batch = 1;
    if (t.status != COMPAR_OK) c->stats.failed++;
    release_task_events(c, t);
    if (t.status == COMPAR_OK) return COMPAR_OK;
    return t.status == COMPAR_E_NCCL ? COMPAR_E_NCCL : COMPAR_E_TASK_FAILED;
}

// ---------------------------------------------------------------- running a variant on a panel
compar_status run_builtin(Ctx *c, compar_target t, const compar_gemm_desc *d, const compar_panel &p,
                          cudaStream_t s, int sms = 0, const WorldLaunch *wl = nullptr) {
    GemmLaunch g;
    g.knobs = &c->knobs;
    g.world = wl;
    g.m = p.rows, g.n = d->n, g.k = d->k;
    g.alpha = d->alpha, g.beta = d->beta;
    g.A = p.A, g.lda = d->lda, g.B = p.B, g.ldb = d->ldb, g.transB = d->transB;
    g.C_in = p.C_in, g.ldc_in = d->ldc_in, g.C_out = p.C_out, g.ldc_out = d->ldc_out;
    g.stream = s;
    g.num_sms = sms > 0 ? sms : c->num_sms;
    cudaError_t e;
    switch (t) {
        case COMPAR_TGT_SIMT_F32: e = launch_simt_f32(g); break;
        case COMPAR_TGT_TMA_F32: e = launch_tma_f32(g); break;
        case COMPAR_TGT_TC_TF32: e = launch_tc_gemm(g, false); break;
        case COMPAR_TGT_TC_BF16: e = launch_tc_gemm(g, true); break;
        case COMPAR_TGT_TC2_TF32: e = launch_tc_gemm_2sm(g, false); break;
        case COMPAR_TGT_TC2_BF16: e = launch_tc_gemm_2sm(g, true); break;
        case COMPAR_TGT_TCW_TF32: e = launch_tc_gemm_2sm_wide(g, false); break;
        case COMPAR_TGT_TCW_BF16: e = launch_tc_gemm_2sm_wide(g, true); break;
        case COMPAR_TGT_TCS_TF32: e = launch_tc_gemm_splitk(g, false); break;
        case COMPAR_TGT_TCS_BF16: e = launch_tc_gemm_splitk(g, true); break;
        case COMPAR_TGT_TCK_TF32: e = launch_tc_gemm_ck(g, false); break;
        case COMPAR_TGT_TCK_BF16: e = launch_tc_gemm_ck(g, true); break;
        case COMPAR_TGT_TCX_F32: e = launch_tc_gemm_f32x3(g); break;
        case COMPAR_TGT_SIMT_BF16: e = launch_simt_bf16(g); break;
        default: return fail(COMPAR_E_INVALID, "not a built-in target");
    }
    c->stats.launches++;
    if (e != cudaSuccess) return fail(COMPAR_E_TASK_FAILED, std::string("launch: ") + cudaGetErrorString(e));
    return COMPAR_OK;
}

compar_status run_scale(Ctx *c, const compar_gemm_desc *d, const compar_panel &p, cudaStream_t s) {
    GemmLaunch g{};
    g.m = p.rows, g.n = d->n, g.beta = d->beta;
    g.C_in = p.C_in, g.ldc_in = d->ldc_in, g.C_out = p.C_out, g.ldc_out = d->ldc_out;
    g.stream = s;
    g.num_sms = c->num_sms;
    g.knobs = &c->knobs;
    cudaError_t e = launch_scale(g);
    c->stats.launches++;
    if (e != cudaSuccess) return fail(COMPAR_E_TASK_FAILED, std::string("scale: ") + cudaGetErrorString(e));
    return COMPAR_OK;
}

// ---------------------------------------------------------------- world mode: B broadcast + panel GEMM
// SURVEY §8(a) a5 / §8(e); DESIGN.md §6.  B (on rank 0) is packed into contiguous N-slabs by the
// copy engine (row-major B: slab j is a K x w_j row-major block; transB: rows of B^T, pitch K) and
// each slab is broadcast (ncclBroadcast on the library's comm stream, or the copy-engine chain).
// A receiver consumes slab j as soon as it landed:
//   * fused (wide-pair variant, uniform slabs of a multiple of 512 columns dividing N): ONE
//     persistent launch whose producers wait per tile on the slab's flag word (written on the comm
//     stream after the slab landed) and visit the tiles column-major;
//   * otherwise one launch per slab after the slab's event (geometric widths: a small first slab,
//     then doubling, so the exposed first-slab latency is short and the launches few).
// Every C element still sums its full K in order, so C is bitwise the single-GPU result.  The root
// multiplies with its own B.  GEMMs that overlap an NCCL broadcast leave bcast_reserve_sms SMs to
// NCCL's kernels (the communicator is capped at bcast_ctas CTAs); the wide variant gets them back
// through a helper launch after the broadcast ends.

constexpr int kMaxSlabs = 64;

// Slab plan of a world task.
struct SlabPlan {
    std::vector<int64_t> col0;   // slab j = columns [col0[j], col0[j+1]) of B (size nslab + 1)
    bool fused = false;          // uniform slabs read by one flag-waiting launch
    int64_t w = 0;               // fused: slab width
    int64_t pitch1 = 0;          // nslab == 1: packed row pitch (elements; >= width, TMA-aligned)
    int nslab() const { return static_cast<int>(col0.size()) - 1; }
};

// fused_ok: the variant is the wide pair kernel.  chunks: the non-fused slab count.
SlabPlan plan_slabs(int64_t N, int64_t K, int eb, bool transB, bool fused_ok, int chunks) {
    SlabPlan sp;
    const int64_t width = transB ? K : N;   // row width of a packed slab's rows (transB: B^T rows)
    if (fused_ok) {   // smallest multiple of 512 dividing N with at most kMaxSlabs slabs
        for (int64_t w = 512; w <= N; w += 512) {
            if (N % w == 0 && N / w <= kMaxSlabs && (transB || (w * eb) % 16 == 0)) {
                sp.fused = true;
                sp.w = w;
                for (int64_t c0 = 0; c0 <= N; c0 += w) sp.col0.push_back(c0);
                break;
            }
        }
        if (sp.fused && sp.nslab() >= 1 && (transB ? (K * eb) % 16 == 0 : true)) return sp;
        sp = SlabPlan{};
    }
    // geometric: boundaries at N / 2^(S-j), rounded up to 256 columns
    const int S = std::max(1, std::min(chunks, 16));
    sp.col0.push_back(0);
    for (int j = 1; j < S; ++j) {
        int64_t b = (N >> (S - j));
        b = (b + 255) / 256 * 256;
        if (b > sp.col0.back() && b < N) sp.col0.push_back(b);
    }
    sp.col0.push_back(N);
    // every packed slab pitch must be TMA-usable (16-byte rows); else a single padded slab
    bool ok = true;
    for (int j = 0; j < sp.nslab(); ++j) {
        const int64_t pitch = transB ? K : sp.col0[j + 1] - sp.col0[j];
        if ((pitch * eb) % 16 != 0) ok = false;
    }
    if (!ok) sp.col0 = {0, N};
    const int64_t unit = 16 / eb;
    sp.pitch1 = (width + unit - 1) / unit * unit;
    return sp;
}

// Bytes of the packed replica for a plan (all slabs; a single slab may carry row padding).
size_t packed_bytes(const SlabPlan &sp, int64_t N, int64_t K, int eb, bool transB) {
    if (sp.nslab() == 1) return static_cast<size_t>(transB ? N : K) * sp.pitch1 * eb;
    return static_cast<size_t>(K) * N * eb;
}

// Packed geometry of slab j: byte offset, rows, row pitch (elements).
struct SlabGeo {
    size_t off;
    int64_t rows, pitch, cols;
};
SlabGeo slab_geo(const SlabPlan &sp, int j, int64_t K, int eb, bool transB) {
    const int64_t c0 = sp.col0[j], wj = sp.col0[j + 1] - c0;
    if (sp.nslab() == 1)
        return {0, transB ? wj : K, sp.pitch1, transB ? K : wj};
    if (transB) return {static_cast<size_t>(c0) * K * eb, wj, K, K};
    return {static_cast<size_t>(K) * c0 * eb, K, wj, wj};
}

// Copy-engine pack of slab j from the caller's B (any ld) into `dst`.
void pack_slab(const SlabPlan &sp, int j, const compar_gemm_desc *d, const void *Bsrc, void *dst, int eb,
               cudaStream_t s) {
    const SlabGeo g = slab_geo(sp, j, d->k, eb, d->transB);
    const int64_t c0 = sp.col0[j];
    const char *src = static_cast<const char *>(Bsrc);
    char *out = static_cast<char *>(dst) + g.off;
    if (d->transB)   // rows [c0, c0 + w) of B^T
        cudaMemcpy2DAsync(out, g.pitch * eb, src + c0 * d->ldb * eb, d->ldb * eb, g.cols * eb, g.rows,
                          cudaMemcpyDeviceToDevice, s);
    else             // columns [c0, c0 + w) of every row of B
        cudaMemcpy2DAsync(out, g.pitch * eb, src + c0 * eb, d->ldb * eb, g.cols * eb, g.rows, cudaMemcpyDeviceToDevice,
                          s);
}

template <class F>
compar_status world_gemms(Ctx *c, const compar_gemm_desc *d, Task &t, cudaStream_t st, const void *replica,
                          const SlabPlan &sp, const std::vector<cudaEvent_t> &landed, const unsigned *flags,
                          unsigned seq, int reserve, F &&launch_on);

// ---------------------------------------------------------------- copy-engine chain broadcast
// Stream memory operations on IPC-mapped flag words (driver entry points; no SM involvement).
using PfnWaitValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using PfnWriteValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PfnWaitValue32 g_wait32 = nullptr;
PfnWriteValue32 g_write32 = nullptr;
bool resolve_stream_memops() {
    static std::once_flag once;
    std::call_once(once, [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_wait32 = reinterpret_cast<PfnWaitValue32>(fn);
        fn = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_write32 = reinterpret_cast<PfnWriteValue32>(fn);
    });
    return g_wait32 && g_write32;
}
constexpr int kCeMax = 64;                      // chunks per broadcast
inline CUdeviceptr dptr(const uint32_t *p) { return static_cast<CUdeviceptr>(reinterpret_cast<uintptr_t>(p)); }

// World task with the copy-engine chain: slab j travels root -> 1 -> ... -> P-1, each hop a
// cudaMemcpyAsync from the upstream rank's IPC-mapped buffer, started by a GPU-side wait on the
// upstream's ready[j] >= seq and followed by consumed[j] = seq in the upstream's flags (it may
// then overwrite slab j for the next broadcast) and ready[j] = seq in our own — which is also the
// slab flag the fused GEMM waits on.  Every rank runs the same broadcast sequence (SPMD), so seq
// agrees everywhere; nothing runs on the SMs.
template <class F>
compar_status ce_pipeline(Ctx *c, const compar_gemm_desc *d, Task &t, cudaStream_t st, const void *Bloc,
                          bool fused_ok, F &&launch_on) {
    const int eb = elem_bytes(d->in_dtype);
    const bool root = c->rank == 0;
    const bool has_down = c->rank + 1 < c->nranks;
    const int64_t K = d->k, N = d->n;
    // the last rank's first slab arrives after P - 1 hops: at least 4 slabs per hop
    const int chunks = std::min(16, std::max(c->cfg.bcast_chunks > 0 ? c->cfg.bcast_chunks : 1, 4 * (c->nranks - 1)));
    const SlabPlan sp = plan_slabs(N, K, eb, d->transB, fused_ok, chunks);
    const int nslab = sp.nslab();
    if (nslab > kCeMax) return fail(COMPAR_E_INVALID, "too many slabs");
    const size_t total = packed_bytes(sp, N, K, eb, d->transB);
    if (total > c->ce_cap) return fail(COMPAR_E_INVALID, "B larger than the copy-engine chain buffer (max_b_bytes)");
    const uint32_t seq = ++c->ce_seq;
    cudaStream_t cs = c->comm_stream;
    CUstream cus = reinterpret_cast<CUstream>(cs);
    t.bc0 = get_event(c);
    t.bc1 = get_event(c);
    cudaEvent_t ready = get_event(c);
    t.extra.push_back(ready);
    cudaEventRecord(ready, st);
    cudaStreamWaitEvent(cs, ready, 0);
    if (c->bcast_free_set) cudaStreamWaitEvent(cs, c->bcast_free, 0);
    cudaEventRecord(t.bc0, cs);
    std::vector<cudaEvent_t> landed;
    for (int j = 0; j < nslab; ++j) {
        const SlabGeo g = slab_geo(sp, j, K, eb, d->transB);
        const size_t bytes = static_cast<size_t>(g.rows) * g.pitch * eb;
        char *mine = static_cast<char *>(c->ce_buf) + g.off;
        if (has_down)  // the downstream rank has copied slab j of the previous broadcast out
            g_wait32(cus, dptr(c->ce_flags + kCeMax + j), seq - 1, CU_STREAM_WAIT_VALUE_GEQ);
        if (root) {
            pack_slab(sp, j, d, Bloc, c->ce_buf, eb, cs);
        } else {
            g_wait32(cus, dptr(c->ce_up_flags + j), seq, CU_STREAM_WAIT_VALUE_GEQ);
            cudaMemcpyAsync(mine, static_cast<const char *>(c->ce_up_buf) + g.off, bytes, cudaMemcpyDefault, cs);
            g_write32(cus, dptr(c->ce_up_flags + kCeMax + j), seq, CU_STREAM_WRITE_VALUE_DEFAULT);
        }
        g_write32(cus, dptr(c->ce_flags + j), seq, CU_STREAM_WRITE_VALUE_DEFAULT);
        cudaEvent_t ev = get_event(c);
        t.extra.push_back(ev);
        landed.push_back(ev);
        cudaEventRecord(ev, cs);
    }
    cudaEventRecord(t.bc1, cs);
    // no SMs to spare: the copy engines move B
    return world_gemms(c, d, t, st, c->ce_buf, sp, landed, c->ce_flags, seq, 0, launch_on);
}

template <class F>
compar_status world_pipeline(Ctx *c, const compar_gemm_desc *d, Task &t, cudaStream_t st, const void *Bloc,
                             bool fused_ok, F &&launch_on) {
    Range range("compar.bcast");
    if (c->ce && c->nranks > 1) return ce_pipeline(c, d, t, st, Bloc, fused_ok, launch_on);
    const int eb = elem_bytes(d->in_dtype);
    const bool loop = c->nranks == 1;              // loopback emulation on one GPU
    const bool root = !loop && c->rank == 0;
    const bool use_nccl = c->comm != nullptr;      // loopback with a 1-rank communicator still calls NCCL
    const int64_t K = d->k, N = d->n;
    const SlabPlan sp = plan_slabs(N, K, eb, d->transB, fused_ok, c->cfg.bcast_chunks > 0 ? c->cfg.bcast_chunks : 1);
    const int nslab = sp.nslab();
    if (nslab > kMaxSlabs) return fail(COMPAR_E_INVALID, "too many slabs");
    const size_t total = packed_bytes(sp, N, K, eb, d->transB);
    compar_status s;
    // buffers: the root (or loopback) packs into bpacked; receivers (or loopback) fill the replica —
    // the caller's B_replica when the packed layout fits its k * n elements, else the library's
    void *packed = nullptr;
    void *replica = nullptr;
    if (root || loop) {
        if ((s = ensure_buffer(&c->bpacked, &c->bpacked_bytes, total)) != COMPAR_OK) return s;
        packed = c->bpacked;
    }
    if (!root) {
        if (!loop && d->B_replica && total <= static_cast<size_t>(K) * N * eb) {
            replica = d->B_replica;
        } else {
            if ((s = ensure_buffer(&c->breplica, &c->breplica_bytes, total)) != COMPAR_OK) return s;
            replica = c->breplica;
        }
    }
    if (!c->slab_flags) {
        cudaError_t e = cudaMalloc(&c->slab_flags, kMaxSlabs * sizeof(uint32_t));
        if (e == cudaSuccess) e = cudaMemset(c->slab_flags, 0, kMaxSlabs * sizeof(uint32_t));
        if (e != cudaSuccess) return cuda_fail(e, "slab flags");
    }
    if (sp.fused && !resolve_stream_memops()) return fail(COMPAR_E_CUDA, "cuStreamWriteValue32 unavailable");
    const uint32_t seq = ++c->slab_seq;
    cudaStream_t cs = c->comm_stream;
    t.bc0 = get_event(c);
    t.bc1 = get_event(c);
    cudaEvent_t ready = get_event(c);
    t.extra.push_back(ready);
    cudaEventRecord(ready, st);                     // inputs of this task are ready
    cudaStreamWaitEvent(cs, ready, 0);
    if (c->bcast_free_set) cudaStreamWaitEvent(cs, c->bcast_free, 0);   // previous world task's GEMMs
    cudaEventRecord(t.bc0, cs);
    std::vector<cudaEvent_t> landed;
    ncclResult_t nr = ncclSuccess;
    for (int j = 0; j < nslab; ++j) {
        const SlabGeo g = slab_geo(sp, j, K, eb, d->transB);
        const size_t bytes = static_cast<size_t>(g.rows) * g.pitch * eb;
        char *pk = packed ? static_cast<char *>(packed) + g.off : nullptr;
        char *rp = replica ? static_cast<char *>(replica) + g.off : nullptr;
        if (root || loop) pack_slab(sp, j, d, Bloc, packed, eb, cs);
        if (loop && !use_nccl)
            cudaMemcpyAsync(rp, pk, bytes, cudaMemcpyDeviceToDevice, cs);
        else if (nr == ncclSuccess)
            nr = ncclBroadcast(pk, root ? pk : rp, bytes, ncclChar, 0, c->comm, cs);
        if (sp.fused && !root)
            g_write32(reinterpret_cast<CUstream>(cs), dptr(c->slab_flags + j), seq, CU_STREAM_WRITE_VALUE_DEFAULT);
        cudaEvent_t ev = get_event(c);
        t.extra.push_back(ev);
        landed.push_back(ev);
        cudaEventRecord(ev, cs);
    }
    cudaEventRecord(t.bc1, cs);
    if (nr != ncclSuccess) {
        make_sticky(c, std::string("ncclBroadcast: ") + ncclGetErrorString(nr));
        return fail(COMPAR_E_NCCL, c->sticky_msg);
    }
    return world_gemms(c, d, t, st, replica, sp, landed, c->slab_flags, seq,
                       (use_nccl && !loop) || c->bcast_loopback >= 2 ? c->bcast_reserve_sms : 0, launch_on);
}

// GEMMs of a world task (shared by the NCCL and copy-engine broadcasts).  The root multiplies with
// its own B; receivers read the replica (fused: one flag-waiting launch; else one launch per slab).
// reserve: SMs the broadcast's kernels need while it runs (0: copy engines only).
template <class F>
compar_status world_gemms(Ctx *c, const compar_gemm_desc *d, Task &t, cudaStream_t st, const void *replica,
                          const SlabPlan &sp, const std::vector<cudaEvent_t> &landed, const unsigned *flags,
                          unsigned seq, int reserve, F &&launch_on) {
    const int eb = elem_bytes(d->in_dtype);
    const bool root = c->nranks > 1 && c->rank == 0;
    const int64_t K = d->k;
    const int nslab = sp.nslab();
    // the wide kernel returns the reserved SMs through a helper launch once the broadcast is over
    WorldLaunch split;
    if (reserve >= 2) {
        split.helper_sms = reserve;
        split.helper_stream = c->aux_stream;
        split.helper_after = t.bc1;
        split.helper_done = get_event(c);
        t.extra.push_back(split.helper_done);
    }
    const int main_sms = reserve > 0 ? std::max(2, c->num_sms - reserve) : 0;
    for (auto &pr : t.panels) {
        pr.start = get_event(c);
        pr.stop = get_event(c);
        cudaEventRecord(pr.start, st);
        compar_status r = COMPAR_OK;
        if (root) {
            // the root already holds B: one launch (helper SMs join after the broadcast)
            r = launch_on(d, pr.p, main_sms, reserve >= 2 ? &split : nullptr);
        } else if (sp.fused) {
            WorldLaunch wl = split;
            wl.flags = flags;
            wl.seq = seq;
            wl.slab_w = static_cast<int>(sp.w);
            wl.nslab = nslab;
            compar_gemm_desc dd = *d;
            dd.ldb = d->transB ? K : sp.w;      // (row-major: the 3-D map's row pitch)
            compar_panel pp = pr.p;
            pp.B = replica;
            r = launch_on(&dd, pp, main_sms, &wl);
        } else {
            for (int j = 0; j < nslab && r == COMPAR_OK; ++j) {
                const SlabGeo g = slab_geo(sp, j, K, eb, d->transB);
                const int64_t col0 = sp.col0[j], wj = sp.col0[j + 1] - col0;
                cudaStreamWaitEvent(st, landed[j], 0);
                compar_gemm_desc dj = *d;
                dj.n = wj;
                dj.ldb = g.pitch;
                compar_panel pj = pr.p;
                pj.B = static_cast<const char *>(replica) + g.off;
                pj.C_in = pr.p.C_in ? pr.p.C_in + col0 : nullptr;
                pj.C_out = pr.p.C_out + col0;
                r = launch_on(&dj, pj, j + 1 < nslab ? main_sms : 0, nullptr);
            }
        }
        if (r != COMPAR_OK) t.status = COMPAR_E_TASK_FAILED;
        cudaEventRecord(pr.stop, st);
    }
    cudaStreamWaitEvent(st, t.bc1, 0);              // the task ends after its broadcast (B reusable)
    cudaEventRecord(c->bcast_free, st);             // the next world task may overwrite the slabs
    c->bcast_free_set = true;
    return COMPAR_OK;
}

// ---------------------------------------------------------------- host-memory tasks: copy/compute overlap
// mem = HOST (the end-to-end path): B goes up first, then A and C_in row chunks stream host->device
// on one copy engine while the GEMM runs on the previous chunk and finished C chunks stream back on
// the other copy engine.  Every C element is computed by exactly one chunk launch over its full K,
// so the result equals the unchunked call bitwise.  The history sample is the sum of the chunk
// kernel times.
template <class F>
compar_status host_pipeline(Ctx *c, const compar_gemm_desc *d, Task &t, cudaStream_t st, const void *A,
                            const void *B, const float *Cin, float *Cout, size_t b_bytes, F &&launch_on) {
    const int eb = elem_bytes(d->in_dtype);
    const int64_t M = d->m, K = d->k, N = d->n;
    const int64_t per = (M + c->host_chunks - 1) / c->host_chunks;
    const int64_t rows = std::max<int64_t>(256, (per + 255) / 256 * 256);
    // chunk boundaries: uniform chunks of `rows`, the last one cut into halving pieces (>= 256 rows)
    // so the exposed tail — the last chunk's GEMM and its copy back — is a fraction of a chunk
    std::vector<int64_t> bounds{0};
    while (bounds.back() < M) {
        const int64_t left = M - bounds.back();
        int64_t step = std::min(rows, left);
        if (left <= rows && c->host_tail_split) step = std::max<int64_t>(256, (left / 2 + 255) / 256 * 256);
        bounds.push_back(std::min(M, bounds.back() + step));
    }
    const int nchunk = static_cast<int>(bounds.size()) - 1;
    // the host C buffer's device alias when it is mapped pinned memory (else nullptr: copy engine)
    float *cout_host_dev = nullptr;
    {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, d->C_out) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer)
            cout_host_dev = static_cast<float *>(pa.devicePointer);
        else
            cudaGetLastError();   // (clear a lookup error on pageable memory)
    }
    cudaEvent_t ready = get_event(c);
    t.extra.push_back(ready);
    cudaEventRecord(ready, st);
    cudaStreamWaitEvent(c->h2d_stream, ready, 0);
    cudaStreamWaitEvent(c->d2h_stream, ready, 0);
    cudaMemcpyAsync(const_cast<void *>(B), d->B, b_bytes, cudaMemcpyHostToDevice, c->h2d_stream);
    c->stats.bytes_h2d += static_cast<int64_t>(b_bytes);
    PanelRun &pr = t.panels[0];
    pr.start = get_event(c);
    pr.stop = get_event(c);
    cudaEventRecord(pr.start, st);
    compar_status r = COMPAR_OK;
    for (int i = 0; i < nchunk && r == COMPAR_OK; ++i) {
        const int64_t r0 = bounds[i], ri = bounds[i + 1] - bounds[i];
        const size_t a_off = static_cast<size_t>(r0) * d->lda * eb;
        const size_t a_len = static_cast<size_t>(ri - 1) * d->lda * eb + static_cast<size_t>(K) * eb;
        cudaMemcpyAsync(static_cast<char *>(const_cast<void *>(A)) + a_off, static_cast<const char *>(d->A) + a_off,
                        a_len, cudaMemcpyHostToDevice, c->h2d_stream);
        c->stats.bytes_h2d += static_cast<int64_t>(a_len);
        if (d->beta != 0.f) {
            const size_t c_len = static_cast<size_t>(ri - 1) * d->ldc_in * 4 + static_cast<size_t>(N) * 4;
            cudaMemcpyAsync(const_cast<float *>(Cin) + r0 * d->ldc_in, d->C_in + r0 * d->ldc_in, c_len,
                            cudaMemcpyHostToDevice, c->h2d_stream);
            c->stats.bytes_h2d += static_cast<int64_t>(c_len);
        }
        cudaEvent_t in = get_event(c);
        t.extra.push_back(in);
        cudaEventRecord(in, c->h2d_stream);
        cudaStreamWaitEvent(st, in, 0);
        compar_panel pc = pr.p;
        pc.row0 = r0;
        pc.rows = ri;
        pc.A = static_cast<const char *>(A) + a_off;
        pc.C_in = Cin ? Cin + r0 * d->ldc_in : nullptr;
        pc.C_out = Cout + r0 * d->ldc_out;
        std::pair<cudaEvent_t, cudaEvent_t> span{get_event(c), get_event(c)};
        cudaEventRecord(span.first, st);
        r = launch_on(d, pc, 0);
        cudaEventRecord(span.second, st);
        pr.sub.push_back(span);
        cudaStreamWaitEvent(c->d2h_stream, span.second, 0);
        // 2-D copy: only the n valid columns of each row go back (the ld gap on the host is untouched).
        // Into mapped pinned memory the copy is a kernel of a few CTAs: a copy engine runs D2H at
        // full rate and takes the H2D direction down to ~52 GB/s while it does; a 4-CTA kernel moves
        // ~47 GB/s and leaves H2D ~53.4 (tools/pcie_mix.cu) — H2D is this pipeline's bound
        if (cout_host_dev && c->d2h_kernel_ctas > 0) {
            const compar_status ks = launch_rows_to_host(cout_host_dev + r0 * d->ldc_out, d->ldc_out, Cout + r0 * d->ldc_out,
                                                         d->ldc_out, ri, N, c->d2h_kernel_ctas, c->d2h_stream) == cudaSuccess
                                         ? COMPAR_OK : COMPAR_E_TASK_FAILED;
            if (ks != COMPAR_OK) r = ks;
        } else {
            cudaMemcpy2DAsync(d->C_out + r0 * d->ldc_out, d->ldc_out * 4, Cout + r0 * d->ldc_out, d->ldc_out * 4, N * 4,
                              ri, cudaMemcpyDeviceToHost, c->d2h_stream);
        }
        c->stats.bytes_d2h += static_cast<int64_t>(ri * N * 4);
    }
    cudaEventRecord(pr.stop, st);
    cudaEvent_t out = get_event(c);
    t.extra.push_back(out);
    cudaEventRecord(out, c->d2h_stream);
    cudaStreamWaitEvent(st, out, 0);                // the task ends when C is back on the host
    if (r != COMPAR_OK) return COMPAR_E_TASK_FAILED;
    return COMPAR_OK;
}

}  // namespace
}  // namespace compar

using namespace compar;

extern "C" {

void compar_config_default(compar_config *cfg) {
    if (!cfg) return;
    cfg->ngpu = -1;
    cfg->device = -1;
    cfg->sched = -1;
    cfg->calib_k = -1;
    cfg->calib_warmup = -1;
    cfg->perf_model_path = nullptr;
    cfg->bcast_chunks = -1;
    cfg->builtins = -1;
    cfg->virtual_clock = 0;
    cfg->variant_mask = -1;
    cfg->calib_order = -1;
    cfg->lanes = -1;
    cfg->calib_prune = -1;
    cfg->bcast_ctas = -1;
    cfg->sync_timeout_ms = -1;
}

const char *compar_last_error(void *) { return t_err.c_str(); }

compar_status compar_register_variant(void *ctx, const char *iface, const char *name, compar_target target,
                                      compar_gemm_fn fn, void *user, int *out_id);

compar_status compar_init(const compar_config *cfg_in, void **ctx) {
    if (!ctx) return fail(COMPAR_E_INVALID, "ctx out-pointer is NULL");
    if (*ctx && as_ctx(*ctx)) return fail(COMPAR_E_STATE, "context already initialised");
    compar_config cfg;
    compar_config_default(&cfg);
    if (cfg_in) cfg = *cfg_in;
    if (cfg.ngpu < 0) cfg.ngpu = env_int("COMPAR_NGPU", 1);
    if (cfg.ngpu == 0) return fail(COMPAR_E_INVALID, "COMPAR_NGPU=0: no GPU class and no CPU fallback");
    if (cfg.ngpu != 1) return fail(COMPAR_E_INVALID, "one GPU per process (use compar_comm_init for SPMD)");
    if (cfg.sched < 0) {
        const char *s = std::getenv("COMPAR_SCHED");
        cfg.sched = (s && std::strcmp(s, "eager") == 0) ? 1 : (s && std::strcmp(s, "predict") == 0) ? 2 : 0;
    }
    if (cfg.calib_k < 0) cfg.calib_k = env_int("COMPAR_CALIB_K", 3);
    if (cfg.calib_warmup < 0) cfg.calib_warmup = env_int("COMPAR_CALIB_WARMUP", 1);
    if (cfg.bcast_chunks < 0) cfg.bcast_chunks = env_int("COMPAR_BCAST_CHUNKS", 8);
    if (cfg.calib_order < 0) {  // (batch threshold read below)
        const char *s = std::getenv("COMPAR_CALIB_ORDER");
        cfg.calib_order = (s && std::strcmp(s, "interleaved") == 0) ? COMPAR_CALIB_INTERLEAVED : COMPAR_CALIB_BLOCKED;
    }
    if (cfg.lanes < 1) cfg.lanes = env_int("COMPAR_LANES", 1);
    if (cfg.lanes < 1 || cfg.lanes > 16) return fail(COMPAR_E_INVALID, "lanes must be in 1..16");
    if (cfg.calib_order != COMPAR_CALIB_INTERLEAVED && cfg.calib_order != COMPAR_CALIB_BLOCKED)
        return fail(COMPAR_E_INVALID, "calib_order must be INTERLEAVED (0) or BLOCKED (1)");
    if (cfg.builtins < 0) cfg.builtins = 1;
    if (cfg.calib_prune < 0) cfg.calib_prune = env_int("COMPAR_CALIB_PRUNE", 150);
    if (cfg.calib_prune != 0 && cfg.calib_prune < 100)
        return fail(COMPAR_E_INVALID, "calib_prune must be 0 (off) or >= 100 (percent of the best mean)");
    if (cfg.bcast_ctas < 0) cfg.bcast_ctas = env_int("COMPAR_BCAST_CTAS", 4);
    if (cfg.bcast_ctas < 1 || cfg.bcast_ctas > 64) return fail(COMPAR_E_INVALID, "bcast_ctas must be in 1..64");
    if (cfg.sync_timeout_ms < 0) cfg.sync_timeout_ms = env_int("COMPAR_SYNC_TIMEOUT_MS", 600000);
    if (cfg.variant_mask < 0) {
        const char *s = std::getenv("COMPAR_VARIANT_MASK");
        cfg.variant_mask = s ? std::strtoll(s, nullptr, 0) : 0;
    }
    auto *c = new Ctx();
    c->cfg = cfg;
    c->virt = cfg.virtual_clock != 0;
    c->hist.calib_k = cfg.calib_k;
    c->hist.calib_warmup = cfg.calib_warmup;
    c->hist.calib_blocked = cfg.calib_order == COMPAR_CALIB_BLOCKED;
    c->hist.prune_pct = cfg.calib_prune;
    c->sync_timeout_ms = cfg.sync_timeout_ms;
    c->knobs = read_knobs();
    c->batch_below_ns = env_int("COMPAR_CALIB_BATCH_NS", 100000);
    const char *pp = cfg.perf_model_path ? cfg.perf_model_path : std::getenv("COMPAR_PERF_MODEL");
    if (pp) c->perf_path = pp;
    c->cfg.perf_model_path = nullptr;
    if (!c->virt) {
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess || n == 0) {
            delete c;
            return fail(COMPAR_E_CUDA, "no CUDA device (the library has no CPU fallback)");
        }
        if (cfg.device >= 0) {
            if (cfg.device >= n || (e = cudaSetDevice(cfg.device)) != cudaSuccess) {
                delete c;
                return fail(COMPAR_E_CUDA, "cannot select device");
            }
        }
        // every CUDA call of the set-up is checked; a failure releases what was created
        auto undo = [c]() {
            for (cudaStream_t s : {c->stream, c->comm_stream, c->aux_stream, c->h2d_stream, c->d2h_stream})
                if (s) cudaStreamDestroy(s);
            for (cudaEvent_t ev : {c->staging_free, c->bcast_free})
                if (ev) cudaEventDestroy(ev);
            if (c->red_buf) cudaFree(c->red_buf);
            delete c;
        };
        if ((e = cudaGetDevice(&c->device)) != cudaSuccess ||
            (e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device)) != cudaSuccess) {
            undo();
            return cuda_fail(e, "device query");
        }
        if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) != cudaSuccess) {
            undo();
            return cuda_fail(e, "cudaStreamCreate");
        }
        if ((e = preload_kernels()) != cudaSuccess) {
            undo();
            return cuda_fail(e, "kernel preload (is this an sm_100 device?)");
        }
        if ((e = cudaMalloc(reinterpret_cast<void **>(&c->red_buf), sizeof(int64_t))) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&c->h2d_stream, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&c->staging_free, cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&c->bcast_free, cudaEventDisableTiming)) != cudaSuccess) {
            undo();
            return cuda_fail(e, "runtime streams / events / buffers");
        }
        c->bcast_loopback = env_int("COMPAR_BCAST_LOOPBACK", 0);
        // measurement aid: run the persistent kernels on fewer SMs (e.g. the SMs left beside an
        // NCCL broadcast), read once here
        const int sms_cap = env_int("COMPAR_NUM_SMS", 0);
        if (sms_cap >= 2 && sms_cap < c->num_sms) c->num_sms = sms_cap;
        c->bcast_reserve_sms = env_int("COMPAR_BCAST_RESERVE_SMS", cfg.bcast_ctas);
        c->host_chunks = env_int("COMPAR_HOST_CHUNKS", 32);
        c->host_tail_split = env_int("COMPAR_HOST_TAIL_SPLIT", 1);
        c->d2h_kernel_ctas = env_int("COMPAR_D2H_KERNEL_CTAS", 4);
    }
    {
        std::lock_guard<std::mutex> lk(g_live_mu);
        g_live.insert(c);
    }
    if (!c->virt && cfg.builtins) {
        int id;
        compar_register_variant(c, "gemm", "simt_f32", COMPAR_TGT_SIMT_F32, nullptr, nullptr, &id);
        compar_register_variant(c, "gemm", "tma_f32", COMPAR_TGT_TMA_F32, nullptr, nullptr, &id);
        compar_register_variant(c, "gemm", "tc_tf32", COMPAR_TGT_TC_TF32, nullptr, nullptr, &id);
        compar_register_variant(c, "gemm", "tc_bf16", COMPAR_TGT_TC_BF16, nullptr, nullptr, &id);
        compar_register_variant(c, "gemm", "tc_tf32_2sm", COMPAR_TGT_TC2_TF32, nullptr, nullptr, &id);
        compar_register_variant(c, "gemm", "tc_bf16_2sm", COMPAR_TGT_TC2_BF16, nullptr, nullptr, &id);
        compar_register_variant(c, "gemm", "tc_tf32_2sm_w", COMPAR_TGT_TCW_TF32, nullptr, nullptr, &id);
        compar_register_variant(c, "gemm", "tc_bf16_2sm_w", COMPAR_TGT_TCW_BF16, nullptr, nullptr, &id);
        compar_register_variant(c, "gemm", "simt_bf16", COMPAR_TGT_SIMT_BF16, nullptr, nullptr, &id);
        compar_register_variant(c, "gemm", "tc_tf32_sk", COMPAR_TGT_TCS_TF32, nullptr, nullptr, &id);
        compar_register_variant(c, "gemm", "tc_bf16_sk", COMPAR_TGT_TCS_BF16, nullptr, nullptr, &id);
        compar_register_variant(c, "gemm", "tc_tf32_ck", COMPAR_TGT_TCK_TF32, nullptr, nullptr, &id);
        compar_register_variant(c, "gemm", "tc_bf16_ck", COMPAR_TGT_TCK_BF16, nullptr, nullptr, &id);
        compar_register_variant(c, "gemm", "tc_f32x3", COMPAR_TGT_TCX_F32, nullptr, nullptr, &id);
        compar_register_sort_variant(c, "sort_radix", COMPAR_TGT_SORT_RADIX, nullptr, nullptr, &id);
        compar_register_sort_variant(c, "sort_bitonic", COMPAR_TGT_SORT_BITONIC, nullptr, nullptr, &id);
    }
    *ctx = c;
    if (!c->perf_path.empty()) {
        std::ifstream f(c->perf_path);
        if (f.good()) {
            compar_status s = compar_perf_load(c, c->perf_path.c_str());
            if (s != COMPAR_OK) return s;
        }
    }
    return COMPAR_OK;
}

compar_status compar_terminate(void *ctx) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    compar_status st = COMPAR_OK;
    {
        std::lock_guard<std::mutex> lk(c->mu);
        for (auto &kv : c->tasks) {
            compar_report rep;
            finish_task(c, kv.second, &rep);
        }
        c->tasks.clear();
        c->done.clear();
    }
    if (!c->perf_path.empty()) st = compar_perf_save(c, c->perf_path.c_str());
    bool last_ctx = false;
    {
        std::lock_guard<std::mutex> lk(g_live_mu);
        g_live.erase(c);
        last_ctx = g_live.empty();
    }
    if (!c->virt) {
        cudaStreamSynchronize(c->stream);
        if (last_ctx) {   // no context can have work in flight: drop the large kernel workspaces
            release_f32x3_workspaces();
            release_split_workspaces();
        }
        for (auto &b : c->staging)
            if (b) cudaFree(b);
        if (c->breplica) cudaFree(c->breplica);
        if (c->bpacked) cudaFree(c->bpacked);
        if (c->ce_up_buf) cudaIpcCloseMemHandle(c->ce_up_buf);
        if (c->ce_up_flags) cudaIpcCloseMemHandle(c->ce_up_flags);
        if (c->ce_buf) cudaFree(c->ce_buf);
        if (c->ce_flags) cudaFree(c->ce_flags);
        if (c->scratch) cudaFree(c->scratch);
        if (c->sort_scratch) cudaFree(c->sort_scratch);
        if (c->sort_done) cudaEventDestroy(c->sort_done);
        for (cudaEvent_t ev : {c->staging_free, c->bcast_free})
            if (ev) cudaEventDestroy(ev);
        if (c->slab_flags) cudaFree(c->slab_flags);
        for (cudaStream_t s : {c->comm_stream, c->aux_stream, c->h2d_stream, c->d2h_stream}) {
            if (s) {
                cudaStreamSynchronize(s);
                cudaStreamDestroy(s);
            }
        }
        if (c->red_buf) cudaFree(c->red_buf);
        if (c->xbuf) cudaFree(c->xbuf);
        for (size_t l = 0; l < c->lane_streams.size(); ++l) {
            cudaStreamSynchronize(c->lane_streams[l]);
            cudaStreamDestroy(c->lane_streams[l]);
            cudaEventDestroy(c->lane_done[l]);
        }
        if (c->sub_event) cudaEventDestroy(c->sub_event);
        if (c->cal_fence) cudaEventDestroy(c->cal_fence);
        for (auto e : c->pool) cudaEventDestroy(e);
        if (c->comm) ncclCommDestroy(c->comm);
        cudaStreamDestroy(c->stream);
    }
    delete c;
    return st;
}

compar_status compar_register_variant(void *ctx, const char *iface, const char *name, compar_target target,
                                      compar_gemm_fn fn, void *user, int *out_id) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    if (!iface || std::strcmp(iface, "gemm") != 0) return fail(COMPAR_E_INVALID, "unknown interface (only \"gemm\")");
    if (!name || !*name || std::strlen(name) > 63) return fail(COMPAR_E_INVALID, "bad variant name");
    for (const char *p = name; *p; ++p)
        if (*p == ' ' || *p == '\t' || *p == '\n') return fail(COMPAR_E_INVALID, "variant name has whitespace");
    if (target < COMPAR_TGT_SIMT_F32 || target > COMPAR_TGT_TCX_F32) return fail(COMPAR_E_INVALID, "unknown target");
    if (target == COMPAR_TGT_USER && !fn) return fail(COMPAR_E_INVALID, "USER variant needs a launch function");
    if (target != COMPAR_TGT_USER && c->virt) return fail(COMPAR_E_INVALID, "built-in targets need CUDA");
    std::lock_guard<std::mutex> lk(c->mu);
    for (const auto &v : c->variants)
        if (v.name == name) return fail(COMPAR_E_DUPLICATE, std::string("duplicate variant ") + name);
    if (c->variants.size() >= 64) return fail(COMPAR_E_INVALID, "too many variants");
    c->variants.push_back(Variant{name, target, fn, user, c->hist.intern(name)});
    if (out_id) *out_id = static_cast<int>(c->variants.size()) - 1;
    return COMPAR_OK;
}

compar_status compar_register_sort_variant(void *ctx, const char *name, compar_target target, compar_sort_fn fn,
                                           void *user, int *out_id) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    if (!name || !*name || std::strlen(name) > 63) return fail(COMPAR_E_INVALID, "bad variant name");
    for (const char *p = name; *p; ++p)
        if (*p == ' ' || *p == '\t' || *p == '\n') return fail(COMPAR_E_INVALID, "variant name has whitespace");
    if (target != COMPAR_TGT_SORT_RADIX && target != COMPAR_TGT_SORT_BITONIC && target != COMPAR_TGT_USER)
        return fail(COMPAR_E_INVALID, "not a sort target");
    if (target == COMPAR_TGT_USER && !fn) return fail(COMPAR_E_INVALID, "USER variant needs a sort function");
    if (target != COMPAR_TGT_USER && c->virt) return fail(COMPAR_E_INVALID, "built-in targets need CUDA");
    std::lock_guard<std::mutex> lk(c->mu);
    for (const auto &v : c->variants)
        if (v.name == name) return fail(COMPAR_E_DUPLICATE, std::string("duplicate variant ") + name);
    if (c->variants.size() >= 64) return fail(COMPAR_E_INVALID, "too many variants");
    Variant v{name, target, nullptr, user, c->hist.intern(name)};
    v.iface = kSort;
    v.sfn = fn;
    c->variants.push_back(v);
    if (out_id) *out_id = static_cast<int>(c->variants.size()) - 1;
    return COMPAR_OK;
}

compar_status compar_variant_count(void *ctx, int *n) {
    Ctx *c = as_ctx(ctx);
    if (!c || !n) return fail(c ? COMPAR_E_INVALID : COMPAR_E_STATE, "bad arguments");
    std::lock_guard<std::mutex> lk(c->mu);
    *n = static_cast<int>(c->variants.size());
    return COMPAR_OK;
}

compar_status compar_variant_info(void *ctx, int id, char *name, int name_len, int *target) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    std::lock_guard<std::mutex> lk(c->mu);
    if (id < 0 || id >= static_cast<int>(c->variants.size())) return fail(COMPAR_E_INVALID, "bad variant id");
    if (name && name_len > 0) {
        std::strncpy(name, c->variants[id].name.c_str(), static_cast<size_t>(name_len) - 1);
        name[name_len - 1] = 0;
    }
    if (target) *target = c->variants[id].target;
    return COMPAR_OK;
}

namespace {

// Decide (variant, mode) for a plan; `commit` accounts the execution in the history.
// Task-parallel world: the lane streams, their "last work" events, the submission event and the
// calibration fence, created on first use.
compar_status ensure_lanes(Ctx *c) {
    if (!c->lane_streams.empty()) return COMPAR_OK;
    const int L = c->placer.lanes();
    for (int l = 0; l < L; ++l) {
        cudaStream_t s = nullptr;
        cudaEvent_t e = nullptr;
        cudaError_t err = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        if (err == cudaSuccess) err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        if (err != cudaSuccess) return cuda_fail(err, "lane stream");
        c->lane_streams.push_back(s);
        c->lane_done.push_back(e);
    }
    cudaError_t err = cudaEventCreateWithFlags(&c->sub_event, cudaEventDisableTiming);
    if (err == cudaSuccess) err = cudaEventCreateWithFlags(&c->cal_fence, cudaEventDisableTiming);
    return err == cudaSuccess ? COMPAR_OK : cuda_fail(err, "lane events");
}

// Batched calibration timing (reading c13; R25): a timed calibration
// execution of a built-in on a key whose work is below batch_below_ns (100 us) repeats the launch
// r = ceil(200 us / t) times (<= 64), each between its own event pair, and records the median
// single-launch time, so launch / clock jitter does not decide between variants a few percent
// apart (with 3 single-launch samples, 1024^3 TF32 picked a 6 % slower variant) while the sample
// stays the quantity a model-mode execution measures (a batch's span / r hides launch overhead
// that differs between kernels: it ranked tma_f32 over tc_tf32 at 64^3).
// t is a static estimate from the key alone (5 us floor + FLOPs at 100 TFLOP/s + compulsory bytes
// at 3 TB/s), so every variant of a key is sampled with the same r: deriving r from each variant's
// own warm-up made the first-ever launch of a kernel (module/workspace set-up, tens of us) switch
// batching off for that variant only, and unbatched samples lost to batched ones by the launch
// overhead (config 1: 18 % regret).
int calib_batch(Ctx *c, const Task &t) {
    if (c->batch_below_ns <= 0 || t.mode != kCalib || t.variant < 0) return 1;
    if (c->variants[t.variant].target == COMPAR_TGT_USER) return 1;
    const Key &k = t.key;
    const double flops = 2.0 * static_cast<double>(k.m) * static_cast<double>(k.n) * static_cast<double>(k.k);
    const double sin = k.dtype == COMPAR_BF16 ? 2.0 : 4.0;
    const double bytes = sin * (static_cast<double>(k.m) * k.k + static_cast<double>(k.k) * k.n) +
                         4.0 * static_cast<double>(k.m) * k.n * (k.beta0 ? 1.0 : 2.0);
    const double est = 5000.0 + flops / 100e12 * 1e9 + bytes / 3e12 * 1e9;
    if (est >= static_cast<double>(c->batch_below_ns)) return 1;
    return static_cast<int>(std::min(64.0, std::ceil(200000.0 / est)));
}

// Static lower bound (ns) of a built-in GEMM variant on a key (R32): FLOPs at the
// nominal dense peak of its arithmetic class, compulsory bytes at the nominal HBM bandwidth —
// both datasheet figures above anything measured, so the bound is below the true time.
// FFMA class: SMs x 128 FMA/clk x 2 FLOP x 1965 MHz; tensor cores: 2.25 PFLOP/s BF16, half for
// TF32; HBM3e 8 TB/s.  0 (no bound) for USER variants and other interfaces.
double static_lb_ns(const Ctx *c, compar_target t, const Key &k) {
    double peak;
    switch (t) {
        case COMPAR_TGT_SIMT_F32:
        case COMPAR_TGT_TMA_F32:
        case COMPAR_TGT_SIMT_BF16: peak = static_cast<double>(c->num_sms) * 128.0 * 2.0 * 1.965e9; break;
        case COMPAR_TGT_TC_BF16:
        case COMPAR_TGT_TC2_BF16:
        case COMPAR_TGT_TCW_BF16:
        case COMPAR_TGT_TCS_BF16:
        case COMPAR_TGT_TCK_BF16: peak = 2.25e15; break;
        case COMPAR_TGT_TC_TF32:
        case COMPAR_TGT_TC2_TF32:
        case COMPAR_TGT_TCW_TF32:
        case COMPAR_TGT_TCS_TF32:
        case COMPAR_TGT_TCK_TF32: peak = 1.125e15; break;
        case COMPAR_TGT_TCX_F32: peak = 1.125e15 / 3.0; break;   // three TF32 products per FP32 product
        default: return 0.0;
    }
    const double m = static_cast<double>(k.m), n = static_cast<double>(k.n), kk = static_cast<double>(k.k);
    const double flops = 2.0 * m * n * kk;
    const double eb = k.dtype == COMPAR_BF16 ? 2.0 : 4.0;
    const double bytes = eb * (m * kk + kk * n) + 4.0 * m * n * (k.beta0 ? 1.0 : 2.0);
    return std::max(flops / peak, bytes / 8.0e12) * 1e9;
}

// Steps 3-7 over an eligible set (registry indices idx, history ids names), any interface.
compar_status choose_core(Ctx *c, const std::vector<int> &idx, const std::vector<int> &names, const Key &key,
                          int hint, bool commit, int *variant, int *mode, bool *warm);

compar_status choose(Ctx *c, const compar_gemm_desc *d, const Plan &plan, bool commit, int *variant, int *mode,
                     bool *warm) {
    std::vector<int> idx;
    std::vector<int> names;  // interned history ids, in registry order
    eligible_set(c, d, plan, idx, names);
    return choose_core(c, idx, names, plan.key, d->variant_hint, commit, variant, mode, warm);
}

compar_status choose_core(Ctx *c, const std::vector<int> &idx, const std::vector<int> &names, const Key &key,
                          int hint, bool commit, int *variant, int *mode, bool *warm) {
    Range range("compar.select");
    Plan plan;  // (only .key is used below)
    plan.key = key;
    *warm = false;
    if (hint >= 0) {
        if (std::find(idx.begin(), idx.end(), hint) == idx.end())
            return fail(COMPAR_E_INVALID, "variant_hint is not eligible for this task");
        *variant = hint;
        *mode = kHint;
        return COMPAR_OK;
    }
    if (idx.empty()) return fail(COMPAR_E_NO_VARIANT, "no eligible variant for this dtype/compute/layout");
    if (c->cfg.sched == 1) {
        *variant = idx[0];
        *mode = kEager;
        return COMPAR_OK;
    }
    std::vector<double> lb(idx.size(), 0.0);   // R32 static lower bounds (GEMM keys only)
    if (key.compute >= 0)
        for (size_t i = 0; i < idx.size(); ++i) lb[i] = static_lb_ns(c, c->variants[idx[i]].target, key);
    if (c->cfg.sched == 2 && key.compute >= 0) {
        // "predict" scheduler (NEXT-2; GEMM keys — its features are FLOPs and bytes): every pending sample is harvested first (the fit reads all
        // keys), then measured means / model predictions decide; unknown variants fall back to
        // calibration below.
        harvest_all(c);
        Mode pm;
        const int ppos = c->hist.decide_predict(names, plan.key, &pm, &lb);
        if (ppos >= 0) {
            *variant = idx[ppos];
            *mode = pm;
            if (commit) *warm = c->hist.commit(names[ppos], plan.key, c->hist.warm_count(lb[ppos]));
            return COMPAR_OK;
        }
        // Only the variants with neither a sample nor a model are calibrated for this key (a
        // variant eligible on too few keys to fit, e.g. the split-K one, must not send every
        // other variant back to calibration).
        const std::vector<int> unk = c->hist.unknown_predict(names, plan.key, &lb);
        std::vector<int> uidx, unames;
        std::vector<double> ulb;
        for (int u : unk) {
            uidx.push_back(idx[u]);
            unames.push_back(names[u]);
            ulb.push_back(lb[u]);
        }
        if (!unames.empty() && unames.size() < names.size()) {
            Mode m;
            const int pos = c->hist.decide(unames, plan.key, &m, &ulb);
            *variant = uidx[pos];
            *mode = m;
            if (commit) *warm = c->hist.commit(unames[pos], plan.key, c->hist.warm_count(ulb[pos]));
            return COMPAR_OK;
        }
    }
    // Step 6: pending samples of the key are harvested (blocking) before a model decision — and,
    // with pruning on, before a calibration decision too, since R32 reads the key's best mean
    // (so every decision stays a function of the submission sequence and the measured values).
    if (c->hist.prune_pct > 0 || !c->hist.calibrating(names, plan.key, &lb)) harvest_key(c, plan.key);
    Mode m;
    const int pos = c->hist.decide(names, plan.key, &m, &lb);
    *variant = idx[pos];
    *mode = m;
    if (commit) *warm = c->hist.commit(names[pos], plan.key, c->hist.warm_count(lb[pos]));
    return COMPAR_OK;
}

}  // namespace

compar_status compar_select(void *ctx, const compar_gemm_desc *d, int *variant, int *mode) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    std::lock_guard<std::mutex> lk(c->mu);
    compar_status s = validate(c, d);
    if (s != COMPAR_OK) return s;
    Plan plan;
    build_plan(c, d, plan, d->A, d->B, d->C_in, d->C_out);
    int v = -1, m = kNoop;
    bool warm;
    if (d->m > 0 && d->n > 0 && d->k > 0 && d->alpha != 0.f) {
        c->in_select = true;    // never a collective harvest from a query
        s = choose(c, d, plan, false, &v, &m, &warm);
        c->in_select = false;
        if (s != COMPAR_OK) return s;
    }
    if (variant) *variant = v;
    if (mode) *mode = m;
    return COMPAR_OK;
}

compar_status compar_gemm_submit(void *ctx, const compar_gemm_desc *d, uint64_t *task_out) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    std::lock_guard<std::mutex> lk(c->mu);
    compar_status s = validate(c, d);
    if (s != COMPAR_OK) return s;
    c->stats.submits++;
    if (c->sticky != COMPAR_OK && d->world != COMPAR_WORLD_LOCAL && c->nranks > 1)
        return fail(c->sticky, "cross-rank path failed earlier: " + c->sticky_msg);
    Task t;
    t.id = c->next_task++;
    t.world = d->world == COMPAR_WORLD_PANELS;
    t.tasks = d->world == COMPAR_WORLD_TASKS;
    // NULL is the CUDA legacy default stream (the CUDA convention, and torch's default stream),
    // so a task is ordered after work the caller queued there.
    cudaStream_t st = static_cast<cudaStream_t>(d->stream);
    const int eb = elem_bytes(d->in_dtype);
    const bool work = d->m > 0 && d->n > 0;
    const bool gemm = work && d->k > 0 && d->alpha != 0.f;

    // Operand pointers the kernels use (host mode: library staging buffers).
    const void *A = d->A, *B = d->B;
    const float *Cin = d->C_in;
    float *Cout = d->C_out;
    const bool host = d->mem == COMPAR_MEM_HOST && !c->virt;
    // Rows this process owns: the whole m, or this rank's panel in world mode.
    int64_t mloc = d->m;
    if (t.world) {
        std::vector<int64_t> offs;
        partition(d->m, c->nranks, offs);
        mloc = offs[c->rank + 1] - offs[c->rank];
    }
    const bool root_b = !t.world || c->rank == 0;  // this process holds B
    const size_t a_bytes =
        (gemm && mloc > 0) ? static_cast<size_t>(mloc - 1) * d->lda * eb + static_cast<size_t>(d->k) * eb : 0;
    const size_t b_rows = d->transB ? d->n : d->k;
    const size_t b_width = d->transB ? d->k : d->n;
    const size_t b_bytes = gemm ? (b_rows - 1) * d->ldb * eb + b_width * eb : 0;
    const size_t cin_bytes = (work && mloc > 0 && d->beta != 0.f)
                                 ? static_cast<size_t>(mloc - 1) * d->ldc_in * 4 + static_cast<size_t>(d->n) * 4
                                 : 0;
    const size_t cout_bytes =
        (work && mloc > 0) ? static_cast<size_t>(mloc - 1) * d->ldc_out * 4 + static_cast<size_t>(d->n) * 4 : 0;
    if (host && work) {
        if ((s = ensure_buffer(&c->staging[0], &c->staging_bytes[0], a_bytes)) != COMPAR_OK) return s;
        if (root_b && (s = ensure_buffer(&c->staging[1], &c->staging_bytes[1], b_bytes)) != COMPAR_OK) return s;
        if ((s = ensure_buffer(&c->staging[3], &c->staging_bytes[3], cout_bytes)) != COMPAR_OK) return s;
        const bool inplace = d->C_in == d->C_out && d->ldc_in == d->ldc_out;
        if (cin_bytes && !inplace && (s = ensure_buffer(&c->staging[2], &c->staging_bytes[2], cin_bytes)) != COMPAR_OK)
            return s;
        A = c->staging[0];
        if (root_b) B = c->staging[1];
        Cout = static_cast<float *>(c->staging[3]);
        Cin = cin_bytes ? (inplace ? Cout : static_cast<float *>(c->staging[2])) : nullptr;
    }
    // World mode, non-root ranks: B arrives in a replica.
    if (!root_b && gemm && !c->virt) {
        if (d->B_replica) {
            B = d->B_replica;
        } else {
            if ((s = ensure_buffer(&c->breplica, &c->breplica_bytes, b_bytes)) != COMPAR_OK) return s;
            B = c->breplica;
        }
    }

    Plan plan;
    build_plan(c, d, plan, A, B, Cin, Cout);
    t.key = plan.key;
    if (gemm) {
        bool warm = false;
        // task-parallel world: the history is charged only once the placement succeeded
        s = choose(c, d, plan, !t.tasks, &t.variant, &t.mode, &warm);
        if (s != COMPAR_OK) {
            c->stats.failed++;
            return s;
        }
        t.warm = warm;
        t.history = (t.mode == kWarmup || t.mode == kCalib || t.mode == kModel || t.mode == kPredict);
    } else {
        t.mode = kNoop;
    }
    std::vector<uint64_t> deps;  // task-parallel world: earlier tasks on other lanes to wait for
    if (t.tasks) {
        // dmda placement (dmda.h): worker = argmin predicted end over the allowed workers
        if (!c->placer_ready) {
            c->placer.configure(c->nranks, c->cfg.lanes);
            c->placer_ready = true;
        }
        Access acc;
        auto span = [](const void *p, size_t bytes) {
            const uintptr_t lo = reinterpret_cast<uintptr_t>(p);
            return Span{lo, lo + bytes};
        };
        // a caller data handle (non-zero id) maps to its own disjoint range of a synthetic space,
        // identical on every rank; otherwise the operand's byte range (per-process pointers)
        auto span_h = [&](int i, const void *p, size_t bytes) {
            if (d->handles[i] == 0) return span(p, bytes);
            const uintptr_t lo = (uintptr_t(1) << 63) + static_cast<uintptr_t>(d->handles[i] % (uint64_t(1) << 22)) *
                                                            (uintptr_t(1) << 40);
            return Span{lo, lo + bytes};
        };
        if (gemm && (d->A || d->handles[0]) && a_bytes) acc.reads.push_back(span_h(0, d->A, a_bytes));
        if (gemm && (d->B || d->handles[1]) && b_bytes) acc.reads.push_back(span_h(1, d->B, b_bytes));
        if ((d->C_in || d->handles[2]) && cin_bytes) acc.reads.push_back(span_h(2, d->C_in, cin_bytes));
        if ((d->C_out || d->handles[3]) && cout_bytes) acc.writes.push_back(span_h(3, d->C_out, cout_bytes));
        int64_t exec = 0;  // predicted ns: the variant's measured mean for the key, else unknown (0)
        if (gemm) {
            const Record *r = c->hist.find(c->variants[t.variant].hid, plan.key);
            if (r && r->count > 0) exec = static_cast<int64_t>(r->sum_ns / static_cast<unsigned __int128>(r->count));
        }
        int64_t end = 0;
        const int w = c->placer.place(acc, exec, &end, &deps);
        if (w < 0) {
            c->stats.failed++;
            return fail(COMPAR_E_INVALID, "task reads data last written by pending tasks on different ranks");
        }
        t.owner = c->placer.rank_of(w);
        t.lane = w % c->placer.lanes();
        t.remote = t.owner != c->rank;
        c->placer.commit(t.id, w, end, acc);
        if (t.history)
            t.warm = c->hist.commit(c->variants[t.variant].hid, plan.key,
                                    c->hist.warm_count(static_lb_ns(c, c->variants[t.variant].target, plan.key)));
        // lanes > 1: model-mode executions overlap other lanes, so their times are not samples
        if (c->placer.lanes() > 1 && (t.mode == kModel || t.mode == kPredict)) t.history = false;
    }
    for (const auto &p : plan.panels) {
        PanelRun pr;
        pr.p = p;
        t.panels.push_back(pr);
    }

    if (c->virt) {
        // Virtual clock: USER variants report synthetic ns; nothing touches CUDA.
        if (gemm && !t.remote) {
            const Variant &var = c->variants[t.variant];
            for (auto &pr : t.panels) {
                compar_status r = var.fn(d, &pr.p, nullptr, var.user, &pr.virtual_ns);
                if (r != COMPAR_OK) t.status = COMPAR_E_TASK_FAILED;
            }
        }
    } else if (work && !t.remote) {
        const bool calib_task = t.mode == kWarmup || t.mode == kCalib;
        if (t.tasks) {  // run on this worker's lane stream, after `stream` and the dependencies
            if ((s = ensure_lanes(c)) != COMPAR_OK) return s;
            cudaStream_t ls = c->lane_streams[t.lane];
            cudaEventRecord(c->sub_event, st);
            cudaStreamWaitEvent(ls, c->sub_event, 0);
            for (uint64_t dep : deps) {
                auto it = c->tasks.find(dep);
                if (it == c->tasks.end() || it->second.remote) continue;
                const Task &dt = it->second;
                cudaEvent_t ev = dt.end ? dt.end : (dt.panels.empty() ? nullptr : dt.panels.back().stop);
                if (ev) cudaStreamWaitEvent(ls, ev, 0);
            }
            if (c->placer.lanes() > 1) {  // calibration runs alone on the GPU
                if (calib_task) {
                    for (int l = 0; l < c->placer.lanes(); ++l)
                        if (l != t.lane) cudaStreamWaitEvent(ls, c->lane_done[l], 0);
                } else if (c->cal_fence_set) {
                    cudaStreamWaitEvent(ls, c->cal_fence, 0);
                }
            }
            st = ls;
        }
        // The plain single-launch task (device memory, one panel, no broadcast) uses the panel's
        // start/stop events as the task span: two event records per task instead of four.
        const bool simple = !host && t.panels.size() == 1 && !(t.world && gemm && (c->nranks > 1 || c->bcast_loopback));
        if (!simple) {
            t.begin = get_event(c);
            t.end = get_event(c);
            cudaEventRecord(t.begin, st);
        }
        const bool pipelined = host && gemm && !t.world && t.panels.size() == 1 && c->host_chunks > 1 && d->m >= 512;
        // the staging buffers are shared by every host-mode task of the context: a task on another
        // stream must not overwrite them while the previous host task still reads or returns them
        if (host && c->staging_free_set) cudaStreamWaitEvent(st, c->staging_free, 0);
        if (host && !pipelined) {
            if (a_bytes) cudaMemcpyAsync(const_cast<void *>(A), d->A, a_bytes, cudaMemcpyHostToDevice, st);
            if (b_bytes && root_b) cudaMemcpyAsync(const_cast<void *>(B), d->B, b_bytes, cudaMemcpyHostToDevice, st);
            if (cin_bytes) cudaMemcpyAsync(const_cast<float *>(Cin), d->C_in, cin_bytes, cudaMemcpyHostToDevice, st);
            c->stats.bytes_h2d += static_cast<int64_t>(a_bytes + (root_b ? b_bytes : 0) + cin_bytes);
        }
        const Variant *var = gemm ? &c->variants[t.variant] : nullptr;
        Range launch_range("compar.launch");
        // sms: SMs a launch may use (0 = all; world mode leaves the broadcast's share); wl: the
        // wide variant's world-mode extras (slab flags; helper launch that returns the reserve)
        auto launch_on = [&](const compar_gemm_desc *dd, const compar_panel &pp, int sms,
                             const WorldLaunch *wl = nullptr) -> compar_status {
            if (!gemm) return run_scale(c, dd, pp, st);
            if (var->target == COMPAR_TGT_USER) {
                c->stats.launches++;
                return var->fn(dd, &pp, st, var->user, nullptr);
            }
            const bool wide = var->target == COMPAR_TGT_TCW_TF32 || var->target == COMPAR_TGT_TCW_BF16;
            if (wide && wl && wl->helper_sms > 0) sms = 0;      // the launcher splits main / helper itself
            const compar_status rs = run_builtin(c, var->target, dd, pp, st, sms, wide ? wl : nullptr);
            if (rs == COMPAR_OK && wide && wl && wl->launches > 1) c->stats.launches += wl->launches - 1;   // helper
            return rs;
        };
        const bool bcast = t.world && gemm && (c->nranks > 1 || c->bcast_loopback);
        if (pipelined) {
            compar_status r = host_pipeline(c, d, t, st, A, B, Cin, Cout, b_bytes, launch_on);
            if (r != COMPAR_OK && t.status == COMPAR_OK) t.status = r;
        } else if (!bcast) {
            int batch = (simple && gemm) ? calib_batch(c, t) : 1;
            if (batch > 1 && ensure_buffer(&c->scratch, &c->scratch_bytes, cout_bytes) != COMPAR_OK) batch = 1;
            for (auto &pr : t.panels) {
                pr.start = get_event(c);
                pr.stop = get_event(c);
                pr.batch = batch;
                cudaEventRecord(pr.start, st);
                compar_panel extra = pr.p;   // the r - 1 timing repeats write the scratch C
                extra.C_out = static_cast<float *>(c->scratch);
                for (int i = 1; i < batch; ++i) {
                    // one event pair per launch: the sample is the median single-launch time
                    // (the quantity model-mode samples measure), not the batch's span / r
                    std::pair<cudaEvent_t, cudaEvent_t> span{get_event(c), get_event(c)};
                    cudaEventRecord(span.first, st);
                    if (launch_on(d, extra, 0) != COMPAR_OK) t.status = COMPAR_E_TASK_FAILED;
                    cudaEventRecord(span.second, st);
                    pr.sub.push_back(span);
                }
                if (batch > 1) {
                    std::pair<cudaEvent_t, cudaEvent_t> span{get_event(c), get_event(c)};
                    cudaEventRecord(span.first, st);
                    if (launch_on(d, pr.p, 0) != COMPAR_OK) t.status = COMPAR_E_TASK_FAILED;
                    cudaEventRecord(span.second, st);
                    pr.sub.push_back(span);
                } else if (launch_on(d, pr.p, 0) != COMPAR_OK) {
                    t.status = COMPAR_E_TASK_FAILED;
                }
                cudaEventRecord(pr.stop, st);
            }
        } else {
            const bool fused_ok = var && (var->target == COMPAR_TGT_TCW_TF32 || var->target == COMPAR_TGT_TCW_BF16);
            compar_status r = world_pipeline(c, d, t, st, B, fused_ok, launch_on);
            if (r != COMPAR_OK && t.status == COMPAR_OK) t.status = r;
        }
        if (host && !pipelined && mloc > 0) {
            cudaMemcpy2DAsync(d->C_out, d->ldc_out * 4, Cout, d->ldc_out * 4, d->n * 4, mloc, cudaMemcpyDeviceToHost, st);
            c->stats.bytes_d2h += static_cast<int64_t>(mloc * d->n * 4);
            (void)cout_bytes;
        }
        if (t.end) cudaEventRecord(t.end, st);
        if (host) {
            cudaEventRecord(c->staging_free, st);
            c->staging_free_set = true;
        }
        if (t.tasks) {
            cudaEventRecord(c->lane_done[t.lane], st);
            if (calib_task && c->placer.lanes() > 1) {
                cudaEventRecord(c->cal_fence, st);
                c->cal_fence_set = true;
            }
        }
    }
    if (task_out) *task_out = t.id;
    c->tasks.emplace(t.id, std::move(t));
    return COMPAR_OK;
}

compar_status compar_sort_submit(void *ctx, const compar_sort_desc *d, uint64_t *task_out) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    std::lock_guard<std::mutex> lk(c->mu);
    if (!d) return fail(COMPAR_E_INVALID, "desc is NULL");
    if (d->n < 0 || d->n >= (int64_t(1) << 30)) return fail(COMPAR_E_INVALID, "n out of range [0, 2^30)");
    if (d->key_type < COMPAR_KEY_U32 || d->key_type > COMPAR_KEY_F32) return fail(COMPAR_E_INVALID, "bad key_type");
    if (d->n > 0 && !d->keys && !c->virt) return fail(COMPAR_E_INVALID, "keys NULL");
    if (d->variant_hint < -1 || d->variant_hint >= static_cast<int>(c->variants.size()))
        return fail(COMPAR_E_INVALID, "variant_hint out of range");
    c->stats.submits++;
    Task t;
    t.id = c->next_task++;
    t.key = Key{d->n, 0, 0, 100 + static_cast<int>(d->key_type), -1, 0, 0};
    cudaStream_t st = static_cast<cudaStream_t>(d->stream);
    const bool work = d->n > 1;  // 0 or 1 keys are sorted already
    if (work) {
        std::vector<int> idx, names;
        for (size_t v = 0; v < c->variants.size(); ++v) {
            if (v < 63 && (c->cfg.variant_mask >> v) & 1) continue;
            const Variant &var = c->variants[v];
            if (var.iface != kSort) continue;
            if (var.target == COMPAR_TGT_SORT_BITONIC && d->n > sort_bitonic_max()) continue;
            idx.push_back(static_cast<int>(v));
            names.push_back(var.hid);
        }
        if (idx.empty() && d->variant_hint < 0) return fail(COMPAR_E_NO_VARIANT, "no eligible sort variant");
        bool warm = false;
        compar_status s = choose_core(c, idx, names, t.key, d->variant_hint, true, &t.variant, &t.mode, &warm);
        if (s != COMPAR_OK) {
            c->stats.failed++;
            return s;
        }
        t.warm = warm;
        t.history = (t.mode == kWarmup || t.mode == kCalib || t.mode == kModel || t.mode == kPredict);
        PanelRun pr;
        pr.p.rows = d->n;
        const Variant &var = c->variants[t.variant];
        if (c->virt) {
            if (var.sfn(d, nullptr, var.user, &pr.virtual_ns) != COMPAR_OK) t.status = COMPAR_E_TASK_FAILED;
        } else {
            if (var.target == COMPAR_TGT_SORT_RADIX) {
                s = ensure_buffer(&c->sort_scratch, &c->sort_scratch_bytes, sort_radix_scratch_bytes(d->n));
                if (s != COMPAR_OK) return s;
            }
            if (!c->sort_done) cudaEventCreateWithFlags(&c->sort_done, cudaEventDisableTiming);
            if (c->sort_done_set) cudaStreamWaitEvent(st, c->sort_done, 0);
            pr.start = get_event(c);
            pr.stop = get_event(c);
            cudaEventRecord(pr.start, st);
            cudaError_t e = cudaSuccess;
            if (var.target == COMPAR_TGT_SORT_RADIX) {
                e = launch_sort_radix(d->keys, d->n, d->key_type, c->sort_scratch, st, c->num_sms);
                c->stats.launches += 5;
            } else if (var.target == COMPAR_TGT_SORT_BITONIC) {
                e = launch_sort_bitonic(d->keys, d->n, d->key_type, st);
                c->stats.launches += 1;
            } else {
                c->stats.launches++;
                if (var.sfn(d, st, var.user, nullptr) != COMPAR_OK) t.status = COMPAR_E_TASK_FAILED;
            }
            if (e != cudaSuccess) {
                t.status = COMPAR_E_TASK_FAILED;
                t_err = std::string("sort launch: ") + cudaGetErrorString(e);
            }
            cudaEventRecord(pr.stop, st);
            cudaEventRecord(c->sort_done, st);
            c->sort_done_set = true;
        }
        t.panels.push_back(pr);
    } else {
        t.mode = kNoop;
    }
    if (task_out) *task_out = t.id;
    c->tasks.emplace(t.id, std::move(t));
    return COMPAR_OK;
}

compar_status compar_register_generic_variant(void *ctx, const char *iface, const char *name, compar_generic_fn fn,
                                              void *user, int *out_id) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    if (!iface || !*iface || std::strlen(iface) > 63) return fail(COMPAR_E_INVALID, "bad interface name");
    if (!std::strcmp(iface, "gemm") || !std::strcmp(iface, "sort"))
        return fail(COMPAR_E_INVALID, "gemm / sort are built-in interfaces (compar_register_variant / _sort_variant)");
    if (!name || !*name || std::strlen(name) > 63) return fail(COMPAR_E_INVALID, "bad variant name");
    if (!fn) return fail(COMPAR_E_INVALID, "a generic variant needs a function");
    std::lock_guard<std::mutex> lk(c->mu);
    for (const auto &v : c->variants)
        if (v.name == name) return fail(COMPAR_E_DUPLICATE, std::string("duplicate variant ") + name);
    if (c->variants.size() >= 64) return fail(COMPAR_E_INVALID, "too many variants");
    Variant v{name, COMPAR_TGT_USER, nullptr, user, c->hist.intern(name)};
    v.iface = kGeneric;
    v.giface = iface;
    v.gfn = fn;
    c->variants.push_back(v);
    if (out_id) *out_id = static_cast<int>(c->variants.size()) - 1;
    return COMPAR_OK;
}

void *compar_current_stream(void) { return t_current_stream; }

compar_status compar_generic_submit(void *ctx, const compar_generic_desc *d, uint64_t *task_out) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    std::lock_guard<std::mutex> lk(c->mu);
    if (!d || !d->iface) return fail(COMPAR_E_INVALID, "desc / interface is NULL");
    if (d->nargs < 0 || (d->nargs > 0 && !d->args)) return fail(COMPAR_E_INVALID, "bad args");
    if (d->nsizes < 0 || d->nsizes > 8 || (d->nsizes > 0 && !d->sizes)) return fail(COMPAR_E_INVALID, "bad sizes");
    if (d->variant_hint < -1 || d->variant_hint >= static_cast<int>(c->variants.size()))
        return fail(COMPAR_E_INVALID, "variant_hint out of range");
    if (c->virt) return fail(COMPAR_E_INVALID, "generic interfaces need CUDA");
    int64_t sz[3] = {1, 1, 1};
    for (int i = 0; i < d->nsizes; ++i) {
        if (d->sizes[i] < 0) return fail(COMPAR_E_INVALID, "negative size");
        if (i < 2) sz[i] = d->sizes[i];
        else sz[2] *= d->sizes[i];
    }
    c->stats.submits++;
    Task t;
    t.id = c->next_task++;
    // key: the sizes plus the interface (its name's history id in the dtype slot, apart from the
    // GEMM / sort keys)
    t.key = Key{sz[0], sz[1], sz[2], 1000 + c->hist.intern(std::string("iface:") + d->iface), -3, 0, 0};
    cudaStream_t st = static_cast<cudaStream_t>(d->stream);
    std::vector<int> idx, names;
    for (size_t v = 0; v < c->variants.size(); ++v) {
        if (v < 63 && (c->cfg.variant_mask >> v) & 1) continue;
        const Variant &var = c->variants[v];
        if (var.iface != kGeneric || var.giface != d->iface) continue;
        idx.push_back(static_cast<int>(v));
        names.push_back(var.hid);
    }
    if (idx.empty()) return fail(COMPAR_E_NO_VARIANT, std::string("no variant of interface ") + d->iface);
    bool warm = false;
    compar_status s = choose_core(c, idx, names, t.key, d->variant_hint, true, &t.variant, &t.mode, &warm);
    if (s != COMPAR_OK) {
        c->stats.failed++;
        return s;
    }
    t.warm = warm;
    t.history = (t.mode == kWarmup || t.mode == kCalib || t.mode == kModel || t.mode == kPredict);
    const Variant &var = c->variants[t.variant];
    PanelRun pr;
    pr.p.rows = sz[0];
    pr.start = get_event(c);
    pr.stop = get_event(c);
    cudaEventRecord(pr.start, st);
    t_current_stream = d->stream;
    if (var.gfn(d->args, d->sizes, d->nsizes, var.user) != COMPAR_OK) t.status = COMPAR_E_TASK_FAILED;
    t_current_stream = nullptr;
    c->stats.launches++;
    cudaEventRecord(pr.stop, st);
    t.panels.push_back(pr);
    if (task_out) *task_out = t.id;
    c->tasks.emplace(t.id, std::move(t));
    return COMPAR_OK;
}

compar_status compar_sync(void *ctx, uint64_t task, compar_report *out) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    std::lock_guard<std::mutex> lk(c->mu);
    compar_report rep;
    std::memset(&rep, 0, sizeof(rep));
    compar_status st = COMPAR_OK;
    Range range("compar.sync");
    if (task == COMPAR_TASK_ALL) {
        std::vector<uint64_t> ids;
        for (auto &kv : c->tasks) ids.push_back(kv.first);
        compar_status xs = exchange_ids(c, ids);  // collective in the task-parallel world
        if (xs != COMPAR_OK) return xs;
        for (auto &kv : c->done) {                // implicitly harvested, not yet synced
            rep = kv.second.second;
            if (kv.second.first != COMPAR_OK) st = kv.second.first;
        }
        c->done.clear();
        for (auto &kv : c->tasks) {
            compar_status s = finish_task(c, kv.second, &rep);
            if (s != COMPAR_OK) st = s;
        }
        c->tasks.clear();
        // a full sync drains every worker: ready times and tracked accesses restart from zero
        c->placer.reset();
        c->cal_fence_set = false;
    } else {
        auto it = c->tasks.find(task);
        if (it == c->tasks.end()) {
            auto dn = c->done.find(task);         // harvested by the selector: its stored report
            if (dn == c->done.end()) return fail(COMPAR_E_UNKNOWN_TASK, "unknown or already-synced task");
            rep = dn->second.second;
            st = dn->second.first;
            c->done.erase(dn);
            if (out) *out = rep;
            if (st != COMPAR_OK) t_err = "task failed (harvested before this sync)";
            return st;
        }
        compar_status xs = exchange_ids(c, {task});
        if (xs != COMPAR_OK) return xs;
        st = finish_task(c, it->second, &rep);
        c->tasks.erase(it);
    }
    if (out) *out = rep;
    return st;
}

compar_status compar_perf_save(void *ctx, const char *path) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    if (!path) return fail(COMPAR_E_INVALID, "path is NULL");
    std::lock_guard<std::mutex> lk(c->mu);
    std::ofstream f(path);
    if (!f.good()) return fail(COMPAR_E_IO, std::string("cannot write ") + path);
    f << "# compar perf model v1: variant m n k dtype compute transB beta0 seen count sum_ns sumsq_ns min_ns\n";
    for (const auto &kv : c->hist.table()) {
        const Key &k = kv.first.second;
        const Record &r = kv.second;
        f << c->hist.name(kv.first.first) << ' ' << k.m << ' ' << k.n << ' ' << k.k << ' ' << k.dtype << ' ' << k.compute << ' '
          << k.transB << ' ' << k.beta0 << ' ' << r.seen << ' ' << r.count << ' ' << u128_str(r.sum_ns) << ' '
          << u128_str(r.sumsq_ns) << ' ' << r.min_ns << '\n';
    }
    return f.good() ? COMPAR_OK : fail(COMPAR_E_IO, "write failed");
}

compar_status compar_perf_load(void *ctx, const char *path) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    if (!path) return fail(COMPAR_E_INVALID, "path is NULL");
    std::lock_guard<std::mutex> lk(c->mu);
    std::ifstream f(path);
    if (!f.good()) return fail(COMPAR_E_IO, std::string("cannot open ") + path);
    std::string line;
    int ln = 0;
    std::vector<std::pair<std::pair<std::string, Key>, Record>> parsed;
    while (std::getline(f, line)) {
        ++ln;
        size_t p = line.find_first_not_of(" \t\r");
        if (p == std::string::npos || line[p] == '#') continue;
        std::istringstream is(line);
        std::string name, sum_s, sq_s;
        Key k{};
        Record r;
        if (!(is >> name >> k.m >> k.n >> k.k >> k.dtype >> k.compute >> k.transB >> k.beta0 >> r.seen >> r.count >>
              sum_s >> sq_s >> r.min_ns) ||
            !parse_u128(sum_s, &r.sum_ns) || !parse_u128(sq_s, &r.sumsq_ns) || r.seen < 0 || r.count < 0) {
            return fail(COMPAR_E_FORMAT, std::string(path) + ":" + std::to_string(ln) + ": malformed record");
        }
        std::string extra;
        if (is >> extra) return fail(COMPAR_E_FORMAT, std::string(path) + ":" + std::to_string(ln) + ": trailing data");
        parsed.push_back({{name, k}, r});
    }
    for (const auto &e : parsed) c->hist.merge(e.first.first, e.first.second, e.second);
    return COMPAR_OK;
}

compar_status compar_history_get(void *ctx, int variant, const compar_gemm_desc *d, compar_record *out) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    if (!d || !out) return fail(COMPAR_E_INVALID, "NULL argument");
    std::lock_guard<std::mutex> lk(c->mu);
    if (variant < 0 || variant >= static_cast<int>(c->variants.size())) return fail(COMPAR_E_INVALID, "bad variant");
    Plan plan;
    build_plan(c, d, plan, d->A, d->B, d->C_in, d->C_out);
    std::memset(out, 0, sizeof(*out));
    const Record *r = c->hist.find(c->variants[variant].hid, plan.key);
    if (r) {
        out->seen = r->seen;
        out->count = r->count;
        out->min_ns = r->min_ns;
        out->sum_ns = r->sum_ns > static_cast<unsigned __int128>(INT64_MAX) ? INT64_MAX : static_cast<int64_t>(r->sum_ns);
        out->mean_ns = r->count ? static_cast<double>(r->sum_ns) / static_cast<double>(r->count) : 0.0;
    }
    return COMPAR_OK;
}

compar_status compar_partition_rows(int64_t m, int p, int64_t *offsets) {
    if (m < 0 || p < 1 || !offsets) return fail(COMPAR_E_INVALID, "bad partition arguments");
    std::vector<int64_t> offs;
    partition(m, p, offs);
    std::copy(offs.begin(), offs.end(), offsets);
    return COMPAR_OK;
}

compar_status compar_comm_unique_id(void *out, int len) {
    if (!out || len < static_cast<int>(sizeof(ncclUniqueId))) return fail(COMPAR_E_INVALID, "buffer too small");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return fail(COMPAR_E_NCCL, ncclGetErrorString(r));
    std::memcpy(out, &id, sizeof(id));
    return COMPAR_OK;
}

compar_status compar_comm_init(void *ctx, int nranks, int rank, const void *id, int len) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    if (nranks < 1 || rank < 0 || rank >= nranks || !id || len < static_cast<int>(sizeof(ncclUniqueId)))
        return fail(COMPAR_E_INVALID, "bad communicator arguments");
    std::lock_guard<std::mutex> lk(c->mu);
    if (c->comm) return fail(COMPAR_E_STATE, "communicator already initialised");
    c->placer_ready = false;  // workers = nranks x lanes from the next task-parallel submit
    if (c->virt) {
        c->nranks = nranks;
        c->rank = rank;
        return COMPAR_OK;
    }
    cudaSetDevice(c->device);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    // The broadcast of B overlaps the GEMMs, so NCCL's kernels get a bounded SM budget: maxCTAs =
    // bcast_ctas, which is also the SM reserve a GEMM overlapping a broadcast leaves free.
    ncclConfig_t config = NCCL_CONFIG_INITIALIZER;
    config.blocking = 1;
    config.minCTAs = 1;
    config.maxCTAs = c->cfg.bcast_ctas;
    ncclResult_t r = ncclCommInitRankConfig(&c->comm, nranks, uid, rank, &config);
    if (r != ncclSuccess) return fail(COMPAR_E_NCCL, std::string("ncclCommInitRankConfig: ") + ncclGetErrorString(r));
    c->sticky = COMPAR_OK;
    c->sticky_msg.clear();
    c->nranks = nranks;
    c->rank = rank;
    return COMPAR_OK;
}

compar_status compar_world_init(void *ctx, int nranks, int rank) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(COMPAR_E_INVALID, "bad world arguments");
    std::lock_guard<std::mutex> lk(c->mu);
    if (c->comm || c->ce_buf) return fail(COMPAR_E_STATE, "a world communicator is already set up");
    c->nranks = nranks;
    c->rank = rank;
    c->placer_ready = false;
    return COMPAR_OK;
}

compar_status compar_ce_export(void *ctx, int nranks, int rank, uint64_t max_b_bytes, void *blob, int len) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    if (nranks < 2 || rank < 0 || rank >= nranks || !blob || len < COMPAR_CE_BLOB_BYTES || max_b_bytes == 0)
        return fail(COMPAR_E_INVALID, "bad copy-engine broadcast arguments");
    if (c->virt) return fail(COMPAR_E_INVALID, "the copy-engine broadcast needs CUDA");
    std::lock_guard<std::mutex> lk(c->mu);
    if (c->comm || c->ce_buf) return fail(COMPAR_E_STATE, "a world communicator is already set up");
    if (!resolve_stream_memops()) return fail(COMPAR_E_CUDA, "cuStreamWaitValue32 / WriteValue32 unavailable");
    cudaSetDevice(c->device);
    cudaError_t e = cudaMalloc(&c->ce_buf, max_b_bytes);
    if (e == cudaSuccess) e = cudaMalloc(&c->ce_flags, 2 * kCeMax * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(c->ce_flags, 0, 2 * kCeMax * sizeof(uint32_t));
    cudaIpcMemHandle_t hb{}, hf{};
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hb, c->ce_buf);
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hf, c->ce_flags);
    if (e != cudaSuccess) return cuda_fail(e, "copy-engine chain buffers");
    std::memset(blob, 0, len);
    std::memcpy(blob, &hb, sizeof(hb));
    std::memcpy(static_cast<char *>(blob) + sizeof(hb), &hf, sizeof(hf));
    c->ce_cap = max_b_bytes;
    c->nranks = nranks;
    c->rank = rank;
    c->placer_ready = false;
    return COMPAR_OK;
}

compar_status compar_ce_import(void *ctx, const void *blobs, int len) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    std::lock_guard<std::mutex> lk(c->mu);
    if (!c->ce_buf) return fail(COMPAR_E_STATE, "compar_ce_export first");
    if (!blobs || len < c->nranks * COMPAR_CE_BLOB_BYTES) return fail(COMPAR_E_INVALID, "need nranks blobs");
    if (c->rank > 0) {
        const char *up = static_cast<const char *>(blobs) + static_cast<size_t>(c->rank - 1) * COMPAR_CE_BLOB_BYTES;
        cudaIpcMemHandle_t hb, hf;
        std::memcpy(&hb, up, sizeof(hb));
        std::memcpy(&hf, up + sizeof(hb), sizeof(hf));
        cudaError_t e = cudaIpcOpenMemHandle(&c->ce_up_buf, hb, cudaIpcMemLazyEnablePeerAccess);
        void *f = nullptr;
        if (e == cudaSuccess) e = cudaIpcOpenMemHandle(&f, hf, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle (upstream rank)");
        c->ce_up_flags = static_cast<uint32_t *>(f);
    }
    c->ce = true;
    return COMPAR_OK;
}

compar_status compar_stats_get(void *ctx, compar_stats *out) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    if (!out) return fail(COMPAR_E_INVALID, "NULL argument");
    std::lock_guard<std::mutex> lk(c->mu);
    *out = c->stats;
    return COMPAR_OK;
}

compar_status compar_set_reduce_hook(void *ctx, compar_reduce_fn fn, void *user) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    std::lock_guard<std::mutex> lk(c->mu);
    c->reduce_hook = fn;
    c->reduce_user = user;
    return COMPAR_OK;
}

compar_status compar_set_reduce_n_hook(void *ctx, compar_reduce_n_fn fn, void *user) {
    Ctx *c = as_ctx(ctx);
    if (!c) return fail(COMPAR_E_STATE, "not an initialised context");
    std::lock_guard<std::mutex> lk(c->mu);
    c->reduce_n_hook = fn;
    c->reduce_n_user = user;
    return COMPAR_OK;
}

compar_status compar_debug_spin(void *stream, int64_t ns) {
    cudaError_t e = launch_spin(static_cast<cudaStream_t>(stream), ns);
    return e == cudaSuccess ? COMPAR_OK : cuda_fail(e, "spin");
}

}  // extern "C"
