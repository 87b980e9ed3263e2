/*
 * compar.h — C ABI of the B200-native COMPAR GEMM component runtime (libcompar.so).
 *
 * What the library is (PAPER.md = /root/reference/PAPER.md, "P:n [§x]"):
 *   * one INTERFACE, "gemm":  C_out = alpha * A * B + beta * C_in  — the paper's
 *     matrix-multiply component (P:76-80 [§2.1]; P:201-205 [Table 2, "Matrix
 *     multiply: BLAS, OMP, CUDA, CUBLAS"]) read with xGEMM semantics
 *     (BASELINE.json north_star; reading R1);
 *   * several IMPLEMENTATION VARIANTS of it, registered in an ordered registry
 *     (P:56-60 [§2.1, method_declare: interface/target/name]; P:118 [§2.2.2,
 *     "a codelet ... corresponds to a variant implementation"]);
 *   * TASKS: each submit creates a task whose variant is chosen at run time by a
 *     history-based performance model (P:118, P:224 [§3.2]);
 *   * lifecycle calls compar_init / compar_terminate (P:89-91 [§2.1]).
 * No GPU work happens outside the library's own CUDA kernels; torch (or any
 * caller) only supplies device memory, streams and process groups.
 *
 * Conventions for every call:
 *   * All functions return compar_status; nothing throws across the ABI.
 *     On failure a thread-local message is available from compar_last_error().
 *   * All matrices are ROW-MAJOR with explicit leading dimensions in ELEMENTS:
 *       A: m x k (lda >= k);  B: k x n (ldb >= n) or, with transB, stored n x k
 *       (ldb >= k);  C_in, C_out: m x n FP32 (ldc >= n).  (R2)
 *   * A and B are FP32 (in_dtype = COMPAR_F32) or BF16 bit patterns
 *     (COMPAR_BF16); C is always FP32 (R5).
 *   * OWNERSHIP: the caller owns A, B, C_in, C_out (and, in SPMD mode, its panels
 *     and optional B replica).  They must stay allocated and unmodified (C_out
 *     unread) until compar_sync() on that task returns — the analogue of StarPU's
 *     "unregister after wait".  The library owns its workspaces: events,
 *     streams, TMA descriptors, B replica caches, host-mode staging buffers, the
 *     NCCL communicator and the history.
 *   * ORDER: work submitted on one stream executes in submission order.
 */
#ifndef COMPAR_H
#define COMPAR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    COMPAR_OK = 0,
    COMPAR_E_INVALID = 1,       /* bad argument: negative dim, short ld, NULL where read, bad enum   */
    COMPAR_E_STATE = 2,         /* not initialised / double init / call after terminate / no comm    */
    COMPAR_E_DUPLICATE = 3,     /* variant name already registered for the interface                  */
    COMPAR_E_NO_VARIANT = 4,    /* eligible set E is empty (SPEC S:357 SubmitError)                   */
    COMPAR_E_CUDA = 5,          /* a CUDA runtime/driver call failed (message has the CUDA string)    */
    COMPAR_E_NCCL = 6,          /* an NCCL call failed                                                */
    COMPAR_E_TASK_FAILED = 7,   /* the variant returned an error; no retry               */
    COMPAR_E_UNKNOWN_TASK = 8,  /* task id never issued or already synced                            */
    COMPAR_E_IO = 9,            /* perf-model file cannot be opened/written                           */
    COMPAR_E_FORMAT = 10,       /* perf-model file malformed; message carries the line number        */
    COMPAR_E_OOM = 11           /* device or host allocation failed                                   */
} compar_status;

typedef enum { COMPAR_F32 = 0, COMPAR_BF16 = 1 } compar_dtype;             /* storage type of A, B */

/* Arithmetic the caller accepts (precision class, R4):
 *   F32_STRICT: FP32 FFMA only  -> eligible targets SIMT_F32, TMA_F32
 *   TF32:       FP32 storage, TF32 tensor cores allowed -> SIMT_F32, TMA_F32, TC_TF32
 *   BF16:       BF16 storage (in_dtype must be BF16)    -> TC_BF16 (+ pair forms), SIMT_BF16
 *   F32_SPLIT:  FP32 storage, FP32 accuracy for finite inputs (every element inside the FP32
 *               dot-product error bound, R38) -> SIMT_F32, TMA_F32, TCX_F32 (three
 *               TF32 tensor-core products per FP32 product).  Unlike F32_STRICT it does not
 *               promise IEEE FFMA semantics: a non-finite A / B entry may turn an FP32 +-inf
 *               result into NaN (the hi*lo cross terms multiply it by zero).
 * The tcgen05 and TMA targets further require the TMA alignment rule (16-byte aligned bases and
 * row pitches); SIMT_F32 / SIMT_BF16 accept any shape and alignment, so every valid descriptor
 * has at least one eligible built-in.                                                        */
typedef enum {
    COMPAR_COMPUTE_F32_STRICT = 0,
    COMPAR_COMPUTE_TF32 = 1,
    COMPAR_COMPUTE_BF16 = 2,
    COMPAR_COMPUTE_F32_SPLIT = 3
} compar_compute;

/* Target of a variant (the paper's `target` clause).  USER variants are
 * caller-supplied launch functions, eligible for every dtype/compute. */
typedef enum {
    COMPAR_TGT_SIMT_F32 = 0,    /* built-in (a): SMEM-tiled FP32 FFMA, float4 loads             */
    COMPAR_TGT_TMA_F32 = 1,     /* built-in (b): TMA + mbarrier pipeline, FP32 FFMA             */
    COMPAR_TGT_TC_TF32 = 2,     /* built-in (c): tcgen05/TMEM tensor cores, TF32 in, FP32 acc    */
    COMPAR_TGT_TC_BF16 = 3,     /* built-in (c): tcgen05/TMEM tensor cores, BF16 in, FP32 acc    */
    COMPAR_TGT_USER = 4,
    COMPAR_TGT_TC2_TF32 = 5,    /* built-in (c), CTA-pair form: tcgen05.mma.cta_group::2, 256x256 tiles */
    COMPAR_TGT_TC2_BF16 = 6,    /* built-in (c), CTA-pair form, BF16                                    */
    COMPAR_TGT_TCW_TF32 = 7,    /* built-in (c), wide CTA-pair form: 256x512 pair tile, 2 accumulators  */
    COMPAR_TGT_TCW_BF16 = 8,    /* built-in (c), wide CTA-pair form, BF16                               */
    COMPAR_TGT_SIMT_BF16 = 9,   /* built-in (a), BF16 operands widened to FP32, FFMA; any shape/alignment */
    COMPAR_TGT_TCS_TF32 = 10,   /* built-in (c), split-K CTA-pair form: K cut into 2..8 ranges (a function */
                                /*   of K only), partials summed in split order; small-M*N / deep-K shapes */
    COMPAR_TGT_TCS_BF16 = 11,   /* built-in (c), split-K CTA-pair form, BF16                              */
    COMPAR_TGT_TCK_TF32 = 12,   /* built-in (c), cluster split-K form: the 2 CTAs of a cluster split one  */
                                /*   1-SM tile's K (at ceil(kb/2), a function of K only) and reduce   */
                                /*   through distributed shared memory; single-wave shapes only       */
                                /*   (ceil(m/128) * ceil(n/256) <= SMs, K > one k-block)              */
    COMPAR_TGT_TCK_BF16 = 13,   /* built-in (c), cluster split-K form, BF16                               */
    COMPAR_TGT_TCX_F32 = 14,    /* built-in (c), FP32-accuracy form (class F32_SPLIT): A, B split into  */
                                /*   TF32 hi + lo in a library workspace (12 (mk + kn) bytes), one TF32 */
                                /*   tcgen05 GEMM over 3K (hi*hi + hi*lo + lo*hi) in 1024-k chunks      */
                                /*   combined by round-to-nearest epilogues; K >= 64, TMA alignment,  */
                                /*   not in host-memory tasks                                          */
    /* the "sort" interface */
    COMPAR_TGT_SORT_RADIX = 20,   /* built-in: onesweep LSD radix sort, 4 x 8-bit passes, any n      */
    COMPAR_TGT_SORT_BITONIC = 21  /* built-in: single-CTA shared-memory bitonic network, n <= 16384  */
} compar_target;

/* Why a task ran the variant it ran. */
typedef enum {
    COMPAR_MODE_WARMUP = 0,     /* calibration, first W executions of (variant,key): sample dropped */
    COMPAR_MODE_CALIB = 1,      /* calibration: least-sampled eligible variant                      */
    COMPAR_MODE_MODEL = 2,      /* model: argmin of the mean measured ns                            */
    COMPAR_MODE_EAGER = 3,      /* eager scheduler: first eligible variant, no history              */
    COMPAR_MODE_HINT = 4,       /* caller forced variant_hint; history untouched                    */
    COMPAR_MODE_NOOP = 5,       /* quick return (m==0 or n==0) or scale-only (k==0 or alpha==0)     */
    COMPAR_MODE_PREDICT = 6     /* predict scheduler: argmin of fitted-model predictions for a key
                                   this variant has no samples of yet                              */
} compar_mode;

typedef enum { COMPAR_MEM_DEVICE = 0, COMPAR_MEM_HOST = 1 } compar_mem;

#define COMPAR_TASK_ALL (~(uint64_t)0)
#define COMPAR_MAX_PANELS 8
#define COMPAR_UNIQUE_ID_BYTES 128

/* Runtime configuration.  Fill with compar_config_default() first; a field left
 * negative / NULL takes the environment variable named, else the default.
 * (SURVEY.md §5 Config; SPEC S:423 environment conventions.) */
typedef struct {
    int ngpu;                   /* GPUs driven by THIS process; must be 1 (SPMD: one process per
                                   GPU, see compar_comm_init).  <0: COMPAR_NGPU or 1.  0: E_INVALID
                                   — there is no CPU class to fall back to (R15).      */
    int device;                 /* CUDA ordinal; <0: the caller's current device                */
    int sched;                  /* 0 history, 1 eager, 2 predict (history + per-variant cost model for
                                   unseen shapes); <0: COMPAR_SCHED=history|eager|predict */
    int calib_k;                /* timed calibration samples per (variant,key); <0: COMPAR_CALIB_K or 3 */
    int calib_warmup;           /* discarded first executions per (variant,key); <0: COMPAR_CALIB_WARMUP or 1 */
    const char *perf_model_path;/* NULL: COMPAR_PERF_MODEL; if the file exists it is merged at init */
    int bcast_chunks;           /* SPMD broadcast of B in this many N-slabs; <0: COMPAR_BCAST_CHUNKS or 8 */
    int builtins;               /* <0 or 1: register simt_f32, tma_f32, tc_tf32, tc_bf16 at init */
    int virtual_clock;          /* 1: host-only mode, no CUDA call at all: USER variants report
                                   synthetic ns through their virtual_ns argument (tests) */
    int64_t variant_mask;       /* bit v set: variant v is masked (never eligible); <0: COMPAR_VARIANT_MASK or 0 */
    int calib_order;            /* calibration order over the eligible variants of an unseen key:
                                   COMPAR_CALIB_INTERLEAVED: least-seen first (v0 v1 v2 v0 v1 v2 ...,
                                   SPEC S:369); COMPAR_CALIB_BLOCKED: W + K executions of v0, then
                                   of v1, ... so every timed sample follows a run of the same
                                   variant (R19: on the power-capped B200 a sample taken
                                   right after a low-power kernel runs at boost clocks).
                                   <0: COMPAR_CALIB_ORDER=interleaved|blocked, else BLOCKED        */
    int lanes;                  /* task-parallel world: library streams (workers) per GPU; model-
                                   mode samples of lanes > 1 are not added to the history (they
                                   overlap other lanes) and calibration executions run alone.
                                   <1: COMPAR_LANES or 1                                           */
    int calib_prune;            /* calibration pruning threshold in percent (R32): a variant
                                   stops calibrating for a key once its mean, or its static lower
                                   bound (FLOPs at its class's nominal peak, compulsory bytes at
                                   nominal HBM bandwidth), exceeds calib_prune/100 x the key's best
                                   mean; blocked calibration visits variants by increasing lower
                                   bound.  0: off.  <0: COMPAR_CALIB_PRUNE or 150 */
    int bcast_ctas;             /* world mode, NCCL broadcast: the communicator's maxCTAs (NCCL
                                   config), and the SMs a GEMM overlapping a broadcast leaves free.
                                   <0: COMPAR_BCAST_CTAS or 4                                        */
    int sync_timeout_ms;        /* world-mode waits (compar_sync on a task with a collective) poll
                                   ncclCommGetAsyncError; an NCCL error, or no completion within this
                                   many ms, aborts the communicator: E_NCCL, and every later world
                                   task fails with E_NCCL (sticky).  0: no timeout.
                                   <0: COMPAR_SYNC_TIMEOUT_MS or 600000                              */
} compar_config;

enum { COMPAR_WORLD_LOCAL = 0, COMPAR_WORLD_PANELS = 1, COMPAR_WORLD_TASKS = 2 };

enum { COMPAR_CALIB_INTERLEAVED = 0, COMPAR_CALIB_BLOCKED = 1 };

/* One GEMM task.  Sizes are the FULL problem; see `world` for SPMD panels. */
typedef struct {
    int64_t m, n, k;
    float alpha, beta;          /* beta == 0: C_in is never read (BLAS rule, R3)        */
    compar_dtype in_dtype;
    compar_compute compute;
    int transB;                 /* 0: B is k x n (ldb >= n); 1: B is stored n x k (ldb >= k)     */
    const void *A;  int64_t lda;
    const void *B;  int64_t ldb;
    const float *C_in;  int64_t ldc_in;   /* may alias C_out exactly (in place)                 */
    float *C_out;       int64_t ldc_out;
    compar_mem mem;             /* HOST: A, B, C_in, C_out are host pointers (pinned for overlap);
                                   the library stages them through its own device buffers: B
                                   first, then A / C_in row chunks up and C_out chunks down on two
                                   copy streams while the GEMM runs on the previous chunk; only the
                                   n valid columns of each C_out row are written on the host (by a
                                   4-CTA copy kernel when C_out is mapped pinned memory, which
                                   leaves the H2D direction more of the link; else by the copy
                                   engine).  The task's end event follows the last D2H copy.     */
    void *stream;               /* cudaStream_t to order the task on; NULL: the CUDA legacy default
                                   stream (ordered after the caller's default-stream work)        */
    int panels;                 /* loopback row panels on this device (1..COMPAR_MAX_PANELS);
                                   0 or 1: a single launch over all m rows                       */
    int world;                  /* 1: SPMD row-panel split across the ranks of compar_comm_init.
                                   A and C_* then point at THIS rank's panel (rows
                                   [o_r, o_{r+1}) of compar_partition_rows(m, nranks)), B is read
                                   on rank 0, packed into contiguous N-slabs (geometric widths: a
                                   small first slab, doubling) and broadcast with NCCL to the other
                                   ranks; a receiver's GEMM consumes slab j as soon as it landed
                                   (one persistent launch that waits per slab on device flags, or
                                   one launch per slab).  Without a
                                   communicator world = 1 is a 1-rank world.  Combines with HOST.
                                   2 (COMPAR_WORLD_TASKS): task-parallel world:
                                   the WHOLE task runs on one worker = (rank, lane) chosen by the
                                   dmda placer (expected completion = worker ready time +
                                   predicted ns, dependencies tracked on the byte ranges of A, B,
                                   C_in (read) and C_out (written)).  Every rank submits the same
                                   task sequence with pointers to its own copies; only the owner
                                   launches, on a library lane stream that first waits for
                                   `stream`.  C_out is then valid on the owner rank only
                                   (report.rank).  compar_sync is collective in this mode (all
                                   ranks, same order).  Device memory only.                     */
    void *B_replica;            /* world mode, rank != 0: device workspace of >= k*n elements that
                                   receives B (its layout afterwards is the library's slab layout,
                                   unspecified to the caller); NULL: a library-owned buffer.  (When
                                   the packed layout needs more than k*n elements — a row pitch that
                                   TMA cannot use — the library uses its own buffer instead.)     */
    int variant_hint;           /* -1: run the selector; >= 0: force that registry index          */
    uint64_t handles[4];        /* task-parallel world: caller ids of the A, B, C_in, C_out data
                                   (StarPU-style data handles, R21); a non-zero id makes
                                   dependency tracking use that id instead of the pointer's byte
                                   range — required for rank-consistent placement when the
                                   processes' allocations differ (pointers are per process); the
                                   same id on C_in and C_out marks an in-place update.  0: range */
} compar_gemm_desc;

/* ---- the "sort" interface ----
 * "the sort function, two parameters are utilized: an array of floats and a
 * scalar integer".  sort(keys, n) rearranges keys[0..n) IN PLACE into ascending order (DESIGN.md
 * R24): FP32 in IEEE 754 totalOrder (-NaN < -Inf < ... < -0 < +0 < ... < +Inf < +NaN, so the
 * result is unique as bit patterns), or uint32 / int32.  Same registry, selector, history
 * (key = (n, key type)), tasks and reports as the GEMM interface. */
typedef enum { COMPAR_KEY_U32 = 0, COMPAR_KEY_I32 = 1, COMPAR_KEY_F32 = 2 } compar_key_type;

typedef struct {
    int64_t n;                  /* number of keys, 0 <= n < 2^30                                    */
    compar_key_type key_type;
    void *keys;                 /* device array of n 4-byte keys, sorted in place; the caller
                                   keeps it alive and unmodified until compar_sync              */
    void *stream;               /* cudaStream_t; NULL: the legacy default stream                 */
    int variant_hint;           /* -1: run the selector; >= 0: force that registry index          */
} compar_sort_desc;

/* User sort variant: sort d->keys on `stream` (virtual-clock mode: store a synthetic cost in
 * *virtual_ns and touch no CUDA). */
typedef compar_status (*compar_sort_fn)(const compar_sort_desc *d, void *stream, void *user, int64_t *virtual_ns);

/* The rows one variant launch covers (a loopback panel, or this rank's panel). */
typedef struct {
    int index;                  /* panel number r                                                  */
    int64_t row0, rows;         /* rows [row0, row0 + rows) of the full m                          */
    const void *A;              /* first row of the panel (device pointers, ld from the desc)      */
    const void *B;              /* B (or the local replica in world mode)                          */
    const float *C_in;
    float *C_out;
} compar_panel;

/* User variant: launch the panel's GEMM on `stream` and return.  In virtual-clock
 * mode `virtual_ns` is non-NULL and the function stores its synthetic cost there
 * (and must not touch CUDA); otherwise it is NULL. */
typedef compar_status (*compar_gemm_fn)(const compar_gemm_desc *d, const compar_panel *p,
                                        void *stream, void *user, int64_t *virtual_ns);

typedef struct {
    uint64_t task;
    int variant;                /* registry index that ran (-1 for NOOP)                           */
    int mode;                   /* compar_mode                                                     */
    int warmup;                 /* 1 if this execution's sample was discarded                      */
    compar_status status;
    int npanels;
    int64_t ns;                 /* the history sample: max over panels (and ranks) of kernel ns    */
    int64_t panel_ns[COMPAR_MAX_PANELS];
    int64_t bcast_ns;           /* world mode: broadcast of B, start -> last chunk landed          */
    int64_t total_ns;           /* first start event -> last stop event of the task on its stream  */
    int batch;                  /* launches timed by one event pair: a calibration execution on a
                                   key whose static cost estimate t (5 us + FLOPs at 100 TFLOP/s +
                                   compulsory bytes at 3 TB/s) is < COMPAR_CALIB_BATCH_NS (default
                                   100 us) repeats the kernel r = ceil(200 us / t) times (<= 64, the
                                   same r for every variant of the key), each launch between its
                                   own event pair, and records the median launch (SURVEY §8(a) a8 /
                                   c13, R25); the r - 1 extra launches write a library
                                   scratch C, so C_out is written once */
    int rank, lane;             /* worker that ran the task (task-parallel world); else rank, 0    */
} compar_report;

typedef struct {
    int64_t seen, count, min_ns;
    int64_t sum_ns;             /* saturating copy of the 128-bit internal sum                     */
    double mean_ns;
} compar_record;

typedef struct {
    int64_t submits, launches, harvested, failed;
    int64_t bytes_h2d, bytes_d2h;
} compar_stats;

/* ---- lifecycle (P:89-91 [§2.1]: `initialize` -> compar_init(), `terminate` -> compar_terminate()) ---- */
void          compar_config_default(compar_config *cfg);
/* E_STATE if ctx already points at a live context; E_INVALID ngpu != 1; E_CUDA if no GPU (unless
 * virtual_clock); built-in kernels are pre-loaded so lazy loading never pollutes calibration. */
compar_status compar_init(const compar_config *cfg, void **ctx);
/* Synchronises every outstanding task, frees workspaces/comms; *ctx invalid afterwards. */
compar_status compar_terminate(void *ctx);

/* ---- variants (P:56-60 method_declare interface/target/name; P:118 codelet) ---- */
/* iface must be "gemm"; name unique (E_DUPLICATE); target USER requires fn (E_INVALID);
 * built-in targets ignore fn.  *out_id = registry index = tie-break order. */
compar_status compar_register_variant(void *ctx, const char *iface, const char *name,
                                      compar_target target, compar_gemm_fn fn, void *user,
                                      int *out_id);
/* A variant of the "sort" interface: target SORT_RADIX / SORT_BITONIC (built-ins, fn ignored) or
 * USER with fn.  Same registry (indices, names, mask) as the GEMM variants. */
compar_status compar_register_sort_variant(void *ctx, const char *name, compar_target target,
                                           compar_sort_fn fn, void *user, int *out_id);
/* ---- generic interfaces (the target of the #pragma compar pre-compiler) ----
 * An interface declared with `#pragma compar method_declare interface(I) ...`: its
 * variants are user functions that enqueue GPU work on the task's stream, which they obtain with
 * compar_current_stream() while the runtime calls them (like StarPU's
 * starpu_cuda_get_local_stream).  args[i] points at the i-th interface argument; sizes[] are the
 * values of the size clauses ("size"), the history key is (I, sizes[0], sizes[1], product of
 * the rest).  Selection, calibration, history, tasks and reports are those of the GEMM interface. */
typedef compar_status (*compar_generic_fn)(void *const *args, const int64_t *sizes, int nsizes, void *user);
typedef struct {
    const char *iface;          /* interface name (variants registered under it compete)          */
    int nargs;
    void *const *args;          /* args[i]: address of the i-th argument value                     */
    int nsizes;                 /* 0..8 */
    const int64_t *sizes;
    void *stream;               /* cudaStream_t the variant's work is ordered on (NULL: default)   */
    int variant_hint;           /* -1: selector; >= 0: that registry index                          */
} compar_generic_desc;
compar_status compar_register_generic_variant(void *ctx, const char *iface, const char *name, compar_generic_fn fn,
                                              void *user, int *out_id);
compar_status compar_generic_submit(void *ctx, const compar_generic_desc *d, uint64_t *task);
/* The stream of the task whose variant the calling thread is running (NULL outside a variant). */
void *compar_current_stream(void);

compar_status compar_variant_count(void *ctx, int *n);
compar_status compar_variant_info(void *ctx, int id, char *name, int name_len, int *target);

/* ---- tasks (P:128 task create + submit) ---- */
/* Validates d (E_INVALID), selects a variant (E_NO_VARIANT), launches asynchronously and returns
 * the monotone task id.  m==0 or n==0: no launch, mode NOOP.  k==0 or alpha==0: a scale-only
 * kernel C_out = beta*C_in, mode NOOP (no history).  In model mode the submit first harvests
 * pending samples of the same key (blocking on them) so decisions are a pure function of the
 * submission sequence. */
compar_status compar_gemm_submit(void *ctx, const compar_gemm_desc *d, uint64_t *task);
/* The sort interface: validates (E_INVALID: n out of range, bad key type, NULL keys), selects
 * among the eligible sort variants (history key = (n, key type); sort_bitonic needs n <= 16384),
 * launches asynchronously.  n <= 1: no launch, mode NOOP.  Sort tasks of one context are
 * serialised with each other (they share the library's radix scratch). */
compar_status compar_sort_submit(void *ctx, const compar_sort_desc *d, uint64_t *task);
/* Blocks until the task's stop event(s); harvests its sample into the history; fills *out
 * (may be NULL).  task == COMPAR_TASK_ALL syncs every outstanding task (out gets the last).
 * A failed variant -> E_TASK_FAILED (status also in out).  After return the library holds no
 * reference to the task's buffers.  A task the selector already harvested implicitly (step 6,
 * before a decision) keeps its report until this call returns it (same status, same report).
 * World-mode tasks: the wait polls NCCL's asynchronous error state (see sync_timeout_ms). */
compar_status compar_sync(void *ctx, uint64_t task, compar_report *out);
/* Query: the (variant, mode) the next submit of d would get.  No launch, no history change.  Like
 * a submit it may first harvest (block on) pending LOCAL samples of the key — their reports stay
 * available to compar_sync — but it never harvests tasks whose harvest is collective (world
 * tasks on several ranks), so it is safe to call on one rank; with such tasks pending, the answer
 * reflects the samples harvested so far. */
compar_status compar_select(void *ctx, const compar_gemm_desc *d, int *variant, int *mode);

/* ---- performance model persistence ("additional training") ---- */
/* Text, one record per line:
 *   <variant_name> <m> <n> <k> <dtype> <compute> <transB> <beta0> <seen> <count> <sum_ns> <sumsq_ns> <min_ns>
 * Load MERGES by (variant_name, key): counts and sums add, min takes the min.  Unknown variant
 * names are kept and apply if that name is registered later. */
compar_status compar_perf_save(void *ctx, const char *path);
compar_status compar_perf_load(void *ctx, const char *path);
compar_status compar_history_get(void *ctx, int variant, const compar_gemm_desc *key_of,
                                 compar_record *out);

/* ---- partitioning and multi-GPU (north star: row panels + NCCL broadcast of B) ---- */
/* offsets[0..p]: base = ceil(ceil(m/p)/128)*128, offsets[r] = min(m, r*base), offsets[p] = m. */
compar_status compar_partition_rows(int64_t m, int p, int64_t *offsets);
/* NCCL unique id for SPMD init (rank 0 creates it, the caller distributes it, e.g. with a
 * torch.distributed broadcast); len >= COMPAR_UNIQUE_ID_BYTES. */
compar_status compar_comm_unique_id(void *out, int len);
/* Joins the nranks-process communicator (one process per GPU).  Required before world = 1. */
compar_status compar_comm_init(void *ctx, int nranks, int rank, const void *id, int len);

/* Joins an nranks-process SPMD world WITHOUT an NCCL communicator: the task-parallel world's sample
 * exchange then goes through compar_set_reduce_n_hook (and world = 1 needs compar_ce_* for B and
 * compar_set_reduce_hook).  E_STATE if a communicator is already set up. */
compar_status compar_world_init(void *ctx, int nranks, int rank);

/* Copy-engine chain broadcast of B for world = 1, instead of NCCL: slab j of B travels
 * root -> rank 1 -> ... -> rank P-1, each hop one cudaMemcpyAsync from the upstream rank's buffer
 * (CUDA IPC; NVLink between GPUs), started by a GPU-side wait (cuStreamWaitValue32) on the
 * upstream's "slab j ready" word and followed by "slab j consumed" (cuStreamWriteValue32) in the
 * upstream's flags, so the hops are pipelined slab by slab, no host round trip and no SM is used
 * (the slab GEMMs keep all SMs).  Setup, on every rank: compar_ce_export allocates the chain
 * buffer (B up to max_b_bytes) and the flag words and writes an opaque blob
 * (len >= COMPAR_CE_BLOB_BYTES); the caller all-gathers the blobs (rank-major) and passes them to
 * compar_ce_import.  Without an NCCL communicator, world-mode samples need compar_set_reduce_hook.
 * The ranks may share one GPU (separate processes), which is how the tests exercise it. */
#define COMPAR_CE_BLOB_BYTES 256
compar_status compar_ce_export(void *ctx, int nranks, int rank, uint64_t max_b_bytes, void *blob, int len);
compar_status compar_ce_import(void *ctx, const void *blobs, int len);

/* Replace the NCCL max-all-reduce that makes world-mode samples rank-consistent by a caller
 * hook (in-place max of *value over all ranks).  Used by the host-only SPMD tests (gloo) in
 * virtual-clock mode; fn = NULL restores the default. */
typedef void (*compar_reduce_fn)(int64_t *value, void *user);
compar_status compar_set_reduce_hook(void *ctx, compar_reduce_fn fn, void *user);
/* Same for the task-parallel world's sample exchange: in-place element-wise max of buf[0..n)
 * over all ranks (the owner of each task contributes its ns, the others -1). */
typedef void (*compar_reduce_n_fn)(int64_t *buf, int n, void *user);
compar_status compar_set_reduce_n_hook(void *ctx, compar_reduce_n_fn fn, void *user);

/* ---- introspection / fixtures ---- */
compar_status compar_stats_get(void *ctx, compar_stats *out);
const char   *compar_last_error(void *ctx);
/* Synthetic-cost fixture: one-thread kernel spinning on %globaltimer for ns nanoseconds on
 * `stream` (SURVEY §4 spin_ns; used by USER test variants with closed-form costs). */
compar_status compar_debug_spin(void *stream, int64_t ns);

#ifdef __cplusplus
}
#endif
#endif /* COMPAR_H */
