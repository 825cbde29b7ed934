/*
 * eclip.h — C-ABI of the B200-native ECLIP resource-allocation planner.
 *
 * The operation is the resource-allocation optimizer of ECLIP (arXiv 2506.12598,
 * PAPER.md §IV-B "Resource Allocation Optimizer"): for every kernel group of
 * every co-located worker (one model per worker) choose one pre-allocated CU/SM pool
 * size (decision x_{k,c}, one configuration per kernel), with at most switchMax
 * configuration switches per worker and request, minimising the predicted
 * co-located execution time e_k = beta_k (1 + alpha_k), alpha_k = CUOverlap_w / N
 * (P:309), CUAverage_w / CUOverlap_w, with equal weight per worker.
 * The paper solves it offline with an ILP solver and stores a lookup table; this
 * library solves it exactly and exhaustively on the GPU.  DESIGN.md fixes every reading
 * (slowdown modes, objectives, QoS, ties) with citations; SURVEY.md §8(b) is the contract.
 *
 * Conventions
 *   - Every function returns ECLIP_OK (0) or a negative ECLIP_E_* code; eclip_last_error()
 *     returns a thread-local message for the last failure on the calling thread.
 *   - Inputs are borrowed for the duration of the call.  eclip_profiles objects are created
 *     and freed by the library, immutable after creation and safe to share between threads.
 *     All result arrays are allocated by the caller.  There is no global mutable state
 *     except the per-thread error message: calls on different threads are independent.
 *   - Times are integer nanoseconds inside the library (profile files carry decimal
 *     microseconds, rounded to the nearest ns, ties to even).
 *   - The planner never falls back to the CPU: without a usable CUDA device every planning
 *     call fails with ECLIP_E_CUDA.
 */
#ifndef ECLIP_H
#define ECLIP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status / error codes ---------------------------------------------------------- */
#define ECLIP_OK 0
#define ECLIP_INFEASIBLE 1          /* result status (not an error): no plan meets every QoS bound */
#define ECLIP_E_PARSE -1            /* profile text is not the SPEC format */
#define ECLIP_E_MISSING_CONFIG -2   /* a kernel row lacks a size column */
#define ECLIP_E_NONMONOTONE -3      /* exec time increases with CUs / is <= 0; message names model and kernel */
#define ECLIP_E_INVALID_ARG -4      /* bad problem (see eclip_problem field comments) */
#define ECLIP_E_TOO_LARGE -5        /* search space / integer ranges beyond the engine's limits */
#define ECLIP_E_CUDA -6             /* CUDA runtime failure, or no CUDA device */
#define ECLIP_E_OOM -7              /* device or host allocation failed */
#define ECLIP_E_IO -8               /* file cannot be read */

/* ---- slowdown modes (CUOverlap_w; readings in DESIGN.md §3.3) ---------------- */
#define ECLIP_EXCLUDE_SELF 0        /* sum_{w' != w} CUAverage_w'  (default) */
#define ECLIP_PAPER_AS_WRITTEN 1    /* CUAverage_w + sum_{w' != w} CUAverage_w'  (P:314 verbatim) */
#define ECLIP_EXCESS_OVER_CAPACITY 2/* max(0, sum_w' CUAverage_w' - N) */
#define ECLIP_MATRIX 3              /* sum_{w' != w} M[w][w'] CUAverage_w'  (BASELINE C3) */

/* ---- objectives ("one identically weighted objective per worker") ------------- */
#define ECLIP_SUM 0                 /* sum_w sum_{k in w} e_k  (default) */
#define ECLIP_MAX 1                 /* max_w sum_{k in w} e_k  (makespan) */
#define ECLIP_ENERGY 2              /* power x makespan, power linear in sum_w CUAverage_w / N */

/* ---- engines ------------------------------------------------------------------------ */
#define ECLIP_ENGINE_AUTO 0
#define ECLIP_ENGINE_ENUM 1         /* level-tuple enumeration: every candidate is classified exactly (QoS range
                                       cuts, branch-and-bound lower bounds) and the rest scored */
#define ECLIP_ENGINE_SLICE 2        /* exact T'-sliced DP (linear slowdown modes only) */
#define ECLIP_ENGINE_BASELINE 3     /* result of eclip_baseline_plan (a fixed comparison plan, no search) */

/* ---- comparison planners (eclip_baseline_plan) ----------------------------------------- */
#define ECLIP_BASELINE_ALL_MAX 0     /* every group at the worker's largest allowed size ("Baseline") */
#define ECLIP_BASELINE_MODEL_WISE 1  /* one size per model (Model-Wise right-sizing) */
#define ECLIP_BASELINE_KERNEL_WISE 2 /* every group at its minimum-CU threshold (KW) */

/* ---- profiles ------------------------------------------------------------------------ */
typedef struct eclip_profiles eclip_profiles;

/* Parse a profile file (SPEC "External Interfaces"): per model a JSON header
 * line {"model": name, "kernels": N, "configs": [c_0, ..., c_{C-1}]} followed by N CSV rows
 * "kernel_id, t_0, ..., t_{C-1}" in decimal microseconds; several models may follow each
 * other.  All models of one profiles object must share the same ascending size list.
 * Errors: ECLIP_E_IO, ECLIP_E_PARSE, ECLIP_E_MISSING_CONFIG, ECLIP_E_NONMONOTONE. */
int eclip_load_profiles(const char* path, eclip_profiles** out);
int eclip_load_profiles_mem(const char* text, size_t len, eclip_profiles** out);

/* Build from arrays: model m has n_kernels[m] kernels; exec_ns holds, model after model,
 * n_kernels[m] rows of n_sizes integer-ns times; sizes_sm ascending (SM or CU counts). */
int eclip_profiles_from_arrays(int32_t n_models, const int32_t* n_kernels, int32_t n_sizes,
                               const int32_t* sizes_sm, const int64_t* exec_ns, eclip_profiles** out);
void eclip_free_profiles(eclip_profiles* p);

/* Introspection: number of models and sizes; copies of sizes [n_sizes], kernel counts
 * [n_models] and exec times (same layout as eclip_profiles_from_arrays) when non-NULL. */
int eclip_profiles_info(const eclip_profiles* p, int32_t* n_models, int32_t* n_sizes,
                        int32_t* sizes_sm, int32_t* n_kernels, int64_t* exec_ns, char* names, size_t names_cap);

const char* eclip_last_error(void);
const char* eclip_version(void);

/* ---- one planning problem (one co-location mix) ------------------------------------- */
typedef struct {
    int32_t n_models;             /* W >= 1 workers (<= 16; ENUM <= 8) */
    const int32_t* model_ids;     /* [W] indices into the profiles (repeats allowed: P:378 Mix 1 = 2x albert) */
    const int32_t* group_bounds;  /* NULL => one group per kernel (the paper's formulation).  Else, for each
                                     worker w in order, G_w+1 ascending kernel offsets 0 = b_0 < ... < b_G = K_w
                                     (concatenated).  Group g = kernels [b_g, b_{g+1}); beta_g = sum of its
                                     kernels' times; switches are counted between groups. */
    int32_t total_sms;            /* N: total CUs/SMs (60 for MI50-shaped, 148 for B200-shaped); sizes must be <= N */
    const uint32_t* allowed_mask; /* [W] bitmask over size columns (pool layouts); NULL => all sizes */
    const double* qos_ns;         /* [W] latency bound Q_w on sum_{k in w} e_k (inclusive); NULL or +inf => none */
    int32_t switch_max;           /* R >= 0 switches per worker per request (the paper uses 14) */
    int32_t slowdown;             /* ECLIP_EXCLUDE_SELF | ECLIP_PAPER_AS_WRITTEN | ECLIP_EXCESS_OVER_CAPACITY | ECLIP_MATRIX */
    const float* slowdown_matrix; /* [W*W] row-major, entries >= 0 (MATRIX only; diagonal ignored) */
    int32_t objective;            /* ECLIP_SUM | ECLIP_MAX | ECLIP_ENERGY */
    float p_idle_w, p_max_w;      /* power model, 0 <= p_idle <= p_max (75 / 225 W) */
    const double* weights;        /* [W] per-worker objective weights omega_w in (0, 1000] ("weights:
                                     per-worker scalar (default all 1)"), or NULL = all 1, the paper's "identically
                                     weighted objective function per worker".  SUM minimises
                                     sum_w omega_w L_w, MAX minimises max_w omega_w L_w; each weight is taken at 1e-6
                                     resolution, round(omega 1e6) / 1e6 (R20).  ENERGY: weights must be
                                     equal (energy is physical).  Errors: ECLIP_E_INVALID_ARG. */
} eclip_problem;

/* Result of one problem.  Arrays are caller-allocated and may be NULL when not wanted:
 * group_sm / group_latency_ns need sum_w G_w entries, the per-worker arrays W entries. */
typedef struct {
    int32_t status;               /* ECLIP_OK or ECLIP_INFEASIBLE */
    int32_t engine_used;          /* ECLIP_ENGINE_ENUM | ECLIP_ENGINE_SLICE */
    int32_t* group_sm;            /* [sum G] chosen pool size per group: the lookup table */
    double* group_latency_ns;     /* [sum G] e_g = beta_g (1 + alpha_w) */
    double* model_latency_ns;     /* [W] L_w = sum_{k in w} e_k */
    int32_t* model_switches;      /* [W] switchTotal_w */
    int32_t* winner_levels;       /* [W] canonical level rank per worker */
    double objective;             /* SUM / MAX: ns;  ENERGY: W*ns (= nJ) */
    double makespan_ns;           /* max_w L_w */
    double power_w;               /* p_idle + (p_max - p_idle) min(1, sum_w CUAverage_w / N) */
    double energy_j;              /* power x makespan */
    double throughput_rps;        /* sum_w 1e9 / L_w (each worker back to back) */
    uint64_t winner_index;        /* mixed-radix index of the winning level tuple (worker 0 most significant);
                                     UINT64_MAX when prod_w L_w exceeds 2^64 (winner_levels is always exact) */
    uint64_t candidates;          /* level tuples in the search space (prod_w L_w; UINT64_MAX if >= 2^64) */
    uint64_t units_scored;        /* ENUM: level tuples covered (= candidates: each one classified exactly or scored);
                                     SLICE: lattice points evaluated */
    uint64_t candidates_evaluated;/* ENUM: tuples whose FP32 key pass 1 actually computed (the rest were classified
                                     without arithmetic: QoS range cuts, lower bounds); SLICE: 0 */
    uint64_t exact_key[4];        /* the winner's exact integer key, little-endian limbs */
    double energy_busy_j;         /* busy-SM energy integral of the plan's predicted run (SPEC integrate_energy
                                     S:416-419 with power_at S:406-409; R21): workers start together and
                                     run their groups back to back (group g for e_g on its pool size), power
                                     p_idle + (p_max - p_idle) min(N, sum of running pool sizes) / N, integrated over
                                     [0, makespan] (J) */
} eclip_result;

typedef struct {
    int32_t engine;               /* ECLIP_ENGINE_AUTO (default) | ENUM | SLICE */
    int32_t device;               /* CUDA device ordinal (default 0) */
    void* cuda_stream;            /* cudaStream_t to run on (NULL => the library's own stream) */
    double tie_tol;               /* tau: ties within key <= m (1 + tau) go to the lowest index (default 1e-5) */
    int32_t shard, n_shards;      /* candidate-space shard of this call (default 0 / 1); see eclip_session_* */
    int32_t no_prune;             /* ENUM, SUM, linear modes, W >= 3: 0 (default) = skip rows of candidates whose
                                     proven lower bound exceeds the tolerance band of the best key found so far
                                     (same answer); 1 = score every QoS-feasible candidate */
    int32_t timing;               /* eclip_planner_create: 1 = record CUDA events around every phase of each plan
                                     (eclip_planner_phase_ms); default 0 */
    void* comm;                   /* eclip_comm* (below) or NULL: shard eclip_plan / eclip_plan_batch over the
                                     communicator's ranks (shard = rank, n_shards = size, device = its device) with
                                     the exchanges inside the library; every rank returns the same result */
} eclip_options;

void eclip_default_options(eclip_options* o);

/* Plan one problem.  Every level tuple is covered on the GPU: ENUM classifies each one exactly
 * (infeasible by exact QoS range cuts, provably outside the tolerance band by exact lower bounds,
 * DESIGN.md §3.9) and scores the rest; SLICE covers them with the exact T'-slice DP.  The winner is the lowest-index tuple whose exact key is within (1+tau) of the exact
 * minimum.  Errors: ECLIP_E_INVALID_ARG, ECLIP_E_TOO_LARGE, ECLIP_E_CUDA, ECLIP_E_OOM. */
int eclip_plan(const eclip_profiles* prof, const eclip_problem* problem, const eclip_options* opt,
               eclip_result* result);

/* Plan many independent problems in one launch sequence (serving-loop replanning, BASELINE
 * config 5).  All problems must share W, total_sms, switch_max, slowdown, objective, power
 * model and group layout; model_ids / qos / masks / matrices differ per problem. */
typedef struct {
    int32_t n_problems;
    int32_t n_models;             /* W, same for every problem */
    const int32_t* model_ids;     /* [n_problems * W] */
    const double* qos_ns;         /* [n_problems * W] or NULL */
    const uint32_t* allowed_mask; /* [n_models_in_profiles] per-model mask, or NULL => all sizes */
    const float* slowdown_matrix; /* [n_problems * W * W] (MATRIX only) */
    int32_t total_sms, switch_max, slowdown, objective;
    float p_idle_w, p_max_w;
    int32_t on_device;            /* 0: the arrays above and below are host memory.
                                     1: model_ids, qos_ns, slowdown_matrix and every eclip_batch_out array are
                                     CUDA device pointers; the call then performs no host<->device copy of
                                     per-problem data and does not synchronise the stream before returning. */
    const double* weights;        /* [n_problems * W] per-worker objective weights (as eclip_problem.weights), or
                                     NULL = all 1 (host or device memory per on_device) */
} eclip_batch;

typedef struct {                  /* struct-of-arrays results, caller-allocated (host or device per on_device) */
    int32_t* status;              /* [n] */
    int32_t* winner_levels;       /* [n * W] */
    uint64_t* winner_index;       /* [n] */
    double* objective;            /* [n] */
    double* makespan_ns;          /* [n] */
    double* power_w;              /* [n] */
    double* energy_j;             /* [n] */
    double* throughput_rps;       /* [n] */
    double* model_latency_ns;     /* [n * W] */
    int32_t* model_switches;      /* [n * W] */
    int32_t* group_sm;            /* [n * W * Gmax] (row of worker w at (i*W + w)*Gmax; unused tail = 0), or NULL */
    int32_t group_stride;         /* Gmax used for group_sm */
    double* energy_busy_j;        /* [n] busy-SM energy integral of the predicted run (eclip_result.energy_busy_j),
                                     or NULL */
} eclip_batch_out;

int eclip_plan_batch(const eclip_profiles* prof, const eclip_batch* batch, const eclip_options* opt,
                     eclip_batch_out* out);

/* ---- persistent planner (serving-loop replanning, BASELINE config 5) --------------------
 * A co-location mix's candidates are built from per-model level tables that depend only on the
 * profiles, the allowed sizes and the switch budget — the paper's runtime "simply references"
 * precomputed results.  A planner builds those tables once (K1, per-table hulls; the only
 * host synchronisation of its life), keeps device workspaces for up to max_problems mixes, and then
 * plans batch after batch running only the per-mix work (staging, pass 1, pass 2, materialise).
 *   eclip_planner_create(prof, shape, max_problems, opt, &pl)
 *       shape: an eclip_batch whose n_models, total_sms, switch_max, slowdown, objective, p_idle_w,
 *       p_max_w and allowed_mask fix the planner; shape->qos_ns != NULL declares that every batch
 *       carries QoS bounds (the array is not read); model_ids / n_problems / on_device are ignored.
 *       opt: engine AUTO or ENUM, n_shards 1; opt->cuda_stream = the stream every plan runs on
 *       (NULL: the planner's own stream).
 *   eclip_planner_plan(pl, batch, out)
 *       batch: n_problems in [1, max_problems], model_ids, qos_ns (NULL iff the shape had none),
 *       slowdown_matrix (MATRIX) and on_device as for eclip_plan_batch; every other field must equal
 *       the shape's.  Host batches are copied into the planner's device buffers on its stream, host
 *       results copied back, and the call synchronises.  Device batches with device outputs
 *       (on_device = 1) perform no copy and, on a caller's stream, no synchronisation.  Results are
 *       identical to eclip_plan_batch's.  Errors: ECLIP_E_INVALID_ARG, ECLIP_E_TOO_LARGE,
 *       ECLIP_E_CUDA, ECLIP_E_OOM.
 *   eclip_planner_phase_ms(pl, ms, n)  needs opt->timing = 1 at creation: CUDA-event times (ms) of the
 *       last plan's phases, ms[0..5): [0] input H2D copies, [1] per-mix staging (k_prep_prob, k_prep_lev,
 *       k_prep_aux), [2] pass 1 (row bounds, pruned scoring, reduction), [3] pass 2 (exact band re-check
 *       and tie-break), [4] materialise (+ result D2H copies); waits for the last event.
 *   eclip_planner_counters(pl, out, n)  the pass-1 counters of eclip_session_counters for the last plan.
 * A planner is not thread-safe: one planner per host thread / stream. */
typedef struct eclip_planner eclip_planner;
int eclip_planner_create(const eclip_profiles* prof, const eclip_batch* shape, int32_t max_problems,
                         const eclip_options* opt, eclip_planner** out);
int eclip_planner_plan(eclip_planner* pl, const eclip_batch* batch, eclip_batch_out* out);
int eclip_planner_phase_ms(eclip_planner* pl, float* ms, int32_t n);
int eclip_planner_counters(eclip_planner* pl, uint64_t* out, int32_t n);
void eclip_planner_free(eclip_planner* pl);

/* ---- multi-GPU inside the library (SURVEY §8(b) nccl_comm, §8(e)) ------------------------
 * One process per GPU.  A sharded plan (rank r scores shard r of every problem's candidate space:
 * ENUM a contiguous range of pass-1 items, SLICE the T' slices = r mod size) needs three per-problem
 * exchanges ("minimize" over all workers' joint plans = one global arg-min): the FP32 filter
 * minima (MIN), the exact 256-bit minimum key and the lowest qualifying level tuple (lexicographic
 * MIN; the tuple's packed order is the candidate-index order).  With options.comm the library runs
 * them itself: an NCCL all-gather of the per-rank values on the planning stream plus an on-device
 * reduction kernel on every rank — no host round trip.
 *   eclip_comm_unique_id(id[128])   rank 0: a new NCCL unique id; the caller broadcasts the 128 bytes
 *                                   to the other ranks (e.g. torch.distributed.broadcast_object_list).
 *   eclip_comm_create(id, n_ranks, rank, device, &c)   collective over the n_ranks processes.
 *   eclip_comm_create_local(n_ranks, device, comms[n_ranks])   n linked communicators in ONE process on
 *                                   one device (testing the sharded protocol on one GPU: drive rank r's
 *                                   plan call from its own host thread; the exchange is device copies).
 *   eclip_comm_info / eclip_comm_free.
 * NCCL is loaded at run time (dlopen libnccl.so.2, reusing the one already in the process).
 * Errors: ECLIP_E_INVALID_ARG, ECLIP_E_CUDA (no device / NCCL failure), ECLIP_E_OOM. */
typedef struct eclip_comm eclip_comm;
int eclip_comm_unique_id(uint8_t* id);
int eclip_comm_create(const uint8_t* id, int32_t n_ranks, int32_t rank, int32_t device, eclip_comm** out);
int eclip_comm_create_local(int32_t n_ranks, int32_t device, eclip_comm** comms);
int eclip_comm_info(const eclip_comm* c, int32_t* rank, int32_t* size, int32_t* device);
void eclip_comm_free(eclip_comm* c);

/* ---- split API for multi-GPU / process-group runs -------------------------------------
 * A session plans a batch (n_problems >= 1) restricted to candidate shard opt->shard of
 * opt->n_shards.  Between the steps the caller combines per-problem values across shards:
 *   pass1      -> float m[n]        : combine with MIN
 *   pass2_min  -> uint64 key[4n]    : combine with lexicographic MIN on (key[3],key[2],key[1],key[0])
 *   pass2_first-> uint64 tuple[4n]  : the lowest qualifying level tuple, packed as a 256-bit integer
 *                                     sum_w l_w << 16(15-w) (little-endian limbs); combine with the same
 *                                     lexicographic MIN as pass2_min (all-ones = none in this shard)
 * then finish() materialises the results (identical on every shard).  All buffers are host
 * memory.  eclip_plan / eclip_plan_batch are exactly session(shard 0 of 1) + these steps. */
typedef struct eclip_session eclip_session;
int eclip_session_create(const eclip_profiles* prof, const eclip_batch* batch, const eclip_options* opt,
                         eclip_session** out);
int eclip_session_pass1(eclip_session* s, float* min_key32);
int eclip_session_pass2_min(eclip_session* s, const float* global_min_key32, uint64_t* exact_min);
int eclip_session_pass2_first(eclip_session* s, const uint64_t* global_exact_min, uint64_t* first_tuple);
int eclip_session_finish(eclip_session* s, const uint64_t* global_first_tuple, eclip_batch_out* out);
void eclip_session_free(eclip_session* s);
/* Counters of the last pass 1 of this session: candidates whose FP32 key was evaluated
 * (QoS-feasible; the others are classified infeasible by exact range cuts without
 * arithmetic) — used by bench.py to report the roofline on the work actually done. */
int eclip_session_stats(eclip_session* s, uint64_t* evaluated_candidates);
/* All pass-1 counters of this session, out[0..n): [0] candidates whose FP32 key was evaluated,
 * [1] pass-1 units (rows x segments) fetched within the band of their row bound under row pruning (0 when
 * pruning is off; the rest were proven outside the tolerance band by their lower bound),
 * [2] device time in ns of the last launch of the dominant pass-1 kernel (k_pass1_fast or
 * k_pass1_gen), from CUDA events recorded around it on the launching stream (0 for SLICE),
 * [3] pruned pass 1: units in which at least one step entry survived the chunk / entry bounds and
 * was swept, [4] entries swept, [5] units that passed the exact QoS range cut and the unit bound,
 * [6] units with at least one step chunk kept by the chunk bound, [7] chunks kept.
 * Entries beyond the defined ones are set to 0.  Errors: ECLIP_E_INVALID_ARG, ECLIP_E_CUDA. */
int eclip_session_counters(eclip_session* s, uint64_t* out, int32_t n);

/* Single-problem sessions (the per-worker masks / groups of eclip_problem; used to shard
 * one large problem, e.g. BASELINE config 4, across GPUs).  Same steps as above with
 * n = 1; finish_problem fills an eclip_result exactly like eclip_plan. */
int eclip_session_create_problem(const eclip_profiles* prof, const eclip_problem* problem,
                                 const eclip_options* opt, eclip_session** out);
int eclip_session_finish_problem(eclip_session* s, const uint64_t* global_first_tuple, eclip_result* result);

/* ---- level-1 tables (introspection) --------------------------------
 * eclip_level_table: the level table K1 builds on the GPU for ONE worker — model `model` of the
 * profiles with kernel groups `group_bounds` (NULL => one group per kernel; else G+1 ascending
 * kernel offsets 0 = b_0 < ... < b_G = K), allowed size columns `allowed_mask` (0 => all) and
 * switch budget R >= 0.  For every attained CU-sum S (SMs): B*(S) = the minimum solo
 * time sum_g beta_g (ns) over plans with <= R switches and the canonical witness (lexicographically
 * smallest size-column sequence among the minimisers), levels in witness (rank) order — the
 * candidate order of eclip_plan.  Outputs (caller-allocated host arrays, `cap`
 * levels): S[cap] int64, B[cap] int64, witness[cap * G] uint8 size columns (level-major);
 * *n_levels receives L (if L > cap nothing is copied and ECLIP_E_INVALID_ARG is returned with
 * *n_levels = L, so a call with cap = 0 queries L).  *n_groups (optional) receives G.
 * Errors: ECLIP_E_INVALID_ARG, ECLIP_E_TOO_LARGE, ECLIP_E_CUDA, ECLIP_E_OOM. */
int eclip_level_table(const eclip_profiles* prof, int32_t model, const int32_t* group_bounds, uint32_t allowed_mask,
                      int32_t switch_max, const eclip_options* opt, int32_t cap, int64_t* S, int64_t* B,
                      uint8_t* witness, int32_t* n_levels, int32_t* n_groups);

/* ---- comparison planners and the lookup table -----------------------
 * eclip_baseline_plan: the paper's comparison plans (§V), evaluated on the GPU with
 * the same model as eclip_plan (slowdown mode, objective, power, exact QoS check):
 *   ECLIP_BASELINE_ALL_MAX     param ignored
 *   ECLIP_BASELINE_MODEL_WISE  param = latency factor f >= 1 (the paper's 3x): the smallest
 *                              allowed size c with sum_g beta_g(c) <= f sum_g beta_g(c_max)
 *   ECLIP_BASELINE_KERNEL_WISE param = tolerance t >= 0 (SPEC default 0.05): per group the
 *                              smallest allowed size c with beta_g(c) <= (1 + t) beta_g(c_max)
 * f and t are taken as the rationals round(x 1e9) / 1e9 and compared exactly.  The switch budget
 * is NOT enforced (the baselines do not have one; model_switches reports what the plan uses).
 * result: status ECLIP_OK, or ECLIP_INFEASIBLE when the plan violates a QoS bound (every other
 * field still describes the plan); engine_used = ECLIP_ENGINE_BASELINE; winner_levels = -1;
 * winner_index = UINT64_MAX; candidates = units_scored = 1; candidates_evaluated = 0; exact_key = 0.
 * Errors: as eclip_plan (ECLIP_E_INVALID_ARG for an unknown kind / out-of-range param). */
int eclip_baseline_plan(const eclip_profiles* prof, const eclip_problem* problem, int32_t kind, double param,
                        const eclip_options* opt, eclip_result* result);

/* Serialize a plan as the lookup table ("store the results in a lookup table"; SPEC
 * S:225-233): every (worker, kernel) -> its pool size, as the JSON text
 *   {"meta":{"hash":"0x<16 hex>","mode":"exclude_self|paper|excess|matrix","switch_max":R},
 *    "workers":[{"worker_id":w,"configs":[c_0,...,c_{K_w-1}]},...]}
 * (no whitespace).  hash = 64-bit FNV-1a over the same text without the "hash" member.
 * group_sm: [sum_w G_w] sizes per group (eclip_result.group_sm); problem gives the workers,
 * models and group bounds.  buf may be NULL to query the length; *len receives the text length
 * (excluding the terminating NUL); buf must hold len + 1 bytes.  Host-only (no GPU work).
 * Errors: ECLIP_E_INVALID_ARG. */
int eclip_lookup_table_json(const eclip_profiles* prof, const eclip_problem* problem, const int32_t* group_sm,
                            char* buf, size_t cap, size_t* len, uint64_t* hash);

/* ---- batched co-location simulator (SPEC simulator + metrics S:266-430) ----
 * Evaluates lookup tables (plans) by simulating co-located execution, many scenarios per launch
 * (one GPU thread per scenario; the event loop of one scenario is serial and deterministic).
 * Per scenario: W workers run n_requests requests each, closed loop (R19); kernel k of
 * worker w runs on pool table[k] (a set of SM groups, mask[w][j]; j = n_sizes-1 is the full device =
 * the default stream, one FIFO shared by every worker when shared_default); kernel
 * k waits for kernel k-1 plus, in ECLIP_SIM_PREALLOC mode, barrier_ns when it changes
 * stream, or in ECLIP_SIM_IOCTL mode a repartition cost ~ triangular(lo, mode, hi) when
 * it changes pool size (SplitMix64 counter-based draws keyed by (seed, scenario,
 * worker, request, kernel)); it runs beta x oversub ns of solo work at rate 1/(1 + alpha(t)),
 * alpha = sum over co-running kernels of shared SMs / N.  Outputs: throughput
 * (requests / the worker's finish time), nearest-rank p95 and mean request latency, makespan,
 * energy = integral of p_idle + (p_max - p_idle) busy/N over [0, makespan], requests/J.
 * All arrays are host memory, row-major, caller-owned. */
#define ECLIP_SIM_PREALLOC 0
#define ECLIP_SIM_IOCTL 1
typedef struct {
    int32_t n_scenarios;      /* S >= 1 */
    int32_t n_workers;        /* W in [1, 8] */
    int32_t max_kernels;      /* K >= 1 (row stride of beta_ns / table) */
    int32_t n_sizes;          /* C in [1, 32]; pool C-1 is the full device */
    int32_t n_groups;         /* G in [1, 32] */
    const int32_t* n_kernels; /* [S*W] kernels per request, in [1, K] */
    const double* beta_ns;    /* [S*W*K*C] solo time (ns, finite, > 0) of kernel k on pool j */
    const int32_t* table;     /* [S*W*K] pool index per kernel (the lookup table) */
    const uint32_t* mask;     /* [W*C] group bitset of worker w's pool j (bits < G) */
    const int32_t* group_sm;  /* [G] SMs per group (>= 0; include any remainder group in the full mask) */
    int32_t total_sms;        /* N >= 1 */
    int32_t n_requests;       /* per worker, in [1, 4096] */
    int32_t shared_default;   /* 1: pool C-1 is ONE stream shared by every worker (FIFO) */
    int32_t mode;             /* ECLIP_SIM_PREALLOC | ECLIP_SIM_IOCTL */
    double barrier_ns;        /* PREALLOC: delay of a kernel that changes stream */
    double ioctl_lo_ns, ioctl_mode_ns, ioctl_hi_ns;  /* IOCTL: triangular repartition cost */
    double oversub;           /* >= 1: queue-oversubscription multiplier */
    double p_idle_w, p_max_w; /* 0 <= p_idle <= p_max */
    uint64_t seed;
} eclip_sim_batch;
typedef struct {
    double* throughput_rps;   /* [S*W] */
    double* p95_ns;           /* [S*W] */
    double* mean_ns;          /* [S*W] */
    double* makespan_ns;      /* [S] */
    double* energy_j;         /* [S] */
    double* req_per_j;        /* [S] */
    int32_t* barriers;        /* [S] barriers inserted (PREALLOC) */
    int64_t* events;          /* [S] kernel completions simulated */
} eclip_sim_out;
/* opt: device (other fields ignored; NULL = device 0).  Errors: ECLIP_E_INVALID_ARG, ECLIP_E_CUDA,
 * ECLIP_E_OOM. */
int eclip_simulate(const eclip_sim_batch* batch, const eclip_options* opt, eclip_sim_out* out);

#ifdef __cplusplus
}
#endif
#endif /* ECLIP_H */
