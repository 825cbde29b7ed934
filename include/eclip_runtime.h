/*
 * eclip_runtime.h — C-ABI of the B200 analogue of ECLIP's runtime scheduler.
 *
 * PAPER.md §IV-A "Runtime Scheduler":
 *   - "ECLIP pre-allocates seven CU-masked streams ... This approach avoids costly CU masking
 *     IOCTL calls at runtime"; "streams are created with CU increments of 15, as each
 *     Shader Engine (SE) on the GPU has exactly 15 CUs ... CUs are assigned in complete SE units"
 *     (P:221); per-worker masks that overlap as little as possible; "the 60 CU allocation is the
 *     default stream".
 *   - "It intercepts kernels and uses a lookup table to determine which CU-masked stream each
 *     kernel should use. The incoming kernel is then removed from its original stream and
 *     redirected to the selected CU-masked stream".
 *   - "A barrier packet is required when (i) the kernel has a dependency on a previous kernel
 *     from the same stream, and (ii) that previous kernel has not yet completed execution"
 *     (P:239-241); completion signals tracked per user stream.
 *
 * B200 mapping: a CU mask becomes an SM partition made of whole "groups" (the
 * SE analogue: equal SM groups from ONE split of the device by CUDA green contexts, unions of
 * groups via one resource descriptor); a CU-masked stream becomes a stream of a green context;
 * the full-size pool is a stream of the primary context (all SMs); a barrier packet becomes a
 * cudaStreamWaitEvent on the predecessor's completion event, inserted only when the predecessor
 * ran on another stream and its event has not completed yet.  The driver API is reached through
 * cudaGetDriverEntryPoint (no link-time libcuda dependency).
 *
 * Conventions are those of eclip.h: ECLIP_OK / negative ECLIP_E_* codes, eclip_last_error(),
 * caller-owned output arrays.  One eclip_rt belongs to one device.  Per-worker calls
 * (dispatch / signal) must come from one host thread per worker (the paper's "designated worker
 * thread"); different workers may call concurrently.
 */
#ifndef ECLIP_RUNTIME_H
#define ECLIP_RUNTIME_H

#include <stdint.h>

#include "eclip.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct eclip_rt eclip_rt;

typedef struct {
    int32_t device;          /* CUDA device ordinal */
    int32_t n_workers;       /* 1..8 co-located workers (one model each) */
    int32_t group_sms;       /* requested SMs per group (the SE analogue); rounded up by the driver to its
                                green-context granularity (8 on sm_90+); >= 1 */
    int32_t shared_default;  /* 1: the full-size pool is ONE primary-context stream shared by every worker
                                (the paper's default stream); 0: one full-device stream per worker */
} eclip_rt_config;

/* Pre-allocate the stream pool: one split of the device into G equal groups, and for every worker
 * w and every j = 1..G-1 a green context over groups {(s_w + t) mod G : t < j}, s_w = floor(w G / W)
 * (reading R17: the paper's 2-worker SE layout generalised as a rotation -- small pools of
 * different workers are disjoint, larger ones overlap in as few groups as the count allows), each
 * with one non-blocking stream; plus the full-size stream(s).  Pool sizes in SMs are therefore
 * {sum of j group sizes : j < G} and, last, the device's SM count.
 * Errors: ECLIP_E_INVALID_ARG (config), ECLIP_E_CUDA (no device / green contexts unsupported). */
int eclip_rt_create(const eclip_rt_config* cfg, eclip_rt** out);
void eclip_rt_free(eclip_rt* rt);

/* Pool geometry.  n_groups = G; group_sm[G] SMs of each group (may be NULL); n_sizes = G (pool
 * sizes j = 1..G-1 plus the full device); sizes[n_sizes] in SMs, ascending (may be NULL);
 * total_sms = the device's SM count (N of the planner). */
int eclip_rt_info(const eclip_rt* rt, int32_t* n_groups, int32_t* group_sm, int32_t* n_sizes, int32_t* sizes,
                  int32_t* total_sms);

/* Layout of (worker, size index j in [0, n_sizes)): group_mask = bit g set iff group g belongs to the
 * pool (all bits for the full size); stream_id = index of the stream in the pool (shared full-size
 * stream: the same id for every worker); sm_count = SMs of the pool. */
int eclip_rt_layout(const eclip_rt* rt, int32_t worker, int32_t size_index, uint32_t* group_mask,
                    int32_t* stream_id, int32_t* sm_count);

/* Install worker w's lookup table: kernel k of every request runs on the pool whose size is
 * kernel_sm[k] SMs (must be one of eclip_rt_info's sizes).  Errors: ECLIP_E_INVALID_ARG. */
int eclip_rt_set_table(eclip_rt* rt, int32_t worker, int32_t n_kernels, const int32_t* kernel_sm);

/* Redirect kernel k of worker w: *stream = the pool stream of table[k] (a cudaStream_t);
 * if the worker's previous kernel ran on another stream and its completion event has not completed
 * (cudaEventQuery), a wait on that event is enqueued on *stream first (the barrier packet)
 * and *barrier = 1, else 0.  The caller launches kernel k on *stream, then calls eclip_rt_signal.
 * kernel = 0 starts a new request (no predecessor dependency is needed after the worker observed the
 * previous request's completion; a pending predecessor still gets a barrier).
 * Errors: ECLIP_E_INVALID_ARG (no table / k out of range), ECLIP_E_CUDA. */
int eclip_rt_dispatch(eclip_rt* rt, int32_t worker, int32_t kernel, void** stream, int32_t* barrier);
/* Record the completion signal of the kernel just launched on the stream of the last dispatch. */
int eclip_rt_signal(eclip_rt* rt, int32_t worker);

/* ---- synthetic profiled kernels (measurement harness of the runtime) -------------------------
 * Kernel k of a model = ctas[k] CTAs of 256 threads, one CTA per SM at a time (large dynamic shared
 * memory), each running iters[k] dependent FP32 FMAs per thread: a knee-shaped latency-vs-SMs curve
 * (flat down to ctas[k] SMs, ~ceil(ctas/SMs) below), like the paper's kernels (Fig. 3). */
typedef struct {
    int32_t n_kernels;
    const int32_t* ctas;     /* [n_kernels] >= 1 */
    const int32_t* iters;    /* [n_kernels] >= 1 */
} eclip_rt_model;

/* Offline profiling (the paper's per-configuration latency profiles): the solo device
 * time of every kernel on every pool size (worker 0's pools, full-size stream last), median of reps
 * CUDA-event timings.  exec_ns[k * n_sizes + j]. */
int eclip_rt_profile(eclip_rt* rt, const eclip_rt_model* model, int32_t reps, double* exec_ns);

#define ECLIP_RT_RECORD 1        /* record per-kernel device timestamps + SM sets (validation) */
#define ECLIP_RT_REPARTITION 2   /* no pre-allocation: on every pool switch create a fresh green context +
                                    stream for the new size (the IOCTL repartition of Obs. 1) */

typedef struct {
    /* per worker w (arrays sized by the caller): */
    int64_t* latency_ns;     /* [W * n_requests] host wall time from a request's first dispatch to its
                                completion (cudaEventSynchronize of the last kernel) */
    /* ECLIP_RT_RECORD only (else may be NULL), per (w, request, kernel), row-major: */
    int64_t* t_start;        /* [W * n_requests * Kmax] device globaltimer (ns) at the first CTA's start */
    int64_t* t_end;          /* [W * n_requests * Kmax] at the last CTA's end */
    int32_t* stream_id;      /* [W * n_requests * Kmax] pool stream the kernel ran on (-1: repartitioned) */
    int32_t* barrier;        /* [W * n_requests * Kmax] 1 if a barrier (event wait) preceded it */
    int32_t* sm_used;        /* [W * n_requests * Kmax] distinct SMs that ran its CTAs */
    uint32_t* sm_mask;       /* [W * n_requests * Kmax * 5] bitset of those SMs (148 bits) */
    int64_t wall_ns;         /* all workers: first dispatch to last completion (host clock) */
    int64_t repartition_ns;  /* ECLIP_RT_REPARTITION: total host time spent creating partitions */
    int32_t barriers;        /* total barriers inserted */
} eclip_rt_run_out;

/* Closed-loop co-location run (P:219 one worker thread per model): every worker thread issues
 * n_requests requests of its model back to back through dispatch / launch / signal, waiting for
 * each request's completion before the next.  models[W]; Kmax = max n_kernels.  Every worker needs
 * a table (eclip_rt_set_table) covering its model's kernels. */
int eclip_rt_run(eclip_rt* rt, const eclip_rt_model* models, int32_t n_requests, int32_t flags,
                 eclip_rt_run_out* out);

#ifdef __cplusplus
}
#endif
#endif /* ECLIP_RUNTIME_H */
