// engine.h — internal structures shared by the host planner (api.cpp) and the CUDA
// kernels (levels.cu, enum.cu, slice.cu).  Not part of the C-ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "exact.cuh"

namespace eclip {

// host-side checkpoints for diagnosing per-call overhead: with ECLIP_HOST_TIMING set in the environment,
// host_mark("label") prints the microseconds since the last host_mark(nullptr) reset to stderr
void host_mark(const char* label);

constexpr int MAXW = 16;        // workers per problem (API limit)
constexpr int MAXW_ENUM = 8;    // workers per problem on the ENUM engine
constexpr int P1_THREADS = 256; // pass-1 CTA size
constexpr int KIN = 16;         // inner-worker levels held in registers per thread (fast pass 1)
constexpr int P1_CS = 4;        // step-level chunk of the pass-1 chunk filter
#ifndef P1_TABN_N
#define P1_TABN_N 6144
#endif
constexpr int P1_TABN = P1_TABN_N;   // entries of each QoS range lookup table (fast pass 1)
// hull slope tables (enum.cu hull_arg): bins of the query ratio z / y by its float bits, 8 per octave
constexpr int HT_NB = 256;
constexpr int HT_F2 = 2 * HT_NB / 8;   // the two tables (step, inner) of a problem, in float2 slots
// per-problem stride of the row-bound hull buffer (float2): [2][2][Lmax] vertices + edges, then the tables
__host__ __device__ __forceinline__ size_t hull_stride(int Lmax) { return (size_t)4 * Lmax + HT_F2; }

enum Mode { M_EXCL = 0, M_PAPER = 1, M_EXCESS = 2, M_MATRIX = 3 };

// Programmatic dependent launch (sm_90+): kernels of the planner's chain are launched with programmatic
// stream serialisation (launch_pdl), so a kernel's CTAs are scheduled while its predecessor's last wave
// still runs.  Every kernel so launched calls pdl_wait() before it reads anything its predecessor wrote
// (and before it exits, so that its completion implies the predecessor's), then pdl_trigger() to let its
// own successor be scheduled.  Outside such a launch both are no-ops.
// ECLIP_CHECK: device-side bounds checks of a test build (-DECLIP_BOUNDS; compute-sanitizer is not available on
// the GPU pool): a failed check prints its site and traps, so the calling test fails.  Nothing otherwise.
#ifdef ECLIP_BOUNDS
#define ECLIP_CHECK(c)                                                                                      \
    do {                                                                                                    \
        if (!(c)) {                                                                                         \
            printf("ECLIP_CHECK failed: %s (%s:%d) block %d thread %d\n", #c, __FILE__, __LINE__,          \
                   (int)blockIdx.x, (int)threadIdx.x);                                                      \
            __trap();                                                                                       \
        }                                                                                                   \
    } while (0)
#else
#define ECLIP_CHECK(c) do { } while (0)
#endif

#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, ((KArgs)args)...);
}
#endif
enum Obj { O_SUM = 0, O_MAX = 1, O_ENERGY = 2 };

// ---------------------------------------------------------------------------------------
// Level-1 DP job (one per level table; §8(a) a2, DESIGN.md §4 K1)
// ---------------------------------------------------------------------------------------
struct LevelJob {
    int32_t G, C, R;            // groups, size columns, effective switch budget min(R, G-1)
    int32_t smax;               // max level in units of u
    int64_t u;                  // gcd of the allowed sizes (SMs)
    uint32_t mask;              // allowed size columns
    int32_t Lcap;               // capacity of the outputs
    const int64_t* beta;        // [G*C] group solo times (ns)
    const int32_t* need;        // [G*C] n_g c_j / u
    int32_t ncp;                // cells (r, s) of a layer, (R+1)(smax+1), padded to a multiple of 32 (each
                                //   layer's slabs 128-byte aligned: layer data is read through L1, see levels.cu)
    void* V;                    // workspace [G][C][ncp] suffix optima (int32 when v32, else int64)
    void* best;                 // workspace [G][ncp][2]: best / second best over j, per layer
    uint8_t* barg;              // workspace [G][ncp] arg-best (255: none)
    int64_t* bstar;             // workspace [smax+1] B*(s)
    int32_t* sidx;              // workspace [smax+1] compacted level -> s
    uint64_t* wtmp;             // workspace [(smax+1) * ceil(G/8)] packed witnesses in s order
    // outputs (rank order)
    int64_t* outS;              // [Lcap] level CU-sum in SMs
    int64_t* outB;              // [Lcap] B*(S) ns
    uint8_t* outW;              // [Lcap*G] witness size columns
    int32_t* outL;              // [1]
};

// v32: every table's suffix sums fit int32 (V / best stored as int32, half the traffic of the layers)
cudaError_t launch_levels(LevelJob* d_jobs, const LevelJob* h_jobs, int n_jobs, bool v32, cudaStream_t st);

// ---------------------------------------------------------------------------------------
// Staged per-level record of one worker inside one problem (written by the prep kernel).
// ---------------------------------------------------------------------------------------
struct Lev {
    int64_t B;        // exact solo time B*(level) (ns)
    int64_t BS;       // exact B * S' (narrow problems; 0 in wide ones, where it may not fit)
    int64_t S;        // S' = S Lambda / K  (Lambda-scaled CU-sum)
    int32_t Tmax;     // largest T' at which this worker meets its QoS (linear modes, narrow problems); -1 never
    float Bk;         // (float)((double)B / (Lambda N))
};
static_assert(sizeof(Lev) == 32, "Lev must be 32 bytes");

// ---------------------------------------------------------------------------------------
// Per-problem descriptor (written by the prep kernel; read by every later kernel)
// ---------------------------------------------------------------------------------------
struct Prob {
    int32_t status;             // 0 ok, 1 infeasible, <0 ECLIP_E_* error
    int32_t W;
    int32_t table[MAXW];        // level table per worker
    int32_t L[MAXW];
    int32_t E;                  // fraction bits of the slowdown matrix (MATRIX), else 0
    int32_t k_pow;              // fraction bits of the power model
    int64_t lam, lamN;          // Lambda = lcm K_w, Lambda N
    uint64_t P;                 // prefix count prod_{w<W-1} L_w
    uint64_t total;             // prod_w L_w
    uint64_t units;             // pass-1 units = rows x nseg (see enum.cu geometry)
    uint64_t n_items;           // pass-1 CTA work items (upi units each)
    int32_t Lstep, nseg, seglen, pad0;
    float inv;                  // (float)(1 / (Lambda N))
    float lamNf;                // (float)(Lambda N)
    float p_idle, p_dyn;        // power model floats (p_dyn = fl(p_max - p_idle))
    float Qlo[MAXW], Qhi[MAXW]; // MATRIX+QoS: surely / maybe feasible float bounds on L_w
    float Mf[MAXW_ENUM * MAXW_ENUM];     // slowdown matrix (float)
    int64_t Mi[MAXW_ENUM * MAXW_ENUM];   // M 2^E (exact)
    u128 Hq[MAXW];              // floor(Q_w D) (exact QoS on h_w); all-ones = none
    u128 D;                     // Lambda N 2^E
    u128 pi_idle, pi_dyn;       // power model p 2^k (exact)
    int32_t has_qos;
    float p_max;                // power model float (for FP64 reporting)
    // per-worker objective weights (R20): wt = round(omega 1e6) / gcd (exact keys),
    // wf = (float)wt (FP32 filters), wv = round(omega 1e6) / 1e6 (FP64 objective); all 1 when unweighted
    uint64_t wt[MAXW];
    float wf[MAXW];
    double wv[MAXW];
    // representative problem of this one's step / inner-worker precomputation (fast pass 1): the aux block,
    // hulls, row-feasibility table and row-bound header depend only on (step table, inner table, their QoS
    // thresholds, Lambda, the hi workers' S' range), so problems of a batch with equal keys share the first
    // one's (k_akey / k_arep); rep == own index otherwise
    int32_t rep;
    int32_t pad_rep;
};

// Settings shared by all problems of one launch sequence
struct Setup {
    int32_t n_problems, W, N, mode, obj, has_qos;
    int32_t Lmax;               // max levels over the tables
    int32_t items_max;          // max pass-1 items over problems
    int32_t nseg;               // segments per row (units = rows x nseg)
    int32_t upi;                // units per pass-1 item (CTA)
    int64_t units_max;          // max units over problems (submin stride)
    int32_t table_bytes;        // fast pass-1 per-CTA table budget (per-warp prefix tables)
    int32_t aux_bytes;          // fast pass-1 per-problem aux block (after the Lev records)
    int32_t lev_stride;         // Lev records per problem block (W*Lmax + aux_bytes/32)
    int32_t wide;               // 1: Lambda N (W+1) may reach 2^24 (heterogeneous kernel counts): S', T' exceed
                                //    the int32 / exact-float ranges of the narrow kernels; pass 1 runs the generic
                                //    kernel with FP32 QoS bounds (maybe / surely feasible, as MATRIX), decisions
                                //    stay exact (u128 / u256) — DESIGN.md §3.10
    int32_t shard, n_shards;
    uint64_t tol_num, tol_den;
    double delta;               // FP32 filter relative error bound
    int32_t prune;              // fast pass 1: skip rows whose lower bound exceeds the incumbent's band (§3.9)
    int32_t weighted;           // per-worker objective weights given (SUM / MAX): the generic pass 1 and the
                                //   weighted FP32 / exact keys (the fast bilinear kernels assume equal weights)
    int64_t rows_max;           // max rows (hi-digit combinations) over problems (rowlb stride)
};

// QoS decided in pass 1 by FP32 bounds on L_w (maybe / surely feasible minima) instead of exact integer
// T' thresholds: the MATRIX mode, and every mode of a wide problem
__host__ __device__ __forceinline__ bool qos_float(const Setup& su) {
    return su.has_qos != 0 && (su.mode == M_MATRIX || su.wide != 0);
}
// T' bound of the narrow problems (Lambda N (W+1) < 2^24: exact in FP32 and int32)
constexpr int64_t NARROW_T = (int64_t)1 << 24;

// Device view of all level tables
struct Tables {
    int32_t n;
    const int32_t* L;           // [n]
    const int64_t* K;           // [n] kernels per table
    const int32_t* G;           // [n]
    const int64_t* const* S;    // [n] -> [L] level CU-sums (SMs)
    const int64_t* const* B;    // [n] -> [L]
    const uint8_t* const* wit;  // [n] -> [L*G]
    const int64_t* const* beta; // [n] -> [G*C]
};

struct PrepIn {
    const int32_t* table_of;    // [n*W] table id per (problem, worker)
    const double* qos;          // [n*W] or null
    const float* M;             // [n*W*W] or null
    float p_idle, p_max;
    const double* weights;      // [n*W] per-worker objective weights or null (all 1)
};

// Device-side outputs / scratch of one launch sequence
struct Work {
    Prob* probs;                // [n]
    Lev* levs;                  // [n * W * Lmax]
    float* submin;              // [n * units_max]  pass-1 minima per unit (maybe-feasible)
    float* submin_sure;         // [n * units_max]  MATRIX+QoS: surely-feasible minima
    float* m32;                 // [n] local (then global) minimum
    float* m32_sure;            // [n]
    U256* hstar;                // [n] exact minimum
    U256* first;                // [n] winner: lowest tuple within tolerance, packed (pack_tuple); all-ones = none
    uint64_t* scored;           // [n]
    unsigned long long* feasible;  // [1] QoS-feasible candidates evaluated by the fast pass 1
    // row-level bound pruning (fast pass 1, W >= 3)
    float* rowlb;               // [n * rows_max] lower bound of every exact key in the row (+inf: no feasible candidate)
    unsigned* lbmin;            // [n] min over rows of rowlb (float bits)
    unsigned* inc;              // [n] incumbent: smallest FP32 key found so far (float bits)
    float2* hull;               // [n][2][2][Lmax]: step / inner worker lower-left hull vertices {B, S'}, then its
                                //   edges {B_i - B_i+1, S'_i+1 - S'_i}
    int32_t* ftab;              // [n * FT_CAP] exact row feasibility: F(t0 + i) (see k_prep_bound)
    uint2* ulist;               // [pass-1 grid][upi] bucket-ordered candidate units of each item (k_bucket)
    int32_t* ulist_n;           // [pass-1 grid]
    struct RowHdr* rowhdr;      // [n]
    unsigned long long* rows_done;  // [1] rows (units) pass 1 actually processed
    int32_t* bandn;             // [n] units in the pass-2 band list (-1: more than BAND_CAP, rescan all)
    uint64_t* bandlist;         // [n * BAND_CAP] band units in index order (k_reduce_min)
    uint32_t* plist;            // [n * PL_CAP] units pass 1 processed with a finite minimum (pruned pass 1)
    int32_t* plist_n;           // [n] their count (> PL_CAP: overflow, reduce_min scans every unit)
    uint32_t* wbits;            // [n * ceil(units_max / 32)] pruned pass 1: units whose submin was written
                                //   (every other unit reads as +inf; replaces a +inf fill of submin)
    uint16_t* thull;            // [tables * Lmax] hull vertex levels of every level table (k_table_hull)
    int32_t* thull_n;           // [tables]
    uint16_t* tord;             // [tables * Lmax] level indices of every level table in S order (k_table_hull)
    const int32_t* table_of;    // [n * W] table of each (problem, worker) (PrepIn.table_of)
    struct AKey* akey;          // [n] the precomputation key of every problem (k_akey)
    unsigned long long* aslot;  // [2 * aslots] hash table {hash, min problem index} of the keys
    int32_t aslots;             // slot count (power of two, >= 2 n); 0: no deduplication
    Tables tb;                  // the level tables
    cudaEvent_t kev[2];         // recorded on the launching stream around the dominant pass-1 kernel (or null)
};

constexpr int FT_CAP = 8192;    // entries of the exact row-feasibility table per problem

struct AKey {                   // what a problem's step / inner-worker precomputation depends on (Prob::rep)
    int32_t tab_step, tab_inner, t0, t1;   // level tables; range of the hi workers' S' sums
    int64_t lam;
    u128 hq_step, hq_inner;                // exact QoS thresholds floor(Q D)
};
#ifndef BAND_CAP_N
#define BAND_CAP_N 1024
#endif
#ifndef PL_CAP_N
#define PL_CAP_N 4096
#endif
constexpr int BAND_CAP = BAND_CAP_N;   // pass-2 band list capacity per problem
constexpr int BAND_SORTED = 64;       // band lists up to this length are in index order (pass 2 stops at the first hit)
constexpr int PL_CAP = PL_CAP_N;       // processed-unit list capacity per problem (tiny values in test builds
                                       // exercise the overflow paths)

struct RowHdr {                 // per-problem constants of the row bound (k_prep_bound)
    int32_t nh[2];              // hull sizes (step, inner)
    int32_t smin_in, umax_in;   // inner worker: min S', max (Tmax - S')
    int32_t smin_st, umax_st;   // step worker:  min S', max (Tmax - S')
    float Sminf_in, Bminf_in;   // inner worker: (float) min S', (float) min B
    int32_t t0, tn;             // feasibility table covers hT in [t0, t0 + tn); tn = 0: no table
    int32_t htb[2];             // slope-table bases (step, inner; hull_arg)
};

// batched co-location simulator (simulate.cu)
struct SimJob {
    long long S;
    int32_t W, K, C, G, N, n_requests, shared_default, ioctl;
    const int32_t* n_kernels;   // [S*W]
    const double* beta;         // [S*W*K*C]
    const int32_t* table;       // [S*W*K]
    const uint32_t* mask;       // [W*C]
    const int32_t* group_sm;    // [G]
    double barrier_ns, io_lo, io_mode, io_hi, oversub, p_idle, p_max;
    unsigned long long seed;
};
struct SimOut {
    double *throughput_rps, *p95_ns, *mean_ns;   // [S*W]
    double *makespan_ns, *energy_j, *req_per_j;  // [S]
    int32_t* barriers;
    long long* events;
    int32_t* status;
};
cudaError_t launch_simulate(const SimJob& J, const SimOut& o, double* latbuf, cudaStream_t st);

// per-problem constants, level records and (fast pass 1) aux blocks; table_hull = also build the
// per-table S orders and hulls (k_table_hull) — a persistent planner builds those once
cudaError_t launch_prep(const Setup& su, const Tables& tb, const PrepIn& in, Work& wk, int C, const int32_t* sizes,
                        cudaStream_t st, bool table_hull = true);
cudaError_t launch_table_hull(const Setup& su, const Tables& tb, Work& wk, cudaStream_t st);
cudaError_t launch_pass1(const Setup& su, Work& wk, cudaStream_t st);
cudaError_t launch_reduce_min(const Setup& su, Work& wk, cudaStream_t st);
cudaError_t launch_pass2_min(const Setup& su, Work& wk, cudaStream_t st);
cudaError_t launch_pass2_first(const Setup& su, Work& wk, cudaStream_t st);
cudaError_t launch_pass2_both(const Setup& su, Work& wk, cudaStream_t st);   // unsharded: one rescan

struct MatOut {                 // materialisation outputs (device pointers, may be null)
    int32_t* status; int32_t* levels; uint64_t* index; double* objective; double* makespan;
    double* power; double* energy; double* thr; double* latency; int32_t* switches; int32_t* group_sm;
    double* group_lat; int32_t group_stride; uint64_t* key;
    double* energy_busy;        // [n] busy-SM energy integral of the predicted run (J; R21)
    int32_t gsum;               // >= sum over workers of the group counts (busy-energy staging)
};
cudaError_t launch_materialize(const Setup& su, const Tables& tb, Work& wk, const int32_t* sizes, int C,
                               MatOut out, cudaStream_t st);

// pass-1 dynamic shared memory for a setup (host helper)
size_t pass1_smem(const Setup& su, bool fast);
bool pass1_fast(int L_inner);
int pass1_fast_team(int L_inner);
size_t pass1_aux_bytes(int Lmax);
bool pass1_prunable(const Setup& su);


// ---- comparison planners (baseline.cu) ----
struct BaseJob {
    int32_t W, C, N, mode, obj, kind;
    uint64_t num, den;                 // tol (KERNEL_WISE) or factor (MODEL_WISE) = num / den
    float p_idle, p_max;
    const int32_t* sizes;              // [C]
    int32_t G[MAXW];
    int64_t K[MAXW];
    uint32_t mask[MAXW];
    const int64_t* exec[MAXW];         // [K_w * C] the worker's per-kernel profile rows (ns)
    const int32_t* bounds[MAXW];       // [G_w + 1] group kernel offsets
    double Q[MAXW];
    float M[MAXW_ENUM * MAXW_ENUM];
    double wv[MAXW];                   // objective weights round(omega 1e6) / 1e6 (1 = unweighted)
};

struct BaseOut {
    int32_t* status;                   // [1] 0 = meets every QoS bound, 1 = does not
    int32_t* group_sm;                 // [W * stride]
    double* group_lat;                 // [W * stride]
    int32_t stride;
    double* latency;                   // [W]
    int32_t* switches;                 // [W]
    double* scalars;                   // [5] objective, makespan, power, energy, throughput
};

cudaError_t launch_baseline(const BaseJob& j, BaseOut o, cudaStream_t st);

}  // namespace eclip

// ---- multi-GPU exchange (comm.cu; the C-ABI's eclip_comm) ----
struct eclip_comm;
namespace eclip {
int comm_min_f32(eclip_comm* c, float* buf, int n, cudaStream_t st);        // in place: global MIN (ECLIP_* code)
int comm_lexmin_u256(eclip_comm* c, U256* buf, int n, cudaStream_t st);     // in place: global lexicographic MIN
int comm_rank(const eclip_comm* c);
int comm_size(const eclip_comm* c);
int comm_device(const eclip_comm* c);

}  // namespace eclip
