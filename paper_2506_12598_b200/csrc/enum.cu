// enum.cu — the ENUM engine: every level tuple of every problem is scored on the GPU.
//
//   prep     per problem constants (Lambda, D, exact QoS bounds, power integers) and the
//            staged per-level records
//   pass 1   K2: mixed-radix enumeration (a4) + FP32 scoring (a5) + per-sub-chunk minima (a6).
//            Every candidate is one joint allocation: a level tuple (l_0..l_{W-1}).  The
//            last worker's levels live in registers (KIN per thread); the other workers form
//            the "prefix", advanced by an odometer (no index decode in the hot loop, no
//            candidate list in HBM).  FP32 keys are a FILTER with relative error <= delta
//            (DESIGN.md §3.5); SUM uses the aggregated form
//               sum_w B_w (1 + O_w / (Lambda N)) = B + (T' B - sum_w B_w S'_w) / (Lambda N)
//            evaluated with packed f32x2 FMA/ADD (two candidates per instruction).
//   pass 2   K5: per problem, rescan only the sub-chunks whose pass-1 minimum is within the
//            band  m (1+tau)(1+delta)/(1-delta); evaluate those candidates EXACTLY (integers)
//            to get the exact minimum H*, then the lowest index with key <= H* (1+tau).
//   materialize (a9): winner -> witnesses -> per-group pool sizes, FP64 latency / power /
//            energy / throughput.
#include <cfloat>
#include <climits>
#include <cstdio>

#include <algorithm>

#include "engine.h"

namespace eclip {

// ------------------------------------------------------------------------------------------
// small helpers
// ------------------------------------------------------------------------------------------
typedef unsigned long long u64;

__device__ __forceinline__ u64 f2pack(float lo, float hi) {
    u64 r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2unpack(u64 v, float& lo, float& hi) {
    asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
    u64 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
    u64 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// 1-D TMA bulk copy global -> shared, completion on an mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    unsigned d = (unsigned)__cvta_generic_to_shared(dst), b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(a), "r"(phase) : "memory");
}

// two pieces (level records, then an aux block from elsewhere) into consecutive shared memory, one barrier
__device__ __forceinline__ void stage_levels2(Lev* sl, const Lev* g1, unsigned b1, const Lev* g2, unsigned b2,
                                              uint64_t* bar) {
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_expect_tx(bar, b1 + b2);
        const unsigned CH = 32768;
        for (unsigned off = 0; off < b1; off += CH)
            bulk_g2s((char*)sl + off, (const char*)g1 + off, b1 - off < CH ? b1 - off : CH, bar);
        for (unsigned off = 0; off < b2; off += CH)
            bulk_g2s((char*)sl + b1 + off, (const char*)g2 + off, b2 - off < CH ? b2 - off : CH, bar);
    }
    __syncthreads();
    mbar_wait(bar, 0);
}

// stage the problem's level records (W x Lmax x 32 B, contiguous) into shared memory
__device__ __forceinline__ void stage_levels(Lev* sl, const Lev* gl, unsigned bytes, uint64_t* bar) {
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_expect_tx(bar, bytes);
        const unsigned CH = 32768;
        for (unsigned off = 0; off < bytes; off += CH) {
            unsigned n = bytes - off < CH ? bytes - off : CH;
            bulk_g2s((char*)sl + off, (const char*)gl + off, n, bar);
        }
    }
    __syncthreads();
    mbar_wait(bar, 0);
}

// ------------------------------------------------------------------------------------------
// pass-1 geometry (shared with pass 2 and the host).
//   The last worker is "inner" (its levels are the per-thread register set), worker W-2 is the
//   "step" worker (walked inside a unit), workers 0..W-3 are "hi" (fixed inside a unit).
//   row  = one combination of hi digits; unit = (row, segment of the step worker's levels);
//   submin[prob][unit] = FP32 minimum over the unit (the pass-2 granularity).
// ------------------------------------------------------------------------------------------
__host__ __device__ __forceinline__ int pow2ceil(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}
__host__ __device__ __forceinline__ int fast_team(int L_in) { return pow2ceil((L_in + KIN - 1) / KIN); }
__host__ __device__ __forceinline__ bool fast_ok(int L_in) { return fast_team(L_in) <= 32; }
__host__ __device__ __forceinline__ uint64_t rows_of(const int* L, int W) {
    uint64_t h = 1;
    for (int w = 0; w < W - 2; w++) h *= (uint64_t)L[w];
    return h;
}
__host__ __device__ __forceinline__ int lstep_of(const int* L, int W) { return W >= 2 ? L[W - 2] : 1; }

// a / b and a % b for b < 2^31: the 32-bit operations when a fits (the 64-bit ones are a software routine)
__host__ __device__ __forceinline__ uint64_t udiv_small(uint64_t a, uint32_t b, uint32_t* rem) {
    if ((a >> 32) == 0) {
        const uint32_t x = (uint32_t)a, q = x / b;
        *rem = x - q * b;
        return q;
    }
    const uint64_t q = a / b;
    *rem = (uint32_t)(a - q * b);
    return q;
}

__host__ __device__ __forceinline__ void shard_items(uint64_t n_items, int shard, int n_shards, uint64_t* lo,
                                                     uint64_t* hi) {
    if (n_shards == 1) {
        *lo = 0;
        *hi = n_items;
        return;
    }
    *lo = n_items * (uint64_t)shard / (uint64_t)n_shards;
    *hi = n_items * (uint64_t)(shard + 1) / (uint64_t)n_shards;
}

// unit -> (row, step-digit range [e0, e1))
__device__ __forceinline__ void unit_range(const Prob& P, uint64_t unit, uint64_t* row, int* e0, int* e1) {
    uint32_t sg;
    *row = udiv_small(unit, (uint32_t)P.nseg, &sg);
    int a = (int)sg * P.seglen, b = a + P.seglen;
    if (b > P.Lstep) b = P.Lstep;
    *e0 = a;
    *e1 = b;
}

// row -> hi digits d[0..W-3] (worker 0 most significant)
__device__ __forceinline__ void decode_row(uint64_t row, const int* L, int W, int* d) {
    for (int w = W - 3; w >= 0; w--) {
        uint32_t r;
        row = udiv_small(row, (uint32_t)L[w], &r);
        d[w] = (int)r;
    }
}

// ------------------------------------------------------------------------------------------
// prep
// ------------------------------------------------------------------------------------------
__global__ void k_prep_prob(Setup su, Tables tb, PrepIn in, Prob* probs) {
    pdl_wait();      // (programmatic dependent launch: the predecessor's results are visible)
    pdl_trigger();
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= su.n_problems) return;
    Prob P;
    memset(&P, 0, sizeof(P));
    P.W = su.W;
    P.status = 0;
    P.rep = p;
    const int W = su.W;
    u64 lam = 1;
    for (int w = 0; w < W; w++) {
        int t = in.table_of[(size_t)p * W + w];
        if (t < 0 || t >= tb.n) { P.status = -4; break; }
        P.table[w] = t;
        P.L[w] = tb.L[t];
        if (P.L[w] <= 0) P.status = 1;  // a worker without any budget-feasible plan
        u64 K = (u64)tb.K[t];
        u64 g = gcd_u64(lam, K);
        lam = lam / g * K;
        if (lam > ((u64)1 << 40)) P.status = -5;
    }
    P.lam = (int64_t)lam;
    P.lamN = (int64_t)(lam * (u64)su.N);
    // narrow problems: S', T' < 2^24 (exact in FP32 / int32, the fast kernels' integer QoS thresholds);
    // wide launches (su.wide, heterogeneous kernel counts): T' in int64
    if ((u128)P.lamN * (u128)(W + 1) >= ((u128)1 << (su.wide ? 62 : 24))) P.status = P.status < 0 ? P.status : -5;
    // index-space sizes, saturating (only the ENUM engine needs them; the host checks its limits)
    uint64_t Pn = 1, tot = 1;
    const uint64_t SAT = (uint64_t)1 << 62;
    for (int w = 0; w < W; w++) {
        uint64_t Lw = (uint64_t)(P.L[w] > 0 ? P.L[w] : 1);
        tot = (tot >= SAT / Lw) ? SAT : tot * Lw;
        if (w < W - 1) Pn = (Pn >= SAT / Lw) ? SAT : Pn * Lw;
    }
    P.P = Pn;
    P.total = tot;
    {   // pass-1 units (see geometry above); rows saturate like the index space
        uint64_t H = 1;
        for (int w = 0; w < W - 2; w++) {
            uint64_t Lw = (uint64_t)(P.L[w] > 0 ? P.L[w] : 1);
            H = (H >= SAT / Lw) ? SAT : H * Lw;
        }
        P.Lstep = W >= 2 ? (P.L[W - 2] > 0 ? P.L[W - 2] : 1) : 1;
        P.nseg = su.nseg < P.Lstep ? su.nseg : P.Lstep;
        P.seglen = (P.Lstep + P.nseg - 1) / P.nseg;
        P.nseg = (P.Lstep + P.seglen - 1) / P.seglen;
        P.units = H * (uint64_t)P.nseg;
        P.n_items = (P.units + (uint64_t)su.upi - 1) / (uint64_t)su.upi;
    }
    P.inv = (float)(1.0 / (double)P.lamN);
    P.lamNf = (float)P.lamN;
    P.p_idle = in.p_idle;
    P.p_dyn = in.p_max - in.p_idle;
    P.p_max = in.p_max;
    // power model as exact integers p 2^k
    int k1 = frac_bits_d((double)in.p_idle, 40), k2 = frac_bits_d((double)in.p_max, 40);
    if (k1 < 0 || k2 < 0) P.status = -4;
    int k = k1 > k2 ? k1 : k2;
    P.k_pow = k;
    double pi_i = ldexp((double)in.p_idle, k), pi_m = ldexp((double)in.p_max, k);
    if (pi_m >= 4.6e18) P.status = -5;
    P.pi_idle = (u128)(u64)pi_i;
    P.pi_dyn = (u128)((u64)pi_m - (u64)pi_i);
    // slowdown matrix
    P.E = 0;
    if (su.mode == M_MATRIX) {
        for (int a = 0; a < W; a++)
            for (int b = 0; b < W; b++) {
                float m = a == b ? 0.0f : in.M[(size_t)p * W * W + a * W + b];
                if (!(m >= 0.0f) || m >= 1024.0f) { P.status = -4; m = 0.0f; }
                int kb = frac_bits_d((double)m, 32);
                if (kb < 0) P.status = -5;
                if (kb > P.E) P.E = kb;
                P.Mf[a * MAXW_ENUM + b] = m;
            }
        for (int a = 0; a < W; a++)
            for (int b = 0; b < W; b++) P.Mi[a * MAXW_ENUM + b] = (int64_t)ldexp((double)P.Mf[a * MAXW_ENUM + b], P.E);
    }
    P.D = (u128)P.lamN << P.E;
    // per-worker objective weights ("weights: per-worker scalar (default all 1)", "strictly
    // positive"; R20): n_w = round-half-up(omega_w 1e6), exact keys use n_w / gcd_w n_w
    {
        u64 g = 0, n[MAXW];
        for (int w = 0; w < W; w++) {
            n[w] = 1000000ull;
            if (in.weights) {
                const double x = in.weights[(size_t)p * W + w];
                if (!(x > 0.0 && x <= 1000.0)) { P.status = -4; break; }
                const double y = x * 1e6;
                const long long r = llround(y);   // half away from zero == half up (y > 0)
                if (r < 1) { P.status = -4; break; }
                n[w] = (u64)r;
            }
            g = gcd_u64(g, n[w]);
        }
        for (int w = 0; w < W; w++) {
            const u64 v = (P.status == -4 || g == 0) ? 1 : n[w] / g;
            P.wt[w] = v;
            P.wf[w] = (float)v;
            P.wv[w] = P.status == -4 ? 1.0 : (double)n[w] / 1e6;
            if (su.obj == O_ENERGY && v != 1) P.status = -4;   // energy is physical: no per-worker weights
        }
    }
    P.has_qos = 0;
    for (int w = 0; w < W; w++) {
        double q = in.qos ? in.qos[(size_t)p * W + w] : (double)INFINITY;
        if (!(q >= 0.0)) P.status = -4;
        P.Hq[w] = floor_qD(q, P.D);
        if (!isinf(q)) P.has_qos = 1;
        // FP32 QoS bounds on L_w (MATRIX, and wide problems): relative error of L32 <= (W+2) 2^-24 (MATRIX),
        // <= (3W+3) 2^-24 (wide EXCESS: T' - Lambda N rounded; the others <= (W+2)); margins 2W+8 / 4W+8
        double marg = (double)((su.wide ? 4 : 2) * W + 8) * 5.9604644775390625e-08;
        P.Qhi[w] = isinf(q) ? INFINITY : __double2float_ru(q * (1.0 + marg));
        P.Qlo[w] = isinf(q) ? INFINITY : __double2float_rd(q * (1.0 - marg));
    }
    probs[p] = P;
}

// one thread per (problem, worker, level)
__global__ void k_prep_lev(Setup su, Tables tb, const Prob* probs, Lev* levs) {
    pdl_wait();      // (programmatic dependent launch: the predecessor's results are visible)
    pdl_trigger();
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    size_t n = (size_t)su.n_problems * su.W * su.Lmax;
    if (i >= n) return;
    int l = (int)(i % su.Lmax);
    int w = (int)((i / su.Lmax) % su.W);
    int p = (int)(i / ((size_t)su.Lmax * su.W));
    const Prob& P = probs[p];
    Lev r;
    r.B = 0; r.BS = 0; r.S = 0; r.Tmax = -1; r.Bk = 0.0f;
    Lev* dst = levs + (size_t)p * su.lev_stride + (size_t)w * su.Lmax + l;
    if (P.status >= 0 && l < P.L[w]) {
        int t = P.table[w];
        int64_t B = tb.B[t][l];
        int64_t Sp = tb.S[t][l] * (P.lam / tb.K[t]);
        r.B = B;
        r.S = Sp;
        r.BS = su.wide ? 0 : B * Sp;   // wide: B S' may exceed int64 (only the narrow fast kernels read it)
        r.Bk = (float)((double)B / (double)P.lamN);
        int64_t T = NARROW_T;
        if (P.has_qos && !qos_float(su) && ~P.Hq[w] != 0) {
            u128 hq = P.Hq[w];
            int64_t hb;  // floor(Hq / B), saturated at 2^30
            if ((hq >> 64) != 0) hb = (int64_t)1 << 30;
            else {
                u64 q = (u64)hq / (u64)B;
                hb = q > ((u64)1 << 30) ? ((int64_t)1 << 30) : (int64_t)q;
            }
            if (su.mode == M_EXCL) T = Sp - P.lamN + hb;
            else if (su.mode == M_PAPER) T = hb - P.lamN;
            else T = ((u128)B * (u128)P.lamN > hq) ? -1 : hb;
            if (T < -1) T = -1;
            if (T > NARROW_T) T = NARROW_T;
        }
        r.Tmax = (int32_t)T;
    }
    *dst = r;
}


// ------------------------------------------------------------------------------------------
// Sharing of the step / inner-worker precomputation inside a batch.  A problem's aux block (k_prep_aux),
// hulls, row-feasibility table and row-bound header (k_prep_bound) are functions of its AKey only; the
// problems of a batch with equal keys (mixes drawn from one model library share worker pairs) use the
// first one's.  k_akey: one warp per problem computes the key (the hi workers' S' sum range from their
// level records) and inserts its hash into an open-addressing table with the minimum problem index;
// k_arep: each problem looks its hash up and takes that index as its representative when the two keys
// are equal (any hash collision falls back to itself).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long akey_hash(const AKey& k) {
    unsigned long long h = 0x9E3779B97F4A7C15ull;
    auto mix = [&](unsigned long long v) {
        h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
        h *= 0xff51afd7ed558ccdull;
        h ^= h >> 33;
    };
    mix(((unsigned long long)(uint32_t)k.tab_step << 32) | (uint32_t)k.tab_inner);
    mix(((unsigned long long)(uint32_t)k.t0 << 32) | (uint32_t)k.t1);
    mix((unsigned long long)k.lam);
    mix((unsigned long long)k.hq_step); mix((unsigned long long)(k.hq_step >> 64));
    mix((unsigned long long)k.hq_inner); mix((unsigned long long)(k.hq_inner >> 64));
    return h | 1ull;   // 0 marks an empty slot
}
__device__ __forceinline__ bool akey_eq(const AKey& a, const AKey& b) {
    return a.tab_step == b.tab_step && a.tab_inner == b.tab_inner && a.t0 == b.t0 && a.t1 == b.t1 && a.lam == b.lam &&
           a.hq_step == b.hq_step && a.hq_inner == b.hq_inner;
}

__global__ void __launch_bounds__(256) k_akey(Setup su, const Prob* probs, const Lev* levs, AKey* keys,
                                              unsigned long long* slot, int nslots) {
    pdl_wait();      // (programmatic dependent launch: the predecessor's results are visible)
    pdl_trigger();
    const int p = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (p >= su.n_problems) return;
    const Prob& P = probs[p];
    const int W = su.W, Lmax = su.Lmax;
    AKey k;
    k.t0 = -1;   // no sharing (invalid problem)
    if (P.status == 0) {
        const Lev* base = levs + (size_t)p * su.lev_stride;
        int t0 = 0, t1 = 0;
        for (int w = 0; w < W - 2; w++) {
            int mn = 1 << 30, mx = 0;
            for (int l = lane; l < P.L[w]; l += 32) {
                const int v = (int)base[(size_t)w * Lmax + l].S;
                mn = min(mn, v); mx = max(mx, v);
            }
            mn = __reduce_min_sync(0xffffffffu, mn);
            mx = __reduce_max_sync(0xffffffffu, mx);
            t0 += mn; t1 += mx;
        }
        k.tab_step = P.table[W >= 2 ? W - 2 : 0]; k.tab_inner = P.table[W - 1];
        k.t0 = t0; k.t1 = t1; k.lam = P.lam;
        k.hq_step = P.Hq[W >= 2 ? W - 2 : 0]; k.hq_inner = P.Hq[W - 1];
    }
    if (lane != 0) return;
    keys[p] = k;
    if (k.t0 < 0) return;
    const unsigned long long h = akey_hash(k);
    unsigned long long* hs = slot;
    unsigned long long* ix = slot + nslots;
    for (int i = (int)(h & (unsigned long long)(nslots - 1)), n = 0; n < nslots; i = (i + 1) & (nslots - 1), n++) {
        const unsigned long long prev = atomicCAS(hs + i, 0ull, h);
        if (prev == 0ull || prev == h) {
            atomicMin(ix + i, (unsigned long long)p);
            return;
        }
    }
}

__global__ void k_arep(Setup su, Prob* probs, const AKey* keys, const unsigned long long* slot, int nslots) {
    pdl_wait();      // (programmatic dependent launch: the predecessor's results are visible)
    pdl_trigger();
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= su.n_problems) return;
    const AKey k = keys[p];
    int rep = p;
    if (k.t0 >= 0) {
        const unsigned long long h = akey_hash(k);
        for (int i = (int)(h & (unsigned long long)(nslots - 1)), n = 0; n < nslots; i = (i + 1) & (nslots - 1), n++) {
            const unsigned long long hv = slot[i];
            if (hv == 0ull) break;
            if (hv == h) {
                const int q = (int)slot[nslots + i];
                if (q < p && akey_eq(keys[q], k)) rep = q;
                break;
            }
        }
    }
    probs[p].rep = rep;
}

// Slope table of a lower-left hull (n vertices, edges ed[0..n-2] = {B_i - B_i+1, S'_i+1 - S'_i}):
// the minimiser of B y + S' z is the count of leading edges with ed.x y > ed.y z, which does not
// increase with q = z / y.  Bin b holds the queries whose float bits satisfy (bits >> 20) = base + b
// (8 bins per octave); T[b] = that count at the upper end of bin b + 1, so T[b] <= the count of every
// query of bin b even when q is computed with a few ulps of error (one bin of slack = 9 %); the last
// bin starts at 0, queries outside the table are clamped to its ends.  The query scans forward from T[b] with the exact predicate (hull_arg): one or two
// steps instead of a binary search.  Built by threads t < nt of the caller (edge counts by binary search).
__device__ __forceinline__ void build_slope_table(const float2* ed, int n, uint8_t* T, int* base, int lane, int nt = 32) {
    int b0 = 0;
    if (n >= 2) {   // the table spans HT_NB / 8 octaves below the first (largest) slope; smaller queries start
                    // from bin 0's count (still a valid start)
        const float smax = ed[0].x / ed[0].y;
        b0 = (__float_as_int(smax) >> 20) - (HT_NB - 3);
    }
    for (int b = lane; b < HT_NB; b += nt) {
        const int qb = b0 + b + 2;   // bits >> 20 of the upper end of bin b + 1
        const float q = qb <= 0 ? 0.0f : (qb >= (0x7f800000 >> 20) ? INFINITY : __int_as_float(qb << 20));
        int lo = 0, hi = max(n - 1, 0);   // the slopes decrease: count = first edge with ed.x <= ed.y q
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (ed[mid].x > ed[mid].y * q) lo = mid + 1; else hi = mid;
        }
        T[b] = (uint8_t)(b == HT_NB - 1 ? 0 : min(lo, 255));
    }
    if (lane == 0) *base = b0;
}
__device__ __forceinline__ int hull_arg(const float2* ed, int n, const uint8_t* T, int base, float y, float z) {
    int b = (__float_as_int(__fdividef(z, y)) >> 20) - base;
    b = min(max(b, 0), HT_NB - 1);
    int lo = T[b];
    while (lo < n - 1) {
        const float2 e = ed[lo];
        if (!(e.x * y > e.y * z)) break;
        lo++;
    }
    return lo;
}

// ------------------------------------------------------------------------------------------
// fast pass-1 aux block (per problem, right after its Lev records; staged with them)
//   ip    float4[LP]   inner levels sorted by S', in pairs {B_k, B_k+1, S'_k, S'_k+1}
//   iu    float2[LP]   {u_k, u_k+1},  u = Tmax - S'  (inner worker's own QoS: Tp <= u)
//   iD    float2[LP]   PAPER: {B_k S'_k/(Lambda N), ...}
//   ssort int[Lmax+1]  sorted S';  usuf int[Lmax+1] suffix min of u;  umaxp int[Lmax+1] prefix max
//   perm  u16[Lmax]    inner sorted by S';  sperm u16[Lmax] step worker sorted by S' per segment
//   khi   u16[TABN]    #{k : S'_k <= s0 + v};   klo u16[TABN]  min{k : usuf[k] >= u0 + v}
//   hdr   int[4]       s0, u0, khi_ok, klo_ok
// ------------------------------------------------------------------------------------------
struct AuxView {
    float4* ip; float2* iu; float2* iD; int* ssort; int* usuf; int* umaxp; uint16_t* perm; uint16_t* sperm;
    uint8_t* khi; uint8_t* klo;       // inner worker: #{k : S'_k <= s0 + v};  min{k : usuf[k] >= u0 + v}
    uint8_t* shi; uint8_t* slo;       // step worker (one segment): same two tables
    int* hdr;                         // s0, u0, khi_ok, klo_ok, ss0, su0, shi_ok, slo_ok
    int* stS; int* stU; int* stUmax;  // step worker, sorted per segment: S', suffix-min of u, prefix-max of u
    float* preminB;                   // inner worker, S'-sorted: preminB[k] = (float) min_{j<k} B_j (+inf at 0)
    float* chB;                       // step worker, S'-sorted: (float) min B over each aligned chunk of P1_CS
    float2* ih;                       // inner worker's lower-left hull: vertices {B, S'} in S' order
    float2* ie;                       //   edges {B_i - B_i+1, S'_i+1 - S'_i}
    int* ihn;                         //   [1] vertex count
    uint16_t* hpos;                   // inner, S'-sorted position k -> last hull vertex with S' <= S'_k
    float* chBs;                      // step worker: suffix minimum of chB over the chunks
    uint8_t* ht;                      // inner hull's slope table [HT_NB] (build_slope_table)
    int* htb;                         //   [1] its base
};
__host__ __device__ __forceinline__ size_t aux_bytes_of(int Lmax) {
    const size_t LP = (size_t)(Lmax + 1) / 2;
    size_t b = ((LP * 32 + (size_t)(Lmax + 1) * 12 + (size_t)Lmax * 4 + 15) & ~(size_t)15) + 4 * (size_t)P1_TABN + 32 +
               (size_t)Lmax * 12 +
               (size_t)(Lmax + 1) * 4 + (size_t)((Lmax + P1_CS - 1) / P1_CS) * 4;
    b = (b + 7) & ~(size_t)7;
    b += (size_t)Lmax * 16 + 4 + (size_t)Lmax * 2;   // ih, ie, ihn, hpos
    b = (b + 3) & ~(size_t)3;
    b += (size_t)((Lmax + P1_CS - 1) / P1_CS) * 4;   // chBs
    b += 4 + HT_NB;                                   // htb, ht
    return (b + 31) / 32 * 32;
}
size_t pass1_aux_bytes(int Lmax) { return aux_bytes_of(Lmax); }
__device__ __forceinline__ AuxView aux_view(unsigned char* base, int Lmax) {
    AuxView a;
    const int LP = (Lmax + 1) / 2;
    a.ip = reinterpret_cast<float4*>(base);
    a.iu = reinterpret_cast<float2*>(a.ip + LP);
    a.iD = a.iu + LP;
    a.ssort = reinterpret_cast<int*>(a.iD + LP);
    a.usuf = a.ssort + (Lmax + 1);
    a.umaxp = a.usuf + (Lmax + 1);
    a.perm = reinterpret_cast<uint16_t*>(a.umaxp + (Lmax + 1));
    a.sperm = a.perm + Lmax;
    a.khi = base + ((reinterpret_cast<unsigned char*>(a.sperm + Lmax) - base + 15) & ~(size_t)15);   // 16-aligned tables
    a.klo = a.khi + P1_TABN;
    a.shi = a.klo + P1_TABN;
    a.slo = a.shi + P1_TABN;
    a.hdr = reinterpret_cast<int*>(a.slo + P1_TABN);
    a.stS = a.hdr + 8;
    a.stU = a.stS + Lmax;
    a.stUmax = a.stU + Lmax;
    a.preminB = reinterpret_cast<float*>(a.stUmax + Lmax);
    a.chB = a.preminB + (Lmax + 1);
    unsigned char* q = reinterpret_cast<unsigned char*>(a.chB + (Lmax + P1_CS - 1) / P1_CS);
    q = base + ((q - base + 7) & ~(size_t)7);
    a.ih = reinterpret_cast<float2*>(q);
    a.ie = a.ih + Lmax;
    a.ihn = reinterpret_cast<int*>(a.ie + Lmax);
    a.hpos = reinterpret_cast<uint16_t*>(a.ihn + 1);
    q = reinterpret_cast<unsigned char*>(a.hpos + Lmax);
    a.chBs = reinterpret_cast<float*>(base + ((q - base + 3) & ~(size_t)3));
    a.htb = reinterpret_cast<int*>(a.chBs + (Lmax + P1_CS - 1) / P1_CS);
    a.ht = reinterpret_cast<uint8_t*>(a.htb + 1);
    return a;
}

// one CTA per problem: sort, pair up, and tabulate the inner / step workers once
template <int MODE>
__global__ void __launch_bounds__(256) k_prep_aux(Setup su, const Prob* probs, Lev* levs, const int32_t* table_of,
                                                  const uint16_t* tord, const uint16_t* thull, const int32_t* thull_n) {
    pdl_wait();      // (programmatic dependent launch: the predecessor's results are visible)
    pdl_trigger();
    const int prob = blockIdx.x;
    const Prob& P = probs[prob];
    if (P.status != 0 || P.rep != prob) return;   // a representative's block serves this problem
    const int W = su.W, Lmax = su.Lmax;
    Lev* base = levs + (size_t)prob * su.lev_stride;
    // the block is built in shared memory from shared copies of the two workers' records, then
    // written out once (coalesced)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Lev* inner_s = reinterpret_cast<Lev*>(smem_raw);
    Lev* step_s = inner_s + Lmax;
    unsigned char* aux_s = reinterpret_cast<unsigned char*>(step_s + Lmax);
    {
        const Lev* gi = base + (W - 1) * Lmax;
        const Lev* gs = base + (W >= 2 ? (W - 2) : 0) * Lmax;
        for (int i = threadIdx.x; i < Lmax; i += blockDim.x) { inner_s[i] = gi[i]; step_s[i] = gs[i]; }
    }
    __syncthreads();
    const Lev* inner = inner_s;
    const Lev* stepw = step_s;
    AuxView A = aux_view(aux_s, Lmax);
    const int Lin = P.L[W - 1], Lst = P.Lstep, segl = P.seglen;
    const double invd = 1.0 / (double)P.lamN;
    // S' order of the inner and step workers: the level tables' S order (k_table_hull; a positive scaling)
    // with whole-row units, else rank sorts (per segment for the step worker)
    const bool tab_order = su.nseg == 1;
    if (tab_order) {
        const uint16_t* oi = tord + (size_t)table_of[(size_t)prob * W + W - 1] * Lmax;
        for (int i = threadIdx.x; i < Lin; i += blockDim.x) A.perm[i] = oi[i];
        if (W >= 2) {
            const uint16_t* os = tord + (size_t)table_of[(size_t)prob * W + W - 2] * Lmax;
            for (int i = threadIdx.x; i < Lst; i += blockDim.x) A.sperm[i] = os[i];
        }
    } else {
    for (int i = threadIdx.x; i < Lin; i += blockDim.x) {
        const int si = inner[i].S;
        int rk = 0;
        for (int j = 0; j < Lin; j++) rk += inner[j].S < si;
        A.perm[rk] = (uint16_t)i;
    }
    }
    if (W >= 2 && !tab_order) {
        for (int i = threadIdx.x; i < Lst; i += blockDim.x) {
            const int b0 = (i / segl) * segl, b1 = min(b0 + segl, Lst);
            const int si = stepw[i].S;
            int rk = 0;
            for (int j = b0; j < b1; j++) rk += stepw[j].S < si;
            A.sperm[b0 + rk] = (uint16_t)i;
        }
    }
    __syncthreads();
    for (int p = threadIdx.x; p < (Lin + 1) / 2; p += blockDim.x) {
        const Lev& a = inner[A.perm[2 * p]];
        const Lev& b = inner[A.perm[min(2 * p + 1, Lin - 1)]];
        A.ip[p] = make_float4(__ll2float_rn(a.B), __ll2float_rn(b.B), (float)a.S, (float)b.S);
        A.iu[p] = make_float2((float)(a.Tmax - a.S), (float)(b.Tmax - b.S));
        if (MODE == M_PAPER) A.iD[p] = make_float2((float)((double)a.BS * invd), (float)((double)b.BS * invd));
    }
    for (int k = threadIdx.x; k < Lin; k += blockDim.x) A.ssort[k] = inner[A.perm[k]].S;
    __syncthreads();
    // warp scans (S'-sorted order): warp 0 preminB (exclusive prefix min of B), warp 1 usuf (suffix min
    // of u = Tmax - S'), warp 2 umaxp (exclusive prefix max of u), warps 3/4 the step worker's
    // per-segment suffix min / inclusive prefix max of u
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        float carry = INFINITY;
        if (lane == 0) A.preminB[0] = INFINITY;
        for (int b = 0; b < Lin; b += 32) {
            float v = b + lane < Lin ? __ll2float_rn(inner[A.perm[b + lane]].B) : INFINITY;
            for (int o = 1; o < 32; o <<= 1) { const float y = __shfl_up_sync(0xffffffffu, v, o); if (lane >= o) v = fminf(v, y); }
            v = fminf(v, carry);
            if (b + lane < Lin) A.preminB[b + lane + 1] = v;
            carry = __shfl_sync(0xffffffffu, v, 31);
        }
    } else if (warp == 1) {
        int carry = 1 << 30;
        if (lane == 0) A.usuf[Lin] = 1 << 30;
        for (int e = Lin; e > 0; e -= 32) {   // chunk [e-32, e)
            const int k = e - 32 + lane;
            int v = k >= 0 ? inner[A.perm[k]].Tmax - A.ssort[k] : (1 << 30);
            for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_down_sync(0xffffffffu, v, o); if (lane + o < 32) v = min(v, y); }
            v = min(v, carry);
            if (k >= 0) A.usuf[k] = v;
            carry = __shfl_sync(0xffffffffu, v, 0);
        }
    } else if (warp == 2) {
        int carry = -(1 << 30);
        if (lane == 0) A.umaxp[0] = -(1 << 30);
        for (int b = 0; b < Lin; b += 32) {
            int v = b + lane < Lin ? inner[A.perm[b + lane]].Tmax - A.ssort[b + lane] : -(1 << 30);
            for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, v, o); if (lane >= o) v = max(v, y); }
            v = max(v, carry);
            if (b + lane < Lin) A.umaxp[b + lane + 1] = v;
            carry = __shfl_sync(0xffffffffu, v, 31);
        }
    } else if (W >= 2 && (warp == 3 || warp == 4)) {
        for (int b0 = 0; b0 < Lst; b0 += segl) {   // segments
            const int b1 = min(b0 + segl, Lst);
            if (warp == 3) {
                int carry = 1 << 30;
                for (int e = b1; e > b0; e -= 32) {
                    const int i = e - 32 + lane;
                    int v = i >= b0 ? stepw[A.sperm[i]].Tmax - stepw[A.sperm[i]].S : (1 << 30);
                    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_down_sync(0xffffffffu, v, o); if (lane + o < 32) v = min(v, y); }
                    v = min(v, carry);
                    if (i >= b0) { A.stU[i] = v; A.stS[i] = stepw[A.sperm[i]].S; }
                    carry = __shfl_sync(0xffffffffu, v, 0);
                }
            } else {
                int carry = -(1 << 30);
                for (int b = b0; b < b1; b += 32) {
                    const int i = b + lane;
                    int v = i < b1 ? stepw[A.sperm[i]].Tmax - stepw[A.sperm[i]].S : -(1 << 30);
                    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, v, o); if (lane >= o) v = max(v, y); }
                    v = max(v, carry);
                    if (i < b1) A.stUmax[i] = v;
                    carry = __shfl_sync(0xffffffffu, v, 31);
                }
            }
        }
    }
    {   // the inner worker's hull (its table's vertex set, k_table_hull) and the clamp positions
        const int ti = table_of[(size_t)prob * W + W - 1];
        const uint16_t* hx = thull + (size_t)ti * Lmax;
        const int nh = thull_n[ti];
        for (int i = threadIdx.x; i < nh; i += blockDim.x) {
            const Lev& v = inner[hx[i]];
            A.ih[i] = make_float2(__ll2float_rn(v.B), (float)v.S);
            if (i + 1 < nh) {
                const Lev& x = inner[hx[i + 1]];
                A.ie[i] = make_float2(__ll2float_rn(v.B - x.B), (float)(x.S - v.S));
            }
        }
        if (threadIdx.x == 0) *A.ihn = nh;
        __syncthreads();
        ECLIP_CHECK((size_t)(A.ht + HT_NB - aux_s) <= su.aux_bytes && nh <= Lmax);
        build_slope_table(A.ie, nh, A.ht, A.htb, threadIdx.x, blockDim.x);
        for (int k = threadIdx.x; k < Lin; k += blockDim.x) {   // last vertex with S' <= S'_k (exact ints)
            const int sk = inner[A.perm[k]].S;
            int lo = 0, hi = nh - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (inner[hx[mid]].S <= sk) lo = mid; else hi = mid - 1;
            }
            A.hpos[k] = (uint16_t)lo;
        }
    }
    if (W >= 2)
        for (int c = threadIdx.x; c * P1_CS < Lst; c += blockDim.x) {
            float m = INFINITY;
            for (int i = c * P1_CS; i < min(Lst, c * P1_CS + P1_CS); i++) m = fminf(m, __ll2float_rn(stepw[A.sperm[i]].B));
            A.chB[c] = m;
        }
    __syncthreads();
    if (W >= 2 && threadIdx.x == 0) {   // suffix minimum of the chunk minima
        float m = INFINITY;
        for (int c = (Lst + P1_CS - 1) / P1_CS - 1; c >= 0; c--) { m = fminf(m, A.chB[c]); A.chBs[c] = m; }
    }
    const int s0 = A.ssort[0], u0 = A.usuf[0];
    const bool khi_ok = Lin <= 255 && A.ssort[Lin - 1] - s0 + 1 <= P1_TABN;
    const bool klo_ok = Lin <= 255 && A.usuf[Lin - 1] - u0 + 1 <= P1_TABN;
    if (khi_ok)
        for (int k = threadIdx.x; k < Lin; k += blockDim.x)
            for (int v = A.ssort[k]; v < (k + 1 < Lin ? A.ssort[k + 1] : A.ssort[k] + 1); v++) A.khi[v - s0] = (uint8_t)(k + 1);
    if (klo_ok)
        for (int k = threadIdx.x; k < Lin; k += blockDim.x)
            for (int v = (k == 0 ? A.usuf[0] : A.usuf[k - 1] + 1); v <= A.usuf[k]; v++) A.klo[v - u0] = (uint8_t)k;
    // step-worker lookup tables (whole-row units only): #{e : S'_e <= ss0 + v}, min{e : stU[e] >= su0 + v}
    bool shi_ok = false, slo_ok = false;
    int ss0 = 0, su0 = 0;
    if (W >= 2 && P.nseg == 1 && Lst <= 255) {
        ss0 = A.stS[0]; su0 = A.stU[0];
        shi_ok = A.stS[Lst - 1] - ss0 + 1 <= P1_TABN;
        slo_ok = A.stU[Lst - 1] - su0 + 1 <= P1_TABN;
        if (shi_ok)
            for (int e = threadIdx.x; e < Lst; e += blockDim.x)
                for (int v = A.stS[e]; v < (e + 1 < Lst ? A.stS[e + 1] : A.stS[e] + 1); v++) A.shi[v - ss0] = (uint8_t)(e + 1);
        if (slo_ok)
            for (int e = threadIdx.x; e < Lst; e += blockDim.x)
                for (int v = (e == 0 ? A.stU[0] : A.stU[e - 1] + 1); v <= A.stU[e]; v++) A.slo[v - su0] = (uint8_t)e;
    }
    if (threadIdx.x == 0) {
        A.hdr[0] = s0; A.hdr[1] = u0; A.hdr[2] = khi_ok; A.hdr[3] = klo_ok;
        A.hdr[4] = ss0; A.hdr[5] = su0; A.hdr[6] = shi_ok; A.hdr[7] = slo_ok;
    }
    __syncthreads();
    // write out the fixed arrays, the used span of each lookup table (the rest is never read) and
    // the header / step arrays
    const uint4* src = reinterpret_cast<const uint4*>(aux_s);
    uint4* dst = reinterpret_cast<uint4*>(base + (size_t)W * Lmax);
    auto cp = [&](size_t off, size_t bytes) {   // off is 16-aligned (aux layout)
        const int n = (int)((bytes + 15) / 16), o = (int)(off / 16);
        for (int i = threadIdx.x; i < n; i += blockDim.x) dst[o + i] = src[o + i];
    };
    const size_t o_khi = (size_t)(A.khi - aux_s), o_hdr = (size_t)(reinterpret_cast<unsigned char*>(A.hdr) - aux_s);
    cp(0, o_khi);
    if (khi_ok) cp(o_khi, (size_t)(A.ssort[Lin - 1] - s0 + 1));
    if (klo_ok) cp(o_khi + P1_TABN, (size_t)(A.usuf[Lin - 1] - u0 + 1));
    if (shi_ok) cp(o_khi + 2 * P1_TABN, (size_t)(A.stS[Lst - 1] - ss0 + 1));
    if (slo_ok) cp(o_khi + 3 * P1_TABN, (size_t)(A.stU[Lst - 1] - su0 + 1));
    cp(o_hdr, (size_t)su.aux_bytes - o_hdr);
}

// ------------------------------------------------------------------------------------------
// Row lower bound.  For a row (hi digits fixed: exact sums hB, hT, hBS), every
// EXCLUDE_SELF key of the row is, exactly (step level e, inner level k),
//   K = Xh + B_e Yh + S'_e Zh + B_k Yh + S'_k Zh + (S'_e B_k + S'_k B_e) / (Lambda N)
// with Xh = hB + (hT hB - hBS)/(Lambda N), Yh = 1 + hT/(Lambda N), Zh = hB/(Lambda N), every term
// >= 0 (PAPER keys are larger by sum_w B_w S'_w/(Lambda N) >= 0, so the bound holds there too).
// Bounding the cross term below by S'_e Bmin_k + Smin_k B_e separates the two workers:
//   K >= Xh + min_e [B_e (Yh + Smin_k/ΛN) + S'_e (Zh + Bmin_k/ΛN)] + min_k [B_k Yh + S'_k Zh]
// and each minimum of a positive linear form over a point set is attained on its lower-left
// convex hull (built exactly here, once per problem).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ bool hull_pop(const Lev& a, const Lev& b, const Lev& c) {
    // drop b unless it lies strictly below the segment a-c (points (S', B), S' increasing)
    const __int128 cr = (__int128)(b.S - a.S) * (__int128)(c.B - a.B) - (__int128)(b.B - a.B) * (__int128)(c.S - a.S);
    return cr <= 0;
}

// One CTA per problem (256 threads):
//  * rank-sort the step and inner workers by (S', B, index); one thread per worker builds the
//    lower-left hull (Pareto staircase + lower convex chain, exact integer orientation tests)
//    and its edges {B_i - B_i+1 > 0, S'_i+1 - S'_i > 0}, whose slopes decrease along the chain;
//  * the exact row-feasibility table.  A candidate (row, e, k) meets every QoS bound iff
//    T' = hT + S'_e + S'_k <= min(hTm, Tmax_e, Tmax_k), i.e. iff
//        hT <= min(u_e - S'_k, u_k - S'_e)  (u = Tmax - S')   and   S'_e + S'_k <= hTm - hT.
//    With F(t) = min { S'_e + S'_k : min(u_e - S'_k, u_k - S'_e) >= t } (non-decreasing in t), a
//    row has a feasible candidate iff F(hT) <= hTm - hT.  F is tabulated for hT in [t0, t1]
//    (sums of the hi workers' min / max S'), when that range fits FT_CAP entries.
// Lower-left hull of every level table in (S, B*) (one CTA per table).  A problem's step / inner worker
// uses its table's levels with S' = S Lambda / K: a positive scaling of S keeps every orientation test,
// so the vertex set (level indices, in S order) is the table's and is computed once per table instead
// of once per problem.  Exact O(L^2) interval test, one point per thread: point p is a vertex iff no
// point before it (smaller S) has B <= B_p and max over later points with smaller B of
// (B_p - B_j)/(S_j - S_p)  <  min over earlier points of (B_j - B_p)/(S_p - S_j) (cross products of
// B < 2^36 and S < 2^24 differences fit in int64); collinear middle points are dropped.
__global__ void __launch_bounds__(256) k_table_hull(Tables tb, int Lmax, uint16_t* thull, int32_t* thull_n,
                                                    uint16_t* tord) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    long long* sB = reinterpret_cast<long long*>(smem_raw);    // [Lmax] B in S order
    int* sS = reinterpret_cast<int*>(sB + Lmax);               // [Lmax] S in S order
    uint16_t* ord = reinterpret_cast<uint16_t*>(sS + Lmax);    // [Lmax] level index in S order
    uint8_t* vf = reinterpret_cast<uint8_t*>(ord + Lmax);      // [Lmax] vertex flags
    const int t = blockIdx.x, L = tb.L[t];
    const int64_t* S = tb.S[t];
    const int64_t* B = tb.B[t];
    for (int l = threadIdx.x; l < L; l += blockDim.x) {   // levels have distinct S: rank = #{smaller S}
        const int64_t sl = S[l];
        int rk = 0;
        for (int j = 0; j < L; j++) rk += S[j] < sl;
        ord[rk] = (uint16_t)l;
        tord[(size_t)t * Lmax + rk] = (uint16_t)l;   // the table's S order (= every problem's S' order)
        sS[rk] = (int)sl;
        sB[rk] = (long long)B[l];
    }
    __syncthreads();
    for (int p = threadIdx.x; p < L; p += blockDim.x) {
        const int pS = sS[p];
        const long long pB = sB[p];
        bool vert = true;
        int64_t lo_n = 0, lo_d = 1, hi_n = 1, hi_d = 0;   // lo = 0, hi = +inf
        for (int r = 0; r < p; r++) {
            const long long qB = sB[r];
            if (qB <= pB) { vert = false; break; }
            const int64_t n = qB - pB, d = (int64_t)(pS - sS[r]);
            if (hi_d == 0 || n * hi_d < hi_n * d) { hi_n = n; hi_d = d; }
        }
        for (int r = p + 1; r < L && vert; r++) {
            const long long qB = sB[r];
            if (qB < pB) {
                const int64_t n = pB - qB, d = (int64_t)(sS[r] - pS);
                if (n * lo_d > lo_n * d) { lo_n = n; lo_d = d; }
            }
        }
        if (vert && hi_d != 0) vert = lo_n * hi_d < hi_n * lo_d;
        vf[p] = vert ? 1 : 0;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        int n = 0;
        for (int b0 = 0; b0 < L; b0 += 32) {
            const int p = b0 + (int)threadIdx.x;
            const bool f = p < L && vf[p];
            const unsigned bal = __ballot_sync(0xffffffffu, f);
            if (f) thull[(size_t)t * Lmax + n + __popc(bal & ((1u << threadIdx.x) - 1u))] = ord[p];
            n += __popc(bal);
        }
        if (threadIdx.x == 0) thull_n[t] = n;
    }
}

__global__ void __launch_bounds__(256) k_prep_bound(Setup su, const Prob* probs, const Lev* levs, float2* hull,
                                                    int32_t* ftab, RowHdr* hdr, const int32_t* table_of,
                                                    const uint16_t* thull, const int32_t* thull_n) {
    pdl_wait();      // (programmatic dependent launch: the predecessor's results are visible)
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int* G = reinterpret_cast<int*>(smem_raw);                          // [FT_CAP]
    Lev* sv = reinterpret_cast<Lev*>(G + FT_CAP);                      // [2][Lmax] step, inner records
    __shared__ int s_t0, s_t1, s_part[256];
    const int prob = blockIdx.x;
    const Prob& P = probs[prob];
    if (P.status != 0 || su.W < 3 || P.rep != prob) return;   // a representative's tables serve this problem
    const int W = su.W, Lmax = su.Lmax;
    const Lev* gbase = levs + (size_t)prob * su.lev_stride;
    for (int i = threadIdx.x; i < 2 * Lmax; i += blockDim.x) sv[i] = gbase[(size_t)(W - 2) * Lmax + i];
    __syncthreads();
    if (threadIdx.x < 32) {   // range of hT over the hi workers (warp 0; sums in registers, one write)
        int t0 = 0, t1 = 0;
        for (int w = 0; w < W - 2; w++) {
            int mn = 1 << 30, mx = 0;
            for (int l = threadIdx.x; l < P.L[w]; l += 32) {
                const int v = (int)gbase[(size_t)w * Lmax + l].S;
                mn = min(mn, v); mx = max(mx, v);
            }
            for (int o = 16; o; o >>= 1) {
                mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            }
            t0 += mn; t1 += mx;
        }
        if (threadIdx.x == 0) { s_t0 = t0; s_t1 = t1; }
    }
    __syncthreads();
    const int t0 = s_t0, tn = (s_t1 - s_t0 + 1 <= FT_CAP && su.has_qos) ? s_t1 - s_t0 + 1 : 0;
    if (threadIdx.x < 64) {   // warp w: worker w's hull (the vertices of its level table, k_table_hull) + edges
        const int which = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const Lev* lv = sv + (size_t)which * Lmax;
        const int L = P.L[W - 2 + which];
        const int tab = table_of[(size_t)prob * W + W - 2 + which];
        const uint16_t* hx = thull + (size_t)tab * Lmax;
        const int n = thull_n[tab];
        int umax = -(1 << 30), smin = INT_MAX;
        long long bmin = LLONG_MAX;
        for (int l = lane; l < L; l += 32) {
            umax = max(umax, (int)(lv[l].Tmax - lv[l].S));   // narrow problems: S' < 2^24
            bmin = min(bmin, (long long)lv[l].B);
            smin = min(smin, (int)lv[l].S);
        }
        for (int off = 16; off; off >>= 1) {
            umax = max(umax, __shfl_xor_sync(0xffffffffu, umax, off));
            bmin = min(bmin, __shfl_xor_sync(0xffffffffu, bmin, off));
            smin = min(smin, __shfl_xor_sync(0xffffffffu, smin, off));
        }
        float2* h = hull + (size_t)prob * hull_stride(Lmax) + (size_t)which * 2 * Lmax;
        for (int i = lane; i < n; i += 32) {
            const Lev& v = lv[hx[i]];
            h[i] = make_float2(__ll2float_rn(v.B), (float)v.S);
            if (i + 1 < n) {
                const Lev& x = lv[hx[i + 1]];
                h[Lmax + i] = make_float2(__ll2float_rn(v.B - x.B), (float)(x.S - v.S));
            }
        }
        __syncwarp();
        int htb = 0;
        build_slope_table(h + Lmax, n, reinterpret_cast<uint8_t*>(hull + (size_t)prob * hull_stride(Lmax) + 4 * (size_t)Lmax) +
                                           which * HT_NB, &htb, lane);
        if (lane == 0) {
            RowHdr* H = hdr + prob;
            H->nh[which] = n;
            H->htb[which] = htb;
            if (which == 0) { H->smin_st = smin; H->umax_st = umax; H->t0 = t0; H->tn = tn; }
            else { H->smin_in = smin; H->umax_in = umax; H->Sminf_in = (float)smin; H->Bminf_in = __ll2float_rn(bmin); }
        }
    }
    if (tn == 0) return;
    // F(t) for t in [t0, t0 + tn): bucket every (e, k) pair at its last valid t, then a suffix minimum
    for (int i = threadIdx.x; i < tn; i += blockDim.x) G[i] = INT_MAX;
    __syncthreads();
    const Lev* st = sv;
    const Lev* in = sv + Lmax;
    const int Le = P.L[W - 2], Lk = P.L[W - 1];
    for (int pidx = threadIdx.x; pidx < Le * Lk; pidx += blockDim.x) {
        const Lev& e = st[pidx / Lk];
        const Lev& k = in[pidx % Lk];
        const int tm = min(e.Tmax - e.S - k.S, k.Tmax - k.S - e.S);
        if (tm < t0) continue;
        atomicMin(&G[min(tm, t0 + tn - 1) - t0], e.S + k.S);
    }
    __syncthreads();
    const int chunk = (tn + blockDim.x - 1) / blockDim.x;
    const int c0 = threadIdx.x * chunk, c1 = min(tn, c0 + chunk);
    int m = INT_MAX;
    for (int i = c1 - 1; i >= c0; i--) { m = min(m, G[i]); G[i] = m; }
    s_part[threadIdx.x] = m;
    __syncthreads();
    if (threadIdx.x < 32) {   // suffix minimum of the 256 chunk minima (8 per lane + a warp scan)
        int v[8], x = INT_MAX;
        for (int q = 7; q >= 0; q--) { x = min(x, s_part[threadIdx.x * 8 + q]); v[q] = x; }
        int y = x;
        for (int off = 1; off < 32; off <<= 1) {
            const int z = __shfl_down_sync(0xffffffffu, y, off);
            if (threadIdx.x + off < 32) y = min(y, z);
        }
        const int after = __shfl_down_sync(0xffffffffu, y, 1);
        const int tail = threadIdx.x < 31 ? after : INT_MAX;
        for (int q = 0; q < 8; q++) s_part[threadIdx.x * 8 + q] = min(v[q], tail);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < tn; i += blockDim.x) {   // coalesced
        const int c = i / chunk;
        ftab[(size_t)prob * FT_CAP + i] = min(G[i], c + 1 < (int)blockDim.x ? s_part[c + 1] : INT_MAX);
    }
}

// min over a lower-left hull of B y + S' z (y, z > 0): the edge slopes (B_i - B_i+1)/(S'_i+1 - S'_i)
// decrease along the chain, so the minimiser is the first vertex whose outgoing edge has
// slope <= z / y (binary search); its neighbours are evaluated too.  A vertex picked wrongly
// because of FP32 rounding of the slope test differs from the minimum by <= ~1e-6 relative
// (the misjudged edges have slopes within rounding of z/y), far inside the bound's margin.
__device__ __forceinline__ float hull_min(const float2* v, const float2* ed, int n, float y, float z) {
    int lo = 0, hi = n - 1;   // first edge index i in [0, n-1) with slope_i <= z/y, else n-1
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const float2 e = ed[mid];
        if (e.x * y > e.y * z) lo = mid + 1; else hi = mid;
    }
    float m = fmaf(v[lo].x, y, v[lo].y * z);
    if (lo > 0) m = fminf(m, fmaf(v[lo - 1].x, y, v[lo - 1].y * z));
    if (lo + 1 < n) m = fminf(m, fmaf(v[lo + 1].x, y, v[lo + 1].y * z));
    return m;
}
// the same with the minimiser found through the hull's slope table
__device__ __forceinline__ float hull_min_t(const float2* v, const float2* ed, int n, const uint8_t* T, int base, float y,
                                           float z) {
    const int lo = hull_arg(ed, n, T, base, y, z);
    float m = fmaf(v[lo].x, y, v[lo].y * z);
    if (lo > 0) m = fminf(m, fmaf(v[lo - 1].x, y, v[lo - 1].y * z));
    if (lo + 1 < n) m = fminf(m, fmaf(v[lo + 1].x, y, v[lo + 1].y * z));
    return m;
}

// min over the points of a lower-left hull's point set with S' in [slo, shi] of B y + S' z (y, z >= 0),
// bounded below: the objective along the hull is convex in S', so the constrained minimum is at the
// unconstrained minimiser when it lies in the range, else at the nearer end, where the hull's B is
// interpolated (beyond the last vertex -- the minimum-B point -- every point has B >= its B).  An
// argmin misjudged by FP32 rounding moves the value by ~1e-7 relative (adjacent vertices then have
// equal objectives up to rounding), far inside the callers' 1 - 2^-16 margin.
__device__ __forceinline__ float hull_min_in(const float2* v, const float2* ed, int n, float y, float z, float slo,
                                            float shi) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const float2 e = ed[mid];
        if (e.x * y > e.y * z) lo = mid + 1; else hi = mid;
    }
    const float s = v[lo].y;
    if (s >= slo && s <= shi) {
        float m = fmaf(v[lo].x, y, s * z);
        if (lo > 0) m = fminf(m, fmaf(v[lo - 1].x, y, v[lo - 1].y * z));
        if (lo + 1 < n) m = fminf(m, fmaf(v[lo + 1].x, y, v[lo + 1].y * z));
        return m;
    }
    const float c = s < slo ? slo : shi;
    if (c >= v[n - 1].y) return fmaf(v[n - 1].x, y, c * z);
    if (c <= v[0].y) return fmaf(v[0].x, y, c * z);
    int a = 0, b = n - 1;   // last vertex with S' <= c
    while (a < b) {
        const int mid = (a + b + 1) >> 1;
        if (v[mid].y <= c) a = mid; else b = mid - 1;
    }
    const float2 p = v[a], q = v[a + 1];
    const float B = fmaf(q.x - p.x, __fdividef(c - p.y, q.y - p.y), p.x);   // (2 ulp: inside the bound's margin)
    return fmaf(B, y, c * z);
}

// hull_min_in with the range ends given as inner S'-sorted positions ka <= kb: their S' (ssort) and
// the last hull vertex at or below each (hpos) are tabulated, so the clamp needs no search
__device__ __forceinline__ float hull_min_pos(const AuxView& A, int n, float y, float z, int ka, int kb) {
    const float2* v = A.ih;
    const int lo = hull_arg(A.ie, n, A.ht, *A.htb, y, z);
    const float s = v[lo].y, slo = (float)A.ssort[ka], shi = (float)A.ssort[kb];
    if (s >= slo && s <= shi) {
        float m = fmaf(v[lo].x, y, s * z);
        if (lo > 0) m = fminf(m, fmaf(v[lo - 1].x, y, v[lo - 1].y * z));
        if (lo + 1 < n) m = fminf(m, fmaf(v[lo + 1].x, y, v[lo + 1].y * z));
        return m;
    }
    const bool below = s < slo;
    const float c = below ? slo : shi;
    const int a = A.hpos[below ? ka : kb];
    if (a >= n - 1) return fmaf(v[n - 1].x, y, c * z);
    const float2 p = v[a], q = v[a + 1];
    const float B = fmaf(q.x - p.x, __fdividef(c - p.y, q.y - p.y), p.x);   // (2 ulp: inside the bound's margin)
    return fmaf(fmaxf(B, q.x), y, c * z);
}

// one thread per row: the bound above, times (1 - 2^-16) (covers its FP32 rounding, <= 16u, and
// the hull search), or +inf when no candidate of the row meets every QoS bound (exact)
template <int NW, bool QOS>
__global__ void __launch_bounds__(256) k_rowlb(Setup su, const Prob* probs, const Lev* levs, const float2* hull,
                                               const int32_t* ftab, const RowHdr* hdr, float* rowlb,
                                               unsigned* lbmin) {
    constexpr int NH = NW - 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* sh = reinterpret_cast<float2*>(smem_raw);   // [2][2][Lmax] + slope tables (hull_stride)
    __shared__ float red[8];
    const int prob = blockIdx.y;
    const Prob& P = probs[prob];
    if (P.status != 0) return;
    const int rp = P.rep;   // hulls, feasibility table and header of the representative (k_arep)
    const RowHdr H = hdr[rp];
    const int Lmax = su.Lmax;
    for (int i = threadIdx.x; i < (int)hull_stride(Lmax); i += blockDim.x) sh[i] = hull[(size_t)rp * hull_stride(Lmax) + i];
    const uint8_t* sht = reinterpret_cast<const uint8_t*>(sh + 4 * Lmax);
    __syncthreads();
    const Lev* base = levs + (size_t)prob * su.lev_stride;
    const uint64_t rows = P.units / (uint64_t)P.nseg;
    const int32_t* ft = ftab + (size_t)rp * FT_CAP;
    const float invf = P.inv;
    uint32_t Lh[NH > 0 ? NH : 1];
#pragma unroll
    for (int w = 0; w < NH; w++) Lh[w] = (uint32_t)P.L[w];
    float bm = INFINITY;
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (uint64_t)gridDim.x * blockDim.x) {
        int64_t hB = 0, hBS = 0;
        int hT = 0, hTm = 1 << 24;
        if (rows <= 0xffffffffull) {
            uint32_t x = (uint32_t)r;
#pragma unroll
            for (int w = NH - 1; w >= 0; w--) {
                const uint32_t d = x % Lh[w];
                x /= Lh[w];
                const Lev& v = base[(size_t)w * Lmax + d];
                hB += v.B; hBS += v.BS; hT += v.S; hTm = min(hTm, v.Tmax);
            }
        } else {
            uint64_t x = r;
#pragma unroll
            for (int w = NH - 1; w >= 0; w--) {
                const int d = (int)(x % (uint64_t)Lh[w]);
                x /= (uint64_t)Lh[w];
                const Lev& v = base[(size_t)w * Lmax + d];
                hB += v.B; hBS += v.BS; hT += v.S; hTm = min(hTm, v.Tmax);
            }
        }
        bool feas = true;
        if (QOS) {
            if (H.tn > 0) feas = ft[hT - H.t0] <= hTm - hT;
            else feas = !(H.smin_st > min(hTm - hT - H.smin_in, H.umax_in - hT) || H.umax_st < hT + H.smin_in);
        }
        float lb = INFINITY;
        if (feas) {
            const float hBf = __ll2float_rn(hB), hTf = (float)hT;
            const float Yh = fmaf(hTf, invf, 1.0f), Zh = hBf * invf;
            const u128 Dh = (u128)hT * (u128)hB - (u128)hBS;
            const float Dhf = (Dh >> 64) ? (float)(double)Dh : __ull2float_rn((unsigned long long)Dh);
            const float Xh = fmaf(Dhf, invf, hBf);
            const float Y2 = fmaf(H.Sminf_in, invf, Yh), Z2 = fmaf(H.Bminf_in, invf, Zh);
            lb = (Xh + hull_min_t(sh, sh + Lmax, H.nh[0], sht, H.htb[0], Y2, Z2) +
                  hull_min_t(sh + 2 * Lmax, sh + 3 * Lmax, H.nh[1], sht + HT_NB, H.htb[1], Yh, Zh)) *
                 0.99998474121f;   // 1 - 2^-16
        }
        rowlb[(size_t)prob * su.rows_max + r] = lb;
        bm = fminf(bm, lb);
    }
    for (int o = 16; o; o >>= 1) bm = fminf(bm, __shfl_xor_sync(0xffffffffu, bm, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = bm;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); i++) bm = fminf(bm, red[i]);
        if (bm < INFINITY) atomicMin(lbmin + prob, __float_as_uint(bm));
    }
}

constexpr int BB_NB = 256;
constexpr float BB_SCALE = 1024.0f;
// bucket of a bound: floor((lb / lbm - 1) BB_SCALE), the quotient as lb times the correctly rounded reciprocal of
// lbm (every caller passes inv = __frcp_rn(lbm), so list building and the stop test agree exactly; the product's
// rounding is far inside bb_edge's one bucket of slack)
__device__ __forceinline__ int bb_bucket(float lb, float inv) {
    const float r = __fmul_rn(__fsub_rn(__fmul_rn(lb, inv), 1.0f), BB_SCALE);
    return r <= 0.0f ? 0 : (r >= (float)(BB_NB - 1) ? BB_NB - 1 : (int)r);
}
// a value <= every bound in bucket b (one bucket of slack covers the rounding of bb_bucket)
__device__ __forceinline__ float bb_edge(int b, float lbm) { return b <= 1 ? 0.0f : lbm * (1.0f + (float)(b - 1) / BB_SCALE); }

// Row bound + best-first list in one kernel, for batches where one pass-1 item is a whole
// problem (nseg = 1, one item per problem, unsharded) and its rows fit in shared memory (C5):
// one CTA per problem computes every row's bound into shared memory (hi records and hull staged
// there), the problem's minimum bound, and the bucket-ordered unit list -- the bounds never go
// to global memory.  Same arithmetic as k_rowlb + k_bucket.
#ifndef RLF_THREADS_N
#define RLF_THREADS_N 512
#endif
constexpr int RLF_THREADS = RLF_THREADS_N;
constexpr int RLF_ROWS_CAP = 24576;
template <int NW, bool QOS>
__global__ void __launch_bounds__(RLF_THREADS) k_rowlb_fused(Setup su, const Prob* probs, const Lev* levs,
                                                             const float2* hull, const int32_t* ftab,
                                                             const RowHdr* hdr, unsigned* lbmin, uint2* ulist,
                                                             int32_t* ulist_n) {
    pdl_wait();      // (programmatic dependent launch: the predecessor's results are visible)
    pdl_trigger();
    constexpr int NH = NW - 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int Lmax = su.Lmax;
    // hulls + edges + slope tables; the hi workers' records as separate arrays (lanes read consecutive
    // levels: one bank per lane); every row's bound; a bit per row with a finite bound
    float2* sh = reinterpret_cast<float2*>(smem_raw);
    int64_t* hB = reinterpret_cast<int64_t*>(sh + hull_stride(Lmax));   // [NH][Lmax]
    int64_t* hBS = hB + NH * Lmax;                                      // [NH][Lmax]
    int32_t* hS = reinterpret_cast<int32_t*>(hBS + NH * Lmax);          // [NH][Lmax]
    int32_t* hTx = hS + NH * Lmax;                                      // [NH][Lmax]
    float* lbs = reinterpret_cast<float*>(hTx + NH * Lmax);             // [rows]
    uint32_t* fbit = reinterpret_cast<uint32_t*>(lbs + su.rows_max);    // [ceil(rows / 32)]
    __shared__ float red[RLF_THREADS / 32];
    __shared__ int hist[BB_NB], cur[BB_NB];
    const int prob = blockIdx.x;
    const Prob& P = probs[prob];
    if (P.status != 0) {
        if (threadIdx.x == 0) ulist_n[prob] = 0;
        return;
    }
    const int rp = P.rep;   // hulls, feasibility table and header of the representative (k_arep)
    const RowHdr H = hdr[rp];
    const Lev* base = levs + (size_t)prob * su.lev_stride;
    for (int i = threadIdx.x; i < (int)hull_stride(Lmax); i += blockDim.x) sh[i] = hull[(size_t)rp * hull_stride(Lmax) + i];
    const uint8_t* sht = reinterpret_cast<const uint8_t*>(sh + 4 * Lmax);
    for (int i = threadIdx.x; i < NH * Lmax; i += blockDim.x) {
        const Lev v = base[i];
        hB[i] = v.B; hBS[i] = v.BS; hS[i] = (int32_t)v.S; hTx[i] = v.Tmax;
    }
    for (int i = threadIdx.x; i < BB_NB; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t rows = (uint32_t)P.units;
    const int32_t* ft = ftab + (size_t)rp * FT_CAP;
    const float invf = P.inv;
    uint32_t Lh[NH > 0 ? NH : 1];
#pragma unroll
    for (int w = 0; w < NH; w++) Lh[w] = (uint32_t)P.L[w];
    ECLIP_CHECK(rows <= (uint32_t)su.rows_max && (NH != 2 || rows == Lh[0] * Lh[NH > 1 ? 1 : 0]));
    auto feasible = [&](int hT, int hTm) -> bool {
        if (!QOS) return true;
        if (H.tn > 0) return ft[hT - H.t0] <= hTm - hT;
        return !(H.smin_st > min(hTm - hT - H.smin_in, H.umax_in - hT) || H.umax_st < hT + H.smin_in);
    };
    // Dhf: (float) sum over the hi workers of B_w (hT - S'_w) >= 0 (computed by the caller)
    auto row_lb = [&](int64_t hBv, float Dhf, int hT) -> float {
        const float hBf = __ll2float_rn(hBv), hTf = (float)hT;
        const float Yh = fmaf(hTf, invf, 1.0f), Zh = hBf * invf;
        const float Xh = fmaf(Dhf, invf, hBf);
        const float Y2 = fmaf(H.Sminf_in, invf, Yh), Z2 = fmaf(H.Bminf_in, invf, Zh);
        return (Xh + hull_min_t(sh, sh + Lmax, H.nh[0], sht, H.htb[0], Y2, Z2) +
                hull_min_t(sh + 2 * Lmax, sh + 3 * Lmax, H.nh[1], sht + HT_NB, H.htb[1], Yh, Zh)) *
               0.99998474121f;   // 1 - 2^-16
    };
    // rows strided over every thread: warp w of pass it handles the 32 consecutive rows of bitmap word
    // it * (RLF_THREADS / 32) + w
    float bm = INFINITY;
    const int nwords = (int)((rows + 31) >> 5);
    const int lane = threadIdx.x & 31;
    const float rL1 = __frcp_rn((float)Lh[NH > 1 ? 1 : 0]);
    for (int r0 = threadIdx.x - lane; r0 < (int)rows; r0 += RLF_THREADS) {
        const int r = r0 + lane;
        float lb = INFINITY;
        if (r < (int)rows) {
            if (NH == 2) {
                // rows = (d0, d1), d1 least significant; d0 = r / L1 from a float quotient corrected by one
                // step (r < 2^24)
                const int L1 = (int)Lh[1];
                int d0 = __float2int_rz((float)r * rL1);
                if (d0 * L1 > r) d0--;
                else if ((d0 + 1) * L1 <= r) d0++;
                const int d1 = r - d0 * L1 + Lmax;
                ECLIP_CHECK(d0 >= 0 && d0 < (int)Lh[0] && d1 >= Lmax && d1 < Lmax + L1);
                const int hT = hS[d0] + hS[d1];
                if (feasible(hT, min(hTx[d0], hTx[d1]))) {
                    // two hi workers: sum_w B_w (hT - S'_w) = B_0 S'_1 + B_1 S'_0, non-negative terms (rounding
                    // <= 3u, inside the bound's 1 - 2^-16 margin)
                    const int64_t b0 = hB[d0], b1 = hB[d1];
                    const float Dhf = fmaf(__ll2float_rn(b0), (float)hS[d1], __ll2float_rn(b1) * (float)hS[d0]);
                    lb = row_lb(b0 + b1, Dhf, hT);
                }
            } else {
                int64_t sB = 0, sBS = 0;
                int hT = 0, hTm = 1 << 24;
                uint32_t x = (uint32_t)r;
#pragma unroll
                for (int w = NH - 1; w >= 0; w--) {
                    const uint32_t d = x % Lh[w];
                    x /= Lh[w];
                    const int i = w * Lmax + (int)d;
                    sB += hB[i]; sBS += hBS[i]; hT += hS[i]; hTm = min(hTm, hTx[i]);
                }
                if (feasible(hT, hTm)) {
                    const u128 Dh = (u128)hT * (u128)sB - (u128)sBS;
                    const float Dhf = (Dh >> 64) ? (float)(double)Dh : __ull2float_rn((unsigned long long)Dh);
                    lb = row_lb(sB, Dhf, hT);
                }
            }
            lbs[r] = lb;
            bm = fminf(bm, lb);
        }
        const unsigned fb = __ballot_sync(0xffffffffu, lb < INFINITY);
        if (lane == 0 && r0 < (int)rows) fbit[r0 >> 5] = fb;
    }
    for (int o = 16; o; o >>= 1) bm = fminf(bm, __shfl_xor_sync(0xffffffffu, bm, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = bm;
    __syncthreads();
    bm = red[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); i++) bm = fminf(bm, red[i]);
    if (threadIdx.x == 0) lbmin[prob] = __float_as_uint(bm);   // +inf bits when no row is feasible
    if (!(bm < INFINITY)) {
        if (threadIdx.x == 0) ulist_n[prob] = 0;
        return;
    }
    const float bminv = __frcp_rn(bm);
    // bucket histogram and scatter over the rows with a finite bound, a row per lane (warp w takes bitmap words
    // w, w + 16, ...); the last bucket -- every bound >= 1.249 x the smallest, most rows -- counted and placed with
    // one atomic per warp, the others with one per row
    const int warp = threadIdx.x >> 5;
    for (int wd = warp; wd < nwords; wd += RLF_THREADS / 32) {
        const uint32_t fw = fbit[wd];
        if (!fw) continue;
        const bool has = (fw >> lane) & 1u;
        const int b = has ? bb_bucket(lbs[wd * 32 + lane], bminv) : -1;
        ECLIP_CHECK(!has || (wd * 32 + lane < (int)rows && b >= 0 && b < BB_NB));
        const unsigned top = __ballot_sync(0xffffffffu, b == BB_NB - 1);
        if (has && b != BB_NB - 1) atomicAdd(&hist[b], 1);
        if (lane == 0 && top) atomicAdd(&hist[BB_NB - 1], __popc(top));
    }
    __syncthreads();
    if (threadIdx.x < 32) {   // exclusive scan of the 256 counts (8 per lane)
        int v[BB_NB / 32], t = 0;
        for (int i = 0; i < BB_NB / 32; i++) { v[i] = hist[threadIdx.x * (BB_NB / 32) + i]; t += v[i]; }
        int xx = t;
        for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, xx, o); if (threadIdx.x >= o) xx += y; }
        int run = xx - t;
        for (int i = 0; i < BB_NB / 32; i++) { cur[threadIdx.x * (BB_NB / 32) + i] = run; run += v[i]; }
        if (threadIdx.x == 31) ulist_n[prob] = xx;
    }
    __syncthreads();
    uint2* out = ulist + (size_t)prob * su.upi;
    for (int wd = warp; wd < nwords; wd += RLF_THREADS / 32) {
        const uint32_t fw = fbit[wd];
        if (!fw) continue;
        const bool has = (fw >> lane) & 1u;
        const uint32_t r = (uint32_t)(wd * 32 + lane);
        const float lb = has ? lbs[r] : INFINITY;
        const int b = has ? bb_bucket(lb, bminv) : -1;
        const unsigned top = __ballot_sync(0xffffffffu, b == BB_NB - 1);
        int p0 = 0;
        if (lane == 0 && top) p0 = atomicAdd(&cur[BB_NB - 1], __popc(top));
        p0 = __shfl_sync(0xffffffffu, p0, 0);
        if (has) {
            const int pos = b == BB_NB - 1 ? p0 + __popc(top & ((1u << lane) - 1u)) : atomicAdd(&cur[b], 1);
            ECLIP_CHECK(pos >= 0 && pos < (int)rows && (size_t)pos < (size_t)su.upi);
            out[pos] = make_uint2(r, __float_as_uint(lb));
        }
    }
}

__global__ void k_fill_u32(unsigned* p, size_t n, unsigned v) {
    pdl_wait();      // (programmatic dependent launch: the predecessor's results are visible)
    pdl_trigger();
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

// up to four fills in one launch (the planner chain: no memset between programmatically serialised kernels)
struct Fill4 {
    unsigned* p[4];
    size_t n[4];
    unsigned v[4];
};
__global__ void k_fill4(Fill4 f) {
    pdl_wait();
    pdl_trigger();
    for (int j = 0; j < 4; j++)
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < f.n[j]; i += (size_t)gridDim.x * blockDim.x)
            f.p[j][i] = f.v[j];
}
static cudaError_t fill4(const Fill4& f, cudaStream_t st) {
    size_t mx = 0;
    for (int j = 0; j < 4; j++) mx = std::max(mx, f.p[j] ? f.n[j] : 0);
    if (mx == 0) return cudaSuccess;
    const size_t blocks = std::min<size_t>((mx + 255) / 256, 148 * 8);
    return launch_pdl(k_fill4, dim3((unsigned)blocks), dim3(256), 0, st, f);
}

// ------------------------------------------------------------------------------------------
// pass 1
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned team_mask(int T) {
    if (T >= 32) return 0xffffffffu;
    unsigned base = ((threadIdx.x & 31u) / (unsigned)T) * (unsigned)T;
    return ((1u << T) - 1u) << base;
}
__device__ __forceinline__ float team_min(float m, int T, unsigned mask) {
    for (int o = T / 2; o > 0; o >>= 1) m = fminf(m, __shfl_xor_sync(mask, m, o));
    return m;
}

__device__ float band_bound(const Setup& su, float m, float ms) {
    // every candidate with exact key <= H*(1+tau) has key32 <= bound; H* <= ms / (1 - delta)
    double base = qos_float(su) ? (double)ms : (double)m;
    if (isinf(base)) return INFINITY;
    double tau = (double)su.tol_num / (double)su.tol_den;
    double b = base * (1.0 + tau) * (1.0 + su.delta) / (1.0 - su.delta) * (1.0 + 1e-12);
    return __double2float_ru(b);
}

// inner worker (S'-sorted): khi = #{k : S'_k <= c1}; klo = min{k : usuf[k] >= Tp}
__device__ __forceinline__ int inner_khi(const AuxView& A, int c1, int s0, int slast, bool khi_ok, int Lin) {
    if (c1 < s0) return 0;
    if (c1 >= slast) return Lin;
    if (khi_ok) return (int)A.khi[c1 - s0];
    int lo = 0, hi = Lin;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (A.ssort[mid] <= c1) lo = mid + 1; else hi = mid; }
    return lo;
}
__device__ __forceinline__ int inner_klo(const AuxView& A, int Tp, int u0v, int ulast, bool klo_ok, int Lin) {
    if (Tp <= u0v) return 0;
    if (Tp > ulast) return Lin;
    if (klo_ok) return (int)A.klo[Tp - u0v];
    int lo = 0, hi = Lin;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (A.usuf[mid] >= Tp) hi = mid; else lo = mid + 1; }
    return lo;
}

struct HiSums {
    int64_t B, BS;
    int32_t T, Tm;
};
// exact sums over the hi workers 0..W-3
__device__ __forceinline__ HiSums hi_sums(const Lev* sl, int Lmax, const int* d, int W) {
    HiSums h;
    h.B = 0; h.BS = 0; h.T = 0; h.Tm = 1 << 24;
    for (int w = 0; w < W - 2; w++) {
        const Lev& r = sl[w * Lmax + d[w]];
        h.B += r.B; h.BS += r.BS; h.T += r.S; h.Tm = min(h.Tm, r.Tmax);
    }
    return h;
}

__device__ __forceinline__ void item_of_block(const Setup& su, const Prob& P, int li, uint64_t* item, bool* ok) {
    uint64_t slo, shi;
    shard_items(P.n_items, su.shard, su.n_shards, &slo, &shi);
    *item = slo + (uint64_t)li;
    *ok = *item < shi;
}

// Fast filter: SUM objective with EXCLUDE_SELF or PAPER_AS_WRITTEN.
// With exact prefix sums (Bp, BSp, Tp) over workers 0..W-2 and the inner level (B_i, S'_i),
// the SUM key  sum_w B_w (1 + O_w / (Lambda N))  is, exactly,
//   EXCLUDE_SELF:  K = X_p + B_i Y_p + S'_i Z_p,         X_p = Bp + (Tp Bp - BSp) / (Lambda N)
//   PAPER:         K = X_p + B_i Y_p + S'_i Z_p + D_i,   X_p = Bp (1 + Tp / (Lambda N))
//   Y_p = 1 + Tp / (Lambda N),   Z_p = Bp / (Lambda N),   D_i = B_i S'_i / (Lambda N),
// every term >= 0.  Per candidate: 2 FMAs (packed f32x2: one issue slot per two candidates)
// + a 3-input min; FP32 relative error <= 8u.
// Mapping: a warp owns a unit (one hi-digit row x one segment of the step worker).  Its
// lanes build a compacted table of the usable step levels, then each lane takes its own
// entries and sweeps the inner worker's levels (S'-sorted, broadcast from shared memory)
// over the exact QoS-feasible range:
//   prefix workers' QoS:  S'_k <= c1 = min_w Tmax_w - Tp   ->  k < k_hi   (prefix of sorted order)
//   inner worker's QoS:   Tp <= u_k = Tmax_k - S'_k        ->  k >= k_lo where k_lo is the first
//       index of the suffix-minimum of u that reaches Tp (exact when u is non-decreasing in S',
//       i.e. B* non-increasing; otherwise the earlier levels are swept with a mask).
// Both ends come from lookup tables indexed by value (binary search if a range is too wide).
// Row pruning (BB): a unit is processed only if its row bound lies in this
// wave's window (lbmin*lo_f, lbmin*hi_f] and below the band of the problem's incumbent `inc`
// (the smallest FP32 key found so far, updated here); skipped units keep submin = +inf.
// pruned pass 1: submin[prob][u] holds a value only if bit u of the problem's written-unit bitmap is set
__device__ __forceinline__ size_t wbits_words(const Setup& su) { return (size_t)((su.units_max + 31) >> 5); }
__device__ __forceinline__ float sub_at(const Setup& su, const float* sp, const uint32_t* wb, int p, uint64_t u) {
    if (wb && !((wb[(size_t)p * wbits_words(su) + (u >> 5)] >> (u & 31)) & 1u)) return INFINITY;
    return sp[u];
}
struct BBArgs {
    const uint2* ulist;         // [grid][upi] this item's candidate units {unit - ua, bound bits}, bucket-ordered
    const int32_t* ulist_n;     // [grid]
    const unsigned* lbmin;      // [n] smallest row bound of the problem (float bits)
    unsigned* inc;              // [n] global incumbent (float bits)
    unsigned long long* rows_done;  // [6]: units fetched within the band, units with >= 1 swept entry, entries swept, units past
                                    //   the unit bound, units with >= 1 chunk kept, chunks kept
    uint32_t* plist;            // [n * PL_CAP] processed units with a finite minimum
    int32_t* plist_n;
    uint32_t* wbits;            // [n][ceil(units_max / 32)] units whose submin this launch wrote
    const float2* hull;         // [n][2][2][Lmax] (k_prep_bound): the inner worker's hull at [2][0], edges [2][1]
    const RowHdr* rowhdr;       // [n] hull sizes
};
// Best-first order: each item's units with a finite row bound are listed by
// bucket of bound / (smallest bound of the problem) - 1 in steps of 1/BB_SCALE (counting sort,
// k_bucket), so the rows most likely to hold the optimum set the incumbent first, and the list
// can be abandoned as soon as a bucket's lower edge leaves the incumbent's band.
// one CTA per pass-1 item: counting sort of the item's units with a finite row bound by bucket
__global__ void __launch_bounds__(256) k_bucket(Setup su, const Prob* probs, const float* rowlb, const unsigned* lbmin,
                                                uint2* ulist, int32_t* ulist_n) {
    __shared__ int hist[BB_NB], cur[BB_NB];
    const int ipS = (su.items_max + su.n_shards - 1) / su.n_shards;
    const int prob = blockIdx.x / ipS;
    const Prob& P = probs[prob];
    uint64_t item = 0;
    bool ok = P.status == 0;
    if (ok) item_of_block(su, P, blockIdx.x % ipS, &item, &ok);
    if (!ok) {
        if (threadIdx.x == 0) ulist_n[blockIdx.x] = 0;
        return;
    }
    uint64_t ua = item * (uint64_t)su.upi, ub = ua + (uint64_t)su.upi;
    if (ub > P.units) ub = P.units;
    const int nseg = P.nseg;
    const float* rlb = rowlb + (size_t)prob * su.rows_max;
    const float lbm = __uint_as_float(lbmin[prob]);
    const float lbminv = __frcp_rn(lbm);
    for (int i = threadIdx.x; i < BB_NB; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (uint64_t u = ua + threadIdx.x; u < ub; u += blockDim.x) {
        const float lb = rlb[nseg == 1 ? u : u / (uint64_t)nseg];
        if (lb < INFINITY) atomicAdd(&hist[bb_bucket(lb, lbminv)], 1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {   // exclusive scan of the 256 counts (8 per lane)
        int v[BB_NB / 32], t = 0;
        for (int i = 0; i < BB_NB / 32; i++) { v[i] = hist[threadIdx.x * (BB_NB / 32) + i]; t += v[i]; }
        int x = t;
        for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, x, o); if (threadIdx.x >= o) x += y; }
        int run = x - t;
        for (int i = 0; i < BB_NB / 32; i++) { cur[threadIdx.x * (BB_NB / 32) + i] = run; run += v[i]; }
        if (threadIdx.x == 31) ulist_n[blockIdx.x] = x;
    }
    __syncthreads();
    uint2* out = ulist + (size_t)blockIdx.x * su.upi;
    for (uint64_t u = ua + threadIdx.x; u < ub; u += blockDim.x) {
        const float lb = rlb[nseg == 1 ? u : u / (uint64_t)nseg];
        if (lb < INFINITY) out[atomicAdd(&cur[bb_bucket(lb, lbminv)], 1)] = make_uint2((unsigned)(u - ua), __float_as_uint(lb));
    }
}

template <int NW, int MODE, bool QOS, bool BB>
#ifndef P1_MINB
#define P1_MINB 4
#endif
#ifndef P1_NE
#define P1_NE 4   // entries per lane in the exhaustive pass without QoS
#endif
#ifndef P1_MINB_EXH
#define P1_MINB_EXH 3   // that pass: registers for independent temporaries of its 4 entries (ILP) over a 4th CTA
#endif
__global__ void __launch_bounds__(P1_THREADS, (!QOS && !BB && NW >= 2) ? P1_MINB_EXH : P1_MINB)
k_pass1_fast(Setup su, const Prob* __restrict__ probs, const Lev* __restrict__ levs, float* __restrict__ submin,
             unsigned long long* __restrict__ feasible, BBArgs bb) {
    pdl_wait();      // (programmatic dependent launch: the predecessor's results are visible)
    pdl_trigger();
    constexpr int NH = NW >= 2 ? NW - 2 : 0;   // hi workers (fixed inside a unit)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ uint64_t bar;
    const int ipS = (su.items_max + su.n_shards - 1) / su.n_shards;
    const int prob = blockIdx.x / ipS;
    const Prob& P = probs[prob];
    if (P.status != 0) return;
    uint64_t item;
    bool ok;
    item_of_block(su, P, blockIdx.x % ipS, &item, &ok);
    if (!ok) return;
    const int W = NW, Lmax = su.Lmax;
    const uint64_t units = P.units;
    uint64_t ua = item * (uint64_t)su.upi, ub = ua + (uint64_t)su.upi;
    if (ub > units) ub = units;
    const int nseg = P.nseg;
    __shared__ unsigned s_inc;
    __shared__ int s_next;   // next list entry to fetch; raised to the list length to stop every warp
    __shared__ uint8_t s_chunk[P1_THREADS / 32][32];
    float lbm = 0.0f;
    int lcnt = 0;
    const uint2* lst = nullptr;
    if (BB) {   // leave before staging if no unit of this item can hold a feasible candidate
        lcnt = bb.ulist_n[blockIdx.x];
        if (lcnt == 0) return;
        lst = bb.ulist + (size_t)blockIdx.x * su.upi;
        lbm = __uint_as_float(bb.lbmin[prob]);
        if (threadIdx.x == 0) { s_inc = 0x7f800000u; s_next = 0; }
    }
    Lev* sl = reinterpret_cast<Lev*>(smem_raw);
    // level records + the aux block (this problem's, or its representative's) by TMA bulk copies
    if (P.rep == prob)
        stage_levels(sl, levs + (size_t)prob * su.lev_stride, (unsigned)(W * Lmax * sizeof(Lev) + su.aux_bytes), &bar);
    else
        stage_levels2(sl, levs + (size_t)prob * su.lev_stride, (unsigned)(W * Lmax * sizeof(Lev)),
                      levs + (size_t)P.rep * su.lev_stride + (size_t)W * Lmax, (unsigned)su.aux_bytes, &bar);
    const AuxView A = aux_view(smem_raw + (size_t)W * Lmax * sizeof(Lev), Lmax);
    const int nhv = *A.ihn;   // inner hull vertex count (staged with the aux block)

    int L[NW];
#pragma unroll
    for (int w = 0; w < NW; w++) L[w] = P.L[w];
    const int Lin = L[NW - 1];
    const Lev* stepw = sl + (W >= 2 ? (W - 2) : 0) * Lmax;
    const int segl = P.seglen, Lstep = P.Lstep;
    float4* tab0 = reinterpret_cast<float4*>(smem_raw + (size_t)W * Lmax * sizeof(Lev) + su.aux_bytes);
    const int warp = threadIdx.x >> 5, wl = threadIdx.x & 31;
    constexpr int NWARP = P1_THREADS / 32;
    // exhaustive without QoS: two table entries per lane (one read of an inner pair serves both)
    constexpr bool TWO = !QOS && !BB && NW >= 2;   // (W = 1: no step worker; the table path)
    constexpr int TABN = 32;   // (TWO keeps its entries in registers)
    float4* tab = tab0 + (size_t)warp * TABN;                                                    // {X,Y,Z,Tp}
    int2* tabk = reinterpret_cast<int2*>(tab0 + (size_t)NWARP * TABN) + (size_t)warp * TABN;     // {k_lo, k_hi}
    const float invf = P.inv;
    const double invd = 1.0 / (double)P.lamN;
    const int s0 = A.hdr[0], u0v = A.hdr[1];
    const bool khi_ok = A.hdr[2] != 0, klo_ok = A.hdr[3] != 0;
    const int smin_i = A.ssort[0], umax_i = A.umaxp[Lin], slast = A.ssort[Lin - 1], ulast = A.usuf[Lin - 1];
    const int ss0 = A.hdr[4], su0 = A.hdr[5];
    const bool step_tab = W >= 2 && A.hdr[6] != 0 && A.hdr[7] != 0;
    const int shi_n = step_tab ? A.stS[P.Lstep - 1] - ss0 + 1 : 0;
    const int sulast = step_tab ? A.stU[P.Lstep - 1] : 0;
    float* subp = submin + (size_t)prob * su.units_max;

    // BB: warps take 32 list entries at a time (best-first), process the ones within the band of the
    // incumbent, and stop when the rest of the list is provably outside it.  Otherwise: 32
    // consecutive units per round, rounds strided by NWARP * 32.
    unsigned long long nfeas = 0;
    unsigned ndone = 0, nue = 0, nent = 0, nuok = 0, nuch = 0, nch = 0;   // per-lane counts (32-bit: registers)
    float bnd = INFINITY, incv = INFINITY, bnd_of = -1.0f;
    // band factor of the linear modes, rounded up once: bnd = m x bandf (rounded up) >= band_bound(m)
    const float bandf = __double2float_ru((1.0 + (double)su.tol_num / (double)su.tol_den) * (1.0 + su.delta) /
                                          (1.0 - su.delta) * (1.0 + 1e-12));
    // unit constants (row decode, exact QoS range cut on the step worker, row constants X_h, Y_h, Z_h),
    // computed by one lane per unit right after a fetch and broadcast to the warp when the unit is
    // processed; false: no step level of the unit is usable (its minimum stays +inf)
    // chunk bound of aligned chunk c of the S'-sorted step levels: for a chunk with smallest
    // S' = Sa and smallest B = Bm, every key of its entries is
    //   >= (Xh + Bm Yh + Sa Zh) + (Yh + Sa/LN) minB_k + (Zh + Bm/LN) minS_k
    // over the inner range that is QoS-feasible at T' = hT + Sa (a superset of every entry's); true: keep
    auto chunk_keep = [&](int c, int hT, int hTm, float Xh, float Yh, float Zh) -> bool {
        const int Sa = A.stS[c * P1_CS];
        const float Bm = A.chB[c];
        const int Tp = hT + Sa;
        const int khi2 = inner_khi(A, hTm - Tp, s0, slast, khi_ok, Lin);
        const int klo2 = inner_klo(A, Tp, u0v, ulast, klo_ok, Lin);
        const int ka = A.umaxp[klo2] >= Tp ? 0 : klo2;
        if (khi2 <= ka) return false;
        const float Sf = (float)Sa;
        const float Xc = fmaf(Bm, Yh, fmaf(Sf, Zh, Xh));
        const float Yc = fmaf(Sf, invf, Yh), Zc = fmaf(Bm, invf, Zh);
        float lbc = fmaf(Yc, A.preminB[khi2], fmaf(Zc, (float)A.ssort[ka], Xc));
        if (!(lbc * 0.99998474121f > bnd)) lbc = fmaxf(lbc, Xc + hull_min_pos(A, nhv, Yc, Zc, ka, khi2 - 1));
        return !(lbc * 0.99998474121f > bnd);   // 1 - 2^-16
    };
    auto unit_consts = [&](uint64_t unit, int& oT, int& oTm, int& oSb, int& oEa, int& oNe, float& oX, float& oY,
                           float& oZ, uint32_t& oCm, bool& oCh) -> bool {
            int seg;
            HiSums h;
            h.B = 0; h.BS = 0; h.T = 0; h.Tm = 1 << 24;
            int64_t hb[2] = {0, 0};
            int hs[2] = {0, 0};
            bool two = false;   // two hi workers decoded by the 32-bit path: the cross term in FP32 below
            if (units <= 0xffffffffull) {   // 32-bit decode (the common case)
                two = NH == 2;
                uint32_t row = (uint32_t)unit;
                if (nseg > 1) { seg = (int)(row % (uint32_t)nseg); row /= (uint32_t)nseg; } else seg = 0;
    #pragma unroll
                for (int w = NH - 1; w >= 0; w--) {
                    uint32_t dw = row;   // worker 0 is the most significant digit: row < L[0] there
                    if (w > 0) {
                        dw = row % (uint32_t)L[w];
                        row /= (uint32_t)L[w];
                    }
                    const Lev& r = sl[w * Lmax + dw];
                    h.B += r.B; h.BS += r.BS; h.T += r.S; h.Tm = min(h.Tm, r.Tmax);
                    if (NH == 2) { hb[w] = r.B; hs[w] = r.S; }
                }
            } else {
                seg = (int)(unit % (uint64_t)nseg);
                uint64_t row = unit / (uint64_t)nseg;
    #pragma unroll
                for (int w = NH - 1; w >= 0; w--) {
                    const int dw = (int)(row % (uint64_t)L[w]);
                    row /= (uint64_t)L[w];
                    const Lev& r = sl[w * Lmax + dw];
                    h.B += r.B; h.BS += r.BS; h.T += r.S; h.Tm = min(h.Tm, r.Tmax);
                }
            }
            const int e0 = seg * segl, e1 = min(Lstep, e0 + segl);
            int ne = e1 - e0;
            int sb = 1 << 30;
            int ea = e0;
            if (QOS) {
                sb = min(h.Tm - h.T - smin_i, umax_i - h.T);
                if (W >= 2 && A.stS[e0] > sb) return false;   // even the smallest step level is infeasible
                if (step_tab) {
                    // usable step levels: S'_e <= sb (a prefix) and u_e >= hT + min S'_k (a suffix of the
                    // suffix-minimum; the prefix maximum says whether earlier levels could qualify)
                    const int eb = (sb - ss0 >= shi_n) ? Lstep : (int)A.shi[sb - ss0];
                    const int need = h.T + smin_i;
                    int lo = (need <= su0) ? 0 : ((need > sulast) ? Lstep : (int)A.slo[need - su0]);
                    if (lo > 0 && A.stUmax[lo - 1] >= need) lo = 0;
                    ea = lo;
                    ne = eb - lo;
                    if (ne <= 0) return false;
                }
            }
            // row constants: the prefix terms are bilinear in the step level (BS_e = B_e S'_e):
            //   X_e = Xh + B_e Yh + S'_e Zh (+ D_e for PAPER),  Y_e = Yh + S'_e inv,  Z_e = Zh + B_e inv
            const float hBf = __ll2float_rn(h.B), hTf = (float)h.T;
            const float Yh = fmaf(hTf, invf, 1.0f), Zh = hBf * invf;
            float Xh;
            if (MODE == M_EXCL) {
                float Dhf;   // = sum_hi B_w (hT - S'_w) >= 0
                if (NH == 2 && two) {   // B_0 S'_1 + B_1 S'_0: non-negative terms, <= 4u (inside delta)
                    Dhf = fmaf(__ll2float_rn(hb[0]), (float)hs[1], __ll2float_rn(hb[1]) * (float)hs[0]);
                } else {
                    const u128 Dh = (u128)h.T * (u128)h.B - (u128)h.BS;
                    Dhf = (Dh >> 64) ? (float)(double)Dh : __ull2float_rn((unsigned long long)Dh);
                }
                Xh = fmaf(Dhf, invf, hBf);
            } else {
                Xh = hBf * Yh;
            }
        oT = h.T; oTm = h.Tm; oSb = sb; oEa = ea; oNe = ne; oX = Xh; oY = Yh; oZ = Zh;
        if (BB && QOS && step_tab && W >= 2) {
            // unit bound: the chunk bound with every usable step level as one chunk (smallest S' = S'_ea,
            // smallest B >= the suffix minimum from ea's chunk); decided against the band at fetch time
            // (the band only tightens afterwards)
            const int Sa = A.stS[ea];
            const float Bm = A.chBs[ea / P1_CS];
            const int Tp = h.T + Sa;
            const int khi2 = inner_khi(A, h.Tm - Tp, s0, slast, khi_ok, Lin);
            const int klo2 = inner_klo(A, Tp, u0v, ulast, klo_ok, Lin);
            const int ka = A.umaxp[klo2] >= Tp ? 0 : klo2;
            if (khi2 <= ka) return false;
            const float Sf = (float)Sa;
            const float Xc = fmaf(Bm, Yh, fmaf(Sf, Zh, Xh));
            const float Yc = fmaf(Sf, invf, Yh), Zc = fmaf(Bm, invf, Zh);
            float lbu = fmaf(Yc, A.preminB[khi2], fmaf(Zc, (float)A.ssort[ka], Xc));
            if (!(lbu * 0.99998474121f > bnd)) lbu = fmaxf(lbu, Xc + hull_min_pos(A, nhv, Yc, Zc, ka, khi2 - 1));
            if (lbu * 0.99998474121f > bnd) return false;
            // the chunk filter, by this lane for its own unit (at fetch time: units whose every chunk is out of the
            // band never reach the warp-wide processing below)
            const int c_lo = ea / P1_CS, c_hi = (ea + ne + P1_CS - 1) / P1_CS;
            if (c_hi - c_lo <= 32) {
                uint32_t m = 0;
                for (int c = c_lo; c < c_hi; c++)
                    if (chunk_keep(c, h.T, h.Tm, Xh, Yh, Zh)) m |= 1u << (c - c_lo);
                if (!m) return false;
                oCm = m;
                oCh = true;
            }
        }
        return true;
    };
    constexpr uint64_t RSTEP = (uint64_t)NWARP * 32;
    uint64_t rbase = ua + (uint64_t)warp * 32;
    int nfetch = 0;
    for (;;) {
        unsigned pend;
        uint32_t loff = 0;
        float lbv = INFINITY;
        uint64_t base = 0;
        if (BB) {
            int b0 = 0;
            if (wl == 0) {
                b0 = atomicAdd(&s_next, 32);
                if ((nfetch++ & 3) == 0) atomicMin(&s_inc, *(volatile const unsigned*)(bb.inc + prob));
            }
            b0 = __shfl_sync(0xffffffffu, b0, 0);
            if (b0 >= lcnt) break;
            const int e = b0 + wl;
            const uint2 en = e < lcnt ? lst[e] : make_uint2(0u, 0x7f800000u);
            ECLIP_CHECK(lcnt <= su.upi && (e >= lcnt || ua + en.x < ub));
            loff = en.x;
            const float lb = __uint_as_float(en.y);
            lbv = lb;
            unsigned ci = 0;   // one read, broadcast (warp-uniform bound)
            if (wl == 0) ci = *(volatile unsigned*)&s_inc;
            incv = __uint_as_float(__shfl_sync(0xffffffffu, ci, 0));
            if (incv != bnd_of) { bnd = __fmul_ru(incv, bandf); bnd_of = incv; }
            // spare lanes of the list's last batch (e >= lcnt) are masked out explicitly: with no
            // incumbent yet bnd is +inf and their +inf filler bound would pass the comparison
            pend = __ballot_sync(0xffffffffu, e < lcnt && lb <= bnd);
            if (!pend && b0 + 32 >= lcnt) break;   // last batch and nothing of it is in the band
            if (!pend) {   // entries are bucket-ordered: the rest of the list lies above this bucket's edge
                float mn = lb;
                for (int o = 16; o; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                if (wl == 0 && bb_edge(bb_bucket(mn, __frcp_rn(lbm)), lbm) > bnd) atomicMax(&s_next, lcnt);   // stop the CTA
                continue;
            }
        } else {
            if (rbase >= ub) break;
            base = rbase;
            rbase += RSTEP;
            pend = __ballot_sync(0xffffffffu, base + wl < ub);
        }
        const float bnd_f = bnd;   // the band the fetch-time filters below use (warp-uniform)
        int uT = 0, uTm = 0, uSb = 0, uEa = 0, uNe = 0;
        float uX = 0.0f, uY = 0.0f, uZ = 0.0f;
        uint32_t uCm = 0;
        bool uok = false, uCh = false;
        if ((pend >> wl) & 1u) {   // this lane's own unit
            const uint64_t myunit = BB ? ua + (uint64_t)loff : base + (uint64_t)wl;
            uok = unit_consts(myunit, uT, uTm, uSb, uEa, uNe, uX, uY, uZ, uCm, uCh);
        }
        if (BB) {   // units fetched within the band; those the fetch-time bounds cleared are not visited below
            if (wl == 0) ndone += __popc(pend);
            pend &= __ballot_sync(0xffffffffu, uok);
        }
      while (pend) {
        const int jl = __ffs(pend) - 1;
        pend &= pend - 1;
        const uint32_t lo_j = __shfl_sync(0xffffffffu, loff, jl);
        const uint64_t unit = BB ? ua + (uint64_t)lo_j : base + (uint64_t)jl;
        if (BB) {   // re-check the unit against the incumbent found since the batch was fetched
            const float lbj = __shfl_sync(0xffffffffu, lbv, jl);
            unsigned ci = 0;   // one read, broadcast: every lane must take the same decision
            if (wl == 0) ci = *(volatile unsigned*)&s_inc;
            const float cur = __uint_as_float(__shfl_sync(0xffffffffu, ci, 0));
            if (cur < incv) {
                incv = cur;
                bnd = __fmul_ru(incv, bandf);
                bnd_of = incv;
            }
            if (lbj > bnd) continue;
        }
        const int cT = __shfl_sync(0xffffffffu, uT, jl), cTm = __shfl_sync(0xffffffffu, uTm, jl);
        const int sb = __shfl_sync(0xffffffffu, uSb, jl), ea = __shfl_sync(0xffffffffu, uEa, jl);
        const int ne = __shfl_sync(0xffffffffu, uNe, jl);
        const float Xh = __shfl_sync(0xffffffffu, uX, jl), Yh = __shfl_sync(0xffffffffu, uY, jl);
        const float Zh = __shfl_sync(0xffffffffu, uZ, jl);
        if (!__shfl_sync(0xffffffffu, (int)uok, jl)) {   // no usable step level
            if (!BB && wl == 0) subp[unit] = INFINITY;
            continue;
        }
        nuok++;
        if (TWO) {
            // exhaustive pass without QoS: every step level of the unit is an entry and every inner level is in
            // range, so lane wl builds its entries ea + kb + wl + 32 i (i < P1_NE) in registers and sweeps all inner
            // pairs with them: one broadcast read of a pair feeds 2 P1_NE candidates (no table round trip)
            float acc[2 * P1_NE];
#pragma unroll
            for (int i = 0; i < 2 * P1_NE; i++) acc[i] = INFINITY;
            const int np2 = Lin >> 1;
            for (int kb = 0; kb < ne; kb += 32 * P1_NE) {
                u64 X2[P1_NE], Y2[P1_NE], Z2[P1_NE];
                float Xs[P1_NE], Ys[P1_NE], Zs[P1_NE];
                int nv = 0;
#pragma unroll
                for (int i = 0; i < P1_NE; i++) {
                    const int k = kb + wl + 32 * i;
                    float X = INFINITY, Y = 0.0f, Z = 0.0f;
                    if (k < ne) {
                        const Lev& r = stepw[A.sperm[ea + k]];
                        const float Be = __ll2float_rn(r.B), Sf = (float)r.S;
                        X = fmaf(Be, Yh, fmaf(Sf, Zh, Xh));
                        if (MODE == M_PAPER) X += (float)((double)r.BS * invd);
                        Y = fmaf(Sf, invf, Yh);
                        Z = fmaf(Be, invf, Zh);
                        nv++;
                    }
                    Xs[i] = X; Ys[i] = Y; Zs[i] = Z;
                    X2[i] = f2pack(X, X); Y2[i] = f2pack(Y, Y); Z2[i] = f2pack(Z, Z);
                }
                nfeas += (unsigned long long)nv * (unsigned long long)Lin;
                // pairs p and p + 1 per iteration: accumulator 2i takes even pairs, 2i + 1 odd ones (static register
                // indices; an index computed from p would put the accumulators in local memory)
                auto pair = [&](int p, int par) {
                    const float4 r = A.ip[p];
                    const u64 Bp = f2pack(r.x, r.y), Sp = f2pack(r.z, r.w);
                    u64 dd = 0;
                    if (MODE == M_PAPER) { const float2 d = A.iD[p]; dd = f2pack(d.x, d.y); }
#pragma unroll
                    for (int i = 0; i < P1_NE; i++) {
                        const u64 base = MODE == M_PAPER ? add2(X2[i], dd) : X2[i];
                        float k0, k1;
                        f2unpack(fma2(Bp, Y2[i], fma2(Sp, Z2[i], base)), k0, k1);
                        acc[2 * i + par] = fminf(acc[2 * i + par], fminf(k0, k1));
                    }
                };
                int p = 0;
                for (; p + 2 <= np2; p += 2) {
                    pair(p, 0);
                    pair(p + 1, 1);
                }
                if (p < np2) pair(p, 0);
                if (Lin & 1) {  // trailing odd element
                    const float4 r = A.ip[Lin >> 1];
                    const float d = MODE == M_PAPER ? A.iD[Lin >> 1].x : 0.0f;
#pragma unroll
                    for (int i = 0; i < P1_NE; i++) acc[2 * i] = fminf(acc[2 * i], fmaf(r.x, Ys[i], fmaf(r.z, Zs[i], Xs[i] + d)));
                }
            }
            float m = acc[0];
#pragma unroll
            for (int i = 1; i < 2 * P1_NE; i++) m = fminf(m, acc[i]);
            for (int o = 16; o; o >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (wl == 0) subp[unit] = m;
            continue;
        }
        const struct { int T, Tm; } h = {cT, cTm};
        int nc = 0;
        bool had = false;
        float m0 = INFINITY, m1 = INFINITY;
        // sweep the warp's table (<= 32 entries, one per lane): packed FMAs over each entry's exact
        // QoS-feasible inner range; called after every entry pass (surviving entries are rare)
        // The warp's table holds <= 32 entries, one per lane; each lane sweeps its entry's inner range with packed
        // FMAs.  Without QoS bounds every range is [0, L_inner): the lanes run in lockstep (broadcast reads of
        // the inner pairs; lanes without an entry score +inf).
        auto sweep_qos = [&]() {   // per-lane ranges (QoS): each lane its own entry's exact feasible range
            for (int i = wl; i < nc; i += 32) {
                const float4 t4 = tab[i];
                int2 kk = tabk[i];
                if (QOS && kk.x < 0) {   // masked sweep of [0, min(k_lo, k_hi)) (non-monotone u)
                    kk.x = -1 - kk.x;
                    const int kend = min(kk.x, kk.y);
                    for (int k = 0; k < kend; k++) {
                        const float4 r = A.ip[k >> 1];
                        const float2 uu2 = A.iu[k >> 1];
                        const float bk = (k & 1) ? r.y : r.x, sk = (k & 1) ? r.w : r.z, uk = (k & 1) ? uu2.y : uu2.x;
                        float b0 = t4.x;
                        if (MODE == M_PAPER) { const float2 dd = A.iD[k >> 1]; b0 += (k & 1) ? dd.y : dd.x; }
                        if (t4.w <= uk) { m0 = fminf(m0, fmaf(bk, t4.y, fmaf(sk, t4.z, b0))); nfeas++; }
                    }
                }
                const int ka = max(kk.x, 0), kb2 = kk.y;
                if (ka >= kb2) continue;
                nfeas += (unsigned long long)(kb2 - ka);
                const u64 X2 = f2pack(t4.x, t4.x), Y2 = f2pack(t4.y, t4.y), Z2 = f2pack(t4.z, t4.z);
                int k = ka;
                if (k & 1) {   // leading odd element
                    const float4 r = A.ip[k >> 1];
                    float b0 = t4.x;
                    if (MODE == M_PAPER) b0 += A.iD[k >> 1].y;
                    m0 = fminf(m0, fmaf(r.y, t4.y, fmaf(r.w, t4.z, b0)));
                    k++;
                }
                const int pend = kb2 >> 1;
    #pragma unroll 4
                for (int p = k >> 1; p < pend; p++) {
                    const float4 r = A.ip[p];
                    u64 base = X2;
                    if (MODE == M_PAPER) { const float2 dd = A.iD[p]; base = add2(X2, f2pack(dd.x, dd.y)); }
                    const u64 key = fma2(f2pack(r.x, r.y), Y2, fma2(f2pack(r.z, r.w), Z2, base));
                    float k0, k1;
                    f2unpack(key, k0, k1);
                    m0 = fminf(m0, fminf(k0, k1));
                }
                if (kb2 & 1) {  // trailing odd element
                    const float4 r = A.ip[kb2 >> 1];
                    float b0 = t4.x;
                    if (MODE == M_PAPER) b0 += A.iD[kb2 >> 1].x;
                    m1 = fminf(m1, fmaf(r.x, t4.y, fmaf(r.z, t4.z, b0)));
                }
            }
        };
        // Without QoS bounds every entry's range is [0, L_inner): the lanes sweep in lockstep (broadcast reads of
        // the inner pairs; lanes without an entry score +inf).  (The exhaustive pass keeps its entries in
        // registers instead, TWO above.)
        auto sweep = [&]() {
            if (QOS) { sweep_qos(); return; }
            const float4 ta = wl < nc ? tab[wl] : make_float4(INFINITY, 0.0f, 0.0f, 0.0f);
            nfeas += (unsigned long long)(wl < nc) * (unsigned long long)Lin;
            if (Lin & 1) {  // trailing odd element
                const float4 r = A.ip[Lin >> 1];
                const float d = MODE == M_PAPER ? A.iD[Lin >> 1].x : 0.0f;
                m1 = fminf(m1, fmaf(r.x, ta.y, fmaf(r.z, ta.z, ta.x + d)));
            }
            const int np2 = Lin >> 1;
            const u64 Xa = f2pack(ta.x, ta.x), Ya = f2pack(ta.y, ta.y), Za = f2pack(ta.z, ta.z);
            float ma = INFINITY, mb = INFINITY;   // two independent minima
            auto key = [&](int q) -> float {
                const float4 r = A.ip[q];
                u64 base = Xa;
                if (MODE == M_PAPER) { const float2 dd = A.iD[q]; base = add2(Xa, f2pack(dd.x, dd.y)); }
                const u64 k2 = fma2(f2pack(r.x, r.y), Ya, fma2(f2pack(r.z, r.w), Za, base));
                float k0, k1;
                f2unpack(k2, k0, k1);
                return fminf(k0, k1);
            };
            int p = 0;
            for (; p + 2 <= np2; p += 2) {
                ma = fminf(ma, key(p));
                mb = fminf(mb, key(p + 1));
            }
            if (p < np2) ma = fminf(ma, key(p));
            m0 = fminf(m0, fminf(ma, mb));
        };
        // one step entry per lane (relative index k in [ea, ea + ne)); appends the usable ones to
        // the warp's table; returns whether the lane's level lies past the QoS prefix
        auto entry = [&](int k, bool valid) -> bool {
            bool use = false, past = true;
            int Sp = 0, Tme = 1 << 24;
            float Be = 0.0f, De = 0.0f;
            if (valid) {
                if (W >= 2) {
                    const Lev& r = stepw[A.sperm[ea + k]];
                    Sp = r.S; Tme = r.Tmax;
                    past = QOS && r.S > sb;
                    use = !past && (!QOS || (r.Tmax - r.S - h.T >= smin_i));
                    if (use) {
                        Be = __ll2float_rn(r.B);
                        if (MODE == M_PAPER) De = (float)((double)r.BS * invd);
                    }
                } else {
                    past = false;
                    use = true;
                }
            }
            float4 ent = make_float4(0.f, 0.f, 0.f, 0.f);
            int klo = 0, khi = Lin;
            if (use) {
                const int Tp = h.T + Sp, Tm = min(h.Tm, Tme);
                const float Sf = (float)Sp;
                float X = fmaf(Be, Yh, fmaf(Sf, Zh, Xh));
                if (MODE == M_PAPER) X += De;
                ent = make_float4(X, fmaf(Sf, invf, Yh), fmaf(Be, invf, Zh), (float)Tp);
                if (QOS) {
                    khi = inner_khi(A, Tm - Tp, s0, slast, khi_ok, Lin);
                    klo = inner_klo(A, Tp, u0v, ulast, klo_ok, Lin);
                    // levels before klo: none qualifies unless u is non-monotone there (rare)
                    const bool pre = A.umaxp[min(klo, khi)] >= Tp;
                    use = khi > klo || pre;
                    if (BB && use) {   // entry bound: every swept key >= X + Y minB + Z minS,
                        // and >= X + min over the inner hull restricted to the entry's S' range
                        const int ka = pre ? 0 : klo;
                        float lbe = fmaf(ent.y, A.preminB[khi], fmaf(ent.z, (float)A.ssort[ka], ent.x));
                        if (!(lbe * 0.99998474121f > bnd))
                            lbe = fmaxf(lbe, ent.x + hull_min_pos(A, nhv, ent.y, ent.z, ka, khi - 1));
                        use = !(lbe * 0.99998474121f > bnd);   // 1 - 2^-16
                    }
                    if (pre) klo = -1 - klo;   // flag: sweep [0, |klo|) with a mask first
                }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, use);
            if (use) {
                const int pos = nc + __popc(bal & ((1u << wl) - 1u));
                tab[pos] = ent;
                tabk[pos] = make_int2(klo, khi);
            }
            nc += __popc(bal);
            if (wl == 0) nent += __popc(bal);
            if (nc) {
                had = true;
                __syncwarp();
                sweep();
                __syncwarp();   // the table is rewritten by the next pass
                nc = 0;
            }
            return past;
        };
        bool chunked = false;
        if (BB && QOS && step_tab && __shfl_sync(0xffffffffu, (int)uCh, jl)) {
            // the chunk filter: the unit's lane evaluated every chunk at fetch time (chunk_keep; a unit with no chunk
            // in the band never gets here); lane wl re-checks chunk c_lo + wl if it was kept
            {
                const int c_lo = ea / P1_CS;
                chunked = true;
                const unsigned cm0 = __shfl_sync(0xffffffffu, uCm, jl);
                // re-checked against the band as it is now if it tightened since the fetch (the same test
                // against the same band would repeat the fetch-time result)
                const bool keep = ((cm0 >> wl) & 1u) && (bnd == bnd_f || chunk_keep(c_lo + wl, h.T, h.Tm, Xh, Yh, Zh));
                const unsigned cm = __ballot_sync(0xffffffffu, keep);
                nch += __popc(cm);
                nuch += cm != 0u;
                if (keep) s_chunk[warp][__popc(cm & ((1u << wl) - 1u))] = (uint8_t)wl;   // surviving chunks, in order
                __syncwarp();
                const int nk = __popc(cm), q = wl / P1_CS, j = wl % P1_CS;
                for (int p0 = 0; p0 < nk; p0 += 32 / P1_CS) {   // 32 / P1_CS surviving chunks per pass, one entry per lane
                    const int k = p0 + q < nk ? (c_lo + s_chunk[warp][p0 + q]) * P1_CS + j - ea : -1;
                    entry(k, k >= 0 && k < ne);
                }
                __syncwarp();
            }
        }
        if (!chunked)
            for (int kb = 0; kb < ne; kb += 32)
                if (__all_sync(0xffffffffu, entry(kb + wl, kb + wl < ne))) break;   // the rest of the sorted segment is unusable
        __syncwarp();
        if (BB && wl == 0 && had) nue++;
        float m = fminf(m0, m1);
        if (BB && !__any_sync(0xffffffffu, m < INFINITY)) {   // nothing feasible swept: submin stays +inf
            __syncwarp();
            continue;
        }
        for (int o = 16; o; o >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (wl == 0) {
            subp[unit] = m;
            if (BB) atomicOr(bb.wbits + (size_t)prob * wbits_words(su) + (unit >> 5), 1u << (unit & 31));
            if (BB && m < INFINITY) {
                const int pos = atomicAdd(bb.plist_n + prob, 1);
                if (pos < PL_CAP) bb.plist[(size_t)prob * PL_CAP + pos] = (uint32_t)unit;
            }
            if (BB && m < incv) {
                atomicMin(&s_inc, __float_as_uint(m));
                atomicMin(bb.inc + prob, __float_as_uint(m));
            }
        }
        if (BB && m < incv) {   // every lane (m and incv are warp-uniform): a tighter band at once
            incv = m;
            bnd = __fmul_ru(incv, bandf);
            bnd_of = incv;
        }
        __syncwarp();   // the table is rewritten for the next unit
      }
    }
    for (int o = 16; o; o >>= 1) nfeas += __shfl_xor_sync(0xffffffffu, nfeas, o);
    if (wl == 0 && nfeas) atomicAdd(feasible, nfeas);
    if (BB && wl == 0 && ndone) {
        atomicAdd(bb.rows_done, (unsigned long long)ndone);
        atomicAdd(bb.rows_done + 1, (unsigned long long)nue);
        atomicAdd(bb.rows_done + 2, (unsigned long long)nent);
        atomicAdd(bb.rows_done + 3, (unsigned long long)nuok);
        atomicAdd(bb.rows_done + 4, (unsigned long long)nuch);
        atomicAdd(bb.rows_done + 5, (unsigned long long)nch);
    }
}

// Generic (unpacked) filter: MAX / ENERGY objectives, EXCESS, MATRIX (any objective), and
// SUM with large inner-level counts.  One warp per unit; inner levels read from shared memory.
template <int NP, int MODE, int OBJ, bool QOS>
__global__ void __launch_bounds__(P1_THREADS, 2)
k_pass1_gen(Setup su, const Prob* __restrict__ probs, const Lev* __restrict__ levs, float* __restrict__ submin,
            float* __restrict__ submin_sure) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ uint64_t bar;
    const int ipS = (su.items_max + su.n_shards - 1) / su.n_shards;
    const int prob = blockIdx.x / ipS;
    const Prob& P = probs[prob];
    if (P.status != 0) return;
    uint64_t item;
    bool ok;
    item_of_block(su, P, blockIdx.x % ipS, &item, &ok);
    if (!ok) return;
    constexpr int W = NP + 1;
    const int Lmax = su.Lmax;
    const bool wide = su.wide != 0;
    Lev* sl = reinterpret_cast<Lev*>(smem_raw);
    stage_levels(sl, levs + (size_t)prob * su.lev_stride, (unsigned)(W * Lmax * sizeof(Lev)), &bar);
    int L[W];
#pragma unroll
    for (int w = 0; w < W; w++) L[w] = P.L[w];
    const int Lin = L[NP];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nwarps = P1_THREADS / 32;
    float Mcol[W];
#pragma unroll
    for (int w = 0; w < W; w++) Mcol[w] = P.Mf[w * MAXW_ENUM + NP];
    const Lev* inner = sl + NP * Lmax;
    const bool weighted = su.weighted != 0;
    float wf[W];
#pragma unroll
    for (int w = 0; w < W; w++) wf[w] = P.wf[w];

    uint64_t u0 = item * (uint64_t)su.upi, u1 = u0 + (uint64_t)su.upi;
    if (u1 > P.units) u1 = P.units;
    int d[W];
    for (uint64_t unit = u0 + (uint64_t)warp; unit < u1; unit += (uint64_t)nwarps) {
        uint64_t row;
        int e0, e1;
        unit_range(P, unit, &row, &e0, &e1);
        decode_row(row, L, W, d);
        float m = INFINITY, ms = INFINITY;
        for (int e = e0; e < e1; e++) {
            if (NP >= 1) d[NP - 1] = e;
            float pBf[W], pBk[W], psf[W];
            int64_t pB = 0, pT = 0;
            int32_t pTm = (int32_t)NARROW_T;
#pragma unroll
            for (int w = 0; w < NP; w++) {
                const Lev& r = sl[w * Lmax + d[w]];
                pBf[w] = __ll2float_rn(r.B);
                pBk[w] = r.Bk;
                psf[w] = __ll2float_rn(r.S);
                pB += r.B; pT += r.S; pTm = min(pTm, r.Tmax);
            }
            const float Tpf = __ll2float_rn(pT);
            const float c1 = wide ? 0.0f : (float)(pTm - pT);
            float Opre[W];
            if (MODE != M_MATRIX && wide) {
                // wide problems: S', T' beyond 2^24, so T' - S'_w is not exact in FP32; the overlap of
                // prefix worker w is summed from the others' rounded S' (non-negative terms, <= (W-1) u)
#pragma unroll
                for (int w = 0; w < NP; w++) {
                    float o = (MODE == M_EXCL) ? 0.0f : psf[w];
#pragma unroll
                    for (int v = 0; v < NP; v++)
                        if (v != w) o += psf[v];
                    Opre[w] = o;
                }
            }
            if (MODE == M_MATRIX) {
#pragma unroll
                for (int w = 0; w < W; w++) {
                    float o = 0.0f;
#pragma unroll
                    for (int v = 0; v < NP; v++)
                        if (v != w) o = fmaf(P.Mf[w * MAXW_ENUM + v], psf[v], o);
                    Opre[w] = o;
                }
            }
            const float Bpf = __ll2float_rn(pB);
            for (int j = lane; j < Lin; j += 32) {
                const Lev& a = inner[j];
                const float iBf = __ll2float_rn(a.B), iBk = a.Bk, isf = __ll2float_rn(a.S);
                const float Tf = Tpf + isf;
                float Lw[W];
                float num = 0.0f;
#pragma unroll
                for (int w = 0; w < W; w++) {
                    const float bf = (w == NP) ? iBf : pBf[w];
                    const float bk = (w == NP) ? iBk : pBk[w];
                    float O;
                    if (MODE == M_EXCL) O = (w == NP) ? Tpf : (wide ? Opre[w] + isf : Tf - psf[w]);
                    else if (MODE == M_PAPER) O = (wide && w < NP) ? Opre[w] + isf : Tf;
                    else if (MODE == M_EXCESS) O = fmaxf(Tf - P.lamNf, 0.0f);
                    else O = (w == NP) ? Opre[w] : fmaf(Mcol[w], isf, Opre[w]);
                    Lw[w] = fmaf(O, bk, bf);
                    if (OBJ == O_SUM) num = fmaf(bf, O, num);
                }
                float key;
                if (weighted && OBJ != O_ENERGY) {   // weights (R20): sum / max of omega_w L_w
                    key = OBJ == O_SUM ? 0.0f : Lw[0] * wf[0];
#pragma unroll
                    for (int w = 0; w < W; w++) key = OBJ == O_SUM ? fmaf(wf[w], Lw[w], key) : fmaxf(key, Lw[w] * wf[w]);
                } else if (OBJ == O_SUM) {
                    key = fmaf(num, P.inv, Bpf + iBf);
                } else {
                    float mx = Lw[0];
#pragma unroll
                    for (int w = 1; w < W; w++) mx = fmaxf(mx, Lw[w]);
                    if (OBJ == O_MAX) key = mx;
                    else key = fmaf(P.p_dyn, fminf(1.0f, Tf * P.inv), P.p_idle) * mx;
                }
                if (QOS) {
                    if (MODE == M_MATRIX || wide) {
                        bool maybe = true, sure = true;
#pragma unroll
                        for (int w = 0; w < W; w++) {
                            maybe = maybe && (Lw[w] <= P.Qhi[w]);
                            sure = sure && (Lw[w] <= P.Qlo[w]);
                        }
                        if (maybe) m = fminf(m, key);
                        if (sure) ms = fminf(ms, key);
                    } else {
                        if (isf <= c1 && Tpf <= (float)(a.Tmax - a.S)) m = fminf(m, key);
                    }
                } else {
                    m = fminf(m, key);
                }
            }
        }
        m = team_min(m, 32, 0xffffffffu);
        if ((MODE == M_MATRIX || wide) && QOS) ms = team_min(ms, 32, 0xffffffffu);
        if (lane == 0) {
            submin[(size_t)prob * su.units_max + unit] = m;
            if ((MODE == M_MATRIX || wide) && QOS) submin_sure[(size_t)prob * su.units_max + unit] = ms;
        }
    }
}

// ------------------------------------------------------------------------------------------
// pass-1 dispatch
// ------------------------------------------------------------------------------------------
typedef void (*P1Fast)(Setup, const Prob*, const Lev*, float*, unsigned long long*, BBArgs);
typedef void (*P1Gen)(Setup, const Prob*, const Lev*, float*, float*);
typedef void (*RowLB)(Setup, const Prob*, const Lev*, const float2*, const int32_t*, const RowHdr*, float*, unsigned*);

template <int NW, bool BB>
static P1Fast pick_fast(int mode, bool qos) {
    if (mode == M_EXCL) return qos ? k_pass1_fast<NW, M_EXCL, true, BB> : k_pass1_fast<NW, M_EXCL, false, BB>;
    return qos ? k_pass1_fast<NW, M_PAPER, true, BB> : k_pass1_fast<NW, M_PAPER, false, BB>;
}
template <int NW>
static RowLB pick_rowlb(bool qos) { return qos ? k_rowlb<NW, true> : k_rowlb<NW, false>; }
typedef void (*RowLBF)(Setup, const Prob*, const Lev*, const float2*, const int32_t*, const RowHdr*, unsigned*, uint2*,
                       int32_t*);
template <int NW>
static RowLBF pick_rowlbf(bool qos) { return qos ? k_rowlb_fused<NW, true> : k_rowlb_fused<NW, false>; }
// one pass-1 item per problem (whole rows), unsharded, rows within the shared-memory cap
static bool rowlb_fused_ok(const Setup& su) {
    return su.n_shards == 1 && su.nseg == 1 && su.items_max == 1 && su.rows_max <= RLF_ROWS_CAP && su.upi >= su.rows_max;
}

template <int NP, int MODE>
static P1Gen pick_gen_m(int obj, bool qos) {
    if (obj == O_SUM) return qos ? k_pass1_gen<NP, MODE, O_SUM, true> : k_pass1_gen<NP, MODE, O_SUM, false>;
    if (obj == O_MAX) return qos ? k_pass1_gen<NP, MODE, O_MAX, true> : k_pass1_gen<NP, MODE, O_MAX, false>;
    return qos ? k_pass1_gen<NP, MODE, O_ENERGY, true> : k_pass1_gen<NP, MODE, O_ENERGY, false>;
}
template <int NP>
static P1Gen pick_gen(int mode, int obj, bool qos) {
    if (mode == M_EXCL) return pick_gen_m<NP, M_EXCL>(obj, qos);
    if (mode == M_PAPER) return pick_gen_m<NP, M_PAPER>(obj, qos);
    if (mode == M_EXCESS) return pick_gen_m<NP, M_EXCESS>(obj, qos);
    return pick_gen_m<NP, M_MATRIX>(obj, qos);
}

bool pass1_fast(int L_inner) { return fast_ok(L_inner); }
int pass1_fast_team(int L_inner) { return fast_team(L_inner); }

// the fast kernel applies when every problem's inner worker fits a warp team
static bool use_fast(const Setup& su) {   // (the host's plan_geometry takes the same decision)
    return su.obj == O_SUM && (su.mode == M_EXCL || su.mode == M_PAPER) && fast_ok(su.Lmax) && !su.wide &&
           !su.weighted;
}

bool pass1_prunable(const Setup& su) { return su.prune != 0 && su.W >= 3 && use_fast(su); }

static cudaError_t fill_u32(void* p, size_t n, unsigned v, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    size_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_fill_u32<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<unsigned*>(p), n, v);
    return cudaGetLastError();
}


size_t pass1_smem(const Setup& su, bool fast) {
    size_t s = (size_t)su.W * su.Lmax * sizeof(Lev);
    if (fast) s += (size_t)su.aux_bytes + (size_t)su.table_bytes;   // aux block + per-warp prefix tables
    return s;
}

cudaError_t launch_pass1(const Setup& su, Work& wk, cudaStream_t st) {
    const int NP = su.W - 1;
    const bool qos = su.has_qos != 0;
    const int ipS = (su.items_max + su.n_shards - 1) / su.n_shards;
    const size_t grid = (size_t)su.n_problems * ipS;
    if (grid == 0) return cudaSuccess;
    const bool fast = use_fast(su);
    const size_t smem = pass1_smem(su, fast);
    if (fast && pass1_prunable(su)) {
        P1Fast f = nullptr;
        RowLB r = nullptr;
        switch (su.W) {
            case 3: f = pick_fast<3, true>(su.mode, qos); r = pick_rowlb<3>(qos); break;
            case 4: f = pick_fast<4, true>(su.mode, qos); r = pick_rowlb<4>(qos); break;
            case 5: f = pick_fast<5, true>(su.mode, qos); r = pick_rowlb<5>(qos); break;
            case 6: f = pick_fast<6, true>(su.mode, qos); r = pick_rowlb<6>(qos); break;
            case 7: f = pick_fast<7, true>(su.mode, qos); r = pick_rowlb<7>(qos); break;
            case 8: f = pick_fast<8, true>(su.mode, qos); r = pick_rowlb<8>(qos); break;
            default: return cudaErrorInvalidValue;
        }
        cudaError_t e;
        const size_t n = (size_t)su.n_problems;
        // unwritten units read as +inf through the bitmap (sub_at), so submin itself is not filled
        {
            Fill4 f{};
            f.p[0] = wk.wbits; f.n[0] = n * (size_t)((su.units_max + 31) >> 5); f.v[0] = 0u;
            f.p[1] = wk.inc; f.n[1] = n; f.v[1] = 0x7f800000u;
            f.p[2] = wk.lbmin; f.n[2] = n; f.v[2] = 0x7f800000u;
            f.p[3] = reinterpret_cast<unsigned*>(wk.plist_n); f.n[3] = n; f.v[3] = 0u;
            if ((e = fill4(f, st)) != cudaSuccess) return e;
        }
        const size_t bsm = (size_t)FT_CAP * 4 + (size_t)su.Lmax * 2 * sizeof(Lev);

        if ((e = cudaFuncSetAttribute((const void*)k_prep_bound, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm)) != cudaSuccess)
            return e;
        if ((e = launch_pdl(k_prep_bound, dim3(su.n_problems), dim3(256), bsm, st, su, wk.probs, wk.levs, wk.hull, wk.ftab,
                            wk.rowhdr, wk.table_of, wk.thull, wk.thull_n)) != cudaSuccess)
            return e;
        const size_t fsm = hull_stride(su.Lmax) * sizeof(float2) + (size_t)su.Lmax * (size_t)(su.W - 2) * 24 +
                           (size_t)su.rows_max * 4 + (size_t)((su.rows_max + 31) / 32) * 4;
        if (rowlb_fused_ok(su) && fsm <= 160 * 1024) {
            RowLBF rf = nullptr;
            switch (su.W) {
                case 3: rf = pick_rowlbf<3>(qos); break;
                case 4: rf = pick_rowlbf<4>(qos); break;
                case 5: rf = pick_rowlbf<5>(qos); break;
                case 6: rf = pick_rowlbf<6>(qos); break;
                case 7: rf = pick_rowlbf<7>(qos); break;
                case 8: rf = pick_rowlbf<8>(qos); break;
                default: return cudaErrorInvalidValue;
            }
            if ((e = cudaFuncSetAttribute((const void*)rf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm)) != cudaSuccess)
                return e;
            if ((e = launch_pdl(rf, dim3(su.n_problems), dim3(RLF_THREADS), fsm, st, su, wk.probs, wk.levs, wk.hull, wk.ftab,
                                wk.rowhdr, wk.lbmin, wk.ulist, wk.ulist_n)) != cudaSuccess)
                return e;
            if ((e = cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
                return e;
            BBArgs bb{wk.ulist, wk.ulist_n, wk.lbmin, wk.inc, wk.rows_done, wk.plist, wk.plist_n, wk.wbits, wk.hull, wk.rowhdr};
            if (wk.kev[0]) cudaEventRecord(wk.kev[0], st);
            if ((e = launch_pdl(f, dim3((unsigned)grid), dim3(P1_THREADS), smem, st, su, wk.probs, wk.levs, wk.submin,
                                wk.feasible, bb)) != cudaSuccess)
                return e;
            if (wk.kev[1]) cudaEventRecord(wk.kev[1], st);
            return cudaGetLastError();
        }
        // enough CTAs to fill the GPU (8 per SM), each looping over many rows of its problem
        const long long want = std::max<long long>(1, (148LL * 8 + su.n_problems - 1) / su.n_problems);
        const long long gx = std::min<long long>((su.rows_max + 255) / 256, want);
        const size_t rsm = hull_stride(su.Lmax) * sizeof(float2);
        if ((e = cudaFuncSetAttribute((const void*)r, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm)) != cudaSuccess)
            return e;
        r<<<dim3((unsigned)gx, (unsigned)su.n_problems), 256, rsm, st>>>(
            su, wk.probs, wk.levs, wk.hull, wk.ftab, wk.rowhdr, wk.rowlb, wk.lbmin);
        if ((e = cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
            return e;
        k_bucket<<<(unsigned)grid, 256, 0, st>>>(su, wk.probs, wk.rowlb, wk.lbmin, wk.ulist, wk.ulist_n);
        BBArgs bb{wk.ulist, wk.ulist_n, wk.lbmin, wk.inc, wk.rows_done, wk.plist, wk.plist_n, wk.wbits, wk.hull, wk.rowhdr};
        if (wk.kev[0]) cudaEventRecord(wk.kev[0], st);
        f<<<(unsigned)grid, P1_THREADS, smem, st>>>(su, wk.probs, wk.levs, wk.submin, wk.feasible, bb);
        if (wk.kev[1]) cudaEventRecord(wk.kev[1], st);
    } else if (fast) {
        P1Fast f = nullptr;
        switch (su.W) {
            case 1: f = pick_fast<1, false>(su.mode, qos); break;
            case 2: f = pick_fast<2, false>(su.mode, qos); break;
            case 3: f = pick_fast<3, false>(su.mode, qos); break;
            case 4: f = pick_fast<4, false>(su.mode, qos); break;
            case 5: f = pick_fast<5, false>(su.mode, qos); break;
            case 6: f = pick_fast<6, false>(su.mode, qos); break;
            case 7: f = pick_fast<7, false>(su.mode, qos); break;
            case 8: f = pick_fast<8, false>(su.mode, qos); break;
            default: return cudaErrorInvalidValue;
        }
        cudaError_t e = cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        BBArgs bb{};
        if (wk.kev[0]) cudaEventRecord(wk.kev[0], st);
        f<<<(unsigned)grid, P1_THREADS, smem, st>>>(su, wk.probs, wk.levs, wk.submin, wk.feasible, bb);
        if (wk.kev[1]) cudaEventRecord(wk.kev[1], st);
    } else {
        P1Gen f = nullptr;
        switch (NP) {
            case 0: f = pick_gen<0>(su.mode, su.obj, qos); break;
            case 1: f = pick_gen<1>(su.mode, su.obj, qos); break;
            case 2: f = pick_gen<2>(su.mode, su.obj, qos); break;
            case 3: f = pick_gen<3>(su.mode, su.obj, qos); break;
            case 4: f = pick_gen<4>(su.mode, su.obj, qos); break;
            case 5: f = pick_gen<5>(su.mode, su.obj, qos); break;
            case 6: f = pick_gen<6>(su.mode, su.obj, qos); break;
            case 7: f = pick_gen<7>(su.mode, su.obj, qos); break;
            default: return cudaErrorInvalidValue;
        }
        cudaError_t e = cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        if (wk.kev[0]) cudaEventRecord(wk.kev[0], st);
        f<<<(unsigned)grid, P1_THREADS, smem, st>>>(su, wk.probs, wk.levs, wk.submin, wk.submin_sure);
        if (wk.kev[1]) cudaEventRecord(wk.kev[1], st);
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// local minimum per problem over this shard's units (one warp per problem)
// ------------------------------------------------------------------------------------------
// one CTA (256 threads) per problem: this shard's minimum over its units' pass-1 minima, then the
// units pass 2 must rescan (submin within the band of this shard's minimum; the global minimum is
// never larger, so its band is a subset), in index order when at most BAND_SORTED long; bandn = -1: more than BAND_CAP
__global__ void __launch_bounds__(256) k_reduce_min(Setup su, const Prob* probs, const float* submin,
                                                    const float* submin_sure, float* m32, float* m32_sure,
                                                    int32_t* bandn, uint64_t* bandlist, const uint32_t* plist,
                                                    const int32_t* plist_n, const uint32_t* wbits) {
    pdl_wait();      // (programmatic dependent launch: the predecessor's results are visible)
    pdl_trigger();
    __shared__ float rm[8], rs[8];
    __shared__ int s_cnt;
    __shared__ uint64_t s_list[BAND_CAP];
    const int p = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
    const Prob& P = probs[p];
    float m = INFINITY, ms = INFINITY;
    uint64_t a = 0, b = 0;
    // units listed by the pruned pass 1 (every other unit kept submin = +inf); unsharded, no overflow
    const int nl = plist_n ? plist_n[p] : -1;
    const uint32_t* lst = (plist && su.n_shards == 1 && !submin_sure && nl >= 0 && nl <= PL_CAP) ? plist + (size_t)p * PL_CAP
                                                                                                  : nullptr;
    if (P.status == 0) {
        uint64_t slo, shi;
        shard_items(P.n_items, su.shard, su.n_shards, &slo, &shi);
        a = slo * (uint64_t)su.upi;
        b = shi * (uint64_t)su.upi;
        if (b > P.units) b = P.units;
        const float* sp = submin + (size_t)p * su.units_max;
        if (lst) {   // pruned pass 1: only the listed units can be finite
            for (int i = tid; i < nl; i += blockDim.x) m = fminf(m, sp[lst[i]]);
        } else {
            for (uint64_t u = a + tid; u < b; u += blockDim.x) {
                m = fminf(m, sub_at(su, sp, wbits, p, u));
                if (submin_sure) ms = fminf(ms, submin_sure[(size_t)p * su.units_max + u]);
            }
        }
    }
    for (int o = 16; o; o >>= 1) {
        m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
        ms = fminf(ms, __shfl_xor_sync(0xffffffffu, ms, o));
    }
    if (lane == 0) { rm[tid >> 5] = m; rs[tid >> 5] = ms; }
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    m = rm[0]; ms = rs[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); i++) { m = fminf(m, rm[i]); ms = fminf(ms, rs[i]); }
    if (tid == 0) {
        m32[p] = m;
        if (m32_sure) m32_sure[p] = submin_sure ? ms : m;
    }
    if (!bandn) return;
    if (P.status == 0 && !isinf(m)) {
        const float bound = band_bound(su, m, submin_sure ? ms : m);
        const float* sp = submin + (size_t)p * su.units_max;
        if (lst) {
            for (int i = tid; i < nl; i += blockDim.x)
                if (sp[lst[i]] <= bound) {
                    const int pos = atomicAdd(&s_cnt, 1);
                    if (pos < BAND_CAP) s_list[pos] = lst[i];
                }
        } else {
            for (uint64_t u = a + tid; u < b; u += blockDim.x)
                if (sub_at(su, sp, wbits, p, u) <= bound) {
                    const int pos = atomicAdd(&s_cnt, 1);
                    if (pos < BAND_CAP) s_list[pos] = u;
                }
        }
    }
    __syncthreads();
    if (tid == 0) {
        const int n = s_cnt;
        if (n <= BAND_CAP) {
            for (int i = 1; i < n && n <= BAND_SORTED; i++) {   // insertion sort: index order (short lists)
                const uint64_t v = s_list[i];
                int j = i - 1;
                while (j >= 0 && s_list[j] > v) { s_list[j + 1] = s_list[j]; j--; }
                s_list[j + 1] = v;
            }
            for (int i = 0; i < n; i++) bandlist[(size_t)p * BAND_CAP + i] = s_list[i];
        }
        bandn[p] = n <= BAND_CAP ? n : -1;
    }
}

cudaError_t launch_reduce_min(const Setup& su, Work& wk, cudaStream_t st) {
    const bool two = qos_float(su);
    cudaError_t e = launch_pdl(k_reduce_min, dim3(su.n_problems), dim3(256), 0, st, su, wk.probs, wk.submin, two ? wk.submin_sure : nullptr, wk.m32,
                                                wk.m32_sure, wk.bandn, wk.bandlist, wk.plist, wk.plist_n,
                                                pass1_prunable(su) ? wk.wbits : nullptr);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// exact evaluation (pass 2)
// ------------------------------------------------------------------------------------------
// exact key of tuple lv (staged records sl); returns false if a QoS bound fails
__device__ bool exact_key(const Setup& su, const Prob& P, const Lev* sl, const int* lv, U256& key) {
    const int W = su.W;
    int64_t Tp = 0;
    for (int w = 0; w < W; w++) Tp += sl[w * su.Lmax + lv[w]].S;
    u128 sum = 0, mx = 0;
    U256 wsum = u256_zero(), wmx = u256_zero();
    for (int w = 0; w < W; w++) {
        const Lev& r = sl[w * su.Lmax + lv[w]];
        u128 O;
        if (su.mode == M_EXCL) O = (u128)(Tp - r.S);
        else if (su.mode == M_PAPER) O = (u128)Tp;
        else if (su.mode == M_EXCESS) O = Tp > P.lamN ? (u128)(Tp - P.lamN) : (u128)0;
        else {
            O = 0;
            for (int v = 0; v < W; v++)
                if (v != w) O += (u128)P.Mi[w * MAXW_ENUM + v] * (u128)sl[v * su.Lmax + lv[v]].S;
        }
        u128 h = (u128)r.B * (P.D + O);
        if (h > P.Hq[w]) return false;
        if (su.weighted) {   // omega_w h_w may exceed 128 bits (R20)
            const U256 wh = u256_mul128((u128)P.wt[w], h);
            wsum = u256_add(wsum, wh);
            if (u256_cmp(wh, wmx) > 0) wmx = wh;
        }
        sum += h;
        if (h > mx) mx = h;
    }
    if (su.weighted && su.obj != O_ENERGY) key = su.obj == O_SUM ? wsum : wmx;
    else if (su.obj == O_SUM) key = u256_of(sum);
    else if (su.obj == O_MAX) key = u256_of(mx);
    else {
        int64_t occ = Tp < P.lamN ? Tp : P.lamN;
        u128 pn = P.pi_idle * (u128)P.lamN + P.pi_dyn * (u128)occ;
        key = u256_mul128(pn, mx);
    }
    return true;
}

// scalar FP32 filter key (error <= delta) and maybe-feasibility, for pass 2
__device__ bool key32_scalar(const Setup& su, const Prob& P, const Lev* sl, const int* lv, float& key) {
    const int W = su.W;
    int64_t Tp = 0, SB = 0, SBS = 0;
    for (int w = 0; w < W; w++) {
        const Lev& r = sl[w * su.Lmax + lv[w]];
        Tp += r.S; SB += r.B; SBS += r.BS;
    }
    const float Tf = __ll2float_rn(Tp);
    float Lw[MAXW_ENUM];
    float num = 0.0f;
    bool feas = true;
    for (int w = 0; w < W; w++) {
        const Lev& r = sl[w * su.Lmax + lv[w]];
        const float bf = __ll2float_rn(r.B);
        float O;
        if (su.wide && (su.mode == M_EXCL || su.mode == M_PAPER)) {   // sum of rounded S' (see k_pass1_gen)
            O = 0.0f;
            for (int v = 0; v < W; v++)
                if (v != w || su.mode == M_PAPER) O += __ll2float_rn(sl[v * su.Lmax + lv[v]].S);
        } else if (su.mode == M_EXCL) O = Tf - (float)r.S;
        else if (su.mode == M_PAPER) O = Tf;
        else if (su.mode == M_EXCESS) O = fmaxf(Tf - P.lamNf, 0.0f);
        else {
            O = 0.0f;
            for (int v = 0; v < W; v++)
                if (v != w) O = fmaf(P.Mf[w * MAXW_ENUM + v], (float)sl[v * su.Lmax + lv[v]].S, O);
        }
        Lw[w] = fmaf(O, r.Bk, bf);
        num = fmaf(bf, O, num);
        if (su.has_qos) {
            if (qos_float(su)) feas = feas && (Lw[w] <= P.Qhi[w]);
            else feas = feas && (Tp <= (int64_t)r.Tmax);
        }
    }
    if (su.weighted && su.obj != O_ENERGY) {   // sum / max of omega_w L_w: <= (2W + 4) u
        key = su.obj == O_SUM ? 0.0f : Lw[0] * P.wf[0];
        for (int w = 0; w < W; w++)
            key = su.obj == O_SUM ? fmaf(P.wf[w], Lw[w], key) : fmaxf(key, Lw[w] * P.wf[w]);
    } else if (su.obj == O_SUM) {
        if (su.mode == M_EXCL && !su.wide) {
            const float bsum = __ll2float_rn(SB);
            key = fmaf(fmaf(Tf, bsum, -__ll2float_rn(SBS)), P.inv, bsum);
        } else {
            key = fmaf(num, P.inv, __ll2float_rn(SB));
        }
    } else {
        float mx = Lw[0];
        for (int w = 1; w < W; w++) mx = fmaxf(mx, Lw[w]);
        key = (su.obj == O_MAX) ? mx : fmaf(P.p_dyn, fminf(1.0f, Tf * P.inv), P.p_idle) * mx;
    }
    return feas;
}


// One CTA per problem.  PASS 0: exact minimum H* over the band.  PASS 1: lowest index whose exact
// key is within tol of the (global) H*.  PASS 2 (unsharded runs): both in one rescan -- the band's
// exactly evaluated candidates are kept in shared memory (a second rescan only on overflow).
constexpr int P2_CAP = 256;
#ifndef P2_THREADS_N
#define P2_THREADS_N 128
#endif
constexpr int P2_THREADS = P2_THREADS_N;
constexpr int P2_ELIST = 1024;   // step levels per unit the pass-2 entry filter handles
#ifndef P2_MINB
#define P2_MINB 6   // 80 registers: 6 CTAs per SM (the band scans are latency-bound; measured 125 -> 109 us on C5)
#endif
template <int PASS>
__global__ void __launch_bounds__(P2_THREADS, P2_MINB) k_pass2(Setup su, Prob* probs, const Lev* __restrict__ levs,
                                               const float* __restrict__ submin, const float* m32,
                                               const float* m32_sure, U256* hstar, U256* first,
                                               const int32_t* bandn, const uint64_t* bandlist,
                                               const float2* hull, const RowHdr* rowhdr, const uint32_t* wbits) {
    pdl_wait();      // (programmatic dependent launch: the predecessor's results are visible)
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ uint64_t bar;
    __shared__ U256 red[P2_THREADS];
    __shared__ uint64_t redi[P2_THREADS];
    __shared__ uint32_t list[P2_THREADS];
    __shared__ int nlist;
    __shared__ int wcount[16], woff[16];
    __shared__ uint64_t c_idx[P2_CAP];
    __shared__ U256 c_key[P2_CAP];
    __shared__ int c_n;
    __shared__ U256 s_hs;
    __shared__ int16_t s_elist[P2_ELIST];
    __shared__ int s_ne;
    Lev* sl = reinterpret_cast<Lev*>(smem_raw);
    const int prob = blockIdx.x;
    Prob& P = probs[prob];
    if (P.status != 0) return;
    if (isinf(m32[prob])) {  // nothing feasible anywhere (global minimum is +inf)
        if (threadIdx.x == 0) {
            if (PASS != 1) hstar[prob] = u256_max();
            if (PASS != 0) first[prob] = u256_max();
        }
        return;
    }
    const int W = su.W;
    stage_levels(sl, levs + (size_t)prob * su.lev_stride, (unsigned)(W * su.Lmax * sizeof(Lev)), &bar);
    const float bound = band_bound(su, m32[prob], m32_sure ? m32_sure[prob] : m32[prob]);
    const int Lin = P.L[W - 1];
    uint64_t slo, shi;
    shard_items(P.n_items, su.shard, su.n_shards, &slo, &shi);
    uint64_t ua = slo * (uint64_t)su.upi, ub = shi * (uint64_t)su.upi;
    if (ub > P.units) ub = P.units;
    int L[MAXW_ENUM];
    for (int w = 0; w < W; w++) L[w] = P.L[w];
    if (threadIdx.x == 0) {
        c_n = 0;
        s_hs = (PASS == 1) ? hstar[prob] : u256_max();
    }
    __syncthreads();
    if (PASS == 1 && u256_is_max(s_hs)) {  // no exactly-feasible candidate
        if (threadIdx.x == 0) first[prob] = u256_max();
        return;
    }

    // phase 0: exact minimum (+ record the band when PASS 2);  phase 1: lowest index within tol
    auto unit_scan = [&](int phase, uint64_t unit, const U256& hs, U256& best, uint64_t& besti) {
        uint64_t row;
        int e0, e1;
        unit_range(P, unit, &row, &e0, &e1);
        int lv[MAXW_ENUM];
        decode_row(row, L, W, lv);
        const uint32_t ncand = (uint32_t)(e1 - e0) * (uint32_t)Lin;
        // exact integer QoS test first (the same predicate as key32_scalar's in the linear modes):
        // hi sums once per unit, then T' = hT + S'_e + S'_k <= min(hTm, Tmax_e, Tmax_k)
        const bool qlin = su.has_qos && !qos_float(su);
        int64_t hT = 0;
        int hTm = 1 << 30;
        if (qlin)
            for (int w = 0; w < W - 2; w++) {
                const Lev& r = sl[w * su.Lmax + lv[w]];
                hT += r.S;
                hTm = min(hTm, r.Tmax);
            }
        const Lev* se = sl + (W >= 2 ? (W - 2) : 0) * su.Lmax;
        const Lev* sk = sl + (W - 1) * su.Lmax;
        auto cand = [&](int ke, int kk) {
            if (qlin) {
                const Lev& rk = sk[kk];
                int64_t Tp = hT + rk.S;
                int Tm = min(hTm, rk.Tmax);
                if (W >= 2) { Tp += se[ke].S; Tm = min(Tm, se[ke].Tmax); }
                if (Tp > (int64_t)Tm) return;
            }
            int lvc[MAXW_ENUM];
            for (int w = 0; w < W - 2; w++) lvc[w] = lv[w];
            if (W >= 2) lvc[W - 2] = ke;
            lvc[W - 1] = kk;
            float k32;
            if (!key32_scalar(su, P, sl, lvc, k32)) return;
            if (!(k32 <= bound)) return;
            U256 k;
            if (!exact_key(su, P, sl, lvc, k)) return;
            uint64_t idx = 0;   // index within the problem (fits: ENUM limits)
            for (int w = 0; w < W; w++) idx = idx * (uint64_t)L[w] + (uint64_t)lvc[w];
            if (phase == 0) {
                if (u256_cmp(k, best) < 0) best = k;
                if (PASS == 2) {
                    const int slot = atomicAdd(&c_n, 1);
                    if (slot < P2_CAP) { c_idx[slot] = idx; c_key[slot] = k; }
                }
            } else if (within_tol(k, hs, su.tol_num, su.tol_den)) {
                if (idx < besti) besti = idx;
            }
        };
        // entry filter (SUM, EXCLUDE_SELF / PAPER with QoS, W >= 3): a step level whose QoS-feasible
        // inner range is empty, or whose every key is provably above the band (the pass-1 entry bound,
        // DESIGN.md §3.9), is not scanned
        int ne_list = -1;
        if (su.aux_bytes > 0 && W >= 3 && su.obj == O_SUM && (su.mode == M_EXCL || su.mode == M_PAPER) && su.has_qos &&
            e1 - e0 <= P2_ELIST) {
            const AuxView A = aux_view(reinterpret_cast<unsigned char*>(const_cast<Lev*>(levs) +
                                                                          (size_t)P.rep * su.lev_stride + (size_t)W * su.Lmax),
                                       su.Lmax);
            int64_t rB = 0, rBS = 0;
            int rT = 0, rTm = 1 << 24;
            for (int w = 0; w < W - 2; w++) {
                const Lev& r = sl[w * su.Lmax + lv[w]];
                rB += r.B; rBS += r.BS; rT += r.S; rTm = min(rTm, r.Tmax);
            }
            const float invf = P.inv;
            const float hBf = __ll2float_rn(rB), hTf = (float)rT;
            const float Yh = fmaf(hTf, invf, 1.0f), Zh = hBf * invf;
            float Xh;
            if (su.mode == M_EXCL) {
                const u128 Dh = (u128)rT * (u128)rB - (u128)rBS;
                const float Dhf = (Dh >> 64) ? (float)(double)Dh : __ull2float_rn((unsigned long long)Dh);
                Xh = fmaf(Dhf, invf, hBf);
            } else {
                Xh = hBf * Yh;
            }
            const int s0 = A.hdr[0], u0v = A.hdr[1], slast = A.ssort[Lin - 1], ulast = A.usuf[Lin - 1];
            const bool khi_ok = A.hdr[2] != 0, klo_ok = A.hdr[3] != 0;
            const double invd = 1.0 / (double)P.lamN;
            __syncthreads();   // the previous unit's list is no longer read
            if (threadIdx.x == 0) s_ne = 0;
            __syncthreads();
            for (int e = e0 + (int)threadIdx.x; e < e1; e += blockDim.x) {
                const Lev& r = se[e];
                const int Tp = rT + r.S, Tm = min(rTm, r.Tmax);
                const int khi = inner_khi(A, Tm - Tp, s0, slast, khi_ok, Lin);
                const int klo = inner_klo(A, Tp, u0v, ulast, klo_ok, Lin);
                const bool pre = A.umaxp[min(klo, khi)] >= Tp;
                bool keep = false;
                if (khi > klo || pre) {
                    const int ka = pre ? 0 : klo;
                    const float Be = __ll2float_rn(r.B), Sf = (float)r.S;
                    float X = fmaf(Be, Yh, fmaf(Sf, Zh, Xh));
                    if (su.mode == M_PAPER) X += (float)((double)r.BS * invd);
                    const float Ye = fmaf(Sf, invf, Yh), Ze = fmaf(Be, invf, Zh);
                    float lbe = fmaf(Ye, A.preminB[khi], fmaf(Ze, (float)A.ssort[ka], X));
                    if (!(lbe * 0.99998474121f > bound))   // the inner hull restricted to the S' range (aux block)
                        lbe = fmaxf(lbe, X + hull_min_pos(A, *A.ihn, Ye, Ze, ka, khi - 1));
                    keep = !(lbe * 0.99998474121f > bound);   // 1 - 2^-16
                }
                if (keep) s_elist[atomicAdd(&s_ne, 1)] = (int16_t)e;
            }
            __syncthreads();
            ne_list = s_ne;
        }
        // 2-D thread map (inner level fixed per thread, step levels strided) when a padded row of
        // inner levels fits the block: no division per candidate
        const int KP = (Lin + 31) & ~31;
        if (KP <= (int)blockDim.x && ne_list >= 0) {
            const int EP = (int)blockDim.x / KP, kk = (int)threadIdx.x % KP, eo = (int)threadIdx.x / KP;
            if (kk < Lin && eo < EP)
                for (int i = eo; i < ne_list; i += EP) cand(s_elist[i], kk);
        } else if (KP <= (int)blockDim.x) {
            const int EP = (int)blockDim.x / KP, kk = (int)threadIdx.x % KP, eo = (int)threadIdx.x / KP;
            if (kk < Lin && eo < EP)
                for (int ke = e0 + eo; ke < e1; ke += EP) cand(ke, kk);
        } else {
            for (uint32_t c = threadIdx.x; c < ncand; c += blockDim.x)
                cand(W >= 2 ? e0 + (int)(c / (uint32_t)Lin) : 0, (int)(c % (uint32_t)Lin));
        }
    };
    const int nband = bandn ? bandn[prob] : -1;
    ECLIP_CHECK(nband <= BAND_CAP);
    auto scan = [&](int phase, U256& best, uint64_t& besti) {
        const U256 hs = s_hs;
        if (nband >= 0) {   // the band's units, listed in index order by k_reduce_min
            for (int i = 0; i < nband; i++) {
                const uint64_t unit = bandlist[(size_t)prob * BAND_CAP + i];
                if (!(sub_at(su, submin + (size_t)prob * su.units_max, wbits, prob, unit) <= bound)) continue;
                unit_scan(phase, unit, hs, best, besti);
                // in an index-ordered list the first unit with a hit holds the winner
                if (phase == 1 && nband <= BAND_SORTED && __syncthreads_or(besti != ~0ull)) break;
            }
            __syncthreads();
            return;
        }
        bool done = false;
        for (uint64_t blk = ua; blk < ub && !done; blk += blockDim.x) {
            const uint64_t u = blk + threadIdx.x;
            const bool in_band = u < ub && sub_at(su, submin + (size_t)prob * su.units_max, wbits, prob, u) <= bound;
            if (threadIdx.x == 0) nlist = 0;
            __syncthreads();
            const unsigned bal = __ballot_sync(0xffffffffu, in_band);
            if ((threadIdx.x & 31) == 0) wcount[threadIdx.x >> 5] = __popc(bal);
            __syncthreads();
            if (threadIdx.x == 0) {
                int acc = 0;
                for (int w = 0; w < (int)(blockDim.x >> 5); w++) { woff[w] = acc; acc += wcount[w]; }
                nlist = acc;
            }
            __syncthreads();
            if (in_band) list[woff[threadIdx.x >> 5] + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u))] = (uint32_t)(u - blk);
            __syncthreads();
            const int nl = nlist;
            for (int li = 0; li < nl; li++) {   // units in candidate-index order
                const uint64_t unit = blk + list[li];
                unit_scan(phase, unit, hs, best, besti);
                if (phase == 1 && __syncthreads_or(besti != ~0ull)) {   // first unit with a hit holds the winner
                    done = true;
                    break;
                }
            }
            __syncthreads();
        }
    };
    auto write_first = [&](uint64_t idx) {
        if (idx == ~0ull) first[prob] = u256_max();
        else {
            int lv[MAXW_ENUM];
            for (int w = W - 1; w >= 0; w--) {
                uint32_t r;
                idx = udiv_small(idx, (uint32_t)L[w], &r);
                lv[w] = (int)r;
            }
            first[prob] = pack_tuple(lv, W);
        }
    };

    U256 best = u256_max();
    uint64_t besti = ~0ull;
    const int nwp = (int)(blockDim.x >> 5), wlane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (PASS != 1) {
        scan(0, best, besti);
        // block minimum: warp shuffles, then the warps' minima
        for (int o = 16; o; o >>= 1) {
            U256 y;
            for (int i = 0; i < 4; i++) y.w[i] = __shfl_xor_sync(0xffffffffu, best.w[i], o);
            if (u256_cmp(y, best) < 0) best = y;
        }
        if (wlane == 0) red[wid] = best;
        __syncthreads();
        if (threadIdx.x == 0) {
            U256 m = red[0];
            for (int i = 1; i < nwp; i++)
                if (u256_cmp(red[i], m) < 0) m = red[i];
            hstar[prob] = m;
            s_hs = m;
        }
        __syncthreads();
        if (PASS == 0) return;
        if (u256_is_max(s_hs)) {
            if (threadIdx.x == 0) first[prob] = u256_max();
            return;
        }
    }
    if (PASS == 2 && c_n <= P2_CAP) {   // the whole band is in shared memory
        const U256 hs = s_hs;
        for (int i = threadIdx.x; i < c_n; i += blockDim.x)
            if (within_tol(c_key[i], hs, su.tol_num, su.tol_den) && c_idx[i] < besti) besti = c_idx[i];
    } else {
        scan(1, best, besti);
    }
    for (int o = 16; o; o >>= 1) {
        const uint64_t y = __shfl_xor_sync(0xffffffffu, besti, o);
        besti = y < besti ? y : besti;
    }
    if (wlane == 0) redi[wid] = besti;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t m = redi[0];
        for (int i = 1; i < nwp; i++) m = redi[i] < m ? redi[i] : m;
        write_first(m);
    }
}

cudaError_t launch_pass2_min(const Setup& su, Work& wk, cudaStream_t st) {
    size_t smem = (size_t)su.W * su.Lmax * sizeof(Lev);
    cudaError_t e = cudaFuncSetAttribute((const void*)k_pass2<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_pass2<0><<<su.n_problems, P2_THREADS, smem, st>>>(su, wk.probs, wk.levs, wk.submin, wk.m32,
                                                 qos_float(su) ? wk.m32_sure : nullptr,
                                                 wk.hstar, wk.first, wk.bandn, wk.bandlist, wk.hull, wk.rowhdr,
                                                 pass1_prunable(su) ? wk.wbits : nullptr);
    return cudaGetLastError();
}
cudaError_t launch_pass2_both(const Setup& su, Work& wk, cudaStream_t st) {
    size_t smem = (size_t)su.W * su.Lmax * sizeof(Lev);
    cudaError_t e = cudaFuncSetAttribute((const void*)k_pass2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = launch_pdl(k_pass2<2>, dim3(su.n_problems), dim3(P2_THREADS), smem, st, su, wk.probs, wk.levs, wk.submin, wk.m32,
                   qos_float(su) ? wk.m32_sure : nullptr, wk.hstar, wk.first, wk.bandn, wk.bandlist, wk.hull, wk.rowhdr,
                   pass1_prunable(su) ? wk.wbits : nullptr);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}
cudaError_t launch_pass2_first(const Setup& su, Work& wk, cudaStream_t st) {
    size_t smem = (size_t)su.W * su.Lmax * sizeof(Lev);
    cudaError_t e = cudaFuncSetAttribute((const void*)k_pass2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_pass2<1><<<su.n_problems, P2_THREADS, smem, st>>>(su, wk.probs, wk.levs, wk.submin, wk.m32,
                                                 qos_float(su) ? wk.m32_sure : nullptr,
                                                 wk.hstar, wk.first, wk.bandn, wk.bandlist, wk.hull, wk.rowhdr,
                                                 pass1_prunable(su) ? wk.wbits : nullptr);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// materialisation (a9): one CTA per problem (thread 0: per-worker scalars; all threads: groups)
// ------------------------------------------------------------------------------------------
// LPP = 32: one warp per problem, several problems per CTA (batches: the work is a short latency chain, so
// more problems in flight is what matters); LPP = 128: a CTA per problem (few problems with many groups)
constexpr int MZ_MAXPPC = 4;
template <int LPP>
__global__ void __launch_bounds__(128) k_materialize(Setup su, Tables tb, const Prob* probs, const Lev* levs,
                                                     const U256* hstar, const U256* first, const int32_t* sizes, int C,
                                                     MatOut o) {
    pdl_wait();      // (programmatic dependent launch: the predecessor's results are visible)
    pdl_trigger();
    const int wp = LPP == 32 ? (int)(threadIdx.x >> 5) : 0, lane = LPP == 32 ? (int)(threadIdx.x & 31) : (int)threadIdx.x;
    const int p = LPP == 32 ? (int)(blockIdx.x * (blockDim.x >> 5)) + wp : (int)blockIdx.x;
    auto gsync = [&]() { if (LPP == 32) __syncwarp(); else __syncthreads(); };
    if (p >= su.n_problems) return;   // (whole warps / CTAs)
    const Prob& P = probs[p];
    const int W = su.W;
    __shared__ int lv_s[MZ_MAXPPC][MAXW];
    __shared__ double alpha_s[MZ_MAXPPC][MAXW];
    __shared__ int goff_s[MZ_MAXPPC][MAXW + 1];
    int* lv = lv_s[wp];
    double* alpha_w = alpha_s[wp];
    int status = P.status;
    if (status == 0 && (u256_is_max(first[p]) || u256_is_max(hstar[p]))) status = 1;  // infeasible
    if (lane == 0 && o.status) o.status[p] = status;
    if (status != 0) {
        if (lane == 0) {
            if (o.index) o.index[p] = 0;
            if (o.energy_busy) o.energy_busy[p] = 0.0;
            if (o.objective) o.objective[p] = 0.0;
            if (o.makespan) o.makespan[p] = 0.0;
            if (o.power) o.power[p] = 0.0;
            if (o.energy) o.energy[p] = 0.0;
            if (o.thr) o.thr[p] = 0.0;
        }
        for (int i = lane; i < W; i += LPP) {
            if (o.levels) o.levels[(size_t)p * W + i] = -1;
            if (o.latency) o.latency[(size_t)p * W + i] = 0.0;
            if (o.switches) o.switches[(size_t)p * W + i] = 0;
        }
        if (o.group_sm)
            for (int i = lane; i < W * o.group_stride; i += LPP) o.group_sm[(size_t)p * W * o.group_stride + i] = 0;
        return;
    }
    if (lane == 0) {
        int l[MAXW];
        unpack_tuple(first[p], W, l);
        // mixed-radix candidate index (worker 0 most significant); all-ones if it needs > 64 bits
        uint64_t idx = 0;
        bool fits = true;
        for (int w = 0; w < W; w++) {
            u128 t = (u128)idx * (u128)P.L[w] + (u128)l[w];
            if (t >> 64) fits = false;
            idx = (uint64_t)t;
            lv[w] = l[w];
        }
        // FP64 values from exact integers
        double avg[MAXW], Bw[MAXW], sum_avg = 0.0;
        for (int w = 0; w < W; w++) {
            const int t = P.table[w];
            avg[w] = (double)tb.S[t][l[w]] / (double)tb.K[t];
            Bw[w] = (double)tb.B[t][l[w]];
            sum_avg += avg[w];
        }
        const double N = (double)su.N;
        double mk = 0.0, wmk = 0.0, obj = 0.0, thr = 0.0;
        for (int w = 0; w < W; w++) {
            double ov;
            if (su.mode == M_EXCL) ov = sum_avg - avg[w];
            else if (su.mode == M_PAPER) ov = sum_avg;
            else if (su.mode == M_EXCESS) ov = sum_avg - N > 0.0 ? sum_avg - N : 0.0;
            else {
                ov = 0.0;
                for (int v = 0; v < W; v++)
                    if (v != w) ov += (double)P.Mf[w * MAXW_ENUM + v] * avg[v];
            }
            const double alpha = ov / N;
            const double Lw = Bw[w] * (1.0 + alpha);
            alpha_w[w] = alpha;
            mk = Lw > mk ? Lw : mk;
            obj += P.wv[w] * Lw;
            wmk = P.wv[w] * Lw > wmk ? P.wv[w] * Lw : wmk;
            thr += 1e9 / Lw;
            if (o.latency) o.latency[(size_t)p * W + w] = Lw;
            if (o.levels) o.levels[(size_t)p * W + w] = l[w];
        }
        double frac = sum_avg / N;
        if (frac > 1.0) frac = 1.0;
        const double pw = (double)P.p_idle + ((double)P.p_max - (double)P.p_idle) * frac;
        if (su.obj == O_MAX) obj = wmk;
        else if (su.obj == O_ENERGY) obj = pw * mk;
        if (o.index) o.index[p] = fits ? idx : ~0ull;
        if (o.objective) o.objective[p] = obj;
        if (o.makespan) o.makespan[p] = mk;
        if (o.power) o.power[p] = pw;
        if (o.energy) o.energy[p] = pw * mk * 1e-9;
        if (o.thr) o.thr[p] = thr;
        if (o.key) {
            U256 k;
            exact_key(su, P, levs + (size_t)p * su.lev_stride, l, k);
            for (int i = 0; i < 4; i++) o.key[(size_t)p * 4 + i] = k.w[i];
        }
    }
    gsync();
    // per worker: switch count; per group: pool size and e_g = beta_g (1 + alpha_w)
    for (int w = lane; w < W; w += LPP) {
        const int t = P.table[w], G = tb.G[t];
        const uint8_t* wit = tb.wit[t] + (size_t)lv[w] * G;
        int sw = 0;
        for (int g = 1; g < G; g++) sw += wit[g] != wit[g - 1];
        if (o.switches) o.switches[(size_t)p * W + w] = sw;
    }
    for (int w = 0; w < W; w++) {
        const int t = P.table[w], G = tb.G[t];
        const uint8_t* wit = tb.wit[t] + (size_t)lv[w] * G;
        for (int g = lane; g < o.group_stride; g += LPP) {
            const size_t at = ((size_t)p * W + w) * o.group_stride + g;
            if (o.group_sm) o.group_sm[at] = g < G ? sizes[wit[g]] : 0;
            if (o.group_lat && g < G) o.group_lat[at] = (double)tb.beta[t][g * C + wit[g]] * (1.0 + alpha_w[w]);
        }
    }
    // busy-SM energy integral of the predicted run (SPEC integrate_energy S:416-419, power_at S:406-409;
    // DESIGN.md R21): every worker starts at 0 and runs its groups back to back; between consecutive group
    // boundaries the power is p_idle + (p_max - p_idle) min(N, sum of the running groups' SMs) / N
    if (o.energy_busy) {
        // the workers' group end times (sequential sums, as the run) and pool sizes in shared memory, the
        // ends ranked into time order, then one elementary interval per lane: its busy SMs from a binary
        // search of each worker's ends, its energy, and a warp sum
        extern __shared__ __align__(8) unsigned char msm[];
        const int gs = o.gsum;
        double* ends = reinterpret_cast<double*>(msm + (size_t)wp * (((size_t)gs * 20 + 7) & ~(size_t)7));   // [gs] per worker
        double* srt = ends + gs;                                               // [gs] all ends in time order
        int* csz = reinterpret_cast<int*>(srt + gs);                           // [gs] pool size of each group
        int* goff = goff_s[wp];
        if (lane == 0) {
            goff[0] = 0;
            for (int w = 0; w < W; w++) goff[w + 1] = goff[w] + tb.G[P.table[w]];
        }
        gsync();
        const int n = goff[W];
        for (int w = 0; w < W; w++) {   // every group's duration and pool size, in parallel
            const int t = P.table[w], G = tb.G[t];
            const uint8_t* wt = tb.wit[t] + (size_t)lv[w] * G;
            for (int g = lane; g < G; g += LPP) {
                ends[goff[w] + g] = (double)tb.beta[t][g * C + wt[g]] * (1.0 + alpha_w[w]);
                csz[goff[w] + g] = sizes[wt[g]];
            }
        }
        gsync();
        for (int w = lane; w < W; w += LPP) {   // one lane per worker: its run, in order
            double e = 0.0;
            for (int i = goff[w]; i < goff[w + 1]; i++) { e += ends[i]; ends[i] = e; }
        }
        gsync();
        for (int i = lane; i < n; i += LPP) {   // rank of end i (ties by position): each worker's ends ascend, so
            const double v = ends[i];           // count by binary search
            int wi = 0;
            while (goff[wi + 1] <= i) wi++;
            int rk = i - goff[wi];
            for (int w = 0; w < W; w++) {
                if (w == wi) continue;
                int lo = goff[w], hi = goff[w + 1];   // count of ends < v, or <= v for earlier workers
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (ends[mid] < v || (w < wi && ends[mid] == v)) lo = mid + 1; else hi = mid;
                }
                rk += lo - goff[w];
            }
            ECLIP_CHECK(rk >= 0 && rk < n && n <= gs);
            srt[rk] = v;
        }
        gsync();
        const double Nd = (double)su.N, pi = (double)P.p_idle, pd = (double)P.p_max - (double)P.p_idle;
        double E = 0.0;
        for (int k = lane; k < n; k += LPP) {   // interval [srt[k-1], srt[k])
            const double t0 = k ? srt[k - 1] : 0.0, t1 = srt[k];
            if (!(t1 > t0)) continue;
            int busy = 0;
            for (int w = 0; w < W; w++) {   // the worker's group running at t0: first end > t0
                int lo = goff[w], hi = goff[w + 1];
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (ends[mid] <= t0) lo = mid + 1; else hi = mid;
                }
                if (lo < goff[w + 1]) busy += csz[lo];
            }
            E += (pi + pd * (double)min(busy, su.N) / Nd) * (t1 - t0);
        }
        for (int off = 16; off; off >>= 1) E += __shfl_xor_sync(0xffffffffu, E, off);
        if (LPP == 32) {
            if (lane == 0) o.energy_busy[p] = E * 1e-9;
        } else {
            __shared__ double red_e[4];
            if ((threadIdx.x & 31) == 0) red_e[threadIdx.x >> 5] = E;
            __syncthreads();
            if (threadIdx.x == 0) o.energy_busy[p] = (red_e[0] + red_e[1] + red_e[2] + red_e[3]) * 1e-9;
        }
    }
}

cudaError_t launch_materialize(const Setup& su, const Tables& tb, Work& wk, const int32_t* sizes, int C, MatOut out,
                               cudaStream_t st) {
    const size_t per = out.energy_busy ? (((size_t)out.gsum * 20 + 7) & ~(size_t)7) : 0;   // busy-energy staging per problem
    cudaError_t e;
    if (su.n_problems < 148 * 4) {   // few problems: a CTA each
        if (per > 48 * 1024 &&
            (e = cudaFuncSetAttribute((const void*)k_materialize<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per)) !=
                cudaSuccess)
            return e;
        e = launch_pdl(k_materialize<128>, dim3(su.n_problems), dim3(128), per, st, su, tb, wk.probs, wk.levs, wk.hstar,
                       wk.first, sizes, C, out);
        if (e != cudaSuccess) return e;
        return cudaGetLastError();
    }
    int ppc = MZ_MAXPPC;
    while (ppc > 1 && per * (size_t)ppc > 48 * 1024) ppc--;
    const size_t sm = per * (size_t)ppc;
    if (sm > 48 * 1024) {
        e = cudaFuncSetAttribute((const void*)k_materialize<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
    }
    e = launch_pdl(k_materialize<32>, dim3((su.n_problems + ppc - 1) / ppc), dim3(32 * ppc), sm, st, su, tb, wk.probs,
                   wk.levs, wk.hstar, wk.first, sizes, C, out);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// per level table: S order and lower-left hull vertices (shared by every problem using the table)
cudaError_t launch_table_hull(const Setup& su, const Tables& tb, Work& wk, cudaStream_t st) {
    if (su.aux_bytes <= 0) return cudaSuccess;
    const size_t hsm = (size_t)su.Lmax * (8 + 4 + 2 + 1) + 16;
    cudaError_t e = cudaFuncSetAttribute((const void*)k_table_hull, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
    if (e != cudaSuccess) return e;
    k_table_hull<<<tb.n, 256, hsm, st>>>(tb, su.Lmax, wk.thull, wk.thull_n, wk.tord);
    return cudaGetLastError();
}

cudaError_t launch_prep(const Setup& su, const Tables& tb, const PrepIn& in, Work& wk, int C, const int32_t* sizes,
                        cudaStream_t st, bool table_hull) {
    (void)C; (void)sizes;
    cudaError_t e;
    // one warp per block: all SMs
    if ((e = launch_pdl(k_prep_prob, dim3((su.n_problems + 31) / 32), dim3(32), 0, st, su, tb, in, wk.probs)) != cudaSuccess)
        return e;
    size_t n = (size_t)su.n_problems * su.W * su.Lmax;
    if ((e = launch_pdl(k_prep_lev, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, su, tb, wk.probs, wk.levs)) !=
        cudaSuccess)
        return e;
    if (su.aux_bytes > 0) {
        if (su.n_problems > 1 && wk.aslots > 0) {   // representatives of the step / inner precomputation
            const size_t ns = (size_t)wk.aslots;
            Fill4 f{};
            f.p[0] = reinterpret_cast<unsigned*>(wk.aslot); f.n[0] = 2 * ns; f.v[0] = 0u;
            f.p[1] = reinterpret_cast<unsigned*>(wk.aslot + ns); f.n[1] = 2 * ns; f.v[1] = 0xffffffffu;
            if ((e = fill4(f, st)) != cudaSuccess) return e;
            if ((e = launch_pdl(k_akey, dim3((su.n_problems + 7) / 8), dim3(256), 0, st, su, wk.probs, wk.levs, wk.akey,
                                wk.aslot, wk.aslots)) != cudaSuccess)
                return e;
            if ((e = launch_pdl(k_arep, dim3((su.n_problems + 255) / 256), dim3(256), 0, st, su, wk.probs, wk.akey, wk.aslot,
                                wk.aslots)) != cudaSuccess)
                return e;
        }
        if (table_hull && (e = launch_table_hull(su, tb, wk, st)) != cudaSuccess) return e;
        const size_t sm = (size_t)2 * su.Lmax * sizeof(Lev) + (size_t)su.aux_bytes;
        auto f = su.mode == M_PAPER ? k_prep_aux<M_PAPER> : k_prep_aux<M_EXCL>;
        e = cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        if ((e = launch_pdl(f, dim3(su.n_problems), dim3(256), sm, st, su, wk.probs, wk.levs, in.table_of, wk.tord, wk.thull,
                            wk.thull_n)) != cudaSuccess)
            return e;
    }
    return cudaGetLastError();
}

}  // namespace eclip
