/*
 * oracle/eclip_oracle.c — O-B, the reduced EXACT oracle for the ECLIP resource-allocation
 * optimizer (§IV-B "Optimization Formulation").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code, header,
 * constant or table generator with paper_2506_12598_b200/ (the product path), and the
 * product never loads it.  Its own pins: tests/test_oracle_*.py (against O-A, the literal
 * brute force of oracle/brute.py, App. B worked examples, SPEC printed values, closed forms).
 *
 * Plain, single-threaded, written for checkability, not speed.  All decisions are EXACT
 * (integers):
 *
 *   or_levels    level table of ONE worker: for every attained CU-sum S,
 *                B*(S) = min solo time and the canonical witness (lexicographically
 *                smallest minimiser), by memoised recursion best(g, prev, used, rem) over
 *                the paper's constraints (one config per kernel P:300, switchTotal_w <=
 *                switchMax P:302-303).  Levels are returned in witness (rank) order.
 *   or_enum      every level tuple in index order; exact key per tuple; m = exact min;
 *                winner = lowest index with key <= m (1 + tau)   (tau rational).
 *   or_slice     the same answer by T'-slicing (linear slowdown modes): exact suffix
 *                (min,+) / (min,max) DP per slice, then the lexicographic walk.
 *   or_eval_f64  FP64 values of a chosen plan (latency, objective, power, energy, RPS).
 *
 * Exact key of a tuple:
 *   Lambda = lcm_w K_w,  S'_w = S_w Lambda / K_w  (so CUAverage_w = S'_w / Lambda),
 *   T' = sum_w S'_w,  D = Lambda N 2^E  (E = fraction bits of the slowdown matrix, else 0),
 *   O^_w = CUOverlap_w * Lambda * 2^E:  EXCLUDE_SELF (T'-S'_w) | PAPER T' | EXCESS
 *          max(0, T' - Lambda N) | MATRIX sum_{v!=w} M_wv 2^E S'_v,
 *   h_w  = B_w (D + O^_w)            so  L_w = sum_k e_k = B_w (1 + alpha_w) = h_w / D,
 *   SUM: sum_w omega_w h_w;  MAX: max_w omega_w h_w  (omega_w = per-worker weight integers, SPEC S:130;
 *        all 1 = the paper's "identically weighted" objective);
 *   ENERGY: (p_idle Lambda N + (p_max - p_idle) min(Lambda N, T')) 2^k * max_w h_w
 *   QoS: L_w <= Q_w  <=>  h_w <= Q_w D (exact dyadic compare).
 * All keys share one positive denominator per problem, so comparing these integers is
 * comparing the paper's quantities exactly.
 *
 * Build: gcc -O2 -std=gnu11 -ffp-contract=off -shared -fPIC -lm
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef __int128 i128;

/* ------------------------------------------------------------------------------------ */
/* 256-bit unsigned integers (4 little-endian 64-bit limbs), for exact keys.              */
/* ------------------------------------------------------------------------------------ */
typedef struct { uint64_t w[4]; } u256;

static u256 u256_zero(void) { u256 r; memset(&r, 0, sizeof r); return r; }
static u256 u256_from128(u128 a) { u256 r = u256_zero(); r.w[0] = (uint64_t)a; r.w[1] = (uint64_t)(a >> 64); return r; }
static int u256_cmp(u256 a, u256 b) {
    for (int i = 3; i >= 0; i--) { if (a.w[i] < b.w[i]) return -1; if (a.w[i] > b.w[i]) return 1; }
    return 0;
}
static u256 u256_add(u256 a, u256 b) {
    u256 r; u128 c = 0;
    for (int i = 0; i < 4; i++) { c += (u128)a.w[i] + b.w[i]; r.w[i] = (uint64_t)c; c >>= 64; }
    return r;
}
/* a (u256, assumed < 2^192) times b (< 2^64) */
static u256 u256_mul64(u256 a, uint64_t b) {
    u256 r; u128 c = 0;
    for (int i = 0; i < 4; i++) { c += (u128)a.w[i] * b; r.w[i] = (uint64_t)c; c >>= 64; }
    return r;
}
static u256 u256_mul128(u128 a, u128 b) {
    uint64_t a0 = (uint64_t)a, a1 = (uint64_t)(a >> 64), b0 = (uint64_t)b, b1 = (uint64_t)(b >> 64);
    u256 r = u256_zero();
    u128 p00 = (u128)a0 * b0, p01 = (u128)a0 * b1, p10 = (u128)a1 * b0, p11 = (u128)a1 * b1;
    u256 t;
    t = u256_zero(); t.w[0] = (uint64_t)p00; t.w[1] = (uint64_t)(p00 >> 64); r = u256_add(r, t);
    t = u256_zero(); t.w[1] = (uint64_t)p01; t.w[2] = (uint64_t)(p01 >> 64); r = u256_add(r, t);
    t = u256_zero(); t.w[1] = (uint64_t)p10; t.w[2] = (uint64_t)(p10 >> 64); r = u256_add(r, t);
    t = u256_zero(); t.w[2] = (uint64_t)p11; t.w[3] = (uint64_t)(p11 >> 64); r = u256_add(r, t);
    return r;
}
static u256 u256_shl(u256 a, int s) {
    u256 r = u256_zero();
    int q = s / 64, m = s % 64;
    for (int i = 3; i >= 0; i--) {
        int src = i - q;
        if (src < 0) continue;
        uint64_t v = a.w[src] << m;
        if (m && src - 1 >= 0) v |= a.w[src - 1] >> (64 - m);
        r.w[i] = v;
    }
    return r;
}
static int u256_bits(u256 a) {
    for (int i = 3; i >= 0; i--) if (a.w[i]) { int b = 64; while (!((a.w[i] >> (b - 1)) & 1)) b--; return 64 * i + b; }
    return 0;
}
double or_u256_to_double(const uint64_t* w) {
    return ldexp((double)w[3], 192) + ldexp((double)w[2], 128) + ldexp((double)w[1], 64) + (double)w[0];
}

/* exact test  h <= q * D  for a double q >= 0 (may be +inf) and integers h, D >= 1 */
static int le_dyadic(u128 h, double q, u128 D) {
    if (isinf(q)) return 1;
    if (q <= 0.0) return h == 0;
    int ex;
    double f = frexp(q, &ex);                 /* q = f 2^ex, f in [0.5, 1) */
    uint64_t mant = (uint64_t)ldexp(f, 53);   /* exact: q = mant 2^(ex-53) */
    int e = ex - 53;
    u256 rhs = u256_mul128((u128)mant, D);
    u256 lhs = u256_from128(h);
    if (e >= 0) {
        if (u256_bits(rhs) + e > 250) return 1;
        rhs = u256_shl(rhs, e);
    } else {
        if (u256_bits(lhs) + (-e) > 250) return 0;
        lhs = u256_shl(lhs, -e);
    }
    return u256_cmp(lhs, rhs) <= 0;
}

/* ------------------------------------------------------------------------------------ */
/* Level table of one worker.                                                             */
/* A plan is sigma in A^G (A = allowed size columns) with sw(sigma) = #{g>=1 : sigma_g !=  */
/* sigma_{g-1}} <= R.  Level S = sum_g n_g c_{sigma_g}; solo B = sum_g      */
/* beta[g][sigma_g].  For every attained S: B*(S) and wit(S) = lexicographically  */
/* smallest minimiser (group 0 most significant, smaller size column first).              */
/* ------------------------------------------------------------------------------------ */
#define OR_INF64 INT64_MAX

typedef struct {
    int G, C, R, NONE;
    long smax;
    const int64_t* beta;
    const int32_t* need;
    uint32_t mask;
    int64_t* memoB;        /* -2 = not computed, OR_INF64 = unreachable */
    int8_t* memoJ;
} lv_ctx;

static size_t lv_key(const lv_ctx* c, int g, int prev, int used, long rem) {
    return ((((size_t)g * (size_t)(c->C + 1) + (size_t)prev) * (size_t)(c->R + 1) + (size_t)used)
            * (size_t)(c->smax + 1)) + (size_t)rem;
}

/* best(g, prev, used, rem): min of sum_{g'>=g} beta over completions with level exactly rem
 * and at most R switches in total; ties -> smallest sigma_g, which applied recursively
 * yields the lexicographically smallest minimiser. */
static int64_t lv_best(lv_ctx* c, int g, int prev, int used, long rem) {
    if (g == c->G) return rem == 0 ? 0 : OR_INF64;
    size_t k = lv_key(c, g, prev, used, rem);
    if (c->memoB[k] != -2) return c->memoB[k];
    int64_t bestB = OR_INF64;
    int bestJ = -1;
    for (int j = 0; j < c->C; j++) {
        if (!((c->mask >> j) & 1u)) continue;
        int u2 = used + ((prev != c->NONE && j != prev) ? 1 : 0);
        if (u2 > c->R) continue;
        long nd = c->need[g * c->C + j];
        if (nd > rem) continue;
        int64_t child = lv_best(c, g + 1, j, u2, rem - nd);
        if (child == OR_INF64) continue;
        int64_t tot = c->beta[g * c->C + j] + child;
        if (tot < bestB) { bestB = tot; bestJ = j; }
    }
    c->memoB[k] = bestB;
    c->memoJ[k] = (int8_t)bestJ;
    return bestB;
}

static int lv_G_for_sort;
static int lv_cmp(const void* a, const void* b) {
    return memcmp(*(const uint8_t* const*)a, *(const uint8_t* const*)b, (size_t)lv_G_for_sort);
}
static long gcd_l(long a, long b) { while (b) { long t = a % b; a = b; b = t; } return a; }

/* Returns L (>= 1), 0 if no plan exists, -1 bad input, -2 cap too small, -3 out of memory.
 * Outputs in rank order: out_S[L] (SM units), out_B[L] (ns), out_wit[L*G] (size column). */
int or_levels(int G, int C, const int64_t* beta, const int32_t* weight, const int32_t* sizes,
              uint32_t mask, int R, int64_t* out_S, int64_t* out_B, uint8_t* out_wit, int cap) {
    if (G < 1 || C < 1 || C > 32 || R < 0) return -1;
    int Reff = R < G - 1 ? R : G - 1;          /* at most G-1 switches can occur */
    long u = 0;
    for (int j = 0; j < C; j++) if ((mask >> j) & 1u) u = gcd_l(u, sizes[j]);
    if (u == 0) return 0;
    lv_ctx c;
    c.G = G; c.C = C; c.R = Reff; c.NONE = C; c.beta = beta; c.mask = mask;
    int32_t* need = (int32_t*)malloc(sizeof(int32_t) * (size_t)G * (size_t)C);
    long smax = 0;
    for (int g = 0; g < G; g++) {
        long mx = 0;
        for (int j = 0; j < C; j++) {
            need[g * C + j] = (int32_t)((long)weight[g] * sizes[j] / u);
            if (((mask >> j) & 1u) && need[g * C + j] > mx) mx = need[g * C + j];
        }
        smax += mx;
    }
    c.need = need; c.smax = smax;
    size_t n = (size_t)G * (size_t)(C + 1) * (size_t)(Reff + 1) * (size_t)(smax + 1);
    c.memoB = (int64_t*)malloc(n * sizeof(int64_t));
    c.memoJ = (int8_t*)malloc(n);
    if (!c.memoB || !c.memoJ) { free(need); free(c.memoB); free(c.memoJ); return -3; }
    for (size_t i = 0; i < n; i++) c.memoB[i] = -2;

    int L = 0;
    int64_t* tS = (int64_t*)malloc(sizeof(int64_t) * (size_t)(smax + 1));
    int64_t* tB = (int64_t*)malloc(sizeof(int64_t) * (size_t)(smax + 1));
    uint8_t* tW = (uint8_t*)malloc((size_t)(smax + 1) * (size_t)G);
    for (long s = 0; s <= smax; s++) {
        int64_t b = lv_best(&c, 0, c.NONE, 0, s);
        if (b == OR_INF64) continue;
        int prev = c.NONE, used = 0;
        long rem = s;
        for (int g = 0; g < G; g++) {
            int j = c.memoJ[lv_key(&c, g, prev, used, rem)];
            tW[(size_t)L * G + g] = (uint8_t)j;
            used += (prev != c.NONE && j != prev) ? 1 : 0;
            rem -= need[g * C + j];
            prev = j;
        }
        tS[L] = s * u;
        tB[L] = b;
        L++;
    }
    int rc = L;
    if (L > cap) rc = -2;
    else if (L > 0) {
        const uint8_t** ptr = (const uint8_t**)malloc(sizeof(uint8_t*) * (size_t)L);
        for (int i = 0; i < L; i++) ptr[i] = tW + (size_t)i * G;
        lv_G_for_sort = G;
        qsort(ptr, (size_t)L, sizeof(uint8_t*), lv_cmp);   /* canonical rank order */
        for (int r = 0; r < L; r++) {
            int i = (int)((ptr[r] - tW) / G);
            out_S[r] = tS[i];
            out_B[r] = tB[i];
            memcpy(out_wit + (size_t)r * G, tW + (size_t)i * G, (size_t)G);
        }
        free(ptr);
    }
    free(tS); free(tB); free(tW); free(need); free(c.memoB); free(c.memoJ);
    return rc;
}

/* ------------------------------------------------------------------------------------ */
/* Exact keys.                                                                            */
/* ------------------------------------------------------------------------------------ */
enum { OR_EXCLUDE_SELF = 0, OR_PAPER = 1, OR_EXCESS = 2, OR_MATRIX = 3 };
enum { OR_SUM = 0, OR_MAX = 1, OR_ENERGY = 2 };
#define OR_MAXW 16

typedef struct {
    int32_t W, N, mode, objective;
    const int32_t* L;       /* [W] level counts */
    const int64_t* S;       /* [sum L] level CU-sums (SM units), rank order, worker-major */
    const int64_t* B;       /* [sum L] level solo times B* (ns) */
    const int64_t* K;       /* [W] kernels per worker (sum n_g) */
    const double* Q;        /* [W] QoS bound (ns); +inf = none */
    const float* M;         /* [W*W] slowdown matrix (MATRIX only), entries >= 0 */
    float p_idle, p_max;
    int64_t tol_num, tol_den;   /* tau = tol_num / tol_den */
    const int64_t* wt;      /* [W] per-worker objective weights as positive integers ("weights: per-worker
                               scalar (default all 1)"; reading R20: round(omega 1e6) divided by the gcd
                               over workers); NULL = all 1 (the paper's equal weights) */
    const double* wval;     /* [W] the weights' values round(omega 1e6) / 1e6 (FP64 objective), NULL = all 1 */
} or_problem;

typedef struct {
    int32_t status;         /* 0 ok, 1 infeasible (no plan meets QoS), <0 error */
    int32_t levels[OR_MAXW];/* winner level ranks */
    uint64_t index;         /* winner mixed-radix index (worker 0 most significant) */
    uint64_t key[4];        /* exact key of the winner (u256 limbs) */
    uint64_t min_key[4];    /* exact minimum key m */
    uint64_t scored;        /* units evaluated */
} or_result;

typedef struct {
    int W, mode, obj;
    int64_t lam, lamN;
    int E;                  /* matrix fraction bits */
    u128 D;                 /* Lambda N 2^E */
    int64_t Mi[OR_MAXW * OR_MAXW];   /* M * 2^E (exact integers) */
    int64_t* off;
    int64_t* Sp;            /* S' per level */
    const int64_t* B;
    const int32_t* L;
    const double* Q;
    u128 pi_idle, pi_dyn;   /* p * 2^k  (exact integers) */
    int64_t tol_num, tol_den;
    int64_t wt[OR_MAXW];    /* objective weights (integers, 1 = unweighted) */
} or_ctx;

static int64_t gcd64(int64_t a, int64_t b) { while (b) { int64_t t = a % b; a = b; b = t; } return a; }

/* smallest k >= 0 with x 2^k integral (x >= 0 finite), or -1 if k > limit */
static int frac_bits(double x, int limit) {
    for (int k = 0; k <= limit; k++) { double y = ldexp(x, k); if (y == floor(y)) return k; }
    return -1;
}

static int or_ctx_init(const or_problem* p, or_ctx* c) {
    memset(c, 0, sizeof(*c));
    if (p->W < 1 || p->W > OR_MAXW || p->N < 1) return -1;
    c->W = p->W; c->mode = p->mode; c->obj = p->objective; c->B = p->B; c->L = p->L; c->Q = p->Q;
    int64_t lam = 1;
    for (int w = 0; w < p->W; w++) { if (p->K[w] < 1) return -1; lam = lam / gcd64(lam, p->K[w]) * p->K[w]; }
    c->lam = lam; c->lamN = lam * (int64_t)p->N;
    c->E = 0;
    if (p->mode == OR_MATRIX) {
        for (int i = 0; i < p->W * p->W; i++) {
            if (i / p->W == i % p->W) continue;
            double m = (double)p->M[i];
            if (!(m >= 0.0) || m >= 1024.0) return -1;
            int k = frac_bits(m, 60);
            if (k < 0) return -1;
            if (k > c->E) c->E = k;
        }
        for (int i = 0; i < p->W * p->W; i++)
            c->Mi[i] = (i / p->W == i % p->W) ? 0 : (int64_t)ldexp((double)p->M[i], c->E);
    }
    c->D = (u128)c->lamN << c->E;
    int64_t tot = 0;
    c->off = (int64_t*)malloc(sizeof(int64_t) * (size_t)p->W);
    for (int w = 0; w < p->W; w++) { c->off[w] = tot; tot += p->L[w]; }
    c->Sp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(tot > 0 ? tot : 1));
    for (int w = 0; w < p->W; w++)
        for (int l = 0; l < p->L[w]; l++) c->Sp[c->off[w] + l] = p->S[c->off[w] + l] * (lam / p->K[w]);
    /* power model as exact integers p 2^k (c3-E) */
    double pi = p->p_idle, pm = p->p_max;
    if (!(pi >= 0.0) || !(pm >= pi)) return -1;
    int k1 = frac_bits(pi, 60), k2 = frac_bits(pm, 60);
    if (k1 < 0 || k2 < 0) return -1;
    int k = k1 > k2 ? k1 : k2;
    c->pi_idle = (u128)ldexp(pi, k);
    c->pi_dyn = (u128)ldexp(pm, k) - c->pi_idle;
    c->tol_num = p->tol_num; c->tol_den = p->tol_den;
    /* weights: SUM and MAX only (energy is a physical quantity: no per-worker weights) */
    for (int w = 0; w < p->W; w++) {
        c->wt[w] = p->wt ? p->wt[w] : 1;
        if (c->wt[w] < 1 || c->wt[w] > ((int64_t)1 << 30)) return -1;
        if (p->objective == OR_ENERGY && c->wt[w] != c->wt[0]) return -1;
    }
    return 0;
}
static void or_ctx_free(or_ctx* c) { free(c->off); free(c->Sp); }

/* O^_w (overlap scaled by Lambda 2^E) for worker w of tuple lv with total Tp */
static u128 or_overlap(const or_ctx* c, const int32_t* lv, int w, int64_t Tp) {
    int64_t spw = c->Sp[c->off[w] + lv[w]];
    switch (c->mode) {
    case OR_EXCLUDE_SELF: return (u128)(Tp - spw);                   /* sum_{w'!=w} CUAverage */
    case OR_PAPER: return (u128)Tp;                                  /* P:314 as printed */
    case OR_EXCESS: return Tp > c->lamN ? (u128)(Tp - c->lamN) : 0;  /* excess over capacity */
    default: {
        u128 o = 0;
        for (int v = 0; v < c->W; v++) if (v != w) o += (u128)c->Mi[w * c->W + v] * (u128)c->Sp[c->off[v] + lv[v]];
        return o;
    }
    }
}

/* exact key of a tuple; returns 0 if every QoS holds, 1 otherwise */
static int or_key(const or_ctx* c, const int32_t* lv, u256* key) {
    int64_t Tp = 0;
    for (int w = 0; w < c->W; w++) Tp += c->Sp[c->off[w] + lv[w]];
    u256 sum = u256_zero(), wmx = u256_zero();
    u128 mx = 0;
    for (int w = 0; w < c->W; w++) {
        u128 h = (u128)c->B[c->off[w] + lv[w]] * (c->D + or_overlap(c, lv, w, Tp));   /* h_w = B_w (D + O^_w) */
        if (!le_dyadic(h, c->Q[w], c->D)) return 1;                                   /* L_w <= Q_w */
        u256 wh = u256_mul128((u128)c->wt[w], h);                                     /* omega_w h_w */
        sum = u256_add(sum, wh);
        if (u256_cmp(wh, wmx) > 0) wmx = wh;
        if (h > mx) mx = h;
    }
    if (c->obj == OR_SUM) *key = sum;
    else if (c->obj == OR_MAX) *key = wmx;
    else {
        int64_t occ = Tp < c->lamN ? Tp : c->lamN;                                    /* min(Lambda N, T') */
        u128 pn = c->pi_idle * (u128)c->lamN + c->pi_dyn * (u128)occ;
        *key = u256_mul128(pn, mx);
    }
    return 0;
}

/* key <= m (1 + tol_num / tol_den)  <=>  key tol_den <= m (tol_den + tol_num) */
static int within_tol(const or_ctx* c, u256 key, u256 m) {
    return u256_cmp(u256_mul64(key, (uint64_t)c->tol_den), u256_mul64(m, (uint64_t)(c->tol_den + c->tol_num))) <= 0;
}

static void or_decode(uint64_t idx, int W, const int32_t* L, int32_t* lv) {
    for (int w = W - 1; w >= 0; w--) { lv[w] = (int32_t)(idx % (uint64_t)L[w]); idx /= (uint64_t)L[w]; }
}

/* Exhaustive enumeration over indices [lo, hi): pass 1 exact minimum, pass 2 lowest index
 * with key <= m (1 + tau).  (hi is clamped to prod L.) */
int or_enum_range(const or_problem* p, uint64_t lo, uint64_t hi, or_result* r) {
    memset(r, 0, sizeof(*r));
    or_ctx c;
    if (or_ctx_init(p, &c)) { r->status = -1; or_ctx_free(&c); return -1; }
    int W = p->W;
    uint64_t total = 1;
    for (int w = 0; w < W; w++) total *= (uint64_t)p->L[w];
    if (hi > total) hi = total;
    int32_t lv[OR_MAXW];
    u256 m, k;
    int have = 0;
    for (uint64_t idx = lo; idx < hi; idx++) {
        or_decode(idx, W, p->L, lv);
        if (or_key(&c, lv, &k)) continue;
        if (!have || u256_cmp(k, m) < 0) { m = k; have = 1; }
    }
    r->scored = hi > lo ? hi - lo : 0;
    if (!have) { r->status = 1; or_ctx_free(&c); return 0; }
    memcpy(r->min_key, m.w, sizeof m.w);
    for (uint64_t idx = lo; idx < hi; idx++) {
        or_decode(idx, W, p->L, lv);
        if (or_key(&c, lv, &k)) continue;
        if (within_tol(&c, k, m)) {
            r->index = idx;
            memcpy(r->key, k.w, sizeof k.w);
            for (int w = 0; w < W; w++) r->levels[w] = lv[w];
            break;
        }
    }
    or_ctx_free(&c);
    return 0;
}
int or_enum(const or_problem* p, or_result* r) { return or_enum_range(p, 0, UINT64_MAX, r); }

/* exact minimum over [lo, hi) only (sharded pass 1); status 1 if nothing feasible */
int or_enum_min_range(const or_problem* p, uint64_t lo, uint64_t hi, or_result* r) {
    memset(r, 0, sizeof(*r));
    or_ctx c;
    if (or_ctx_init(p, &c)) { r->status = -1; or_ctx_free(&c); return -1; }
    uint64_t total = 1;
    for (int w = 0; w < p->W; w++) total *= (uint64_t)p->L[w];
    if (hi > total) hi = total;
    int32_t lv[OR_MAXW];
    u256 m, k;
    int have = 0;
    for (uint64_t idx = lo; idx < hi; idx++) {
        or_decode(idx, p->W, p->L, lv);
        if (or_key(&c, lv, &k)) continue;
        if (!have || u256_cmp(k, m) < 0) { m = k; have = 1; }
    }
    r->status = have ? 0 : 1;
    if (have) memcpy(r->min_key, m.w, sizeof m.w);
    or_ctx_free(&c);
    return 0;
}

/* lowest index in [lo, hi) with key <= m (1 + tau) for a given exact m (sharded pass 2) */
int or_enum_first_within(const or_problem* p, uint64_t lo, uint64_t hi, const uint64_t* mkey, or_result* r) {
    memset(r, 0, sizeof(*r));
    or_ctx c;
    if (or_ctx_init(p, &c)) { r->status = -1; or_ctx_free(&c); return -1; }
    uint64_t total = 1;
    for (int w = 0; w < p->W; w++) total *= (uint64_t)p->L[w];
    if (hi > total) hi = total;
    u256 m; memcpy(m.w, mkey, sizeof m.w);
    int32_t lv[OR_MAXW];
    u256 k;
    r->status = 1;
    for (uint64_t idx = lo; idx < hi; idx++) {
        or_decode(idx, p->W, p->L, lv);
        if (or_key(&c, lv, &k)) continue;
        if (within_tol(&c, k, m)) {
            r->status = 0; r->index = idx; memcpy(r->key, k.w, sizeof k.w);
            for (int w = 0; w < p->W; w++) r->levels[w] = lv[w];
            break;
        }
    }
    or_ctx_free(&c);
    return 0;
}

/* exact key of one tuple (returns 1 if infeasible) */
int or_key_of(const or_problem* p, const int32_t* lv, uint64_t* key_out) {
    or_ctx c;
    if (or_ctx_init(p, &c)) { or_ctx_free(&c); return -1; }
    u256 k = u256_zero();
    int rc = or_key(&c, lv, &k);
    memcpy(key_out, k.w, sizeof k.w);
    or_ctx_free(&c);
    return rc;
}

/* ------------------------------------------------------------------------------------ */
/* T'-slicing (linear modes).  For fixed T' = sum_w S'_w every O^_w depends on (T', S'_w)   */
/* only, so h_w(l; T') is a per-worker table and                                          */
/*   SUM:  J(T') = min over tuples with sum S' = T' of sum_w h_w  — a (min,+) knapsack;    */
/*   MAX/ENERGY: (min,max) knapsack (ENERGY multiplies the slice's constant power).        */
/* Suffix DP:  D_{W-1}[P] = h_{W-1}(l) with S'_{W-1}(l) = P;                               */
/*             D_w[P] = min_l ( h_w(l) (+) D_{w+1}[P - S'_w(l)] );   J(T') = D_0[T'].       */
/* Infeasible (QoS) entries are +inf.  Then the lexicographic walk per qualifying slice.  */
/* ------------------------------------------------------------------------------------ */
#define OR_U128_INF (~(u128)0)

typedef struct {
    const or_problem* p;
    const or_ctx* c;
    int64_t gS;
    int64_t *smin, *smax, *slo, *shi;
    u128** D;
    int64_t *dlo, *dhi;
    u128* h;
} or_slice_ctx;

static u128 comb(int obj, u128 a, u128 b) {
    if (a == OR_U128_INF || b == OR_U128_INF) return OR_U128_INF;
    return obj == OR_SUM ? a + b : (a > b ? a : b);
}

static u128 or_slice_dp(or_slice_ctx* s, int64_t T) {
    const or_problem* p = s->p; const or_ctx* c = s->c;
    int W = p->W;
    int64_t Tp = T * s->gS;
    int32_t lv[OR_MAXW];
    memset(lv, 0, sizeof lv);
    for (int w = 0; w < W; w++) {
        for (int l = 0; l < p->L[w]; l++) {
            lv[w] = l;
            u128 h = (u128)c->B[c->off[w] + l] * (c->D + or_overlap(c, lv, w, Tp));
            /* the weighted term omega_w h_w (or_slice checked that it fits with room for W of them) */
            s->h[c->off[w] + l] = le_dyadic(h, c->Q[w], c->D) ? h * (u128)c->wt[w] : OR_U128_INF;
        }
        lv[w] = 0;
    }
    for (int w = W - 1; w >= 1; w--) {
        int64_t pre_lo = 0, pre_hi = 0;
        for (int v = 0; v < w; v++) { pre_lo += s->smin[v]; pre_hi += s->smax[v]; }
        int64_t lo = T - pre_hi, hi = T - pre_lo;
        if (lo < s->slo[w]) lo = s->slo[w];
        if (hi > s->shi[w]) hi = s->shi[w];
        s->dlo[w] = lo; s->dhi[w] = hi;
        for (int64_t P = lo; P <= hi; P++) {
            u128 best = OR_U128_INF;
            for (int l = 0; l < p->L[w]; l++) {
                int64_t i = c->off[w] + l;
                int64_t rest = P - c->Sp[i] / s->gS;
                u128 v;
                if (w == W - 1) {
                    if (rest != 0) continue;
                    v = s->h[i];
                } else {
                    if (rest < s->dlo[w + 1] || rest > s->dhi[w + 1]) continue;
                    v = comb(p->objective, s->h[i], s->D[w + 1][rest - s->dlo[w + 1]]);
                }
                if (v < best) best = v;
            }
            s->D[w][P - lo] = best;
        }
    }
    u128 J = OR_U128_INF;
    for (int l = 0; l < p->L[0]; l++) {
        int64_t i = c->off[0] + l;
        int64_t rest = T - c->Sp[i] / s->gS;
        u128 v;
        if (W == 1) {
            if (rest != 0) continue;
            v = s->h[i];
        } else {
            if (rest < s->dlo[1] || rest > s->dhi[1]) continue;
            v = comb(p->objective, s->h[i], s->D[1][rest - s->dlo[1]]);
        }
        if (v < J) J = v;
    }
    return J;
}

static u256 or_slice_key(const or_ctx* c, int obj, int64_t Tp, u128 v) {
    if (obj != OR_ENERGY) return u256_from128(v);
    v /= (u128)c->wt[0];   /* ENERGY: uniform weights (or_ctx_init), the DP carried wt[0] max h */
    int64_t occ = Tp < c->lamN ? Tp : c->lamN;
    u128 pn = c->pi_idle * (u128)c->lamN + c->pi_dyn * (u128)occ;
    return u256_mul128(pn, v);
}

int or_slice(const or_problem* p, or_result* r) {
    memset(r, 0, sizeof(*r));
    if (p->mode == OR_MATRIX) { r->status = -1; return -1; }
    or_ctx c;
    if (or_ctx_init(p, &c)) { r->status = -1; or_ctx_free(&c); return -1; }
    int W = p->W;
    or_slice_ctx s;
    s.p = p; s.c = &c;
    int64_t tot = 0;
    for (int w = 0; w < W; w++) tot += p->L[w];
    int64_t gS = 0;
    for (int64_t i = 0; i < tot; i++) gS = gcd64(gS, c.Sp[i]);
    if (gS == 0) gS = 1;
    s.gS = gS;
    s.smin = (int64_t*)malloc(sizeof(int64_t) * W); s.smax = (int64_t*)malloc(sizeof(int64_t) * W);
    s.slo = (int64_t*)malloc(sizeof(int64_t) * (W + 1)); s.shi = (int64_t*)malloc(sizeof(int64_t) * (W + 1));
    for (int w = 0; w < W; w++) {
        s.smin[w] = INT64_MAX; s.smax[w] = 0;
        for (int l = 0; l < p->L[w]; l++) {
            int64_t v = c.Sp[c.off[w] + l] / gS;
            if (v < s.smin[w]) s.smin[w] = v;
            if (v > s.smax[w]) s.smax[w] = v;
        }
    }
    s.slo[W] = 0; s.shi[W] = 0;
    for (int w = W - 1; w >= 0; w--) { s.slo[w] = s.slo[w + 1] + s.smin[w]; s.shi[w] = s.shi[w + 1] + s.smax[w]; }
    s.D = (u128**)calloc((size_t)W, sizeof(u128*));
    s.dlo = (int64_t*)calloc((size_t)W + 1, sizeof(int64_t)); s.dhi = (int64_t*)calloc((size_t)W + 1, sizeof(int64_t));
    for (int w = 1; w < W; w++) s.D[w] = (u128*)malloc(sizeof(u128) * (size_t)(s.shi[w] - s.slo[w] + 1));
    s.h = (u128*)malloc(sizeof(u128) * (size_t)tot);
    {   /* every weighted term must fit u128 with room for the sum over W workers */
        u128 lim = (~(u128)0) / (u128)(W + 1);
        for (int w = 0; w < W; w++)
            for (int l = 0; l < p->L[w]; l++) {
                u128 hmax = (u128)p->B[c.off[w] + l] * (c.D + (u128)(s.shi[0] * gS) + (u128)c.lamN);
                if (hmax > lim / (u128)c.wt[w]) {
                    r->status = -1;
                    free(s.h);
                    for (int v = 1; v < W; v++) free(s.D[v]);
                    free(s.D); free(s.dlo); free(s.dhi); free(s.smin); free(s.smax); free(s.slo); free(s.shi);
                    or_ctx_free(&c);
                    return -1;
                }
            }
    }

    int64_t Tlo = s.slo[0], Thi = s.shi[0];
    u256* J = (u256*)malloc(sizeof(u256) * (size_t)(Thi - Tlo + 1));
    char* okJ = (char*)calloc((size_t)(Thi - Tlo + 1), 1);
    u256 m = u256_zero();
    int have = 0;
    for (int64_t T = Tlo; T <= Thi; T++) {
        u128 v = or_slice_dp(&s, T);
        if (v == OR_U128_INF) continue;
        J[T - Tlo] = or_slice_key(&c, p->objective, T * gS, v);
        okJ[T - Tlo] = 1;
        if (!have || u256_cmp(J[T - Tlo], m) < 0) { m = J[T - Tlo]; have = 1; }
    }
    if (!have) { r->status = 1; goto done; }
    memcpy(r->min_key, m.w, sizeof m.w);
    {
        int haveb = 0;
        int32_t best[OR_MAXW], cur[OR_MAXW];
        u128 hp[OR_MAXW];
        for (int64_t T = Tlo; T <= Thi; T++) {
            if (!okJ[T - Tlo] || !within_tol(&c, J[T - Tlo], m)) continue;
            (void)or_slice_dp(&s, T);
            int64_t rem = T;
            int ok = 1;
            for (int w = 0; w < W && ok; w++) {
                int found = 0;
                for (int l = 0; l < p->L[w]; l++) {
                    int64_t i = c.off[w] + l;
                    int64_t rest = rem - c.Sp[i] / gS;
                    u128 v;
                    if (w == W - 1) {
                        if (rest != 0) continue;
                        v = s.h[i];
                    } else {
                        if (rest < s.dlo[w + 1] || rest > s.dhi[w + 1]) continue;
                        v = comb(p->objective, s.h[i], s.D[w + 1][rest - s.dlo[w + 1]]);
                    }
                    for (int v2 = w - 1; v2 >= 0; v2--) v = comb(p->objective, hp[v2], v);
                    if (v == OR_U128_INF) continue;
                    if (within_tol(&c, or_slice_key(&c, p->objective, T * gS, v), m)) {
                        cur[w] = l; hp[w] = s.h[i]; rem = rest; found = 1; break;
                    }
                }
                if (!found) ok = 0;
            }
            if (!ok) { r->status = -4; goto done; }
            int less = !haveb;
            for (int w = 0; w < W && !less; w++) {
                if (cur[w] < best[w]) { less = 1; break; }
                if (cur[w] > best[w]) break;
            }
            if (less) { memcpy(best, cur, sizeof(int32_t) * W); haveb = 1; }
        }
        u128 idx = 0;
        int fits = 1;
        for (int w = 0; w < W; w++) {
            idx = idx * (u128)p->L[w] + (u128)best[w];
            if (idx >> 64) fits = 0;
            r->levels[w] = best[w];
        }
        r->index = fits ? (uint64_t)idx : UINT64_MAX;   /* index needs more than 64 bits */
        u256 k;
        or_key(&c, best, &k);
        memcpy(r->key, k.w, sizeof k.w);
        r->status = 0;
    }
done:
    free(J); free(okJ); free(s.h);
    for (int w = 1; w < W; w++) free(s.D[w]);
    free(s.D); free(s.dlo); free(s.dhi); free(s.smin); free(s.smax); free(s.slo); free(s.shi);
    or_ctx_free(&c);
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* FP64 values of a plan (values parity):                                  */
/*   CUAverage_w = S_w / K_w; CUOverlap_w per mode (c3-O/c3-M);             */
/*   alpha_w = CUOverlap_w / N; L_w = B_w (1 + alpha_w) = sum_k e_k;        */
/*   power = p_idle + (p_max - p_idle) min(1, sum_w CUAverage_w / N) (c3-E);    */
/*   makespan = max_w L_w; energy = power x makespan; throughput = sum_w 1e9 / L_w;        */
/*   objective SUM = sum_w omega_w L_w, MAX = max_w omega_w L_w (omega = wval, default 1). */
/* out: [0..W-1] L_w (ns); [W] objective; [W+1] makespan (ns); [W+2] power (W);             */
/*      [W+3] energy (J); [W+4] throughput (1/s); [W+5+w] alpha_w.                          */
/* ------------------------------------------------------------------------------------ */
int or_eval_f64(const or_problem* p, const int32_t* lv, double* out) {
    int W = p->W;
    if (W < 1 || W > OR_MAXW) return -1;
    int64_t off = 0;
    double avg[OR_MAXW], Bw[OR_MAXW];
    double sum_avg = 0.0;
    for (int w = 0; w < W; w++) {
        int64_t i = off + lv[w];
        avg[w] = (double)p->S[i] / (double)p->K[w];
        Bw[w] = (double)p->B[i];
        sum_avg += avg[w];
        off += p->L[w];
    }
    double mk = 0.0, wmk = 0.0, obj = 0.0, thr = 0.0;
    for (int w = 0; w < W; w++) {
        double ov;
        if (p->mode == OR_EXCLUDE_SELF) ov = sum_avg - avg[w];
        else if (p->mode == OR_PAPER) ov = sum_avg;
        else if (p->mode == OR_EXCESS) ov = sum_avg - (double)p->N > 0 ? sum_avg - (double)p->N : 0.0;
        else {
            ov = 0.0;
            for (int v = 0; v < W; v++) if (v != w) ov += (double)p->M[w * W + v] * avg[v];
        }
        double alpha = ov / (double)p->N;
        double Lw = Bw[w] * (1.0 + alpha);
        out[w] = Lw;
        out[W + 5 + w] = alpha;
        if (Lw > mk) mk = Lw;
        double om = p->wval ? p->wval[w] : 1.0;     /* objective weight (SUM / MAX) */
        obj += om * Lw;
        if (om * Lw > wmk) wmk = om * Lw;
        thr += 1e9 / Lw;
    }
    double frac = sum_avg / (double)p->N;
    if (frac > 1.0) frac = 1.0;
    double pw = (double)p->p_idle + ((double)p->p_max - (double)p->p_idle) * frac;
    if (p->objective == OR_MAX) obj = wmk;
    else if (p->objective == OR_ENERGY) obj = pw * mk;
    out[W] = obj;
    out[W + 1] = mk;
    out[W + 2] = pw;
    out[W + 3] = pw * mk * 1e-9;
    out[W + 4] = thr;
    return 0;
}
