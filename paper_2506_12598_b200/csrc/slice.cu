// slice.cu — SLICE engine kernels (K3 FP32 slice DP, exact slice DP, K4 lexicographic walk).
// See slice.h and DESIGN.md §4.  Derivation (App. A.2 of SURVEY.md): in
// the linear modes (EXCLUDE_SELF, PAPER_AS_WRITTEN, EXCESS) O_w depends on the tuple only
// through (T', S'_w), so with T' fixed the SUM objective separates into per-worker terms.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "slice.h"

namespace eclip {

static constexpr uint64_t UINF = ~0ull;
static constexpr int SL_THREADS = 256;
static constexpr int SLX = 1024;   // exact DP / walk: one CTA per band slice, a wide block (few band slices, each latency-bound)

SliceState::~SliceState() { release(); }
void SliceState::release() {
    for (void* p : allocs) cudaFreeAsync(p, st);
    allocs.clear();
}

uint64_t slice_units(const SliceState& s) {
    unsigned long long u = 0;
    if (s.d_units) cudaMemcpy(&u, s.d_units, sizeof u, cudaMemcpyDeviceToHost);
    return u;
}

// per-slice D range of worker w (w >= 1): P values reachable from T with workers w..W-1
__device__ __forceinline__ void drange(const SliceDev& S, int64_t T, int w, int64_t* lo, int64_t* hi) {
    int64_t a = T - S.phi[w], b = T - S.plo[w];
    *lo = a > S.slo[w] ? a : S.slo[w];
    *hi = b < S.shi[w] ? b : S.shi[w];
}

__device__ __forceinline__ int64_t overlap_exact(int mode, int64_t Tp, int64_t Sp, int64_t lamN) {
    if (mode == M_EXCL) return Tp - Sp;
    if (mode == M_PAPER) return Tp;
    return Tp > lamN ? Tp - lamN : 0;
}

// ------------------------------------------------------------------------------------------
// K3: FP32 filter DP, one CTA per slice (interleaved over shards).
// D buffers carry PAD = max level span of +inf on both sides, so the inner (min,+) loop has no
// bounds checks.  Each thread owns RB consecutive outputs P; the k loop is unrolled by KU: per
// block of KU levels it loads a window of RB + KU - 1 D values and the KU g values into registers
// and does RB x KU adds with the mins folded in pairs (FMNMX3).  RB is odd: a warp's windows start
// RB floats apart, so its window loads fall on 32 distinct banks (an even RB = 8 put 8 lanes on a bank).
// ------------------------------------------------------------------------------------------
constexpr int RB = 9;
constexpr int KU = 8;
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

template <int OBJ>
__device__ __forceinline__ float comb_f(float g, float d) { return OBJ == O_SUM ? g + d : fmaxf(g, d); }

template <int OBJ>
__global__ void __launch_bounds__(SL_THREADS) k_slice_f32(SliceDev S, const Prob* probs, const Lev* __restrict__ levs,
                                                          const int16_t* __restrict__ dense, float* J32,
                                                          unsigned long long* units) {
    unsigned long long cnt = 0;
    extern __shared__ float sm[];
    const Prob& P = probs[0];
    int64_t T = S.Tlo + S.shard + (int64_t)S.n_shards * blockIdx.x;
    if (T > S.Thi) return;
    const int W = S.W;
    const int PAD = S.pad;
    const int BUF = S.maxrange + 2 * PAD + RB;          // entries [-PAD, maxrange + PAD + RB)
    const int BUFS = BUF;
    int gspan = 1;
    for (int w = 0; w < W; w++) gspan = max(gspan, S.smax[w] - S.smin[w] + 1);
    // g_w(level; T') of one worker at a time (the stage that uses it): a small buffer keeps the block's shared
    // memory low enough for more CTAs per SM, whose warps fill the issue slots while a stage's barrier waits
    float* g = sm;                                      // [gspan]
    float* Da = g + gspan;
    float* Db = Da + BUFS;
    const int64_t Tp = T * S.gS;
    const float Tpf = (float)Tp;
    auto fill_g = [&](int w) {
        const int span = S.smax[w] - S.smin[w] + 1;
        for (int i = threadIdx.x; i < span; i += blockDim.x) {
            const int l = dense[S.doff[w] + i];
            float v = INFINITY;
            if (l >= 0) {
                const Lev& r = levs[w * S.Lmax + l];
                if (Tp <= (int64_t)r.Tmax) {
                    float O = (float)overlap_exact(S.mode, Tp, r.S, P.lamN);
                    v = fmaf(O, r.Bk, __ll2float_rn(r.B)) * P.wf[w];   // omega_w L_w (weights: DESIGN.md R20)
                }
            }
            g[i] = v;
        }
    };
    for (int i = threadIdx.x; i < 2 * BUFS; i += blockDim.x) Da[i] = INFINITY;
    fill_g(W - 1);
    __syncthreads();
    float* Dn = Da;   // D_{w+1}
    float* Dc = Db;   // D_w
    auto at = [&](float* D, int i) -> float& { return D[i + PAD]; };   // index i >= -PAD
    int64_t nlo = 0, nhi = -1;
    if (W >= 2) {
        drange(S, T, W - 1, &nlo, &nhi);
        const float* gw = g;
        for (int64_t p = nlo + threadIdx.x; p <= nhi; p += blockDim.x) at(Dn, (int)(p - nlo)) = gw[p - S.smin[W - 1]];
        __syncthreads();
        if (W >= 3) {   // g of the first stage
            fill_g(W - 2);
            __syncthreads();
        }
        for (int w = W - 2; w >= 1; w--) {
            int64_t lo, hi;
            drange(S, T, w, &lo, &hi);
            const float* gw2 = g;   // g_w (filled before the barrier that ended the previous stage)
            const int nk = S.smax[w] - S.smin[w] + 1;
            const int np = (int)(hi - lo + 1);
            const int nprev = (int)(nhi - nlo + 1);
            for (int c = threadIdx.x * RB; c < np; c += blockDim.x * RB) {
                // outputs p = lo + c + j (j < RB) read Dn[b + j - k], b = lo + c - smin_w - nlo
                const int b = (int)(lo + c - S.smin[w] - nlo);
                const int ks = max(0, b - (nprev - 1)), ke = min(nk, b + RB);   // k outside is +inf
                float best[RB];
#pragma unroll
                for (int j = 0; j < RB; j++) best[j] = INFINITY;
                int k = ks;
                for (; k + KU <= ke; k += KU) {
                    float win[RB + KU - 1], gg[KU];   // win[i] = Dn[b - k - KU + 1 + i]
#pragma unroll
                    for (int i = 0; i < RB + KU - 1; i++) win[i] = at(Dn, b - k - KU + 1 + i);
#pragma unroll
                    for (int u = 0; u < KU; u++) gg[u] = gw2[k + u];
                    if (OBJ == O_SUM) {
                        // packed adds: output j at level k+u reads win[j + KU-1-u]; the window is consumed as the
                        // aligned pairs (win[2q], win[2q+1]) for both parities of u (j even / odd), so each level
                        // is 4 add.f32x2 (g broadcast) + 1 scalar add for the 9 outputs
#pragma unroll
                        for (int u = 0; u < KU; u += 2) {
                            float s0[RB], s1[RB];
                            auto sums = [&](int uu, float* sv) {
                                const int off = KU - 1 - uu;   // win index of output j = j + off
                                const u64 g2 = f2pack(gg[uu], gg[uu]);
#pragma unroll
                                for (int j = (off & 1); j + 1 < RB; j += 2) {
                                    float lo, hi;
                                    f2unpack(add2(f2pack(win[j + off], win[j + off + 1]), g2), lo, hi);
                                    sv[j] = lo; sv[j + 1] = hi;
                                }
                                if (off & 1) sv[0] = gg[uu] + win[off];                  // j = 0 alone
                                else sv[RB - 1] = gg[uu] + win[RB - 1 + off];            // j = RB-1 alone
                            };
                            sums(u, s0);
                            sums(u + 1, s1);
#pragma unroll
                            for (int j = 0; j < RB; j++) best[j] = fminf(best[j], fminf(s0[j], s1[j]));
                        }
                    } else {
#pragma unroll
                        for (int u = 0; u < KU; u += 2)
#pragma unroll
                            for (int j = 0; j < RB; j++)   // Dn[b + j - (k + u)] = win[j + KU - 1 - u]
                                best[j] = fminf(best[j], fminf(comb_f<OBJ>(gg[u], win[j + KU - 1 - u]),
                                                               comb_f<OBJ>(gg[u + 1], win[j + KU - 2 - u])));
                    }
                }
                for (; k < ke; k++) {
                    const float gk = gw2[k];
#pragma unroll
                    for (int j = 0; j < RB; j++) best[j] = fminf(best[j], comb_f<OBJ>(gk, at(Dn, b + j - k)));
                }
                if (ks < ke) cnt += (unsigned long long)(ke - ks) * RB;
#pragma unroll
                for (int j = 0; j < RB; j++)
                    if (c + j < np) at(Dc, c + j) = best[j];
            }
            __syncthreads();
            // clear the stale part of the buffer that becomes D_{w+1} next stage (outside [0, np): left over from
            // two stages ago); the next stage writes every entry of [0, np') of the other buffer, so that one needs
            // no clearing.  And the next stage's g_{w-1}, under the same barrier.
            for (int i = threadIdx.x; i < BUF; i += blockDim.x)
                if (i - PAD < 0 || i - PAD >= np) at(Dc, i - PAD) = INFINITY;
            fill_g(w - 1);
            float* t = Dn; Dn = Dc; Dc = t;
            __syncthreads();
            nlo = lo; nhi = hi;
        }
    }
    // J = min_k g_0[k] (+) D_1[T - smin_0 - k]
    if (W == 2) {   // (W >= 3: the last stage filled g_0; W = 1: g holds worker 0 already)
        fill_g(0);
        __syncthreads();
    }
    float J = INFINITY;
    const int nk0 = S.smax[0] - S.smin[0] + 1;
    for (int k = threadIdx.x; k < nk0; k += blockDim.x) {
        int64_t rest = T - S.smin[0] - k;
        float v;
        if (W == 1) {
            if (rest != 0) continue;
            v = g[k];
        } else {
            if (rest < nlo || rest > nhi) continue;
            float d = at(Dn, (int)(rest - nlo));
            v = (OBJ == O_SUM) ? g[k] + d : fmaxf(g[k], d);
        }
        J = fminf(J, v);
    }
    if (threadIdx.x == 0) cnt += (unsigned long long)nk0;
    if (cnt) atomicAdd(units, cnt);
    __shared__ float red[SL_THREADS];
    red[threadIdx.x] = J;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = fminf(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        float j = red[0];
        if (OBJ == O_ENERGY && j < INFINITY) j = fmaf(P.p_dyn, fminf(1.0f, Tpf * P.inv), P.p_idle) * j;
        J32[T - S.Tlo] = j;
    }
}

// min over this shard's slices -> m32[0]; and the band list
__global__ void k_slice_min(SliceDev S, const float* J32, float* m32) {
    __shared__ float red[1024];
    float m = INFINITY;
    for (int64_t i = S.shard + (int64_t)S.n_shards * threadIdx.x; i < S.n_slices; i += (int64_t)S.n_shards * blockDim.x)
        m = fminf(m, J32[i]);
    red[threadIdx.x] = m;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = fminf(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) m32[0] = red[0];
}

__global__ void k_slice_band(SliceDev S, const float* J32, const float* m32, int32_t* band, int32_t* nband) {
    __shared__ int cnt;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    float m = m32[0];
    float bound = INFINITY;
    if (!isinf(m)) {
        double tau = (double)S.tol_num / (double)S.tol_den;
        bound = __double2float_ru((double)m * (1.0 + tau) * (1.0 + S.delta) / (1.0 - S.delta) * (1.0 + 1e-12));
    }
    for (int64_t i = S.shard + (int64_t)S.n_shards * threadIdx.x; i < S.n_slices; i += (int64_t)S.n_shards * blockDim.x) {
        if (!isinf(m) && J32[i] <= bound) {
            int pos = atomicAdd(&cnt, 1);
            band[pos] = (int32_t)i;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) *nband = cnt;
}

// ------------------------------------------------------------------------------------------
// exact DP of one slice into scratch (u64 per entry, UINF = infeasible); returns J via smem
// layout of scratch: [g: gtot][D_1 .. D_{W-1}: maxrange each]
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t comb_u(int obj, uint64_t a, uint64_t b) {
    if (a == UINF || b == UINF) return UINF;
    return obj == O_SUM ? a + b : (a > b ? a : b);
}

__device__ void slice_exact_dp(const SliceDev& S, const Prob& P, const Lev* levs, const int16_t* dense, int64_t T,
                               uint64_t* scr, int64_t* dlo, int64_t* dhi) {
    const int W = S.W;
    uint64_t* h = scr;
    const int64_t Tp = T * S.gS;
    for (int i = threadIdx.x; i < S.gtot; i += blockDim.x) {
        int w = 0;
        while (w + 1 < W && S.doff[w + 1] <= i) w++;
        int l = dense[i];
        uint64_t v = UINF;
        if (l >= 0) {
            const Lev& r = levs[w * S.Lmax + l];
            if (Tp <= (int64_t)r.Tmax)   // omega_w h_w (slice_setup checked the u64 range)
                v = (uint64_t)r.B * (uint64_t)(P.lamN + overlap_exact(S.mode, Tp, r.S, P.lamN)) * P.wt[w];
        }
        h[i] = v;
    }
    if (threadIdx.x == 0)
        for (int w = 1; w < W; w++) drange(S, T, w, &dlo[w], &dhi[w]);
    __syncthreads();
    if (W >= 2) {
        uint64_t* D = scr + S.gtot + (size_t)(W - 1 - 1) * S.maxrange;
        const uint64_t* hw = h + S.doff[W - 1];
        for (int64_t p = dlo[W - 1] + threadIdx.x; p <= dhi[W - 1]; p += blockDim.x) D[p - dlo[W - 1]] = hw[p - S.smin[W - 1]];
        __syncthreads();
        for (int w = W - 2; w >= 1; w--) {
            uint64_t* Dc = scr + S.gtot + (size_t)(w - 1) * S.maxrange;
            const uint64_t* Dn = scr + S.gtot + (size_t)w * S.maxrange;
            const uint64_t* hw2 = h + S.doff[w];
            const int nk = S.smax[w] - S.smin[w] + 1;
            for (int64_t p = dlo[w] + threadIdx.x; p <= dhi[w]; p += blockDim.x) {
                uint64_t best = UINF;
                // rest = p - smin_w - k must lie in [dlo[w+1], dhi[w+1]]
                const int64_t k0 = p - S.smin[w] - dhi[w + 1], k1 = p - S.smin[w] - dlo[w + 1];
                const int ka = (int)(k0 > 0 ? k0 : 0), kb = (int)(k1 < nk - 1 ? k1 : nk - 1);
                const uint64_t* dn = Dn + (p - S.smin[w] - dlo[w + 1]);
                for (int k = ka; k <= kb; k++) {
                    const uint64_t v = comb_u(S.obj, hw2[k], dn[-k]);
                    if (v < best) best = v;
                }
                Dc[p - dlo[w]] = best;
            }
            __syncthreads();
        }
    }
}

__device__ U256 slice_key(const SliceDev& S, const Prob& P, int64_t Tp, uint64_t v) {
    if (S.obj != O_ENERGY) return u256_of((u128)v);
    int64_t occ = Tp < P.lamN ? Tp : P.lamN;
    u128 pn = P.pi_idle * (u128)P.lamN + P.pi_dyn * (u128)occ;
    return u256_mul128(pn, (u128)v);
}

// pass 2a: exact J for every band slice
__global__ void __launch_bounds__(SLX) k_slice_exact(SliceDev S, const Prob* probs, const Lev* levs,
                                                            const int16_t* dense, const int32_t* band,
                                                            const int32_t* nband, uint64_t* scratch, U256* Jex) {
    const Prob& P = probs[0];
    __shared__ int64_t dlo[MAXW + 1], dhi[MAXW + 1];
    __shared__ uint64_t red[SLX];
    uint64_t* scr = scratch + (size_t)blockIdx.x * (S.gtot + (size_t)(S.W) * S.maxrange);
    for (int bi = blockIdx.x; bi < *nband; bi += gridDim.x) {
        int64_t T = S.Tlo + band[bi];
        slice_exact_dp(S, P, levs, dense, T, scr, dlo, dhi);
        const int W = S.W;
        const uint64_t* h = scr;
        uint64_t J = UINF;
        const int nk0 = S.smax[0] - S.smin[0] + 1;
        for (int k = threadIdx.x; k < nk0; k += blockDim.x) {
            int64_t rest = T - S.smin[0] - k;
            uint64_t v;
            if (W == 1) {
                if (rest != 0) continue;
                v = h[k];
            } else {
                if (rest < dlo[1] || rest > dhi[1]) continue;
                v = comb_u(S.obj, h[k], scr[S.gtot + (rest - dlo[1])]);
            }
            if (v < J) J = v;
        }
        red[threadIdx.x] = J;
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s && red[threadIdx.x + s] < red[threadIdx.x]) red[threadIdx.x] = red[threadIdx.x + s];
            __syncthreads();
        }
        if (threadIdx.x == 0) Jex[band[bi]] = red[0] == UINF ? u256_max() : slice_key(S, P, T * S.gS, red[0]);
        __syncthreads();
    }
}

// lexicographically smallest qualifying tuple over the band slices
__global__ void k_slice_first(const int32_t* nband, const U256* wtup, U256* first) {
    if (threadIdx.x != 0) return;
    U256 m = u256_max();
    for (int i = 0; i < *nband; i++)
        if (u256_cmp(wtup[i], m) < 0) m = wtup[i];
    first[0] = m;
}

__global__ void k_slice_hstar(const int32_t* band, const int32_t* nband, const U256* Jex, U256* hstar) {
    if (threadIdx.x != 0) return;
    U256 m = u256_max();
    for (int i = 0; i < *nband; i++)
        if (u256_cmp(Jex[band[i]], m) < 0) m = Jex[band[i]];
    hstar[0] = m;
}

// pass 2b: exact DP + lexicographic walk in every slice whose exact J is within tolerance.
// The walk is block-parallel: for worker w = 0..W-1 every level l (rank order) is tested at
// once -- "does some completion of (prefix, l) inside this slice reach key <= H*(1+tau)?",
// exact by the DP tables -- and the smallest qualifying rank is kept.
__global__ void __launch_bounds__(SLX) k_slice_walk(SliceDev S, const Prob* probs, const Lev* levs,
                                                           const int16_t* dense, const int32_t* band,
                                                           const int32_t* nband, uint64_t* scratch, const U256* Jex,
                                                           const U256* hstar, U256* wtup) {
    const Prob& P = probs[0];
    __shared__ int64_t dlo[MAXW + 1], dhi[MAXW + 1];
    __shared__ int s_pick;
    __shared__ int64_t s_rem;
    __shared__ uint64_t s_hp[MAXW];
    __shared__ int s_lv[MAXW];
    uint64_t* scr = scratch + (size_t)blockIdx.x * (S.gtot + (size_t)(S.W) * S.maxrange);
    const U256 hs = hstar[0];
    for (int bi = blockIdx.x; bi < *nband; bi += gridDim.x) {
        if (threadIdx.x == 0) wtup[bi] = u256_max();
        if (u256_is_max(hs) || u256_is_max(Jex[band[bi]]) || !within_tol(Jex[band[bi]], hs, S.tol_num, S.tol_den))
            continue;
        const int64_t T = S.Tlo + band[bi];
        if (*nband <= (int)gridDim.x) {
            // pass 2a left this slice's exact tables in this CTA's scratch slot (same grid mapping)
            if (threadIdx.x == 0)
                for (int w = 1; w < S.W; w++) drange(S, T, w, &dlo[w], &dhi[w]);
            __syncthreads();
        } else {
            slice_exact_dp(S, P, levs, dense, T, scr, dlo, dhi);
        }
        const int W = S.W;
        const int64_t Tp = T * S.gS;
        if (threadIdx.x == 0) s_rem = T;
        __syncthreads();
        bool ok = true;
        for (int w = 0; w < W && ok; w++) {
            if (threadIdx.x == 0) s_pick = INT_MAX;
            __syncthreads();
            const int64_t rem = s_rem;
            for (int l = threadIdx.x; l < P.L[w]; l += blockDim.x) {
                const Lev& r = levs[w * S.Lmax + l];
                const int64_t s = r.S / S.gS;
                const int64_t rest = rem - s;
                const uint64_t hw = scr[S.doff[w] + (s - S.smin[w])];
                if (hw == UINF) continue;
                uint64_t v;
                if (w == W - 1) {
                    if (rest != 0) continue;
                    v = hw;
                } else {
                    if (rest < dlo[w + 1] || rest > dhi[w + 1]) continue;
                    v = comb_u(S.obj, hw, scr[S.gtot + (size_t)w * S.maxrange + (rest - dlo[w + 1])]);
                }
                for (int u = 0; u < w; u++) v = comb_u(S.obj, s_hp[u], v);
                if (v == UINF) continue;
                if (within_tol(slice_key(S, P, Tp, v), hs, S.tol_num, S.tol_den)) atomicMin(&s_pick, l);
            }
            __syncthreads();
            const int pick = s_pick;
            ok = pick != INT_MAX;
            if (ok && threadIdx.x == 0) {
                const Lev& r = levs[w * S.Lmax + pick];
                const int64_t s = r.S / S.gS;
                s_lv[w] = pick;
                s_hp[w] = scr[S.doff[w] + (s - S.smin[w])];
                s_rem = rem - s;
            }
            __syncthreads();
        }
        if (ok && threadIdx.x == 0) wtup[bi] = pack_tuple(s_lv, W);
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------
template <class T>
static cudaError_t salloc(SliceState& s, T** p, size_t n) {
    void* q = nullptr;
    cudaError_t e = cudaMallocAsync(&q, std::max<size_t>(n, 1) * sizeof(T), s.st);
    if (e == cudaSuccess) s.allocs.push_back(q);
    *p = (T*)q;
    return e;
}

#define CK(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) return _e; } while (0)

cudaError_t slice_setup(SliceState& s, const Setup& su, const Tables& tb, Work& wk, const int32_t* tabL,
                        const int32_t* table_of, cudaStream_t st) {
    (void)tb; (void)tabL; (void)table_of;
    s.st = st;
    const int W = su.W;
    Prob P;
    std::vector<Lev> lev((size_t)W * su.Lmax);
    CK(cudaMemcpyAsync(&P, wk.probs, sizeof(Prob), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(lev.data(), wk.levs, lev.size() * sizeof(Lev), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    host_mark("slice_setup: records on host");
    SliceDev& S = s.h;
    S.W = W; S.Lmax = su.Lmax; S.mode = su.mode; S.obj = su.obj;
    S.shard = su.shard; S.n_shards = su.n_shards;
    S.tol_num = su.tol_num; S.tol_den = su.tol_den;
    S.delta = (double)(4 * W + 16) * std::ldexp(1.0, -24);
    if (P.status != 0) {  // nothing to slice; the kernels see n_slices = 0
        S.n_slices = 0; S.gtot = 1; S.maxrange = 1; S.gS = 1; S.Tlo = 0; S.Thi = -1;
        CK(salloc(s, &s.dense, 1)); CK(salloc(s, &s.J32, 1)); CK(salloc(s, &s.Jex, 1));
        CK(salloc(s, &s.band, 1)); CK(salloc(s, &s.nband, 1)); CK(salloc(s, &s.scratch, 1));
        CK(salloc(s, &s.wtup, 1));
        CK(salloc(s, &s.d_units, 1));
        CK(cudaMemsetAsync(s.nband, 0, 4, st));
        s.slots = 1;
        return cudaSuccess;
    }
    int64_t g = 0;
    for (int w = 0; w < W; w++)
        for (int l = 0; l < P.L[w]; l++) {
            const int64_t v = lev[(size_t)w * su.Lmax + l].S;
            if (g == 0 || v % g != 0) g = std::gcd(g, v);   // (one division for the common multiples)
        }
    if (g == 0) g = 1;
    S.gS = g;
    host_mark("slice_setup: gcd");
    std::vector<int16_t> dense;
    std::vector<int32_t> q((size_t)W * su.Lmax);   // S' / g (exact quotients, one division each)
    for (int w = 0; w < W; w++) {
        int mn = INT32_MAX, mx = 0;
        for (int l = 0; l < P.L[w]; l++) {
            const int v = (int)(lev[(size_t)w * su.Lmax + l].S / g);
            q[(size_t)w * su.Lmax + l] = v;
            mn = std::min(mn, v); mx = std::max(mx, v);
        }
        S.smin[w] = mn; S.smax[w] = mx;
        S.doff[w] = (int32_t)dense.size();
        size_t base = dense.size();
        dense.resize(base + (mx - mn + 1), -1);
        for (int l = 0; l < P.L[w]; l++) dense[base + q[(size_t)w * su.Lmax + l] - mn] = (int16_t)l;
    }
    if (su.Lmax > 32767) return cudaErrorInvalidValue;
    S.gtot = (int32_t)dense.size();
    host_mark("slice_setup: dense");
    {
        static const bool on = std::getenv("ECLIP_HOST_TIMING") != nullptr;
        if (on) std::fprintf(stderr, "[eclip host] slice W %d Lmax %d gtot %d g %lld\n", W, su.Lmax, S.gtot, (long long)g);
    }
    S.plo[0] = 0; S.phi[0] = 0;
    for (int w = 0; w < W; w++) { S.plo[w + 1] = S.plo[w] + S.smin[w]; S.phi[w + 1] = S.phi[w] + S.smax[w]; }
    S.slo[W] = 0; S.shi[W] = 0;
    for (int w = W - 1; w >= 0; w--) { S.slo[w] = S.slo[w + 1] + S.smin[w]; S.shi[w] = S.shi[w + 1] + S.smax[w]; }
    S.Tlo = S.slo[0]; S.Thi = S.shi[0];
    S.n_slices = S.Thi - S.Tlo + 1;
    {   // the exact DP sums W weighted terms omega_w B (Lambda N + O) in u64 (O <= T'max in every linear mode)
        const unsigned __int128 lim = (~(unsigned __int128)0 >> 64) / (unsigned __int128)(W + 1);
        for (int w = 0; w < W; w++)
            for (int l = 0; l < P.L[w]; l++) {
                const unsigned __int128 h = (unsigned __int128)lev[(size_t)w * su.Lmax + l].B *
                                            (unsigned __int128)(P.lamN + S.Thi * g) * (unsigned __int128)P.wt[w];
                if (h > lim) return cudaErrorNotSupported;   // -> ECLIP_E_TOO_LARGE (use ENUM)
            }
    }
    // the widest D range over all slices: per worker, hi(T) - lo(T) + 1 = min(shi, T - plo) - max(slo, T - phi) + 1
    // is concave and piecewise linear in T, so its maximum over [Tlo, Thi] is at an end or a breakpoint
    int64_t mr = 1;
    for (int w = 1; w < W; w++) {
        const int64_t cand[4] = {S.Tlo, S.Thi, S.shi[w] + S.plo[w], S.slo[w] + S.phi[w]};
        for (int64_t T : cand) {
            T = std::min<int64_t>(std::max<int64_t>(T, S.Tlo), S.Thi);
            int64_t lo = std::max(S.slo[w], T - S.phi[w]), hi = std::min(S.shi[w], T - S.plo[w]);
            mr = std::max<int64_t>(mr, hi - lo + 1);
        }
    }
    S.maxrange = (int32_t)mr;
    host_mark("slice_setup: ranges");
    int pad = 1;
    for (int w = 0; w < W; w++) pad = std::max(pad, S.smax[w] - S.smin[w] + 1);
    S.pad = pad + RB + KU;
    // every buffer in one allocation (256-byte aligned pieces)
    s.slots = 148 * 2;
    size_t off = 0;
    auto take = [&](size_t bytes) { const size_t o = off; off = (off + std::max<size_t>(bytes, 1) + 255) & ~(size_t)255; return o; };
    const size_t o_units = take(8), o_dense = take(dense.size() * 2), o_J32 = take(4 * (size_t)S.n_slices);
    const size_t o_Jex = take(sizeof(U256) * (size_t)S.n_slices), o_band = take(4 * (size_t)S.n_slices);
    const size_t o_wtup = take(sizeof(U256) * (size_t)S.n_slices), o_nband = take(4);
    const size_t o_scr = take(8 * (size_t)s.slots * (S.gtot + (size_t)W * S.maxrange));
    unsigned char* blk = nullptr;
    CK(salloc(s, &blk, off));
    s.d_units = (unsigned long long*)(blk + o_units);
    s.dense = (int16_t*)(blk + o_dense);
    s.J32 = (float*)(blk + o_J32);
    s.Jex = (U256*)(blk + o_Jex);
    s.band = (int32_t*)(blk + o_band);
    s.wtup = (U256*)(blk + o_wtup);
    s.nband = (int32_t*)(blk + o_nband);
    s.scratch = (uint64_t*)(blk + o_scr);
    CK(cudaMemcpyAsync(s.dense, dense.data(), dense.size() * 2, cudaMemcpyHostToDevice, st));
    host_mark("slice_setup: done");
    return cudaSuccess;
}

cudaError_t slice_pass1(SliceState& s, const Setup& su, const Tables& tb, Work& wk, cudaStream_t st) {
    (void)su; (void)tb;
    const SliceDev& S = s.h;
    int64_t mine = S.n_slices > S.shard ? (S.n_slices - S.shard + S.n_shards - 1) / S.n_shards : 0;
    const size_t BUF = (size_t)S.maxrange + 2 * (size_t)S.pad + RB;
    size_t gspan = 1;
    for (int w = 0; w < S.W; w++) gspan = std::max<size_t>(gspan, (size_t)(S.smax[w] - S.smin[w] + 1));
    size_t smem = sizeof(float) * (gspan + 2 * BUF);   // one worker's g at a time (k_slice_f32)
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    const void* f = S.obj == O_SUM ? (const void*)k_slice_f32<O_SUM> : (S.obj == O_MAX ? (const void*)k_slice_f32<O_MAX>
                                                                                       : (const void*)k_slice_f32<O_ENERGY>);
    CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaMemsetAsync(s.d_units, 0, sizeof(unsigned long long), st));
    if (mine > 0) {
        if (S.obj == O_SUM) k_slice_f32<O_SUM><<<(unsigned)mine, SL_THREADS, smem, st>>>(S, wk.probs, wk.levs, s.dense, s.J32, s.d_units);
        else if (S.obj == O_MAX) k_slice_f32<O_MAX><<<(unsigned)mine, SL_THREADS, smem, st>>>(S, wk.probs, wk.levs, s.dense, s.J32, s.d_units);
        else k_slice_f32<O_ENERGY><<<(unsigned)mine, SL_THREADS, smem, st>>>(S, wk.probs, wk.levs, s.dense, s.J32, s.d_units);
    }
    k_slice_min<<<1, 1024, 0, st>>>(S, s.J32, wk.m32);
    return cudaGetLastError();
}

cudaError_t slice_pass2_min(SliceState& s, const Setup& su, const Tables& tb, Work& wk, cudaStream_t st) {
    (void)su; (void)tb;
    const SliceDev& S = s.h;
    k_slice_band<<<1, 1024, 0, st>>>(S, s.J32, wk.m32, s.band, s.nband);
    k_slice_exact<<<s.slots, SLX, 0, st>>>(S, wk.probs, wk.levs, s.dense, s.band, s.nband, s.scratch, s.Jex);
    k_slice_hstar<<<1, 32, 0, st>>>(s.band, s.nband, s.Jex, wk.hstar);
    return cudaGetLastError();
}

cudaError_t slice_pass2_first(SliceState& s, const Setup& su, const Tables& tb, Work& wk, cudaStream_t st) {
    (void)su; (void)tb;
    const SliceDev& S = s.h;
    k_slice_walk<<<s.slots, SLX, 0, st>>>(S, wk.probs, wk.levs, s.dense, s.band, s.nband, s.scratch, s.Jex,
                                                 wk.hstar, s.wtup);
    k_slice_first<<<1, 32, 0, st>>>(s.nband, s.wtup, wk.first);
    return cudaGetLastError();
}

cudaError_t slice_decode_winner(SliceState& s, const Setup& su, Work& wk, cudaStream_t st) {
    (void)s; (void)su; (void)wk; (void)st;
    return cudaSuccess;
}

}  // namespace eclip
