// levels.cu — K1: level-1 DP on the GPU (DESIGN.md §4 "K1").
//
// For one worker (model, grouping, allowed sizes, switch budget R) compute, for every
// attainable CU-sum S = sum_g n_g c_{sigma_g}, the minimum solo time
//     B*(S) = min { sum_g beta[g][sigma_g] : sigma in A^G, sw(sigma) <= R }
// (one configuration per kernel group P:299-300; switchTotal_w <= switchMax P:302-303;
//  beta = profile P:308) and its canonical witness (lexicographically smallest minimiser),
// then order the levels by witness (the canonical rank order that defines candidate
// indices).
//
// Suffix DP (a different recurrence from the oracle's memoised forward recursion):
//   V[g][j][r][s] = min over sigma_g..sigma_{G-1} with sigma_g = j, at most r switches
//                   inside g..G-1, and suffix level s (units of u = gcd of allowed sizes)
//   V[G-1][j][r][s] = beta[G-1][j]            if s == need[G-1][j]
//   V[g][j][r][s]   = beta[g][j] + min( V[g+1][j][r][s-need_gj],
//                                       min_{j' != j} V[g+1][j'][r-1][s-need_gj] ).
// One thread owns a (table, r, s) cell of a layer: it computes all C sizes j and, from
// them, the best / second-best / arg-best over j that the next layer needs, so each layer
// costs one grid-wide barrier.  All layers stay in global memory (L2-resident) for the
// greedy witness reconstruction.  Witnesses are packed 8 groups per 64-bit word (group 0
// in the top byte) so ranking compares words.  One cooperative launch covers every table.
#include <cooperative_groups.h>

#include <cstdio>

#include "engine.h"

namespace cg = cooperative_groups;

namespace eclip {

static constexpr int MAXJ = 64;      // tables per launch (host splits larger sets)

template <class VT> struct VPair;
template <> struct VPair<int32_t> { typedef int2 T; };
template <> struct VPair<int64_t> { typedef longlong2 T; };
template <class VT> __device__ __forceinline__ VT vinf() { return VT(~(unsigned long long)0 >> (65 - 8 * sizeof(VT))); }

__device__ __forceinline__ size_t vidx(const LevelJob& J, int g, int j, int k) {
    return ((size_t)g * J.C + j) * J.ncp + k;
}
__device__ __forceinline__ int nwords(const LevelJob& J) { return (J.G + 7) / 8; }

// one (r, s) cell k of layer g = G-1-step: V for all sizes j, and best / second best / arg over j.
// Layer g+1's V, best and arg are read through L1 (plain loads): every layer has its own 128-byte
// aligned region, written completely in its step and read only after the grid barrier that ends it,
// so no SM can hold a line of it from before it was written; neighbouring cells read overlapping
// best / arg entries (s - need_j for the C sizes j), which L1 then serves.
template <int CM, class VT>   // CM >= J.C: the loops over sizes are unrolled, so their loads are issued together
__device__ __forceinline__ void dp_cell(const LevelJob& J, int step, int k) {
    typedef typename VPair<VT>::T P2;
    const VT INF = vinf<VT>();
    const int S1 = J.smax + 1;
    const int r = k / S1, s = k - r * S1;
    const int g = J.G - 1 - step;
    VT* V = reinterpret_cast<VT*>(J.V);
    const P2* bestp = reinterpret_cast<const P2*>(J.best);
    VT b1 = INF, b2 = INF;
    int a1 = 255;
    // Branch-free: every load of the cell is issued unconditionally at a clamped (valid) address and the
    // unused values are discarded by selects, so the C sizes' loads are all in flight together (with a
    // branch per size the compiler keeps them inside the branches: one L2 round trip per size).
    const int gn = g + 1 < J.G ? g + 1 : g;   // (layer G-1 reads nothing)
    const bool last = g == J.G - 1;
    const int rm = r >= 1 ? r - 1 : 0;
    VT lv[CM], lb1[CM], lb2[CM];
    int la[CM], lnd[CM];
#pragma unroll
    for (int j = 0; j < CM; j++) {   // loads only
        const int jc = j < J.C ? j : J.C - 1;
        const int nd = J.need[g * J.C + jc];
        const int sp = nd <= s ? s - nd : 0;
        lnd[j] = nd;
        lv[j] = V[vidx(J, gn, jc, r * S1 + sp)];
        const size_t bi = (size_t)gn * J.ncp + rm * S1 + sp;
        la[j] = J.barg[bi];
        const P2 bb2 = bestp[bi];
        lb1[j] = bb2.x; lb2[j] = bb2.y;
    }
    VT outv[CM];
#pragma unroll
    for (int j = 0; j < CM; j++) {   // then the arithmetic, as selects
        const int jc = j < J.C ? j : J.C - 1;
        const bool act = j < J.C && ((J.mask >> j) & 1u);
        const VT b = (VT)J.beta[g * J.C + jc];
        const VT w = la[j] != j ? lb1[j] : lb2[j];
        const VT v = (r >= 1 && w < lv[j]) ? w : lv[j];
        const VT o_last = (act && s == lnd[j]) ? b : INF;
        const VT o_in = (act && lnd[j] <= s && v != INF) ? b + v : INF;
        outv[j] = last ? o_last : o_in;
    }
#pragma unroll
    for (int j = 0; j < CM; j++) {
        if (j >= J.C) break;
        const VT out = outv[j];
        V[vidx(J, g, j, k)] = out;
        if (out < b1) { b2 = b1; b1 = out; a1 = j; }
        else if (out < b2) { b2 = out; }
    }
    const size_t bo = (size_t)g * J.ncp + k;
    P2 o;
    o.x = b1; o.y = b2;
    reinterpret_cast<P2*>(J.best)[bo] = o;
    J.barg[bo] = (uint8_t)a1;
}

// greedy reconstruction of level l's canonical witness (packed words)
template <int CM, class VT>
__device__ __forceinline__ void reconstruct(const LevelJob& J, int l) {
    const VT* V = reinterpret_cast<const VT*>(J.V);
    const int S1 = J.smax + 1;
    int rem = J.sidx[l];
    int64_t opt = J.bstar[rem];
    int r = J.R, prev = -1;
    const int nw = nwords(J);
    uint64_t word = 0;
    for (int g = 0; g < J.G; g++) {
        int pick = -1;
        // the candidates' values are loaded together (independent), then the first match is taken
        VT cv[CM];
#pragma unroll
        for (int j = 0; j < CM; j++) {   // branch-free: every load issued (clamped address), then selected
            const int jc = j < J.C ? j : J.C - 1;
            const int nd = J.need[g * J.C + jc];
            const int rr = (g == 0 || j == prev) ? r : r - 1;
            const bool ok = j < J.C && ((J.mask >> j) & 1u) && nd <= rem && rr >= 0;
            const VT v = V[vidx(J, g, jc, (rr >= 0 ? rr : 0) * S1 + rem)];
            cv[j] = ok ? v : vinf<VT>();
        }
#pragma unroll
        for (int j = CM - 1; j >= 0; j--)   // the smallest matching j
            if (j < J.C && (int64_t)cv[j] == opt) pick = j;
        if (pick < 0) pick = 0;   // unreachable: opt is attained
        if (g > 0 && pick != prev) r--;
        opt -= J.beta[g * J.C + pick];
        rem -= J.need[g * J.C + pick];
        prev = pick;
        word |= (uint64_t)pick << (8 * (7 - (g & 7)));
        if ((g & 7) == 7 || g == J.G - 1) {
            J.wtmp[(size_t)l * nw + (g >> 3)] = word;
            word = 0;
        }
    }
}

// rank of level l = number of lexicographically smaller witnesses; scatter to rank order
__device__ __forceinline__ void rank_level(const LevelJob& J, int l, int L) {
    const int nw = nwords(J);
    const uint64_t* a = J.wtmp + (size_t)l * nw;
    int rk = 0;
    for (int m = 0; m < L; m++) {
        const uint64_t* b = J.wtmp + (size_t)m * nw;
        for (int q = 0; q < nw; q++) {
            if (b[q] != a[q]) { rk += (b[q] < a[q]); break; }
        }
    }
    const int s = J.sidx[l];
    J.outS[rk] = (int64_t)s * J.u;
    J.outB[rk] = J.bstar[s];
    for (int g = 0; g < J.G; g++) J.outW[(size_t)rk * J.G + g] = (uint8_t)(a[g >> 3] >> (8 * (7 - (g & 7))));
}

// the same with one warp per level: the lanes split the comparisons (L / 32 each) and the witness bytes
__device__ __forceinline__ void rank_level_warp(const LevelJob& J, int l, int L, int lane) {
    const int nw = nwords(J);
    const uint64_t* a = J.wtmp + (size_t)l * nw;
    int rk = 0;
    for (int m = lane; m < L; m += 32) {
        const uint64_t* b = J.wtmp + (size_t)m * nw;
        for (int q = 0; q < nw; q++) {
            const uint64_t bq = b[q], aq = a[q];
            if (bq != aq) { rk += (bq < aq); break; }
        }
    }
    for (int o = 16; o; o >>= 1) rk += __shfl_xor_sync(0xffffffffu, rk, o);
    const int s = J.sidx[l];
    if (lane == 0) {
        J.outS[rk] = (int64_t)s * J.u;
        J.outB[rk] = J.bstar[s];
    }
    for (int g = lane; g < J.G; g += 32) J.outW[(size_t)rk * J.G + g] = (uint8_t)(a[g >> 3] >> (8 * (7 - (g & 7))));
}

// B*(s) = best over j of layer 0 at r = R; compact the attained levels (one CTA per table)
template <class VT>
__device__ __forceinline__ void compact_table(const LevelJob& J) {
    __shared__ int s_count;
    __shared__ int s_warp[32];
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    const int S1 = J.smax + 1;
    for (int base = 0; base <= J.smax; base += blockDim.x) {
        const int s = base + threadIdx.x;
        int64_t b = INT64_MAX;
        if (s <= J.smax) {
            const VT v = reinterpret_cast<const VT*>(J.best)[2 * ((size_t)J.R * S1 + s)];   // layer 0, r = R
            b = v == vinf<VT>() ? INT64_MAX : (int64_t)v;
            J.bstar[s] = b;
        }
        const int valid = (s <= J.smax) && (b != INT64_MAX);
        const unsigned bal = __ballot_sync(0xffffffffu, valid);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (lane == 0) s_warp[warp] = __popc(bal);
        __syncthreads();
        if (threadIdx.x == 0) {
            int acc = s_count;
            for (int w = 0; w < (int)(blockDim.x >> 5); w++) { int c = s_warp[w]; s_warp[w] = acc; acc += c; }
            s_count = acc;
        }
        __syncthreads();
        if (valid) J.sidx[s_warp[warp] + __popc(bal & ((1u << lane) - 1u))] = s;
        __syncthreads();
    }
    if (threadIdx.x == 0) *J.outL = s_count;
    __syncthreads();
}

#ifdef K1_DEBUG
__device__ unsigned long long k1_dbg[80];
#define K1_STAMP(i)                                                                                  \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                                      \
        unsigned long long t_;                                                                      \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                     \
        k1_dbg[i] = t_;                                                                             \
    }
#else
#define K1_STAMP(i)
#endif
template <int CM, class VT>
__global__ void __launch_bounds__(256) k_levels(const LevelJob* __restrict__ jobs, int n_jobs, int gmax,
                                                size_t wsm_words) {
    cg::grid_group grid = cg::this_grid();
    __shared__ LevelJob sj[MAXJ];
    __shared__ int off[MAXJ + 1];
    for (int t = threadIdx.x; t < n_jobs; t += blockDim.x) sj[t] = jobs[t];
    __syncthreads();
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int gstride = gridDim.x * blockDim.x;
    // level reconstructions: an order that spreads them over every SM (consecutive levels on different CTAs);
    // each is a latency-bound chain of dependent loads, so fewer per SM is faster
    const int sid = threadIdx.x * gridDim.x + blockIdx.x;

    K1_STAMP(0)
    // ---- DP layers G-1 .. 0 (one cell = (table, r, s); all C sizes per cell) ----
    for (int step = 0; step < gmax; step++) {
        K1_STAMP(1 + step)
        if (threadIdx.x == 0) {
            off[0] = 0;
            for (int t = 0; t < n_jobs; t++)
                off[t + 1] = off[t] + ((sj[t].G - 1 - step >= 0) ? (sj[t].R + 1) * (sj[t].smax + 1) : 0);
        }
        __syncthreads();
        const int total = off[n_jobs];
        for (int i = gtid; i < total; i += gstride) {   // consecutive cells on consecutive threads (coalesced)
            int t = 0;
            while (off[t + 1] <= i) t++;
            const LevelJob& J = sj[t];
            const int k = i - off[t];
            dp_cell<CM, VT>(J, step, k);
        }
        // the next layer's profile rows (need, beta) into this SM's L1 while the grid barrier completes:
        // the first loads of every cell of the next layer then hit L1
        if (threadIdx.x < n_jobs) {
            const LevelJob& J = sj[threadIdx.x];
            const int gn = J.G - 2 - step;
            if (gn >= 0) {
                asm volatile("prefetch.global.L1 [%0];" ::"l"(J.need + gn * J.C));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(J.beta + gn * J.C));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(J.beta + gn * J.C + 8));
            }
        }
        grid.sync();
    }

    K1_STAMP(70)
    // ---- per table (one CTA each): B*(s) = best over j of layer 0 at r = R; compact ----
    for (int t = blockIdx.x; t < n_jobs; t += gridDim.x) compact_table<VT>(sj[t]);
    grid.sync();
    K1_STAMP(71)

    // flattened (table, level) work for the remaining phases
    if (threadIdx.x == 0) {
        off[0] = 0;
        for (int t = 0; t < n_jobs; t++) off[t + 1] = off[t] + *sj[t].outL;
    }
    __syncthreads();
    const int nlev = off[n_jobs];

    // ---- greedy reconstruction of every level's canonical witness (packed words) ----
    for (int i = sid; i < nlev; i += gstride) {
        int t = 0;
        while (off[t + 1] <= i) t++;
        const LevelJob& J = sj[t];
        const int l = i - off[t];
        reconstruct<CM, VT>(J, l);
    }
    grid.sync();
    K1_STAMP(72)

    // ---- rank = number of lexicographically smaller witnesses; scatter to rank order.  One CTA
    // per table with the table's witness words staged in shared memory (the comparisons are
    // O(L^2); from global memory each thread would walk L dependent L2 loads) ----
    extern __shared__ uint64_t wsm[];
    if (wsm_words == 0) {   // large tables: one warp per level over the whole grid, from global memory (L1-resident)
        const int lane = threadIdx.x & 31;
        for (int i = gtid >> 5; i < nlev; i += gstride >> 5) {
            int t = 0;
            while (off[t + 1] <= i) t++;
            rank_level_warp(sj[t], i - off[t], off[t + 1] - off[t], lane);
        }
        return;
    }
    for (int t = blockIdx.x; t < n_jobs; t += gridDim.x) {
        const LevelJob& J = sj[t];
        const int L = off[t + 1] - off[t], nw = nwords(J);
        if ((size_t)L * nw <= wsm_words) {
            for (int i = threadIdx.x; i < L * nw; i += blockDim.x) wsm[i] = J.wtmp[i];
            __syncthreads();
            for (int l = threadIdx.x; l < L; l += blockDim.x) {
                const uint64_t* a = wsm + (size_t)l * nw;
                int rk = 0;
                for (int m = 0; m < L; m++) {
                    const uint64_t* b = wsm + (size_t)m * nw;
                    for (int q = 0; q < nw; q++)
                        if (b[q] != a[q]) { rk += (b[q] < a[q]); break; }
                }
                const int s = J.sidx[l];
                J.outS[rk] = (int64_t)s * J.u;
                J.outB[rk] = J.bstar[s];
                for (int g = 0; g < J.G; g++) J.outW[(size_t)rk * J.G + g] = (uint8_t)(a[g >> 3] >> (8 * (7 - (g & 7))));
            }
            __syncthreads();
        } else {
            for (int l = threadIdx.x; l < L; l += blockDim.x) rank_level(J, l, L);
        }
    }
    K1_STAMP(73)
}

cudaError_t launch_levels(LevelJob* d_jobs, const LevelJob* h_jobs, int n_jobs, bool v32, cudaStream_t st) {
    if (n_jobs > MAXJ) return cudaErrorInvalidValue;
    int gmax = 0;
    for (int i = 0; i < n_jobs; i++) gmax = h_jobs[i].G > gmax ? h_jobs[i].G : gmax;
    int dev = 0, nsm = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    // shared memory for the ranking phase: the largest table's witness words (level count <= Lcap)
    size_t wsm = 0;
    for (int i = 0; i < n_jobs; i++) {
        const size_t w = (size_t)h_jobs[i].Lcap * ((h_jobs[i].G + 7) / 8);
        if (w > wsm) wsm = w;
    }
    if (wsm > 2048) wsm = 0;   // large tables (many levels, e.g. BASELINE C4) rank from global memory (measured faster)
    size_t wsm_words = wsm;
    int cmax = 0;
    for (int i = 0; i < n_jobs; i++) cmax = h_jobs[i].C > cmax ? h_jobs[i].C : cmax;
    const void* kf = v32 ? (cmax <= 8    ? (const void*)k_levels<8, int32_t>
                            : cmax <= 12 ? (const void*)k_levels<12, int32_t>
                            : cmax <= 16 ? (const void*)k_levels<16, int32_t>
                                         : (const void*)k_levels<32, int32_t>)
                         : (cmax <= 8    ? (const void*)k_levels<8, int64_t>
                            : cmax <= 12 ? (const void*)k_levels<12, int64_t>
                            : cmax <= 16 ? (const void*)k_levels<16, int64_t>
                                         : (const void*)k_levels<32, int64_t>);
    e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(wsm * 8));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kf, 256, wsm * 8);
    if (e != cudaSuccess) return e;
    if (per_sm > 4) per_sm = 4;   // more resident threads: fewer cells per thread on a layer's critical path
    int grid = nsm * (per_sm > 0 ? per_sm : 1);
    void* args[] = {(void*)&d_jobs, (void*)&n_jobs, (void*)&gmax, (void*)&wsm_words};
#ifdef K1_DEBUG
    e = cudaLaunchCooperativeKernel(kf, dim3(grid), dim3(256), args, wsm * 8, st);
    unsigned long long h[80];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, k1_dbg, sizeof h);
    fprintf(stderr, "K1 grid %d gmax %d: layers", grid, gmax);
    for (int i = 1; i <= gmax; i++) fprintf(stderr, " %.1f", (h[i] - h[i - 1]) * 1e-3);
    fprintf(stderr, " | last layer->compact %.1f compact %.1f reconstruct %.1f rank %.1f us\n", (h[70] - h[gmax]) * 1e-3,
            (h[71] - h[70]) * 1e-3, (h[72] - h[71]) * 1e-3, (h[73] - h[72]) * 1e-3);
    return e;
#else
    return cudaLaunchCooperativeKernel(kf, dim3(grid), dim3(256), args, wsm * 8, st);
#endif
}

}  // namespace eclip
