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
//                                       min_{j' != j} V[g+1][j'][r-1][s-need_gj] )
// using the best / second-best over j' (O(1) per state).  All G layers are kept (global
// memory, L2-resident) for the greedy witness reconstruction.
//
// One cooperative launch covers every table; layers are separated by grid-wide barriers.
#include <cooperative_groups.h>

#include "engine.h"

namespace cg = cooperative_groups;

namespace eclip {

static constexpr int64_t INF64 = INT64_MAX;

__device__ __forceinline__ size_t vidx(const LevelJob& J, int g, int j, int r, int s) {
    return ((((size_t)g * J.C + j) * (J.R + 1) + r) * (size_t)(J.smax + 1)) + s;
}

__global__ void __launch_bounds__(256) k_levels(const LevelJob* __restrict__ jobs, int n_jobs, int gmax) {
    cg::grid_group grid = cg::this_grid();
    const size_t gtid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t gstride = (size_t)gridDim.x * blockDim.x;

    for (int step = 0; step < gmax; step++) {
        // ---- phase A: best / second-best over j' of layer g+1 (for steps >= 1) ----
        if (step > 0) {
            for (int t = 0; t < n_jobs; t++) {
                const LevelJob& J = jobs[t];
                int g = J.G - 1 - step;
                if (g < 0) continue;
                size_t n = (size_t)(J.R + 1) * (J.smax + 1);
                for (size_t i = gtid; i < n; i += gstride) {
                    int r = (int)(i / (J.smax + 1)), s = (int)(i % (J.smax + 1));
                    int64_t b1 = INF64, b2 = INF64;
                    int a1 = -1;
                    for (int j = 0; j < J.C; j++) {
                        if (!((J.mask >> j) & 1u)) continue;
                        int64_t v = J.V[vidx(J, g + 1, j, r, s)];
                        if (v < b1) { b2 = b1; b1 = v; a1 = j; }
                        else if (v < b2) { b2 = v; }
                    }
                    J.best[2 * i] = b1;
                    J.best[2 * i + 1] = b2;
                    J.barg[i] = a1;
                }
            }
            grid.sync();
        }
        // ---- phase B: layer g ----
        for (int t = 0; t < n_jobs; t++) {
            const LevelJob& J = jobs[t];
            int g = J.G - 1 - step;
            if (g < 0) continue;
            size_t n = (size_t)J.C * (J.R + 1) * (J.smax + 1);
            for (size_t i = gtid; i < n; i += gstride) {
                int s = (int)(i % (J.smax + 1));
                size_t q = i / (J.smax + 1);
                int r = (int)(q % (J.R + 1));
                int j = (int)(q / (J.R + 1));
                int64_t out = INF64;
                if ((J.mask >> j) & 1u) {
                    int nd = J.need[g * J.C + j];
                    int64_t b = J.beta[g * J.C + j];
                    if (g == J.G - 1) {
                        if (s == nd) out = b;
                    } else if (nd <= s) {
                        int sp = s - nd;
                        int64_t v = J.V[vidx(J, g + 1, j, r, sp)];
                        if (r >= 1) {
                            size_t bi = (size_t)(r - 1) * (J.smax + 1) + sp;
                            int64_t w = (J.barg[bi] != j) ? J.best[2 * bi] : J.best[2 * bi + 1];
                            if (w < v) v = w;
                        }
                        if (v != INF64) out = b + v;
                    }
                }
                J.V[vidx(J, g, j, r, s)] = out;
            }
        }
        grid.sync();
    }

    // ---- phase C/D: per job (one CTA each): B*(s), compaction of attained levels ----
    for (int t = blockIdx.x; t < n_jobs; t += gridDim.x) {
        const LevelJob& J = jobs[t];
        __shared__ int s_count;
        __shared__ int s_warp[32];
        if (threadIdx.x == 0) s_count = 0;
        __syncthreads();
        for (int base = 0; base <= J.smax; base += blockDim.x) {
            int s = base + threadIdx.x;
            int64_t b = INF64;
            if (s <= J.smax) {
                for (int j = 0; j < J.C; j++) {
                    if (!((J.mask >> j) & 1u)) continue;
                    int64_t v = J.V[vidx(J, 0, j, J.R, s)];
                    if (v < b) b = v;
                }
                J.best[s] = b;  // reuse workspace: B*(s)
            }
            int valid = (s <= J.smax) && (b != INF64);
            unsigned bal = __ballot_sync(0xffffffffu, valid);
            int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
            if (lane == 0) s_warp[warp] = __popc(bal);
            __syncthreads();
            if (threadIdx.x == 0) {
                int acc = s_count;
                for (int w = 0; w < (int)(blockDim.x >> 5); w++) { int c = s_warp[w]; s_warp[w] = acc; acc += c; }
                s_count = acc;
            }
            __syncthreads();
            if (valid) {
                int pos = s_warp[warp] + __popc(bal & ((1u << lane) - 1u));
                J.sidx[pos] = s;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) *J.outL = s_count;
        __syncthreads();
    }
    grid.sync();

    // ---- phase E: greedy reconstruction of the canonical witness of every level ----
    for (int t = 0; t < n_jobs; t++) {
        const LevelJob& J = jobs[t];
        int L = *J.outL;
        for (size_t l = gtid; l < (size_t)L; l += gstride) {
            int rem = J.sidx[l];
            int64_t opt = J.best[rem];
            int r = J.R, prev = -1;
            for (int g = 0; g < J.G; g++) {
                int pick = -1;
                for (int j = 0; j < J.C && pick < 0; j++) {
                    if (!((J.mask >> j) & 1u)) continue;
                    int nd = J.need[g * J.C + j];
                    if (nd > rem) continue;
                    int rr = (g == 0 || j == prev) ? r : r - 1;
                    if (rr < 0) continue;
                    if (J.V[vidx(J, g, j, rr, rem)] == opt) pick = j;
                }
                // pick >= 0 always holds (opt is attained); guard anyway
                if (pick < 0) pick = 0;
                if (g > 0 && pick != prev) r--;
                opt -= J.beta[g * J.C + pick];
                rem -= J.need[g * J.C + pick];
                prev = pick;
                J.wtmp[l * J.G + g] = (uint8_t)pick;
            }
        }
    }
    grid.sync();

    // ---- phase F: rank of every level = number of lexicographically smaller witnesses ----
    for (int t = 0; t < n_jobs; t++) {
        const LevelJob& J = jobs[t];
        int L = *J.outL;
        for (size_t l = gtid; l < (size_t)L; l += gstride) {
            const uint8_t* a = J.wtmp + l * J.G;
            int rk = 0;
            for (int m = 0; m < L; m++) {
                const uint8_t* b = J.wtmp + (size_t)m * J.G;
                for (int g = 0; g < J.G; g++) {
                    if (b[g] != a[g]) { rk += (b[g] < a[g]); break; }
                }
            }
            J.rank[l] = rk;
        }
    }
    grid.sync();

    // ---- phase G: scatter to rank order ----
    for (int t = 0; t < n_jobs; t++) {
        const LevelJob& J = jobs[t];
        int L = *J.outL;
        for (size_t l = gtid; l < (size_t)L; l += gstride) {
            int rk = J.rank[l];
            int s = J.sidx[l];
            J.outS[rk] = (int64_t)s * J.u;
            J.outB[rk] = J.best[s];
            for (int g = 0; g < J.G; g++) J.outW[(size_t)rk * J.G + g] = J.wtmp[l * J.G + g];
        }
    }
}

cudaError_t launch_levels(LevelJob* d_jobs, const LevelJob* h_jobs, int n_jobs, cudaStream_t st) {
    int gmax = 0;
    for (int i = 0; i < n_jobs; i++) gmax = h_jobs[i].G > gmax ? h_jobs[i].G : gmax;
    int dev = 0, nsm = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_levels, 256, 0);
    if (e != cudaSuccess) return e;
    if (per_sm > 4) per_sm = 4;
    int grid = nsm * (per_sm > 0 ? per_sm : 1);
    void* args[] = {(void*)&d_jobs, (void*)&n_jobs, (void*)&gmax};
    return cudaLaunchCooperativeKernel((void*)k_levels, dim3(grid), dim3(256), args, 0, st);
}

}  // namespace eclip
