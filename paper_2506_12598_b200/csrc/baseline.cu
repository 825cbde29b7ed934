// baseline.cu — the paper's comparison planners, evaluated on the GPU under the
// same model as the optimizer:
//   ALL_MAX      every kernel group at the worker's largest allowed size ("Baseline": "send all
//                incoming kernels to the default stream that uses all 60 CUs", PAPER §V)
//   MODEL_WISE   one size per model: smallest c with sum_g t_g(c) <= factor sum_g t_g(max)
//                (Model-Wise right-sizing P:396; SPEC model_wise_rightsize S:90-98)
//   KERNEL_WISE  every group at its threshold: smallest c with t_g(c) <= (1 + tol) t_g(max)
//                ("minimum number of CUs needed without noticeable slowdown" P:264; SPEC
//                min_cu_threshold S:80-88; the KW^IOCTL / KW^Prealloc scenarios P:400-404)
// Predicates are exact: tol / factor are the rationals num/den with den = 1e9.
#include "engine.h"

namespace eclip {

// solo time of group g at size column j: beta_g(c_j) = sum of its kernels' times
__device__ __forceinline__ int64_t group_beta(const BaseJob& J, int w, int g, int j) {
    int64_t b = 0;
    for (int k = J.bounds[w][g]; k < J.bounds[w][g + 1]; k++) b += J.exec[w][(size_t)k * J.C + j];
    return b;
}

__global__ void k_baseline(BaseJob J, BaseOut o) {
    __shared__ int64_t sS[MAXW], sB[MAXW];
    __shared__ double alpha_w[MAXW];
    const int w = threadIdx.x;
    if (w < J.W) {
        const int G = J.G[w], C = J.C;
        int jmax = 0;
        for (int j = 0; j < C; j++)
            if ((J.mask[w] >> j) & 1u) jmax = j;
        int model_col = jmax;
        if (J.kind == 1) {   // model-wise right-size
            int64_t tmax = 0;
            for (int g = 0; g < G; g++) tmax += group_beta(J, w, g, jmax);
            for (int j = 0; j < C; j++) {
                if (!((J.mask[w] >> j) & 1u)) continue;
                int64_t t = 0;
                for (int g = 0; g < G; g++) t += group_beta(J, w, g, j);
                if ((u128)t * J.den <= (u128)tmax * J.num) { model_col = j; break; }
            }
        }
        int64_t S = 0, B = 0;
        int prev = -1, sw = 0;
        for (int g = 0; g < G; g++) {
            int col = jmax;
            if (J.kind == 1) col = model_col;
            else if (J.kind == 2) {   // kernel-wise threshold
                const int64_t tm = group_beta(J, w, g, jmax);
                for (int j = 0; j < C; j++) {
                    if (!((J.mask[w] >> j) & 1u)) continue;
                    if ((u128)group_beta(J, w, g, j) * J.den <= (u128)tm * (J.den + J.num)) { col = j; break; }
                }
            }
            if (g > 0 && col != prev) sw++;
            prev = col;
            S += (int64_t)(J.bounds[w][g + 1] - J.bounds[w][g]) * J.sizes[col];
            B += group_beta(J, w, g, col);
            if (o.group_sm) o.group_sm[w * o.stride + g] = J.sizes[col];
        }
        sS[w] = S;
        sB[w] = B;
        if (o.switches) o.switches[w] = sw;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int W = J.W;
        const double N = (double)J.N;
        double avg[MAXW], sum_avg = 0.0;
        for (int v = 0; v < W; v++) { avg[v] = (double)sS[v] / (double)J.K[v]; sum_avg += avg[v]; }
        double mk = 0.0, wmk = 0.0, obj = 0.0, thr = 0.0;
        // exact QoS check: h_w = B_w (D + O^_w) <= floor(Q_w D)
        uint64_t lam = 1;
        for (int v = 0; v < W; v++) { const uint64_t g = gcd_u64(lam, (uint64_t)J.K[v]); lam = lam / g * (uint64_t)J.K[v]; }
        const int64_t lamN = (int64_t)lam * J.N;
        int E = 0;
        if (J.mode == M_MATRIX)
            for (int a = 0; a < W; a++)
                for (int b = 0; b < W; b++)
                    if (a != b) { const int kb = frac_bits_d((double)J.M[a * MAXW_ENUM + b], 32); E = kb > E ? kb : E; }
        const u128 D = (u128)lamN << E;
        int64_t Tp = 0;
        for (int v = 0; v < W; v++) Tp += sS[v] * (int64_t)(lam / (uint64_t)J.K[v]);
        int status = 0;
        for (int v = 0; v < W; v++) {
            double ov;
            u128 Oh;
            const int64_t Sp = sS[v] * (int64_t)(lam / (uint64_t)J.K[v]);
            if (J.mode == M_EXCL) { ov = sum_avg - avg[v]; Oh = (u128)(Tp - Sp); }
            else if (J.mode == M_PAPER) { ov = sum_avg; Oh = (u128)Tp; }
            else if (J.mode == M_EXCESS) { ov = sum_avg - N > 0.0 ? sum_avg - N : 0.0; Oh = Tp > lamN ? (u128)(Tp - lamN) : 0; }
            else {
                ov = 0.0;
                Oh = 0;
                for (int u = 0; u < W; u++) {
                    if (u == v) continue;
                    ov += (double)J.M[v * MAXW_ENUM + u] * avg[u];
                    Oh += (u128)(int64_t)ldexp((double)J.M[v * MAXW_ENUM + u], E) *
                          (u128)(sS[u] * (int64_t)(lam / (uint64_t)J.K[u]));
                }
            }
            const u128 h = (u128)sB[v] * (D + Oh);
            if (h > floor_qD(J.Q[v], D)) status = 1;
            const double alpha = ov / N;
            alpha_w[v] = alpha;
            const double Lw = (double)sB[v] * (1.0 + alpha);
            mk = Lw > mk ? Lw : mk;
            obj += J.wv[w] * Lw;                       // per-worker weights (R20), 1 by default
            wmk = J.wv[w] * Lw > wmk ? J.wv[w] * Lw : wmk;
            thr += 1e9 / Lw;
            if (o.latency) o.latency[v] = Lw;
        }
        double frac = sum_avg / N;
        if (frac > 1.0) frac = 1.0;
        const double pw = (double)J.p_idle + ((double)J.p_max - (double)J.p_idle) * frac;
        if (J.obj == O_MAX) obj = wmk;
        else if (J.obj == O_ENERGY) obj = pw * mk;
        o.scalars[0] = obj;
        o.scalars[1] = mk;
        o.scalars[2] = pw;
        o.scalars[3] = pw * mk * 1e-9;
        o.scalars[4] = thr;
        *o.status = status;
    }
    __syncthreads();
    if (w < J.W && o.group_lat) {
        for (int g = 0; g < J.G[w]; g++) {
            int col = 0;
            for (int j = 0; j < J.C; j++)
                if (J.sizes[j] == o.group_sm[w * o.stride + g]) col = j;
            o.group_lat[w * o.stride + g] = (double)group_beta(J, w, g, col) * (1.0 + alpha_w[w]);
        }
    }
}

cudaError_t launch_baseline(const BaseJob& j, BaseOut o, cudaStream_t st) {
    k_baseline<<<1, 32 * ((j.W + 31) / 32), 0, st>>>(j, o);
    return cudaGetLastError();
}

}  // namespace eclip
