// simulate.cu — batched discrete-event co-location simulator (SPEC simulator
// and metrics modules S:266-430; C-ABI eclip_simulate in include/eclip.h).
//
// One thread simulates one scenario (a co-location mix + a lookup table per worker + an overhead
// model): closed-loop requests per worker, kernels redirected to pools of SM groups, a shared FIFO
// default stream, barrier / repartition delays, processor-sharing slowdown alpha(t) = sum of shared
// SMs with co-runners / N recomputed at every start and completion, exact energy integral of the
// linear power model, nearest-rank p95.  The event loop is serial per scenario (SPEC "strictly
// single-threaded and deterministic"); the batch is the parallel dimension.  Every floating-
// point step is an explicit IEEE binary64 round-to-nearest operation in the oracle's order
// (oracle/simulator.py), so results are reproducible bit for bit.
#include <cuda_runtime.h>

#include "engine.h"

namespace eclip {

constexpr int SIM_W = 8;

__device__ __forceinline__ unsigned long long sm64(unsigned long long x) {
    x += 0x9E3779B97F4A7C15ull;
    unsigned long long z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double sim_uniform(unsigned long long seed, long long s, int w, int r, int k) {
    const unsigned long long key = seed + ((((((unsigned long long)s * 8ull + (unsigned long long)w) << 20) +
                                             (unsigned long long)r) << 8) + (unsigned long long)k);
    return __dmul_rn((double)(sm64(key) >> 11), 1.0 / 9007199254740992.0);
}
__device__ __forceinline__ double sim_tri(double u, double lo, double mode, double hi) {
    if (hi <= lo) return lo;
    const double fc = __ddiv_rn(__dsub_rn(mode, lo), __dsub_rn(hi, lo));
    if (u < fc) return __dadd_rn(lo, __dsqrt_rn(__dmul_rn(__dmul_rn(u, __dsub_rn(hi, lo)), __dsub_rn(mode, lo))));
    return __dsub_rn(hi, __dsqrt_rn(__dmul_rn(__dmul_rn(__dsub_rn(1.0, u), __dsub_rn(hi, lo)), __dsub_rn(hi, mode))));
}

__device__ __forceinline__ int sms_of(uint32_t m, const int32_t* gsm, int G) {
    int s = 0;
    for (int g = 0; g < G; g++)
        if ((m >> g) & 1u) s += gsm[g];
    return s;
}

__global__ void __launch_bounds__(128) k_simulate(SimJob J, SimOut o, double* latbuf) {
    const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= J.S) return;
    const int W = J.W, K = J.K, C = J.C, full = C - 1;
    const int32_t* nk = J.n_kernels + s * W;
    const double* beta = J.beta + s * (long long)W * K * C;
    const int32_t* tab = J.table + s * (long long)W * K;
    double* lat = latbuf + s * (long long)W * J.n_requests;
    int req[SIM_W], kk[SIM_W];
    bool running[SIM_W], fin[SIM_W];
    double ready[SIM_W], rem[SIM_W], rstart[SIM_W], disp[SIM_W], tfin[SIM_W], lsum[SIM_W], alpha[SIM_W];
    for (int w = 0; w < W; w++) {
        req[w] = 0; kk[w] = 0; running[w] = false; fin[w] = false;
        ready[w] = 0.0; rem[w] = 0.0; rstart[w] = 0.0; disp[w] = 0.0; tfin[w] = 0.0; lsum[w] = 0.0;
    }
    auto stream_of = [&](int w, int j) -> int { return j == full ? (J.shared_default ? -1 : -2 - w) : w * C + j; };
    double t = 0.0, energy = 0.0;
    int barriers = 0;
    long long events = 0;
    const double N = (double)J.N;
    for (;;) {
        // 1. start every startable kernel (shared default stream: FIFO head only)
        bool dbusy = false;
        int hw = -1, hk = -1;
        if (J.shared_default) {
            double bd = 0.0;
            for (int w = 0; w < W; w++) {
                if (running[w] && tab[w * K + kk[w]] == full) dbusy = true;
                if (fin[w]) continue;
                int d = -1;
                for (int k = kk[w]; k < nk[w]; k++)
                    if (tab[w * K + k] == full) { d = k; break; }
                if (d < 0 || (running[w] && kk[w] == d)) continue;
                if (hw < 0 || disp[w] < bd) { bd = disp[w]; hw = w; hk = d; }   // ties: lowest worker
            }
        }
        for (int w = 0; w < W; w++) {
            if (fin[w] || running[w] || ready[w] > t) continue;
            const int j = tab[w * K + kk[w]];
            if (j == full && J.shared_default) {
                if (dbusy || hw != w || hk != kk[w]) continue;
                dbusy = true;
            }
            running[w] = true;
            rem[w] = __dmul_rn(beta[((long long)w * K + kk[w]) * C + j], J.oversub);
        }
        // 2. rates and busy SMs
        bool any = false, all_fin = true;
        uint32_t busy_m = 0;
        for (int a = 0; a < W; a++) {
            all_fin &= fin[a];
            if (!running[a]) continue;
            any = true;
            const uint32_t ma = J.mask[a * C + tab[a * K + kk[a]]];
            busy_m |= ma;
            int sh = 0;
            for (int b = 0; b < W; b++)
                if (b != a && running[b]) sh += sms_of(ma & J.mask[b * C + tab[b * K + kk[b]]], J.group_sm, J.G);
            alpha[a] = __ddiv_rn((double)sh, N);
        }
        if (!any && all_fin) break;
        const double busy = (double)sms_of(busy_m, J.group_sm, J.G);
        // 3. next event
        double tc = INFINITY, tr = INFINITY;
        for (int a = 0; a < W; a++)
            if (running[a]) tc = fmin(tc, __dadd_rn(t, __dmul_rn(rem[a], __dadd_rn(1.0, alpha[a]))));
        for (int w = 0; w < W; w++)
            if (!fin[w] && !running[w] && ready[w] > t) tr = fmin(tr, ready[w]);
        const double tn = fmin(tc, tr);
        if (isinf(tn)) { o.status[s] = -1; return; }   // deadlock (cannot happen for valid inputs)
        const double dt = __dsub_rn(tn, t);
        energy = __dadd_rn(energy, __dmul_rn(__dadd_rn(J.p_idle, __dmul_rn(__dsub_rn(J.p_max, J.p_idle), __ddiv_rn(busy, N))), dt));
        uint32_t done = 0;
        for (int a = 0; a < W; a++) {
            if (!running[a]) continue;
            if (__dadd_rn(t, __dmul_rn(rem[a], __dadd_rn(1.0, alpha[a]))) == tc && tc == tn) done |= 1u << a;
            else rem[a] = __dsub_rn(rem[a], __ddiv_rn(dt, __dadd_rn(1.0, alpha[a])));
        }
        t = tn;
        // 4. completions (worker order)
        for (int a = 0; a < W; a++) {
            if (!((done >> a) & 1u)) continue;
            events++;
            running[a] = false;
            const int jprev = tab[a * K + kk[a]];
            kk[a]++;
            if (kk[a] == nk[a]) {
                const double l = __dsub_rn(t, rstart[a]);
                lat[(long long)a * J.n_requests + req[a]] = l;
                lsum[a] = __dadd_rn(lsum[a], l);
                req[a]++;
                kk[a] = 0;
                if (req[a] == J.n_requests) { fin[a] = true; tfin[a] = t; continue; }
                rstart[a] = t; disp[a] = t; ready[a] = t;
            } else {
                const int jn = tab[a * K + kk[a]];
                double extra = 0.0;
                if (J.ioctl) {
                    if (jn != jprev) extra = sim_tri(sim_uniform(J.seed, s, a, req[a], kk[a]), J.io_lo, J.io_mode, J.io_hi);
                } else if (stream_of(a, jn) != stream_of(a, jprev)) {
                    barriers++;
                    extra = J.barrier_ns;
                }
                ready[a] = __dadd_rn(t, extra);
            }
        }
    }
    const double R = (double)J.n_requests;
    for (int w = 0; w < W; w++) {
        o.throughput_rps[s * W + w] = __ddiv_rn(R, __dmul_rn(tfin[w], 1e-9));
        o.mean_ns[s * W + w] = __ddiv_rn(lsum[w], R);
        // nearest-rank p95: the smallest value with at least ceil(0.95 n) values <= it
        const int rank = (int)ceil(0.95 * (double)J.n_requests);
        const double* L = lat + (long long)w * J.n_requests;
        double best = INFINITY;
        for (int i = 0; i < J.n_requests; i++) {
            int le = 0;
            for (int q = 0; q < J.n_requests; q++) le += L[q] <= L[i];
            if (le >= rank && L[i] < best) best = L[i];
        }
        o.p95_ns[s * W + w] = best;
    }
    o.makespan_ns[s] = t;
    const double ej = __dmul_rn(energy, 1e-9);
    o.energy_j[s] = ej;
    o.req_per_j[s] = __ddiv_rn((double)W * R, ej);
    o.barriers[s] = barriers;
    o.events[s] = events;
    o.status[s] = 0;
}

cudaError_t launch_simulate(const SimJob& J, const SimOut& o, double* latbuf, cudaStream_t st) {
    const long long blocks = (J.S + 127) / 128;
    k_simulate<<<(unsigned)blocks, 128, 0, st>>>(J, o, latbuf);
    return cudaGetLastError();
}

}  // namespace eclip
