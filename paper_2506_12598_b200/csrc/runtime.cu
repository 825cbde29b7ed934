// runtime.cu — the B200 analogue of ECLIP's runtime scheduler (§IV-A, P:213-251;
// SURVEY.md §8(f) f2; C-ABI in include/eclip_runtime.h; design in DESIGN.md §10).
//
//   pool      one split of the device's SMs into G equal groups (CUDA green contexts, the SE
//             analogue of P:221); per worker and size j < G a green context over j groups
//             (rotation layout, reading R17) with one stream; the full size = primary-context
//             stream(s) over all SMs ("the 60 CU allocation is the default stream")
//   redirect  kernel k of worker w -> the pool stream of lookup-table entry k
//   barrier   an event wait on the predecessor's completion event, only when the predecessor ran
//             on another stream and has not completed
//   harness   synthetic knee-shaped kernels (k_spin), offline profiling of every pool size, and
//             closed-loop co-location runs with one host thread per worker, optionally
//             repartitioning on every switch instead of pre-allocating (the IOCTL path)
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "eclip_runtime.h"

namespace eclip {
int set_error(int code, const char* msg);
}

namespace {

int rt_fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    return eclip::set_error(code, buf);
}

#define RT_CU(x)                                                                                         \
    do {                                                                                                 \
        cudaError_t _e = (x);                                                                            \
        if (_e != cudaSuccess)                                                                           \
            return rt_fail(ECLIP_E_CUDA, "CUDA: %s (%s:%d)", cudaGetErrorString(_e), __FILE__, __LINE__); \
    } while (0)
#define RT_DRV(x)                                                                                        \
    do {                                                                                                 \
        CUresult _r = (x);                                                                               \
        if (_r != CUDA_SUCCESS)                                                                          \
            return rt_fail(ECLIP_E_CUDA, "CUDA driver error %d (%s:%d)", (int)_r, __FILE__, __LINE__);  \
    } while (0)

// driver entry points (no link-time libcuda dependency)
struct Drv {
    CUresult (*DeviceGet)(CUdevice*, int);
    CUresult (*DeviceGetDevResource)(CUdevice, CUdevResource*, CUdevResourceType);
    CUresult (*DevSmResourceSplitByCount)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*,
                                          unsigned int, unsigned int);
    CUresult (*DevResourceGenerateDesc)(CUdevResourceDesc*, CUdevResource*, unsigned int);
    CUresult (*GreenCtxCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int);
    CUresult (*GreenCtxDestroy)(CUgreenCtx);
    CUresult (*GreenCtxStreamCreate)(CUstream*, CUgreenCtx, unsigned int, int);
    CUresult (*StreamDestroy)(CUstream);
};

int load_drv(Drv* d) {
    struct E { const char* name; void** fn; } es[] = {
        {"cuDeviceGet", (void**)&d->DeviceGet},
        {"cuDeviceGetDevResource", (void**)&d->DeviceGetDevResource},
        {"cuDevSmResourceSplitByCount", (void**)&d->DevSmResourceSplitByCount},
        {"cuDevResourceGenerateDesc", (void**)&d->DevResourceGenerateDesc},
        {"cuGreenCtxCreate", (void**)&d->GreenCtxCreate},
        {"cuGreenCtxDestroy", (void**)&d->GreenCtxDestroy},
        {"cuGreenCtxStreamCreate", (void**)&d->GreenCtxStreamCreate},
        {"cuStreamDestroy", (void**)&d->StreamDestroy},
    };
    for (auto& e : es) {
        cudaDriverEntryPointQueryResult q;
        cudaError_t r = cudaGetDriverEntryPoint(e.name, e.fn, cudaEnableDefault, &q);
        if (r != cudaSuccess || q != cudaDriverEntryPointSuccess || !*e.fn)
            return rt_fail(ECLIP_E_CUDA, "driver entry point %s unavailable (green contexts need CUDA 12.4+)", e.name);
    }
    return ECLIP_OK;
}

constexpr int SPIN_THREADS = 256;
constexpr int SPIN_SMEM = 160 * 1024;   // > half an SM's shared memory: one CTA per SM at a time
constexpr int MAXW_RT = 8;

struct KRec {                 // per launched kernel (ECLIP_RT_RECORD)
    unsigned long long t0, t1;
    unsigned int sm[5];
    unsigned int pad[3];
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// iters dependent FMAs per thread; the result is kept live through shared memory
__global__ void __launch_bounds__(SPIN_THREADS) k_spin(int iters, KRec* rec) {
    extern __shared__ float spin_sm[];
    unsigned long long t0 = 0;
    if (rec && threadIdx.x == 0) t0 = gtimer();
    float a = (float)threadIdx.x * 1e-3f, b = 0.999f;
    for (int i = 0; i < iters; i++) a = fmaf(a, b, 1e-3f);
    spin_sm[threadIdx.x] = a;
    __syncthreads();
    if (rec && threadIdx.x == 0) {
        const unsigned long long t1 = gtimer();
        unsigned int smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        atomicMin(&rec->t0, t0);
        atomicMax(&rec->t1, t1);
        if (smid < 160) atomicOr(&rec->sm[smid >> 5], 1u << (smid & 31));
        if (spin_sm[0] == -1.0f) rec->pad[0] = 1;   // never true; keeps the chain live
    }
}

struct Pool {
    cudaStream_t stream = nullptr;
    CUgreenCtx ctx = nullptr;   // null for the full-size (primary context) stream
    uint32_t groups = 0;
    int sms = 0;
};

struct WorkerState {
    std::vector<int32_t> table;   // kernel -> size index
    int prev_stream = -1;         // stream id of the previous kernel (-1: none)
    int cur_stream = -1;          // stream id of the last dispatch
    cudaStream_t cur = nullptr;
    std::vector<cudaEvent_t> ring;   // completion signals
    int ring_pos = 0;
    cudaEvent_t prev_ev = nullptr;
};

}  // namespace

struct eclip_rt {
    int device = 0, W = 0, G = 0, N = 0;
    bool shared_default = true;
    Drv drv{};
    CUdevice cudev = 0;
    std::vector<CUdevResource> groups;   // from one split
    std::vector<int> group_sm;
    std::vector<int> sizes;              // [G] pool sizes in SMs (j groups for j < G, then N)
    std::vector<Pool> pools;             // stream ids: worker-major (w * (G-1) + j-1), then full-size stream(s)
    std::vector<WorkerState> ws;
    ~eclip_rt() {
        cudaSetDevice(device);
        cudaDeviceSynchronize();
        for (auto& w : ws)
            for (cudaEvent_t e : w.ring) cudaEventDestroy(e);
        for (auto& p : pools) {
            if (p.ctx) {
                if (p.stream) drv.StreamDestroy((CUstream)p.stream);
                drv.GreenCtxDestroy(p.ctx);
            } else if (p.stream) {
                cudaStreamDestroy(p.stream);
            }
        }
    }
    int stream_of(int w, int j) const {   // j = size index
        if (j < G - 1) return w * (G - 1) + j;
        return W * (G - 1) + (shared_default ? 0 : w);
    }
    uint32_t mask_of(int w, int j) const {
        if (j >= G - 1) return G >= 32 ? 0xffffffffu : ((1u << G) - 1u);
        const int s = (w * G) / W;
        uint32_t m = 0;
        for (int t = 0; t <= j; t++) m |= 1u << ((s + t) % G);
        return m;
    }
    int make_green(uint32_t m, Pool* p) {   // green context + stream over the groups in m
        std::vector<CUdevResource> rs;
        int sms = 0;
        for (int g = 0; g < G; g++)
            if ((m >> g) & 1u) { rs.push_back(groups[g]); sms += group_sm[g]; }
        CUdevResourceDesc desc;
        RT_DRV(drv.DevResourceGenerateDesc(&desc, rs.data(), (unsigned)rs.size()));
        RT_DRV(drv.GreenCtxCreate(&p->ctx, desc, cudev, CU_GREEN_CTX_DEFAULT_STREAM));
        CUstream st;
        RT_DRV(drv.GreenCtxStreamCreate(&st, p->ctx, CU_STREAM_NON_BLOCKING, 0));
        p->stream = (cudaStream_t)st;
        p->groups = m;
        p->sms = sms;
        return ECLIP_OK;
    }
};

extern "C" int eclip_rt_create(const eclip_rt_config* cfg, eclip_rt** out) {
    if (!cfg || !out) return rt_fail(ECLIP_E_INVALID_ARG, "null argument");
    *out = nullptr;
    if (cfg->n_workers < 1 || cfg->n_workers > MAXW_RT) return rt_fail(ECLIP_E_INVALID_ARG, "n_workers must be in [1, 8]");
    if (cfg->group_sms < 1) return rt_fail(ECLIP_E_INVALID_ARG, "group_sms must be >= 1");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return rt_fail(ECLIP_E_CUDA, "no CUDA device available; the runtime has no CPU fallback");
    if (cfg->device < 0 || cfg->device >= ndev) return rt_fail(ECLIP_E_INVALID_ARG, "device out of range");
    auto rt = std::make_unique<eclip_rt>();
    rt->device = cfg->device;
    rt->W = cfg->n_workers;
    rt->shared_default = cfg->shared_default != 0;
    RT_CU(cudaSetDevice(rt->device));
    RT_CU(cudaFree(0));   // primary context
    int rc = load_drv(&rt->drv);
    if (rc) return rc;
    RT_DRV(rt->drv.DeviceGet(&rt->cudev, rt->device));
    CUdevResource all;
    RT_DRV(rt->drv.DeviceGetDevResource(rt->cudev, &all, CU_DEV_RESOURCE_TYPE_SM));
    rt->N = (int)all.sm.smCount;
    unsigned n = 0;
    RT_DRV(rt->drv.DevSmResourceSplitByCount(nullptr, &n, &all, nullptr, 0, (unsigned)cfg->group_sms));
    if (n < 2) return rt_fail(ECLIP_E_INVALID_ARG, "group_sms %d leaves fewer than 2 groups", cfg->group_sms);
    if (n > 31) n = 31;
    rt->groups.resize(n);
    CUdevResource rem;
    RT_DRV(rt->drv.DevSmResourceSplitByCount(rt->groups.data(), &n, &all, &rem, 0, (unsigned)cfg->group_sms));
    rt->groups.resize(n);
    rt->G = (int)n;
    for (auto& g : rt->groups) rt->group_sm.push_back((int)g.sm.smCount);
    for (int j = 1; j < rt->G; j++) {
        int s = 0;
        for (int g = 0; g < j; g++) s += rt->group_sm[g];
        rt->sizes.push_back(s);
    }
    rt->sizes.push_back(rt->N);
    // the pool: W * (G-1) green-context streams, then the full-size stream(s)
    rt->pools.resize((size_t)rt->W * (rt->G - 1) + (rt->shared_default ? 1 : rt->W));
    for (int w = 0; w < rt->W; w++)
        for (int j = 0; j < rt->G - 1; j++) {
            rc = rt->make_green(rt->mask_of(w, j), &rt->pools[rt->stream_of(w, j)]);
            if (rc) return rc;
        }
    for (size_t i = (size_t)rt->W * (rt->G - 1); i < rt->pools.size(); i++) {
        Pool& p = rt->pools[i];
        RT_CU(cudaStreamCreateWithFlags(&p.stream, cudaStreamNonBlocking));
        p.groups = rt->mask_of(0, rt->G - 1);
        p.sms = rt->N;
    }
    rt->ws.resize(rt->W);
    for (auto& w : rt->ws) {
        w.ring.resize(64);
        for (auto& e : w.ring) RT_CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    RT_CU(cudaFuncSetAttribute((const void*)k_spin, cudaFuncAttributeMaxDynamicSharedMemorySize, SPIN_SMEM));
    *out = rt.release();
    return ECLIP_OK;
}

extern "C" void eclip_rt_free(eclip_rt* rt) { delete rt; }

extern "C" int eclip_rt_info(const eclip_rt* rt, int32_t* n_groups, int32_t* group_sm, int32_t* n_sizes, int32_t* sizes,
                             int32_t* total_sms) {
    if (!rt) return rt_fail(ECLIP_E_INVALID_ARG, "null runtime");
    if (n_groups) *n_groups = rt->G;
    if (group_sm) for (int g = 0; g < rt->G; g++) group_sm[g] = rt->group_sm[g];
    if (n_sizes) *n_sizes = (int32_t)rt->sizes.size();
    if (sizes) for (size_t j = 0; j < rt->sizes.size(); j++) sizes[j] = rt->sizes[j];
    if (total_sms) *total_sms = rt->N;
    return ECLIP_OK;
}

extern "C" int eclip_rt_layout(const eclip_rt* rt, int32_t worker, int32_t j, uint32_t* group_mask, int32_t* stream_id,
                               int32_t* sm_count) {
    if (!rt || worker < 0 || worker >= rt->W || j < 0 || j >= (int)rt->sizes.size())
        return rt_fail(ECLIP_E_INVALID_ARG, "worker / size index out of range");
    const int s = rt->stream_of(worker, j);
    if (group_mask) *group_mask = rt->pools[s].groups;
    if (stream_id) *stream_id = s;
    if (sm_count) *sm_count = rt->pools[s].sms;
    return ECLIP_OK;
}

extern "C" int eclip_rt_set_table(eclip_rt* rt, int32_t worker, int32_t n_kernels, const int32_t* kernel_sm) {
    if (!rt || worker < 0 || worker >= rt->W || n_kernels < 1 || !kernel_sm)
        return rt_fail(ECLIP_E_INVALID_ARG, "bad table arguments");
    std::vector<int32_t> t(n_kernels);
    for (int k = 0; k < n_kernels; k++) {
        auto it = std::find(rt->sizes.begin(), rt->sizes.end(), kernel_sm[k]);
        if (it == rt->sizes.end())
            return rt_fail(ECLIP_E_INVALID_ARG, "kernel %d: %d SMs is not a pool size of this runtime", k, kernel_sm[k]);
        t[k] = (int32_t)(it - rt->sizes.begin());
    }
    rt->ws[worker].table = t;
    return ECLIP_OK;
}

extern "C" int eclip_rt_dispatch(eclip_rt* rt, int32_t worker, int32_t kernel, void** stream, int32_t* barrier) {
    if (!rt || worker < 0 || worker >= rt->W) return rt_fail(ECLIP_E_INVALID_ARG, "worker out of range");
    WorkerState& w = rt->ws[worker];
    if (kernel < 0 || kernel >= (int)w.table.size()) return rt_fail(ECLIP_E_INVALID_ARG, "kernel not in the lookup table");
    const int sid = rt->stream_of(worker, w.table[kernel]);
    cudaStream_t s = rt->pools[sid].stream;
    int b = 0;
    if (w.prev_ev && w.prev_stream != sid) {   // (i) dependency on the previous kernel of the user stream
        const cudaError_t q = cudaEventQuery(w.prev_ev);
        if (q == cudaErrorNotReady) {          // (ii) not completed: barrier packet
            RT_CU(cudaStreamWaitEvent(s, w.prev_ev, 0));
            b = 1;
        } else if (q != cudaSuccess) {
            RT_CU(q);
        }
    }
    w.cur_stream = sid;
    w.cur = s;
    if (stream) *stream = (void*)s;
    if (barrier) *barrier = b;
    return ECLIP_OK;
}

extern "C" int eclip_rt_signal(eclip_rt* rt, int32_t worker) {
    if (!rt || worker < 0 || worker >= rt->W) return rt_fail(ECLIP_E_INVALID_ARG, "worker out of range");
    WorkerState& w = rt->ws[worker];
    if (w.cur_stream < 0) return rt_fail(ECLIP_E_INVALID_ARG, "signal without dispatch");
    cudaEvent_t e = w.ring[w.ring_pos];
    w.ring_pos = (w.ring_pos + 1) % (int)w.ring.size();
    RT_CU(cudaEventRecord(e, w.cur));
    w.prev_ev = e;
    w.prev_stream = w.cur_stream;
    return ECLIP_OK;
}

static int check_model(const eclip_rt_model* m) {
    if (!m || m->n_kernels < 1 || !m->ctas || !m->iters) return rt_fail(ECLIP_E_INVALID_ARG, "bad model");
    for (int k = 0; k < m->n_kernels; k++)
        if (m->ctas[k] < 1 || m->iters[k] < 1) return rt_fail(ECLIP_E_INVALID_ARG, "model kernel %d: ctas, iters >= 1", k);
    return ECLIP_OK;
}

extern "C" int eclip_rt_profile(eclip_rt* rt, const eclip_rt_model* model, int32_t reps, double* exec_ns) {
    if (!rt || !exec_ns || reps < 1) return rt_fail(ECLIP_E_INVALID_ARG, "bad profile arguments");
    int rc = check_model(model);
    if (rc) return rc;
    RT_CU(cudaSetDevice(rt->device));
    const int J = (int)rt->sizes.size();
    cudaEvent_t a, b;
    RT_CU(cudaEventCreate(&a));
    RT_CU(cudaEventCreate(&b));
    std::vector<float> t(reps);
    for (int j = 0; j < J; j++) {
        cudaStream_t s = rt->pools[rt->stream_of(0, j)].stream;
        for (int k = 0; k < model->n_kernels; k++) {
            k_spin<<<model->ctas[k], SPIN_THREADS, SPIN_SMEM, s>>>(model->iters[k], nullptr);   // warm-up
            for (int r = 0; r < reps; r++) {
                RT_CU(cudaEventRecord(a, s));
                k_spin<<<model->ctas[k], SPIN_THREADS, SPIN_SMEM, s>>>(model->iters[k], nullptr);
                RT_CU(cudaEventRecord(b, s));
                RT_CU(cudaEventSynchronize(b));
                RT_CU(cudaEventElapsedTime(&t[r], a, b));
            }
            std::sort(t.begin(), t.end());
            exec_ns[(size_t)k * J + j] = (double)t[reps / 2] * 1e6;
        }
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ECLIP_OK;
}

extern "C" int eclip_rt_run(eclip_rt* rt, const eclip_rt_model* models, int32_t n_requests, int32_t flags,
                            eclip_rt_run_out* out) {
    if (!rt || !models || !out || n_requests < 1 || !out->latency_ns) return rt_fail(ECLIP_E_INVALID_ARG, "bad run arguments");
    const int W = rt->W;
    int Kmax = 0;
    for (int w = 0; w < W; w++) {
        int rc = check_model(&models[w]);
        if (rc) return rc;
        if ((int)rt->ws[w].table.size() < models[w].n_kernels)
            return rt_fail(ECLIP_E_INVALID_ARG, "worker %d: lookup table does not cover its model", w);
        Kmax = std::max(Kmax, models[w].n_kernels);
    }
    const bool rec = (flags & ECLIP_RT_RECORD) != 0, repart = (flags & ECLIP_RT_REPARTITION) != 0;
    if (rec && !(out->t_start && out->t_end && out->stream_id && out->barrier && out->sm_used && out->sm_mask))
        return rt_fail(ECLIP_E_INVALID_ARG, "ECLIP_RT_RECORD needs every record array");
    RT_CU(cudaSetDevice(rt->device));
    const size_t nrec = (size_t)W * n_requests * Kmax;
    KRec* d_rec = nullptr;
    if (rec) {
        RT_CU(cudaMalloc(&d_rec, nrec * sizeof(KRec)));
        std::vector<KRec> init(nrec);
        for (auto& r : init) { std::memset(&r, 0, sizeof r); r.t0 = ~0ull; }
        RT_CU(cudaMemcpy(d_rec, init.data(), nrec * sizeof(KRec), cudaMemcpyHostToDevice));
        std::fill(out->barrier, out->barrier + nrec, 0);
        std::fill(out->stream_id, out->stream_id + nrec, -2);
    }
    for (auto& w : rt->ws) { w.prev_ev = nullptr; w.prev_stream = -1; w.cur_stream = -1; }
    RT_CU(cudaDeviceSynchronize());
    std::atomic<int> ready{0}, errs{0}, nbar{0};
    std::atomic<long long> rep_ns{0};
    std::string err0;
    std::mutex emu;
    using clk = std::chrono::steady_clock;
    clk::time_point t_begin;
    std::vector<clk::time_point> t_done(W);
    auto worker = [&](int w) {
        cudaSetDevice(rt->device);
        const eclip_rt_model& m = models[w];
        const int K = m.n_kernels;
        WorkerState& st = rt->ws[w];
        auto fail_w = [&](const char* what, cudaError_t e) {
            std::lock_guard<std::mutex> g(emu);
            if (errs++ == 0) err0 = std::string(what) + ": " + cudaGetErrorString(e);
        };
        ready++;
        while (ready.load() < W) std::this_thread::yield();
        if (w == 0) t_begin = clk::now();
        std::vector<Pool> fresh;   // ECLIP_RT_REPARTITION: partitions created on the fly
        for (int r = 0; r < n_requests && errs.load() == 0; r++) {
            const auto t0 = clk::now();
            int cur_j = -1;
            cudaStream_t rs = nullptr;
            for (int k = 0; k < K; k++) {
                cudaStream_t s;
                int b = 0, sid;
                if (!repart) {
                    void* sp;
                    if (eclip_rt_dispatch(rt, w, k, &sp, &b) != ECLIP_OK) { fail_w("dispatch", cudaErrorUnknown); return; }
                    s = (cudaStream_t)sp;
                    sid = st.cur_stream;
                } else {
                    // repartition on every switch: a fresh partition for the new size (the IOCTL path);
                    // a stream switch still needs the dependency (an event wait)
                    const int j = st.table[k];
                    if (j != cur_j) {
                        const auto c0 = clk::now();
                        Pool p;
                        if (j < rt->G - 1) {
                            if (rt->make_green(rt->mask_of(w, j), &p) != ECLIP_OK) { fail_w("green context", cudaErrorUnknown); return; }
                        } else {
                            p.stream = rt->pools[rt->stream_of(w, j)].stream;
                        }
                        rep_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(clk::now() - c0).count();
                        if (rs && st.prev_ev) {
                            cudaError_t e = cudaStreamWaitEvent(p.stream, st.prev_ev, 0);
                            if (e != cudaSuccess) { fail_w("wait", e); return; }
                            b = 1;
                        }
                        fresh.push_back(p);
                        rs = p.stream;
                        cur_j = j;
                    }
                    s = rs;
                    sid = -1;
                    st.cur = s;
                    st.cur_stream = 1000000 + (int)fresh.size();
                }
                KRec* kr = rec ? d_rec + ((size_t)w * n_requests + r) * Kmax + k : nullptr;
                k_spin<<<m.ctas[k], SPIN_THREADS, SPIN_SMEM, s>>>(m.iters[k], kr);
                cudaError_t e = cudaGetLastError();
                if (e != cudaSuccess) { fail_w("launch", e); return; }
                if (eclip_rt_signal(rt, w) != ECLIP_OK) { fail_w("signal", cudaErrorUnknown); return; }
                if (rec) {
                    const size_t i = ((size_t)w * n_requests + r) * Kmax + k;
                    out->stream_id[i] = sid;
                    out->barrier[i] = b;
                }
                nbar += b;
            }
            cudaError_t e = cudaEventSynchronize(st.prev_ev);
            if (e != cudaSuccess) { fail_w("sync", e); return; }
            out->latency_ns[(size_t)w * n_requests + r] =
                std::chrono::duration_cast<std::chrono::nanoseconds>(clk::now() - t0).count();
            for (Pool& p : fresh)
                if (p.ctx) { rt->drv.StreamDestroy((CUstream)p.stream); rt->drv.GreenCtxDestroy(p.ctx); }
            fresh.clear();
        }
        t_done[w] = clk::now();
    };
    std::vector<std::thread> th;
    for (int w = 0; w < W; w++) th.emplace_back(worker, w);
    for (auto& t : th) t.join();
    if (errs.load()) {
        if (d_rec) cudaFree(d_rec);
        return rt_fail(ECLIP_E_CUDA, "runtime worker failed: %s", err0.c_str());
    }
    clk::time_point t_end = t_done[0];
    for (auto& t : t_done) t_end = std::max(t_end, t);
    out->wall_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t_end - t_begin).count();
    out->repartition_ns = rep_ns.load();
    out->barriers = nbar.load();
    if (rec) {
        std::vector<KRec> h(nrec);
        RT_CU(cudaMemcpy(h.data(), d_rec, nrec * sizeof(KRec), cudaMemcpyDeviceToHost));
        cudaFree(d_rec);
        for (size_t i = 0; i < nrec; i++) {
            out->t_start[i] = (int64_t)h[i].t0;
            out->t_end[i] = (int64_t)h[i].t1;
            int c = 0;
            for (int q = 0; q < 5; q++) { out->sm_mask[i * 5 + q] = h[i].sm[q]; c += __builtin_popcount(h[i].sm[q]); }
            out->sm_used[i] = c;
        }
    }
    return ECLIP_OK;
}
