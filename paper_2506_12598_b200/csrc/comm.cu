// comm.cu — the multi-GPU exchange of a sharded plan.
//
// A sharded plan (every rank scores its part of the candidate space) needs three per-problem
// exchanges, all tiny (4-32 B per problem) and latency-bound:
//   pass 1   FP32 filter minima                         -> global MIN
//   pass 2a  exact minimum key (256-bit)                -> global lexicographic MIN
//   pass 2b  lowest qualifying level tuple (packed, 256-bit, its order is the index order) -> lexicographic MIN
// Each is one all-gather of the per-rank values on the planning stream followed by a reduction
// kernel that every rank runs on the gathered values (so every rank holds the same global value in
// device memory, no host round trip).  The all-gather is NCCL's (one process per GPU, NVLink /
// NVSwitch; NCCL is loaded with dlopen so the process shares whatever libnccl.so.2 torch loaded),
// or, for tests on one GPU, a local group of communicators in one process (one host thread per
// rank, device-to-device copies ordered by CUDA events).
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/eclip.h"
#include "engine.h"

namespace eclip {
int set_error(int code, const char* msg);
}

using namespace eclip;

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        // reuse the libnccl.so.2 already in the process (torch's), else load it
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) { a.why = dlerror() ? dlerror() : "dlopen(libnccl.so.2) failed"; return; }
        a.getUniqueId = (decltype(a.getUniqueId))dlsym(h, "ncclGetUniqueId");
        a.commInitRank = (decltype(a.commInitRank))dlsym(h, "ncclCommInitRank");
        a.allGather = (decltype(a.allGather))dlsym(h, "ncclAllGather");
        a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
        a.errorString = (decltype(a.errorString))dlsym(h, "ncclGetErrorString");
        a.ok = a.getUniqueId && a.commInitRank && a.allGather && a.commDestroy && a.errorString;
        if (!a.ok) a.why = "libnccl.so.2 lacks an expected symbol";
    });
    return a;
}

int nccl_fail(const char* what, ncclResult_t r) {
    std::string m = std::string("NCCL ") + what + ": " + (nccl().errorString ? nccl().errorString(r) : "error");
    return set_error(ECLIP_E_CUDA, m.c_str());
}

// a group of communicators inside one process (tests: several ranks on one GPU, one host thread each)
struct LocalGroup {
    int n = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long gen = 0;
    std::vector<const void*> send;
    std::vector<cudaEvent_t> ready, done;
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const unsigned long g = gen;
        if (++arrived == n) {
            arrived = 0;
            gen++;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
    ~LocalGroup() {
        for (cudaEvent_t e : ready) if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : done) if (e) cudaEventDestroy(e);
    }
};

}  // namespace

struct eclip_comm {
    int rank = 0, size = 1, device = 0;
    ncclComm_t nc = nullptr;
    std::shared_ptr<LocalGroup> local;
    unsigned char* recv = nullptr;   // gather buffer [size][bytes] (grown on demand, stream-ordered)
    size_t recv_cap = 0;
    cudaStream_t recv_st = nullptr;
    ~eclip_comm() {
        if (recv) cudaFree(recv);
        if (nc && nccl().commDestroy) nccl().commDestroy(nc);
    }
};

// ------------------------------------------------------------------------------------------
// reductions over the gathered per-rank values (every rank runs them on identical inputs)
// ------------------------------------------------------------------------------------------
__global__ void k_gather_min_f32(const float* g, int ranks, int n, float* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        float m = g[i];
        for (int r = 1; r < ranks; r++) m = fminf(m, g[(size_t)r * n + i]);
        out[i] = m;
    }
}

__global__ void k_gather_lexmin_u256(const U256* g, int ranks, int n, U256* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        U256 m = g[i];
        for (int r = 1; r < ranks; r++) {
            const U256 v = g[(size_t)r * n + i];
            if (u256_cmp(v, m) < 0) m = v;
        }
        out[i] = m;
    }
}

namespace eclip {

// all-gather `bytes` from every rank into the communicator's gather buffer; returns it
static int comm_allgather(eclip_comm* c, const void* send, size_t bytes, cudaStream_t st, unsigned char** out) {
    const size_t need = bytes * (size_t)c->size;
    if (need > c->recv_cap) {
        if (c->recv) { cudaStreamSynchronize(st); cudaFree(c->recv); c->recv = nullptr; c->recv_cap = 0; }
        cudaError_t e = cudaMalloc((void**)&c->recv, need);
        if (e != cudaSuccess) return set_error(ECLIP_E_OOM, "comm gather buffer");
        c->recv_cap = need;
    }
    if (c->nc) {
        ncclResult_t r = nccl().allGather(send, c->recv, bytes, ncclUint8, c->nc, st);
        if (r != ncclSuccess) return nccl_fail("all-gather", r);
    } else {
        LocalGroup& g = *c->local;
        g.send[c->rank] = send;
        if (cudaEventRecord(g.ready[c->rank], st) != cudaSuccess) return set_error(ECLIP_E_CUDA, "event record");
        g.barrier();
        for (int r = 0; r < c->size; r++) {
            cudaStreamWaitEvent(st, g.ready[r], 0);
            cudaMemcpyAsync(c->recv + (size_t)r * bytes, g.send[r], bytes, cudaMemcpyDeviceToDevice, st);
        }
        cudaEventRecord(g.done[c->rank], st);
        g.barrier();
        for (int r = 0; r < c->size; r++) cudaStreamWaitEvent(st, g.done[r], 0);   // peers read my send buffer
        if (cudaGetLastError() != cudaSuccess) return set_error(ECLIP_E_CUDA, "local all-gather");
    }
    *out = c->recv;
    return ECLIP_OK;
}

int comm_min_f32(eclip_comm* c, float* buf, int n, cudaStream_t st) {
    if (c->size == 1 && !c->nc) return ECLIP_OK;
    unsigned char* g;
    int rc = comm_allgather(c, buf, sizeof(float) * (size_t)n, st, &g);
    if (rc) return rc;
    k_gather_min_f32<<<(n + 255) / 256, 256, 0, st>>>((const float*)g, c->size, n, buf);
    return cudaGetLastError() == cudaSuccess ? ECLIP_OK : set_error(ECLIP_E_CUDA, "k_gather_min_f32");
}

int comm_lexmin_u256(eclip_comm* c, U256* buf, int n, cudaStream_t st) {
    if (c->size == 1 && !c->nc) return ECLIP_OK;
    unsigned char* g;
    int rc = comm_allgather(c, buf, sizeof(U256) * (size_t)n, st, &g);
    if (rc) return rc;
    k_gather_lexmin_u256<<<(n + 127) / 128, 128, 0, st>>>((const U256*)g, c->size, n, buf);
    return cudaGetLastError() == cudaSuccess ? ECLIP_OK : set_error(ECLIP_E_CUDA, "k_gather_lexmin_u256");
}

int comm_rank(const eclip_comm* c) { return c->rank; }
int comm_size(const eclip_comm* c) { return c->size; }
int comm_device(const eclip_comm* c) { return c->device; }

}  // namespace eclip

// ------------------------------------------------------------------------------------------
// C-ABI
// ------------------------------------------------------------------------------------------
extern "C" int eclip_comm_unique_id(uint8_t* id) {
    if (!id) return set_error(ECLIP_E_INVALID_ARG, "null id");
    NcclApi& a = nccl();
    if (!a.ok) return set_error(ECLIP_E_CUDA, ("NCCL unavailable: " + a.why).c_str());
    ncclUniqueId u;
    ncclResult_t r = a.getUniqueId(&u);
    if (r != ncclSuccess) return nccl_fail("get unique id", r);
    memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    return ECLIP_OK;
}

extern "C" int eclip_comm_create(const uint8_t* id, int32_t n_ranks, int32_t rank, int32_t device, eclip_comm** out) {
    if (!id || !out || n_ranks < 1 || rank < 0 || rank >= n_ranks || device < 0)
        return set_error(ECLIP_E_INVALID_ARG, "bad arguments to eclip_comm_create");
    NcclApi& a = nccl();
    if (!a.ok) return set_error(ECLIP_E_CUDA, ("NCCL unavailable: " + a.why).c_str());
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device >= ndev)
        return set_error(ECLIP_E_CUDA, "no such CUDA device for the communicator");
    if (cudaSetDevice(device) != cudaSuccess) return set_error(ECLIP_E_CUDA, "cudaSetDevice");
    auto c = std::make_unique<eclip_comm>();
    c->rank = rank; c->size = n_ranks; c->device = device;
    ncclUniqueId u;
    memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    ncclResult_t r = a.commInitRank(&c->nc, n_ranks, u, rank);
    if (r != ncclSuccess) { c->nc = nullptr; return nccl_fail("comm init", r); }
    *out = c.release();
    return ECLIP_OK;
}

extern "C" int eclip_comm_create_local(int32_t n_ranks, int32_t device, eclip_comm** comms) {
    if (!comms || n_ranks < 1 || device < 0) return set_error(ECLIP_E_INVALID_ARG, "bad arguments to eclip_comm_create_local");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device >= ndev)
        return set_error(ECLIP_E_CUDA, "no such CUDA device for the communicator");
    if (cudaSetDevice(device) != cudaSuccess) return set_error(ECLIP_E_CUDA, "cudaSetDevice");
    auto g = std::make_shared<LocalGroup>();
    g->n = n_ranks;
    g->send.assign(n_ranks, nullptr);
    g->ready.assign(n_ranks, nullptr);
    g->done.assign(n_ranks, nullptr);
    for (int r = 0; r < n_ranks; r++)
        if (cudaEventCreateWithFlags(&g->ready[r], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&g->done[r], cudaEventDisableTiming) != cudaSuccess)
            return set_error(ECLIP_E_CUDA, "event create");
    for (int r = 0; r < n_ranks; r++) {
        eclip_comm* c = new eclip_comm();
        c->rank = r; c->size = n_ranks; c->device = device; c->local = g;
        comms[r] = c;
    }
    return ECLIP_OK;
}

extern "C" int eclip_comm_info(const eclip_comm* c, int32_t* rank, int32_t* size, int32_t* device) {
    if (!c) return set_error(ECLIP_E_INVALID_ARG, "null communicator");
    if (rank) *rank = c->rank;
    if (size) *size = c->size;
    if (device) *device = c->device;
    return ECLIP_OK;
}

extern "C" void eclip_comm_free(eclip_comm* c) { delete c; }
