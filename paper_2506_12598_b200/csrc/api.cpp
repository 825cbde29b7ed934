// api.cpp — the C-ABI (include/eclip.h): profile ingest, validation,
// level-table jobs, engine orchestration and result marshalling.  Every step of the
// planning path runs in the CUDA kernels of levels.cu / enum.cu / slice.cu; this file only
// prepares inputs, launches, and copies results.  There is no CPU fallback.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdarg>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <atomic>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/eclip.h"
#include "engine.h"
#include "slice.h"

using namespace eclip;

// ------------------------------------------------------------------------------------------
// errors
// ------------------------------------------------------------------------------------------
static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

namespace eclip {
// the same thread-local message for the other translation units (runtime.cu)
int set_error(int code, const char* msg) {
    g_err = msg;
    return code;
}
}  // namespace eclip

#define CU(x)                                                                                       \
    do {                                                                                            \
        cudaError_t _e = (x);                                                                       \
        if (_e != cudaSuccess) {                                                                    \
            return fail(_e == cudaErrorMemoryAllocation ? ECLIP_E_OOM : ECLIP_E_CUDA, "CUDA: %s (%s:%d)", \
                        cudaGetErrorString(_e), __FILE__, __LINE__);                                \
        }                                                                                           \
    } while (0)

extern "C" const char* eclip_last_error(void) { return g_err.c_str(); }
extern "C" const char* eclip_version(void) { return "eclip-b200 0.1 (sm_100a)"; }

// ------------------------------------------------------------------------------------------
// profiles
// ------------------------------------------------------------------------------------------
struct eclip_profiles {
    std::vector<std::string> names;
    std::vector<int32_t> sizes;
    std::vector<int32_t> nk;
    std::vector<int64_t> row0;   // first row of each model
    std::vector<int64_t> exec;   // [sum nk][C]
    int C() const { return (int)sizes.size(); }
    int n() const { return (int)nk.size(); }
    const int64_t* row(int m, int k) const { return exec.data() + (size_t)(row0[m] + k) * sizes.size(); }
};

// decimal microseconds -> integer ns, round half to even
static bool us_to_ns(const std::string& cell, int64_t* out) {
    size_t i = 0, n = cell.size();
    while (i < n && isspace((unsigned char)cell[i])) i++;
    while (n > i && isspace((unsigned char)cell[n - 1])) n--;
    if (i >= n) return false;
    bool neg = false;
    if (cell[i] == '+' || cell[i] == '-') { neg = cell[i] == '-'; i++; }
    std::string ip, fp;
    while (i < n && isdigit((unsigned char)cell[i])) ip += cell[i++];
    if (i < n && cell[i] == '.') {
        i++;
        while (i < n && isdigit((unsigned char)cell[i])) fp += cell[i++];
    }
    if (i != n || (ip.empty() && fp.empty())) return false;
    if (ip.size() > 12) return false;
    int64_t whole = 0;
    for (char c : ip) whole = whole * 10 + (c - '0');
    int64_t ns = whole * 1000;
    std::string f3 = fp.substr(0, std::min<size_t>(3, fp.size()));
    while (f3.size() < 3) f3 += '0';
    ns += (f3[0] - '0') * 100 + (f3[1] - '0') * 10 + (f3[2] - '0');
    // remaining digits decide rounding: > half up, == half to even
    if (fp.size() > 3) {
        std::string rest = fp.substr(3);
        int cmp;
        if (rest[0] > '5') cmp = 1;
        else if (rest[0] < '5') cmp = -1;
        else {
            cmp = 0;
            for (size_t k = 1; k < rest.size(); k++)
                if (rest[k] != '0') { cmp = 1; break; }
        }
        if (cmp > 0 || (cmp == 0 && (ns & 1))) ns += 1;
    }
    *out = neg ? -ns : ns;
    return true;
}

static int parse_profiles(const char* text, size_t len, eclip_profiles** out) {
    std::string s(text, len);
    std::istringstream in(s);
    std::string line;
    std::vector<std::string> lines;
    while (std::getline(in, line)) {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        bool blank = true;
        for (char c : line)
            if (!isspace((unsigned char)c)) { blank = false; break; }
        if (!blank) lines.push_back(line);
    }
    auto P = std::make_unique<eclip_profiles>();
    size_t i = 0;
    while (i < lines.size()) {
        // minimal JSON header parse: {"model": "...", "kernels": N, "configs": [..]}
        const std::string& h = lines[i];
        auto key = [&](const char* k) -> size_t {
            size_t p = h.find(std::string("\"") + k + "\"");
            if (p == std::string::npos) return p;
            p = h.find(':', p);
            return p == std::string::npos ? p : p + 1;
        };
        size_t pm = key("model"), pk = key("kernels"), pc = key("configs");
        if (h.find('{') == std::string::npos || pm == std::string::npos || pk == std::string::npos || pc == std::string::npos)
            return fail(ECLIP_E_PARSE, "parse failure: line %zu is not a profile header", i + 1);
        size_t q1 = h.find('"', pm), q2 = q1 == std::string::npos ? q1 : h.find('"', q1 + 1);
        if (q2 == std::string::npos) return fail(ECLIP_E_PARSE, "parse failure: bad model name on line %zu", i + 1);
        std::string name = h.substr(q1 + 1, q2 - q1 - 1);
        long nk = strtol(h.c_str() + pk, nullptr, 10);
        size_t b1 = h.find('[', pc), b2 = h.find(']', pc);
        if (nk < 1 || b1 == std::string::npos || b2 == std::string::npos)
            return fail(ECLIP_E_PARSE, "parse failure: model %s: bad kernels/configs", name.c_str());
        std::vector<int32_t> cfg;
        {
            std::string c = h.substr(b1 + 1, b2 - b1 - 1);
            std::stringstream cs(c);
            std::string tok;
            while (std::getline(cs, tok, ',')) {
                char* e = nullptr;
                long v = strtol(tok.c_str(), &e, 10);
                if (v <= 0) return fail(ECLIP_E_PARSE, "parse failure: model %s: bad config %s", name.c_str(), tok.c_str());
                cfg.push_back((int32_t)v);
            }
        }
        if (cfg.empty()) return fail(ECLIP_E_PARSE, "parse failure: model %s: empty configs", name.c_str());
        if (cfg.size() > 32) return fail(ECLIP_E_PARSE, "parse failure: model %s: more than 32 configs", name.c_str());
        if (P->sizes.empty()) P->sizes = cfg;
        else if (P->sizes != cfg)
            return fail(ECLIP_E_PARSE, "parse failure: model %s: configs differ from the first model's", name.c_str());
        for (size_t j = 1; j < cfg.size(); j++)
            if (cfg[j] <= cfg[j - 1]) return fail(ECLIP_E_PARSE, "parse failure: configs must ascend");
        if (i + 1 + (size_t)nk > lines.size())
            return fail(ECLIP_E_PARSE, "parse failure: model %s: expected %ld kernel rows", name.c_str(), nk);
        P->names.push_back(name);
        P->nk.push_back((int32_t)nk);
        P->row0.push_back((int64_t)(P->exec.size() / cfg.size()));
        for (long k = 0; k < nk; k++) {
            const std::string& r = lines[i + 1 + k];
            std::vector<std::string> cells;
            std::stringstream rs(r);
            std::string tok;
            while (std::getline(rs, tok, ',')) cells.push_back(tok);
            if (cells.size() != cfg.size() + 1)
                return fail(ECLIP_E_MISSING_CONFIG, "missing config column: model %s, kernel %ld", name.c_str(), k);
            std::vector<int64_t> row;
            for (size_t j = 1; j < cells.size(); j++) {
                int64_t v;
                if (!us_to_ns(cells[j], &v))
                    return fail(ECLIP_E_PARSE, "parse failure: model %s, kernel %ld: not a decimal: %s", name.c_str(), k,
                                cells[j].c_str());
                if (v <= 0) return fail(ECLIP_E_NONMONOTONE, "non-positive exec_time: model %s, kernel %ld", name.c_str(), k);
                row.push_back(v);
            }
            for (size_t j = 0; j + 1 < row.size(); j++)
                if (row[j] < row[j + 1])
                    return fail(ECLIP_E_NONMONOTONE, "non-monotone exec_time: model %s, kernel %ld", name.c_str(), k);
            P->exec.insert(P->exec.end(), row.begin(), row.end());
        }
        i += 1 + nk;
    }
    if (P->nk.empty()) return fail(ECLIP_E_PARSE, "parse failure: empty profile file");
    *out = P.release();
    return ECLIP_OK;
}

extern "C" int eclip_load_profiles_mem(const char* text, size_t len, eclip_profiles** out) {
    if (!text || !out) return fail(ECLIP_E_INVALID_ARG, "null argument");
    return parse_profiles(text, len, out);
}

extern "C" int eclip_load_profiles(const char* path, eclip_profiles** out) {
    if (!path || !out) return fail(ECLIP_E_INVALID_ARG, "null argument");
    std::ifstream f(path, std::ios::binary);
    if (!f) return fail(ECLIP_E_IO, "cannot read %s: %s", path, strerror(errno));
    std::stringstream ss;
    ss << f.rdbuf();
    std::string s = ss.str();
    return parse_profiles(s.data(), s.size(), out);
}

extern "C" int eclip_profiles_from_arrays(int32_t n_models, const int32_t* n_kernels, int32_t n_sizes,
                                          const int32_t* sizes_sm, const int64_t* exec_ns, eclip_profiles** out) {
    if (n_models < 1 || !n_kernels || n_sizes < 1 || n_sizes > 32 || !sizes_sm || !exec_ns || !out)
        return fail(ECLIP_E_INVALID_ARG, "bad arguments to eclip_profiles_from_arrays");
    auto P = std::make_unique<eclip_profiles>();
    P->sizes.assign(sizes_sm, sizes_sm + n_sizes);
    for (int j = 0; j < n_sizes; j++) {
        if (sizes_sm[j] <= 0) return fail(ECLIP_E_INVALID_ARG, "size %d is not positive", j);
        if (j && sizes_sm[j] <= sizes_sm[j - 1]) return fail(ECLIP_E_INVALID_ARG, "sizes must ascend");
    }
    int64_t r = 0;
    for (int m = 0; m < n_models; m++) {
        if (n_kernels[m] < 1) return fail(ECLIP_E_INVALID_ARG, "model %d has no kernels", m);
        P->names.push_back("model" + std::to_string(m));
        P->nk.push_back(n_kernels[m]);
        P->row0.push_back(r);
        for (int k = 0; k < n_kernels[m]; k++, r++) {
            const int64_t* row = exec_ns + (size_t)r * n_sizes;
            for (int j = 0; j < n_sizes; j++) {
                if (row[j] <= 0) return fail(ECLIP_E_NONMONOTONE, "non-positive exec_time: model %d, kernel %d", m, k);
                if (j && row[j - 1] < row[j]) return fail(ECLIP_E_NONMONOTONE, "non-monotone exec_time: model %d, kernel %d", m, k);
            }
            P->exec.insert(P->exec.end(), row, row + n_sizes);
        }
    }
    *out = P.release();
    return ECLIP_OK;
}

extern "C" void eclip_free_profiles(eclip_profiles* p) { delete p; }

extern "C" int eclip_profiles_info(const eclip_profiles* p, int32_t* n_models, int32_t* n_sizes, int32_t* sizes_sm,
                                   int32_t* n_kernels, int64_t* exec_ns, char* names, size_t names_cap) {
    if (!p) return fail(ECLIP_E_INVALID_ARG, "null profiles");
    if (n_models) *n_models = p->n();
    if (n_sizes) *n_sizes = p->C();
    if (sizes_sm) std::copy(p->sizes.begin(), p->sizes.end(), sizes_sm);
    if (n_kernels) std::copy(p->nk.begin(), p->nk.end(), n_kernels);
    if (exec_ns) std::copy(p->exec.begin(), p->exec.end(), exec_ns);
    if (names && names_cap) {
        std::string all;
        for (auto& s : p->names) all += s + "\n";
        size_t n = std::min(all.size(), names_cap - 1);
        memcpy(names, all.data(), n);
        names[n] = 0;
    }
    return ECLIP_OK;
}

extern "C" void eclip_default_options(eclip_options* o) {
    memset(o, 0, sizeof(*o));
    o->engine = ECLIP_ENGINE_AUTO;
    o->device = 0;
    o->cuda_stream = nullptr;
    o->tie_tol = 1e-5;
    o->shard = 0;
    o->n_shards = 1;
}

// ------------------------------------------------------------------------------------------
// level tables (host descriptions; built on the GPU by K1)
// ------------------------------------------------------------------------------------------
struct TableSpec {
    int model;
    std::vector<int32_t> bounds;  // kernel offsets (G+1)
    uint32_t mask;
    int R;
    bool operator<(const TableSpec& o) const {
        return std::tie(model, bounds, mask, R) < std::tie(o.model, o.bounds, o.mask, o.R);
    }
};

struct HostTable {
    int G, C, Reff, smax, Lcap;
    int64_t u, K;
    uint32_t mask;
    std::vector<int64_t> beta;  // [G*C]
    std::vector<int32_t> need;  // [G*C]
    size_t v_elems;
};

static int64_t gcd64(int64_t a, int64_t b) {
    while (b) { int64_t t = a % b; a = b; b = t; }
    return a;
}

static int build_host_table(const eclip_profiles* P, const TableSpec& sp, HostTable* t) {
    const int C = P->C();
    const int G = (int)sp.bounds.size() - 1;
    t->G = G; t->C = C; t->mask = sp.mask;
    t->Reff = std::min(sp.R, G - 1);
    t->beta.assign((size_t)G * C, 0);
    t->need.assign((size_t)G * C, 0);
    int64_t u = 0;
    for (int j = 0; j < C; j++)
        if ((sp.mask >> j) & 1u) u = gcd64(u, P->sizes[j]);
    t->u = u;
    int64_t smax = 0, bmax = 0;
    for (int g = 0; g < G; g++) {
        int64_t ng = sp.bounds[g + 1] - sp.bounds[g];
        int64_t mx = 0, bm = 0;
        for (int j = 0; j < C; j++) {
            int64_t b = 0;
            for (int k = sp.bounds[g]; k < sp.bounds[g + 1]; k++) b += P->row(sp.model, k)[j];
            t->beta[(size_t)g * C + j] = b;
            if ((sp.mask >> j) & 1u) {
                t->need[(size_t)g * C + j] = (int32_t)(ng * P->sizes[j] / u);
                mx = std::max<int64_t>(mx, t->need[(size_t)g * C + j]);
                bm = std::max<int64_t>(bm, b);
            }
        }
        smax += mx;
        bmax += bm;
    }
    if (bmax >= ((int64_t)1 << 36))
        return fail(ECLIP_E_TOO_LARGE, "model %d: solo request time %lld ns exceeds 2^36 ns", sp.model, (long long)bmax);
    if (smax > (1 << 22)) return fail(ECLIP_E_TOO_LARGE, "model %d: CU-sum range too large", sp.model);
    if ((double)G * C * (std::min(sp.R, G - 1) + 1) * (smax + 1) >= 2147483647.0)
        return fail(ECLIP_E_TOO_LARGE, "model %d: level-DP state space exceeds 2^31", sp.model);
    t->smax = (int)smax;
    t->K = sp.bounds.back();
    t->Lcap = (int)smax + 1;
    t->v_elems = (size_t)G * C * (t->Reff + 1) * (smax + 1);
    return ECLIP_OK;
}

// ------------------------------------------------------------------------------------------
// device allocation helpers (stream-ordered)
// ------------------------------------------------------------------------------------------
struct DevArena {
    cudaStream_t st = nullptr;
    std::vector<void*> ptrs;
    template <class T>
    cudaError_t alloc(T** p, size_t n) {
        void* q = nullptr;
        cudaError_t e = cudaMallocAsync(&q, std::max<size_t>(n, 1) * sizeof(T), st);
        if (e == cudaSuccess) ptrs.push_back(q);
        *p = (T*)q;
        return e;
    }
    void release() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
        ptrs.clear();
    }
    ~DevArena() { release(); }
};

// ------------------------------------------------------------------------------------------
// the session: everything one planning call needs on the device
// ------------------------------------------------------------------------------------------
struct eclip_session {
    const eclip_profiles* prof = nullptr;
    cudaStream_t st = nullptr;
    bool own_stream = false;
    bool keep_stream = false;            // own_stream shared by the thread's sessions (not destroyed)
    int device = 0;
    DevArena arena;
    // problem description
    Setup su{};
    int W = 0, n = 0, C = 0;
    bool on_device = false;
    std::vector<HostTable> tabs;
    std::vector<int32_t> tabL;
    std::vector<int32_t> tabG;
    std::vector<int32_t> h_table_of;     // host copy (single-problem path)
    int32_t* d_sizes = nullptr;
    Tables tb{};
    Work wk{};
    PrepIn pin{};
    int engine = ECLIP_ENGINE_ENUM;
    int gmax = 0;
    uint64_t scored_local = 0;
    eclip_comm* comm = nullptr;          // in-library exchange of a sharded plan (opt->comm)
    SliceState slice;
    ~eclip_session() {
        slice.release();
        arena.release();
        for (cudaEvent_t& e : wk.kev)
            if (e) cudaEventDestroy(e);
        if (own_stream && st) {
            cudaStreamSynchronize(st);
            if (!keep_stream) cudaStreamDestroy(st);
        }
    }
};

static int setup_device(eclip_session* s, const eclip_options* opt) {
    s->device = opt ? opt->device : 0;
    if (opt && opt->comm) {   // the communicator fixes the device and the shard
        s->comm = (eclip_comm*)opt->comm;
        s->device = comm_device(s->comm);
    }
    // device count and the pool setting are queried once per process (per device)
    static int ndev = -1;
    static cudaError_t ndev_err = cudaSuccess;
    static std::once_flag once;
    std::call_once(once, [] { ndev_err = cudaGetDeviceCount(&ndev); });
    if (ndev_err != cudaSuccess || ndev <= 0)
        return fail(ECLIP_E_CUDA, "no CUDA device available (%s); the planner has no CPU fallback",
                    ndev_err == cudaSuccess ? "0 devices" : cudaGetErrorString(ndev_err));
    if (s->device < 0 || s->device >= ndev) return fail(ECLIP_E_INVALID_ARG, "device %d out of range", s->device);
    CU(cudaSetDevice(s->device));
    static std::atomic<uint64_t> pool_set{0};   // bit d: device d's pool configured
    if (s->device < 64 && !((pool_set.load() >> s->device) & 1ull)) {
        // keep freed workspace in the device's stream-ordered pool between calls (no re-mapping)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, s->device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        pool_set.fetch_or(1ull << s->device);
    }
    if (opt && opt->cuda_stream) {
        s->st = (cudaStream_t)opt->cuda_stream;
    } else if (!s->comm && s->device < 64) {
        // the library's own stream: one per (host thread, device), created once and kept (a stream per call costs
        // more than the small plans it serves); sessions of a communicator group get their own (their collectives
        // must not queue behind each other)
        static thread_local cudaStream_t cached[64] = {};
        if (!cached[s->device]) CU(cudaStreamCreateWithFlags(&cached[s->device], cudaStreamNonBlocking));
        s->st = cached[s->device];
        s->own_stream = true;
        s->keep_stream = true;
    } else {
        CU(cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking));
        s->own_stream = true;
    }
    s->arena.st = s->st;
    for (cudaEvent_t& e : s->wk.kev) CU(cudaEventCreate(&e));
    return ECLIP_OK;
}

// One device block carved into 256-byte aligned pieces (one cudaMallocAsync instead of dozens).
struct Bump {
    size_t off = 0;
    template <class T>
    size_t take(size_t n) {
        const size_t o = off;
        off = (off + std::max<size_t>(n, 1) * sizeof(T) + 255) & ~(size_t)255;
        return o;
    }
};

// Build tables with K1 on the GPU and fetch their level counts.  Inputs (group times, level
// steps, job descriptors, table views) are packed host-side into the front of one device block
// and sent with a single copy; the K1 workspaces and outputs follow in the same block.
static int build_tables(eclip_session* s, const std::vector<TableSpec>& specs) {
    const eclip_profiles* P = s->prof;
    s->tabs.resize(specs.size());
    for (size_t i = 0; i < specs.size(); i++) {
        int rc = build_host_table(P, specs[i], &s->tabs[i]);
        if (rc) return rc;
    }
    host_mark("host tables");
    const int nt = (int)specs.size();
    struct Off { size_t beta, need, V, best, barg, bstar, sidx, wtmp, outS, outB, outW; };
    std::vector<Off> off(nt);
    Bump bp;
    for (int i = 0; i < nt; i++) {   // inputs first (the copied prefix)
        off[i].beta = bp.take<int64_t>(s->tabs[i].beta.size());
        off[i].need = bp.take<int32_t>(s->tabs[i].need.size());
    }
    const size_t o_jobs = bp.take<LevelJob>(nt), o_K = bp.take<int64_t>(nt), o_G = bp.take<int32_t>(nt);
    const size_t o_S = bp.take<int64_t*>(nt), o_B = bp.take<int64_t*>(nt), o_W = bp.take<uint8_t*>(nt);
    const size_t o_beta = bp.take<int64_t*>(nt);
    const size_t in_bytes = bp.off;
    const size_t o_L = bp.take<int32_t>(nt);
    // K1 stores its layers as int32 when every table's largest plan time fits (sum over groups of the
    // slowest size < 2^31 - 1), else int64
    bool v32 = true;
    for (int i = 0; i < nt; i++) {
        const HostTable& t = s->tabs[i];
        int64_t mx = 0;
        for (int g = 0; g < t.G; g++) {
            int64_t m = 0;
            for (int j = 0; j < t.C; j++) m = std::max(m, t.beta[(size_t)g * t.C + j]);
            mx += m;
        }
        if (mx >= INT32_MAX) v32 = false;
    }
    const size_t vb = v32 ? 4 : 8;
    std::vector<int32_t> ncp(nt);
    for (int i = 0; i < nt; i++) {
        const HostTable& t = s->tabs[i];
        const size_t ns = (size_t)(t.Reff + 1) * (t.smax + 1);
        ncp[i] = (int32_t)((ns + 31) & ~(size_t)31);   // 128-byte aligned layer slabs (levels.cu)
        off[i].V = bp.take<unsigned char>((size_t)t.G * t.C * ncp[i] * vb);
        off[i].best = bp.take<unsigned char>((size_t)t.G * ncp[i] * 2 * vb);
        off[i].barg = bp.take<uint8_t>((size_t)t.G * ncp[i]);
        off[i].bstar = bp.take<int64_t>(t.smax + 1);
        off[i].sidx = bp.take<int32_t>(t.smax + 1);
        off[i].wtmp = bp.take<uint64_t>((size_t)(t.smax + 1) * ((t.G + 7) / 8));
        off[i].outS = bp.take<int64_t>(t.Lcap);
        off[i].outB = bp.take<int64_t>(t.Lcap);
        off[i].outW = bp.take<uint8_t>((size_t)t.Lcap * t.G);
    }
    unsigned char* base;
    CU(s->arena.alloc(&base, bp.off));
    std::vector<unsigned char> h(in_bytes);
    auto at = [&](size_t o) { return base + o; };
    std::vector<LevelJob> jobs(nt);
    std::vector<int64_t> hK(nt);
    std::vector<const void*> hS(nt), hB(nt), hW(nt), hbeta(nt);
    s->tabG.resize(nt);
    s->gmax = 0;
    for (int i = 0; i < nt; i++) {
        const HostTable& t = s->tabs[i];
        std::memcpy(h.data() + off[i].beta, t.beta.data(), t.beta.size() * 8);
        std::memcpy(h.data() + off[i].need, t.need.data(), t.need.size() * 4);
        LevelJob& J = jobs[i];
        J.G = t.G; J.C = t.C; J.R = t.Reff; J.smax = t.smax; J.u = t.u; J.mask = t.mask; J.Lcap = t.Lcap;
        J.beta = (const int64_t*)at(off[i].beta);
        J.need = (const int32_t*)at(off[i].need);
        J.ncp = ncp[i];
        J.V = at(off[i].V);
        J.best = at(off[i].best);
        J.barg = (uint8_t*)at(off[i].barg);
        J.bstar = (int64_t*)at(off[i].bstar);
        J.sidx = (int32_t*)at(off[i].sidx);
        J.wtmp = (uint64_t*)at(off[i].wtmp);
        J.outS = (int64_t*)at(off[i].outS);
        J.outB = (int64_t*)at(off[i].outB);
        J.outW = (uint8_t*)at(off[i].outW);
        J.outL = (int32_t*)at(o_L) + i;
        hK[i] = t.K; s->tabG[i] = t.G;
        hS[i] = J.outS; hB[i] = J.outB; hW[i] = J.outW; hbeta[i] = J.beta;
        s->gmax = std::max(s->gmax, t.G);
    }
    std::memcpy(h.data() + o_jobs, jobs.data(), sizeof(LevelJob) * nt);
    std::memcpy(h.data() + o_K, hK.data(), 8 * nt);
    std::memcpy(h.data() + o_G, s->tabG.data(), 4 * nt);
    std::memcpy(h.data() + o_S, hS.data(), 8 * nt);
    std::memcpy(h.data() + o_B, hB.data(), 8 * nt);
    std::memcpy(h.data() + o_W, hW.data(), 8 * nt);
    std::memcpy(h.data() + o_beta, hbeta.data(), 8 * nt);
    CU(cudaMemcpyAsync(base, h.data(), in_bytes, cudaMemcpyHostToDevice, s->st));
    LevelJob* djobs = (LevelJob*)at(o_jobs);
    for (int c0 = 0; c0 < nt; c0 += 64)   // K1 handles up to 64 tables per cooperative launch
        CU(launch_levels(djobs + c0, jobs.data() + c0, std::min(64, nt - c0), v32, s->st));
    int32_t* dL = (int32_t*)at(o_L);
    s->tabL.resize(nt);
    CU(cudaMemcpyAsync(s->tabL.data(), dL, 4 * nt, cudaMemcpyDeviceToHost, s->st));
    host_mark("K1 launched");
    CU(cudaStreamSynchronize(s->st));   // level counts size the enumeration
    s->tb.n = nt; s->tb.L = dL; s->tb.K = (const int64_t*)at(o_K); s->tb.G = (const int32_t*)at(o_G);
    s->tb.S = (const int64_t* const*)at(o_S); s->tb.B = (const int64_t* const*)at(o_B);
    s->tb.wit = (const uint8_t* const*)at(o_W); s->tb.beta = (const int64_t* const*)at(o_beta);
    return ECLIP_OK;
}

static int check_common(const eclip_profiles* P, int W, int N, int R, int mode, int obj, float pi, float pm,
                        double tol) {
    if (!P) return fail(ECLIP_E_INVALID_ARG, "null profiles");
    if (W < 1 || W > MAXW) return fail(ECLIP_E_INVALID_ARG, "n_models must be in [1, %d]", MAXW);
    if (N < 1) return fail(ECLIP_E_INVALID_ARG, "total_sms must be >= 1");
    if (P->sizes.back() > N) return fail(ECLIP_E_INVALID_ARG, "pool size %d exceeds total_sms %d", P->sizes.back(), N);
    if (R < 0) return fail(ECLIP_E_INVALID_ARG, "switch_max must be >= 0");
    if (mode < 0 || mode > 3) return fail(ECLIP_E_INVALID_ARG, "unknown slowdown mode %d", mode);
    if (obj < 0 || obj > 2) return fail(ECLIP_E_INVALID_ARG, "unknown objective %d", obj);
    if (!(std::isfinite(pi) && std::isfinite(pm) && pi >= 0.0f && pm >= pi))
        return fail(ECLIP_E_INVALID_ARG, "power model needs 0 <= p_idle <= p_max");
    if (!(tol >= 0.0 && tol < 1.0)) return fail(ECLIP_E_INVALID_ARG, "tie_tol must be in [0, 1)");
    return ECLIP_OK;
}

// per-worker objective weights (R20): finite, in (0, 1000], >= 5e-7 (so that
// round(omega 1e6) >= 1); ENERGY needs equal weights.  Returns whether they differ (the weighted kernels).
static int check_weights(const double* wt, size_t n, int W, int obj, bool* unequal) {
    *unequal = false;
    if (!wt) return ECLIP_OK;
    for (size_t i = 0; i < n * (size_t)W; i++) {
        if (!(wt[i] > 0.0 && wt[i] <= 1000.0) || llround(wt[i] * 1e6) < 1)
            return fail(ECLIP_E_INVALID_ARG, "weights must lie in (0, 1000] (1e-6 resolution)");
        if (llround(wt[i] * 1e6) != llround(wt[i - i % W] * 1e6)) *unequal = true;
    }
    if (*unequal && obj == ECLIP_ENERGY)
        return fail(ECLIP_E_INVALID_ARG, "the ENERGY objective takes no per-worker weights (they must be equal)");
    return ECLIP_OK;
}

static void fill_setup(eclip_session* s, int n, int W, int N, int R, int mode, int obj, bool has_qos,
                       const eclip_options* opt) {
    (void)R;
    Setup& su = s->su;
    su.n_problems = n; su.W = W; su.N = N; su.mode = mode; su.obj = obj; su.has_qos = has_qos ? 1 : 0;
    double tol = opt ? opt->tie_tol : 1e-5;
    su.tol_den = 1000000000ull;
    su.tol_num = (uint64_t)llround(tol * 1e9);
    su.delta = (double)(8 * W + 16) * std::ldexp(1.0, -24);
    su.shard = opt ? opt->shard : 0;
    su.n_shards = opt ? std::max(1, opt->n_shards) : 1;
    if (s->comm) {
        su.shard = comm_rank(s->comm);
        su.n_shards = comm_size(s->comm);
    }
    su.prune = (opt && opt->no_prune) ? 0 : 1;
}

// Narrow or wide launch (Setup::wide): Lambda = lcm of the kernel counts of the tables a problem can
// use (a batch: every table, an upper bound of each problem's Lambda); wide when Lambda N (W+1) reaches
// 2^24, the range of the narrow kernels' exact FP32 / int32 T' arithmetic.
static void set_wide(eclip_session* s, const std::vector<int32_t>& tables) {
    long double lam = 1;
    uint64_t l = 1;
    for (int t : tables) {
        const uint64_t K = (uint64_t)s->tabs[t].K;
        const uint64_t g = (uint64_t)gcd64((int64_t)l, (int64_t)K);
        lam = lam / (long double)g * (long double)K;
        l = lam < 1.8e19L ? l / g * K : l;
    }
    s->su.wide = (lam * (long double)s->su.N * (long double)(s->su.W + 1) >= 16777216.0L) ? 1 : 0;
}

// choose the engine and size the work (pass-1 geometry: see enum.cu)
static int plan_geometry(eclip_session* s, const eclip_options* opt) {
    Setup& su = s->su;
    int Lmax = 1, Lmin = 1 << 30;
    for (int L : s->tabL) {
        Lmax = std::max(Lmax, L);
        Lmin = std::min(Lmin, std::max(L, 1));
    }
    su.Lmax = Lmax;
    const int W = su.W;
    const long double n = su.n_problems;
    long double H = 1;
    for (int w = 0; w < W - 2; w++) H *= Lmax;
    long double tuples = H * (W >= 2 ? Lmax : 1) * Lmax;
    int want = opt ? opt->engine : ECLIP_ENGINE_AUTO;
    bool enum_ok = W <= MAXW_ENUM && (size_t)W * Lmax * sizeof(Lev) <= 100 * 1024 && tuples < 4e18L && Lmax <= 4096 &&
                   n * H * 4 < 6e9L;
    bool slice_ok = su.mode != M_MATRIX && s->n == 1 && !su.wide;
    if (want == ECLIP_ENGINE_ENUM && !enum_ok)
        return fail(ECLIP_E_TOO_LARGE, "ENUM engine limits exceeded (W=%d, Lmax=%d)", W, Lmax);
    if (want == ECLIP_ENGINE_SLICE && !slice_ok)
        return su.wide ? fail(ECLIP_E_TOO_LARGE, "SLICE engine: the T' range of these kernel counts is too large "
                                                 "(Lambda N (W+1) >= 2^24); use ENUM")
                       : fail(ECLIP_E_INVALID_ARG, "SLICE engine needs a linear slowdown mode and a single problem");
    if (want == ECLIP_ENGINE_AUTO) {
        // ENUM scores every candidate; SLICE when enumeration is far larger than the lattice
        if (!enum_ok || (slice_ok && tuples > 4e10L)) {
            if (!slice_ok) return fail(ECLIP_E_TOO_LARGE, "search space too large for ENUM and SLICE does not apply");
            s->engine = ECLIP_ENGINE_SLICE;
        } else {
            s->engine = ECLIP_ENGINE_ENUM;
        }
    } else {
        s->engine = want;
    }
    if (s->engine != ECLIP_ENGINE_ENUM) {
        su.nseg = 1; su.upi = 1; su.units_max = 1; su.items_max = 1; su.table_bytes = 0; su.aux_bytes = 0;
        su.lev_stride = W * Lmax;
        return ECLIP_OK;
    }
    const int Lstep = W >= 2 ? Lmax : 1;
    int nseg = 1;
    if (n * H < 4096) nseg = (int)std::min<long double>(Lstep, std::ceil(4096.0L / (n * H)));
    const int seglen = (Lstep + nseg - 1) / nseg;
    nseg = (Lstep + seglen - 1) / seglen;
    const bool fast = su.obj == O_SUM && (su.mode == M_EXCL || su.mode == M_PAPER) && pass1_fast(Lmax) && !su.wide &&
                      !su.weighted;
    const int teams_typ = P1_THREADS / 32;   // one unit per warp in both pass-1 kernels
    const long double units = H * nseg;
    const long double cand_unit = (long double)seglen * Lmax;
    long double target = n * units / 592.0L;                    // >= 2 CTAs per SM, 2 waves
    long double upi = std::min<long double>(target, std::max<long double>(1, 16777216.0L / cand_unit));
    upi = std::max<long double>(upi, teams_typ);
    if (su.prune && W >= 3 && fast) {
        // row pruning leaves few units per item: larger items (up to a whole problem) amortise the
        // staging, as long as there are >= 8 CTAs per SM
        upi = std::max<long double>(upi, std::min<long double>(units, std::ceil(n * units / 1184.0L)));
    }
    upi = std::ceil(upi / teams_typ) * teams_typ;
    su.nseg = nseg;
    su.upi = (int32_t)std::min<long double>(upi, 1 << 30);
    su.units_max = (int64_t)units;
    su.rows_max = (int64_t)H;
    su.items_max = (int32_t)std::ceil(units / su.upi);
    su.table_bytes = 0;
    su.aux_bytes = 0;
    if (fast) {   // per-problem aux block (staged with the Lev records) + per-warp prefix tables
        su.aux_bytes = (int32_t)pass1_aux_bytes(Lmax);
        // 32 entries per warp; 64 in the exhaustive pass without QoS (two per lane, k_pass1_fast TWO)
        su.table_bytes = (int32_t)((size_t)(P1_THREADS / 32) * 32 * 24);   // 32 entries per warp
    }
    su.lev_stride = W * Lmax + su.aux_bytes / (int)sizeof(Lev);
    return ECLIP_OK;
}

// Work buffers of the current geometry in one device block.  With `reuse` (a persistent planner)
// the block of the previous call is kept when it is large enough; otherwise a new one is taken.
struct WorkBlock {
    unsigned char* base = nullptr;
    size_t cap = 0;
};

static int alloc_work(eclip_session* s, WorkBlock* reuse = nullptr) {
    Setup& su = s->su;
    Work& wk = s->wk;
    const size_t n = (size_t)su.n_problems;
    const bool en = s->engine == ECLIP_ENGINE_ENUM, bb = en && pass1_prunable(su);
    const size_t ns = n * (size_t)su.units_max;
    const size_t grid = n * (size_t)((su.items_max + su.n_shards - 1) / su.n_shards);
    Bump bp;   // one block; null pieces stay null
    const size_t o_cnt = bp.take<unsigned long long>(8);   // feasible, rows_done[6] (zeroed)
    const size_t o_probs = bp.take<Prob>(n), o_levs = bp.take<Lev>(n * (size_t)su.lev_stride);
    const size_t o_sub = en ? bp.take<float>(ns) : 0, o_bandn = en ? bp.take<int32_t>(n) : 0;
    const size_t o_bandl = en ? bp.take<uint64_t>(n * (size_t)BAND_CAP) : 0;
    const size_t o_sure = (en && qos_float(su)) ? bp.take<float>(ns) : 0;
    const size_t o_m32 = bp.take<float>(n), o_m32s = bp.take<float>(n), o_hs = bp.take<U256>(n), o_first = bp.take<U256>(n);
    size_t o_th = 0, o_thn = 0, o_tord = 0;
    if (en && su.aux_bytes > 0 && !wk.thull) {   // per-table S order and hulls (k_table_hull), unless held elsewhere
        o_th = bp.take<uint16_t>((size_t)s->tb.n * su.Lmax);
        o_thn = bp.take<int32_t>((size_t)s->tb.n);
        o_tord = bp.take<uint16_t>((size_t)s->tb.n * su.Lmax);
    }
    size_t o_rowlb = 0, o_lbmin = 0, o_inc = 0, o_hull = 0, o_ftab = 0, o_ulist = 0, o_uln = 0, o_rh = 0, o_pl = 0, o_pln = 0, o_wb = 0;
    if (bb) {
        o_rowlb = bp.take<float>(n * (size_t)su.rows_max);
        o_lbmin = bp.take<unsigned>(n);
        o_inc = bp.take<unsigned>(n);
        o_hull = bp.take<float2>(n * hull_stride(su.Lmax));
        o_ftab = bp.take<int32_t>(n * (size_t)FT_CAP);
        o_ulist = bp.take<uint2>(grid * (size_t)su.upi);
        o_uln = bp.take<int32_t>(grid);
        o_rh = bp.take<RowHdr>(n);

        o_pl = bp.take<uint32_t>(n * (size_t)PL_CAP);
        o_pln = bp.take<int32_t>(n);
        o_wb = bp.take<uint32_t>(n * (size_t)((su.units_max + 31) >> 5));
    }
    // representatives of the step / inner precomputation (fast pass 1, batches)
    size_t aslots = 0, o_akey = 0, o_aslot = 0;
    if (en && su.aux_bytes > 0 && n > 1) {
        aslots = 1024;
        while (aslots < 2 * n) aslots <<= 1;
        o_akey = bp.take<AKey>(n);
        o_aslot = bp.take<unsigned long long>(2 * aslots);
    }
    unsigned char* base;
    if (reuse && reuse->base && reuse->cap >= bp.off) {
        base = reuse->base;
    } else {
        CU(s->arena.alloc(&base, bp.off));
        if (reuse) { reuse->base = base; reuse->cap = bp.off; }
    }
    wk.feasible = (unsigned long long*)(base + o_cnt);
    wk.rows_done = wk.feasible + 1;
    CU(cudaMemsetAsync(wk.feasible, 0, 8 * sizeof(unsigned long long), s->st));
    wk.probs = (Prob*)(base + o_probs);
    if (o_th) {
        wk.thull = (uint16_t*)(base + o_th);
        wk.thull_n = (int32_t*)(base + o_thn);
        wk.tord = (uint16_t*)(base + o_tord);
    }
    wk.levs = (Lev*)(base + o_levs);
    if (en) {
        wk.submin = (float*)(base + o_sub);
        wk.bandn = (int32_t*)(base + o_bandn);
        wk.bandlist = (uint64_t*)(base + o_bandl);
        if (o_sure) wk.submin_sure = (float*)(base + o_sure);
    }
    wk.aslots = (int32_t)aslots;
    wk.akey = aslots ? (AKey*)(base + o_akey) : nullptr;
    wk.aslot = aslots ? (unsigned long long*)(base + o_aslot) : nullptr;
    wk.m32 = (float*)(base + o_m32);
    wk.m32_sure = (float*)(base + o_m32s);
    wk.hstar = (U256*)(base + o_hs);
    wk.first = (U256*)(base + o_first);
    if (bb) {
        wk.rowlb = (float*)(base + o_rowlb);
        wk.lbmin = (unsigned*)(base + o_lbmin);
        wk.inc = (unsigned*)(base + o_inc);
        wk.hull = (float2*)(base + o_hull);
        wk.ftab = (int32_t*)(base + o_ftab);
        wk.ulist = (uint2*)(base + o_ulist);
        wk.ulist_n = (int32_t*)(base + o_uln);
        wk.rowhdr = (RowHdr*)(base + o_rh);

        wk.plist = (uint32_t*)(base + o_pl);
        wk.plist_n = (int32_t*)(base + o_pln);
        wk.wbits = (uint32_t*)(base + o_wb);
    }
    return ECLIP_OK;
}

static int status_error(const eclip_session* s, int st, int p) {
    (void)s;
    if (st == -5) return fail(ECLIP_E_TOO_LARGE, "problem %d exceeds the exact-arithmetic ranges (Lambda = lcm of kernel counts <= 2^40, Lambda N (W+1) < 2^62, ...)", p);
    return fail(ECLIP_E_INVALID_ARG, "problem %d is invalid (model id / QoS / matrix / power values)", p);
}

// per-worker table specs of a problem (validated: model ids, masks, group bounds, QoS)
static int worker_specs(const eclip_profiles* P, const eclip_problem* pr, std::vector<TableSpec>* out) {
    const int W = pr->n_models;
    const int C = P->C();
    out->assign(W, TableSpec{});
    const int32_t* gb = pr->group_bounds;
    for (int w = 0; w < W; w++) {
        int m = pr->model_ids[w];
        if (m < 0 || m >= P->n()) return fail(ECLIP_E_INVALID_ARG, "model id %d of worker %d out of range", m, w);
        TableSpec& sp = (*out)[w];
        sp.model = m;
        sp.R = pr->switch_max;
        sp.mask = pr->allowed_mask ? pr->allowed_mask[w] : ((C == 32) ? 0xffffffffu : ((1u << C) - 1u));
        if (C < 32) sp.mask &= (1u << C) - 1u;
        if (sp.mask == 0) return fail(ECLIP_E_INVALID_ARG, "worker %d has no allowed size", w);
        for (int j = 0; j < C; j++)
            if (((sp.mask >> j) & 1u) && P->sizes[j] > pr->total_sms)
                return fail(ECLIP_E_INVALID_ARG, "size %d exceeds total_sms", P->sizes[j]);
        int K = P->nk[m];
        if (gb) {
            if (gb[0] != 0) return fail(ECLIP_E_INVALID_ARG, "group_bounds of worker %d must start at 0", w);
            sp.bounds.push_back(0);
            int i = 1;
            while (sp.bounds.back() != K) {
                int b = gb[i];
                if (b <= sp.bounds.back() || b > K)
                    return fail(ECLIP_E_INVALID_ARG, "group_bounds of worker %d must ascend to %d", w, K);
                sp.bounds.push_back(b);
                i++;
            }
            gb += i;
        } else {
            for (int k = 0; k <= K; k++) sp.bounds.push_back(k);
        }
        if (pr->qos_ns && !(pr->qos_ns[w] >= 0.0)) return fail(ECLIP_E_INVALID_ARG, "qos_ns[%d] must be >= 0 or +inf", w);
    }
    if (pr->slowdown == ECLIP_MATRIX) {
        if (!pr->slowdown_matrix) return fail(ECLIP_E_INVALID_ARG, "MATRIX slowdown needs slowdown_matrix");
        if (W > MAXW_ENUM) return fail(ECLIP_E_TOO_LARGE, "MATRIX slowdown supports at most %d workers", MAXW_ENUM);
        for (int i = 0; i < W * W; i++) {
            float m = pr->slowdown_matrix[i];
            if (i / W != i % W && !(std::isfinite(m) && m >= 0.0f && m < 1024.0f))
                return fail(ECLIP_E_INVALID_ARG, "slowdown_matrix entries must be finite, >= 0 and < 1024");
        }
    }
    return ECLIP_OK;
}

// ------------------------------------------------------------------------------------------
// session construction
// ------------------------------------------------------------------------------------------
static int session_from_problem(const eclip_profiles* P, const eclip_problem* pr, const eclip_options* opt,
                                eclip_session** out) {
    if (!pr) return fail(ECLIP_E_INVALID_ARG, "null problem");
    const int W = pr->n_models;
    double tol = opt ? opt->tie_tol : 1e-5;
    int rc = check_common(P, W, pr->total_sms, pr->switch_max, pr->slowdown, pr->objective, pr->p_idle_w, pr->p_max_w, tol);
    if (rc) return rc;
    if (!pr->model_ids) return fail(ECLIP_E_INVALID_ARG, "null model_ids");
    const int C = P->C();
    std::vector<TableSpec> wspec, specs;
    rc = worker_specs(P, pr, &wspec);
    if (rc) return rc;
    std::map<TableSpec, int> ids;
    std::vector<int32_t> table_of(W);
    for (int w = 0; w < W; w++) {
        const TableSpec& sp = wspec[w];
        auto it = ids.find(sp);
        if (it == ids.end()) {
            ids[sp] = (int)specs.size();
            table_of[w] = (int)specs.size();
            specs.push_back(sp);
        } else {
            table_of[w] = it->second;
        }
    }
    auto s = std::make_unique<eclip_session>();
    s->prof = P;
    s->W = W; s->n = 1; s->C = C;
    rc = setup_device(s.get(), opt);
    if (rc) return rc;
    host_mark("setup_device");
    bool has_qos = false;
    if (pr->qos_ns)
        for (int w = 0; w < W; w++) has_qos |= !std::isinf(pr->qos_ns[w]);
    bool unequal = false;
    if ((rc = check_weights(pr->weights, 1, W, pr->objective, &unequal))) return rc;
    fill_setup(s.get(), 1, W, pr->total_sms, pr->switch_max, pr->slowdown, pr->objective, has_qos, opt);
    s->su.weighted = unequal ? 1 : 0;
    rc = build_tables(s.get(), specs);
    if (rc) return rc;
    host_mark("build_tables (K1, synced)");
    s->h_table_of = table_of;
    set_wide(s.get(), table_of);
    rc = plan_geometry(s.get(), opt);
    if (rc) return rc;
    rc = alloc_work(s.get());
    if (rc) return rc;
    host_mark("geometry + alloc_work");
    // per-problem inputs
    int32_t* dtab; double* dq = nullptr; float* dM = nullptr;
    CU(s->arena.alloc(&dtab, W));
    CU(cudaMemcpyAsync(dtab, table_of.data(), 4 * W, cudaMemcpyHostToDevice, s->st));
    if (pr->qos_ns) {
        CU(s->arena.alloc(&dq, W));
        CU(cudaMemcpyAsync(dq, pr->qos_ns, 8 * W, cudaMemcpyHostToDevice, s->st));
    }
    if (pr->slowdown == ECLIP_MATRIX) {
        CU(s->arena.alloc(&dM, (size_t)W * W));
        CU(cudaMemcpyAsync(dM, pr->slowdown_matrix, 4 * W * W, cudaMemcpyHostToDevice, s->st));
    }
    double* dw = nullptr;
    if (pr->weights) {
        CU(s->arena.alloc(&dw, W));
        CU(cudaMemcpyAsync(dw, pr->weights, 8 * W, cudaMemcpyHostToDevice, s->st));
    }
    CU(s->arena.alloc(&s->d_sizes, C));
    CU(cudaMemcpyAsync(s->d_sizes, P->sizes.data(), 4 * C, cudaMemcpyHostToDevice, s->st));
    s->pin.table_of = dtab; s->pin.qos = dq; s->pin.M = dM; s->pin.weights = dw;
    s->wk.table_of = dtab;
    s->wk.tb = s->tb;
    s->pin.p_idle = pr->p_idle_w; s->pin.p_max = pr->p_max_w;
    CU(launch_prep(s->su, s->tb, s->pin, s->wk, C, s->d_sizes, s->st));
    *out = s.release();
    return ECLIP_OK;
}

static int session_from_batch(const eclip_profiles* P, const eclip_batch* b, const eclip_options* opt,
                              eclip_session** out) {
    if (!b) return fail(ECLIP_E_INVALID_ARG, "null batch");
    double tol = opt ? opt->tie_tol : 1e-5;
    int rc = check_common(P, b->n_models, b->total_sms, b->switch_max, b->slowdown, b->objective, b->p_idle_w,
                          b->p_max_w, tol);
    if (rc) return rc;
    if (b->n_problems < 1) return fail(ECLIP_E_INVALID_ARG, "n_problems must be >= 1");
    if (!b->model_ids) return fail(ECLIP_E_INVALID_ARG, "null model_ids");
    if (b->slowdown == ECLIP_MATRIX && !b->slowdown_matrix)
        return fail(ECLIP_E_INVALID_ARG, "MATRIX slowdown needs slowdown_matrix");
    const int W = b->n_models, n = b->n_problems, C = P->C();
    if (!b->on_device) {
        for (int i = 0; i < n * W; i++) {
            if (b->model_ids[i] < 0 || b->model_ids[i] >= P->n())
                return fail(ECLIP_E_INVALID_ARG, "model id %d out of range (problem %d)", b->model_ids[i], i / W);
            if (b->qos_ns && !(b->qos_ns[i] >= 0.0)) return fail(ECLIP_E_INVALID_ARG, "qos_ns must be >= 0 or +inf");
        }
    }
    // one table per model of the profiles (the batch shares the grouping, mask and budget)
    std::vector<TableSpec> specs;
    for (int m = 0; m < P->n(); m++) {
        TableSpec sp;
        sp.model = m;
        sp.R = b->switch_max;
        sp.mask = b->allowed_mask ? b->allowed_mask[m] : ((C == 32) ? 0xffffffffu : ((1u << C) - 1u));
        if (C < 32) sp.mask &= (1u << C) - 1u;
        if (sp.mask == 0) return fail(ECLIP_E_INVALID_ARG, "model %d has no allowed size", m);
        for (int j = 0; j < C; j++)
            if (((sp.mask >> j) & 1u) && P->sizes[j] > b->total_sms)
                return fail(ECLIP_E_INVALID_ARG, "size %d exceeds total_sms", P->sizes[j]);
        for (int k = 0; k <= P->nk[m]; k++) sp.bounds.push_back(k);
        specs.push_back(sp);
    }
    auto s = std::make_unique<eclip_session>();
    s->prof = P;
    s->W = W; s->n = n; s->C = C;
    s->on_device = b->on_device != 0;
    rc = setup_device(s.get(), opt);
    if (rc) return rc;
    bool unequal = b->weights != nullptr && b->on_device;   // device weights: not inspected on the host
    if (b->weights && !b->on_device && (rc = check_weights(b->weights, (size_t)n, W, b->objective, &unequal))) return rc;
    fill_setup(s.get(), n, W, b->total_sms, b->switch_max, b->slowdown, b->objective, b->qos_ns != nullptr, opt);
    s->su.weighted = unequal ? 1 : 0;
    rc = build_tables(s.get(), specs);
    if (rc) return rc;
    {
        std::vector<int32_t> all(specs.size());
        for (size_t i = 0; i < all.size(); i++) all[i] = (int32_t)i;
        set_wide(s.get(), all);
    }
    rc = plan_geometry(s.get(), opt);
    if (rc) return rc;
    if (s->engine != ECLIP_ENGINE_ENUM) return fail(ECLIP_E_TOO_LARGE, "batched planning runs on the ENUM engine only");
    rc = alloc_work(s.get());
    if (rc) return rc;
    const int32_t* dtab = b->model_ids;
    const double* dq = b->qos_ns;
    const float* dM = b->slowdown_matrix;
    const double* dW = b->weights;
    if (!b->on_device) {
        int32_t* t; double* q = nullptr; float* M = nullptr;
        if (b->weights) {
            double* wd;
            CU(s->arena.alloc(&wd, (size_t)n * W));
            CU(cudaMemcpyAsync(wd, b->weights, 8 * (size_t)n * W, cudaMemcpyHostToDevice, s->st));
            dW = wd;
        }
        CU(s->arena.alloc(&t, (size_t)n * W));
        CU(cudaMemcpyAsync(t, b->model_ids, 4 * (size_t)n * W, cudaMemcpyHostToDevice, s->st));
        if (b->qos_ns) {
            CU(s->arena.alloc(&q, (size_t)n * W));
            CU(cudaMemcpyAsync(q, b->qos_ns, 8 * (size_t)n * W, cudaMemcpyHostToDevice, s->st));
        }
        if (b->slowdown == ECLIP_MATRIX) {
            CU(s->arena.alloc(&M, (size_t)n * W * W));
            CU(cudaMemcpyAsync(M, b->slowdown_matrix, 4 * (size_t)n * W * W, cudaMemcpyHostToDevice, s->st));
        }
        dtab = t; dq = q; dM = M;
    }
    CU(s->arena.alloc(&s->d_sizes, C));
    CU(cudaMemcpyAsync(s->d_sizes, P->sizes.data(), 4 * C, cudaMemcpyHostToDevice, s->st));
    s->pin.table_of = dtab; s->pin.qos = dq; s->pin.M = dM; s->pin.weights = dW;
    s->wk.table_of = dtab;
    s->wk.tb = s->tb;
    s->pin.p_idle = b->p_idle_w; s->pin.p_max = b->p_max_w;
    CU(launch_prep(s->su, s->tb, s->pin, s->wk, C, s->d_sizes, s->st));
    *out = s.release();
    return ECLIP_OK;
}

// ------------------------------------------------------------------------------------------
// steps
// ------------------------------------------------------------------------------------------
static int step_pass1(eclip_session* s) {
    if (s->engine == ECLIP_ENGINE_SLICE) {
        CU(slice_pass1(s->slice, s->su, s->tb, s->wk, s->st));
        return ECLIP_OK;
    }
    CU(launch_pass1(s->su, s->wk, s->st));
    CU(launch_reduce_min(s->su, s->wk, s->st));
    return ECLIP_OK;
}
static int step_pass2_min(eclip_session* s) {
    if (s->engine == ECLIP_ENGINE_SLICE) {
        CU(slice_pass2_min(s->slice, s->su, s->tb, s->wk, s->st));
        return ECLIP_OK;
    }
    CU(launch_pass2_min(s->su, s->wk, s->st));
    return ECLIP_OK;
}
static int step_pass2_first(eclip_session* s) {
    if (s->engine == ECLIP_ENGINE_SLICE) {
        CU(slice_pass2_first(s->slice, s->su, s->tb, s->wk, s->st));
        return ECLIP_OK;
    }
    CU(launch_pass2_first(s->su, s->wk, s->st));
    return ECLIP_OK;
}

extern "C" int eclip_session_create(const eclip_profiles* prof, const eclip_batch* batch, const eclip_options* opt,
                                    eclip_session** out) {
    if (!out) return fail(ECLIP_E_INVALID_ARG, "null out");
    if (batch && batch->on_device) return fail(ECLIP_E_INVALID_ARG, "sessions take host batches");
    return session_from_batch(prof, batch, opt, out);
}

extern "C" int eclip_session_pass1(eclip_session* s, float* min_key32) {
    if (!s) return fail(ECLIP_E_INVALID_ARG, "null session");
    int rc = step_pass1(s);
    if (rc) return rc;
    if (min_key32) {
        CU(cudaMemcpyAsync(min_key32, s->wk.m32, 4 * (size_t)s->n, cudaMemcpyDeviceToHost, s->st));
        CU(cudaStreamSynchronize(s->st));
    }
    return ECLIP_OK;
}

extern "C" int eclip_session_pass2_min(eclip_session* s, const float* global_min, uint64_t* exact_min) {
    if (!s) return fail(ECLIP_E_INVALID_ARG, "null session");
    if (global_min) {
        CU(cudaMemcpyAsync(s->wk.m32, global_min, 4 * (size_t)s->n, cudaMemcpyHostToDevice, s->st));
        if (!qos_float(s->su))
            CU(cudaMemcpyAsync(s->wk.m32_sure, global_min, 4 * (size_t)s->n, cudaMemcpyHostToDevice, s->st));
    }
    int rc = step_pass2_min(s);
    if (rc) return rc;
    if (exact_min) {
        CU(cudaMemcpyAsync(exact_min, s->wk.hstar, 32 * (size_t)s->n, cudaMemcpyDeviceToHost, s->st));
        CU(cudaStreamSynchronize(s->st));
    }
    return ECLIP_OK;
}

extern "C" int eclip_session_pass2_first(eclip_session* s, const uint64_t* global_exact_min, uint64_t* first_tuple) {
    if (!s) return fail(ECLIP_E_INVALID_ARG, "null session");
    if (global_exact_min)
        CU(cudaMemcpyAsync(s->wk.hstar, global_exact_min, 32 * (size_t)s->n, cudaMemcpyHostToDevice, s->st));
    int rc = step_pass2_first(s);
    if (rc) return rc;
    if (first_tuple) {
        CU(cudaMemcpyAsync(first_tuple, s->wk.first, 32 * (size_t)s->n, cudaMemcpyDeviceToHost, s->st));
        CU(cudaStreamSynchronize(s->st));
    }
    return ECLIP_OK;
}

// A growable device scratch block (stream-ordered); a persistent planner keeps its result
// staging here instead of allocating per call.
struct Scratch {
    unsigned char* p = nullptr;
    size_t cap = 0;
    cudaStream_t st = nullptr;
    cudaError_t need(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFreeAsync(p, st);
        p = nullptr; cap = 0;
        cudaError_t e = cudaMallocAsync((void**)&p, bytes, st);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    ~Scratch() { if (p) cudaFreeAsync(p, st); }
};

// materialise into device buffers; copy to the caller's host arrays unless on_device
static int finish_batch(eclip_session* s, eclip_batch_out* o, double* glat_host = nullptr, uint64_t* key_host = nullptr,
                        Scratch* stg = nullptr) {
    const size_t n = s->n, W = s->W;
    int stride = o->group_stride > 0 ? o->group_stride : 1;
    MatOut mo{};
    mo.group_stride = stride;
    mo.gsum = s->W * std::max(1, s->gmax);
    if (s->on_device) {
        mo.status = o->status; mo.levels = o->winner_levels; mo.index = o->winner_index; mo.objective = o->objective;
        mo.makespan = o->makespan_ns; mo.power = o->power_w; mo.energy = o->energy_j; mo.thr = o->throughput_rps;
        mo.latency = o->model_latency_ns; mo.switches = o->model_switches; mo.group_sm = o->group_sm;
        mo.energy_busy = o->energy_busy_j;
        if (s->engine == ECLIP_ENGINE_SLICE) CU(slice_decode_winner(s->slice, s->su, s->wk, s->st));
        CU(launch_materialize(s->su, s->tb, s->wk, s->d_sizes, s->C, mo, s->st));
        return ECLIP_OK;
    }
    // staging for every output: one block (the planner's growable scratch, or the session arena)
    Bump bp;
    const size_t o_st = bp.take<int32_t>(n), o_lv = bp.take<int32_t>(n * W), o_sw = bp.take<int32_t>(n * W);
    const size_t o_idx = bp.take<uint64_t>(n), o_obj = bp.take<double>(n), o_mk = bp.take<double>(n);
    const size_t o_pw = bp.take<double>(n), o_en = bp.take<double>(n), o_thr = bp.take<double>(n);
    const size_t o_lat = bp.take<double>(n * W);
    const size_t o_eb = o->energy_busy_j ? bp.take<double>(n) : 0;
    const size_t o_gsm = o->group_sm ? bp.take<int32_t>(n * W * stride) : 0;
    const size_t o_glat = glat_host ? bp.take<double>(n * W * stride) : 0;
    const size_t o_key = key_host ? bp.take<uint64_t>(n * 4) : 0;
    unsigned char* base;
    if (stg) {
        CU(stg->need(bp.off));
        base = stg->p;
    } else {
        CU(s->arena.alloc(&base, bp.off));
    }
    int32_t* st = (int32_t*)(base + o_st); int32_t* lv = (int32_t*)(base + o_lv); int32_t* sw = (int32_t*)(base + o_sw);
    uint64_t* idx = (uint64_t*)(base + o_idx);
    double *obj = (double*)(base + o_obj), *mk = (double*)(base + o_mk), *pw = (double*)(base + o_pw);
    double *en = (double*)(base + o_en), *thr = (double*)(base + o_thr), *lat = (double*)(base + o_lat);
    int32_t* gsm = o->group_sm ? (int32_t*)(base + o_gsm) : nullptr;
    double* glat = glat_host ? (double*)(base + o_glat) : nullptr;
    uint64_t* key = key_host ? (uint64_t*)(base + o_key) : nullptr;
    mo.group_lat = glat; mo.key = key;
    mo.energy_busy = o->energy_busy_j ? (double*)(base + o_eb) : nullptr;
    mo.status = st; mo.levels = lv; mo.index = idx; mo.objective = obj; mo.makespan = mk; mo.power = pw;
    mo.energy = en; mo.thr = thr; mo.latency = lat; mo.switches = sw; mo.group_sm = gsm;
    if (s->engine == ECLIP_ENGINE_SLICE) CU(slice_decode_winner(s->slice, s->su, s->wk, s->st));
    CU(launch_materialize(s->su, s->tb, s->wk, s->d_sizes, s->C, mo, s->st));
    if (!stg && bp.off <= ((size_t)256 << 10)) {
        // small results (one-shot plans): the staging block in one copy, then host copies into the caller's arrays
        std::vector<unsigned char> hb(bp.off);
        CU(cudaMemcpyAsync(hb.data(), base, bp.off, cudaMemcpyDeviceToHost, s->st));
        CU(cudaStreamSynchronize(s->st));
        auto hc = [&](void* dst, const void* src, size_t bytes) {
            if (dst) std::memcpy(dst, hb.data() + ((const unsigned char*)src - base), bytes);
        };
        hc(o->status, st, 4 * n);
        hc(o->winner_levels, lv, 4 * n * W);
        hc(o->winner_index, idx, 8 * n);
        hc(o->objective, obj, 8 * n);
        hc(o->makespan_ns, mk, 8 * n);
        hc(o->power_w, pw, 8 * n);
        hc(o->energy_j, en, 8 * n);
        hc(o->throughput_rps, thr, 8 * n);
        hc(o->model_latency_ns, lat, 8 * n * W);
        hc(o->model_switches, sw, 4 * n * W);
        if (mo.energy_busy) hc(o->energy_busy_j, mo.energy_busy, 8 * n);
        if (gsm) hc(o->group_sm, gsm, 4 * n * W * stride);
        if (glat) hc(glat_host, glat, 8 * n * W * stride);
        if (key) hc(key_host, key, 32 * n);
        if (o->status)
            for (size_t i = 0; i < n; i++)
                if (o->status[i] < 0) return status_error(s, o->status[i], (int)i);
        return ECLIP_OK;
    }
    auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
        return dst ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s->st) : cudaSuccess;
    };
    CU(cp(o->status, st, 4 * n));
    CU(cp(o->winner_levels, lv, 4 * n * W));
    CU(cp(o->winner_index, idx, 8 * n));
    CU(cp(o->objective, obj, 8 * n));
    CU(cp(o->makespan_ns, mk, 8 * n));
    CU(cp(o->power_w, pw, 8 * n));
    CU(cp(o->energy_j, en, 8 * n));
    CU(cp(o->throughput_rps, thr, 8 * n));
    CU(cp(o->model_latency_ns, lat, 8 * n * W));
    CU(cp(o->model_switches, sw, 4 * n * W));
    if (mo.energy_busy) CU(cp(o->energy_busy_j, mo.energy_busy, 8 * n));
    if (gsm) CU(cp(o->group_sm, gsm, 4 * n * W * stride));
    if (glat) CU(cp(glat_host, glat, 8 * n * W * stride));
    if (key) CU(cp(key_host, key, 32 * n));
    CU(cudaStreamSynchronize(s->st));
    if (o->status)
        for (size_t i = 0; i < n; i++)
            if (o->status[i] < 0) return status_error(s, o->status[i], (int)i);
    return ECLIP_OK;
}

extern "C" int eclip_session_finish(eclip_session* s, const uint64_t* global_first_tuple, eclip_batch_out* out) {
    if (!s || !out) return fail(ECLIP_E_INVALID_ARG, "null argument");
    if (global_first_tuple)
        CU(cudaMemcpyAsync(s->wk.first, global_first_tuple, 32 * (size_t)s->n, cudaMemcpyHostToDevice, s->st));
    return finish_batch(s, out);
}

extern "C" void eclip_session_free(eclip_session* s) { delete s; }

extern "C" int eclip_session_stats(eclip_session* s, uint64_t* evaluated) {
    if (!s || !evaluated) return fail(ECLIP_E_INVALID_ARG, "null argument");
    unsigned long long v = 0;
    if (s->wk.feasible) CU(cudaMemcpyAsync(&v, s->wk.feasible, sizeof v, cudaMemcpyDeviceToHost, s->st));
    CU(cudaStreamSynchronize(s->st));
    *evaluated = v;
    return ECLIP_OK;
}

extern "C" int eclip_session_counters(eclip_session* s, uint64_t* out, int32_t n) {
    if (!s || !out || n < 0) return fail(ECLIP_E_INVALID_ARG, "null argument");
    unsigned long long v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (s->wk.feasible) CU(cudaMemcpyAsync(&v[0], s->wk.feasible, sizeof v[0], cudaMemcpyDeviceToHost, s->st));
    if (s->wk.rows_done) CU(cudaMemcpyAsync(&v[1], s->wk.rows_done, sizeof v[1], cudaMemcpyDeviceToHost, s->st));
    if (s->wk.rows_done) CU(cudaMemcpyAsync(&v[3], s->wk.rows_done + 1, 5 * sizeof v[0], cudaMemcpyDeviceToHost, s->st));
    CU(cudaStreamSynchronize(s->st));
    float ms = 0.0f;   // the events exist from session creation; unrecorded (SLICE) -> error -> 0
    if (s->engine == ECLIP_ENGINE_ENUM && cudaEventElapsedTime(&ms, s->wk.kev[0], s->wk.kev[1]) == cudaSuccess)
        v[2] = (unsigned long long)llround((double)ms * 1e6);
    cudaGetLastError();
    for (int i = 0; i < n; i++) out[i] = i < 8 ? v[i] : 0;
    return ECLIP_OK;
}

// ------------------------------------------------------------------------------------------
// one-shot entry points
// ------------------------------------------------------------------------------------------
static int run_all_steps(eclip_session* s) {
    int rc = step_pass1(s);
    if (rc) return rc;
    if (s->comm) {   // sharded over the communicator: the three exchanges on device buffers
        if ((rc = comm_min_f32(s->comm, s->wk.m32, s->n, s->st))) return rc;
        if (qos_float(s->su)) {
            if ((rc = comm_min_f32(s->comm, s->wk.m32_sure, s->n, s->st))) return rc;
        } else {
            CU(cudaMemcpyAsync(s->wk.m32_sure, s->wk.m32, 4 * (size_t)s->n, cudaMemcpyDeviceToDevice, s->st));
        }
        if ((rc = step_pass2_min(s))) return rc;
        if ((rc = comm_lexmin_u256(s->comm, s->wk.hstar, s->n, s->st))) return rc;
        if ((rc = step_pass2_first(s))) return rc;
        return comm_lexmin_u256(s->comm, s->wk.first, s->n, s->st);
    }
    if (s->engine == ECLIP_ENGINE_ENUM && s->su.n_shards == 1) {   // unsharded: one band rescan
        CU(launch_pass2_both(s->su, s->wk, s->st));
        return ECLIP_OK;
    }
    rc = step_pass2_min(s);
    if (rc) return rc;
    return step_pass2_first(s);
}

extern "C" int eclip_plan_batch(const eclip_profiles* prof, const eclip_batch* batch, const eclip_options* opt,
                                eclip_batch_out* out) {
    if (!out) return fail(ECLIP_E_INVALID_ARG, "null out");
    eclip_session* s = nullptr;
    int rc = session_from_batch(prof, batch, opt, &s);
    if (rc) { delete s; return rc; }
    std::unique_ptr<eclip_session> guard(s);
    rc = run_all_steps(s);
    if (rc) return rc;
    rc = finish_batch(s, out);
    if (rc) return rc;
    if (s->on_device && s->own_stream) CU(cudaStreamSynchronize(s->st));
    return ECLIP_OK;
}

// ------------------------------------------------------------------------------------------
// persistent planner (include/eclip.h "persistent planner"): level tables, per-table hulls and
// device workspaces are built once; each plan call runs only the per-mix work
// ------------------------------------------------------------------------------------------
struct eclip_planner {
    std::unique_ptr<eclip_session> s;
    eclip_options opt{};
    int n_max = 0, W = 0, N = 0, R = 0, mode = 0, obj = 0;
    float pi = 0.0f, pm = 0.0f;
    bool has_qos = false, has_w = false, timing = false;
    std::vector<uint32_t> mask;
    WorkBlock wb;
    Scratch stg;
    int32_t* d_ids = nullptr;
    double* d_qos = nullptr;
    float* d_M = nullptr;
    double* d_w = nullptr;
    cudaEvent_t ev[6] = {};
    bool ev_valid = false;
    ~eclip_planner() {
        if (s && s->st) cudaStreamSynchronize(s->st);
        for (cudaEvent_t& e : ev)
            if (e) cudaEventDestroy(e);
    }
};

// table specs of a batch: one table per model of the profiles (shared grouping, mask and budget)
static int batch_specs(const eclip_profiles* P, const eclip_batch* b, std::vector<TableSpec>* specs) {
    const int C = P->C();
    specs->clear();
    for (int m = 0; m < P->n(); m++) {
        TableSpec sp;
        sp.model = m;
        sp.R = b->switch_max;
        sp.mask = b->allowed_mask ? b->allowed_mask[m] : ((C == 32) ? 0xffffffffu : ((1u << C) - 1u));
        if (C < 32) sp.mask &= (1u << C) - 1u;
        if (sp.mask == 0) return fail(ECLIP_E_INVALID_ARG, "model %d has no allowed size", m);
        for (int j = 0; j < C; j++)
            if (((sp.mask >> j) & 1u) && P->sizes[j] > b->total_sms)
                return fail(ECLIP_E_INVALID_ARG, "size %d exceeds total_sms", P->sizes[j]);
        for (int k = 0; k <= P->nk[m]; k++) sp.bounds.push_back(k);
        specs->push_back(sp);
    }
    return ECLIP_OK;
}

extern "C" int eclip_planner_create(const eclip_profiles* P, const eclip_batch* b, int32_t max_problems,
                                    const eclip_options* opt, eclip_planner** out) {
    if (!b || !out) return fail(ECLIP_E_INVALID_ARG, "null argument");
    if (max_problems < 1) return fail(ECLIP_E_INVALID_ARG, "max_problems must be >= 1");
    eclip_options o;
    if (opt) o = *opt; else eclip_default_options(&o);
    if (o.engine != ECLIP_ENGINE_AUTO && o.engine != ECLIP_ENGINE_ENUM)
        return fail(ECLIP_E_INVALID_ARG, "the planner runs the ENUM engine");
    if (o.n_shards > 1 || o.comm) return fail(ECLIP_E_INVALID_ARG, "the planner plans whole batches (n_shards = 1, no comm)");
    o.engine = ECLIP_ENGINE_ENUM;
    o.shard = 0; o.n_shards = 1;
    int rc = check_common(P, b->n_models, b->total_sms, b->switch_max, b->slowdown, b->objective, b->p_idle_w,
                          b->p_max_w, o.tie_tol);
    if (rc) return rc;
    std::vector<TableSpec> specs;
    if ((rc = batch_specs(P, b, &specs))) return rc;
    auto pl = std::make_unique<eclip_planner>();
    pl->opt = o;
    pl->n_max = max_problems;
    pl->W = b->n_models; pl->N = b->total_sms; pl->R = b->switch_max; pl->mode = b->slowdown; pl->obj = b->objective;
    pl->pi = b->p_idle_w; pl->pm = b->p_max_w;
    pl->has_qos = b->qos_ns != nullptr;
    pl->has_w = b->weights != nullptr;
    pl->timing = o.timing != 0;
    for (auto& sp : specs) pl->mask.push_back(sp.mask);
    pl->s = std::make_unique<eclip_session>();
    eclip_session* s = pl->s.get();
    s->prof = P;
    s->W = pl->W; s->n = max_problems; s->C = P->C();
    if ((rc = setup_device(s, &o))) return rc;
    fill_setup(s, max_problems, pl->W, pl->N, pl->R, pl->mode, pl->obj, pl->has_qos, &o);
    s->su.weighted = pl->has_w ? 1 : 0;   // weights may differ from call to call: the weighted kernels
    if (pl->has_w && pl->obj == ECLIP_ENERGY)
        return fail(ECLIP_E_INVALID_ARG, "the ENERGY objective takes no per-worker weights");
    if ((rc = build_tables(s, specs))) return rc;   // K1 once (the only host synchronisation)
    {
        std::vector<int32_t> all(specs.size());
        for (size_t i = 0; i < all.size(); i++) all[i] = (int32_t)i;
        set_wide(s, all);
    }
    if ((rc = plan_geometry(s, &o))) return rc;
    if (s->engine != ECLIP_ENGINE_ENUM) return fail(ECLIP_E_TOO_LARGE, "batched planning runs on the ENUM engine only");
    if (s->su.aux_bytes > 0) {   // per-table S orders and hulls, kept for the planner's lifetime
        CU(s->arena.alloc(&s->wk.thull, (size_t)s->tb.n * s->su.Lmax));
        CU(s->arena.alloc(&s->wk.thull_n, (size_t)s->tb.n));
        CU(s->arena.alloc(&s->wk.tord, (size_t)s->tb.n * s->su.Lmax));
        CU(launch_table_hull(s->su, s->tb, s->wk, s->st));
    }
    const size_t nw = (size_t)max_problems * pl->W;
    CU(s->arena.alloc(&pl->d_ids, nw));
    if (pl->has_qos) CU(s->arena.alloc(&pl->d_qos, nw));
    if (pl->mode == ECLIP_MATRIX) CU(s->arena.alloc(&pl->d_M, nw * pl->W));
    if (pl->has_w) CU(s->arena.alloc(&pl->d_w, nw));
    CU(s->arena.alloc(&s->d_sizes, s->C));
    CU(cudaMemcpyAsync(s->d_sizes, P->sizes.data(), 4 * (size_t)s->C, cudaMemcpyHostToDevice, s->st));
    if ((rc = alloc_work(s, &pl->wb))) return rc;
    pl->stg.st = s->st;
    if (pl->timing)
        for (cudaEvent_t& e : pl->ev) CU(cudaEventCreate(&e));
    CU(cudaStreamSynchronize(s->st));
    *out = pl.release();
    return ECLIP_OK;
}

extern "C" int eclip_planner_plan(eclip_planner* pl, const eclip_batch* b, eclip_batch_out* out) {
    if (!pl || !b || !out) return fail(ECLIP_E_INVALID_ARG, "null argument");
    eclip_session* s = pl->s.get();
    const int n = b->n_problems, W = pl->W;
    if (n < 1 || n > pl->n_max) return fail(ECLIP_E_INVALID_ARG, "n_problems must be in [1, %d]", pl->n_max);
    if (b->n_models != W || b->total_sms != pl->N || b->switch_max != pl->R || b->slowdown != pl->mode ||
        b->objective != pl->obj || b->p_idle_w != pl->pi || b->p_max_w != pl->pm)
        return fail(ECLIP_E_INVALID_ARG, "batch settings differ from the planner's");
    if ((b->qos_ns != nullptr) != pl->has_qos)
        return fail(ECLIP_E_INVALID_ARG, pl->has_qos ? "this planner needs qos_ns" : "this planner was created without QoS");
    if ((b->weights != nullptr) != pl->has_w)
        return fail(ECLIP_E_INVALID_ARG, pl->has_w ? "this planner needs weights" : "this planner was created without weights");
    if (!b->model_ids || (pl->mode == ECLIP_MATRIX && !b->slowdown_matrix))
        return fail(ECLIP_E_INVALID_ARG, "null model_ids / slowdown_matrix");
    if (b->allowed_mask)
        for (size_t m = 0; m < pl->mask.size(); m++) {
            const uint32_t want = b->allowed_mask[m] & (s->C < 32 ? (1u << s->C) - 1u : 0xffffffffu);
            if (want != pl->mask[m]) return fail(ECLIP_E_INVALID_ARG, "allowed_mask differs from the planner's");
        }
    const size_t nw = (size_t)n * W;
    if (!b->on_device) {
        for (size_t i = 0; i < nw; i++) {
            if (b->model_ids[i] < 0 || b->model_ids[i] >= s->prof->n())
                return fail(ECLIP_E_INVALID_ARG, "model id %d out of range (problem %zu)", b->model_ids[i], i / W);
            if (b->qos_ns && !(b->qos_ns[i] >= 0.0)) return fail(ECLIP_E_INVALID_ARG, "qos_ns must be >= 0 or +inf");
        }
        bool unequal;
        int rcw = check_weights(b->weights, (size_t)n, W, pl->obj, &unequal);
        if (rcw) return rcw;
    }
    if (pl->timing) CU(cudaEventRecord(pl->ev[0], s->st));
    const int32_t* dtab = b->model_ids;
    const double* dq = b->qos_ns;
    const float* dM = b->slowdown_matrix;
    const double* dW = b->weights;
    if (!b->on_device) {   // inputs into the planner's device buffers (stream-ordered)
        CU(cudaMemcpyAsync(pl->d_ids, b->model_ids, 4 * nw, cudaMemcpyHostToDevice, s->st));
        if (pl->has_qos) CU(cudaMemcpyAsync(pl->d_qos, b->qos_ns, 8 * nw, cudaMemcpyHostToDevice, s->st));
        if (pl->d_M) CU(cudaMemcpyAsync(pl->d_M, b->slowdown_matrix, 4 * nw * W, cudaMemcpyHostToDevice, s->st));
        if (pl->d_w) CU(cudaMemcpyAsync(pl->d_w, b->weights, 8 * nw, cudaMemcpyHostToDevice, s->st));
        dtab = pl->d_ids; dq = pl->d_qos; dM = pl->d_M; dW = pl->d_w;
    }
    if (pl->timing) CU(cudaEventRecord(pl->ev[1], s->st));
    // geometry of this call's batch size (host arithmetic on the cached level counts; no sync)
    s->n = n;
    s->on_device = b->on_device != 0;
    s->su.n_problems = n;
    int rc = plan_geometry(s, &pl->opt);
    if (rc) return rc;
    if ((rc = alloc_work(s, &pl->wb))) return rc;
    s->pin.table_of = dtab; s->pin.qos = dq; s->pin.M = dM; s->pin.weights = dW;
    s->pin.p_idle = pl->pi; s->pin.p_max = pl->pm;
    s->wk.table_of = dtab;
    s->wk.tb = s->tb;
    CU(launch_prep(s->su, s->tb, s->pin, s->wk, s->C, s->d_sizes, s->st, /*table_hull=*/false));
    if (pl->timing) CU(cudaEventRecord(pl->ev[2], s->st));
    if ((rc = step_pass1(s))) return rc;
    if (pl->timing) CU(cudaEventRecord(pl->ev[3], s->st));
    CU(launch_pass2_both(s->su, s->wk, s->st));
    if (pl->timing) CU(cudaEventRecord(pl->ev[4], s->st));
    pl->ev_valid = false;
    if (b->on_device) {
        if ((rc = finish_batch(s, out))) return rc;
        if (pl->timing) CU(cudaEventRecord(pl->ev[5], s->st));
        if (s->own_stream) CU(cudaStreamSynchronize(s->st));
    } else {
        // finish_batch synchronises after the D2H copies: record the last event before it returns
        // by materialising through the staging block, then timing the copies with it
        if ((rc = finish_batch(s, out, nullptr, nullptr, &pl->stg))) return rc;
        if (pl->timing) CU(cudaEventRecord(pl->ev[5], s->st));
    }
    pl->ev_valid = pl->timing;
    return ECLIP_OK;
}

extern "C" int eclip_planner_phase_ms(eclip_planner* pl, float* ms, int32_t n) {
    if (!pl || !ms || n < 0) return fail(ECLIP_E_INVALID_ARG, "null argument");
    if (!pl->ev_valid) return fail(ECLIP_E_INVALID_ARG, "no timed plan (create the planner with opt->timing = 1)");
    CU(cudaEventSynchronize(pl->ev[5]));
    for (int i = 0; i < n; i++) {
        ms[i] = 0.0f;
        if (i < 5) CU(cudaEventElapsedTime(&ms[i], pl->ev[i], pl->ev[i + 1]));
    }
    return ECLIP_OK;
}

extern "C" int eclip_planner_counters(eclip_planner* pl, uint64_t* out, int32_t n) {
    if (!pl) return fail(ECLIP_E_INVALID_ARG, "null planner");
    return eclip_session_counters(pl->s.get(), out, n);
}

extern "C" void eclip_planner_free(eclip_planner* pl) { delete pl; }

static int plan_one(eclip_session* s, eclip_result* r, const uint64_t* first_override) {
    const int W = s->W;
    int gmax = 1;
    for (int w = 0; w < W; w++) gmax = std::max(gmax, s->tabs[s->h_table_of[w]].G);
    std::vector<int32_t> st(1), lv(W), sw(W), gsm((size_t)W * gmax);
    std::vector<uint64_t> idx(1), key(4);
    std::vector<double> obj(1), mk(1), pw(1), en(1), thr(1), eb(1), lat(W), glat((size_t)W * gmax);
    eclip_batch_out o{};
    o.energy_busy_j = eb.data();
    o.status = st.data(); o.winner_levels = lv.data(); o.winner_index = idx.data(); o.objective = obj.data();
    o.makespan_ns = mk.data(); o.power_w = pw.data(); o.energy_j = en.data(); o.throughput_rps = thr.data();
    o.model_latency_ns = lat.data(); o.model_switches = sw.data(); o.group_sm = gsm.data(); o.group_stride = gmax;
    if (first_override) CU(cudaMemcpyAsync(s->wk.first, first_override, 32, cudaMemcpyHostToDevice, s->st));
    int rc = finish_batch(s, &o, glat.data(), key.data());
    if (rc) return rc;
    r->status = st[0] == 0 ? ECLIP_OK : ECLIP_INFEASIBLE;
    r->engine_used = s->engine;
    r->objective = obj[0]; r->makespan_ns = mk[0]; r->power_w = pw[0]; r->energy_j = en[0];
    r->throughput_rps = thr[0]; r->winner_index = idx[0]; r->energy_busy_j = eb[0];
    for (int i = 0; i < 4; i++) r->exact_key[i] = key[i];
    long double totl = 1;
    for (int w = 0; w < W; w++) totl *= (long double)std::max(1, s->tabL[s->h_table_of[w]]);
    uint64_t total = totl < 1.8e19L ? (uint64_t)totl : ~0ull;   // all-ones: more than 2^64 tuples
    r->candidates = total;
    r->units_scored = s->engine == ECLIP_ENGINE_ENUM ? total : slice_units(s->slice);
    r->candidates_evaluated = 0;
    if (s->engine == ECLIP_ENGINE_ENUM && s->wk.feasible) {
        unsigned long long v = 0;
        CU(cudaMemcpy(&v, s->wk.feasible, sizeof v, cudaMemcpyDeviceToHost));
        r->candidates_evaluated = v;
    }
    size_t off = 0;
    for (int w = 0; w < W; w++) {
        int G = s->tabs[s->h_table_of[w]].G;
        if (r->model_latency_ns) r->model_latency_ns[w] = lat[w];
        if (r->model_switches) r->model_switches[w] = sw[w];
        if (r->winner_levels) r->winner_levels[w] = lv[w];
        for (int g = 0; g < G; g++) {
            if (r->group_sm) r->group_sm[off + g] = gsm[(size_t)w * gmax + g];
            if (r->group_latency_ns) r->group_latency_ns[off + g] = glat[(size_t)w * gmax + g];
        }
        off += G;
    }
    return ECLIP_OK;
}

extern "C" int eclip_session_create_problem(const eclip_profiles* prof, const eclip_problem* problem,
                                            const eclip_options* opt, eclip_session** out) {
    if (!out) return fail(ECLIP_E_INVALID_ARG, "null out");
    eclip_session* s = nullptr;
    int rc = session_from_problem(prof, problem, opt, &s);
    if (rc) { delete s; return rc; }
    host_mark("session_from_problem");
    if (s->engine == ECLIP_ENGINE_SLICE) {
        cudaError_t e = slice_setup(s->slice, s->su, s->tb, s->wk, s->tabL.data(), s->h_table_of.data(), s->st);
        if (e == cudaErrorNotSupported) {
            delete s;
            return fail(ECLIP_E_TOO_LARGE, "SLICE engine: weighted terms exceed its 64-bit exact DP; use ENUM");
        }
        if (e != cudaSuccess) { delete s; return fail(ECLIP_E_CUDA, "SLICE setup: %s", cudaGetErrorString(e)); }
    }
    *out = s;
    return ECLIP_OK;
}

extern "C" int eclip_session_finish_problem(eclip_session* s, const uint64_t* global_first_index, eclip_result* r) {
    if (!s || !r) return fail(ECLIP_E_INVALID_ARG, "null argument");
    return plan_one(s, r, global_first_index);
}

void eclip::host_mark(const char* label) {
    static const bool on = std::getenv("ECLIP_HOST_TIMING") != nullptr;
    static thread_local std::chrono::steady_clock::time_point t0;
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    if (!label) { t0 = t; return; }
    std::fprintf(stderr, "[eclip host] %-28s %9.1f us\n", label,
                 std::chrono::duration<double, std::micro>(t - t0).count());
}

extern "C" int eclip_plan(const eclip_profiles* prof, const eclip_problem* problem, const eclip_options* opt,
                          eclip_result* r) {
    if (!r) return fail(ECLIP_E_INVALID_ARG, "null result");
    host_mark(nullptr);
    eclip_session* s = nullptr;
    int rc = eclip_session_create_problem(prof, problem, opt, &s);
    if (rc) return rc;
    host_mark("session created");
    std::unique_ptr<eclip_session> guard(s);
    rc = run_all_steps(s);
    if (rc) return rc;
    host_mark("steps launched");
    rc = plan_one(s, r, nullptr);
    host_mark("result on host");
    return rc;
}

// ------------------------------------------------------------------------------------------
// level-table introspection (K1 output of one worker)
// ------------------------------------------------------------------------------------------
extern "C" int eclip_level_table(const eclip_profiles* P, int32_t model, const int32_t* gb, uint32_t mask, int32_t R,
                                 const eclip_options* opt, int32_t cap, int64_t* S, int64_t* B, uint8_t* wit,
                                 int32_t* n_levels, int32_t* n_groups) {
    if (!P || !n_levels || cap < 0) return fail(ECLIP_E_INVALID_ARG, "null argument");
    if (model < 0 || model >= P->n()) return fail(ECLIP_E_INVALID_ARG, "model %d out of range", model);
    if (R < 0) return fail(ECLIP_E_INVALID_ARG, "switch_max must be >= 0");
    if (cap > 0 && (!S || !B || !wit)) return fail(ECLIP_E_INVALID_ARG, "null output array");
    const int C = P->C(), K = P->nk[model];
    TableSpec sp;
    sp.model = model;
    sp.R = R;
    sp.mask = mask ? mask : ((C == 32) ? 0xffffffffu : ((1u << C) - 1u));
    if (C < 32) sp.mask &= (1u << C) - 1u;
    if (sp.mask == 0) return fail(ECLIP_E_INVALID_ARG, "no allowed size column");
    if (gb) {
        if (gb[0] != 0) return fail(ECLIP_E_INVALID_ARG, "group_bounds must start at 0");
        sp.bounds.push_back(0);
        for (int i = 1; sp.bounds.back() != K; i++) {
            if (gb[i] <= sp.bounds.back() || gb[i] > K) return fail(ECLIP_E_INVALID_ARG, "group_bounds must ascend to %d", K);
            sp.bounds.push_back(gb[i]);
        }
    } else {
        for (int k = 0; k <= K; k++) sp.bounds.push_back(k);
    }
    eclip_session s;   // device, stream, arena
    s.prof = P;
    int rc = setup_device(&s, opt);
    if (rc) return rc;
    rc = build_tables(&s, std::vector<TableSpec>{sp});
    if (rc) return rc;
    const int L = s.tabL[0], G = (int)sp.bounds.size() - 1;
    *n_levels = L;
    if (n_groups) *n_groups = G;
    if (L > cap) return cap == 0 ? ECLIP_OK : fail(ECLIP_E_INVALID_ARG, "cap %d < %d levels", cap, L);
    std::vector<const void*> ptr(3);
    CU(cudaMemcpyAsync(ptr.data(), s.tb.S, sizeof(void*), cudaMemcpyDeviceToHost, s.st));
    CU(cudaMemcpyAsync(ptr.data() + 1, s.tb.B, sizeof(void*), cudaMemcpyDeviceToHost, s.st));
    CU(cudaMemcpyAsync(ptr.data() + 2, s.tb.wit, sizeof(void*), cudaMemcpyDeviceToHost, s.st));
    CU(cudaStreamSynchronize(s.st));
    CU(cudaMemcpyAsync(S, ptr[0], 8 * (size_t)L, cudaMemcpyDeviceToHost, s.st));
    CU(cudaMemcpyAsync(B, ptr[1], 8 * (size_t)L, cudaMemcpyDeviceToHost, s.st));
    CU(cudaMemcpyAsync(wit, ptr[2], (size_t)L * G, cudaMemcpyDeviceToHost, s.st));
    CU(cudaStreamSynchronize(s.st));
    return ECLIP_OK;
}

// ------------------------------------------------------------------------------------------
// comparison planners and the lookup table
// ------------------------------------------------------------------------------------------
extern "C" int eclip_baseline_plan(const eclip_profiles* P, const eclip_problem* pr, int32_t kind, double param,
                                   const eclip_options* opt, eclip_result* r) {
    if (!pr || !r) return fail(ECLIP_E_INVALID_ARG, "null argument");
    const int W = pr->n_models;
    int rc = check_common(P, W, pr->total_sms, pr->switch_max, pr->slowdown, pr->objective, pr->p_idle_w, pr->p_max_w,
                          0.0);
    if (rc) return rc;
    if (!pr->model_ids) return fail(ECLIP_E_INVALID_ARG, "null model_ids");
    if (kind < ECLIP_BASELINE_ALL_MAX || kind > ECLIP_BASELINE_KERNEL_WISE)
        return fail(ECLIP_E_INVALID_ARG, "unknown baseline kind %d", kind);
    if (kind == ECLIP_BASELINE_KERNEL_WISE && !(param >= 0.0 && param <= 1e6))
        return fail(ECLIP_E_INVALID_ARG, "kernel-wise tolerance must be in [0, 1e6]");
    if (kind == ECLIP_BASELINE_MODEL_WISE && !(param >= 1.0 && param <= 1e6))
        return fail(ECLIP_E_INVALID_ARG, "model-wise latency factor must be in [1, 1e6]");
    std::vector<TableSpec> ws;
    rc = worker_specs(P, pr, &ws);
    if (rc) return rc;
    const int C = P->C();
    // same exact-arithmetic ranges as the optimizer (status -5 in k_prep_prob)
    uint64_t lam = 1;
    for (int w = 0; w < W; w++) {
        const uint64_t K = (uint64_t)P->nk[ws[w].model];
        lam = lam / (uint64_t)gcd64((int64_t)lam, (int64_t)K) * K;
        if (lam > ((uint64_t)1 << 40)) return fail(ECLIP_E_TOO_LARGE, "lcm of kernel counts too large");
    }
    if ((long double)lam * pr->total_sms * (W + 1) >= 4611686018427387904.0L)   // 2^62: int64 T' (baseline.cu)
        return fail(ECLIP_E_TOO_LARGE, "Lambda N (W+1) >= 2^62");
    for (int w = 0; w < W; w++) {
        int64_t bm = 0;
        for (int k = 0; k < P->nk[ws[w].model]; k++) {
            int64_t mx = 0;
            for (int j = 0; j < C; j++) mx = std::max(mx, P->row(ws[w].model, k)[j]);
            bm += mx;
        }
        if (bm >= ((int64_t)1 << 36)) return fail(ECLIP_E_TOO_LARGE, "worker %d: solo time exceeds 2^36 ns", w);
    }
    eclip_session s;   // stream + arena only
    s.prof = P;
    rc = setup_device(&s, opt);
    if (rc) return rc;
    BaseJob J{};
    J.W = W; J.C = C; J.N = pr->total_sms; J.mode = pr->slowdown; J.obj = pr->objective; J.kind = kind;
    J.den = 1000000000ull;
    J.num = (uint64_t)llround(param * 1e9);
    J.p_idle = pr->p_idle_w; J.p_max = pr->p_max_w;
    {
        bool unequal;
        if ((rc = check_weights(pr->weights, 1, W, pr->objective, &unequal))) return rc;
        for (int w = 0; w < W; w++) J.wv[w] = pr->weights ? (double)llround(pr->weights[w] * 1e6) / 1e6 : 1.0;
    }
    int gmax = 1;
    for (int w = 0; w < W; w++) gmax = std::max(gmax, (int)ws[w].bounds.size() - 1);
    int32_t* dsz;
    CU(s.arena.alloc(&dsz, C));
    CU(cudaMemcpyAsync(dsz, P->sizes.data(), 4 * C, cudaMemcpyHostToDevice, s.st));
    J.sizes = dsz;
    for (int w = 0; w < W; w++) {
        const int m = ws[w].model, K = P->nk[m];
        const int G = (int)ws[w].bounds.size() - 1;
        J.G[w] = G; J.K[w] = K; J.mask[w] = ws[w].mask;
        J.Q[w] = pr->qos_ns ? pr->qos_ns[w] : (double)INFINITY;
        int64_t* dex; int32_t* dgb;
        CU(s.arena.alloc(&dex, (size_t)K * C));
        CU(s.arena.alloc(&dgb, G + 1));
        CU(cudaMemcpyAsync(dex, P->row(m, 0), (size_t)K * C * 8, cudaMemcpyHostToDevice, s.st));
        CU(cudaMemcpyAsync(dgb, ws[w].bounds.data(), (size_t)(G + 1) * 4, cudaMemcpyHostToDevice, s.st));
        J.exec[w] = dex; J.bounds[w] = dgb;
    }
    if (pr->slowdown == ECLIP_MATRIX)
        for (int a = 0; a < W; a++)
            for (int b = 0; b < W; b++) J.M[a * MAXW_ENUM + b] = a == b ? 0.0f : pr->slowdown_matrix[a * W + b];
    // one device block for every output: status, switches, group_sm | scalars, latency, group_lat
    const size_t ni = 1 + (size_t)W + (size_t)W * gmax, nd = 5 + (size_t)W + (size_t)W * gmax;
    int32_t* di; double* dd;
    CU(s.arena.alloc(&di, ni));
    CU(s.arena.alloc(&dd, nd));
    BaseOut o{};
    o.status = di; o.switches = di + 1; o.group_sm = di + 1 + W; o.stride = gmax;
    o.scalars = dd; o.latency = dd + 5; o.group_lat = dd + 5 + W;
    CU(launch_baseline(J, o, s.st));
    std::vector<int32_t> hi(ni);
    std::vector<double> hd(nd);
    CU(cudaMemcpyAsync(hi.data(), di, ni * 4, cudaMemcpyDeviceToHost, s.st));
    CU(cudaMemcpyAsync(hd.data(), dd, nd * 8, cudaMemcpyDeviceToHost, s.st));
    CU(cudaStreamSynchronize(s.st));
    r->status = hi[0] == 0 ? ECLIP_OK : ECLIP_INFEASIBLE;
    r->engine_used = ECLIP_ENGINE_BASELINE;
    r->objective = hd[0]; r->makespan_ns = hd[1]; r->power_w = hd[2]; r->energy_j = hd[3]; r->throughput_rps = hd[4];
    r->winner_index = ~0ull;
    r->candidates = 1;
    r->units_scored = 1;
    r->candidates_evaluated = 0;
    for (int i = 0; i < 4; i++) r->exact_key[i] = 0;
    size_t off = 0;
    for (int w = 0; w < W; w++) {
        const int G = J.G[w];
        if (r->model_latency_ns) r->model_latency_ns[w] = hd[5 + w];
        if (r->model_switches) r->model_switches[w] = hi[1 + w];
        if (r->winner_levels) r->winner_levels[w] = -1;
        for (int g = 0; g < G; g++) {
            if (r->group_sm) r->group_sm[off + g] = hi[1 + W + (size_t)w * gmax + g];
            if (r->group_latency_ns) r->group_latency_ns[off + g] = hd[5 + W + (size_t)w * gmax + g];
        }
        off += G;
    }
    return ECLIP_OK;
}

// 64-bit FNV-1a (offset basis 0xcbf29ce484222325, prime 0x100000001b3)
static uint64_t fnv1a64(const std::string& s) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (unsigned char c : s) {
        h ^= c;
        h *= 0x100000001b3ull;
    }
    return h;
}

extern "C" int eclip_lookup_table_json(const eclip_profiles* P, const eclip_problem* pr, const int32_t* group_sm,
                                       char* buf, size_t cap, size_t* len, uint64_t* hash) {
    if (!P || !pr || !group_sm || !pr->model_ids) return fail(ECLIP_E_INVALID_ARG, "null argument");
    const int W = pr->n_models;
    if (W < 1 || W > MAXW) return fail(ECLIP_E_INVALID_ARG, "n_models must be in [1, %d]", MAXW);
    if (pr->slowdown < 0 || pr->slowdown > 3) return fail(ECLIP_E_INVALID_ARG, "unknown slowdown mode");
    std::vector<TableSpec> ws;
    int rc = worker_specs(P, pr, &ws);
    if (rc) return rc;
    static const char* names[4] = {"exclude_self", "paper", "excess", "matrix"};
    std::string body = "\"workers\":[";
    size_t off = 0;
    for (int w = 0; w < W; w++) {
        body += (w ? ",{\"worker_id\":" : "{\"worker_id\":") + std::to_string(w) + ",\"configs\":[";
        const std::vector<int32_t>& b = ws[w].bounds;
        bool first = true;
        for (size_t g = 0; g + 1 < b.size(); g++) {
            const int32_t c = group_sm[off + g];
            for (int k = b[g]; k < b[g + 1]; k++) {
                body += (first ? "" : ",") + std::to_string(c);
                first = false;
            }
        }
        off += b.size() - 1;
        body += "]}";
    }
    body += "]";
    const std::string meta_tail = "\"mode\":\"" + std::string(names[pr->slowdown]) + "\",\"switch_max\":" +
                                  std::to_string(pr->switch_max) + "}";
    const std::string canon = "{\"meta\":{" + meta_tail + "," + body + "}";
    const uint64_t h = fnv1a64(canon);
    char hx[32];
    snprintf(hx, sizeof hx, "0x%016llx", (unsigned long long)h);
    const std::string text = "{\"meta\":{\"hash\":\"" + std::string(hx) + "\"," + meta_tail + "," + body + "}";
    if (hash) *hash = h;
    if (len) *len = text.size();
    if (buf) {
        if (cap < text.size() + 1) return fail(ECLIP_E_INVALID_ARG, "buffer too small: need %zu bytes", text.size() + 1);
        memcpy(buf, text.c_str(), text.size() + 1);
    }
    return ECLIP_OK;
}

// ------------------------------------------------------------------------------------------
// batched co-location simulator (simulate.cu)
// ------------------------------------------------------------------------------------------
extern "C" int eclip_simulate(const eclip_sim_batch* b, const eclip_options* opt, eclip_sim_out* out) {
    if (!b || !out) return fail(ECLIP_E_INVALID_ARG, "null argument");
    const long long S = b->n_scenarios;
    const int W = b->n_workers, K = b->max_kernels, C = b->n_sizes, G = b->n_groups;
    if (S < 1 || W < 1 || W > 8 || K < 1 || C < 1 || C > 32 || G < 1 || G > 32 || b->total_sms < 1 ||
        b->n_requests < 1 || b->n_requests > 4096 || (b->mode != ECLIP_SIM_PREALLOC && b->mode != ECLIP_SIM_IOCTL))
        return fail(ECLIP_E_INVALID_ARG, "simulator batch sizes out of range");
    if (!b->n_kernels || !b->beta_ns || !b->table || !b->mask || !b->group_sm)
        return fail(ECLIP_E_INVALID_ARG, "null simulator input array");
    if (!out->throughput_rps || !out->p95_ns || !out->mean_ns || !out->makespan_ns || !out->energy_j ||
        !out->req_per_j || !out->barriers || !out->events)
        return fail(ECLIP_E_INVALID_ARG, "null simulator output array");
    if (!(b->oversub >= 1.0) || !(b->barrier_ns >= 0.0) || !(b->p_idle_w >= 0.0) || !(b->p_max_w >= b->p_idle_w) ||
        !(b->ioctl_lo_ns >= 0.0 && b->ioctl_mode_ns >= b->ioctl_lo_ns && b->ioctl_hi_ns >= b->ioctl_mode_ns) ||
        !std::isfinite(b->oversub + b->barrier_ns + b->p_max_w + b->ioctl_hi_ns))
        return fail(ECLIP_E_INVALID_ARG, "simulator overhead / power model out of range");
    for (int g = 0; g < G; g++)
        if (b->group_sm[g] < 0) return fail(ECLIP_E_INVALID_ARG, "group_sm must be >= 0");
    const uint32_t gbits = G == 32 ? 0xffffffffu : ((1u << G) - 1u);
    for (int i = 0; i < W * C; i++)
        if (b->mask[i] & ~gbits) return fail(ECLIP_E_INVALID_ARG, "mask %d uses groups beyond n_groups", i);
    for (long long i = 0; i < S * W; i++) {
        const int nk = b->n_kernels[i];
        if (nk < 1 || nk > K) return fail(ECLIP_E_INVALID_ARG, "n_kernels[%lld] must be in [1, max_kernels]", i);
        for (int k = 0; k < nk; k++) {
            const int j = b->table[i * K + k];
            if (j < 0 || j >= C) return fail(ECLIP_E_INVALID_ARG, "table entry out of range (scenario %lld)", i / W);
            const double v = b->beta_ns[(i * K + k) * C + j];
            if (!(std::isfinite(v) && v > 0.0)) return fail(ECLIP_E_INVALID_ARG, "beta_ns must be finite and > 0");
        }
    }
    eclip_session s;   // device, stream and arena only
    int rc = setup_device(&s, opt);
    if (rc) return rc;
    Bump bp;
    const size_t o_nk = bp.take<int32_t>(S * W), o_beta = bp.take<double>((size_t)S * W * K * C);
    const size_t o_tab = bp.take<int32_t>((size_t)S * W * K), o_mask = bp.take<uint32_t>((size_t)W * C);
    const size_t o_gsm = bp.take<int32_t>(G);
    const size_t o_out = bp.take<double>((size_t)S * (3 * W + 3)), o_int = bp.take<int32_t>((size_t)S * 2);
    const size_t o_ev = bp.take<long long>(S), o_lat = bp.take<double>((size_t)S * W * b->n_requests);
    unsigned char* base;
    CU(s.arena.alloc(&base, bp.off));
    CU(cudaMemcpyAsync(base + o_nk, b->n_kernels, 4 * (size_t)S * W, cudaMemcpyHostToDevice, s.st));
    CU(cudaMemcpyAsync(base + o_beta, b->beta_ns, 8 * (size_t)S * W * K * C, cudaMemcpyHostToDevice, s.st));
    CU(cudaMemcpyAsync(base + o_tab, b->table, 4 * (size_t)S * W * K, cudaMemcpyHostToDevice, s.st));
    CU(cudaMemcpyAsync(base + o_mask, b->mask, 4 * (size_t)W * C, cudaMemcpyHostToDevice, s.st));
    CU(cudaMemcpyAsync(base + o_gsm, b->group_sm, 4 * (size_t)G, cudaMemcpyHostToDevice, s.st));
    SimJob J{};
    J.S = S; J.W = W; J.K = K; J.C = C; J.G = G; J.N = b->total_sms; J.n_requests = b->n_requests;
    J.shared_default = b->shared_default ? 1 : 0; J.ioctl = b->mode == ECLIP_SIM_IOCTL;
    J.n_kernels = (const int32_t*)(base + o_nk); J.beta = (const double*)(base + o_beta);
    J.table = (const int32_t*)(base + o_tab); J.mask = (const uint32_t*)(base + o_mask);
    J.group_sm = (const int32_t*)(base + o_gsm);
    J.barrier_ns = b->barrier_ns; J.io_lo = b->ioctl_lo_ns; J.io_mode = b->ioctl_mode_ns; J.io_hi = b->ioctl_hi_ns;
    J.oversub = b->oversub; J.p_idle = b->p_idle_w; J.p_max = b->p_max_w; J.seed = b->seed;
    double* od = (double*)(base + o_out);
    SimOut o{};
    o.throughput_rps = od; o.p95_ns = od + S * W; o.mean_ns = od + 2 * S * W;
    o.makespan_ns = od + 3 * S * W; o.energy_j = od + 3 * S * W + S; o.req_per_j = od + 3 * S * W + 2 * S;
    o.barriers = (int32_t*)(base + o_int); o.status = o.barriers + S; o.events = (long long*)(base + o_ev);
    CU(launch_simulate(J, o, (double*)(base + o_lat), s.st));
    std::vector<int32_t> st(S);
    CU(cudaMemcpyAsync(out->throughput_rps, o.throughput_rps, 8 * (size_t)S * W, cudaMemcpyDeviceToHost, s.st));
    CU(cudaMemcpyAsync(out->p95_ns, o.p95_ns, 8 * (size_t)S * W, cudaMemcpyDeviceToHost, s.st));
    CU(cudaMemcpyAsync(out->mean_ns, o.mean_ns, 8 * (size_t)S * W, cudaMemcpyDeviceToHost, s.st));
    CU(cudaMemcpyAsync(out->makespan_ns, o.makespan_ns, 8 * (size_t)S, cudaMemcpyDeviceToHost, s.st));
    CU(cudaMemcpyAsync(out->energy_j, o.energy_j, 8 * (size_t)S, cudaMemcpyDeviceToHost, s.st));
    CU(cudaMemcpyAsync(out->req_per_j, o.req_per_j, 8 * (size_t)S, cudaMemcpyDeviceToHost, s.st));
    CU(cudaMemcpyAsync(out->barriers, o.barriers, 4 * (size_t)S, cudaMemcpyDeviceToHost, s.st));
    CU(cudaMemcpyAsync(out->events, o.events, 8 * (size_t)S, cudaMemcpyDeviceToHost, s.st));
    CU(cudaMemcpyAsync(st.data(), o.status, 4 * (size_t)S, cudaMemcpyDeviceToHost, s.st));
    CU(cudaStreamSynchronize(s.st));
    for (long long i = 0; i < S; i++)
        if (st[i] != 0) return fail(ECLIP_E_INVALID_ARG, "scenario %lld cannot progress (simulator deadlock)", i);
    return ECLIP_OK;
}
