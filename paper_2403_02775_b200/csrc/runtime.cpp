// Host runtime: error slots, streams, device info, config validation and the
// small C-ABI utilities. No compute happens here.
#include "runtime.hpp"

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <cstdio>
#include <mutex>
#include <cstdlib>
#include <unordered_map>
#include <unordered_set>

namespace ezq {

static std::atomic<int64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
static std::atomic<int64_t> g_ties{0}, g_tie_fallback{0};
void note_ties(int64_t resolved, int64_t fallback) {
    g_ties += resolved;
    g_tie_fallback += fallback;
}

namespace {

struct ProfRec {
    std::string family;
    cudaEvent_t a, b;
    double work;
};
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof;
std::atomic<int> g_prof_on{0};

struct ErrState {
    int code = 0;
    std::string msg;
    int64_t index = -1;
};
thread_local ErrState t_err;
thread_local int t_device = -1;
thread_local std::unordered_map<int, cudaStream_t> t_streams;
thread_local std::unordered_map<int, cudaStream_t> t_copy_streams;
thread_local std::unordered_map<int, cudaStream_t> t_d2h_streams;

std::mutex g_mu;
std::unordered_map<int, DeviceInfo> g_info;
std::unordered_map<int, bool> g_pool_ready;

}  // namespace

int prof_begin(const char* family, cudaStream_t st) {
    if (!g_prof_on.load()) return -1;
    ProfRec r;
    r.family = family;
    r.work = 0.0;
    cudaEventCreate(&r.a);
    cudaEventCreate(&r.b);
    cudaEventRecord(r.a, st);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.push_back(r);
    return static_cast<int>(g_prof.size()) - 1;
}

void prof_end(int token, cudaStream_t st, double work) {
    if (token < 0) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEventRecord(g_prof[token].b, st);
    g_prof[token].work = work;
}

int set_error(int code, const std::string& msg, int64_t index) {
    t_err.code = code;
    t_err.msg = msg;
    t_err.index = index;
    return code;
}

int clear_error() {
    t_err.code = 0;
    t_err.msg.clear();
    t_err.index = -1;
    return EZQ_OK;
}

int cuda_error(cudaError_t e, const char* where) {
    const int code = (e == cudaErrorMemoryAllocation) ? EZQ_ERR_OOM : EZQ_ERR_CUDA;
    return set_error(code, std::string("CUDA error ") + cudaGetErrorString(e) + " at " + where);
}

int bind_device(int* dev) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return set_error(EZQ_ERR_NO_DEVICE,
                         "no CUDA device available (the B200 engine has no CPU fallback)");
    }
    int d = t_device;
    if (d < 0) {
        EZQ_CK(cudaGetDevice(&d));
    } else {
        EZQ_CK(cudaSetDevice(d));
    }
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!g_pool_ready[d]) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
            g_pool_ready[d] = true;
        }
    }
    *dev = d;
    return EZQ_OK;
}

cudaStream_t thread_stream(int dev) {
    auto it = t_streams.find(dev);
    if (it != t_streams.end()) return it->second;
    cudaStream_t s = nullptr;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    t_streams[dev] = s;
    return s;
}

cudaStream_t d2h_stream(int dev) {
    auto it = t_d2h_streams.find(dev);
    if (it != t_d2h_streams.end()) return it->second;
    cudaStream_t s = nullptr;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    t_d2h_streams[dev] = s;
    return s;
}

cudaStream_t copy_stream(int dev) {
    auto it = t_copy_streams.find(dev);
    if (it != t_copy_streams.end()) return it->second;
    // Highest priority: the ingest kernel's CTAs are dispatched ahead of the
    // compute kernels' queued CTAs whenever an SM frees resources.
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStream_t s;
    cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi);
    t_copy_streams[dev] = s;
    return s;
}

const DeviceInfo& device_info(int dev) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_info.find(dev);
    if (it != g_info.end()) return it->second;
    DeviceInfo di;
    cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&di.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&di.smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, dev) == cudaSuccess) di.total_mem = prop.totalGlobalMem;
    else cudaGetLastError();
    return g_info[dev] = di;
}

std::string fmt_double(double v) { return std::to_string(v); }

bool trace_on() {
    static const bool on = std::getenv("EZQ_TRACE") != nullptr;
    return on;
}

void trace(const char* what, long long a) {
    if (!trace_on()) return;
    static const auto t0 = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[ezq %10.3f ms] %s %lld\n", ms, what, a);
}

namespace {
std::mutex g_pin_mu;
std::unordered_map<void*, size_t> g_pin_live;                  // ptr -> size
std::unordered_set<void*> g_malloc_live;                         // pageable fallback (no device)
std::unordered_map<size_t, std::vector<void*>> g_pin_free;     // size -> blocks
size_t g_pin_cached = 0;
constexpr size_t kPinCacheLimit = 16ull << 30;
}  // namespace

void* host_alloc(size_t bytes) {
    bytes = bytes ? bytes : 1;
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        auto it = g_pin_free.find(bytes);
        if (it != g_pin_free.end() && !it->second.empty()) {
            void* p = it->second.back();
            it->second.pop_back();
            g_pin_cached -= bytes;
            g_pin_live[p] = bytes;
            return p;
        }
    }
    void* p = nullptr;
    trace("host_alloc miss", static_cast<long long>(bytes));
    if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) {
        // No device (host-only codec use) or pinned memory exhausted:
        // pageable memory serves host artifacts just as well.
        cudaGetLastError();
        p = std::malloc(bytes);
        if (!p) return nullptr;
        std::lock_guard<std::mutex> lk(g_pin_mu);
        g_malloc_live.insert(p);
        return p;
    }
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_live[p] = bytes;
    return p;
}

void host_free(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (g_malloc_live.erase(p)) {
        std::free(p);
        return;
    }
    auto it = g_pin_live.find(p);
    if (it == g_pin_live.end()) return;
    const size_t bytes = it->second;
    g_pin_live.erase(it);
    if (g_pin_cached + bytes <= kPinCacheLimit) {
        g_pin_free[bytes].push_back(p);
        g_pin_cached += bytes;
    } else {
        cudaFreeHost(p);
    }
}

int validate_config(const ezq_config* c, std::string* msg) {
    if (c->bits < 2 || c->bits > 8) {
        *msg = "bits must be in [2, 8], got " + std::to_string(c->bits);
        return EZQ_ERR_INVALID_ARGUMENT;
    }
    if (!(c->sigma_n >= 0.0f) || !std::isfinite(c->sigma_n)) {
        *msg = "sigma_n must be finite and >= 0";
        return EZQ_ERR_INVALID_ARGUMENT;
    }
    if (!(c->lr > 0.0) || !std::isfinite(c->lr)) {
        *msg = "lr must be finite and > 0";
        return EZQ_ERR_INVALID_ARGUMENT;
    }
    if (!(c->beta1 >= 0.0 && c->beta1 < 1.0)) {
        *msg = "adam_beta1 must be in [0, 1)";
        return EZQ_ERR_INVALID_ARGUMENT;
    }
    if (!(c->beta2 >= 0.0 && c->beta2 < 1.0)) {
        *msg = "adam_beta2 must be in [0, 1)";
        return EZQ_ERR_INVALID_ARGUMENT;
    }
    if (!(c->eps > 0.0)) {
        *msg = "adam_eps must be > 0";
        return EZQ_ERR_INVALID_ARGUMENT;
    }
    if (c->steps < 0) {
        *msg = "steps must be >= 0";
        return EZQ_ERR_INVALID_ARGUMENT;
    }
    if (c->select_step < 0) {
        *msg = "select_step must be >= 0";
        return EZQ_ERR_INVALID_ARGUMENT;
    }
    return EZQ_OK;
}

void bias_tables(const ezq_config* c, std::vector<double>& h) {
    const int n = (c->steps > 0 ? c->steps : 0) + 1;
    h.assign(4 * static_cast<size_t>(n), 1.0);
    for (int t = 1; t < n; ++t) {
        // optimize.cpp:90-91 evaluates exactly these with glibc pow.
        h[t] = 1.0 - std::pow(c->beta1, static_cast<double>(t));
        h[n + t] = 1.0 - std::pow(c->beta2, static_cast<double>(t));
    }
    // correctly rounded reciprocals (IEEE division) for div_by_table
    for (int t = 0; t < 2 * n; ++t) h[2 * n + t] = 1.0 / h[t];
}

CfgDev make_cfg(const ezq_config* c, int mode, const double* bc_dev) {
    CfgDev d{};
    d.bits = c->bits;
    d.lmin = -(1 << (c->bits - 1)) + 1;
    d.lmax = 1 << (c->bits - 1);
    d.mode = mode;
    d.steps = c->steps;
    d.select = c->select;
    d.fixed_at = c->select_step < c->steps ? c->select_step : c->steps;
    d.sigma_n = c->sigma_n;
    d.guard = level_guard(d.lmax);
    d.guard_sat = level_guard_sat(d.lmin, d.lmax);
    d.sat_b = static_cast<float>(static_cast<double>(-d.lmin) / static_cast<double>(d.lmax - d.lmin));
    // EZQ_TIE_CAP (test aid, 0..kTieMax): fewer candidate slots send more
    // near-tie columns down the full reference-order fallback
    static const int tie_cap = [] {
        const char* e = std::getenv("EZQ_TIE_CAP");
        const int v = e ? std::atoi(e) : kTieMax;
        return v < 0 ? 0 : (v > kTieMax ? kTieMax : v);
    }();
    d.tie_cap = tie_cap;
    d.adam.b1 = c->beta1;
    d.adam.b2 = c->beta2;
    d.adam.c1 = 1.0 - c->beta1;
    d.adam.c2 = 1.0 - c->beta2;
    d.adam.lr = c->lr;
    d.adam.eps = c->eps;
    const int n = (c->steps > 0 ? c->steps : 0) + 1;
    d.bc1 = bc_dev;
    d.bc2 = bc_dev ? bc_dev + n : nullptr;
    d.rbc1 = bc_dev ? bc_dev + 2 * n : nullptr;
    d.rbc2 = bc_dev ? bc_dev + 3 * n : nullptr;
    return d;
}

// Device scratch blocks are recycled across calls: cudaMallocAsync of a
// size the pool has not seen maps fresh memory (tens to hundreds of ms for
// GB-sized arenas, measured on B200), which made repeated batch calls
// erratic. A returned block carries an event recorded on its last stream;
// the next user waits on it.
namespace {
struct CachedBlock {
    void* p;
    size_t bytes;
    int dev;
    cudaEvent_t ready;
};
std::mutex g_blk_mu;
std::vector<CachedBlock> g_blk_free;
size_t g_blk_cached = 0;
constexpr size_t kBlkCacheLimit = 12ull << 30;
}  // namespace

void* block_get(size_t need, cudaStream_t st, size_t* got) {
    int dev = 0;
    cudaGetDevice(&dev);
    {  // size classes: 8 per octave (>= 1 MB granules), so similar calls share blocks
        size_t gran = size_t(1) << 20;
        while (gran * 16 <= need) gran <<= 1;
        need = (need + gran - 1) / gran * gran;
    }
    {
        std::lock_guard<std::mutex> lk(g_blk_mu);
        int best = -1;
        for (int i = 0; i < static_cast<int>(g_blk_free.size()); ++i) {
            const CachedBlock& b = g_blk_free[i];
            if (b.dev != dev || b.bytes < need) continue;  // best fit: any cached block that is large enough
            if (best < 0 || b.bytes < g_blk_free[best].bytes) best = i;
        }
        if (best >= 0) {
            CachedBlock b = g_blk_free[best];
            g_blk_free.erase(g_blk_free.begin() + best);
            g_blk_cached -= b.bytes;
            cudaStreamWaitEvent(st, b.ready, 0);
            cudaEventDestroy(b.ready);
            *got = b.bytes;
            return b.p;
        }
    }
    void* p = nullptr;
    if (cudaMallocAsync(&p, need, st) != cudaSuccess) {
        cudaGetLastError();
        // release the cache and retry once
        std::vector<CachedBlock> drop;
        {
            std::lock_guard<std::mutex> lk(g_blk_mu);
            drop.swap(g_blk_free);
            g_blk_cached = 0;
        }
        for (auto& b : drop) {
            cudaStreamWaitEvent(st, b.ready, 0);
            cudaEventDestroy(b.ready);
            cudaFreeAsync(b.p, st);
        }
        if (cudaMallocAsync(&p, need, st) != cudaSuccess) return nullptr;
    }
    *got = need;
    return p;
}

void block_put(void* p, size_t bytes, cudaStream_t st) {
    if (!p) return;
    int dev = 0;
    cudaGetDevice(&dev);
    if (bytes > kBlkCacheLimit) {
        cudaFreeAsync(p, st);
        return;
    }
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventRecord(ev, st);
    std::vector<CachedBlock> evict;
    {
        std::lock_guard<std::mutex> lk(g_blk_mu);
        g_blk_free.push_back({p, bytes, dev, ev});
        g_blk_cached += bytes;
        while (g_blk_cached > kBlkCacheLimit && !g_blk_free.empty()) {  // oldest first
            evict.push_back(g_blk_free.front());
            g_blk_cached -= g_blk_free.front().bytes;
            g_blk_free.erase(g_blk_free.begin());
        }
    }
    for (auto& b : evict) {
        cudaStreamWaitEvent(st, b.ready, 0);
        cudaEventDestroy(b.ready);
        cudaFreeAsync(b.p, st);
    }
}

int Arena::allocate(cudaStream_t st) {
    owner_ = st;
    off_ = 0;
    if (need_ == 0) return EZQ_OK;
    base_ = static_cast<char*>(block_get(need_, st, &cap_));
    if (!base_) return cuda_error(cudaErrorMemoryAllocation, "arena allocation");
    return EZQ_OK;
}

void Arena::release(cudaStream_t st) {
    block_put(base_, cap_, st);
    base_ = nullptr;
}

Arena::~Arena() {
    if (base_) block_put(base_, cap_, owner_);
}

}  // namespace ezq

using namespace ezq;

extern "C" {

void ezq_config_default(ezq_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->bits = 4;
    c->sigma_n = 3.0f;
    c->lr = 1e-3;
    c->beta1 = 0.9;
    c->beta2 = 0.999;
    c->eps = 1e-8;
    c->steps = 200;
    c->select = EZQ_SELECT_BEST;
    c->select_step = 100;
    c->seed = 0;
}

int ezq_config_validate(const ezq_config* cfg) {
    std::string msg;
    const int s = validate_config(cfg, &msg);
    return s ? set_error(s, msg) : clear_error();
}

int ezq_last_error(char* msg, size_t cap, int64_t* index) {
    if (msg && cap) {
        std::strncpy(msg, t_err.msg.c_str(), cap - 1);
        msg[cap - 1] = 0;
    }
    if (index) *index = t_err.index;
    return t_err.code;
}

int ezq_device_count(int* n) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        c = 0;
    }
    *n = c;
    return clear_error();
}

int ezq_set_device(int device) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess || device < 0 || device >= c) {
        cudaGetLastError();
        return set_error(EZQ_ERR_NO_DEVICE, "invalid device " + std::to_string(device));
    }
    t_device = device;
    EZQ_CK(cudaSetDevice(device));
    return clear_error();
}

int ezq_synchronize(void) {
    int dev;
    if (int s = bind_device(&dev)) return s;
    EZQ_CK(cudaStreamSynchronize(thread_stream(dev)));
    return clear_error();
}

const char* ezq_version(void) { return "ezquant-b200 0.1.0 (sm_100a)"; }

int64_t ezq_kernel_launches(void) { return g_launches.load(); }

int ezq_tie_stats(int64_t* resolved, int64_t* fallback) {
    if (resolved) *resolved = g_ties.load();
    if (fallback) *fallback = g_tie_fallback.load();
    return EZQ_OK;
}

int ezq_profile_enable(int on) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto& r : g_prof) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    g_prof.clear();
    g_prof_on.store(on);
    return clear_error();
}

int ezq_profile_read(const char* family, double* ms, int64_t* launches, double* work) {
    *ms = 0.0;
    *launches = 0;
    *work = 0.0;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto& r : g_prof) {
        if (r.family != family) continue;
        EZQ_CK(cudaEventSynchronize(r.b));
        float t = 0.f;
        EZQ_CK(cudaEventElapsedTime(&t, r.a, r.b));
        *ms += t;
        *launches += 1;
        *work += r.work;
    }
    return clear_error();
}

void ezq_free(void* p) { std::free(p); }

int ezq_device_upload(const float* host, int64_t n, float** dev) {
    *dev = nullptr;
    int d;
    if (int s = bind_device(&d)) return s;
    float* p = nullptr;
    const size_t bytes = sizeof(float) * static_cast<size_t>(std::max<int64_t>(n, 1));
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        return set_error(EZQ_ERR_OOM, "device allocation of " + std::to_string(bytes) + " bytes failed");
    }
    if (n > 0) {
        const cudaError_t e = cudaMemcpy(p, host, sizeof(float) * n, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(p);
            return cuda_error(e, "ezq_device_upload");
        }
    }
    *dev = p;
    return clear_error();
}

void ezq_device_free(void* dev) {
    if (dev) cudaFree(dev);
}

int ezq_device_mem_info(size_t* free_bytes, size_t* total_bytes) {
    int d;
    if (int s = bind_device(&d)) return s;
    EZQ_CK(cudaMemGetInfo(free_bytes, total_bytes));
    return clear_error();
}

// ---- host scalar utilities (bookkeeping; identical arithmetic) -----------
double ezq_initial_scale(const float* x, int64_t n, const ezq_config* cfg) {
    double max_abs = 0.0;  // rtn.cpp:81-86
    for (int64_t i = 0; i < n; ++i) {
        const double a = std::fabs(static_cast<double>(x[i]));
        max_abs = (max_abs < a) ? a : max_abs;
    }
    if (max_abs == 0.0) return 1.0;
    return max_abs / static_cast<double>(1 << (cfg->bits - 1));
}

int ezq_adam_step(double* m, double* v, int64_t* t, double scale, double grad,
                  const ezq_config* c, double* out) {
    // optimize.cpp:86-94; volatile temporaries keep the host compiler from
    // contracting into FMAs so the result matches the device update.
    *t += 1;
    volatile double a = c->beta1 * *m;
    volatile double b = (1.0 - c->beta1) * grad;
    *m = a + b;
    volatile double p = (1.0 - c->beta2) * grad;
    volatile double q = p * grad;
    volatile double r = c->beta2 * *v;
    *v = r + q;
    const double mh = *m / (1.0 - std::pow(c->beta1, static_cast<double>(*t)));
    const double vh = *v / (1.0 - std::pow(c->beta2, static_cast<double>(*t)));
    volatile double num = c->lr * mh;
    const double upd = num / (std::sqrt(vh) + c->eps);
    const double updated = scale - upd;
    *out = updated < 1e-12 ? 1e-12 : updated;
    return clear_error();
}

int64_t ezq_packed_size(int64_t count, int bits) { return bits == 4 ? (count + 1) / 2 : count; }

int ezq_pack_levels(const int16_t* lv, int64_t n, int bits, uint8_t* out) {
    const int lmin = -(1 << (bits - 1)) + 1, lmax = 1 << (bits - 1);
    for (int64_t i = 0; i < n; ++i)  // rtn.cpp:127-131
        if (lv[i] < lmin || lv[i] > lmax)
            return set_error(EZQ_ERR_INVALID_ARGUMENT,
                             "level " + std::to_string(lv[i]) + " outside [" +
                                 std::to_string(lmin) + ", " + std::to_string(lmax) + "]");
    const int64_t nb = ezq_packed_size(n, bits);
    std::memset(out, 0, static_cast<size_t>(nb));
    if (bits == 4) {
        for (int64_t i = 0; i < n; ++i) {
            const uint8_t nib = static_cast<uint8_t>(lv[i] - lmin);
            if (i % 2 == 0)
                out[i / 2] = nib;
            else
                out[i / 2] |= static_cast<uint8_t>(nib << 4);
        }
    } else {
        for (int64_t i = 0; i < n; ++i) out[i] = static_cast<uint8_t>(lv[i] - lmin);
    }
    return clear_error();
}

int ezq_unpack_levels(const uint8_t* b, int64_t nbytes, int64_t count, int bits, int16_t* out) {
    if (count < 0) return set_error(EZQ_ERR_INVALID_ARGUMENT, "negative level count");
    const int64_t need = ezq_packed_size(count, bits);
    if (nbytes < need)  // rtn.cpp:153-157
        return set_error(EZQ_ERR_INVALID_ARGUMENT,
                         "packed buffer holds " + std::to_string(nbytes) + " bytes, need " +
                             std::to_string(need) + " for " + std::to_string(count) + " levels");
    const int lmin = -(1 << (bits - 1)) + 1;
    const int span = (1 << (bits - 1)) - lmin;
    if (bits == 4) {
        for (int64_t i = 0; i < count; ++i) {
            const uint8_t v = b[i / 2];
            out[i] = static_cast<int16_t>(lmin + ((i % 2 == 0) ? (v & 0x0f) : (v >> 4)));
        }
    } else {
        for (int64_t i = 0; i < count; ++i) {
            if (b[i] > span)
                return set_error(EZQ_ERR_INVALID_ARGUMENT,
                                 "packed byte " + std::to_string(b[i]) + " exceeds level span " +
                                     std::to_string(span),
                                 i);
            out[i] = static_cast<int16_t>(lmin + b[i]);
        }
    }
    return clear_error();
}

int ezq_dequantize_channel(const int16_t* lv, int64_t n, double scale, float* out) {
    if (!(scale > 0.0) || !std::isfinite(scale))
        return set_error(EZQ_ERR_INVALID_ARGUMENT,
                         "scale must be finite and > 0, got " + fmt_double(scale));
    for (int64_t i = 0; i < n; ++i)
        out[i] = static_cast<float>(scale * static_cast<double>(lv[i]));  // rtn.cpp:101-107
    return clear_error();
}

}  // extern "C"
