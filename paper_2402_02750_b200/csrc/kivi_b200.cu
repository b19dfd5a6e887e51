// C-ABI implementation of include/kivi_b200.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/kivi_b200.h"
#include "common.cuh"
#include "kernels_attend_fast.cuh"
#include "kernels_attend_gqa.cuh"
#include "kernels_attend_gqa_tc.cuh"
#include "kernels_attend_generic.cuh"
#include "kernels_quant.cuh"
#include "kernels_project.cuh"

using namespace kivi_b200;

namespace {

thread_local std::string g_last_error;

kivi_status fail(kivi_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

#define KIVI_CUDA(call)                                                                    \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) {                                                           \
            if (e_ == cudaErrorMemoryAllocation)                                           \
                return fail(KIVI_ERR_OOM, "%s: %s", #call, cudaGetErrorString(e_));       \
            return fail(KIVI_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_));          \
        }                                                                                  \
    } while (0)

#define KIVI_LAUNCHED()                                                                     \
    do {                                                                                    \
        cudaError_t e_ = cudaGetLastError();                                                \
        if (e_ != cudaSuccess) return fail(KIVI_ERR_CUDA, "launch: %s", cudaGetErrorString(e_)); \
    } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int64_t ceil_div(int64_t x, int64_t m) { return (x + m - 1) / m; }

int grid_for(int64_t n, int block = 256) {
    int64_t g = ceil_div(std::max<int64_t>(n, 1), block);
    return (int)std::min<int64_t>(g, 148LL * 32);
}

// RAII-less device buffer helper (the cache owns and frees them).
template <typename T>
cudaError_t dalloc(T** p, size_t count) {
    *p = nullptr;
    if (count == 0) return cudaSuccess;
    return cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
}

// Grow-only per-thread device scratch (standalone entry points): avoids
// cudaMalloc/cudaFree (which synchronises the device) on every call.
struct Scratch {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = 256;
        while (want < bytes) want <<= 1;
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    ~Scratch() {
        if (p) cudaFree(p);
    }
};
// One set per (host thread, device): a thread that drives several GPUs gets
// separate buffers on each.
constexpr int kMaxDevices = 64;
Scratch& scratch(int slot) {
    thread_local Scratch s[kMaxDevices][4];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = 0;
    return s[dev][slot];
}

}  // namespace

struct kivi_cache {
    kivi_config cfg{};
    int device = 0;
    int64_t n_units = 0;
    int64_t cap = 0;  // tokens per unit (multiple of R)
    int64_t l = 0;
    int64_t kres_cap = 0, vres_cap = 0;  // reference residual_capacity
    // Complete 32-row key tiles of the current ring window whose codes are
    // already in kcodes (quantized early by the fast append, see
    // append_flush_fast_kernel); reset at every flush, prefill and import.
    int64_t kq_done = 0;
    int attend_path = 0;
    CacheDev dev{};

    // workspaces (grown lazily)
    float* part_o = nullptr;
    int64_t part_cap = 0;
    float2* part_ml = nullptr;
    int64_t ml_cap = 0;
    float* scratch = nullptr;
    int64_t scratch_cap = 0;
    float* heads_buf = nullptr;  // per-head GQA route: q / out (/ weights) by head
    int64_t heads_cap = 0;
    // launch_fast(defer_combine): the merge left to the caller
    int64_t pending_nsub = 0;
    int pending_cmode = 0;
    float2* stats = nullptr;
    int64_t stats_cap = 0;
    // [B][body, tail, gqa_tc, small_fused, body_vimma, body 512, body_vimma 512,
    //     body 384, body_vimma 384]
    int fast_per_sm[9][9] = {};
    // staging for _host calls
    // host-path staging, double-buffered: call i uploads into stg[i & 1]
    // while call i-1's kernels may still read stg[(i-1) & 1]
    struct HostStage {
        float* q = nullptr;
        float* k = nullptr;
        float* v = nullptr;
        float* out = nullptr;
        float* w = nullptr;
        int64_t cap_q = 0, cap_out = 0, cap_k = 0, cap_v = 0, cap_w = 0;
        cudaEvent_t in_free = nullptr;   // staged inputs consumed by the kernels
        cudaEvent_t out_free = nullptr;  // staged result copied to the host
    } stg[2];
    int stg_i = 0;
    double* xfer = nullptr;  // export/import staging
    int64_t xfer_cap = 0;
    // host-buffer path: inputs are uploaded on a private copy stream so the
    // next call's upload overlaps this call's kernels
    cudaStream_t h2d = nullptr;
    // fast attend: the tail kernel runs on a side stream next to the body kernel
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int* work = nullptr;  // body kernels' dynamic item counters: a ring of WORK_SLOTS
    int64_t work_seq = 0; // body launches so far (slot = work_seq % WORK_SLOTS)
    cudaEvent_t ev_h2d_done = nullptr;  // staged inputs uploaded
    unsigned long long* small_sync = nullptr;  // [1 + n_units] single-launch decode counters
    unsigned long long small_gbar = 0;         // cumulative grid-barrier target
    unsigned int small_units = 0;              // cumulative per-unit item target
    cudaStream_t d2h = nullptr;         // result copies of the host path
    cudaEvent_t ev_out_ready = nullptr; // staged result written by the kernels

    // profiling
    bool profile = false;
    int profile_stride = 1;     // time every profile_stride-th attend launch
    int64_t profile_seq = 0;    // attend launches seen while profiling
    bool prof_now = false;      // the current attend launch is timed
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
    int64_t main_launches = 0;
    int64_t total_launches = 0;

    std::vector<cudaEvent_t> event_pool;
    cudaEvent_t take_event() {
        if (event_pool.empty()) {
            cudaEvent_t e = nullptr;
            cudaEventCreate(&e);
            return e;
        }
        cudaEvent_t e = event_pool.back();
        event_pool.pop_back();
        return e;
    }

    int64_t kg() const { return l - l % cfg.residual_length; }
    int64_t vg() const { return l - std::min<int64_t>(l, cfg.residual_length); }
};

namespace {

kivi_status validate_cfg(const kivi_config* cfg) {
    if (!cfg) return fail(KIVI_ERR_USAGE, "config is NULL");
    // QuantParams::validate (quantize.cpp:13-20)
    if (cfg->bits < 1 || cfg->bits > 8)
        return fail(KIVI_ERR_CONFIG, "bits must be in [1, 8], got %d", cfg->bits);
    if (cfg->group_size < 1)
        return fail(KIVI_ERR_CONFIG, "group_size must be >= 1, got %lld",
                    (long long)cfg->group_size);
    // CacheConfig::validate (kv_cache.cpp:7-21)
    if (cfg->residual_length < 1) return fail(KIVI_ERR_CONFIG, "residual_length must be >= 1");
    if (cfg->residual_length % cfg->group_size != 0)
        return fail(KIVI_ERR_CONFIG, "residual_length %lld must be divisible by group_size %lld",
                    (long long)cfg->residual_length, (long long)cfg->group_size);
    if (cfg->head_dim < 1 || cfg->head_dim % cfg->group_size != 0)
        return fail(KIVI_ERR_CONFIG, "head_dim %lld must be a positive multiple of group_size %lld",
                    (long long)cfg->head_dim, (long long)cfg->group_size);
    // Packed storage (quantize.cpp:173-176)
    if (!(cfg->bits == 1 || cfg->bits == 2 || cfg->bits == 4 || cfg->bits == 8))
        return fail(KIVI_ERR_CONFIG,
                    "packed storage requires bits in {1,2,4,8}; B=%d is fake-quant only", cfg->bits);
    return KIVI_OK;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

void free_cache_buffers(kivi_cache* h) {
    cudaFree(h->dev.kcodes);
    cudaFree(h->dev.kpairs);
    cudaFree(h->dev.vcodes);
    cudaFree(h->dev.vpairs);
    cudaFree(h->dev.kring);
    cudaFree(h->dev.vring);
    h->dev.kcodes = nullptr;
    h->dev.kpairs = nullptr;
    h->dev.vcodes = nullptr;
    h->dev.vpairs = nullptr;
    h->dev.kring = nullptr;
    h->dev.vring = nullptr;
}

struct Layout {
    int64_t cap, k_ustride, kp_ustride, v_ustride, vp_ustride, ring_ustride;
};

Layout make_layout(const kivi_config& cfg, int64_t capacity) {
    Layout L;
    const int64_t R = cfg.residual_length, G = cfg.group_size, d = cfg.head_dim, B = cfg.bits;
    L.cap = std::max<int64_t>(round_up(std::max<int64_t>(capacity, 1), R), R);
    const int64_t tiles = L.cap / G;
    L.k_ustride = round_up(ceil_div(tiles * d * G * B, 8), 256);
    L.kp_ustride = round_up(tiles * d, 32);
    L.v_ustride = round_up(ceil_div(L.cap * d * B, 8), 256);
    L.vp_ustride = round_up(L.cap * (d / G), 32);
    L.ring_ustride = round_up(R * d, 64);
    return L;
}

kivi_status alloc_cache_buffers(kivi_cache* h, const Layout& L, cudaStream_t st) {
    CacheDev& c = h->dev;
    const int64_t U = h->n_units;
    KIVI_CUDA(dalloc(&c.kcodes, (size_t)(U * L.k_ustride)));
    KIVI_CUDA(dalloc(&c.kpairs, (size_t)(U * L.kp_ustride)));
    KIVI_CUDA(dalloc(&c.vcodes, (size_t)(U * L.v_ustride)));
    KIVI_CUDA(dalloc(&c.vpairs, (size_t)(U * L.vp_ustride)));
    KIVI_CUDA(dalloc(&c.kring, (size_t)(U * L.ring_ustride)));
    KIVI_CUDA(dalloc(&c.vring, (size_t)(U * L.ring_ustride)));
    KIVI_CUDA(cudaMemsetAsync(c.kcodes, 0, (size_t)(U * L.k_ustride), st));
    KIVI_CUDA(cudaMemsetAsync(c.vcodes, 0, (size_t)(U * L.v_ustride), st));
    KIVI_CUDA(cudaMemsetAsync(c.kpairs, 0, sizeof(float2) * (size_t)(U * L.kp_ustride), st));
    KIVI_CUDA(cudaMemsetAsync(c.vpairs, 0, sizeof(float2) * (size_t)(U * L.vp_ustride), st));
    KIVI_CUDA(cudaMemsetAsync(c.kring, 0, sizeof(float) * (size_t)(U * L.ring_ustride), st));
    KIVI_CUDA(cudaMemsetAsync(c.vring, 0, sizeof(float) * (size_t)(U * L.ring_ustride), st));
    c.k_ustride = L.k_ustride;
    c.kp_ustride = L.kp_ustride;
    c.v_ustride = L.v_ustride;
    c.vp_ustride = L.vp_ustride;
    c.ring_ustride = L.ring_ustride;
    h->cap = L.cap;
    return KIVI_OK;
}

void init_dev_scalars(kivi_cache* h) {
    h->dev.bits = h->cfg.bits;
    h->dev.G = (int)h->cfg.group_size;
    h->dev.R = (int)h->cfg.residual_length;
    h->dev.d = (int)h->cfg.head_dim;
    h->dev.maxc = (1 << h->cfg.bits) - 1;
    h->dev.n_units = h->n_units;
}

uint64_t grouped_bytes(int64_t tokens, const kivi_config& cfg) {
    // reference grouped_bytes (kv_cache.cpp:110-115): packed bytes + 4 B per group
    const int64_t codes = tokens * cfg.head_dim;
    return (uint64_t)ceil_div(codes * cfg.bits, 8) + 4ull * (uint64_t)(codes / cfg.group_size);
}

template <typename T>
kivi_status ensure(T** p, int64_t* cap, int64_t need) {
    if (need <= *cap) return KIVI_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    KIVI_CUDA(dalloc(p, (size_t)need));
    *cap = need;
    return KIVI_OK;
}

kivi_status ensure_capacity(kivi_cache* h, int64_t tokens, cudaStream_t st) {
    if (tokens <= h->cap) return KIVI_OK;
    return kivi_cache_reserve(h, std::max<int64_t>(tokens, 2 * h->cap), st);
}

// The fast kernels move caller rows as 16-byte vectors and TMA bulk copies:
// they need 16-byte aligned row pointers (d = 128 keeps every row aligned).
bool al16(const void* a, const void* b = nullptr, const void* c = nullptr,
          const void* d = nullptr, const void* e = nullptr) {
    return ((((uintptr_t)a | (uintptr_t)b | (uintptr_t)c | (uintptr_t)d | (uintptr_t)e) & 15) == 0);
}

bool fast_supported(const kivi_cache* h, int qpk) {
    const kivi_config& c = h->cfg;
    if (c.head_dim != 128 || c.group_size != 32) return false;
    if (qpk == 1) return c.bits == 2 || c.bits == 4;
    return c.bits == 2 && (qpk == 2 || qpk == 4);  // GQA kernel
}

// Tuning knobs (read once): KIVI_TAIL_SIDE=0 runs the tail kernel on the
// caller's stream before the body; KIVI_TAIL_CTAS sets its CTAs per SM.
int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}

// Routing / tuning knobs, read from the environment once per process and
// again on kivi_reload_tuning() (tests flip them between cases).  Defaults are
// the measured-best settings.
struct Tuning {
    int fused_append, tail_side, small_items, small_fused, small_sub, combine_parallel;
    int tail_sub, res_sub, res_sub_body, mha_tc, pdl, tail_ctas, tail_warp_ctas, tail_last;
    int gqa_tc, gqa_partial, gqa_tail_ctas, step_graph, zero_copy_bytes, proj_split, vimma;
    int body_prefetch, body_long_l, gqa_heads, step_fuse, body_sub, gqa_item;
    void load() {
        fused_append = env_int("KIVI_FUSED_APPEND", 0);
        tail_side = env_int("KIVI_TAIL_SIDE", 1);
        small_items = env_int("KIVI_SMALL_ITEMS", 1);
        small_fused = env_int("KIVI_SMALL_FUSED", 0);
        small_sub = env_int("KIVI_SMALL_SUB", 0);
        combine_parallel = env_int("KIVI_COMBINE_PARALLEL", -1);
        tail_sub = env_int("KIVI_TAIL_SUB", 256);
        res_sub = env_int("KIVI_RES_SUB", 32);
        res_sub_body = env_int("KIVI_RES_SUB_BODY", 0);
        mha_tc = env_int("KIVI_MHA_TC", 0);
        pdl = env_int("KIVI_PDL", 1);
        tail_ctas = env_int("KIVI_TAIL_CTAS", 1);
        tail_warp_ctas = env_int("KIVI_TAIL_WARP_CTAS", 0);
        tail_last = env_int("KIVI_TAIL_LAST", 0);
        gqa_tc = env_int("KIVI_GQA_TC", 1);
        gqa_partial = env_int("KIVI_GQA_PARTIAL", 1);
        gqa_tail_ctas = env_int("KIVI_GQA_TAIL_CTAS", 8);
        step_graph = env_int("KIVI_STEP_GRAPH", -1);  // -1: single-layer host steps only
        body_prefetch = env_int("KIVI_BODY_PREFETCH", 0);
        body_long_l = env_int("KIVI_BODY_LONG_L", 16384);
        gqa_heads = env_int("KIVI_GQA_HEADS", 1);
        step_fuse = env_int("KIVI_STEP_FUSE", 1);
        body_sub = env_int("KIVI_BODY_SUB", -1);
        gqa_item = env_int("KIVI_GQA_ITEM", 256);
        zero_copy_bytes = env_int("KIVI_ZERO_COPY_BYTES", 65536);
        proj_split = env_int("KIVI_PROJ_SPLIT", 2);
        vimma = env_int("KIVI_VIMMA", 1);
    }
};
Tuning g_tune;
bool g_tune_loaded = false;
const Tuning& tune() {
    if (!g_tune_loaded) {
        g_tune.load();
        g_tune_loaded = true;
    }
    return g_tune;
}

int g_num_sms[kMaxDevices] = {};
// SM count of the current device (callers hold a DeviceGuard for the cache).
int num_sms() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = 0;
    if (!g_num_sms[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        g_num_sms[dev] = n > 0 ? n : 148;
    }
    return g_num_sms[dev];
}

// Whether kivi_decode may fold this step's append into the residual-window
// kernel (the cache holds l tokens; the decision uses the geometry after the
// append, as launch_fast will).
bool fused_append_ok(const kivi_cache* h, int q_per_kv) {
    // off by default: measured C2 8.73 vs 8.49 ms/step (the append lengthens the
    // residual items, which sit on the critical path); read per call (tests flip it)
    const int on = tune().fused_append;
    const int tail_side = tune().tail_side;
    const kivi_config& c = h->cfg;
    if (!on || !tail_side || q_per_kv != 1 || h->attend_path == 1) return false;
    if (c.head_dim != 128 || c.group_size != 32 || (c.bits != 2 && c.bits != 4)) return false;
    const int64_t l = h->l + 1, R = c.residual_length;
    const int64_t vg = l - std::min(l, R);
    const bool latency_bound =
        tune().small_items && h->n_units * ceil_div(l, fast::BSUB) < 4 * num_sms();
    return !latency_bound && vg > 0 && ((vg - 1) / 32 * 32) / fast::BSUB > 0;
}

// Few units (the latency-bound route): one cooperative launch appends,
// attends and merges (no append / combine launches).
bool small_fused_ok(const kivi_cache* h, int q_per_kv) {
    const kivi_config& c = h->cfg;
    // off by default: measured slower on C1 (51.6 vs 22.1 + append + combine us):
    // the grid barrier and the last-warp merges serialise latency-bound phases
    if (!tune().small_fused || q_per_kv != 1 || h->attend_path == 1) return false;
    if (c.head_dim != 128 || c.group_size != 32 || (c.bits != 2 && c.bits != 4)) return false;
    const int64_t l = h->l + 1;
    return tune().small_items && h->n_units * ceil_div(l, fast::BSUB) < 4 * num_sms();
}

template <int B>
kivi_status launch_small_fused(kivi_cache* h, const float* q, const float* tk, const float* tv,
                               float* out, float* weights, float qscale, int64_t l_app,
                               cudaStream_t st) {
    const int64_t U = h->n_units;
    const int tsub = std::max(32, std::min(fast::SUB, tune().small_sub > 0 ? tune().small_sub : 64) / 32 * 32);
    const int64_t n_sub = ceil_div(h->l, tsub);
    if (h->l >= (1LL << 30) || U * n_sub >= (1LL << 30))
        return fail(KIVI_ERR_CONFIG, "fast attend path: cache too large for 32-bit indexing");
    const int64_t n_sub_cap = std::max<int64_t>(n_sub, ceil_div(h->cap, tsub) + 2);
    kivi_status rc = ensure(&h->part_o, &h->part_cap, U * n_sub_cap * fast::D);
    if (rc) return rc;
    rc = ensure(&h->part_ml, &h->ml_cap, U * n_sub_cap);
    if (rc) return rc;
    rc = ensure(&h->stats, &h->stats_cap, U);
    if (rc) return rc;
    if (!h->small_sync) {
        KIVI_CUDA(dalloc(&h->small_sync, (size_t)(1 + U)));
        KIVI_CUDA(cudaMemsetAsync(h->small_sync, 0, sizeof(unsigned long long) * (1 + U), st));
    }
    const int smem = fast::WS2::STRIDE * fast::WARPS;
    // per cache (so per device): the attribute must be set on each device
    int& per_sm = h->fast_per_sm[B][3];
    if (!per_sm) {
        KIVI_CUDA(cudaFuncSetAttribute(fast::attend_tail_kernel<B, fast::WARPS, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        KIVI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, fast::attend_tail_kernel<B, fast::WARPS, true>, fast::WARPS * 32, smem));
        if (per_sm < 1) per_sm = 1;
    }
    fast::FastArgs a{};
    a.c = h->dev;
    a.l = (int)h->l;
    a.kg = (int)h->kg();
    a.vg = (int)h->vg();
    a.n_sub = (int)n_sub;
    a.k_first = 0;
    a.t_first = 0;
    a.sub = tsub;
    a.n_per_unit = (int)n_sub;
    a.n_items = (int)(U * n_sub);
    a.q = q;
    a.qscale = qscale;
    a.part_o = h->part_o;
    a.part_ml = h->part_ml;
    a.wlog = weights;
    a.tk = tk;
    a.tv = tv;
    a.l_app = (int)l_app;
    const int64_t grid = std::min<int64_t>((int64_t)num_sms() * per_sm,
                                           std::max<int64_t>(ceil_div(a.n_items, fast::WARPS),
                                                             ceil_div(U, fast::WARPS)));
    h->small_gbar += (unsigned long long)(grid * fast::WARPS);
    h->small_units += (unsigned int)n_sub;
    a.gbar = h->small_sync;
    a.gbar_target = h->small_gbar;
    a.unit_done = reinterpret_cast<unsigned int*>(h->small_sync + 1);
    a.unit_target = h->small_units;
    a.out = out;
    a.stats = weights ? h->stats : nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    h->prof_now = h->profile && (h->profile_seq++ % h->profile_stride == 0);
    if (h->prof_now) {
        e0 = h->take_event();
        e1 = h->take_event();
        cudaEventRecord(e0, st);
    }
    void* args[] = {&a};
    KIVI_CUDA(cudaLaunchCooperativeKernel((const void*)fast::attend_tail_kernel<B, fast::WARPS, true>, dim3((unsigned)grid),
                                          dim3(fast::WARPS * 32), args, (size_t)smem, st));
    KIVI_LAUNCHED();
    if (h->prof_now) {
        cudaEventRecord(e1, st);
        h->events.emplace_back(e0, e1);
        h->main_launches++;
    }
    h->total_launches++;
    if (weights) {
        fast::normalize_weights_kernel<<<grid_for(U * h->l), 256, 0, st>>>(weights, h->stats, h->l,
                                                                            U);
        KIVI_LAUNCHED();
        h->total_launches++;
    }
    return KIVI_OK;
}

// Body kernels take items from a counter: launch i uses slot i % WORK_SLOTS
// and zeroes slot (i + WORK_SLOTS/2) % WORK_SLOTS for a later launch (that
// slot's last user finished WORK_SLOTS/2 launches ago), so no memset sits
// between the kernels of a decode step.
constexpr int WORK_SLOTS = 64;
static void take_work_slot(kivi_cache* h, fast::FastArgs& a) {
    const int s = (int)(h->work_seq++ % WORK_SLOTS);
    a.work = h->work + s;
    a.work_clear = h->work + (s + WORK_SLOTS / 2) % WORK_SLOTS;
}

// K5 variant: the parallel-over-partials merge (weights computed once per
// partial, then independent loads) measured faster at every config with the
// partials L2-resident after the attend (C1 7.4 vs 12.8 us, C2 8.9 vs 10.0,
// C3 17.7 vs 21.8, C5 13.2 vs 20.7 us per layer); KIVI_COMBINE_PARALLEL=0
// selects the serial per-channel merge.
// K5 merge mode: 0 one serial loop per thread, 1 block-parallel over the
// partials, 2 one warp per row (KIVI_COMBINE_PARALLEL).
// Default (-1): warp per row from 4096 rows (C3: +0.6 % per step; C2, 2048
// rows: neutral; C1, 32 rows: 14 % slower), block-parallel below.
static int combine_parallel(int64_t rows) {
    const int force = tune().combine_parallel;
    if (force >= 0) return force;
    return rows >= 4096 ? 2 : 1;
}

// Launch with programmatic stream serialization (kernel must pdl_wait()
// before reading what the previous kernel in the stream writes).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Tokens per body item.  KIVI_BODY_SUB = 256 / 384 / 512 fixes it; -1 (auto):
// the largest item size whose whole items cover [0, floor32(vg)) within 2 %
// of the best size (what they leave goes to the residual-window kernel);
// larger items = fewer items, less per-item work.  C2 / C4 (vg ~ 3968) ->
// 384 (attend -1.9 %), C5 (vg = 32640) -> 512 (-2.4 %).  -2: the earlier
// rule, 512 from KIVI_BODY_LONG_L tokens, else 256.
static int body_item_tokens(const kivi_cache* h, int64_t body_vg, int64_t l_app) {
    if (l_app >= 0 || tune().mha_tc) return fast::BSUB;
    const int fixed = tune().body_sub;
    if (fixed == 256 || fixed == 384 || fixed == 512) return fixed;
    if (fixed == -2) {
        const int long_l = tune().body_long_l;
        return (long_l > 0 && h->l >= long_l) ? 512 : fast::BSUB;
    }
    const int64_t span = (body_vg / 32) * 32;
    int64_t best_cover = 0;
    for (int bs : {256, 384, 512}) best_cover = std::max(best_cover, (span / bs) * bs);
    // the largest item whose whole items cover within 2 % of the best
    for (int bs : {512, 384}) {
        const int64_t cover = (span / bs) * bs;
        if (cover > 0 && 50 * (best_cover - cover) <= span) return bs;
    }
    return fast::BSUB;
}

template <int B>
kivi_status launch_fast(kivi_cache* h, const float* q, float* out, float* weights, float qscale,
                        cudaStream_t st, const float* tk = nullptr, const float* tv = nullptr,
                        int64_t l_app = -1, bool defer_combine = false) {
    const int64_t U = h->n_units;
    // Items: body = whole BSUB-token sub-chunks below floor32(vg) (all keys and
    // values quantized); tail = TSUB-token items over [nfull * BSUB, l), which
    // hold the fp32 residual rows.  One partial slot per item.
    const int tsub_env = std::max(32, std::min(fast::SUB, tune().tail_sub) / 32 * 32);
    // few-unit route item size: KIVI_SMALL_SUB, or (0, default) sized so the
    // items below the residual window about fill the resident warps once
    // (C1: 32 units x 3968 tokens / 1776 warps -> 96 tokens; 64 measured
    // 18.3 us, 96 16.2 us, 128 18.0 us)
    const int tsub_small_env = tune().small_sub;
    static const int tsub_small_min = 32;
    const int64_t res_warps = (int64_t)num_sms() * 3 * fast::WARPS;  // tail kernel: 3 CTAs / SM
    const int tsub_small =
        tsub_small_env > 0
            ? (int)std::max<int64_t>(32, std::min<int64_t>(fast::SUB, tsub_small_env) / 32 * 32)
            : (int)std::min<int64_t>(fast::SUB,
                                     std::max<int64_t>(tsub_small_min,
                                                       ceil_div(ceil_div(U * std::max<int64_t>(h->vg(), 1),
                                                                         res_warps), 32) * 32));
    // Few units (e.g. one sequence's 32 heads): 256-token body items leave
    // most warps idle and the per-unit residual item becomes the critical
    // path, so every token goes through tsub-token items instead.
    const int small_items = tune().small_items;
    const bool latency_bound = small_items && U * ceil_div(h->l, fast::BSUB) < 4 * num_sms();
    // fused append: the body must not cover the token the append pops into the
    // quantized store (token vg - 1), so it stops at floor32(vg - 1)
    const int64_t body_vg = l_app >= 0 ? h->vg() - 1 : h->vg();
    // body item size: 512 tokens from KIVI_BODY_LONG_L tokens (default 16384;
    // 0 disables), where the wider residual region is a small share
    const int bsub = body_item_tokens(h, body_vg, l_app);
    const int64_t nfull = latency_bound ? 0 : ((body_vg / 32) * 32) / bsub;
    if (l_app >= 0 && (latency_bound || nfull == 0))
        return fail(KIVI_ERR_USAGE, "internal: fused append outside its route");
    const int64_t t_first = nfull * bsub;
    const int tsub = latency_bound ? tsub_small : tsub_env;
    // few-unit route: the residual window [floor32(vg), l) in rsub-token items
    const int rsub_env = tune().res_sub / 32 * 32;
    // (KIVI_RES_SUB_BODY=1: on the body route too; measured slower on C2,
    // within noise on C5)
    const bool rsub_body = tune().res_sub_body != 0;
    const int rsub = ((latency_bound || rsub_body) && l_app < 0 && rsub_env > 0) ? rsub_env : 0;
    const int64_t t_b = rsub ? (h->vg() / 32) * 32 : h->l;
    const int64_t n_a = ceil_div(t_b - t_first, tsub);
    const int64_t n_b = rsub ? ceil_div(h->l - t_b, rsub) : 0;
    const int64_t n_sub = nfull + n_a + n_b;
    if (h->l >= (1LL << 30) || U * n_sub >= (1LL << 30))
        return fail(KIVI_ERR_CONFIG, "fast attend path: cache too large for 32-bit indexing");
    // partials sized for the reserved capacity: growing them mid-decode would
    // cudaFree (a device-wide sync) inside a serving loop
    const int64_t n_sub_cap = std::max<int64_t>(
        n_sub, ceil_div(h->cap, std::min(tsub_env, tsub_small_min)) + 2 +
                   (rsub_env > 0 ? ceil_div(h->cfg.residual_length + 32, std::max(rsub_env, 32)) : 0));
    kivi_status rc = ensure(&h->part_o, &h->part_cap, U * n_sub_cap * fast::D);
    if (rc) return rc;
    rc = ensure(&h->part_ml, &h->ml_cap, U * n_sub_cap);
    if (rc) return rc;
    rc = ensure(&h->stats, &h->stats_cap, U);
    if (rc) return rc;

    fast::FastArgs a{};
    a.l_app = -1;
    a.c = h->dev;
    a.l = (int)h->l;
    a.kg = (int)h->kg();
    a.vg = (int)h->vg();
    a.n_sub = (int)n_sub;
    a.q = q;
    a.qscale = qscale;
    a.part_o = h->part_o;
    a.part_ml = h->part_ml;
    a.wlog = weights;

    const int smem = fast::WS2::STRIDE * fast::WARPS;
    // P.V of the body on the integer tensor cores (2-bit; kernels_vimma.cuh)
    const bool vimma = B == 2 && tune().vimma;
    const int bidx = bsub == 512 ? 1 : (bsub == 384 ? 2 : 0);
    const int smem_body =
        (bidx == 1 ? (vimma ? fast::WarpSmemBody<true, 512>::STRIDE : fast::WarpSmemBody<false, 512>::STRIDE)
         : bidx == 2 ? (vimma ? fast::WarpSmemBody<true, 384>::STRIDE : fast::WarpSmemBody<false, 384>::STRIDE)
                     : (vimma ? fast::WarpSmemBody<true>::STRIDE : fast::WSB::STRIDE)) *
        fast::WARPS;
    void (*body_kernel)(fast::FastArgs) =
        bidx == 1 ? fast::attend_body_kernel<B, false, 512>
                  : (bidx == 2 ? fast::attend_body_kernel<B, false, 384> : fast::attend_body_kernel<B>);
    if constexpr (B == 2)
        if (vimma)
            body_kernel = bidx == 1 ? fast::attend_body_kernel<2, true, 512>
                                    : (bidx == 2 ? fast::attend_body_kernel<2, true, 384>
                                                 : fast::attend_body_kernel<2, true>);
    const int smem_tc = gqa_tc::TS<1>::STRIDE * gqa_tc::WARPS;
    const int mha_tc = tune().mha_tc;  // measured slower on C2
    if (h->fast_per_sm[B][0] == 0) {
        KIVI_CUDA(cudaFuncSetAttribute(gqa_tc::attend_gqa_tc_kernel<1>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem_tc));
        int tc_per_sm = 0;
        KIVI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &tc_per_sm, gqa_tc::attend_gqa_tc_kernel<1>, gqa_tc::WARPS * 32, smem_tc));
        h->fast_per_sm[B][2] = tc_per_sm < 1 ? 1 : tc_per_sm;
        KIVI_CUDA(cudaFuncSetAttribute(fast::attend_body_kernel<B>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem_body));
        KIVI_CUDA(cudaFuncSetAttribute(fast::attend_tail_kernel<B>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        KIVI_CUDA(cudaFuncSetAttribute(fast::attend_tail_kernel<B, fast::WARPS, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        KIVI_CUDA(cudaFuncSetAttribute(fast::attend_tail_kernel<B, 1>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       fast::WS2::STRIDE));
        int per_sm = 0;
        KIVI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, fast::attend_body_kernel<B>, fast::WARPS * 32,
            fast::WSB::STRIDE * fast::WARPS));
        h->fast_per_sm[B][0] = per_sm < 1 ? 1 : per_sm;
        if constexpr (B == 2) {
            const int smem_vi = fast::WarpSmemBody<true>::STRIDE * fast::WARPS;
            KIVI_CUDA(cudaFuncSetAttribute(fast::attend_body_kernel<2, true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem_vi));
            KIVI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &per_sm, fast::attend_body_kernel<2, true>, fast::WARPS * 32, smem_vi));
            h->fast_per_sm[B][4] = per_sm < 1 ? 1 : per_sm;
            const int smem_vi5 = fast::WarpSmemBody<true, 512>::STRIDE * fast::WARPS;
            KIVI_CUDA(cudaFuncSetAttribute(fast::attend_body_kernel<2, true, 512>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem_vi5));
            KIVI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &per_sm, fast::attend_body_kernel<2, true, 512>, fast::WARPS * 32, smem_vi5));
            h->fast_per_sm[B][6] = per_sm < 1 ? 1 : per_sm;
            const int smem_vi3 = fast::WarpSmemBody<true, 384>::STRIDE * fast::WARPS;
            KIVI_CUDA(cudaFuncSetAttribute(fast::attend_body_kernel<2, true, 384>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem_vi3));
            KIVI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &per_sm, fast::attend_body_kernel<2, true, 384>, fast::WARPS * 32, smem_vi3));
            h->fast_per_sm[B][8] = per_sm < 1 ? 1 : per_sm;
        }
        {
            const int smem5 = fast::WarpSmemBody<false, 512>::STRIDE * fast::WARPS;
            KIVI_CUDA(cudaFuncSetAttribute(fast::attend_body_kernel<B, false, 512>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem5));
            KIVI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &per_sm, fast::attend_body_kernel<B, false, 512>, fast::WARPS * 32, smem5));
            h->fast_per_sm[B][5] = per_sm < 1 ? 1 : per_sm;
            const int smem3 = fast::WarpSmemBody<false, 384>::STRIDE * fast::WARPS;
            KIVI_CUDA(cudaFuncSetAttribute(fast::attend_body_kernel<B, false, 384>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem3));
            KIVI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &per_sm, fast::attend_body_kernel<B, false, 384>, fast::WARPS * 32, smem3));
            h->fast_per_sm[B][7] = per_sm < 1 ? 1 : per_sm;
        }
        KIVI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, fast::attend_tail_kernel<B>, fast::WARPS * 32, smem));
        h->fast_per_sm[B][1] = per_sm < 1 ? 1 : per_sm;
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    h->prof_now = h->profile && (h->profile_seq++ % h->profile_stride == 0);
    if (h->prof_now) {
        e0 = h->take_event();
        e1 = h->take_event();
        cudaEventRecord(e0, st);
    }
    if (!h->side) {
        KIVI_CUDA(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
        KIVI_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
        KIVI_CUDA(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
        KIVI_CUDA(dalloc(&h->work, WORK_SLOTS));
        KIVI_CUDA(cudaMemsetAsync(h->work, 0, sizeof(int) * WORK_SLOTS, st));
    }
    const bool has_tail = n_sub > nfull;
    const int use_pdl = tune().pdl;
    const int tail_side = tune().tail_side;
    const int tail_ctas = tune().tail_ctas;
    const int tail_warp_ctas = tune().tail_warp_ctas;
    // Body and tail concurrently.  Default: one stream, programmatic launches
    // (append -> tail -> body -> combine): the tail waits for the append, then
    // triggers, so the body's CTAs start beside it (the body reads only what
    // the append wrote, complete once the tail runs) and wait for the tail
    // only at their end, before the combine.  KIVI_PDL=0: tail on a side
    // stream with fork / join events.
    const bool one_stream = use_pdl && nfull > 0 && has_tail && l_app < 0 && !tail_warp_ctas &&
                            !(B == 2 && mha_tc);
    cudaStream_t tail_st = (tail_side && nfull > 0 && !one_stream) ? h->side : st;
    const int tail_last_env = tune().tail_last;
    const bool tail_last = one_stream && tail_last_env;
    fast::FastArgs a_tail{};
    bool tail_deferred = false;
    if (has_tail) {
        // Tail items (residual fp32 tokens, latency-bound) with 2 CTAs per SM,
        // concurrently with the ALU-bound body kernel.
        if (tail_st != st) {
            KIVI_CUDA(cudaEventRecord(h->ev_fork, st));
            KIVI_CUDA(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
        }
        a.k_first = (int)nfull;
        a.t_first = (int)t_first;
        a.sub = tsub;
        a.sub_b = rsub;
        a.n_a = (int)n_a;
        a.t_b = (int)t_b;
        a.n_per_unit = (int)(n_sub - nfull);
        a.n_items = (int)(U * a.n_per_unit);
        a.tk = tk;
        a.tv = tv;
        a.l_app = (int)l_app;
        a.prefetch = latency_bound ? 1 : 0;
        if (tail_last) {
            // launched after the body (below)
            a_tail = a;
            a_tail.tail_last = 1;
            tail_deferred = true;
        } else if (nfull > 0 && tail_st != st && tail_warp_ctas && l_app < 0) {
            // one-warp CTAs beside the body kernel: every tail item its own warp
            const int64_t grid = std::min<int64_t>((int64_t)num_sms() * tail_warp_ctas,
                                                   a.n_items);
            fast::attend_tail_kernel<B, 1><<<(unsigned)grid, 32, fast::WS2::STRIDE, tail_st>>>(a);
        } else {
            const int per_sm =
                (nfull > 0 && (tail_st != st || one_stream)) ? tail_ctas : h->fast_per_sm[B][1];
            const int64_t grid = std::min<int64_t>((int64_t)num_sms() * per_sm,
                                                   ceil_div(a.n_items, fast::WARPS));
            if (l_app >= 0)  // fused append: the variant carrying the append code
                fast::attend_tail_kernel<B, fast::WARPS, true>
                    <<<(unsigned)grid, fast::WARPS * 32, smem, tail_st>>>(a);
            else if (use_pdl && tail_st == st && !(h->prof_now && !one_stream))
                // few-unit route (append -> attend -> combine) or one_stream
                KIVI_CUDA(launch_pdl(fast::attend_tail_kernel<B>, dim3((unsigned)grid),
                                     dim3(fast::WARPS * 32), (size_t)smem, st, a));
            else
                fast::attend_tail_kernel<B><<<(unsigned)grid, fast::WARPS * 32, smem, tail_st>>>(a);
        }
        if (!tail_deferred) {
            KIVI_LAUNCHED();
            if (tail_st != st) KIVI_CUDA(cudaEventRecord(h->ev_join, tail_st));
            h->total_launches++;
        }
    }
    if (nfull > 0) {
        a.l_app = -1;
        a.k_first = 0;
        a.t_first = 0;
        a.prefetch = tune().body_prefetch;
        a.sub = bsub;
        a.n_per_unit = (int)nfull;
        a.n_items = (int)(U * nfull);
        take_work_slot(h, a);
        if (B == 2 && mha_tc && bsub == fast::SUB) {
            // tensor-core body (kernels_attend_gqa_tc.cuh with one query head):
            // every item is a whole SUB-token sub-chunk below nfull * BSUB
            a.body_end = (int)(nfull * bsub);
            const int64_t grid = std::min<int64_t>((int64_t)num_sms() * h->fast_per_sm[B][2],
                                                   ceil_div(a.n_items, gqa_tc::WARPS));
            gqa_tc::attend_gqa_tc_kernel<1>
                <<<(unsigned)grid, gqa_tc::WARPS * 32, smem_tc, st>>>(a);
        } else {
            const int64_t grid = std::min<int64_t>(
                (int64_t)num_sms() *
                    h->fast_per_sm[B][bidx == 1 ? (vimma ? 6 : 5) : bidx == 2 ? (vimma ? 8 : 7) : (vimma ? 4 : 0)],
                ceil_div(a.n_items, fast::WARPS));
            if (tail_deferred) {
                // body first (normal launch: the append is complete), then the
                // residual-window kernel as its programmatic dependent
                a.tail_last = 1;
                body_kernel<<<(unsigned)grid, fast::WARPS * 32, smem_body, st>>>(a);
            } else if (one_stream)
                KIVI_CUDA(launch_pdl(body_kernel, dim3((unsigned)grid), dim3(fast::WARPS * 32),
                                     (size_t)smem_body, st, a));
            else
                body_kernel<<<(unsigned)grid, fast::WARPS * 32, smem_body, st>>>(a);
        }
        KIVI_LAUNCHED();
        h->total_launches++;
        if (tail_deferred) {
            const int64_t grid = std::min<int64_t>((int64_t)num_sms() * h->fast_per_sm[B][1],
                                                   ceil_div(a_tail.n_items, fast::WARPS));
            KIVI_CUDA(launch_pdl(fast::attend_tail_kernel<B>, dim3((unsigned)grid),
                                 dim3(fast::WARPS * 32), (size_t)smem, st, a_tail));
            KIVI_LAUNCHED();
            h->total_launches++;
        }
    }
    if (has_tail && tail_st != st) KIVI_CUDA(cudaStreamWaitEvent(st, h->ev_join, 0));
    if (h->prof_now) {
        cudaEventRecord(e1, st);
        h->events.emplace_back(e0, e1);
        h->main_launches++;
    }
    // K5: merge the per-item partials (a separate launch keeps the merge work
    // balanced; fusing it into the attend tail serialised it on the last warps)
    const int cmode = combine_parallel(U);
    const unsigned cgrid = (unsigned)(cmode == 2 ? ceil_div(U, 4) : U);
    if (defer_combine) {  // the caller fuses the merge with the next layer's append
        h->pending_nsub = n_sub;
        h->pending_cmode = cmode;
        return KIVI_OK;
    }
    if (use_pdl && ((nfull == 0 && !h->prof_now) || (one_stream && !h->prof_now)))
        KIVI_CUDA(launch_pdl(fast::combine_kernel, dim3(cgrid), dim3(fast::D), 0, st,
                             (const float*)h->part_o, (const float2*)h->part_ml, (int)n_sub, out,
                             weights ? h->stats : (float2*)nullptr, cmode, (int64_t)U));
    else
        fast::combine_kernel<<<cgrid, fast::D, 0, st>>>(h->part_o, h->part_ml, (int)n_sub, out,
                                                        weights ? h->stats : nullptr, cmode,
                                                        (int64_t)U);
    KIVI_LAUNCHED();
    h->total_launches++;
    if (weights) {
        fast::normalize_weights_kernel<<<grid_for(U * h->l), 256, 0, st>>>(weights, h->stats, h->l,
                                                                            U);
        KIVI_LAUNCHED();
        h->total_launches++;
    }
    return KIVI_OK;
}

template <int H>
kivi_status launch_gqa(kivi_cache* h, const float* q, float* out, float* weights, float qscale,
                       cudaStream_t st) {
    using WS = gqa::GS<H>;
    using TWS = gqa_tc::TS<H>;
    const int64_t U = h->n_units;
    if (h->l >= (1LL << 30) || U * ceil_div(h->l, fast::SUB) >= (1LL << 30))
        return fail(KIVI_ERR_CONFIG, "GQA attend path: cache too large for 32-bit indexing");
    const int64_t n_sub = ceil_div(h->l, fast::SUB);
    const int use_tc = tune().gqa_tc;
    // body = [0, floor32(vg)) (partial last item): the CUDA-core residual items
    // then hold fewer than 32 quantized values
    const int partial = tune().gqa_partial;
    // tensor-core body items: 256 tokens, or 384 (KIVI_GQA_ITEM=384: fewer
    // items, C3 +2.3 %, but the tensor core's truncating fp32 accumulation runs
    // 1.5x longer per item: rel-L2 on 50x outlier key channels 9-11e-6 vs 6-7.5e-6
    // against the reference, too close to the 1e-5 bar; off)
    const int git = tune().gqa_item == 384 ? 384 : 256;
    const int64_t body_end =
        use_tc ? (partial ? (h->vg() / 32) * 32 : (h->vg() / 32 * 32) / git * git) : 0;
    const int64_t nfull = ceil_div(body_end, git);
    const int64_t ntail = ceil_div(h->l - body_end, fast::SUB);  // residual-window items
    const int64_t n_parts = nfull + ntail;                       // <= n_sub + 1
    const int64_t n_sub_cap = std::max<int64_t>(n_sub, ceil_div(h->cap, fast::SUB)) + 1;
    kivi_status rc = ensure(&h->part_o, &h->part_cap, U * n_sub_cap * H * fast::D);
    if (rc) return rc;
    rc = ensure(&h->part_ml, &h->ml_cap, U * n_sub_cap * H);
    if (rc) return rc;
    rc = ensure(&h->stats, &h->stats_cap, U * H);
    if (rc) return rc;
    fast::FastArgs a{};
    a.c = h->dev;
    a.l = (int)h->l;
    a.kg = (int)h->kg();
    a.vg = (int)h->vg();
    a.n_sub = (int)n_parts;
    a.q = q;
    a.qscale = qscale;
    a.part_o = h->part_o;
    a.part_ml = h->part_ml;
    a.wlog = weights;
    const int smem = WS::STRIDE * gqa::WARPS;
    const int smem_tc =
        (git == 384 ? gqa_tc::TS<H, 384>::STRIDE : TWS::STRIDE) * gqa_tc::WARPS;
    const int key = 4 + H;
    if (h->fast_per_sm[key][2] == 0) {
        KIVI_CUDA(cudaFuncSetAttribute(gqa::attend_gqa_kernel<H>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        KIVI_CUDA(cudaFuncSetAttribute(gqa_tc::attend_gqa_tc_kernel<H>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem_tc));
        KIVI_CUDA(cudaFuncSetAttribute(gqa::attend_gqa_kernel<H, 1>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, WS::STRIDE));
        int per_sm = 0;
        KIVI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, gqa::attend_gqa_kernel<H>, gqa::WARPS * 32, smem));
        h->fast_per_sm[key][2] = per_sm < 1 ? 1 : per_sm;
        KIVI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, gqa_tc::attend_gqa_tc_kernel<H>, gqa_tc::WARPS * 32,
            TWS::STRIDE * gqa_tc::WARPS));
        h->fast_per_sm[key][3] = per_sm < 1 ? 1 : per_sm;
        const int smem_tc3 = gqa_tc::TS<H, 384>::STRIDE * gqa_tc::WARPS;
        KIVI_CUDA(cudaFuncSetAttribute(gqa_tc::attend_gqa_tc_kernel<H, 384>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem_tc3));
        KIVI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, gqa_tc::attend_gqa_tc_kernel<H, 384>, gqa_tc::WARPS * 32, smem_tc3));
        h->fast_per_sm[key][4] = per_sm < 1 ? 1 : per_sm;
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    h->prof_now = h->profile && (h->profile_seq++ % h->profile_stride == 0);
    if (h->prof_now) {
        e0 = h->take_event();
        e1 = h->take_event();
        cudaEventRecord(e0, st);
    }
    if (!h->side) {
        KIVI_CUDA(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
        KIVI_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
        KIVI_CUDA(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
        KIVI_CUDA(dalloc(&h->work, WORK_SLOTS));
        KIVI_CUDA(cudaMemsetAsync(h->work, 0, sizeof(int) * WORK_SLOTS, st));
    }
    const bool has_tail = ntail > 0;
    const int tail_ctas = tune().gqa_tail_ctas;
    cudaStream_t tail_st = nfull > 0 ? h->side : st;
    if (has_tail) {
        // items holding fp32 residual rows: CUDA-core kernel, concurrently
        if (tail_st != st) {
            KIVI_CUDA(cudaEventRecord(h->ev_fork, st));
            KIVI_CUDA(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
        }
        a.k_first = (int)nfull;
        a.t_first = (int)body_end;
        a.sub = fast::SUB;
        a.n_per_unit = (int)ntail;
        a.n_items = (int)(U * a.n_per_unit);
        if (tail_st != st) {
            // one-warp CTAs (27 KB) so two tensor-core CTAs still fit beside one
            const int64_t grid = std::min<int64_t>((int64_t)num_sms() * tail_ctas, a.n_items);
            gqa::attend_gqa_kernel<H, 1><<<(unsigned)grid, 32, WS::STRIDE, tail_st>>>(a);
        } else {
            const int64_t grid = std::min<int64_t>((int64_t)num_sms() * h->fast_per_sm[key][2],
                                                   ceil_div(a.n_items, gqa::WARPS));
            gqa::attend_gqa_kernel<H><<<(unsigned)grid, gqa::WARPS * 32, smem, tail_st>>>(a);
        }
        KIVI_LAUNCHED();
        if (tail_st != st) KIVI_CUDA(cudaEventRecord(h->ev_join, tail_st));
        h->total_launches++;
    }
    if (nfull > 0) {
        a.k_first = 0;
        a.t_first = 0;
        a.sub = fast::SUB;
        a.body_end = (int)body_end;
        a.n_per_unit = (int)nfull;
        a.n_items = (int)(U * nfull);
        a.prefetch = tune().body_prefetch;
        a.sub = git;
        take_work_slot(h, a);
        const int64_t grid = std::min<int64_t>(
            (int64_t)num_sms() * h->fast_per_sm[key][git == 384 ? 4 : 3],
            ceil_div(a.n_items, gqa_tc::WARPS));
        if (git == 384)
            gqa_tc::attend_gqa_tc_kernel<H, 384><<<(unsigned)grid, gqa_tc::WARPS * 32, smem_tc, st>>>(a);
        else
            gqa_tc::attend_gqa_tc_kernel<H><<<(unsigned)grid, gqa_tc::WARPS * 32, smem_tc, st>>>(a);
        KIVI_LAUNCHED();
        h->total_launches++;
    }
    if (has_tail && tail_st != st) KIVI_CUDA(cudaStreamWaitEvent(st, h->ev_join, 0));
    if (h->prof_now) {
        cudaEventRecord(e1, st);
        h->events.emplace_back(e0, e1);
        h->main_launches++;
    }
    const int cmode = combine_parallel(U * H);
    gqa::combine_heads_kernel<<<(unsigned)(cmode == 2 ? ceil_div(U * H, 4) : U * H), fast::D, 0,
                                st>>>(h->part_o, h->part_ml, (int)n_parts, H, out,
                                      weights ? h->stats : nullptr, cmode, (int64_t)(U * H));
    KIVI_LAUNCHED();
    h->total_launches++;
    if (weights) {
        fast::normalize_weights_kernel<<<grid_for(U * H * h->l), 256, 0, st>>>(weights, h->stats,
                                                                                h->l, U * H);
        KIVI_LAUNCHED();
        h->total_launches++;
    }
    return KIVI_OK;
}

// attend_generic_kernel's dynamic shared memory: q row, reduction scratch,
// and the cached group (scale, zero) pairs
size_t generic_smem(int64_t d) {
    return sizeof(float) * (size_t)((d + 32 + 1) & ~1LL) + (sizeof(double) + sizeof(float)) * GEN_SC_CAP;
}

kivi_status launch_generic(kivi_cache* h, const float* q, int qpk, float* out, float* weights,
                           int scale_logits, cudaStream_t st) {
    const int64_t rows = h->n_units * qpk;
    kivi_status rc = ensure(&h->scratch, &h->scratch_cap, rows * std::max(h->l, h->cap));
    if (rc) return rc;
    AttendGenericArgs a;
    a.c = h->dev;
    a.l = h->l;
    a.kg = h->kg();
    a.vg = h->vg();
    a.ring_mod = h->cfg.residual_length;
    a.q = q;
    a.qpk = qpk;
    a.out = out;
    a.weights = weights;
    a.scratch = h->scratch;
    a.scale_logits = scale_logits;
    const size_t smem = generic_smem(h->cfg.head_dim);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    h->prof_now = h->profile && (h->profile_seq++ % h->profile_stride == 0);
    if (h->prof_now) {
        e0 = h->take_event();
        e1 = h->take_event();
        cudaEventRecord(e0, st);
    }
    attend_generic_kernel<<<(unsigned)rows, 256, smem, st>>>(a);
    KIVI_LAUNCHED();
    if (h->prof_now) {
        cudaEventRecord(e1, st);
        h->events.emplace_back(e0, e1);
        h->main_launches++;
    }
    h->total_launches++;
    return KIVI_OK;
}

}  // namespace

extern "C" {

const char* kivi_last_error(void) { return g_last_error.c_str(); }
int kivi_abi_version(void) { return KIVI_B200_ABI_VERSION; }
kivi_status kivi_config_validate(const kivi_config* cfg) { return validate_cfg(cfg); }

kivi_status kivi_cache_create(const kivi_config* cfg, int device, int64_t n_units,
                              int64_t capacity_tokens, kivi_cache** out) {
    if (!out) return fail(KIVI_ERR_USAGE, "out is NULL");
    *out = nullptr;
    kivi_status rc = validate_cfg(cfg);
    if (rc) return rc;
    if (n_units < 1) return fail(KIVI_ERR_USAGE, "n_units must be >= 1");
    if (capacity_tokens < 0) return fail(KIVI_ERR_USAGE, "capacity_tokens must be >= 0");
    DeviceGuard g(device);
    kivi_cache* h = new kivi_cache();
    h->cfg = *cfg;
    h->device = device;
    h->n_units = n_units;
    init_dev_scalars(h);
    rc = alloc_cache_buffers(h, make_layout(*cfg, capacity_tokens), nullptr);
    if (rc) {
        free_cache_buffers(h);
        delete h;
        return rc;
    }
    cudaError_t e = cudaStreamSynchronize(nullptr);
    if (e != cudaSuccess) {
        free_cache_buffers(h);
        delete h;
        return fail(KIVI_ERR_CUDA, "create: %s", cudaGetErrorString(e));
    }
    *out = h;
    return KIVI_OK;
}

kivi_status kivi_cache_destroy(kivi_cache* h) {
    if (!h) return KIVI_OK;
    DeviceGuard g(h->device);
    // the caller's streams must be done with the cache (as for any free); the
    // cache's own copy / side streams are drained here, not the whole device
    if (h->side) cudaStreamSynchronize(h->side);
    if (h->h2d) cudaStreamSynchronize(h->h2d);
    if (h->d2h) cudaStreamSynchronize(h->d2h);
    free_cache_buffers(h);
    cudaFree(h->part_o);
    cudaFree(h->part_ml);
    cudaFree(h->scratch);
    cudaFree(h->heads_buf);
    cudaFree(h->stats);
    for (auto& sg : h->stg) {
        cudaFree(sg.q);
        cudaFree(sg.k);
        cudaFree(sg.v);
        cudaFree(sg.out);
        cudaFree(sg.w);
        if (sg.in_free) cudaEventDestroy(sg.in_free);
        if (sg.out_free) cudaEventDestroy(sg.out_free);
    }
    cudaFree(h->xfer);
    if (h->h2d) cudaStreamDestroy(h->h2d);
    if (h->side) cudaStreamDestroy(h->side);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    cudaFree(h->work);
    if (h->small_sync) cudaFree(h->small_sync);
    if (h->d2h) cudaStreamDestroy(h->d2h);
    if (h->ev_out_ready) cudaEventDestroy(h->ev_out_ready);
    if (h->ev_h2d_done) cudaEventDestroy(h->ev_h2d_done);
    for (auto& ev : h->events) {
        cudaEventDestroy(ev.first);
        cudaEventDestroy(ev.second);
    }
    for (auto e : h->event_pool) cudaEventDestroy(e);
    delete h;
    return KIVI_OK;
}

kivi_status kivi_cache_reserve(kivi_cache* h, int64_t capacity_tokens, void* stream) {
    if (!h) return fail(KIVI_ERR_USAGE, "cache is NULL");
    DeviceGuard g(h->device);
    Layout L = make_layout(h->cfg, capacity_tokens);
    if (L.cap <= h->cap) return KIVI_OK;
    kivi_cache tmp;
    tmp.cfg = h->cfg;
    tmp.n_units = h->n_units;
    cudaStream_t st = S(stream);
    kivi_status rc = alloc_cache_buffers(&tmp, L, st);
    if (rc) {
        free_cache_buffers(&tmp);
        return rc;
    }
    const CacheDev& o = h->dev;
    CacheDev& n = tmp.dev;
    const int64_t U = h->n_units;
    KIVI_CUDA(cudaMemcpy2DAsync(n.kcodes, n.k_ustride, o.kcodes, o.k_ustride, o.k_ustride, U,
                                cudaMemcpyDeviceToDevice, st));
    KIVI_CUDA(cudaMemcpy2DAsync(n.kpairs, n.kp_ustride * sizeof(float2), o.kpairs,
                                o.kp_ustride * sizeof(float2), o.kp_ustride * sizeof(float2), U,
                                cudaMemcpyDeviceToDevice, st));
    KIVI_CUDA(cudaMemcpy2DAsync(n.vcodes, n.v_ustride, o.vcodes, o.v_ustride, o.v_ustride, U,
                                cudaMemcpyDeviceToDevice, st));
    KIVI_CUDA(cudaMemcpy2DAsync(n.vpairs, n.vp_ustride * sizeof(float2), o.vpairs,
                                o.vp_ustride * sizeof(float2), o.vp_ustride * sizeof(float2), U,
                                cudaMemcpyDeviceToDevice, st));
    KIVI_CUDA(cudaMemcpyAsync(n.kring, o.kring, sizeof(float) * U * o.ring_ustride,
                              cudaMemcpyDeviceToDevice, st));
    KIVI_CUDA(cudaMemcpyAsync(n.vring, o.vring, sizeof(float) * U * o.ring_ustride,
                              cudaMemcpyDeviceToDevice, st));
    KIVI_CUDA(cudaStreamSynchronize(st));
    free_cache_buffers(h);
    h->dev.kcodes = n.kcodes;
    h->dev.kpairs = n.kpairs;
    h->dev.vcodes = n.vcodes;
    h->dev.vpairs = n.vpairs;
    h->dev.kring = n.kring;
    h->dev.vring = n.vring;
    h->dev.k_ustride = n.k_ustride;
    h->dev.kp_ustride = n.kp_ustride;
    h->dev.v_ustride = n.v_ustride;
    h->dev.vp_ustride = n.vp_ustride;
    h->dev.ring_ustride = n.ring_ustride;
    h->cap = tmp.cap;
    return KIVI_OK;
}

kivi_status kivi_cache_clone(const kivi_cache* src, void* stream, kivi_cache** out) {
    if (!src || !out) return fail(KIVI_ERR_USAGE, "NULL argument");
    DeviceGuard g(src->device);
    kivi_cache* h = nullptr;
    kivi_status rc = kivi_cache_create(&src->cfg, src->device, src->n_units, src->cap, &h);
    if (rc) return rc;
    cudaStream_t st = S(stream);
    const CacheDev& o = src->dev;
    CacheDev& n = h->dev;
    const int64_t U = src->n_units;
    KIVI_CUDA(cudaMemcpyAsync(n.kcodes, o.kcodes, (size_t)(U * o.k_ustride),
                              cudaMemcpyDeviceToDevice, st));
    KIVI_CUDA(cudaMemcpyAsync(n.kpairs, o.kpairs, sizeof(float2) * (size_t)(U * o.kp_ustride),
                              cudaMemcpyDeviceToDevice, st));
    KIVI_CUDA(cudaMemcpyAsync(n.vcodes, o.vcodes, (size_t)(U * o.v_ustride),
                              cudaMemcpyDeviceToDevice, st));
    KIVI_CUDA(cudaMemcpyAsync(n.vpairs, o.vpairs, sizeof(float2) * (size_t)(U * o.vp_ustride),
                              cudaMemcpyDeviceToDevice, st));
    KIVI_CUDA(cudaMemcpyAsync(n.kring, o.kring, sizeof(float) * (size_t)(U * o.ring_ustride),
                              cudaMemcpyDeviceToDevice, st));
    KIVI_CUDA(cudaMemcpyAsync(n.vring, o.vring, sizeof(float) * (size_t)(U * o.ring_ustride),
                              cudaMemcpyDeviceToDevice, st));
    KIVI_CUDA(cudaStreamSynchronize(st));
    h->l = src->l;
    h->kq_done = src->kq_done;
    h->kres_cap = src->kres_cap;
    h->vres_cap = src->vres_cap;
    h->attend_path = src->attend_path;
    *out = h;
    return KIVI_OK;
}

kivi_status kivi_cache_get_info(const kivi_cache* h, kivi_cache_info* info) {
    if (!h || !info) return fail(KIVI_ERR_USAGE, "NULL argument");
    const int64_t R = h->cfg.residual_length, d = h->cfg.head_dim;
    info->n_units = h->n_units;
    info->capacity_tokens = h->cap;
    info->total_tokens = h->l;
    info->key_grouped_tokens = h->kg();
    info->key_residual_rows = h->l - h->kg();
    info->key_residual_capacity = h->kres_cap;
    info->value_grouped_tokens = h->vg();
    info->value_residual_rows = h->l - h->vg();
    info->value_residual_capacity = h->vres_cap;
    (void)R;
    // reference memory_bytes (kv_cache.cpp:117-127): residual charged at its
    // high-water capacity x residual.cols() (0 for a never-initialised state).
    const uint64_t kcols = (h->l > 0 || h->kres_cap > 0) ? (uint64_t)d : 0;
    info->key_memory_bytes = grouped_bytes(h->kg(), h->cfg) + 2ull * h->kres_cap * kcols;
    info->value_memory_bytes = grouped_bytes(h->vg(), h->cfg) + 2ull * h->vres_cap * kcols;
    const CacheDev& c = h->dev;
    info->device_bytes = (uint64_t)h->n_units *
                         ((uint64_t)c.k_ustride + (uint64_t)c.v_ustride +
                          sizeof(float2) * (uint64_t)(c.kp_ustride + c.vp_ustride) +
                          2 * sizeof(float) * (uint64_t)c.ring_ustride);
    return KIVI_OK;
}

kivi_status kivi_prefill(kivi_cache* h, const float* keys, const float* values, int64_t l,
                         void* stream) {
    if (!h) return fail(KIVI_ERR_USAGE, "cache is NULL");
    if (l <= 0) return fail(KIVI_ERR_USAGE, "prefill: empty prompt");
    if (!keys || !values) return fail(KIVI_ERR_USAGE, "prefill: NULL keys/values");
    DeviceGuard g(h->device);
    cudaStream_t st = S(stream);
    kivi_status rc = ensure_capacity(h, l, st);
    if (rc) return rc;
    CacheDev& c = h->dev;
    const int64_t U = h->n_units;
    // reset the code streams (appends OR into zeroed words)
    KIVI_CUDA(cudaMemsetAsync(c.kcodes, 0, (size_t)(U * c.k_ustride), st));
    KIVI_CUDA(cudaMemsetAsync(c.vcodes, 0, (size_t)(U * c.v_ustride), st));
    const int64_t R = h->cfg.residual_length;
    const int64_t kg = l - l % R;
    const int64_t vg = l - std::min(l, R);
    const int64_t G = h->cfg.group_size, d = h->cfg.head_dim;
    // the fast kernels read 16-byte vectors of the caller's rows
    const bool rows16 = (((uintptr_t)keys | (uintptr_t)values) & 15) == 0;
    const bool fast = d == 128 && G == 32 && (c.bits == 2 || c.bits == 4) && rows16;
    if (kg > 0) {
        if (fast && c.bits == 2)
            prefill_keys_fast_kernel<2><<<grid_for(U * (kg / G) * d), 256, 0, st>>>(c, keys, l, kg);
        else if (fast)
            prefill_keys_fast_kernel<4><<<grid_for(U * (kg / G) * d), 256, 0, st>>>(c, keys, l, kg);
        else
            prefill_keys_kernel<<<grid_for(U * (kg / G) * d), 256, 0, st>>>(c, keys, l, kg);
        KIVI_LAUNCHED();
        h->total_launches++;
    }
    if (vg > 0) {
        if (fast && c.bits == 2)
            prefill_values_fast_kernel<2><<<grid_for(U * vg * 4), 256, 0, st>>>(c, values, l, vg);
        else if (fast)
            prefill_values_fast_kernel<4><<<grid_for(U * vg * 4), 256, 0, st>>>(c, values, l, vg);
        else
            prefill_values_kernel<<<grid_for(U * vg * (d / G)), 256, 0, st>>>(c, values, l, vg);
        KIVI_LAUNCHED();
        h->total_launches++;
    }
    const int vec = (d % 4 == 0 && rows16) ? 4 : 1;
    prefill_residual_kernel<<<grid_for(U * (2 * l - kg - vg) * (d / vec)), 256, 0, st>>>(
        c, keys, values, l, kg, vg, vec);
    KIVI_LAUNCHED();
    h->total_launches++;
    h->l = l;
    h->kq_done = 0;
    h->kres_cap = l % R;  // kv_cache.cpp:40
    h->vres_cap = std::min(l, R);
    return KIVI_OK;
}

// Host-side counters of one append_token (kv_cache.cpp:66-98).
static void append_bookkeeping(kivi_cache* h) {
    const int64_t R = h->cfg.residual_length;
    // residual_capacity = max(capacity, rows after the push) (kv_cache.cpp:78, 93-94)
    const int64_t krows_after_push = h->l % R + 1;
    h->kres_cap = std::max(h->kres_cap, krows_after_push);
    const int64_t vrows = std::min(h->l, R) == R ? R : std::min(h->l, R) + 1;
    h->vres_cap = std::max(h->vres_cap, vrows);
    h->l += 1;
    if (h->l % R == 0) h->kq_done = 0;  // flushed: a new ring window
}

// Key tiles the fast append of token h->l must quantize: the complete tiles
// of the ring after the push not yet quantized, [kq_done, rows / 32) (one
// tile every 32 steps; after a prefill or import, every complete tile).
static void key_tiles_due(kivi_cache* h, int* tl0, int* ntl) {
    const int64_t rows = h->l % h->cfg.residual_length + 1;
    const int64_t done = rows / 32;
    *tl0 = (int)h->kq_done;
    *ntl = (int)std::max<int64_t>(done - h->kq_done, 0);
    h->kq_done = std::max(h->kq_done, done);
}

// qs: optional query staging by the fast append (QStage); callers check
// append_stages_q() first.
static bool append_stages_q(const kivi_cache* h, const float* t_k, const float* t_v) {
    const kivi_config& cf = h->cfg;
    return cf.head_dim == 128 && cf.group_size == 32 && (cf.bits == 2 || cf.bits == 4) &&
           al16(t_k, t_v);
}

static kivi_status append_launch(kivi_cache* h, const float* t_k, const float* t_v,
                                 cudaStream_t st, QStage qs = QStage{nullptr, nullptr, 0}) {
    const kivi_config& cf = h->cfg;
    if (append_stages_q(h, t_k, t_v)) {
        const unsigned grid = (unsigned)ceil_div(h->n_units, 8);
        int tl0, ntl;
        key_tiles_due(h, &tl0, &ntl);
        if (ntl > 0) {
            // complete key tiles: extra blocks quantize them, one thread per group
            const int64_t groups = h->n_units * ntl * (128 / FLUSH_GPT);
            const unsigned fgrid = (unsigned)ceil_div(groups, 256);
            if (cf.bits == 2)
                append_flush_fast_kernel<2><<<grid + fgrid, 256, 0, st>>>(h->dev, t_k, t_v, h->l,
                                                                         (int)grid, tl0, ntl, qs);
            else
                append_flush_fast_kernel<4><<<grid + fgrid, 256, 0, st>>>(h->dev, t_k, t_v, h->l,
                                                                         (int)grid, tl0, ntl, qs);
        } else if (cf.bits == 2) {
            append_fast_kernel<2><<<grid, 256, 0, st>>>(h->dev, t_k, t_v, h->l, qs);
        } else {
            append_fast_kernel<4><<<grid, 256, 0, st>>>(h->dev, t_k, t_v, h->l, qs);
        }
    } else {
        append_kernel<<<(unsigned)h->n_units, 128, 0, st>>>(h->dev, t_k, t_v, h->l);
    }
    KIVI_LAUNCHED();
    h->total_launches++;
    return KIVI_OK;
}

kivi_status kivi_append(kivi_cache* h, const float* t_k, const float* t_v, void* stream) {
    if (!h) return fail(KIVI_ERR_USAGE, "cache is NULL");
    if (!t_k || !t_v) return fail(KIVI_ERR_SHAPE, "append_token: NULL key/value rows");
    DeviceGuard g(h->device);
    cudaStream_t st = S(stream);
    kivi_status rc = ensure_capacity(h, h->l + 1, st);
    if (rc) return rc;
    rc = append_launch(h, t_k, t_v, st);
    if (rc) return rc;
    append_bookkeeping(h);
    return KIVI_OK;
}

extern "C++" {
namespace {
// rows of `len` floats: dst row (h, u) <- src row (u, h) (to_heads), or the
// reverse; one float4 per thread (len % 4 == 0)
__global__ void permute_heads_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                     int64_t U, int H, int64_t len, int to_heads) {
    const int64_t v4 = len / 4, total = U * H * v4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / v4, c = i - row * v4;  // row in dst order
        int64_t srow;
        if (to_heads) {  // dst (h, u) <- src (u, h)
            const int64_t hh = row / U, u = row - hh * U;
            srow = u * H + hh;
        } else {  // dst (u, h) <- src (h, u)
            const int64_t u = row / H, hh = row - u * H;
            srow = hh * U + u;
        }
        reinterpret_cast<float4*>(dst)[row * v4 + c] =
            reinterpret_cast<const float4*>(src)[srow * v4 + c];
    }
}
}  // namespace

// GQA shapes outside one tensor-core launch (B = 4, or q_per_kv not in
// {2, 4}) when the fast kernels cover the cache (d = 128, G = 32, B in {2, 4}):
// the query heads are split into groups of gs = 4 (or 2) heads for the
// tensor-core kernel at B = 2 (e.g. 8 q heads per kv head: two passes), else
// single heads for the MHA kernels; every pass streams the shared cache once
// (q_per_kv / gs passes, against the generic kernel's reference-order double
// loop: ~270x faster at C3's shape in 4 bits).  q and the outputs are
// permuted to and from group-major rows around the passes.
template <int B>
static kivi_status attend_heads_mha(kivi_cache* h, const float* t_q, int qpk, float* out,
                                    float* weights, float qscale, cudaStream_t st) {
    const int64_t U = h->n_units, d = h->cfg.head_dim, l = h->l;
    const int gs = (B == 2 && qpk % 4 == 0) ? 4 : ((B == 2 && qpk % 2 == 0) ? 2 : 1);
    const int ng = qpk / gs;
    const int64_t need = 2 * qpk * U * d + (weights ? qpk * U * l : 0);
    kivi_status rc = ensure(&h->heads_buf, &h->heads_cap, need);
    if (rc) return rc;
    float* qh = h->heads_buf;
    float* oh = qh + qpk * U * d;
    float* wh = weights ? oh + qpk * U * d : nullptr;
    // rows of gs heads: (u, g) -> (g, u)
    permute_heads_kernel<<<grid_for(qpk * U * d / 4), 256, 0, st>>>(t_q, qh, U, ng, gs * d, 1);
    KIVI_LAUNCHED();
    for (int g = 0; g < ng; ++g) {
        const float* qg = qh + g * U * gs * d;
        float* og = oh + g * U * gs * d;
        float* wg = wh ? wh + g * U * gs * l : nullptr;
        if constexpr (B == 2) {
            if (gs == 4) rc = launch_gqa<4>(h, qg, og, wg, qscale, st);
            else if (gs == 2) rc = launch_gqa<2>(h, qg, og, wg, qscale, st);
            else rc = launch_fast<B>(h, qg, og, wg, qscale, st);
        } else {
            rc = launch_fast<B>(h, qg, og, wg, qscale, st);
        }
        if (rc) return rc;
    }
    permute_heads_kernel<<<grid_for(qpk * U * d / 4), 256, 0, st>>>(oh, out, U, ng, gs * d, 0);
    KIVI_LAUNCHED();
    if (weights) {
        if ((gs * l) % 4 == 0) {
            permute_heads_kernel<<<grid_for(qpk * U * l / 4), 256, 0, st>>>(wh, weights, U, ng,
                                                                            gs * l, 0);
            KIVI_LAUNCHED();
        } else {
            for (int g = 0; g < ng; ++g)
                KIVI_CUDA(cudaMemcpy2DAsync(weights + g * gs * l, sizeof(float) * qpk * l,
                                            wh + g * U * gs * l, sizeof(float) * gs * l,
                                            sizeof(float) * gs * l, U, cudaMemcpyDeviceToDevice,
                                            st));
        }
    }
    h->total_launches += 2 + (weights ? 1 : 0);
    return KIVI_OK;
}
}  // extern "C++"

kivi_status kivi_attend(kivi_cache* h, const float* t_q, int32_t q_per_kv, float* out,
                        float* weights, int32_t scale_logits, void* stream) {
    if (!h) return fail(KIVI_ERR_USAGE, "cache is NULL");
    if (q_per_kv < 1) return fail(KIVI_ERR_SHAPE, "q_per_kv must be >= 1");
    if (!t_q || !out) return fail(KIVI_ERR_SHAPE, "attend: NULL query/output");
    if (h->l < 1) return fail(KIVI_ERR_USAGE, "attend: empty cache");
    DeviceGuard g(h->device);
    cudaStream_t st = S(stream);
    const bool fast_ok = fast_supported(h, q_per_kv) && al16(t_q, out, weights);
    // GQA shapes outside the tensor-core kernel: one MHA fast attend per head
    const bool heads_ok = !fast_ok && q_per_kv > 1 && fast_supported(h, 1) &&
                          al16(t_q, out, weights) && tune().gqa_heads;
    if (h->attend_path == 2 && !fast_ok && !heads_ok)
        return fail(KIVI_ERR_CONFIG,
                    "fast attend path does not support this shape (or rows not 16-byte aligned)");
    if (heads_ok && h->attend_path != 1) {
        const float scale = scale_logits ? 1.0f / sqrtf((float)h->cfg.head_dim) : 1.0f;
        const float qscale = scale * fast::LOG2E;
        if (h->cfg.bits == 2) return attend_heads_mha<2>(h, t_q, q_per_kv, out, weights, qscale, st);
        return attend_heads_mha<4>(h, t_q, q_per_kv, out, weights, qscale, st);
    }
    if (fast_ok && h->attend_path != 1) {
        const float scale = scale_logits ? 1.0f / sqrtf((float)h->cfg.head_dim) : 1.0f;
        const float qscale = scale * fast::LOG2E;
        if (q_per_kv == 4) return launch_gqa<4>(h, t_q, out, weights, qscale, st);
        if (q_per_kv == 2) return launch_gqa<2>(h, t_q, out, weights, qscale, st);
        if (h->cfg.bits == 2) return launch_fast<2>(h, t_q, out, weights, qscale, st);
        return launch_fast<4>(h, t_q, out, weights, qscale, st);
    }
    return launch_generic(h, t_q, q_per_kv, out, weights, scale_logits, st);
}

static kivi_status decode_impl(kivi_cache* h, const float* t_q, const float* t_k,
                               const float* t_v, int32_t q_per_kv, float* out, float* weights,
                               int32_t scale_logits, void* stream, const float* q_src);

kivi_status kivi_decode(kivi_cache* h, const float* t_q, const float* t_k, const float* t_v,
                        int32_t q_per_kv, float* out, float* weights, int32_t scale_logits,
                        void* stream) {
    return decode_impl(h, t_q, t_k, t_v, q_per_kv, out, weights, scale_logits, stream, nullptr);
}

// q_src != NULL: the query rows are in device-mapped host memory at q_src and
// t_q is device scratch; the fast append copies them across (QStage), other
// routes enqueue a copy first.
static kivi_status decode_impl(kivi_cache* h, const float* t_q, const float* t_k,
                               const float* t_v, int32_t q_per_kv, float* out, float* weights,
                               int32_t scale_logits, void* stream, const float* q_src) {
    if (!h) return fail(KIVI_ERR_USAGE, "cache is NULL");
    if (q_per_kv < 1) return fail(KIVI_ERR_SHAPE, "q_per_kv must be >= 1");
    if (!t_q || !out) return fail(KIVI_ERR_SHAPE, "decode_attention: NULL query/output");
    if (!t_k || !t_v) return fail(KIVI_ERR_SHAPE, "append_token: NULL key/value rows");
    const bool aligned = al16(t_q, t_k, t_v, out, weights);
    if (q_src && !(append_stages_q(h, t_k, t_v) && al16(q_src) && !small_fused_ok(h, q_per_kv) &&
                   !fused_append_ok(h, q_per_kv))) {
        DeviceGuard g(h->device);
        KIVI_CUDA(cudaMemcpyAsync(const_cast<float*>(t_q), q_src,
                                  sizeof(float) * h->n_units * q_per_kv * h->cfg.head_dim,
                                  cudaMemcpyDefault, S(stream)));
        q_src = nullptr;
    }
    if (q_src) {  // fast append stages q, then the attend
        DeviceGuard g(h->device);
        cudaStream_t st = S(stream);
        kivi_status rc = ensure_capacity(h, h->l + 1, st);
        if (rc) return rc;
        rc = append_launch(h, t_k, t_v, st, QStage{q_src, const_cast<float*>(t_q), q_per_kv});
        if (rc) return rc;
        append_bookkeeping(h);
        return kivi_attend(h, t_q, q_per_kv, out, weights, scale_logits, stream);
    }
    if (small_fused_ok(h, q_per_kv) && fast_supported(h, q_per_kv) && aligned) {
        DeviceGuard g(h->device);
        cudaStream_t st = S(stream);
        kivi_status rc = ensure_capacity(h, h->l + 1, st);
        if (rc) return rc;
        const int64_t l_app = h->l;
        append_bookkeeping(h);
        const float scale = scale_logits ? 1.0f / sqrtf((float)h->cfg.head_dim) : 1.0f;
        const float qscale = scale * fast::LOG2E;
        if (h->cfg.bits == 2)
            return launch_small_fused<2>(h, t_q, t_k, t_v, out, weights, qscale, l_app, st);
        return launch_small_fused<4>(h, t_q, t_k, t_v, out, weights, qscale, l_app, st);
    }
    if (fused_append_ok(h, q_per_kv) && fast_supported(h, q_per_kv) && aligned) {
        // The append runs inside the residual-window kernel, on each unit right
        // before its residual items; the body items never read what it writes
        // (launch_fast stops the body at floor32(vg - 1)).
        DeviceGuard g(h->device);
        cudaStream_t st = S(stream);
        kivi_status rc = ensure_capacity(h, h->l + 1, st);
        if (rc) return rc;
        const int64_t l_app = h->l;
        append_bookkeeping(h);
        const float scale = scale_logits ? 1.0f / sqrtf((float)h->cfg.head_dim) : 1.0f;
        const float qscale = scale * fast::LOG2E;
        if (h->cfg.bits == 2) return launch_fast<2>(h, t_q, out, weights, qscale, st, t_k, t_v, l_app);
        return launch_fast<4>(h, t_q, out, weights, qscale, st, t_k, t_v, l_app);
    }
    kivi_status rc = kivi_append(h, t_k, t_v, stream);
    if (rc) return rc;
    return kivi_attend(h, t_q, q_per_kv, out, weights, scale_logits, stream);
}

kivi_status kivi_prefill_host(kivi_cache* h, const float* keys, const float* values, int64_t l,
                              void* stream) {
    if (!h) return fail(KIVI_ERR_USAGE, "cache is NULL");
    if (l <= 0) return fail(KIVI_ERR_USAGE, "prefill: empty prompt");
    DeviceGuard g(h->device);
    cudaStream_t st = S(stream);
    const int64_t n = h->n_units * l * h->cfg.head_dim;
    float *dk = nullptr, *dv = nullptr;
    KIVI_CUDA(dalloc(&dk, (size_t)n));
    KIVI_CUDA(dalloc(&dv, (size_t)n));
    KIVI_CUDA(cudaMemcpyAsync(dk, keys, sizeof(float) * n, cudaMemcpyHostToDevice, st));
    KIVI_CUDA(cudaMemcpyAsync(dv, values, sizeof(float) * n, cudaMemcpyHostToDevice, st));
    kivi_status rc = kivi_prefill(h, dk, dv, l, stream);
    cudaError_t e = cudaStreamSynchronize(st);
    cudaFree(dk);
    cudaFree(dv);
    if (rc) return rc;
    if (e != cudaSuccess) return fail(KIVI_ERR_CUDA, "prefill_host: %s", cudaGetErrorString(e));
    return KIVI_OK;
}

// The staging set for this host-path call (alternating), sized for it.  The
// weights buffer is sized for the reserved capacity so a growing context does
// not reallocate it every call (a cudaFree synchronises the device).
static kivi_status stage_rows(kivi_cache* h, int64_t qpk, int64_t wlen, kivi_cache::HostStage** out) {
    const int64_t U = h->n_units, d = h->cfg.head_dim;
    kivi_status rc;
    if (!h->h2d) {
        KIVI_CUDA(cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking));
        KIVI_CUDA(cudaEventCreateWithFlags(&h->ev_h2d_done, cudaEventDisableTiming));
        KIVI_CUDA(cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking));
        KIVI_CUDA(cudaEventCreateWithFlags(&h->ev_out_ready, cudaEventDisableTiming));
        for (auto& sg : h->stg) {
            KIVI_CUDA(cudaEventCreateWithFlags(&sg.in_free, cudaEventDisableTiming));
            KIVI_CUDA(cudaEventRecord(sg.in_free, h->h2d));  // nothing staged yet
            KIVI_CUDA(cudaEventCreateWithFlags(&sg.out_free, cudaEventDisableTiming));
            KIVI_CUDA(cudaEventRecord(sg.out_free, h->d2h));  // nothing to copy yet
        }
    }
    kivi_cache::HostStage& sg = h->stg[h->stg_i];
    h->stg_i ^= 1;
    if ((rc = ensure(&sg.q, &sg.cap_q, U * qpk * d))) return rc;
    if ((rc = ensure(&sg.out, &sg.cap_out, U * qpk * d))) return rc;
    if ((rc = ensure(&sg.k, &sg.cap_k, U * d))) return rc;
    if ((rc = ensure(&sg.v, &sg.cap_v, U * d))) return rc;
    if (wlen > 0 &&
        (rc = ensure(&sg.w, &sg.cap_w, std::max<int64_t>(wlen, U * qpk * (h->cap + 1)))))
        return rc;
    *out = &sg;
    return KIVI_OK;
}

kivi_status kivi_append_host(kivi_cache* h, const float* t_k, const float* t_v, void* stream) {
    if (!h) return fail(KIVI_ERR_USAGE, "cache is NULL");
    if (!t_k || !t_v) return fail(KIVI_ERR_SHAPE, "append_token: NULL key/value rows");
    DeviceGuard g(h->device);
    kivi_cache::HostStage* sg = nullptr;
    kivi_status rc = stage_rows(h, 1, 0, &sg);
    if (rc) return rc;
    cudaStream_t st = S(stream);
    const size_t bytes = sizeof(float) * (size_t)(h->n_units * h->cfg.head_dim);
    KIVI_CUDA(cudaStreamWaitEvent(h->h2d, sg->in_free, 0));
    KIVI_CUDA(cudaMemcpyAsync(sg->k, t_k, bytes, cudaMemcpyHostToDevice, h->h2d));
    KIVI_CUDA(cudaMemcpyAsync(sg->v, t_v, bytes, cudaMemcpyHostToDevice, h->h2d));
    KIVI_CUDA(cudaEventRecord(h->ev_h2d_done, h->h2d));
    KIVI_CUDA(cudaStreamWaitEvent(st, h->ev_h2d_done, 0));
    rc = kivi_append(h, sg->k, sg->v, stream);
    if (rc) return rc;
    KIVI_CUDA(cudaEventRecord(sg->in_free, st));
    return KIVI_OK;
}

kivi_status kivi_decode_host(kivi_cache* h, const float* t_q, const float* t_k, const float* t_v,
                             int32_t q_per_kv, float* out, float* weights, int32_t scale_logits,
                             void* stream) {
    if (!h) return fail(KIVI_ERR_USAGE, "cache is NULL");
    if (q_per_kv < 1) return fail(KIVI_ERR_SHAPE, "q_per_kv must be >= 1");
    if (!t_q || !t_k || !t_v || !out) return fail(KIVI_ERR_SHAPE, "decode_attention: NULL rows");
    DeviceGuard g(h->device);
    const int64_t U = h->n_units, d = h->cfg.head_dim;
    const int64_t wlen = weights ? U * q_per_kv * (h->l + 1) : 0;
    kivi_cache::HostStage* sg = nullptr;
    kivi_status rc = stage_rows(h, q_per_kv, wlen, &sg);
    if (rc) return rc;
    cudaStream_t st = S(stream);
    // upload on the copy stream once the kernels of the call that last used
    // this staging set (two calls ago) consumed it: it overlaps the previous
    // call's kernels
    KIVI_CUDA(cudaStreamWaitEvent(h->h2d, sg->in_free, 0));
    KIVI_CUDA(cudaMemcpyAsync(sg->q, t_q, sizeof(float) * U * q_per_kv * d,
                              cudaMemcpyHostToDevice, h->h2d));
    KIVI_CUDA(cudaMemcpyAsync(sg->k, t_k, sizeof(float) * U * d, cudaMemcpyHostToDevice, h->h2d));
    KIVI_CUDA(cudaMemcpyAsync(sg->v, t_v, sizeof(float) * U * d, cudaMemcpyHostToDevice, h->h2d));
    KIVI_CUDA(cudaEventRecord(h->ev_h2d_done, h->h2d));
    KIVI_CUDA(cudaStreamWaitEvent(st, h->ev_h2d_done, 0));
    // that call's result copy must have left this set's output buffers
    KIVI_CUDA(cudaStreamWaitEvent(st, sg->out_free, 0));
    rc = kivi_decode(h, sg->q, sg->k, sg->v, q_per_kv, sg->out, weights ? sg->w : nullptr,
                     scale_logits, stream);
    if (rc) return rc;
    KIVI_CUDA(cudaEventRecord(sg->in_free, st));
    // result copy on the cache's own stream, so the next layer's kernels on
    // `stream` do not queue behind it (kivi_host_join orders `stream` after it)
    KIVI_CUDA(cudaEventRecord(h->ev_out_ready, st));
    KIVI_CUDA(cudaStreamWaitEvent(h->d2h, h->ev_out_ready, 0));
    KIVI_CUDA(cudaMemcpyAsync(out, sg->out, sizeof(float) * U * q_per_kv * d,
                              cudaMemcpyDeviceToHost, h->d2h));
    if (weights)
        KIVI_CUDA(cudaMemcpyAsync(weights, sg->w, sizeof(float) * wlen, cudaMemcpyDeviceToHost,
                                  h->d2h));
    KIVI_CUDA(cudaEventRecord(sg->out_free, h->d2h));
    return KIVI_OK;
}

// ---- one decode step of a whole model (one cache per layer) -----------------

static kivi_status check_layers(kivi_cache* const* caches, int32_t n_layers) {
    if (!caches || n_layers < 1) return fail(KIVI_ERR_USAGE, "decode_layers: no caches");
    for (int32_t i = 0; i < n_layers; ++i) {
        const kivi_cache* c = caches[i];
        if (!c) return fail(KIVI_ERR_USAGE, "decode_layers: cache %d is NULL", i);
        const kivi_cache* c0 = caches[0];
        if (c->n_units != c0->n_units || c->device != c0->device ||
            c->cfg.head_dim != c0->cfg.head_dim)
            return fail(KIVI_ERR_SHAPE, "decode_layers: cache %d differs in units/device/head_dim",
                        i);
    }
    return KIVI_OK;
}

// Whether a multi-layer step can fuse each layer's merge with the next layer's
// append (combine_append_kernel): MHA on the fast kernels' body route, no
// profiling, every layer at the same length and shape.
static bool step_fusable(kivi_cache* const* caches, int32_t n_layers, int32_t q_per_kv,
                         const float* t_q, const float* t_k, const float* t_v, const float* out) {
    if (!tune().step_fuse || n_layers < 2 || q_per_kv != 1 || !tune().pdl) return false;
    if (!al16(t_q, t_k, t_v, out)) return false;
    const kivi_cache* h0 = caches[0];
    for (int32_t i = 0; i < n_layers; ++i) {
        const kivi_cache* h = caches[i];
        if (!fast_supported(h, 1) || h->attend_path == 1 || h->profile || h->l != h0->l ||
            h->cfg.bits != h0->cfg.bits || h->cfg.residual_length != h0->cfg.residual_length ||
            h->kq_done != h0->kq_done || small_fused_ok(h, 1) || fused_append_ok(h, 1))
            return false;
        // body route after this step's append (the few-unit route has its own chain)
        const int64_t l = h->l + 1;
        if (tune().small_items && h->n_units * ceil_div(l, fast::BSUB) < 4 * num_sms()) return false;
        const int64_t vg = l - std::min<int64_t>(l, h->cfg.residual_length);
        if ((vg / 32 * 32) / fast::BSUB == 0) return false;
    }
    return true;
}

extern "C++" {
template <int B>
static kivi_status decode_layers_fused(kivi_cache* const* caches, int32_t n_layers,
                                       const float* t_q, const float* t_k, const float* t_v,
                                       float* out, int32_t scale_logits, cudaStream_t st) {
    const int64_t U = caches[0]->n_units, d = caches[0]->cfg.head_dim;
    const int64_t krow = U * d;
    const float qscale = (scale_logits ? 1.0f / sqrtf((float)d) : 1.0f) * fast::LOG2E;
    for (int32_t i = 0; i < n_layers; ++i) {
        kivi_status rc = ensure_capacity(caches[i], caches[i]->l + 1, st);
        if (rc) return rc;
    }
    kivi_status rc = append_launch(caches[0], t_k, t_v, st);
    if (rc) return rc;
    append_bookkeeping(caches[0]);
    for (int32_t i = 0; i < n_layers; ++i) {
        kivi_cache* h = caches[i];
        rc = launch_fast<B>(h, t_q + i * krow, out + i * krow, nullptr, qscale, st, nullptr,
                            nullptr, -1, /*defer_combine=*/true);
        if (rc) return rc;
        const int n_sub = (int)h->pending_nsub, cmode = h->pending_cmode;
        const int n_comb = (int)(cmode == 2 ? ceil_div(U, 4) : U);
        if (i + 1 < n_layers) {
            kivi_cache* hn = caches[i + 1];
            int tl0, ntl;
            key_tiles_due(hn, &tl0, &ntl);
            const int n_app = (int)ceil_div(U, 4);
            KIVI_CUDA(launch_pdl(fast::combine_append_kernel<B>, dim3((unsigned)(n_comb + n_app)),
                                 dim3(fast::D), 0, st, (const float*)h->part_o,
                                 (const float2*)h->part_ml, n_sub, out + i * krow, cmode, (int64_t)U,
                                 n_comb, hn->dev, t_k + (i + 1) * krow, t_v + (i + 1) * krow,
                                 (int64_t)hn->l));
            KIVI_LAUNCHED();
            h->total_launches++;
            if (ntl > 0) {  // complete key tiles of layer i+1 (every 32 steps)
                const unsigned fgrid = (unsigned)ceil_div(U * ntl * (128 / FLUSH_GPT), 256);
                append_flush_fast_kernel<B><<<fgrid, 256, 0, st>>>(
                    hn->dev, t_k + (i + 1) * krow, t_v + (i + 1) * krow, hn->l, 0, tl0, ntl,
                    QStage{nullptr, nullptr, 0});
                KIVI_LAUNCHED();
                hn->total_launches++;
            }
            append_bookkeeping(hn);
        } else {
            KIVI_CUDA(launch_pdl(fast::combine_kernel, dim3((unsigned)n_comb), dim3(fast::D), 0, st,
                                 (const float*)h->part_o, (const float2*)h->part_ml, n_sub,
                                 out + i * krow, (float2*)nullptr, cmode, (int64_t)U));
            KIVI_LAUNCHED();
            h->total_launches++;
        }
    }
    return KIVI_OK;
}
}  // extern "C++"

static kivi_status decode_layers_enqueue(kivi_cache* const* caches, int32_t n_layers,
                                         const float* t_q, const float* t_k, const float* t_v,
                                         int32_t q_per_kv, float* out, int32_t scale_logits,
                                         void* stream) {
    const int64_t U = caches[0]->n_units, d = caches[0]->cfg.head_dim;
    const int64_t qrow = U * q_per_kv * d, krow = U * d;
    if (step_fusable(caches, n_layers, q_per_kv, t_q, t_k, t_v, out)) {
        if (caches[0]->cfg.bits == 2)
            return decode_layers_fused<2>(caches, n_layers, t_q, t_k, t_v, out, scale_logits, S(stream));
        return decode_layers_fused<4>(caches, n_layers, t_q, t_k, t_v, out, scale_logits, S(stream));
    }
    for (int32_t i = 0; i < n_layers; ++i) {
        kivi_status rc = kivi_decode(caches[i], t_q + i * qrow, t_k + i * krow, t_v + i * krow,
                                     q_per_kv, out + i * qrow, nullptr, scale_logits, stream);
        if (rc) return rc;
    }
    return KIVI_OK;
}

kivi_status kivi_decode_layers(kivi_cache* const* caches, int32_t n_layers, const float* t_q,
                               const float* t_k, const float* t_v, int32_t q_per_kv, float* out,
                               int32_t scale_logits, void* stream) {
    kivi_status rc = check_layers(caches, n_layers);
    if (rc) return rc;
    if (q_per_kv < 1) return fail(KIVI_ERR_SHAPE, "q_per_kv must be >= 1");
    if (!t_q || !t_k || !t_v || !out) return fail(KIVI_ERR_SHAPE, "decode_layers: NULL rows");
    DeviceGuard g(caches[0]->device);
    return decode_layers_enqueue(caches, n_layers, t_q, t_k, t_v, q_per_kv, out, scale_logits,
                                 stream);
}

namespace {
// Device staging of kivi_decode_layers_host, one per (host thread, device):
// the step's rows for every layer, uploaded in three copies.  Optionally the
// whole step (uploads, every layer's kernels, the result copy) is captured as
// a CUDA graph and replayed: re-captured every step (the kernels' arguments
// follow l) and applied to the instantiated graph with cudaGraphExecUpdate,
// re-instantiated only when the launch topology changes.
struct StepStage {
    float* q = nullptr;
    float* k = nullptr;
    float* v = nullptr;
    float* out = nullptr;
    int64_t cap_q = 0, cap_k = 0, cap_v = 0, cap_out = 0;
    // layer i's rows go up on h2d (gated by ev_in[i]) while earlier layers
    // compute; its output comes back on d2h after ev_out[i]
    cudaStream_t h2d = nullptr, d2h = nullptr;
    std::vector<cudaEvent_t> ev_in, ev_out;
    cudaEvent_t ev_start = nullptr, ev_join = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t graph_steps = 0, graph_updates_failed = 0, graph_capture_failed = 0;
    cudaError_t init(int n_layers) {
        cudaError_t e = cudaSuccess;
        if (!h2d) {
            if ((e = cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking))) return e;
            if ((e = cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking))) return e;
            if ((e = cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming))) return e;
            if ((e = cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming))) return e;
        }
        while ((int)ev_in.size() < n_layers) {
            cudaEvent_t a = nullptr, b = nullptr;
            if ((e = cudaEventCreateWithFlags(&a, cudaEventDisableTiming))) return e;
            if ((e = cudaEventCreateWithFlags(&b, cudaEventDisableTiming))) return e;
            ev_in.push_back(a);
            ev_out.push_back(b);
        }
        return e;
    }
    ~StepStage() {
        cudaFree(q);
        cudaFree(k);
        cudaFree(v);
        cudaFree(out);
        for (auto e : ev_in) cudaEventDestroy(e);
        for (auto e : ev_out) cudaEventDestroy(e);
        if (ev_start) cudaEventDestroy(ev_start);
        if (ev_join) cudaEventDestroy(ev_join);
        if (h2d) cudaStreamDestroy(h2d);
        if (d2h) cudaStreamDestroy(d2h);
        if (exec) cudaGraphExecDestroy(exec);
    }
};
// Device address of pinned, device-mapped host memory (cudaHostAlloc /
// cudaHostRegister; with unified addressing every pinned allocation is
// mapped), or nullptr for pageable memory.
const float* mapped(const float* host) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, host) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (at.type != cudaMemoryTypeHost || at.devicePointer == nullptr) return nullptr;
    return static_cast<const float*>(at.devicePointer);
}
StepStage& step_stage() {
    thread_local StepStage s[kMaxDevices];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = 0;
    return s[dev];
}
}  // namespace

kivi_status kivi_decode_layers_host(kivi_cache* const* caches, int32_t n_layers, const float* t_q,
                                    const float* t_k, const float* t_v, int32_t q_per_kv,
                                    float* out, int32_t scale_logits, void* stream) {
    kivi_status rc = check_layers(caches, n_layers);
    if (rc) return rc;
    if (q_per_kv < 1) return fail(KIVI_ERR_SHAPE, "q_per_kv must be >= 1");
    if (!t_q || !t_k || !t_v || !out) return fail(KIVI_ERR_SHAPE, "decode_layers: NULL rows");
    DeviceGuard g(caches[0]->device);
    const int64_t U = caches[0]->n_units, d = caches[0]->cfg.head_dim;
    const int64_t nq = n_layers * U * q_per_kv * d, nk = n_layers * U * d;
    StepStage& sg = step_stage();
    if ((rc = ensure(&sg.q, &sg.cap_q, nq))) return rc;
    if ((rc = ensure(&sg.k, &sg.cap_k, nk))) return rc;
    if ((rc = ensure(&sg.v, &sg.cap_v, nk))) return rc;
    if ((rc = ensure(&sg.out, &sg.cap_out, nq))) return rc;
    // A step that grows a cache (capacity doubling also regrows its partial
    // buffers) runs directly: allocations are not allowed inside a capture.
    bool grows = false;
    for (int32_t i = 0; i < n_layers; ++i) {
        grows |= caches[i]->l + 1 > caches[i]->cap;
        rc = ensure_capacity(caches[i], caches[i]->l + 1, S(stream));
        if (rc) return rc;
    }
    KIVI_CUDA(sg.init(n_layers));
    cudaStream_t st = S(stream);
    const int64_t qrow = U * q_per_kv * d, krow = U * d;
    // zero-copy rows (one layer, rows <= KIVI_ZERO_COPY_BYTES, default 64 KiB)
    const bool zero_copy =
        n_layers == 1 && (int64_t)sizeof(float) * qrow <= tune().zero_copy_bytes;
    auto enqueue = [&]() -> kivi_status {
        if (n_layers == 1) {
            // one layer: nothing to overlap the copies with; one stream
            // avoids the cross-stream event latencies (C1: a ~25 us step).
            // Small rows in pinned (device-mapped) host memory skip the copy
            // engine: the append kernel reads the key/value rows and the
            // merge kernel writes the outputs across PCIe itself (each copy
            // is a few us of DMA setup on a latency-bound step).  q is read
            // by every item of the attend, so it is uploaded.
            const float* dk = zero_copy ? mapped(t_k) : nullptr;
            const float* dv = zero_copy ? mapped(t_v) : nullptr;
            float* dout = zero_copy ? const_cast<float*>(mapped(out)) : nullptr;
            const float* dq = zero_copy ? mapped(t_q) : nullptr;
            if (!dq)
                KIVI_CUDA(cudaMemcpyAsync(sg.q, t_q, sizeof(float) * qrow, cudaMemcpyHostToDevice, st));
            if (!dk || !dv) {
                KIVI_CUDA(cudaMemcpyAsync(sg.k, t_k, sizeof(float) * krow, cudaMemcpyHostToDevice, st));
                KIVI_CUDA(cudaMemcpyAsync(sg.v, t_v, sizeof(float) * krow, cudaMemcpyHostToDevice, st));
                dk = sg.k;
                dv = sg.v;
            }
            // q is read by every attend item: the append warps stage it from
            // the mapped host rows into device memory (no copy-engine call)
            kivi_status r = decode_impl(caches[0], sg.q, dk, dv, q_per_kv, dout ? dout : sg.out,
                                        nullptr, scale_logits, stream, dq);
            if (r) return r;
            if (!dout)
                KIVI_CUDA(cudaMemcpyAsync(out, sg.out, sizeof(float) * qrow, cudaMemcpyDeviceToHost, st));
            return KIVI_OK;
        }
        // fork the copy streams off `stream` (this call's work starts after
        // what the caller enqueued before it)
        KIVI_CUDA(cudaEventRecord(sg.ev_start, st));
        KIVI_CUDA(cudaStreamWaitEvent(sg.h2d, sg.ev_start, 0));
        KIVI_CUDA(cudaStreamWaitEvent(sg.d2h, sg.ev_start, 0));
        for (int32_t i = 0; i < n_layers; ++i) {
            KIVI_CUDA(cudaMemcpyAsync(sg.q + i * qrow, t_q + i * qrow, sizeof(float) * qrow,
                                      cudaMemcpyHostToDevice, sg.h2d));
            KIVI_CUDA(cudaMemcpyAsync(sg.k + i * krow, t_k + i * krow, sizeof(float) * krow,
                                      cudaMemcpyHostToDevice, sg.h2d));
            KIVI_CUDA(cudaMemcpyAsync(sg.v + i * krow, t_v + i * krow, sizeof(float) * krow,
                                      cudaMemcpyHostToDevice, sg.h2d));
            KIVI_CUDA(cudaEventRecord(sg.ev_in[i], sg.h2d));
        }
        for (int32_t i = 0; i < n_layers; ++i) {
            KIVI_CUDA(cudaStreamWaitEvent(st, sg.ev_in[i], 0));
            kivi_status r = kivi_decode(caches[i], sg.q + i * qrow, sg.k + i * krow,
                                        sg.v + i * krow, q_per_kv, sg.out + i * qrow, nullptr,
                                        scale_logits, stream);
            if (r) return r;
            KIVI_CUDA(cudaEventRecord(sg.ev_out[i], st));
            KIVI_CUDA(cudaStreamWaitEvent(sg.d2h, sg.ev_out[i], 0));
            KIVI_CUDA(cudaMemcpyAsync(out + i * qrow, sg.out + i * qrow, sizeof(float) * qrow,
                                      cudaMemcpyDeviceToHost, sg.d2h));
        }
        // join: `stream` ends after the last result copy
        KIVI_CUDA(cudaEventRecord(sg.ev_join, sg.d2h));
        KIVI_CUDA(cudaStreamWaitEvent(st, sg.ev_join, 0));
        return KIVI_OK;
    };
    bool profiling = false;
    for (int32_t i = 0; i < n_layers; ++i) profiling |= caches[i]->profile;
    // per-step CUDA graph: on by default for one layer (C1 e2e 28.8-29.5k vs
    // 27.3-27.6k tokens/s), off for many (capturing 32 layers costs more host
    // time than the replay saves: C2 e2e 7,526-7,561 vs 7,661-7,675)
    const bool graph = tune().step_graph > 0 || (tune().step_graph < 0 && n_layers == 1);
    if (graph && st != nullptr && !profiling && !grows) {
        // The partial-result buffers must already exist (an allocation inside
        // a capture invalidates it): the first call of a cache runs directly.
        bool warm = true;
        for (int32_t i = 0; i < n_layers; ++i) warm &= caches[i]->part_o != nullptr;
        if (warm) {
            std::vector<int64_t> l0(n_layers), kc(n_layers), vc(n_layers), ws(n_layers),
                kq(n_layers);
            for (int32_t i = 0; i < n_layers; ++i) {
                l0[i] = caches[i]->l;
                kq[i] = caches[i]->kq_done;
                kc[i] = caches[i]->kres_cap;
                vc[i] = caches[i]->vres_cap;
                ws[i] = caches[i]->work_seq;
            }
            KIVI_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            kivi_status r = enqueue();
            cudaGraph_t graph = nullptr;
            cudaError_t ce = cudaStreamEndCapture(st, &graph);
            if (r == KIVI_OK && ce == cudaSuccess && graph) {
                bool ok = false;
                if (sg.exec) {
                    cudaGraphExecUpdateResultInfo info{};
                    ok = cudaGraphExecUpdate(sg.exec, graph, &info) == cudaSuccess;
                    if (!ok) {
                        cudaGetLastError();
                        cudaGraphExecDestroy(sg.exec);
                        sg.exec = nullptr;
                        sg.graph_updates_failed++;
                    }
                }
                if (!ok) ok = cudaGraphInstantiate(&sg.exec, graph, 0) == cudaSuccess;
                cudaGraphDestroy(graph);
                if (ok) {
                    KIVI_CUDA(cudaGraphLaunch(sg.exec, st));
                    KIVI_CUDA(cudaStreamSynchronize(st));
                    sg.graph_steps++;
                    return KIVI_OK;
                }
            }
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();
            // capture failed: undo the host-side step bookkeeping and run directly
            if (getenv("KIVI_DEBUG_GRAPH"))
                fprintf(stderr, "kivi: step graph capture failed (%s / %s); direct launch\n",
                        r ? g_last_error.c_str() : "ok", cudaGetErrorString(ce));
            sg.graph_capture_failed++;
            for (int32_t i = 0; i < n_layers; ++i) {
                caches[i]->l = l0[i];
                caches[i]->kq_done = kq[i];
                caches[i]->kres_cap = kc[i];
                caches[i]->vres_cap = vc[i];
                caches[i]->work_seq = ws[i];
            }
        }
    }
    rc = enqueue();
    if (rc) return rc;
    KIVI_CUDA(cudaStreamSynchronize(st));
    return KIVI_OK;
}

// ---- q/k/v projection on the tensor cores (kernels_project.cuh) ------------

namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 2-D fp32 tensor map over a row-major [rows][cols] matrix, box [box_rows][32]
// with 128-byte swizzle (rows past `rows` read as zeros).
kivi_status make_tmap(CUtensorMap* tm, const float* base, int64_t rows, int64_t cols,
                      int box_rows) {
    EncodeTiledFn fn = encode_tiled();
    if (!fn) return fail(KIVI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)cols * sizeof(float)};
    const cuuint32_t box[2] = {32u, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1u, 1u};
    CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(KIVI_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return KIVI_OK;
}

__global__ void transpose_kernel(const float* __restrict__ in, int64_t rows, int64_t cols,
                                 float* __restrict__ out) {
    __shared__ float tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][i];
    }
}
}  // namespace

struct kivi_proj {
    int device = 0;
    int64_t hidden_in = 0, hidden_out = 0;
    float* wt[3] = {nullptr, nullptr, nullptr};  // W^T: [hidden_out][hidden_in]
    CUtensorMap tm_w[3];
    int64_t launches = 0;
};

kivi_status kivi_proj_create(int device, int64_t hidden_in, int64_t hidden_out, const float* w_q,
                             const float* w_k, const float* w_v, void* stream, kivi_proj** out) {
    if (!out) return fail(KIVI_ERR_USAGE, "out is NULL");
    *out = nullptr;
    if (hidden_in < 32 || hidden_in % 32 != 0 || hidden_out < 128 || hidden_out % 128 != 0)
        return fail(KIVI_ERR_SHAPE,
                    "projection: hidden_in must be a multiple of 32 and hidden_out of 128 "
                    "(got %lld, %lld)",
                    (long long)hidden_in, (long long)hidden_out);
    if (!w_q || !w_k || !w_v) return fail(KIVI_ERR_USAGE, "projection: NULL weights");
    DeviceGuard g(device);
    kivi_proj* p = new kivi_proj();
    p->device = device;
    p->hidden_in = hidden_in;
    p->hidden_out = hidden_out;
    const float* w[3] = {w_q, w_k, w_v};
    cudaStream_t st = S(stream);
    for (int i = 0; i < 3; ++i) {
        if (dalloc(&p->wt[i], (size_t)(hidden_in * hidden_out)) != cudaSuccess) {
            kivi_proj_destroy(p);
            return fail(KIVI_ERR_OOM, "projection: weight allocation failed");
        }
        dim3 grid((unsigned)ceil_div(hidden_out, 32), (unsigned)ceil_div(hidden_in, 32));
        transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(w[i], hidden_in, hidden_out, p->wt[i]);
        kivi_status rc = make_tmap(&p->tm_w[i], p->wt[i], hidden_out, hidden_in, proj::BM);
        if (rc) {
            kivi_proj_destroy(p);
            return rc;
        }
    }
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        kivi_proj_destroy(p);
        return fail(KIVI_ERR_CUDA, "projection: %s", cudaGetErrorString(e));
    }
    *out = p;
    return KIVI_OK;
}

kivi_status kivi_proj_destroy(kivi_proj* p) {
    if (!p) return KIVI_OK;
    DeviceGuard g(p->device);
    for (auto w : p->wt) cudaFree(w);
    delete p;
    return KIVI_OK;
}

namespace {
// One launch of proj_kernel over rows [0, n) of x (N tiles of <= 128 rows).
kivi_status launch_proj(kivi_proj* p, const float* x, int64_t n, proj::ProjArgs a, int bits,
                        cudaStream_t st) {
    if (n < 1) return fail(KIVI_ERR_SHAPE, "projection: no rows");
    // N tiles of <= 128 rows: 4+ TMEM accumulator chunks (kernels_project.cuh)
    const int N = (int)std::min<int64_t>(128, round_up(n, 16));
    CUtensorMap tm_x;
    kivi_status rc = make_tmap(&tm_x, x, n, p->hidden_in, N);
    if (rc) return rc;
    const int a_bytes = proj::BM * proj::BK * 4, b_bytes = N * proj::BK * 4;
    const int stage = 2 * a_bytes + 2 * b_bytes;
    const int nkb = (int)(p->hidden_in / proj::BK);
    a.K = (int)p->hidden_in;
    a.N = N;
    a.tiles_m = (int)(p->hidden_out / proj::BM);
    a.stages = std::max(2, std::min(std::min(6, nkb), proj::SMEM_LIMIT / stage));
    a.hidden_out = (int)p->hidden_out;
    a.split_mode = tune().proj_split;
    const size_t smem = 1024 + (size_t)a.stages * stage + (3 * a.stages + 2) * 8;
    auto kern = bits == 4 ? proj::proj_kernel<4> : proj::proj_kernel<2>;
    // The attribute is per function and device, shared by every host thread
    // driving this device: always set the same value (the device's opt-in
    // maximum), so a thread launching a small tile never lowers the limit
    // under another thread's larger launch (a "too many resources" race).
    {
        int optin = 0;
        KIVI_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device));
        cudaFuncAttributes fa{};
        KIVI_CUDA(cudaFuncGetAttributes(&fa, kern));
        const int lim = optin - (int)fa.sharedSizeBytes;
        if ((int)smem > lim) return fail(KIVI_ERR_CONFIG, "projection: %zu B of shared memory > %d", smem, lim);
        KIVI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, lim));
    }
    const int n_tiles = (int)ceil_div(n, N);
    for (int t = 0; t < n_tiles; ++t) {  // one launch per N tile (n_valid / n_tile0 differ)
        proj::ProjArgs at = a;
        at.n_tile0 = t * N;
        at.n_valid = (int)std::min<int64_t>(N, n - (int64_t)t * N);
        kern<<<dim3((unsigned)(3 * at.tiles_m)), proj::THREADS, smem, st>>>(
            p->tm_w[0], p->tm_w[1], p->tm_w[2], tm_x, at);
        KIVI_LAUNCHED();
        p->launches++;
    }
    return KIVI_OK;
}
}  // namespace

kivi_status kivi_proj_gemm(kivi_proj* p, const float* x, int64_t n, float* out_q, float* out_k,
                           float* out_v, int64_t seq, void* stream) {
    if (!p || !x) return fail(KIVI_ERR_USAGE, "projection: NULL argument");
    if (!out_q || !out_k || !out_v) return fail(KIVI_ERR_USAGE, "projection: NULL output");
    if (seq < 0 || (seq > 0 && (n % seq != 0 || p->hidden_out % 128 != 0)))
        return fail(KIVI_ERR_SHAPE, "projection: rows must be a multiple of seq");
    DeviceGuard g(p->device);
    proj::ProjArgs a{};
    a.mode = seq > 0 ? 2 : 0;
    a.seq = (int)seq;
    a.heads = (int)(p->hidden_out / proj::BM);
    a.out[0] = out_q;
    a.out[1] = out_k;
    a.out[2] = out_v;
    return launch_proj(p, x, n, a, 2, S(stream));
}

kivi_status kivi_proj_append(kivi_proj* p, kivi_cache* h, const float* x, int64_t n, float* q_out,
                             void* stream) {
    if (!p || !h || !x || !q_out) return fail(KIVI_ERR_USAGE, "projection: NULL argument");
    const kivi_config& cf = h->cfg;
    if (cf.head_dim != 128 || cf.group_size != 32 || (cf.bits != 2 && cf.bits != 4))
        return fail(KIVI_ERR_CONFIG,
                    "fused projection-append needs head_dim 128, group 32, 2 or 4 bits");
    const int64_t heads = p->hidden_out / proj::BM;
    if (h->n_units != n * heads)
        return fail(KIVI_ERR_SHAPE, "projection: cache has %lld units, rows x heads = %lld",
                    (long long)h->n_units, (long long)(n * heads));
    if (h->device != p->device) return fail(KIVI_ERR_USAGE, "projection and cache on different devices");
    DeviceGuard g(p->device);
    cudaStream_t st = S(stream);
    kivi_status rc = ensure_capacity(h, h->l + 1, st);
    if (rc) return rc;
    proj::ProjArgs a{};
    a.mode = 1;
    a.out[0] = q_out;
    a.c = h->dev;
    a.l = h->l;
    a.heads = (int)heads;
    rc = launch_proj(p, x, n, a, cf.bits, st);
    if (rc) return rc;
    h->total_launches += ceil_div(n, 256);
    int tl0, ntl;
    key_tiles_due(h, &tl0, &ntl);
    if (ntl > 0) {
        // complete key tiles of this step: the projection wrote token l into the ring
        const int64_t groups = h->n_units * ntl * (128 / FLUSH_GPT);
        const unsigned fgrid = (unsigned)ceil_div(groups, 256);
        if (cf.bits == 2)
            append_flush_fast_kernel<2><<<fgrid, 256, 0, st>>>(h->dev, nullptr, nullptr, h->l, 0,
                                                              tl0, ntl, QStage{nullptr, nullptr, 0});
        else
            append_flush_fast_kernel<4><<<fgrid, 256, 0, st>>>(h->dev, nullptr, nullptr, h->l, 0,
                                                              tl0, ntl, QStage{nullptr, nullptr, 0});
        KIVI_LAUNCHED();
        h->total_launches++;
    }
    append_bookkeeping(h);
    return KIVI_OK;
}

kivi_status kivi_step_graph_stats(int64_t* replayed, int64_t* reinstantiated,
                                  int64_t* capture_failed) {
    StepStage& sg = step_stage();
    if (replayed) *replayed = sg.graph_steps;
    if (reinstantiated) *reinstantiated = sg.graph_updates_failed;
    if (capture_failed) *capture_failed = sg.graph_capture_failed;
    return KIVI_OK;
}

kivi_status kivi_host_join(kivi_cache* h, void* stream) {
    if (!h) return fail(KIVI_ERR_USAGE, "cache is NULL");
    if (!h->d2h) return KIVI_OK;  // no host-path call yet
    DeviceGuard g(h->device);
    for (auto& sg : h->stg) KIVI_CUDA(cudaStreamWaitEvent(S(stream), sg.out_free, 0));
    return KIVI_OK;
}

kivi_status kivi_export_unit(const kivi_cache* h, int64_t unit, kivi_unit_state* dst,
                             void* stream) {
    if (!h || !dst) return fail(KIVI_ERR_USAGE, "NULL argument");
    if (unit < 0 || unit >= h->n_units) return fail(KIVI_ERR_USAGE, "unit out of range");
    DeviceGuard g(h->device);
    cudaStream_t st = S(stream);
    const CacheDev& c = h->dev;
    const int64_t kg = h->kg(), vg = h->vg(), l = h->l;
    const int64_t d = h->cfg.head_dim, G = h->cfg.group_size, B = h->cfg.bits;
    const int64_t kgroups = kg * d / G, vgroups = vg * d / G;
    const int64_t kr = l - kg, vr = l - vg;
    const int64_t ntmp = 2 * (kgroups + vgroups) + (kr + vr) * d / 2 + 8;
    kivi_cache* hm = const_cast<kivi_cache*>(h);
    kivi_status rc = ensure(&hm->xfer, &hm->xfer_cap, ntmp);
    if (rc) return rc;
    double* tmp = hm->xfer;
    double *kz = tmp, *ks = kz + kgroups, *vz = ks + kgroups, *vs = vz + vgroups;
    float* kres = reinterpret_cast<float*>(vs + vgroups);
    float* vres = kres + kr * d;
    if (kgroups)
        pairs_to_zs_kernel<<<grid_for(kgroups), 256, 0, st>>>(c.kpairs + unit * c.kp_ustride,
                                                               kgroups, c.maxc, kz, ks);
    if (vgroups)
        pairs_to_zs_kernel<<<grid_for(vgroups), 256, 0, st>>>(c.vpairs + unit * c.vp_ustride,
                                                               vgroups, c.maxc, vz, vs);
    if (kr)
        KIVI_CUDA(cudaMemcpyAsync(kres, c.kring + unit * c.ring_ustride, sizeof(float) * kr * d,
                                  cudaMemcpyDeviceToDevice, st));
    if (vr)
        ring_gather_kernel<<<grid_for(vr * d), 256, 0, st>>>(c.vring + unit * c.ring_ustride, vg, vr,
                                                             c.R, c.d, vres);
    KIVI_LAUNCHED();
    const size_t kbytes = (size_t)ceil_div(kg * d * B, 8), vbytes = (size_t)ceil_div(vg * d * B, 8);
    if (dst->key_packed && kbytes)
        KIVI_CUDA(cudaMemcpyAsync(dst->key_packed, c.kcodes + unit * c.k_ustride, kbytes,
                                  cudaMemcpyDeviceToHost, st));
    if (dst->value_packed && vbytes)
        KIVI_CUDA(cudaMemcpyAsync(dst->value_packed, c.vcodes + unit * c.v_ustride, vbytes,
                                  cudaMemcpyDeviceToHost, st));
    if (dst->key_zero && kgroups)
        KIVI_CUDA(cudaMemcpyAsync(dst->key_zero, kz, 8 * kgroups, cudaMemcpyDeviceToHost, st));
    if (dst->key_scale && kgroups)
        KIVI_CUDA(cudaMemcpyAsync(dst->key_scale, ks, 8 * kgroups, cudaMemcpyDeviceToHost, st));
    if (dst->value_zero && vgroups)
        KIVI_CUDA(cudaMemcpyAsync(dst->value_zero, vz, 8 * vgroups, cudaMemcpyDeviceToHost, st));
    if (dst->value_scale && vgroups)
        KIVI_CUDA(cudaMemcpyAsync(dst->value_scale, vs, 8 * vgroups, cudaMemcpyDeviceToHost, st));
    if (dst->key_residual && kr)
        KIVI_CUDA(cudaMemcpyAsync(dst->key_residual, kres, sizeof(float) * kr * d,
                                  cudaMemcpyDeviceToHost, st));
    if (dst->value_residual && vr)
        KIVI_CUDA(cudaMemcpyAsync(dst->value_residual, vres, sizeof(float) * vr * d,
                                  cudaMemcpyDeviceToHost, st));
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(KIVI_ERR_CUDA, "export: %s", cudaGetErrorString(e));
    return KIVI_OK;
}

kivi_status kivi_import_unit(kivi_cache* h, int64_t unit, int64_t total_tokens,
                             int64_t key_residual_capacity, int64_t value_residual_capacity,
                             const kivi_unit_state* src, void* stream) {
    if (!h || !src) return fail(KIVI_ERR_USAGE, "NULL argument");
    if (unit < 0 || unit >= h->n_units) return fail(KIVI_ERR_USAGE, "unit out of range");
    if (total_tokens < 0) return fail(KIVI_ERR_USAGE, "negative token count");
    DeviceGuard g(h->device);
    cudaStream_t st = S(stream);
    kivi_status rc = ensure_capacity(h, total_tokens, st);
    if (rc) return rc;
    h->l = total_tokens;
    h->kq_done = 0;
    h->kres_cap = key_residual_capacity;
    h->vres_cap = value_residual_capacity;
    CacheDev& c = h->dev;
    const int64_t kg = h->kg(), vg = h->vg(), l = h->l;
    const int64_t d = h->cfg.head_dim, G = h->cfg.group_size, B = h->cfg.bits;
    const int64_t kgroups = kg * d / G, vgroups = vg * d / G;
    const int64_t kr = l - kg, vr = l - vg;
    const size_t kbytes = (size_t)ceil_div(kg * d * B, 8), vbytes = (size_t)ceil_div(vg * d * B, 8);
    if ((kgroups && (!src->key_packed || !src->key_zero || !src->key_scale)) ||
        (vgroups && (!src->value_packed || !src->value_zero || !src->value_scale)) ||
        (kr && !src->key_residual) || (vr && !src->value_residual))
        return fail(KIVI_ERR_USAGE, "import: missing state buffers");
    KIVI_CUDA(cudaMemsetAsync(c.kcodes + unit * c.k_ustride, 0, (size_t)c.k_ustride, st));
    KIVI_CUDA(cudaMemsetAsync(c.vcodes + unit * c.v_ustride, 0, (size_t)c.v_ustride, st));
    if (kbytes)
        KIVI_CUDA(cudaMemcpyAsync(c.kcodes + unit * c.k_ustride, src->key_packed, kbytes,
                                  cudaMemcpyHostToDevice, st));
    if (vbytes)
        KIVI_CUDA(cudaMemcpyAsync(c.vcodes + unit * c.v_ustride, src->value_packed, vbytes,
                                  cudaMemcpyHostToDevice, st));
    const int64_t ntmp = 2 * (kgroups + vgroups) + (kr + vr) * d / 2 + 8;
    rc = ensure(&h->xfer, &h->xfer_cap, ntmp);
    if (rc) return rc;
    double* tmp = h->xfer;
    double *kz = tmp, *ks = kz + kgroups, *vz = ks + kgroups, *vs = vz + vgroups;
    float* kres = reinterpret_cast<float*>(vs + vgroups);
    float* vres = kres + kr * d;
    if (kgroups) {
        KIVI_CUDA(cudaMemcpyAsync(kz, src->key_zero, 8 * kgroups, cudaMemcpyHostToDevice, st));
        KIVI_CUDA(cudaMemcpyAsync(ks, src->key_scale, 8 * kgroups, cudaMemcpyHostToDevice, st));
        zs_to_pairs_kernel<<<grid_for(kgroups), 256, 0, st>>>(kz, ks, kgroups, c.maxc,
                                                               c.kpairs + unit * c.kp_ustride);
    }
    if (vgroups) {
        KIVI_CUDA(cudaMemcpyAsync(vz, src->value_zero, 8 * vgroups, cudaMemcpyHostToDevice, st));
        KIVI_CUDA(cudaMemcpyAsync(vs, src->value_scale, 8 * vgroups, cudaMemcpyHostToDevice, st));
        zs_to_pairs_kernel<<<grid_for(vgroups), 256, 0, st>>>(vz, vs, vgroups, c.maxc,
                                                               c.vpairs + unit * c.vp_ustride);
    }
    if (kr)
        KIVI_CUDA(cudaMemcpyAsync(c.kring + unit * c.ring_ustride, src->key_residual,
                                  sizeof(float) * kr * d, cudaMemcpyHostToDevice, st));
    if (vr) {
        KIVI_CUDA(cudaMemcpyAsync(vres, src->value_residual, sizeof(float) * vr * d,
                                  cudaMemcpyHostToDevice, st));
        ring_scatter_kernel<<<grid_for(vr * d), 256, 0, st>>>(c.vring + unit * c.ring_ustride, vg, vr,
                                                              c.R, c.d, vres);
    }
    KIVI_LAUNCHED();
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(KIVI_ERR_CUDA, "import: %s", cudaGetErrorString(e));
    return KIVI_OK;
}

kivi_status kivi_materialize(const kivi_cache* h, float* keys_out, float* values_out,
                             void* stream) {
    if (!h) return fail(KIVI_ERR_USAGE, "cache is NULL");
    DeviceGuard g(h->device);
    if (h->l == 0) return KIVI_OK;
    cudaStream_t st = S(stream);
    materialize_kernel<<<grid_for(h->n_units * h->l * h->cfg.head_dim), 256, 0, st>>>(
        h->dev, h->l, h->kg(), h->vg(), keys_out, values_out);
    KIVI_LAUNCHED();
    return KIVI_OK;
}

kivi_status kivi_quantize_matrix(const float* m, int64_t rows, int64_t cols, int32_t bits,
                                 int64_t group_size, kivi_axis axis, uint8_t* packed,
                                 double* zero_points, double* scales, void* stream) {
    if (bits < 1 || bits > 8) return fail(KIVI_ERR_CONFIG, "bits must be in [1, 8], got %d", bits);
    if (group_size < 1) return fail(KIVI_ERR_CONFIG, "group_size must be >= 1");
    if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8))
        return fail(KIVI_ERR_CONFIG,
                    "packed storage requires bits in {1,2,4,8}; B=%d is fake-quant only", bits);
    const int64_t extent = axis == KIVI_PER_CHANNEL ? rows : cols;
    if (extent % group_size != 0)
        return fail(KIVI_ERR_SHAPE,
                    "quantize: %s grouped axis extent %lld not divisible by group size %lld "
                    "(matrix %lldx%lld)",
                    axis == KIVI_PER_CHANNEL ? "per_channel" : "per_token", (long long)extent,
                    (long long)group_size, (long long)rows, (long long)cols);
    if (rows * cols == 0) return KIVI_OK;
    cudaStream_t st = S(stream);
    const int64_t nbytes = ceil_div(rows * cols * bits, 8);
    KIVI_CUDA(scratch(0).ensure((size_t)round_up(nbytes, 4)));
    uint8_t* tmp = static_cast<uint8_t*>(scratch(0).p);
    KIVI_CUDA(cudaMemsetAsync(tmp, 0, (size_t)round_up(nbytes, 4), st));
    quantize_matrix_kernel<<<grid_for(rows * cols / group_size), 256, 0, st>>>(
        m, rows, cols, bits, (int)group_size, axis == KIVI_PER_CHANNEL, tmp, zero_points, scales);
    cudaError_t le = cudaGetLastError();
    cudaError_t ce = cudaMemcpyAsync(packed, tmp, (size_t)nbytes, cudaMemcpyDefault, st);
    cudaError_t se = cudaStreamSynchronize(st);
    if (le != cudaSuccess) return fail(KIVI_ERR_CUDA, "quantize: %s", cudaGetErrorString(le));
    if (ce != cudaSuccess) return fail(KIVI_ERR_CUDA, "quantize: %s", cudaGetErrorString(ce));
    if (se != cudaSuccess) return fail(KIVI_ERR_CUDA, "quantize: %s", cudaGetErrorString(se));
    return KIVI_OK;
}

kivi_status kivi_dequantize_matrix(const uint8_t* packed, const double* zero_points,
                                   const double* scales, int64_t rows, int64_t cols, int32_t bits,
                                   int64_t group_size, kivi_axis axis, float* out, void* stream) {
    if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8))
        return fail(KIVI_ERR_USAGE, "unpack_codes: bits must be one of {1,2,4,8}");
    if (group_size < 1) return fail(KIVI_ERR_CONFIG, "group_size must be >= 1");
    if (rows * cols == 0) return KIVI_OK;
    // read_code views the stream as 32-bit words: stage into a padded buffer.
    cudaStream_t st = S(stream);
    const int64_t nbytes = ceil_div(rows * cols * bits, 8);
    KIVI_CUDA(scratch(1).ensure((size_t)round_up(nbytes, 4)));
    uint8_t* tmp = static_cast<uint8_t*>(scratch(1).p);
    KIVI_CUDA(cudaMemsetAsync(tmp, 0, (size_t)round_up(nbytes, 4), st));
    KIVI_CUDA(cudaMemcpyAsync(tmp, packed, (size_t)nbytes, cudaMemcpyDefault, st));
    dequantize_matrix_kernel<<<grid_for(rows * cols), 256, 0, st>>>(
        tmp, zero_points, scales, rows, cols, bits, (int)group_size, axis == KIVI_PER_CHANNEL, out);
    cudaError_t le = cudaGetLastError();
    cudaError_t se = cudaStreamSynchronize(st);
    if (le != cudaSuccess) return fail(KIVI_ERR_CUDA, "dequantize: %s", cudaGetErrorString(le));
    if (se != cudaSuccess) return fail(KIVI_ERR_CUDA, "dequantize: %s", cudaGetErrorString(se));
    return KIVI_OK;
}

kivi_status kivi_quantize_codes(const float* m, int64_t rows, int64_t cols, int32_t bits,
                                int64_t group_size, kivi_axis axis, uint8_t* codes,
                                double* zero_points, double* scales, void* stream) {
    if (bits < 1 || bits > 8) return fail(KIVI_ERR_CONFIG, "bits must be in [1, 8], got %d", bits);
    if (group_size < 1) return fail(KIVI_ERR_CONFIG, "group_size must be >= 1");
    const int64_t extent = axis == KIVI_PER_CHANNEL ? rows : cols;
    if (extent % group_size != 0)
        return fail(KIVI_ERR_SHAPE,
                    "quantize: %s grouped axis extent %lld not divisible by group size %lld "
                    "(matrix %lldx%lld)",
                    axis == KIVI_PER_CHANNEL ? "per_channel" : "per_token", (long long)extent,
                    (long long)group_size, (long long)rows, (long long)cols);
    if (rows * cols == 0) return KIVI_OK;
    quantize_codes_kernel<<<grid_for(rows * cols / group_size), 256, 0, S(stream)>>>(
        m, rows, cols, bits, (int)group_size, axis == KIVI_PER_CHANNEL, codes, zero_points, scales);
    KIVI_LAUNCHED();
    return KIVI_OK;
}

kivi_status kivi_quantize_group(const float* values, int64_t n, int32_t bits, uint8_t* codes,
                                double* zero_point, double* scale, float* dequantized,
                                void* stream) {
    if (n < 1) return fail(KIVI_ERR_USAGE, "quantize_group: empty group");
    if (bits < 1 || bits > 8) return fail(KIVI_ERR_USAGE, "quantize_group: bits out of range");
    if (n >= (1LL << 31)) return fail(KIVI_ERR_SHAPE, "quantize_group: group too large");
    quantize_group_kernel<<<1, 256, 0, S(stream)>>>(values, (int)n, (1 << bits) - 1, codes,
                                                    zero_point, scale, dequantized);
    KIVI_LAUNCHED();
    return KIVI_OK;
}

kivi_status kivi_dequantize_codes(const uint8_t* codes, const double* zero_points,
                                  const double* scales, int64_t rows, int64_t cols,
                                  int64_t group_size, kivi_axis axis, float* out, void* stream) {
    if (group_size < 1) return fail(KIVI_ERR_CONFIG, "group_size must be >= 1");
    if (rows * cols == 0) return KIVI_OK;
    dequantize_codes_kernel<<<grid_for(rows * cols), 256, 0, S(stream)>>>(
        codes, zero_points, scales, rows, cols, (int)group_size, axis == KIVI_PER_CHANNEL, out);
    KIVI_LAUNCHED();
    return KIVI_OK;
}

kivi_status kivi_pack_codes(const uint8_t* codes, int64_t n, int32_t bits, uint8_t* bytes,
                            void* stream) {
    if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8))
        return fail(KIVI_ERR_USAGE, "pack_codes: bits must be one of {1,2,4,8}, got %d", bits);
    if (n == 0) return KIVI_OK;
    cudaStream_t st = S(stream);
    KIVI_CUDA(scratch(2).ensure(sizeof(int)));
    int* bad = static_cast<int*>(scratch(2).p);
    KIVI_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
    pack_codes_kernel<<<grid_for(ceil_div(n * bits, 8)), 256, 0, st>>>(codes, n, bits, bytes, bad);
    int hbad = 0;
    cudaError_t le = cudaGetLastError();
    cudaError_t ce = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaError_t se = cudaStreamSynchronize(st);
    if (le != cudaSuccess || ce != cudaSuccess || se != cudaSuccess)
        return fail(KIVI_ERR_CUDA, "pack_codes: %s",
                    cudaGetErrorString(le != cudaSuccess ? le : (ce != cudaSuccess ? ce : se)));
    if (hbad) return fail(KIVI_ERR_USAGE, "pack_codes: code exceeds 2^%d-1", bits);
    return KIVI_OK;
}

kivi_status kivi_unpack_codes(const uint8_t* bytes, int64_t n, int32_t bits, uint8_t* codes,
                              void* stream) {
    if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8))
        return fail(KIVI_ERR_USAGE, "unpack_codes: bits must be one of {1,2,4,8}");
    if (n == 0) return KIVI_OK;
    unpack_codes_kernel<<<grid_for(n), 256, 0, S(stream)>>>(bytes, n, bits, codes);
    KIVI_LAUNCHED();
    return KIVI_OK;
}

kivi_status kivi_reference_attention(const float* q, int64_t n_q, const float* keys,
                                     const float* values, int64_t l, int64_t d,
                                     int32_t scale_logits, float* out, void* stream) {
    if (n_q < 1 || d < 1) return fail(KIVI_ERR_SHAPE, "reference_attention: empty query");
    if (l < 1) return fail(KIVI_ERR_SHAPE, "reference_attention: empty keys");
    cudaStream_t st = S(stream);
    KIVI_CUDA(scratch(3).ensure(sizeof(float) * (size_t)(n_q * l)));
    float* lg_scratch = static_cast<float*>(scratch(3).p);
    AttendGenericArgs a{};
    a.c.bits = 2;
    a.c.G = 1;
    a.c.R = (int)l;
    a.c.d = (int)d;
    a.c.maxc = 3;
    a.c.n_units = 1;
    a.c.kring = const_cast<float*>(keys);
    a.c.vring = const_cast<float*>(values);
    a.c.ring_ustride = 0;
    a.l = l;
    a.kg = 0;
    a.vg = 0;
    a.ring_mod = l;
    a.q = q;
    a.qpk = (int)n_q;
    a.out = out;
    a.weights = nullptr;
    a.scratch = lg_scratch;
    a.scale_logits = scale_logits;
    attend_generic_kernel<<<(unsigned)n_q, 256, generic_smem(d), st>>>(a);
    cudaError_t le = cudaGetLastError();
    cudaError_t se = cudaStreamSynchronize(st);
    if (le != cudaSuccess) return fail(KIVI_ERR_CUDA, "reference_attention: %s", cudaGetErrorString(le));
    if (se != cudaSuccess) return fail(KIVI_ERR_CUDA, "reference_attention: %s", cudaGetErrorString(se));
    return KIVI_OK;
}

kivi_status kivi_reload_tuning(void) {
    g_tune.load();
    g_tune_loaded = true;
    return KIVI_OK;
}

kivi_status kivi_set_attend_path(kivi_cache* h, int32_t path) {
    if (!h) return fail(KIVI_ERR_USAGE, "cache is NULL");
    if (path < 0 || path > 2) return fail(KIVI_ERR_USAGE, "path must be 0, 1 or 2");
    h->attend_path = path;
    return KIVI_OK;
}

kivi_status kivi_profile_enable(kivi_cache* h, int32_t enable) {
    if (!h) return fail(KIVI_ERR_USAGE, "cache is NULL");
    if (enable < 0) return fail(KIVI_ERR_USAGE, "profile stride must be >= 0");
    h->profile = enable != 0;
    h->profile_stride = enable > 1 ? enable : 1;
    h->profile_seq = 0;
    return KIVI_OK;
}

kivi_status kivi_profile_read(kivi_cache* h, double* main_kernel_ms, int64_t* main_launches,
                              int64_t* total_launches) {
    if (!h) return fail(KIVI_ERR_USAGE, "cache is NULL");
    DeviceGuard g(h->device);
    double ms = 0.0;
    for (auto& ev : h->events) {
        KIVI_CUDA(cudaEventSynchronize(ev.second));
        float t = 0.f;
        KIVI_CUDA(cudaEventElapsedTime(&t, ev.first, ev.second));
        ms += t;
        h->event_pool.push_back(ev.first);
        h->event_pool.push_back(ev.second);
    }
    h->events.clear();
    if (main_kernel_ms) *main_kernel_ms = ms;
    if (main_launches) *main_launches = h->main_launches;
    if (total_launches) *total_launches = h->total_launches;
    h->main_launches = 0;
    h->total_launches = 0;
    return KIVI_OK;
}

kivi_status kivi_attend_bytes(const kivi_cache* h, int32_t q_per_kv, uint64_t* bytes_per_unit) {
    if (!h || !bytes_per_unit) return fail(KIVI_ERR_USAGE, "NULL argument");
    // ceil(kg*d*B/8) + ceil(vg*d*B/8) + (kg*d/G + vg*d/G)*2*4
    //             + (kr+vr)*d*4 + q_per_kv*d*4*2
    const int64_t d = h->cfg.head_dim, G = h->cfg.group_size, B = h->cfg.bits;
    const int64_t kg = h->kg(), vg = h->vg(), kr = h->l - kg, vr = h->l - vg;
    *bytes_per_unit = (uint64_t)(ceil_div(kg * d * B, 8) + ceil_div(vg * d * B, 8) +
                                 (kg * d / G + vg * d / G) * 8 + (kr + vr) * d * 4 +
                                 (int64_t)q_per_kv * d * 8);
    return KIVI_OK;
}

}  // extern "C"
