// Native decode driver: the reference's run_decode_benchmark
// (proj/src/workload.cpp:145-271) as C++ host code over the C-ABI
// (include/kivi_b200.h), one host thread per device.  See include/kivi_driver.h.
//
// The only device code here is data generation and the output checksum; the
// hot path (projection + append, attend, merge) is the library's.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

#include "kivi_driver.h"

namespace {

thread_local std::string g_err;

kivi_status set_err(kivi_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

// ---- counter-based N(0, 1) draws (splitmix64 + Box-Muller) -----------------
// Element i of draw stream s is a pure function of (seed, s, i): any device
// and any batch split produce the same numbers.
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__global__ void fill_normal_kernel(float* dst, int64_t n, uint64_t seed, uint64_t stream,
                                   int64_t first, float scale) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h = mix64(seed ^ mix64(stream * 0x632be59bd9b4e019ull + (uint64_t)(first + i)));
        const double u1 = ((double)(h >> 11) + 1.0) * (1.0 / 9007199254740993.0);  // (0, 1]
        const double u2 = (double)(mix64(h) >> 11) * (1.0 / 9007199254740992.0);   // [0, 1)
        dst[i] = (float)(sqrt(-2.0 * log(u1)) * cospi(2.0 * u2)) * scale;
    }
}

// sum and |sum| of n floats into acc[0], acc[1] (fp64)
__global__ void checksum_kernel(const float* x, int64_t n, double* acc) {
    double s = 0.0, a = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        s += x[i];
        a += fabs((double)x[i]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        a += __shfl_xor_sync(0xffffffffu, a, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&acc[0], s);
        atomicAdd(&acc[1], a);
    }
}

int blocks_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)); }

enum : uint64_t { STREAM_W = 1, STREAM_PROMPT = 1ull << 40, STREAM_TOKEN = 2ull << 40 };

struct Shard {
    int device = 0;
    int64_t b0 = 0, b1 = 0;            // batch rows [b0, b1)
    kivi_status status = KIVI_OK;
    std::string error;
    std::vector<float> step_ms;        // per decode step
    double checksum = 0.0, abs_sum = 0.0;
    uint64_t peak_bytes = 0;
};

struct Ctx {
    kivi_workload_spec spec;
    kivi_config cfg;
    uint64_t seed;
    const float* weights;
    const float* prompts;
    const float* tokens;
    uint64_t budget;
    // budget accounting across shards: every shard checks its own counted
    // bytes plus the other shards' (same schedule, so the same per-shard
    // growth): total = per-unit bytes x all units
};

#define DRV_CUDA(x)                                                                       \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess) {                                                          \
            sh.status = KIVI_ERR_CUDA;                                                    \
            sh.error = std::string(#x) + ": " + cudaGetErrorString(e_);                   \
            goto done;                                                                    \
        }                                                                                 \
    } while (0)
#define DRV_KIVI(x)                                                                       \
    do {                                                                                  \
        kivi_status s_ = (x);                                                             \
        if (s_ != KIVI_OK) {                                                              \
            sh.status = s_;                                                               \
            sh.error = std::string(#x) + ": " + kivi_last_error();                        \
            goto done;                                                                    \
        }                                                                                 \
    } while (0)

// Counted cache bytes of the whole job (every shard holds the same per-unit
// state: lockstep decode), the reference's memory_bytes summed over states.
uint64_t counted_bytes(const std::vector<kivi_cache*>& caches, int64_t units_total) {
    uint64_t per_unit = 0;
    for (kivi_cache* c : caches) {
        kivi_cache_info in{};
        if (kivi_cache_get_info(c, &in) == KIVI_OK) per_unit += in.key_memory_bytes + in.value_memory_bytes;
    }
    return per_unit * (uint64_t)units_total;
}

void run_shard(const Ctx& cx, Shard& sh) {
    const kivi_workload_spec& sp = cx.spec;
    const int64_t H = sp.kv_heads, D = sp.head_dim, hid = H * D, P = sp.prompt_len;
    const int64_t Bs = sh.b1 - sh.b0, U = Bs * H, units_total = sp.batch * H;
    std::vector<kivi_proj*> projs;
    std::vector<kivi_cache*> caches;
    std::vector<cudaEvent_t> ev;
    cudaStream_t st = nullptr;
    float *w = nullptr, *x = nullptr, *kq = nullptr, *kk = nullptr, *kv = nullptr, *tok = nullptr,
          *q = nullptr, *out = nullptr;
    double* acc = nullptr;
    double host_acc[2] = {0.0, 0.0};
    if (Bs <= 0) return;
    DRV_CUDA(cudaSetDevice(sh.device));
    DRV_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    DRV_CUDA(cudaMalloc(&w, sizeof(float) * 3 * hid * hid));
    DRV_CUDA(cudaMalloc(&x, sizeof(float) * Bs * P * hid));
    DRV_CUDA(cudaMalloc(&kq, sizeof(float) * Bs * P * hid));
    DRV_CUDA(cudaMalloc(&kk, sizeof(float) * Bs * P * hid));
    DRV_CUDA(cudaMalloc(&kv, sizeof(float) * Bs * P * hid));
    DRV_CUDA(cudaMalloc(&tok, sizeof(float) * std::max<int64_t>(1, sp.gen_len) * Bs * hid));
    DRV_CUDA(cudaMalloc(&q, sizeof(float) * U * D));
    DRV_CUDA(cudaMalloc(&out, sizeof(float) * U * D));
    DRV_CUDA(cudaMalloc(&acc, sizeof(double) * 2));
    DRV_CUDA(cudaMemsetAsync(acc, 0, sizeof(double) * 2, st));

    // the shard's prompts [Bs][P][hid] and decode tokens [gen][Bs][hid]
    if (cx.prompts) {
        DRV_CUDA(cudaMemcpyAsync(x, cx.prompts + sh.b0 * P * hid, sizeof(float) * Bs * P * hid,
                                 cudaMemcpyHostToDevice, st));
        for (int64_t s = 0; s < sp.gen_len; ++s)
            DRV_CUDA(cudaMemcpyAsync(tok + s * Bs * hid, cx.tokens + (s * sp.batch + sh.b0) * hid,
                                     sizeof(float) * Bs * hid, cudaMemcpyHostToDevice, st));
    } else {
        fill_normal_kernel<<<blocks_for(Bs * P * hid), 256, 0, st>>>(x, Bs * P * hid, cx.seed,
                                                                      STREAM_PROMPT, sh.b0 * P * hid, 1.0f);
        for (int64_t s = 0; s < sp.gen_len; ++s)
            fill_normal_kernel<<<blocks_for(Bs * hid), 256, 0, st>>>(
                tok + s * Bs * hid, Bs * hid, cx.seed, STREAM_TOKEN, (s * sp.batch + sh.b0) * hid, 1.0f);
        DRV_CUDA(cudaGetLastError());
    }

    // per layer: weights -> projection (its own transposed copy), prompt
    // projection straight into the per-unit layout, bulk prefill
    for (int64_t ly = 0; ly < sp.layers; ++ly) {
        if (cx.weights) {
            DRV_CUDA(cudaMemcpyAsync(w, cx.weights + ly * 3 * hid * hid, sizeof(float) * 3 * hid * hid,
                                     cudaMemcpyHostToDevice, st));
        } else {
            const float scale = 1.0f / std::sqrt((float)hid);
            fill_normal_kernel<<<blocks_for(3 * hid * hid), 256, 0, st>>>(
                w, 3 * hid * hid, cx.seed, STREAM_W + (uint64_t)ly, 0, scale);
            DRV_CUDA(cudaGetLastError());
        }
        kivi_proj* p = nullptr;
        DRV_KIVI(kivi_proj_create(sh.device, hid, hid, w, w + hid * hid, w + 2 * hid * hid, st, &p));
        projs.push_back(p);
        kivi_cache* c = nullptr;
        DRV_KIVI(kivi_cache_create(&cx.cfg, sh.device, U, P + sp.gen_len, &c));
        caches.push_back(c);
        DRV_KIVI(kivi_proj_gemm(p, x, Bs * P, kq, kk, kv, P, st));
        DRV_KIVI(kivi_prefill(c, kk, kv, P, st));
    }
    if (cx.budget) {
        const uint64_t used = counted_bytes(caches, units_total);
        if (used > cx.budget) {
            sh.status = KIVI_ERR_CAPACITY;
            sh.error = "memory budget exceeded at prefill: " + std::to_string(used) + " > " +
                       std::to_string(cx.budget) + " bytes";
            goto done;
        }
    }
    DRV_CUDA(cudaStreamSynchronize(st));

    // decode: per step and layer, projection + append (one launch), attend
    ev.resize(2 * std::max<int64_t>(1, sp.gen_len));
    for (auto& e : ev) DRV_CUDA(cudaEventCreate(&e));
    for (int64_t s = 0; s < sp.gen_len; ++s) {
        DRV_CUDA(cudaEventRecord(ev[2 * s], st));
        for (int64_t ly = 0; ly < sp.layers; ++ly) {
            DRV_KIVI(kivi_proj_append(projs[ly], caches[ly], tok + s * Bs * hid, Bs, q, st));
            DRV_KIVI(kivi_attend(caches[ly], q, 1, out, nullptr, 1, st));
            checksum_kernel<<<blocks_for(U * D), 256, 0, st>>>(out, U * D, acc);
        }
        DRV_CUDA(cudaEventRecord(ev[2 * s + 1], st));
        if (cx.budget) {
            const uint64_t used = counted_bytes(caches, units_total);
            if (used > cx.budget) {
                sh.status = KIVI_ERR_CAPACITY;
                sh.error = "memory budget exceeded at decode step " + std::to_string(s + 1) + ": " +
                           std::to_string(used) + " > " + std::to_string(cx.budget) + " bytes";
                goto done;
            }
        }
    }
    DRV_CUDA(cudaGetLastError());
    DRV_CUDA(cudaStreamSynchronize(st));
    for (int64_t s = 0; s < sp.gen_len; ++s) {
        float ms = 0.f;
        DRV_CUDA(cudaEventElapsedTime(&ms, ev[2 * s], ev[2 * s + 1]));
        sh.step_ms.push_back(ms);
    }
    DRV_CUDA(cudaMemcpy(host_acc, acc, sizeof host_acc, cudaMemcpyDeviceToHost));
    sh.checksum = host_acc[0];
    sh.abs_sum = host_acc[1];
    sh.peak_bytes = counted_bytes(caches, U);
done:
    if (st) cudaStreamSynchronize(st);
    for (auto e : ev)
        if (e) cudaEventDestroy(e);
    for (auto p : projs) kivi_proj_destroy(p);
    for (auto c : caches) kivi_cache_destroy(c);
    for (void* ptr : {(void*)w, (void*)x, (void*)kq, (void*)kk, (void*)kv, (void*)tok, (void*)q,
                      (void*)out, (void*)acc})
        if (ptr) cudaFree(ptr);
    if (st) cudaStreamDestroy(st);
}

double percentile(const std::vector<double>& sorted, double q) {  // workload.cpp:135-141
    if (sorted.empty()) return 0.0;
    const auto idx = (size_t)std::ceil(q * (double)sorted.size()) - 1;
    return sorted[std::min(idx, sorted.size() - 1)];
}

}  // namespace

extern "C" const char* kivi_driver_last_error(void) { return g_err.c_str(); }

extern "C" kivi_status kivi_run_decode_benchmark(const kivi_workload_spec* spec, const kivi_config* cfg,
                                                 const int32_t* devices, int32_t n_devices,
                                                 uint64_t seed, const float* weights,
                                                 const float* prompts, const float* tokens,
                                                 uint64_t budget_bytes, kivi_bench_report* report) {
    g_err.clear();
    if (!spec || !cfg || !devices || !report) return set_err(KIVI_ERR_USAGE, "NULL argument");
    if (n_devices < 1) return set_err(KIVI_ERR_USAGE, "no devices");
    const kivi_workload_spec& sp = *spec;
    // WorkloadSpec::validate (workload.cpp:12-17)
    if (std::min({sp.batch, sp.prompt_len, sp.layers, sp.kv_heads, sp.head_dim}) < 1)
        return set_err(KIVI_ERR_CONFIG, "workload counts must be >= 1");
    if (sp.gen_len < 0) return set_err(KIVI_ERR_CONFIG, "gen_len must be >= 0");
    kivi_status rc = kivi_config_validate(cfg);
    if (rc) return set_err(rc, "%s", kivi_last_error());
    if (cfg->head_dim != sp.head_dim)
        return set_err(KIVI_ERR_CONFIG, "run_decode_benchmark: cfg.head_dim must match spec.head_dim");
    if (sp.head_dim != 128 || cfg->group_size != 32 || (cfg->bits != 2 && cfg->bits != 4))
        return set_err(KIVI_ERR_CONFIG,
                       "native driver: fused projection needs head_dim 128, group 32, 2 or 4 bits");
    if ((weights == nullptr) != (prompts == nullptr) || (weights == nullptr) != (tokens == nullptr))
        return set_err(KIVI_ERR_USAGE, "weights, prompts and tokens: all or none");

    Ctx cx{sp, *cfg, seed, weights, prompts, tokens, budget_bytes};
    std::vector<Shard> shards(n_devices);
    for (int i = 0; i < n_devices; ++i) {
        shards[i].device = devices[i];
        shards[i].b0 = sp.batch * i / n_devices;
        shards[i].b1 = sp.batch * (i + 1) / n_devices;
    }
    std::vector<std::thread> th;
    for (int i = 0; i < n_devices; ++i) th.emplace_back(run_shard, std::cref(cx), std::ref(shards[i]));
    for (auto& t : th) t.join();
    for (auto& s : shards)
        if (s.status != KIVI_OK) return set_err(s.status, "device %d: %s", s.device, s.error.c_str());

    kivi_bench_report r{};
    r.decode_steps = sp.gen_len;
    r.n_devices = n_devices;
    std::vector<double> lat(sp.gen_len, 0.0);
    for (auto& s : shards) {
        for (int64_t k = 0; k < (int64_t)s.step_ms.size(); ++k) lat[k] = std::max(lat[k], (double)s.step_ms[k]);
        r.output_checksum += s.checksum;
        r.output_abs_sum += s.abs_sum;
        r.peak_cache_bytes += s.peak_bytes;
    }
    double total_ms = 0.0;
    for (double v : lat) total_ms += v;
    r.decode_seconds = total_ms / 1e3;
    if (sp.gen_len > 0 && total_ms > 0.0) r.tokens_per_sec = (double)(sp.batch * sp.gen_len) / r.decode_seconds;
    std::sort(lat.begin(), lat.end());
    r.p50_ms = percentile(lat, 0.50);
    r.p90_ms = percentile(lat, 0.90);
    r.p99_ms = percentile(lat, 0.99);
    *report = r;
    return KIVI_OK;
}
