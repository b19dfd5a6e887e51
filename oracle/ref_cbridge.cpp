// TEST INFRASTRUCTURE ONLY — ctypes-callable C bridge over the REFERENCE
// library compiled from /root/reference by oracle/Makefile (oracle/_ref).
// Used by tests/ (parity checker), __graft_entry__.smoke() and bench.py's
// CPU-baseline / --impl reference leg.  Never linked by the product.
//
// Every entry point calls the reference's own API:
//   prefill / append_token / decode_attention / materialize_* / memory_bytes
//   (reference proj/include/kivi/kv_cache.hpp:45-58, attention.hpp:18-27),
//   quantize_group / pack_codes / QuantizedTensor::quantize
//   (reference proj/include/kivi/quantize.hpp:35-70),
//   estimate_memory / max_batch_at_budget / SyntheticLayer /
//   run_decode_benchmark (reference proj/include/kivi/workload.hpp:41-73).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "kivi/analysis.hpp"
#include "kivi/dump_io.hpp"
#include "kivi/attention.hpp"
#include "kivi/kv_cache.hpp"
#include "kivi/quantize.hpp"
#include "kivi/workload.hpp"

using namespace kivi;

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
    if (dynamic_cast<const ShapeError*>(&e)) return 1;
    if (dynamic_cast<const UsageError*>(&e)) return 2;
    if (dynamic_cast<const ConfigError*>(&e)) return 3;
    return 9;
}

#define GUARD(...)                           \
    try {                                    \
        __VA_ARGS__;                         \
        return 0;                            \
    } catch (const std::exception& e) {      \
        g_err = e.what();                    \
        return code_of(e);                   \
    }

Matrix from(const float* p, int64_t rows, int64_t cols) {
    Matrix m(rows, cols);
    if (rows * cols) std::memcpy(m.data(), p, sizeof(float) * rows * cols);
    return m;
}

struct State {
    KeyCacheState key;
    ValueCacheState value;
};

CacheConfig cfg_of(int bits, int64_t G, int64_t R, int64_t d) { return CacheConfig{bits, G, R, d}; }

int code_of_budget(const std::exception& e) {
    if (dynamic_cast<const BudgetError*>(&e)) return 4;
    return code_of(e);
}

#define GUARD_B(...)                         \
    try {                                    \
        __VA_ARGS__;                         \
        return 0;                            \
    } catch (const std::exception& e) {      \
        g_err = e.what();                    \
        return code_of_budget(e);            \
    }

// spec[6] = batch, prompt_len, gen_len, layers, kv_heads, head_dim
WorkloadSpec spec_of(const int64_t* s) {
    WorkloadSpec w;
    w.batch = s[0];
    w.prompt_len = s[1];
    w.gen_len = s[2];
    w.layers = s[3];
    w.kv_heads = s[4];
    w.head_dim = s[5];
    return w;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_state_new() { return new State(); }
void ref_state_free(void* h) { delete static_cast<State*>(h); }
void* ref_state_clone(void* h) { return new State(*static_cast<State*>(h)); }

int ref_prefill(void* h, int bits, int64_t G, int64_t R, int64_t d, const float* K, const float* V,
                int64_t l) {
    GUARD({
        State* s = static_cast<State*>(h);
        PrefillResult r = prefill(from(K, l, d), from(V, l, d), cfg_of(bits, G, R, d));
        s->key = std::move(r.key);
        s->value = std::move(r.value);
    })
}

int ref_append(void* h, int bits, int64_t G, int64_t R, int64_t d, const float* tk,
               const float* tv) {
    GUARD({
        State* s = static_cast<State*>(h);
        append_token(s->key, s->value, from(tk, 1, d), from(tv, 1, d), cfg_of(bits, G, R, d));
    })
}

// out: d floats; weights: l floats after the append (may be NULL).
int ref_decode(void* h, int bits, int64_t G, int64_t R, int64_t d, const float* q, const float* tk,
               const float* tv, int scale_logits, float* out, float* weights) {
    GUARD({
        State* s = static_cast<State*>(h);
        AttentionOptions opts;
        opts.scale_logits = scale_logits != 0;
        DecodeOutput o = decode_attention(from(q, 1, d), from(tk, 1, d), from(tv, 1, d), s->key,
                                          s->value, cfg_of(bits, G, R, d), opts);
        std::memcpy(out, o.output.data(), sizeof(float) * d);
        if (weights) std::memcpy(weights, o.weights.data(), sizeof(float) * o.weights.size());
    })
}

// counters[8] = key.grouped.rows, key.residual.rows, key.total, key.residual_capacity,
//               value.grouped.rows, value.residual.rows, value.total, value.residual_capacity
// sizes[6]    = key packed bytes, key groups, value packed bytes, value groups,
//               memory_bytes(key), memory_bytes(value)
int ref_counters(void* h, int64_t* counters, uint64_t* sizes) {
    GUARD({
        State* s = static_cast<State*>(h);
        counters[0] = s->key.grouped.rows();
        counters[1] = s->key.residual.rows();
        counters[2] = s->key.total_tokens;
        counters[3] = s->key.residual_capacity;
        counters[4] = s->value.grouped.rows();
        counters[5] = s->value.residual.rows();
        counters[6] = s->value.total_tokens;
        counters[7] = s->value.residual_capacity;
        sizes[0] = s->key.grouped.packed().size();
        sizes[1] = (uint64_t)s->key.grouped.group_count();
        sizes[2] = s->value.grouped.packed().size();
        sizes[3] = (uint64_t)s->value.grouped.group_count();
        sizes[4] = memory_bytes(s->key);
        sizes[5] = memory_bytes(s->value);
    })
}

// Any pointer may be NULL.  Residuals are rows x d in token order.
int ref_export(void* h, uint8_t* kp, double* kz, double* ks, float* kr, uint8_t* vp, double* vz,
               double* vs, float* vr) {
    GUARD({
        State* s = static_cast<State*>(h);
        const auto& K = s->key.grouped;
        const auto& V = s->value.grouped;
        if (kp && !K.packed().empty()) std::memcpy(kp, K.packed().data(), K.packed().size());
        if (kz) std::copy(K.zero_points().begin(), K.zero_points().end(), kz);
        if (ks) std::copy(K.scales().begin(), K.scales().end(), ks);
        if (kr && s->key.residual.size())
            std::memcpy(kr, s->key.residual.data(), sizeof(float) * s->key.residual.size());
        if (vp && !V.packed().empty()) std::memcpy(vp, V.packed().data(), V.packed().size());
        if (vz) std::copy(V.zero_points().begin(), V.zero_points().end(), vz);
        if (vs) std::copy(V.scales().begin(), V.scales().end(), vs);
        if (vr && s->value.residual.size())
            std::memcpy(vr, s->value.residual.data(), sizeof(float) * s->value.residual.size());
    })
}

int ref_materialize(void* h, float* keys, float* values) {
    GUARD({
        State* s = static_cast<State*>(h);
        Matrix mk = materialize_keys(s->key), mv = materialize_values(s->value);
        if (keys && mk.size()) std::memcpy(keys, mk.data(), sizeof(float) * mk.size());
        if (values && mv.size()) std::memcpy(values, mv.data(), sizeof(float) * mv.size());
    })
}

int ref_quantize_group(const float* v, int64_t n, int bits, uint8_t* codes, double* z, double* s) {
    GUARD({
        GroupQuant g = quantize_group(std::span<const float>(v, (size_t)n), bits);
        std::copy(g.codes.begin(), g.codes.end(), codes);
        *z = g.zero_point;
        *s = g.scale;
    })
}

int ref_pack_codes(const uint8_t* codes, int64_t n, int bits, uint8_t* bytes) {
    GUARD({
        auto b = pack_codes(std::span<const uint8_t>(codes, (size_t)n), bits);
        std::copy(b.begin(), b.end(), bytes);
    })
}

int ref_quantize_matrix(const float* m, int64_t rows, int64_t cols, int bits, int64_t G,
                        int per_channel, uint8_t* packed, double* z, double* s) {
    GUARD({
        QuantParams p{bits, G, per_channel ? Axis::per_channel : Axis::per_token};
        QuantizedTensor t = QuantizedTensor::quantize(from(m, rows, cols), p);
        std::copy(t.packed().begin(), t.packed().end(), packed);
        std::copy(t.zero_points().begin(), t.zero_points().end(), z);
        std::copy(t.scales().begin(), t.scales().end(), s);
    })
}

int ref_reference_attention(const float* q, int64_t nq, const float* K, const float* V, int64_t l,
                            int64_t d, int scale_logits, float* out) {
    GUARD({
        AttentionOptions opts;
        opts.scale_logits = scale_logits != 0;
        Matrix o = reference_attention(from(q, nq, d), from(K, l, d), from(V, l, d), opts);
        std::memcpy(out, o.data(), sizeof(float) * o.size());
    })
}

// CPU baseline: n_units caches prefilled with uniform(-1,1) data of length
// l_prefill, then `warmup` untimed and `steps` timed decode_attention calls per
// unit (append + attend), spread over `threads` std::threads.  Returns the wall
// seconds of the timed decode loop (prefill excluded) in *seconds and a
// checksum of all outputs.
int ref_bench_decode(int bits, int64_t G, int64_t R, int64_t d, int64_t n_units, int64_t l_prefill,
                     int64_t warmup, int64_t steps, int threads, uint64_t seed, double* seconds,
                     double* checksum) {
    GUARD({
        const CacheConfig cfg = cfg_of(bits, G, R, d);
        std::vector<State> st((size_t)n_units);
        std::vector<std::vector<float>> qkv((size_t)n_units);
        auto worker_prefill = [&](int64_t u0, int64_t u1) {
            for (int64_t u = u0; u < u1; ++u) {
                std::mt19937_64 rng(seed + 7919ull * (uint64_t)u);
                std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
                Matrix K(l_prefill, d), V(l_prefill, d);
                for (Index i = 0; i < K.size(); ++i) K(i) = dist(rng);
                for (Index i = 0; i < V.size(); ++i) V(i) = dist(rng);
                PrefillResult r = prefill(K, V, cfg);
                st[(size_t)u].key = std::move(r.key);
                st[(size_t)u].value = std::move(r.value);
                auto& buf = qkv[(size_t)u];
                buf.resize((size_t)((warmup + steps) * 3 * d));
                for (auto& x : buf) x = dist(rng);
            }
        };
        const int T = std::max(1, threads);
        auto run_pool = [&](auto&& fn) {
            std::vector<std::thread> pool;
            const int64_t per = (n_units + T - 1) / T;
            for (int t = 0; t < T; ++t) {
                const int64_t u0 = t * per, u1 = std::min(n_units, u0 + per);
                if (u0 < u1) pool.emplace_back(fn, u0, u1);
            }
            for (auto& th : pool) th.join();
        };
        run_pool(worker_prefill);
        std::vector<double> sums((size_t)n_units, 0.0);
        int64_t s_begin = 0, s_end = warmup;
        auto worker_decode = [&](int64_t u0, int64_t u1) {
            for (int64_t s = s_begin; s < s_end; ++s) {
                for (int64_t u = u0; u < u1; ++u) {
                    const float* b = qkv[(size_t)u].data() + s * 3 * d;
                    DecodeOutput o = decode_attention(from(b, 1, d), from(b + d, 1, d),
                                                      from(b + 2 * d, 1, d), st[(size_t)u].key,
                                                      st[(size_t)u].value, cfg);
                    sums[(size_t)u] += (double)o.output.sum();
                }
            }
        };
        run_pool(worker_decode);  // untimed warm-up steps
        s_begin = warmup;
        s_end = warmup + steps;
        const auto t0 = std::chrono::steady_clock::now();
        run_pool(worker_decode);
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        double cs = 0.0;
        for (double v : sums) cs += v;
        *checksum = cs;
    })
}

// ---- workload layer (reference workload.cpp) ---------------------------------
// out[5] = fp, kivi, code, scale_zero, residual bytes; *ratio = compression.
int ref_estimate_memory(const int64_t* spec, int bits, int64_t G, int64_t R, uint64_t* out,
                        double* ratio) {
    GUARD({
        const MemoryEstimate e = estimate_memory(spec_of(spec), cfg_of(bits, G, R, spec[5]));
        out[0] = e.fp_bytes;
        out[1] = e.kivi_bytes;
        out[2] = e.code_bytes;
        out[3] = e.scale_zero_bytes;
        out[4] = e.residual_bytes;
        *ratio = e.compression_ratio;
    })
}

int ref_max_batch_at_budget(const int64_t* spec, uint64_t budget, int fp_mode, int bits,
                            int64_t G, int64_t R, int64_t* out) {
    GUARD_B({
        *out = max_batch_at_budget(spec_of(spec), budget, fp_mode ? BenchMode::fp : BenchMode::kivi,
                                   cfg_of(bits, G, R, spec[5]));
    })
}

// The exact synthetic data run_decode_benchmark draws (workload.cpp:157-160,
// 198-201, 222-223): per-layer W_q, W_k, W_v [hidden][hidden] (row-major,
// layers x 3), prompts [batch][prompt_len][hidden], decode tokens
// [gen_len][batch][hidden].
int ref_workload_data(const int64_t* spec, uint64_t seed, float* weights, float* prompts,
                      float* tokens) {
    GUARD({
        const WorkloadSpec w = spec_of(spec);
        const int64_t hidden = w.hidden();
        const size_t hh = (size_t)(hidden * hidden);
        for (int64_t ly = 0; ly < w.layers; ++ly) {
            SyntheticLayer L(hidden, seed + 1000003ull * (uint64_t)ly);
            std::memcpy(weights + (3 * ly + 0) * hh, L.w_q.data(), sizeof(float) * hh);
            std::memcpy(weights + (3 * ly + 1) * hh, L.w_k.data(), sizeof(float) * hh);
            std::memcpy(weights + (3 * ly + 2) * hh, L.w_v.data(), sizeof(float) * hh);
        }
        std::mt19937_64 data_rng(seed ^ 0x9e3779b97f4a7c15ull);
        const size_t ph = (size_t)(w.prompt_len * hidden);
        for (int64_t b = 0; b < w.batch; ++b) {
            const Matrix x = gaussian_matrix(w.prompt_len, hidden, data_rng);
            std::memcpy(prompts + b * ph, x.data(), sizeof(float) * ph);
        }
        for (int64_t step = 0; step < w.gen_len; ++step)
            for (int64_t b = 0; b < w.batch; ++b) {
                const Matrix t = gaussian_matrix(1, hidden, data_rng);
                std::memcpy(tokens + (step * w.batch + b) * hidden, t.data(), sizeof(float) * hidden);
            }
    })
}

// out_d[2] = tokens_per_sec, output_checksum; *peak = peak_cache_bytes.
int ref_run_decode_benchmark(const int64_t* spec, uint64_t seed, int fp_mode, int bits, int64_t G,
                             int64_t R, uint64_t budget, double* out_d, uint64_t* peak) {
    GUARD_B({
        const BenchReport r = run_decode_benchmark(
            spec_of(spec), cfg_of(bits, G, R, spec[5]), seed,
            fp_mode ? BenchMode::fp : BenchMode::kivi,
            budget ? std::optional<std::uint64_t>(budget) : std::nullopt);
        out_d[0] = r.tokens_per_sec;
        out_d[1] = r.output_checksum;
        *peak = r.peak_cache_bytes;
    })
}

// ---- KVQD dumps (reference dump_io.cpp) ---------------------------------------
// write: n tensors of rows x cols; read: dims[3] = heads, rows, cols, then data
// (call with data = NULL to get dims).  Errors: FormatError -> 5 with the byte
// offset in *offset.
int ref_write_dump(const char* path, const float* data, int64_t n, int64_t rows, int64_t cols) {
    GUARD({
        std::vector<Matrix> t;
        for (int64_t i = 0; i < n; ++i) t.push_back(from(data + i * rows * cols, rows, cols));
        write_dump(path, t);
    })
}

int ref_read_dump(const char* path, int64_t* dims, float* data, uint64_t* offset) {
    try {
        const std::vector<Matrix> t = read_dump(path);
        dims[0] = (int64_t)t.size();
        dims[1] = t.empty() ? 0 : t[0].rows();
        dims[2] = t.empty() ? 0 : t[0].cols();
        if (data)
            for (size_t i = 0; i < t.size(); ++i)
                std::memcpy(data + i * t[i].size(), t[i].data(), sizeof(float) * t[i].size());
        return 0;
    } catch (const FormatError& e) {
        g_err = e.what();
        *offset = e.byte_offset;
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

}  // extern "C"
