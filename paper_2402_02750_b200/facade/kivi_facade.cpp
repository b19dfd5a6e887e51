// Drop-in facade: the reference's kivi:: API (reference proj/include/kivi/
// {quantize,kv_cache,attention}.hpp) implemented over the B200 C-ABI
// (include/kivi_b200.h).  Callers and tests written against the reference
// relink unchanged; every quantize / pack / dequantize / append / attention
// computation runs on the GPU.  Host code here only validates arguments (with
// the reference's exception types and messages), moves data, and keeps the
// caller-owned states in the reference layout.
//
// State model: KeyCacheState / ValueCacheState remain plain values.  Each
// call loads the unit into a per-thread device cache (kivi_import_unit), runs
// the kernels, and writes the new state back (kivi_export_unit).  The batched
// C-ABI (one kivi_cache for a whole layer, state resident in HBM) is the
// high-throughput path; this facade is the drop-in for single-unit callers.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "kivi/attention.hpp"
#include "kivi/kv_cache.hpp"
#include "kivi/quantize.hpp"
#include "kivi_b200.h"

namespace kivi {

namespace detail {
struct TensorAccess {
    static QuantizedTensor make(std::vector<std::uint8_t> packed, std::vector<double> z,
                                std::vector<double> s, Index rows, Index cols,
                                const QuantParams& p) {
        QuantizedTensor t(p);
        t.packed_ = std::move(packed);
        t.zero_points_ = std::move(z);
        t.scales_ = std::move(s);
        t.rows_ = rows;
        t.cols_ = cols;
        return t;
    }
    static std::vector<std::uint8_t>& packed(QuantizedTensor& t) { return t.packed_; }
    static std::vector<double>& zeros(QuantizedTensor& t) { return t.zero_points_; }
    static std::vector<double>& scales(QuantizedTensor& t) { return t.scales_; }
    static Index& rows(QuantizedTensor& t) { return t.rows_; }
};
}  // namespace detail

namespace {

using detail::TensorAccess;

[[noreturn]] void raise(kivi_status st) {
    const std::string msg = kivi_last_error();
    switch (st) {
        case KIVI_ERR_SHAPE: throw ShapeError(msg);
        case KIVI_ERR_USAGE: throw UsageError(msg);
        case KIVI_ERR_CONFIG: throw ConfigError(msg);
        default: throw std::runtime_error("kivi_b200: " + msg);
    }
}

inline void check(kivi_status st) {
    if (st != KIVI_OK) raise(st);
}

inline void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("kivi facade: ") + what + ": " +
                                                   cudaGetErrorString(e));
}

// Per-thread pool of device blocks in power-of-two size classes: facade
// calls are small and frequent, and cudaFree synchronises the device.
class BlockPool {
public:
    void* take(std::size_t bytes) {
        const int cls = size_class(bytes);
        auto& fl = free_[cls];
        if (!fl.empty()) {
            void* p = fl.back();
            fl.pop_back();
            return p;
        }
        void* p = nullptr;
        cuda(cudaMalloc(&p, std::size_t(1) << cls), "cudaMalloc");
        return p;
    }
    void give(void* p, std::size_t bytes) { free_[size_class(bytes)].push_back(p); }
    ~BlockPool() {
        for (auto& fl : free_)
            for (void* p : fl) cudaFree(p);
    }

private:
    static int size_class(std::size_t bytes) {
        int c = 8;
        while ((std::size_t(1) << c) < bytes) ++c;
        return c;
    }
    std::vector<void*> free_[64];
};

BlockPool& pool() {
    thread_local BlockPool p;
    return p;
}

// Device buffer (RAII, pooled).
template <typename T>
class DBuf {
public:
    explicit DBuf(std::size_t n) : n_(n) {
        if (n_) p_ = static_cast<T*>(pool().take(n_ * sizeof(T)));
    }
    DBuf(const T* host, std::size_t n) : DBuf(n) { upload(host); }
    ~DBuf() {
        if (p_) pool().give(p_, n_ * sizeof(T));
    }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    T* get() const { return p_; }
    void upload(const T* host) {
        if (n_) cuda(cudaMemcpy(p_, host, n_ * sizeof(T), cudaMemcpyHostToDevice), "upload");
    }
    std::vector<T> download(std::size_t n) const {
        std::vector<T> v(n);
        if (n) cuda(cudaMemcpy(v.data(), p_, n * sizeof(T), cudaMemcpyDeviceToHost), "download");
        return v;
    }

private:
    T* p_ = nullptr;
    std::size_t n_;
};

inline void sync() { cuda(cudaStreamSynchronize(nullptr), "sync"); }

kivi_axis axis_of(Axis a) { return a == Axis::per_channel ? KIVI_PER_CHANNEL : KIVI_PER_TOKEN; }

std::size_t packed_size(std::uint64_t codes, int bits) { return (codes * bits + 7) / 8; }

// ---- per-thread device cache pool (one single-unit kivi_cache per config) --
struct CacheDeleter {
    void operator()(kivi_cache* c) const { kivi_cache_destroy(c); }
};
using CacheKey = std::tuple<int, Index, Index, Index>;

kivi_cache* pooled_cache(const CacheConfig& cfg) {
    thread_local std::map<CacheKey, std::unique_ptr<kivi_cache, CacheDeleter>> pool;
    const CacheKey key{cfg.bits, cfg.group_size, cfg.residual_length, cfg.head_dim};
    auto it = pool.find(key);
    if (it != pool.end()) return it->second.get();
    kivi_config c{cfg.bits, cfg.group_size, cfg.residual_length, cfg.head_dim};
    kivi_cache* h = nullptr;
    int dev = 0;
    cudaGetDevice(&dev);
    check(kivi_cache_create(&c, dev, 1, 0, &h));
    check(kivi_set_attend_path(h, 1));  // reference arithmetic order (generic kernel)
    pool.emplace(key, std::unique_ptr<kivi_cache, CacheDeleter>(h));
    return h;
}

// Loads a caller-owned state pair into the device cache.
void load_state(kivi_cache* h, const KeyCacheState& ks, const ValueCacheState& vs,
                const CacheConfig& cfg) {
    const Index l = ks.total_tokens;
    const Index R = cfg.residual_length;
    if (vs.total_tokens != l)
        throw UsageError("kivi facade: key and value states hold different token counts");
    const Index kr = l % R, vr = std::min(l, R);
    if (ks.grouped.rows() != l - kr || ks.residual.rows() != kr || vs.grouped.rows() != l - vr ||
        vs.residual.rows() != vr)
        throw UsageError("kivi facade: state is not a prefill/append_token state");
    kivi_unit_state st{};
    auto& kq = const_cast<QuantizedTensor&>(ks.grouped);
    auto& vq = const_cast<QuantizedTensor&>(vs.grouped);
    st.key_packed = TensorAccess::packed(kq).data();
    st.key_zero = TensorAccess::zeros(kq).data();
    st.key_scale = TensorAccess::scales(kq).data();
    st.key_residual = const_cast<float*>(ks.residual.data());
    st.value_packed = TensorAccess::packed(vq).data();
    st.value_zero = TensorAccess::zeros(vq).data();
    st.value_scale = TensorAccess::scales(vq).data();
    st.value_residual = const_cast<float*>(vs.residual.data());
    check(kivi_import_unit(h, 0, l, ks.residual_capacity, vs.residual_capacity, &st, nullptr));
}

// Writes the device cache's unit back into the caller-owned states.
void store_state(kivi_cache* h, KeyCacheState& ks, ValueCacheState& vs, const CacheConfig& cfg) {
    kivi_cache_info info{};
    check(kivi_cache_get_info(h, &info));
    const Index d = cfg.head_dim, G = cfg.group_size;
    const int B = cfg.bits;
    const Index kg = info.key_grouped_tokens, vg = info.value_grouped_tokens;
    std::vector<std::uint8_t> kp(packed_size((std::uint64_t)kg * d, B)),
        vp(packed_size((std::uint64_t)vg * d, B));
    std::vector<double> kz(kg * d / G), ksc(kg * d / G), vz(vg * d / G), vsc(vg * d / G);
    Matrix kres(info.key_residual_rows, d), vres(info.value_residual_rows, d);
    kivi_unit_state st{kp.data(), kz.data(), ksc.data(), kres.data(),
                       vp.data(), vz.data(), vsc.data(), vres.data()};
    check(kivi_export_unit(h, 0, &st, nullptr));
    ks.grouped = TensorAccess::make(std::move(kp), std::move(kz), std::move(ksc), kg, d,
                                    cfg.key_params());
    vs.grouped = TensorAccess::make(std::move(vp), std::move(vz), std::move(vsc), vg, d,
                                    cfg.value_params());
    ks.residual = std::move(kres);
    vs.residual = std::move(vres);
    ks.total_tokens = vs.total_tokens = info.total_tokens;
    ks.residual_capacity = info.key_residual_capacity;
    vs.residual_capacity = info.value_residual_capacity;
}

void check_rows(const Matrix& t_K, const Matrix& t_V, const CacheConfig& cfg) {
    // reference append_token shape check (kv_cache.cpp:68-72)
    if (t_K.rows() != 1 || t_V.rows() != 1 || t_K.cols() != cfg.head_dim ||
        t_V.cols() != cfg.head_dim)
        throw ShapeError("append_token: expected 1x" + std::to_string(cfg.head_dim) +
                         " key/value rows");
}

}  // namespace

// ============================ quantizer ======================================

const char* axis_name(Axis axis) { return axis == Axis::per_token ? "per_token" : "per_channel"; }

void QuantParams::validate() const {
    if (bits < 1 || bits > 8) throw ConfigError("bits must be in [1, 8], got " + std::to_string(bits));
    if (group_size < 1)
        throw ConfigError("group_size must be >= 1, got " + std::to_string(group_size));
}

GroupQuant quantize_group(std::span<const float> values, int bits) {
    if (values.empty()) throw UsageError("quantize_group: empty group");
    if (bits < 1 || bits > 8) throw UsageError("quantize_group: bits out of range");
    const std::size_t n = values.size();
    DBuf<float> m(values.data(), n);
    DBuf<std::uint8_t> codes(n);
    DBuf<double> z(1), s(1);
    check(kivi_quantize_codes(m.get(), 1, (int64_t)n, bits, (int64_t)n, KIVI_PER_TOKEN,
                              codes.get(), z.get(), s.get(), nullptr));
    sync();
    GroupQuant g;
    g.codes = codes.download(n);
    g.zero_point = z.download(1)[0];
    g.scale = s.download(1)[0];
    return g;
}

std::vector<float> dequantize_group(std::span<const std::uint8_t> codes, double zero_point,
                                    double scale) {
    const std::size_t n = codes.size();
    if (n == 0) return {};
    DBuf<std::uint8_t> c(codes.data(), n);
    DBuf<double> z(&zero_point, 1), s(&scale, 1);
    DBuf<float> out(n);
    check(kivi_dequantize_codes(c.get(), z.get(), s.get(), 1, (int64_t)n, (int64_t)n,
                                KIVI_PER_TOKEN, out.get(), nullptr));
    sync();
    return out.download(n);
}

std::vector<std::uint8_t> pack_codes(std::span<const std::uint8_t> codes, int bits) {
    if (bits != 1 && bits != 2 && bits != 4 && bits != 8)
        throw UsageError("pack_codes: bits must be one of {1,2,4,8}, got " + std::to_string(bits));
    const std::size_t n = codes.size();
    if (n == 0) return {};
    for (std::uint8_t c : codes)  // message parity with the reference (quantize.cpp:66-70)
        if (c > (1 << bits) - 1)
            throw UsageError("pack_codes: code " + std::to_string(c) + " exceeds 2^" +
                             std::to_string(bits) + "-1");
    DBuf<std::uint8_t> c(codes.data(), n);
    DBuf<std::uint8_t> out(packed_size(n, bits));
    check(kivi_pack_codes(c.get(), (int64_t)n, bits, out.get(), nullptr));
    return out.download(packed_size(n, bits));
}

std::vector<std::uint8_t> unpack_codes(std::span<const std::uint8_t> bytes, std::size_t count,
                                       int bits) {
    if (bits != 1 && bits != 2 && bits != 4 && bits != 8)
        throw UsageError("unpack_codes: bits must be one of {1,2,4,8}");
    if (packed_size(count, bits) > bytes.size())
        throw UsageError("unpack_codes: byte buffer too short for " + std::to_string(count) +
                         " codes");
    if (count == 0) return {};
    DBuf<std::uint8_t> b(bytes.data(), bytes.size());
    DBuf<std::uint8_t> out(count);
    check(kivi_unpack_codes(b.get(), (int64_t)count, bits, out.get(), nullptr));
    sync();
    return out.download(count);
}

QuantizedTensor QuantizedTensor::quantize(const Matrix& m, const QuantParams& params) {
    params.validate();
    if (!params.packable())
        throw ConfigError("packed storage requires bits in {1,2,4,8}; B=" +
                          std::to_string(params.bits) + " is fake-quant only");
    const Index extent = params.axis == Axis::per_channel ? m.rows() : m.cols();
    if (extent % params.group_size != 0)
        throw ShapeError(std::string("quantize: ") + axis_name(params.axis) +
                         " grouped axis extent " + std::to_string(extent) +
                         " not divisible by group size " + std::to_string(params.group_size) +
                         " (matrix " + shape_str(m) + ")");
    const std::uint64_t n = (std::uint64_t)m.size();
    const std::size_t ng = n / params.group_size;
    std::vector<std::uint8_t> packed(packed_size(n, params.bits));
    std::vector<double> z(ng), s(ng);
    if (n) {
        DBuf<float> dm(m.data(), n);
        DBuf<double> dz(ng), ds(ng);
        check(kivi_quantize_matrix(dm.get(), m.rows(), m.cols(), params.bits, params.group_size,
                                   axis_of(params.axis), packed.data(), dz.get(), ds.get(),
                                   nullptr));
        z = dz.download(ng);
        s = ds.download(ng);
    }
    return TensorAccess::make(std::move(packed), std::move(z), std::move(s), m.rows(), m.cols(),
                              params);
}

Matrix QuantizedTensor::dequantize() const {
    if (rows_ == 0) return Matrix(0, cols_);
    const std::size_t n = (std::size_t)code_count(), ng = scales_.size();
    DBuf<std::uint8_t> p(packed_.data(), packed_.size());
    DBuf<double> z(zero_points_.data(), ng), s(scales_.data(), ng);
    DBuf<float> out(n);
    check(kivi_dequantize_matrix(p.get(), z.get(), s.get(), rows_, cols_, params_.bits,
                                 params_.group_size, axis_of(params_.axis), out.get(), nullptr));
    Matrix m(rows_, cols_);
    cuda(cudaMemcpy(m.data(), out.get(), n * sizeof(float), cudaMemcpyDeviceToHost), "download");
    return m;
}

void QuantizedTensor::concat_tokens(const QuantizedTensor& other) {
    if (other.rows_ == 0) return;
    if (rows_ == 0) {
        *this = other;
        return;
    }
    if (cols_ != other.cols_)
        throw ShapeError("concat_tokens: column counts differ (" + std::to_string(cols_) + " vs " +
                         std::to_string(other.cols_) + ")");
    if (params_.bits != other.params_.bits || params_.group_size != other.params_.group_size ||
        params_.axis != other.params_.axis)
        throw ConfigError("concat_tokens: quantization parameters differ");
    // Device unpack of both streams + one repack (the reference's algorithm,
    // quantize.cpp:206-213).
    const std::size_t na = (std::size_t)code_count(), nb = (std::size_t)other.code_count();
    DBuf<std::uint8_t> a(packed_.data(), packed_.size()), b(other.packed_.data(), other.packed_.size());
    DBuf<std::uint8_t> codes(na + nb);
    check(kivi_unpack_codes(a.get(), (int64_t)na, params_.bits, codes.get(), nullptr));
    check(kivi_unpack_codes(b.get(), (int64_t)nb, params_.bits, codes.get() + na, nullptr));
    DBuf<std::uint8_t> out(packed_size(na + nb, params_.bits));
    check(kivi_pack_codes(codes.get(), (int64_t)(na + nb), params_.bits, out.get(), nullptr));
    packed_ = out.download(packed_size(na + nb, params_.bits));
    zero_points_.insert(zero_points_.end(), other.zero_points_.begin(), other.zero_points_.end());
    scales_.insert(scales_.end(), other.scales_.begin(), other.scales_.end());
    rows_ += other.rows_;
}

Matrix fake_quantize(const Matrix& m, const QuantParams& params) {
    params.validate();
    if (m.size() == 0) return m;
    const Index G = params.group_size;
    const bool pc = params.axis == Axis::per_channel;
    const Index extent = pc ? m.rows() : m.cols();
    const Index padded = (extent + G - 1) / G * G;
    Matrix p = pc ? Matrix::Zero(padded, m.cols()) : Matrix::Zero(m.rows(), padded);
    p.block(0, 0, m.rows(), m.cols()) = m;
    const std::size_t n = (std::size_t)p.size(), ng = n / G;
    DBuf<float> dm(p.data(), n);
    DBuf<std::uint8_t> codes(n);
    DBuf<double> z(ng), s(ng);
    DBuf<float> out(n);
    check(kivi_quantize_codes(dm.get(), p.rows(), p.cols(), params.bits, G, axis_of(params.axis),
                              codes.get(), z.get(), s.get(), nullptr));
    check(kivi_dequantize_codes(codes.get(), z.get(), s.get(), p.rows(), p.cols(), G,
                                axis_of(params.axis), out.get(), nullptr));
    Matrix deq(p.rows(), p.cols());
    cuda(cudaMemcpy(deq.data(), out.get(), n * sizeof(float), cudaMemcpyDeviceToHost), "download");
    return deq.block(0, 0, m.rows(), m.cols());
}

// ============================ streaming cache ================================

void CacheConfig::validate() const {
    key_params().validate();
    if (residual_length < 1) throw ConfigError("residual_length must be >= 1");
    if (residual_length % group_size != 0)
        throw ConfigError("residual_length " + std::to_string(residual_length) +
                          " must be divisible by group_size " + std::to_string(group_size));
    if (head_dim < 1 || head_dim % group_size != 0)
        throw ConfigError("head_dim " + std::to_string(head_dim) +
                          " must be a positive multiple of group_size " + std::to_string(group_size));
}

PrefillResult prefill(const Matrix& keys, const Matrix& values, const CacheConfig& cfg) {
    cfg.validate();
    if (keys.rows() == 0) throw UsageError("prefill: empty prompt");
    if (keys.rows() != values.rows()) throw ShapeError("prefill: key/value token counts differ");
    if (keys.cols() != cfg.head_dim || values.cols() != cfg.head_dim)
        throw ShapeError("prefill: head_dim mismatch");
    kivi_cache* h = pooled_cache(cfg);
    check(kivi_prefill_host(h, keys.data(), values.data(), keys.rows(), nullptr));
    PrefillResult out;
    store_state(h, out.key, out.value, cfg);
    out.passthrough_keys = keys;
    out.passthrough_values = values;
    return out;
}

void append_token(KeyCacheState& key_state, ValueCacheState& value_state, const Matrix& t_K,
                  const Matrix& t_V, const CacheConfig& cfg) {
    check_rows(t_K, t_V, cfg);
    kivi_cache* h = pooled_cache(cfg);
    load_state(h, key_state, value_state, cfg);
    check(kivi_append_host(h, t_K.data(), t_V.data(), nullptr));
    sync();
    store_state(h, key_state, value_state, cfg);
}

Matrix materialize_keys(const KeyCacheState& state) {
    return concat_rows(state.grouped.dequantize(), state.residual);
}

Matrix materialize_values(const ValueCacheState& state) {
    return concat_rows(state.grouped.dequantize(), state.residual);
}

namespace {
std::uint64_t grouped_bytes(const QuantizedTensor& t) {
    return (std::uint64_t)t.packed().size() + 4u * (std::uint64_t)t.group_count();
}
}  // namespace

// Byte accounting of the reference (kv_cache.cpp:110-127): 2 bytes per
// zero-point and scale, 2 bytes per residual element at the high-water mark.
std::uint64_t memory_bytes(const KeyCacheState& state) {
    return grouped_bytes(state.grouped) +
           2u * (std::uint64_t)state.residual_capacity * (std::uint64_t)state.residual.cols();
}

std::uint64_t memory_bytes(const ValueCacheState& state) {
    return grouped_bytes(state.grouped) +
           2u * (std::uint64_t)state.residual_capacity * (std::uint64_t)state.residual.cols();
}

// ============================ attention ======================================

Matrix reference_attention(const Matrix& t_Q, const Matrix& K, const Matrix& V,
                           const AttentionOptions& opts) {
    if (K.rows() != V.rows()) throw ShapeError("reference_attention: K/V token counts differ");
    if (t_Q.cols() != K.cols())
        throw ShapeError("matmul: inner dimensions differ (" + std::to_string(t_Q.cols()) + " vs " +
                         std::to_string(K.cols()) + ")");
    if (V.cols() != K.cols())
        throw ShapeError("reference_attention: value width must equal key width on the GPU path");
    if (K.rows() == 0) throw ShapeError("reference_attention: no keys");
    const Index nq = t_Q.rows(), d = t_Q.cols(), l = K.rows();
    DBuf<float> q(t_Q.data(), nq * d), k(K.data(), l * d), v(V.data(), l * d), out(nq * d);
    check(kivi_reference_attention(q.get(), nq, k.get(), v.get(), l, d, opts.scale_logits ? 1 : 0,
                                   out.get(), nullptr));
    Matrix o(nq, d);
    cuda(cudaMemcpy(o.data(), out.get(), sizeof(float) * nq * d, cudaMemcpyDeviceToHost),
         "download");
    return o;
}

DecodeOutput decode_attention(const Matrix& t_Q, const Matrix& t_K, const Matrix& t_V,
                              KeyCacheState& key_state, ValueCacheState& value_state,
                              const CacheConfig& cfg, const AttentionOptions& opts) {
    if (t_Q.rows() != 1 || t_Q.cols() != cfg.head_dim)
        throw ShapeError("decode_attention: query must be 1x" + std::to_string(cfg.head_dim));
    check_rows(t_K, t_V, cfg);
    kivi_cache* h = pooled_cache(cfg);
    load_state(h, key_state, value_state, cfg);
    const Index l = key_state.total_tokens + 1;
    DecodeOutput out;
    out.output = Matrix(1, cfg.head_dim);
    out.weights = Matrix(1, l);
    check(kivi_decode_host(h, t_Q.data(), t_K.data(), t_V.data(), 1, out.output.data(),
                           out.weights.data(), opts.scale_logits ? 1 : 0, nullptr));
    check(kivi_host_join(h, nullptr));
    sync();
    store_state(h, key_state, value_state, cfg);
    return out;
}

}  // namespace kivi
