/*
 * kivi_b200.h — C ABI of the B200-native KIVI KV-cache hot path.
 *
 * One `kivi_cache` holds n_units independent streaming caches (one per
 * (batch element, kv-head) of a layer — a "unit" is the reference's
 * KeyCacheState + ValueCacheState pair, reference
 * proj/include/kivi/kv_cache.hpp:22-35).  All units of a cache advance in
 * lockstep: every append adds exactly one token to every unit, which is how a
 * decode step drives them (reference proj/src/workload.cpp:224-242).
 *
 * Conventions
 *   - Plain C types only; no torch, no C++ in the signatures.
 *   - Every data pointer of a non-`_host` entry point is a DEVICE pointer
 *     (cudaMalloc'd, or any memory the GPU can dereference); work is enqueued
 *     on `stream` (a cudaStream_t passed as void*; NULL = legacy default
 *     stream) and the call returns without synchronising.
 *   - `_host` entry points take HOST pointers and enqueue the host<->device
 *     copies on `stream` together with the kernels (cudaMemcpyAsync
 *     semantics: use pinned buffers for asynchrony and synchronise `stream`
 *     before reading outputs or reusing inputs).  kivi_prefill_host
 *     synchronises before returning.
 *   - Errors mirror the reference's exception types (reference
 *     proj/include/kivi/errors.hpp:10-22): a failing call returns a status
 *     and leaves the cache unchanged; kivi_last_error() returns a
 *     thread-local message.
 *   - Numerics: packed codes and per-group zero-points/maxima are bit-exact
 *     with the reference quantizer (reference proj/src/quantize.cpp:22-48);
 *     attention outputs are fp32 and within the tolerances stated in
 *     DESIGN.md.
 */
#ifndef KIVI_B200_H
#define KIVI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KIVI_B200_ABI_VERSION 1

typedef enum kivi_status {
    KIVI_OK = 0,
    KIVI_ERR_SHAPE = 1,    /* reference ShapeError  (errors.hpp:10)  */
    KIVI_ERR_USAGE = 2,    /* reference UsageError  (errors.hpp:15)  */
    KIVI_ERR_CONFIG = 3,   /* reference ConfigError (errors.hpp:20)  */
    KIVI_ERR_CUDA = 4,     /* CUDA runtime / launch failure          */
    KIVI_ERR_OOM = 5,      /* device or pinned allocation failed     */
    KIVI_ERR_CAPACITY = 6  /* append past a cache's fixed capacity   */
} kivi_status;

/* Mirrors reference CacheConfig (kv_cache.hpp:9-18): B, G, R, d.
 * validate(): 1 <= bits <= 8 and packable (bits in {1,2,4,8}),
 * group_size >= 1, residual_length >= 1, residual_length % group_size == 0,
 * head_dim >= 1, head_dim % group_size == 0 (kv_cache.cpp:7-21,
 * quantize.cpp:13-20, 173-176). */
typedef struct kivi_config {
    int32_t bits;
    int64_t group_size;
    int64_t residual_length;
    int64_t head_dim;
} kivi_config;

/* Quantization axis, reference Axis (quantize.hpp:14). */
typedef enum kivi_axis { KIVI_PER_TOKEN = 0, KIVI_PER_CHANNEL = 1 } kivi_axis;

typedef struct kivi_cache kivi_cache;

/* Counters of one cache (identical for every unit). */
typedef struct kivi_cache_info {
    int64_t n_units;
    int64_t capacity_tokens;
    int64_t total_tokens;             /* l                                    */
    int64_t key_grouped_tokens;       /* l - l % R                            */
    int64_t key_residual_rows;        /* l % R                                */
    int64_t key_residual_capacity;    /* reference KeyCacheState::residual_capacity */
    int64_t value_grouped_tokens;     /* l - min(l, R)                        */
    int64_t value_residual_rows;      /* min(l, R)                            */
    int64_t value_residual_capacity;
    uint64_t key_memory_bytes;        /* reference memory_bytes(KeyCacheState), per unit */
    uint64_t value_memory_bytes;      /* reference memory_bytes(ValueCacheState), per unit */
    uint64_t device_bytes;            /* bytes this cache holds in HBM        */
} kivi_cache_info;

/* Host-side view of one unit's state in the REFERENCE's layout
 * (QuantizedTensor::packed()/zero_points()/scales(), residual rows in token
 * order).  Buffers are caller-owned; sizes follow kivi_cache_info:
 *   key_packed   ceil(key_grouped_tokens*d*B/8) bytes
 *   key_zero/key_scale   key_grouped_tokens*d/G doubles
 *   key_residual key_residual_rows*d floats
 *   value_packed ceil(value_grouped_tokens*d*B/8) bytes
 *   value_zero/value_scale value_grouped_tokens*d/G doubles
 *   value_residual value_residual_rows*d floats
 * Any pointer may be NULL to skip that field (export only). */
typedef struct kivi_unit_state {
    uint8_t* key_packed;
    double* key_zero;
    double* key_scale;
    float* key_residual;
    uint8_t* value_packed;
    double* value_zero;
    double* value_scale;
    float* value_residual;
} kivi_unit_state;

/* Last error message of the calling thread ("" if none). */
const char* kivi_last_error(void);
int kivi_abi_version(void);

/* Validates like CacheConfig::validate (kv_cache.cpp:7-21) + packable. */
kivi_status kivi_config_validate(const kivi_config* cfg);

/* ---- cache lifetime (replaces constructing KeyCacheState/ValueCacheState) */
kivi_status kivi_cache_create(const kivi_config* cfg, int device, int64_t n_units,
                              int64_t capacity_tokens, kivi_cache** out);
kivi_status kivi_cache_destroy(kivi_cache* cache);
/* Grows every unit's capacity (device reallocation + copy); stream-ordered. */
kivi_status kivi_cache_reserve(kivi_cache* cache, int64_t capacity_tokens, void* stream);
/* Deep copy (reference states are copyable, workload.cpp:166-167). */
kivi_status kivi_cache_clone(const kivi_cache* src, void* stream, kivi_cache** out);
kivi_status kivi_cache_get_info(const kivi_cache* cache, kivi_cache_info* info);

/* ---- hot path ------------------------------------------------------------ */

/* Reference prefill (kv_cache.cpp:23-55): resets every unit to the prompt.
 * keys/values: [n_units][l][d] fp32.  l >= 1 else KIVI_ERR_USAGE. */
kivi_status kivi_prefill(kivi_cache* cache, const float* keys, const float* values, int64_t l,
                         void* stream);

/* Reference append_token (kv_cache.cpp:66-98) for every unit.
 * t_k, t_v: [n_units][d] fp32. */
kivi_status kivi_append(kivi_cache* cache, const float* t_k, const float* t_v, void* stream);

/* Attention of the current state (no append) — the second half of the
 * reference decode_attention (attention.cpp:36-99), for q_per_kv query heads
 * per unit (q_per_kv == 1 is the reference's MHA; >1 is GQA, which the
 * reference emulates with one state copy per query head).
 *   t_q:     [n_units][q_per_kv][d] fp32
 *   out:     [n_units][q_per_kv][d] fp32
 *   weights: NULL, or [n_units][q_per_kv][l] fp32 normalised softmax weights
 *            (reference DecodeOutput::weights, attention.hpp:14)
 *   scale_logits: reference AttentionOptions::scale_logits (attention.hpp:7-10) */
kivi_status kivi_attend(kivi_cache* cache, const float* t_q, int32_t q_per_kv, float* out,
                        float* weights, int32_t scale_logits, void* stream);

/* Reference decode_attention (attention.cpp:26-100): append, then attend. */
kivi_status kivi_decode(kivi_cache* cache, const float* t_q, const float* t_k, const float* t_v,
                        int32_t q_per_kv, float* out, float* weights, int32_t scale_logits,
                        void* stream);

/* Host-buffer variants: the copies in and out are enqueued with the work.
 * kivi_decode_host copies its result on the cache's own copy stream (so the
 * next layer's kernels on `stream` do not queue behind it): before reading
 * `out`/`weights`, call kivi_host_join(cache, stream) and synchronise
 * `stream` (or synchronise the device). */
kivi_status kivi_prefill_host(kivi_cache* cache, const float* keys, const float* values,
                              int64_t l, void* stream);
kivi_status kivi_append_host(kivi_cache* cache, const float* t_k, const float* t_v,
                             void* stream);
kivi_status kivi_decode_host(kivi_cache* cache, const float* t_q, const float* t_k,
                             const float* t_v, int32_t q_per_kv, float* out, float* weights,
                             int32_t scale_logits, void* stream);
/* Orders `stream` after every result copy kivi_decode_host has enqueued. */
kivi_status kivi_host_join(kivi_cache* cache, void* stream);

/* ---- one decode step of a whole model ------------------------------------
 * caches[i] holds layer i (all with the same n_units, head_dim and device);
 * the reference's decode loop runs the layers of a step in order
 * (workload.cpp:224-242).  Row layouts, layer-major:
 *   t_q, out: [n_layers][n_units][q_per_kv][d];  t_k, t_v: [n_layers][n_units][d].
 * kivi_decode_layers: device pointers, enqueued on `stream`, no sync.
 * kivi_decode_layers_host: host pointers (pinned for speed); uploads every
 * layer's rows, decodes every layer and copies the outputs back, then
 * synchronises `stream`: the outputs are on the host when it returns.  With
 * KIVI_STEP_GRAPH=1 (and a non-NULL stream) the step is captured as a CUDA
 * graph and replayed (cudaGraphExecUpdate between steps). */
kivi_status kivi_decode_layers(kivi_cache* const* caches, int32_t n_layers, const float* t_q,
                               const float* t_k, const float* t_v, int32_t q_per_kv, float* out,
                               int32_t scale_logits, void* stream);
kivi_status kivi_decode_layers_host(kivi_cache* const* caches, int32_t n_layers, const float* t_q,
                                    const float* t_k, const float* t_v, int32_t q_per_kv,
                                    float* out, int32_t scale_logits, void* stream);

/* ---- q/k/v projection fused with the append ------------
 * The reference projects each decode token per layer, q = t W_q, k = t W_k,
 * v = t W_v in fp32 (workload.cpp:230-232).  kivi_proj holds one layer's
 * three [hidden_in][hidden_out] weight matrices (x @ W convention, device
 * pointers, copied and transposed once); the GEMM runs on the tcgen05 tensor
 * cores in 3xTF32 (fp32-class accuracy).
 * kivi_proj_gemm: x [n][hidden_in] -> out_q/k/v; seq == 0: [n][hidden_out];
 *   seq > 0: rows are (sequence, token) = (r / seq, r % seq) and the outputs
 *   are written per unit, [n / seq * heads][seq][128] (kivi_prefill's layout).
 * kivi_proj_append: the decode step's projection + append in one launch:
 *   q -> q_out [n * heads][128]; k and v are appended to `cache` (n_units =
 *   n * heads, head_dim 128, group 32, 2 or 4 bits) as kivi_append would,
 *   with the value FIFO pop quantized in the GEMM epilogue.  Follow with
 *   kivi_attend (together: the reference decode_attention). */
typedef struct kivi_proj kivi_proj;
kivi_status kivi_proj_create(int device, int64_t hidden_in, int64_t hidden_out, const float* w_q,
                             const float* w_k, const float* w_v, void* stream, kivi_proj** out);
kivi_status kivi_proj_destroy(kivi_proj* proj);
kivi_status kivi_proj_gemm(kivi_proj* proj, const float* x, int64_t n, float* out_q, float* out_k,
                           float* out_v, int64_t seq, void* stream);
kivi_status kivi_proj_append(kivi_proj* proj, kivi_cache* cache, const float* x, int64_t n,
                             float* q_out, void* stream);

/* Step-graph counters of the calling thread on the current device: steps
 * replayed as a graph, graph re-instantiations (topology changed), captures
 * that failed (run directly instead). */
kivi_status kivi_step_graph_stats(int64_t* replayed, int64_t* reinstantiated,
                                  int64_t* capture_failed);

/* ---- state exchange in the reference layout (parity / drop-in facade) ---- */

/* Copies unit `unit` to host buffers; synchronises `stream`. */
kivi_status kivi_export_unit(const kivi_cache* cache, int64_t unit, kivi_unit_state* dst,
                             void* stream);
/* Sets every unit's token count to `total_tokens` and loads unit `unit` from
 * host buffers in the reference layout (all units of the cache must later be
 * loaded, or they hold zeros).  Synchronises `stream`. */
kivi_status kivi_import_unit(kivi_cache* cache, int64_t unit, int64_t total_tokens,
                             int64_t key_residual_capacity, int64_t value_residual_capacity,
                             const kivi_unit_state* src, void* stream);
/* Reference materialize_keys / materialize_values (kv_cache.cpp:100-106):
 * [n_units][l][d] fp32, bit-exact dequantisation (double, quantize.cpp:142-167). */
kivi_status kivi_materialize(const kivi_cache* cache, float* keys_out, float* values_out,
                             void* stream);

/* ---- standalone quantizer (reference quantize.hpp:35-96) ----------------- */

/* QuantizedTensor::quantize (quantize.cpp:171-185) of a rows x cols fp32
 * matrix: packed bytes (ceil(rows*cols*B/8)), per-group zero-points and
 * scales as double (group order quantize.cpp:105-140).  Device pointers. */
kivi_status kivi_quantize_matrix(const float* m, int64_t rows, int64_t cols, int32_t bits,
                                 int64_t group_size, kivi_axis axis, uint8_t* packed,
                                 double* zero_points, double* scales, void* stream);
/* QuantizedTensor::dequantize (quantize.cpp:187-192 -> 142-167). */
kivi_status kivi_dequantize_matrix(const uint8_t* packed, const double* zero_points,
                                   const double* scales, int64_t rows, int64_t cols,
                                   int32_t bits, int64_t group_size, kivi_axis axis, float* out,
                                   void* stream);
/* Reference quantize_group (quantize.cpp:22-48) of one group of n values (any
 * n >= 1, B in [1, 8]): codes[n] (uint8), *zero_point, *scale as the
 * reference's doubles; dequantized (NULL or [n] fp32) receives
 * dequantize_group (quantize.cpp:50-57) of the result.  One launch, all
 * pointers device-accessible (device or mapped host memory).  Empty group or
 * B out of range: KIVI_ERR_USAGE (the reference's UsageError). */
kivi_status kivi_quantize_group(const float* values, int64_t n, int32_t bits, uint8_t* codes,
                                double* zero_point, double* scale, float* dequantized,
                                void* stream);
/* Unpacked-code variants for ANY B in [1, 8] (reference quantize_grouped /
 * dequantize_grouped, quantize.cpp:105-167, used by quantize_group and
 * fake_quantize which accept non-packable B): one uint8 code per element, in
 * group order.  Device pointers. */
kivi_status kivi_quantize_codes(const float* m, int64_t rows, int64_t cols, int32_t bits,
                                int64_t group_size, kivi_axis axis, uint8_t* codes,
                                double* zero_points, double* scales, void* stream);
kivi_status kivi_dequantize_codes(const uint8_t* codes, const double* zero_points,
                                  const double* scales, int64_t rows, int64_t cols,
                                  int64_t group_size, kivi_axis axis, float* out, void* stream);
/* pack_codes / unpack_codes (quantize.cpp:59-93).  pack returns
 * KIVI_ERR_USAGE for bits not in {1,2,4,8} or a code > 2^B-1 (after
 * synchronising `stream` to inspect the device-side range check). */
kivi_status kivi_pack_codes(const uint8_t* codes, int64_t n, int32_t bits, uint8_t* bytes,
                            void* stream);
kivi_status kivi_unpack_codes(const uint8_t* bytes, int64_t n, int32_t bits, uint8_t* codes,
                              void* stream);
/* Reference reference_attention (attention.cpp:16-24): full-precision
 * softmax(scale * q K^T) V for q: [n_q][d], K,V: [l][d] -> out [n_q][d]. */
kivi_status kivi_reference_attention(const float* q, int64_t n_q, const float* keys,
                                     const float* values, int64_t l, int64_t d,
                                     int32_t scale_logits, float* out, void* stream);

/* ---- measurement hooks (bench.py) --------------------------------------- */

/* Re-reads the KIVI_* routing / tuning environment variables (read once per
 * process otherwise; DESIGN.md §4 lists them).  Affects later calls only. */
kivi_status kivi_reload_tuning(void);

/* Selects the attend kernel: 0 = auto (fast sm_100a kernel when the shape is
 * supported, else generic), 1 = force generic, 2 = force fast (error if the
 * shape is unsupported). */
kivi_status kivi_set_attend_path(kivi_cache* cache, int32_t path);
/* enable = 0: off.  enable = k >= 1: kivi_attend / kivi_decode record CUDA
 * events around the main attend kernel of every k-th call (k > 1 keeps the
 * host cost of the events off latency-bound steps). */
kivi_status kivi_profile_enable(kivi_cache* cache, int32_t enable);
/* Synchronises the recorded events and returns the summed main-kernel time,
 * the number of main-kernel launches timed (summed into main_kernel_ms) and
 * the total number of kernels this library launched for the cache since the
 * last reset; then resets. */
kivi_status kivi_profile_read(kivi_cache* cache, double* main_kernel_ms, int64_t* main_launches,
                              int64_t* total_launches);
/* Algorithmic HBM bytes the attend kernel must read + write per unit for the
 * cache's current state and q_per_kv (SURVEY §8d formula). */
kivi_status kivi_attend_bytes(const kivi_cache* cache, int32_t q_per_kv, uint64_t* bytes_per_unit);

#ifdef __cplusplus
}
#endif

#endif /* KIVI_B200_H */
