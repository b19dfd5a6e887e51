/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement ("port") of the reference's
 * KIVI hot path, used as a parity checker by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg.  It is pinned against the reference itself
 * (oracle/_ref, compiled from /root/reference) and against the golden vectors
 * in tests/golden/ (see tests/test_oracle.py).  Never linked by the product.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference/proj).
 */
#ifndef KIVI_ORACLE_H
#define KIVI_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* quantize_group (src/quantize.cpp:22-48).  Returns 0, or 2 (UsageError) for
 * an empty group / bits outside [1,8]. */
int oracle_quantize_group(const float* v, int64_t n, int bits, uint8_t* codes, double* zero,
                          double* scale);
/* dequantize_group (src/quantize.cpp:50-57). */
void oracle_dequantize_group(const uint8_t* codes, int64_t n, double zero, double scale,
                             float* out);
/* pack_codes / unpack_codes (src/quantize.cpp:59-93).  Return 2 on UsageError. */
int oracle_pack_codes(const uint8_t* codes, int64_t n, int bits, uint8_t* bytes);
int oracle_unpack_codes(const uint8_t* bytes, int64_t nbytes, int64_t n, int bits, uint8_t* codes);
/* QuantizedTensor::quantize (src/quantize.cpp:171-185 -> 105-140) of a
 * row-major rows x cols matrix; returns 0, 1 (ShapeError) or 3 (ConfigError). */
int oracle_quantize_matrix(const float* m, int64_t rows, int64_t cols, int bits, int64_t G,
                           int per_channel, uint8_t* packed, double* zero, double* scale);
/* QuantizedTensor::dequantize (src/quantize.cpp:142-167, 187-192). */
void oracle_dequantize_matrix(const uint8_t* packed, const double* zero, const double* scale,
                              int64_t rows, int64_t cols, int bits, int64_t G, int per_channel,
                              float* out);

/* One (KeyCacheState, ValueCacheState) pair (include/kivi/kv_cache.hpp:22-35). */
typedef struct oracle_unit oracle_unit;
oracle_unit* oracle_unit_new(int bits, int64_t G, int64_t R, int64_t d);
void oracle_unit_free(oracle_unit* u);
/* prefill (src/kv_cache.cpp:23-55); 0 or 2 (empty prompt). */
int oracle_prefill(oracle_unit* u, const float* keys, const float* values, int64_t l);
/* append_token (src/kv_cache.cpp:66-98). */
void oracle_append(oracle_unit* u, const float* tk, const float* tv);
/* decode_attention (src/attention.cpp:26-100): append, then attend.
 * out: d floats; weights: l floats (after the append) or NULL. */
void oracle_decode(oracle_unit* u, const float* q, const float* tk, const float* tv,
                   int scale_logits, float* out, float* weights);
/* Attention over the current state only (attention.cpp:36-99). */
void oracle_attend(const oracle_unit* u, const float* q, int scale_logits, float* out,
                   float* weights);
/* materialize_keys / materialize_values (src/kv_cache.cpp:100-106): l x d. */
void oracle_materialize(const oracle_unit* u, float* keys, float* values);
/* reference_attention (src/attention.cpp:16-24): q is nq x d. */
void oracle_reference_attention(const float* q, int64_t nq, const float* K, const float* V,
                                int64_t l, int64_t d, int scale_logits, float* out);

/* Counters: [0] key grouped rows, [1] key residual rows, [2] total tokens,
 * [3] key residual capacity, [4] value grouped rows, [5] value residual rows,
 * [6] value residual capacity, [7] memory_bytes(key) (kv_cache.cpp:117-121),
 * [8] memory_bytes(value) (kv_cache.cpp:123-127). */
void oracle_counters(const oracle_unit* u, int64_t* out9);
/* Views of the packed state in the reference layout. */
const uint8_t* oracle_key_packed(const oracle_unit* u, int64_t* nbytes);
const uint8_t* oracle_value_packed(const oracle_unit* u, int64_t* nbytes);
const double* oracle_key_zero(const oracle_unit* u, int64_t* ngroups);
const double* oracle_key_scale(const oracle_unit* u, int64_t* ngroups);
const double* oracle_value_zero(const oracle_unit* u, int64_t* ngroups);
const double* oracle_value_scale(const oracle_unit* u, int64_t* ngroups);
/* Residual rows in token order (rows x d). */
const float* oracle_key_residual(const oracle_unit* u, int64_t* rows);
const float* oracle_value_residual(const oracle_unit* u, int64_t* rows);

/* Counter-based input generator shared by the harness on every side:
 * uniform in [-1, 1) from splitmix64(seed, index).  Exactly reproducible. */
float oracle_uniform(uint64_t seed, uint64_t index);
void oracle_fill_uniform(float* out, int64_t n, uint64_t seed, uint64_t first_index);

#ifdef __cplusplus
}
#endif

#endif /* KIVI_ORACLE_H */
