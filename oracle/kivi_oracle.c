/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference KIVI hot
 * path (see kivi_oracle.h).  Compiled with -ffp-contract=off so every float
 * and double operation rounds exactly as the reference's Release build on
 * x86-64 (no FMA contraction; reference proj/CMakeLists.txt:9-11).
 * Paths below are relative to /root/reference/proj.
 */
#include "kivi_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- quantizer ---------------------------------------------------------- */

/* src/quantize.cpp:22-48 */
int oracle_quantize_group(const float* v, int64_t n, int bits, uint8_t* codes, double* zero,
                          double* scale) {
    if (n <= 0) return 2;                  /* :23 UsageError("empty group") */
    if (bits < 1 || bits > 8) return 2;    /* :24 */
    /* std::minmax_element: first smallest, last largest (:26) */
    float lo = v[0], hi = v[0];
    for (int64_t i = 1; i < n; ++i) {
        if (v[i] < lo) lo = v[i];
        if (!(v[i] < hi)) hi = v[i];
    }
    const int max_code = (1 << bits) - 1;
    *zero = (double)lo;                    /* :32 */
    if ((double)hi == (double)lo) {        /* :34-38 degenerate group */
        *scale = 1.0;
        memset(codes, 0, (size_t)n);
        return 0;
    }
    const double s = ((double)hi - (double)lo) / (double)max_code; /* :39 */
    *scale = s;
    for (int64_t i = 0; i < n; ++i) {      /* :40-45 */
        double q = nearbyint(((double)v[i] - (double)lo) / s);
        if (q < 0.0) q = 0.0;
        if (q > (double)max_code) q = (double)max_code;
        codes[i] = (uint8_t)q;
    }
    return 0;
}

/* src/quantize.cpp:50-57 */
void oracle_dequantize_group(const uint8_t* codes, int64_t n, double zero, double scale,
                             float* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = (float)((double)codes[i] * scale + zero);
}

static int packable(int bits) { return bits == 1 || bits == 2 || bits == 4 || bits == 8; }

/* src/quantize.cpp:59-76 */
int oracle_pack_codes(const uint8_t* codes, int64_t n, int bits, uint8_t* bytes) {
    if (!packable(bits)) return 2;
    const int max_code = (1 << bits) - 1;
    memset(bytes, 0, (size_t)((n * bits + 7) / 8));
    for (int64_t i = 0; i < n; ++i) {
        if (codes[i] > max_code) return 2;
        const int64_t bit = i * bits;
        bytes[bit >> 3] |= (uint8_t)(codes[i] << (bit & 7));
    }
    return 0;
}

/* src/quantize.cpp:78-93 */
int oracle_unpack_codes(const uint8_t* bytes, int64_t nbytes, int64_t n, int bits,
                        uint8_t* codes) {
    if (!packable(bits)) return 2;
    if ((n * bits + 7) / 8 > nbytes) return 2;
    const uint8_t mask = (uint8_t)((1 << bits) - 1);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t bit = i * bits;
        codes[i] = (uint8_t)((bytes[bit >> 3] >> (bit & 7)) & mask);
    }
    return 0;
}

static uint8_t code_at(const uint8_t* packed, int64_t i, int bits) {
    /* include/kivi/quantize.hpp:79-83 */
    const int64_t bit = i * bits;
    return (uint8_t)((packed[bit >> 3] >> (bit & 7)) & ((1 << bits) - 1));
}

/* Appends `n` codes at code position `pos` of a zero-initialised stream. */
static void put_codes(uint8_t* packed, int64_t pos, const uint8_t* codes, int64_t n, int bits) {
    for (int64_t i = 0; i < n; ++i) {
        const int64_t bit = (pos + i) * bits;
        packed[bit >> 3] |= (uint8_t)(codes[i] << (bit & 7));
    }
}

/* src/quantize.cpp:105-140 (group order) + :171-185 (packing). */
int oracle_quantize_matrix(const float* m, int64_t rows, int64_t cols, int bits, int64_t G,
                           int per_channel, uint8_t* packed, double* zero, double* scale) {
    if (bits < 1 || bits > 8 || G < 1) return 3;            /* QuantParams::validate */
    if (!packable(bits)) return 3;                           /* :173-176 */
    const int64_t extent = per_channel ? rows : cols;
    if (extent % G != 0) return 1;                           /* :109-116 ShapeError */
    memset(packed, 0, (size_t)((rows * cols * bits + 7) / 8));
    uint8_t* codes = (uint8_t*)malloc((size_t)G);
    float* buf = (float*)malloc(sizeof(float) * (size_t)G);
    int64_t g = 0;
    if (per_channel) {
        for (int64_t tg = 0; tg < rows / G; ++tg)
            for (int64_t c = 0; c < cols; ++c, ++g) {
                for (int64_t i = 0; i < G; ++i) buf[i] = m[(tg * G + i) * cols + c];
                oracle_quantize_group(buf, G, bits, codes, &zero[g], &scale[g]);
                put_codes(packed, g * G, codes, G, bits);
            }
    } else {
        for (int64_t r = 0; r < rows; ++r)
            for (int64_t cg = 0; cg < cols / G; ++cg, ++g) {
                for (int64_t i = 0; i < G; ++i) buf[i] = m[r * cols + cg * G + i];
                oracle_quantize_group(buf, G, bits, codes, &zero[g], &scale[g]);
                put_codes(packed, g * G, codes, G, bits);
            }
    }
    free(codes);
    free(buf);
    return 0;
}

/* src/quantize.cpp:142-167 */
void oracle_dequantize_matrix(const uint8_t* packed, const double* zero, const double* scale,
                              int64_t rows, int64_t cols, int bits, int64_t G, int per_channel,
                              float* out) {
    int64_t pos = 0, g = 0;
    if (per_channel) {
        for (int64_t tg = 0; tg < rows / G; ++tg)
            for (int64_t c = 0; c < cols; ++c, ++g)
                for (int64_t i = 0; i < G; ++i, ++pos)
                    out[(tg * G + i) * cols + c] =
                        (float)((double)code_at(packed, pos, bits) * scale[g] + zero[g]);
    } else {
        for (int64_t r = 0; r < rows; ++r)
            for (int64_t cg = 0; cg < cols / G; ++cg, ++g)
                for (int64_t i = 0; i < G; ++i, ++pos)
                    out[r * cols + cg * G + i] =
                        (float)((double)code_at(packed, pos, bits) * scale[g] + zero[g]);
    }
}

/* ---- streaming cache ---------------------------------------------------- */

typedef struct {
    uint8_t* packed;
    int64_t packed_cap;
    double* zero;
    double* scale;
    int64_t groups, groups_cap;
    int64_t rows;
} qstore;

struct oracle_unit {
    int bits;
    int64_t G, R, d;
    qstore kq, vq;
    float* kres; /* up to R rows, token order */
    int64_t kres_rows;
    float* vres; /* FIFO, up to R rows, token order */
    int64_t vres_rows;
    int64_t total;
    int64_t kcap, vcap; /* residual_capacity */
    int initialised;    /* residual.cols() == d once set up */
};

static void qstore_free(qstore* q) {
    free(q->packed);
    free(q->zero);
    free(q->scale);
    memset(q, 0, sizeof(*q));
}

/* Appends `ntok` tokens' worth of groups (QuantizedTensor::concat_tokens,
 * src/quantize.cpp:194-217: a pure append of codes and groups). */
static void qstore_append(qstore* q, const uint8_t* codes, int64_t ncodes, const double* z,
                          const double* s, int64_t ngroups, int64_t ntok, int bits, int64_t d) {
    const int64_t start_pos = q->rows * d; /* codes already stored */
    const int64_t need = ((start_pos + ncodes) * bits + 7) / 8;
    if (need > q->packed_cap) {
        int64_t cap = q->packed_cap ? q->packed_cap : 64;
        while (cap < need) cap *= 2;
        q->packed = (uint8_t*)realloc(q->packed, (size_t)cap);
        memset(q->packed + q->packed_cap, 0, (size_t)(cap - q->packed_cap));
        q->packed_cap = cap;
    }
    put_codes(q->packed, start_pos, codes, ncodes, bits);
    if (q->groups + ngroups > q->groups_cap) {
        int64_t cap = q->groups_cap ? q->groups_cap : 64;
        while (cap < q->groups + ngroups) cap *= 2;
        q->zero = (double*)realloc(q->zero, sizeof(double) * (size_t)cap);
        q->scale = (double*)realloc(q->scale, sizeof(double) * (size_t)cap);
        q->groups_cap = cap;
    }
    memcpy(q->zero + q->groups, z, sizeof(double) * (size_t)ngroups);
    memcpy(q->scale + q->groups, s, sizeof(double) * (size_t)ngroups);
    q->groups += ngroups;
    q->rows += ntok;
}

/* Quantizes a rows x d block with the given axis and appends it. */
static void quantize_append(qstore* q, const float* m, int64_t rows, int64_t d, int bits,
                            int64_t G, int per_channel) {
    if (rows == 0) return;
    const int64_t n = rows * d, ng = n / G;
    uint8_t* packed = (uint8_t*)calloc((size_t)((n * bits + 7) / 8 + 1), 1);
    double* z = (double*)malloc(sizeof(double) * (size_t)ng);
    double* s = (double*)malloc(sizeof(double) * (size_t)ng);
    uint8_t* codes = (uint8_t*)malloc((size_t)n);
    oracle_quantize_matrix(m, rows, d, bits, G, per_channel, packed, z, s);
    oracle_unpack_codes(packed, (n * bits + 7) / 8, n, bits, codes);
    qstore_append(q, codes, n, z, s, ng, rows, bits, d);
    free(packed);
    free(z);
    free(s);
    free(codes);
}

oracle_unit* oracle_unit_new(int bits, int64_t G, int64_t R, int64_t d) {
    oracle_unit* u = (oracle_unit*)calloc(1, sizeof(oracle_unit));
    u->bits = bits;
    u->G = G;
    u->R = R;
    u->d = d;
    u->kres = (float*)calloc((size_t)(R * d), sizeof(float));
    u->vres = (float*)calloc((size_t)(R * d), sizeof(float));
    return u;
}

void oracle_unit_free(oracle_unit* u) {
    if (!u) return;
    qstore_free(&u->kq);
    qstore_free(&u->vq);
    free(u->kres);
    free(u->vres);
    free(u);
}

static void unit_reset(oracle_unit* u) {
    qstore_free(&u->kq);
    qstore_free(&u->vq);
    u->kres_rows = u->vres_rows = 0;
    u->total = u->kcap = u->vcap = 0;
}

/* src/kv_cache.cpp:23-55 */
int oracle_prefill(oracle_unit* u, const float* keys, const float* values, int64_t l) {
    if (l == 0) return 2;
    unit_reset(u);
    const int64_t R = u->R, d = u->d;
    const int64_t key_res = l % R;                          /* :37 */
    quantize_append(&u->kq, keys, l - key_res, d, u->bits, u->G, 1);
    memcpy(u->kres, keys + (l - key_res) * d, sizeof(float) * (size_t)(key_res * d));
    u->kres_rows = key_res;
    u->kcap = key_res;
    const int64_t value_res = l < R ? l : R;               /* :45 */
    quantize_append(&u->vq, values, l - value_res, d, u->bits, u->G, 0);
    memcpy(u->vres, values + (l - value_res) * d, sizeof(float) * (size_t)(value_res * d));
    u->vres_rows = value_res;
    u->vcap = value_res;
    u->total = l;
    u->initialised = 1;
    return 0;
}

/* src/kv_cache.cpp:66-98 */
void oracle_append(oracle_unit* u, const float* tk, const float* tv) {
    const int64_t R = u->R, d = u->d;
    /* key: push, flush the R-row block per-channel (:76-84) */
    memcpy(u->kres + u->kres_rows * d, tk, sizeof(float) * (size_t)d);
    u->kres_rows += 1;
    if (u->kres_rows > u->kcap) u->kcap = u->kres_rows;
    if (u->kres_rows == R) {
        quantize_append(&u->kq, u->kres, R, d, u->bits, u->G, 1);
        u->kres_rows = 0;
    }
    /* value: FIFO pop of the oldest row when full, then push (:87-97) */
    if (u->vres_rows == R) {
        quantize_append(&u->vq, u->vres, 1, d, u->bits, u->G, 0);
        memmove(u->vres, u->vres + d, sizeof(float) * (size_t)((R - 1) * d));
        u->vres_rows = R - 1;
    }
    memcpy(u->vres + u->vres_rows * d, tv, sizeof(float) * (size_t)d);
    u->vres_rows += 1;
    if (u->vres_rows > u->vcap) u->vcap = u->vres_rows;
    u->total += 1;
    u->initialised = 1;
}

static float logit_scale(int64_t d, int scale_logits) {
    /* src/attention.cpp:10-12 */
    return scale_logits ? 1.0f / sqrtf((float)d) : 1.0f;
}

/* src/attention.cpp:36-99 (after the append at :32) */
void oracle_attend(const oracle_unit* u, const float* q, int scale_logits, float* out,
                   float* weights) {
    const int64_t d = u->d, G = u->G, l = u->total;
    const int bits = u->bits;
    const int64_t kg = u->kq.rows, vg = u->vq.rows;
    double* gl = (double*)calloc((size_t)(kg ? kg : 1), sizeof(double));
    float* logits = (float*)malloc(sizeof(float) * (size_t)l);
    float* w = (float*)malloc(sizeof(float) * (size_t)l);
    /* :40-58 grouped key logits, double, channel order per token */
    int64_t pos = 0, group = 0;
    for (int64_t tg = 0; tg < kg / G; ++tg)
        for (int64_t c = 0; c < d; ++c, ++group) {
            const double z = u->kq.zero[group], s = u->kq.scale[group], qc = q[c];
            for (int64_t i = 0; i < G; ++i, ++pos)
                gl[tg * G + i] += qc * ((double)code_at(u->kq.packed, pos, bits) * s + z);
        }
    for (int64_t t = 0; t < kg; ++t) logits[t] = (float)gl[t];        /* :59-62 */
    for (int64_t r = 0; r < u->kres_rows; ++r) {                      /* :63-66 */
        float acc = 0.0f;
        for (int64_t c = 0; c < d; ++c) acc += q[c] * u->kres[r * d + c];
        logits[kg + r] = acc;
    }
    const float sc = logit_scale(d, scale_logits);                    /* :67 */
    for (int64_t t = 0; t < l; ++t) logits[t] *= sc;
    /* :70 softmax_rows (include/kivi/matrix.hpp:31-39) */
    float mx = logits[0];
    for (int64_t t = 1; t < l; ++t) mx = logits[t] > mx ? logits[t] : mx;
    for (int64_t t = 0; t < l; ++t) w[t] = expf(logits[t] - mx);
    float sum = 0.0f;
    for (int64_t t = 0; t < l; ++t) sum += w[t];
    for (int64_t t = 0; t < l; ++t) w[t] /= sum;
    /* :73-90 grouped values, double, token order per channel */
    double* acc = (double*)calloc((size_t)d, sizeof(double));
    pos = 0;
    group = 0;
    for (int64_t t = 0; t < vg; ++t) {
        const double wt = w[t];
        for (int64_t cg = 0; cg < d / G; ++cg, ++group) {
            const double z = u->vq.zero[group], s = u->vq.scale[group];
            for (int64_t i = 0; i < G; ++i, ++pos)
                acc[cg * G + i] += wt * ((double)code_at(u->vq.packed, pos, bits) * s + z);
        }
    }
    /* :91-98 residual product + combine */
    const int64_t vr = u->vres_rows;
    for (int64_t c = 0; c < d; ++c) {
        float r = 0.0f;
        for (int64_t k = 0; k < vr; ++k) r += w[l - vr + k] * u->vres[k * d + c];
        out[c] = r;
        if (vg > 0) out[c] += (float)acc[c];
    }
    if (weights) memcpy(weights, w, sizeof(float) * (size_t)l);
    free(gl);
    free(logits);
    free(w);
    free(acc);
}

/* src/attention.cpp:26-100 */
void oracle_decode(oracle_unit* u, const float* q, const float* tk, const float* tv,
                   int scale_logits, float* out, float* weights) {
    oracle_append(u, tk, tv);
    oracle_attend(u, q, scale_logits, out, weights);
}

/* src/kv_cache.cpp:100-106 */
void oracle_materialize(const oracle_unit* u, float* keys, float* values) {
    const int64_t d = u->d;
    if (keys) {
        if (u->kq.rows)
            oracle_dequantize_matrix(u->kq.packed, u->kq.zero, u->kq.scale, u->kq.rows, d, u->bits,
                                     u->G, 1, keys);
        memcpy(keys + u->kq.rows * d, u->kres, sizeof(float) * (size_t)(u->kres_rows * d));
    }
    if (values) {
        if (u->vq.rows)
            oracle_dequantize_matrix(u->vq.packed, u->vq.zero, u->vq.scale, u->vq.rows, d, u->bits,
                                     u->G, 0, values);
        memcpy(values + u->vq.rows * d, u->vres, sizeof(float) * (size_t)(u->vres_rows * d));
    }
}

/* src/attention.cpp:16-24 */
void oracle_reference_attention(const float* q, int64_t nq, const float* K, const float* V,
                                int64_t l, int64_t d, int scale_logits, float* out) {
    float* lg = (float*)malloc(sizeof(float) * (size_t)l);
    const float sc = logit_scale(d, scale_logits);
    for (int64_t r = 0; r < nq; ++r) {
        for (int64_t t = 0; t < l; ++t) {
            float acc = 0.0f;
            for (int64_t c = 0; c < d; ++c) acc += q[r * d + c] * K[t * d + c];
            lg[t] = acc * sc;
        }
        float mx = lg[0];
        for (int64_t t = 1; t < l; ++t) mx = lg[t] > mx ? lg[t] : mx;
        for (int64_t t = 0; t < l; ++t) lg[t] = expf(lg[t] - mx);
        float sum = 0.0f;
        for (int64_t t = 0; t < l; ++t) sum += lg[t];
        for (int64_t t = 0; t < l; ++t) lg[t] /= sum;
        for (int64_t c = 0; c < d; ++c) {
            float acc = 0.0f;
            for (int64_t t = 0; t < l; ++t) acc += lg[t] * V[t * d + c];
            out[r * d + c] = acc;
        }
    }
    free(lg);
}

/* src/kv_cache.cpp:110-127 */
static uint64_t grouped_bytes(const qstore* q, int64_t d, int bits) {
    return (uint64_t)((q->rows * d * bits + 7) / 8) + 4u * (uint64_t)q->groups;
}

void oracle_counters(const oracle_unit* u, int64_t* o) {
    const int64_t cols = u->initialised ? u->d : 0;
    o[0] = u->kq.rows;
    o[1] = u->kres_rows;
    o[2] = u->total;
    o[3] = u->kcap;
    o[4] = u->vq.rows;
    o[5] = u->vres_rows;
    o[6] = u->vcap;
    o[7] = (int64_t)(grouped_bytes(&u->kq, u->d, u->bits) + 2u * (uint64_t)u->kcap * (uint64_t)cols);
    o[8] = (int64_t)(grouped_bytes(&u->vq, u->d, u->bits) + 2u * (uint64_t)u->vcap * (uint64_t)cols);
}

const uint8_t* oracle_key_packed(const oracle_unit* u, int64_t* nbytes) {
    *nbytes = (u->kq.rows * u->d * u->bits + 7) / 8;
    return u->kq.packed;
}
const uint8_t* oracle_value_packed(const oracle_unit* u, int64_t* nbytes) {
    *nbytes = (u->vq.rows * u->d * u->bits + 7) / 8;
    return u->vq.packed;
}
const double* oracle_key_zero(const oracle_unit* u, int64_t* n) {
    *n = u->kq.groups;
    return u->kq.zero;
}
const double* oracle_key_scale(const oracle_unit* u, int64_t* n) {
    *n = u->kq.groups;
    return u->kq.scale;
}
const double* oracle_value_zero(const oracle_unit* u, int64_t* n) {
    *n = u->vq.groups;
    return u->vq.zero;
}
const double* oracle_value_scale(const oracle_unit* u, int64_t* n) {
    *n = u->vq.groups;
    return u->vq.scale;
}
const float* oracle_key_residual(const oracle_unit* u, int64_t* rows) {
    *rows = u->kres_rows;
    return u->kres;
}
const float* oracle_value_residual(const oracle_unit* u, int64_t* rows) {
    *rows = u->vres_rows;
    return u->vres;
}

/* ---- deterministic inputs ---------------------------------------------- */

static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

float oracle_uniform(uint64_t seed, uint64_t index) {
    const uint64_t h = splitmix64(seed * 0xD1B54A32D192ED03ull ^ splitmix64(index));
    /* 24 random bits -> [0,1) exactly, then to [-1, 1) */
    return (float)(h >> 40) * (1.0f / 16777216.0f) * 2.0f - 1.0f;
}

void oracle_fill_uniform(float* out, int64_t n, uint64_t seed, uint64_t first_index) {
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_uniform(seed, first_index + (uint64_t)i);
}
