// Quantize / append / prefill / materialize kernels (bit-exact with the
// reference quantizer).  Generic over B in {1,2,4,8}, any G, R, d with
// R % G == 0 and d % G == 0.
#pragma once

#include "common.cuh"

namespace kivi_b200 {

// Device layout of one cache (all arrays are [n_units][...], unit strides in
// elements of each array).  See DESIGN.md "HBM layout".
struct CacheDev {
    int bits, G, R, d, maxc;
    int64_t n_units;
    // Key codes: reference per-channel group order — bit ((tg*d + c)*G + i)*B
    // of a unit's stream (quantize.cpp:118-127).  Pairs [tg*d + c] = (lo, hi).
    uint8_t* kcodes;
    int64_t k_ustride;  // bytes
    float2* kpairs;
    int64_t kp_ustride;  // float2 elements
    // Value codes: per-token order — bit (t*d + c)*B (quantize.cpp:128-138).
    // Pairs [t*(d/G) + cg].
    uint8_t* vcodes;
    int64_t v_ustride;
    float2* vpairs;
    int64_t vp_ustride;
    // Residual windows: fp32 rings [R][d]; key token t (>= kg) at row t - kg,
    // value token t (>= vg) at row t % R.
    float* kring;
    float* vring;
    int64_t ring_ustride;  // floats
};

// Quantizes one group of G values read as p[i*stride] (i < G) and ORs its
// codes into `codes` starting at bit `bit0`; returns (lo, hi).
__device__ __forceinline__ float2 quantize_group_dev(const float* p, int64_t stride, int G,
                                                     int bits, int maxc, uint8_t* codes,
                                                     uint64_t bit0) {
    float lo = p[0], hi = p[0];
    for (int i = 1; i < G; ++i) minmax_step(p[(int64_t)i * stride], lo, hi);
    CodeCtx cc = make_code_ctx(lo, hi, maxc);
    if (hi != lo) {
        // Accumulate whole 32-bit words, flush each once.
        uint64_t bit = bit0;
        uint32_t word = 0;
        uint64_t cur = bit >> 5;
        for (int i = 0; i < G; ++i, bit += (uint64_t)bits) {
            uint64_t wi = bit >> 5;
            if (wi != cur) {
                if (word) atomicOr(reinterpret_cast<uint32_t*>(codes) + cur, word);
                word = 0;
                cur = wi;
            }
            word |= quant_code(cc, p[(int64_t)i * stride]) << (bit & 31);
        }
        if (word) atomicOr(reinterpret_cast<uint32_t*>(codes) + cur, word);
    }
    return make_float2(lo, hi);
}

// ---- prefill (reference prefill, kv_cache.cpp:23-55) ----------------------

// One thread per key group (unit, tg, c) of the first kg tokens.
__global__ void prefill_keys_kernel(CacheDev c, const float* __restrict__ keys, int64_t l,
                                    int64_t kg) {
    const int64_t tiles = kg / c.G;
    const int64_t per_unit = tiles * c.d;
    const int64_t total = per_unit * c.n_units;
    for (int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gid < total;
         gid += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = gid / per_unit;
        const int64_t g = gid % per_unit;  // tg*d + ch
        const int64_t tg = g / c.d, ch = g % c.d;
        const float* src = keys + (u * l + tg * c.G) * c.d + ch;
        float2 r = quantize_group_dev(src, c.d, c.G, c.bits, c.maxc, c.kcodes + u * c.k_ustride,
                                      (uint64_t)g * c.G * c.bits);
        c.kpairs[u * c.kp_ustride + g] = r;
    }
}

// One thread per value group (unit, t, cg) of the first vg tokens.
__global__ void prefill_values_kernel(CacheDev c, const float* __restrict__ values, int64_t l,
                                      int64_t vg) {
    const int64_t gpt = c.d / c.G;
    const int64_t per_unit = vg * gpt;
    const int64_t total = per_unit * c.n_units;
    for (int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gid < total;
         gid += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = gid / per_unit;
        const int64_t g = gid % per_unit;  // t*gpt + cg
        const int64_t t = g / gpt, cg = g % gpt;
        const float* src = values + (u * l + t) * c.d + cg * c.G;
        float2 r = quantize_group_dev(src, 1, c.G, c.bits, c.maxc, c.vcodes + u * c.v_ustride,
                                      (uint64_t)g * c.G * c.bits);
        c.vpairs[u * c.vp_ustride + g] = r;
    }
}

// Residual rows: keys [kg, l) -> ring rows [0, l-kg); values [vg, l) -> rows t % R.
// vec = 4 (d % 4 == 0, 16-byte aligned rows): one float4 per thread;
// otherwise (vec = 1) one float per thread.
__global__ void prefill_residual_kernel(CacheDev c, const float* __restrict__ keys,
                                        const float* __restrict__ values, int64_t l, int64_t kg,
                                        int64_t vg, int vec) {
    const int64_t kr = l - kg, vr = l - vg;
    const int64_t rowv = c.d / vec;  // vectors per row
    const int64_t per_unit = (kr + vr) * rowv;
    const int64_t total = per_unit * c.n_units;
    for (int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gid < total;
         gid += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = gid / per_unit;
        const int64_t e = gid - u * per_unit;
        const int64_t row = e / rowv;
        const int64_t ch = (e - row * rowv) * vec;
        const float* src;
        float* dst;
        if (row < kr) {
            src = keys + (u * l + kg + row) * c.d + ch;
            dst = c.kring + u * c.ring_ustride + row * c.d + ch;
        } else {
            const int64_t t = vg + (row - kr);
            src = values + (u * l + t) * c.d + ch;
            dst = c.vring + u * c.ring_ustride + (t % c.R) * c.d + ch;
        }
        if (vec == 4)
            *reinterpret_cast<float4*>(dst) = __ldcs(reinterpret_cast<const float4*>(src));
        else
            *dst = *src;
    }
}

// ---- append (reference append_token, kv_cache.cpp:66-98) -----------------
// One CTA per unit.  `l` = token count BEFORE the append.
__global__ void append_kernel(CacheDev c, const float* __restrict__ tk,
                              const float* __restrict__ tv, int64_t l) {
    const int64_t u = blockIdx.x;
    const int R = c.R, d = c.d, G = c.G;
    float* kring = c.kring + u * c.ring_ustride;
    float* vring = c.vring + u * c.ring_ustride;
    const int slot = (int)(l % R);

    // Key: push the row into the ring (row l - kg == l % R).
    for (int ch = threadIdx.x; ch < d; ch += blockDim.x)
        kring[(int64_t)slot * d + ch] = tk[u * d + ch];

    // Value: the FIFO is full (l >= R): quantize the oldest row (token l - R,
    // ring row l % R) per-token before it is overwritten.
    if (l >= R) {
        const int64_t e = l - R;
        const int gpt = d / G;
        for (int cg = threadIdx.x; cg < gpt; cg += blockDim.x) {
            float2 r = quantize_group_dev(vring + (int64_t)slot * d + cg * G, 1, G, c.bits, c.maxc,
                                          c.vcodes + u * c.v_ustride,
                                          ((uint64_t)e * d + (uint64_t)cg * G) * c.bits);
            c.vpairs[u * c.vp_ustride + e * gpt + cg] = r;
        }
    }
    __syncthreads();
    for (int ch = threadIdx.x; ch < d; ch += blockDim.x)
        vring[(int64_t)slot * d + ch] = tv[u * d + ch];

    // Key flush when the residual reaches R rows: quantize the R x d block
    // per-channel into tiles (l+1-R)/G ... (l+1)/G - 1.
    if ((l + 1) % R == 0) {
        const int64_t tile0 = (l + 1 - R) / G;
        const int ngroups = (R / G) * d;
        for (int g = threadIdx.x; g < ngroups; g += blockDim.x) {
            const int tl = g / d, ch = g % d;
            const int64_t gi = (tile0 + tl) * d + ch;
            float2 r = quantize_group_dev(kring + (int64_t)tl * G * d + ch, d, G, c.bits, c.maxc,
                                          c.kcodes + u * c.k_ustride, (uint64_t)gi * G * c.bits);
            c.kpairs[u * c.kp_ustride + gi] = r;
        }
    }
}

// ---- fast append for d = 128, G = 32, B in {2, 4} (one warp per unit) -----
// Same semantics as append_kernel.  Lane j owns channels 4j..4j+3 of a row;
// a 32-channel value group is 8 lanes.  Ties in the group min / max follow
// std::minmax_element (first smallest, last largest) via the channel index.
__device__ __forceinline__ void minmax_pair_reduce8(float& lo, int& ilo, float& hi, int& ihi) {
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        const float olo = __shfl_xor_sync(0xffffffffu, lo, o);
        const int oilo = __shfl_xor_sync(0xffffffffu, ilo, o);
        const float ohi = __shfl_xor_sync(0xffffffffu, hi, o);
        const int oihi = __shfl_xor_sync(0xffffffffu, ihi, o);
        if (olo < lo || (!(lo < olo) && oilo < ilo)) { lo = olo; ilo = oilo; }
        if (ohi > hi || (!(hi > ohi) && oihi > ihi)) { hi = ohi; ihi = oihi; }
    }
}

// One unit's append_token by one warp (d = 128, G = 32).  Also called by the
// residual-window attend kernel, which appends each unit it owns right before
// streaming that unit's residual items (kivi_decode's fused route).
// One token row (d = 128) quantized per-token into d/32 groups by a warp:
// lane j holds channels 4j..4j+3 (x); writes the row's d*B/32 code words and
// its 4 (lo, hi) pairs.  Ties in the group min / max follow
// std::minmax_element (first smallest, last largest) via the channel index.
template <int B>
__device__ __forceinline__ void value_row_fast(const float4 v, int lane, uint32_t* __restrict__ vw,
                                               float2* __restrict__ vp) {
    const float x[4] = {v.x, v.y, v.z, v.w};
    float lo = fminf(fminf(x[0], x[1]), fminf(x[2], x[3]));
    float hi = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (__any_sync(0xffffffffu, lo == 0.0f || hi == 0.0f)) {
        // a zero extreme: +0 / -0 compare equal, so resolve first smallest /
        // last largest by channel index (rare; warp-uniform branch)
        lo = x[0];
        hi = x[0];
        int ilo = 4 * lane, ihi = 4 * lane;
#pragma unroll
        for (int i = 1; i < 4; ++i) {
            if (x[i] < lo) { lo = x[i]; ilo = 4 * lane + i; }
            if (!(x[i] < hi)) { hi = x[i]; ihi = 4 * lane + i; }
        }
        minmax_pair_reduce8(lo, ilo, hi, ihi);
    }
    const CodeCtx cc = make_code_ctx(lo, hi, (1 << B) - 1);
    uint32_t bits = 0, redo = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        bool ex;
        bits |= quant_code_fast(cc, x[i], ex) << (B * i);
        redo |= (uint32_t)ex << i;
    }
    if (redo) {  // rare: near-tie values decided exactly
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (redo & (1u << i))
                bits = (bits & ~(((1u << B) - 1u) << (B * i))) |
                       (quant_code_exact(lo, hi, (1 << B) - 1, x[i]) << (B * i));
    }
    // lane's 4 codes -> position (4*lane*B) of the token's 128*B-bit row
    uint32_t word = bits << ((4 * lane * B) & 31);
    constexpr int LPW = 32 / (4 * B);  // lanes sharing one 32-bit word
#pragma unroll
    for (int o = 1; o < LPW; o <<= 1) word |= __shfl_xor_sync(0xffffffffu, word, o);
    if ((lane % LPW) == 0) vw[(4 * lane * B) >> 5] = word;
    if ((lane & 7) == 0) vp[lane >> 3] = make_float2(lo, hi);
}

// One group of 32 values in stream order (a key group: 32 tokens of one
// channel; a value group: 32 channels of one token) -> its B code words (token i at bits B*(i % (32/B)) of word i / (32/B)) and
// (lo, hi); sequential over the tokens, so first-min / last-max are exact.
template <int B>
__device__ __forceinline__ float2 key_group_fast(const float (&x)[32], uint32_t (&w)[B]) {
    const float2 lh = minmax_first_last(x);
    const CodeCtx cc = make_code_ctx(lh.x, lh.y, (1 << B) - 1);
    constexpr int CPW = 32 / B;  // codes per word
    uint32_t redo = 0;           // values whose code must be decided exactly
#pragma unroll
    for (int k = 0; k < B; ++k) {
        uint32_t word = 0;
#pragma unroll
        for (int i = 0; i < CPW; ++i) {
            bool ex;
            word |= quant_code_fast(cc, x[k * CPW + i], ex) << (B * i);
            redo |= (uint32_t)ex << (k * CPW + i);
        }
        w[k] = word;
    }
    if (redo) {  // rare (near-tie values, non-finite groups)
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (redo & (1u << j)) {
                const int k = j / CPW, sh = B * (j % CPW);
                const uint32_t q = quant_code_exact(cc.lo, cc.hi, cc.maxc, x[j]);
                w[k] = (w[k] & ~(((1u << B) - 1u) << sh)) | (q << sh);
            }
        }
    }
    return lh;
}

template <int B>
__device__ __forceinline__ void store_key_words(uint32_t* dst, const uint32_t (&w)[B]) {
    if constexpr (B == 2) {
        *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
    } else if constexpr (B == 4) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
#pragma unroll
        for (int k = 0; k < B; ++k) dst[k] = w[k];
    }
}

// FLUSH = false leaves the key flush to the flush warps of
// append_flush_fast_kernel (the serial per-warp flush below takes ~130 us).
template <int B, bool FLUSH = true>
__device__ __forceinline__ void append_unit_fast(const CacheDev& c, const float* __restrict__ tk,
                                                 const float* __restrict__ tv, int64_t l,
                                                 int64_t u, int lane) {
    constexpr int D = 128, G = 32;
    const int R = c.R;
    const int slot = (int)(l % R);
    float* kring = c.kring + u * c.ring_ustride;
    float* vring = c.vring + u * c.ring_ustride;
    const float4 kv = reinterpret_cast<const float4*>(tk + u * D)[lane];
    const float4 vv = reinterpret_cast<const float4*>(tv + u * D)[lane];
    reinterpret_cast<float4*>(kring + (int64_t)slot * D)[lane] = kv;

    if (l >= R) {
        // value FIFO pop: quantize the oldest row (token l - R) per-token
        const int64_t e = l - R;
        const float4 old = reinterpret_cast<const float4*>(vring + (int64_t)slot * D)[lane];
        value_row_fast<B>(old, lane,
                          reinterpret_cast<uint32_t*>(c.vcodes + u * c.v_ustride) + e * (D * B / 32),
                          c.vpairs + u * c.vp_ustride + e * (D / G));
    }
    reinterpret_cast<float4*>(vring + (int64_t)slot * D)[lane] = vv;

    if (FLUSH && (l + 1) % R == 0) {
        // key flush: quantize the R x 128 ring per-channel into R/32 tiles;
        // lane owns channels lane, lane+32, lane+64, lane+96 (sequential over
        // the 32 tokens of a group: exact first-min / last-max order).
        __syncwarp();
        const int64_t tile0 = (l + 1 - R) / G;
        uint32_t* kw = reinterpret_cast<uint32_t*>(c.kcodes + u * c.k_ustride);
        for (int tl = 0; tl < R / G; ++tl) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int ch = lane + 32 * q;
                const float* col = kring + (int64_t)tl * G * D + ch;
                float lo = col[0], hi = col[0];
                for (int i = 1; i < G; ++i) minmax_step(col[(int64_t)i * D], lo, hi);
                const CodeCtx cc = make_code_ctx(lo, hi, (1 << B) - 1);
                const int64_t g = (tile0 + tl) * D + ch;
                constexpr int CPW = 32 / B;  // codes per word
#pragma unroll
                for (int w = 0; w < G / CPW; ++w) {
                    uint32_t word = 0;
                    for (int i = 0; i < CPW; ++i)
                        word |= quant_code(cc, col[(int64_t)(w * CPW + i) * D]) << (B * i);
                    kw[g * (G / CPW) + w] = word;
                }
                c.kpairs[u * c.kp_ustride + g] = make_float2(lo, hi);
            }
        }
    }
}

// Optional query staging (qs.src != NULL): the warp of unit u also copies
// that unit's qs.rows query rows from qs.src (host memory mapped into the
// device: the single-layer host path) to qs.dst, so a latency-bound step
// needs no separate H2D copy (each costs ~15 us of DMA setup for 16 KB).
struct QStage {
    const float* src;
    float* dst;
    int rows;  // query rows (q_per_kv) per unit
};

__device__ __forceinline__ void stage_q_rows(const QStage& qs, int64_t u, int lane) {
    if (!qs.src) return;
    const float4* s4 = reinterpret_cast<const float4*>(qs.src + u * qs.rows * 128);
    float4* d4 = reinterpret_cast<float4*>(qs.dst + u * qs.rows * 128);
    for (int i = lane; i < qs.rows * 32; i += 32) d4[i] = s4[i];
}

template <int B>
__global__ void __launch_bounds__(256) append_fast_kernel(CacheDev c, const float* __restrict__ tk,
                                                          const float* __restrict__ tv, int64_t l,
                                                          QStage qs) {
    pdl_trigger();  // the attend launch may be scheduled behind this one
    const int lane = threadIdx.x & 31;
    const int64_t u = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (u >= c.n_units) return;
    stage_q_rows(qs, u, lane);
    append_unit_fast<B, false>(c, tk, tv, l, u, lane);
}

#ifndef KIVI_FLUSH_GPT
#define KIVI_FLUSH_GPT 1
#endif
#if KIVI_FLUSH_STREAM
constexpr int FLUSH_GPT = KIVI_FLUSH_GPT;  // key groups (channels) per flush thread
#else
constexpr int FLUSH_GPT = 1;
#endif

template <int N>
__device__ __forceinline__ void load_vec(const float* p, float (&v)[N]) {
    if constexpr (N == 4) {
        const float4 t = *reinterpret_cast<const float4*>(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else if constexpr (N == 2) {
        const float2 t = *reinterpret_cast<const float2*>(p);
        v[0] = t.x; v[1] = t.y;
    } else {
        v[0] = *p;
    }
}

// Flush warp fw of an early key-tile quantisation.
// KIVI_FLUSH_STREAM: lane = FLUSH_GPT consecutive channels (groups) of one
// (unit, tile); a warp covers 32 * FLUSH_GPT channels, every ring row one
// coalesced load per warp.  Two streaming passes over the 32 rows (min / max,
// then codes) instead of 32 values per group held in registers; per value ~9
// instructions: FMNMX pairs (+0 / -0 re-resolved in order only when an end
// is zero, as minmax_first_last), the code y = fma(v - lo, r, 1.5 * 2^23)
// read from y's mantissa (one LOP3), the near-tie test on
// fma(v - lo, r, -rint) (fewer roundings than quant_code_fast's x, so its tie
// margin still covers the error) and one flag per group instead of a redo
// mask: a group with a near-tie value (rare) is re-coded value by value with
// quant_code.  Codes are the reference's either way.
// Otherwise: one group per lane, 32 values in registers (key_group_fast).
template <int B>
__device__ __forceinline__ void flush_key_group(const CacheDev& c, const float* __restrict__ tk,
                                                int64_t l, int64_t fw, int tl0, int ntl, int lane) {
    constexpr int D = 128, G = 32;
    const int last = (int)(l % c.R);  // ring row of token l (written by this launch)
#if KIVI_FLUSH_STREAM
    constexpr int NG = FLUSH_GPT, WPT = D / (32 * NG);  // warps per (unit, tile)
    const int64_t u = fw / (ntl * WPT);
    if (u >= c.n_units) return;
    const int rem = (int)(fw % (ntl * WPT));
    const int tl = tl0 + rem / WPT;
    const int ch = (rem % WPT) * 32 * NG + lane * NG;
    const float* col = c.kring + u * c.ring_ustride + (int64_t)tl * G * D + ch;
    // token l is the last row of the tile that completes at this step; its ring
    // row may still be in flight from the append blocks of this launch
    const bool own = tk != nullptr && last == tl * G + (G - 1);
    float xl[NG];
    if (own) {
        load_vec<NG>(tk + u * D + ch, xl);
    } else {
        load_vec<NG>(col + (int64_t)(G - 1) * D, xl);
    }
    auto ld = [&](int i, float (&v)[NG]) {
        if (i == G - 1) {
#pragma unroll
            for (int j = 0; j < NG; ++j) v[j] = xl[j];
        } else {
            load_vec<NG>(col + (int64_t)i * D, v);
        }
    };
    float lo[NG], hi[NG];
    {
        float v[NG];
        ld(0, v);
#pragma unroll
        for (int j = 0; j < NG; ++j) lo[j] = hi[j] = v[j];
    }
#pragma unroll
    for (int i = 1; i < G; ++i) {
        float v[NG];
        ld(i, v);
#pragma unroll
        for (int j = 0; j < NG; ++j) {
            lo[j] = fminf(lo[j], v[j]);
            hi[j] = fmaxf(hi[j], v[j]);
        }
    }
#pragma unroll
    for (int j = 0; j < NG; ++j) {
        if (lo[j] == 0.0f || hi[j] == 0.0f) {  // +0 / -0: first zero for lo, last for hi
            float zf = 0.0f, zl = 0.0f;
            bool seen = false;
#pragma unroll 1
            for (int i = 0; i < G; ++i) {
                float v[NG];
                ld(i, v);
                if (v[j] == 0.0f) {
                    if (!seen) zf = v[j];
                    zl = v[j];
                    seen = true;
                }
            }
            if (lo[j] == 0.0f) lo[j] = zf;
            if (hi[j] == 0.0f) hi[j] = zl;
        }
    }
    asm volatile("" ::: "memory");  // re-read the rows below; do not keep them live
    CodeCtx cc[NG];
#pragma unroll
    for (int j = 0; j < NG; ++j) cc[j] = make_code_ctx(lo[j], hi[j], (1 << B) - 1);
    constexpr int CPW = 32 / B;
    uint32_t w[NG][B];
    bool near_tie[NG];
#pragma unroll
    for (int j = 0; j < NG; ++j) {
        near_tie[j] = false;
#pragma unroll
        for (int k = 0; k < B; ++k) w[j][k] = 0u;
    }
#pragma unroll
    for (int i = 0; i < G; ++i) {
        float v[NG];
        ld(i, v);
#pragma unroll
        for (int j = 0; j < NG; ++j) {
            w[j][i / CPW] += quant_code_fma(cc[j], v[j], near_tie[j]) << (B * (i % CPW));
        }
    }
#pragma unroll
    for (int j = 0; j < NG; ++j) {
        if (near_tie[j]) {
#pragma unroll 1
            for (int k = 0; k < B; ++k) {
                uint32_t word = 0;
#pragma unroll 1
                for (int i = 0; i < CPW; ++i) {
                    float v[NG];
                    ld(k * CPW + i, v);
                    word |= quant_code(cc[j], v[j]) << (B * i);
                }
                w[j][k] = word;
            }
        }
    }
    const int64_t g = ((l - l % c.R) / G + tl) * D + ch;
    uint32_t* dst = reinterpret_cast<uint32_t*>(c.kcodes + u * c.k_ustride) + g * B;
#pragma unroll
    for (int j = 0; j < NG; ++j) store_key_words<B>(dst + j * B, w[j]);
    float2* pd = c.kpairs + u * c.kp_ustride + g;
#pragma unroll
    for (int j = 0; j < NG; ++j) pd[j] = make_float2(lo[j], hi[j]);
#else
    const int64_t u = fw / (ntl * (D / 32));
    if (u >= c.n_units) return;
    const int rem = (int)(fw % (ntl * (D / 32)));
    const int tl = tl0 + rem / (D / 32);
    const int ch = (rem % (D / 32)) * 32 + lane;
    const float* kring = c.kring + u * c.ring_ustride;
    const int64_t g = ((l - l % c.R) / G + tl) * D + ch;
    uint32_t w[B];
    float2 lh;
    float x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const int r = tl * G + i;
        x[i] = (r == last && tk) ? __ldg(tk + u * D + ch) : kring[(int64_t)r * D + ch];
    }
    lh = key_group_fast<B>(x, w);
    store_key_words<B>(reinterpret_cast<uint32_t*>(c.kcodes + u * c.k_ustride) + g * B, w);
    c.kpairs[u * c.kp_ustride + g] = lh;
#endif
}

// Append plus early key-tile quantisation: blocks [0, n_app) append one unit
// per warp (no flush); the remaining blocks quantize ring tiles
// [tl0, tl0 + ntl) of the current window (kg = l - l % R), one thread per
// (unit, 32-token tile, channel) group: lanes are 32 consecutive channels, so
// every token row is one coalesced 128-byte load per warp and the group's
// code words one contiguous store.
//
// A key tile is quantized as soon as its 32 rows are in the ring, not all
// R / 32 at the flush: the attend kernels and every export read codes of
// tiles below kg only, the rows stay fp32 in the ring until the flush
// (kv_cache.cpp:80-90), and a tile's codes depend on its own 32 rows only —
// so the flush step's work is one tile, not R / 32 (kivi_cache::kq_done).
// Row l % R (token l) is read from t_k, which the append warps write
// concurrently; with t_k == NULL (n_app = 0: the projection kernel already
// wrote the row) from the ring.
template <int B>
#ifndef KIVI_FLUSH_MINB
#define KIVI_FLUSH_MINB 1
#endif
__global__ void __launch_bounds__(256, KIVI_FLUSH_MINB) append_flush_fast_kernel(CacheDev c,
                                                                const float* __restrict__ tk,
                                                                const float* __restrict__ tv,
                                                                int64_t l, int n_app, int tl0,
                                                                int ntl, QStage qs) {
    pdl_trigger();
    constexpr int D = 128, G = 32;
    const int lane = threadIdx.x & 31;
    if ((int)blockIdx.x < n_app) {
        const int64_t u = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
        if (u < c.n_units) {
            stage_q_rows(qs, u, lane);
            append_unit_fast<B, false>(c, tk, tv, l, u, lane);
        }
        return;
    }
    const int64_t fw = (int64_t)(blockIdx.x - n_app) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    flush_key_group<B>(c, tk, l, fw, tl0, ntl, lane);
}

// ---- bulk prefill for d = 128, G = 32, B in {2, 4} --------------------------
// Keys: one thread per (unit, tile, channel) group, lanes on consecutive
// channels (coalesced token rows), whole code words stored (no atomics).
template <int B>
__global__ void __launch_bounds__(256) prefill_keys_fast_kernel(CacheDev c,
                                                                const float* __restrict__ keys,
                                                                int64_t l, int64_t kg) {
    constexpr int D = 128, G = 32;
    const int64_t per_unit = (kg / G) * D;
    const int64_t total = per_unit * c.n_units;
    for (int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gid < total;
         gid += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = gid / per_unit;
        const int64_t g = gid % per_unit;  // tg * D + ch
        const int64_t tg = g / D, ch = g % D;
        const float* src = keys + (u * l + tg * G) * D + ch;
        float x[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = __ldcs(src + (int64_t)i * D);
        uint32_t w[B];
        const float2 lh = key_group_fast<B>(x, w);
        store_key_words<B>(reinterpret_cast<uint32_t*>(c.kcodes + u * c.k_ustride) + g * B, w);
        c.kpairs[u * c.kp_ustride + g] = lh;
    }
}

// Values: one thread per (unit, token, 32-channel group): the group's 128
// contiguous bytes as 8 float4 loads (a warp's first load touches 32 lines,
// the next seven hit the sectors L1 already holds), min / max and codes in
// registers exactly as for a key group — no cross-lane reductions, ~1/3 of
// the instructions of a warp-per-row split.  Group g = t * 4 + cg of a unit
// has its codes at word g * B and its pair at g, as a key group does.
template <int B>
__global__ void __launch_bounds__(256) prefill_values_fast_kernel(CacheDev c,
                                                                  const float* __restrict__ values,
                                                                  int64_t l, int64_t vg) {
    constexpr int D = 128, G = 32;
    const int64_t per_unit = vg * (D / G);
    const int64_t total = per_unit * c.n_units;
    for (int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gid < total;
         gid += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = gid / per_unit;
        const int64_t g = gid - u * per_unit;  // t * 4 + cg
        const float4* src = reinterpret_cast<const float4*>(values + u * l * D + g * G);
        float x[32];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float4 v = __ldcs(src + i);
            x[4 * i] = v.x;
            x[4 * i + 1] = v.y;
            x[4 * i + 2] = v.z;
            x[4 * i + 3] = v.w;
        }
        uint32_t w[B];
        const float2 lh = key_group_fast<B>(x, w);
        store_key_words<B>(reinterpret_cast<uint32_t*>(c.vcodes + u * c.v_ustride) + g * B, w);
        c.vpairs[u * c.vp_ustride + g] = lh;
    }
}

// ---- one group, quantized and dequantized in one launch --------------------
// Reference quantize_group (quantize.cpp:22-48) of n values (any n, any B in
// [1, 8]) followed by dequantize_group (quantize.cpp:50-57) of its result: one
// CTA, every value loaded once in parallel (the facade's inputs sit in mapped
// host memory: a serial per-value loop would be one PCIe round trip per value),
// first-smallest / last-largest by index, codes decided exactly as
// quant_code, z / s as the reference's doubles.
__global__ void __launch_bounds__(256) quantize_group_kernel(const float* __restrict__ v, int n,
                                                             int maxc, uint8_t* __restrict__ codes,
                                                             double* __restrict__ zp,
                                                             double* __restrict__ sc,
                                                             float* __restrict__ deq) {
    __shared__ float s_lo[8], s_hi[8];
    __shared__ int s_ilo[8], s_ihi[8];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    float lo = INFINITY, hi = -INFINITY;
    int ilo = INT_MAX, ihi = -1;
    for (int i = t; i < n; i += blockDim.x) {
        const float x = v[i];
        if (x < lo || (!(lo < x) && i < ilo)) { lo = x; ilo = i; }
        if (x > hi || (!(hi > x) && i > ihi)) { hi = x; ihi = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float olo = __shfl_xor_sync(0xffffffffu, lo, o);
        const int oilo = __shfl_xor_sync(0xffffffffu, ilo, o);
        const float ohi = __shfl_xor_sync(0xffffffffu, hi, o);
        const int oihi = __shfl_xor_sync(0xffffffffu, ihi, o);
        if (olo < lo || (!(lo < olo) && oilo < ilo)) { lo = olo; ilo = oilo; }
        if (ohi > hi || (!(hi > ohi) && oihi > ihi)) { hi = ohi; ihi = oihi; }
    }
    if (lane == 0) {
        s_lo[warp] = lo; s_ilo[warp] = ilo;
        s_hi[warp] = hi; s_ihi[warp] = ihi;
    }
    __syncthreads();
    lo = s_lo[0]; ilo = s_ilo[0]; hi = s_hi[0]; ihi = s_ihi[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
        if (s_ilo[w] >= 0 && s_ilo[w] != INT_MAX &&
            (s_lo[w] < lo || (!(lo < s_lo[w]) && s_ilo[w] < ilo))) { lo = s_lo[w]; ilo = s_ilo[w]; }
        if (s_ihi[w] >= 0 && (s_hi[w] > hi || (!(hi > s_hi[w]) && s_ihi[w] > ihi))) {
            hi = s_hi[w]; ihi = s_ihi[w];
        }
    }
    // lo / hi are elements of v (the reference's minmax_element values)
    const CodeCtx cc = make_code_ctx(lo, hi, maxc);
    const double s = group_scale(lo, hi, maxc);
    for (int i = t; i < n; i += blockDim.x) {
        const uint32_t q = hi == lo ? 0u : quant_code(cc, v[i]);
        codes[i] = (uint8_t)q;
        if (deq) deq[i] = dequant_exact(q, s, (double)lo);
    }
    if (t == 0) {
        *zp = (double)lo;
        *sc = s;
    }
}

// ---- materialize (reference materialize_*, kv_cache.cpp:100-106) ---------
__global__ void materialize_kernel(CacheDev c, int64_t l, int64_t kg, int64_t vg,
                                   float* __restrict__ kout, float* __restrict__ vout) {
    const int64_t per_unit = l * c.d;
    const int64_t total = per_unit * c.n_units;
    const int gpt = c.d / c.G;
    for (int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gid < total;
         gid += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = gid / per_unit;
        const int64_t e = gid % per_unit;
        const int64_t t = e / c.d, ch = e % c.d;
        if (kout) {
            float val;
            if (t < kg) {
                const int64_t tg = t / c.G, i = t % c.G;
                const int64_t g = tg * c.d + ch;
                float2 pr = c.kpairs[u * c.kp_ustride + g];
                uint32_t code = read_code(c.kcodes + u * c.k_ustride,
                                          ((uint64_t)g * c.G + i) * c.bits, c.bits);
                val = dequant_exact(code, group_scale(pr.x, pr.y, c.maxc), (double)pr.x);
            } else {
                val = c.kring[u * c.ring_ustride + (t - kg) * c.d + ch];
            }
            kout[gid] = val;
        }
        if (vout) {
            float val;
            if (t < vg) {
                const int64_t g = t * gpt + ch / c.G;
                float2 pr = c.vpairs[u * c.vp_ustride + g];
                uint32_t code = read_code(c.vcodes + u * c.v_ustride,
                                          ((uint64_t)t * c.d + ch) * c.bits, c.bits);
                val = dequant_exact(code, group_scale(pr.x, pr.y, c.maxc), (double)pr.x);
            } else {
                val = c.vring[u * c.ring_ustride + (t % c.R) * c.d + ch];
            }
            vout[gid] = val;
        }
    }
}

// ---- export / import in the reference layout --------------------------------
// (lo, hi) pairs -> reference (zero_point, scale) doubles.
__global__ void pairs_to_zs_kernel(const float2* __restrict__ pairs, int64_t n, int maxc,
                                   double* __restrict__ z, double* __restrict__ s) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float2 p = pairs[i];
        z[i] = (double)p.x;
        s[i] = group_scale(p.x, p.y, maxc);
    }
}

// Reference (zero_point, scale) -> (lo, hi): hi = float(z + s*maxc) recovers
// the group maximum for every state this library exported.
__global__ void zs_to_pairs_kernel(const double* __restrict__ z, const double* __restrict__ s,
                                   int64_t n, int maxc, float2* __restrict__ pairs) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float lo = (float)z[i];
        float hi = (float)__dadd_rn(z[i], __dmul_rn(s[i], (double)maxc));
        // A degenerate group (reference hi == lo: scale 1.0, every code 0) must
        // export scale 1.0 again.  float(z + maxc) need not land exactly maxc
        // above z (z = 0.1f, B = 2 re-exports 0.99999997), so such a group is
        // stored as hi == lo.  A genuine scale-1.0 group has hi - lo == maxc up
        // to double rounding and round-trips through the first branch; its
        // dequantisation is unchanged either way (codes 0 give z).
        if (s[i] == 1.0 && group_scale(lo, hi, maxc) != 1.0) hi = lo;
        pairs[i] = make_float2(lo, hi);
    }
}

// Value ring (tokens [vg, l) at rows t % R) <-> token-ordered rows.
__global__ void ring_gather_kernel(const float* __restrict__ ring, int64_t first_token,
                                   int64_t rows, int R, int d, float* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * d;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / d, ch = i % d;
        out[i] = ring[((first_token + r) % R) * d + ch];
    }
}
__global__ void ring_scatter_kernel(float* __restrict__ ring, int64_t first_token, int64_t rows,
                                    int R, int d, const float* __restrict__ in) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * d;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / d, ch = i % d;
        ring[((first_token + r) % R) * d + ch] = in[i];
    }
}

// ---- standalone matrix quantizer (QuantizedTensor::quantize) --------------
// One thread per group; group order per quantize.cpp:105-140.
__global__ void quantize_matrix_kernel(const float* __restrict__ m, int64_t rows, int64_t cols,
                                       int bits, int G, int per_channel, uint8_t* packed,
                                       double* __restrict__ zp, double* __restrict__ sc) {
    const int maxc = (1 << bits) - 1;
    const int64_t ngroups = rows * cols / G;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngroups;
         g += (int64_t)gridDim.x * blockDim.x) {
        const float* src;
        int64_t stride;
        if (per_channel) {
            const int64_t tg = g / cols, ch = g % cols;
            src = m + tg * G * cols + ch;
            stride = cols;
        } else {
            const int64_t gpr = cols / G;
            const int64_t r = g / gpr, cg = g % gpr;
            src = m + r * cols + cg * G;
            stride = 1;
        }
        float2 r = quantize_group_dev(src, stride, G, bits, maxc, packed, (uint64_t)g * G * bits);
        zp[g] = (double)r.x;
        sc[g] = group_scale(r.x, r.y, maxc);
    }
}

// Unpacked variant for any B in [1, 8]: codes[g*G + i] = code of element i
// of group g (reference quantize_grouped, quantize.cpp:105-140).
__global__ void quantize_codes_kernel(const float* __restrict__ m, int64_t rows, int64_t cols,
                                      int bits, int G, int per_channel, uint8_t* __restrict__ codes,
                                      double* __restrict__ zp, double* __restrict__ sc) {
    const int maxc = (1 << bits) - 1;
    const int64_t ngroups = rows * cols / G;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngroups;
         g += (int64_t)gridDim.x * blockDim.x) {
        const float* src;
        int64_t stride;
        if (per_channel) {
            const int64_t tg = g / cols, ch = g % cols;
            src = m + tg * G * cols + ch;
            stride = cols;
        } else {
            const int64_t gpr = cols / G;
            src = m + (g / gpr) * cols + (g % gpr) * G;
            stride = 1;
        }
        float lo = src[0], hi = src[0];
        for (int i = 1; i < G; ++i) minmax_step(src[(int64_t)i * stride], lo, hi);
        const CodeCtx cc = make_code_ctx(lo, hi, maxc);
        for (int i = 0; i < G; ++i) codes[g * G + i] = (uint8_t)quant_code(cc, src[(int64_t)i * stride]);
        zp[g] = (double)lo;
        sc[g] = group_scale(lo, hi, maxc);
    }
}

__global__ void dequantize_codes_kernel(const uint8_t* __restrict__ codes,
                                        const double* __restrict__ zp,
                                        const double* __restrict__ sc, int64_t rows, int64_t cols,
                                        int G, int per_channel, float* __restrict__ out) {
    const int64_t n = rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / cols, ch = e % cols;
        int64_t g, pos;
        if (per_channel) {
            g = (r / G) * cols + ch;
            pos = g * G + r % G;
        } else {
            g = r * (cols / G) + ch / G;
            pos = e;
        }
        out[e] = dequant_exact(codes[pos], sc[g], zp[g]);
    }
}

// QuantizedTensor::dequantize: one thread per element.
__global__ void dequantize_matrix_kernel(const uint8_t* __restrict__ packed,
                                         const double* __restrict__ zp,
                                         const double* __restrict__ sc, int64_t rows,
                                         int64_t cols, int bits, int G, int per_channel,
                                         float* __restrict__ out) {
    const int64_t n = rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / cols, ch = e % cols;
        int64_t g, pos;
        if (per_channel) {
            const int64_t tg = r / G, i = r % G;
            g = tg * cols + ch;
            pos = g * G + i;
        } else {
            g = r * (cols / G) + ch / G;
            pos = e;  // per-token stream order == row-major order
        }
        uint32_t code = read_code(packed, (uint64_t)pos * bits, bits);
        out[e] = dequant_exact(code, sc[g], zp[g]);
    }
}

// pack_codes: one thread per output byte; flags out-of-range codes.
__global__ void pack_codes_kernel(const uint8_t* __restrict__ codes, int64_t n, int bits,
                                  uint8_t* __restrict__ bytes, int* __restrict__ bad) {
    const int per = 8 / bits;
    const int64_t nbytes = (n * bits + 7) / 8;
    const int maxc = (1 << bits) - 1;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nbytes;
         b += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v = 0;
        for (int k = 0; k < per; ++k) {
            const int64_t i = b * per + k;
            if (i >= n) break;
            uint32_t cd = codes[i];
            if (cd > (uint32_t)maxc) atomicMax(bad, 1);
            v |= (cd & (uint32_t)maxc) << (k * bits);
        }
        bytes[b] = (uint8_t)v;
    }
}

__global__ void unpack_codes_kernel(const uint8_t* __restrict__ bytes, int64_t n, int bits,
                                    uint8_t* __restrict__ codes) {
    const uint32_t mask = (1u << bits) - 1u;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t bit = (uint64_t)i * bits;
        codes[i] = (uint8_t)((bytes[bit >> 3] >> (bit & 7)) & mask);
    }
}

}  // namespace kivi_b200
