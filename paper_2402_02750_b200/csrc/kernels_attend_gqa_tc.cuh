// Fused dequant-attention decode on the tensor cores (mma.sync m16n8k16,
// fp16 operands, fp32 accumulation).  H = 1, 2 or 4 query heads share one kv
// unit (H = 1: MHA, BASELINE configs 1/2/5; H = 4: config 3, Mistral-7B);
// B = 2, d = 128, G = 32.  Body items only (whole 256-token sub-chunks whose keys
// and values are all quantized); items holding fp32 residual rows run on the
// CUDA-core kernel (kernels_attend_gqa.cuh) concurrently.
//
// Why tensor cores for a GEMV: with H heads every code feeds H multiply-adds.
// On CUDA cores that is 1 LOP3 + H/2 FFMA2 per code (3 issue slots at H = 4,
// and the ALU pipe saturates on the extraction at H = 1); the MMA does the
// H-way and the 16-deep reduction in one instruction per 256 codes, leaving
// ~0.6 ALU ops per code for the extraction.  N = 8 columns hold (head, hi/lo)
// pairs, so at H = 1 three quarters of each MMA are zero padding; the tensor
// pipe is otherwise idle, so that costs nothing measurable.
//
// Exactness.  Codes enter the MMA as fp16 SUBNORMALS: a 2-bit code at
// mantissa bit p of a half is code * 2^(p-24) exactly (a LOP3 isolates it; no
// conversion).  p is 6 or 8, the top of the mantissa: the tensor core aligns
// products by nominal exponent, so low subnormal bits would lose precision
// (measured: codes at bits 0-1 cost ~7 bits on 50x outlier channels).  The other operand is x = q'_h * s * 2^E (keys) or
// p_h * s * 2^E (values), split as x = hi + lo with hi = x truncated to 10
// mantissa bits (exact in fp16) and lo = fp16(x - hi): 21 significant bits.
// 2^E (power of two, per job) keeps |x| < 2^14, inside fp16 range.  The MMA
// accumulates in fp32; hi and lo land in two N-columns of the same head and
// are added in the epilogue.
//
// Keys (per 32-token tile T, per 16-channel K step):
//   D[token row][n = 2h + part] += A[row][k] * B[k][n]
//   A = codes: lane (g, t) holds the byte (g & 3) of word (channel, half
//       g >> 2), i.e. tokens 4g..4g+3 of its 4 channels 8s + 2t + {0, 1}
//       and 64 + 8s + 2t + {0, 1} (K step s: channels 8s.., 64+8s..);
//       one PRMT pairs channels (c, c+1) into the two fp16 halves and a
//       LOP3 (after one shared shift) per token position j selects the code:
//       row g <-> token 4g + 2m, row g+8 <-> 4g + 2m + 1 in MMA m (m = 0, 1).
//   B = split(q'_h[c] * s_T[c] * 2^E), built cooperatively per tile (lane L
//       computes the 16 products of channels 2L, 2L+1, 64+2L, 65+2L:
//       conflict-free pair loads) and stored in fragment
//       order in shared memory.
//   The epilogue needs no reduction: lane (g, t) owns head t, tokens 4g+j.
//   bias_h(T) = sum_c q'_h[c] z_T[c] is an fp32 dot product reduced through
//   shared memory once per job.
// Values (per 16-token K step, per 32-channel group cg), transposed:
//   D[channel row][n = 2h + part] += A[row][k = token] * B[k][n]
//   A = codes: lane (g, t) holds byte 8cg + g (channels 32cg + 4g + {0..3})
//       of tokens 16s + t + 4i; PRMT pairs two tokens, LOP3 picks channel j.
//   B = split(p_h[t] * s[t][cg] * 2^E), built cooperatively per K step.
//   sum_t p_h[t] z[t][cg] is an fp32 FMA chain reduced per item.
#pragma once

#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels_attend_fast.cuh"

namespace kivi_b200 {
namespace gqa_tc {

using fast::D;
// Job geometry: a key job is KT 32-token tiles (KT KB codes + KT KB (lo, hi)),
// a value job VT tokens (VT x 32 B codes + VT x 32 B pairs).  Small jobs keep
// the per-warp shared memory at ~19 KB, so 3 CTAs x 4 warps fit an SM: the
// kernel is latency-bound and needs the warps more than the larger jobs.
#ifndef KIVI_GQA_TC_KT
#define KIVI_GQA_TC_KT 2
#endif
constexpr int KT = KIVI_GQA_TC_KT;
constexpr int VT = KT * 32;
constexpr int SLOT = KT * 2048;
using fast::SUB;
#ifndef KIVI_GQA_TC_WARPS
#define KIVI_GQA_TC_WARPS 4
#endif
constexpr int WARPS = KIVI_GQA_TC_WARPS;   // warps per CTA
#ifndef KIVI_GQA_TC_MIN_CTAS
#define KIVI_GQA_TC_MIN_CTAS (KT == 2 ? 3 : 2)
#endif
constexpr int MIN_CTAS = KIVI_GQA_TC_MIN_CTAS;
#ifndef KIVI_GQA_UNROLL
#define KIVI_GQA_UNROLL 1
#endif
#ifndef KIVI_GQA_KEY_SPLIT
#define KIVI_GQA_KEY_SPLIT 1
#endif
constexpr int KEY_SPLIT = KIVI_GQA_KEY_SPLIT;  // 1: two accumulator chains per key tile
constexpr int BFK_ROW = 9;        // uint2 per consumer lane in the key B buffer (8 K steps + pad)
constexpr int BFV_CG = 72;        // 32-bit words per channel group in the value B buffer (64 + pad)
constexpr int BIAS_ROW = 17;      // floats per lane row of the key-bias transpose
constexpr uint32_t FULL = 0xffffffffu;

// probs layout: token pairs (t, t+4) with t & 4 == 0 side by side per head,
// so the value producer reads (p_h[t], p_h[t+4]) as one float2:
//   pidx(t, h) = ((t >> 3) * 4 + (t & 3)) * 2H + 2h + ((t >> 2) & 1)
// H = 4: the four pair blocks of a 32-word row are XOR-swizzled by the row
// (bits 3-4 ^= (t >> 3) & 3): the key epilogue's stores (lanes g = 0..7 on
// tokens 4g + j) then spread over 32 banks instead of 8.
template <int H>
__device__ __forceinline__ int pidx(int t, int h) {
    const int i = ((t >> 3) * 4 + (t & 3)) * (2 * H) + 2 * h + ((t >> 2) & 1);
    return H == 4 ? i ^ (((t >> 3) & 3) << 3) : i;
}
// logical pair block of physical block p (the swizzle is an involution)
template <int H>
__device__ __forceinline__ int pblock(int p) {
    return H == 4 ? p ^ ((p >> 2) & 3) : p;
}

// IT: tokens per item.  IT = 384 keeps the per-warp footprint inside 3 CTAs x
// 4 warps per SM by single-buffering the B fragments (one more warp barrier
// per tile / K step).
template <int H, int IT = SUB>
struct TS {  // per-warp shared memory
    // q rows are staged (TMA) into the key-bias scratch: q is consumed at the
    // start of an item, the scratch only afterwards, and the next item's q
    // is issued only after this item's key jobs are done.
    static constexpr int QB_OFF = 2 * SLOT;                   // [H][128] q | [32][17] bias
    static constexpr int QB_BYTES = (32 * BIAS_ROW * 4 > H * D * 4) ? 32 * BIAS_ROW * 4 : H * D * 4;
    static constexpr int PROBS_OFF = QB_OFF + ((QB_BYTES + 15) & ~15);  // [256 x H] p (pidx)
    static constexpr int BF_OFF = PROBS_OFF + IT * H * 4;      // B fragments (keys | values)
    static constexpr int BFK_BYTES = 32 * BFK_ROW * 8;         // 2304 = 2 x 4 x 72 x 4
    static constexpr bool DB = IT <= SUB;                     // double-buffered fragments
    static constexpr int BF_BYTES = (DB ? 2 : 1) * BFK_BYTES;
    static constexpr int ZS_OFF = BF_OFF + BF_BYTES;           // [H][4] value z sums
    static constexpr int BAR_OFF = ZS_OFF + 16 * 4;
    static constexpr int BYTES = BAR_OFF + 16;
    static constexpr int STRIDE = (BYTES + 127) & ~127;
    static_assert((DB ? 2 : 1) * 4 * BFV_CG * 4 <= BF_BYTES, "value B buffers overflow");
    static_assert(BFK_BYTES % 16 == 0, "key B buffer alignment");
};

__device__ __forceinline__ void mma_f16(float4& d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d.x), "+f"(d.y), "+f"(d.z), "+f"(d.w)
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// x = (x0, x1) -> fp16x2 words (hi, lo) with x = hi + lo to ~2^-21 relative:
// hi = x truncated to 10 mantissa bits (exact in fp16), lo = x - hi (exact in
// fp32, one packed FFMA2), rounded to fp16.
__device__ __forceinline__ void split_pair(float2 x, uint32_t& whi, uint32_t& wlo) {
    const float2 h = make_float2(__uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u),
                                 __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u));
    const float2 l = __ffma2_rn(h, make_float2(-1.0f, -1.0f), x);
    __half2 hh = __floats2half2_rn(h.x, h.y);
    __half2 ll = __floats2half2_rn(l.x, l.y);
    whi = *reinterpret_cast<uint32_t*>(&hh);
    wlo = *reinterpret_cast<uint32_t*>(&ll);
}

// Biased exponent byte of a bound m (clamped >= 13): 2^(140 - eb) * m < 2^14.
__device__ __forceinline__ int exp_byte(float m) {
    return max((int)((__float_as_uint(m) >> 23) & 0xFFu), 13);
}
__device__ __forceinline__ float scale_up(int eb) { return __uint_as_float((uint32_t)(267 - eb) << 23); }
// 2^(24 - p - E) with 2^E = scale_up(eb): undoes the subnormal code position
// (code * 2^(p-24), code at mantissa bits p, p+1) and the 2^E operand scale.
__device__ __forceinline__ float unscale(int eb, int p) {
    return __uint_as_float((uint32_t)(eb + 11 - p) << 23);
}

// The four codes of a PRMT'd word x = [byte, byte | byte', byte'] (each fp16
// half holds one code byte twice) as fp16 subnormal pairs.  The tensor core
// aligns products by their NOMINAL exponent, so a subnormal operand loses as
// many bits as it has leading mantissa zeros: every code is taken from the
// top of the mantissa (bits 8-9, or 6-7), never from the bottom.  Code j of
// the byte -> mantissa position code_pos(j) = {8, 6, 8, 6}.
__host__ __device__ constexpr int code_pos(int j) { return (j & 1) ? 6 : 8; }
struct CodeQuad {
    uint32_t c[4];
};
__device__ __forceinline__ CodeQuad code_quad(uint32_t x) {
    const uint32_t y = x >> 4;
    CodeQuad q;
    q.c[0] = x & 0x03000300u;  // upper copy, bits 0-1 of the byte -> mantissa 8-9
    q.c[1] = y & 0x00C000C0u;  // upper copy, bits 2-3 -> 6-7
    q.c[2] = y & 0x03000300u;  // upper copy, bits 4-5 -> 8-9
    q.c[3] = x & 0x00C000C0u;  // lower copy, bits 6-7 -> 6-7
    return q;
}

// Two MMAs sharing B in one asm statement: the eight A registers are live at
// once, so ptxas gives them distinct quads (with one MMA per statement it
// funnelled every MMA through the same four registers, serialising the
// extraction LOP3s behind the previous MMA's operand read).
__device__ __forceinline__ void mma_f16_x2(float4& d0, float4& d1, const CodeQuad& ca,
                                           const CodeQuad& cb, uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%8,%9,%10,%11}, "
        "{%16,%17}, {%0,%1,%2,%3};\n\t"
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%4,%5,%6,%7}, {%12,%13,%14,%15}, "
        "{%16,%17}, {%4,%5,%6,%7};"
        : "+f"(d0.x), "+f"(d0.y), "+f"(d0.z), "+f"(d0.w), "+f"(d1.x), "+f"(d1.y), "+f"(d1.z),
          "+f"(d1.w)
        : "r"(ca.c[0]), "r"(ca.c[1]), "r"(cb.c[0]), "r"(cb.c[1]), "r"(ca.c[2]), "r"(ca.c[3]),
          "r"(cb.c[2]), "r"(cb.c[3]), "r"(b0), "r"(b1));
}


// -------------------------------------------------------------------------
// One key job: KT tiles (codes [KT][1024 B], pairs [KT][128] (lo, hi)) -> the
// log2-domain logits of tokens tok0 .. tok0+32KT-1 x H heads at probs[pidx].
// -------------------------------------------------------------------------
template <int H, bool DB = true>
__device__ __forceinline__ void key_job(const uint8_t* slot, const float2 (&qv)[H][2], float qmax,
                                        float* probs, int tok0, uint8_t* bf, float* biasm, int lane,
                                        uint32_t sel, int ntl) {
    const int g = lane >> 2, t = lane & 3;
    const float4* pairs4 = reinterpret_cast<const float4*>(slot + KT * 1024);
    // pre-pass over this lane's channels (2L, 2L+1, 64+2L, 65+2L) of the KT tiles: spans,
    // bias partials, job-wide span maximum
    float dmax = 0.f;
#pragma unroll
    for (int T = 0; T < KT; ++T) {
        if (T < ntl) {  // tiles past a partial item's end were not loaded
            const float4 p01 = pairs4[T * 64 + lane];
            const float4 p23 = pairs4[T * 64 + 32 + lane];
            const float lo[4] = {p01.x, p01.z, p23.x, p23.z};
            dmax = fmaxf(dmax, fmaxf(fmaxf(p01.y - p01.x, p01.w - p01.z),
                                     fmaxf(p23.y - p23.x, p23.w - p23.z)));
#pragma unroll
            for (int h = 0; h < H; ++h) {
                float b = qv[h][0].x * lo[0];
                b = fmaf(qv[h][0].y, lo[1], b);
                b = fmaf(qv[h][1].x, lo[2], b);
                b = fmaf(qv[h][1].y, lo[3], b);
                biasm[lane * BIAS_ROW + T * H + h] = b;
            }
        } else {
#pragma unroll
            for (int h = 0; h < H; ++h) biasm[lane * BIAS_ROW + T * H + h] = 0.f;
        }
    }
    dmax = warp_max_redux(dmax);
    const int eb = exp_byte(qmax * dmax * (1.0f / 3.0f));
    const float f = scale_up(eb) * (1.0f / 3.0f);
    __syncwarp();
    // bias column sums: lane L sums column L & 15 over 16 rows, then xor 16
    float bs = 0.f;
    {
        // KT * H <= 16 columns; lane L sums column L % NC over rows of its share
        constexpr int NC = (KT * H <= 8) ? 8 : 16;
        constexpr int RPL = NC;  // rows per lane
        const int col = lane & (NC - 1), r0 = (lane / NC) * RPL;
#pragma unroll
        for (int r = 0; r < RPL; ++r) bs += biasm[(r0 + r) * BIAS_ROW + col];
#pragma unroll
        for (int o = NC; o < 32; o <<= 1) bs += __shfl_xor_sync(FULL, bs, o);
    }
    const int s_p = lane >> 2, t_p = lane & 3;  // producer -> consumer K step / lane slot
    // producer: B fragments of tile T into buffer T & 1
    auto produce = [&](int T) {
        uint2* bfk = reinterpret_cast<uint2*>(bf + (DB ? (T & 1) : 0) * TS<H>::BFK_BYTES);
        const float4 p01 = pairs4[T * 64 + lane];
        const float4 p23 = pairs4[T * 64 + 32 + lane];
        const float2 f2 = make_float2(f, f);
        const float2 d01 = __fmul2_rn(make_float2(p01.y - p01.x, p01.w - p01.z), f2);
        const float2 d23 = __fmul2_rn(make_float2(p23.y - p23.x, p23.w - p23.z), f2);
#pragma unroll
        for (int h = 0; h < H; ++h) {
            uint32_t hi01, lo01, hi23, lo23;
            split_pair(__fmul2_rn(qv[h][0], d01), hi01, lo01);
            split_pair(__fmul2_rn(qv[h][1], d23), hi23, lo23);
            bfk[((2 * h) * 4 + t_p) * BFK_ROW + s_p] = make_uint2(hi01, hi23);
            bfk[((2 * h + 1) * 4 + t_p) * BFK_ROW + s_p] = make_uint2(lo01, lo23);
        }
    };
    // consumer: 8 K steps x 2 MMAs of tile T, then its logits
    auto consume = [&](int T) {
        const uint2* bfk = reinterpret_cast<const uint2*>(bf + (DB ? (T & 1) : 0) * TS<H>::BFK_BYTES);
        // even / odd K steps accumulate separately: two independent HMMA
        // chains per token half
        float4 acc[2][2];
#pragma unroll
        for (int e = 0; e < 2; ++e) acc[e][0] = acc[e][1] = make_float4(0.f, 0.f, 0.f, 0.f);
        const uint8_t* ct = slot + T * 1024 + 4 * (g >> 2);
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            // K step s: channels 8s .. 8s+7 (K 2t, 2t+1 <-> 8s + 2t + {0, 1})
            // and 64 + 8s .. 64 + 8s + 7 (K 2t+8, 2t+9), as the producer lane
            // 4s + t built them (its pairs: channels 2L, 2L+1, 64+2L, 65+2L)
            const int cb = (8 * s + 2 * t) * 8;
            const uint32_t w0 = *reinterpret_cast<const uint32_t*>(ct + cb);
            const uint32_t w1 = *reinterpret_cast<const uint32_t*>(ct + cb + 8);
            const uint32_t w2 = *reinterpret_cast<const uint32_t*>(ct + cb + 512);
            const uint32_t w3 = *reinterpret_cast<const uint32_t*>(ct + cb + 520);
            const CodeQuad c01 = code_quad(__byte_perm(w0, w1, sel));
            const CodeQuad c23 = code_quad(__byte_perm(w2, w3, sel));
            uint2 b = make_uint2(0u, 0u);
            if (g < 2 * H) b = bfk[lane * BFK_ROW + s];
            mma_f16_x2(acc[s & KEY_SPLIT][0], acc[s & KEY_SPLIT][1], c01, c23, b.x, b.y);
        }
        float4 acc0 = acc[0][0], acc1 = acc[0][1];
        if (KEY_SPLIT) {
            acc0.x += acc[1][0].x; acc0.y += acc[1][0].y; acc0.z += acc[1][0].z; acc0.w += acc[1][0].w;
            acc1.x += acc[1][1].x; acc1.y += acc[1][1].y; acc1.z += acc[1][1].z; acc1.w += acc[1][1].w;
        }
        const float bias = __shfl_sync(FULL, bs, (T * H + t) & 15);  // column T*H+t
        if (t < H) {
            // tokens tb + j, j = 0..3 share the pair block of tb (tb & 3 == 0)
            const int tb = tok0 + T * 32 + 4 * g;
            // tokens tb + j sit in pair blocks j of one row (swizzled: j ^ r)
            probs[pidx<H>(tb + 0, t)] = fmaf(acc0.x + acc0.y, unscale(eb, code_pos(0)), bias);
            probs[pidx<H>(tb + 1, t)] = fmaf(acc0.z + acc0.w, unscale(eb, code_pos(1)), bias);
            probs[pidx<H>(tb + 2, t)] = fmaf(acc1.x + acc1.y, unscale(eb, code_pos(2)), bias);
            probs[pidx<H>(tb + 3, t)] = fmaf(acc1.z + acc1.w, unscale(eb, code_pos(3)), bias);
        }
    };
    // two fragment buffers: one warp barrier per tile orders producer and
    // consumer (tile T+1's producer writes the buffer tile T-1 read before
    // the barrier of tile T).  Building tile T+1 during tile T's MMAs measured
    // slower (374 vs 360 us on C3): register pressure, no extra overlap.
#if KIVI_GQA_UNROLL
#pragma unroll
    for (int T = 0; T < KT; ++T) {
        if (T < ntl) {
            produce(T);
            __syncwarp();
            consume(T);
            if (!DB) __syncwarp();  // one buffer: the next producer overwrites it
        }
    }
#else
#pragma unroll 1
    for (int T = 0; T < ntl; ++T) {
        produce(T);
        __syncwarp();
        consume(T);
        if (!DB) __syncwarp();
    }
#endif
    __syncwarp();  // the next job's producer overwrites the buffers
}

// Softmax of each head over the item's 256 tokens (probs in pidx layout, in
// place, log2 domain) -> p in (0, 1]; ml[h] = (max, sum).  Lane L owns the
// pair blocks L + 32i (tokens tb, tb+4 with tb = (b >> 2) * 8 + (b & 3)).
template <int H, int IT = SUB>
__device__ __forceinline__ void softmax_heads(float* probs, float* wlog, int64_t wstride, float2* ml,
                                              int lane, int ntok = IT) {
    constexpr int NP = IT / 64;  // pair blocks per lane
    __syncwarp();
    float2 v[NP][H];
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        if constexpr (H == 1) {
            v[i][0] = reinterpret_cast<const float2*>(probs)[lane + 32 * i];
        } else {
            const float4* src = reinterpret_cast<const float4*>(probs + (lane + 32 * i) * 2 * H);
#pragma unroll
            for (int h2 = 0; h2 < H / 2; ++h2) {
                const float4 x = src[h2];
                v[i][2 * h2] = make_float2(x.x, x.y);
                v[i][2 * h2 + 1] = make_float2(x.z, x.w);
            }
        }
    }
    float m[H], sm[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
        m[h] = fmaxf(v[0][h].x, v[0][h].y);
#pragma unroll
        for (int i = 1; i < NP; ++i) m[h] = fmaxf(m[h], fmaxf(v[i][h].x, v[i][h].y));
        m[h] = warp_max_redux(m[h]);
        sm[h] = 0.f;
    }
    if (wlog) {
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            const int b = pblock<H>(lane + 32 * i);
            const int tb = (b >> 2) * 8 + (b & 3);
#pragma unroll
            for (int h = 0; h < H; ++h) {
                if (tb < ntok) wlog[h * wstride + tb] = v[i][h].x;
                if (tb + 4 < ntok) wlog[h * wstride + tb + 4] = v[i][h].y;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < NP; ++i) {
#pragma unroll
        for (int h = 0; h < H; ++h) {
            v[i][h].x = fast::ex2_approx(v[i][h].x - m[h]);
            v[i][h].y = fast::ex2_approx(v[i][h].y - m[h]);
            sm[h] += v[i][h].x + v[i][h].y;
        }
        if constexpr (H == 1) {
            reinterpret_cast<float2*>(probs)[lane + 32 * i] = v[i][0];
        } else {
            float4* dst = reinterpret_cast<float4*>(probs + (lane + 32 * i) * 2 * H);
#pragma unroll
            for (int h2 = 0; h2 < H / 2; ++h2)
                dst[h2] = make_float4(v[i][2 * h2].x, v[i][2 * h2].y, v[i][2 * h2 + 1].x,
                                      v[i][2 * h2 + 1].y);
        }
    }
#pragma unroll
    for (int h = 0; h < H; ++h) ml[h] = make_float2(m[h], warp_sum(sm[h]));
    __syncwarp();
}

// -------------------------------------------------------------------------
// One value job: VT tokens (codes [VT][32 B], pairs [VT][4] (lo, hi)),
// probabilities p_src (pidx layout, job-relative) -> vacc[cg][m], zs[h]
// (this lane's share of sum_t p_h[t] z[t][cg = lane & 3], token pair halves).  eb_run is the running
// exponent byte (the larger of all jobs so far: smaller 2^E).
// -------------------------------------------------------------------------
template <int H, bool FULL = true, bool DB = true>
__device__ __forceinline__ void value_job(const uint8_t* slot, const float* p_src, float4 (&vacc)[4][2],
                                          float2 (&zs)[H], int& eb_run, bool first, uint8_t* bf,
                                          int lane, uint32_t sel, int ntok = VT) {
    if constexpr (FULL) ntok = VT;
    const int g = lane >> 2, t = lane & 3;
    const float4* pairs4 = reinterpret_cast<const float4*>(slot + VT * 32);
    const float2* pairs2 = reinterpret_cast<const float2*>(slot + VT * 32);
    float dmax = 0.f;
#pragma unroll
    for (int i = 0; i < VT / 16; ++i) {
        if (FULL || (lane + 32 * i) / 2 < ntok) {  // float4 f holds token f / 2
            const float4 pr = pairs4[lane + 32 * i];
            dmax = fmaxf(dmax, fmaxf(pr.y - pr.x, pr.w - pr.z));
        }
    }
    dmax = warp_max_redux(dmax);
    const int eb = exp_byte(dmax * (1.0f / 3.0f));
    if (first) {
        eb_run = eb;
    } else if (eb > eb_run) {  // larger spans: drop the accumulators to the new scale
        const float r = __uint_as_float((uint32_t)(127 - min(eb - eb_run, 126)) << 23);
#pragma unroll
        for (int cg = 0; cg < 4; ++cg)
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                vacc[cg][m].x *= r; vacc[cg][m].y *= r; vacc[cg][m].z *= r; vacc[cg][m].w *= r;
            }
        eb_run = eb;
    }
    const float f = scale_up(eb_run) * (1.0f / 3.0f);
    const int p = lane >> 2, cgp = lane & 3;
    const int tcons = p & 3, which = p >> 2;
    const int toff = (p < 4) ? p : p + 4;  // this producer's token pair: (toff, toff + 4)
    // producer: B fragments of K step s into buffer s & 1
    auto produce = [&](int s) {
        uint32_t* bv = reinterpret_cast<uint32_t*>(bf) + (DB ? (s & 1) : 0) * (4 * BFV_CG);
        const int ta = 16 * s + toff, tb = ta + 4;
        // tokens past a partial item's end: zero operands (their slot bytes
        // were not loaded)
        const float2 pa = (FULL || ta < ntok) ? pairs2[ta * 4 + cgp] : make_float2(0.f, 0.f);
        const float2 pb = (FULL || tb < ntok) ? pairs2[tb * 4 + cgp] : make_float2(0.f, 0.f);
        const float2 d2 = __fmul2_rn(make_float2(pa.y - pa.x, pb.y - pb.x), make_float2(f, f));
        const float2 z2 = make_float2(pa.x, pb.x);
        float2 P[H];  // (p_h[ta], p_h[tb])
        if constexpr (H == 1) {
            P[0] = *reinterpret_cast<const float2*>(p_src + pidx<H>(ta, 0));
        } else {
            const float4* pp = reinterpret_cast<const float4*>(p_src + pidx<H>(ta, 0));
#pragma unroll
            for (int h2 = 0; h2 < H / 2; ++h2) {
                const float4 x = pp[h2];
                P[2 * h2] = make_float2(x.x, x.y);
                P[2 * h2 + 1] = make_float2(x.z, x.w);
            }
        }
#pragma unroll
        for (int h = 0; h < H; ++h) {
            uint32_t whi, wlo;
            split_pair(__fmul2_rn(P[h], d2), whi, wlo);
            // scalar FMAs: z2 = (pa.x, pb.x) is not a register pair, and
            // FFMA2 on it cost ~6 register moves per step
            zs[h].x = fmaf(P[h].x, z2.x, zs[h].x);
            zs[h].y = fmaf(P[h].y, z2.y, zs[h].y);
            bv[cgp * BFV_CG + 2 * ((2 * h) * 4 + tcons) + which] = whi;
            bv[cgp * BFV_CG + 2 * ((2 * h + 1) * 4 + tcons) + which] = wlo;
        }
    };
    // consumer: 4 channel groups x 2 MMAs of K step s
    auto consume = [&](int s) {
        const uint32_t* bv = reinterpret_cast<const uint32_t*>(bf) + (DB ? (s & 1) : 0) * (4 * BFV_CG);
#pragma unroll
        for (int cg = 0; cg < 4; ++cg) {
            const uint8_t* cw = slot + 4 * (2 * cg + (g >> 2)) + (16 * s + t) * 32;
            const uint32_t w0 = *reinterpret_cast<const uint32_t*>(cw);
            const uint32_t w1 = *reinterpret_cast<const uint32_t*>(cw + 4 * 32);
            const uint32_t w2 = *reinterpret_cast<const uint32_t*>(cw + 8 * 32);
            const uint32_t w3 = *reinterpret_cast<const uint32_t*>(cw + 12 * 32);
            const CodeQuad c01 = code_quad(__byte_perm(w0, w1, sel));
            const CodeQuad c23 = code_quad(__byte_perm(w2, w3, sel));
            uint2 b = make_uint2(0u, 0u);
            if (g < 2 * H) b = reinterpret_cast<const uint2*>(bv + cg * BFV_CG)[lane];
            mma_f16_x2(vacc[cg][0], vacc[cg][1], c01, c23, b.x, b.y);
        }
    };
    // one warp barrier per K step (two buffers, as in key_job)
#if KIVI_GQA_UNROLL
    if constexpr (FULL) {
#pragma unroll
        for (int s = 0; s < VT / 16; ++s) {
            produce(s);
            __syncwarp();
            consume(s);
            if (!DB) __syncwarp();  // one buffer: the next producer overwrites it
        }
    } else
#endif
    {
#pragma unroll 1
        for (int s = 0; s < (ntok + 15) / 16; ++s) {
            produce(s);
            __syncwarp();
            consume(s);
            if (!DB) __syncwarp();
        }
    }
}

// Write the item's H partials: lane (g, t) owns head t, channels
// 32cg + 4g + {0..3}.
template <int H>
__device__ __forceinline__ void value_finalize(const float4 (&vacc)[4][2], const float2 (&zs2)[H],
                                               int eb, const float2* ml, float* zsm, float* part_o,
                                               float2* part_ml, int lane) {
    const int g = lane >> 2, t = lane & 3;
    float zs[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
        zs[h] = zs2[h].x + zs2[h].y;
        zs[h] += __shfl_xor_sync(FULL, zs[h], 4);
        zs[h] += __shfl_xor_sync(FULL, zs[h], 8);
        zs[h] += __shfl_xor_sync(FULL, zs[h], 16);
    }
    __syncwarp();
    if (lane < 4) {
#pragma unroll
        for (int h = 0; h < H; ++h) zsm[h * 4 + lane] = zs[h];
    }
    __syncwarp();
    if (t < H) {
        const float4 z = reinterpret_cast<const float4*>(zsm)[t];
        const float zc[4] = {z.x, z.y, z.z, z.w};
        float* po = part_o + (int64_t)t * D + 4 * g;
#pragma unroll
        for (int cg = 0; cg < 4; ++cg) {
            float4 o;
            o.x = fmaf(vacc[cg][0].x + vacc[cg][0].y, unscale(eb, code_pos(0)), zc[cg]);
            o.y = fmaf(vacc[cg][0].z + vacc[cg][0].w, unscale(eb, code_pos(1)), zc[cg]);
            o.z = fmaf(vacc[cg][1].x + vacc[cg][1].y, unscale(eb, code_pos(2)), zc[cg]);
            o.w = fmaf(vacc[cg][1].z + vacc[cg][1].w, unscale(eb, code_pos(3)), zc[cg]);
            *reinterpret_cast<float4*>(po + 32 * cg) = o;
        }
    }
#pragma unroll
    for (int h = 0; h < H; ++h)
        if (lane == h) part_ml[h] = ml[h];
}

// -------------------------------------------------------------------------
// Body kernel: persistent warps take items (unit, 256-token sub-chunk of
// [0, body_end) — all keys and values quantized; the last item of a unit may
// be partial) from an atomic counter; key and value jobs stream through two TMA
// slots per warp (as fast::attend_body_kernel).  A partial item's missing
// tiles / tokens are never loaded nor computed: zero-byte jobs complete their
// barrier at once, their logits are -inf and their value operands zero.
// -------------------------------------------------------------------------
template <int H, int IT = SUB>
__global__ void __launch_bounds__(WARPS * 32, MIN_CTAS) attend_gqa_tc_kernel(fast::FastArgs a) {
    using WS = TS<H, IT>;
    using PB = fast::P<2>;
    constexpr int NKJ = (IT / 32) / KT, NVJ = IT / VT, NJ = NKJ + NVJ;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* wbase = smem_raw + warp * WS::STRIDE;
    float* qraw = reinterpret_cast<float*>(wbase + WS::QB_OFF);
    float* biasm = qraw;
    float* probs = reinterpret_cast<float*>(wbase + WS::PROBS_OFF);
    uint8_t* bf = wbase + WS::BF_OFF;
    float* zsm = reinterpret_cast<float*>(wbase + WS::ZS_OFF);
    uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + WS::BAR_OFF);
    if (lane == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const uint64_t policy = make_evict_first_policy();
    const CacheDev& c = a.c;
    const int nper = a.n_per_unit;
    const uint32_t sel = (uint32_t)(lane >> 2 & 3) * 0x1111u + 0x4400u;
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.work_clear) *a.work_clear = 0;

    auto grab = [&]() -> int {
        int v = 0;
        if (lane == 0) v = atomicAdd(a.work, 1);
        return __shfl_sync(FULL, v, 0);
    };
    // a.prefetch: L2 bulk prefetch of the item after next as soon as it is
    // grabbed (its 4 x 8 KB of codes and pairs; a partial item's tail too)
    auto prefetch_item = [&](int it) {
        if (!a.prefetch || it >= a.n_items || lane != 0) return;
        const int pu = it / nper, pkk = it - pu * nper, pk = a.k_first + pkk;
        const int Ti = min(IT, a.body_end - pkk * IT);
        if (Ti <= 0) return;
        bulk_prefetch_l2(c.kcodes + pu * c.k_ustride + (int64_t)pk * (IT / 32) * PB::TILE_CODE,
                         (uint32_t)(Ti / 32) * PB::TILE_CODE);
        bulk_prefetch_l2(c.kpairs + pu * c.kp_ustride + (int64_t)pk * (IT / 32) * D,
                         (uint32_t)(Ti / 32) * D * 8);
        bulk_prefetch_l2(c.vcodes + pu * c.v_ustride + (int64_t)pk * IT * PB::TOK_CODE,
                         (uint32_t)Ti * PB::TOK_CODE);
        bulk_prefetch_l2(c.vpairs + pu * c.vp_ustride + (int64_t)pk * IT * (D / fast::G),
                         (uint32_t)Ti * (D / fast::G) * 8);
    };
    int f_item = grab(), f_job = 0;
    int f_ahead = grab();
    prefetch_item(f_ahead);
    // The claim of the item after f_ahead is issued with f_item's first job
    // and read (broadcast from lane 0) only when f_item's jobs are all issued:
    // the atomic's round trip overlaps a whole item instead of stalling the
    // warp at the broadcast.
    int pend = 0;
    int c_next = f_item;
    int f_u = f_item / nper, f_k = f_item - f_u * nper;
    // the item's source addresses and token count, once per item; the
    // addresses advance by a constant per job
    const uint8_t *src_kc, *src_vc;
    const float2 *src_kp, *src_vp;
    int f_ti;
    auto item_sources = [&]() {
        const int64_t kk = a.k_first + f_k;
        f_ti = min(IT, a.body_end - f_k * IT);  // item tokens (partial last item)
        src_kc = c.kcodes + f_u * c.k_ustride + kk * (IT / 32) * PB::TILE_CODE;
        src_kp = c.kpairs + f_u * c.kp_ustride + kk * (IT / 32) * D;
        src_vc = c.vcodes + f_u * c.v_ustride + kk * IT * PB::TOK_CODE;
        src_vp = c.vpairs + f_u * c.vp_ustride + kk * IT * (D / fast::G);
    };
    item_sources();
    auto issue_next = [&](int s) {
        if (f_item >= a.n_items) return;
        if (lane == 0) {
            if (KIVI_DEFER_CLAIM && f_job == 0 && f_ahead < a.n_items) pend = atomicAdd(a.work, 1);
            uint8_t* slot = wbase + s * SLOT;
            uint64_t* bar = &bars[s];
            const int Ti = f_ti;
            fence_proxy_async_smem();
            if (f_job < NKJ) {
                const int ntl = min(KT, max(0, Ti / 32 - f_job * KT));
                const uint32_t cb = (uint32_t)ntl * PB::TILE_CODE;
                const uint32_t pb = (uint32_t)ntl * D * 8;
                constexpr uint32_t qb = H * D * 4;
                mbar_arrive_expect_tx(bar, cb + pb + (f_job == 0 ? qb : 0));
                if (ntl) {
                    bulk_g2s_evict_first(slot, src_kc, cb, bar, policy);
                    bulk_g2s_evict_first(slot + KT * PB::TILE_CODE, src_kp, pb, bar, policy);
                }
                if (f_job == 0) bulk_g2s(qraw, a.q + (int64_t)f_u * H * D, qb, bar);
                src_kc += KT * PB::TILE_CODE;
                src_kp += KT * D;
            } else {
                const int ntok = min(VT, max(0, Ti - (f_job - NKJ) * VT));
                const uint32_t cb = (uint32_t)ntok * PB::TOK_CODE;
                const uint32_t pb = (uint32_t)ntok * (D / fast::G) * 8;
                mbar_arrive_expect_tx(bar, cb + pb);
                if (ntok) {
                    bulk_g2s_evict_first(slot, src_vc, cb, bar, policy);
                    bulk_g2s_evict_first(slot + VT * PB::TOK_CODE, src_vp, pb, bar, policy);
                }
                src_vc += VT * PB::TOK_CODE;
                src_vp += VT * (D / fast::G);
            }
        }
        if (++f_job == NJ) {
            f_job = 0;
            f_item = f_ahead;
            c_next = f_item;
            if (f_item < a.n_items) {
                f_ahead = KIVI_DEFER_CLAIM ? __shfl_sync(0xffffffffu, pend, 0) : grab();
                prefetch_item(f_ahead);
            }
            f_u = f_item / nper;
            f_k = f_item - f_u * nper;
            item_sources();
        }
    };
    issue_next(0);
    issue_next(1);

    uint32_t phase = 0;
    int cs = 0;
    auto wait_slot = [&]() -> uint8_t* {
        mbar_wait(&bars[cs], (phase >> cs) & 1u);
        phase ^= (1u << cs);
        return wbase + cs * SLOT;
    };
    auto release_slot = [&]() {
        __syncwarp();
        issue_next(cs);
        cs ^= 1;
    };

    for (int item = c_next; item < a.n_items; item = c_next) {
        const int u = item / nper;
        const int k = a.k_first + (item - u * nper);
        const int Ti = min(IT, a.body_end - (item - u * nper) * IT);
        float2 qv[H][2];
        float qmax = 0.f;
#pragma unroll 1
        for (int jk = 0; jk < NKJ; ++jk) {
            uint8_t* slot = wait_slot();
            if (jk == 0) {
                const float2 qs2 = make_float2(a.qscale, a.qscale);
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    // this lane's key channels: 2L, 2L+1 and 64+2L, 65+2L
                    const float2 q01 = reinterpret_cast<const float2*>(qraw + h * D)[lane];
                    const float2 q23 = reinterpret_cast<const float2*>(qraw + h * D + 64)[lane];
                    qv[h][0] = __fmul2_rn(q01, qs2);
                    qv[h][1] = __fmul2_rn(q23, qs2);
                    qmax = fmaxf(qmax, fmaxf(fmaxf(fabsf(qv[h][0].x), fabsf(qv[h][0].y)),
                                             fmaxf(fabsf(qv[h][1].x), fabsf(qv[h][1].y))));
                }
                qmax = warp_max_redux(qmax);
                __syncwarp();  // qraw is reused as the bias scratch below
            }
            const int ntl = min(KT, max(0, Ti / 32 - jk * KT));
            if (ntl) key_job<H, WS::DB>(slot, qv, qmax, probs, jk * KT * 32, bf, biasm, lane, sel, ntl);
            release_slot();
        }
        if (Ti < IT) {  // partial item: tokens past its end get zero probability
            for (int i = lane; i < (IT - Ti) * H; i += 32) {
                const int t = Ti + i / H;
                probs[pidx<H>(t, i % H)] = -INFINITY;
            }
        }
        float2 ml[H];
        softmax_heads<H, IT>(probs, a.wlog ? a.wlog + (int64_t)u * H * a.l + (int64_t)k * IT : nullptr,
                         a.l, ml, lane, Ti);
        float4 vacc[4][2];
#pragma unroll
        for (int cg = 0; cg < 4; ++cg)
#pragma unroll
            for (int m = 0; m < 2; ++m) vacc[cg][m] = make_float4(0.f, 0.f, 0.f, 0.f);
        float2 zs[H];
#pragma unroll
        for (int h = 0; h < H; ++h) zs[h] = make_float2(0.f, 0.f);
        int eb_run = 0;
#pragma unroll 1
        for (int jv = 0; jv < NVJ; ++jv) {
            uint8_t* slot = wait_slot();
            const int ntok = min(VT, max(0, Ti - jv * VT));
            if (ntok == VT)
                value_job<H, true, WS::DB>(slot, probs + jv * VT * H, vacc, zs, eb_run, jv == 0, bf, lane,
                                   sel);
            else if (ntok)
                value_job<H, false, WS::DB>(slot, probs + jv * VT * H, vacc, zs, eb_run, jv == 0, bf, lane,
                                    sel, ntok);
            if (jv == NVJ - 1) {
                const int64_t pi = ((int64_t)u * a.n_sub + k) * H;
                value_finalize<H>(vacc, zs, eb_run, ml, zsm, a.part_o + pi * D, a.part_ml + pi, lane);
            }
            release_slot();
        }
    }
}

}  // namespace gqa_tc
}  // namespace kivi_b200
