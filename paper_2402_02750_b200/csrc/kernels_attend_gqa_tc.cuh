// Grouped-query fused dequant-attention decode on the tensor cores
// (mma.sync m16n8k16, fp16 operands, fp32 accumulation).  H = 2 or 4 query
// heads share one kv unit (BASELINE config 3: Mistral-7B, H = 4); B = 2,
// d = 128, G = 32.  Body items only (whole 256-token sub-chunks whose keys
// and values are all quantized); items holding fp32 residual rows run on the
// CUDA-core kernel (kernels_attend_gqa.cuh) concurrently.
//
// Why tensor cores here and not for MHA: with H heads every code feeds H
// multiply-adds.  On CUDA cores that is 1 LOP3 + H/2 FFMA2 per code (3 issue
// slots at H = 4); the MMA does the H-way (and the 16-deep) reduction in one
// instruction per 256 codes, leaving ~1 ALU op per code for the extraction.
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
//       g >> 2), i.e. tokens 4g..4g+3 of its 4 channels 16s + 4t + {0..3};
//       one PRMT pairs channels (c, c+1) into the two fp16 halves and a
//       LOP3 (after one shared shift) per token position j selects the code:
//       row g <-> token 4g + 2m, row g+8 <-> 4g + 2m + 1 in MMA m (m = 0, 1).
//   B = split(q'_h[c] * s_T[c] * 2^E), built cooperatively per tile (lane L
//       computes the 16 products of channels 4L..4L+3) and stored in fragment
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
using fast::SLOT;
using fast::SUB;
constexpr int WARPS = 4;
constexpr int BFK_ROW = 9;        // uint2 per consumer lane in the key B buffer (8 K steps + pad)
constexpr int BFV_CG = 72;        // 32-bit words per channel group in the value B buffer (64 + pad)
constexpr int BIAS_ROW = 17;      // floats per lane row of the key-bias transpose
constexpr uint32_t FULL = 0xffffffffu;

template <int H>
struct TS {  // per-warp shared memory
    static constexpr int QRAW_OFF = 2 * SLOT;                  // [H][128] staged q rows
    static constexpr int PROBS_OFF = QRAW_OFF + H * D * 4;     // [256][H] logits -> p
    static constexpr int BF_OFF = PROBS_OFF + SUB * H * 4;     // B fragments (keys | values)
    static constexpr int BF_BYTES = 32 * BFK_ROW * 8;          // 2304 = 2 x 4 x 72 x 4
    static constexpr int BIAS_OFF = BF_OFF + BF_BYTES;         // [32][17] key-bias partials
    static constexpr int ZS_OFF = BIAS_OFF + 32 * BIAS_ROW * 4;  // [H][4] value z sums
    static constexpr int BAR_OFF = ZS_OFF + 16 * 4;
    static constexpr int BYTES = BAR_OFF + 16;
    static constexpr int STRIDE = (BYTES + 127) & ~127;
    static_assert(2 * 4 * BFV_CG * 4 <= BF_BYTES, "value B buffers overflow");
};

__device__ __forceinline__ void mma_f16(float4& d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d.x), "+f"(d.y), "+f"(d.z), "+f"(d.w)
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// (x0, x1) -> fp16x2 words (hi, lo) with x = hi + lo to ~2^-21 relative.
__device__ __forceinline__ void split_pair(float x0, float x1, uint32_t& whi, uint32_t& wlo) {
    const float h0 = __uint_as_float(__float_as_uint(x0) & 0xFFFFE000u);
    const float h1 = __uint_as_float(__float_as_uint(x1) & 0xFFFFE000u);
    __half2 hh = __floats2half2_rn(h0, h1);
    __half2 ll = __floats2half2_rn(x0 - h0, x1 - h1);
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

// -------------------------------------------------------------------------
// One key job: 4 tiles (codes [4][1024 B], pairs [4][128] (lo, hi)) -> the
// log2-domain logits of 128 tokens x H heads at probs_dst[token * H + h].
// -------------------------------------------------------------------------
template <int H>
__device__ __forceinline__ void key_job(const uint8_t* slot, const float (&qv)[H][4], float qmax,
                                        float* probs_dst, uint8_t* bf, float* biasm, int lane,
                                        uint32_t sel) {
    const int g = lane >> 2, t = lane & 3;
    const float4* pairs4 = reinterpret_cast<const float4*>(slot + 4 * 1024);
    // pre-pass over this lane's channels 4L..4L+3 of the 4 tiles: spans,
    // bias partials, job-wide span maximum
    float dmax = 0.f;
#pragma unroll
    for (int T = 0; T < 4; ++T) {
        const float4 p01 = pairs4[T * 64 + 2 * lane];
        const float4 p23 = pairs4[T * 64 + 2 * lane + 1];
        const float lo[4] = {p01.x, p01.z, p23.x, p23.z};
        dmax = fmaxf(dmax, fmaxf(fmaxf(p01.y - p01.x, p01.w - p01.z),
                                 fmaxf(p23.y - p23.x, p23.w - p23.z)));
#pragma unroll
        for (int h = 0; h < H; ++h) {
            float b = qv[h][0] * lo[0];
            b = fmaf(qv[h][1], lo[1], b);
            b = fmaf(qv[h][2], lo[2], b);
            b = fmaf(qv[h][3], lo[3], b);
            biasm[lane * BIAS_ROW + T * H + h] = b;
        }
    }
    dmax = warp_max(dmax);
    const int eb = exp_byte(qmax * dmax * (1.0f / 3.0f));
    const float f = scale_up(eb) * (1.0f / 3.0f);
    __syncwarp();
    // bias column sums: lane L sums column L & 15 over 16 rows, then xor 16
    float bs = 0.f;
    {
        const int col = lane & 15, r0 = (lane >> 4) * 16;
#pragma unroll
        for (int r = 0; r < 16; ++r) bs += biasm[(r0 + r) * BIAS_ROW + col];
        bs += __shfl_xor_sync(FULL, bs, 16);
    }
    uint2* bfk = reinterpret_cast<uint2*>(bf);
    const int s_p = lane >> 2, t_p = lane & 3;  // producer -> consumer K step / lane slot
#pragma unroll 1
    for (int T = 0; T < 4; ++T) {
        // ---- producer: B fragments of tile T ----
        const float4 p01 = pairs4[T * 64 + 2 * lane];
        const float4 p23 = pairs4[T * 64 + 2 * lane + 1];
        const float d0 = (p01.y - p01.x) * f, d1 = (p01.w - p01.z) * f;
        const float d2 = (p23.y - p23.x) * f, d3 = (p23.w - p23.z) * f;
#pragma unroll
        for (int h = 0; h < H; ++h) {
            uint32_t hi01, lo01, hi23, lo23;
            split_pair(qv[h][0] * d0, qv[h][1] * d1, hi01, lo01);
            split_pair(qv[h][2] * d2, qv[h][3] * d3, hi23, lo23);
            bfk[((2 * h) * 4 + t_p) * BFK_ROW + s_p] = make_uint2(hi01, hi23);
            bfk[((2 * h + 1) * 4 + t_p) * BFK_ROW + s_p] = make_uint2(lo01, lo23);
        }
        __syncwarp();
        // ---- consumer: 8 K steps x 2 MMAs ----
        float4 acc0 = make_float4(0.f, 0.f, 0.f, 0.f), acc1 = acc0;
        const uint8_t* ct = slot + T * 1024 + 4 * (g >> 2);
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const int cb = (16 * s + 4 * t) * 8;
            const uint32_t w0 = *reinterpret_cast<const uint32_t*>(ct + cb);
            const uint32_t w1 = *reinterpret_cast<const uint32_t*>(ct + cb + 8);
            const uint32_t w2 = *reinterpret_cast<const uint32_t*>(ct + cb + 16);
            const uint32_t w3 = *reinterpret_cast<const uint32_t*>(ct + cb + 24);
            const CodeQuad c01 = code_quad(__byte_perm(w0, w1, sel));
            const CodeQuad c23 = code_quad(__byte_perm(w2, w3, sel));
            uint2 b = make_uint2(0u, 0u);
            if (g < 2 * H) b = bfk[lane * BFK_ROW + s];
            mma_f16(acc0, c01.c[0], c01.c[1], c23.c[0], c23.c[1], b.x, b.y);
            mma_f16(acc1, c01.c[2], c01.c[3], c23.c[2], c23.c[3], b.x, b.y);
        }
        const float bias = __shfl_sync(FULL, bs, (T * H + t) & 15);
        __syncwarp();  // the next tile's producer overwrites bfk
        if (t < H) {
            float* dst = probs_dst + (T * 32 + 4 * g) * H + t;
            dst[0 * H] = fmaf(acc0.x + acc0.y, unscale(eb, code_pos(0)), bias);
            dst[1 * H] = fmaf(acc0.z + acc0.w, unscale(eb, code_pos(1)), bias);
            dst[2 * H] = fmaf(acc1.x + acc1.y, unscale(eb, code_pos(2)), bias);
            dst[3 * H] = fmaf(acc1.z + acc1.w, unscale(eb, code_pos(3)), bias);
        }
    }
}

// Softmax of each head over the item's 256 tokens (probs [token][H], in
// place, log2 domain) -> p in (0, 1]; ml[h] = (max, sum).
template <int H>
__device__ __forceinline__ void softmax_heads(float* probs, float* wlog, int64_t wstride, float2* ml,
                                              int lane) {
    __syncwarp();
    float v[8][H];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float* src = probs + (lane + 32 * i) * H;
        if constexpr (H == 4) {
            const float4 x = *reinterpret_cast<const float4*>(src);
            v[i][0] = x.x; v[i][1] = x.y; v[i][2] = x.z; v[i][3] = x.w;
        } else {
            const float2 x = *reinterpret_cast<const float2*>(src);
            v[i][0] = x.x; v[i][1] = x.y;
        }
    }
    float m[H], sm[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
        m[h] = v[0][h];
#pragma unroll
        for (int i = 1; i < 8; ++i) m[h] = fmaxf(m[h], v[i][h]);
        m[h] = warp_max(m[h]);
        sm[h] = 0.f;
    }
    if (wlog) {
#pragma unroll
        for (int h = 0; h < H; ++h)
#pragma unroll
            for (int i = 0; i < 8; ++i) wlog[h * wstride + lane + 32 * i] = v[i][h];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#pragma unroll
        for (int h = 0; h < H; ++h) {
            v[i][h] = fast::ex2_approx(v[i][h] - m[h]);
            sm[h] += v[i][h];
        }
        float* dst = probs + (lane + 32 * i) * H;
        if constexpr (H == 4)
            *reinterpret_cast<float4*>(dst) = make_float4(v[i][0], v[i][1], v[i][2], v[i][3]);
        else
            *reinterpret_cast<float2*>(dst) = make_float2(v[i][0], v[i][1]);
    }
#pragma unroll
    for (int h = 0; h < H; ++h) ml[h] = make_float2(m[h], warp_sum(sm[h]));
    __syncwarp();
}

// -------------------------------------------------------------------------
// One value job: 128 tokens (codes [128][32 B], pairs [128][4] (lo, hi)),
// probabilities p_src[token * H + h] -> vacc[cg][m], zs[h] (this lane's
// share of sum_t p_h[t] z[t][cg = lane & 3]).  eb_run is the running
// exponent byte (the larger of all jobs so far: smaller 2^E).
// -------------------------------------------------------------------------
template <int H>
__device__ __forceinline__ void value_job(const uint8_t* slot, const float* p_src, float4 (&vacc)[4][2],
                                          float (&zs)[H], int& eb_run, bool first, uint8_t* bf,
                                          int lane, uint32_t sel) {
    const int g = lane >> 2, t = lane & 3;
    const float4* pairs4 = reinterpret_cast<const float4*>(slot + 4096);
    const float2* pairs2 = reinterpret_cast<const float2*>(slot + 4096);
    float dmax = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float4 pr = pairs4[lane + 32 * i];
        dmax = fmaxf(dmax, fmaxf(pr.y - pr.x, pr.w - pr.z));
    }
    dmax = warp_max(dmax);
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
#pragma unroll 1
    for (int s = 0; s < 8; ++s) {
        uint32_t* bv = reinterpret_cast<uint32_t*>(bf) + (s & 1) * (4 * BFV_CG);
        // ---- producer: B fragments of K step s ----
        {
            const int ta = 16 * s + toff, tb = ta + 4;
            const float2 pa = pairs2[ta * 4 + cgp], pb = pairs2[tb * 4 + cgp];
            const float da = (pa.y - pa.x) * f, db = (pb.y - pb.x) * f;
            float Pa[H], Pb[H];
            if constexpr (H == 4) {
                const float4 xa = *reinterpret_cast<const float4*>(p_src + ta * 4);
                const float4 xb = *reinterpret_cast<const float4*>(p_src + tb * 4);
                Pa[0] = xa.x; Pa[1] = xa.y; Pa[2] = xa.z; Pa[3] = xa.w;
                Pb[0] = xb.x; Pb[1] = xb.y; Pb[2] = xb.z; Pb[3] = xb.w;
            } else {
                const float2 xa = *reinterpret_cast<const float2*>(p_src + ta * 2);
                const float2 xb = *reinterpret_cast<const float2*>(p_src + tb * 2);
                Pa[0] = xa.x; Pa[1] = xa.y;
                Pb[0] = xb.x; Pb[1] = xb.y;
            }
#pragma unroll
            for (int h = 0; h < H; ++h) {
                uint32_t whi, wlo;
                split_pair(Pa[h] * da, Pb[h] * db, whi, wlo);
                zs[h] = fmaf(Pa[h], pa.x, fmaf(Pb[h], pb.x, zs[h]));
                bv[cgp * BFV_CG + 2 * ((2 * h) * 4 + tcons) + which] = whi;
                bv[cgp * BFV_CG + 2 * ((2 * h + 1) * 4 + tcons) + which] = wlo;
            }
        }
        __syncwarp();
        // ---- consumer: 4 channel groups x 2 MMAs ----
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
            mma_f16(vacc[cg][0], c01.c[0], c01.c[1], c23.c[0], c23.c[1], b.x, b.y);
            mma_f16(vacc[cg][1], c01.c[2], c01.c[3], c23.c[2], c23.c[3], b.x, b.y);
        }
    }
}

// Write the item's H partials: lane (g, t) owns head t, channels
// 32cg + 4g + {0..3}.
template <int H>
__device__ __forceinline__ void value_finalize(const float4 (&vacc)[4][2], float (&zs)[H], int eb,
                                               const float2* ml, float* zsm, float* part_o,
                                               float2* part_ml, int lane) {
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int h = 0; h < H; ++h) {
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
// Body kernel: persistent warps take items (unit, fully quantized 256-token
// sub-chunk) from an atomic counter; 2 key jobs + 2 value jobs per item,
// streamed through two TMA slots per warp (as fast::attend_body_kernel).
// -------------------------------------------------------------------------
template <int H>
__global__ void __launch_bounds__(WARPS * 32, 2) attend_gqa_tc_kernel(fast::FastArgs a) {
    using WS = TS<H>;
    using PB = fast::P<2>;
    constexpr int NKJ = 2, NVJ = 2, NJ = 4;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* wbase = smem_raw + warp * WS::STRIDE;
    float* qraw = reinterpret_cast<float*>(wbase + WS::QRAW_OFF);
    float* probs = reinterpret_cast<float*>(wbase + WS::PROBS_OFF);
    uint8_t* bf = wbase + WS::BF_OFF;
    float* biasm = reinterpret_cast<float*>(wbase + WS::BIAS_OFF);
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

    auto grab = [&]() -> int {
        int v = 0;
        if (lane == 0) v = atomicAdd(a.work, 1);
        return __shfl_sync(FULL, v, 0);
    };
    int f_item = grab(), f_job = 0;
    int f_ahead = grab();
    int c_next = f_item;
    int f_u = f_item / nper, f_k = f_item - f_u * nper;
    auto issue_next = [&](int s) {
        if (f_item >= a.n_items) return;
        if (lane == 0) {
            uint8_t* slot = wbase + s * SLOT;
            uint64_t* bar = &bars[s];
            const int kk = a.k_first + f_k;
            fence_proxy_async_smem();
            if (f_job < NKJ) {
                const int64_t tile0 = (int64_t)kk * (SUB / 32) + f_job * PB::KQ_TILES;
                constexpr uint32_t cb = PB::KQ_TILES * PB::TILE_CODE;
                constexpr uint32_t pb = PB::KQ_TILES * D * 8;
                constexpr uint32_t qb = H * D * 4;
                mbar_arrive_expect_tx(bar, cb + pb + (f_job == 0 ? qb : 0));
                bulk_g2s_evict_first(slot, c.kcodes + f_u * c.k_ustride + tile0 * PB::TILE_CODE, cb,
                                     bar, policy);
                bulk_g2s_evict_first(slot + cb, c.kpairs + f_u * c.kp_ustride + tile0 * D, pb, bar,
                                     policy);
                if (f_job == 0) bulk_g2s(qraw, a.q + (int64_t)f_u * H * D, qb, bar);
            } else {
                const int64_t ts = (int64_t)kk * SUB + (f_job - NKJ) * PB::VQ_TOK;
                constexpr uint32_t cb = PB::VQ_TOK * PB::TOK_CODE;
                constexpr uint32_t pb = PB::VQ_TOK * (D / fast::G) * 8;
                mbar_arrive_expect_tx(bar, cb + pb);
                bulk_g2s_evict_first(slot, c.vcodes + f_u * c.v_ustride + ts * PB::TOK_CODE, cb, bar,
                                     policy);
                bulk_g2s_evict_first(slot + cb, c.vpairs + f_u * c.vp_ustride + ts * (D / fast::G),
                                     pb, bar, policy);
            }
        }
        if (++f_job == NJ) {
            f_job = 0;
            f_item = f_ahead;
            c_next = f_item;
            if (f_item < a.n_items) f_ahead = grab();
            f_u = f_item / nper;
            f_k = f_item - f_u * nper;
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
        float qv[H][4];
        float qmax = 0.f;
#pragma unroll 1
        for (int jk = 0; jk < NKJ; ++jk) {
            uint8_t* slot = wait_slot();
            if (jk == 0) {
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    const float4 q4 = reinterpret_cast<const float4*>(qraw + h * D)[lane];
                    qv[h][0] = q4.x * a.qscale;
                    qv[h][1] = q4.y * a.qscale;
                    qv[h][2] = q4.z * a.qscale;
                    qv[h][3] = q4.w * a.qscale;
#pragma unroll
                    for (int i = 0; i < 4; ++i) qmax = fmaxf(qmax, fabsf(qv[h][i]));
                }
                qmax = warp_max(qmax);
            }
            key_job<H>(slot, qv, qmax, probs + jk * 128 * H, bf, biasm, lane, sel);
            release_slot();
        }
        float2 ml[H];
        softmax_heads<H>(probs, a.wlog ? a.wlog + (int64_t)u * H * a.l + (int64_t)k * SUB : nullptr,
                         a.l, ml, lane);
        float4 vacc[4][2];
#pragma unroll
        for (int cg = 0; cg < 4; ++cg)
#pragma unroll
            for (int m = 0; m < 2; ++m) vacc[cg][m] = make_float4(0.f, 0.f, 0.f, 0.f);
        float zs[H];
#pragma unroll
        for (int h = 0; h < H; ++h) zs[h] = 0.f;
        int eb_run = 0;
#pragma unroll 1
        for (int jv = 0; jv < NVJ; ++jv) {
            uint8_t* slot = wait_slot();
            value_job<H>(slot, probs + jv * 128 * H, vacc, zs, eb_run, jv == 0, bf, lane, sel);
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
