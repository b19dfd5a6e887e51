// Fast fused dequant-attention decode for the headline shape family
// (d = 128, G = 32, B in {2, 4}, one query head per kv unit).
//
// Work decomposition:
//   item  = (unit, 256-token sub-chunk); a persistent grid of warps walks the
//           item list, each warp owning its items end to end (logits ->
//           softmax -> P.V) and writing one partial (m, L, o[128]) per item;
//           K5 (combine_kernel) merges partials with an LSE rescale.
//   job   = <= 8 KB of one kind of data for one item: quantized key tiles
//           (KQ), fp32 key residual rows (KF), quantized value tokens (VQ),
//           fp32 value residual rows (VF).  Each warp streams its jobs through
//           NSLOT shared-memory slots filled by cp.async.bulk (TMA 1-D) with
//           one mbarrier per slot, so the next jobs are in flight while the
//           current one is computed.  The item's query row rides along with
//           its first job.
//
// Arithmetic (exact dequantisation, fp32 accumulation):
//   key logit  t = sum_c q_c (code*s_c + z_c) = sum_c (q_c s_c) code + sum_c q_c z_c
//   value out  c = sum_t p_t (code*s_t + z_t) = sum_t (p_t s_t) code + sum_t p_t z_t
// A B-bit code at bit position e of a word is read as the fp32 DENORMAL whose
// bits are (word & (mask << e)), i.e. code * 2^(e-149), exactly.  The
// per-group multiplier carries 2^64 so products land in the normal range,
// and each accumulator (one per token for keys, per channel for values) has a
// fixed position e, undone once at the end.  So each code costs one LOP3 and
// half an FFMA2 — no shifts, no int->float conversion.
#pragma once

#include "common.cuh"
#include "kernels_quant.cuh"
#include "kernels_vimma.cuh"

namespace kivi_b200 {
namespace fast {

constexpr int D = 128;
constexpr int G = 32;
constexpr int SUB = 256;       // tokens per item (tail / GQA items; max tail item)
// Tokens per MHA body item.  512 measured: body 3.5 % faster per token, but
// the residual-window region (tail items) grows by 256 tokens per unit and
// the launch got slower (C2 266 vs 247 us), so 256.
#ifndef KIVI_MHA_BSUB
#define KIVI_MHA_BSUB 256
#endif
constexpr int BSUB = KIVI_MHA_BSUB;
constexpr int WARPS = 4;       // warps per CTA
constexpr int SLOT = 8192;     // bytes per pipeline slot
constexpr int F_ROWS = 16;     // fp32 residual rows per job (16 * 512 B)
constexpr float TWO_POW_64 = 18446744073709551616.0f;
constexpr float LOG2E = 1.4426950408889634f;

#define KIVI_F(x) __uint_as_float(x)

// Unroll factor of the key-tile loop (8 iterations).  Full unrolling costs
// ~14 KB of SASS; see DESIGN.md for the measured trade-off.
#ifndef KIVI_KQ_UNROLL
#define KIVI_KQ_UNROLL 2
#endif
constexpr int KQ_UNROLL = KIVI_KQ_UNROLL;

// w >> K on the FMA pipe (IMAD.HI) instead of the ALU pipe (SHF): the body
// kernel is ALU-bound on the code extraction, the FMA pipe has headroom.
#ifndef KIVI_COMBINE_UNROLL
#define KIVI_COMBINE_UNROLL 8
#endif
constexpr int COMBINE_UNROLL = KIVI_COMBINE_UNROLL;  // K5 partial loop (x2 loads)
#ifndef KIVI_VQ_UNROLL
#define KIVI_VQ_UNROLL 1
#endif
#ifndef KIVI_SHR_FMA
#define KIVI_SHR_FMA 1
#endif
template <int K>
__device__ __forceinline__ uint32_t shr_fma(uint32_t w) {
#if KIVI_SHR_FMA
    uint32_t r;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(w), "r"(1u << (32 - K)));
    return r;
#else
    return w >> K;
#endif
}
template <int B>
struct P;
template <>
struct P<2> {
    static constexpr int CB = 8;                // bytes per (tile, channel)
    static constexpr int TILE_CODE = D * CB;    // 1024
    static constexpr int KQ_TILES = 4;          // tiles per KQ job (4 KB codes + 4 KB pairs)
    static constexpr int LPT = 8;               // lanes per key tile
    static constexpr int TOK_CODE = D * 2 / 8;  // 32 bytes of codes per token
    static constexpr int VQ_TOK = 128;          // tokens per VQ job (4 KB codes + 4 KB pairs)
    static constexpr int TPW = 16;              // codes per 32-bit word
    // denormal bit position of code k of a word (after the one shift below)
    static __host__ __device__ constexpr int epos(int k) { return k <= 10 ? 2 * k : 2 * k - 10; }
    // acc[0..7] (+)= M * codes of w (codes 2j, 2j+1 in acc[j])
    static __device__ __forceinline__ void fma_word(float2* acc, uint32_t w, float M) {
        const float2 m2 = make_float2(M, M);
        const uint32_t s = shr_fma<10>(w);
        acc[0] = __ffma2_rn(m2, make_float2(KIVI_F(w & 0x3u), KIVI_F(w & 0xCu)), acc[0]);
        acc[1] = __ffma2_rn(m2, make_float2(KIVI_F(w & 0x30u), KIVI_F(w & 0xC0u)), acc[1]);
        acc[2] = __ffma2_rn(m2, make_float2(KIVI_F(w & 0x300u), KIVI_F(w & 0xC00u)), acc[2]);
        acc[3] = __ffma2_rn(m2, make_float2(KIVI_F(w & 0x3000u), KIVI_F(w & 0xC000u)), acc[3]);
        acc[4] = __ffma2_rn(m2, make_float2(KIVI_F(w & 0x30000u), KIVI_F(w & 0xC0000u)), acc[4]);
        acc[5] = __ffma2_rn(m2, make_float2(KIVI_F(w & 0x300000u), KIVI_F(s & 0x3000u)), acc[5]);
        acc[6] = __ffma2_rn(m2, make_float2(KIVI_F(s & 0xC000u), KIVI_F(s & 0x30000u)), acc[6]);
        acc[7] = __ffma2_rn(m2, make_float2(KIVI_F(s & 0xC0000u), KIVI_F(s & 0x300000u)), acc[7]);
    }
};
template <>
struct P<4> {
    static constexpr int CB = 16;
    static constexpr int TILE_CODE = D * CB;    // 2048
    static constexpr int KQ_TILES = 2;          // 4 KB codes + 2 KB pairs
    static constexpr int LPT = 16;
    static constexpr int TOK_CODE = D * 4 / 8;  // 64
    static constexpr int VQ_TOK = 64;           // 4 KB codes + 2 KB pairs
    static constexpr int TPW = 8;
    static __host__ __device__ constexpr int epos(int k) { return k <= 4 ? 4 * k : 4 * k - 12; }
    static __device__ __forceinline__ void fma_word(float2* acc, uint32_t w, float M) {
        const float2 m2 = make_float2(M, M);
        const uint32_t s = shr_fma<12>(w);
        acc[0] = __ffma2_rn(m2, make_float2(KIVI_F(w & 0xFu), KIVI_F(w & 0xF0u)), acc[0]);
        acc[1] = __ffma2_rn(m2, make_float2(KIVI_F(w & 0xF00u), KIVI_F(w & 0xF000u)), acc[1]);
        acc[2] = __ffma2_rn(m2, make_float2(KIVI_F(w & 0xF0000u), KIVI_F(s & 0xF00u)), acc[2]);
        acc[3] = __ffma2_rn(m2, make_float2(KIVI_F(s & 0xF000u), KIVI_F(s & 0xF0000u)), acc[3]);
    }
};

// 2^(149 - 64 - e): undoes the denormal position e and the 2^64 multiplier.
__device__ __forceinline__ float unscale_pos(int e) {
    return __int_as_float((127 + 149 - 64 - e) << 23);
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct FastArgs {
    CacheDev c;
    int l, kg, vg;
    int n_sub;          // partial slots per unit
    int k_first;        // first partial slot (sub-chunk index) of this launch
    int t_first;        // first token of this launch's items
    int sub;            // tokens per item of this launch (plan_item)
    int n_per_unit;     // sub-chunks per unit handled by this launch
    int n_items;        // n_units * n_per_unit
    const float* q;     // [units][128]
    float qscale;       // logit scale * log2(e)
    float* part_o;      // [units][n_sub][128]
    float2* part_ml;    // [units][n_sub]   (max, sum) in log2 domain
    float* wlog;        // [units][l] log2-domain logits, or null
    int* work;          // body kernel: dynamic item counter (zero at launch)
    int* work_clear;    // body kernel: a later launch's counter, zeroed here
    int prefetch;       // tail kernel: L2-prefetch each item's fp32 rows
    int tail_last;      // one-stream order body -> tail (tail needs only the append,
                        // which finished before the body started)
    // tail kernel, two item sizes per unit (few-unit route): items
    // [0, n_a) are `sub` tokens from t_first up to t_b, items [n_a, n_per_unit)
    // are sub_b tokens from t_b (the residual window's fp32 rows in short
    // items, so no item is a long chain of dependent row jobs).  sub_b = 0:
    // uniform items.
    int sub_b, n_a, t_b;
    int body_end;       // tensor-core GQA body: tokens it covers (multiple of 32;
                        // its last item per unit may be partial)
    // fused append (tail kernel only): when l_app >= 0 the tail kernel first
    // appends token rows tk/tv [units][128] to each unit it owns (the cache
    // held l_app tokens), then streams that unit's items.
    const float* tk;
    const float* tv;
    int l_app;
    // single-launch decode (few units, tail kernel only; gbar != null): every
    // warp < n_units appends its unit, a grid-wide counter barrier (cooperative
    // launch: all CTAs resident) orders the appends before any item, and the
    // warp that writes a unit's last partial merges the unit (combine_kernel's
    // arithmetic).  Counters are cumulative over launches: targets are passed.
    unsigned long long* gbar;
    unsigned long long gbar_target;
    unsigned int* unit_done;
    unsigned int unit_target;
    float* out;
    float2* stats;
};

// Merge unit u's n_sub partials (LSE rescale, log2 domain) by one warp: lane
// owns channels 4*lane .. 4*lane+3.  Same arithmetic as combine_kernel.  The
// partial weights are computed once by their owner lane (k mod 32) and
// broadcast; the partial loads are independent and unrolled so they overlap.
__device__ __forceinline__ void combine_unit_warp(const float* __restrict__ part_o,
                                                  const float2* __restrict__ part_ml, int n_sub,
                                                  int64_t u, float* __restrict__ out,
                                                  float2* __restrict__ stats, int lane) {
    const float2* ml = part_ml + u * n_sub;
    const float4* po = reinterpret_cast<const float4*>(part_o + u * n_sub * D) + lane;
    float M = -INFINITY;
    for (int k = lane; k < n_sub; k += 32) M = fmaxf(M, __ldcg(&ml[k]).x);
    M = warp_max_redux(M);
    float L = 0.f;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k0 = 0; k0 < n_sub; k0 += 32) {
        float w = 0.f;
        if (k0 + lane < n_sub) {
            const float2 m = __ldcg(&ml[k0 + lane]);
            w = exp2f(m.x - M);
            L = fmaf(m.y, w, L);
        }
        const int nk = min(32, n_sub - k0);
#pragma unroll 8
        for (int i = 0; i < nk; ++i) {
            const float wi = __shfl_sync(0xffffffffu, w, i);
            const float4 p = __ldcg(po + (int64_t)(k0 + i) * (D / 4));
            o.x = fmaf(p.x, wi, o.x);
            o.y = fmaf(p.y, wi, o.y);
            o.z = fmaf(p.z, wi, o.z);
            o.w = fmaf(p.w, wi, o.w);
        }
    }
    L = warp_sum(L);
    reinterpret_cast<float4*>(out + u * D)[lane] = make_float4(o.x / L, o.y / L, o.z / L, o.w / L);
    if (stats && lane == 0) stats[u] = make_float2(M, L);
}

// Per-warp shared memory.  One q staging buffer suffices for NSLOT == 2: the
// next item's first job is issued only after the current item's job 0 (which
// consumes the staged q) has been computed, since every item has >= 2 jobs.
template <int NSLOT>
struct WarpSmem {
    static_assert(NSLOT == 2, "q staging assumes two slots");
    static constexpr int QRAW_OFF = NSLOT * SLOT;            // 128 fp32 (staged q)
    static constexpr int QQ_OFF = QRAW_OFF + D * 4;          // 128 fp32 (q * scale * log2e)
    static constexpr int PROBS_OFF = QQ_OFF + D * 4;         // SUB fp32
    static constexpr int BAR_OFF = PROBS_OFF + SUB * 4;
    static constexpr int BYTES = BAR_OFF + 8 * NSLOT;
    static constexpr int STRIDE = (BYTES + 127) & ~127;
};
using WS2 = WarpSmem<2>;

// Body kernel layout: BSUB probabilities, and the staged q row aliased onto
// the first 128 of them.  Safe because the next item's first job (which
// carries q) is issued when the second-to-last value job is released; by
// then only the last value job still reads p, and it reads tokens
// >= BSUB - VQ_TOK >= 128 (NVJ >= 2).  Keeps 3 CTAs x 4 warps per SM.
// (VI, the tensor-core value jobs, keeps their B digits in the job's slot.)
template <bool VI = false, int BS = BSUB>
struct WarpSmemBody {
    static constexpr int QQ_OFF = 2 * SLOT;
    static constexpr int PROBS_OFF = QQ_OFF + D * 4;
    static constexpr int QRAW_OFF = PROBS_OFF;
    static constexpr int BAR_OFF = PROBS_OFF + BS * 4;
    static constexpr int BYTES = BAR_OFF + 16;
    static constexpr int STRIDE = (BYTES + 127) & ~127;
};
using WSB = WarpSmemBody<false>;

// ===================== shared compute bodies ===============================

// q row (staged by TMA) -> q * scale * log2(e) table.
// The table holds (q * qscale) * ksc: the key loops' per-channel multiplier
// (q s ksc) is then one multiply, and the logits' bias / fp32-row dots are
// scaled back by 1 / ksc once per token.
__device__ __forceinline__ void load_q_table(const float* qraw, float* qq, float qscale, float ksc,
                                             int lane) {
    const float4 qv = reinterpret_cast<const float4*>(qraw)[lane];
    reinterpret_cast<float4*>(qq)[lane] =
        make_float4((qv.x * qscale) * ksc, (qv.y * qscale) * ksc, (qv.z * qscale) * ksc,
                    (qv.w * qscale) * ksc);
    __syncwarp();
}

// Quantized key tiles -> logits.  The slot holds KQ_TILES tiles of codes
// followed by KQ_TILES tiles of (lo, hi) pairs; lanes split as (tile, channel
// slice); the 32 per-token partials are transpose-reduced through the slot.
// Writes the logits of tiles [0, ntiles) to probs_dst[tile * 32 + token].
template <int B>
__device__ __forceinline__ void kq_tiles_to_logits(uint8_t* slot, const float* qq, float* probs_dst,
                                                   int ntiles, float ksc, int lane) {
    using PB = P<B>;
    const int tl = lane / PB::LPT;  // tile within job
    const int b = lane % PB::LPT;
    float2 acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = make_float2(0.f, 0.f);
    float bias = 0.f;
    if (tl < ntiles) {
        const uint8_t* codes = slot + tl * PB::TILE_CODE;
        const uint8_t* pairs = slot + PB::KQ_TILES * PB::TILE_CODE + tl * D * 8;
        if constexpr (B == 2) {
            // software-pipelined: the loads of iteration it+1 are issued
            // before the 64 LOP3 + 32 FFMA2 of iteration it
            uint4 cw = *reinterpret_cast<const uint4*>(codes + b * 16);
            float4 pr = *reinterpret_cast<const float4*>(pairs + b * 16);
            float2 qv = *reinterpret_cast<const float2*>(qq + 2 * b);
#pragma unroll KQ_UNROLL
            for (int it = 0; it < 8; ++it) {
                uint4 cw_n = cw;
                float4 pr_n = pr;
                float2 qv_n = qv;
                if (it < 7) {
                    const int ci = (it + 1) * PB::LPT + b;
                    cw_n = *reinterpret_cast<const uint4*>(codes + ci * 16);
                    pr_n = *reinterpret_cast<const float4*>(pairs + ci * 16);
                    qv_n = *reinterpret_cast<const float2*>(qq + 2 * ci);
                }
                const float m0 = qv.x * (pr.y - pr.x);
                const float m1 = qv.y * (pr.w - pr.z);
                bias = fmaf(qv.x, pr.x, bias);
                bias = fmaf(qv.y, pr.z, bias);
                PB::fma_word(acc, cw.x, m0);
                PB::fma_word(acc + 8, cw.y, m0);
                PB::fma_word(acc, cw.z, m1);
                PB::fma_word(acc + 8, cw.w, m1);
                cw = cw_n;
                pr = pr_n;
                qv = qv_n;
            }
        } else {
#pragma unroll
            for (int it = 0; it < 8; ++it) {
                const int ci = it * PB::LPT + b;
                const uint4 cw = *reinterpret_cast<const uint4*>(codes + ci * 16);
                const float2 pr = *reinterpret_cast<const float2*>(pairs + ci * 8);
                const float qv = qq[ci];
                const float m0 = qv * (pr.y - pr.x);
                bias = fmaf(qv, pr.x, bias);
                PB::fma_word(acc, cw.x, m0);
                PB::fma_word(acc + 4, cw.y, m0);
                PB::fma_word(acc + 8, cw.z, m0);
                PB::fma_word(acc + 12, cw.w, m0);
            }
        }
    }
#pragma unroll
    for (int o = 1; o < PB::LPT; o <<= 1) bias += __shfl_xor_sync(0xffffffffu, bias, o);
    __syncwarp();
    float* red = reinterpret_cast<float*>(slot);
    {
        float4* row = reinterpret_cast<float4*>(red + lane * 36);
#pragma unroll
        for (int i = 0; i < 8; ++i)
            row[i] = make_float4(acc[2 * i].x, acc[2 * i].y, acc[2 * i + 1].x, acc[2 * i + 1].y);
    }
    __syncwarp();
    constexpr int TPL = 32 / PB::LPT;  // tokens per lane after the reduce
    float sum[TPL];
#pragma unroll
    for (int i = 0; i < TPL; ++i) sum[i] = 0.f;
#pragma unroll
    for (int bb = 0; bb < PB::LPT; ++bb) {
        const float* src = red + (tl * PB::LPT + bb) * 36 + TPL * b;
        if constexpr (TPL == 4) {
            const float4 v = *reinterpret_cast<const float4*>(src);
            sum[0] += v.x; sum[1] += v.y; sum[2] += v.z; sum[3] += v.w;
        } else {
            const float2 v = *reinterpret_cast<const float2*>(src);
            sum[0] += v.x; sum[1] += v.y;
        }
    }
    if (tl < ntiles) {
        float lg[TPL];
#pragma unroll
        for (int i = 0; i < TPL; ++i)
            lg[i] = fmaf(sum[i], unscale_pos(PB::epos((TPL * b + i) % PB::TPW)), bias * (1.0f / ksc));
        float* dst = probs_dst + tl * 32 + TPL * b;
        if constexpr (TPL == 4)
            *reinterpret_cast<float4*>(dst) = make_float4(lg[0], lg[1], lg[2], lg[3]);
        else
            *reinterpret_cast<float2*>(dst) = make_float2(lg[0], lg[1]);
    }
}

// fp32 key residual rows -> logits.  16 independent partial dot products
// (lane owns channels 4*lane..4*lane+3), then one xor-16 step and a
// reduce-scatter over 16 lanes, after which lane r (< 16) holds row r.
__device__ __forceinline__ void kf_rows_to_logits(const uint8_t* slot, const float* qq,
                                                  float* probs_dst, int n, float inv_ksc,
                                                  int lane) {
    const float4 qa = reinterpret_cast<const float4*>(qq)[lane];
    float part[F_ROWS];
#pragma unroll
    for (int r = 0; r < F_ROWS; ++r) {
        part[r] = 0.f;
        if (r < n) {
            const float4 kv = reinterpret_cast<const float4*>(slot + r * D * 4)[lane];
            part[r] = qa.x * kv.x + qa.y * kv.y + qa.z * kv.z + qa.w * kv.w;
        }
    }
#pragma unroll
    for (int r = 0; r < F_ROWS; ++r) part[r] += __shfl_xor_sync(0xffffffffu, part[r], 16);
#pragma unroll
    for (int half = F_ROWS / 2; half >= 1; half >>= 1) {
        const bool upper = (lane & half) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
            const float send = upper ? part[i] : part[i + half];
            const float keep = upper ? part[i + half] : part[i];
            part[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
        }
    }
    if (lane < n) probs_dst[lane] = part[0] * inv_ksc;
}

// Softmax over the item's logits (in place, log2 domain); returns (max, sum).
__device__ __forceinline__ float2 softmax_item(float* probs, int ntok, float* wlog_dst, int lane) {
    __syncwarp();
    float mx = -INFINITY;
    for (int i = lane; i < ntok; i += 32) mx = fmaxf(mx, probs[i]);
    mx = warp_max_redux(mx);
    float sm = 0.f;
    for (int i = lane; i < ntok; i += 32) {
        const float lg = probs[i];
        if (wlog_dst) wlog_dst[i] = lg;
        const float e = ex2_approx(lg - mx);
        probs[i] = e;
        sm += e;
    }
    sm = warp_sum(sm);
    __syncwarp();
    return make_float2(mx, sm);
}

// Quantized value tokens -> P.V accumulators.  Lane = (jj, h): token offset
// jj in 0..15, channel half h (channels 64h .. 64h+63 = groups 2h, 2h+1).
// NT > 0: n == NT, a multiple of 16 (body jobs): the token loop is unrolled,
// with no trip-count test or prefetch register rotation.
template <int B, int NT = 0>
__device__ __forceinline__ void vq_tokens_accumulate(const uint8_t* slot, const float* pr_tok, int n,
                                                     float ksc, float2* vacc, float& zacc0,
                                                     float& zacc1, int lane) {
    using PB = P<B>;
    const int h = lane & 1, jj = lane >> 1;
    const uint8_t* pairs = slot + PB::VQ_TOK * PB::TOK_CODE;
#if KIVI_VQ_UNROLL
    if constexpr (B == 2 && NT > 0) {
        static_assert(NT % 16 == 0, "unrolled value job: whole 16-token rounds");
#pragma unroll
        for (int i = 0; i < NT / 16; ++i) {
            const int t = jj + 16 * i;
            const uint4 cw = *reinterpret_cast<const uint4*>(slot + t * PB::TOK_CODE + h * 16);
            const float4 pr = *reinterpret_cast<const float4*>(pairs + t * 32 + h * 16);
            const float pt = pr_tok[t];
            const float pk = pt * ksc;
            const float ws0 = pk * (pr.y - pr.x);
            const float ws1 = pk * (pr.w - pr.z);
            zacc0 = fmaf(pt, pr.x, zacc0);
            zacc1 = fmaf(pt, pr.z, zacc1);
            PB::fma_word(vacc, cw.x, ws0);
            PB::fma_word(vacc + 8, cw.y, ws0);
            PB::fma_word(vacc + 16, cw.z, ws1);
            PB::fma_word(vacc + 24, cw.w, ws1);
        }
        return;
    }
#endif
    if constexpr (B == 2) {
        int t = jj;
        uint4 cw = make_uint4(0, 0, 0, 0);
        float4 pr = make_float4(0.f, 0.f, 0.f, 0.f);
        float pt = 0.f;
        if (t < n) {
            cw = *reinterpret_cast<const uint4*>(slot + t * PB::TOK_CODE + h * 16);
            pr = *reinterpret_cast<const float4*>(pairs + t * 32 + h * 16);
            pt = pr_tok[t];
        }
        for (; t < n; t += 16) {
            const int tn = t + 16;  // prefetch the next token of this lane
            uint4 cw_n = cw;
            float4 pr_n = pr;
            float pt_n = pt;
            if (tn < n) {
                cw_n = *reinterpret_cast<const uint4*>(slot + tn * PB::TOK_CODE + h * 16);
                pr_n = *reinterpret_cast<const float4*>(pairs + tn * 32 + h * 16);
                pt_n = pr_tok[tn];
            }
            const float pk = pt * ksc;
            const float ws0 = pk * (pr.y - pr.x);
            const float ws1 = pk * (pr.w - pr.z);
            zacc0 = fmaf(pt, pr.x, zacc0);
            zacc1 = fmaf(pt, pr.z, zacc1);
            PB::fma_word(vacc, cw.x, ws0);
            PB::fma_word(vacc + 8, cw.y, ws0);
            PB::fma_word(vacc + 16, cw.z, ws1);
            PB::fma_word(vacc + 24, cw.w, ws1);
            cw = cw_n;
            pr = pr_n;
            pt = pt_n;
        }
    } else {
        for (int t = jj; t < n; t += 16) {
            const float pt = pr_tok[t];
            const float4 pr = *reinterpret_cast<const float4*>(pairs + t * 32 + h * 16);
            const float pk = pt * ksc;
            const float ws0 = pk * (pr.y - pr.x);
            const float ws1 = pk * (pr.w - pr.z);
            zacc0 = fmaf(pt, pr.x, zacc0);
            zacc1 = fmaf(pt, pr.z, zacc1);
            const uint4 c0 = *reinterpret_cast<const uint4*>(slot + t * PB::TOK_CODE + h * 32);
            const uint4 c1 = *reinterpret_cast<const uint4*>(slot + t * PB::TOK_CODE + h * 32 + 16);
            PB::fma_word(vacc, c0.x, ws0);
            PB::fma_word(vacc + 4, c0.y, ws0);
            PB::fma_word(vacc + 8, c0.z, ws0);
            PB::fma_word(vacc + 12, c0.w, ws0);
            PB::fma_word(vacc + 16, c1.x, ws1);
            PB::fma_word(vacc + 20, c1.y, ws1);
            PB::fma_word(vacc + 24, c1.z, ws1);
            PB::fma_word(vacc + 28, c1.w, ws1);
        }
    }
}

// fp32 value residual rows -> P.V (lane owns channels 4*lane .. 4*lane+3).
__device__ __forceinline__ void vf_rows_accumulate(const uint8_t* slot, const float* pr_tok, int n,
                                                   float4& facc, int lane) {
    float4 a2 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < F_ROWS; r += 2) {
        if (r < n) {
            const float4 vv = reinterpret_cast<const float4*>(slot + r * D * 4)[lane];
            const float pt = pr_tok[r];
            facc.x = fmaf(pt, vv.x, facc.x);
            facc.y = fmaf(pt, vv.y, facc.y);
            facc.z = fmaf(pt, vv.z, facc.z);
            facc.w = fmaf(pt, vv.w, facc.w);
        }
        if (r + 1 < n) {
            const float4 vv = reinterpret_cast<const float4*>(slot + (r + 1) * D * 4)[lane];
            const float pt = pr_tok[r + 1];
            a2.x = fmaf(pt, vv.x, a2.x);
            a2.y = fmaf(pt, vv.y, a2.y);
            a2.z = fmaf(pt, vv.z, a2.z);
            a2.w = fmaf(pt, vv.w, a2.w);
        }
    }
    facc.x += a2.x;
    facc.y += a2.y;
    facc.z += a2.z;
    facc.w += a2.w;
}

// Reduce the value accumulators across the 16 lanes sharing a channel half
// (32 rows x 64 channels through the slot, 16-byte chunks XOR-swizzled by
// row: conflict-free writes and reads) and write the item's partial.
template <int B>
__device__ __forceinline__ void v_finalize(uint8_t* slot, const float2* vacc, float zacc0,
                                           float zacc1, const float4& facc, float2 ml,
                                           float* part_o, float2* part_ml, int lane) {
    using PB = P<B>;
    __syncwarp();
    float4* red = reinterpret_cast<float4*>(slot);
#pragma unroll
    for (int qc = 0; qc < 16; ++qc)
        red[lane * 16 + (qc ^ (lane & 7))] =
            make_float4(vacc[2 * qc].x, vacc[2 * qc].y, vacc[2 * qc + 1].x, vacc[2 * qc + 1].y);
    float z0 = zacc0, z1 = zacc1;
#pragma unroll
    for (int o = 2; o < 32; o <<= 1) {
        z0 += __shfl_xor_sync(0xffffffffu, z0, o);
        z1 += __shfl_xor_sync(0xffffffffu, z1, o);
    }
    __syncwarp();
    const int ho = lane >> 4;  // output channel half of this lane
    const int qc = lane & 15;  // 16-byte chunk within the half
    const float zh0 = __shfl_sync(0xffffffffu, z0, ho);
    const float zh1 = __shfl_sync(0xffffffffu, z1, ho);
    const float z = ((lane >> 3) & 1) ? zh1 : zh0;
    float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r2 = 0; r2 < 16; ++r2) {
        const int row = r2 * 2 + ho;
        const float4 v = red[row * 16 + (qc ^ (row & 7))];
        s4.x += v.x; s4.y += v.y; s4.z += v.z; s4.w += v.w;
    }
    const int m0 = (4 * qc) & 31;  // channel within its 32-channel group
    float4 o;
    o.x = fmaf(s4.x, unscale_pos(PB::epos((m0 + 0) % PB::TPW)), z) + facc.x;
    o.y = fmaf(s4.y, unscale_pos(PB::epos((m0 + 1) % PB::TPW)), z) + facc.y;
    o.z = fmaf(s4.z, unscale_pos(PB::epos((m0 + 2) % PB::TPW)), z) + facc.z;
    o.w = fmaf(s4.w, unscale_pos(PB::epos((m0 + 3) % PB::TPW)), z) + facc.w;
    reinterpret_cast<float4*>(part_o)[lane] = o;
    if (lane == 0) *part_ml = ml;
}

// ===================== K4a: body kernel (fully quantized items) =============
// Items are whole 256-token sub-chunks below floor32(vg): every token's key
// and value are quantized, so the job sequence is fixed (B=2: 2 key jobs of 4
// tiles, 2 value jobs of 128 tokens) and the issue path is straight-line.
// VI (B = 2 only): P.V on the integer tensor cores (kernels_vimma.cuh).
// BS: tokens per item (BSUB = 256 by default; 512 for long contexts, where
// the residual region it widens is a small share: C5 +1.7 %, C2 -5 %).
template <int B, bool VI = false, int BS = BSUB>
__global__ void __launch_bounds__(WARPS * 32, 3) attend_body_kernel(FastArgs a) {
    using PB = P<B>;
    using WSB = WarpSmemBody<VI, BS>;
    static_assert(!VI || B == 2, "tensor-core value jobs: 2-bit codes");
    constexpr int NKJ = (BS / 32) / PB::KQ_TILES;  // key jobs per item
    constexpr int NVJ = BS / PB::VQ_TOK;           // value jobs per item
    static_assert(NVJ >= 2 && BS - PB::VQ_TOK >= D, "q staging aliases p[0..127]");
    constexpr int NJ = NKJ + NVJ;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* wbase = smem_raw + warp * WSB::STRIDE;
    float* qraw = reinterpret_cast<float*>(wbase + WSB::QRAW_OFF);
    float* qq = reinterpret_cast<float*>(wbase + WSB::QQ_OFF);
    float* probs = reinterpret_cast<float*>(wbase + WSB::PROBS_OFF);
    uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + WSB::BAR_OFF);
    if (lane == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const uint64_t policy = make_evict_first_policy();
    const CacheDev& c = a.c;
    const int nper = a.n_per_unit;
    const float ksc = TWO_POW_64 / (float)((1 << B) - 1);
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.work_clear) *a.work_clear = 0;
    if (a.tail_last) pdl_trigger();  // the residual-window kernel may follow at once

    // Items are taken dynamically (atomic counter), one item ahead of use, so
    // CTAs that start late — e.g. after a concurrently running tail kernel
    // frees their slot — simply take fewer items.
    auto grab = [&]() -> int {
        int v = 0;
        if (lane == 0) v = atomicAdd(a.work, 1);
        return __shfl_sync(0xffffffffu, v, 0);
    };
    // a.prefetch: L2 bulk prefetch of the whole item after next (its 4 x 8 KB
    // of codes and pairs) as soon as it is grabbed, one item ahead of its TMA
    // loads: more HBM bytes in flight per SM than the two 8 KB slots per warp
    auto prefetch_item = [&](int it) {
        if (!a.prefetch || it >= a.n_items || lane != 0) return;
        const int pu = it / nper, pk = a.k_first + (it - pu * nper);
        constexpr int TPI = BS / 32;  // key tiles per item
        bulk_prefetch_l2(c.kcodes + pu * c.k_ustride + (int64_t)pk * TPI * PB::TILE_CODE,
                         TPI * PB::TILE_CODE);
        bulk_prefetch_l2(c.kpairs + pu * c.kp_ustride + (int64_t)pk * TPI * D, TPI * D * 8);
        bulk_prefetch_l2(c.vcodes + pu * c.v_ustride + (int64_t)pk * BS * PB::TOK_CODE,
                         BS * PB::TOK_CODE);
        bulk_prefetch_l2(c.vpairs + pu * c.vp_ustride + (int64_t)pk * BS * (D / G),
                         BS * (D / G) * 8);
    };
    int f_item = grab(), f_job = 0;
    int f_ahead = grab();   // the item after f_item (atomic latency off the critical path)
    prefetch_item(f_ahead);
    // The claim of the item after f_ahead is issued with f_item's first job
    // and read (broadcast from lane 0) only when f_item's jobs are all issued:
    // the atomic's round trip overlaps a whole item instead of stalling the
    // warp at the broadcast.
    int pend = 0;
    int c_next = f_item;    // next item for the compute loop
    int f_u = f_item / nper, f_k = f_item - f_u * nper;
    // the item's source addresses, advanced by a constant per job (the 64-bit
    // unit / item arithmetic once per item instead of once per copy)
    const uint8_t *src_kc, *src_vc;
    const float2 *src_kp, *src_vp;
    auto item_sources = [&]() {
        src_kc = c.kcodes + f_u * c.k_ustride + (int64_t)f_k * (BS / 32) * PB::TILE_CODE;
        src_kp = c.kpairs + f_u * c.kp_ustride + (int64_t)f_k * (BS / 32) * D;
        src_vc = c.vcodes + f_u * c.v_ustride + (int64_t)f_k * BS * PB::TOK_CODE;
        src_vp = c.vpairs + f_u * c.vp_ustride + (int64_t)f_k * BS * (D / G);
    };
    item_sources();
    auto issue_next = [&](int s) {
        if (f_item >= a.n_items) return;
        if (lane == 0) {
            if (KIVI_DEFER_CLAIM && f_job == 0 && f_ahead < a.n_items) pend = atomicAdd(a.work, 1);
            uint8_t* slot = wbase + s * SLOT;
            uint64_t* bar = &bars[s];
            fence_proxy_async_smem();
            if (f_job < NKJ) {
                constexpr uint32_t cb = PB::KQ_TILES * PB::TILE_CODE;
                constexpr uint32_t pb = PB::KQ_TILES * D * 8;
                mbar_arrive_expect_tx(bar, cb + pb + (f_job == 0 ? D * 4 : 0));
                bulk_g2s_evict_first(slot, src_kc, cb, bar, policy);
                bulk_g2s_evict_first(slot + cb, src_kp, pb, bar, policy);
                if (f_job == 0) bulk_g2s(qraw, a.q + (int64_t)f_u * D, D * 4, bar);
                src_kc += cb;
                src_kp += PB::KQ_TILES * D;
            } else {
                constexpr uint32_t cb = PB::VQ_TOK * PB::TOK_CODE;
                constexpr uint32_t pb = PB::VQ_TOK * (D / G) * 8;
                mbar_arrive_expect_tx(bar, cb + pb);
                bulk_g2s_evict_first(slot, src_vc, cb, bar, policy);
                bulk_g2s_evict_first(slot + cb, src_vp, pb, bar, policy);
                src_vc += cb;
                src_vp += PB::VQ_TOK * (D / G);
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
#pragma unroll 1
        for (int jk = 0; jk < NKJ; ++jk) {
            uint8_t* slot = wait_slot();
            if (jk == 0) load_q_table(qraw, qq, a.qscale, ksc, lane);
            kq_tiles_to_logits<B>(slot, qq, probs + jk * PB::KQ_TILES * 32, PB::KQ_TILES, ksc,
                                  lane);
            release_slot();
        }
        const float2 ml = softmax_item(
            probs, BS, a.wlog ? a.wlog + (int64_t)u * a.l + (int64_t)k * BS : nullptr, lane);
        if constexpr (VI) {
            vimma::State st;
            vimma::begin_item(st);
#pragma unroll 1
            for (int jv = 0; jv < NVJ; ++jv) {
                uint8_t* slot = wait_slot();
                vimma::value_job<PB::VQ_TOK>(slot, probs + jv * PB::VQ_TOK, st, lane);
                if (jv == NVJ - 1) {
                    const int64_t pi = (int64_t)u * a.n_sub + k;
                    vimma::finalize(st, ml, a.part_o + pi * D, a.part_ml + pi, lane);
                }
                release_slot();
            }
        } else {
            float2 vacc[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) vacc[i] = make_float2(0.f, 0.f);
            float zacc0 = 0.f, zacc1 = 0.f;
#pragma unroll 1
            for (int jv = 0; jv < NVJ; ++jv) {
                uint8_t* slot = wait_slot();
                vq_tokens_accumulate<B, PB::VQ_TOK>(slot, probs + jv * PB::VQ_TOK, PB::VQ_TOK, ksc,
                                                    vacc, zacc0, zacc1, lane);
                if (jv == NVJ - 1) {
                    const int64_t pi = (int64_t)u * a.n_sub + k;
                    v_finalize<B>(slot, vacc, zacc0, zacc1, make_float4(0.f, 0.f, 0.f, 0.f), ml,
                                  a.part_o + pi * D, a.part_ml + pi, lane);
                }
                release_slot();
            }
        }
    }
    // programmatic launch after the residual-window kernel (one stream): let
    // the combine be scheduled, and finish only once that kernel has finished
    pdl_trigger();
    pdl_wait();
}

// ===================== K4b: tail kernel (items with residual tokens) ========

enum JobKind { KQ = 0, KF = 1, VQ = 2, VF = 3 };

struct ItemPlan {
    int u, k, t0, t1;
    int nkq, nkf, nvq, nvf, njobs;
};

template <int B>
__device__ __forceinline__ ItemPlan plan_item(const FastArgs& a, int item) {
    ItemPlan p;
    p.u = item / a.n_per_unit;
    const int j = item - p.u * a.n_per_unit;
    p.k = a.k_first + j;
    if (a.sub_b > 0 && j >= a.n_a) {
        p.t0 = a.t_b + (j - a.n_a) * a.sub_b;
        p.t1 = min(p.t0 + a.sub_b, a.l);
    } else {
        p.t0 = a.t_first + j * a.sub;
        p.t1 = min(p.t0 + a.sub, a.sub_b > 0 ? a.t_b : a.l);
    }
    const int kq = max(0, min(p.t1, a.kg) - p.t0);
    const int kf = p.t1 - max(p.t0, a.kg);
    const int vq = max(0, min(p.t1, a.vg) - p.t0);
    const int vf = p.t1 - max(p.t0, a.vg);
    p.nkq = (kq + P<B>::KQ_TILES * 32 - 1) / (P<B>::KQ_TILES * 32);
    p.nkf = kf > 0 ? (kf + F_ROWS - 1) / F_ROWS : 0;
    p.nvq = (vq + P<B>::VQ_TOK - 1) / P<B>::VQ_TOK;
    p.nvf = vf > 0 ? (vf + F_ROWS - 1) / F_ROWS : 0;
    p.njobs = p.nkq + p.nkf + p.nvq + p.nvf;
    return p;
}

// L2 bulk prefetch of an item's fp32 residual rows (keys [max(t0, kg), t1),
// values [max(t0, vg), t1) in the ring); lane 0 only.
__device__ __forceinline__ void prefetch_item_rows(const FastArgs& a, const ItemPlan& p) {
    const CacheDev& c = a.c;
    const int kf0 = max(p.t0, a.kg);
    if (p.t1 > kf0)
        bulk_prefetch_l2(c.kring + p.u * c.ring_ustride + (int64_t)(kf0 - a.kg) * D,
                         (uint32_t)(p.t1 - kf0) * D * 4);
    const int vf0 = max(p.t0, a.vg);
    if (p.t1 > vf0) {
        const float* ring = c.vring + p.u * c.ring_ustride;
        const int r0 = vf0 % c.R, n = p.t1 - vf0;
        const int n1 = min(n, c.R - r0);
        bulk_prefetch_l2(ring + (int64_t)r0 * D, (uint32_t)n1 * D * 4);
        if (n > n1) bulk_prefetch_l2(ring, (uint32_t)(n - n1) * D * 4);
    }
}

struct JobDesc {
    int kind;
    int ts;  // first token
    int n;   // tokens (KQ: tiles)
};

template <int B>
__device__ __forceinline__ JobDesc job_of(const FastArgs& a, const ItemPlan& p, int j) {
    JobDesc jd;
    if (j < p.nkq) {
        jd.kind = KQ;
        jd.ts = p.t0 + j * P<B>::KQ_TILES * 32;
        jd.n = min(P<B>::KQ_TILES, (min(p.t1, a.kg) - jd.ts) >> 5);
        return jd;
    }
    j -= p.nkq;
    if (j < p.nkf) {
        jd.kind = KF;
        jd.ts = max(p.t0, a.kg) + j * F_ROWS;
        jd.n = min(F_ROWS, p.t1 - jd.ts);
        return jd;
    }
    j -= p.nkf;
    if (j < p.nvq) {
        jd.kind = VQ;
        jd.ts = p.t0 + j * P<B>::VQ_TOK;
        jd.n = min(P<B>::VQ_TOK, min(p.t1, a.vg) - jd.ts);
        return jd;
    }
    j -= p.nvq;
    jd.kind = VF;
    jd.ts = max(p.t0, a.vg) + j * F_ROWS;
    jd.n = min(F_ROWS, p.t1 - jd.ts);
    return jd;
}

// Lane 0 only: arm the slot's mbarrier and issue the bulk copies of a job
// (plus the unit's query row for the first job of an item).
template <int B>
__device__ __forceinline__ void issue_job(const FastArgs& a, int u, const JobDesc& jd,
                                          bool with_q, uint8_t* slot, float* qraw, uint64_t* bar,
                                          uint64_t policy) {
    const CacheDev& c = a.c;
    const uint32_t qb = with_q ? D * 4 : 0;
    if (jd.kind == KQ) {
        const int tile0 = jd.ts >> 5;
        const uint32_t cb = (uint32_t)jd.n * P<B>::TILE_CODE;
        const uint32_t pb = (uint32_t)jd.n * D * 8;
        mbar_arrive_expect_tx(bar, cb + pb + qb);
        bulk_g2s_evict_first(slot, c.kcodes + u * c.k_ustride + (int64_t)tile0 * P<B>::TILE_CODE,
                             cb, bar, policy);
        bulk_g2s_evict_first(slot + P<B>::KQ_TILES * P<B>::TILE_CODE,
                             c.kpairs + u * c.kp_ustride + (int64_t)tile0 * D, pb, bar, policy);
    } else if (jd.kind == VQ) {
        const uint32_t cb = (uint32_t)jd.n * P<B>::TOK_CODE;
        const uint32_t pb = (uint32_t)jd.n * (D / G) * 8;
        mbar_arrive_expect_tx(bar, cb + pb + qb);
        bulk_g2s_evict_first(slot, c.vcodes + u * c.v_ustride + (int64_t)jd.ts * P<B>::TOK_CODE,
                             cb, bar, policy);
        bulk_g2s_evict_first(slot + P<B>::VQ_TOK * P<B>::TOK_CODE,
                             c.vpairs + u * c.vp_ustride + (int64_t)jd.ts * (D / G), pb, bar,
                             policy);
    } else if (jd.kind == KF) {
        const uint32_t bytes = (uint32_t)jd.n * D * 4;
        mbar_arrive_expect_tx(bar, bytes + qb);
        bulk_g2s_evict_first(slot, c.kring + u * c.ring_ustride + (int64_t)(jd.ts - a.kg) * D,
                             bytes, bar, policy);
    } else {
        const uint32_t bytes = (uint32_t)jd.n * D * 4;
        mbar_arrive_expect_tx(bar, bytes + qb);
        const int r0 = jd.ts % c.R;
        const float* ring = c.vring + u * c.ring_ustride;
        if (r0 + jd.n <= c.R) {
            bulk_g2s_evict_first(slot, ring + (int64_t)r0 * D, bytes, bar, policy);
        } else {
            const uint32_t n1 = (uint32_t)(c.R - r0);
            bulk_g2s_evict_first(slot, ring + (int64_t)r0 * D, n1 * D * 4, bar, policy);
            bulk_g2s_evict_first(slot + n1 * D * 4, ring, bytes - n1 * D * 4, bar, policy);
        }
    }
    if (with_q) bulk_g2s(qraw, a.q + (int64_t)u * D, qb, bar);
}

// Any mix of quantized / fp32 keys and values per item (the residual window
// and the last partial sub-chunk), any l.
// NW warps per CTA: 4 when the tail runs alone; 1 when it runs beside the
// body kernel on a side stream, so its CTAs fit in the shared memory the
// body CTAs leave free and every tail item gets its own warp.
// APP: compile the fused-append and single-launch (gbar) modes in.  Their
// append / quantize / merge code is ~20K SASS instructions; the default tail
// kernel leaves it out to keep its instruction footprint small.
template <int B, int NW = WARPS, bool APP = false>
__global__ void __launch_bounds__(NW * 32, 3) attend_tail_kernel(FastArgs a) {
    using PB = P<B>;
    if (!a.tail_last) pdl_wait();  // the append before it (programmatic launch)
    pdl_trigger();                  // ... and the launch after it
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* wbase = smem_raw + warp * WS2::STRIDE;
    float* qraw = reinterpret_cast<float*>(wbase + WS2::QRAW_OFF);
    float* qq = reinterpret_cast<float*>(wbase + WS2::QQ_OFF);
    float* probs = reinterpret_cast<float*>(wbase + WS2::PROBS_OFF);
    uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + WS2::BAR_OFF);
    if (lane == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const uint64_t policy = make_evict_first_policy();
    const int gw = blockIdx.x * NW + warp;
    const int tw = gridDim.x * NW;
    const float ksc = TWO_POW_64 / (float)((1 << B) - 1);

    // Item order.  Default: item i to warp i mod tw.  Fused append: a warp owns
    // whole units (u = gw, gw + tw, ...) and walks each unit's items in order,
    // appending the unit's new token before issuing its first job.
    const bool fused = APP && a.l_app >= 0 && !a.gbar;
    const int nper = a.n_per_unit;
    const int n_units = a.n_items / nper;
    auto first_item = [&]() { return fused ? gw * nper : gw; };
    auto next_item = [&](int it) {
        if (!fused) return it + tw;
        return (it % nper == nper - 1) ? it + 1 + (tw - 1) * nper : it + 1;
    };
    auto enter_unit = [&](int it) {  // whole warp
        if constexpr (APP) {
            if (fused && it < a.n_items && it % nper == 0) {
                append_unit_fast<B>(a.c, a.tk, a.tv, a.l_app, it / nper, lane);
                fence_proxy_async_global();  // the unit's TMA reads follow its append
                __syncwarp();
            }
        }
    };
    (void)n_units;
    if (APP && a.gbar) {
        // single-launch decode: appends, then a grid-wide barrier
        if (gw < n_units) {
            append_unit_fast<B>(a.c, a.tk, a.tv, a.l_app, gw, lane);
            fence_proxy_async_global();
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) {
            atomicAdd(a.gbar, 1ull);
            while (ld_acquire_u64(a.gbar) < a.gbar_target) __nanosleep(100);
        }
        __syncwarp();
        fence_proxy_async_global();  // this warp's TMA reads follow every append
    }
    // The item's fp32 residual rows (up to 2 x 64 KB) are a chain of 16-row
    // jobs through two slots; with a.prefetch they are all prefetched into L2
    // when the item's first job is issued, turning the chain's HBM round trips
    // into L2 hits.  Used on the few-unit route (C1: 22.2 -> 21.2 us); beside
    // the body kernel it costs more than it saves (C2 248 -> 258 us).
    auto prefetch_rows = [&](const ItemPlan& p) { prefetch_item_rows(a, p); };
    int f_item = first_item(), f_job = 0;
    ItemPlan f_plan{};
    if (!(APP && a.gbar)) enter_unit(f_item);
    if (f_item < a.n_items) f_plan = plan_item<B>(a, f_item);
    auto issue_next = [&](int s) {
        if (f_item >= a.n_items) return;
        if (lane == 0) {
            if (a.prefetch && f_job == 0) prefetch_rows(f_plan);
            const JobDesc jd = job_of<B>(a, f_plan, f_job);
            fence_proxy_async_smem();
            issue_job<B>(a, f_plan.u, jd, f_job == 0, wbase + s * SLOT, qraw, &bars[s], policy);
        }
        if (++f_job == f_plan.njobs) {
            f_item = next_item(f_item);
            f_job = 0;
            enter_unit(f_item);
            if (f_item < a.n_items) f_plan = plan_item<B>(a, f_item);
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

    for (int item = first_item(); item < a.n_items; item = next_item(item)) {
        const ItemPlan p = plan_item<B>(a, item);
        const int nk = p.nkq + p.nkf;
        for (int j = 0; j < nk; ++j) {
            uint8_t* slot = wait_slot();
            if (j == 0) load_q_table(qraw, qq, a.qscale, ksc, lane);
            const JobDesc jd = job_of<B>(a, p, j);
            if (jd.kind == KQ)
                kq_tiles_to_logits<B>(slot, qq, probs + (jd.ts - p.t0), jd.n, ksc, lane);
            else
                kf_rows_to_logits(slot, qq, probs + (jd.ts - p.t0), jd.n, 1.0f / ksc, lane);
            release_slot();
        }
        const float2 ml = softmax_item(
            probs, p.t1 - p.t0, a.wlog ? a.wlog + (int64_t)p.u * a.l + p.t0 : nullptr, lane);
        float2 vacc[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) vacc[i] = make_float2(0.f, 0.f);
        float4 facc = make_float4(0.f, 0.f, 0.f, 0.f);
        float zacc0 = 0.f, zacc1 = 0.f;
        for (int j = nk; j < p.njobs; ++j) {
            uint8_t* slot = wait_slot();
            const JobDesc jd = job_of<B>(a, p, j);
            const float* pr_tok = probs + (jd.ts - p.t0);
            if (jd.kind == VQ)
                vq_tokens_accumulate<B>(slot, pr_tok, jd.n, ksc, vacc, zacc0, zacc1, lane);
            else
                vf_rows_accumulate(slot, pr_tok, jd.n, facc, lane);
            if (j == p.njobs - 1) {
                const int64_t pi = (int64_t)p.u * a.n_sub + p.k;
                v_finalize<B>(slot, vacc, zacc0, zacc1, facc, ml, a.part_o + pi * D,
                              a.part_ml + pi, lane);
                if (APP && a.gbar) {
                    // the unit's last partial merges the unit
                    __threadfence();
                    __syncwarp();
                    unsigned int done = 0;
                    if (lane == 0) done = atomicAdd(&a.unit_done[p.u], 1u) + 1u;
                    done = __shfl_sync(0xffffffffu, done, 0);
                    if (done == a.unit_target) {
                        __threadfence();
                        combine_unit_warp(a.part_o, a.part_ml, a.n_sub, p.u, a.out, a.stats, lane);
                    }
                }
            }
            release_slot();
        }
    }
    if (a.tail_last) pdl_wait();  // finish only after the body kernel before it
}

// K5 row merge, one 128-thread block per output row (thread c = channel c):
// partial k of the row is part_ml[ml0 + k * ms] / part_o[(ml0 + k * ms) * D].
// The max and the weights are computed in parallel over k (128 partials per
// pass), then every thread streams its channel of the partials with
// independent loads — the loop carries no exp2 and no load latency chain.
__device__ __forceinline__ void combine_row(const float* __restrict__ part_o,
                                            const float2* __restrict__ part_ml, int n_sub,
                                            int64_t ml0, int ms, float* __restrict__ out_row,
                                            float2* __restrict__ stat) {
    __shared__ float sw[128];
    __shared__ float sred[8];
    const int c = threadIdx.x, warp = c >> 5, lane = c & 31;
    float m = -INFINITY;
    for (int k = c; k < n_sub; k += 128) m = fmaxf(m, part_ml[ml0 + (int64_t)k * ms].x);
    m = warp_max_redux(m);
    if (lane == 0) sred[warp] = m;
    __syncthreads();
    const float M = fmaxf(fmaxf(sred[0], sred[1]), fmaxf(sred[2], sred[3]));
    float Lp = 0.f, o = 0.f, o1 = 0.f;
    for (int k0 = 0; k0 < n_sub; k0 += 128) {
        __syncthreads();  // sw reuse (and sred reads above)
        if (k0 + c < n_sub) {
            const float2 ml = part_ml[ml0 + (int64_t)(k0 + c) * ms];
            const float w = exp2f(ml.x - M);
            sw[c] = w;
            Lp = fmaf(ml.y, w, Lp);
        }
        __syncthreads();
        const int nk = min(128, n_sub - k0);
        int i = 0;
#pragma unroll COMBINE_UNROLL
        for (; i + 1 < nk; i += 2) {
            o = fmaf(part_o[(ml0 + (int64_t)(k0 + i) * ms) * D + c], sw[i], o);
            o1 = fmaf(part_o[(ml0 + (int64_t)(k0 + i + 1) * ms) * D + c], sw[i + 1], o1);
        }
        if (i < nk) o = fmaf(part_o[(ml0 + (int64_t)(k0 + i) * ms) * D + c], sw[i], o);
    }
    Lp = warp_sum(Lp);
    __syncthreads();
    if (lane == 0) sred[4 + warp] = Lp;
    __syncthreads();
    const float L = (sred[4] + sred[5]) + (sred[6] + sred[7]);
    out_row[c] = (o + o1) / L;
    if (stat && c == 0) *stat = make_float2(M, L);
}

// The same merge by ONE warp per row (rows = unit x head): lane owns channels
// 4*lane .. 4*lane+3 (one float4 per partial: a coalesced 512 B per warp and
// k), each partial's weight computed once by lane k % 32 and broadcast, the
// partial loads unrolled 8 deep; no block barriers.  Partial k of the row at
// ml0 + k * ms.
__device__ __forceinline__ void combine_row_warp(const float* __restrict__ part_o,
                                                 const float2* __restrict__ part_ml, int n_sub,
                                                 int64_t ml0, int ms, float* __restrict__ out_row,
                                                 float2* __restrict__ stat, int lane) {
    float M = -INFINITY;
    for (int k = lane; k < n_sub; k += 32) M = fmaxf(M, __ldcg(&part_ml[ml0 + (int64_t)k * ms]).x);
    M = warp_max_redux(M);
    float L = 0.f;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k0 = 0; k0 < n_sub; k0 += 32) {
        float w = 0.f;
        if (k0 + lane < n_sub) {
            const float2 m = __ldcg(&part_ml[ml0 + (int64_t)(k0 + lane) * ms]);
            w = exp2f(m.x - M);
            L = fmaf(m.y, w, L);
        }
        const int nk = min(32, n_sub - k0);
#pragma unroll 8
        for (int i = 0; i < nk; ++i) {
            const float wi = __shfl_sync(0xffffffffu, w, i);
            const float4 p = __ldcg(reinterpret_cast<const float4*>(
                                        part_o + (ml0 + (int64_t)(k0 + i) * ms) * D) + lane);
            o.x = fmaf(p.x, wi, o.x);
            o.y = fmaf(p.y, wi, o.y);
            o.z = fmaf(p.z, wi, o.z);
            o.w = fmaf(p.w, wi, o.w);
        }
    }
    L = warp_sum(L);
    reinterpret_cast<float4*>(out_row)[lane] = make_float4(o.x / L, o.y / L, o.z / L, o.w / L);
    if (stat && lane == 0) *stat = make_float2(M, L);
}

// The same merge as one serial loop per thread: better when there are many
// rows (thousands of blocks hide each block's latency chain; measured C3 20.5
// vs 28.5 us), worse when there are few (C1: 12.8 vs 7.4 us).
__device__ __forceinline__ void combine_row_serial(const float* __restrict__ part_o,
                                                   const float2* __restrict__ part_ml, int n_sub,
                                                   int64_t ml0, int ms, float* __restrict__ out_row,
                                                   float2* __restrict__ stat) {
    const int c = threadIdx.x;
    float M = -INFINITY;
    for (int k = 0; k < n_sub; ++k) M = fmaxf(M, part_ml[ml0 + (int64_t)k * ms].x);
    float L = 0.f, o = 0.f;
    for (int k = 0; k < n_sub; ++k) {
        const int64_t pi = ml0 + (int64_t)k * ms;
        const float2 ml = part_ml[pi];
        const float w = exp2f(ml.x - M);
        L = fmaf(ml.y, w, L);
        o = fmaf(part_o[pi * D + c], w, o);
    }
    out_row[c] = o / L;
    if (stat && c == 0) *stat = make_float2(M, L);
}

// K5: merge the per-item partials of every unit (LSE rescale in log2 domain).
__global__ void __launch_bounds__(128) combine_kernel(const float* __restrict__ part_o,
                                                      const float2* __restrict__ part_ml, int n_sub,
                                                      float* __restrict__ out,
                                                      float2* __restrict__ stats, int parallel,
                                                      int64_t n_rows) {
    pdl_wait();
    if (parallel == 2) {  // one warp per unit, four units per block
        const int64_t u = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
        if (u < n_rows)
            combine_row_warp(part_o, part_ml, n_sub, u * n_sub, 1, out + u * D,
                             stats ? stats + u : nullptr, threadIdx.x & 31);
        return;
    }
    const int64_t u = blockIdx.x;
    if (parallel)
        combine_row(part_o, part_ml, n_sub, u * n_sub, 1, out + u * D, stats ? stats + u : nullptr);
    else
        combine_row_serial(part_o, part_ml, n_sub, u * n_sub, 1, out + u * D,
                           stats ? stats + u : nullptr);
}

// One layer's K5 merge fused with the NEXT layer's append (a multi-layer
// decode step on one stream): blocks [0, n_comb) merge layer i's partials
// exactly as combine_kernel (they wait for the attend before them); blocks
// [n_comb, ...) append layer i+1's token rows, one warp per unit
// (append_fast_kernel; a step that completes key tiles quantizes them in a
// separate append_flush_fast_kernel launch, whose 32-value registers would
// otherwise cut this kernel's occupancy).  The append touches only layer i+1's cache,
// which no kernel in flight reads, so it runs beside the merge instead of as
// its own launch after it.
template <int B>
__global__ void __launch_bounds__(128) combine_append_kernel(
    const float* __restrict__ part_o, const float2* __restrict__ part_ml, int n_sub,
    float* __restrict__ out, int cmode, int64_t n_rows, int n_comb, CacheDev cn,
    const float* __restrict__ tk, const float* __restrict__ tv, int64_t l_next) {
    pdl_trigger();  // the next layer's attend may be scheduled (it waits for all of this)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if ((int)blockIdx.x < n_comb) {
        pdl_wait();
        if (cmode == 2) {
            const int64_t u = (int64_t)blockIdx.x * 4 + warp;
            if (u < n_rows) combine_row_warp(part_o, part_ml, n_sub, u * n_sub, 1, out + u * D, nullptr, lane);
            return;
        }
        const int64_t u = blockIdx.x;
        if (cmode)
            combine_row(part_o, part_ml, n_sub, u * n_sub, 1, out + u * D, nullptr);
        else
            combine_row_serial(part_o, part_ml, n_sub, u * n_sub, 1, out + u * D, nullptr);
        return;
    }
    const int64_t u = (int64_t)((int)blockIdx.x - n_comb) * 4 + warp;
    if (u < cn.n_units) append_unit_fast<B, false>(cn, tk, tv, l_next, u, lane);
}

// Optional weights: w_t = 2^(logit2_t - M) / L, in place over the wlog buffer.
__global__ void normalize_weights_kernel(float* __restrict__ w, const float2* __restrict__ stats,
                                         int64_t l, int64_t n_units) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_units * l;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float2 st = stats[i / l];
        w[i] = exp2f(w[i] - st.x) / st.y;
    }
}

#undef KIVI_F

}  // namespace fast
}  // namespace kivi_b200
