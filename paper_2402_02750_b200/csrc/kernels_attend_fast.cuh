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
//           current one is computed.
//
// Arithmetic (exact dequantisation, fp32 accumulation):
//   key logit  t = sum_c q_c (code*s_c + z_c) = sum_c (q_c s_c) code + sum_c q_c z_c
//   value out  c = sum_t p_t (code*s_t + z_t) = sum_t (p_t s_t) code + sum_t p_t z_t
// A 2-bit code at bit position e of a word is read as the fp32 DENORMAL
// whose bits are (word & (3 << e)), i.e. code * 2^(e-149), exactly.  The
// per-group multiplier carries 2^64 so products land in the normal range,
// and each accumulator (one per token for keys, per channel for values) has a
// fixed position e, undone once at the end.  So each code costs one LOP3 and
// half an FFMA2 — no shifts, no int->float conversion.
#pragma once

#include "common.cuh"
#include "kernels_quant.cuh"

namespace kivi_b200 {
namespace fast {

constexpr int D = 128;
constexpr int G = 32;
constexpr int SUB = 256;       // tokens per item
constexpr int WARPS = 4;       // warps per CTA
constexpr int SLOT = 8192;     // bytes per pipeline slot
constexpr int F_ROWS = 16;     // fp32 residual rows per job (16 * 512 B)
constexpr float TWO_POW_64 = 18446744073709551616.0f;
constexpr float LOG2E = 1.4426950408889634f;

template <int B>
struct P;
template <>
struct P<2> {
    static constexpr int CB = 8;             // bytes per (tile, channel)
    static constexpr int TILE_CODE = D * CB; // 1024
    static constexpr int KQ_TILES = 4;       // tiles per KQ job (4 KB codes + 4 KB pairs)
    static constexpr int LPT = 8;            // lanes per tile
    static constexpr int TOK_CODE = D * 2 / 8;  // 32
    static constexpr int VQ_TOK = 128;       // tokens per VQ job (4 KB codes + 4 KB pairs)
    static constexpr int TPW = 16;           // codes per 32-bit word
    // denormal bit position of code k of a word (after the one shift below)
    static __host__ __device__ constexpr int epos(int k) { return k <= 10 ? 2 * k : 2 * k - 10; }
    // acc[0..7] (+)= M * codes of w (codes 2j, 2j+1 in acc[j])
    static __device__ __forceinline__ void fma_word(float2* acc, uint32_t w, float M) {
        const float2 m2 = make_float2(M, M);
        const uint32_t s = w >> 10;
#define KIVI_F(x) __uint_as_float(x)
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
    static constexpr int TILE_CODE = D * CB;  // 2048
    static constexpr int KQ_TILES = 2;        // 4 KB codes + 2 KB pairs
    static constexpr int LPT = 16;
    static constexpr int TOK_CODE = D * 4 / 8;  // 64
    static constexpr int VQ_TOK = 64;           // 4 KB codes + 2 KB pairs
    static constexpr int TPW = 8;
    static __host__ __device__ constexpr int epos(int k) { return k <= 4 ? 4 * k : 4 * k - 12; }
    static __device__ __forceinline__ void fma_word(float2* acc, uint32_t w, float M) {
        const float2 m2 = make_float2(M, M);
        const uint32_t s = w >> 12;
        acc[0] = __ffma2_rn(m2, make_float2(KIVI_F(w & 0xFu), KIVI_F(w & 0xF0u)), acc[0]);
        acc[1] = __ffma2_rn(m2, make_float2(KIVI_F(w & 0xF00u), KIVI_F(w & 0xF000u)), acc[1]);
        acc[2] = __ffma2_rn(m2, make_float2(KIVI_F(w & 0xF0000u), KIVI_F(s & 0xF00u)), acc[2]);
        acc[3] = __ffma2_rn(m2, make_float2(KIVI_F(s & 0xF000u), KIVI_F(s & 0xF0000u)), acc[3]);
#undef KIVI_F
    }
};

// 2^(149 - 64 - e): undoes the denormal position e and the 2^64 multiplier.
__device__ __forceinline__ float unscale_pos(int e) {
    return __int_as_float((127 + 149 - 64 - e) << 23);
}

struct FastArgs {
    CacheDev c;
    int64_t l, kg, vg;
    const float* q;     // [units][128]
    float qscale;       // logit scale * log2(e)
    float* part_o;      // [units][n_sub][128]
    float2* part_ml;    // [units][n_sub]   (max, sum) in log2 domain
    float* wlog;        // [units][l] log2-domain logits, or null
    int64_t n_sub;
};

enum JobKind { KQ = 0, KF = 1, VQ = 2, VF = 3 };

struct ItemPlan {
    int64_t u, t0, t1;
    int nkq, nkf, nvq, nvf;
};

template <int B>
__device__ __forceinline__ ItemPlan plan_item(const FastArgs& a, int64_t item) {
    ItemPlan p;
    p.u = item / a.n_sub;
    p.t0 = (item % a.n_sub) * SUB;
    p.t1 = min(p.t0 + SUB, a.l);
    const int64_t kq = max((int64_t)0, min(p.t1, a.kg) - p.t0);
    const int64_t kf = p.t1 - max(p.t0, a.kg);
    const int64_t vq = max((int64_t)0, min(p.t1, a.vg) - p.t0);
    const int64_t vf = p.t1 - max(p.t0, a.vg);
    p.nkq = (int)((kq + P<B>::KQ_TILES * 32 - 1) / (P<B>::KQ_TILES * 32));
    p.nkf = kf > 0 ? (int)((kf + F_ROWS - 1) / F_ROWS) : 0;
    p.nvq = (int)((vq + P<B>::VQ_TOK - 1) / P<B>::VQ_TOK);
    p.nvf = vf > 0 ? (int)((vf + F_ROWS - 1) / F_ROWS) : 0;
    return p;
}

struct JobDesc {
    int kind;
    int64_t ts;  // first token
    int n;       // tokens (KQ: tiles)
};

template <int B>
__device__ __forceinline__ JobDesc job_of(const FastArgs& a, const ItemPlan& p, int j) {
    JobDesc jd;
    if (j < p.nkq) {
        jd.kind = KQ;
        jd.ts = p.t0 + (int64_t)j * P<B>::KQ_TILES * 32;
        const int64_t end = min(p.t1, a.kg);
        jd.n = (int)min((int64_t)P<B>::KQ_TILES, (end - jd.ts) / 32);
        return jd;
    }
    j -= p.nkq;
    if (j < p.nkf) {
        jd.kind = KF;
        jd.ts = max(p.t0, a.kg) + (int64_t)j * F_ROWS;
        jd.n = (int)min((int64_t)F_ROWS, p.t1 - jd.ts);
        return jd;
    }
    j -= p.nkf;
    if (j < p.nvq) {
        jd.kind = VQ;
        jd.ts = p.t0 + (int64_t)j * P<B>::VQ_TOK;
        jd.n = (int)min((int64_t)P<B>::VQ_TOK, min(p.t1, a.vg) - jd.ts);
        return jd;
    }
    j -= p.nvq;
    jd.kind = VF;
    jd.ts = max(p.t0, a.vg) + (int64_t)j * F_ROWS;
    jd.n = (int)min((int64_t)F_ROWS, p.t1 - jd.ts);
    return jd;
}

// Lane 0 only: arm the slot's mbarrier and issue the bulk copies of a job.
template <int B>
__device__ __forceinline__ void issue_job(const FastArgs& a, int64_t u, const JobDesc& jd,
                                          uint8_t* slot, uint64_t* bar, uint64_t policy) {
    const CacheDev& c = a.c;
    if (jd.kind == KQ) {
        const int64_t tile0 = jd.ts / 32;
        const uint32_t cb = (uint32_t)jd.n * P<B>::TILE_CODE;
        const uint32_t pb = (uint32_t)jd.n * D * 8;
        mbar_arrive_expect_tx(bar, cb + pb);
        bulk_g2s_evict_first(slot, c.kcodes + u * c.k_ustride + tile0 * P<B>::TILE_CODE, cb, bar,
                             policy);
        bulk_g2s_evict_first(slot + P<B>::KQ_TILES * P<B>::TILE_CODE,
                             c.kpairs + u * c.kp_ustride + tile0 * D, pb, bar, policy);
    } else if (jd.kind == VQ) {
        const uint32_t cb = (uint32_t)jd.n * P<B>::TOK_CODE;
        const uint32_t pb = (uint32_t)jd.n * (D / G) * 8;
        mbar_arrive_expect_tx(bar, cb + pb);
        bulk_g2s_evict_first(slot, c.vcodes + u * c.v_ustride + jd.ts * P<B>::TOK_CODE, cb, bar,
                             policy);
        bulk_g2s_evict_first(slot + P<B>::VQ_TOK * P<B>::TOK_CODE,
                             c.vpairs + u * c.vp_ustride + jd.ts * (D / G), pb, bar, policy);
    } else if (jd.kind == KF) {
        const uint32_t bytes = (uint32_t)jd.n * D * 4;
        mbar_arrive_expect_tx(bar, bytes);
        bulk_g2s_evict_first(slot, c.kring + u * c.ring_ustride + (jd.ts - a.kg) * D, bytes, bar,
                             policy);
    } else {
        const uint32_t bytes = (uint32_t)jd.n * D * 4;
        mbar_arrive_expect_tx(bar, bytes);
        const int64_t r0 = jd.ts % c.R;
        const float* ring = c.vring + u * c.ring_ustride;
        if (r0 + jd.n <= c.R) {
            bulk_g2s_evict_first(slot, ring + r0 * D, bytes, bar, policy);
        } else {
            const uint32_t n1 = (uint32_t)(c.R - r0);
            bulk_g2s_evict_first(slot, ring + r0 * D, n1 * D * 4, bar, policy);
            bulk_g2s_evict_first(slot + n1 * D * 4, ring, bytes - n1 * D * 4, bar, policy);
        }
    }
}

template <int NSLOT>
struct WarpSmem {
    static constexpr int PROBS_OFF = NSLOT * SLOT;
    static constexpr int Q_OFF = PROBS_OFF + SUB * 4;
    static constexpr int BAR_OFF = Q_OFF + D * 4;
    static constexpr int BYTES = BAR_OFF + 8 * NSLOT + 8;
};

template <int B, int NSLOT>
__global__ void __launch_bounds__(WARPS * 32) attend_fast_kernel(FastArgs a) {
    using PB = P<B>;
    using WS = WarpSmem<NSLOT>;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* wbase = smem_raw + warp * ((WS::BYTES + 127) & ~127);
    float* probs = reinterpret_cast<float*>(wbase + WS::PROBS_OFF);
    float* qs = reinterpret_cast<float*>(wbase + WS::Q_OFF);
    uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + WS::BAR_OFF);

    if (lane == 0) {
        for (int s = 0; s < NSLOT; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const uint64_t policy = make_evict_first_policy();

    const int64_t total = a.c.n_units * a.n_sub;
    const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
    const int64_t tw = (int64_t)gridDim.x * WARPS;

    // Fetch cursor (uniform across the warp).
    int64_t f_item = gw;
    int f_job = 0;
    ItemPlan f_plan;
    int f_njobs = 0;
    if (f_item < total) {
        f_plan = plan_item<B>(a, f_item);
        f_njobs = f_plan.nkq + f_plan.nkf + f_plan.nvq + f_plan.nvf;
    }
    auto issue_next = [&](int s) {
        if (f_item >= total) return;
        if (lane == 0) {
            JobDesc jd = job_of<B>(a, f_plan, f_job);
            fence_proxy_async_smem();
            issue_job<B>(a, f_plan.u, jd, wbase + s * SLOT, &bars[s], policy);
        }
        if (++f_job == f_njobs) {
            f_item += tw;
            f_job = 0;
            if (f_item < total) {
                f_plan = plan_item<B>(a, f_item);
                f_njobs = f_plan.nkq + f_plan.nkf + f_plan.nvq + f_plan.nvf;
            }
        }
    };
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) issue_next(s);

    uint32_t phase = 0;
    int cs = 0;  // compute slot
    const float ksc = TWO_POW_64 / (float)((1 << B) - 1);

    for (int64_t item = gw; item < total; item += tw) {
        const ItemPlan p = plan_item<B>(a, item);
        const int njobs = p.nkq + p.nkf + p.nvq + p.nvf;
        const int64_t u = p.u;
        const int ntok = (int)(p.t1 - p.t0);
        {
            const float4 qv = reinterpret_cast<const float4*>(a.q + u * D)[lane];
            reinterpret_cast<float4*>(qs)[lane] =
                make_float4(qv.x * a.qscale, qv.y * a.qscale, qv.z * a.qscale, qv.w * a.qscale);
        }
        __syncwarp();

        float2 vacc[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) vacc[i] = make_float2(0.f, 0.f);
        float4 facc = make_float4(0.f, 0.f, 0.f, 0.f);
        float zacc = 0.f;
        float m_item = 0.f, l_item = 0.f;

        for (int j = 0; j < njobs; ++j) {
            uint8_t* slot = wbase + cs * SLOT;
            mbar_wait(&bars[cs], (phase >> cs) & 1u);
            phase ^= (1u << cs);
            const JobDesc jd = job_of<B>(a, p, j);

            if (jd.kind == KQ) {
                // ---- quantized key tiles -> logits --------------------------
                const int tl = lane / PB::LPT;  // tile within job
                const int b = lane % PB::LPT;
                float2 acc[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) acc[i] = make_float2(0.f, 0.f);
                float bias = 0.f;
                if (tl < jd.n) {
                    const uint8_t* codes = slot + tl * PB::TILE_CODE;
                    const uint8_t* pairs = slot + PB::KQ_TILES * PB::TILE_CODE + tl * D * 8;
#pragma unroll
                    for (int it = 0; it < 8; ++it) {
                        const int ci = it * PB::LPT + b;  // 16-byte chunk index
                        const uint4 cw = *reinterpret_cast<const uint4*>(codes + ci * 16);
                        if constexpr (B == 2) {
                            const float4 pr = *reinterpret_cast<const float4*>(pairs + ci * 16);
                            const float2 qq = *reinterpret_cast<const float2*>(qs + 2 * ci);
                            const float m0 = qq.x * (pr.y - pr.x) * ksc;
                            const float m1 = qq.y * (pr.w - pr.z) * ksc;
                            bias = fmaf(qq.x, pr.x, bias);
                            bias = fmaf(qq.y, pr.z, bias);
                            PB::fma_word(acc, cw.x, m0);
                            PB::fma_word(acc + 8, cw.y, m0);
                            PB::fma_word(acc, cw.z, m1);
                            PB::fma_word(acc + 8, cw.w, m1);
                        } else {
                            const float2 pr = *reinterpret_cast<const float2*>(pairs + ci * 8);
                            const float qq = qs[ci];
                            const float m0 = qq * (pr.y - pr.x) * ksc;
                            bias = fmaf(qq, pr.x, bias);
                            PB::fma_word(acc, cw.x, m0);
                            PB::fma_word(acc + 4, cw.y, m0);
                            PB::fma_word(acc + 8, cw.z, m0);
                            PB::fma_word(acc + 12, cw.w, m0);
                        }
                    }
                }
                // bias over the LPT lanes of a tile
#pragma unroll
                for (int o = 1; o < PB::LPT; o <<= 1) bias += __shfl_xor_sync(0xffffffffu, bias, o);
                // transpose-reduce the 32 per-token partials through the slot
                __syncwarp();
                float* red = reinterpret_cast<float*>(slot);
                {
                    float4* row = reinterpret_cast<float4*>(red + lane * 36);
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        row[i] = make_float4(acc[2 * i].x, acc[2 * i].y, acc[2 * i + 1].x,
                                             acc[2 * i + 1].y);
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
                if (tl < jd.n) {
                    const int tok_in_item = (int)(jd.ts - p.t0) + tl * 32;
                    float lg[TPL];
#pragma unroll
                    for (int i = 0; i < TPL; ++i) {
                        const int tok = TPL * b + i;  // token within tile
                        lg[i] = fmaf(sum[i], unscale_pos(PB::epos(tok % PB::TPW)), bias);
                    }
                    if constexpr (TPL == 4)
                        *reinterpret_cast<float4*>(probs + tok_in_item + TPL * b) =
                            make_float4(lg[0], lg[1], lg[2], lg[3]);
                    else
                        *reinterpret_cast<float2*>(probs + tok_in_item + TPL * b) =
                            make_float2(lg[0], lg[1]);
                }
            } else if (jd.kind == KF) {
                // ---- fp32 key residual rows -> logits -----------------------
                const float4 qv = reinterpret_cast<const float4*>(qs)[lane];
                float mine = 0.f;
                for (int r = 0; r < jd.n; ++r) {
                    const float4 kv = reinterpret_cast<const float4*>(slot + r * D * 4)[lane];
                    float v = qv.x * kv.x + qv.y * kv.y + qv.z * kv.z + qv.w * kv.w;
                    v = warp_sum(v);
                    if (lane == r) mine = v;
                }
                if (lane < jd.n) probs[jd.ts - p.t0 + lane] = mine;
            } else if (jd.kind == VQ) {
                // ---- quantized value tokens -> P.V --------------------------
                const int cg = lane & 3, jj = lane >> 2;
                const uint8_t* pairs = slot + PB::VQ_TOK * PB::TOK_CODE;
                const float* pr_tok = probs + (jd.ts - p.t0);
                for (int t = jj; t < jd.n; t += 8) {
                    const float pt = pr_tok[t];
                    const float2 pr =
                        *reinterpret_cast<const float2*>(pairs + t * (D / G) * 8 + cg * 8);
                    const float ws = pt * (pr.y - pr.x) * ksc;
                    zacc = fmaf(pt, pr.x, zacc);
                    if constexpr (B == 2) {
                        const uint2 cw =
                            *reinterpret_cast<const uint2*>(slot + t * PB::TOK_CODE + cg * 8);
                        PB::fma_word(vacc, cw.x, ws);
                        PB::fma_word(vacc + 8, cw.y, ws);
                    } else {
                        const uint4 cw =
                            *reinterpret_cast<const uint4*>(slot + t * PB::TOK_CODE + cg * 16);
                        PB::fma_word(vacc, cw.x, ws);
                        PB::fma_word(vacc + 4, cw.y, ws);
                        PB::fma_word(vacc + 8, cw.z, ws);
                        PB::fma_word(vacc + 12, cw.w, ws);
                    }
                }
            } else {
                // ---- fp32 value residual rows -> P.V ------------------------
                const float* pr_tok = probs + (jd.ts - p.t0);
                for (int r = 0; r < jd.n; ++r) {
                    const float4 vv = reinterpret_cast<const float4*>(slot + r * D * 4)[lane];
                    const float pt = pr_tok[r];
                    facc.x = fmaf(pt, vv.x, facc.x);
                    facc.y = fmaf(pt, vv.y, facc.y);
                    facc.z = fmaf(pt, vv.z, facc.z);
                    facc.w = fmaf(pt, vv.w, facc.w);
                }
            }

            if (j == p.nkq + p.nkf - 1) {
                // ---- all logits of the item are in `probs`: softmax (log2) --
                __syncwarp();
                float mx = -INFINITY;
                for (int i = lane; i < ntok; i += 32) mx = fmaxf(mx, probs[i]);
                mx = warp_max(mx);
                float sm = 0.f;
                for (int i = lane; i < ntok; i += 32) {
                    const float lg = probs[i];
                    if (a.wlog) a.wlog[u * a.l + p.t0 + i] = lg;
                    const float e = exp2f(lg - mx);
                    probs[i] = e;
                    sm += e;
                }
                m_item = mx;
                l_item = warp_sum(sm);
                __syncwarp();
            }

            if (j == njobs - 1) {
                // ---- finalize: reduce value accumulators, write the partial -
                __syncwarp();
                float* red = reinterpret_cast<float*>(slot);
                {
                    const int cg = lane & 3, jj = lane >> 2;
                    float4* row = reinterpret_cast<float4*>(red + (jj * 4 + cg) * 36);
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        row[i] = make_float4(vacc[2 * i].x, vacc[2 * i].y, vacc[2 * i + 1].x,
                                             vacc[2 * i + 1].y);
                }
                float zt = zacc;
                zt += __shfl_xor_sync(0xffffffffu, zt, 4);
                zt += __shfl_xor_sync(0xffffffffu, zt, 8);
                zt += __shfl_xor_sync(0xffffffffu, zt, 16);
                __syncwarp();
                const int cgo = lane >> 3;         // output channel group of this lane
                const int m0 = 4 * (lane & 7);     // first channel within the group
                const float z = __shfl_sync(0xffffffffu, zt, cgo);
                float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    const float4 v = *reinterpret_cast<const float4*>(red + (jj * 4 + cgo) * 36 + m0);
                    s4.x += v.x; s4.y += v.y; s4.z += v.z; s4.w += v.w;
                }
                float4 o;
                o.x = fmaf(s4.x, unscale_pos(PB::epos((m0 + 0) % PB::TPW)), z) + facc.x;
                o.y = fmaf(s4.y, unscale_pos(PB::epos((m0 + 1) % PB::TPW)), z) + facc.y;
                o.z = fmaf(s4.z, unscale_pos(PB::epos((m0 + 2) % PB::TPW)), z) + facc.z;
                o.w = fmaf(s4.w, unscale_pos(PB::epos((m0 + 3) % PB::TPW)), z) + facc.w;
                const int64_t pi = u * a.n_sub + (p.t0 / SUB);
                reinterpret_cast<float4*>(a.part_o + pi * D)[lane] = o;
                if (lane == 0) a.part_ml[pi] = make_float2(m_item, l_item);
            }

            __syncwarp();
            issue_next(cs);
            cs = (cs + 1 == NSLOT) ? 0 : cs + 1;
        }
    }
}

// K5: merge the per-item partials of every unit (LSE rescale in log2 domain).
__global__ void combine_kernel(const float* __restrict__ part_o, const float2* __restrict__ part_ml,
                               int64_t n_sub, float* __restrict__ out, float2* __restrict__ stats) {
    const int64_t u = blockIdx.x;
    const int c = threadIdx.x;  // 128 threads
    float M = -INFINITY;
    for (int64_t k = 0; k < n_sub; ++k) M = fmaxf(M, part_ml[u * n_sub + k].x);
    float L = 0.f, o = 0.f;
    for (int64_t k = 0; k < n_sub; ++k) {
        const float2 ml = part_ml[u * n_sub + k];
        const float w = exp2f(ml.x - M);
        L = fmaf(ml.y, w, L);
        o = fmaf(part_o[(u * n_sub + k) * D + c], w, o);
    }
    out[u * D + c] = o / L;
    if (stats && c == 0) stats[u] = make_float2(M, L);
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

}  // namespace fast
}  // namespace kivi_b200
