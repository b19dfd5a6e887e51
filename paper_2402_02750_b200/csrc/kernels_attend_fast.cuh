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

#define KIVI_F(x) __uint_as_float(x)

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
        const uint32_t s = w >> 10;
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
        const uint32_t s = w >> 12;
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
    int n_sub;          // items per unit
    int n_items;        // n_units * n_sub
    const float* q;     // [units][128]
    float qscale;       // logit scale * log2(e)
    float* part_o;      // [units][n_sub][128]
    float2* part_ml;    // [units][n_sub]   (max, sum) in log2 domain
    float* wlog;        // [units][l] log2-domain logits, or null
};

enum JobKind { KQ = 0, KF = 1, VQ = 2, VF = 3 };

struct ItemPlan {
    int u, t0, t1;
    int nkq, nkf, nvq, nvf, njobs;
};

template <int B>
__device__ __forceinline__ ItemPlan plan_item(const FastArgs& a, int item) {
    ItemPlan p;
    p.u = item / a.n_sub;
    p.t0 = (item - p.u * a.n_sub) * SUB;
    p.t1 = min(p.t0 + SUB, a.l);
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

// Per-warp shared memory.  One q staging buffer suffices for NSLOT == 2: the
// next item's first job is issued only after the current item's job 0 (which
// consumes the staged q) has been computed, since every item has >= 2 jobs.
template <int NSLOT>
struct WarpSmem {
    static_assert(NSLOT == 2, "q staging assumes two slots");
    static constexpr int QRAW_OFF = NSLOT * SLOT;            // 128 fp32 (staged q)
    static constexpr int QQ_OFF = QRAW_OFF + D * 4;          // 128 fp32 (q * scale * log2e)
    static constexpr int PROBS_OFF = QQ_OFF + D * 4;         // 256 fp32
    static constexpr int BAR_OFF = PROBS_OFF + SUB * 4;
    static constexpr int BYTES = BAR_OFF + 8 * NSLOT;
    static constexpr int STRIDE = (BYTES + 127) & ~127;
};

template <int B, int NSLOT>
__global__ void __launch_bounds__(WARPS * 32, 3) attend_fast_kernel(FastArgs a) {
    using PB = P<B>;
    using WS = WarpSmem<NSLOT>;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* wbase = smem_raw + warp * WS::STRIDE;
    float* qraw = reinterpret_cast<float*>(wbase + WS::QRAW_OFF);
    float* qq = reinterpret_cast<float*>(wbase + WS::QQ_OFF);
    float* probs = reinterpret_cast<float*>(wbase + WS::PROBS_OFF);
    uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + WS::BAR_OFF);

    if (lane == 0) {
        for (int s = 0; s < NSLOT; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const uint64_t policy = make_evict_first_policy();

    const int gw = blockIdx.x * WARPS + warp;
    const int tw = gridDim.x * WARPS;
    const float ksc = TWO_POW_64 / (float)((1 << B) - 1);

    // ---- fetch cursor (uniform across the warp) ----------------------------
    int f_item = gw, f_job = 0;
    ItemPlan f_plan{};
    if (f_item < a.n_items) f_plan = plan_item<B>(a, f_item);
    auto issue_next = [&](int s) {
        if (f_item >= a.n_items) return;
        if (lane == 0) {
            const JobDesc jd = job_of<B>(a, f_plan, f_job);
            fence_proxy_async_smem();
            issue_job<B>(a, f_plan.u, jd, f_job == 0, wbase + s * SLOT, qraw, &bars[s], policy);
        }
        if (++f_job == f_plan.njobs) {
            f_item += tw;
            f_job = 0;
            if (f_item < a.n_items) f_plan = plan_item<B>(a, f_item);
        }
    };
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) issue_next(s);

    uint32_t phase = 0;
    int cs = 0;  // compute slot

    auto wait_slot = [&]() -> uint8_t* {
        mbar_wait(&bars[cs], (phase >> cs) & 1u);
        phase ^= (1u << cs);
        return wbase + cs * SLOT;
    };
    auto release_slot = [&](bool) {
        __syncwarp();
        issue_next(cs);
        cs = (cs + 1 == NSLOT) ? 0 : cs + 1;
    };

    for (int item = gw; item < a.n_items; item += tw) {
        const ItemPlan p = plan_item<B>(a, item);
        const int u = p.u;
        const int ntok = p.t1 - p.t0;
        const int nk = p.nkq + p.nkf;

        // ================= phase 1: logits of the item's tokens =============
        for (int j = 0; j < nk; ++j) {
            uint8_t* slot = wait_slot();
            if (j == 0) {
                // query row arrived with the item's first job
                const float4 qv = reinterpret_cast<const float4*>(qraw)[lane];
                reinterpret_cast<float4*>(qq)[lane] = make_float4(
                    qv.x * a.qscale, qv.y * a.qscale, qv.z * a.qscale, qv.w * a.qscale);
                __syncwarp();
            }
            const JobDesc jd = job_of<B>(a, p, j);
            if (jd.kind == KQ) {
                const int tl = lane / PB::LPT;  // tile within job
                const int b = lane % PB::LPT;
                float2 acc[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) acc[i] = make_float2(0.f, 0.f);
                float bias = 0.f;
                if (tl < jd.n) {
                    const uint8_t* codes = slot + tl * PB::TILE_CODE;
                    const uint8_t* pairs = slot + PB::KQ_TILES * PB::TILE_CODE + tl * D * 8;
                    if constexpr (B == 2) {
                        // software-pipelined: loads of iteration it+1 issued before
                        // the 64 LOP3 + 32 FFMA2 of iteration it
                        uint4 cw = *reinterpret_cast<const uint4*>(codes + b * 16);
                        float4 pr = *reinterpret_cast<const float4*>(pairs + b * 16);
                        float2 qv = *reinterpret_cast<const float2*>(qq + 2 * b);
#pragma unroll
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
                            const float m0 = qv.x * ksc * (pr.y - pr.x);
                            const float m1 = qv.y * ksc * (pr.w - pr.z);
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
                            const float m0 = qv * ksc * (pr.y - pr.x);
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
                    const int tok_in_item = (jd.ts - p.t0) + tl * 32;
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
            } else {
                // ---- fp32 key residual rows -> logits -----------------------
                const float4 qa = reinterpret_cast<const float4*>(qq)[lane];
                float mine = 0.f;
                for (int r = 0; r < jd.n; ++r) {
                    const float4 kv = reinterpret_cast<const float4*>(slot + r * D * 4)[lane];
                    float v = qa.x * kv.x + qa.y * kv.y + qa.z * kv.z + qa.w * kv.w;
                    v = warp_sum(v);
                    if (lane == r) mine = v;
                }
                if (lane < jd.n) probs[jd.ts - p.t0 + lane] = mine;
            }
            release_slot(jd.kind == KQ);
        }

        // ================= softmax over the item (log2 domain) ===============
        __syncwarp();
        float m_item, l_item;
        {
            float mx = -INFINITY;
            for (int i = lane; i < ntok; i += 32) mx = fmaxf(mx, probs[i]);
            mx = warp_max(mx);
            float sm = 0.f;
            for (int i = lane; i < ntok; i += 32) {
                const float lg = probs[i];
                if (a.wlog) a.wlog[(int64_t)u * a.l + p.t0 + i] = lg;
                const float e = ex2_approx(lg - mx);
                probs[i] = e;
                sm += e;
            }
            m_item = mx;
            l_item = warp_sum(sm);
        }
        __syncwarp();

        // ================= phase 2: P.V ======================================
        // VQ lanes: (jj, h) = token offset jj in 0..15, channel half h
        // (channels 64h .. 64h+63 = value groups 2h, 2h+1).
        const int h = lane & 1, jj = lane >> 1;
        float2 vacc[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) vacc[i] = make_float2(0.f, 0.f);
        float4 facc = make_float4(0.f, 0.f, 0.f, 0.f);
        float zacc0 = 0.f, zacc1 = 0.f;
        for (int j = nk; j < p.njobs; ++j) {
            uint8_t* slot = wait_slot();
            const JobDesc jd = job_of<B>(a, p, j);
            const float* pr_tok = probs + (jd.ts - p.t0);
            if (jd.kind == VQ) {
                const uint8_t* pairs = slot + PB::VQ_TOK * PB::TOK_CODE;
                if constexpr (B == 2) {
                    int t = jj;
                    uint4 cw = make_uint4(0, 0, 0, 0);
                    float4 pr = make_float4(0.f, 0.f, 0.f, 0.f);
                    float pt = 0.f;
                    if (t < jd.n) {
                        cw = *reinterpret_cast<const uint4*>(slot + t * PB::TOK_CODE + h * 16);
                        pr = *reinterpret_cast<const float4*>(pairs + t * 32 + h * 16);
                        pt = pr_tok[t];
                    }
                    for (; t < jd.n; t += 16) {
                        // prefetch the next token of this lane
                        const int tn = t + 16;
                        uint4 cw_n = cw;
                        float4 pr_n = pr;
                        float pt_n = pt;
                        if (tn < jd.n) {
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
                    for (int t = jj; t < jd.n; t += 16) {
                        const float pt = pr_tok[t];
                        const float4 pr = *reinterpret_cast<const float4*>(pairs + t * 32 + h * 16);
                        const float pk = pt * ksc;
                        const float ws0 = pk * (pr.y - pr.x);
                        const float ws1 = pk * (pr.w - pr.z);
                        zacc0 = fmaf(pt, pr.x, zacc0);
                        zacc1 = fmaf(pt, pr.z, zacc1);
                        const uint4 c0 =
                            *reinterpret_cast<const uint4*>(slot + t * PB::TOK_CODE + h * 32);
                        const uint4 c1 =
                            *reinterpret_cast<const uint4*>(slot + t * PB::TOK_CODE + h * 32 + 16);
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
            } else {
                // ---- fp32 value residual rows -> P.V ------------------------
                for (int r = 0; r < jd.n; ++r) {
                    const float4 vv = reinterpret_cast<const float4*>(slot + r * D * 4)[lane];
                    const float pt = pr_tok[r];
                    facc.x = fmaf(pt, vv.x, facc.x);
                    facc.y = fmaf(pt, vv.y, facc.y);
                    facc.z = fmaf(pt, vv.z, facc.z);
                    facc.w = fmaf(pt, vv.w, facc.w);
                }
            }

            if (j == p.njobs - 1) {
                // ---- finalize: reduce value accumulators, write the partial -
                // 32 rows (one per lane) x 64 channels, 16-byte chunks XOR-
                // swizzled by row so both the writes and the reads are
                // bank-conflict free.
                __syncwarp();
                float4* red = reinterpret_cast<float4*>(slot);
#pragma unroll
                for (int qc = 0; qc < 16; ++qc)
                    red[lane * 16 + (qc ^ (lane & 7))] =
                        make_float4(vacc[2 * qc].x, vacc[2 * qc].y, vacc[2 * qc + 1].x,
                                    vacc[2 * qc + 1].y);
                float z0 = zacc0, z1 = zacc1;
#pragma unroll
                for (int o = 2; o < 32; o <<= 1) {
                    z0 += __shfl_xor_sync(0xffffffffu, z0, o);
                    z1 += __shfl_xor_sync(0xffffffffu, z1, o);
                }
                __syncwarp();
                const int ho = lane >> 4;      // output channel half of this lane
                const int qc = lane & 15;      // 16-byte chunk within the half
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
                reinterpret_cast<float4*>(a.part_o + (int64_t)item * D)[lane] = o;
                if (lane == 0) a.part_ml[item] = make_float2(m_item, l_item);
            }
            release_slot(j == p.njobs - 1);
        }
    }
}

// K5: merge the per-item partials of every unit (LSE rescale in log2 domain).
__global__ void combine_kernel(const float* __restrict__ part_o, const float2* __restrict__ part_ml,
                               int n_sub, float* __restrict__ out, float2* __restrict__ stats) {
    const int64_t u = blockIdx.x;
    const int c = threadIdx.x;  // 128 threads
    float M = -INFINITY;
    for (int k = 0; k < n_sub; ++k) M = fmaxf(M, part_ml[u * n_sub + k].x);
    float L = 0.f, o = 0.f;
    for (int k = 0; k < n_sub; ++k) {
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

#undef KIVI_F

}  // namespace fast
}  // namespace kivi_b200
