// Fast fused dequant-attention decode for grouped-query attention: H query
// heads share one kv unit (BASELINE config 3: Mistral-7B, H = 4).  B = 2,
// d = 128, G = 32.
//
// Every code is extracted ONCE (denormal LOP3, as in kernels_attend_fast.cuh)
// and reused by all H heads: FFMA2 pairs heads (h, h+1) with the code
// broadcast, so a code costs ~1 LOP3 + H/2 FFMA2.
//
// Same item / job / TMA-slot machinery as the MHA tail kernel; the lane maps
// keep 16 x H accumulators per lane:
//   key tiles   lane = (tile 0..3, token half 0..1, channel slice 0..3); a
//               lane walks 32 channels of its slice (rotated so the 32 word
//               loads of a warp hit 32 distinct banks) over 16 tokens;
//               the 4 slices are transpose-reduced through the slot.
//   value rows  lane = (token offset 0..3, 16-channel slice 0..7).
#pragma once

#include "common.cuh"
#include "kernels_attend_fast.cuh"

namespace kivi_b200 {
namespace gqa {

using fast::D;
using fast::F_ROWS;
using fast::G;
using fast::SLOT;
using fast::SUB;
constexpr int WARPS = 4;

// q table row stride: 2H + 2 floats.  A key-tile step reads 16 distinct
// channels c (c mod 16 all different); with stride 2H+2 (10 or 6 floats) the
// 64-bit loads of those rows cover 32 distinct banks.
template <int H>
constexpr int QT_STRIDE = 2 * H + 2;

template <int H>
struct GS {  // per-warp shared memory
    static constexpr int QRAW_OFF = 2 * SLOT;                 // [H][128] staged q rows
    static constexpr int QT_OFF = QRAW_OFF + H * D * 4;        // [128][QT_STRIDE]: qs_h, qk_h
    static constexpr int PROBS_OFF = QT_OFF + D * QT_STRIDE<H> * 4;  // [256][H]
    static constexpr int BAR_OFF = PROBS_OFF + SUB * H * 4;
    static constexpr int BYTES = BAR_OFF + 16;
    static constexpr int STRIDE = (BYTES + 127) & ~127;
};

// acc[k * (H/2) + hp] (+)= (M[2hp], M[2hp+1]) * code_k for the 16 codes of w.
template <int H>
__device__ __forceinline__ void fma_word_heads(float2* acc, uint32_t w, const float2* M) {
    const uint32_t s = w >> 10;
    uint32_t bits[16];
#pragma unroll
    for (int k = 0; k <= 10; ++k) bits[k] = w & (3u << (2 * k));
#pragma unroll
    for (int k = 11; k < 16; ++k) bits[k] = s & (3u << (2 * k - 10));
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const float x = __uint_as_float(bits[k]);
#pragma unroll
        for (int hp = 0; hp < H / 2; ++hp)
            acc[k * (H / 2) + hp] = __ffma2_rn(M[hp], make_float2(x, x), acc[k * (H / 2) + hp]);
    }
}

template <int H>
__device__ __forceinline__ void issue_gqa_job(const fast::FastArgs& a, int u, const fast::JobDesc& jd,
                                              bool with_q, uint8_t* slot, float* qraw, uint64_t* bar,
                                              uint64_t policy) {
    // identical to the MHA tail issue, except the q copy carries H rows
    const CacheDev& c = a.c;
    const uint32_t qb = with_q ? H * D * 4 : 0;
    using PB = fast::P<2>;
    if (jd.kind == fast::KQ) {
        const int tile0 = jd.ts >> 5;
        const uint32_t cb = (uint32_t)jd.n * PB::TILE_CODE;
        const uint32_t pb = (uint32_t)jd.n * D * 8;
        mbar_arrive_expect_tx(bar, cb + pb + qb);
        bulk_g2s_evict_first(slot, c.kcodes + u * c.k_ustride + (int64_t)tile0 * PB::TILE_CODE, cb,
                             bar, policy);
        bulk_g2s_evict_first(slot + PB::KQ_TILES * PB::TILE_CODE,
                             c.kpairs + u * c.kp_ustride + (int64_t)tile0 * D, pb, bar, policy);
    } else if (jd.kind == fast::VQ) {
        const uint32_t cb = (uint32_t)jd.n * PB::TOK_CODE;
        const uint32_t pb = (uint32_t)jd.n * (D / G) * 8;
        mbar_arrive_expect_tx(bar, cb + pb + qb);
        bulk_g2s_evict_first(slot, c.vcodes + u * c.v_ustride + (int64_t)jd.ts * PB::TOK_CODE, cb,
                             bar, policy);
        bulk_g2s_evict_first(slot + PB::VQ_TOK * PB::TOK_CODE,
                             c.vpairs + u * c.vp_ustride + (int64_t)jd.ts * (D / G), pb, bar,
                             policy);
    } else if (jd.kind == fast::KF) {
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
    if (with_q) bulk_g2s(qraw, a.q + (int64_t)u * H * D, qb, bar);
}

// Quantized key tiles -> logits of H heads (probs layout [token][H]).
template <int H>
__device__ __forceinline__ void kq_tiles_heads(uint8_t* slot, const float* qt, float* probs_dst,
                                               int ntiles, int lane) {
    const int tl = lane >> 3, hf = (lane >> 2) & 1, sl = lane & 3;
    const int rot = tl * 4 + sl;  // bank rotation (see file comment)
    float2 acc[16 * H / 2];
#pragma unroll
    for (int i = 0; i < 16 * H / 2; ++i) acc[i] = make_float2(0.f, 0.f);
    float2 bias[H / 2];
#pragma unroll
    for (int hp = 0; hp < H / 2; ++hp) bias[hp] = make_float2(0.f, 0.f);
    if (tl < ntiles) {
        const uint8_t* codes = slot + tl * 1024;
        const uint8_t* pairs = slot + 4 * 1024 + tl * 1024;
#pragma unroll 2
        for (int i = 0; i < 32; ++i) {
            const int c = sl * 32 + ((i + rot) & 31);
            const uint32_t w = *reinterpret_cast<const uint32_t*>(codes + c * 8 + hf * 4);
            const float2 pr = *reinterpret_cast<const float2*>(pairs + c * 8);
            const float* q = qt + c * QT_STRIDE<H>;
            float2 M[H / 2];
            const float diff = pr.y - pr.x;
#pragma unroll
            for (int hp = 0; hp < H / 2; ++hp) {
                const float2 qs = *reinterpret_cast<const float2*>(q + 2 * hp);
                const float2 qk = *reinterpret_cast<const float2*>(q + H + 2 * hp);
                M[hp] = __fmul2_rn(qk, make_float2(diff, diff));
                bias[hp] = __ffma2_rn(qs, make_float2(pr.x, pr.x), bias[hp]);
            }
            fma_word_heads<H>(acc, w, M);
        }
    }
    // bias over the 4 channel slices of a (tile, half)
#pragma unroll
    for (int hp = 0; hp < H / 2; ++hp) {
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
            bias[hp].x += __shfl_xor_sync(0xffffffffu, bias[hp].x, o);
            bias[hp].y += __shfl_xor_sync(0xffffffffu, bias[hp].y, o);
        }
    }
    // transpose-reduce: row = lane, 16*H floats (value k*H + h), XOR-swizzled
    // 16-byte chunks; lane sl then owns tokens 4sl..4sl+3 of its (tile, half)
    __syncwarp();
    float4* red = reinterpret_cast<float4*>(slot);
    constexpr int CH = 4 * H;  // 16-byte chunks per row
#pragma unroll
    for (int q4 = 0; q4 < CH; ++q4)
        red[lane * CH + (q4 ^ (lane & 7))] = make_float4(acc[2 * q4].x, acc[2 * q4].y,
                                                         acc[2 * q4 + 1].x, acc[2 * q4 + 1].y);
    __syncwarp();
    if (tl < ntiles) {
        const int row0 = lane & ~3;
#pragma unroll
        for (int kk0 = 0; kk0 < 4; ++kk0) {
            // lane-dependent order: the 8 lanes of a load phase hit 8 slots
            const int kk = kk0 ^ (sl >> 1) ^ (hf << 1);
            const int k = 4 * sl + kk;  // token within the half
            float v[H];
#pragma unroll
            for (int h = 0; h < H; ++h) v[h] = 0.f;
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                const int row = row0 + s2;
#pragma unroll
                for (int h4 = 0; h4 < H; h4 += 4 > H ? H : 4) {
                    // values k*H .. k*H+H-1 live in chunk(s) (k*H)/4 ..
                    const int q4 = (k * H + h4) >> 2;
                    const float4 t4 = red[row * CH + (q4 ^ (row & 7))];
                    if constexpr (H == 4) {
                        v[0] += t4.x; v[1] += t4.y; v[2] += t4.z; v[3] += t4.w;
                    } else {
                        const bool hi = ((k * H) & 3) != 0;
                        v[0] += hi ? t4.z : t4.x;
                        v[1] += hi ? t4.w : t4.y;
                    }
                }
            }
            const float sc = fast::unscale_pos(fast::P<2>::epos(k));
            float* dst = probs_dst + (tl * 32 + hf * 16 + k) * H;
#pragma unroll
            for (int hp = 0; hp < H / 2; ++hp) {
                dst[2 * hp] = fmaf(v[2 * hp], sc, bias[hp].x);
                dst[2 * hp + 1] = fmaf(v[2 * hp + 1], sc, bias[hp].y);
            }
        }
    }
}

// fp32 key residual rows -> logits of H heads.  Lane = (row r = lane / 2,
// e = lane % 2): at H = 4, e picks the head pair and the lane runs the whole
// 128-channel dot product for both heads with FFMA2 (no cross-lane reduction);
// at H = 2, e picks a channel half and one shuffle adds the halves.  The
// row's float4 chunks are visited from a row-rotated start so the 16 rows
// of a job (512 B apart) hit distinct banks.  (Was: per-head lane-per-channel
// partials + a 16-way shuffle reduce-scatter, ~4x the instructions.)
template <int H>
__device__ __forceinline__ void kf_rows_heads(const uint8_t* slot, const float* qt, float* probs_dst,
                                              int n, int lane) {
    static_assert(H == 2 || H == 4, "kf_rows_heads: H in {2, 4}");
    const int r = lane >> 1, e = lane & 1;
    const float4* row = reinterpret_cast<const float4*>(slot + r * D * 4);
    constexpr int NCH = H == 4 ? 32 : 16;   // float4 chunks per lane
    const int hp = H == 4 ? e : 0;          // head pair
    const int c0 = H == 4 ? 0 : 16 * e;     // first chunk of this lane's half
    float2 acc = make_float2(0.f, 0.f), acc1 = acc;
    if (r < n) {
#pragma unroll 4
        for (int i = 0; i < NCH; ++i) {
            const int c4 = c0 + ((i + r) & (NCH - 1));
            const float4 kv = row[c4];
            const float* q = qt + (4 * c4) * QT_STRIDE<H> + 2 * hp;
            acc = __ffma2_rn(*reinterpret_cast<const float2*>(q), make_float2(kv.x, kv.x), acc);
            acc1 = __ffma2_rn(*reinterpret_cast<const float2*>(q + QT_STRIDE<H>),
                              make_float2(kv.y, kv.y), acc1);
            acc = __ffma2_rn(*reinterpret_cast<const float2*>(q + 2 * QT_STRIDE<H>),
                             make_float2(kv.z, kv.z), acc);
            acc1 = __ffma2_rn(*reinterpret_cast<const float2*>(q + 3 * QT_STRIDE<H>),
                              make_float2(kv.w, kv.w), acc1);
        }
    }
    acc.x += acc1.x;
    acc.y += acc1.y;
    if constexpr (H == 2) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
        if (r < n && e == 0) *reinterpret_cast<float2*>(probs_dst + r * H) = acc;
    } else {
        if (r < n) *reinterpret_cast<float2*>(probs_dst + r * H + 2 * hp) = acc;
    }
}

// Softmax of each head over the item (in place, log2 domain).
template <int H>
__device__ __forceinline__ void softmax_heads(float* probs, int ntok, float* wlog, int64_t wrow_stride,
                                              float2* ml, int lane) {
    __syncwarp();
#pragma unroll
    for (int h = 0; h < H; ++h) {
        float mx = -INFINITY;
        for (int i = lane; i < ntok; i += 32) mx = fmaxf(mx, probs[i * H + h]);
        mx = warp_max(mx);
        float sm = 0.f;
        for (int i = lane; i < ntok; i += 32) {
            const float lg = probs[i * H + h];
            if (wlog) wlog[h * wrow_stride + i] = lg;
            const float e = fast::ex2_approx(lg - mx);
            probs[i * H + h] = e;
            sm += e;
        }
        ml[h] = make_float2(mx, warp_sum(sm));
    }
    __syncwarp();
}

// Quantized value tokens -> P.V for H heads.
template <int H>
__device__ __forceinline__ void vq_tokens_heads(const uint8_t* slot, const float* pr_tok, int n,
                                                float ksc, float2* vacc, float* zacc, int lane) {
    const int jj = lane >> 3, cs = lane & 7;
    const uint8_t* pairs = slot + 128 * 32;
    for (int t = jj; t < n; t += 4) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(slot + t * 32 + cs * 4);
        const float2 pr = *reinterpret_cast<const float2*>(pairs + t * 32 + (cs >> 1) * 8);
        const float* p = pr_tok + t * H;
        const float dk = (pr.y - pr.x) * ksc;
        float2 ws[H / 2];
#pragma unroll
        for (int hp = 0; hp < H / 2; ++hp) {
            const float2 p2 = *reinterpret_cast<const float2*>(p + 2 * hp);
            ws[hp] = __fmul2_rn(p2, make_float2(dk, dk));
            zacc[2 * hp] = fmaf(p2.x, pr.x, zacc[2 * hp]);
            zacc[2 * hp + 1] = fmaf(p2.y, pr.x, zacc[2 * hp + 1]);
        }
        fma_word_heads<H>(vacc, w, ws);
    }
}

// fp32 value residual rows -> P.V (lane owns channels 4*lane..4*lane+3).
template <int H>
__device__ __forceinline__ void vf_rows_heads(const uint8_t* slot, const float* pr_tok, int n,
                                              float* facc, int lane) {
    for (int r = 0; r < n; ++r) {
        const float4 vv = reinterpret_cast<const float4*>(slot + r * D * 4)[lane];
#pragma unroll
        for (int h = 0; h < H; ++h) {
            const float pt = pr_tok[r * H + h];
            facc[h * 4 + 0] = fmaf(pt, vv.x, facc[h * 4 + 0]);
            facc[h * 4 + 1] = fmaf(pt, vv.y, facc[h * 4 + 1]);
            facc[h * 4 + 2] = fmaf(pt, vv.z, facc[h * 4 + 2]);
            facc[h * 4 + 3] = fmaf(pt, vv.w, facc[h * 4 + 3]);
        }
    }
}

// Reduce the value accumulators over the 4 token offsets and write the item's
// H partials (lane L owns channels 4L..4L+3 of every head).
template <int H>
__device__ __forceinline__ void v_finalize_heads(uint8_t* slot, const float2* vacc, const float* zacc,
                                                 const float* facc, const float2* ml, float* part_o,
                                                 float2* part_ml, int lane) {
    __syncwarp();
    float4* red = reinterpret_cast<float4*>(slot);
    constexpr int CH = 4 * H;  // chunks per row: value index m*H + h (m = channel in slice)
#pragma unroll
    for (int q4 = 0; q4 < CH; ++q4)
        red[lane * CH + (q4 ^ (lane & 7))] = make_float4(vacc[2 * q4].x, vacc[2 * q4].y,
                                                         vacc[2 * q4 + 1].x, vacc[2 * q4 + 1].y);
    float z[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
        float zz = zacc[h];
        zz += __shfl_xor_sync(0xffffffffu, zz, 8);
        zz += __shfl_xor_sync(0xffffffffu, zz, 16);
        // output lane L's group is L >> 3; lane (jj=0, cs=2*group) holds it
        z[h] = __shfl_sync(0xffffffffu, zz, 2 * (lane >> 3));
    }
    __syncwarp();
    const int cs = lane >> 2;         // 16-channel slice holding channels 4L..4L+3
    const int m0 = 4 * (lane & 3);    // first channel within the slice
    float out[H][4];
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
        for (int i = 0; i < 4; ++i) out[h][i] = 0.f;
#pragma unroll
    for (int j2 = 0; j2 < 4; ++j2) {
        const int row = j2 * 8 + cs;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int m = m0 + i;
            if constexpr (H == 4) {
                const float4 t4 = red[row * CH + (m ^ (row & 7))];
                out[0][i] += t4.x; out[1][i] += t4.y; out[2][i] += t4.z; out[3][i] += t4.w;
            } else {
                const int q4 = (m * H) >> 2;
                const float4 t4 = red[row * CH + (q4 ^ (row & 7))];
                const bool hi = ((m * H) & 3) != 0;
                out[0][i] += hi ? t4.z : t4.x;
                out[1][i] += hi ? t4.w : t4.y;
            }
        }
    }
#pragma unroll
    for (int h = 0; h < H; ++h) {
        float4 o;
        o.x = fmaf(out[h][0], fast::unscale_pos(fast::P<2>::epos(m0 + 0)), z[h]) + facc[h * 4 + 0];
        o.y = fmaf(out[h][1], fast::unscale_pos(fast::P<2>::epos(m0 + 1)), z[h]) + facc[h * 4 + 1];
        o.z = fmaf(out[h][2], fast::unscale_pos(fast::P<2>::epos(m0 + 2)), z[h]) + facc[h * 4 + 2];
        o.w = fmaf(out[h][3], fast::unscale_pos(fast::P<2>::epos(m0 + 3)), z[h]) + facc[h * 4 + 3];
        reinterpret_cast<float4*>(part_o + h * D)[lane] = o;
    }
#pragma unroll
    for (int h = 0; h < H; ++h)
        if (lane == h) part_ml[h] = ml[h];
}

// Item order: sub-chunk-major with the LAST sub-chunk first.  Item i -> unit
// i mod U, sub-chunk n_per_unit-1 - i/U.  The heavy items (the ones holding
// fp32 residual rows) are then the first U items and spread over U warps; in
// unit-major order with a static stride they all landed on the few warps
// whose index is = n_per_unit-1 (mod n_per_unit) and idled 31 % of the SMs.
__device__ __forceinline__ fast::ItemPlan plan_gqa(const fast::FastArgs& a, int i) {
    const int nu = a.n_items / a.n_per_unit;
    const int kk = i / nu;
    const int u = i - kk * nu;
    return fast::plan_item<2>(a, u * a.n_per_unit + (a.n_per_unit - 1 - kk));
}

// NW warps per CTA: 4 when this kernel runs every item; 1 when it runs only
// the residual-window items beside the tensor-core body kernel, so its
// shared memory leaves room for two body CTAs on the same SM.
template <int H, int NW = WARPS>
__global__ void __launch_bounds__(NW * 32, 2) attend_gqa_kernel(fast::FastArgs a) {
    using WS = GS<H>;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* wbase = smem_raw + warp * WS::STRIDE;
    float* qraw = reinterpret_cast<float*>(wbase + WS::QRAW_OFF);
    float* qt = reinterpret_cast<float*>(wbase + WS::QT_OFF);
    float* probs = reinterpret_cast<float*>(wbase + WS::PROBS_OFF);
    uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + WS::BAR_OFF);
    if (lane == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const uint64_t policy = make_evict_first_policy();
    const int gw = blockIdx.x * NW + warp;
    const int tw = gridDim.x * NW;
    const float ksc = fast::TWO_POW_64 / 3.0f;

    int f_item = gw, f_job = 0;
    fast::ItemPlan f_plan{};
    if (f_item < a.n_items) f_plan = plan_gqa(a, f_item);
    auto issue_next = [&](int s) {
        if (f_item >= a.n_items) return;
        if (lane == 0) {
            const fast::JobDesc jd = fast::job_of<2>(a, f_plan, f_job);
            fence_proxy_async_smem();
            issue_gqa_job<H>(a, f_plan.u, jd, f_job == 0, wbase + s * SLOT, qraw, &bars[s], policy);
        }
        if (++f_job == f_plan.njobs) {
            f_item += tw;
            f_job = 0;
            if (f_item < a.n_items) f_plan = plan_gqa(a, f_item);
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

    for (int item = gw; item < a.n_items; item += tw) {
        const fast::ItemPlan p = plan_gqa(a, item);
        const int nk = p.nkq + p.nkf;
        for (int j = 0; j < nk; ++j) {
            uint8_t* slot = wait_slot();
            if (j == 0) {
                // q table: qt[c][h] = q_h,c * scale * log2e, qt[c][H+h] = that * ksc
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    const float4 qv = reinterpret_cast<const float4*>(qraw + h * D)[lane];
                    const float v[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float qs = v[i] * a.qscale;
                        qt[(4 * lane + i) * QT_STRIDE<H> + h] = qs;
                        qt[(4 * lane + i) * QT_STRIDE<H> + H + h] = qs * ksc;
                    }
                }
                __syncwarp();
            }
            const fast::JobDesc jd = fast::job_of<2>(a, p, j);
            if (jd.kind == fast::KQ)
                kq_tiles_heads<H>(slot, qt, probs + (jd.ts - p.t0) * H, jd.n, lane);
            else
                kf_rows_heads<H>(slot, qt, probs + (jd.ts - p.t0) * H, jd.n, lane);
            release_slot();
        }
        float2 ml[H];
        softmax_heads<H>(probs, p.t1 - p.t0,
                         a.wlog ? a.wlog + ((int64_t)p.u * H) * a.l + p.t0 : nullptr, a.l, ml,
                         lane);
        float2 vacc[16 * H / 2];
#pragma unroll
        for (int i = 0; i < 16 * H / 2; ++i) vacc[i] = make_float2(0.f, 0.f);
        float zacc[H], facc[4 * H];
#pragma unroll
        for (int h = 0; h < H; ++h) zacc[h] = 0.f;
#pragma unroll
        for (int i = 0; i < 4 * H; ++i) facc[i] = 0.f;
        for (int j = nk; j < p.njobs; ++j) {
            uint8_t* slot = wait_slot();
            const fast::JobDesc jd = fast::job_of<2>(a, p, j);
            const float* pr_tok = probs + (jd.ts - p.t0) * H;
            if (jd.kind == fast::VQ)
                vq_tokens_heads<H>(slot, pr_tok, jd.n, ksc, vacc, zacc, lane);
            else
                vf_rows_heads<H>(slot, pr_tok, jd.n, facc, lane);
            if (j == p.njobs - 1) {
                const int64_t pi = ((int64_t)p.u * a.n_sub + p.k) * H;
                v_finalize_heads<H>(slot, vacc, zacc, facc, ml, a.part_o + pi * D, a.part_ml + pi,
                                    lane);
            }
            release_slot();
        }
    }
}

// K5 for H heads: rows r = u*H + h; partial (u, k, h) at (u*n_sub + k)*H + h.
__global__ void __launch_bounds__(128) combine_heads_kernel(const float* __restrict__ part_o,
                                                            const float2* __restrict__ part_ml,
                                                            int n_sub, int H,
                                                            float* __restrict__ out,
                                                            float2* __restrict__ stats,
                                                            int parallel, int64_t n_rows) {
    if (parallel == 2) {  // one warp per row, four rows per block
        const int64_t r = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
        if (r < n_rows)
            fast::combine_row_warp(part_o, part_ml, n_sub, (r / H) * n_sub * H + r % H, H,
                                   out + r * D, stats ? stats + r : nullptr, threadIdx.x & 31);
        return;
    }
    const int64_t r = blockIdx.x;
    const int64_t u = r / H, h = r % H;
    if (parallel)
        fast::combine_row(part_o, part_ml, n_sub, u * n_sub * H + h, H, out + r * D,
                          stats ? stats + r : nullptr);
    else
        fast::combine_row_serial(part_o, part_ml, n_sub, u * n_sub * H + h, H, out + r * D,
                                 stats ? stats + r : nullptr);
}

}  // namespace gqa
}  // namespace kivi_b200
