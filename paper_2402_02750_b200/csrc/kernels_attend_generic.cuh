// Generic decode attention: any B, G, R, d, q_per_kv.  Follows the reference
// arithmetic order of decode_attention (proj/src/attention.cpp:36-99):
//   * grouped key logits accumulated in double over channels c = 0..d-1,
//     term q_c * (code*s + z), cast to float                       (:40-62)
//   * residual key logits: sequential float dot product             (:63-66)
//   * logits *= 1/sqrt(d) in float                                  (:67)
//   * softmax: max, exp(x - max), sequential float sum, divide      (:70, matrix.hpp:31-39)
//   * grouped values: double accumulation over tokens t = 0..vg-1   (:73-90)
//   * residual values: sequential float sum; out = resid + float(acc) (:91-98)
// One CTA per (unit, query head).  Used for shapes the fast kernel does not
// cover, for the C++ drop-in facade, and for reference_attention (kg=vg=0).
#pragma once

#include "common.cuh"
#include "kernels_quant.cuh"

namespace kivi_b200 {

struct AttendGenericArgs {
    CacheDev c;
    int64_t l, kg, vg;
    int64_t ring_mod;  // value residual row of token t = t % ring_mod (R, or l for ref attention)
    const float* q;    // [units][qpk][d]
    int qpk;
    float* out;        // [units][qpk][d]
    float* weights;    // [units][qpk][l] or null
    float* scratch;    // [units][qpk][l]
    int scale_logits;
};

// exp rounded from a double evaluation (closest float to e^x in practice).
__device__ __forceinline__ float expf_accurate(float x) { return (float)exp((double)x); }

// Group scales (the reference's double (hi - lo) / maxc) are computed once per
// group into shared memory, a batch of key tiles / value tokens at a time,
// instead of once per code (a DDIV per element): the same doubles, the same
// summation order, so the outputs are unchanged bit for bit.
constexpr int GEN_SC_CAP = 1024;  // cached (scale, zero) entries: 12 KB

__global__ void attend_generic_kernel(AttendGenericArgs a) {
    extern __shared__ float smem[];
    const CacheDev& c = a.c;
    const int d = c.d, G = c.G;
    const int64_t u = blockIdx.x / a.qpk;
    const int h = blockIdx.x % a.qpk;
    const int64_t row = u * a.qpk + h;
    float* sq = smem;             // d
    float* red = smem + d;        // 32 floats
    double* sS = reinterpret_cast<double*>(smem + ((d + 32 + 1) & ~1));  // GEN_SC_CAP
    float* sZ = reinterpret_cast<float*>(sS + GEN_SC_CAP);                // GEN_SC_CAP
    const float* q = a.q + row * d;
    for (int ch = threadIdx.x; ch < d; ch += blockDim.x) sq[ch] = q[ch];
    __syncthreads();

    const float scale = a.scale_logits ? __fdiv_rn(1.0f, __fsqrt_rn((float)d)) : 1.0f;
    const int64_t l = a.l, kg = a.kg, vg = a.vg;
    float* lg = a.scratch + row * l;
    const uint8_t* kc = c.kcodes + u * c.k_ustride;
    const float2* kp = c.kpairs + u * c.kp_ustride;
    const uint8_t* vc = c.vcodes + u * c.v_ustride;
    const float2* vp = c.vpairs + u * c.vp_ustride;
    const float* kr = c.kring + u * c.ring_ustride;
    const float* vr = c.vring + u * c.ring_ustride;

    // 1. logits of the grouped keys: nt tiles at a time (their d x nt scales
    //    cached), one thread per token, channels in order
    {
        const int T = max(1, min((int)blockDim.x / G, GEN_SC_CAP / d));
        const int64_t ntiles = kg / G;
        for (int64_t tg0 = 0; tg0 < ntiles; tg0 += T) {
            const int nt = (int)(ntiles - tg0 < T ? ntiles - tg0 : T);
            if (d <= GEN_SC_CAP) {
                for (int e = threadIdx.x; e < nt * d; e += blockDim.x) {
                    const float2 pr = kp[(tg0 + e / d) * d + e % d];
                    sS[e] = group_scale(pr.x, pr.y, c.maxc);
                    sZ[e] = pr.x;
                }
            }
            __syncthreads();
            for (int j = threadIdx.x; j < nt * G; j += blockDim.x) {
                const int tt = j / G, i = j % G;
                const int64_t tg = tg0 + tt, t = tg * G + i;
                double acc = 0.0;
                for (int ch = 0; ch < d; ++ch) {
                    const int64_t g = tg * d + ch;
                    double s;
                    float z;
                    if (d <= GEN_SC_CAP) {
                        s = sS[tt * d + ch];
                        z = sZ[tt * d + ch];
                    } else {
                        const float2 pr = kp[g];
                        s = group_scale(pr.x, pr.y, c.maxc);
                        z = pr.x;
                    }
                    const uint32_t code = read_code(kc, ((uint64_t)g * G + i) * c.bits, c.bits);
                    const double deq = __dadd_rn(__dmul_rn((double)code, s), (double)z);
                    acc = __dadd_rn(acc, __dmul_rn((double)sq[ch], deq));
                }
                lg[t] = __fmul_rn((float)acc, scale);
            }
            __syncthreads();
        }
    }
    // residual keys
    for (int64_t t = kg + threadIdx.x; t < l; t += blockDim.x) {
        const float* kv = kr + (t - kg) * d;
        float acc = 0.0f;
        for (int ch = 0; ch < d; ++ch) acc = __fadd_rn(acc, __fmul_rn(sq[ch], kv[ch]));
        lg[t] = __fmul_rn(acc, scale);
    }
    __syncthreads();

    // 2. max (order-independent)
    float m = -INFINITY;
    for (int64_t t = threadIdx.x; t < l; t += blockDim.x) m = fmaxf(m, lg[t]);
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
        v = warp_max(v);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    m = red[0];
    __syncthreads();

    // 3. exponentials, then the reference's sequential sum and divide
    for (int64_t t = threadIdx.x; t < l; t += blockDim.x) lg[t] = expf_accurate(__fsub_rn(lg[t], m));
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.0f;
        for (int64_t t = 0; t < l; ++t) s = __fadd_rn(s, lg[t]);
        red[1] = s;
    }
    __syncthreads();
    const float sum = red[1];
    for (int64_t t = threadIdx.x; t < l; t += blockDim.x) {
        const float w = __fdiv_rn(lg[t], sum);
        lg[t] = w;
        if (a.weights) a.weights[row * l + t] = w;
    }
    __syncthreads();

    // 4. outputs: grouped values in token chunks (their scales cached), one
    //    thread per channel (up to 8 channels per thread), tokens in order
    const int gpt = d / G;
    constexpr int CPT = 8;
    if (d <= CPT * (int)blockDim.x && gpt <= GEN_SC_CAP) {
        double acc[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) acc[k] = 0.0;
        const int TC = max(1, GEN_SC_CAP / gpt);
        for (int64_t t0 = 0; t0 < vg; t0 += TC) {
            const int nt = (int)(vg - t0 < TC ? vg - t0 : TC);
            for (int e = threadIdx.x; e < nt * gpt; e += blockDim.x) {
                const float2 pr = vp[t0 * gpt + e];
                sS[e] = group_scale(pr.x, pr.y, c.maxc);
                sZ[e] = pr.x;
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                const int ch = threadIdx.x + k * blockDim.x;
                if (ch < d) {
                    double ac = acc[k];
                    for (int tt = 0; tt < nt; ++tt) {
                        const int64_t t = t0 + tt;
                        const double w = (double)lg[t];
                        const int e = tt * gpt + ch / G;
                        const uint32_t code = read_code(vc, ((uint64_t)t * d + ch) * c.bits, c.bits);
                        ac = __dadd_rn(ac, __dmul_rn(w, __dadd_rn(__dmul_rn((double)code, sS[e]),
                                                                  (double)sZ[e])));
                    }
                    acc[k] = ac;
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const int ch = threadIdx.x + k * blockDim.x;
            if (ch < d) {
                float r = 0.0f;
                for (int64_t t = vg; t < l; ++t)
                    r = __fadd_rn(r, __fmul_rn(lg[t], vr[(t % a.ring_mod) * d + ch]));
                a.out[row * d + ch] = vg > 0 ? __fadd_rn(r, (float)acc[k]) : r;
            }
        }
        return;
    }
    for (int ch = threadIdx.x; ch < d; ch += blockDim.x) {
        double acc = 0.0;
        for (int64_t t = 0; t < vg; ++t) {
            const double w = (double)lg[t];
            const int64_t g = t * gpt + ch / G;
            const float2 pr = vp[g];
            const double s = group_scale(pr.x, pr.y, c.maxc);
            const uint32_t code = read_code(vc, ((uint64_t)t * d + ch) * c.bits, c.bits);
            acc = __dadd_rn(acc, __dmul_rn(w, __dadd_rn(__dmul_rn((double)code, s), (double)pr.x)));
        }
        float r = 0.0f;
        for (int64_t t = vg; t < l; ++t)
            r = __fadd_rn(r, __fmul_rn(lg[t], vr[(t % a.ring_mod) * d + ch]));
        a.out[row * d + ch] = vg > 0 ? __fadd_rn(r, (float)acc) : r;
    }
}

}  // namespace kivi_b200
