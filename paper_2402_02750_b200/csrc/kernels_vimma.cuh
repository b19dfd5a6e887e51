// P.V of the MHA body on the integer tensor cores (B = 2, d = 128, G = 32):
// mma.sync m16n8k32 u8 x u8 -> s32, exact integer accumulation.
//
//   out_c = sum_t p_t (code_tc * s_t,cg + z_t,cg)
//         = (1/3) sum_t code_tc * (p_t * (hi - lo)_t,cg) + sum_t p_t lo_t,cg
//
// A = the 2-bit value codes as u8 (exact), M = 16 channels x K = 32 tokens.
// B = x_t,cg = round(p_t (hi - lo)_t,cg 2^(31 - E)) split into its four
//     bytes (digits d = 0..3, x = sum_d byte_d 256^d), N = 8 columns =
//     (channel-group half, digit); 2^E bounds the item's spans (all channel
//     groups), so x < 2^31 and the four digit products sum exactly in int32
//     (<= 255 * 3 * 256 per column per item).
// The fixed point carries 31 bits below the item's largest span (p <= 1):
// its error is ~2^-31 of the largest term, below fp32 accumulation's.
//
// Why: the CUDA-core value loop spends one LOP3 per code (ALU pipe, half
// rate) plus half an FFMA2 and is what keeps the body ALU-bound.  Here
// ldmatrix.trans + two PRMTs put 4 tokens x 8 channels of one lane's codes in
// K order and one shift + LOP3 yields FOUR codes (one u8 per byte): ~0.5
// issue slots per code for the operands, 1/16 MMA per code.
//
// Fragment mapping (lane = (g, t4), g = lane / 4, t4 = lane % 4):
//   ldmatrix.x4.trans over a 32-token K block, matrix m = tokens 8m..8m+7,
//   row = token, 16 bytes = channels 64e..64e+63 (half e): register R_m =
//   [tok 8m+2t4: channels 64e+8g..+3, +4..+7 | tok 8m+2t4+1: same].
//   PRMT(R0, R1) -> the K-group tokens (2t4, 2t4+1, 8+2t4, 9+2t4) of one
//   4-channel byte; (P >> 2i) & 0x03030303 = channel 64e+8g+i' of those 4
//   tokens = one A register (row = channel, 4 K = 4 tokens).
//   M-block j (0..3): rows g <-> channel 64e+8g+2j, g+8 <-> 64e+8g+2j+1;
//   its rows span two channel groups (2e + g/4), hence the (cg half, digit)
//   columns: a row's value uses the 4 columns of its own group half.
#pragma once

#include "common.cuh"

namespace kivi_b200 {
namespace vimma {

constexpr uint32_t FULL = 0xffffffffu;

__device__ __forceinline__ void imma(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                     uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                              uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

// x >> 2, x >> 4 as IMAD.HI (FMA pipe; the ALU pipe carries the masks)
__device__ __forceinline__ uint32_t shr2(uint32_t x) { return __umulhi(x, 1u << 30); }
__device__ __forceinline__ uint32_t shr4(uint32_t x) { return __umulhi(x, 1u << 28); }

// 2^k as a float for k in [-126, 127]
__device__ __forceinline__ float pow2f(int k) { return __uint_as_float((uint32_t)(k + 127) << 23); }

// Per-warp state of an item's value phase (registers).
struct State {
    int D[2][4][4];   // [channel half e][M-block j][mma regs]
    float F[2][4][2]; // [e][j][row g, g + 8]: D flushed at an exponent change
    int E;            // running span exponent of the item (all channel groups)
    float z;          // producer lane's share of sum_t p_t lo_t,cg (cg = lane % 4)
    bool first;
};

// Digit weights of this lane's two D columns (2 t4, 2 t4 + 1 = digits
// 2 (t4 % 2), 2 (t4 % 2) + 1) and the full value sum_d D_d 256^d of rows g
// and g + 8 (the partner lane t4 ^ 1 holds the other two digits).
__device__ __forceinline__ void combine_digits(const int (&d)[4], int t4, float& a, float& b) {
    const float dw0 = (t4 & 1) ? 65536.f : 1.f;
    const float dw1 = (t4 & 1) ? 16777216.f : 256.f;
    a = fmaf((float)d[1], dw1, (float)d[0] * dw0);
    b = fmaf((float)d[3], dw1, (float)d[2] * dw0);
    a += __shfl_xor_sync(FULL, a, 1);
    b += __shfl_xor_sync(FULL, b, 1);
}

__device__ __forceinline__ void begin_item(State& st) {
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int r = 0; r < 4; ++r) st.D[e][j][r] = 0;
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int j = 0; j < 4; ++j) st.F[e][j][0] = st.F[e][j][1] = 0.f;
    st.z = 0.f;
    st.first = true;
}

// Digit words of one 32-token K block: 8 K-group rows x 16 words (4 channel
// groups x 4 digits); rows 2, 3, 6, 7 XOR the word index with 8, so the
// consumer reads (lane (g, t4): row t4 or 4 + t4, word 8e + g) hit 32
// distinct banks.
__device__ __forceinline__ int dig_word(int kg, int w) { return kg * 16 + (w ^ (((kg >> 1) & 1) << 3)); }

// One value job: NTOK (multiple of 32) tokens, slot = [NTOK][32 B] codes then
// [NTOK][4] (lo, hi) pairs; p = the job's probabilities.  The pairs are read
// once into registers; their space then holds the B digits of every K block
// (NTOK / 32 x 512 B), so producing and consuming need a single warp barrier.
template <int NTOK>
__device__ __forceinline__ void value_job(uint8_t* slot, const float* p, State& st, int lane) {
    static_assert(NTOK % 32 == 0, "whole 32-token K blocks");
    static_assert(NTOK * 16 <= NTOK * 32, "digits fit in the pairs region");
    constexpr int NKB = NTOK / 32;
    const float2* pairs = reinterpret_cast<const float2*>(slot + NTOK * 32);
    uint32_t* dig = reinterpret_cast<uint32_t*>(slot + NTOK * 32);
    // producer role: lane = (K-group kg, channel group cg)
    const int kg = lane >> 2, cg = lane & 3;
    const int tk0 = 16 * (kg >> 2) + 2 * (kg & 3);  // K-group tokens: tk0 + {0, 1, 8, 9}
    // spans of this lane's tokens (all K blocks), job-wide max per cg
    float span[NKB][4], pt[NKB][4];
    float smax = 0.f;
#pragma unroll
    for (int kb = 0; kb < NKB; ++kb)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int t = 32 * kb + tk0 + (i & 1) + 8 * (i >> 1);
            const float2 pr = pairs[t * 4 + cg];
            pt[kb][i] = p[t];
            span[kb][i] = pr.y - pr.x;
            smax = fmaxf(smax, span[kb][i]);
            st.z = fmaf(pt[kb][i], pr.x, st.z);
        }
    // one exponent for the job's four channel groups: a warp max (CREDUX).  A
    // group whose spans are 2^k below the job's largest keeps 31 - k bits of
    // fixed point, still far below the fp32 rounding it replaces.
    smax = warp_max_redux(smax);
    // smax < 2^E; E >= -90 keeps 2^(31 - E) and 2^(E - 31) normal floats
    // (all-constant groups have smax = 0 and x = 0)
    const int ej = max((int)((__float_as_uint(smax) >> 23) & 0xFFu) - 126, -90);
    // consumer role: lane = (g, t4)
    const int g = lane >> 2, t4 = lane & 3;
    if (!st.first && ej > st.E) {  // warp-uniform, rare
        // larger spans than the item's earlier jobs: the integer sums move to
        // fp32 at the old scale (digit columns cannot be shifted one by one:
        // the bits a digit column drops belong to the column below), then
        // restart at 0
        const float sc_old = pow2f(st.E - 31);
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float a, b;
                combine_digits(st.D[e][j], t4, a, b);
                st.F[e][j][0] = fmaf(a, sc_old, st.F[e][j][0]);
                st.F[e][j][1] = fmaf(b, sc_old, st.F[e][j][1]);
#pragma unroll
                for (int r = 0; r < 4; ++r) st.D[e][j][r] = 0;
            }
    }
    st.E = st.first ? ej : max(st.E, ej);
    const int eprod = st.E;
    st.first = false;
    const float xscale = pow2f(31 - eprod);
    __syncwarp();  // every lane has read its pairs: the region now takes the digits
    // ---- producer: digits of x for (K-group kg, group cg), every K block ----
#pragma unroll
    for (int kb = 0; kb < NKB; ++kb) {
        uint32_t x[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = __float2uint_rn((pt[kb][i] * span[kb][i]) * xscale);
        const uint32_t lo01 = __byte_perm(x[0], x[1], 0x5140), lo23 = __byte_perm(x[2], x[3], 0x5140);
        const uint32_t hi01 = __byte_perm(x[0], x[1], 0x7362), hi23 = __byte_perm(x[2], x[3], 0x7362);
        *reinterpret_cast<uint4*>(dig + kb * 128 + dig_word(kg, 4 * cg)) =
            make_uint4(__byte_perm(lo01, lo23, 0x5410), __byte_perm(lo01, lo23, 0x7632),
                       __byte_perm(hi01, hi23, 0x5410), __byte_perm(hi01, hi23, 0x7632));
    }
    __syncwarp();
    // ---- consumer: codes of both channel halves, 4 M-blocks each ----
    const uint32_t slot_s = smem_u32(slot);
#pragma unroll
    for (int kb = 0; kb < NKB; ++kb) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int w = 8 * e + g;  // (group 2e + g / 4, digit g % 4)
            const uint32_t b0 = dig[kb * 128 + dig_word(t4, w)];
            const uint32_t b1 = dig[kb * 128 + dig_word(4 + t4, w)];
            uint32_t r0, r1, r2, r3;
            ldsm_x4_trans(slot_s + (uint32_t)((32 * kb + lane) * 32 + 16 * e), r0, r1, r2, r3);
            const uint32_t P0 = __byte_perm(r0, r1, 0x6420), P1 = __byte_perm(r0, r1, 0x7531);
            const uint32_t P2 = __byte_perm(r2, r3, 0x6420), P3 = __byte_perm(r2, r3, 0x7531);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                // channel 8g + i of the K groups: (P >> 2 (i % 4)) & 0x03030303;
                // the shifts run on the FMA pipe (IMAD.HI), the masks on the ALU
                const uint32_t lo = j < 2 ? P0 : P1, hi = j < 2 ? P2 : P3;
                const bool odd = j & 1;  // i = 2j, 2j + 1: shifts {0, 2} or {4, 6}
                const uint32_t l0 = odd ? shr4(lo) : lo, h0 = odd ? shr4(hi) : hi;
                imma(st.D[e][j], l0 & 0x03030303u, shr2(l0) & 0x03030303u, h0 & 0x03030303u,
                     shr2(h0) & 0x03030303u, b0, b1);
            }
        }
    }
}

// The item's partial: channel values (1/3) (2^(E - 31) sum_d D_d 256^d + F)
// + z_cg, written as part_o[128]; ml = (max, sum) of the item's softmax.
__device__ __forceinline__ void finalize(const State& st, float2 ml, float* part_o, float2* part_ml,
                                         int lane) {
    const int g = lane >> 2, t4 = lane & 3;
    // z per group: producer lanes with lane % 4 == cg hold the shares
    float z = st.z;
    z += __shfl_xor_sync(FULL, z, 4);
    z += __shfl_xor_sync(FULL, z, 8);
    z += __shfl_xor_sync(FULL, z, 16);
    const bool writer = (t4 == 0 && g < 4) || (t4 == 2 && g >= 4);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int cgc = 2 * e + (g >> 2);
        const float zc = __shfl_sync(FULL, z, cgc);
        const float sc = pow2f(st.E - 31);
        float v[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float a, b;
            combine_digits(st.D[e][j], t4, a, b);
            v[2 * j] = fmaf(fmaf(a, sc, st.F[e][j][0]), 1.0f / 3.0f, zc);
            v[2 * j + 1] = fmaf(fmaf(b, sc, st.F[e][j][1]), 1.0f / 3.0f, zc);
        }
        if (writer) {
            float4* dst = reinterpret_cast<float4*>(part_o + 64 * e + 8 * g);
            dst[0] = make_float4(v[0], v[1], v[2], v[3]);
            dst[1] = make_float4(v[4], v[5], v[6], v[7]);
        }
    }
    if (lane == 0) *part_ml = ml;
}

}  // namespace vimma
}  // namespace kivi_b200
