// q/k/v projection of the decode step on the 5th-generation tensor cores,
// fused with the KV-cache append (the reference projects
// t * W per layer in fp32, workload.cpp:230-232, and the paper names fusing
// the quantization with the preceding op as the speed-up it left undone,
// PAPER.md:690-694).
//
// Swap-AB tiling for a skinny GEMM: the MMA's M is 128 output channels (one
// head at d = 128), N the batch rows (padded to 16..256, the padding is TMA
// zero fill), K the hidden size:
//     D[m][n] = sum_k Wt[m][k] * x[n][k]        (Wt = W^T, prepared once)
// fp32 accuracy from TF32 tensor cores with the 3xTF32 split
//     x*w ~= x_hi*w_hi + x_hi*w_lo + x_lo*w_hi
// where x_hi = x rounded to tf32 and x_lo = the rounded remainder, computed
// in shared memory (in place over the TMA'd tile) by the epilogue warps while
// the TMA streams the next tiles.  The three products accumulate in one fp32 TMEM accumulator.
//
// Warp roles (one CTA per 128-channel tile of q, k or v, 6 warps):
//   warp 0, one lane : TMA producer (Wt tile 128 x 32 fp32, x tile N x 32),
//                      SWIZZLE_128B, a ring of STAGES stages;
//   warp 1, one lane : tcgen05.mma issuer (kind::tf32, 3 x 4 MMAs per stage),
//                      tcgen05.commit frees the stage / signals the epilogue;
//   warps 2-5        : lo-part split of every stage, then the epilogue:
//                      tcgen05.ld of the accumulator (lane = output channel),
//                      and per batch row either a plain store (q rows, prefill
//                      projections) or the append of the new token into the
//                      KIVI cache (key row into the ring; value FIFO pop:
//                      quantize the evicted row per-token across the warp's 32
//                      channels, then write the new row) -- no k/v round trip
//                      through HBM and no separate append launch.
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "kernels_quant.cuh"

namespace kivi_b200 {
namespace proj {

constexpr int BM = 128;       // output channels per CTA
constexpr int BK = 32;        // fp32 per 128-byte swizzle row
constexpr int UK = 8;         // K per tf32 MMA
constexpr int THREADS = 192;  // 6 warps
constexpr int SMEM_LIMIT = 200 * 1024;

struct ProjArgs {
    int K;           // hidden_in (multiple of 32)
    int N;           // MMA N: batch rows padded to a multiple of 16 (16..256)
    int n_valid;     // real rows of this CTA's N tile
    int n_tile0;     // first row of this CTA's N tile (blockIdx.y * N)
    int tiles_m;     // 128-channel tiles per matrix (hidden_out / 128)
    int stages;
    int mode;        // 0: store rows  1: decode append (k, v) + q store  2: store per unit
    int split_mode;  // hi/lo split (see the split warps)
    // mode 0: out[which] is [rows][hidden_out] row-major
    // mode 1: out[0] = q rows [n * heads + h][128]; k / v go into the cache
    // mode 2: row = b * seq + t -> out[which][((b * heads + h) * seq + t)][128]
    //         (the [units][l][d] layout kivi_prefill takes)
    float* out[3];
    int hidden_out;
    int seq;
    // mode 1
    CacheDev c;
    int64_t l;       // tokens in the cache before the append
    int heads;       // kv heads (units = rows * heads)
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
        "{%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* tm) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(tm) : "memory");
}

// K-major operand tile with 128-byte rows, SWIZZLE_128B (as the TMA writes
// it): SBO = 1024 B between 8-row groups, LBO unused (1), version 1 (sm_100).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, M = 128.
__host__ __device__ constexpr uint32_t tf32_idesc(int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Round-to-nearest tf32 split x = hi + lo: hi = x rounded to 10 mantissa
// bits (what the tensor core reads of it exactly), lo = x - hi (exact in fp32,
// |lo| <= 2^-11 |x|) rounded the same way.  The three products hi*hi, hi*lo,
// lo*hi then carry x*w to ~2^-22 relative (the dropped lo*lo is < 2^-22);
// with a truncating split (hi = x as the tensor core truncates it) both the
// lo operand's own truncation and lo*lo were ~2^-20, several times the error
// of an fp32 SIMT product.
__device__ __forceinline__ float rn_tf32(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
__device__ __forceinline__ float trunc_tf32(float x) {
    return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
__device__ __forceinline__ float4 trunc4(float4 x) {
    return make_float4(trunc_tf32(x.x), trunc_tf32(x.y), trunc_tf32(x.z), trunc_tf32(x.w));
}
__device__ __forceinline__ float4 lo_part4(float4 x) {
    return make_float4(x.x - trunc_tf32(x.x), x.y - trunc_tf32(x.y), x.z - trunc_tf32(x.z),
                       x.w - trunc_tf32(x.w));
}
__device__ __forceinline__ void split_tf32(float4& x, float4& lo) {
    float4 h = make_float4(rn_tf32(x.x), rn_tf32(x.y), rn_tf32(x.z), rn_tf32(x.w));
    lo = make_float4(rn_tf32(x.x - h.x), rn_tf32(x.y - h.y), rn_tf32(x.z - h.z), rn_tf32(x.w - h.w));
    x = h;
}

// The value FIFO pop for one 32-channel group held one channel per lane: the
// reference quantize_group (quantize.cpp:22-48) over the warp, ties in the
// min / max by channel index (std::minmax_element semantics).
template <int B>
__device__ __forceinline__ void value_group_lane(float x, int lane, uint32_t* vw_group,
                                                 float2* vp_group) {
    float lo = x, hi = x;
    int ilo = lane, ihi = lane;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float olo = __shfl_xor_sync(0xffffffffu, lo, o);
        const int oilo = __shfl_xor_sync(0xffffffffu, ilo, o);
        const float ohi = __shfl_xor_sync(0xffffffffu, hi, o);
        const int oihi = __shfl_xor_sync(0xffffffffu, ihi, o);
        if (olo < lo || (!(lo < olo) && oilo < ilo)) { lo = olo; ilo = oilo; }
        if (ohi > hi || (!(hi > ohi) && oihi > ihi)) { hi = ohi; ihi = oihi; }
    }
    const CodeCtx cc = make_code_ctx(lo, hi, (1 << B) - 1);
    constexpr int CPW = 32 / B;  // codes per 32-bit word
    uint32_t word = quant_code(cc, x) << (B * (lane % CPW));
#pragma unroll
    for (int o = 1; o < CPW; o <<= 1) word |= __shfl_xor_sync(0xffffffffu, word, o);
    if (lane % CPW == 0) vw_group[lane / CPW] = word;
    if (lane == 0) *vp_group = make_float2(lo, hi);
}

template <int B>
__global__ void __launch_bounds__(THREADS, 1)
    proj_kernel(const __grid_constant__ CUtensorMap tm_w0, const __grid_constant__ CUtensorMap tm_w1,
                const __grid_constant__ CUtensorMap tm_w2, const __grid_constant__ CUtensorMap tm_x,
                ProjArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte aligned operand tiles (SWIZZLE_128B atoms)
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const int N = a.N;
    const uint32_t a_bytes = BM * BK * 4, b_bytes = (uint32_t)N * BK * 4;
    const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;  // A, A_lo, B, B_lo
    const int S = a.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(base + S * stage_bytes);
    uint64_t* split = full + S;
    uint64_t* empty = split + S;
    uint64_t* tmem_full = empty + S;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int which = blockIdx.x / a.tiles_m, tile_m = blockIdx.x % a.tiles_m;
    const CUtensorMap* tm_w = which == 0 ? &tm_w0 : (which == 1 ? &tm_w1 : &tm_w2);
    const int nkb = a.K / BK;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(tm_w);
        prefetch_tmap(&tm_x);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&split[s], 128);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        fence_mbar_init();
    }
    // Accumulator chunks: the tensor core's fp32 accumulation rounds once per
    // MMA against the running sum, so its error grows with the number of MMAs
    // folded into one accumulator (measured: 1.3e-6 relative at K = 128,
    // 3e-5 at K = 4096).  K is split over up to 8 accumulators in TMEM (as
    // many as 512 columns hold) that the epilogue adds in fp32.
    uint32_t ncols_per = 32;
    while ((int)ncols_per < N) ncols_per <<= 1;
    int nchunk = 1;
    while (nchunk < 8 && (uint32_t)(2 * nchunk) * ncols_per <= 512u && 2 * nchunk <= nkb) nchunk <<= 1;
    const uint32_t ncols = (uint32_t)nchunk * ncols_per;
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(ncols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ===== TMA producer =====
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % S;
                if (kb >= S) mbar_wait(&empty[s], ((kb / S) - 1) & 1);
                uint8_t* st = base + s * stage_bytes;
                mbar_arrive_expect_tx(&full[s], a_bytes + b_bytes);
                tma_load_2d(st, tm_w, kb * BK, tile_m * BM, &full[s]);
                tma_load_2d(st + 2 * a_bytes, &tm_x, kb * BK, a.n_tile0, &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ===== MMA issuer =====
            const uint32_t idesc = tf32_idesc(N);
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % S;
                const int chunk = kb * nchunk / nkb;
                const bool first = kb == (chunk * nkb + nchunk - 1) / nchunk;  // chunk's first kb
                const uint32_t acc = tmem + (uint32_t)chunk * ncols_per;
                mbar_wait(&split[s], (kb / S) & 1);
                tc_fence_after();
                const uint32_t st = smem_u32(base + s * stage_bytes);
                const uint32_t sa = st, sa_lo = st + a_bytes, sb = st + 2 * a_bytes,
                               sb_lo = sb + b_bytes;
#pragma unroll
                for (int kk = 0; kk < BK / UK; ++kk) {
                    const uint32_t off = kk * UK * 4;  // 32 bytes per K step inside the atom
                    const uint64_t da = sw128_desc(sa + off), dal = sw128_desc(sa_lo + off);
                    const uint64_t db = sw128_desc(sb + off), dbl = sw128_desc(sb_lo + off);
                    mma_tf32(acc, da, db, idesc, !(first && kk == 0));
                    mma_tf32(acc, da, dbl, idesc, 1);
                    mma_tf32(acc, dal, db, idesc, 1);
                }
                umma_commit(&empty[s]);  // the stage is free once these MMAs completed
            }
            umma_commit(tmem_full);
        }
    } else {
        // ===== lo-part split of each stage (warps 2-5, 128 threads) =====
        const int t = threadIdx.x - 64;
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % S;
            mbar_wait(&full[s], (kb / S) & 1);
            uint8_t* st = base + s * stage_bytes;
            float4* A = reinterpret_cast<float4*>(st);
            float4* Alo = reinterpret_cast<float4*>(st + a_bytes);
            float4* Bx = reinterpret_cast<float4*>(st + 2 * a_bytes);
            float4* Blo = reinterpret_cast<float4*>(st + 2 * a_bytes + b_bytes);
            // split_mode 0: hi = the TMA'd tile itself (the tensor core
            // truncates it), lo = x - trunc(x); 1: hi = trunc(x) written in
            // place; 2: round-to-nearest hi and lo (split_tf32)
            if (a.split_mode == 0) {
#pragma unroll 4
                for (int i = t; i < (int)(a_bytes / 16); i += 128) Alo[i] = lo_part4(A[i]);
                for (int i = t; i < (int)(b_bytes / 16); i += 128) Blo[i] = lo_part4(Bx[i]);
            } else if (a.split_mode == 1) {
                for (int i = t; i < (int)(a_bytes / 16); i += 128) {
                    const float4 x = A[i];
                    Alo[i] = lo_part4(x);
                    A[i] = trunc4(x);
                }
                for (int i = t; i < (int)(b_bytes / 16); i += 128) {
                    const float4 x = Bx[i];
                    Blo[i] = lo_part4(x);
                    Bx[i] = trunc4(x);
                }
            } else {
                for (int i = t; i < (int)(a_bytes / 16); i += 128) {
                    float4 x = A[i], lo;
                    split_tf32(x, lo);
                    A[i] = x;
                    Alo[i] = lo;
                }
                for (int i = t; i < (int)(b_bytes / 16); i += 128) {
                    float4 x = Bx[i], lo;
                    split_tf32(x, lo);
                    Bx[i] = x;
                    Blo[i] = lo;
                }
            }
            fence_proxy_async_smem();  // generic-proxy writes -> tensor-core (async) reads
            mbar_arrive(&split[s]);
        }
        // ===== epilogue =====
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        const int q = warp & 3;            // TMEM lane quarter of this warp
        const int m = q * 32 + lane;       // output channel in the tile
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16);
        for (int c0 = 0; c0 < N; c0 += 16) {
            float v[16];
            tmem_ld16(taddr + c0, v);
            for (int ch = 1; ch < nchunk; ++ch) {
                float w[16];
                tmem_ld16(taddr + (uint32_t)ch * ncols_per + c0, w);
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] += w[j];
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int n = c0 + j;
                if (n >= a.n_valid) break;
                const int row = a.n_tile0 + n;
                if (a.mode == 0) {
                    a.out[which][(int64_t)row * a.hidden_out + tile_m * BM + m] = v[j];
                } else if (a.mode == 2) {
                    const int b = row / a.seq, tt = row - b * a.seq;
                    a.out[which][(((int64_t)b * a.heads + tile_m) * a.seq + tt) * BM + m] = v[j];
                } else if (which == 0) {
                    a.out[0][((int64_t)row * a.heads + tile_m) * BM + m] = v[j];
                } else {
                    const CacheDev& c = a.c;
                    const int64_t u = (int64_t)row * a.heads + tile_m;
                    const int slot = (int)(a.l % c.R);
                    if (which == 1) {
                        c.kring[u * c.ring_ustride + (int64_t)slot * BM + m] = v[j];
                    } else {
                        float* vrow = c.vring + u * c.ring_ustride + (int64_t)slot * BM;
                        if (a.l >= c.R) {
                            // FIFO pop of token l - R (its row is in this slot)
                            const int64_t e = a.l - c.R;
                            uint32_t* vw = reinterpret_cast<uint32_t*>(c.vcodes + u * c.v_ustride) +
                                           e * (BM * B / 32) + q * B;
                            value_group_lane<B>(vrow[m], lane, vw,
                                                c.vpairs + u * c.vp_ustride + e * (BM / 32) + q);
                        }
                        vrow[m] = v[j];
                    }
                }
            }
        }
        tc_fence_before();
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols)
                     : "memory");
    }
}

}  // namespace proj
}  // namespace kivi_b200
