// Shared device helpers for the KIVI B200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

// Persistent attend kernels: claim the item after next with the current
// item's first job and broadcast it one item later (1), or claim and
// broadcast at once (0, default: 1 measured 0.5-1 % slower on C2 / C3
// although the broadcast shuffle was the body's most-stalled instruction).
#ifndef KIVI_DEFER_CLAIM
#define KIVI_DEFER_CLAIM 0
#endif
// Key-tile flush: two streaming passes over the ring rows (see flush_key_group).
#ifndef KIVI_FLUSH_STREAM
#define KIVI_FLUSH_STREAM 1
#endif

namespace kivi_b200 {

// ---------------------------------------------------------------------------
// Exact group quantizer.
//
// Reference quantize_group (proj/src/quantize.cpp:22-48):
//   lo, hi  = float min / max of the group (first smallest, last largest —
//             std::minmax_element semantics; only visible for +0/-0 ties)
//   if hi == lo: scale 1, all codes 0
//   s       = (double(hi) - double(lo)) / (2^B - 1)              (double)
//   code    = clamp(nearbyint((double(v) - lo) / s), 0, 2^B - 1) (ties-even)
//
// The device version stores the group as the float pair (lo, hi), from which
// the reference's double scale is recomputed bit-exactly anywhere.  Codes are
// decided in fp32 with an error bound (|x - X| < 1e-4 for B <= 8) and only
// values within 1e-3 of a rounding tie take the exact double path, so every
// code equals the reference's.
// ---------------------------------------------------------------------------
struct GroupRange {
    float lo;
    float hi;
};

__device__ __forceinline__ void minmax_step(float v, float& lo, float& hi) {
    if (v < lo) lo = v;     // first smallest
    if (!(v < hi)) hi = v;  // last largest
}

__device__ __forceinline__ double group_scale(float lo, float hi, int maxc) {
    if (hi == lo) return 1.0;
    return __ddiv_rn(__dsub_rn((double)hi, (double)lo), (double)maxc);
}

struct CodeCtx {
    float lo;
    float hi;
    float r;        // maxc / (hi - lo) in fp32; 0 for a degenerate group, NaN
                    // when the fp32 path cannot be used (every code exact)
    float tie;      // 0.5 - maxc * 2^-20: fp32 decisions closer to a tie go exact
    int maxc;
};

__device__ __forceinline__ CodeCtx make_code_ctx(float lo, float hi, int maxc) {
    CodeCtx c;
    c.lo = lo;
    c.hi = hi;
    c.maxc = maxc;
    const float r = (float)maxc / (hi - lo);
    c.r = (hi == lo) ? 0.0f : ((isfinite(r) && r > 0.0f) ? r : __int_as_float(0x7fc00000));
    c.tie = 0.5f - (float)maxc * 0x1p-20f;
    return c;
}

// The reference's own expression, rint((double(v) - lo) / s) clamped, with
// the exact double scale (a DDIV: only for the rare near-tie values).
__device__ __noinline__ uint32_t quant_code_exact(float lo, float hi, int maxc, float v) {
    double q = rint(__ddiv_rn(__dsub_rn((double)v, (double)lo), group_scale(lo, hi, maxc)));
    q = fmin(fmax(q, 0.0), (double)maxc);
    return (uint32_t)q;
}

// Branch-free fp32 decision.  x = (v - lo) * r carries at most ~4 fp32
// roundings relative to the exact quotient X <= maxc (|x - X| < 4.1 * 2^-24 *
// maxc), so rint(x) is the reference's code unless x lies within maxc * 2^-20
// (4x that bound) of a .5 tie; then *exact is set and the caller re-decides
// the code by quant_code_exact.  rint by the 1.5 * 2^23 magic add
// (round-to-nearest-even, |x| < 2^22), the code read from the sum's mantissa:
// full-rate FADD / IADD only (floorf, rintf and F2I run on the quarter-rate
// conversion pipe).  NaN x (r = NaN, inf inputs) always fails the test.
__device__ __forceinline__ uint32_t quant_code_fast(const CodeCtx& c, float v, bool& exact) {
    const float x = __fmul_rn(__fsub_rn(v, c.lo), c.r);
    const float y = __fadd_rn(x, 12582912.0f);
    const float rx = __fsub_rn(y, 12582912.0f);
    exact = !(fabsf(__fsub_rn(x, rx)) < c.tie);
    return (uint32_t)min(max(__float_as_int(y) - 0x4B400000, 0), c.maxc);
}

// The same decision with one FFMA: y = fma(v - lo, r, 1.5 * 2^23) rounds the
// exact product (v - lo) * r to the nearest even integer in its mantissa (one
// LOP3 reads the code), and d = fma(v - lo, r, -rint) is its distance to that
// integer; fewer roundings than quant_code_fast's x, so the same tie margin
// covers the error.  near_tie |= the decision needs the exact path (NaN r or
// inputs included); the caller then re-codes the group with quant_code.  The
// returned code is only meaningful when near_tie stays false.
__device__ __forceinline__ uint32_t quant_code_fma(const CodeCtx& c, float v, bool& near_tie) {
    constexpr float MAGIC = 12582912.0f;  // 1.5 * 2^23
    const float t = __fsub_rn(v, c.lo);
    const float y = __fmaf_rn(t, c.r, MAGIC);
    const float d = __fmaf_rn(t, c.r, -__fsub_rn(y, MAGIC));
    near_tie |= !(fabsf(d) < c.tie);
    return (uint32_t)__float_as_int(y) & (uint32_t)c.maxc;
}

__device__ __forceinline__ uint32_t quant_code(const CodeCtx& c, float v) {
    bool exact;
    const uint32_t q = quant_code_fast(c, v, exact);
    return exact ? quant_code_exact(c.lo, c.hi, c.maxc, v) : q;
}

// std::minmax_element over x[0..N) (first smallest, last largest) for finite
// inputs: FMNMX chains, then the only case where equal-comparing values have
// different bits, +0 / -0, re-resolved in order.  (Non-finite groups are out
// of contract: the reference's own codes are undefined for NaN.)
template <int N>
__device__ __forceinline__ float2 minmax_first_last(const float (&x)[N]) {
    float lo = x[0], hi = x[0];
#pragma unroll
    for (int i = 1; i < N; ++i) {
        lo = fminf(lo, x[i]);
        hi = fmaxf(hi, x[i]);
    }
    if (lo == 0.0f || hi == 0.0f) {
        float zf = 0.0f, zl = 0.0f;
        bool seen = false;
#pragma unroll
        for (int i = N - 1; i >= 0; --i) {
            if (x[i] == 0.0f) {
                zf = x[i];            // ends as the first zero
                if (!seen) zl = x[i];  // the last zero
                seen = true;
            }
        }
        if (lo == 0.0f) lo = zf;
        if (hi == 0.0f) hi = zl;
    }
    return make_float2(lo, hi);
}

// Reference dequantisation: float(double(code) * s + z), no contraction
// (quantize.cpp:50-57, 142-167).
__device__ __forceinline__ float dequant_exact(uint32_t code, double s, double z) {
    return (float)__dadd_rn(__dmul_rn((double)code, s), z);
}

// ---------------------------------------------------------------------------
// Little-endian bit streams (reference pack_codes, quantize.cpp:59-76): code
// i occupies bits [i*B, i*B+B) of the byte stream.  With B in {1,2,4,8} a
// code never straddles a 32-bit word, so a 32-bit little-endian word view
// addresses it as bit (i*B) & 31 of word (i*B) >> 5.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t read_code(const uint8_t* base, uint64_t bit, int bits) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(base);
    return (w[bit >> 5] >> (bit & 31)) & ((1u << bits) - 1u);
}

// OR `code` into a zero-initialised stream (concurrent writers of one word
// are fine).
__device__ __forceinline__ void or_code(uint8_t* base, uint64_t bit, int bits, uint32_t code) {
    (void)bits;
    if (code == 0u) return;
    uint32_t* w = reinterpret_cast<uint32_t*>(base);
    atomicOr(&w[bit >> 5], code << (bit & 31));
}

// ---------------------------------------------------------------------------
// Bulk-copy (TMA, cp.async.bulk) + mbarrier helpers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Generic-proxy global writes (e.g. an append) before async-proxy (TMA)
// reads of the same memory.
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Plain arrive (consumer releases a slot).
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Non-blocking probe of a phase: true when the phase with `parity` completed.
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// 1-D bulk global->shared copy completing on `bar` (bytes % 16 == 0,
// both addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Same with an L2 evict-first policy: the cache is streamed exactly once per
// decode step, so it should not displace other lines.
__device__ __forceinline__ void bulk_g2s_evict_first(void* dst, const void* src, uint32_t bytes,
                                                     uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
        "[%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// Programmatic dependent launch.  A kernel launched with the
// programmatic-serialization attribute may start before its predecessor in
// the stream has finished; it must pdl_wait() before touching memory the
// predecessor writes (a no-op for a normal launch).  pdl_trigger() lets the
// dependent's CTAs be scheduled once every CTA of this grid has issued it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

// Bulk prefetch of [src, src + bytes) into L2 (no shared memory, no
// completion tracking); bytes a multiple of 16, src 16-byte aligned.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint64_t make_evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Warp max in one instruction (CREDUX.MAX.F32, sm_100a) instead of a
// 5-step shuffle chain; every lane gets the result.
__device__ __forceinline__ float warp_max_redux(float v) {
    float r;
    asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
    return r;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace kivi_b200
