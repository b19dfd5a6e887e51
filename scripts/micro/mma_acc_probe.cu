// Probe the internal accumulation precision of mma.sync m16n8k16 f16->f32:
// D = sum_k A[0][k] B[k][0] + C with one large and one small product.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
__global__ void k(const float* avals, float cin, float* out) {
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    auto A = [&](int m, int kk) -> __half { return m == 0 ? __float2half(avals[kk]) : __float2half(0.f); };
    auto pk = [](__half lo, __half hi) { return (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16); };
    uint32_t a0 = pk(A(g, 2 * t), A(g, 2 * t + 1)), a1 = pk(A(g + 8, 2 * t), A(g + 8, 2 * t + 1));
    uint32_t a2 = pk(A(g, 2 * t + 8), A(g, 2 * t + 9)), a3 = pk(A(g + 8, 2 * t + 8), A(g + 8, 2 * t + 9));
    __half one = __float2half(g == 0 ? 1.f : 0.f);
    uint32_t b0 = pk(one, one), b1 = pk(one, one);
    float d0 = (g == 0 && t == 0) ? cin : 0.f, d1 = 0, d2 = 0, d3 = 0;
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d0), "+f"(d1), "+f"(d2), "+f"(d3) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    if (lane == 0) out[0] = d0;
}
int main() {
    float *da, *dout; cudaMalloc(&da, 64); cudaMalloc(&dout, 4);
    auto run = [&](float* a, float c) { cudaMemcpy(da, a, 64, cudaMemcpyHostToDevice); k<<<1, 32>>>(da, c, dout); float r; cudaMemcpy(&r, dout, 4, cudaMemcpyDeviceToHost); return r; };
    printf("two products: big=1024, small=1+2^-10*m (fp16 exact), expect exact sum\n");
    for (int e = 0; e <= 30; e += 2) {
        float a[16] = {0}; a[0] = 1024.f; a[1] = ldexpf(1.f, -e) * (1.f + 1.f / 1024.f);
        float r = run(a, 0.f); double want = 1024.0 + (double)ldexpf(1.f, -e) * (1.0 + 1.0 / 1024.0);
        printf("  small=2^-%-2d*(1+2^-10): got %.10g want %.10g relerr %.3g\n", e, r, want, fabs(r - want) / want);
    }
    printf("accumulator C=1024 + product small\n");
    for (int e = 0; e <= 30; e += 2) {
        float a[16] = {0}; a[0] = ldexpf(1.f, -e) * (1.f + 1.f / 1024.f);
        float r = run(a, 1024.f); double want = 1024.0 + (double)a[0];
        printf("  small=2^-%-2d: got %.10g want %.10g relerr %.3g\n", e, r, want, fabs(r - want) / want);
    }
    printf("subnormal A products: 1 * 2^-24 * 1024 + ... \n");
    {
        float a[16] = {0}; a[0] = 1024.f; a[1] = ldexpf(3.f, -24); a[2] = ldexpf(1.f, -20);
        float r = run(a, 0.f); double want = 1024.0 + ldexp(3.0, -24) + ldexp(1.0, -20);
        printf("  got %.12g want %.12g relerr %.3g\n", r, want, fabs(r - want) / want);
    }
    return 0;
}
