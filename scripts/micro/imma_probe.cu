// Probe: mma.sync m16n8k32 u8 x s8 -> s32 on sm_100a: correctness + throughput.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void imma(int* d, const uint32_t* a, const uint32_t* b) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__global__ void test(int* out) {
    // A[m][k] = (m + k) % 200 (u8), B[k][n] = (k - n) % 100 - 50 (s8)
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    auto A = [](int m, int k) { return (uint32_t)((m + k) % 200); };
    auto B = [](int k, int n) { return (int)((k * 7 + n * 3) % 100) - 50; };
    uint32_t a[4], b[2];
    int rows[4] = {g, g + 8, g, g + 8}, c0[4] = {4 * t, 4 * t, 4 * t + 16, 4 * t + 16};
    for (int i = 0; i < 4; ++i) { a[i] = 0; for (int j = 0; j < 4; ++j) a[i] |= A(rows[i], c0[i] + j) << (8 * j); }
    for (int i = 0; i < 2; ++i) { b[i] = 0; for (int j = 0; j < 4; ++j) b[i] |= ((uint32_t)(B(4 * t + 16 * i + j, g) & 0xFF)) << (8 * j); }
    int d[4] = {0, 0, 0, 0};
    imma(d, a, b);
    out[g * 8 + 2 * t] = d[0]; out[g * 8 + 2 * t + 1] = d[1]; out[(g + 8) * 8 + 2 * t] = d[2]; out[(g + 8) * 8 + 2 * t + 1] = d[3];
}
__global__ void tput(int* out, int iters) {
    uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, 7u, 9u}, b[2] = {0x01010101u, 0x01010101u};
    int d[8][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) imma(d[j], a, b);
    }
    int s = 0; for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    if (s == 1234567) out[0] = s;
}
int main() {
    int* dout; cudaMalloc(&dout, 128 * 4);
    test<<<1, 32>>>(dout);
    int h[128]; cudaMemcpy(h, dout, 512, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 16; ++m) for (int n = 0; n < 8; ++n) {
        long ref = 0; for (int k = 0; k < 32; ++k) ref += (long)((m + k) % 200) * (((k * 7 + n * 3) % 100) - 50);
        if (ref != h[m * 8 + n]) bad++;
    }
    printf("imma u8.s8 correctness: bad %d / 128 (%s)\n", bad, cudaGetErrorString(cudaGetLastError()));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int wpb : {4, 8}) {
        int iters = 4096; cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        tput<<<sms * 2, wpb * 32>>>(dout, 16);
        cudaEventRecord(e0); tput<<<sms * 2, wpb * 32>>>(dout, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = 2.0 * 16 * 8 * 32 * 8.0 * iters * sms * 2 * wpb;
        printf("mma.sync m16n8k32 u8.s8: %d warps/CTA: %.1f TOP/s (%s)\n", wpb, ops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
}
