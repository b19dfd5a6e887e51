// Read-bandwidth probe: how fast can this part stream HBM with the attend
// kernels' access pattern (per-warp 8 KB TMA bulk copies into 2..4 smem slots,
// evict_first), vs plain 128-bit loads.  usage: read_bw [GB=4]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}"
                 ::"r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}

template <int NSLOT>
__global__ void __launch_bounds__(128) tma_read(const uint8_t* src, int64_t nchunks, int chunk, float* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* base = sm + warp * (NSLOT * chunk + 64);
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + NSLOT * chunk);
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if (lane == 0) for (int s = 0; s < NSLOT; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncwarp();
    const int64_t gw = blockIdx.x * 4 + warp, tw = (int64_t)gridDim.x * 4;
    int64_t next = gw;
    auto issue = [&](int s) {
        if (next < nchunks && lane == 0) {
            expect_tx(&bars[s], chunk);
            bulk(base + s * chunk, src + next * chunk, chunk, &bars[s], pol);
        }
        next += tw;
    };
    for (int s = 0; s < NSLOT; ++s) issue(s);
    float acc = 0.f;
    uint32_t ph = 0;
    int s = 0;
    for (int64_t c = gw; c < nchunks; c += tw) {
        wait(&bars[s], (ph >> s) & 1);
        ph ^= 1u << s;
        acc += reinterpret_cast<const float*>(base + s * chunk)[lane];
        __syncwarp();
        issue(s);
        s = (s + 1 == NSLOT) ? 0 : s + 1;
    }
    if (acc == 1234.5f) sink[0] = acc;
}

__global__ void ldg_read(const float4* src, int64_t n, float* sink) {
    float acc = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float4 v = __ldcs(src + i);
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 1234.5f) sink[0] = acc;
}

int main(int argc, char** argv) {
    const double gb = argc > 1 ? atof(argv[1]) : 4.0;
    const int64_t bytes = (int64_t)(gb * 1e9) / 65536 * 65536;
    uint8_t* buf; float* sink;
    cudaMalloc(&buf, bytes); cudaMalloc(&sink, 4);
    cudaMemset(buf, 1, bytes);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto time = [&](auto launch) {
        launch(); cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        return bytes / (best * 1e-3) / 1e9;
    };
    for (int chunk : {4096, 8192, 16384}) {
        for (int ctas : {2, 3, 4}) {
            const int sm2 = 4 * (2 * chunk + 64), sm3 = 4 * (3 * chunk + 64), sm4 = 4 * (4 * chunk + 64);
            cudaFuncSetAttribute(tma_read<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
            cudaFuncSetAttribute(tma_read<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm3);
            cudaFuncSetAttribute(tma_read<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4);
            const int64_t nch = bytes / chunk;
            if (sm2 * ctas <= 227 * 1024)
                printf("tma chunk %5d slots 2 ctas/SM %d: %7.0f GB/s\n", chunk, ctas,
                       time([&] { tma_read<2><<<sms * ctas, 128, sm2>>>(buf, nch, chunk, sink); }));
            if (sm3 * ctas <= 227 * 1024)
                printf("tma chunk %5d slots 3 ctas/SM %d: %7.0f GB/s\n", chunk, ctas,
                       time([&] { tma_read<3><<<sms * ctas, 128, sm3>>>(buf, nch, chunk, sink); }));
            if (sm4 * ctas <= 227 * 1024)
                printf("tma chunk %5d slots 4 ctas/SM %d: %7.0f GB/s\n", chunk, ctas,
                       time([&] { tma_read<4><<<sms * ctas, 128, sm4>>>(buf, nch, chunk, sink); }));
        }
    }
    for (int blocks : {4, 8, 16})
        printf("ldg.128 streaming, %2d x 256-thread blocks/SM: %7.0f GB/s\n", blocks,
               time([&] { ldg_read<<<sms * blocks, 256>>>((const float4*)buf, bytes / 16, sink); }));
    printf("copy (cudaMemcpy D2D, read+write bytes): %7.0f GB/s\n",
           2 * time([&] { cudaMemcpyAsync(buf, buf + bytes / 2, bytes / 2, cudaMemcpyDeviceToDevice); }) / 2);
    return 0;
}
