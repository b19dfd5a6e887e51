// Probe: tcgen05.mma kind::i8 with MN-major (transposed) shared-memory operands,
// no swizzle.  Finds which descriptor field (LBO / SBO) holds the MN-block and the
// K-block stride for MN-major u8 operands, and checks that u8 x u8 -> s32 is exact.
// One CTA, M = 128, N = 64, K = 32 (one MMA).  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o umma_i8_probe umma_i8_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
// element (r, k) of an R x K u8 operand -> byte offset in shared memory.
//  K-major : core matrix = 8 rows (R) x 16 B (K);  R-blocks at rb, K-blocks at kb
//  MN-major: core matrix = 8 rows (K) x 16 B (R);  R-blocks at rb, K-blocks at kb
__device__ __forceinline__ int off(int major, int r, int k, int rb, int kb) {
    if (major == 0) return (r >> 3) * rb + (k >> 4) * kb + (r & 7) * 16 + (k & 15);
    return (r >> 4) * rb + (k >> 3) * kb + (k & 7) * 16 + (r & 15);
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version 1 (sm_100), layout SWIZZLE_NONE (0)
    return d;
}

constexpr int M = 128, N = 64, K = 32;

// cfg: bit0 A major, bit1 B major, bit2 swap (LBO,SBO) roles for MN-major operands,
// bit3 B signed (s8)
__global__ void probe(const uint8_t* A, const uint8_t* B, int32_t* D, int cfg) {
    __shared__ __align__(1024) uint8_t sa[M * K];
    __shared__ __align__(1024) uint8_t sb[N * K];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x;
    const int amaj = cfg & 1, bmaj = (cfg >> 1) & 1, swap = (cfg >> 2) & 1, bsig = (cfg >> 3) & 1;
    // strides: K-major: K-blocks (16 B) adjacent (128 B), R-blocks after all K-blocks
    //          MN-major: K-blocks (8 rows) adjacent (128 B), R-blocks after all K-blocks
    const int a_kb = 128, a_rb = amaj ? (K / 8) * 128 : (K / 16) * 128;
    const int b_kb = 128, b_rb = bmaj ? (K / 8) * 128 : (K / 16) * 128;
    for (int i = tid; i < M * K; i += blockDim.x) {
        int r = i / K, k = i % K;
        sa[off(amaj, r, k, a_rb, a_kb)] = A[i];
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        int n = i / K, k = i % K;  // B given as [N][K]
        sb[off(bmaj, n, k, b_rb, b_kb)] = B[i];
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         su32(&tmem_base)),
                     "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tmem_base;
    if (tid == 0) {
        // K-major: LBO = K-block stride, SBO = R-block stride (as the SW128 path);
        // MN-major: hypothesis 0 LBO = K-block, SBO = R-block; hypothesis 1 swapped.
        uint32_t al = a_kb, as = a_rb, bl = b_kb, bs = b_rb;
        if (amaj && swap) { al = a_rb; as = a_kb; }
        if (bmaj && swap) { bl = b_rb; bs = b_kb; }
        const uint64_t da = desc(su32(sa), al, as), db = desc(su32(sb), bl, bs);
        const uint32_t idesc = (2u << 4) | (0u << 7) | ((uint32_t)bsig << 10) |
                               ((uint32_t)amaj << 15) | ((uint32_t)bmaj << 16) |
                               ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
            "l"(da), "l"(db), "r"(idesc), "r"(0)
            : "memory");
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                su32(&bar))
            : "memory");
    }
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}\n"
                : "=r"(done)
                : "r"(su32(&bar)));
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int w = tid >> 5;
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
            "%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
              "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(tm + ((uint32_t)(w * 32) << 16) + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 16; ++j) D[tid * N + c0 + j] = (int32_t)r[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(64));
}

int main() {
    std::vector<uint8_t> A(M * K), B(N * K);
    srand(7);
    for (auto& x : A) x = rand() % 4;
    for (auto& x : B) x = rand() % 256;
    uint8_t *dA, *dB;
    int32_t* dD;
    cudaMalloc(&dA, M * K);
    cudaMalloc(&dB, N * K);
    cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, A.data(), M * K, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), N * K, cudaMemcpyHostToDevice);
    const int cfgs[] = {0, 1, 5, 2, 6, 3, 7, 8, 11, 15};
    for (int cfg : cfgs) {
        cudaMemset(dD, 0, M * N * 4);
        probe<<<1, 128>>>(dA, dB, dD, cfg);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<int32_t> D(M * N);
        cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
        long bad = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                long ref = 0;
                for (int k = 0; k < K; ++k)
                    ref += (long)A[m * K + k] * ((cfg & 8) ? (long)(int8_t)B[n * K + k] : (long)B[n * K + k]);
                if (ref != D[m * N + n]) ++bad;
            }
        printf("cfg %2d (A %s, B %s, %s, B %s): %s, %ld / %d mismatches  D[0..3] %d %d %d %d\n", cfg,
               (cfg & 1) ? "MN" : "K", (cfg & 2) ? "MN" : "K", (cfg & 4) ? "swapped" : "LBO=K-blk",
               (cfg & 8) ? "s8" : "u8", cudaGetErrorString(e), bad, M * N, D[0], D[1], D[2], D[3]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
