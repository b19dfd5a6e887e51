// Isolates gqa_tc::key_job on one warp: 4 key tiles with optional outlier
// channels -> logits vs exact double.  Not product code.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include "../../paper_2402_02750_b200/csrc/kernels_attend_gqa_tc.cuh"
using namespace kivi_b200;
__global__ void run(const uint8_t* job, const float* q, float* probs_out, int mode) {
    __shared__ __align__(128) uint8_t slot[8192];
    __shared__ __align__(16) float probs[128 * 4];
    __shared__ __align__(16) uint8_t bf[4608];
    __shared__ float biasm[32 * 17];
    const int lane = threadIdx.x;
    for (int i = lane; i < 2048; i += 32) reinterpret_cast<uint32_t*>(slot)[i] = reinterpret_cast<const uint32_t*>(job)[i];
    __syncwarp();
    float2 qv[4][2]; float qmax = 0.f;
    for (int h = 0; h < 4; ++h) for (int i = 0; i < 2; ++i) { qv[h][i] = make_float2(q[h * 128 + 4 * lane + 2 * i], q[h * 128 + 4 * lane + 2 * i + 1]); qmax = fmaxf(qmax, fmaxf(fabsf(qv[h][i].x), fabsf(qv[h][i].y))); }
    qmax = warp_max(qmax);
    const uint32_t sel = (uint32_t)(lane >> 2 & 3) * 0x1111u + 0x4400u;
    gqa_tc::key_job<4>(slot, qv, qmax, probs, 0, bf, biasm, lane, sel);
    __syncwarp();
    for (int i = lane; i < 512; i += 32) probs_out[i] = probs[gqa_tc::pidx<4>(i >> 2, i & 3)];
}
int main(int argc, char** argv) {
    std::mt19937 rng(1);
    std::uniform_real_distribution<float> U(-1.f, 1.f);
    for (int outl = 0; outl < 2; ++outl) {
        double sum_err = 0, max_err = 0, sum_mag = 0; int n = 0;
        double ej[4] = {0,0,0,0}; int nj[4] = {0,0,0,0};
        for (int trial = 0; trial < 20; ++trial) {
            std::vector<uint8_t> job(8192, 0);
            std::vector<float> q(512);
            for (auto& v : q) v = U(rng) * 0.1275f;
            std::vector<double> exact(128 * 4, 0.0);
            for (int T = 0; T < 4; ++T) {
                for (int c = 0; c < 128; ++c) {
                    float k[32];
                    for (int i = 0; i < 32; ++i) { k[i] = U(rng); if (outl && (c == 1 || c == 17 || c == 40)) k[i] *= 50.f; }
                    float lo = k[0], hi = k[0];
                    for (int i = 0; i < 32; ++i) { lo = fminf(lo, k[i]); hi = fmaxf(hi, k[i]); }
                    double s = ((double)hi - lo) / 3.0;
                    float* pr = reinterpret_cast<float*>(job.data() + 4096 + T * 1024 + c * 8);
                    pr[0] = lo; pr[1] = hi;
                    for (int i = 0; i < 32; ++i) {
                        int code = (int)std::nearbyint(((double)k[i] - lo) / s); code = code < 0 ? 0 : code > 3 ? 3 : code;
                        job[T * 1024 + c * 8 + (i >> 2)] |= (uint8_t)(code << (2 * (i & 3)));
                        for (int h = 0; h < 4; ++h) exact[(T * 32 + i) * 4 + h] += (double)q[h * 128 + c] * (code * s + lo);
                    }
                }
            }
            uint8_t* dj; float *dq, *dout;
            cudaMalloc(&dj, 8192); cudaMalloc(&dq, 2048); cudaMalloc(&dout, 2048);
            cudaMemcpy(dj, job.data(), 8192, cudaMemcpyHostToDevice); cudaMemcpy(dq, q.data(), 2048, cudaMemcpyHostToDevice);
            run<<<1, 32>>>(dj, dq, dout, 0);
            std::vector<float> got(512); cudaMemcpy(got.data(), dout, 2048, cudaMemcpyDeviceToHost);
            for (int i = 0; i < 512; ++i) { double e = fabs(got[i] - exact[i]); int j = (i / 4) % 4; ej[j] += e * e; nj[j]++; sum_err += e * e; max_err = fmax(max_err, e); sum_mag += exact[i] * exact[i]; ++n; }
            cudaFree(dj); cudaFree(dq); cudaFree(dout);
        }
        printf("  per token position j: %.3g %.3g %.3g %.3g\n", sqrt(ej[0]/nj[0]), sqrt(ej[1]/nj[1]), sqrt(ej[2]/nj[2]), sqrt(ej[3]/nj[3]));
        printf("outliers=%d: logit rms err %.3g, max err %.3g, rms logit %.3g (%s)\n", outl, sqrt(sum_err / n), max_err, sqrt(sum_mag / n), cudaGetErrorString(cudaGetLastError()));
    }
}
