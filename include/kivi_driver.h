/*
 * kivi_driver.h — native decode driver over the C-ABI (libkivi_driver.so).
 *
 * The reference's only in-tree caller of the hot path is
 * run_decode_benchmark (reference proj/src/workload.cpp:145-271): prefill a
 * prompt into one cache per (batch element, layer, kv-head), then gen_len
 * decode steps that project each token (t @ W_q/k/v, workload.cpp:230-232)
 * and call decode_attention on every state.  This is that driver as C++ host
 * code calling the B200 library only through include/kivi_b200.h:
 *
 *   - one host thread per listed device, each with its own stream, driving
 *     a contiguous block of the batch (batch-major sharding over
 *     (batch, kv-head) units; no collective on the decode path);
 *   - per layer and step ONE kivi_proj_append (tcgen05 tensor-core q/k/v
 *     projection fused with the cache append, value FIFO pop quantized in
 *     the GEMM epilogue) and ONE kivi_attend over all of the shard's units;
 *   - the prompt is projected by kivi_proj_gemm straight into the per-unit
 *     layout kivi_prefill takes;
 *   - step latency from CUDA events on each device's stream; a step's
 *     latency is the maximum over devices.
 *
 * Shapes: head_dim 128, group 32, 2 or 4 bits, hidden = kv_heads * 128 (the
 * fused projection's constraints); anything else returns KIVI_ERR_CONFIG.
 * The device list may repeat a device (several host threads sharing one GPU).
 */
#ifndef KIVI_DRIVER_H
#define KIVI_DRIVER_H

#include "kivi_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* reference WorkloadSpec (workload.hpp:14-24) */
typedef struct kivi_workload_spec {
    int64_t batch;
    int64_t prompt_len;
    int64_t gen_len;
    int64_t layers;
    int64_t kv_heads;
    int64_t head_dim;
} kivi_workload_spec;

/* reference BenchReport (workload.hpp:38-47) plus the device-side detail */
typedef struct kivi_bench_report {
    int64_t decode_steps;
    double tokens_per_sec;      /* batch * gen_len / sum of step latencies     */
    double p50_ms, p90_ms, p99_ms;
    uint64_t peak_cache_bytes;  /* memory_bytes of every state, all devices    */
    double output_checksum;     /* sum of every decode output (fp64)           */
    double output_abs_sum;      /* sum of |output|: scale for tolerances       */
    double decode_seconds;      /* sum of step latencies (max over devices)    */
    int32_t n_devices;
} kivi_bench_report;

/*
 * Runs the benchmark.  devices[0..n_devices) are CUDA ordinals (repeats
 * allowed); batch rows are split into n_devices contiguous blocks.
 * weights/prompts/tokens: optional HOST fp32 data, all three or none —
 *   weights [layers][3][hidden][hidden] (W_q, W_k, W_v of each layer,
 *   x @ W), prompts [batch][prompt_len][hidden], tokens [gen_len][batch][hidden];
 * with none, N(0,1) data is drawn on the devices from `seed` by a
 * counter-based generator (weights scaled by 1/sqrt(hidden) as the
 * reference's SyntheticLayer, workload.cpp:116-122), identical for any
 * device list.  budget_bytes > 0: the counted cache bytes are checked after
 * the prefill and after every step (workload.cpp:175-192); exceeding it
 * returns KIVI_ERR_CAPACITY ("memory budget exceeded at ...").
 */
kivi_status kivi_run_decode_benchmark(const kivi_workload_spec* spec, const kivi_config* cfg,
                                      const int32_t* devices, int32_t n_devices, uint64_t seed,
                                      const float* weights, const float* prompts,
                                      const float* tokens, uint64_t budget_bytes,
                                      kivi_bench_report* report);

/* Last error of the calling thread for this library ("" if none). */
const char* kivi_driver_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* KIVI_DRIVER_H */
