// B200 cells of the reference simulator's cost model (simulator.py:57-127,
// REFERENCE_LATENCY_US / REFERENCE_THROUGHPUT_GBS), measured here:
//   plain : one pinned cudaMemcpyAsync H2D (api latency = host time of the
//           call; throughput = back-to-back copies, device-timed)
//   cc    : one confidential transfer as the B200 data plane performs it on
//           the on-the-fly path (SyncCc: every transfer sealed and opened on
//           the fly): H2D copy + seal (H2D counter) + receiver open, waited
//           for synchronously (api latency), or pipelined back to back
//           (throughput).
// Prints one JSON object; tools/sim_calibrated.py fits the CostModel.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

#include "spgcm.h"

static double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
    uint8_t key[32];
    for (int i = 0; i < 32; ++i) key[i] = (uint8_t)(11 * i + 1);
    sp_ctx *ctx = nullptr;
    if (sp_ctx_create(key, &ctx) != SP_OK) {
        printf("{\"error\": \"%s\"}\n", sp_last_error());
        return 1;
    }
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    const size_t sizes[] = {32, 128 * 1024, 1 << 20, 32 << 20};
    const size_t maxn = 32 << 20;
    uint8_t *h, *d, *d2, *tags;
    int32_t *st;
    cudaHostAlloc(&h, maxn, 0);
    for (size_t i = 0; i < maxn; ++i) h[i] = (uint8_t)(i * 13);
    cudaMalloc(&d, maxn);
    cudaMalloc(&d2, maxn);
    cudaMalloc(&tags, 16);
    cudaMalloc(&st, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    printf("{\"device\": \"B200\", \"cells\": [");
    bool first = true;
    for (size_t n : sizes) {
        const int reps = n >= (16u << 20) ? 30 : 300;
        // ---- plain: API latency and sustained throughput
        for (int w = 0; w < 10; ++w) cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        double t0 = now_us();
        for (int r = 0; r < reps; ++r) cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s);
        double api_plain = (now_us() - t0) / reps;
        cudaStreamSynchronize(s);
        cudaEventRecord(a, s);
        for (int r = 0; r < reps; ++r) cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        double gbs_plain = (double)n * reps / (ms * 1e6);
        // ---- cc: copy + seal + open
        sp_desc sd{SP_DIR_H2D, 0, 0, n, d, d, tags, nullptr};
        sp_desc od{SP_DIR_H2D, 0, 0, n, d, d2, tags, st};
        auto transfer = [&](uint64_t iv) {
            cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s);
            sd.iv = od.iv = iv;
            sp_seal_batch(ctx, &sd, 1, s);
            sp_open_batch(ctx, &od, 1, s);
        };
        for (int w = 0; w < 10; ++w) transfer((uint64_t)w);
        cudaStreamSynchronize(s);
        t0 = now_us();
        for (int r = 0; r < reps; ++r) {
            transfer((uint64_t)r);
            cudaStreamSynchronize(s);  // synchronous, like the CC driver's inline path
        }
        double api_cc = (now_us() - t0) / reps;
        cudaEventRecord(a, s);
        for (int r = 0; r < reps; ++r) transfer((uint64_t)r);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double gbs_cc = (double)n * reps / (ms * 1e6);
        // ---- crypto alone (seal + open of device-resident data)
        cudaEventRecord(a, s);
        for (int r = 0; r < reps; ++r) {
            sd.iv = od.iv = (uint64_t)r;
            sp_seal_batch(ctx, &sd, 1, s);
            sp_open_batch(ctx, &od, 1, s);
        }
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double gbs_crypto = (double)n * reps / (ms * 1e6);
        printf("%s{\"size\": %zu, \"plain_api_us\": %.3f, \"plain_gbs\": %.3f, \"cc_api_us\": %.3f, \"cc_gbs\": %.3f, "
               "\"crypto_seal_open_gbs\": %.3f}",
               first ? "" : ", ", n, api_plain, gbs_plain, api_cc, gbs_cc, gbs_crypto);
        first = false;
    }
    printf("]}\n");
    return 0;
}
