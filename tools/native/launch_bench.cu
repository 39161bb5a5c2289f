// Per-launch cost of small seal batches from C (no Python in the loop).
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <vector>
#include "spgcm.h"

__global__ void k_empty() {}

int main() {
    uint8_t key[32];
    for (int i = 0; i < 32; ++i) key[i] = (uint8_t)i;
    sp_ctx *ctx = nullptr;
    if (sp_ctx_create(key, &ctx) != SP_OK) { printf("ctx: %s\n", sp_last_error()); return 1; }
    cudaStream_t s;
    cudaStreamCreate(&s);
    const size_t sizes[] = {1, 2048, 65536, 229376, 1 << 20, 4 << 20, 32 << 20};
    uint8_t *buf, *out, *tags;
    cudaMalloc(&buf, 64u << 20);
    cudaMalloc(&out, 64u << 20);
    cudaMalloc(&tags, 16 * 64);
    cudaMemset(buf, 7, 64u << 20);
    {
        for (int w = 0; w < 20; ++w) k_empty<<<148, 512, 0, s>>>();
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a, s);
        for (int r = 0; r < 200; ++r) k_empty<<<148, 512, 0, s>>>();
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("empty kernel 148x512: %8.2f us/launch\n", ms * 1000 / 200);
    }
    {
        // host-side issue cost per launch: inline descriptors (<= 32) vs the pinned ring
        std::vector<sp_desc> d(256);
        for (int i = 0; i < 256; ++i) d[i] = sp_desc{0, 0, (uint64_t)i, 16, buf + 16 * i, out + 16 * i, tags + 16 * (i % 64), nullptr};
        for (int nmsg : {1, 32, 33, 64, 256}) {
            for (int w = 0; w < 50; ++w) sp_seal_batch(ctx, d.data(), nmsg, s);
            cudaStreamSynchronize(s);
            auto t0 = std::chrono::steady_clock::now();
            for (int r = 0; r < 200; ++r) sp_seal_batch(ctx, d.data(), nmsg, s);
            double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / 200;
            cudaStreamSynchronize(s);
            printf("host issue cost, %3d msgs: %6.2f us/launch\n", nmsg, us);
        }
    }
    for (size_t n : sizes) {
        for (int nmsg : {1, 8, 32}) {
            if (n * nmsg > (64u << 20)) continue;
            std::vector<sp_desc> d(nmsg);
            for (int i = 0; i < nmsg; ++i) d[i] = sp_desc{0, 0, (uint64_t)i, n, buf + i * n, out + i * n, tags + 16 * i, nullptr};
            for (int w = 0; w < 20; ++w) sp_seal_batch(ctx, d.data(), nmsg, s);
            cudaStreamSynchronize(s);
            const int reps = 200;
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a, s);
            for (int r = 0; r < reps; ++r) sp_seal_batch(ctx, d.data(), nmsg, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("msgs=%2d x %9zu B : %8.2f us/launch  %8.2f GB/s\n", nmsg, n, ms * 1000 / reps,
                   (double)n * nmsg * reps / (ms * 1e6));
        }
    }
    sp_ctx_destroy(ctx);
    return 0;
}
