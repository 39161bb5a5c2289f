// Latency of the host-buffer entry points (encrypt_at / decrypt_at shape).
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <vector>
#include "spgcm.h"

int main() {
    uint8_t key[32];
    for (int i = 0; i < 32; ++i) key[i] = (uint8_t)(3 * i);
    sp_ctx *ctx = nullptr;
    if (sp_ctx_create(key, &ctx) != SP_OK) { printf("ctx: %s\n", sp_last_error()); return 1; }
    for (size_t n : {(size_t)1, (size_t)2048, (size_t)229376, (size_t)1 << 20, (size_t)32 << 20}) {
        uint8_t *p, *c, *q;
        cudaHostAlloc(&p, n, 0); cudaHostAlloc(&c, n, 0); cudaHostAlloc(&q, n, 0);
        for (size_t i = 0; i < n; ++i) p[i] = (uint8_t)(i * 7);
        uint8_t tag[16];
        for (int w = 0; w < 5; ++w) { sp_seal_host(ctx, 0, 1, p, n, c, tag); sp_open_host(ctx, 0, 1, c, n, tag, q); }
        const int reps = n > (1 << 22) ? 20 : 200;
        auto t0 = std::chrono::steady_clock::now();
        for (int r = 0; r < reps; ++r) sp_seal_host(ctx, 0, (uint64_t)r, p, n, c, tag);
        auto t1 = std::chrono::steady_clock::now();
        for (int r = 0; r < reps; ++r) sp_open_host(ctx, 0, (uint64_t)(reps - 1), c, n, tag, q);
        auto t2 = std::chrono::steady_clock::now();
        double us_s = std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
        double us_o = std::chrono::duration<double, std::micro>(t2 - t1).count() / reps;
        printf("%9zu B: sp_seal_host %8.1f us (%6.2f GB/s)  sp_open_host %8.1f us\n", n, us_s, n / us_s / 1e3, us_o);
        cudaFreeHost(p); cudaFreeHost(c); cudaFreeHost(q);
    }
    return 0;
}
