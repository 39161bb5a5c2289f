// Host-side cost of the CUDA calls the engine's issuing thread makes (no
// device back-pressure: each batch of N calls starts on drained streams and
// N is far below the launch queue depth).  Prints microseconds per call.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include tools/native/host_api_cost.cu \
//        -L paper_2411_03357_b200/lib -lspgcm -Xlinker -rpath,'$ORIGIN/../../paper_2411_03357_b200/lib' \
//        -o tools/native/host_api_cost
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <functional>
#include <vector>

#include "spgcm.h"

__global__ void k_empty() {}
struct Big {
    unsigned char b[2400];
};
__global__ void k_big_params(const __grid_constant__ Big p) {
    if (p.b[0] == 17 && threadIdx.x == 999) printf("x");
}

static void measure(const char *name, int n, cudaStream_t s, const std::function<void(int)> &fn) {
    double best = 1e30;
    for (int rep = 0; rep < 5; ++rep) {
        cudaDeviceSynchronize();
        const auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < n; ++i) fn(i);
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        best = std::min(best, us / n);
        cudaDeviceSynchronize();
    }
    printf("%-44s %7.2f us/call\n", name, best);
    (void)s;
}

int main() {
    cudaStream_t s, s2;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    uint8_t key[32] = {1};
    sp_ctx *ctx;
    if (sp_ctx_create(key, &ctx)) return 1;
    uint8_t *dbuf, *hbuf, *tags;
    cudaMalloc(&dbuf, 64 << 20);
    cudaMalloc(&tags, 1 << 16);
    cudaHostAlloc(&hbuf, 64 << 20, cudaHostAllocDefault);
    std::vector<cudaEvent_t> ev(256);
    for (auto &e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    const int N = 100;
    measure("cudaLaunchKernel (empty, <<<1,32>>>)", N, s, [&](int) { k_empty<<<1, 32, 0, s>>>(); });
    measure("cudaLaunchKernel (2.4 KB params)", N, s, [&](int) { k_big_params<<<1, 32, 0, s>>>(Big{}); });
    measure("cudaEventRecord", N, s, [&](int i) { cudaEventRecord(ev[i], s); });
    measure("cudaStreamWaitEvent", N, s, [&](int i) { cudaStreamWaitEvent(s2, ev[i], 0); });
    measure("cudaEventQuery (completed)", N, s, [&](int i) { cudaEventQuery(ev[i]); });
    measure("cudaMemcpyAsync H2D 224 KiB pinned", N, s,
            [&](int i) { cudaMemcpyAsync(dbuf + i * 229376, hbuf + i * 229376, 229376, cudaMemcpyHostToDevice, s); });
    measure("cudaMemcpyAsync D2H 224 KiB pinned", N, s,
            [&](int i) { cudaMemcpyAsync(hbuf + i * 229376, dbuf + i * 229376, 229376, cudaMemcpyDeviceToHost, s); });
    auto seal = [&](int n, size_t len, int i) {
        std::vector<sp_desc> d(n);
        for (int k = 0; k < n; ++k)
            d[k] = sp_desc{SP_DIR_H2D, 0u, (uint64_t)(i * n + k), len, dbuf + k * len, dbuf + k * len, tags + 16 * k,
                           nullptr};
        sp_seal_batch(ctx, d.data(), n, s);
    };
    measure("sp_seal_batch 1 NOP (SmallTabs)", N, s, [&](int i) { seal(1, 1, i); });
    measure("sp_seal_batch 1 x 224 KiB (BigTabs)", N, s, [&](int i) { seal(1, 229376, i); });
    measure("sp_seal_batch 4 x 224 KiB (BigTabs)", N, s, [&](int i) { seal(4, 229376, i); });
    measure("sp_seal_batch 32 x 224 KiB (BigTabs)", 20, s, [&](int i) { seal(32, 229376, i); });
    printf("launches %llu\n", (unsigned long long)sp_launch_count());
    return 0;
}
