// Device time per k_gcm launch for small batches (NOP pads, tokens, KV
// blocks), back to back on one stream and with a cross-stream event wait
// between launches (the engine's small-batch pattern), via libspgcm's C-ABI.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include tools/native/launch_latency.cu \
//        -L paper_2411_03357_b200/lib -lspgcm -Xlinker -rpath,$PWD/paper_2411_03357_b200/lib -o /tmp/ll
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
    if (sp_ctx_create(key, &ctx) != SP_OK) return 1;
    cudaStream_t s, s2;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    uint8_t *buf, *tags;
    cudaMalloc(&buf, 64 << 20);
    cudaMalloc(&tags, 16 * 1024);
    cudaMemset(buf, 0, 64 << 20);
    cudaEvent_t a, b, x;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
    {  // launch floor: an empty kernel back to back
        cudaEvent_t a0, b0;
        cudaEventCreate(&a0);
        cudaEventCreate(&b0);
        for (int w = 0; w < 100; ++w) k_empty<<<1, 32, 0, s>>>();
        cudaEventRecord(a0, s);
        for (int r = 0; r < 2000; ++r) k_empty<<<1, 32, 0, s>>>();
        cudaEventRecord(b0, s);
        cudaEventSynchronize(b0);
        float ms = 0;
        cudaEventElapsedTime(&ms, a0, b0);
        printf("%-18s %-16s %7.2f us/launch\n", "empty kernel", "back-to-back", ms * 1e3 / 2000);
    }
    struct Case {
        const char *name;
        int n;
        size_t size;
    } cases[] = {{"1 NOP (1 B)", 1, 1},       {"8 NOPs", 8, 1},           {"1 x 2 KiB token", 1, 2048},
                 {"1 x 16 KiB", 1, 16384}, {"1 x 64 KiB", 1, 65536}, {"1 x 224 KiB KV", 1, 229376}, {"4 x 224 KiB KV", 4, 229376}, {"32 x 224 KiB KV", 32, 229376},
                 {"1 x 1 MiB", 1, 1 << 20}};
    for (auto &c : cases) {
        std::vector<sp_desc> d(c.n);
        for (int i = 0; i < c.n; ++i) {
            d[i] = sp_desc{SP_DIR_H2D, 0u, (uint64_t)i, c.size, buf + i * c.size, buf + i * c.size, tags + 16 * i, nullptr};
        }
        {  // device time alone: the same launches captured once in a CUDA graph, replayed
            const int reps = 200;
            cudaGraph_t g;
            cudaGraphExec_t ge;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
            for (int r = 0; r < reps; ++r) sp_seal_batch(ctx, d.data(), c.n, s);
            cudaStreamEndCapture(s, &g);
            if (cudaGraphInstantiate(&ge, g, 0) == cudaSuccess) {
                cudaGraphLaunch(ge, s);
                cudaStreamSynchronize(s);
                cudaEventRecord(a, s);
                for (int k = 0; k < 5; ++k) cudaGraphLaunch(ge, s);
                cudaEventRecord(b, s);
                cudaEventSynchronize(b);
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                printf("%-18s %-16s %7.2f us/launch\n", c.name, "graph (device)", ms * 1e3 / (5 * reps));
                cudaGraphExecDestroy(ge);
            } else {
                printf("%-18s %-16s   n/a (capture failed: %s)\n", c.name, "graph (device)", cudaGetErrorString(cudaGetLastError()));
            }
            cudaGraphDestroy(g);
            cudaGetLastError();
        }
        for (int mode = 0; mode < 2; ++mode) {
            const int reps = 2000;
            for (int w = 0; w < 50; ++w) sp_seal_batch(ctx, d.data(), c.n, s);
            cudaStreamSynchronize(s);
            const auto h0 = std::chrono::steady_clock::now();
            cudaEventRecord(a, s);
            for (int r = 0; r < reps; ++r) {
                if (mode == 1) {  // event hop through a second stream before every launch
                    cudaEventRecord(x, s);
                    cudaStreamWaitEvent(s2, x, 0);
                    cudaEventRecord(x, s2);
                    cudaStreamWaitEvent(s, x, 0);
                }
                sp_seal_batch(ctx, d.data(), c.n, s);
            }
            cudaEventRecord(b, s);
            const double host_us =
                std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count() / reps;
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("%-18s %-16s %7.2f us/launch  (host issue %.2f us/launch)\n", c.name,
                   mode ? "event-hop" : "back-to-back", ms * 1e3 / reps, host_us);
        }
    }
    printf("launches %llu\n", (unsigned long long)sp_launch_count());
    return 0;
}
