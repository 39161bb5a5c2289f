// Probe: k_gcm reading plaintext from and writing ciphertext to pinned host
// memory directly (UVA zero-copy, no copy engines) vs the copy-engine host
// pipeline (sp_seal_host_batch), on the OPT-13B layer (19 messages).
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

#include "spgcm.h"

int main() {
    uint8_t key[32];
    for (int i = 0; i < 32; ++i) key[i] = (uint8_t)i;
    sp_ctx *ctx = nullptr;
    if (sp_ctx_create(key, &ctx) != SP_OK) return 1;
    std::vector<size_t> sizes(18, 32u << 20);
    sizes.push_back(25298944);
    size_t total = 0;
    for (auto s : sizes) total += s;
    uint8_t *h_in, *h_out, *h_tags;
    cudaHostAlloc(&h_in, total, 0);
    cudaHostAlloc(&h_out, total, 0);
    cudaHostAlloc(&h_tags, 16 * sizes.size(), 0);
    for (size_t i = 0; i < total; i += 4096) h_in[i] = (uint8_t)i;
    std::vector<sp_desc> d(sizes.size());
    size_t off = 0;
    for (size_t i = 0; i < sizes.size(); ++i) {
        d[i] = sp_desc{SP_DIR_H2D, 0u, 100 + i, sizes[i], h_in + off, h_out + off, h_tags + 16 * i, nullptr};
        off += sizes[i];
    }
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) sp_seal_batch(ctx, d.data(), (int)d.size(), s);
    cudaStreamSynchronize(s);
    const int reps = 5;
    cudaEventRecord(a, s);
    for (int r = 0; r < reps; ++r) sp_seal_batch(ctx, d.data(), (int)d.size(), s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("zero-copy seal (kernel reads/writes pinned host): %.2f ms per layer, %.1f GB/s each way (err %s)\n",
           ms / reps, total / (ms / reps) / 1e6, cudaGetErrorString(cudaGetLastError()));
    std::vector<uint8_t> ref_out(total), ref_tags(16 * sizes.size());
    for (size_t i = 0; i < total; ++i) ref_out[i] = h_out[i];
    for (size_t i = 0; i < ref_tags.size(); ++i) ref_tags[i] = h_tags[i];
    // copy-engine pipeline
    sp_seal_host_batch(ctx, d.data(), (int)d.size());
    auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; ++r) sp_seal_host_batch(ctx, d.data(), (int)d.size());
    double pms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() / reps;
    printf("copy-engine pipeline seal_host_batch: %.2f ms per layer, %.1f GB/s each way\n", pms, total / pms / 1e6);
    size_t diff = 0;
    for (size_t i = 0; i < total; ++i) diff += ref_out[i] != h_out[i];
    for (size_t i = 0; i < ref_tags.size(); ++i) diff += ref_tags[i] != h_tags[i];
    printf("outputs identical: %s\n", diff ? "NO" : "yes");
    return 0;
}
