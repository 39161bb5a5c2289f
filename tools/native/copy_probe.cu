// Device time of host<->device transfers of many small blocks (KV blocks,
// 64 KiB .. 1 MiB chunks), three ways:
//   (a) one cudaMemcpyAsync per block, back to back on one stream;
//   (b) the same split round-robin over 2 / 4 streams;
//   (c) one gather kernel per batch: SMs load/store the pinned host blocks
//       directly over PCIe (mapped memory, 16 B per lane, several loads in
//       flight per lane), `ctas` CTAs.
// CUDA events around each variant; host call cost beside it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/native/copy_probe.cu -o tools/native/copy_probe
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

struct Job {
    const uint4 *src;
    uint4 *dst;
    uint64_t n16;  // 16-byte words
};

// each warp takes 16 KiB pieces round-robin across the whole batch; 4 loads in
// flight per lane (2 KiB per warp per step)
__global__ void k_gather(const Job *jobs, int njobs, uint64_t piece16) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t p = warp;
    int j = 0;
    uint64_t base = 0;  // first piece of job j
    for (;; p += nwarps) {
        while (j < njobs && p >= base + (jobs[j].n16 + piece16 - 1) / piece16) {
            base += (jobs[j].n16 + piece16 - 1) / piece16;
            ++j;
        }
        if (j >= njobs) return;
        const Job jb = jobs[j];
        const uint64_t lo = (p - base) * piece16, hi = min(jb.n16, lo + piece16);
        for (uint64_t i = lo + lane; i < hi; i += 128) {
            uint4 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (i + 32 * k < hi) v[k] = __ldcv(jb.src + i + 32 * k);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (i + 32 * k < hi) __stcs(jb.dst + i + 32 * k, v[k]);
        }
    }
}

int main() {
    CK(cudaSetDevice(0));
    const size_t total = 256ull << 20;
    uint8_t *h, *d;
    CK(cudaHostAlloc(&h, total, cudaHostAllocMapped));
    CK(cudaMalloc(&d, total));
    uint8_t *hd;
    CK(cudaHostGetDevicePointer(&hd, h, 0));
    for (size_t i = 0; i < total; i += 4096) h[i] = (uint8_t)i;
    cudaStream_t st[4];
    for (auto &s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t a, b, f[4];
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (auto &e : f) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    Job *djobs;
    CK(cudaMalloc(&djobs, 8192 * sizeof(Job)));
    auto now = [] { return std::chrono::steady_clock::now(); };
    for (size_t sz : {16384ul, 65536ul, 229376ul, 1048576ul, 4194304ul}) {
        const int n = (int)std::min<size_t>(4096, total / sz / 2);
        for (int dir = 0; dir < 2; ++dir) {
            const bool h2d = dir == 0;
            auto src = [&](int i) -> void * { return h2d ? (void *)(h + i * sz) : (void *)(d + i * sz); };
            auto dst = [&](int i) -> void * { return h2d ? (void *)(d + i * sz) : (void *)(h + i * sz); };
            const char *dn = h2d ? "H2D" : "D2H";
            for (int ns : {1, 2, 4}) {
                for (int rep = 0; rep < 2; ++rep) {
                    CK(cudaDeviceSynchronize());
                    CK(cudaEventRecord(a, st[0]));
                    for (int k = 1; k < ns; ++k) CK(cudaStreamWaitEvent(st[k], a, 0));
                    auto t0 = now();
                    for (int i = 0; i < n; ++i)
                        CK(cudaMemcpyAsync(dst(i), src(i), sz, h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                                           st[i % ns]));
                    auto t1 = now();
                    for (int k = 1; k < ns; ++k) {
                        CK(cudaEventRecord(f[k], st[k]));
                        CK(cudaStreamWaitEvent(st[0], f[k], 0));
                    }
                    CK(cudaEventRecord(b, st[0]));
                    CK(cudaEventSynchronize(b));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, a, b));
                    if (rep)
                        printf("%s %8zu B x %4d  memcpy/%d-stream  %7.2f us/block  %6.2f GB/s  host %5.2f us/call\n", dn,
                               sz, n, ns, ms * 1e3 / n, sz * (double)n / ms / 1e6,
                               std::chrono::duration<double, std::micro>(t1 - t0).count() / n);
                }
            }
            std::vector<Job> jobs(n);
            for (int i = 0; i < n; ++i)
                jobs[i] = Job{(const uint4 *)(h2d ? hd + i * sz : d + i * sz),
                              (uint4 *)(h2d ? d + i * sz : hd + i * sz), sz / 16};
            CK(cudaMemcpy(djobs, jobs.data(), n * sizeof(Job), cudaMemcpyHostToDevice));
            for (int ctas : {16, 32, 74, 148, 296}) {
                for (int batch : {4, 32, n}) {
                    if (batch > n) continue;
                    float ms = 0;
                    for (int rep = 0; rep < 2; ++rep) {
                        CK(cudaDeviceSynchronize());
                        CK(cudaEventRecord(a, st[0]));
                        for (int i = 0; i + batch <= n; i += batch)
                            k_gather<<<ctas, 512, 0, st[0]>>>(djobs + i, batch, 1024);
                        CK(cudaEventRecord(b, st[0]));
                        CK(cudaEventSynchronize(b));
                        CK(cudaEventElapsedTime(&ms, a, b));
                    }
                    CK(cudaGetLastError());
                    const int done = n / batch * batch;
                    printf("%s %8zu B x %4d  gather %3d CTAs, %4d blocks/launch  %7.2f us/block  %6.2f GB/s\n", dn, sz,
                           done, ctas, batch, ms * 1e3 / done, sz * (double)done / ms / 1e6);
                }
            }
        }
    }
    return 0;
}
