// Primitives of a persistent crypto server: what a stream-ordered
// hand-off to a resident kernel costs compared with a kernel launch.
//   stream s:  [writeValue(ready[k] = k), waitValue(done[k] >= k)]  (one cuStreamBatchMemOp)
//   server:    one warp polls ready[], answers done[]
// Reports device time per item on s (CUDA events, back to back and behind a
// cross-stream event), the host cost of the memop call, and the same for an
// empty kernel launch.  The server exits on a host-mapped stop word or after
// a hard 20 s deadline (globaltimer), so a lost hand-off cannot hang the box.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/native/server_probe.cu -o tools/native/server_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

typedef CUresult (*PFN_batch)(CUstream, unsigned int, CUstreamBatchMemOpParams *, unsigned int);

constexpr uint32_t kSlots = 1024;

__device__ __forceinline__ uint64_t gtime() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t ld_acq(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// one lane polls the next slot; answers in order
__global__ void k_server(const uint32_t *ready, uint32_t *done, const volatile uint32_t *stop, uint32_t *served) {
    if (threadIdx.x != 0) return;
    const uint64_t deadline = gtime() + 20ull * 1000000000ull;
    uint32_t k = 1;
    uint32_t spins = 0;
    for (;;) {
        const uint32_t slot = k % kSlots;
        if (ld_acq(ready + slot) == k) {
            st_rel(done + slot, k);
            ++k;
            continue;
        }
        if ((++spins & 255u) == 0) {
            if (*stop) break;
            if (gtime() > deadline) break;
        }
    }
    *served = k - 1;
}

__global__ void k_empty() {}

int main() {
    CK(cudaSetDevice(0));
    PFN_batch batch = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuStreamBatchMemOp", reinterpret_cast<void **>(&batch), cudaEnableDefault, &q));
    if (!batch) {
        printf("no cuStreamBatchMemOp\n");
        return 1;
    }
    uint32_t *ready, *done, *served;
    CK(cudaMalloc(&ready, kSlots * 4));
    CK(cudaMalloc(&done, kSlots * 4));
    CK(cudaMalloc(&served, 4));
    CK(cudaMemset(ready, 0, kSlots * 4));
    CK(cudaMemset(done, 0, kSlots * 4));
    uint32_t *stop_h, *stop_d;
    CK(cudaHostAlloc(&stop_h, 4, cudaHostAllocMapped));
    *stop_h = 0;
    CK(cudaHostGetDevicePointer(&stop_d, stop_h, 0));
    cudaStream_t s, s2, srv;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&srv, cudaStreamNonBlocking));
    uint8_t *hbuf, *dbuf;
    CK(cudaHostAlloc(&hbuf, 64 << 20, cudaHostAllocDefault));
    CK(cudaMalloc(&dbuf, 64 << 20));
    cudaEvent_t a, b, x;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    CK(cudaDeviceSynchronize());

    auto now = [] { return std::chrono::steady_clock::now(); };
    auto us = [](auto t0, auto t1) { return std::chrono::duration<double, std::micro>(t1 - t0).count(); };

    // empty kernel chain
    {
        for (int w = 0; w < 100; ++w) k_empty<<<1, 32, 0, s>>>();
        CK(cudaEventRecord(a, s));
        auto t0 = now();
        for (int r = 0; r < 2000; ++r) k_empty<<<1, 32, 0, s>>>();
        auto t1 = now();
        CK(cudaEventRecord(b, s));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        printf("empty kernel        back-to-back  device %6.2f us/item  host %5.2f us/call\n", ms * 1e3 / 2000,
               us(t0, t1) / 2000);
        for (int r = 0; r < 2000; ++r) {
            CK(cudaEventRecord(x, s2));
            CK(cudaStreamWaitEvent(s, x, 0));
            k_empty<<<1, 32, 0, s>>>();
        }
        CK(cudaEventRecord(a, s));
        for (int r = 0; r < 2000; ++r) {
            CK(cudaEventRecord(x, s2));
            CK(cudaStreamWaitEvent(s, x, 0));
            k_empty<<<1, 32, 0, s>>>();
        }
        CK(cudaEventRecord(b, s));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms, a, b));
        printf("empty kernel        event-hop     device %6.2f us/item\n", ms * 1e3 / 2000);
    }

    k_server<<<1, 32, 0, srv>>>(ready, done, stop_d, served);
    uint32_t k = 0;
    auto item = [&](cudaStream_t st) {
        ++k;
        CUstreamBatchMemOpParams ops[2];
        memset(ops, 0, sizeof ops);
        ops[0].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
        ops[0].writeValue.address = (CUdeviceptr)(ready + k % kSlots);
        ops[0].writeValue.value = k;
        ops[0].writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
        ops[1].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
        ops[1].waitValue.address = (CUdeviceptr)(done + k % kSlots);
        ops[1].waitValue.value = k;
        ops[1].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
        CUresult r = batch((CUstream)st, 2, ops, 0);
        if (r != CUDA_SUCCESS) {
            printf("batch memop failed %d\n", (int)r);
            *stop_h = 1;
            exit(1);
        }
    };
    const int N = 2000;
    for (int w = 0; w < 100; ++w) item(s);
    CK(cudaEventRecord(a, s));
    auto t0 = now();
    for (int r = 0; r < N; ++r) item(s);
    auto t1 = now();
    CK(cudaEventRecord(b, s));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("server hand-off     back-to-back  device %6.2f us/item  host %5.2f us/call\n", ms * 1e3 / N, us(t0, t1) / N);

    CK(cudaEventRecord(a, s));
    t0 = now();
    for (int r = 0; r < N; ++r) {
        CK(cudaEventRecord(x, s2));
        CK(cudaStreamWaitEvent(s, x, 0));
        item(s);
    }
    t1 = now();
    CK(cudaEventRecord(b, s));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("server hand-off     event-hop     device %6.2f us/item  host %5.2f us/iter\n", ms * 1e3 / N, us(t0, t1) / N);

    // with a 224 KiB H2D copy ahead of every item (swap-in then open)
    CK(cudaEventRecord(a, s));
    for (int r = 0; r < N / 4; ++r) {
        CK(cudaMemcpyAsync(dbuf + (r % 64) * 229376, hbuf + (r % 64) * 229376, 229376, cudaMemcpyHostToDevice, s));
        item(s);
    }
    CK(cudaEventRecord(b, s));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("copy 224K + server  back-to-back  device %6.2f us/item\n", ms * 1e3 / (N / 4));
    CK(cudaEventRecord(a, s));
    for (int r = 0; r < N / 4; ++r) {
        CK(cudaMemcpyAsync(dbuf + (r % 64) * 229376, hbuf + (r % 64) * 229376, 229376, cudaMemcpyHostToDevice, s));
        k_empty<<<1, 32, 0, s>>>();
    }
    CK(cudaEventRecord(b, s));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("copy 224K + kernel  back-to-back  device %6.2f us/item\n", ms * 1e3 / (N / 4));
    CK(cudaEventRecord(a, s));
    for (int r = 0; r < N / 4; ++r)
        CK(cudaMemcpyAsync(dbuf + (r % 64) * 229376, hbuf + (r % 64) * 229376, 229376, cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(b, s));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("copy 224K alone     back-to-back  device %6.2f us/item\n", ms * 1e3 / (N / 4));

    *stop_h = 1;
    CK(cudaStreamSynchronize(srv));
    uint32_t sv = 0;
    CK(cudaMemcpy(&sv, served, 4, cudaMemcpyDeviceToHost));
    printf("served %u items (posted %u)\n", sv, k);
    return 0;
}
