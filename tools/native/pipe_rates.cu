// Issue rates of the SM pipes k_gcm lives on, measured on the B200 itself
// ("measure the sm_100 INT32/LOP3 lane count, do not assume it").
// Each case runs a fully occupied grid (148 x 4 CTAs x 512 threads) of
// unrolled, independent chains of one instruction and reports
//   ops per SM per clock = (threads x ops per thread) / (SMs x cycles),
// cycles from clock64() on each CTA (max over CTAs), i.e. lanes per SM per
// clock of that pipe.  LDS cases use lane-private addresses (conflict-free,
// as k_gcm's replicated tables) with a data-dependent address chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/native/pipe_rates.cu -o /tmp/pipe_rates
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kThreads = 512;
constexpr int kIters = 4096;
constexpr int kChains = 8;

__device__ unsigned long long g_cycles[148 * 8];
__device__ uint32_t g_sink[1];

#define CHAIN_LOOP(...)                                                   \
    _Pragma("unroll 1") for (int it = 0; it < kIters; ++it) {              \
        _Pragma("unroll") for (int c = 0; c < kChains; ++c) { __VA_ARGS__; }      \
    }

template <int OP>
__global__ void __launch_bounds__(kThreads, 4) k_alu(uint32_t seed, int per_sm_slot) {
    uint32_t v[kChains], w = seed ^ threadIdx.x, z = seed * 3u + 1u;
#pragma unroll
    for (int c = 0; c < kChains; ++c) v[c] = seed + c * 0x9e3779b9u + threadIdx.x;
    __syncthreads();
    const unsigned long long t0 = clock64();
    if (OP == 0) {  // LOP3 (3-input xor, the AES column merge)
        CHAIN_LOOP(asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(w), "r"(z)));
    } else if (OP == 1) {  // PRMT (byte extract / lookup offset)
        CHAIN_LOOP(asm volatile("prmt.b32 %0, %0, %1, 0x5504;" : "+r"(v[c]) : "r"(w)));
    } else if (OP == 2) {  // IADD3
        CHAIN_LOOP(asm volatile("add.u32 %0, %0, %1;" : "+r"(v[c]) : "r"(w)));
    } else if (OP == 3) {  // SHF (funnel shift, GHASH byte shift)
        CHAIN_LOOP(asm volatile("shf.l.wrap.b32 %0, %0, %1, 8;" : "+r"(v[c]) : "r"(w)));
    } else if (OP == 4) {  // LOP (2-input and, last-round masks)
        CHAIN_LOOP(asm volatile("and.b32 %0, %0, %1;" : "+r"(v[c]) : "r"(w | 0x80000000u)));
    }
    const unsigned long long t1 = clock64();
    __syncthreads();
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc ^= v[c];
    if (acc == 0x12345678u) g_sink[0] = acc;
    if (threadIdx.x == 0 && per_sm_slot >= 0) g_cycles[blockIdx.x] = t1 - t0;
}

// LDS.32 / LDS.128 from a lane-private copy of a 256-entry table (entry
// stride 256 B as k_gcm's T tables), next address from the loaded value.
template <int WIDE>
__global__ void __launch_bounds__(kThreads, 1) k_lds(uint32_t seed, int per_sm_slot) {
    extern __shared__ __align__(16) uint32_t tab[];  // 64 KiB: 256 entries x 256 B
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) tab[i] = ((i * 2654435761u) >> 8) & 0xffu;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    // k_gcm's lookup: one PRMT forms (byte << 8) | lane constant, then
    // LDS [reg + imm] at the absolute dynamic-smem base (0x400, checked)
    if (static_cast<uint32_t>(__cvta_generic_to_shared(tab)) != 0x400u) __trap();
    const uint32_t lc = WIDE ? (lane & 7u) * 16u : lane * 4u;
    uint32_t v[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) v[c] = (seed + c * 77u + threadIdx.x) & 0xffu;
    const unsigned long long t0 = clock64();
    if (!WIDE) {
        CHAIN_LOOP({
            uint32_t r;
            const uint32_t a = __byte_perm(v[c], lc, 0x5504u);
            asm volatile("ld.shared.u32 %0, [%1+0x400];" : "=r"(r) : "r"(a));
            v[c] = r;
        });
    } else {
        CHAIN_LOOP({
            uint32_t r0, r1, r2, r3;
            const uint32_t a = __byte_perm(v[c], lc, 0x5504u);
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4+0x400];" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a));
            v[c] = r0 ^ r1 ^ r2 ^ r3;
        });
    }
    const unsigned long long t1 = clock64();
    __syncthreads();
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc ^= v[c];
    if (acc == 0x12345678u) g_sink[0] = acc;
    if (threadIdx.x == 0 && per_sm_slot >= 0) g_cycles[blockIdx.x] = t1 - t0;
}

static double run(const char *name, void (*k)(uint32_t, int), int ctas_per_sm, int smem, int sms) {
    const int grid = sms * ctas_per_sm;
    if (smem) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<grid, kThreads, smem>>>(1u, 0);  // warm
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<grid, kThreads, smem>>>(7u, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    static unsigned long long cyc[148 * 8];
    cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * grid);
    unsigned long long mx = 0;
    for (int i = 0; i < grid; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
    const double ops = (double)grid * kThreads * kIters * kChains;
    // CTAs of one SM run concurrently: per-SM rate = ops per SM / max cycles
    const double per_sm_clk = ops / sms / (double)mx;
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    printf("{\"op\": \"%s\", \"lanes_per_sm_per_clk\": %.2f, \"kernel_ms\": %.3f, \"ctas_per_sm\": %d, "
           "\"gops_per_s\": %.1f}\n",
           name, per_sm_clk, ms, ctas_per_sm, ops / (ms * 1e-3) / 1e9);
    return per_sm_clk;
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    const int sms = prop.multiProcessorCount;
    printf("{\"device\": \"%s\", \"sms\": %d}\n", prop.name, sms);
    run("LOP3.LUT", k_alu<0>, 4, 0, sms);
    run("PRMT", k_alu<1>, 4, 0, sms);
    run("IADD3", k_alu<2>, 4, 0, sms);
    run("SHF", k_alu<3>, 4, 0, sms);
    run("LOP (and)", k_alu<4>, 4, 0, sms);
    run("LDS.32 lane-private", k_lds<0>, 1, 65536, sms);
    run("LDS.128 8-copy", k_lds<1>, 1, 65536, sms);
    return 0;
}
