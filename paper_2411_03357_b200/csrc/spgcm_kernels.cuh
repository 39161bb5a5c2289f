// sm_100a device code for the AES-256-GCM seal/open path.
//
// Replaces the arithmetic the reference reaches through
// `AESGCM(key).encrypt/decrypt` (channel.py:96 and channel.py:111-113).
//
// Design:
//  * One persistent CTA per SM (512 threads, 192 KB of shared tables):
//      [0,   64K)  AES T0/T1, entry v at v*256, T0 copy c at +4c, T1 at +128+4c
//      [64K,128K)  AES T2/T3, same layout
//      [128K,192K) GHASH: entry v at v*256, M_G[v] copy c (c<8) at +16c,
//                  R8[v] copy c (c<32) at +128+4c
//    Every lane reads its own copy, so the random-index lookups are
//    bank-conflict free (LDS.32: bank = lane; LDS.128: bank group = lane&7).
//    The 256-byte entry stride lets one PRMT build the full lookup offset
//    (byte << 8 | lane constant).
//  * Work unit = a "row" of 32 consecutive 16-byte GCM blocks, rows aligned
//    to the END of each message.  Each warp takes a contiguous range of rows
//    (whole batch flattened), so loads/stores are 512-byte coalesced and the
//    GHASH Horner chain per lane runs with stride multiplier G = H^32.
//  * A run of rows of one message ends with: lane multiply by H^(32-lane)
//    (nibble tables in HBM), warp XOR-reduce, multiply by H^(32*r_end+1) =
//    F[r_end/16] * H^(32*(r_end%16)) (lane-parallel nibble lookups), then
//    either the final tag (run covers the message) or an atomic XOR into a
//    per-message accumulator with a rows-done counter (last finisher tags).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace spgcm {

constexpr int kThreads = 512;
constexpr int kThreadsSmall = 128;  // latency variant (SmallTabs): 4 warps, up to 4 CTAs per SM
constexpr int kWarpsPerCta = kThreads / 32;
constexpr uint64_t kMaxMsg = 32ull << 20;
constexpr uint32_t kMaxRows = (uint32_t)((kMaxMsg / 16 + 31) / 32);  // 65536
constexpr uint32_t kNumF = (kMaxRows + 15) / 16;                     // 4096
// nibble-table index layout (each table: 32 positions x 16 values x uint4 = 8 KiB)
constexpr uint32_t kNtLane = 0;          // H^e, e = 1..33 -> index e-1 (H^(33-l): runs ending at their message's end)
constexpr uint32_t kNtF = 33;            // F_a = H^(512a+1), a < kNumF
constexpr uint32_t kNtP32 = kNtF + kNumF;  // H^(32b), b = 1..15 -> kNtP32 + b - 1
// Short tails: a run ending r_end < kNumG rows before its message's end
// scales by H^(32 r_end + 1) in ONE lookup (instead of F then H^(32b)), and
// the tree's last step folds that scaling in: W = D0 H^17 + D1 H, so
// W x H^(32 r_end + 1) = D0 x H^(32 r_end + 18) + D1 x H^(32 r_end + 2).
constexpr uint32_t kNumG = 512;
constexpr uint32_t kNtG1 = kNtP32 + 15;        // H^(32r + 1),  r < kNumG
constexpr uint32_t kNtG2 = kNtG1 + kNumG;      // H^(32r + 2)
constexpr uint32_t kNtG18 = kNtG2 + kNumG;     // H^(32r + 18)
constexpr uint32_t kNumNt = kNtG18 + kNumG;
constexpr uint32_t kNtEntries = 32 * 16;

constexpr uint32_t kSmAes0 = 0;
constexpr uint32_t kSmAes1 = 65536;
constexpr uint32_t kSmGh = 131072;
constexpr uint32_t kSmemBytes = 196608;
// Lane-combine tree (KParamsT.reserved & kTreeBit): nibble tables of H^1,
// H^2, H^4, H^8 (8 KiB each, same layout as the HBM nibble tables) after
// the BigTabs tables.
constexpr uint32_t kSmTree = 196608;
constexpr uint32_t kSmemBytesTree = kSmemBytes + 4u * 8192u;  // 224 KiB (of 227)
constexpr uint32_t kTreeBit = 1u;

struct MsgDev {
    const uint8_t *src;
    uint8_t *dst;
    uint8_t *tag;
    int32_t *status;
    uint64_t len;
    uint64_t iv;
    uint64_t row_begin;  // global row index of this message's first row
    uint32_t rows;
    uint32_t dir;
};

// Batches of up to kInline messages travel inside the kernel parameters (no
// descriptor copy, no host staging on the launch path).  Two parameter
// blocks: 32 inline descriptors (2.4 KiB) for the common case, 256 (16.6
// KiB) for 33-256 message batches (host issue 3.5 us vs ~17 us through the
// pinned staging ring + copy + event).  Keeping most launches small matters:
// the driver's ring of pending launch parameters is finite, and with 16 KiB
// blocks a deep queue of pending launches blocks the issuing thread.
constexpr uint32_t kInline = 32;
constexpr uint32_t kInlineBig = 256;
constexpr uint32_t kInlineTiny = 4;  // 0.5 KiB of parameters: the common KV / NOP-run / token launch

// MsgDev.dir: low byte = channel direction (nonce word 0), this bit = open
// (verify + decrypt) instead of seal, so one launch can mix both.
constexpr uint32_t kOpenBit = 0x100u;
// MsgDev.dir: this bit = write *status only on failure (SP_STATUS_ON_FAILURE)
constexpr uint32_t kStickyBit = 0x200u;

// Fused levels (sp_crypt_levels): up to kMaxLevels dependent batches in ONE
// launch.  Level L's rows split into lvl_unit[L+1]-lvl_unit[L] units; warps
// claim units in global order from ctl[0], and a unit of level L > 0 starts
// once every unit of level L-1 is done (ctl[2+L-1]).  Claiming in order makes
// it deadlock-free without co-residency: every unit a waiter depends on was
// claimed earlier by a warp that is already running.  The last warp to exit
// (ctl[1]) resets the counters for the next launch on the stream.
constexpr uint32_t kMaxLevels = 8;
constexpr uint32_t kCtlWords = 2 + kMaxLevels;

template <uint32_t INL>
struct KParamsT {
    MsgDev inl[INL];
    uint32_t rk[60];
    const uint32_t *ttab;  // T0..T3 [4][256] then R8[256]
    const uint4 *mg;       // M_G[256], G = H^32
    const uint4 *nt;       // nibble tables [kNumNt][32][16]
    const MsgDev *msgs;
    uint32_t *acc;         // per message: 4 words XOR accumulator + rows done (stride 8)
    uint64_t row_begin;    // rows [row_begin, row_end) of the flattened batch
    uint64_t row_end;
    uint32_t nmsgs;
    uint32_t reserved;
    uint32_t warps_used;   // warps per CTA that own rows (<= kWarpsPerCta)
    uint32_t nlevels;      // fused launches only (k_gcm<.., true>)
    uint32_t lvl_unit[kMaxLevels + 1];
    uint64_t lvl_row[kMaxLevels + 1];
    uint32_t *ctl;         // claim, exit, done[kMaxLevels]
};
using KParams = KParamsT<kInline>;
using KParamsTiny = KParamsT<kInlineTiny>;
using KParamsBig = KParamsT<kInlineBig>;

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

__device__ __forceinline__ uint32_t word_of(const uint4 &v, int k) {
    return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}

__device__ __forceinline__ uint4 xor4(uint4 a, uint4 b) {
    return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w);
}

// ---- AES-256 on lane-replicated T-tables ------------------------------------
// PRMT selector building (w.byte_k << 8) | lane*4: out b0 = lc.b0, b1 = w.bk,
// b2 = b3 = lc.b1 (= 0).
#define SP_SEL(k) (0x5504u | ((uint32_t)(k) << 4))

// The dynamic shared window of a non-cluster launch starts at shared address
// kSmBase (checked at kernel entry).  Lookups use absolute addresses so one
// PRMT + one LDS [reg+imm] is the whole lookup (no base add per access).
constexpr uint32_t kSmBase = 0x400;

__device__ __forceinline__ uint32_t lds32(uint32_t addr, uint32_t off_unused = 0) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

template <uint32_t OFF>
__device__ __forceinline__ uint32_t lds32_at(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(OFF + kSmBase));
    return v;
}

template <uint32_t OFF>
__device__ __forceinline__ uint4 lds128_at(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4+%5];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr), "n"(OFF + kSmBase));
    return v;
}

// ---- table policies -----------------------------------------------------------
// Big: the lane-replicated layout above (conflict-free LDS, one PRMT per
// lookup; 192 KB per CTA).  Small: one copy of each table (T0..T3 1 KB each,
// M_G 4 KB, R8 1 KB = 10 KB per CTA) for latency-bound launches: the fill is
// 19x smaller, lookups cost one more ALU op and some bank conflicts.
constexpr uint32_t kSmallT = 0;        // T0..T3: table t entry v at t*1024 + v*4
constexpr uint32_t kSmallMG = 4096;    // M_G[v] at 4096 + v*16
constexpr uint32_t kSmallR8 = 8192;    // R8[v]  at 8192 + v*4
constexpr uint32_t kSmallSmem = 9216;

template <int K>
__device__ __forceinline__ uint32_t byte_x4(uint32_t w) {  // byte K of w, times 4
    return K == 0 ? (w << 2) & 0x3fcu : (w >> (8 * K - 2)) & 0x3fcu;
}
template <int K>
__device__ __forceinline__ uint32_t byte_x16(uint32_t w) {  // byte K of w, times 16
    return K == 0 ? (w << 4) & 0xff0u : (w >> (8 * K - 4)) & 0xff0u;
}

struct BigTabs {
    static constexpr bool kSmall = false;
    template <int T, int K>
    static __device__ __forceinline__ uint32_t t(uint32_t w, uint32_t lc) {
        return lds32_at<(T < 2 ? kSmAes0 : kSmAes1) + (T & 1) * 128u>(__byte_perm(w, lc, SP_SEL(K)));
    }
    template <int K>
    static __device__ __forceinline__ uint4 mg(uint32_t w, uint32_t lcm) {
        return lds128_at<kSmGh>(__byte_perm(w, lcm, SP_SEL(K)));
    }
    static __device__ __forceinline__ uint32_t r8(uint32_t w, uint32_t lcr) {
        return lds32_at<kSmGh>(__byte_perm(w, lcr, SP_SEL(3)));
    }
};

struct SmallTabs {
    static constexpr bool kSmall = true;
    template <int T, int K>
    static __device__ __forceinline__ uint32_t t(uint32_t w, uint32_t) {
        return lds32_at<kSmallT + T * 1024u>(byte_x4<K>(w));
    }
    template <int K>
    static __device__ __forceinline__ uint4 mg(uint32_t w, uint32_t) {
        return lds128_at<kSmallMG>(byte_x16<K>(w));
    }
    static __device__ __forceinline__ uint32_t r8(uint32_t w, uint32_t) { return lds32_at<kSmallR8>(byte_x4<3>(w)); }
};

#define T0L(w, b) TB::template t<0, b>(w, lc)
#define T1L(w, b) TB::template t<1, b>(w, lc)
#define T2L(w, b) TB::template t<2, b>(w, lc)
#define T3L(w, b) TB::template t<3, b>(w, lc)

// Rounds r0..13 (full T-table rounds) on state s0..s3, then the final round.
template <class TB>
__device__ __forceinline__ uint4 aes256_from_round(int r0, const uint32_t *rk, uint32_t lc, uint32_t s0,
                                                   uint32_t s1, uint32_t s2, uint32_t s3) {
#pragma unroll
    for (int r = 1; r < 14; ++r) {
        if (r < r0) continue;
        const uint32_t t0 = T0L(s0, 0) ^ T1L(s1, 1) ^ T2L(s2, 2) ^ T3L(s3, 3) ^ rk[4 * r + 0];
        const uint32_t t1 = T0L(s1, 0) ^ T1L(s2, 1) ^ T2L(s3, 2) ^ T3L(s0, 3) ^ rk[4 * r + 1];
        const uint32_t t2 = T0L(s2, 0) ^ T1L(s3, 1) ^ T2L(s0, 2) ^ T3L(s1, 3) ^ rk[4 * r + 2];
        const uint32_t t3 = T0L(s3, 0) ^ T1L(s0, 1) ^ T2L(s1, 2) ^ T3L(s2, 3) ^ rk[4 * r + 3];
        s0 = t0; s1 = t1; s2 = t2; s3 = t3;
    }
    // Final round: S-box bytes come out of the T-tables: T2 has S at byte 0,
    // T3 at byte 1, T0 at byte 2, T1 at byte 3.
    uint4 o;
#define SP_LAST(ca, cb, cc, cd, k)                                                       \
    ((T2L(ca, 0) & 0x000000ffu) | (T3L(cb, 1) & 0x0000ff00u) | (T0L(cc, 2) & 0x00ff0000u) | \
     (T1L(cd, 3) & 0xff000000u)) ^ rk[56 + k]
    o.x = SP_LAST(s0, s1, s2, s3, 0);
    o.y = SP_LAST(s1, s2, s3, s0, 1);
    o.z = SP_LAST(s2, s3, s0, s1, 2);
    o.w = SP_LAST(s3, s0, s1, s2, 3);
#undef SP_LAST
    return o;
}

// s0..s3: counter block words already XORed with round key 0.
template <class TB>
__device__ __forceinline__ uint4 aes256_rounds(const uint32_t *rk, uint32_t lc, uint32_t s0, uint32_t s1,
                                               uint32_t s2, uint32_t s3) {
    return aes256_from_round<TB>(1, rk, lc, s0, s1, s2, s3);
}

// ---- counter-mode caching ----------------------------------------------------
// After round 0 only column 3 (the 32-bit counter) varies.  With counters
// < 2^24 (messages <= 32 MiB), round-1 column 3 is message-constant, columns
// 1-2 change only when ctr >> 8 changes, and round 2 has one varying input
// column.  Per block that is 5 lookups for rounds 1-2 instead of 32.
struct CtrConst {
    uint32_t c0, c1, c2, t3;  // round-1 partial columns (message constants)
};

struct CtrCache {
    uint32_t gid;             // ctr >> 8 the d-values belong to
    uint32_t d0, d1, d2, d3;  // round-2 partial columns (group constants)
};

template <class TB>
__device__ __forceinline__ CtrConst ctr_const(const uint32_t *rk, uint32_t lc, uint32_t x0, uint32_t x1,
                                              uint32_t x2) {
    CtrConst c;
    const uint32_t s3hi = rk[3];  // byte 0 of (bswap(ctr) ^ rk3) for ctr < 2^24
    c.c0 = T0L(x0, 0) ^ T1L(x1, 1) ^ T2L(x2, 2) ^ rk[4];
    c.c1 = T0L(x1, 0) ^ T1L(x2, 1) ^ T3L(x0, 3) ^ rk[5];
    c.c2 = T0L(x2, 0) ^ T2L(x0, 2) ^ T3L(x1, 3) ^ rk[6];
    c.t3 = T0L(s3hi, 0) ^ T1L(x0, 1) ^ T2L(x1, 2) ^ T3L(x2, 3) ^ rk[7];
    return c;
}

template <class TB>
__device__ __forceinline__ void ctr_refresh(CtrCache &k, const CtrConst &c, const uint32_t *rk, uint32_t lc,
                                            uint32_t s3, uint32_t gid) {
    const uint32_t t1 = c.c1 ^ T2L(s3, 2);
    const uint32_t t2 = c.c2 ^ T1L(s3, 1);
    const uint32_t t3 = c.t3;
    k.d0 = T1L(t1, 1) ^ T2L(t2, 2) ^ T3L(t3, 3) ^ rk[8];
    k.d1 = T0L(t1, 0) ^ T1L(t2, 1) ^ T2L(t3, 2) ^ rk[9];
    k.d2 = T0L(t2, 0) ^ T1L(t3, 1) ^ T3L(t1, 3) ^ rk[10];
    k.d3 = T0L(t3, 0) ^ T2L(t1, 2) ^ T3L(t2, 3) ^ rk[11];
    k.gid = gid;
}

template <class TB>
__device__ __forceinline__ uint4 aes256_ctr(const uint32_t *rk, uint32_t lc, const CtrConst &c, CtrCache &k,
                                            uint32_t ctr) {
    const uint32_t s3 = bswap32(ctr) ^ rk[3];
    const uint32_t gid = ctr >> 8;
    if (gid != k.gid) ctr_refresh<TB>(k, c, rk, lc, s3, gid);
    const uint32_t t0 = c.c0 ^ T3L(s3, 3);
    const uint32_t u0 = T0L(t0, 0) ^ k.d0;
    const uint32_t u1 = T3L(t0, 3) ^ k.d1;
    const uint32_t u2 = T2L(t0, 2) ^ k.d2;
    const uint32_t u3 = T1L(t0, 1) ^ k.d3;
    return aes256_from_round<TB>(3, rk, lc, u0, u1, u2, u3);
}

// ---- GHASH: Y * G with an 8-bit Shoup table in shared memory ----------------
// Element layout: little-endian 32-bit words of the 16-byte GCM string
// (byte 0 holds coefficients x^0..x^7, MSB first).  Multiplying by x^8 moves
// every byte one position up; byte 15 falls off and is folded back with R8.
// (Measured alternative, r1: computing R8 with IMAD/IMAD.HI shifts on the FMA
// pipe and moving the byte shifts there too removes 15 shared wavefronts per
// row but lengthens every Horner step's dependency chain; it ran at 422 GB/s
// vs 483 GB/s for the table version, so the table stays.)
template <class TB>
__device__ __forceinline__ uint4 gmul_g(uint4 y, uint32_t lcm, uint32_t lcr) {
    uint4 z = TB::template mg<3>(y.w, lcm);
#pragma unroll
    for (int b = 14; b >= 0; --b) {
        const uint32_t r = TB::r8(z.w, lcr);
        z.w = __funnelshift_l(z.z, z.w, 8);
        z.z = __funnelshift_l(z.y, z.z, 8);
        z.y = __funnelshift_l(z.x, z.y, 8);
        z.x = z.x << 8;
        uint4 m;
        switch (b & 3) {
            case 0: m = TB::template mg<0>(word_of(y, b >> 2), lcm); break;
            case 1: m = TB::template mg<1>(word_of(y, b >> 2), lcm); break;
            case 2: m = TB::template mg<2>(word_of(y, b >> 2), lcm); break;
            default: m = TB::template mg<3>(word_of(y, b >> 2), lcm); break;
        }
        z.x ^= r ^ m.x;
        z.y ^= m.y;
        z.z ^= m.z;
        z.w ^= m.w;
    }
    return z;
}

// ---- nibble-table multiplies (HBM/L2 resident tables) ----------------------
__device__ __forceinline__ uint32_t nibble_of(const uint4 &v, int q) {
    const uint32_t byte = (word_of(v, q >> 3) >> (8 * ((q >> 1) & 3))) & 0xffu;
    return (q & 1) ? (byte & 15u) : (byte >> 4);
}

// Full multiply by the table's element, done by one lane (32 lookups).
__device__ __forceinline__ uint4 nt_mul_lane(const uint4 *tab, uint4 v) {
    uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int q = 0; q < 32; ++q) acc = xor4(acc, __ldg(tab + q * 16 + nibble_of(v, q)));
    return acc;
}

// v x H^(2^K) with the shared-memory nibble table K of the tree: 32
// independent LDS.128, no global traffic.
template <int K>
__device__ __forceinline__ uint4 tree_mul(uint4 v) {
    uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int q = 0; q < 32; ++q) {
        const uint32_t w = word_of(v, q >> 3);
        const int sh = 8 * ((q >> 1) & 3) - ((q & 1) ? 4 : 0);  // nibble q of the string, times 16
        const uint32_t off = (sh >= 0 ? (w >> sh) : (w << (-sh))) & 0xf0u;
        acc = xor4(acc, lds128_at<kSmTree + (uint32_t)K * 8192u>(off + (uint32_t)q * 256u));
    }
    return acc;
}

__device__ __forceinline__ uint4 warp_xor(uint4 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x ^= __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y ^= __shfl_xor_sync(0xffffffffu, v.y, o);
        v.z ^= __shfl_xor_sync(0xffffffffu, v.z, o);
        v.w ^= __shfl_xor_sync(0xffffffffu, v.w, o);
    }
    return v;
}

// Lane-parallel partial product: lane q looks up nibble q (v warp-uniform).
__device__ __forceinline__ uint4 nt_part(const uint4 *tab, uint4 v, int lane) {
    return __ldg(tab + lane * 16 + nibble_of(v, lane));
}

// ---- block load / store ------------------------------------------------------
__device__ __forceinline__ uint4 load_bytes(const uint8_t *p, int n) {
    uint32_t w[4] = {0, 0, 0, 0};
    for (int k = 0; k < n; ++k) w[k >> 2] |= (uint32_t)p[k] << (8 * (k & 3));
    return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ void store_bytes(uint8_t *p, uint4 v, int n) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    for (int k = 0; k < n; ++k) p[k] = (uint8_t)(w[k >> 2] >> (8 * (k & 3)));
}

__device__ __forceinline__ uint4 mask_bytes(uint4 v, int n) {
    // keep bytes [0, n), zero the rest (n in 1..15)
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int keep = n - 4 * k;
        w[k] = keep >= 4 ? w[k] : (keep <= 0 ? 0u : (w[k] & ((1u << (8 * keep)) - 1u)));
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

}  // namespace spgcm
