// libspgcm: AES-256-GCM seal/open for B200 (sm_100a) behind the C-ABI of
// include/spgcm.h.  See DESIGN.md §3 for the layout and the roofline.
//
// Reference seam replaced: specpipe.channel.encrypt_at / decrypt_at
// (/root/reference/pkg/src/specpipe/channel.py:85-115).

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "spgcm.h"
#include "spgcm_kernels.cuh"

using namespace spgcm;

// =============================================================================
// Device: the batched seal/open kernel
// =============================================================================

template <class P>
__device__ __forceinline__ void fill_tables(uint8_t *sm, const P &p) {
    // 8192 AES stores + 4096 GHASH stores of 16 B = 24 per thread.  All global
    // loads are issued before any store so their latencies overlap (the tables
    // are usually evicted from L2 by the payload stream: one DRAM round trip
    // per CTA instead of 24 dependent ones).
    static_assert((2u * 256u * 2u * 8u) % kThreads == 0 && (256u * 16u) % kThreads == 0, "fill split");
    constexpr int kA = (2 * 256 * 2 * 8) / kThreads, kG = (256 * 16) / kThreads;
    uint32_t aval[kA];
    uint4 gval[kG];
#pragma unroll
    for (int j = 0; j < kA; ++j) {
        const uint32_t f = threadIdx.x + (uint32_t)j * kThreads;
        const uint32_t t = (f >> 3) & 1u, v = (f >> 4) & 255u, pr = f >> 12;
        aval[j] = __ldg(p.ttab + (2u * pr + t) * 256u + v);
    }
#pragma unroll
    for (int j = 0; j < kG; ++j) {
        const uint32_t f = threadIdx.x + (uint32_t)j * kThreads;
        const uint32_t sidx = f & 15u, v = f >> 4;
        if (sidx < 8u) {
            gval[j] = __ldg(p.mg + v);
        } else {
            const uint32_t r = __ldg(p.ttab + 4u * 256u + v);
            gval[j] = make_uint4(r, r, r, r);
        }
    }
#pragma unroll
    for (int j = 0; j < kA; ++j) {
        const uint32_t f = threadIdx.x + (uint32_t)j * kThreads;
        const uint32_t c4 = f & 7u, t = (f >> 3) & 1u, v = (f >> 4) & 255u, pr = f >> 12;
        *reinterpret_cast<uint4 *>(sm + pr * 65536u + v * 256u + t * 128u + c4 * 16u) =
            make_uint4(aval[j], aval[j], aval[j], aval[j]);
    }
#pragma unroll
    for (int j = 0; j < kG; ++j) {
        const uint32_t f = threadIdx.x + (uint32_t)j * kThreads;
        *reinterpret_cast<uint4 *>(sm + kSmGh + (f >> 4) * 256u + (f & 15u) * 16u) = gval[j];
    }
}

// Compact tables for latency-bound launches (SmallTabs layout): 10 KB.
template <class P>
__device__ __forceinline__ void fill_tables_small(uint8_t *sm, const P &p) {
    // T0..T3 (4 x 256 words) + R8 (256 words) = 1280 words; M_G = 256 x 16 B
    for (uint32_t f = threadIdx.x; f < 1280u; f += blockDim.x) {
        const uint32_t v = __ldg(p.ttab + f);  // ttab = T0..T3 then R8, contiguous
        if (f < 1024u) *reinterpret_cast<uint32_t *>(sm + kSmallT + f * 4u) = v;
        else *reinterpret_cast<uint32_t *>(sm + kSmallR8 + (f - 1024u) * 4u) = v;
    }
    for (uint32_t f = threadIdx.x; f < 256u; f += blockDim.x)
        *reinterpret_cast<uint4 *>(sm + kSmallMG + f * 16u) = __ldg(p.mg + f);
}

__device__ __forceinline__ uint32_t atom_add_acq_rel_gpu(uint32_t *p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ uint4 len_block(uint64_t len) {
    const uint64_t bits = len * 8u;
    return make_uint4(0u, 0u, bswap32((uint32_t)(bits >> 32)), bswap32((uint32_t)bits));
}

// Tag finalisation for one message; T = GHASH xor E_K(J0) (the warp that
// covered the message's first row folded E_K(J0) in).  Warp-uniform.
template <bool COH>
__device__ __forceinline__ uint4 load_tag(const uint8_t *t) {
    if ((reinterpret_cast<uintptr_t>(t) & 15u) != 0) return load_bytes(t, 16);
    return COH ? __ldcg(reinterpret_cast<const uint4 *>(t)) : __ldg(reinterpret_cast<const uint4 *>(t));
}

// want: the expected tag, already loaded by lane 0 (have_want) or loaded here.
__device__ __forceinline__ void finish_message(const MsgDev &md, uint4 tag, int lane, uint4 want, bool have_want) {
    if (!(md.dir & kOpenBit)) {
        if (lane == 0) {
            if ((reinterpret_cast<uintptr_t>(md.tag) & 15u) == 0)
                *reinterpret_cast<uint4 *>(md.tag) = tag;
            else
                store_bytes(md.tag, tag, 16);
        }
        return;
    }
    uint32_t bad = 0;
    if (lane == 0) {
        if (!have_want) want = load_tag<true>(md.tag);  // after the message's rows: coherent
        bad = (want.x ^ tag.x) | (want.y ^ tag.y) | (want.z ^ tag.z) | (want.w ^ tag.w);
        if (md.status && (bad || !(md.dir & kStickyBit))) *md.status = bad ? 1 : 0;
    }
    bad = __shfl_sync(0xffffffffu, bad, 0);
    if (bad) {
        // unverified plaintext never leaves: zero the whole output, 16 B per
        // lane store where aligned
        uint64_t k = 0;
        const uint64_t head = (16u - (reinterpret_cast<uintptr_t>(md.dst) & 15u)) & 15u;
        for (uint64_t j = (uint64_t)lane; j < min(head, md.len); j += 32) md.dst[j] = 0;
        k = min(head, md.len);
        const uint64_t nvec = (md.len - k) >> 4;
        uint4 *v = reinterpret_cast<uint4 *>(md.dst + k);
        for (uint64_t j = (uint64_t)lane; j < nvec; j += 32) v[j] = make_uint4(0, 0, 0, 0);
        for (uint64_t j = k + (nvec << 4) + (uint64_t)lane; j < md.len; j += 32) md.dst[j] = 0;
    }
}

// Unit [k, k+1) of `n` equal shares of `total` rows starting at `base`.
__device__ __forceinline__ void share_of(uint64_t base, uint64_t total, uint64_t k, uint64_t n, uint64_t &g,
                                         uint64_t &g_end) {
    if (total * n <= 0xffffffffull) {  // 32-bit division (the common case; 64-bit is a long software routine)
        const uint32_t t32 = (uint32_t)total, k32 = (uint32_t)k, n32 = (uint32_t)n;
        g = base + (t32 * k32) / n32;
        g_end = base + (t32 * (k32 + 1u)) / n32;
    } else {
        g = base + (total * k) / n;
        g_end = base + (total * (k + 1)) / n;
    }
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Rows [g, g_end) of the flattened batch: keystream + XOR, GHASH, and the
// tags of the messages whose last row this range completes.  COH: the
// range may read what an earlier level of the same launch wrote, so no
// read goes through the non-coherent (read-only) path.
template <uint32_t INL, class TB, bool COH>
__device__ __forceinline__ void gcm_rows(const KParamsT<INL> &p, uint64_t g, const uint64_t g_end, const int lane,
                                         const uint32_t lct, const uint32_t lcm, const uint32_t lcr) {
    const MsgDev *msgs = p.nmsgs <= INL ? p.inl : p.msgs;
    // first message containing row g (binary search on row_begin)
    uint32_t lo = 0, hi = p.nmsgs - 1;
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (msgs[mid].row_begin <= g) lo = mid; else hi = mid - 1;
    }
    uint32_t m = lo;

    while (g < g_end) {
        const MsgDev md = msgs[m];
        const uint64_t t_a = g - md.row_begin;
        const uint64_t t_b = min((uint64_t)md.rows, g_end - md.row_begin);
        const int64_t nblk = (int64_t)((md.len + 15u) >> 4);
        const int tail = (int)(md.len & 15u);
        const bool vec = ((reinterpret_cast<uintptr_t>(md.src) | reinterpret_cast<uintptr_t>(md.dst)) & 15u) == 0;
        const uint32_t x0 = bswap32(md.dir & 0xffu) ^ p.rk[0];
        const bool opening = (md.dir & kOpenBit) != 0;
        const uint32_t x1 = bswap32((uint32_t)(md.iv >> 32)) ^ p.rk[1];
        const uint32_t x2 = bswap32((uint32_t)md.iv) ^ p.rk[2];
        const int64_t base_i = nblk - 32 * (int64_t)md.rows + lane;  // block of this lane in local row 0

        auto load_row = [&](uint64_t t) -> uint4 {
            const int64_t i = base_i + 32 * (int64_t)t;
            if (i < 0) return make_uint4(0, 0, 0, 0);
            const int nb = (i == nblk - 1 && tail) ? tail : 16;
            const uint8_t *ptr = md.src + 16 * i;
            if (vec && nb == 16)
                return COH ? __ldcg(reinterpret_cast<const uint4 *>(ptr)) : __ldcs(reinterpret_cast<const uint4 *>(ptr));
            return load_bytes(ptr, nb);
        };

        // Prefetch into L2 the F / H^(32b) rows this lane's epilogue reads
        // (2 lines each; cold in HBM otherwise): overlaps two of the
        // epilogue's dependent DRAM round trips with the row loop.  A run
        // that ends at its message's end (r_end = 0) needs neither.
        const uint32_t r_end = md.rows - (uint32_t)t_b;
        const bool tree = !TB::kSmall && (p.reserved & kTreeBit);
        const bool short_tail = r_end < kNumG;
        if (r_end && short_tail) {
            const char *ga = reinterpret_cast<const char *>(p.nt + (size_t)((tree ? kNtG2 : kNtG1) + r_end) * kNtEntries + lane * 16);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ga));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ga + 128));
            if (tree) {
                const char *gb = reinterpret_cast<const char *>(p.nt + (size_t)(kNtG18 + r_end) * kNtEntries + lane * 16);
                asm volatile("prefetch.global.L2 [%0];" ::"l"(gb));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(gb + 128));
            }
        } else if (r_end) {
            const char *ft = reinterpret_cast<const char *>(p.nt + (size_t)(kNtF + (r_end >> 4)) * kNtEntries + lane * 16);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ft));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ft + 128));
            if (r_end & 15u) {
                const char *pt = reinterpret_cast<const char *>(
                    p.nt + (size_t)(kNtP32 + (r_end & 15u) - 1u) * kNtEntries + lane * 16);
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pt));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pt + 128));
            }
        }
        // the expected tag of an open whose last row this run covers: read
        // now, not after the epilogue
        const bool have_want = opening && t_b == md.rows && lane == 0;
        const uint4 want = have_want ? load_tag<COH>(md.tag) : make_uint4(0, 0, 0, 0);
        const uint4 lh_part = nt_part(p.nt + (size_t)kNtLane * kNtEntries, len_block(md.len), lane);  // L x H
        const CtrConst cc = ctr_const<TB>(p.rk, lct, x0, x1, x2);
        CtrCache ck;
        ck.gid = 0xffffffffu;
        ck.d0 = ck.d1 = ck.d2 = ck.d3 = 0;
        uint4 y = make_uint4(0, 0, 0, 0);
        uint4 cur = load_row(t_a);
        for (uint64_t t = t_a; t < t_b; ++t) {
            const uint4 nxt = (t + 1 < t_b) ? load_row(t + 1) : make_uint4(0, 0, 0, 0);
            const int64_t i = base_i + 32 * (int64_t)t;
            const uint32_t ctr = (uint32_t)(i + 2);
            const uint4 ks = aes256_ctr<TB>(p.rk, lct, cc, ck, ctr);
            uint4 out = xor4(cur, ks);
            uint4 gin = cur;
            if (i >= 0) {
                const int nb = (i == nblk - 1 && tail) ? tail : 16;
                if (nb != 16) out = mask_bytes(out, nb);
                uint8_t *dptr = md.dst + 16 * i;
                if (vec && nb == 16) __stcs(reinterpret_cast<uint4 *>(dptr), out);
                else store_bytes(dptr, out, nb);
                if (!opening) gin = out;
            } else {
                gin = make_uint4(0, 0, 0, 0);
            }
            y = (t == t_a) ? gin : xor4(gmul_g<TB>(y, lcm, lcr), gin);
            cur = nxt;
        }

        // combine lanes: W = sum_l Y_l * H^(32 - l), then x H^(32 r_end + 1).
        // A run that ends at its message's end (r_end = 0) walks the tables
        // of H^(33 - l) and is done (one dependent round trip fewer).  The
        // lane-table loads are in flight while the warp covering the
        // message's first row computes E_K(J0) (folded into W: XOR is
        // order-free, so the finisher needs no AES of its own).
        uint4 lanes_w;
        bool scaled = r_end == 0;  // W already carries H^(32 r_end + 1)
        if (tree) {
            // binary tree over lanes in shared memory: level k folds pairs
            // 2^k apart as left x H^(2^k) + right, so lane 0 ends with
            // D0 = sum_{l<16} Y_l H^(15-l) and lane 16 with D1 (lanes 16..31);
            // then W = D0 H^(17|18) + D1 H^(1|2), lane-parallel (two HBM
            // nibble loads per lane): 128 global loads per warp instead of
            // 1,024 (the L2 request rate bounded launches of many warps).
            uint4 v = y;
#define SP_TREE_LEVEL(K)                                                         \
    {                                                                            \
        uint4 r;                                                                 \
        r.x = __shfl_down_sync(0xffffffffu, v.x, 1 << K);                        \
        r.y = __shfl_down_sync(0xffffffffu, v.y, 1 << K);                        \
        r.z = __shfl_down_sync(0xffffffffu, v.z, 1 << K);                        \
        r.w = __shfl_down_sync(0xffffffffu, v.w, 1 << K);                        \
        if ((lane & ((2 << K) - 1)) == 0) v = xor4(tree_mul<K>(v), r);           \
    }
            SP_TREE_LEVEL(0)
            SP_TREE_LEVEL(1)
            SP_TREE_LEVEL(2)
            SP_TREE_LEVEL(3)
#undef SP_TREE_LEVEL
            uint4 d0, d1;
            d0.x = __shfl_sync(0xffffffffu, v.x, 0);
            d0.y = __shfl_sync(0xffffffffu, v.y, 0);
            d0.z = __shfl_sync(0xffffffffu, v.z, 0);
            d0.w = __shfl_sync(0xffffffffu, v.w, 0);
            d1.x = __shfl_sync(0xffffffffu, v.x, 16);
            d1.y = __shfl_sync(0xffffffffu, v.y, 16);
            d1.z = __shfl_sync(0xffffffffu, v.z, 16);
            d1.w = __shfl_sync(0xffffffffu, v.w, 16);
            uint32_t t0, t1;  // tables scaling D0 and D1
            if (r_end == 0) {
                t0 = kNtLane + 17u;  // H^18
                t1 = kNtLane + 1u;   // H^2
            } else if (short_tail) {
                t0 = kNtG18 + r_end;  // H^(32 r_end + 18)
                t1 = kNtG2 + r_end;   // H^(32 r_end + 2)
                scaled = true;
            } else {
                t0 = kNtLane + 16u;  // H^17
                t1 = kNtLane;        // H^1
            }
            lanes_w = xor4(nt_part(p.nt + (size_t)t0 * kNtEntries, d0, lane),
                           nt_part(p.nt + (size_t)t1 * kNtEntries, d1, lane));
        } else {
            lanes_w = nt_mul_lane(p.nt + (size_t)(kNtLane + (r_end ? 31u : 32u) - (uint32_t)lane) * kNtEntries, y);
        }
        uint4 ek = make_uint4(0, 0, 0, 0);
        if (t_a == 0 && lane == 0) ek = aes256_rounds<TB>(p.rk, lct, x0, x1, x2, bswap32(1u) ^ p.rk[3]);
        uint4 w = warp_xor(lanes_w);
        if (!scaled) {  // scale by H^(32 r_end + 1)
            if (short_tail) {
                w = warp_xor(nt_part(p.nt + (size_t)(kNtG1 + r_end) * kNtEntries, w, lane));
            } else {  // = F[r_end / 16] x H^(32 (r_end mod 16))
                w = warp_xor(nt_part(p.nt + (size_t)(kNtF + (r_end >> 4)) * kNtEntries, w, lane));
                if (r_end & 15u)
                    w = warp_xor(nt_part(p.nt + (size_t)(kNtP32 + (r_end & 15u) - 1u) * kNtEntries, w, lane));
            }
        }
        if (t_a == 0) {
            ek.x = __shfl_sync(0xffffffffu, ek.x, 0);
            ek.y = __shfl_sync(0xffffffffu, ek.y, 0);
            ek.z = __shfl_sync(0xffffffffu, ek.z, 0);
            ek.w = __shfl_sync(0xffffffffu, ek.w, 0);
            w = xor4(w, ek);
        }

        if (t_a == 0 && t_b == md.rows) {
            finish_message(md, xor4(w, warp_xor(lh_part)), lane, want, have_want);
        } else {
            uint32_t *acc = p.acc + (size_t)m * 8u;
            // XOR-accumulate (order-free, so deterministic) and count rows:
            // the count is a release/acquire RMW, no full fence.
            if (lane < 4) atomicXor(acc + lane, word_of(w, lane));
            __syncwarp();
            uint32_t old = 0;
            if (lane == 0) old = atom_add_acq_rel_gpu(acc + 4, (uint32_t)(t_b - t_a));
            old = __shfl_sync(0xffffffffu, old, 0);
            if (old + (uint32_t)(t_b - t_a) == md.rows) {
                __syncwarp();
                uint32_t v = 0;
                if (lane < 4) v = atomicExch(acc + lane, 0u);
                if (lane == 0) atomicExch(acc + 4, 0u);
                uint4 a;
                a.x = __shfl_sync(0xffffffffu, v, 0);
                a.y = __shfl_sync(0xffffffffu, v, 1);
                a.z = __shfl_sync(0xffffffffu, v, 2);
                a.w = __shfl_sync(0xffffffffu, v, 3);
                finish_message(md, xor4(a, warp_xor(lh_part)), lane, want, have_want);
            }
        }
        g = md.row_begin + t_b;
        ++m;
    }
}

template <uint32_t INL, class TB, bool LV>
__global__ void __launch_bounds__(TB::kSmall ? kThreadsSmall : kThreads, TB::kSmall ? 4 : 1)
    k_gcm(const __grid_constant__ KParamsT<INL> p) {
    extern __shared__ __align__(16) uint8_t sm[];
    if (static_cast<uint32_t>(__cvta_generic_to_shared(sm)) != kSmBase) __trap();  // absolute lookups
    // let a dependent launch on this stream be scheduled now: its CTAs take
    // idle SMs and fill their tables while this grid runs (they read no data
    // before their own griddepcontrol.wait, which waits for this grid to end)
    asm volatile("griddepcontrol.launch_dependents;");
    if (TB::kSmall) fill_tables_small(sm, p);
    else fill_tables(sm, p);  // per-key constants only: may overlap the previous launch (PDL)
    if (!TB::kSmall && (p.reserved & kTreeBit)) {
        // tree tables: H^(2^k) = HBM nibble table kNtLane + 2^k - 1, k = 0..3
        uint4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t f = threadIdx.x + (uint32_t)j * kThreads, k = f >> 9;
            v[j] = __ldg(p.nt + (size_t)(kNtLane + (1u << k) - 1u) * kNtEntries + (f & 511u));
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            reinterpret_cast<uint4 *>(sm + kSmTree)[threadIdx.x + (uint32_t)j * kThreads] = v[j];
    }
    __syncthreads();
    // programmatic dependent launch: everything below may read what the
    // previous kernel on this stream wrote (messages, accumulators)
    asm volatile("griddepcontrol.wait;" ::: "memory");

    const int lane = threadIdx.x & 31;
    const uint32_t lct = (uint32_t)lane * 4u;                  // T tables
    const uint32_t lcm = (uint32_t)(lane & 7) * 16u;           // M_G copies
    const uint32_t lcr = 128u + (uint32_t)lane * 4u;           // R8 copies

    const uint32_t warp = threadIdx.x >> 5;
    if (warp >= p.warps_used) return;
    if (!LV) {
        // contiguous, balanced row range for this warp
        uint64_t g, g_end;
        share_of(p.row_begin, p.row_end - p.row_begin, (uint64_t)blockIdx.x * p.warps_used + warp,
                 (uint64_t)gridDim.x * p.warps_used, g, g_end);
        if (g < g_end) gcm_rows<INL, TB, false>(p, g, g_end, lane, lct, lcm, lcr);
        return;
    }

    // fused levels: claim units in order (see KParamsT)
    uint32_t *ctl = p.ctl;
    const uint32_t units = p.lvl_unit[p.nlevels];
    for (;;) {
        uint32_t u = 0;
        if (lane == 0) u = atomicAdd(ctl, 1u);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= units) break;
        uint32_t lv = 0;
        while (u >= p.lvl_unit[lv + 1]) ++lv;
        if (lv > 0) {
            if (lane == 0) {
                const uint32_t need = p.lvl_unit[lv] - p.lvl_unit[lv - 1];
                uint32_t ns = 32, spins = 0;
                while (ld_acquire_gpu(ctl + 2 + lv - 1) < need) {
                    __nanosleep(ns);
                    ns = ns < 512 ? ns * 2 : ns;
                    if (++spins > (1u << 22)) __trap();  // a lost level (bug): fail loudly, never hang
                }
            }
            __syncwarp();
        }
        const uint32_t k = u - p.lvl_unit[lv], n = p.lvl_unit[lv + 1] - p.lvl_unit[lv];
        uint64_t g, g_end;
        share_of(p.lvl_row[lv], p.lvl_row[lv + 1] - p.lvl_row[lv], k, n, g, g_end);
        if (g < g_end) gcm_rows<INL, TB, true>(p, g, g_end, lane, lct, lcm, lcr);
        __threadfence();
        __syncwarp();
        if (lane == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctl + 2 + lv) : "memory");
    }
    if (lane == 0) {
        const uint32_t e = atomicAdd(ctl + 1, 1u);
        if (e == gridDim.x * p.warps_used - 1u) {  // every warp is past its last claim
            ctl[0] = 0;
            ctl[1] = 0;
            for (uint32_t l = 0; l < p.nlevels; ++l) ctl[2 + l] = 0;
        }
    }
}

// =============================================================================
// Device: context setup (H, powers of H, tables) — runs once per key
// =============================================================================

struct G128 {
    uint64_t hi, lo;  // big-endian halves of the 16-byte GCM string
};

__host__ __device__ inline G128 g_mulx(G128 v) {
    const uint64_t lsb = v.lo & 1u;
    v.lo = (v.lo >> 1) | (v.hi << 63);
    v.hi >>= 1;
    if (lsb) v.hi ^= 0xe100000000000000ull;
    return v;
}

__host__ __device__ inline G128 g_mul(G128 x, G128 y) {
    G128 z = {0, 0};
    G128 v = y;
    for (int i = 0; i < 128; ++i) {
        const uint64_t bit = i < 64 ? (x.hi >> (63 - i)) & 1u : (x.lo >> (127 - i)) & 1u;
        if (bit) { z.hi ^= v.hi; z.lo ^= v.lo; }
        v = g_mulx(v);
    }
    return z;
}

__host__ __device__ inline uint32_t bs32(uint32_t x) {
    return (x >> 24) | ((x >> 8) & 0xff00u) | ((x << 8) & 0xff0000u) | (x << 24);
}

__host__ __device__ inline uint4 g_to_words(G128 v) {
    return make_uint4(bs32((uint32_t)(v.hi >> 32)), bs32((uint32_t)v.hi), bs32((uint32_t)(v.lo >> 32)),
                      bs32((uint32_t)v.lo));
}

__host__ __device__ inline G128 g_from_words(uint4 w) {
    G128 v;
    v.hi = ((uint64_t)bs32(w.x) << 32) | bs32(w.y);
    v.lo = ((uint64_t)bs32(w.z) << 32) | bs32(w.w);
    return v;
}

__host__ __device__ inline G128 g_pow(G128 h, uint64_t e) {
    G128 r = {0x8000000000000000ull, 0};  // 1 = x^0
    G128 b = h;
    while (e) {
        if (e & 1u) r = g_mul(r, b);
        b = g_mul(b, b);
        e >>= 1;
    }
    return r;
}

// H = E_K(0^128): plain byte-wise AES in one thread.
__global__ void k_setup_h(KParams p, const uint8_t *sbox, uint4 *out_h) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint8_t s[16];
    const uint8_t *rk = reinterpret_cast<const uint8_t *>(p.rk);
    for (int i = 0; i < 16; ++i) s[i] = rk[i];
    auto xt = [](uint8_t a) -> uint8_t { return (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1b : 0)); };
    for (int r = 1; r <= 14; ++r) {
        uint8_t t[16];
        for (int c = 0; c < 4; ++c)
            for (int q = 0; q < 4; ++q) t[q + 4 * c] = sbox[s[q + 4 * ((c + q) & 3)]];
        if (r != 14) {
            for (int c = 0; c < 4; ++c) {
                const uint8_t a0 = t[4 * c], a1 = t[4 * c + 1], a2 = t[4 * c + 2], a3 = t[4 * c + 3];
                s[4 * c + 0] = xt(a0) ^ (xt(a1) ^ a1) ^ a2 ^ a3;
                s[4 * c + 1] = a0 ^ xt(a1) ^ (xt(a2) ^ a2) ^ a3;
                s[4 * c + 2] = a0 ^ a1 ^ xt(a2) ^ (xt(a3) ^ a3);
                s[4 * c + 3] = (xt(a0) ^ a0) ^ a1 ^ a2 ^ xt(a3);
            }
        } else {
            for (int i = 0; i < 16; ++i) s[i] = t[i];
        }
        for (int i = 0; i < 16; ++i) s[i] ^= rk[16 * r + i];
    }
    uint32_t w[4];
    for (int k = 0; k < 4; ++k)
        w[k] = (uint32_t)s[4 * k] | ((uint32_t)s[4 * k + 1] << 8) | ((uint32_t)s[4 * k + 2] << 16) |
               ((uint32_t)s[4 * k + 3] << 24);
    *out_h = make_uint4(w[0], w[1], w[2], w[3]);
}

// powers[idx] for every nibble table, plus G = H^32 at powers[kNumNt]
__global__ void k_setup_powers(const uint4 *hptr, uint4 *powers) {
    const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx > kNumNt) return;
    const G128 h = g_from_words(*hptr);
    uint64_t e;
    if (idx < kNtF) e = idx + 1;                                   // H^1..H^33
    else if (idx < kNtP32) e = 512ull * (idx - kNtF) + 1;          // F_a
    else if (idx < kNtG1) e = 32ull * (idx - kNtP32 + 1);          // H^(32b)
    else if (idx < kNtG2) e = 32ull * (idx - kNtG1) + 1;           // short tails
    else if (idx < kNtG18) e = 32ull * (idx - kNtG2) + 2;
    else if (idx < kNumNt) e = 32ull * (idx - kNtG18) + 18;
    else e = 32;                                                    // G
    powers[idx] = g_to_words(g_pow(h, e));
}

// nibble tables: nt[t][q][v] = (nibble v at position q) * powers[t]
__global__ void k_setup_nt(const uint4 *powers, uint4 *nt) {
    const uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (uint64_t)kNumNt * kNtEntries) return;
    const uint32_t t = (uint32_t)(idx / kNtEntries), q = (uint32_t)(idx % kNtEntries) / 16u, v = (uint32_t)idx & 15u;
    // element with nibble v at nibble position q (MSB of the nibble = lowest degree)
    const uint32_t shift_in_string = 124u - 4u * q;  // bit position from the right in a 128-bit BE int
    G128 x = {0, 0};
    if (shift_in_string >= 64) x.hi = (uint64_t)v << (shift_in_string - 64);
    else x.lo = (uint64_t)v << shift_in_string;
    nt[idx] = g_to_words(g_mul(x, g_from_words(powers[t])));
}

// M_G[v] = (byte v at position 0) * G
__global__ void k_setup_mg(const uint4 *powers, uint4 *mg) {
    const uint32_t v = threadIdx.x;
    G128 x = {(uint64_t)v << 56, 0};
    mg[v] = g_to_words(g_mul(x, g_from_words(powers[kNumNt])));
}

// =============================================================================
// Host
// =============================================================================

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char *where) {
    return fail(e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver || e == cudaErrorNoKernelImageForDevice
                    ? SP_ENODEV
                    : SP_ECUDA,
                std::string(where) + ": " + cudaGetErrorString(e));
}

#define SP_CUDA(call, where)                          \
    do {                                              \
        cudaError_t e_ = (call);                      \
        if (e_ != cudaSuccess) return cuda_fail(e_, where); \
    } while (0)

// FIPS-197 constants derived, not tabulated: S-box from GF(2^8) inverse + affine.
struct Consts {
    uint8_t sbox[256];
    uint32_t t[4][256];
    uint32_t r8[256];
    Consts() {
        auto mul = [](uint8_t a, uint8_t b) {
            uint8_t r = 0;
            for (int i = 0; i < 8; ++i) {
                if (b & 1) r ^= a;
                const uint8_t h = a & 0x80;
                a <<= 1;
                if (h) a ^= 0x1b;
                b >>= 1;
            }
            return r;
        };
        for (int x = 0; x < 256; ++x) {
            uint8_t inv = 0;
            for (int y = 1; x && y < 256; ++y)
                if (mul((uint8_t)x, (uint8_t)y) == 1) { inv = (uint8_t)y; break; }
            uint8_t s = inv, r = inv;
            for (int k = 0; k < 4; ++k) { r = (uint8_t)((r << 1) | (r >> 7)); s ^= r; }
            sbox[x] = s ^ 0x63;
        }
        for (int x = 0; x < 256; ++x) {
            const uint32_t s = sbox[x], s2 = mul(sbox[x], 2), s3 = mul(sbox[x], 3);
            t[0][x] = s2 | (s << 8) | (s << 16) | (s3 << 24);
            t[1][x] = s3 | (s2 << 8) | (s << 16) | (s << 24);
            t[2][x] = s | (s3 << 8) | (s2 << 16) | (s << 24);
            t[3][x] = s | (s << 8) | (s3 << 16) | (s2 << 24);
        }
        for (int v = 0; v < 256; ++v) {
            // byte 15 = v, multiplied by x^8: result lives in bytes 0,1
            G128 e = {0, (uint64_t)v};
            for (int k = 0; k < 8; ++k) e = g_mulx(e);
            const uint4 w = g_to_words(e);
            r8[v] = w.x;
        }
    }
};

const Consts &consts() {
    static Consts c;
    return c;
}

void key_expand(const uint8_t key[32], uint32_t rk[60]) {
    const Consts &c = consts();
    uint8_t w[240];
    memcpy(w, key, 32);
    uint8_t rcon = 1;
    for (int i = 8; i < 60; ++i) {
        uint8_t t[4];
        memcpy(t, w + 4 * (i - 1), 4);
        if (i % 8 == 0) {
            const uint8_t t0 = t[0];
            t[0] = c.sbox[t[1]] ^ rcon;
            t[1] = c.sbox[t[2]];
            t[2] = c.sbox[t[3]];
            t[3] = c.sbox[t0];
            rcon = (uint8_t)((rcon << 1) ^ ((rcon & 0x80) ? 0x1b : 0));
        } else if (i % 8 == 4) {
            for (int k = 0; k < 4; ++k) t[k] = c.sbox[t[k]];
        }
        for (int k = 0; k < 4; ++k) w[4 * i + k] = w[4 * (i - 8) + k] ^ t[k];
    }
    memcpy(rk, w, 240);  // little-endian words == AES state column words
}

// Pinned descriptor-staging slots per stream: a slot is reused only after the
// copy that read it completed, so the host can run this many large batches
// ahead of the device before it blocks.
constexpr int kPinSlots = 32;

struct Workspace {
    std::mutex mu;  // calls on one stream from several host threads serialise here
    MsgDev *d_msgs = nullptr;
    size_t cap_msgs = 0;
    uint32_t *d_acc = nullptr;
    size_t cap_acc = 0;
    uint32_t *d_ctl = nullptr;  // fused-level launches: claim / exit / per-level done counters
    std::vector<MsgDev> h_msgs;
    // pinned staging ring for descriptor arrays larger than kInline
    MsgDev *h_pin[kPinSlots] = {};
    cudaEvent_t ev_pin[kPinSlots] = {};
    bool ev_live[kPinSlots] = {};
    size_t cap_pin = 0;
    int slot = 0;
};

std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, Workspace *> g_ws;

}  // namespace

struct sp_ctx {
    int device = 0;
    int num_sms = 148;
    std::atomic<int> max_sms{0};  // SM budget (0: all); sp_ctx_set_max_sms
    std::atomic<int> small_sms{0};  // SM cap of small launches (0: none); sp_ctx_set_small_sms
    int sms() const {
        const int m = max_sms.load(std::memory_order_relaxed);
        return m > 0 && m < num_sms ? m : num_sms;
    }
    uint32_t rk[60];
    uint32_t *d_ttab = nullptr;  // T[4][256] + R8[256]
    uint4 *d_mg = nullptr;
    uint4 *d_nt = nullptr;
    uint4 *d_pow = nullptr;      // kNumNt + 1 powers
    uint8_t *d_sbox = nullptr;
    uint4 *d_h = nullptr;
};

namespace {

Workspace *workspace_for(int device, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    auto &w = g_ws[{device, s}];
    if (!w) w = new Workspace();
    return w;
}

KParams base_params(const sp_ctx *ctx) {
    KParams p;
    memset(&p, 0, sizeof(p));
    memcpy(p.rk, ctx->rk, sizeof(p.rk));
    p.ttab = ctx->d_ttab;
    p.mg = ctx->d_mg;
    p.nt = ctx->d_nt;
    return p;
}

int check_desc(const sp_desc &d) {
    if (d.len < 1 || d.len > SP_MAX_MESSAGE_BYTES) return fail(SP_EINVAL, "message length must be in 1..32 MiB");
    if (d.dir > 1u) return fail(SP_EINVAL, "direction must be 0 (H2D) or 1 (D2H)");
    if (!d.src || !d.dst || !d.tag) return fail(SP_EINVAL, "null buffer");
    return SP_OK;
}

uint32_t rows_of(uint64_t len) { return (uint32_t)((((len + 15u) >> 4) + 31u) >> 5); }

// Launch shape.  Every warp that owns rows ends its run with a 32-lane GHASH
// combine whose nibble-table lookups hit 32 different L2 lines per load
// (1,024 L2 requests per warp): fine for big batches (one combine per ~260
// rows), but for small batches it is the whole cost if 16 warps of one SM do
// it at once.  So batches that do not fill the GPU spread their working
// warps over many SMs first (rows per warp per the policy above
// launch_rows); big ones use all 16 warps of every SM.
// Tiny messages (NOP pads, tokens) are latency-bound in their epilogue, so a
// batch also gets at least one warp per message.
// Minimum rows per working warp of a BigTabs batch above the tiny range
// (SPGCM_ROWS_PER_WARP overrides, for launch-shape sweeps).
uint64_t rows_per_warp() {
    static const uint64_t v = [] {
        const char *e = getenv("SPGCM_ROWS_PER_WARP");
        const long x = e ? atol(e) : 0;
        return x > 0 ? (uint64_t)x : (uint64_t)4;
    }();
    return v;
}

// Minimum working warps per CTA of a launch that does not fill the GPU
// (SPGCM_PACK, default 1 = spread one warp per SM first).  Spreading gives
// the lowest latency for a launch alone; packing keeps a small launch on few
// SMs, so the small launches of several streams run side by side instead of
// each occupying most SMs with one 192 KiB-table CTA per working warp.
uint32_t pack_warps() {
    static const uint32_t v = [] {
        const char *e = getenv("SPGCM_PACK");
        const long x = e ? atol(e) : 1;
        return (uint32_t)std::max(1L, std::min<long>(x, kWarpsPerCta));
    }();
    return v;
}

uint64_t env_u64(const char *name, uint64_t dflt);

// SMs a launch of `rows` rows may use.  Small launches (<= SPGCM_SMALL_SMS_ROWS
// rows, default 4096 = 2 MiB: KV batches, tokens, NOP pads) are latency-
// bound, not throughput-bound, yet each 512-thread CTA holds a whole SM's
// register file while it runs; spread over up to 148 SMs they take SMs from
// the model's compute and from the k_xfer transfers beside them.  A context
// can cap them (sp_ctx_set_small_sms; libsppipe sets 32 on its pipes): the
// OPT-30B KV trace then runs 0.947 -> 0.964 of plain with compute and
// 0.77 -> 0.79 swap-only, 64 KiB chunks 0.89 -> 0.91 / 0.80 -> 0.85
// (profiles/r2_ab_kv_sms.txt, r2_ab_small_sms.txt), while one launch alone
// gets slower (1 x 224 KiB 7.3 -> 10.1 us), so direct callers stay uncapped
// by default.  SPGCM_SMALL_SMS overrides every context (0 = no cap).  The
// context's SM budget (sp_ctx_set_max_sms) still applies.
uint64_t launch_sms(const sp_ctx *ctx, uint64_t rows) {
    static const char *env = getenv("SPGCM_SMALL_SMS");  // overrides every context's setting (A/B)
    static const uint64_t env_cap = env ? (uint64_t)atoll(env) : 0;
    static const uint64_t cap_rows = env_u64("SPGCM_SMALL_SMS_ROWS", 4096);
    const uint64_t cap = env ? env_cap : (uint64_t)ctx->small_sms.load(std::memory_order_relaxed);
    const uint64_t sms = (uint64_t)ctx->sms();
    return cap && rows <= cap_rows ? std::min(sms, cap) : sms;
}

void launch_shape(const sp_ctx *ctx, uint64_t rows, uint64_t nmsgs, int &grid, uint32_t &warps_used, uint64_t rpw,
                  uint64_t cap_rows = ~0ull) {
    const uint64_t sms = launch_sms(ctx, cap_rows == ~0ull ? rows : cap_rows);
    const uint64_t want_warps =
        std::max<uint64_t>(1, std::min<uint64_t>(std::max(rows / rpw, std::min(nmsgs, rows)),
                                                 sms * kWarpsPerCta));
    warps_used = (uint32_t)std::max<uint64_t>((want_warps + sms - 1) / sms, std::min<uint64_t>(pack_warps(), want_warps));
    grid = (int)((want_warps + warps_used - 1) / warps_used);
}

// Launch policy by the batch's rows:
//   <= SPGCM_TINY_ROWS (default 512 rows = 256 KiB: NOP pads, tokens, one KV
//      block): BigTabs at 1 row per warp (2 above 256 rows) — the shortest
//      serial chain per warp wins despite the 192 KiB table fill
//      (profiles/r2_launch_shape_sweep.txt, device time per launch in a CUDA
//      graph: 1 x 64 KiB 8.9 -> 6.2 us, 1 x 224 KiB 9.5 -> 7.6 us, 2 KiB
//      token 8.2 -> 6.1 us against SmallTabs).  Such a launch holds up to
//      148 SMs for a few us; while the model's compute outranked the data
//      plane that slowed the traces (r2_ab_tiny.txt), with the data plane's
//      streams on top it is neutral to slightly faster (64 KiB chunks with
//      compute 0.89 -> 0.91 of plain, r2_ab_tiny_prio.txt);
//   <= SPGCM_SMALL_ROWS (default 256; only reached with SPGCM_TINY_ROWS=0):
//      the SmallTabs variant, 10 KB of tables per CTA, 128-thread CTAs, up
//      to 4 per SM, SPGCM_SMALL_RPW (default 2) rows per warp;
//   above: BigTabs, SPGCM_ROWS_PER_WARP (default 4) rows per warp (SmallTabs
//      above 256 rows lost everywhere: 4 x 224 KiB 11.3 -> 15.4 us).
uint64_t env_u64(const char *name, uint64_t dflt) {
    const char *e = getenv(name);
    return e ? (uint64_t)atoll(e) : dflt;
}
uint64_t small_rows_max() {
    static const uint64_t v = env_u64("SPGCM_SMALL_ROWS", 256);
    return v;
}
uint64_t tiny_rows_max() {
    static const uint64_t v = env_u64("SPGCM_TINY_ROWS", 512);
    return v;
}
uint64_t small_rows_per_warp() {
    static const uint64_t v = std::max<uint64_t>(1, env_u64("SPGCM_SMALL_RPW", 2));
    return v;
}

void launch_shape_small(const sp_ctx *ctx, uint64_t rows, uint64_t nmsgs, int &grid, uint32_t &warps_used) {
    const uint64_t sms = launch_sms(ctx, rows);
    // under an SM budget the grid stays within `sms` CTAs (the scheduler
    // may place co-resident CTAs on different SMs)
    const uint64_t per_cta = kThreadsSmall / 32, ctas_per_sm = sms < (uint64_t)ctx->num_sms ? 1 : 4;
    // one-row messages (NOP pads) get one warp each; longer ones split
    // small_rows_per_warp() rows per warp (SPGCM_SMALL_SINGLE_ROWS=k keeps
    // messages of up to k rows on one warp: measured slower for k = 8 on
    // 2 KiB tokens, 9.8 vs 7.9 us per launch, profiles/r2_launch_latency.txt)
    static const uint64_t single = env_u64("SPGCM_SMALL_SINGLE_ROWS", 1);  // >1: measured slower (r2)
    const uint64_t spread = rows <= single * nmsgs ? std::min(nmsgs, rows)
                                              : std::max(rows / small_rows_per_warp(), std::min(nmsgs, rows));
    const uint64_t want_warps = std::max<uint64_t>(1, std::min<uint64_t>(spread, sms * ctas_per_sm * per_cta));
    warps_used = (uint32_t)std::min<uint64_t>(
        per_cta, std::max<uint64_t>((want_warps + sms * ctas_per_sm - 1) / (sms * ctas_per_sm),
                                    std::min<uint64_t>(pack_warps(), want_warps)));
    grid = (int)((want_warps + warps_used - 1) / warps_used);
}

int ensure_ws(Workspace *ws, size_t nmsgs, cudaStream_t s) {
    if (ws->cap_msgs < nmsgs) {
        if (ws->d_msgs) SP_CUDA(cudaFree(ws->d_msgs), "cudaFree");
        size_t cap = std::max<size_t>(nmsgs, 256);
        SP_CUDA(cudaMalloc(&ws->d_msgs, cap * sizeof(MsgDev)), "cudaMalloc(msgs)");
        ws->cap_msgs = cap;
    }
    if (ws->cap_acc < nmsgs) {
        if (ws->d_acc) SP_CUDA(cudaFree(ws->d_acc), "cudaFree");
        size_t cap = std::max<size_t>(nmsgs, 256);
        SP_CUDA(cudaMalloc(&ws->d_acc, cap * 8 * sizeof(uint32_t)), "cudaMalloc(acc)");
        SP_CUDA(cudaMemsetAsync(ws->d_acc, 0, cap * 8 * sizeof(uint32_t), s), "cudaMemsetAsync(acc)");
        ws->cap_acc = cap;
    }
    if (!ws->d_ctl) {
        SP_CUDA(cudaMalloc(&ws->d_ctl, kCtlWords * sizeof(uint32_t)), "cudaMalloc(ctl)");
        SP_CUDA(cudaMemsetAsync(ws->d_ctl, 0, kCtlWords * sizeof(uint32_t), s), "cudaMemsetAsync(ctl)");
    }
    return SP_OK;
}

// Lane combine of a BigTabs launch: with many working warps the 1,024
// nibble-table loads per warp of nt_mul_lane bound the launch on L2
// requests; the shared-memory tree (kTreeBit) replaces them with 32 KiB of
// tables per CTA and 128 loads per warp, at ~0.3-0.5 us more latency per
// warp (four dependent levels, 32 KiB more fill).  Graph-replayed device
// time per launch, tree vs nibble tables (profiles/r2_tree_small.txt):
// 32 x 224 KiB 26.7 vs 32.2 us, 4 x 224 KiB 10.5 vs 11.2, 1 MiB 10.3 vs
// 10.8; 1 x 224 KiB (224 warps) 7.9 vs 7.6, NOP 5.4 vs 4.9.  So from 256
// working warps on, for launches of short runs (<= 16 rows per warp: a big
// batch combines once per ~500 rows and keeps 192 KiB of shared memory);
// SPGCM_TREE_WARPS overrides the warp count (0: always, huge: never).
bool use_tree(uint64_t warps, uint64_t rows) {
    static const uint64_t v = env_u64("SPGCM_TREE_WARPS", 256);
    return warps >= v && (v == 0 || rows <= 16 * warps);
}

template <uint32_t INL>
int launch_rows(const sp_ctx *ctx, KParamsT<INL> p, uint64_t row_begin, uint64_t row_end, cudaStream_t s) {
    if (row_end <= row_begin) return SP_OK;
    p.row_begin = row_begin;
    p.row_end = row_end;
    int grid = 1;
    const uint64_t rows = row_end - row_begin;
    const bool tiny = rows <= tiny_rows_max();
    const bool small = !tiny && rows <= small_rows_max();
    if (small) launch_shape_small(ctx, rows, p.nmsgs, grid, p.warps_used);
    else launch_shape(ctx, rows, p.nmsgs, grid, p.warps_used, tiny ? (rows <= 256 ? 1 : 2) : rows_per_warp());
    // Programmatic dependent launch: a launch that directly follows another
    // kernel on the stream starts (and fills its shared-memory tables)
    // while that kernel's last CTAs drain; it waits in griddepcontrol.wait
    // before touching any data.  SPGCM_PDL=0 disables.
    static const bool pdl = [] {
        const char *e = getenv("SPGCM_PDL");
        return !(e && e[0] == '0');
    }();
    const bool tree = !small && use_tree((uint64_t)grid * p.warps_used, rows);
    if (tree) p.reserved |= kTreeBit;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(small ? kThreadsSmall : kThreads);
    cfg.dynamicSmemBytes = small ? kSmallSmem : (tree ? kSmemBytesTree : kSmemBytes);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    if (small)
        SP_CUDA(cudaLaunchKernelEx(&cfg, k_gcm<INL, SmallTabs, false>, p), "k_gcm launch");
    else
        SP_CUDA(cudaLaunchKernelEx(&cfg, k_gcm<INL, BigTabs, false>, p), "k_gcm launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SP_OK;
}

// One launch for `nlevels` dependent levels (p.lvl_row filled, rows grouped
// by level).  Each level gets the units its own launch would have had
// warps (the tiny-batch policy of launch_rows); the grid covers the
// largest level in one wave and warps loop over claimed units.
template <uint32_t INL>
int launch_levels(const sp_ctx *ctx, KParamsT<INL> p, uint32_t nlevels, cudaStream_t s) {
    const uint64_t all_rows = p.lvl_row[nlevels] - p.lvl_row[0];
    const uint64_t sms = launch_sms(ctx, all_rows);
    int grid = 1;
    uint32_t wu = 1;
    p.nlevels = nlevels;
    p.lvl_unit[0] = 0;
    for (uint32_t l = 0; l < nlevels; ++l) {
        const uint64_t rows = p.lvl_row[l + 1] - p.lvl_row[l];
        const uint64_t rpw = rows <= tiny_rows_max() ? (rows <= 256 ? 1 : 2) : rows_per_warp();
        const uint64_t want = std::max<uint64_t>(1, std::min<uint64_t>(std::max<uint64_t>(rows / rpw, 1),
                                                                       sms * kWarpsPerCta));
        int g = 1;
        uint32_t w = 1;
        launch_shape(ctx, rows, 1, g, w, rpw, all_rows);
        grid = std::max(grid, g);
        wu = std::max(wu, w);
        p.lvl_unit[l + 1] = p.lvl_unit[l] + (uint32_t)want;
    }
    p.warps_used = wu;
    p.row_begin = p.lvl_row[0];
    p.row_end = p.lvl_row[nlevels];
    static const bool pdl = [] {
        const char *e = getenv("SPGCM_PDL");
        return !(e && e[0] == '0');
    }();
    const bool tree = use_tree((uint64_t)grid * wu, p.lvl_row[nlevels] - p.lvl_row[0]);
    if (tree) p.reserved |= kTreeBit;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = tree ? kSmemBytesTree : kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    SP_CUDA(cudaLaunchKernelEx(&cfg, k_gcm<INL, BigTabs, true>, p), "k_gcm levels launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SP_OK;
}

// Build device message table for a batch; returns total rows.  mode: 0 all
// seal, 1 all open, 2 per message (desc.reserved = SP_OP_SEAL / SP_OP_OPEN).
// SPGCM_INLINE_BIG=0: batches above kInline always use the staging ring (A/B).
bool inline_big_enabled() {
    static const bool on = [] {
        const char *e = getenv("SPGCM_INLINE_BIG");
        return !(e && e[0] == '0');
    }();
    return on;
}

// SPGCM_TINY_PARAMS=0: batches of <= kInlineTiny messages use the 32-slot parameter block (A/B).
bool tiny_params_enabled() {
    static const bool on = [] {
        const char *e = getenv("SPGCM_TINY_PARAMS");
        return !(e && e[0] == '0');
    }();
    return on;
}

// SPGCM_FUSE_LEVELS=0: sp_crypt_levels issues one launch per level (A/B).
bool fuse_levels_enabled() {
    static const bool on = [] {
        const char *e = getenv("SPGCM_FUSE_LEVELS");
        return !(e && e[0] == '0');
    }();
    return on;
}

// With `big` non-null, a batch of kInline+1 .. kInlineBig messages goes
// inline in *big (and *use_big is set) instead of through the staging ring.
int stage_batch(const sp_ctx *ctx, const sp_desc *d, int n, cudaStream_t s, Workspace *ws, KParams &p,
                uint64_t &rows, int mode, KParamsBig *big = nullptr, bool *use_big = nullptr) {
    ws->h_msgs.resize((size_t)n);
    rows = 0;
    for (int i = 0; i < n; ++i) {
        int rc = check_desc(d[i]);
        if (rc) return rc;
        const uint32_t op = d[i].reserved & ~SP_STATUS_ON_FAILURE;
        if (mode == 2 && op > SP_OP_OPEN) return fail(SP_EINVAL, "op must be SP_OP_SEAL or SP_OP_OPEN");
        const bool open = mode == 1 || (mode == 2 && op == SP_OP_OPEN);
        if (open && !d[i].status) return fail(SP_EINVAL, "open needs a status pointer");
        MsgDev &m = ws->h_msgs[(size_t)i];
        m.src = static_cast<const uint8_t *>(d[i].src);
        m.dst = static_cast<uint8_t *>(d[i].dst);
        m.tag = static_cast<uint8_t *>(d[i].tag);
        m.status = d[i].status;
        m.len = d[i].len;
        m.iv = d[i].iv;
        m.dir = d[i].dir | (open ? kOpenBit : 0u) | ((d[i].reserved & SP_STATUS_ON_FAILURE) ? kStickyBit : 0u);
        m.rows = rows_of(d[i].len);
        m.row_begin = rows;
        rows += m.rows;
    }
    int rc = ensure_ws(ws, (size_t)n, s);
    if (rc) return rc;
    p = base_params(ctx);
    if (use_big) *use_big = false;
    if ((uint32_t)n <= kInline) {
        memcpy(p.inl, ws->h_msgs.data(), (size_t)n * sizeof(MsgDev));
    } else if (big && (uint32_t)n <= kInlineBig && inline_big_enabled()) {
        memcpy(big->rk, p.rk, sizeof(p.rk));
        big->ttab = p.ttab;
        big->mg = p.mg;
        big->nt = p.nt;
        big->msgs = ws->d_msgs;
        big->acc = ws->d_acc;
        big->nmsgs = (uint32_t)n;
        big->reserved = 0;
        big->row_begin = big->row_end = 0;
        big->warps_used = 0;
        memcpy(big->inl, ws->h_msgs.data(), (size_t)n * sizeof(MsgDev));
        *use_big = true;
    } else {
        // pinned ring slot: wait only for the copy that last used this slot
        const int k = ws->slot;
        ws->slot = (k + 1) % kPinSlots;
        if (ws->cap_pin < (size_t)n) {
            for (int j = 0; j < kPinSlots; ++j) {
                if (ws->ev_live[j]) SP_CUDA(cudaEventSynchronize(ws->ev_pin[j]), "cudaEventSynchronize");
                if (ws->h_pin[j]) cudaFreeHost(ws->h_pin[j]);
                ws->h_pin[j] = nullptr;
                ws->ev_live[j] = false;
            }
            const size_t cap = std::max<size_t>((size_t)n, 1024);
            for (int j = 0; j < kPinSlots; ++j) {
                SP_CUDA(cudaHostAlloc(reinterpret_cast<void **>(&ws->h_pin[j]), cap * sizeof(MsgDev),
                                      cudaHostAllocDefault), "cudaHostAlloc(msgs)");
                if (!ws->ev_pin[j])
                    SP_CUDA(cudaEventCreateWithFlags(&ws->ev_pin[j], cudaEventDisableTiming), "event");
            }
            ws->cap_pin = cap;
        }
        if (ws->ev_live[k]) SP_CUDA(cudaEventSynchronize(ws->ev_pin[k]), "cudaEventSynchronize");
        memcpy(ws->h_pin[k], ws->h_msgs.data(), (size_t)n * sizeof(MsgDev));
        SP_CUDA(cudaMemcpyAsync(ws->d_msgs, ws->h_pin[k], (size_t)n * sizeof(MsgDev), cudaMemcpyHostToDevice, s),
                "cudaMemcpyAsync(msgs)");
        SP_CUDA(cudaEventRecord(ws->ev_pin[k], s), "cudaEventRecord");
        ws->ev_live[k] = true;
    }
    p.msgs = ws->d_msgs;
    p.acc = ws->d_acc;
    p.nmsgs = (uint32_t)n;
    return SP_OK;
}

int run_batch(sp_ctx *ctx, const sp_desc *d, int n, cudaStream_t s, int mode) {
    if (!ctx) return fail(SP_EINVAL, "null context");
    if (n <= 0) return n == 0 ? SP_OK : fail(SP_EINVAL, "negative batch size");
    if (!d) return fail(SP_EINVAL, "null descriptors");
    SP_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    Workspace *ws = workspace_for(ctx->device, s);
    std::lock_guard<std::mutex> lk(ws->mu);
    KParams p;
    static thread_local KParamsBig big;  // 16.6 KiB: off the stack
    bool use_big = false;
    uint64_t rows = 0;
    int rc = stage_batch(ctx, d, n, s, ws, p, rows, mode, &big, &use_big);
    if (rc) return rc;
    if (use_big) return launch_rows(ctx, big, 0, rows, s);
    if ((uint32_t)n <= kInlineTiny && tiny_params_enabled()) {
        // the driver copies every parameter byte into the launch: 0.5 KiB
        // instead of 2.4 KiB for the few-message launches the engine issues
        // most (KV blocks, NOP runs, tokens)
        KParamsTiny t;
        memcpy(t.inl, p.inl, (size_t)n * sizeof(MsgDev));
        memcpy(t.rk, p.rk, sizeof(t.rk));
        t.ttab = p.ttab;
        t.mg = p.mg;
        t.nt = p.nt;
        t.msgs = p.msgs;
        t.acc = p.acc;
        t.nmsgs = p.nmsgs;
        t.reserved = 0;
        t.row_begin = t.row_end = 0;
        t.warps_used = 0;
        return launch_rows(ctx, t, 0, rows, s);
    }
    return launch_rows(ctx, p, 0, rows, s);
}

// ---- host-buffer pipeline ----------------------------------------------------
// Pieces of ~kPieceBytes (whole rows) flow H2D (stream a) -> kernel (stream b)
// -> D2H (stream c); each stage waits on the previous stage's event.
// Piece schedule of the host pipeline: pieces double from kPieceMinRows up to
// max_piece_rows() (the first one twice) and halve again over the tail, so the H2D of the first
// piece and the D2H of the last one (the only un-overlapped transfers) are
// small while the steady state runs on large copies.
constexpr uint64_t kPieceMinRows = (1ull << 20) / 512u;  // 1 MiB

uint64_t max_piece_rows() {
    // 32 MiB by default; SPGCM_PIECE_MIB overrides (tuning)
    static const uint64_t rows = [] {
        const char *e = getenv("SPGCM_PIECE_MIB");
        const long mib = e ? atol(e) : 32;
        return (uint64_t)std::max(1L, mib) * (1ull << 20) / 512u;
    }();
    return rows;
}

std::vector<uint64_t> piece_schedule(uint64_t rows) {
    std::vector<uint64_t> out;
    const uint64_t cap = max_piece_rows();
    uint64_t done = 0, cur = std::min(kPieceMinRows, cap);
    // ramp 1, 1, 2, 4, ... cap/2 MiB sums to cap: the steady-state pieces then
    // start on multiples of cap, i.e. on 32 MiB message boundaries, so each
    // moves as ONE copy per direction instead of a 1 MiB + 31 MiB pair (a
    // 1 MiB copy runs at ~20 GB/s and opened a ~40 us gap per piece)
    if (cap >= 2 * cur && rows > 2 * cur) {
        out.push_back(cur);
        done = cur;
    }
    while (done < rows) {
        const uint64_t left = rows - done;
        uint64_t take = std::min(cur, left);
        if (left > take && left < 2 * take) take = std::max<uint64_t>(kPieceMinRows, left / 2);  // taper
        take = std::min(take, left);
        out.push_back(take);
        done += take;
        cur = std::min(cap, cur * 2);
        if (rows - done < 2 * cur) cur = std::max<uint64_t>(kPieceMinRows, (rows - done) / 2);
    }
    return out;
}

struct HostPipe {
    int device = -1;
    cudaStream_t s_in = nullptr, s_k = nullptr, s_out = nullptr;
    uint8_t *d_in = nullptr, *d_out = nullptr, *d_tags = nullptr;
    int32_t *d_status = nullptr;
    uint8_t *h_tags = nullptr;  // pinned staging: all tags of a batch cross PCIe in one copy
    size_t cap_bytes = 0, cap_msgs = 0;
    std::vector<cudaEvent_t> ev_in, ev_k;
    std::mutex mu;
};

std::mutex g_pipes_mu;
std::map<int, HostPipe *> g_pipes;

HostPipe *pipe_for(int device) {
    std::lock_guard<std::mutex> lk(g_pipes_mu);
    auto &p = g_pipes[device];
    if (!p) p = new HostPipe();
    return p;
}

int ensure_pipe(HostPipe *hp, int device, size_t bytes, size_t nmsgs, size_t npieces) {
    if (!hp->s_in) {
        SP_CUDA(cudaStreamCreateWithFlags(&hp->s_in, cudaStreamNonBlocking), "stream");
        SP_CUDA(cudaStreamCreateWithFlags(&hp->s_k, cudaStreamNonBlocking), "stream");
        SP_CUDA(cudaStreamCreateWithFlags(&hp->s_out, cudaStreamNonBlocking), "stream");
        hp->device = device;
    }
    if (hp->cap_bytes < bytes) {
        if (hp->d_in) { cudaFree(hp->d_in); cudaFree(hp->d_out); }
        size_t cap = std::max<size_t>(bytes, 1u << 20);
        SP_CUDA(cudaMalloc(&hp->d_in, cap), "cudaMalloc(pipe in)");
        SP_CUDA(cudaMalloc(&hp->d_out, cap), "cudaMalloc(pipe out)");
        hp->cap_bytes = cap;
    }
    if (hp->cap_msgs < nmsgs) {
        if (hp->d_tags) { cudaFree(hp->d_tags); cudaFree(hp->d_status); cudaFreeHost(hp->h_tags); }
        size_t cap = std::max<size_t>(nmsgs, 64);
        SP_CUDA(cudaMalloc(&hp->d_tags, cap * 16), "cudaMalloc(pipe tags)");
        SP_CUDA(cudaHostAlloc(reinterpret_cast<void **>(&hp->h_tags), cap * 16, cudaHostAllocDefault),
                "cudaHostAlloc(pipe tags)");
        SP_CUDA(cudaMalloc(&hp->d_status, cap * sizeof(int32_t)), "cudaMalloc(pipe status)");
        hp->cap_msgs = cap;
    }
    while (hp->ev_in.size() < npieces) {
        cudaEvent_t a, b;
        SP_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming), "event");
        SP_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming), "event");
        hp->ev_in.push_back(a);
        hp->ev_k.push_back(b);
    }
    return SP_OK;
}

// byte range [lo, hi) of local rows [t0, t1) of a message of `len` bytes
inline void rows_to_bytes(uint64_t len, uint32_t rows, uint64_t t0, uint64_t t1, uint64_t &lo, uint64_t &hi) {
    const int64_t nblk = (int64_t)((len + 15u) >> 4);
    const int64_t b0 = nblk - 32 * (int64_t)(rows - t0);
    const int64_t b1 = nblk - 32 * (int64_t)(rows - t1);
    lo = (uint64_t)std::max<int64_t>(0, b0) * 16u;
    hi = std::min<uint64_t>(len, (uint64_t)std::max<int64_t>(0, b1) * 16u);
}

int run_host_batch(sp_ctx *ctx, const sp_desc *d, int n, bool open) {
    if (!ctx) return fail(SP_EINVAL, "null context");
    if (n <= 0) return n == 0 ? SP_OK : fail(SP_EINVAL, "negative batch size");
    if (!d) return fail(SP_EINVAL, "null descriptors");
    for (int i = 0; i < n; ++i) {
        int rc = check_desc(d[i]);
        if (rc) return rc;
    }
    SP_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    HostPipe *hp = pipe_for(ctx->device);
    std::lock_guard<std::mutex> lk(hp->mu);

    // device staging layout: messages packed at 256-byte aligned offsets
    std::vector<uint64_t> off((size_t)n);
    uint64_t total = 0, rows = 0;
    for (int i = 0; i < n; ++i) {
        off[(size_t)i] = total;
        total += (d[i].len + 255u) & ~255ull;
        rows += rows_of(d[i].len);
    }
    const std::vector<uint64_t> sched = piece_schedule(rows);
    const size_t npieces = sched.size();
    int rc = ensure_pipe(hp, ctx->device, total, (size_t)n, npieces);
    if (rc) return rc;

    std::vector<sp_desc> dd((size_t)n);
    for (int i = 0; i < n; ++i) {
        dd[(size_t)i] = d[i];
        dd[(size_t)i].src = hp->d_in + off[(size_t)i];
        dd[(size_t)i].dst = hp->d_out + off[(size_t)i];
        dd[(size_t)i].tag = hp->d_tags + 16u * (size_t)i;
        dd[(size_t)i].status = hp->d_status + i;
    }
    if (open) {
        // the previous call's tag D2H out of h_tags finished at its stream sync
        for (int i = 0; i < n; ++i) memcpy(hp->h_tags + 16u * (size_t)i, d[i].tag, 16);
        SP_CUDA(cudaMemcpyAsync(hp->d_tags, hp->h_tags, 16u * (size_t)n, cudaMemcpyHostToDevice, hp->s_in),
                "cudaMemcpyAsync(tags)");
    }
    Workspace *ws = workspace_for(ctx->device, hp->s_k);
    std::lock_guard<std::mutex> wlk(ws->mu);
    KParams p;
    uint64_t rows_chk = 0;
    rc = stage_batch(ctx, dd.data(), n, hp->s_k, ws, p, rows_chk, open ? 1 : 0);
    if (rc) return rc;

    // walk pieces of whole rows across the flattened batch
    int mi = 0;
    uint64_t g = 0;
    size_t k = 0;
    const std::vector<MsgDev> &msgs = ws->h_msgs;
    while (g < rows) {
        const uint64_t g_end = std::min(rows, g + sched[k]);
        const cudaStream_t s_in = hp->s_in;
        // H2D for every message slice in [g, g_end)
        int mj = mi;
        uint64_t gg = g;
        while (gg < g_end) {
            const MsgDev &m = msgs[(size_t)mj];
            const uint64_t t0 = gg - m.row_begin, t1 = std::min<uint64_t>(m.rows, g_end - m.row_begin);
            uint64_t lo, hi;
            rows_to_bytes(m.len, m.rows, t0, t1, lo, hi);
            if (hi > lo)
                SP_CUDA(cudaMemcpyAsync(hp->d_in + off[(size_t)mj] + lo, static_cast<const uint8_t *>(d[mj].src) + lo,
                                        hi - lo, cudaMemcpyHostToDevice, s_in),
                        "cudaMemcpyAsync(H2D)");
            gg = m.row_begin + t1;
            if (t1 == m.rows) ++mj;
        }
        SP_CUDA(cudaEventRecord(hp->ev_in[k], s_in), "event record");
        SP_CUDA(cudaStreamWaitEvent(hp->s_k, hp->ev_in[k], 0), "wait");
        rc = launch_rows(ctx, p, g, g_end, hp->s_k);
        if (rc) return rc;
        SP_CUDA(cudaEventRecord(hp->ev_k[k], hp->s_k), "event record");
        SP_CUDA(cudaStreamWaitEvent(hp->s_out, hp->ev_k[k], 0), "wait");
        // D2H of the same slices.  An open releases a message's plaintext
        // only once its tag is verified: its bytes cross to the caller in
        // one copy after the piece that holds its last row (where the
        // finisher checks the tag and, on a mismatch, zeroes the device
        // copy), so unverified plaintext never reaches host memory
        // (channel.py:110-115 returns none on failure).
        gg = g;
        while (gg < g_end) {
            const MsgDev &m = msgs[(size_t)mi];
            const uint64_t t0 = gg - m.row_begin, t1 = std::min<uint64_t>(m.rows, g_end - m.row_begin);
            uint64_t lo, hi;
            if (open) {
                lo = 0;
                hi = t1 == m.rows ? m.len : 0;
            } else {
                rows_to_bytes(m.len, m.rows, t0, t1, lo, hi);
            }
            if (hi > lo)
                SP_CUDA(cudaMemcpyAsync(static_cast<uint8_t *>(d[mi].dst) + lo, hp->d_out + off[(size_t)mi] + lo,
                                        hi - lo, cudaMemcpyDeviceToHost, hp->s_out),
                        "cudaMemcpyAsync(D2H)");
            gg = m.row_begin + t1;
            if (t1 == m.rows) ++mi;
        }
        g = g_end;
        ++k;
    }
    if (!open)
        SP_CUDA(cudaMemcpyAsync(hp->h_tags, hp->d_tags, 16u * (size_t)n, cudaMemcpyDeviceToHost, hp->s_out),
                "cudaMemcpyAsync(tags D2H)");
    std::vector<int32_t> st;
    if (open) {
        st.resize((size_t)n);
        SP_CUDA(cudaMemcpyAsync(st.data(), hp->d_status, (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                hp->s_out),
                "cudaMemcpyAsync(status)");
    }
    SP_CUDA(cudaStreamSynchronize(hp->s_out), "cudaStreamSynchronize");
    if (!open)
        for (int i = 0; i < n; ++i) memcpy(d[i].tag, hp->h_tags + 16u * (size_t)i, 16);
    if (open) {
        int bad = 0;
        for (int i = 0; i < n; ++i) {
            if (d[i].status) *d[i].status = st[(size_t)i];
            if (st[(size_t)i]) bad = 1;  // the device zeroed the message before it crossed
        }
        if (bad) return fail(SP_EAUTH, "authentication failed");
    }
    return SP_OK;
}

}  // namespace

// =============================================================================
// C ABI
// =============================================================================

extern "C" {

const char *sp_last_error(void) { return g_err.c_str(); }
const char *sp_version(void) { return "spgcm 0.1.0 sm_100a"; }
uint64_t sp_launch_count(void) { return g_launches.load(); }

int sp_ctx_create(const uint8_t key[SP_KEY_BYTES], sp_ctx **out) {
    if (!key || !out) return fail(SP_EINVAL, "null argument");
    *out = nullptr;
    int dev = 0;
    SP_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    cudaDeviceProp prop;
    SP_CUDA(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
    if (prop.major != 10) return fail(SP_ENODEV, "libspgcm is built for sm_100a (B200) only");
    SP_CUDA(cudaFuncSetAttribute(k_gcm<kInline, BigTabs, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kSmemBytesTree), "cudaFuncSetAttribute(k_gcm)");
    SP_CUDA(cudaFuncSetAttribute(k_gcm<kInlineTiny, BigTabs, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kSmemBytesTree), "cudaFuncSetAttribute(k_gcm tiny)");
    SP_CUDA(cudaFuncSetAttribute(k_gcm<kInlineBig, BigTabs, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kSmemBytesTree), "cudaFuncSetAttribute(k_gcm big)");
    SP_CUDA(cudaFuncSetAttribute(k_gcm<kInline, BigTabs, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kSmemBytesTree), "cudaFuncSetAttribute(k_gcm levels)");
    SP_CUDA(cudaFuncSetAttribute(k_gcm<kInlineTiny, BigTabs, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kSmemBytesTree), "cudaFuncSetAttribute(k_gcm tiny levels)");
    SP_CUDA(cudaFuncSetAttribute(k_gcm<kInlineBig, BigTabs, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kSmemBytesTree), "cudaFuncSetAttribute(k_gcm big levels)");
    sp_ctx *c = new sp_ctx();
    c->device = dev;
    c->num_sms = prop.multiProcessorCount;
    key_expand(key, c->rk);
    const Consts &k = consts();
    auto bail = [&](int rc) {
        sp_ctx_destroy(c);
        return rc;
    };
    cudaError_t e;
    if ((e = cudaMalloc(&c->d_ttab, 5 * 256 * sizeof(uint32_t))) ||
        (e = cudaMalloc(&c->d_mg, 256 * sizeof(uint4))) ||
        (e = cudaMalloc(&c->d_nt, (size_t)kNumNt * kNtEntries * sizeof(uint4))) ||
        (e = cudaMalloc(&c->d_pow, (size_t)(kNumNt + 1) * sizeof(uint4))) ||
        (e = cudaMalloc(&c->d_sbox, 256)) || (e = cudaMalloc(&c->d_h, sizeof(uint4))))
        return bail(cuda_fail(e, "cudaMalloc(ctx)"));
    if ((e = cudaMemcpy(c->d_ttab, k.t, sizeof(k.t), cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(c->d_ttab + 4 * 256, k.r8, sizeof(k.r8), cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(c->d_sbox, k.sbox, 256, cudaMemcpyHostToDevice)))
        return bail(cuda_fail(e, "cudaMemcpy(ctx)"));
    KParams p = base_params(c);
    k_setup_h<<<1, 1>>>(p, c->d_sbox, c->d_h);
    k_setup_powers<<<(kNumNt + 1 + 127) / 128, 128>>>(c->d_h, c->d_pow);
    k_setup_nt<<<(unsigned)(((uint64_t)kNumNt * kNtEntries + 255) / 256), 256>>>(c->d_pow, c->d_nt);
    k_setup_mg<<<1, 256>>>(c->d_pow, c->d_mg);
    g_launches.fetch_add(4, std::memory_order_relaxed);
    if ((e = cudaGetLastError()) || (e = cudaDeviceSynchronize())) return bail(cuda_fail(e, "ctx setup kernels"));
    *out = c;
    return SP_OK;
}

void sp_ctx_destroy(sp_ctx *c) {
    if (!c) return;
    cudaFree(c->d_ttab);
    cudaFree(c->d_mg);
    cudaFree(c->d_nt);
    cudaFree(c->d_pow);
    cudaFree(c->d_sbox);
    cudaFree(c->d_h);
    delete c;
}

int sp_ctx_round_keys(const sp_ctx *c, uint8_t out[240]) {
    if (!c || !out) return fail(SP_EINVAL, "null argument");
    memcpy(out, c->rk, 240);
    return SP_OK;
}

int sp_ctx_set_max_sms(sp_ctx *c, int max_sms) {
    if (!c || max_sms < 0) return fail(SP_EINVAL, "max_sms must be >= 0");
    c->max_sms.store(max_sms, std::memory_order_relaxed);
    return SP_OK;
}

int sp_ctx_max_sms(const sp_ctx *c) { return c ? c->sms() : 0; }

int sp_ctx_set_small_sms(sp_ctx *c, int small_sms) {
    if (!c || small_sms < 0) return fail(SP_EINVAL, "small_sms must be >= 0");
    c->small_sms.store(small_sms, std::memory_order_relaxed);
    return SP_OK;
}

int sp_ctx_hash_key(const sp_ctx *c, uint8_t out[16]) {
    if (!c || !out) return fail(SP_EINVAL, "null argument");
    SP_CUDA(cudaMemcpy(out, c->d_h, 16, cudaMemcpyDeviceToHost), "cudaMemcpy(H)");
    return SP_OK;
}

int sp_seal_batch(sp_ctx *ctx, const sp_desc *d, int n, sp_stream_t stream) {
    return run_batch(ctx, d, n, static_cast<cudaStream_t>(stream), 0);
}

int sp_open_batch(sp_ctx *ctx, const sp_desc *d, int n, sp_stream_t stream) {
    return run_batch(ctx, d, n, static_cast<cudaStream_t>(stream), 1);
}

int sp_crypt_batch(sp_ctx *ctx, const sp_desc *d, int n, sp_stream_t stream) {
    return run_batch(ctx, d, n, static_cast<cudaStream_t>(stream), 2);
}

int sp_crypt_levels(sp_ctx *ctx, const sp_desc *d, int n, const int *level_start, int nlevels,
                    sp_stream_t stream) {
    if (!ctx) return fail(SP_EINVAL, "null context");
    if (!d || n <= 0) return fail(SP_EINVAL, "null or empty descriptor array");
    if (nlevels < 1 || !level_start) return fail(SP_EINVAL, "need at least one level");
    if (level_start[0] != 0 || level_start[nlevels] != n) return fail(SP_EINVAL, "levels must cover the batch");
    for (int l = 0; l < nlevels; ++l)
        if (level_start[l + 1] <= level_start[l]) return fail(SP_EINVAL, "empty level");
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (nlevels == 1) return run_batch(ctx, d, n, s, 2);
    if ((uint32_t)nlevels > kMaxLevels || (uint32_t)n > kInlineBig || !fuse_levels_enabled()) {
        for (int l = 0; l < nlevels; ++l) {  // one launch per level, in stream order
            const int rc = run_batch(ctx, d + level_start[l], level_start[l + 1] - level_start[l], s, 2);
            if (rc) return rc;
        }
        return SP_OK;
    }
    SP_CUDA(cudaSetDevice(ctx->device), "cudaSetDevice");
    Workspace *ws = workspace_for(ctx->device, s);
    std::lock_guard<std::mutex> lk(ws->mu);
    KParams p;
    static thread_local KParamsBig big;
    bool use_big = false;
    uint64_t rows = 0;
    int rc = stage_batch(ctx, d, n, s, ws, p, rows, 2, &big, &use_big);
    if (rc) return rc;
    auto fill = [&](auto &q) {
        q.ctl = ws->d_ctl;
        for (int l = 0; l < nlevels; ++l) q.lvl_row[l] = ws->h_msgs[(size_t)level_start[l]].row_begin;
        q.lvl_row[nlevels] = rows;
    };
    if (use_big) {
        fill(big);
        return launch_levels(ctx, big, (uint32_t)nlevels, s);
    }
    if ((uint32_t)n <= kInlineTiny && tiny_params_enabled()) {
        KParamsTiny t;
        memset(&t, 0, sizeof(t));
        memcpy(t.inl, p.inl, (size_t)n * sizeof(MsgDev));
        memcpy(t.rk, p.rk, sizeof(t.rk));
        t.ttab = p.ttab;
        t.mg = p.mg;
        t.nt = p.nt;
        t.msgs = p.msgs;
        t.acc = p.acc;
        t.nmsgs = p.nmsgs;
        fill(t);
        return launch_levels(ctx, t, (uint32_t)nlevels, s);
    }
    fill(p);
    return launch_levels(ctx, p, (uint32_t)nlevels, s);
}

int sp_seal(sp_ctx *ctx, uint32_t dir, uint64_t iv, const void *src, size_t len, void *dst, void *tag16,
            sp_stream_t stream) {
    sp_desc d{dir, 0, iv, len, src, dst, tag16, nullptr};
    return sp_seal_batch(ctx, &d, 1, stream);
}

int sp_open(sp_ctx *ctx, uint32_t dir, uint64_t iv, const void *src, size_t len, const void *tag16, void *dst,
            int32_t *status_dev, sp_stream_t stream) {
    sp_desc d{dir, 0, iv, len, src, dst, const_cast<void *>(tag16), status_dev};
    return sp_open_batch(ctx, &d, 1, stream);
}

int sp_seal_host_batch(sp_ctx *ctx, const sp_desc *d, int n) { return run_host_batch(ctx, d, n, false); }

int sp_open_host_batch(sp_ctx *ctx, const sp_desc *d, int n) { return run_host_batch(ctx, d, n, true); }

int sp_seal_host(sp_ctx *ctx, uint32_t dir, uint64_t iv, const void *src, size_t len, void *dst,
                 uint8_t tag16[SP_TAG_BYTES]) {
    sp_desc d{dir, 0, iv, len, src, dst, tag16, nullptr};
    return run_host_batch(ctx, &d, 1, false);
}

int sp_open_host(sp_ctx *ctx, uint32_t dir, uint64_t iv, const void *src, size_t len,
                 const uint8_t tag16[SP_TAG_BYTES], void *dst) {
    int32_t status = 0;
    sp_desc d{dir, 0, iv, len, src, dst, const_cast<uint8_t *>(tag16), &status};
    return run_host_batch(ctx, &d, 1, true);
}

}  // extern "C"
