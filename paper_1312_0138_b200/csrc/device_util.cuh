// Device helpers shared by the sm_100a kernels (bucket.cu, scan.cu): warp
// scans, TMA bulk copies with mbarriers, and the bitset-word extraction
// primitives used by every scan/extraction path.
#pragma once

#include <cstdint>

#include "kernels.h"

namespace bws_gpu {
namespace dev {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, unsigned lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(kFull, v, off);
        if (lane >= static_cast<unsigned>(off)) v += o;
    }
    return v;
}

// ---- TMA bulk copy + mbarrier helpers (PTX) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// One thread: expect `bytes` on `bar` and start a bulk global->shared copy.
__device__ __forceinline__ void tma_load_bytes(void* dst, const void* src, unsigned bytes,
                                               unsigned long long* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// A bulk global->shared copy completing `bytes` of a transaction the caller
// has already announced on `bar` (mbarrier.arrive.expect_tx).
__device__ __forceinline__ void tma_copy_bytes(void* dst, const void* src, unsigned bytes,
                                               unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// L2 eviction-priority policies (createpolicy) for cache-hinted accesses.
__device__ __forceinline__ unsigned long long l2_policy_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long l2_policy_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// tma_load_bytes with an L2 cache policy (e.g. evict_first for a stream read once).
__device__ __forceinline__ void tma_load_bytes_hint(void* dst, const void* src, unsigned bytes,
                                                    unsigned long long* bar, unsigned long long policy) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void st_hint(uint32_t* p, uint32_t v, unsigned long long policy) {
    asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(policy) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 16-byte streaming load that does not allocate in L1 (kernels that keep
// ~200 KB of SMEM per SM leave a small L1 for the loads in flight)
__device__ __forceinline__ uint4 ld_na(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// Writes kb + bit for every set bit of x, ascending, to the padded stage.
__device__ __forceinline__ void stage_bits(uint32_t x, uint32_t kb, uint32_t& p, uint32_t* stage) {
    while (x) {
        const int bt = __ffs(x) - 1;
        x &= x - 1;
        stage[p + (p >> 5)] = kb + static_cast<uint32_t>(bt);
        ++p;
    }
}

// Copies `count` staged keys to o[0, count) with coalesced stores. Staged key
// i = lane + 32 r sits at stage[lane + 33 r] (one pad word per 32), so both
// sides advance by a constant stride: no per-key index arithmetic.
__device__ __forceinline__ void drain_stage(const uint32_t* stage, uint32_t count,
                                            uint32_t* __restrict__ o, unsigned lane) {
    __syncwarp();
    const uint32_t* sp = stage + lane;
    uint32_t* gp = o + lane;
    const uint32_t rows = count >> 5;  // full rows of 32 keys
    uint32_t r = 0;
#pragma unroll 1
    for (; r + 4 <= rows; r += 4, sp += 4 * 33, gp += 4 * 32) {
        const uint32_t a = sp[0], b = sp[33], c = sp[66], d = sp[99];
        __stcs(gp, a);
        __stcs(gp + 32, b);
        __stcs(gp + 64, c);
        __stcs(gp + 96, d);
    }
#pragma unroll 1
    for (; r < rows; ++r, sp += 33, gp += 32) __stcs(gp, sp[0]);
    if (lane < (count & 31u)) __stcs(gp, sp[0]);
    __syncwarp();
}

// Extracts the 32 words at s_bits[w .. w+32) (word per lane) to o[0 ..) and
// returns the number of keys: a chunk with more than BUCKET_STAGE keys goes
// word by word with a ballot (lane = bit, coalesced 128-byte stores), others
// through the warp's stage.
template <int STAGE = BUCKET_STAGE>
__device__ __forceinline__ uint32_t extract_words32(const uint32_t* s_bits, uint32_t w,
                                                    uint32_t key_hi, uint32_t* __restrict__ o,
                                                    uint32_t* s_stage, unsigned lane) {
    const uint32_t x = s_bits[w + lane];
    const uint32_t cx = __popc(x);
    const uint32_t incl = warp_incl_scan(cx, lane);
    const uint32_t ctot = __shfl_sync(kFull, incl, 31);
    if (ctot == 0) return 0;
    if (ctot > static_cast<uint32_t>(STAGE)) {
        const unsigned lt = lanemask_lt();
        uint32_t q = 0;
        const uint32_t kb = key_hi + (w << 5) + lane;
        for (int j = 0; j < 32; ++j) {
            const uint32_t xj = __shfl_sync(kFull, x, j);
            const bool bit = (xj >> lane) & 1u;
            const unsigned m = __ballot_sync(kFull, bit);
            if (bit) __stcs(o + q + __popc(m & lt), kb + (static_cast<uint32_t>(j) << 5));
            q += __popc(m);
        }
        return ctot;
    }
    uint32_t p = incl - cx;
    stage_bits(x, key_hi + ((w + lane) << 5), p, s_stage);
    drain_stage(s_stage, ctot, o, lane);
    return ctot;
}


// Extracts the 64 words at s_bits[w .. w+64) (w a multiple of 64; lane l
// holds words 2l, 2l+1) to o[0 ..) in order; returns the number of keys. Half
// the per-chunk overhead (load, popcount, warp scan, drain) of two 32-word
// chunks and a little less lane divergence (two words per lane). Chunks with
// more than STAGE keys go through extract_words32 (ballots when dense).
template <int STAGE>
__device__ __forceinline__ uint32_t extract_words64(const uint32_t* s_bits, uint32_t w, uint32_t key_hi,
                                                    uint32_t* __restrict__ o, uint32_t* s_stage,
                                                    unsigned lane) {
    const uint2 xx = reinterpret_cast<const uint2*>(s_bits + w)[lane];
    const uint32_t c0 = __popc(xx.x);
    const uint32_t c = c0 + __popc(xx.y);
    const uint32_t incl = warp_incl_scan(c, lane);
    const uint32_t ctot = __shfl_sync(kFull, incl, 31);
    if (ctot == 0) return 0;
    if (ctot > static_cast<uint32_t>(STAGE)) {
        const uint32_t n0 = extract_words32<STAGE>(s_bits, w, key_hi, o, s_stage, lane);
        return n0 + extract_words32<STAGE>(s_bits, w + 32, key_hi, o + n0, s_stage, lane);
    }
    uint32_t p = incl - c;
    const uint32_t kb = key_hi + ((w + 2 * lane) << 5);
    stage_bits(xx.x, kb, p, s_stage);
    stage_bits(xx.y, kb + 32, p, s_stage);
    drain_stage(s_stage, ctot, o, lane);
    return ctot;
}

// Extracts the `nwords` (multiple of 128) SMEM bitset words at s_bits[w0 ..)
// to o[0 ..) in order; returns the number of keys. 128-word steps, lane-major
// (lane owns 4 words); a step with <= STAGE keys is extracted in one pass
// through the warp's stage, denser steps as two 64-word sub-steps (two words
// per lane), and very dense ones word by word with ballots.
template <int STAGE>
__device__ __forceinline__ uint32_t extract_seg128(const uint32_t* s_bits, uint32_t w0, uint32_t nwords,
                                                   uint32_t key_hi, uint32_t* __restrict__ o,
                                                   uint32_t* s_stage, unsigned lane) {
    const uint4* s4 = reinterpret_cast<const uint4*>(s_bits);
    uint32_t total = 0;
    for (uint32_t w = w0; w < w0 + nwords; w += 128) {
        const uint4 v = s4[w / 4 + lane];
        const uint32_t cl = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
        const uint32_t incl = warp_incl_scan(cl, lane);
        const uint32_t ctot = __shfl_sync(kFull, incl, 31);
        if (ctot == 0) continue;
        uint32_t* od = o + total;
        total += ctot;
        if (ctot <= static_cast<uint32_t>(STAGE)) {
            uint32_t p = incl - cl;
            const uint32_t kb = key_hi + ((w + 4 * lane) << 5);
            stage_bits(v.x, kb, p, s_stage);
            stage_bits(v.y, kb + 32, p, s_stage);
            stage_bits(v.z, kb + 64, p, s_stage);
            stage_bits(v.w, kb + 96, p, s_stage);
            drain_stage(s_stage, ctot, od, lane);
            continue;
        }
        if (ctot > 2u * STAGE) {  // dense: word-by-word ballots
#pragma unroll 1
            for (uint32_t q = 0; q < 128; q += 32) od += extract_words32<STAGE>(s_bits, w + q, key_hi, od, s_stage, lane);
            continue;
        }
        const uint32_t n0 = extract_words64<STAGE>(s_bits, w, key_hi, od, s_stage, lane);
        extract_words64<STAGE>(s_bits, w + 64, key_hi, od + n0, s_stage, lane);
    }
    return total;
}

// Extracts the `nwords` (multiple of 512) SMEM bitset words at s_bits[w0 ..)
// to o[0 ..) in order; returns the number of keys. 512-word steps: lane l
// owns words [16l, 16l+16) of a step (4 LDS.128 in a lane-rotated order, so
// the reads are bank-conflict free). An empty step costs ~40 instructions; a
// sparse step (<= 128 keys) writes each lane's keys straight to its output
// range, visiting only nonzero words; a denser step is extracted as four
// 128-word steps (per-warp stage, or word-by-word ballots when dense).
template <int STAGE>
__device__ __forceinline__ uint32_t extract_span512(uint32_t* s_bits, uint32_t w0, uint32_t nwords,
                                                    uint32_t key_hi, uint32_t* __restrict__ o,
                                                    uint32_t* s_stage, unsigned lane,
                                                    bool consume, uint32_t* gclear) {
    const uint4* s4 = reinterpret_cast<const uint4*>(s_bits);
    uint32_t total = 0;
    for (uint32_t st = 0; st < nwords; st += 512) {
        const uint32_t lw = w0 + st + 16 * lane;  // this lane's first word (SMEM index)
        uint32_t c = 0, nz = 0;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const uint32_t q = (static_cast<uint32_t>(s) + lane) & 3u;
            const uint4 v = s4[lw / 4 + q];
            c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
            nz |= ((v.x != 0u ? 1u : 0u) | (v.y != 0u ? 2u : 0u) | (v.z != 0u ? 4u : 0u) |
                   (v.w != 0u ? 8u : 0u)) << (4 * q);
            // gclear: the global copy of these words is consumed (zeroed)
            if (gclear && (v.x | v.y | v.z | v.w))
                *reinterpret_cast<uint4*>(gclear + lw + 4 * q) = make_uint4(0, 0, 0, 0);
        }
        const uint32_t incl = warp_incl_scan(c, lane);
        const uint32_t ctot = __shfl_sync(kFull, incl, 31);
        if (ctot == 0) continue;
        if (ctot <= 128u) {
            uint32_t* ol = o + total + (incl - c);
            while (nz) {
                const uint32_t j = static_cast<uint32_t>(__ffs(nz) - 1);
                nz &= nz - 1;
                uint32_t x = s_bits[lw + j];
                if (consume) s_bits[lw + j] = 0u;
                const uint32_t kb = key_hi + ((lw + j) << 5);
                while (x) {
                    const int bt = __ffs(x) - 1;
                    x &= x - 1;
                    __stcs(ol++, kb + static_cast<uint32_t>(bt));
                }
            }
            total += ctot;
            continue;
        }
        uint32_t* od = o + total;
#pragma unroll 1
        for (uint32_t sub = 0; sub < 512; sub += 128) {
            const uint32_t sw = w0 + st + sub;
            const uint4 v = s4[sw / 4 + lane];
            const uint32_t cl = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
            const uint32_t in2 = warp_incl_scan(cl, lane);
            const uint32_t ct = __shfl_sync(kFull, in2, 31);
            if (ct == 0) continue;
            if (ct <= static_cast<uint32_t>(STAGE)) {
                uint32_t p = in2 - cl;
                const uint32_t kb = key_hi + ((sw + 4 * lane) << 5);
                stage_bits(v.x, kb, p, s_stage);
                stage_bits(v.y, kb + 32, p, s_stage);
                stage_bits(v.z, kb + 64, p, s_stage);
                stage_bits(v.w, kb + 96, p, s_stage);
                drain_stage(s_stage, ct, od, lane);
                od += ct;
            } else if (ct > 2u * STAGE) {  // dense: word-by-word ballots
#pragma unroll 1
                for (uint32_t q = 0; q < 128; q += 32)
                    od += extract_words32<STAGE>(s_bits, sw + q, key_hi, od, s_stage, lane);
            } else {
                const uint32_t n0 = extract_words64<STAGE>(s_bits, sw, key_hi, od, s_stage, lane);
                od += n0 + extract_words64<STAGE>(s_bits, sw + 64, key_hi, od + n0, s_stage, lane);
            }
            if (consume && cl) reinterpret_cast<uint4*>(s_bits)[sw / 4 + lane] = make_uint4(0, 0, 0, 0);
        }
        total += ctot;
    }
    return total;
}

}  // namespace dev
}  // namespace bws_gpu
