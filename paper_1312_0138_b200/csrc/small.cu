// KS: a whole small sort in ONE cooperative launch, bitset words kept in
// registers (SURVEY.md §8(a) G2+G3 fused for sorts below the bucketed
// threshold; §7.7 "one persistent kernel: scatter, grid barrier, scan").
//
// For n < 2^21 keys the two-launch direct path (K2 scatter, K3 lookback scan)
// is latency-bound: C1 (10^6 keys, M = 2^24) spends ~14 us in K2 and ~19 us in
// K3, most of it launch latency, the 64-tile lookback chain and tile setup.
// KS does the same work with two grid-wide waits and no shared-memory bitset:
//
//   A  every thread ORs its keys into the cached global bitset (all-zero
//      between sorts, L2-resident: one RED per key; the CTA's slice of it is
//      prefetched into L2 first) and counts them per owning slice in a
//      shared-memory histogram, which the CTA then adds to a global one (G
//      REDs); keys >= the range are counted as bad;
//   B  grid barrier (all CTAs are co-resident: cooperative launch, one CTA
//      per SM; a monotonic 64-bit arrival counter, no reset: the launch
//      generation is the counter / G read at kernel start, so nothing
//      launch-specific comes from the host and captured graphs replay);
//   C  CTA c takes slice c of the bitset — thread t the `per` consecutive
//      16-byte vectors [t per, (t + 1) per) of it, kept in registers when
//      per == 1 — and popcounts it; its output offset is the histogram's
//      prefix (keys of the slices before c), known right after the barrier:
//      no second grid-wide wait for the other CTAs' popcounts. For distinct
//      keys the two agree; repeated keys only leave gaps in the output, and
//      ctrl->total (the sum of popcounts) reports them as usual;
//   E  a block scan of the thread counts, then every thread writes the keys of
//      its vectors to its output slots — through an SMEM stage and coalesced
//      stores when the CTA has at most 10240 keys, else directly — and zeroes
//      the nonzero words, so the cached bitset is all-zero again.
//
// HBM traffic: 4n (keys) + 4n (output); the bitset stays in L2. CTA 0 zeroes
// the control block before the barrier (no memset precedes the launch); the
// histogram has two parities (generation & 1) and each launch zeroes the next one's. A wait
// that exceeds 2 s is a protocol fault: ctrl->error, and the host resets the
// state (capi.cpp read_ctrl).
#include <cuda_runtime.h>

#include <cstdint>

#include "device_util.cuh"
#include "kernels.h"

namespace bws_gpu {
using namespace dev;

namespace {

constexpr int KS_THREADS = 1024;
constexpr uint32_t KS_STAGE = 10240;  // keys a CTA stages in SMEM for coalesced output stores
constexpr unsigned long long kKsTimeoutNs = 2000000000ull;

__device__ __forceinline__ unsigned long long ks_ld_acquire64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ks_ld_relaxed64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void ks_st_relaxed64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ks_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

}  // namespace

__global__ void __launch_bounds__(KS_THREADS, 1) small_sort_kernel(SmallArgs a) {
    __shared__ uint32_t s_hist[KS_MAXG];  // keys of this CTA per owning slice
    __shared__ uint32_t s_stage[KS_STAGE];
    __shared__ uint32_t s_warp[KS_THREADS / 32];
    __shared__ uint32_t s_bad;
    __shared__ uint32_t s_max;
    __shared__ uint32_t s_fail;
    __shared__ unsigned long long s_base;
    __shared__ unsigned long long s_gen;
    const uint32_t G = gridDim.x, c = blockIdx.x;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long* tr = a.trace ? a.trace + static_cast<size_t>(c) * KS_TRACE_WORDS : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = ks_now();
    for (uint32_t i = threadIdx.x; i < G; i += KS_THREADS) s_hist[i] = 0;
    if (threadIdx.x == 0) {
        s_bad = 0;
        s_max = 0;
        s_fail = 0;
        s_base = 0;
        // The launch generation, from the arrival counter itself: every earlier
        // launch added exactly G, and a CTA reads it before it arrives, so all
        // CTAs of this launch see a value in [gen G, (gen + 1) G). Nothing
        // launch-specific comes from the host: a captured graph replays correctly.
        s_gen = ks_ld_relaxed64(a.sync) / G;
        if (c == 0) {  // the whole control block: no memset before the launch
            Ctrl r = {};
            *a.ctrl = r;
        }
    }
    __syncthreads();
    const unsigned long long gen = s_gen;
    uint32_t* ghist = a.ghist + (gen & 1u) * KS_MAXG;          // this launch's slice histogram
    if (threadIdx.x == 0) a.ghist[((gen & 1u) ^ 1u) * KS_MAXG + c] = 0;  // the next launch's: zeroed here

    // ------------------------------------------------------------ A: scatter
    // the CTA's slice of the bitset into L2 first (cold after an L2 flush: a
    // RED to a sector that is not resident waits for its DRAM fetch)
    const uint32_t per = a.per;
    if (a.prefetch) {
        const uint32_t v0 = c * per * KS_THREADS + threadIdx.x * per;
        for (uint32_t i = 0; i < per; i += 8) {  // 128-byte lines
            const uint32_t v = v0 + i;
            if (v < a.total_v)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const uint4*>(a.gbits) + v));
        }
    }
    {
        const size_t vlo = a.ks.nv * c / G, vhi = a.ks.nv * (c + 1) / G;
        uint32_t bad = 0, kmax = 0;
        auto put = [&](uint32_t k) {
            const uint32_t x = (k ^ a.ks.xr) - a.lo;
            kmax = max(kmax, k ^ a.ks.xr);  // like K0 / K2: the host tracks the range of unhinted sorts
            if (x > a.range_m1) {
                ++bad;
                return;
            }
            atomicOr(a.gbits + (x >> 5), 1u << (x & 31));
            atomicAdd(s_hist + (per == 1 ? x >> 17 : __umulhi(x >> 17, a.per_magic)), 1u);  // (x >> 17) / per
        };
        for (size_t v = vlo + threadIdx.x; v < vhi; v += 2 * KS_THREADS) {
            const bool two = v + KS_THREADS < vhi;
            const uint4 q0 = ld_na(a.ks.body + v);
            const uint4 q1 = two ? ld_na(a.ks.body + v + KS_THREADS) : make_uint4(0, 0, 0, 0);
            put(q0.x);
            put(q0.y);
            put(q0.z);
            put(q0.w);
            if (two) {
                put(q1.x);
                put(q1.y);
                put(q1.z);
                put(q1.w);
            }
        }
        if (threadIdx.x == 0) {
            if (c == 0)
                for (int i = 0; i < a.ks.n_head; ++i) put(a.ks.head[i]);
            if (c == G - 1)
                for (int i = 0; i < a.ks.n_tail; ++i) put(a.ks.tail[i]);
        }
        bad = __reduce_add_sync(kFull, bad);
        if (lane == 0 && bad) atomicAdd(&s_bad, bad);
        kmax = __reduce_max_sync(kFull, kmax);
        if (lane == 0 && kmax) atomicMax(&s_max, kmax);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < G; i += KS_THREADS) {
        const uint32_t h = s_hist[i];
        if (h) atomicAdd(ghist + i, h);
    }
    __syncthreads();
    if (tr && threadIdx.x == 0) tr[1] = ks_now();

    // ------------------------------------------------------- B: grid barrier
    // (the grid.sync() pattern: the CTA barrier orders every thread's REDs
    // before thread 0's fence, which is cumulative; one fence per CTA instead
    // of one per thread — the per-thread fences were 3.4 stalled warps per
    // issued instruction in the KS ncu capture)
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(a.sync, 1ull);
        const unsigned long long target = (gen + 1ull) * G;
        const unsigned long long t0 = ks_now();
        uint32_t spins = 0;
        while (ks_ld_acquire64(a.sync) < target) {
            if ((++spins & 1023u) == 0 && ks_now() - t0 > kKsTimeoutNs) {
                s_fail = 1;
                break;
            }
        }
        __threadfence();
        if (tr) tr[2] = ks_now();
    }
    __syncthreads();
    if (s_fail) {
        if (threadIdx.x == 0) atomicExch(&a.ctrl->error, 1u);
        return;
    }

    // ---------------- C: the CTA's slice counted; its output offset from the
    // slice histogram (keys before slice c; equal to the set bits before it
    // when the keys are distinct — with repeats the offsets only leave gaps,
    // and the total below, a popcount, reports them)
    const uint32_t slice_v = per * KS_THREADS;
    const uint32_t v_begin = c * slice_v + threadIdx.x * per;  // first vector of this thread
    uint4* g4 = reinterpret_cast<uint4*>(a.gbits);
    uint32_t before_cta = 0;
    for (uint32_t i = threadIdx.x; i < c; i += KS_THREADS) before_cta += __ldcg(ghist + i);
    uint32_t cnt = 0;
    uint4 w0 = make_uint4(0, 0, 0, 0);  // the thread's vector when per == 1
    if (per == 1) {
        if (v_begin < a.total_v) w0 = __ldcg(g4 + v_begin);
        cnt = __popc(w0.x) + __popc(w0.y) + __popc(w0.z) + __popc(w0.w);
    } else {
        for (uint32_t i = 0; i < per; ++i) {
            const uint32_t v = v_begin + i;
            if (v >= a.total_v) break;
            const uint4 w = __ldcg(g4 + v);
            cnt += __popc(w.x) + __popc(w.y) + __popc(w.z) + __popc(w.w);
        }
    }
    if (threadIdx.x < ((c + 31u) & ~31u)) {  // whole warps that hold histogram entries
        before_cta = __reduce_add_sync(kFull, before_cta);
        if (lane == 0 && before_cta) atomicAdd(&s_base, static_cast<unsigned long long>(before_cta));
    }
    const uint32_t incl = warp_incl_scan(cnt, lane);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint32_t before_thread;  // keys of this CTA before this thread's vectors
    uint32_t cta_total;
    {
        const uint32_t wv = s_warp[lane];
        const uint32_t wi = warp_incl_scan(wv, lane);
        before_thread = __shfl_sync(kFull, wi - wv, warp) + (incl - cnt);
        cta_total = __shfl_sync(kFull, wi, 31);
    }
    if (threadIdx.x == 0) {  // (after the barrier: CTA 0 zeroed the control block before it arrived)
        if (cta_total) atomicAdd(&a.ctrl->total, static_cast<unsigned long long>(cta_total));
        if (s_bad) atomicAdd(&a.ctrl->bad_keys, s_bad);
        if (s_max) atomicMax(&a.ctrl->max_key, s_max);
    }
    const unsigned long long base = s_base;
    if (tr && threadIdx.x == 0) tr[3] = ks_now();

    // ---------------------------------------------------------- E: extraction
    // A thread's keys are few and its neighbours' slots lie apart: direct
    // stores would cost a sector per lane. Up to KS_STAGE keys per CTA go
    // through SMEM and leave with coalesced stores; denser slices store directly.
    const bool staged = cta_total <= KS_STAGE;
    if (cnt != 0) {
        uint32_t* o = staged ? s_stage + before_thread : a.out + base + before_thread;
        auto emit = [&](uint32_t w, uint32_t key_hi) {
            while (w) {
                const uint32_t b = __ffs(w) - 1;
                w &= w - 1;
                *o++ = (key_hi + b + a.lo) ^ a.ks.xr;
            }
        };
        const uint4 zero = make_uint4(0, 0, 0, 0);
        if (per == 1) {
            const uint32_t kb = v_begin * 128u;
            emit(w0.x, kb);
            emit(w0.y, kb + 32u);
            emit(w0.z, kb + 64u);
            emit(w0.w, kb + 96u);
            __stcg(g4 + v_begin, zero);
        } else {
            for (uint32_t i = 0; i < per; ++i) {
                const uint32_t v = v_begin + i;
                if (v >= a.total_v) break;
                const uint4 w = __ldcg(g4 + v);
                if ((w.x | w.y | w.z | w.w) == 0u) continue;
                const uint32_t kb = v * 128u;
                emit(w.x, kb);
                emit(w.y, kb + 32u);
                emit(w.z, kb + 64u);
                emit(w.w, kb + 96u);
                __stcg(g4 + v, zero);
            }
        }
    }
    if (staged) {
        __syncthreads();
        uint32_t* o = a.out + base;
        for (uint32_t i = threadIdx.x; i < cta_total; i += KS_THREADS) o[i] = s_stage[i];
    }
    if (tr) {
        __syncwarp();
        if (lane == 0) atomicMax(tr + 5, ks_now());
    }
}

// The KS plan for a hinted sort: G CTAs, `per` vectors of 128 bits per thread.
// ok only for ranges a slice of which a CTA holds in <= KS_MAX_PER vectors per
// thread (2^27 keys on 148 SMs).
SmallPlan plan_small(std::uint64_t key_range, int ctas) {
    SmallPlan p;
    if (ctas <= 0 || ctas > KS_MAXG || key_range == 0 || key_range > (std::uint64_t(1) << 32)) return p;
    const std::uint64_t total_v = (key_range + 127) / 128;
    const std::uint64_t per = (total_v + static_cast<std::uint64_t>(ctas) * KS_THREADS - 1) /
                              (static_cast<std::uint64_t>(ctas) * KS_THREADS);
    if (per > KS_MAX_PER) return p;
    p.ok = true;
    p.G = ctas;
    p.per = static_cast<std::uint32_t>(per);
    p.total_v = static_cast<std::uint32_t>(total_v);
    return p;
}

std::size_t small_state_bytes() { return 64 + 2 * static_cast<std::size_t>(KS_MAXG) * 4; }

cudaError_t configure_small(int device, LaunchGeometry* geo) {
    int sms = 0, coop = 0;
    cudaError_t err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (err != cudaSuccess) return err;
    err = cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
    if (err != cudaSuccess) return err;
    geo->small_ctas = coop && sms <= KS_MAXG ? sms : 0;
    return cudaSuccess;
}

cudaError_t launch_small_sort(const KeySplit& ks, std::uint64_t key_range, std::uint32_t key_lo,
                              std::uint32_t* out, Ctrl* ctrl, void* state,
                              const SmallPlan& plan, std::uint32_t* gbits, cudaStream_t stream,
                              unsigned long long* trace, int prefetch) {
    if (!plan.ok) return cudaErrorInvalidValue;
    SmallArgs a;
    a.ks = ks;
    a.lo = key_lo;
    a.range_m1 = static_cast<std::uint32_t>(key_range - 1);
    a.gbits = gbits;
    a.per = plan.per;
    a.total_v = plan.total_v;
    a.out = out;
    a.ctrl = ctrl;
    a.sync = static_cast<unsigned long long*>(state);
    a.ghist = reinterpret_cast<std::uint32_t*>(static_cast<unsigned char*>(state) + 64);
    a.per_magic = static_cast<std::uint32_t>(((std::uint64_t(1) << 32) + plan.per - 1) / plan.per);
    a.trace = trace;
    a.prefetch = prefetch;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(plan.G));
    cfg.blockDim = dim3(KS_THREADS);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, small_sort_kernel, a);
}

}  // namespace bws_gpu
