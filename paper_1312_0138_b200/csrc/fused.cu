// KF: the whole sort in ONE persistent kernel for key ranges whose bitset
// fits in the SMs' shared memory in at most two passes (M <= ~2^28 on a
// 148-SM B200: C1, C2). SURVEY.md §8(a) G2+G3 fused; §8(d) bytes.
//
// Why: the bucketed pipeline (bucket.cu KB3 -> KB4) moves every key through
// HBM twice (16n bytes) because KB4 needs a bucket's keys complete before it
// can build the bucket's bitset. Here the bitset of a pass is split into one
// slice per SM, held in that SM's shared memory for the whole pass, and keys
// travel from the SM that reads them to the SM that owns their slice through
// small per-owner ring buffers that stay in the 126 MB L2:
//
//   producer warps  stream the CTA's share of the keys (TMA ring), counting-
//                   sort each tile by owner in SMEM, claim a run in every
//                   owner's ring (one global atomicAdd per non-empty owner)
//                   and write each run with one cp.async.bulk store;
//   consumer warps  poll the CTA's own ring and OR each entry into the SMEM
//                   bitset slice (atomicOr, no global atomics per key);
//   end             every CTA publishes its popcounts, reads the others'
//                   (all CTAs are co-resident: cooperative launch), and
//                   extracts its slices straight to the output at its prefix.
//
// HBM traffic: P reads of the keys (P = passes, 1 or 2) + one write of the
// output = 4n(P + 1) bytes (C2: 12n instead of the bucketed 16n; C1: 8n in
// one launch instead of K2 + K3). Ring traffic (write + read of every key)
// stays in L2; its lines are reused lap after lap.
//
// Ring protocol. Ring (set s, owner o) has C = 2^KF_LOGC entries; tail[s][o]
// counts claimed entries and head[s][o] consumed ones, both monotonic mod 2^32
// across launches (the ring memory persists, initialised to 0xFFFFFFFF). An
// entry is the key's offset inside the owner's slice (< 2^24) with bit 31 =
// the parity of its lap, (position >> KF_LOGC) & 1, so a consumer recognises a
// written entry by its lap bit alone: no reset writes, no per-run flags, and a
// run torn by a bulk store in flight is simply not yet valid. Producers wait
// before storing until claim + len - head <= C. Pass p uses ring set p & 1, so
// a producer already in pass 1 never mixes entries into a ring its consumer
// is still draining for pass 0. A consumer learns the final tail of a pass
// when all G producers have counted themselves done for it (their claims
// precede that count). Deadlock freedom: a consumer waits only for entries
// below head + RW; any run claimed below that point ends below head + RW +
// KF_TILE + 4 <= head + C, so its producer never waits for space.
//
// Passes: with P == 2 the keys are read twice; pass p keeps keys in
// [p H, (p + 1) H), H = G S. At the end of pass 0 the consumer saves its
// slice to global memory (L2-resident, S/8 bytes per SM) and clears it;
// extraction of both passes happens at the end with all 32 warps.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_util.cuh"
#include "kernels.h"

namespace bws_gpu {
using namespace dev;

namespace {

constexpr int KF_THREADS = 1024;
constexpr int KF_CONS_WARPS = 8;
constexpr int KF_CONS = KF_CONS_WARPS * 32;    // consumer threads
constexpr int KF_PROD = KF_THREADS - KF_CONS;  // producer threads (24 warps)
constexpr int KF_PWARPS = KF_PROD / 32;
constexpr int KF_KPT = 16;
constexpr int KF_TILE = KF_PROD * KF_KPT;      // 12288 keys per producer tile
constexpr int KF_REG = KF_TILE + 4 * KF_MAXG;  // words per tile region (runs padded to 4)
constexpr int KF_NSUB = KF_CONS_WARPS;         // sub-rings per owner: one per consumer warp
constexpr int KF_LOGC = 12;
constexpr uint32_t KF_C = 1u << KF_LOGC;       // entries per sub-ring
constexpr uint32_t KF_CHUNK = 512;             // entries per consumer-warp step (4 uint4 per lane)
constexpr uint32_t KF_WINDOW = 2 * KF_CHUNK;   // entries a consumer warp waits on at once
constexpr uint32_t KF_PIECE = 1024;            // max entries per producer store
constexpr int KF_STAGE = 640;                  // extraction stage keys per warp
constexpr uint32_t KF_MARK = 0x40000000u;      // end-of-pass marker | producer CTA (data entries < 2^24)
static_assert(KF_C >= KF_WINDOW + KF_PIECE, "sub-ring too small for the deadlock-freedom bound");
static_assert(KF_MAXG <= KF_PROD, "one owner per producer thread");

constexpr std::size_t kRingSets = 2;
constexpr std::size_t kCtrWords = 2 * kRingSets * KF_MAXG * KF_NSUB + 64;  // tail, head, sync, trace ctl

constexpr int kBarProd = 1;
constexpr int kBarCons = 2;

__device__ __forceinline__ void bar_prod() {
    asm volatile("bar.sync %0, %1;" ::"n"(kBarProd), "n"(KF_PROD) : "memory");
}
__device__ __forceinline__ void bar_cons() {
    asm volatile("bar.sync %0, %1;" ::"n"(kBarCons), "n"(KF_CONS) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// the published counts carry no other data: relaxed stores (no release fence)
__device__ __forceinline__ void st_relaxed64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// ring entries are read from L2 (another SM wrote them)
__device__ __forceinline__ uint4 ld_ring(const uint32_t* p) {
    uint4 v;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
constexpr unsigned long long kTimeoutNs = 2000000000ull;  // 2 s: a protocol fault, not a slow sort

// lap parity bit of ring position q (bit 31 of an entry written there)
__device__ __forceinline__ uint32_t lap_bit(uint32_t q) { return ((q >> KF_LOGC) & 1u) << 31; }
// all four entries of the uint4 at position q written in q's lap
__device__ __forceinline__ bool written(const uint4& v, uint32_t q) {
    return lap_bit(q) ? ((v.x & v.y & v.z & v.w) >> 31) != 0u : ((v.x | v.y | v.z | v.w) >> 31) == 0u;
}

// Phase trace (BITSORT_KF_TRACE): per CTA, globaltimer at phase ends + spin counts.
enum : int { kTrStart, kTrProd0, kTrCons0, kTrProd1, kTrCons1, kTrCounts, kTrEnd, kTrProdSpin, kTrConsSpin,
              kTrPhase0, kTrN = kTrPhase0 + 6 };  // + producer thread 0's clocks: wait, rank, A, scan, scatter, store
// producer phase clocks in the trace: build with -DKF_PHASE_CLOCKS (costs registers)
#ifdef KF_PHASE_CLOCKS
__device__ __forceinline__ unsigned long long clk() { return clock64(); }
#define KF_PH(i, v) (ph[i] += (v))
#else
__device__ __forceinline__ unsigned long long clk() { return 0; }
#define KF_PH(i, v) ((void)0)
#endif
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

}  // namespace

// Producer SMEM (after the bitset slice): TMA ring, sorted tile, 16 copies of
// every run start, counters, cached sub-ring heads; the extraction stages
// reuse it after both passes.
constexpr std::size_t kf_prod_only_bytes() {
    return 2 * std::size_t(KF_REG) * 4 +                                           // two tile regions
           16 * std::size_t(KF_MAXG) * 2 +                                        // start copies
           (std::size_t(KF_MAXG) + 1) * 4 + 2 * std::size_t(KF_MAXG) * 4;          // counts + heads
}
constexpr std::size_t kf_stage_bytes() { return std::size_t(32) * (KF_STAGE + KF_STAGE / 32) * 4; }
constexpr std::size_t kf_prod_bytes() {
    return kf_prod_only_bytes() > kf_stage_bytes() ? kf_prod_only_bytes() : kf_stage_bytes();
}

std::size_t fused_smem_bytes(std::uint32_t slice_bits) { return slice_bits / 8 + kf_prod_bytes(); }

__global__ void __launch_bounds__(KF_THREADS, 1) fused_sort_kernel(FusedArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t G = gridDim.x, c = blockIdx.x;
    const uint32_t Sw = a.S >> 5;  // words per slice
    uint32_t* s_bits = reinterpret_cast<uint32_t*>(smem_raw);
    // two tile regions: tile g arrives in region g & 1 (TMA), its keys go to
    // registers, and the same region then holds the tile sorted by owner until
    // its bulk stores have read it (while tile g + 1 arrives in the other)
    uint32_t* s_ring = s_bits + Sw;                      // 2 x KF_REG
    uint16_t* s_start16 = reinterpret_cast<uint16_t*>(s_ring + 2 * KF_REG);
    uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_start16 + 16 * KF_MAXG);  // KF_MAXG + 1
    uint32_t* s_headc = s_cnt + KF_MAXG + 1;            // 2 x KF_MAXG: heads of this CTA's sub-rings
    uint32_t* s_stage_all = s_ring;                      // extraction (after both passes)
    __shared__ __align__(8) unsigned long long s_bar[2];
    __shared__ unsigned long long s_scratch[33];
    __shared__ uint32_t s_warp[32];
    __shared__ unsigned long long s_base[2];
    __shared__ uint32_t s_bad;
    __shared__ uint32_t s_cons_cnt[KF_CONS_WARPS];
    __shared__ uint32_t s_mk[2 * KF_CONS_WARPS];
    __shared__ unsigned long long s_spin[2];

    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t P = static_cast<uint32_t>(a.P);
    const uint32_t sub = c % KF_NSUB;  // the sub-ring this CTA writes in every owner's ring
    auto ring_index = [&](uint32_t p, uint32_t o, uint32_t sr) { return ((p & 1u) * G + o) * KF_NSUB + sr; };
    unsigned long long* tr = a.trace ? a.trace + static_cast<size_t>(c) * kTrN : nullptr;
    if (tr && threadIdx.x == 0) tr[kTrStart] = now_ns();

    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        fence_mbar_init();
        s_bad = 0;
        s_spin[0] = s_spin[1] = 0;
    }
    if (!a.gbits) {  // ring mode (KD overwrites its slice from the global bitset)
        uint4* b4 = reinterpret_cast<uint4*>(s_bits);
        for (uint32_t i = threadIdx.x; i < Sw / 4; i += KF_THREADS) b4[i] = make_uint4(0, 0, 0, 0);
        for (uint32_t i = threadIdx.x; i <= G; i += KF_THREADS) s_cnt[i] = 0;
        for (uint32_t i = threadIdx.x; i < 2 * G; i += KF_THREADS)
            s_headc[i] = ld_relaxed(a.head + ring_index(i / G, i % G, sub));
    }
    __syncthreads();

    if (a.gbits) {
        // ------------------------------------------------ direct mode (KD)
        // small sorts: every thread ORs its keys straight into the global
        // bitset (L2-resident; one RED per key), a grid barrier, then every
        // CTA takes its slice of the bitset into SMEM (and zeroes it, so the
        // cached bitset stays all-zero) for the common count/extract tail
        const size_t vlo = a.ks.nv * c / G, vhi = a.ks.nv * (c + 1) / G;
        uint32_t bad = 0;
        auto put = [&](uint32_t k) {
            const uint32_t x = (k ^ a.ks.xr) - a.lo;
            if (x > a.range_m1) {
                ++bad;
                return;
            }
            atomicOr(a.gbits + (x >> 5), 1u << (x & 31));
        };
        for (size_t v = vlo + threadIdx.x; v < vhi; v += KF_THREADS) {
            const uint4 q = ld_na(a.ks.body + v);
            put(q.x);
            put(q.y);
            put(q.z);
            put(q.w);
        }
        if (threadIdx.x == 0) {
            if (c == 0)
                for (int i = 0; i < a.ks.n_head; ++i) put(a.ks.head[i]);
            if (c == G - 1)
                for (int i = 0; i < a.ks.n_tail; ++i) put(a.ks.tail[i]);
        }
        if (bad) atomicAdd(&s_bad, bad);
        __syncthreads();
        if (threadIdx.x == 0) {  // grid barrier (all CTAs are co-resident)
            __threadfence();
            atomicAdd(a.sync + 0, 1u);
            const unsigned long long t0 = now_ns();
            while (ld_relaxed(a.sync + 0) < G) {
                if (now_ns() - t0 > kTimeoutNs) {
                    atomicExch(a.sync + 3, 1u);
                    break;
                }
            }
            __threadfence();
            if (tr) tr[kTrProd0] = now_ns();
        }
        __syncthreads();
        uint4* g4 = reinterpret_cast<uint4*>(a.gbits + static_cast<size_t>(c) * Sw);
        uint4* b4 = reinterpret_cast<uint4*>(s_bits);
        uint32_t cnt = 0;
        for (uint32_t i = threadIdx.x; i < Sw / 4; i += KF_THREADS) {
            const uint4 w = __ldcg(g4 + i);
            b4[i] = w;
            if (w.x | w.y | w.z | w.w) __stcg(g4 + i, make_uint4(0, 0, 0, 0));
            cnt += __popc(w.x) + __popc(w.y) + __popc(w.z) + __popc(w.w);
        }
        cnt = __reduce_add_sync(kFull, cnt);
        if (lane == 0) s_warp[warp] = cnt;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
            for (int w = 0; w < KF_THREADS / 32; ++w) tot += s_warp[w];
            st_relaxed64(a.counts + c, (1ull << 63) | tot);
            if (tr) tr[kTrCons0] = now_ns();
        }
    } else if (threadIdx.x < KF_PROD) {
        // ------------------------------------------------------------ producers
        const size_t vlo = a.ks.nv * c / G, vhi = a.ks.nv * (c + 1) / G;
        constexpr size_t kTileVec = KF_TILE / 4;
        const uint32_t ntiles = static_cast<uint32_t>((vhi - vlo + kTileVec - 1) / kTileVec);
        const uint32_t total_tiles = ntiles * P;
        const unsigned long long pol_first = l2_policy_evict_first();
        auto load_tile = [&](uint32_t g) {  // one thread
            const size_t v0 = vlo + static_cast<size_t>(g % ntiles) * kTileVec;
            const size_t nvec = min(kTileVec, vhi - v0);
            fence_proxy_async_smem();
            tma_load_bytes_hint(s_ring + (g & 1u) * KF_REG, a.ks.body + v0, static_cast<unsigned>(nvec * 16),
                                &s_bar[g & 1u], pol_first);
        };
        if (threadIdx.x == 0)
            if (total_tiles > 0) load_tile(0);

        bool timed_out = false;
        unsigned long long spins = 0;
        // space in sub-ring (p, o) for entries up to position `end`: wait for its consumer
        auto wait_space = [&](uint32_t p, uint32_t o, uint32_t end) {
            uint32_t& hc = s_headc[(p & 1u) * G + o];
            if (static_cast<int32_t>(end - hc) <= static_cast<int32_t>(KF_C)) return;
            const uint32_t* hp = a.head + ring_index(p, o, sub);
            const unsigned long long t0 = now_ns();
            for (;;) {
                const uint32_t h = ld_relaxed(hp);
                hc = h;
                if (static_cast<int32_t>(end - h) <= static_cast<int32_t>(KF_C)) return;
                ++spins;
                if (timed_out || now_ns() - t0 > kTimeoutNs || ((spins & 255) == 0 && ld_relaxed(a.sync + 3))) {
                    timed_out = true;
                    atomicExch(a.sync + 3, 1u);
                    return;
                }
            }
        };
        // one key outside the 16-byte body (<= 3 per end of the array): a
        // padded run of four copies, plain stores
        auto put_single = [&](uint32_t p, uint32_t k) {
            const uint32_t x = (k ^ a.ks.xr) - a.lo;
            if (x > a.range_m1) {
                if (p == 0) atomicAdd(&s_bad, 1u);
                return;
            }
            const uint32_t pp = P == 2 && x >= a.H ? 1u : 0u;
            if (pp != p) return;
            const uint32_t xp = x - p * a.H;
            const uint32_t o = __umulhi(xp >> 12, a.mag);
            const uint32_t r = xp - o * a.S;
            const uint32_t claim = atomicAdd(a.tail + ring_index(p, o, sub), 4u);
            wait_space(p, o, claim + 4);
            uint32_t* ring = a.rings + static_cast<size_t>(ring_index(p, o, sub)) * KF_C;
            for (uint32_t i = 0; i < 4; ++i) __stcg(ring + ((claim + i) & (KF_C - 1)), r | lap_bit(claim + i));
        };

        const uint32_t nb = G;  // owners; slot nb = not in this pass / out of range
        // owner o's counter, claim and stores belong to producer thread o * ostride
        // (spread over the producer warps, in owner order for the run-start scan)
        const uint32_t ostride = KF_PROD / G;
        const uint32_t o_mine = threadIdx.x % ostride == 0 ? threadIdx.x / ostride : nb;
        uint32_t g = 0;
        unsigned long long ph[6] = {0, 0, 0, 0, 0, 0};
        for (uint32_t p = 0; p < P; ++p) {
            const uint32_t plo = p * a.H;
            if (threadIdx.x == 0) {
                if (c == 0)
                    for (int i = 0; i < a.ks.n_head; ++i) put_single(p, a.ks.head[i]);
                if (c == G - 1)
                    for (int i = 0; i < a.ks.n_tail; ++i) put_single(p, a.ks.tail[i]);
            }
            for (uint32_t t = 0; t < ntiles; ++t, ++g) {
                const uint32_t slot = g & 1u;
                uint32_t* buf = s_ring + slot * KF_REG;
                const size_t v0 = vlo + static_cast<size_t>(t) * kTileVec;
                const uint32_t nvec = static_cast<uint32_t>(min(kTileVec, vhi - v0));
                // this tile's view of its owner's sub-ring head, loaded now and
                // used at copy time (its latency hides behind the tile's work)
                const uint32_t hpre = o_mine < nb ? ld_relaxed(a.head + ring_index(p, o_mine, sub)) : 0u;
                unsigned long long c0 = clk();
                mbar_wait(&s_bar[slot], (g >> 1) & 1u);
                unsigned long long c1 = clk();
                KF_PH(0, c1 - c0);

                uint32_t k[KF_KPT];  // offset inside the owner's slice
                uint32_t rb[KF_KPT]; // owner << 16 | rank
                uint32_t bad = 0;
#pragma unroll
                for (int j = 0; j < KF_KPT / 4; ++j) {
                    const uint32_t vi = j * KF_PROD + threadIdx.x;
                    const bool in = vi < nvec;
                    const uint4 v = in ? reinterpret_cast<const uint4*>(buf)[vi] : make_uint4(0, 0, 0, 0);
                    const uint32_t kk[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t x = (kk[q] ^ a.ks.xr) - a.lo;
                        const bool ok = in && x <= a.range_m1;
                        bad += (in && !ok) ? 1u : 0u;
                        const uint32_t pp = P == 2 && x >= a.H ? 1u : 0u;
                        const uint32_t xp = x - plo;
                        const uint32_t o = __umulhi(xp >> 12, a.mag);
                        const bool mine = ok && pp == p;
                        k[4 * j + q] = xp - o * a.S;
                        rb[4 * j + q] = mine ? o : nb;
                    }
                }
                if (p == 0 && bad) atomicAdd(&s_bad, bad);
                // ranks: one SMEM atomic per key, or one per warp step when all of
                // the warp's keys go to one owner (sorted or clustered input)
                {
                    uint32_t omin = 0xffffffffu, omax = 0;
#pragma unroll
                    for (int q = 0; q < KF_KPT; ++q) {
                        omin = min(omin, rb[q]);
                        omax = max(omax, rb[q]);
                    }
                    omin = __reduce_min_sync(kFull, omin);
                    omax = __reduce_max_sync(kFull, omax);
                    if (omin == omax) {
                        if (omin != nb) {
                            uint32_t base = 0;
                            if (lane == 0) base = atomicAdd(s_cnt + omin, 32u * KF_KPT);
                            base = __shfl_sync(kFull, base, 0) + lane * KF_KPT;
#pragma unroll
                            for (int q = 0; q < KF_KPT; ++q) rb[q] = (omin << 16) | (base + q);
                        } else {
#pragma unroll
                            for (int q = 0; q < KF_KPT; ++q) rb[q] = nb << 16;
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < KF_KPT; ++q)
                            rb[q] = (rb[q] << 16) | (rb[q] != nb ? atomicAdd(s_cnt + rb[q], 1u) : 0u);
                    }
                }
                c0 = clk();
                KF_PH(1, c0 - c1);
                bar_prod();  // A: counts complete; this tile's keys are in registers
                c1 = clk();
                KF_PH(2, c1 - c0);
                if (threadIdx.x == KF_PROD - 32 && g + 1 < total_tiles) load_tile(g + 1);
                // padded run starts (multiples of 4) and the claims (consumed after the scatter)
                uint32_t claim = 0, cb = 0, st = 0;
                {
                    const uint32_t o = o_mine;
                    if (o < nb) {
                        cb = s_cnt[o];
                        s_cnt[o] = 0;
                    }
                    const uint32_t local = (cb + 3u) & ~3u;
                    const uint32_t incl = warp_incl_scan(local, lane);
                    if (lane == 31) s_scratch[warp] = incl;
                    bar_prod();
                    const uint32_t w = lane < KF_PWARPS ? static_cast<uint32_t>(s_scratch[lane]) : 0u;
                    const uint32_t wi = warp_incl_scan(w, lane);
                    st = __shfl_sync(kFull, wi - w, warp) + (incl - local);
                    if (cb) {
                        claim = atomicAdd(a.tail + ring_index(p, o, sub), local);
                        uint4 rep;
                        rep.x = rep.y = rep.z = rep.w = st | (st << 16);
                        reinterpret_cast<uint4*>(s_start16 + 16 * o)[0] = rep;
                        reinterpret_cast<uint4*>(s_start16 + 16 * o)[1] = rep;
                    }
                }
                bar_prod();  // B
                c0 = clk();
                KF_PH(3, c0 - c1);
#pragma unroll
                for (int q = 0; q < KF_KPT; ++q) {
                    const uint32_t o = rb[q] >> 16;
                    if (o != nb) buf[s_start16[(o << 4) | (lane & 15u)] + (rb[q] & 0xffffu)] = k[q];
                }
                fence_proxy_async_smem();
                bar_prod();  // C
                c1 = clk();
                KF_PH(4, c1 - c0);
                // every run of this warp's owners, copied by the whole warp with
                // 16-byte stores (lap bit applied), in pieces of <= KF_PIECE
                // entries each written once its consumer has made room for it
                const uint32_t pc = (cb + 3u) & ~3u;
                for (uint32_t i = cb; i < pc; ++i) buf[st + i] = buf[st];  // pad with a repeat
                if (o_mine < nb) {
                    uint32_t& hc = s_headc[(p & 1u) * G + o_mine];
                    if (static_cast<int32_t>(hpre - hc) > 0) hc = hpre;
                }
                __syncwarp();
                for (unsigned todo = __ballot_sync(kFull, cb != 0); todo; todo &= todo - 1) {
                    const int src = __ffs(todo) - 1;
                    const uint32_t r_st = __shfl_sync(kFull, st, src), r_pc = __shfl_sync(kFull, pc, src);
                    const uint32_t r_claim = __shfl_sync(kFull, claim, src), r_o = __shfl_sync(kFull, o_mine, src);
                    uint32_t* ring = a.rings + static_cast<size_t>(ring_index(p, r_o, sub)) * KF_C;
                    for (uint32_t off = 0; off < r_pc; off += KF_PIECE) {
                        const uint32_t len = min(KF_PIECE, r_pc - off);
                        if (lane == 0) wait_space(p, r_o, r_claim + off + len);
                        __syncwarp();
                        for (uint32_t u = lane; u < len / 4; u += 32) {
                            uint4 v = reinterpret_cast<const uint4*>(buf + r_st + off)[u];
                            const uint32_t q = r_claim + off + 4 * u;
                            const uint32_t lb = lap_bit(q);
                            v.x |= lb;
                            v.y |= lb;
                            v.z |= lb;
                            v.w |= lb;
                            __stcg(reinterpret_cast<uint4*>(ring + (q & (KF_C - 1))), v);
                        }
                    }
                }
                KF_PH(5, clk() - c1);
            }
            // pass done: an end marker after this CTA's last claim in every
            // owner's sub-ring (its consumer stops once it has seen the
            // markers of all its producers and everything before them)
            bar_prod();  // every claim of this pass (incl. thread 0's single keys) precedes the markers
            if (o_mine < nb) {
                const uint32_t ri = ring_index(p, o_mine, sub);
                const uint32_t claim = atomicAdd(a.tail + ri, 4u);
                wait_space(p, o_mine, claim + 4);
                const uint32_t m = KF_MARK | c | lap_bit(claim);
                __stcg(reinterpret_cast<uint4*>(a.rings + static_cast<size_t>(ri) * KF_C + (claim & (KF_C - 1))),
                       make_uint4(m, m, m, m));
            }
            if (tr && threadIdx.x == 0) tr[p == 0 ? kTrProd0 : kTrProd1] = now_ns();
        }
        if (tr && threadIdx.x == 0)
            for (int i = 0; i < 6; ++i) tr[kTrPhase0 + i] = ph[i];
    } else {
        // ------------------------------------------------------------ consumers
        // consumer warp w drains sub-ring w of this CTA's ring: 512-entry steps
        // (lane l: uint4 l + 32 i, i < 4), the next step's loads in flight
        const uint32_t cw = warp - KF_PWARPS;
        // producers writing this warp's sub-ring: CTAs c' with c' % KF_NSUB == cw
        const uint32_t expect = (G > cw) ? (G - cw + KF_NSUB - 1) / KF_NSUB : 0u;
        volatile uint32_t* mk_cnt = s_mk + 2 * cw;      // markers seen (this pass)
        volatile uint32_t* mk_max = s_mk + 2 * cw + 1;  // last marker's offset from h0, + 1
        bool abort = false;
        uint32_t polls = 0;
        for (uint32_t p = 0; p < P; ++p) {
            const uint32_t ri = ring_index(p, c, cw);
            uint32_t* ring = a.rings + static_cast<size_t>(ri) * KF_C;
            const uint32_t h0 = ld_acquire(a.head + ri);  // this warp is the sub-ring's only consumer
            if (lane == 0) {
                *mk_cnt = 0;
                *mk_max = 0;
            }
            __syncwarp();
            const unsigned long long t0 = now_ns();
            uint4 va[4], vb[4];
            auto pos_of = [&](uint32_t step, int i) { return step * KF_CHUNK + 4u * (lane + 32u * i); };
            auto issue = [&](uint32_t step, uint4 (&buf)[4]) {
#pragma unroll
                for (int i = 0; i < 4; ++i) buf[i] = ld_ring(ring + ((h0 + pos_of(step, i)) & (KF_C - 1)));
            };
            // drained: every producer's marker seen, and nothing is written past the last
            auto past_end = [&](uint32_t rel) { return *mk_cnt == expect && rel + 1 > *mk_max; };
            // consumes step `step` from cur; true when the pass is drained
            auto consume = [&](uint32_t step, uint4 (&cur)[4]) -> bool {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t rel = pos_of(step, i);
                    for (;;) {
                        if (written(cur[i], h0 + rel)) {
                            if (cur[i].x & KF_MARK) {
                                atomicMax(const_cast<uint32_t*>(mk_max), rel + 1);
                                __threadfence_block();
                                atomicAdd(const_cast<uint32_t*>(mk_cnt), 1u);
                            } else {
                                const uint32_t e[4] = {cur[i].x & 0x7fffffffu, cur[i].y & 0x7fffffffu,
                                                       cur[i].z & 0x7fffffffu, cur[i].w & 0x7fffffffu};
#pragma unroll
                                for (int j = 0; j < 4; ++j) atomicOr(s_bits + (e[j] >> 5), 1u << (e[j] & 31));
                            }
                            break;
                        }
                        if (past_end(rel)) break;  // never written
                        if (abort || now_ns() - t0 > kTimeoutNs || ((++polls & 255) == 0 && ld_relaxed(a.sync + 3))) {
                            abort = true;
                            atomicExch(a.sync + 3, 1u);
                            break;
                        }
                        cur[i] = ld_ring(ring + ((h0 + rel) & (KF_C - 1)));
                    }
                }
                __syncwarp();
                const bool any_abort = __any_sync(kFull, abort);
                const uint32_t next = (step + 1) * KF_CHUNK;
                const bool fin = *mk_cnt == expect;  // then the last marker lies in this or an earlier step
                // consumed (the reads have returned: a producer may now overwrite)
                if (lane == 0) st_relaxed(a.head + ri, h0 + (fin ? *mk_max + 3 : next));
                return fin || any_abort;
            };
            issue(0, va);
            issue(1, vb);
            for (uint32_t step = 0;; step += 2) {
                if (consume(step, va)) break;
                issue(step + 2, va);
                if (consume(step + 1, vb)) break;
                issue(step + 3, vb);
            }
            bar_cons();  // every sub-ring of this pass drained
            // the pass's popcount, published for every CTA's output offsets
            const uint32_t ct = threadIdx.x - KF_PROD;
            uint32_t cnt = 0;
            {
                const uint4* b4 = reinterpret_cast<const uint4*>(s_bits);
                for (uint32_t i = ct; i < Sw / 4; i += KF_CONS) {
                    const uint4 w = b4[i];
                    cnt += __popc(w.x) + __popc(w.y) + __popc(w.z) + __popc(w.w);
                }
            }
            cnt = __reduce_add_sync(kFull, cnt);
            if (lane == 0) s_cons_cnt[cw] = cnt;
            bar_cons();
            if (ct == 0) {
                uint32_t tot = 0;
                for (int w = 0; w < KF_CONS_WARPS; ++w) tot += s_cons_cnt[w];
                st_relaxed64(a.counts + p * G + c, (1ull << 63) | tot);
                if (tr) tr[p == 0 ? kTrCons0 : kTrCons1] = now_ns();
            }
            if (p + 1 < P) {  // keep the pass-0 slice for the end; clear for pass 1
                uint4* b4 = reinterpret_cast<uint4*>(s_bits);
                uint4* g4 = reinterpret_cast<uint4*>(a.saved + static_cast<size_t>(c) * Sw);
                for (uint32_t i = ct; i < Sw / 4; i += KF_CONS) {
                    __stcg(g4 + i, b4[i]);
                    b4[i] = make_uint4(0, 0, 0, 0);
                }
            }
            bar_cons();
        }
    }
    __syncthreads();

    // ---------------------------------------------------------------- offsets
    if (warp == 0) {
        if (tr && lane == 0) tr[kTrProdSpin] = now_ns();  // (slot reused: offsets phase entered)
        // publish the bad-key count with the counts, then read every CTA's
        if (lane == 0) st_relaxed64(a.counts + 2 * G + c, (1ull << 63) | s_bad);
        unsigned long long before[2] = {0, 0}, tot[2] = {0, 0}, bad = 0;
        constexpr int kPer = (3 * KF_MAXG + 31) / 32;
        unsigned long long w[kPer];
        uint32_t missing = 0;  // bit j: word lane + 32 j not yet published
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const uint32_t i = lane + 32u * j;
            const bool want = i < 3 * G && !(P == 1 && i >= G && i < 2 * G);  // P == 1: no pass 1
            w[j] = want ? ld_relaxed64(a.counts + i) : (1ull << 63);
        }
        {
            const unsigned long long t0 = now_ns();
            for (;;) {
                missing = 0;
#pragma unroll
                for (int j = 0; j < kPer; ++j) missing |= (w[j] >> 63) ? 0u : (1u << j);
                if (!missing) {
                    if (tr && lane == 0) tr[kTrConsSpin] = now_ns();  // (slot reused: every count seen)
                    break;
                }
                if (now_ns() - t0 > kTimeoutNs) {
                    atomicExch(a.sync + 3, 1u);
                    break;
                }
#pragma unroll
                for (int j = 0; j < kPer; ++j)
                    if (missing & (1u << j))
                        w[j] = ld_relaxed64(a.counts + lane + 32u * j);
            }
        }
        unsigned long long t0s = 0, t1s = 0, b0s = 0, b1s = 0;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const uint32_t i = lane + 32u * j;
            if (i >= 3 * G || (P == 1 && i >= G && i < 2 * G)) continue;
            const unsigned long long val = w[j] & ~(1ull << 63);
            const uint32_t pp = i / G, cc = i % G;
            const bool lt = cc < c;
            if (pp == 0) {
                t0s += val;
                b0s += lt ? val : 0ull;
            } else if (pp == 1) {
                t1s += val;
                b1s += lt ? val : 0ull;
            } else {
                bad += val;
            }
        }
        for (int off = 16; off; off >>= 1) {
            t0s += __shfl_xor_sync(kFull, t0s, off);
            t1s += __shfl_xor_sync(kFull, t1s, off);
            b0s += __shfl_xor_sync(kFull, b0s, off);
            b1s += __shfl_xor_sync(kFull, b1s, off);
            bad += __shfl_xor_sync(kFull, bad, off);
        }
        before[0] = b0s;
        before[1] = b1s;
        tot[0] = t0s;
        tot[1] = t1s;
        if (lane == 0) {
            s_base[0] = before[0];
            s_base[1] = tot[0] + before[1];
            if (c == 0) {
                a.ctrl->total = tot[0] + tot[1];
                a.ctrl->bad_keys = static_cast<uint32_t>(bad);
                a.ctrl->ticket = 0;
                a.ctrl->done_ctas = 0;
                a.ctrl->error = *reinterpret_cast<volatile uint32_t*>(a.sync + 3);
            }
            if (tr) {
                tr[kTrCounts] = now_ns();
            }
        }
    }
    __syncthreads();

    // ------------------------------------------------------------- extraction
    uint32_t* s_stage = s_stage_all + warp * (KF_STAGE + KF_STAGE / 32);
    const uint32_t seg_words = Sw / 32;  // multiple of 128
    const bool failed = *reinterpret_cast<volatile uint32_t*>(a.sync + 3) != 0;
    for (int pi = static_cast<int>(P) - 1; pi >= 0 && !failed; --pi) {
        const uint32_t p = static_cast<uint32_t>(pi);
        if (p + 1 < P) {  // the saved pass-0 slice back into SMEM
            __syncthreads();
            const uint4* g4 = reinterpret_cast<const uint4*>(a.saved + static_cast<size_t>(c) * Sw);
            uint4* b4 = reinterpret_cast<uint4*>(s_bits);
            for (uint32_t i = threadIdx.x; i < Sw / 4; i += KF_THREADS) b4[i] = __ldcg(g4 + i);
            __syncthreads();
        }
        const uint32_t seg = warp * seg_words;
        uint32_t cwd = 0;
        {
            const uint4* s4 = reinterpret_cast<const uint4*>(s_bits);
            for (uint32_t i = lane; i < seg_words / 4; i += 32) {
                const uint4 v = s4[seg / 4 + i];
                cwd += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
            }
            cwd = __reduce_add_sync(kFull, cwd);
        }
        if (lane == 0) s_warp[warp] = cwd;
        __syncthreads();
        const uint32_t wv = s_warp[lane];
        const uint32_t wi = warp_incl_scan(wv, lane);
        const uint32_t wprefix = __shfl_sync(kFull, wi - wv, warp);
        uint32_t* o = a.out + s_base[p] + wprefix;
        const uint32_t key_hi = a.lo + p * a.H + c * a.S;
        extract_seg128<KF_STAGE>(s_bits, seg, seg_words, key_hi, o, s_stage, lane);
    }

    // --------------------------------------------------------------- teardown
    __syncthreads();
    if (warp == 0) {
        uint32_t last = 0;
        if (lane == 0) {
            if (tr) tr[kTrEnd] = now_ns();
            __threadfence();
            last = atomicAdd(a.sync + 2, 1u) == G - 1;
        }
        if (__shfl_sync(kFull, last, 0)) {  // last CTA out: reset the per-launch counters
            for (uint32_t i = lane; i < 3 * G; i += 32) a.counts[i] = 0;
            if (lane == 0) {
                a.sync[0] = 0;
                a.sync[1] = 0;
                a.sync[2] = 0;
            }
            __threadfence();
        }
    }
}

FusedPlan plan_fused(std::uint64_t key_range, int sms, std::size_t smem_limit) {
    FusedPlan pl;
    if (sms <= 0 || sms > KF_MAXG || key_range == 0) return pl;
    for (int P = 1; P <= 2; ++P) {
        const std::uint64_t per = (key_range + static_cast<std::uint64_t>(P) * sms - 1) / (static_cast<std::uint64_t>(P) * sms);
        const std::uint64_t S = ((per + (1u << 17) - 1) >> 17) << 17;
        if (S >= (std::uint64_t(1) << 24)) continue;
        if (fused_smem_bytes(static_cast<std::uint32_t>(S)) > smem_limit) continue;
        const std::uint64_t H = S * static_cast<std::uint64_t>(sms);
        if (P == 2 && H >= (std::uint64_t(1) << 32)) continue;
        pl.ok = true;
        pl.P = P;
        pl.G = sms;
        pl.S = static_cast<std::uint32_t>(S);
        pl.H = P == 2 ? static_cast<std::uint32_t>(H) : 0xffffffffu;
        const std::uint64_t sq = S >> 12;
        pl.mag = static_cast<std::uint32_t>(((std::uint64_t(1) << 32) + sq - 1) / sq);
        pl.smem = fused_smem_bytes(pl.S);
        return pl;
    }
    return pl;
}

std::size_t fused_ring_bytes(int sms) { return kRingSets * static_cast<std::size_t>(sms) * KF_NSUB * KF_C * 4; }

std::size_t fused_state_bytes(int sms) {
    return fused_ring_bytes(sms) +
           kCtrWords * 4 +                                  // counters (tail, head, sync)
           3 * static_cast<std::size_t>(KF_MAXG) * 8;       // counts
}

cudaError_t configure_fused(int device, LaunchGeometry* geo) {
    int sms = 0, optin = 0;
    cudaError_t err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (err != cudaSuccess) return err;
    err = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (err != cudaSuccess) return err;
    int coop = 0;
    err = cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
    if (err != cudaSuccess) return err;
    const std::size_t limit = static_cast<std::size_t>(optin) - 2048;  // static SMEM
    err = cudaFuncSetAttribute(fused_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(limit));
    if (err != cudaSuccess) return err;
    geo->fused_ctas = coop ? sms : 0;
    geo->fused_smem_limit = limit;
    return cudaSuccess;
}

cudaError_t init_fused_state(void* state, int sms, cudaStream_t stream) {
    unsigned char* s = static_cast<unsigned char*>(state);
    const std::size_t ring_bytes = fused_ring_bytes(sms);
    cudaError_t err = cudaMemsetAsync(s, 0xff, ring_bytes, stream);  // every entry EMPTY
    if (err != cudaSuccess) return err;
    return cudaMemsetAsync(s + ring_bytes, 0, fused_state_bytes(sms) - ring_bytes, stream);
}

cudaError_t launch_fused_sort(const KeySplit& ks, std::uint64_t key_range, std::uint32_t key_lo,
                              std::uint32_t* out, Ctrl* ctrl, void* state, std::uint32_t* saved,
                              const FusedPlan& plan, cudaStream_t stream, unsigned long long* trace,
                              std::uint32_t* gbits) {
    if (!plan.ok) return cudaErrorInvalidValue;
    unsigned char* s = static_cast<unsigned char*>(state);
    const std::size_t ring_bytes = fused_ring_bytes(plan.G);
    uint32_t* ctr = reinterpret_cast<uint32_t*>(s + ring_bytes);
    FusedArgs a;
    a.ks = ks;
    a.range_m1 = static_cast<std::uint32_t>(key_range - 1);
    a.lo = key_lo;
    a.H = plan.H;
    a.S = plan.S;
    a.mag = plan.mag;
    a.P = plan.P;
    a.out = out;
    a.ctrl = ctrl;
    a.rings = reinterpret_cast<uint32_t*>(s);
    a.tail = ctr;                                    // per sub-ring claim counters
    a.head = ctr + kRingSets * KF_MAXG * KF_NSUB;    // per sub-ring consumed counters
    a.sync = ctr + 2 * kRingSets * KF_MAXG * KF_NSUB;  // done[0], done[1], exit, error
    a.trace = trace;
    a.gbits = plan.P == 1 ? gbits : nullptr;
    a.counts = reinterpret_cast<unsigned long long*>(s + ring_bytes + kCtrWords * 4);
    a.saved = saved;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(plan.G));
    cfg.blockDim = dim3(KF_THREADS);
    cfg.dynamicSmemBytes = plan.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fused_sort_kernel, a);
}

}  // namespace bws_gpu
