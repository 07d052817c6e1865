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
constexpr int KF_CONS_WARPS = 4;
constexpr int KF_CONS = KF_CONS_WARPS * 32;   // consumer threads
constexpr int KF_PROD = KF_THREADS - KF_CONS;  // producer threads (28 warps)
constexpr int KF_PWARPS = KF_PROD / 32;
constexpr int KF_KPT = 8;
constexpr int KF_TILE = KF_PROD * KF_KPT;      // 7168 keys per producer tile
constexpr int KF_U = 4;                        // uint4 per consumer thread per round
constexpr uint32_t KF_RW = KF_CONS * KF_U * 4; // entries per consumer round
constexpr int KF_LOGC = 14;
constexpr uint32_t KF_C = 1u << KF_LOGC;       // ring entries per owner
constexpr int KF_STAGE = 640;                  // extraction stage keys per warp
static_assert(KF_C >= KF_RW + KF_TILE + 4 * 2, "ring too small for the deadlock-freedom bound");
static_assert(KF_MAXG <= KF_PROD, "one owner per producer thread");

constexpr std::size_t kCtrWords = 4 * KF_MAXG + 64;  // tail[2G], head[2G], sync[4], padding

constexpr int kBarProd = 1;
constexpr int kBarCons = 2;

__device__ __forceinline__ void bar_prod() {
    asm volatile("bar.sync %0, %1;" ::"n"(kBarProd), "n"(KF_PROD) : "memory");
}
__device__ __forceinline__ void bar_cons() {
    asm volatile("bar.sync %0, %1;" ::"n"(kBarCons), "n"(KF_CONS) : "memory");
}
// consumer barrier that also ORs a predicate over the consumer threads
__device__ __forceinline__ bool bar_cons_or(bool v) {
    uint32_t r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.u32 p, %1, 0;\n\t"
        "bar.red.or.pred q, %2, %3, p;\n\t"
        "selp.u32 %0, 1, 0, q;\n\t}"
        : "=r"(r)
        : "r"(static_cast<uint32_t>(v)), "n"(kBarCons), "n"(KF_CONS)
        : "memory");
    return r != 0;
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
__device__ __forceinline__ void st_release64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
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
__device__ __forceinline__ unsigned long long now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
constexpr unsigned long long kTimeoutNs = 2000000000ull;  // 2 s: a protocol fault, not a slow sort

// entries of a uint4 written in the lap of position q
__device__ __forceinline__ bool lap_valid(const uint4& v, uint32_t q) {
    const uint32_t par = (q >> KF_LOGC) & 1u;
    return par ? ((v.x & v.y & v.z & v.w) >> 31) != 0u : ((v.x | v.y | v.z | v.w) >> 31) == 0u;
}

}  // namespace

// Producer SMEM (after the bitset slice): TMA ring, sorted tile, 16 copies of
// every run start, counters, cached ring heads. Also the extraction stages.
constexpr std::size_t kf_prod_bytes() {
    return (2 * std::size_t(KF_TILE) + KF_TILE + 4 * std::size_t(KF_MAXG)) * 4 +  // ring + sorted
           16 * std::size_t(KF_MAXG) * 2 +                                        // start copies
           (std::size_t(KF_MAXG) + 1) * 4 + 2 * std::size_t(KF_MAXG) * 4;          // counts + heads
}
static_assert(kf_prod_bytes() >= std::size_t(32) * (KF_STAGE + KF_STAGE / 32) * 4, "stages fit");

std::size_t fused_smem_bytes(std::uint32_t slice_bits) { return slice_bits / 8 + kf_prod_bytes(); }

__global__ void __launch_bounds__(KF_THREADS, 1) fused_sort_kernel(FusedArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t G = gridDim.x, c = blockIdx.x;
    const uint32_t Sw = a.S >> 5;  // words per slice
    uint32_t* s_bits = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* s_ring = s_bits + Sw;                      // 2 x KF_TILE (TMA destination)
    uint32_t* s_sorted = s_ring + 2 * KF_TILE;           // KF_TILE + 4 * KF_MAXG
    uint16_t* s_start16 = reinterpret_cast<uint16_t*>(s_sorted + KF_TILE + 4 * KF_MAXG);
    uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_start16 + 16 * KF_MAXG);  // KF_MAXG + 1
    uint32_t* s_headc = s_cnt + KF_MAXG + 1;            // 2 x KF_MAXG (producers' view of heads)
    uint32_t* s_stage_all = s_ring;                      // extraction (after both passes)
    __shared__ __align__(8) unsigned long long s_bar[2];
    __shared__ unsigned long long s_scratch[33];
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_T;
    __shared__ unsigned long long s_base[2];
    __shared__ uint32_t s_bad;

    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t P = static_cast<uint32_t>(a.P);

    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        fence_mbar_init();
        s_bad = 0;
    }
    {
        uint4* b4 = reinterpret_cast<uint4*>(s_bits);
        for (uint32_t i = threadIdx.x; i < Sw / 4; i += KF_THREADS) b4[i] = make_uint4(0, 0, 0, 0);
    }
    for (uint32_t i = threadIdx.x; i <= G; i += KF_THREADS) s_cnt[i] = 0;
    for (uint32_t i = threadIdx.x; i < 2 * G; i += KF_THREADS) s_headc[i] = ld_acquire(a.head + i);
    __syncthreads();

    if (threadIdx.x < KF_PROD) {
        // ------------------------------------------------------------ producers
        const size_t vlo = a.ks.nv * c / G, vhi = a.ks.nv * (c + 1) / G;
        constexpr size_t kTileVec = KF_TILE / 4;
        const uint32_t ntiles = static_cast<uint32_t>((vhi - vlo + kTileVec - 1) / kTileVec);
        const uint32_t total_tiles = ntiles * P;
        const unsigned long long pol_first = l2_policy_evict_first();
        const unsigned long long pol_last = l2_policy_evict_last();
        auto load_tile = [&](uint32_t g) {  // one thread
            const size_t v0 = vlo + static_cast<size_t>(g % ntiles) * kTileVec;
            const size_t nvec = min(kTileVec, vhi - v0);
            fence_proxy_async_smem();
            tma_load_bytes_hint(s_ring + (g & 1u) * KF_TILE, a.ks.body + v0, static_cast<unsigned>(nvec * 16),
                                &s_bar[g & 1u], pol_first);
        };
        if (threadIdx.x == 0)
            for (uint32_t g = 0; g < 2 && g < total_tiles; ++g) load_tile(g);

        bool timed_out = false;
        // space in ring ri for a run ending at position `end`: wait for the consumer
        auto wait_space = [&](uint32_t ri, uint32_t end) {
            if (static_cast<int32_t>(end - s_headc[ri]) <= static_cast<int32_t>(KF_C)) return;
            const unsigned long long t0 = now_ns();
            unsigned ns = 32;
            for (;;) {
                const uint32_t h = ld_acquire(a.head + ri);
                s_headc[ri] = h;
                if (static_cast<int32_t>(end - h) <= static_cast<int32_t>(KF_C)) return;
                if (timed_out || now_ns() - t0 > kTimeoutNs || *reinterpret_cast<volatile uint32_t*>(a.sync + 3)) {
                    timed_out = true;
                    atomicExch(a.sync + 3, 1u);
                    return;
                }
                __nanosleep(ns);
                ns = ns < 1024 ? 2 * ns : ns;
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
            const uint32_t ri = (p & 1u) * G + o;
            const uint32_t claim = atomicAdd(a.tail + ri, 4u);
            wait_space(ri, claim + 4);
            uint32_t* ring = a.rings + static_cast<size_t>(ri) * KF_C;
            for (uint32_t i = 0; i < 4; ++i) {
                const uint32_t q = claim + i;
                __stcg(ring + (q & (KF_C - 1)), r | (((q >> KF_LOGC) & 1u) << 31));
            }
        };

        const uint32_t nb = G;  // owners; slot nb = not in this pass / out of range
        // owner o's counter, claim and stores belong to producer thread o * ostride
        // (spread over the producer warps, in owner order for the run-start scan)
        const uint32_t ostride = KF_PROD / G;
        bool stores_pending = false;
        uint32_t g = 0;
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
                const uint32_t* buf = s_ring + slot * KF_TILE;
                const size_t v0 = vlo + static_cast<size_t>(t) * kTileVec;
                const uint32_t nvec = static_cast<uint32_t>(min(kTileVec, vhi - v0));
                mbar_wait(&s_bar[slot], (g >> 1) & 1u);

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
                bar_prod();  // A: counts complete; the TMA slot is free
                if (threadIdx.x == KF_PROD - 32 && g + 2 < total_tiles) load_tile(g + 2);
                // padded run starts (multiples of 4), claims, lap parity of each claim
                uint32_t claim = 0, cb = 0, st = 0;
                const uint32_t o_mine = threadIdx.x % ostride == 0 ? threadIdx.x / ostride : nb;
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
                        claim = atomicAdd(a.tail + (p & 1u) * G + o, local);
                        const uint32_t v16 = st | (((claim >> KF_LOGC) & 1u) << 15);
                        uint4 rep;
                        rep.x = rep.y = rep.z = rep.w = v16 | (v16 << 16);
                        reinterpret_cast<uint4*>(s_start16 + 16 * o)[0] = rep;
                        reinterpret_cast<uint4*>(s_start16 + 16 * o)[1] = rep;
                    }
                }
                if (stores_pending) {  // the previous tile's stores must have read s_sorted
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    stores_pending = false;
                }
                bar_prod();  // B
#pragma unroll
                for (int q = 0; q < KF_KPT; ++q) {
                    const uint32_t o = rb[q] >> 16;
                    if (o != nb) {
                        const uint32_t v16 = s_start16[(o << 4) | (lane & 15u)];
                        s_sorted[(v16 & 0x7fffu) + (rb[q] & 0xffffu)] = k[q] | ((v16 >> 15) << 31);
                    }
                }
                fence_proxy_async_smem();
                bar_prod();  // C
                if (cb) {
                    const uint32_t o = o_mine;
                    const uint32_t pc = (cb + 3u) & ~3u;
                    for (uint32_t i = cb; i < pc; ++i) s_sorted[st + i] = s_sorted[st];  // pad with a repeat
                    const uint32_t pos0 = claim & (KF_C - 1);
                    const uint32_t len1 = min(pc, KF_C - pos0);
                    // a run crossing the ring end continues in the next lap: flip its lap bit
                    for (uint32_t i = len1; i < pc; ++i) s_sorted[st + i] ^= 0x80000000u;
                    fence_proxy_async_smem();
                    const uint32_t ri = (p & 1u) * G + o;
                    wait_space(ri, claim + pc);
                    uint32_t* ring = a.rings + static_cast<size_t>(ri) * KF_C;
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                                     ring + pos0),
                                 "r"(smem_u32(s_sorted + st)), "r"(len1 * 4), "l"(pol_last)
                                 : "memory");
                    if (pc > len1)
                        asm volatile(
                            "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(ring),
                            "r"(smem_u32(s_sorted + st + len1)), "r"((pc - len1) * 4), "l"(pol_last)
                            : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    stores_pending = true;
                }
            }
            // pass done: this CTA's runs are written; count it for the consumers
            if (stores_pending) {
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                stores_pending = false;
            }
            bar_prod();
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(a.sync + p, 1u);
            }
        }
    } else {
        // ------------------------------------------------------------ consumers
        const uint32_t ct = threadIdx.x - KF_PROD;
        for (uint32_t p = 0; p < P; ++p) {
            const uint32_t ri = (p & 1u) * G + c;
            const uint32_t* ring = a.rings + static_cast<size_t>(ri) * KF_C;
            uint32_t h = ld_acquire(a.head + ri);  // this CTA is the ring's only consumer
            uint32_t T = 0;
            bool tknown = false;
            const unsigned long long t0 = now_ns();
            bool abort = false;
            for (;;) {
                uint4 v[KF_U];
                uint32_t q[KF_U];
#pragma unroll
                for (int u = 0; u < KF_U; ++u) {
                    q[u] = h + 4u * (ct + static_cast<uint32_t>(u) * KF_CONS);
                    v[u] = (tknown && static_cast<int32_t>(q[u] - T) >= 0) ? make_uint4(0, 0, 0, 0)
                                                                             : ld_ring(ring + (q[u] & (KF_C - 1)));
                }
#pragma unroll
                for (int u = 0; u < KF_U; ++u) {
                    unsigned ns = 32;
                    int spins = 0;
                    for (;;) {
                        if (tknown && static_cast<int32_t>(q[u] - T) >= 0) break;  // never written
                        if (lap_valid(v[u], q[u])) {
                            const uint32_t e[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const uint32_t r = e[i] & 0x7fffffffu;
                                atomicOr(s_bits + (r >> 5), 1u << (r & 31));
                            }
                            break;
                        }
                        if (!tknown && (++spins & 3) == 0 && ld_acquire(a.sync + p) >= G) {
                            T = ld_acquire(a.tail + ri);
                            tknown = true;
                            continue;
                        }
                        if (abort || now_ns() - t0 > kTimeoutNs ||
                            *reinterpret_cast<volatile uint32_t*>(a.sync + 3)) {
                            abort = true;
                            atomicExch(a.sync + 3, 1u);
                            break;
                        }
                        __nanosleep(ns);
                        ns = ns < 512 ? 2 * ns : ns;
                        v[u] = ld_ring(ring + (q[u] & (KF_C - 1)));
                    }
                }
                if (tknown) s_T = T;
                const bool any_known = bar_cons_or(tknown);
                const bool any_abort = bar_cons_or(abort);
                if (any_known && !tknown) {
                    T = s_T;
                    tknown = true;
                }
                h += KF_RW;
                const bool fin = tknown && static_cast<int32_t>(h - T) >= 0;
                if (ct == 0) st_release(a.head + ri, fin ? T : h);
                if (fin || any_abort) break;
            }
            bar_cons();
            // the pass's popcount, published for every CTA's output offsets
            {
                uint32_t cnt = 0;
                const uint4* b4 = reinterpret_cast<const uint4*>(s_bits);
                for (uint32_t i = ct; i < Sw / 4; i += KF_CONS) {
                    const uint4 w = b4[i];
                    cnt += __popc(w.x) + __popc(w.y) + __popc(w.z) + __popc(w.w);
                }
                cnt = __reduce_add_sync(kFull, cnt);
                if (lane == 0) s_warp[warp] = cnt;
                bar_cons();
                if (ct == 0) {
                    uint32_t tot = 0;
                    for (int w = 0; w < KF_CONS_WARPS; ++w) tot += s_warp[KF_PWARPS + w];
                    st_release64(a.counts + p * G + c, (1ull << 63) | tot);
                }
            }
            if (p + 1 < P) {  // keep the pass-0 slice for the end; clear for pass 1
                uint4* b4 = reinterpret_cast<uint4*>(s_bits);
                uint4* g4 = reinterpret_cast<uint4*>(a.saved + static_cast<size_t>(c) * Sw);
                for (uint32_t i = ct; i < Sw / 4; i += KF_CONS) {
                    __stcg(g4 + i, b4[i]);
                    b4[i] = make_uint4(0, 0, 0, 0);
                }
                bar_cons();
            }
        }
    }
    __syncthreads();

    // ---------------------------------------------------------------- offsets
    if (warp == 0) {
        // publish the bad-key count with the counts, then read every CTA's
        if (lane == 0) st_release64(a.counts + 2 * G + c, (1ull << 63) | s_bad);
        unsigned long long before[2] = {0, 0}, tot[2] = {0, 0}, bad = 0;
        const unsigned long long t0 = now_ns();
        for (uint32_t i = lane; i < 3 * G; i += 32) {
            if (P == 1 && i >= G && i < 2 * G) continue;  // no pass 1
            unsigned long long w;
            unsigned ns = 32;
            for (;;) {
                w = ld_acquire64(a.counts + i);
                if (w >> 63) break;
                if (now_ns() - t0 > kTimeoutNs || *reinterpret_cast<volatile uint32_t*>(a.sync + 3)) {
                    atomicExch(a.sync + 3, 1u);
                    w = 1ull << 63;
                    break;
                }
                __nanosleep(ns);
                ns = ns < 512 ? 2 * ns : ns;
            }
            const unsigned long long val = w & ~(1ull << 63);
            const uint32_t pp = i / G, cc = i % G;
            if (pp < 2) {
                tot[pp] += val;
                if (cc < c) before[pp] += val;
            } else {
                bad += val;
            }
        }
#pragma unroll
        for (int pp = 0; pp < 2; ++pp) {
            for (int off = 16; off; off >>= 1) {
                tot[pp] += __shfl_xor_sync(kFull, tot[pp], off);
                before[pp] += __shfl_xor_sync(kFull, before[pp], off);
            }
        }
        for (int off = 16; off; off >>= 1) bad += __shfl_xor_sync(kFull, bad, off);
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
        uint32_t cw = 0;
        {
            const uint4* s4 = reinterpret_cast<const uint4*>(s_bits);
            for (uint32_t i = lane; i < seg_words / 4; i += 32) {
                const uint4 v = s4[seg / 4 + i];
                cw += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
            }
            cw = __reduce_add_sync(kFull, cw);
        }
        if (lane == 0) s_warp[warp] = cw;
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
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(a.sync + 2, 1u) == G - 1) {  // last CTA out: reset the per-launch counters
            a.sync[0] = 0;
            a.sync[1] = 0;
            for (uint32_t i = 0; i < 3 * G; ++i) a.counts[i] = 0;
            a.sync[2] = 0;
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

std::size_t fused_state_bytes(int sms) {
    return 2 * static_cast<std::size_t>(sms) * KF_C * 4 +  // rings
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
    const std::size_t ring_bytes = 2 * static_cast<std::size_t>(sms) * KF_C * 4;
    cudaError_t err = cudaMemsetAsync(s, 0xff, ring_bytes, stream);  // lap bit 1: nothing written in lap 0
    if (err != cudaSuccess) return err;
    return cudaMemsetAsync(s + ring_bytes, 0, fused_state_bytes(sms) - ring_bytes, stream);
}

cudaError_t launch_fused_sort(const KeySplit& ks, std::uint64_t key_range, std::uint32_t key_lo,
                              std::uint32_t* out, Ctrl* ctrl, void* state, std::uint32_t* saved,
                              const FusedPlan& plan, cudaStream_t stream) {
    if (!plan.ok) return cudaErrorInvalidValue;
    unsigned char* s = static_cast<unsigned char*>(state);
    const std::size_t ring_bytes = 2 * static_cast<std::size_t>(plan.G) * KF_C * 4;
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
    a.tail = ctr;                 // 2G
    a.head = ctr + 2 * KF_MAXG;   // 2G
    a.sync = ctr + 4 * KF_MAXG;   // done[0], done[1], exit, error
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
