// Bucketed bitset sort (sm_100a): the K2 scatter with SHARED-MEMORY STAGING
// made applicable to every input, including shuffled ones.
//
// Why: a random-address atomicOr (RED) to global memory costs one L2 request
// per key. Measured on B200 (profiles/r01_microbench_primitives.jsonl) that
// caps the direct scatter at ~188 G keys/s for an L2-resident bitset and
// ~25 G keys/s for a 512 MiB one, while shared-memory atomicOr runs at
// ~1.7 T keys/s. So the keys are first moved, with coalesced traffic, into
// key-range buckets whose bitset fits in SMEM (2^shift bits, shift <= 20):
//
//   KB1 bucket_hist      per-CTA histogram of bucket ids over a contiguous
//                        chunk of the keys                       (read 4n)
//   KB2 bucket_colscan   column prefix over CTAs -> each CTA's first slot
//                        in every bucket; bucket totals
//   KB3 bucket_partition per tile: SMEM counting sort by bucket, then
//                        coalesced run writes to the bucket slots (read 4n,
//                        write 4n)
//   KB4 bucket_sort      per bucket: SMEM bitset (atomicOr), popcount, and
//                        set-bit extraction straight to the output; the
//                        output offset of a bucket is the prefix of bucket
//                        totals, so no cross-CTA scan is needed (read 4n,
//                        write 4n)
//
// The global bitset is never materialised: 20n bytes of HBM traffic and no
// M-proportional term. Duplicate keys are detected by sum(popcount) < n.
#include "kernels.h"
#include "device_util.cuh"

#ifndef KB4_RING
#define KB4_RING 4  // packed-layout KB4: bulk-copy ring slots in the stage area (C5 KB4: 2 slots 830 us, 4 slots 816, 8 slots 849)
#endif

#include <cstdlib>
#include <string>

namespace bws_gpu {
namespace {

using namespace dev;

// Block-wide exclusive scan of `count` (<= MAX_BUCKETS) uint32 values in
// `vals` (SMEM), written as 64-bit prefixes to `out64` (SMEM or global) and
// returning the total. blockDim.x must be a multiple of 32; `scratch` holds
// 33 uint64.
__device__ unsigned long long block_exclusive_scan_u64(const uint32_t* vals, int count,
                                                       unsigned long long* out64,
                                                       unsigned long long* scratch) {
    const int per = (count + blockDim.x - 1) / blockDim.x;
    const int begin = threadIdx.x * per;
    unsigned long long local = 0;
    for (int i = 0; i < per; ++i)
        if (begin + i < count) local += vals[begin + i];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned long long o = __shfl_up_sync(kFull, incl, off);
        if (lane >= static_cast<unsigned>(off)) incl += o;
    }
    if (lane == 31) scratch[warp] = incl;
    __syncthreads();
    const int nwarps = blockDim.x >> 5;
    if (warp == 0) {
        unsigned long long w = lane < static_cast<unsigned>(nwarps) ? scratch[lane] : 0ull;
        unsigned long long wi = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned long long o = __shfl_up_sync(kFull, wi, off);
            if (lane >= static_cast<unsigned>(off)) wi += o;
        }
        if (lane < static_cast<unsigned>(nwarps)) scratch[lane] = wi - w;
        if (lane == 31) scratch[32] = wi;  // total (nwarps <= 32)
    }
    __syncthreads();
    unsigned long long run = scratch[warp] + (incl - local);
    const unsigned long long total = scratch[32];
    for (int i = 0; i < per; ++i) {
        if (begin + i < count) {
            out64[begin + i] = run;
            run += vals[begin + i];
        }
    }
    __syncthreads();
    return total;
}

// ---------------------------------------------------------------------------
// KB1/KB3 see the keys as a 16-byte-aligned body of nv uint4 split evenly
// over the P CTAs, plus <= 3 head keys (CTA 0) and <= 3 tail keys (CTA P-1),
// so both kernels assign every key to the same CTA.

// Slot of a key in KB1/KB3: its bucket, clamped to the spill slot `nb` for
// keys beyond the last bucket; padding lanes (`in` false) also spill. KB1 and
// KB3 apply the same rule, so slot counts always match. A key in
// [key_range, nb * width) (ranges that are not a multiple of the width) lands in the last bucket;
// KB1 counts it in ctrl->bad_keys exactly, and the host then rejects the sort.
__device__ __forceinline__ uint32_t bucket_id(uint32_t k, const BucketMap& m) {
    return __umulhi(((k - m.lo) >> m.ms) << 12, m.mq);
}
__device__ __forceinline__ uint32_t bucket_or_spill(uint32_t k, bool in, const BucketMap& m, int nb) {
    return in ? min(bucket_id(k, m), static_cast<uint32_t>(nb)) : static_cast<uint32_t>(nb);
}

// KB1: histogram of bucket ids over partition CTA c's share, computed by
// HIST_SPLIT CTAs per share (more loads in flight) that add into the zeroed,
// bucket-major H[b * P + c] (KB2 scans contiguous rows).
__global__ void __launch_bounds__(BUCKET_HIST_THREADS)
    bucket_hist_kernel(KeySplit ks, BucketMap bm, int nb, uint32_t limit, int check,
                       uint32_t* __restrict__ H, Ctrl* __restrict__ ctrl) {
    __shared__ uint32_t s_h[MAX_BUCKETS + 1];
    for (int b = threadIdx.x; b <= nb; b += blockDim.x) s_h[b] = 0;
    __syncthreads();
    const unsigned P = gridDim.x / HIST_SPLIT, c = blockIdx.x / HIST_SPLIT;
    const unsigned part = blockIdx.x % HIST_SPLIT;
    const size_t clo = ks.nv * c / P, chi = ks.nv * (c + 1) / P;
    const size_t vlo = clo + (chi - clo) * part / HIST_SPLIT;
    const size_t vhi = clo + (chi - clo) * (part + 1) / HIST_SPLIT;
    const unsigned lane = threadIdx.x & 31;
    uint32_t mx = 0, bad = 0;
    // largest key - lo that is in range and in a real bucket (fast path bound)
    const uint64_t bucket_end = static_cast<uint64_t>(nb) * bm.width;
    uint64_t fl = bucket_end - 1;
    if (check && limit - 1ull < fl) fl = limit - 1ull;
    const uint32_t fast_last = fl > 0xffffffffull ? 0xffffffffu : static_cast<uint32_t>(fl);
    constexpr int U = 4;  // uint4 per thread per step: 16 keys
    const size_t step = static_cast<size_t>(blockDim.x) * U;
    // software pipelined: the next step's loads are in flight while this
    // step's buckets are counted
    uint4 v[U];
    bool in[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const size_t i = vlo + static_cast<size_t>(u) * blockDim.x + threadIdx.x;
        in[u] = i < vhi;
        v[u] = in[u] ? __ldcs(ks.body + i) : make_uint4(0, 0, 0, 0);
    }
    for (size_t base = vlo; base < vhi; base += step) {
        uint4 vn[U];
        bool inn[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = base + step + static_cast<size_t>(u) * blockDim.x + threadIdx.x;
            inn[u] = i < vhi;
            vn[u] = inn[u] ? __ldcs(ks.body + i) : make_uint4(0, 0, 0, 0);
        }
        uint32_t bk[U * 4];
        uint32_t rmin = 0xffffffffu, rmax = 0;  // over key - lo
        bool all_in = true;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t kk[4] = {v[u].x ^ ks.xr, v[u].y ^ ks.xr, v[u].z ^ ks.xr, v[u].w ^ ks.xr};
            all_in &= in[u];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                bk[u * 4 + q] = kk[q];
                rmin = min(rmin, kk[q] - bm.lo);
                rmax = max(rmax, kk[q] - bm.lo);
            }
        }
        rmin = __reduce_min_sync(kFull, rmin);
        rmax = __reduce_max_sync(kFull, rmax);
        if (__all_sync(kFull, all_in) && rmax <= fast_last) {
            // every key in range and in a real bucket: no per-key checks
            mx = max(mx, rmax + bm.lo);
            const uint32_t blo = __umulhi((rmin >> bm.ms) << 12, bm.mq);
            if (blo == __umulhi((rmax >> bm.ms) << 12, bm.mq)) {
                // sorted / clustered input: one bucket for the whole warp step
                if (lane == 0) atomicAdd(s_h + blo, 32u * U * 4);
            } else {
#pragma unroll
                for (int q = 0; q < U * 4; ++q) atomicAdd(s_h + __umulhi(((bk[q] - bm.lo) >> bm.ms) << 12, bm.mq), 1u);
            }
        } else {
            uint32_t kmax = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t kq = bk[u * 4 + q];
                    kmax = max(kmax, in[u] ? kq : 0u);
                    bad += (check && in[u] && kq - bm.lo >= limit) ? 1u : 0u;
                    atomicAdd(s_h + bucket_or_spill(kq, in[u], bm, nb), 1u);
                }
            }
            mx = max(mx, kmax);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            v[u] = vn[u];
            in[u] = inn[u];
        }
    }
    if (threadIdx.x == 0 && part == 0) {  // misaligned head (share 0) / tail (last share)
        const uint32_t* extra = c == 0 ? ks.head : nullptr;
        int ne = c == 0 ? ks.n_head : 0;
        for (int pass = 0; pass < 2; ++pass) {
            for (int i = 0; i < ne; ++i) {
                const uint32_t e = extra[i] ^ ks.xr;
                atomicAdd(s_h + bucket_or_spill(e, true, bm, nb), 1u);
                mx = max(mx, e);
                bad += (check && e - bm.lo >= limit) ? 1u : 0u;
            }
            extra = c == P - 1 ? ks.tail : nullptr;
            ne = c == P - 1 ? ks.n_tail : 0;
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x)
        if (s_h[b]) atomicAdd(H + static_cast<size_t>(b) * P + c, s_h[b]);
    const uint32_t wm = __reduce_max_sync(kFull, mx);
    const uint32_t wb = __reduce_add_sync(kFull, bad);
    if (lane == 0) {
        if (wm) atomicMax(&ctrl->max_key, wm);
        if (wb) atomicAdd(&ctrl->bad_keys, wb);
    }
}

// KB2: one warp per bucket row: H[b][c] <- sum_{c' < c} H[b][c']; tot[b] <- row sum.
__global__ void bucket_colscan_kernel(uint32_t* __restrict__ H, int P, int nb,
                                      uint32_t* __restrict__ tot) {
    const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (b >= nb) return;
    const unsigned lane = threadIdx.x & 31;
    uint32_t* row = H + static_cast<size_t>(b) * P;
    const int per = (P + 31) / 32;
    const int begin = lane * per;
    uint32_t local = 0;
    for (int i = 0; i < per; ++i)
        if (begin + i < P) local += row[begin + i];
    uint32_t incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(kFull, incl, off);
        if (lane >= static_cast<unsigned>(off)) incl += o;
    }
    uint32_t run = incl - local;
    for (int i = 0; i < per; ++i) {
        if (begin + i < P) {
            const uint32_t v = row[begin + i];
            row[begin + i] = run;
            run += v;
        }
    }
    if (lane == 31) tot[b] = incl;
}

// KB2b (packed layout, i.e. wide sparse ranges with skewed bucket sizes such
// as C5's Zipf clusters): KB4's ticket order, largest buckets first (by
// power-of-two size class; the order inside a class is arbitrary). KB4 takes
// buckets by dynamic ticket, so a big bucket ticketed last would run alone
// at the end: measured C5 counts give a ~17% longer KB4 in index order than
// with this approximate longest-processing-time-first order.
// Run by one whole CTA (CTA 0 of the packed KB3, once the totals are known);
// order[nb] = 1 if the order is not the identity (KB4 reads it once).
__device__ void compute_kb4_order(const uint32_t* __restrict__ tot, int nb, uint32_t* __restrict__ order) {
    __shared__ uint32_t s_cls[33];
    __shared__ unsigned long long s_sum;
    __shared__ uint32_t s_max;
    if (threadIdx.x < 33) s_cls[threadIdx.x] = 0u;
    if (threadIdx.x == 0) {
        s_sum = 0;
        s_max = 0;
    }
    __syncthreads();
    unsigned long long sum = 0;
    uint32_t mx = 0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        const uint32_t c = tot[b];
        sum += c;
        mx = max(mx, c);
        atomicAdd(&s_cls[c ? 32 - __clz(c) : 0], 1u);
    }
    sum = __reduce_add_sync(0xffffffffu, static_cast<uint32_t>(sum));  // per-warp (< 2^32 keys)
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&s_sum, sum);
        atomicMax(&s_max, mx);
    }
    __syncthreads();
    // near-uniform sizes (C4: uniform draws) keep the index order: LPT buys
    // nothing there and the permuted order measured 3% slower
    if (static_cast<unsigned long long>(s_max) * nb <= 2 * s_sum) {
        if (threadIdx.x == 0) order[nb] = 0u;
        return;
    }
    if (threadIdx.x == 0) order[nb] = 1u;
    if (threadIdx.x == 0) {  // exclusive prefix in descending class order
        uint32_t run = 0;
        for (int k = 32; k >= 0; --k) {
            const uint32_t v = s_cls[k];
            s_cls[k] = run;
            run += v;
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        const uint32_t c = tot[b];
        order[atomicAdd(&s_cls[c ? 32 - __clz(c) : 0], 1u)] = static_cast<uint32_t>(b);
    }
}

// Chunked layout (packed sorts without KB1/KB2): a bucket's keys live in
// 2^chunk_shift-slot chunks of a pool. Chunk 0 of bucket b is pool chunk b
// (implicit); chunk j >= 1 is pool chunk chunk_tab[b * max_chunks + j] - 1
// (0: not allocated yet), allocated from pool chunk nb upwards. Tiles claim
// runs in a bucket with one atomicAdd on its fill counter, as in the slab
// layout; the claim that holds a chunk's first slot allocates it, others wait.
__device__ __forceinline__ uint32_t chunk_base(uint32_t id, uint32_t cs, uint32_t pad) {
    return (id << cs) + id * pad;  // (pool slots stay below 2^32: chunk_slots)
}
__device__ __forceinline__ uint32_t chunk_alloc(const SlabArgs& sa, int nb, uint32_t b, uint32_t j) {
    if (j == 0) return b;
    const uint32_t id = static_cast<uint32_t>(nb) + atomicAdd(sa.pool_next, 1u);
    atomicExch(sa.chunk_tab + static_cast<size_t>(b) * sa.max_chunks + j, id + 1u);
    return id;
}
__device__ __forceinline__ uint32_t chunk_get(const SlabArgs& sa, uint32_t b, uint32_t j) {
    if (j == 0) return b;
    const volatile uint32_t* t = sa.chunk_tab + static_cast<size_t>(b) * sa.max_chunks + j;
    uint32_t v = *t;
    if (v) return v - 1u;
    // the allocating claim precedes ours and every KB3 CTA is resident, so the
    // entry appears within microseconds; a protocol fault must not hang the
    // GPU: after 2 s the sort is flagged (Ctrl.error) and this run goes to chunk 0
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while ((v = *t) == 0u) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > 2000000000ull) {
            atomicExch(&sa.ctrl->error, 1u);
            return 0u;
        }
    }
    return v - 1u;
}

// Slab epilogue shared by the slab KB3 variants: folds the CTA's bad-key
// count into ctrl, and the last CTA to finish turns the fill counters into
// bucket totals (0 for an overflowed bucket: its keys are lost, so the sort
// sees fewer set bits than keys) and output offsets for KB4. `s_vals` holds
// nb uint32, `s_out64` nb uint64 (both SMEM).
__device__ __forceinline__ void slab_finish(const SlabArgs& sa, int nb, uint32_t bad, uint32_t kmax,
                                            uint32_t* s_vals, unsigned long long* s_out64,
                                            unsigned long long* s_scratch, uint32_t* s_last) {
    const unsigned lane = threadIdx.x & 31;
    const uint32_t wb = __reduce_add_sync(kFull, bad);
    if (lane == 0 && wb) atomicAdd(&sa.ctrl->bad_keys, wb);
    // the largest key seen (biased key, like K0's ctrl->max_key): the host
    // learns the true range of a sort that ran on a speculated one
    const uint32_t wm = __reduce_max_sync(kFull, kmax);
    if (lane == 0 && wm) atomicMax(&sa.ctrl->max_key, wm);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        *s_last = atomicAdd(&sa.ctrl->done_ctas, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!*s_last) return;
    __threadfence();
    // keys beyond the range were left out of the slabs: an in-place KB4 must
    // write nothing then (the caller redoes the sort from the intact keys)
    if (threadIdx.x == 0 && *reinterpret_cast<volatile const uint32_t*>(&sa.ctrl->bad_keys)) sa.ctrl->overflow = 1u;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        const uint32_t v = __ldcg(sa.gcnt + b);
        const bool ok = v <= sa.cap;
        if (!ok) sa.ctrl->overflow = 1u;  // some runs were dropped: the slab lost keys
        sa.tot[b] = ok ? v : 0u;  // slots KB4 reads
        s_vals[b] = ok ? (sa.gtrue ? __ldcg(sa.gtrue + b) : v) : 0u;  // keys, for the offsets
        sa.gcnt[b] = 0u;  // the counters start the next sort at zero
        if (sa.gtrue) sa.gtrue[b] = 0u;
    }
    __syncthreads();
    const unsigned long long total = block_exclusive_scan_u64(s_vals, nb, s_out64, s_scratch);
    for (int b = threadIdx.x; b < nb; b += blockDim.x) sa.g_base[b] = s_out64[b];
    if (threadIdx.x == 0) sa.g_base[nb] = total;
    if (sa.order) {  // chunked layout: KB4's ticket order from the totals
        __syncthreads();
        compute_kb4_order(sa.tot, nb, sa.order);
    }
}

// KB3: partition, one persistent CTA per SM. CTA c streams its share in
// 16384-key tiles through a double-buffered SMEM ring filled by TMA bulk copies
// (the next tile lands while the current one is processed). Per tile: ranks
// from SMEM atomicAdd on per-bucket counters (order inside a bucket is
// irrelevant to a bitset; out-of-range keys rank in the spill slot nb, which
// sorts last), an exclusive scan, an in-place counting-sort scatter into the
// tile buffer, then thread i stores sorted key i to parted[delta[bucket] + i]:
// consecutive threads write consecutive addresses within each bucket run.
// Slot positions are 32-bit (the bucketed path requires n < 2^32).
//
// Packed layout (SLAB false): a CTA's slots in every bucket come from KB1/KB2.
// Slab layout (SLAB true, see SlabArgs): each tile claims its run in every
// bucket with one global atomicAdd per non-empty bucket; the claims are
// issued before the tile's SMEM scatter and consumed after it, so their
// latency overlaps that work. The last CTA to finish turns the fill counters
// into bucket totals and output offsets for KB4.
// L2 hints (packed layout only, i.e. !SLAB): the key stream is loaded
// evict_first and the scattered run stores are evict_last, so the partially
// written 32-byte sectors of ~4096 short runs per tile stay in L2 until
// complete instead of being evicted half-written (measured: C5 KB3 1570 ->
// 1462 us, C4 116 -> 104 us; the slab layout's longer runs (C3) got slower).
template <int THREADS, int KPT, int MAXB, int LAYOUT>
__global__ void __launch_bounds__(THREADS, 1024 / THREADS)
    bucket_partition_kernel(KeySplit ks, BucketMap bm, int nb,
                            const uint32_t* __restrict__ H, const uint32_t* __restrict__ tot,
                            uint32_t* __restrict__ parted, unsigned long long* __restrict__ g_base,
                            SlabArgs sa) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // LAYOUT 0: packed (KB1/KB2 offsets); 1: slab (fixed per-bucket capacity,
    // claims); 2: chunked (claims into pool chunks allocated on first touch)
    constexpr bool SLAB = LAYOUT != 0;
    constexpr bool CHUNK = LAYOUT == 2;
    constexpr int kSlots = MAXB + 1;
    constexpr int TILE = THREADS * KPT;
    static_assert(!CHUNK || TILE <= 32767, "chunked crossings are 15-bit tile positions");
    constexpr int NWARPS = THREADS / 32;
    constexpr int PER_MAX = (kSlots + THREADS - 1) / THREADS;
    uint32_t* s_buf = reinterpret_cast<uint32_t*>(smem_raw);  // 2 x TILE
    uint32_t* s_cnt = s_buf + 2 * TILE;                   // keys per bucket in the tile
    uint32_t* s_start = s_cnt + kSlots;                        // tile-local bucket start
    uint32_t* s_cur = s_start + kSlots;                        // next free global slot
    uint32_t* s_delta = s_cur + kSlots;                        // global slot - local index
    __shared__ unsigned long long s_scratch[33];
    __shared__ __align__(8) unsigned long long s_bar[2];
    __shared__ uint32_t s_tile_valid;
    __shared__ uint32_t s_last;

    const unsigned P = gridDim.x, c = blockIdx.x;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t vlo = ks.nv * c / P, vhi = ks.nv * (c + 1) / P;
    constexpr size_t kTileVec = TILE / 4;
    const size_t ntiles = (vhi - vlo + kTileVec - 1) / kTileVec;
    const uint32_t spill = static_cast<uint32_t>(nb);
    // Slot of a key: its bucket, or the spill slot for padding lanes and (slab
    // layout, which has no KB1 to count them) keys beyond the range, so the
    // spill count of a tile gives the out-of-range keys for free.
    const uint32_t last = SLAB && sa.check ? sa.limit - 1u : 0xffffffffu;
    // largest key - lo that maps to a real bucket under slot_of: the slab's
    // range limit, or (packed layout) the end of the last bucket
    const uint64_t bucket_end = static_cast<uint64_t>(nb) * bm.width;
    const uint32_t fast_last = SLAB ? last : (bucket_end > 0xffffffffull ? 0xffffffffu
                                                                         : static_cast<uint32_t>(bucket_end - 1));
    auto slot_of = [&](uint32_t key, bool in) -> uint32_t {
        if constexpr (SLAB) return in && key - bm.lo <= last ? bucket_id(key, bm) : spill;
        else return bucket_or_spill(key, in, bm, nb);
    };

    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (size_t t = 0; t < 2 && t < ntiles; ++t) {
            const size_t v0 = vlo + t * kTileVec;
            const size_t nvec = min(kTileVec, vhi - v0);
            if (!SLAB || CHUNK)
                tma_load_bytes_hint(s_buf + t * TILE, ks.body + v0, static_cast<unsigned>(nvec * 16), &s_bar[t],
                                    l2_policy_evict_first());
            else
                tma_load_bytes(s_buf + t * TILE, ks.body + v0, static_cast<unsigned>(nvec * 16), &s_bar[t]);
        }
    }

    unsigned long long* s_base64 = reinterpret_cast<unsigned long long*>(s_cnt);  // spans cnt+start
    uint32_t bad = 0;  // slab: keys >= sa.limit (KB1 counts them in the packed layout)
    uint32_t kmax = 0;  // slab: largest (biased) key this thread saw
    if constexpr (!SLAB) {
        // bucket bases (exclusive prefix of totals) + this CTA's first slot per bucket
        for (int b = threadIdx.x; b < nb; b += blockDim.x) s_cur[b] = tot[b];
        __syncthreads();
        const unsigned long long total = block_exclusive_scan_u64(s_cur, nb, s_base64, s_scratch);
        for (int b = threadIdx.x; b < nb; b += blockDim.x) {
            if (c == 0) g_base[b] = s_base64[b];
            s_delta[b] = static_cast<uint32_t>(s_base64[b] + H[static_cast<size_t>(b) * P + c]);
        }
        if (c == 0 && threadIdx.x == 0) g_base[nb] = total;
        __syncthreads();
        if (c == 0 && sa.order) compute_kb4_order(tot, nb, sa.order);  // KB4's ticket order
    }
    for (int b = threadIdx.x; b <= nb; b += blockDim.x) {
        if constexpr (!SLAB) s_cur[b] = b < nb ? s_delta[b] : 0u;
        s_cnt[b] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // misaligned head (CTA 0) / tail (CTA P-1) keys
        const uint32_t* extra = c == 0 ? ks.head : nullptr;
        int ne = c == 0 ? ks.n_head : 0;
        for (int pass = 0; pass < 2; ++pass) {
            for (int i = 0; i < ne; ++i) {
                const uint32_t e = extra[i] ^ ks.xr;
                const uint32_t b = slot_of(e, true);
                kmax = max(kmax, e);
                if constexpr (CHUNK) {
                    bad += (sa.check && e - bm.lo >= sa.limit) ? 1u : 0u;
                    if (b != spill) {
                        const uint32_t pos = atomicAdd(sa.gcnt + b, 1u);
                        const uint32_t cs = sa.chunk_shift, cm = (1u << cs) - 1u;
                        const uint32_t j = pos >> cs;
                        if (j < sa.max_chunks) {
                            const uint32_t id = (pos & cm) == 0 ? chunk_alloc(sa, nb, b, j) : chunk_get(sa, b, j);
                            parted[static_cast<size_t>(chunk_base(id, cs, sa.chunk_pad)) + (pos & cm)] = e;
                        } else {
                            sa.ctrl->overflow = 1u;
                        }
                    }
                } else if constexpr (SLAB) {
                    bad += (sa.check && e - bm.lo >= sa.limit) ? 1u : 0u;
                    if (b != spill) {
                        const uint32_t pos = atomicAdd(sa.gcnt + b, 1u);
                        if (pos < sa.cap) parted[b * sa.cap + pos] = e;
                    }
                } else {
                    if (b != spill) parted[s_cur[b]++] = e;
                }
            }
            extra = c == P - 1 ? ks.tail : nullptr;
            ne = c == P - 1 ? ks.n_tail : 0;
        }
    }
    __syncthreads();

    constexpr int VPT = KPT / 4;
    const int slots = nb + 1;
    const int per = (slots + THREADS - 1) / THREADS;
    const int sb = threadIdx.x * per;
    for (size_t t = 0; t < ntiles; ++t) {
        const int p = static_cast<int>(t & 1);
        uint32_t* buf = s_buf + p * TILE;
        const size_t v0 = vlo + t * kTileVec;
        const uint32_t nvec = static_cast<uint32_t>(min(kTileVec, vhi - v0));
        mbar_wait(&s_bar[p], static_cast<unsigned>((t >> 1) & 1));

        uint32_t k[KPT];
        uint32_t rb[KPT];  // bucket << 16 | rank inside the bucket (rank < TILE)
        uint32_t rmin = 0xffffffffu, rmax = 0;  // over key - lo
        bool all_in = true;
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
            const uint32_t vi = j * THREADS + threadIdx.x;
            const bool in = vi < nvec;
            all_in &= in;
            const uint4 v = in ? reinterpret_cast<const uint4*>(buf)[vi] : make_uint4(0, 0, 0, 0);
            const uint32_t kk[4] = {v.x ^ ks.xr, v.y ^ ks.xr, v.z ^ ks.xr, v.w ^ ks.xr};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                k[4 * j + q] = kk[q];
                rmin = min(rmin, kk[q] - bm.lo);
                rmax = max(rmax, kk[q] - bm.lo);
            }
        }
        rmin = __reduce_min_sync(kFull, rmin);
        rmax = __reduce_max_sync(kFull, rmax);
        // every key of the warp step below the fast limit (and no padding
        // lanes): buckets without per-key range checks
        if (__all_sync(kFull, all_in) && rmax <= fast_last) {
            if constexpr (SLAB) kmax = max(kmax, rmax + bm.lo);
#pragma unroll
            for (int q = 0; q < KPT; ++q) rb[q] = __umulhi(((k[q] - bm.lo) >> bm.ms) << 12, bm.mq);
        } else {
#pragma unroll
            for (int j = 0; j < VPT; ++j) {
                const bool in = j * THREADS + threadIdx.x < nvec;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    rb[4 * j + q] = slot_of(k[4 * j + q], in);
                    if constexpr (SLAB) kmax = max(kmax, in ? k[4 * j + q] : 0u);
                }
            }
        }
        const uint32_t blo = slot_of(rmin + bm.lo, true);
        const uint32_t bhi = slot_of(rmax + bm.lo, true);
        if (blo == bhi && __all_sync(kFull, all_in)) {
            // the whole warp step lies in one bucket: one atomic, ranks by lane
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(s_cnt + blo, 32u * KPT);
            base = __shfl_sync(kFull, base, 0) + lane * KPT;
#pragma unroll
            for (int q = 0; q < KPT; ++q) rb[q] = (blo << 16) | (base + q);
        } else {
#pragma unroll
            for (int q = 0; q < KPT; ++q) rb[q] = (rb[q] << 16) | atomicAdd(s_cnt + rb[q], 1u);
        }
        __syncthreads();  // A: tile counts complete; every thread has read buf
        uint32_t claim[SLAB ? PER_MAX : 1];  // slab: first claimed slot per bucket (in flight)
        uint32_t ccnt[SLAB ? PER_MAX : 1];
        {
            uint32_t local = 0;
            for (int q = 0; q < per; ++q)
                if (sb + q < slots) local += s_cnt[sb + q];
            const uint32_t incl = warp_incl_scan(local, lane);
            if (lane == 31) s_scratch[warp] = incl;
            __syncthreads();
            uint32_t run;
            {  // every warp scans the warp totals itself (one barrier less per tile)
                const uint32_t w = lane < NWARPS ? static_cast<uint32_t>(s_scratch[lane]) : 0u;
                const uint32_t wi = warp_incl_scan(w, lane);
                run = __shfl_sync(kFull, wi - w, warp) + (incl - local);
            }
            if constexpr (SLAB) {
#pragma unroll
                for (int q = 0; q < PER_MAX; ++q) {
                    const int b = sb + q;
                    ccnt[q] = 0;
                    if (q < per && b < slots) {
                        const uint32_t cb = s_cnt[b];
                        s_start[b] = run;
                        s_cnt[b] = 0;
                        if (b == nb) {
                            s_tile_valid = run;  // spill keys sort after every bucket
                            bad += cb - (TILE - 4 * nvec);  // out-of-range keys (padding lanes spill too)
                        } else if (cb) {
                            claim[q] = atomicAdd(sa.gcnt + b, cb);
                        }
                        ccnt[q] = b < nb ? cb : 0u;
                        run += cb;
                    }
                }
            } else {
                for (int q = 0; q < per; ++q) {
                    const int b = sb + q;
                    if (b < slots) {
                        const uint32_t cb = s_cnt[b];
                        s_start[b] = run;
                        s_delta[b] = s_cur[b] - run;
                        s_cur[b] += cb;
                        s_cnt[b] = 0;
                        if (b == nb) s_tile_valid = run;  // spill keys sort after every bucket
                        run += cb;
                    }
                }
            }
        }
        __syncthreads();  // B
        // all 16 bucket-start lookups first (independent SMEM loads), then the stores
#pragma unroll
        for (int q = 0; q < KPT; ++q) rb[q] = s_start[rb[q] >> 16] + (rb[q] & 0xffffu);
#pragma unroll
        for (int q = 0; q < KPT; ++q) buf[rb[q]] = k[q];
        if constexpr (CHUNK) {
            // every chunk whose first slot lies in this tile's run is allocated
            // here (allocation never waits); the run's first chunk, when an
            // earlier claim owns it, is waited for (all KB3 CTAs are resident).
            // Two passes: all of this thread's allocations and table loads are
            // issued before any result is waited for (the loads' L2 latency
            // overlaps instead of adding up per bucket).
            uint32_t id0[PER_MAX];
            const uint32_t cs = sa.chunk_shift, cm = (1u << cs) - 1u;
#pragma unroll
            for (int q = 0; q < PER_MAX; ++q) {
                id0[q] = 0u;
                if (!ccnt[q]) continue;
                const uint32_t b = sb + q;
                const uint32_t cl = claim[q], cb = ccnt[q];
                const uint32_t j0 = cl >> cs, j1 = (cl + cb - 1) >> cs;
                if (j1 >= sa.max_chunks) continue;  // overflow: handled below
                for (uint32_t j = j0; j <= j1; ++j) {
                    if ((j << cs) >= cl) {
                        const uint32_t id = chunk_alloc(sa, nb, b, j);
                        if (j == j0) id0[q] = id + 1u;
                    }
                }
                if ((cl & cm) != 0)  // owned by an earlier claim: look it up (0 = not yet)
                    id0[q] = j0 == 0 ? b + 1u
                                     : *reinterpret_cast<const volatile uint32_t*>(
                                           sa.chunk_tab + static_cast<size_t>(b) * sa.max_chunks + j0);
            }
#pragma unroll
            for (int q = 0; q < PER_MAX; ++q) {
                if (!ccnt[q]) continue;
                const uint32_t b = sb + q;
                const uint32_t cl = claim[q], cb = ccnt[q];
                const uint32_t j0 = cl >> cs, j1 = (cl + cb - 1) >> cs;
                if (j1 >= sa.max_chunks) {  // repeated keys overflowed the bucket
                    sa.ctrl->overflow = 1u;
                    s_cur[b] = KC_DROP;  // (any 32-bit delta is a valid slot offset)
                    continue;
                }
                const uint32_t id = id0[q] ? id0[q] - 1u : chunk_get(sa, b, j0);
                const uint32_t st = s_start[b];
                s_delta[b] = chunk_base(id, cs, sa.chunk_pad) + (cl & cm) - st;
                // tile position where the run leaves its first chunk (0x7fff: never;
                // a crossing lies inside the tile, so it fits 15 bits), with the
                // next chunk's index above it for the slow path
                const uint32_t room = (1u << cs) - (cl & cm);
                s_cur[b] = cb > room ? (st + room) | ((j0 + 1) << 15) : 0x7fffu;
            }
        } else if constexpr (SLAB) {
#pragma unroll
            for (int q = 0; q < PER_MAX; ++q) {
                if (ccnt[q]) {
                    const uint32_t b = sb + q;
                    // a claim past the bucket's capacity (only duplicates can cause
                    // one) is aimed at the dump tile, whose stores are then skipped
                    // (a bucket that overflowed sorts nothing; repeated keys can
                    // overflow every tile's run, and concurrent stores to one dump
                    // tile measured 3 ms on 2^26 keys)
                    const uint32_t dst = claim[q] + ccnt[q] <= sa.cap ? b * sa.cap + claim[q] : sa.dump;
                    s_delta[b] = dst - s_start[b];
                }
            }
        }
        __syncthreads();  // C
        const uint32_t tile_valid = s_tile_valid;
        if (!SLAB) {
            const unsigned long long pol = l2_policy_evict_last();
#pragma unroll 4
            for (uint32_t i = threadIdx.x; i < tile_valid; i += THREADS) {
                const uint32_t key = buf[i];
                st_hint(parted + s_delta[bucket_id(key, bm)] + i, key, pol);
            }
        } else if constexpr (CHUNK) {
            const unsigned long long pol = l2_policy_evict_last();
#pragma unroll 4
            for (uint32_t i = threadIdx.x; i < tile_valid; i += THREADS) {
                const uint32_t key = buf[i];
                const uint32_t b = bucket_id(key, bm);
                const uint32_t d = s_delta[b];
                const uint32_t x = s_cur[b];
                if (x == KC_DROP) continue;  // an overflowed (repeated-key) run
                size_t dst = d + i;  // (32-bit wrap: d is the slot minus the tile position)
                if (i >= (x & 0x7fffu)) {  // past the run's first chunk (rare)
                    const uint32_t k2 = i - (x & 0x7fffu);
                    const uint32_t id = chunk_get(sa, b, (x >> 15) + (k2 >> sa.chunk_shift));
                    dst = static_cast<size_t>(chunk_base(id, sa.chunk_shift, sa.chunk_pad)) + (k2 & ((1u << sa.chunk_shift) - 1u));
                }
                st_hint(parted + dst, key, pol);
            }
        } else {
#pragma unroll 4
            for (uint32_t i = threadIdx.x; i < tile_valid; i += THREADS) {
                const uint32_t key = buf[i];
                const uint32_t pos = s_delta[bucket_id(key, bm)] + i;
                if (pos < sa.dump) parted[pos] = key;  // dump-tile runs are dropped
            }
        }
        __syncthreads();  // D: buf free again
        if (threadIdx.x == 0 && t + 2 < ntiles) {
            const size_t v2 = vlo + (t + 2) * kTileVec;
            const size_t nv2 = min(kTileVec, vhi - v2);
            fence_proxy_async_smem();
            if (!SLAB || CHUNK)
                tma_load_bytes_hint(buf, ks.body + v2, static_cast<unsigned>(nv2 * 16), &s_bar[p],
                                    l2_policy_evict_first());
            else
                tma_load_bytes(buf, ks.body + v2, static_cast<unsigned>(nv2 * 16), &s_bar[p]);
        }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if constexpr (SLAB) slab_finish(sa, nb, bad, kmax, s_cur, s_base64, s_scratch, &s_last);
}


// KB3, slab layout with bulk-copy (TMA) run stores — the default for <= 1024
// buckets. Same tile pipeline as bucket_partition_kernel, but the tile is
// counting-sorted into a separate SMEM buffer whose bucket runs start on
// 16-byte boundaries, and each bucket's run leaves with ONE cp.async.bulk
// store issued by the thread owning the bucket, instead of every thread
// copying keys and looking up their bucket's destination (that write loop was
// ~20% of KB3's instructions; 293 bulk stores of ~224 B per SM per tile
// measured ~2 us, tools/tma_store_bench.cu). The stores drain while the next
// tile is ranked; their SMEM reads are waited for just before the next
// scatter. Runs are padded to a multiple of 4 keys with copies of the run's
// first key (a bitset ignores repeats: KB4 reads the padded slot count, the
// output offsets use the true count), so every claim in the slab is 16-byte
// aligned. The TMA ring is freed as soon as a tile's keys are in registers,
// so the next-but-one tile's load starts a phase earlier than in the
// in-place variant.
template <int MAXB, int THREADS_ = PART_THREADS, int KPT_ = PART_KPT>
__global__ void __launch_bounds__(THREADS_, 1)
    bucket_partition_tma_kernel(KeySplit ks, BucketMap bm, int nb, uint32_t* __restrict__ parted, SlabArgs sa) {
    constexpr int THREADS = THREADS_;
    constexpr int KPT = KPT_;
    static_assert(THREADS * KPT == PART_TILE, "the SMEM layout is sized for PART_TILE keys");
    constexpr int TILE = THREADS * KPT;
    constexpr int NWARPS = THREADS / 32;
    constexpr int kSlots = MAXB + 1;
    constexpr int PER_MAX = (kSlots + THREADS - 1) / THREADS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint32_t* s_ring = reinterpret_cast<uint32_t*>(smem_raw);  // 2 x TILE (TMA destination)
    uint32_t* s_sorted = s_ring + 2 * TILE;                     // TILE + 4 * kSlots (runs 16B-aligned)
    uint32_t* s_cnt = s_sorted + TILE + 4 * kSlots;             // keys per bucket in the tile
    uint32_t* s_start = s_cnt + kSlots;                         // run start in s_sorted (multiple of 4)
    // 16 copies of every run start (16-bit): lane l reads copy l & 15, so a
    // warp's 32 random lookups spread over 8x more banks than one copy allows
    // (offset from the 128-byte-aligned SMEM base rounded up to 16 bytes at
    // compile time: no integer round trip, so the compiler keeps LDS addressing)
    constexpr int kStart16Words = (3 * TILE + 6 * kSlots + 3) & ~3;
    uint16_t* s_start16 = reinterpret_cast<uint16_t*>(reinterpret_cast<uint32_t*>(smem_raw) + kStart16Words);
    __shared__ unsigned long long s_scratch[33];
    __shared__ __align__(8) unsigned long long s_bar[2];
    __shared__ uint32_t s_last;

    const unsigned P = gridDim.x, c = blockIdx.x;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t vlo = ks.nv * c / P, vhi = ks.nv * (c + 1) / P;
    constexpr size_t kTileVec = TILE / 4;
    const size_t ntiles = (vhi - vlo + kTileVec - 1) / kTileVec;
    const uint32_t spill = static_cast<uint32_t>(nb);
    const uint32_t last = sa.check ? sa.limit - 1u : 0xffffffffu;
    auto slot_of = [&](uint32_t key, bool in) -> uint32_t {
        return in && key - bm.lo <= last ? bucket_id(key, bm) : spill;
    };
    auto load_tile = [&](size_t t, int p) {  // thread 0
        const size_t v0 = vlo + t * kTileVec;
        const size_t nvec = min(kTileVec, vhi - v0);
        fence_proxy_async_smem();
        // the key stream is read once: evict_first keeps L2 for the runs KB4
        // reads next (measured C2 KB4 146.6 -> 144.2 us)
        tma_load_bytes_hint(s_ring + p * TILE, ks.body + v0, static_cast<unsigned>(nvec * 16), &s_bar[p],
                            l2_policy_evict_first());
    };

    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        fence_mbar_init();
    }
    for (int b = threadIdx.x; b < kSlots; b += THREADS) s_cnt[b] = 0;
    __syncthreads();
    if (threadIdx.x == 0)
        for (size_t t = 0; t < 2 && t < ntiles; ++t) load_tile(t, static_cast<int>(t));
    uint32_t bad = 0;
    uint32_t kmax = 0;  // largest (biased) key this thread saw
    if (threadIdx.x == 0) {  // misaligned head (CTA 0) / tail (CTA P-1): one padded claim each
        const uint32_t* extra = c == 0 ? ks.head : nullptr;
        int ne = c == 0 ? ks.n_head : 0;
        for (int pass = 0; pass < 2; ++pass) {
            for (int i = 0; i < ne; ++i) {
                const uint32_t e = extra[i] ^ ks.xr;
                bad += (sa.check && e - bm.lo >= sa.limit) ? 1u : 0u;
                kmax = max(kmax, e);
                const uint32_t b = slot_of(e, true);
                if (b == spill) continue;
                atomicAdd(sa.gtrue + b, 1u);
                const uint32_t pos = atomicAdd(sa.gcnt + b, 4u);
                if (pos + 4 <= sa.cap) {
                    parted[b * sa.cap + pos] = e;
                    for (int q = 1; q < 4; ++q) parted[b * sa.cap + pos + q] = bm.lo + (b + 1u) * bm.width;
                }
            }
            extra = c == P - 1 ? ks.tail : nullptr;
            ne = c == P - 1 ? ks.n_tail : 0;
        }
    }

    constexpr int VPT = KPT / 4;
    const int slots = nb + 1;
    const int per = (slots + THREADS - 1) / THREADS;
    const int sb = threadIdx.x * per;
    bool stores_pending = false;  // this thread has bulk stores reading s_sorted
    for (size_t t = 0; t < ntiles; ++t) {
        const int p = static_cast<int>(t & 1);
        const uint32_t* buf = s_ring + p * TILE;
        const size_t v0 = vlo + t * kTileVec;
        const uint32_t nvec = static_cast<uint32_t>(min(kTileVec, vhi - v0));
        mbar_wait(&s_bar[p], static_cast<unsigned>((t >> 1) & 1));

        uint32_t k[KPT];
        uint32_t rb[KPT];  // bucket << 16 | rank inside the bucket (rank < TILE)
        uint32_t rmin = 0xffffffffu, rmax = 0;  // over key - lo
        bool all_in = true;
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
            const uint32_t vi = j * THREADS + threadIdx.x;
            const bool in = vi < nvec;
            all_in &= in;
            const uint4 v = in ? reinterpret_cast<const uint4*>(buf)[vi] : make_uint4(0, 0, 0, 0);
            const uint32_t kk[4] = {v.x ^ ks.xr, v.y ^ ks.xr, v.z ^ ks.xr, v.w ^ ks.xr};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                k[4 * j + q] = kk[q];
                rmin = min(rmin, kk[q] - bm.lo);
                rmax = max(rmax, kk[q] - bm.lo);
            }
        }
        rmin = __reduce_min_sync(kFull, rmin);
        rmax = __reduce_max_sync(kFull, rmax);
        // a warp step with every key in range (and no padding lanes) needs no
        // per-key range check: the common case
        if (__all_sync(kFull, all_in) && rmax <= last) {
            kmax = max(kmax, rmax + bm.lo);
#pragma unroll
            for (int q = 0; q < KPT; ++q) rb[q] = __umulhi(((k[q] - bm.lo) >> bm.ms) << 12, bm.mq);
        } else {
#pragma unroll
            for (int j = 0; j < VPT; ++j) {
                const bool in = j * THREADS + threadIdx.x < nvec;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    rb[4 * j + q] = slot_of(k[4 * j + q], in);
                    kmax = max(kmax, in ? k[4 * j + q] : 0u);
                }
            }
        }
        const uint32_t blo = slot_of(rmin + bm.lo, true);
        const uint32_t bhi = slot_of(rmax + bm.lo, true);
        if (blo == bhi && __all_sync(kFull, all_in)) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(s_cnt + blo, 32u * KPT);
            base = __shfl_sync(kFull, base, 0) + lane * KPT;
#pragma unroll
            for (int q = 0; q < KPT; ++q) rb[q] = (blo << 16) | (base + q);
        } else {
#pragma unroll
            for (int q = 0; q < KPT; ++q) rb[q] = (rb[q] << 16) | atomicAdd(s_cnt + rb[q], 1u);
        }
        __syncthreads();  // A: counts complete; the ring slot is free
        // the refill is issued by the last warp: warp 0 is on the scan's critical path
        if (threadIdx.x == THREADS - 32 && t + 2 < ntiles) load_tile(t + 2, p);
        // padded run starts (multiples of 4) and the slab claims
        uint32_t claim[PER_MAX];
        uint32_t ccnt[PER_MAX];
        {
            uint32_t local = 0;
            for (int q = 0; q < per; ++q)
                if (sb + q < nb) local += (s_cnt[sb + q] + 3u) & ~3u;
            const uint32_t incl = warp_incl_scan(local, lane);
            if (lane == 31) s_scratch[warp] = incl;
            __syncthreads();
            uint32_t run;
            {  // every warp scans the warp totals itself (one barrier less per tile)
                const uint32_t w = lane < NWARPS ? static_cast<uint32_t>(s_scratch[lane]) : 0u;
                const uint32_t wi = warp_incl_scan(w, lane);
                run = __shfl_sync(kFull, wi - w, warp) + (incl - local);
            }
#pragma unroll
            for (int q = 0; q < PER_MAX; ++q) {
                const int b = sb + q;
                ccnt[q] = 0;
                if (q < per && b < slots) {
                    const uint32_t cb = s_cnt[b];
                    s_cnt[b] = 0;
                    if (b == nb) {
                        bad += cb - (TILE - 4 * nvec);  // out-of-range keys (padding lanes spill too)
                    } else {
                        s_start[b] = run;
                        if (cb) {
                            uint4 rep;  // 8 x 16-bit copies
                            rep.x = rep.y = rep.z = rep.w = run | (run << 16);
                            reinterpret_cast<uint4*>(s_start16 + 16 * b)[0] = rep;
                            reinterpret_cast<uint4*>(s_start16 + 16 * b)[1] = rep;
                            const uint32_t pc = (cb + 3u) & ~3u;
                            claim[q] = atomicAdd(sa.gcnt + b, pc);
                            atomicAdd(sa.gtrue + b, cb);
                            ccnt[q] = cb;
                        }
                        run += (cb + 3u) & ~3u;
                    }
                }
            }
        }
        // the previous tile's bulk stores must have read s_sorted before it is rewritten
        if (stores_pending) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            stores_pending = false;
        }
        __syncthreads();  // B
        // (a branch-free version — all 16 run-start lookups, then 16 stores, no
        // spill checks on tiles without spill keys — cut this loop from 14 to 7
        // instructions per key and measured C2 KB3 166.5 -> 171.7 us: the LSU
        // data pipe, not instruction issue, bounds the kernel, and the
        // interleaved lookup/store pairs pace it better)
#pragma unroll
        for (int q = 0; q < KPT; ++q) {
            const uint32_t b = rb[q] >> 16;
            if (b != spill) s_sorted[s_start16[(b << 4) | (lane & 15u)] + (rb[q] & 0xffffu)] = k[q];
        }
        fence_proxy_async_smem();  // generic-proxy writes -> visible to the bulk copies
        __syncthreads();  // C
#pragma unroll
        for (int q = 0; q < PER_MAX; ++q) {
            if (ccnt[q]) {
                const uint32_t b = sb + q;
                const uint32_t cb = ccnt[q], pc = (cb + 3u) & ~3u;
                const uint32_t st = s_start[b];
                // pad to 4 with the first key past the bucket (KB4 and KB4m drop it):
                // the slab then holds the exact key multiset (in-place recovery)
                const uint32_t padv = bm.lo + (b + 1u) * bm.width;
                for (uint32_t i = cb; i < pc; ++i) s_sorted[st + i] = padv;
                fence_proxy_async_smem();
                // a claim past the bucket's capacity (only duplicates cause one) is
                // dropped: that bucket then sorts nothing and the popcount total
                // reports the repeats
                if (claim[q] + pc <= sa.cap) {
                    uint32_t* dst = parted + static_cast<size_t>(b) * sa.cap + claim[q];
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                                 "r"(smem_u32(s_sorted + st)), "r"(pc * 4)
                                 : "memory");
                    stores_pending = true;
                }
            }
        }
        if (stores_pending) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    // the dependent KB4 may start its prologue (it waits for this grid's completion
    // before reading anything KB3 wrote)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (stores_pending) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    slab_finish(sa, nb, bad, kmax, s_cnt, reinterpret_cast<unsigned long long*>(s_sorted), s_scratch, &s_last);
}

constexpr std::size_t part_tma_smem_bytes(int maxb) {
    return (2 * std::size_t(PART_TILE) + PART_TILE + 4 * std::size_t(maxb + 1) + 2 * std::size_t(maxb + 1) +
            8 * std::size_t(maxb + 1) + 4) * 4;  // ... + 16 x 16-bit start copies (16B-aligned)
}


// KB4 scatter of one bucket's keys into the SMEM bitset (and, for SPARSE
// buckets, the summary of touched words): misaligned head, 16-byte loads
// with 4 per thread in flight, tail. Slab runs are padded with the first key
// past the bucket (x == width), which is dropped.

template <bool SPARSE, int NT = BUCKET_THREADS>
__device__ __forceinline__ void scatter_bucket_keys(const uint32_t* __restrict__ src, uint32_t cnt,
                                                    uint32_t key_lo, uint32_t width, uint32_t* s_bits,
                                                    uint32_t* s_sum) {
    // Predicated reductions on 32-bit shared addresses instead of `if (x >= width)
    // return; atomicOr(...)`: the branch cost a BSSY/BRA/BSYNC per key and the
    // compiler rebuilt the shared-window base inside every conditional block
    // (12 instructions per key in the round-2 ncu SASS view, 5 now).
    const uint32_t bits32 = smem_u32(s_bits), sum32 = SPARSE ? smem_u32(s_sum) : 0u;
    auto set_key = [&](uint32_t key) {
        const uint32_t x = key - key_lo;  // < width: the key's bucket is this one (== width: padding)
        const uint32_t w = x >> 5;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.lt.u32 p, %0, %1;\n\t@p red.shared.or.b32 [%2], %3;\n\t}"
            ::"r"(x), "r"(width), "r"(bits32 + (w << 2)), "r"(1u << (x & 31))
            : "memory");
        if (SPARSE)
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.lt.u32 p, %0, %1;\n\t@p red.shared.or.b32 [%2], %3;\n\t}"
                ::"r"(x), "r"(width), "r"(sum32 + ((w >> 5) << 2)), "r"(1u << (w & 31))
                : "memory");
    };
    const uint32_t head = min(cnt, static_cast<uint32_t>(
                                       ((16 - (reinterpret_cast<uintptr_t>(src) & 15)) & 15) / 4));
    if (threadIdx.x < head) set_key(__ldcs(src + threadIdx.x));
    const uint4* v4 = reinterpret_cast<const uint4*>(src + head);
    const uint32_t nv = (cnt - head) / 4;
    constexpr int U = 4;
    constexpr uint32_t kBatch = NT * U;
    uint32_t i0 = 0;
    for (; i0 + kBatch <= nv; i0 += kBatch) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_na(v4 + i0 + u * NT + threadIdx.x);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            set_key(v[u].x);
            set_key(v[u].y);
            set_key(v[u].z);
            set_key(v[u].w);
        }
    }
    for (uint32_t i = i0 + threadIdx.x; i < nv; i += NT) {
        const uint4 v = ld_na(v4 + i);
        set_key(v.x);
        set_key(v.y);
        set_key(v.z);
        set_key(v.w);
    }
    const uint32_t done = head + 4 * nv;
    if (threadIdx.x < cnt - done) set_key(__ldcs(src + done + threadIdx.x));
}

// KB4: one bucket per CTA iteration (dynamic ticket). SMEM bitset of 2^shift
// bits; warp w owns words [w*W/32, (w+1)*W/32) and extracts them in order
// straight to the output slots of the bucket. Every key of a bucket lands in
// [base_b, base_b + tot_b) (tot_b counts duplicates too), so no output bounds
// checks are needed.
//
// Dense buckets zero the whole bitset up front and scan every word. Sparse
// buckets (< 1 key per 4 words: e.g. C4, and the thin tails of C5) also mark
// each touched word in a summary bitset (one bit per word), visit only
// touched words, and zero exactly those words again, so a sparse bucket costs
// O(keys) SMEM work instead of O(2^shift / 32) and leaves the bitset clean.
template <int STAGE, int NT = BUCKET_THREADS>
__global__ void __launch_bounds__(NT, NT >= 1024 ? 1 : 2)
    bucket_sort_kernel(const uint32_t* __restrict__ parted, const uint32_t* __restrict__ tot,
                       const unsigned long long* __restrict__ g_base, BucketMap bm, int nb,
                       uint32_t src_cap, uint32_t* __restrict__ out, Ctrl* __restrict__ ctrl,
                       const uint32_t* __restrict__ order, int all_or_nothing,
                       const uint32_t* __restrict__ chunk_tab, uint32_t max_chunks, uint32_t chunk_shift,
                       uint32_t chunk_pad) {
    // in-place sorts: a slab that lost runs (repeated keys overflowed a
    // bucket) writes nothing, so the input stays intact for the counting pass
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t W = bm.width >> 5;  // words per bucket bitset (>= 1024; 2^k or a multiple of 4096)
    uint32_t* s_bits = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* s_sum = s_bits + W;             // bit w set <=> word w touched (sparse buckets)
    uint32_t* s_stage_all = s_sum + W / 32;   // NT/32 x stage pitch
    __shared__ uint32_t s_warp[NT / 32];
    // next bucket (ticket, offset, count), fetched by thread 0 one bucket ahead
    // so its latency hides behind the current bucket (sparse buckets are short)
    __shared__ unsigned s_b[2];
    __shared__ unsigned long long s_bbase[2];
    __shared__ uint32_t s_bcnt[2];
    __shared__ __align__(8) unsigned long long s_lbar[KB4_RING];  // dense scatter: bulk-load ring (full)
    __shared__ __align__(8) unsigned long long s_ebar[KB4_RING];  // ... and its slots consumed (NT arrivals)

    const unsigned lane = threadIdx.x & 31;
    const unsigned warp = threadIdx.x >> 5;
    constexpr int kStagePitch = STAGE + STAGE / 32;
    uint32_t* s_stage = s_stage_all + warp * kStagePitch;
    // Dense buckets stream their keys through the (then idle) stage area with
    // bulk copies: two chunks in flight, no L1 or registers tied up by the
    // loads (the SMEM bitset + stage leave KB4 a small L1).
    constexpr uint32_t kChunk = ((NT / 32) * kStagePitch * 4 / KB4_RING) / 16 * 4;  // keys per ring slot
    // (measured: the ring takes C5's packed-layout KB4 from 1025 to 959 us and
    // makes C2's and C3's slab-layout KB4 2-5% slower, so slab buckets keep
    // register loads)
    unsigned chunk_seq = 0;  // bulk chunks this CTA has consumed (block-uniform)
    if (threadIdx.x == 0) {
        for (int q = 0; q < KB4_RING; ++q) {
            mbar_init(&s_lbar[q], 1);
            mbar_init(&s_ebar[q], NT);
        }
        fence_mbar_init();
    }
    const uint32_t seg_words = W / (NT / 32);
    const uint4* s4 = reinterpret_cast<const uint4*>(s_bits);

    auto fetch = [&](int slot) {  // thread 0
        unsigned nbk = atomicAdd(&ctrl->ticket, 1u);
        if (order && nbk < static_cast<unsigned>(nb)) nbk = order[nbk];  // largest buckets first
        s_b[slot] = nbk;
        if (nbk < static_cast<unsigned>(nb)) {
            s_bbase[slot] = g_base[nbk];
            s_bcnt[slot] = tot[nbk];
        }
    };
    for (uint32_t i = threadIdx.x; i < W / 32; i += NT) s_sum[i] = 0u;
    {  // the first bucket's clean bitset
        uint4* b4 = reinterpret_cast<uint4*>(s_bits);
        for (uint32_t i = threadIdx.x; i < W / 4; i += NT) b4[i] = make_uint4(0, 0, 0, 0);
    }
    // Programmatic dependent launch: everything above (barrier init, 100+ KB of
    // SMEM zeroing) ran while KB3's last CTAs were finishing; KB3's results
    // (totals, offsets, order, the control block) are read only below this
    // wait. Without the launch attribute the wait returns at once.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (all_or_nothing && *reinterpret_cast<volatile const uint32_t*>(&ctrl->overflow)) return;
    if (threadIdx.x == 0) {
        if (order && order[nb] == 0u) order = nullptr;  // identity: no per-ticket lookup
        fetch(0);
    }
    bool dirty = false;  // block-uniform: bitset needs zeroing before the next bucket
    for (unsigned it = 0;; ++it) {
        const int slot = static_cast<int>(it & 1u);
        if (dirty) {  // the previous bucket's readers finished at the loop-end barrier
            uint4* b4 = reinterpret_cast<uint4*>(s_bits);
            for (uint32_t i = threadIdx.x; i < W / 4; i += NT) b4[i] = make_uint4(0, 0, 0, 0);
        }
        __syncthreads();
        const unsigned b = s_b[slot];
        if (b >= static_cast<unsigned>(nb)) break;
        const unsigned long long base = s_bbase[slot];
        const uint32_t cnt = s_bcnt[slot];
        if (threadIdx.x == 0) fetch(slot ^ 1);  // read again only after two more barriers
        const uint32_t* src = parted + (src_cap ? static_cast<size_t>(b) * src_cap : base);  // slab / packed
        const bool sparse = static_cast<unsigned long long>(cnt) * 4 < W;
        const uint32_t key_lo = bm.lo + static_cast<uint32_t>(b) * bm.width;
        // chunked layout: the bucket's keys are 2^chunk_shift-slot pool chunks
        const uint32_t CH = 1u << chunk_shift;
        auto chunk_src = [&](uint32_t j) {
            const uint32_t id = j == 0 ? b : chunk_tab[static_cast<size_t>(b) * max_chunks + j] - 1u;
            return parted + static_cast<size_t>(chunk_base(id, chunk_shift, chunk_pad));
        };
        if (chunk_tab && (sparse || cnt <= 2 * CH)) {
            for (uint32_t j = 0; j * CH < cnt; ++j) {
                const uint32_t cj = min(CH, cnt - j * CH);
                if (sparse)
                    scatter_bucket_keys<true, NT>(chunk_src(j), cj, key_lo, bm.width, s_bits, s_sum);
                else
                    scatter_bucket_keys<false, NT>(chunk_src(j), cj, key_lo, bm.width, s_bits, s_sum);
            }
        } else if (sparse) {
            scatter_bucket_keys<true, NT>(src, cnt, key_lo, bm.width, s_bits, s_sum);
        } else if (src_cap) {  // slab-layout buckets: register loads measured faster (C2, C3)
            scatter_bucket_keys<false, NT>(src, cnt, key_lo, bm.width, s_bits, s_sum);
        } else {
            // packed: one contiguous range; chunked: the same ring pieces, each
            // loaded as at most two bulk copies (one per pool chunk it touches)
            const uint32_t piece = kChunk;
            static_assert(KC_CHUNK_MIN >= kChunk, "a ring piece touches at most two pool chunks");
            const uint32_t head = chunk_tab ? 0u : min(cnt, static_cast<uint32_t>(
                                                               ((16 - (reinterpret_cast<uintptr_t>(src) & 15)) & 15) / 4));
            const uint32_t body = (cnt - head) & ~3u;
            const uint32_t nchunks = (body + piece - 1) / piece;
            auto set_key = [&](uint32_t key) {
                const uint32_t x = key - key_lo;
                atomicOr(s_bits + (x >> 5), 1u << (x & 31));
            };
            auto at = [&](uint32_t k) {  // address of the bucket's k-th key slot
                return chunk_tab ? chunk_src(k >> chunk_shift) + (k & (CH - 1u)) : src + k;
            };
            auto issue = [&](uint32_t c) {  // thread 0
                const unsigned g = chunk_seq + c;
                const uint32_t len = min(piece, body - c * piece);
                uint32_t* dst = s_stage_all + (g % KB4_RING) * kChunk;
                fence_proxy_async_smem();
                const uint32_t k0 = head + c * piece;
                const uint32_t first = chunk_tab ? min(len, CH - (k0 & (CH - 1u))) : len;
                if (first == len) {
                    tma_load_bytes(dst, at(k0), len * 4, &s_lbar[g % KB4_RING]);
                } else {  // the piece crosses into the next pool chunk: one arrival, two copies
                    unsigned long long* bar = &s_lbar[g % KB4_RING];
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                                 "r"(len * 4)
                                 : "memory");
                    tma_copy_bytes(dst, at(k0), first * 4, bar);
                    tma_copy_bytes(dst + first, at(k0 + first), (len - first) * 4, bar);
                }
            };
            if (threadIdx.x == 0) {
                for (uint32_t q = 0; q < KB4_RING && q < nchunks; ++q) issue(q);
            }
            if (threadIdx.x < head) set_key(__ldcs(src + threadIdx.x));
            if (threadIdx.x < cnt - head - body) set_key(__ldcs(at(head + body + threadIdx.x)));
            for (uint32_t c = 0; c < nchunks; ++c) {
                const unsigned g = chunk_seq + c;
                mbar_wait(&s_lbar[g % KB4_RING], (g / KB4_RING) & 1u);
                const uint4* r4 = reinterpret_cast<const uint4*>(s_stage_all + (g % KB4_RING) * kChunk);
                const uint32_t nv = min(piece, body - c * piece) / 4;
                for (uint32_t i = threadIdx.x; i < nv; i += NT) {
                    const uint4 v = r4[i];
                    set_key(v.x);
                    set_key(v.y);
                    set_key(v.z);
                    set_key(v.w);
                }
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&s_ebar[g % KB4_RING])) : "memory");
                if (threadIdx.x == 0 && c + KB4_RING < nchunks) {  // refill once every thread is done with the slot
                    mbar_wait(&s_ebar[g % KB4_RING], (g / KB4_RING) & 1u);
                    issue(c + KB4_RING);
                }
            }
            chunk_seq += nchunks;
        }
        __syncthreads();
        // phase 1: per-warp popcount of its segment (128-bit SMEM reads; sparse
        // buckets read only the touched words, found through the summary)
        const uint32_t seg = warp * seg_words;
        uint32_t c = 0;
        uint32_t c_first = 0;  // sparse: this lane's count of its first summary word (reused below)
        if (sparse) {
            for (uint32_t i = lane; i < seg_words / 32; i += 32) {
                const uint32_t si = seg / 32 + i;
                uint32_t ci = 0;
                for (uint32_t m = s_sum[si]; m; m &= m - 1) ci += __popc(s_bits[si * 32 + (__ffs(m) - 1)]);
                if (i == lane) c_first = ci;
                c += ci;
            }
        } else {
            for (uint32_t i = lane; i < seg_words / 4; i += 32) {
                const uint4 v = s4[seg / 4 + i];
                c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
            }
        }
        c = __reduce_add_sync(kFull, c);
        if (lane == 0) s_warp[warp] = c;
        __syncthreads();
        // every warp scans the (<= 32) segment counts itself: no second barrier
        uint32_t wprefix;
        {
            constexpr unsigned NWARP = NT / 32;
            const uint32_t v = lane < NWARP ? s_warp[lane] : 0u;
            const uint32_t incl = warp_incl_scan(v, lane);
            wprefix = __shfl_sync(kFull, incl - v, warp);
            if (warp == 0 && lane == 31 && incl) atomicAdd(&ctrl->total, static_cast<unsigned long long>(incl));
        }
        uint32_t* o = out + base + wprefix;
        // output keys: bucket base + bit index, mapped back by the XOR (signed sorts use
        // power-of-two widths, so no bucket straddles 2^31 and the XOR commutes with the add)
        const uint32_t key_hi = (bm.lo + static_cast<uint32_t>(b) * bm.width) ^ bm.xr;
        if (sparse) {
            // lane-major over summary words: lane owns 32 consecutive bitset
            // words (one summary word) per round; its keys are contiguous in
            // the output at its prefix offset. Touched words are zeroed.
            for (uint32_t i0 = 0; i0 < seg_words / 32; i0 += 32) {
                const uint32_t si = seg / 32 + i0 + lane;
                uint32_t m = i0 + lane < seg_words / 32 ? s_sum[si] : 0u;
                uint32_t cl = c_first;  // the first round's counts come from phase 1
                if (i0 > 0) {
                    cl = 0;
                    for (uint32_t mm = m; mm; mm &= mm - 1) cl += __popc(s_bits[si * 32 + (__ffs(mm) - 1)]);
                }
                const uint32_t incl = warp_incl_scan(cl, lane);
                const uint32_t ctot = __shfl_sync(kFull, incl, 31);
                if (ctot == 0) continue;
                uint32_t* ol = o + (incl - cl);
                if (m) s_sum[si] = 0u;
                while (m) {
                    const uint32_t t = static_cast<uint32_t>(__ffs(m) - 1);
                    m &= m - 1;
                    const uint32_t wi = si * 32 + t;
                    uint32_t x = s_bits[wi];
                    s_bits[wi] = 0u;
                    const uint32_t kb = key_hi + (wi << 5);
                    while (x) {
                        const int bt = __ffs(x) - 1;
                        x &= x - 1;
                        __stcs(ol++, kb + static_cast<uint32_t>(bt));
                    }
                }
                o += ctot;
            }
        } else if (seg_words % 512 == 0) {
            extract_span512<STAGE>(s_bits, seg, seg_words, key_hi, o, s_stage, lane, false, nullptr);
        } else if (seg_words % 128 == 0) {
            // 128-word steps, lane-major (lane owns 4 words); a step with
            // <= STAGE keys is extracted in one pass, denser steps as two
            // 64-word sub-steps (two words per lane)
            for (uint32_t w0 = 0; w0 < seg_words; w0 += 128) {
                const uint4 v = s4[(seg + w0) / 4 + lane];
                const uint32_t cl = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
                const uint32_t incl = warp_incl_scan(cl, lane);
                const uint32_t ctot = __shfl_sync(kFull, incl, 31);
                if (ctot == 0) continue;
                if (ctot <= static_cast<uint32_t>(STAGE)) {
                    uint32_t p = incl - cl;
                    const uint32_t kb = key_hi + ((seg + w0 + 4 * lane) << 5);
                    stage_bits(v.x, kb, p, s_stage);
                    stage_bits(v.y, kb + 32, p, s_stage);
                    stage_bits(v.z, kb + 64, p, s_stage);
                    stage_bits(v.w, kb + 96, p, s_stage);
                    drain_stage(s_stage, ctot, o, lane);
                    o += ctot;
                    continue;
                }
                if (ctot > 2u * STAGE) {  // dense: word-by-word ballots
#pragma unroll 1
                    for (uint32_t q = 0; q < 128; q += 32)
                        o += extract_words32<STAGE>(s_bits, seg + w0 + q, key_hi, o, s_stage, lane);
                    continue;
                }
                const uint32_t n0 = extract_words64<STAGE>(s_bits, seg + w0, key_hi, o, s_stage, lane);
                o += n0 + extract_words64<STAGE>(s_bits, seg + w0 + 64, key_hi, o + n0, s_stage, lane);
            }
        } else {
            for (uint32_t w0 = 0; w0 < seg_words; w0 += 32)
                o += extract_words32<STAGE>(s_bits, seg + w0, key_hi, o, s_stage, lane);
        }
        dirty = !sparse;
        __syncthreads();
    }
}


// KB4m (multiset sorts, bws_sort on input with repeated keys): the counting
// sort of a bucket (baselines.hpp:99-122's counting_sort with the bucket as its
// span) in shared memory. The bucket's width is covered by windows of values
// with SMEM counters — 16-bit counters over 2^16 values when the bucket holds
// fewer than 2^16 keys (no counter can overflow), else 32-bit counters over
// 2^15 values. Per window: one counting pass over the bucket's keys (staged in
// SMEM once when they fit, else 16-byte-batched loads), a block-wide
// inclusive prefix of the counters (lane-rotated LDS.128, conflict-free) and
// the expansion — output slot i of the window takes the value whose prefix
// first exceeds i (binary search), so a value repeated 2^26 times is written by
// all threads, coalesced. Windows with no keys are skipped (per-window counts
// from a first pass). The output range of a bucket is the prefix of the bucket
// totals (packed layout: the same slots the bucket occupies in `parted`).
// Adds every key it writes to ctrl->total.
constexpr int MS_THREADS = 1024;
constexpr int MS_CNT_BYTES = 128 << 10;          // counter area
constexpr int MS_STAGE_KEYS = 16384;             // keys staged in SMEM (64 KB)
constexpr int MS_MAX_WIN = (1 << MAX_BUCKET_SHIFT) / (1 << 15);  // 32
constexpr std::size_t ms_smem_bytes() { return MS_CNT_BYTES + MS_STAGE_KEYS * 4; }
__global__ void __launch_bounds__(MS_THREADS, 1)
    bucket_multiset_kernel(const uint32_t* __restrict__ parted, const uint32_t* __restrict__ tot,
                           const unsigned long long* __restrict__ g_base, BucketMap bm, int nb,
                           uint32_t* __restrict__ out, Ctrl* __restrict__ ctrl, uint32_t src_cap) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem_raw);  // counters, then inclusive prefix
    uint16_t* s_cnt16 = reinterpret_cast<uint16_t*>(smem_raw);
    uint32_t* s_keys = reinterpret_cast<uint32_t*>(smem_raw + MS_CNT_BYTES);
    __shared__ uint32_t s_wc[MS_MAX_WIN];                     // keys per window of the bucket
    __shared__ uint32_t s_warp[MS_THREADS / 32];
    __shared__ unsigned s_b;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long written = 0;  // thread 0
    for (;;) {
        if (threadIdx.x == 0) s_b = atomicAdd(&ctrl->ticket, 1u);
        if (threadIdx.x < MS_MAX_WIN) s_wc[threadIdx.x] = 0u;
        __syncthreads();
        const unsigned b = s_b;
        if (b >= static_cast<unsigned>(nb)) break;
        const uint32_t cnt = tot[b];
        const unsigned long long base = g_base[b];
        // packed layout: the bucket's keys sit where its output goes; slab
        // layout (in-place recovery): its slab, padding (x == width) dropped
        const uint32_t* src = parted + (src_cap ? static_cast<size_t>(b) * src_cap : base);
        const uint32_t key_lo = bm.lo + static_cast<uint32_t>(b) * bm.width;
        const bool c16 = cnt < 65536u;           // block-uniform
        const int wshift = c16 ? 16 : 15;
        const uint32_t win = 1u << wshift;
        const uint32_t nwin = (bm.width + win - 1) >> wshift;
        const bool staged = cnt <= static_cast<uint32_t>(MS_STAGE_KEYS);
        if (staged)
            for (uint32_t i = threadIdx.x; i < cnt; i += MS_THREADS) s_keys[i] = src[i] - key_lo;
        // visits every key of the bucket (offset from key_lo) in batches of
        // four independent loads per thread
        auto for_keys = [&](auto&& f) {
            if (staged) {
                for (uint32_t i = threadIdx.x; i < cnt; i += MS_THREADS)
                    if (s_keys[i] < bm.width) f(s_keys[i], true);
                return;
            }
            uint32_t i0 = 0;
            for (; i0 + 4 * MS_THREADS <= cnt; i0 += 4 * MS_THREADS) {
                uint32_t v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldcg(src + i0 + u * MS_THREADS + threadIdx.x);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (v[u] - key_lo < bm.width) f(v[u] - key_lo, true);
            }
            for (uint32_t i = i0 + threadIdx.x; i < cnt; i += MS_THREADS)
                if (src[i] - key_lo < bm.width) f(src[i] - key_lo, true);
        };
        __syncthreads();
        // pass 0: keys per window (warp-aggregated: one SMEM atomic per window per warp step)
        if (nwin == 1 && !src_cap) {  // (slab slots also hold padding: counted below)
            if (threadIdx.x == 0) s_wc[0] = cnt;
        } else {
            const uint32_t rounds = (cnt + MS_THREADS - 1) / MS_THREADS;  // every lane takes part in the match
            for (uint32_t r = 0; r < rounds; ++r) {
                const uint32_t i = r * MS_THREADS + threadIdx.x;
                const uint32_t x = i < cnt ? (staged ? s_keys[i] : src[i] - key_lo) : 0u;
                const uint32_t w = i < cnt && x < bm.width ? x >> wshift : 0xffffffffu;
                const unsigned peers = __match_any_sync(kFull, w);
                if (w != 0xffffffffu && lane == static_cast<unsigned>(__ffs(peers) - 1))
                    atomicAdd(&s_wc[w], static_cast<uint32_t>(__popc(peers)));
            }
        }
        __syncthreads();
        unsigned long long o = base;
        for (uint32_t w = 0; w < nwin; ++w) {
            const uint32_t wk = s_wc[w];  // block-uniform
            if (wk == 0) continue;
            uint4* c4 = reinterpret_cast<uint4*>(s_cnt);
            for (uint32_t i = threadIdx.x; i < MS_CNT_BYTES / 16; i += MS_THREADS) c4[i] = make_uint4(0, 0, 0, 0);
            __syncthreads();
            const uint32_t wlo = w << wshift;
            if (c16) {
                for_keys([&](uint32_t x, bool) {
                    x -= wlo;
                    if (x < win) atomicAdd(s_cnt + (x >> 1), 1u << ((x & 1u) << 4));
                });
            } else {
                for_keys([&](uint32_t x, bool) {
                    x -= wlo;
                    if (x < win) atomicAdd(s_cnt + x, 1u);
                });
            }
            __syncthreads();
            // inclusive prefix of the counters: warp w owns words [1024w, 1024w + 1024),
            // lane l the words 1024w + 32j + l (conflict-free); pass A: warp
            // totals; pass B: row-by-row warp scans carrying the running sum
            const uint32_t* wrow = s_cnt + warp * 1024 + lane;
            uint32_t part = 0;
#pragma unroll 8
            for (int j = 0; j < 32; ++j) {
                const uint32_t x = wrow[32 * j];
                part += c16 ? (x & 0xffffu) + (x >> 16) : x;
            }
            part = __reduce_add_sync(kFull, part);
            if (lane == 0) s_warp[warp] = part;
            __syncthreads();
            if (warp == 0) {
                const uint32_t x = s_warp[lane];
                s_warp[lane] = warp_incl_scan(x, lane) - x;
            }
            __syncthreads();
            uint32_t carry = s_warp[warp];
            uint32_t* wrow_w = s_cnt + warp * 1024 + lane;
#pragma unroll 4
            for (int j = 0; j < 32; ++j) {
                const uint32_t x = wrow_w[32 * j];
                const uint32_t sum = c16 ? (x & 0xffffu) + (x >> 16) : x;
                const uint32_t incl = warp_incl_scan(sum, lane);
                const uint32_t excl = carry + incl - sum;
                wrow_w[32 * j] = c16 ? ((excl + (x & 0xffffu)) | ((excl + sum) << 16)) : excl + sum;
                carry += __shfl_sync(kFull, incl, 31);
            }
            __syncthreads();
            // expansion: slot i holds the smallest value whose inclusive prefix exceeds i
            const uint32_t kbase = key_lo + wlo;
            for (uint32_t i = threadIdx.x; i < wk; i += MS_THREADS) {
                uint32_t lo = 0, len = win;
#pragma unroll 1
                while (len > 1) {
                    const uint32_t half = len >> 1;
                    const uint32_t pv = c16 ? s_cnt16[lo + half - 1] : s_cnt[lo + half - 1];
                    if (pv <= i) lo += half;
                    len -= half;
                }
                __stcs(out + o + i, (kbase + lo) ^ bm.xr);
            }
            o += wk;
            __syncthreads();
        }
        if (threadIdx.x == 0) written += o - base;  // keys written (slab padding excluded)
    }
    if (threadIdx.x == 0 && written) atomicAdd(&ctrl->total, written);
}

// KB4b (multi-GPU per-rank build): like KB4, but instead of extracting keys
// each bucket's SMEM bitset is written to the global bitset, coalesced and
// without atomics; every word below n_words is written, so the caller's
// bitset needs no clearing.
__global__ void __launch_bounds__(BUCKET_THREADS, 1)
    bucket_bitset_kernel(const uint32_t* __restrict__ parted, const uint32_t* __restrict__ tot,
                         const unsigned long long* __restrict__ g_base, BucketMap bm, int nb,
                         uint32_t src_cap, uint32_t* __restrict__ bits, unsigned long long n_words,
                         uint32_t last_mask, Ctrl* __restrict__ ctrl) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t W = bm.width >> 5;
    uint32_t* s_bits = reinterpret_cast<uint32_t*>(smem_raw);
    __shared__ unsigned s_b;
    uint4* s4 = reinterpret_cast<uint4*>(s_bits);
    for (;;) {
        if (threadIdx.x == 0) s_b = atomicAdd(&ctrl->ticket, 1u);
        for (uint32_t i = threadIdx.x; i < W / 4; i += BUCKET_THREADS) s4[i] = make_uint4(0, 0, 0, 0);
        __syncthreads();
        const unsigned b = s_b;
        if (b >= static_cast<unsigned>(nb)) break;
        scatter_bucket_keys<false>(parted + (src_cap ? static_cast<size_t>(b) * src_cap : g_base[b]), tot[b],
                                   bm.lo + static_cast<uint32_t>(b) * bm.width, bm.width, s_bits, nullptr);
        __syncthreads();
        const unsigned long long w0 = static_cast<unsigned long long>(b) * W;
        // keys in [key_range, 32 * n_words) of a non-multiple-of-32 range never appear
        if (threadIdx.x == 0 && n_words - 1 >= w0 && n_words - 1 < w0 + W) s_bits[n_words - 1 - w0] &= last_mask;
        __syncthreads();
        if (w0 + W <= n_words && (reinterpret_cast<uintptr_t>(bits) & 15) == 0) {
            uint4* g4 = reinterpret_cast<uint4*>(bits + w0);
            for (uint32_t i = threadIdx.x; i < W / 4; i += BUCKET_THREADS) __stcs(g4 + i, s4[i]);
        } else {
            for (uint32_t i = threadIdx.x; i < W; i += BUCKET_THREADS)
                if (w0 + i < n_words) bits[w0 + i] = s_bits[i];
        }
        __syncthreads();
    }
}


// KB4p (multi-GPU push build, the exchange fused into the build): like KB4b,
// but each bucket's finished SMEM bitset leaves with one bulk OR-reduction
// per destination slice (cp.reduce.async.bulk ... .or.b32) straight into the
// owner rank's slice buffer — peer memory over NVLink/NVSwitch through CUDA
// IPC, or local memory for the rank's own slice. The L2 of the owner applies
// the OR, so pushes from all ranks into one slice need no other
// synchronisation; distinct keys set disjoint bits, so OR is exact, and
// repeats only lose bits (the popcount total reports them). Slice r covers
// words [r * slice_words, (r + 1) * slice_words) (slice_words a multiple of
// 4: bulk operations move 16-byte units).
__global__ void __launch_bounds__(BUCKET_THREADS, 1)
    bucket_push_kernel(const uint32_t* __restrict__ parted, const uint32_t* __restrict__ tot,
                       const unsigned long long* __restrict__ g_base, BucketMap bm, int nb, uint32_t src_cap,
                       OrSources slices, unsigned long long slice_words, unsigned long long n_words,
                       uint32_t last_mask, Ctrl* __restrict__ ctrl) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t W = bm.width >> 5;
    uint32_t* s_bits = reinterpret_cast<uint32_t*>(smem_raw);
    __shared__ unsigned s_b;
    uint4* s4 = reinterpret_cast<uint4*>(s_bits);
    const unsigned long long total_words = slice_words * static_cast<unsigned long long>(slices.n);
    for (;;) {
        if (threadIdx.x == 0) {
            // the previous bucket's bulk reductions must have read s_bits
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            s_b = atomicAdd(&ctrl->ticket, 1u);
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < W / 4; i += BUCKET_THREADS) s4[i] = make_uint4(0, 0, 0, 0);
        __syncthreads();
        const unsigned b = s_b;
        if (b >= static_cast<unsigned>(nb)) break;
        scatter_bucket_keys<false>(parted + (src_cap ? static_cast<size_t>(b) * src_cap : g_base[b]), tot[b],
                                   bm.lo + static_cast<uint32_t>(b) * bm.width, bm.width, s_bits, nullptr);
        __syncthreads();
        const unsigned long long w0 = static_cast<unsigned long long>(b) * W;
        if (threadIdx.x == 0 && n_words - 1 >= w0 && n_words - 1 < w0 + W) s_bits[n_words - 1 - w0] &= last_mask;
        fence_proxy_async_smem();  // generic-proxy SMEM writes -> visible to the bulk reductions
        __syncthreads();
        if (threadIdx.x == 0) {
            // one bulk OR per slice the bucket's words [w0, w0 + W) overlap
            const unsigned long long end = min(w0 + W, total_words);
            unsigned long long w = w0;
#pragma unroll 1
            while (w < end) {
                const int r = static_cast<int>(w / slice_words);
                const unsigned long long seg_end = min(end, static_cast<unsigned long long>(r + 1) * slice_words);
                uint32_t* dst = const_cast<uint32_t*>(slices.p[r]) + (w - static_cast<unsigned long long>(r) * slice_words);
                const uint32_t bytes = static_cast<uint32_t>(seg_end - w) * 4u;
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.or.b32 [%0], [%1], %2;" ::"l"(dst),
                             "r"(smem_u32(s_bits + (w - w0))), "r"(bytes)
                             : "memory");
                w = seg_end;
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // reductions performed
        __threadfence_system();
    }
}

// K0: max key (only when no key-range hint is given).
__global__ void key_max_kernel(const uint32_t* __restrict__ keys, size_t n, Ctrl* __restrict__ ctrl,
                               uint32_t xr) {
    uint32_t mx = 0, mn = 0xffffffffu;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t tid = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    auto fold = [&](uint32_t k) {
        k ^= xr;
        mx = max(mx, k);
        mn = min(mn, k);
    };
    // 16-byte loads over the aligned body, four in flight per thread
    size_t head = ((16 - (reinterpret_cast<uintptr_t>(keys) & 15)) & 15) / 4;
    if (head > n) head = n;
    const uint4* v4 = reinterpret_cast<const uint4*>(keys + head);
    const size_t nv = (n - head) / 4;
    size_t i = tid;
    for (; i + 3 * stride < nv; i += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcs(v4 + i + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            fold(v[u].x);
            fold(v[u].y);
            fold(v[u].z);
            fold(v[u].w);
        }
    }
    for (; i < nv; i += stride) {
        const uint4 v = __ldcs(v4 + i);
        fold(v.x);
        fold(v.y);
        fold(v.z);
        fold(v.w);
    }
    if (tid < head) fold(keys[tid]);
    for (size_t j = head + 4 * nv + tid; j < n; j += stride) fold(keys[j]);
    mx = __reduce_max_sync(kFull, mx);
    mn = __reduce_min_sync(kFull, mn);
    if ((threadIdx.x & 31) == 0) {
        if (mx) atomicMax(&ctrl->max_key, mx);
        if (~mn) atomicMax(&ctrl->min_inv, ~mn);
    }
}

}  // namespace

// The narrow KB3 variant (2 CTAs/SM, 8192-key tiles) measured slower than the
// wide one on C2 (profiles/r01_*): shorter bucket runs add partial-sector
// DRAM traffic. It stays selectable for experiments (BITSORT_PART=narrow).
static bool narrow_partition(const BucketPlan& plan) {
    static const bool want = [] {
        const char* e = std::getenv("BITSORT_PART");
        return e && std::string(e) == "narrow";
    }();
    return want && plan.nb <= PART_NARROW_MAXB;
}

cudaError_t launch_key_max(const uint32_t* keys, size_t n, Ctrl* ctrl, const LaunchGeometry& geo,
                           cudaStream_t stream, uint32_t xr) {
    key_max_kernel<<<geo.fill_blocks, 256, 0, stream>>>(keys, n, ctrl, xr);
    return cudaGetLastError();
}

static BucketMap pow2_map(int shift) {
    BucketMap m;
    m.ms = shift;
    m.mq = 1u << 20;
    m.width = 1u << shift;
    return m;
}

BucketPlan plan_buckets(uint64_t key_range, int kb4_ctas) {
    BucketPlan p;
    int log2m = 0;
    while ((1ull << log2m) < key_range) ++log2m;
    // About 256 buckets: KB3 runs faster with fewer buckets (longer runs per
    // tile; measured C2: 256 buckets 177 us vs 1024 buckets 256 us) and KB4
    // still has enough of them. Ranges above 2^28 take 2^20-key buckets (the
    // largest SMEM bitset) and more of them, up to MAX_BUCKETS. (A cluster
    // KB4 with DSMEM bitsets for wider buckets measured 6.7x slower on C3:
    // profiles/r01_cluster_kb4_experiment.json.)
    int shift = log2m - 8;
    const char* env = std::getenv("BITSORT_BUCKET_SHIFT");  // experiments
    if (env) shift = std::atoi(env);
    while (shift < MAX_BUCKET_SHIFT && ((key_range + (1ull << shift) - 1) >> shift) > MAX_BUCKETS) ++shift;
    if (shift > MAX_BUCKET_SHIFT) shift = MAX_BUCKET_SHIFT;
    if (shift < MIN_BUCKET_SHIFT) shift = MIN_BUCKET_SHIFT;
    p.shift = shift;
    p.map = pow2_map(shift);
    const uint64_t nb = (key_range + (1ull << shift) - 1) >> shift;
    p.nb = static_cast<int>(nb < 1 ? 1 : nb);
    // Widest buckets: KB4 runs ceil(nb / CTAs) rounds of one bucket per CTA,
    // so 256 buckets on 148 SMs leave 40 SMs idle in the second round. Widths
    // q * 2^17 (q = 5..7; KB4's warp segments need multiples of 2^17 keys)
    // can fill the rounds better: C2 (2^28 keys) -> 293 buckets of 7 * 2^17,
    // two full rounds at 7/8 of the work each. Ties keep the wider buckets
    // (fewer KB3 runs).
    if (shift == MAX_BUCKET_SHIFT && kb4_ctas > 0 && !env && !std::getenv("BITSORT_POW2_BUCKETS")) {
        auto rounds = [&](uint64_t n) { return (n + kb4_ctas - 1) / kb4_ctas; };
        uint64_t best = rounds(nb) * 8;
        for (uint32_t q = 7; q >= 5; --q) {
            const uint64_t w = static_cast<uint64_t>(q) << 17;
            const uint64_t nq = (key_range + w - 1) / w;
            if (nq > static_cast<uint64_t>(MAX_BUCKETS)) break;
            if (rounds(nq) * q < best) {
                best = rounds(nq) * q;
                p.map.ms = 17;
                p.map.mq = ((1u << 20) + q - 1) / q;
                p.map.width = static_cast<uint32_t>(w);
                p.nb = static_cast<int>(nq);
            }
        }
    }
    return p;
}

BucketPlan plan_multiset(uint64_t key_range) {
    // KB4m covers a bucket in 2^15-value windows, one pass over the bucket's
    // keys per window: the narrowest buckets KB3 allows (<= MAX_BUCKETS) keep
    // that at one or two passes below 2^28 values, and give KB4m more
    // buckets than SMs
    int log2m = 0;
    while ((1ull << log2m) < key_range) ++log2m;
    int shift = log2m - 12;
    if (shift < MIN_BUCKET_SHIFT) shift = MIN_BUCKET_SHIFT;
    if (shift > MAX_BUCKET_SHIFT) shift = MAX_BUCKET_SHIFT;
    BucketPlan p;
    p.shift = shift;
    p.map = pow2_map(shift);
    const uint64_t nb = (key_range + (1ull << shift) - 1) >> shift;
    p.nb = static_cast<int>(nb < 1 ? 1 : nb);
    return p;
}

BucketPlan plan_range_split(uint64_t key_range, int parts) {
    BucketPlan p;
    const uint64_t want = (key_range + parts - 1) / parts;
    uint64_t best = 0;
    int best_s = 12;
    uint32_t best_q = 1;
    for (int s = 12; s <= 31; ++s) {  // (key >> 32 would be undefined)
        for (uint32_t q = 1; q <= 8; ++q) {
            const uint64_t w = static_cast<uint64_t>(q) << s;
            if (w < want || (q > 1 && s < 15)) continue;  // q > 1 needs s >= 15 for an exact map
            if (best == 0 || w < best) {
                best = w;
                best_s = s;
                best_q = q;
            }
        }
    }
    p.map.ms = best_s;
    p.map.mq = ((1u << 20) + best_q - 1) / best_q;
    p.map.width = best >= (1ull << 32) ? 0xffffffffu : static_cast<uint32_t>(best);
    p.shift = MAX_BUCKET_SHIFT;
    p.nb = parts;
    p.partition_only = true;
    return p;
}

const uint32_t* bucket_totals(const void* scratch, const BucketPlan& plan, const LaunchGeometry& geo) {
    const int P = narrow_partition(plan) ? geo.part_blocks_narrow : geo.part_blocks;
    return static_cast<const uint32_t*>(scratch) + 2 * MAX_BUCKETS + static_cast<size_t>(P) * plan.nb;
}

// The bulk-store KB3 (bucket_partition_tma_kernel) takes slab sorts with <= 1024 buckets.
static bool tma_store_kb3(const BucketPlan& plan) {
    static const bool off = [] {
        const char* e = std::getenv("BITSORT_TMA_STORE");
        return e && std::string(e) == "0";
    }();
    // runs average TILE / nb keys per tile: at 1024 buckets (C3, 16-key runs)
    // the padding and ~1000 small copies per tile cost more than they save
    return !off && plan.nb <= 512 && !narrow_partition(plan);
}

uint64_t slab_slots(const BucketPlan& plan, size_t n) {
    static const bool off = [] {
        const char* e = std::getenv("BITSORT_SLAB");
        return e && std::string(e) == "0";
    }();
    if (off || plan.partition_only) return 0;
    uint64_t cap = (static_cast<uint64_t>(n) + 3) & ~uint64_t(3);
    if (cap > plan.map.width) cap = plan.map.width;
    // bulk-store runs are padded to multiples of 4: at most 3 extra slots per
    // bucket per tile (KB3 CTAs <= 1024) plus the head/tail claims
    if (tma_store_kb3(plan)) cap += 3 * (static_cast<uint64_t>(n) / PART_TILE + 1024 + 8);
    cap = (cap + 3) & ~uint64_t(3);  // bucket slabs and the dump tile stay 16-byte aligned
    const uint64_t slots = static_cast<uint64_t>(plan.nb) * cap + PART_DUMP;  // + dump tile
    // the slab trades memory (up to 4.5 slots per key, or 256 MiB for small
    // sorts) for the histogram pass
    const bool small = slots * 4 <= (uint64_t(256) << 20);
    if ((!small && slots > 4 * static_cast<uint64_t>(n) + n / 2 + PART_DUMP) || slots >= (1ull << 32)) return 0;
    return slots;
}

// Chunked layout (the packed layout's replacement for distinct-key sorts:
// no KB1 histogram read, no KB2): pool slots for n keys in nb buckets.
// Pool chunk id starts at slot id * (2^shift + pad), pad = BITSORT_CHUNK_PAD
// slots (default 0). An experiment knob: C4's KB3 measures 105 us when the
// pool is allocated before the 512 MiB cached bitset and 151 us when after it
// (a C1 sort first); taking the chunk starts off their power-of-two stride
// (pad 32 .. 1056) changed neither figure, so the stride is not the cause
// (profiles/r02_order_probe.log).
uint32_t chunk_pad_slots() {
    static const uint32_t pad = [] {
        const char* e = std::getenv("BITSORT_CHUNK_PAD");
        const long v = e ? std::atol(e) : 0;
        return static_cast<uint32_t>(v < 0 ? 0 : (v > 4096 ? 4096 : v)) & ~3u;
    }();
    return pad;
}
constexpr uint32_t kMaxChunksPerBucket = (1u << MAX_BUCKET_SHIFT) / KC_CHUNK_MIN + 2;
// Chunk size: about a quarter of a bucket's mean key count (few allocations,
// at most a quarter-bucket of pool slots wasted per bucket), 2^13 .. 2^16.
uint32_t chunk_shift(const BucketPlan& plan, size_t n) {
    const uint64_t per = static_cast<uint64_t>(n) / (4ull * static_cast<uint64_t>(plan.nb));
    uint32_t s = 13;
    while (s < 16 && (uint64_t(1) << (s + 1)) <= per) ++s;
    return s;
}
uint32_t chunk_max(const BucketPlan& plan, size_t n) {
    const uint64_t cap = std::min<uint64_t>(plan.map.width, n);
    const uint64_t ch = uint64_t(1) << chunk_shift(plan, n);
    return static_cast<uint32_t>((cap + ch - 1) / ch + 1);
}
uint64_t chunk_slots(const BucketPlan& plan, size_t n) {
    static const bool off = [] {
        const char* e = std::getenv("BITSORT_CHUNK");
        return e && std::string(e) == "0";
    }();
    if (off || plan.partition_only || plan.nb > MAX_BUCKETS) return 0;
    const uint64_t ch = uint64_t(1) << chunk_shift(plan, n);
    const uint64_t chunks = static_cast<uint64_t>(n) / ch + plan.nb + 2;  // implicit chunk 0 per bucket
    const uint64_t slots = chunks * (ch + chunk_pad_slots());
    return slots < (1ull << 32) - ch ? slots : 0;
}

bool slab_in_use(const BucketPlan& plan, size_t n, uint64_t parted_cap) {
    const uint64_t slab = slab_slots(plan, n);
    return slab != 0 && slab <= parted_cap;
}

size_t bucket_scratch_bytes(const BucketPlan& plan, int hist_blocks) {
    return static_cast<size_t>(hist_blocks) * plan.nb * sizeof(uint32_t)  // H
           + (MAX_BUCKETS + 1) * sizeof(uint32_t)                          // tot
           + (MAX_BUCKETS + 2) * sizeof(unsigned long long)                // base (8-aligned)
           + MAX_BUCKETS * sizeof(uint32_t)                                // KB4 ticket order
           + 2 * MAX_BUCKETS * sizeof(uint32_t)                            // slab fill + true counts
           + (8 + static_cast<size_t>(MAX_BUCKETS) * kMaxChunksPerBucket) * sizeof(uint32_t);  // chunks
}

cudaError_t launch_bucket_sort(const uint32_t* keys, size_t n, uint64_t key_range, uint32_t* out,
                               uint32_t* parted, void* scratch, Ctrl* ctrl, const BucketPlan& plan,
                               const LaunchGeometry& geo, cudaStream_t stream, int* launches,
                               KernelTimer* timer, uint32_t* bits_out, uint64_t n_words,
                               uint64_t parted_cap, bool multiset, const OrSources* push,
                               uint64_t push_slice_words, int inplace_mode) {
    if (n == 0) return cudaSuccess;
    const int P = narrow_partition(plan) ? geo.part_blocks_narrow : geo.part_blocks;
    // scratch: slab fill counters (fixed place: they persist across sorts), then H, tot, base
    uint32_t* gcnt = static_cast<uint32_t*>(scratch);  // then the true counts (bulk-store KB3)
    uint32_t* H = gcnt + 2 * MAX_BUCKETS;
    uint32_t* tot = H + static_cast<size_t>(P) * plan.nb;
    unsigned long long* base =
        reinterpret_cast<unsigned long long*>(reinterpret_cast<uintptr_t>(tot + MAX_BUCKETS + 1) & ~uintptr_t(7));
    // KB4 ticket order (packed layout only; slab buckets are uniform in C2/C3)
    uint32_t* order_buf = reinterpret_cast<uint32_t*>(base + MAX_BUCKETS + 2);
    const int check = key_range < (1ull << 32);
    const uint32_t limit = check ? static_cast<uint32_t>(key_range) : 0u;
    KeySplit ks;
    const uintptr_t addr = reinterpret_cast<uintptr_t>(keys);
    size_t n_head = ((16 - (addr & 15)) & 15) / 4;
    if (n_head > n) n_head = n;
    ks.nv = (n - n_head) / 4;
    ks.body = reinterpret_cast<const uint4*>(keys + n_head);
    ks.head = keys;
    ks.n_head = static_cast<int>(n_head);
    ks.tail = keys + n_head + 4 * ks.nv;
    ks.n_tail = static_cast<int>(n - n_head - 4 * ks.nv);
    ks.xr = plan.map.xr;

    const uint64_t slab = slab_slots(plan, n);
    // multiset sorts take the packed layout: exact for any key multiplicity
    const bool use_slab = !multiset && slab != 0 && slab <= parted_cap;
    // distinct-key sorts that do not fit the slab: the chunked layout (no
    // KB1/KB2); the multiset, range-split and multi-GPU builds keep the packed one
    const uint64_t cslots = chunk_slots(plan, n);
    const bool use_chunk = !use_slab && !multiset && !bits_out && !push && !plan.partition_only &&
                           inplace_mode == 0 && cslots != 0 && cslots <= parted_cap;
    uint32_t* pool_next = order_buf + MAX_BUCKETS + 4;  // (order[nb] is written) then the chunk table
    uint32_t* chunk_tab = pool_next + 4;
    static const bool order_off = [] {
        const char* e = std::getenv("BITSORT_KB4_ORDER");
        return e && std::string(e) == "0";
    }();
    uint32_t* kb4_order =
        (!use_slab && !plan.partition_only && !multiset && !bits_out && !push && !order_off && plan.nb > 1) ? order_buf
                                                                                                    : nullptr;
    SlabArgs sa;
    int nlaunch = 0;
    cudaError_t err;
    if (inplace_mode == 2) {
        // recovery of an in-place sort whose keys repeat: the previous slab
        // KB3 (same keys, plan, buffers) left the exact multiset in its slabs
        // (padding is out of bucket) and the totals/offsets in the scratch;
        // KB4m counting-sorts every bucket from its slab into out
        if (!use_slab) return cudaErrorInvalidValue;
        const uint32_t cap = static_cast<uint32_t>((slab - PART_DUMP) / plan.nb) & ~3u;
        if (timer) timer->before(stream);
        bucket_multiset_kernel<<<geo.multiset_blocks, MS_THREADS, ms_smem_bytes(), stream>>>(
            parted, tot, base, plan.map, plan.nb, out, ctrl, cap);
        if (timer) timer->after("bucket_multiset", stream);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        if (launches) *launches = 1;
        return cudaSuccess;
    }
    if (use_chunk) {
        const uint32_t maxc = chunk_max(plan, n);
        err = cudaMemsetAsync(pool_next, 0, (4 + static_cast<size_t>(plan.nb) * maxc) * sizeof(uint32_t), stream);
        if (err != cudaSuccess) return err;
        sa.gcnt = gcnt;
        sa.gtrue = nullptr;
        sa.chunk_shift = chunk_shift(plan, n);
        sa.chunk_pad = chunk_pad_slots();
        sa.cap = maxc << sa.chunk_shift;  // more slots means repeated keys: the bucket sorts nothing
        sa.dump = 0xffffffffu;
        sa.limit = limit;
        sa.check = check;
        sa.ctrl = ctrl;
        sa.tot = tot;
        sa.g_base = base;
        sa.order = kb4_order;
        sa.chunk_tab = chunk_tab;
        sa.max_chunks = maxc;
        sa.pool_next = pool_next;
        if (timer) timer->before(stream);
        if (n >= (size_t(1) << 26))  // long shares: 20480-key tiles
            bucket_partition_kernel<PART_THREADS, PART_KPT_SLAB, MAX_BUCKETS, 2>
                <<<P, PART_THREADS, part_smem_bytes(PART_THREADS, MAX_BUCKETS, PART_KPT_SLAB), stream>>>(
                    ks, plan.map, plan.nb, nullptr, nullptr, parted, nullptr, sa);
        else
            bucket_partition_kernel<PART_THREADS, PART_KPT, MAX_BUCKETS, 2>
                <<<P, PART_THREADS, part_smem_bytes(PART_THREADS, MAX_BUCKETS), stream>>>(
                    ks, plan.map, plan.nb, nullptr, nullptr, parted, nullptr, sa);
        if (timer) timer->after("bucket_partition", stream);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        nlaunch = 1;
    } else if (use_slab) {
        // KB3 (slab) claims slots with fill counters: no KB1/KB2. The counters
        // are zeroed once at allocation and re-zeroed by the last KB3 CTA.
        sa.gcnt = gcnt;
        sa.gtrue = tma_store_kb3(plan) ? gcnt + MAX_BUCKETS : nullptr;
        sa.cap = static_cast<uint32_t>((slab - PART_DUMP) / plan.nb) & ~3u;
        sa.dump = static_cast<uint32_t>(plan.nb) * sa.cap;  // 16-byte aligned (bulk-store runs)
        sa.limit = limit;
        sa.check = check;
        sa.ctrl = ctrl;
        sa.tot = tot;
        sa.g_base = base;
        if (timer) timer->before(stream);
        static const bool half_threads = [] {  // experiment: 512 threads x 32 keys (same tile)
            const char* e = std::getenv("BITSORT_PART_TMA");
            return e && std::string(e) == "512";
        }();
        if (sa.gtrue && half_threads)
            bucket_partition_tma_kernel<512, 512, 32>
                <<<P, 512, part_tma_smem_bytes(512), stream>>>(ks, plan.map, plan.nb, parted, sa);
        else if (sa.gtrue)
            bucket_partition_tma_kernel<512>
                <<<P, PART_THREADS, part_tma_smem_bytes(512), stream>>>(ks, plan.map, plan.nb, parted, sa);
        else if (narrow_partition(plan))
            bucket_partition_kernel<PART_NARROW_THREADS, PART_KPT, PART_NARROW_MAXB, 1>
                <<<P, PART_NARROW_THREADS, part_smem_bytes(PART_NARROW_THREADS, PART_NARROW_MAXB), stream>>>(
                    ks, plan.map, plan.nb, nullptr, nullptr, parted, nullptr, sa);
        else if (plan.nb <= PART_NARROW_MAXB)  // fewer slot-scan iterations per thread
            bucket_partition_kernel<PART_THREADS, PART_KPT_SLAB, PART_NARROW_MAXB, 1>
                <<<P, PART_THREADS, part_smem_bytes(PART_THREADS, PART_NARROW_MAXB, PART_KPT_SLAB), stream>>>(
                    ks, plan.map, plan.nb, nullptr, nullptr, parted, nullptr, sa);
        else
            bucket_partition_kernel<PART_THREADS, PART_KPT, MAX_BUCKETS, 1>
                <<<P, PART_THREADS, part_smem_bytes(PART_THREADS, MAX_BUCKETS), stream>>>(
                    ks, plan.map, plan.nb, nullptr, nullptr, parted, nullptr, sa);
        if (timer) timer->after("bucket_partition", stream);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        nlaunch = 1;
    } else {
        err = cudaMemsetAsync(H, 0, static_cast<size_t>(P) * plan.nb * sizeof(uint32_t), stream);
        if (err != cudaSuccess) return err;
        if (timer) timer->before(stream);
        bucket_hist_kernel<<<P * HIST_SPLIT, BUCKET_HIST_THREADS, 0, stream>>>(ks, plan.map, plan.nb,
                                                                               limit, check, H, ctrl);
        if (timer) timer->after("bucket_hist", stream);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
        if (timer) timer->before(stream);
        bucket_colscan_kernel<<<(plan.nb * 32 + 255) / 256, 256, 0, stream>>>(H, P, plan.nb, tot);
        if (timer) timer->after("bucket_colscan", stream);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        sa.order = kb4_order;
        if (timer) timer->before(stream);
        if (narrow_partition(plan))
            bucket_partition_kernel<PART_NARROW_THREADS, PART_KPT, PART_NARROW_MAXB, 0>
                <<<P, PART_NARROW_THREADS, part_smem_bytes(PART_NARROW_THREADS, PART_NARROW_MAXB), stream>>>(
                    ks, plan.map, plan.nb, H, tot, parted, base, sa);
        else if (n >= (size_t(1) << 26))  // long shares: 20480-key tiles (C5 KB3 1449 -> 1376 us)
            bucket_partition_kernel<PART_THREADS, PART_KPT_SLAB, MAX_BUCKETS, 0>
                <<<P, PART_THREADS, part_smem_bytes(PART_THREADS, MAX_BUCKETS, PART_KPT_SLAB), stream>>>(
                    ks, plan.map, plan.nb, H, tot, parted, base, sa);
        else  // short shares (C4: ~7 tiles per CTA): 16384-key tiles keep the tail short
            bucket_partition_kernel<PART_THREADS, PART_KPT, MAX_BUCKETS, 0>
                <<<P, PART_THREADS, part_smem_bytes(PART_THREADS, MAX_BUCKETS), stream>>>(
                    ks, plan.map, plan.nb, H, tot, parted, base, sa);
        if (timer) timer->after("bucket_partition", stream);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        nlaunch += 3;
    }
    if (plan.partition_only) {  // range split: the packed groups are the result
        if (launches) *launches = nlaunch;
        return cudaSuccess;
    }
    const uint32_t src_cap = use_slab ? sa.cap : 0u;
    if (push) {  // multi-GPU push build: bucket bitsets ORed into the owners' slices
        if (timer) timer->before(stream);
        bucket_push_kernel<<<geo.bucket_blocks[plan.shift], BUCKET_THREADS, std::size_t(1) << (plan.shift - 3),
                             stream>>>(parted, tot, base, plan.map, plan.nb, src_cap, *push, push_slice_words,
                                       n_words, (key_range & 31) ? (1u << (key_range & 31)) - 1u : 0xffffffffu,
                                       ctrl);
        if (timer) timer->after("bucket_push", stream);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        if (launches) *launches = nlaunch + 1;
        return cudaSuccess;
    }
    if (bits_out) {  // multi-GPU per-rank build: write the bitset instead of sorted keys
        if (timer) timer->before(stream);
        bucket_bitset_kernel<<<geo.bucket_blocks[plan.shift], BUCKET_THREADS,
                               std::size_t(1) << (plan.shift - 3), stream>>>(
            parted, tot, base, plan.map, plan.nb, src_cap, bits_out, n_words,
            (key_range & 31) ? (1u << (key_range & 31)) - 1u : 0xffffffffu, ctrl);
        if (timer) timer->after("bucket_bitset", stream);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        if (launches) *launches = nlaunch + 1;
        return cudaSuccess;
    }
    if (multiset) {
        if (timer) timer->before(stream);
        bucket_multiset_kernel<<<geo.multiset_blocks, MS_THREADS, ms_smem_bytes(), stream>>>(
            parted, tot, base, plan.map, plan.nb, out, ctrl, 0u);
        if (timer) timer->after("bucket_multiset", stream);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        if (launches) *launches = nlaunch + 1;
        return cudaSuccess;
    }
    if (timer) timer->before(stream);
    const size_t smem = bucket_sort_smem_bytes(plan.shift);
    // KB4 directly after KB3 on the stream: programmatic dependent launch (its
    // prologue overlaps KB3's tail). Not with per-kernel timing events in between.
    static const bool pdl_off = [] {
        const char* e = std::getenv("BITSORT_PDL");
        return e && std::string(e) == "0";
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(geo.bucket_blocks[plan.shift]));
    cfg.blockDim = dim3(plan.shift >= MAX_BUCKET_SHIFT ? BUCKET_THREADS : 512);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute pdl_attr[1];
    pdl_attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl_attr[0].val.programmaticStreamSerializationAllowed = 1;
    if (!timer && !pdl_off && nlaunch > 0) {
        cfg.attrs = pdl_attr;
        cfg.numAttrs = 1;
    }
    const int aon = inplace_mode == 1 && use_slab;
    const uint32_t* ctab = use_chunk ? sa.chunk_tab : nullptr;
    if (plan.shift >= MAX_BUCKET_SHIFT)
        err = cudaLaunchKernelEx(&cfg, bucket_sort_kernel<BUCKET_STAGE>, static_cast<const uint32_t*>(parted),
                                 static_cast<const uint32_t*>(tot), static_cast<const unsigned long long*>(base),
                                 plan.map, plan.nb, src_cap, out, ctrl, static_cast<const uint32_t*>(kb4_order), aon,
                                 ctab, sa.max_chunks, sa.chunk_shift, sa.chunk_pad);
    else  // narrower buckets: two 512-thread CTAs per SM
        err = cudaLaunchKernelEx(&cfg, bucket_sort_kernel<BUCKET_STAGE, 512>, static_cast<const uint32_t*>(parted),
                                 static_cast<const uint32_t*>(tot), static_cast<const unsigned long long*>(base),
                                 plan.map, plan.nb, src_cap, out, ctrl, static_cast<const uint32_t*>(kb4_order), aon,
                                 ctab, sa.max_chunks, sa.chunk_shift, sa.chunk_pad);
    if (err != cudaSuccess) return err;
    if (timer) timer->after("bucket_sort", stream);
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
    if (launches) *launches = nlaunch + 1;
    return cudaSuccess;
}

cudaError_t launch_bucket_push(const uint32_t* keys, size_t n, uint64_t key_range, uint32_t* parted, void* scratch,
                               Ctrl* ctrl, const BucketPlan& plan, const LaunchGeometry& geo, cudaStream_t stream,
                               int* launches, const OrSources& slices, uint64_t slice_words, uint64_t parted_cap,
                               KernelTimer* timer) {
    return launch_bucket_sort(keys, n, key_range, nullptr, parted, scratch, ctrl, plan, geo, stream, launches, timer,
                              nullptr, (key_range + 31) / 32, parted_cap, false, &slices, slice_words);
}

cudaError_t configure_bucket_kernels(int device, LaunchGeometry* geo) {
    int sms = 0;
    cudaError_t err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (err != cudaSuccess) return err;
    for (auto kern : {bucket_partition_kernel<PART_THREADS, PART_KPT_SLAB, MAX_BUCKETS, 2>}) {
        err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(part_smem_bytes(PART_THREADS, MAX_BUCKETS, PART_KPT_SLAB)));
        if (err != cudaSuccess) return err;
    }
    err = cudaFuncSetAttribute(bucket_partition_kernel<PART_THREADS, PART_KPT, MAX_BUCKETS, 2>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(part_smem_bytes(PART_THREADS, MAX_BUCKETS)));
    if (err != cudaSuccess) return err;
    err = cudaFuncSetAttribute(bucket_partition_kernel<PART_THREADS, PART_KPT_SLAB, MAX_BUCKETS, 0>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(part_smem_bytes(PART_THREADS, MAX_BUCKETS, PART_KPT_SLAB)));
    if (err != cudaSuccess) return err;
    auto wide = bucket_partition_kernel<PART_THREADS, PART_KPT, MAX_BUCKETS, 0>;
    auto narrow = bucket_partition_kernel<PART_NARROW_THREADS, PART_KPT, PART_NARROW_MAXB, 0>;
    err = cudaFuncSetAttribute(wide, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(part_smem_bytes(PART_THREADS, MAX_BUCKETS)));
    if (err != cudaSuccess) return err;
    err = cudaFuncSetAttribute(bucket_partition_kernel<PART_THREADS, PART_KPT, MAX_BUCKETS, 1>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(part_smem_bytes(PART_THREADS, MAX_BUCKETS)));
    if (err != cudaSuccess) return err;
    err = cudaFuncSetAttribute(bucket_partition_tma_kernel<512, 512, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(part_tma_smem_bytes(512)));
    if (err != cudaSuccess) return err;
    err = cudaFuncSetAttribute(bucket_partition_tma_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(part_tma_smem_bytes(512)));
    if (err != cudaSuccess) return err;
    err = cudaFuncSetAttribute(bucket_partition_kernel<PART_THREADS, PART_KPT_SLAB, PART_NARROW_MAXB, 1>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(part_smem_bytes(PART_THREADS, PART_NARROW_MAXB, PART_KPT_SLAB)));
    if (err != cudaSuccess) return err;
    err = cudaFuncSetAttribute(bucket_partition_kernel<PART_NARROW_THREADS, PART_KPT, PART_NARROW_MAXB, 1>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(part_smem_bytes(PART_NARROW_THREADS, PART_NARROW_MAXB)));
    if (err != cudaSuccess) return err;
    err = cudaFuncSetAttribute(narrow, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(part_smem_bytes(PART_NARROW_THREADS, PART_NARROW_MAXB)));
    if (err != cudaSuccess) return err;
    err = cudaFuncSetAttribute(bucket_bitset_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               1 << (MAX_BUCKET_SHIFT - 3));
    if (err != cudaSuccess) return err;
    err = cudaFuncSetAttribute(bucket_push_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               1 << (MAX_BUCKET_SHIFT - 3));
    if (err != cudaSuccess) return err;
    err = cudaFuncSetAttribute(bucket_multiset_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(ms_smem_bytes()));
    if (err != cudaSuccess) return err;
    geo->multiset_blocks = sms;
    err = cudaFuncSetAttribute(bucket_sort_kernel<BUCKET_STAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(bucket_sort_smem_bytes(20)));
    if (err != cudaSuccess) return err;
    err = cudaFuncSetAttribute(bucket_sort_kernel<BUCKET_STAGE, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(bucket_sort_smem_bytes(19)));
    if (err != cudaSuccess) return err;
    int per = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, wide, PART_THREADS,
                                                        part_smem_bytes(PART_THREADS, MAX_BUCKETS));
    if (err != cudaSuccess) return err;
    geo->part_blocks = sms * (per > 0 ? per : 1);
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per, narrow, PART_NARROW_THREADS, part_smem_bytes(PART_NARROW_THREADS, PART_NARROW_MAXB));
    if (err != cudaSuccess) return err;
    geo->part_blocks_narrow = sms * (per > 0 ? per : 1);
    for (int shift = MIN_BUCKET_SHIFT; shift <= MAX_BUCKET_SHIFT; ++shift) {
        err = shift >= MAX_BUCKET_SHIFT
                  ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bucket_sort_kernel<BUCKET_STAGE>,
                                                                  BUCKET_THREADS, bucket_sort_smem_bytes(shift))
                  : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bucket_sort_kernel<BUCKET_STAGE, 512>,
                                                                  512, bucket_sort_smem_bytes(shift));
        if (err != cudaSuccess) return err;
        geo->bucket_blocks[shift] = sms * (per > 0 ? per : 1);
    }
    return cudaSuccess;
}

}  // namespace bws_gpu
