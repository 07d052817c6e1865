// K3 bitset scan, v2 (sm_100a): single-pass decoupled-lookback scan of a
// global bitset into sorted keys.
//
// v1 (kernels.cu) used 2048-word tiles: at B200 bandwidth that is ~800 tiles
// per microsecond, and the lookback chain (32 predecessors per L2 round trip)
// could not keep up — a sparse 512 MiB bitset scanned at 0.6 TB/s. v2:
//  - 8192-word (32 KB) tiles fetched by TMA bulk copies into a double-buffered
//    SMEM ring, the next tile's copy in flight while the current one is
//    scanned (tiles by dynamic ticket, so lookback never waits on a CTA that
//    has not started);
//  - lookback windows of 128 predecessors per round trip (4 packed 64-bit
//    {flag, count} status words per lane);
//  - extraction from SMEM with the shared 128-word step (per-warp stage or
//    ballot; empty steps skipped), coalesced stores;
//  - optional consumption (zeroing of nonzero 16-byte chunks) to keep a cached
//    bitset all-zero between sorts.
#include "device_util.cuh"
#include "kernels.h"

namespace bws_gpu {
namespace {

using namespace dev;

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPrefix = 2ull << 62;
constexpr unsigned long long kValueMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    return v;
}

// Warp 0: exclusive prefix of `tile` given its aggregate (64-bit status words,
// 128 predecessors per round trip: lane l reads tiles end-1-4l-j, j = 0..3).
__device__ unsigned long long lookback(unsigned long long* status, unsigned tile,
                                       unsigned long long agg, unsigned lane) {
    if (tile == 0) {
        if (lane == 0) st_relaxed_u64(status, kFlagPrefix | agg);
        return 0;
    }
    if (lane == 0) st_relaxed_u64(status + tile, kFlagAgg | agg);
    unsigned long long prefix = 0;
    long long end = tile;
    for (;;) {
        unsigned long long s[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long long idx = end - 1 - 4 * static_cast<long long>(lane) - j;
            s[j] = idx >= 0 ? ld_relaxed_u64(status + idx) : kFlagPrefix;
        }
        for (;;) {
            bool ready = true;
#pragma unroll
            for (int j = 0; j < 4; ++j) ready &= (s[j] >> 62) != 0;
            if (__all_sync(kFull, ready)) break;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const long long idx = end - 1 - 4 * static_cast<long long>(lane) - j;
                if ((s[j] >> 62) == 0) s[j] = ld_relaxed_u64(status + idx);
            }
        }
        int first = 4;  // first PREFIX among this lane's 4, nearest first
#pragma unroll
        for (int j = 3; j >= 0; --j)
            if ((s[j] >> 62) == 2) first = j;
        const unsigned pm = __ballot_sync(kFull, first < 4);
        unsigned long long mine = 0;
        if (pm) {
            const unsigned fl = __ffs(pm) - 1;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (lane < fl || (lane == fl && j <= first)) mine += s[j] & kValueMask;
            prefix += warp_sum_u64(mine);
            break;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) mine += s[j] & kValueMask;
        prefix += warp_sum_u64(mine);
        end -= 128;
    }
    if (lane == 0) st_relaxed_u64(status + tile, kFlagPrefix | (prefix + agg));
    return prefix;
}

// Stores at most `room` of the warp's `count` keys from the stage (the output
// capacity guard of the multi-GPU slice scan; normally room >= count).
__device__ __forceinline__ void drain_stage_capped(const uint32_t* stage, uint32_t count,
                                                   uint32_t* __restrict__ o, long long room,
                                                   unsigned lane) {
    __syncwarp();
    const uint32_t lim = room < static_cast<long long>(count) ? (room > 0 ? static_cast<uint32_t>(room) : 0u) : count;
    for (uint32_t i = lane; i < lim; i += 32) __stcs(o + i, stage[i + (i >> 5)]);
    __syncwarp();
}

// Bounds-checked extraction of one 512-word warp segment into o[0, room)
// (used only near the end of an output buffer).
__device__ void extract_segment_capped(const uint32_t* t32, uint32_t seg, uint32_t key_hi,
                                       uint32_t* __restrict__ o, long long room, uint32_t* s_stage,
                                       unsigned lane) {
    constexpr uint32_t kSeg = SCAN2_TILE_WORDS / (SCAN2_THREADS / 32);
    const uint4* s4 = reinterpret_cast<const uint4*>(t32);
    long long left = room;
    for (uint32_t s0 = 0; s0 < kSeg; s0 += 128) {
        const uint4 v = s4[(seg + s0) / 4 + lane];
        const uint32_t cl = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
        const uint32_t incl = warp_incl_scan(cl, lane);
        const uint32_t ctot = __shfl_sync(kFull, incl, 31);
        if (ctot == 0) continue;
        if (ctot <= static_cast<uint32_t>(SCAN2_STAGE)) {
            uint32_t p = incl - cl;
            const uint32_t kb = key_hi + ((seg + s0 + 4 * lane) << 5);
            stage_bits(v.x, kb, p, s_stage);
            stage_bits(v.y, kb + 32, p, s_stage);
            stage_bits(v.z, kb + 64, p, s_stage);
            stage_bits(v.w, kb + 96, p, s_stage);
            drain_stage_capped(s_stage, ctot, o, left, lane);
        } else if (left >= static_cast<long long>(ctot)) {
            uint32_t* oq = o;
#pragma unroll 1
            for (uint32_t q = 0; q < 128; q += 32)
                oq += extract_words32<SCAN2_STAGE>(t32, seg + s0 + q, key_hi, oq, s_stage, lane);
        }
        o += ctot;
        left -= ctot;
    }
}

// Two-pass variant, pass 1: popcount of every 8192-word tile (streaming reads).
__global__ void __launch_bounds__(SCAN2_THREADS)
    tile_count_kernel(const uint32_t* __restrict__ bits, unsigned long long n_words,
                      uint32_t* __restrict__ counts, uint32_t* __restrict__ seg_counts) {
    __shared__ uint32_t s_w[SCAN2_THREADS / 32];
    const unsigned n_tiles = static_cast<unsigned>((n_words + SCAN2_TILE_WORDS - 1) / SCAN2_TILE_WORDS);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (unsigned t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const unsigned long long w0 = static_cast<unsigned long long>(t) * SCAN2_TILE_WORDS;
        // warp w counts the tile's 512-word segment w (the scan's warp segment)
        const unsigned long long sw0 = w0 + warp * (SCAN2_TILE_WORDS / (SCAN2_THREADS / 32));
        constexpr int kV = SCAN2_TILE_WORDS / (SCAN2_THREADS / 32) / 4 / 32;  // uint4 per lane
        uint32_t c = 0;
        if (sw0 + 32 * 4 * kV <= n_words) {
            const uint4* v4 = reinterpret_cast<const uint4*>(bits + sw0);
            uint4 v[kV];
#pragma unroll
            for (int j = 0; j < kV; ++j) v[j] = __ldcs(v4 + j * 32 + lane);
#pragma unroll
            for (int j = 0; j < kV; ++j) c += __popc(v[j].x) + __popc(v[j].y) + __popc(v[j].z) + __popc(v[j].w);
        } else {
            for (unsigned long long i = sw0 + lane; i < min(n_words, sw0 + 32 * 4 * kV); i += 32) c += __popc(bits[i]);
        }
        c = __reduce_add_sync(kFull, c);
        if (lane == 0) {
            s_w[warp] = c;
            seg_counts[static_cast<size_t>(t) * (SCAN2_THREADS / 32) + warp] = c;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t sum = 0;
            for (int q = 0; q < SCAN2_THREADS / 32; ++q) sum += s_w[q];
            counts[t] = sum;
        }
        __syncthreads();
    }
}

// Two-pass variant, pass 2: exclusive prefix of the tile counts (one CTA).
__global__ void __launch_bounds__(1024)
    tile_offsets_kernel(const uint32_t* __restrict__ counts, unsigned long long n_words,
                        unsigned long long* __restrict__ offsets, Ctrl* __restrict__ ctrl,
                        unsigned long long* __restrict__ d_total) {
    __shared__ unsigned long long s_w[32];
    const unsigned n_tiles = static_cast<unsigned>((n_words + SCAN2_TILE_WORDS - 1) / SCAN2_TILE_WORDS);
    const unsigned per = (n_tiles + 1023) / 1024;
    const unsigned b0 = threadIdx.x * per;
    unsigned long long local = 0;
    for (unsigned i = 0; i < per; ++i)
        if (b0 + i < n_tiles) local += counts[b0 + i];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned long long o = __shfl_up_sync(kFull, incl, off);
        if (lane >= static_cast<unsigned>(off)) incl += o;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const unsigned long long w = s_w[lane];
        unsigned long long wi = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned long long o = __shfl_up_sync(kFull, wi, off);
            if (lane >= static_cast<unsigned>(off)) wi += o;
        }
        s_w[lane] = wi - w;
        if (lane == 31) {
            ctrl->total = wi;
            if (d_total) *d_total = wi;
        }
    }
    __syncthreads();
    unsigned long long run = s_w[warp] + incl - local;
    for (unsigned i = 0; i < per; ++i) {
        if (b0 + i < n_tiles) {
            offsets[b0 + i] = run;
            run += counts[b0 + i];
        }
    }
}

// MULTI: the scanned bitset is the OR of srcs.p[0 .. srcs.n) (bits == srcs.p[0],
// the local one, arrives by TMA; the others — peer GPUs' memory over
// NVLink/NVSwitch through CUDA IPC — are loaded with 16-byte loads while that
// copy is in flight and ORed into the SMEM tile). This fuses the multi-GPU
// exchange into the scan: no gathered slice is written or re-read.
template <bool CLEAR, bool PRECOUNT, bool MULTI = false>
__global__ void __launch_bounds__(SCAN2_THREADS, 2)
    scan2_kernel(uint32_t* __restrict__ bits, unsigned long long n_words_param, uint32_t key_base,
                 uint32_t* __restrict__ out, unsigned long long out_cap, Ctrl* __restrict__ ctrl,
                 unsigned long long* __restrict__ status, unsigned long long* __restrict__ d_total,
                 OrSources srcs = OrSources{}) {
    static_assert(!(MULTI && (CLEAR || PRECOUNT)), "the source-OR scan is lookback-only and read-only");
    constexpr int NW = SCAN2_THREADS / 32;
    constexpr uint32_t kSeg = SCAN2_TILE_WORDS / NW;  // words per warp segment (512)
    constexpr int kPitch = SCAN2_STAGE + SCAN2_STAGE / 32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint32_t* s_tiles = reinterpret_cast<uint32_t*>(smem_raw);  // 2 x SCAN2_TILE_WORDS
    uint32_t* s_stage = s_tiles + 2 * SCAN2_TILE_WORDS + (threadIdx.x >> 5) * kPitch;
    __shared__ __align__(8) unsigned long long s_bar[2];
    __shared__ uint32_t s_tile[2], s_par[2], s_issued[2];
    __shared__ uint32_t s_warp[NW];
    __shared__ unsigned long long s_prefix;

    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned long long n_words =
        n_words_param ? n_words_param
                      : (static_cast<unsigned long long>(
                             *reinterpret_cast<volatile unsigned int*>(&ctrl->max_key)) >> 5) + 1;
    const unsigned n_tiles = static_cast<unsigned>((n_words + SCAN2_TILE_WORDS - 1) / SCAN2_TILE_WORDS);

    // thread 0: take a ticket and start the tile's bulk copy. Tickets are
    // taken just in time (never ahead of the tile being worked on): a tile
    // ticketed early would publish its aggregate late and stall every later
    // tile's lookback (measured: 4x slower with one-ahead prefetch).
    // PRECOUNT (no lookback chain): static tiles, the next one prefetched
    // into the other buffer while the current one is extracted.
    unsigned next_static = blockIdx.x;
    auto fetch = [&](int slot) {
        unsigned t;
        if (PRECOUNT) {
            t = next_static;
            next_static += gridDim.x;
        } else {
            t = atomicAdd(&ctrl->ticket, 1u);
        }
        s_tile[slot] = t;
        if (t >= n_tiles) return;
        const unsigned long long w0 = static_cast<unsigned long long>(t) * SCAN2_TILE_WORDS;
        const unsigned long long len = min(static_cast<unsigned long long>(SCAN2_TILE_WORDS), n_words - w0);
        const uint32_t bulk = static_cast<uint32_t>(len & ~3ull) * 4;  // 16-byte multiple
        s_par[slot] = s_issued[slot] & 1;
        s_issued[slot] += 1;
        if (bulk) {
            fence_proxy_async_smem();
            tma_load_bytes(s_tiles + slot * SCAN2_TILE_WORDS, bits + w0, bulk, &s_bar[slot]);
        } else {  // nothing for the TMA: complete the phase by hand
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&s_bar[slot])) : "memory");
        }
    };
    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        fence_mbar_init();
        s_issued[0] = s_issued[1] = 0;
        if (PRECOUNT) fetch(0);
    }
    __syncthreads();

    for (uint32_t it = 0;; ++it) {
        const int slot = PRECOUNT ? static_cast<int>(it & 1) : 0;
        if (!PRECOUNT) {
            if (threadIdx.x == 0) fetch(slot);
            __syncthreads();
        }
        const unsigned tile = s_tile[slot];
        if (tile >= n_tiles) break;
        if (PRECOUNT && threadIdx.x == 0) fetch(slot ^ 1);  // released at the previous loop end
        const unsigned long long w0 = static_cast<unsigned long long>(tile) * SCAN2_TILE_WORDS;
        const uint32_t len = static_cast<uint32_t>(min(static_cast<unsigned long long>(SCAN2_TILE_WORDS), n_words - w0));
        uint32_t* t32 = s_tiles + slot * SCAN2_TILE_WORDS;
        constexpr int kPV = SCAN2_TILE_WORDS / 4 / SCAN2_THREADS;  // uint4 per thread per tile
        uint4 acc[kPV];
        uint32_t acc_tail = 0u;
        if (MULTI) {
            // the other sources' words of this tile, ORed in registers while
            // the local copy is in flight (one round trip per source)
            const uint32_t nv = len >> 2;
#pragma unroll
            for (int k = 0; k < kPV; ++k) acc[k] = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
            for (int s = 1; s < MAX_OR_SOURCES; ++s) {  // static indices: srcs stays in param space
                if (s >= srcs.n) break;
                const uint4* p4 = reinterpret_cast<const uint4*>(srcs.p[s] + w0);
                uint4 v[kPV];
#pragma unroll
                for (int k = 0; k < kPV; ++k) {
                    const uint32_t i = threadIdx.x + k * SCAN2_THREADS;
                    v[k] = i < nv ? __ldcs(p4 + i) : make_uint4(0u, 0u, 0u, 0u);
                }
#pragma unroll
                for (int k = 0; k < kPV; ++k) {
                    acc[k].x |= v[k].x;
                    acc[k].y |= v[k].y;
                    acc[k].z |= v[k].z;
                    acc[k].w |= v[k].w;
                }
                if (threadIdx.x < (len & 3u)) acc_tail |= srcs.p[s][w0 + (len & ~3u) + threadIdx.x];
            }
        }
        mbar_wait(&s_bar[slot], s_par[slot]);
        // tail words (< 4) the bulk copy did not cover; zero padding past the end
        if (threadIdx.x < 4) {
            const uint32_t i = (len & ~3u) + threadIdx.x;
            if (i < SCAN2_TILE_WORDS) t32[i] = i < len ? (bits[w0 + i] | acc_tail) : 0u;
        }
        if (MULTI) {
            uint4* t4 = reinterpret_cast<uint4*>(t32);
            const uint32_t nv = len >> 2;
#pragma unroll
            for (int k = 0; k < kPV; ++k) {
                const uint32_t i = threadIdx.x + k * SCAN2_THREADS;
                if (i < nv) {
                    uint4 t = t4[i];
                    t.x |= acc[k].x;
                    t.y |= acc[k].y;
                    t.z |= acc[k].z;
                    t.w |= acc[k].w;
                    t4[i] = t;
                }
            }
        }
        if (len < SCAN2_TILE_WORDS)
            for (uint32_t i = (len & ~3u) + 4 + threadIdx.x; i < SCAN2_TILE_WORDS; i += SCAN2_THREADS) t32[i] = 0u;
        __syncthreads();
        const uint32_t seg = warp * kSeg;
        const uint4* s4 = reinterpret_cast<const uint4*>(t32);
        if (PRECOUNT) {
            // no cross-warp dependency: this warp's first output slot is the
            // tile prefix plus the counts of the segments before it
            const uint32_t* segc = reinterpret_cast<const uint32_t*>(status + n_tiles + n_tiles / 2 + 1);
            const uint32_t sc = lane < static_cast<unsigned>(warp) ? segc[static_cast<size_t>(tile) * NW + lane] : 0u;
            const unsigned long long first = status[tile] + __reduce_add_sync(kFull, sc);
            const long long room = static_cast<long long>(out_cap) - static_cast<long long>(first);
            const uint32_t key_hi = key_base + static_cast<uint32_t>(w0 << 5);
            if (room >= static_cast<long long>(kSeg) * 32) {
                extract_span512<SCAN2_STAGE>(t32, seg, kSeg, key_hi, out + first, s_stage, lane, false,
                                             CLEAR ? bits + w0 : nullptr);
            } else {
                if (CLEAR) {
                    for (uint32_t i = lane; i < kSeg / 4; i += 32) {
                        const uint4 v = s4[seg / 4 + i];
                        const unsigned long long gw = w0 + seg + 4 * i;
                        if ((v.x | v.y | v.z | v.w) && gw < n_words) {
                            if (gw + 4 <= n_words)
                                *reinterpret_cast<uint4*>(bits + gw) = make_uint4(0, 0, 0, 0);
                            else
                                for (unsigned long long q = gw; q < n_words; ++q) bits[q] = 0u;
                        }
                    }
                }
                if (room > 0) extract_segment_capped(t32, seg, key_hi, out + first, room, s_stage, lane);
            }
            __syncthreads();
            continue;
        }

        // phase 1: per-warp popcount of its 512-word segment (+ consumption)
        uint32_t c = 0;
        for (uint32_t i = lane; i < kSeg / 4; i += 32) {
            const uint4 v = s4[seg / 4 + i];
            c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
            if (CLEAR && (v.x | v.y | v.z | v.w)) {
                const unsigned long long gw = w0 + seg + 4 * i;
                if (gw + 4 <= n_words)
                    *reinterpret_cast<uint4*>(bits + gw) = make_uint4(0, 0, 0, 0);
                else
                    for (unsigned long long q = gw; q < n_words; ++q) bits[q] = 0u;
            }
        }
        c = __reduce_add_sync(kFull, c);
        if (lane == 0) s_warp[warp] = c;
        __syncthreads();
        if (warp == 0) {
            const uint32_t v = lane < NW ? s_warp[lane] : 0u;
            const uint32_t incl = warp_incl_scan(v, lane);
            if (lane < NW) s_warp[lane] = incl - v;
            const unsigned long long agg = __shfl_sync(kFull, incl, 31);
            // PRECOUNT: `status` holds the tile offsets of the two-pass variant
            const unsigned long long prefix = PRECOUNT ? status[tile] : lookback(status, tile, agg, lane);
            if (lane == 0) {
                s_prefix = prefix;
                if (!PRECOUNT && tile == n_tiles - 1) {
                    ctrl->total = prefix + agg;
                    if (d_total) *d_total = prefix + agg;
                }
            }
        }
        __syncthreads();

        // phase 2: extraction of the warp's 512-word segment
        const unsigned long long first = s_prefix + s_warp[warp];
        const long long room = static_cast<long long>(out_cap) - static_cast<long long>(first);
        const uint32_t key_hi = key_base + static_cast<uint32_t>(w0 << 5);
        if (room >= static_cast<long long>(kSeg) * 32) {
            extract_span512<SCAN2_STAGE>(t32, seg, kSeg, key_hi, out + first, s_stage, lane, false, nullptr);
        } else if (room > 0) {  // near the end of the output buffer: bounds-checked slow path
            extract_segment_capped(t32, seg, key_hi, out + first, room, s_stage, lane);
        }
        __syncthreads();  // buffer free for the next tile's copy
    }
}

}  // namespace

cudaError_t launch_scan2_sources(const OrSources& srcs, uint64_t n_words, uint32_t key_base, uint32_t* out,
                                 uint64_t out_capacity, Ctrl* ctrl, unsigned long long* status,
                                 unsigned long long* d_total, const LaunchGeometry& geo,
                                 cudaStream_t stream) {
    if (n_words == 0) return cudaSuccess;
    int blocks = geo.scan2_blocks;
    const uint64_t tiles = (n_words + SCAN2_TILE_WORDS - 1) / SCAN2_TILE_WORDS;
    if (tiles < static_cast<uint64_t>(blocks)) blocks = static_cast<int>(tiles);
    scan2_kernel<false, false, true><<<blocks, SCAN2_THREADS, scan2_smem_bytes(), stream>>>(
        const_cast<uint32_t*>(srcs.p[0]), n_words, key_base, out, out_capacity, ctrl, status, d_total, srcs);
    return cudaGetLastError();
}

bool scan2_supported(const uint32_t* bits) { return (reinterpret_cast<uintptr_t>(bits) & 15) == 0; }

cudaError_t configure_scan2(int device, LaunchGeometry* geo) {
    int sms = 0;
    cudaError_t err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (err != cudaSuccess) return err;
    const int smem = static_cast<int>(scan2_smem_bytes());
    for (auto k : {scan2_kernel<true, false>, scan2_kernel<false, false>, scan2_kernel<true, true>,
                   scan2_kernel<false, true>, scan2_kernel<false, false, true>}) {
        err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (err != cudaSuccess) return err;
    }
    int per = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, scan2_kernel<true, false>, SCAN2_THREADS, smem);
    if (err != cudaSuccess) return err;
    geo->scan2_blocks = sms * (per > 0 ? per : 1);
    return cudaSuccess;
}

cudaError_t launch_scan2(uint32_t* bits, uint64_t n_words, uint32_t key_base, uint32_t* out,
                         uint64_t out_capacity, Ctrl* ctrl, unsigned long long* status,
                         unsigned long long* d_total, int clear, const LaunchGeometry& geo,
                         cudaStream_t stream, int two_pass, int* launches) {
    int blocks = geo.scan2_blocks;
    const uint64_t tiles = (n_words + SCAN2_TILE_WORDS - 1) / SCAN2_TILE_WORDS;
    if (n_words != 0 && tiles < static_cast<uint64_t>(blocks)) blocks = static_cast<int>(tiles);
    if (launches) *launches = 1;
    if (two_pass && n_words != 0) {
        // counts in the upper half of `status` (tiles <= 16384 words of 8 B each
        // were reserved; 2048-word granularity reserves 4x that)
        // layout: offsets u64[tiles] | counts u32[tiles] | seg counts u32[16 * tiles]
        uint32_t* counts = reinterpret_cast<uint32_t*>(status + tiles);
        uint32_t* segc = reinterpret_cast<uint32_t*>(status + tiles + tiles / 2 + 1);
        tile_count_kernel<<<geo.scan2_blocks, SCAN2_THREADS, 0, stream>>>(bits, n_words, counts, segc);
        tile_offsets_kernel<<<1, 1024, 0, stream>>>(counts, n_words, status, ctrl, d_total);
        if (clear)
            scan2_kernel<true, true><<<blocks, SCAN2_THREADS, scan2_smem_bytes(), stream>>>(
                bits, n_words, key_base, out, out_capacity, ctrl, status, d_total);
        else
            scan2_kernel<false, true><<<blocks, SCAN2_THREADS, scan2_smem_bytes(), stream>>>(
                bits, n_words, key_base, out, out_capacity, ctrl, status, d_total);
        if (launches) *launches = 3;
        return cudaGetLastError();
    }
    if (clear)
        scan2_kernel<true, false><<<blocks, SCAN2_THREADS, scan2_smem_bytes(), stream>>>(
            bits, n_words, key_base, out, out_capacity, ctrl, status, d_total);
    else
        scan2_kernel<false, false><<<blocks, SCAN2_THREADS, scan2_smem_bytes(), stream>>>(
            bits, n_words, key_base, out, out_capacity, ctrl, status, d_total);
    return cudaGetLastError();
}

}  // namespace bws_gpu
