// sm_100a kernels of the bitset sort.
//
// The reference sorts with 32 stable LSD partition passes
// (proj/src/bitsort.hpp:84-103 partition_pass, :111-129 sort_same_sign_impl).
// For distinct keys in [0, M) the sorted order is unique, so the same output is
// produced here by
//   K2 bitset_scatter : bits[x >> 5] |= 1 << (x & 31)        (reads 4n bytes)
//   K3 bitset_scan    : popcount -> decoupled-lookback prefix -> set-bit
//                       extraction -> SMEM-staged coalesced store (reads M/8,
//                       writes 4n bytes)
// Both kernels are persistent (grid = SMs x resident blocks) and HBM-bound; no
// tensor cores are involved.
#include "kernels.h"

namespace bws_gpu {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPrefix = 2ull << 62;
constexpr unsigned long long kValueMask = (1ull << 62) - 1;
// A warp whose 512 keys span fewer words than this aggregates its atomics.
constexpr uint32_t kWarpAggSpanWords = 2048;

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

// Lanes holding keys of the same word OR their bits together (match.any +
// redux.or, the labeled-partition reduction); one lane per distinct word issues
// the global RED. Invalid lanes get a tag no real word can have (words < 2^27).
__device__ __forceinline__ void or_warp_aggregated(uint32_t* bits, uint32_t key, bool valid,
                                                   unsigned lane) {
    const uint32_t word = key >> 5;
    const uint32_t tag = valid ? word : (0x80000000u | lane);
    const unsigned peers = __match_any_sync(kFull, tag);
    const uint32_t agg = __reduce_or_sync(peers, 1u << (key & 31));
    if (valid && static_cast<unsigned>(__ffs(peers) - 1) == lane) atomicOr(bits + word, agg);
}

// ---------------------------------------------------------------------------
// K2: bitset scatter.
//
// A block tile is SCATTER_VEC coalesced uint4 loads per thread (4096 keys).
// MODE kAuto : block min/max -> if the tile's word span fits the SMEM window,
//              OR into shared memory and flush each nonzero word with one RED;
//              otherwise a warp whose span is narrow uses warp aggregation,
//              a wide (shuffled) warp issues one RED per key.
// The body is 16-byte aligned; the <=3 leading and <=3 trailing keys of a
// misaligned array are handled by block 0 (head/tail).
template <int MODE, bool CHECK>
__global__ void __launch_bounds__(SCATTER_THREADS)
    scatter_kernel(const uint4* __restrict__ vec, size_t n_vec, const uint32_t* __restrict__ head,
                   int n_head, const uint32_t* __restrict__ tail, int n_tail,
                   uint32_t* __restrict__ bits, uint32_t limit, Ctrl* __restrict__ ctrl) {
    extern __shared__ uint32_t s_bits[];  // SCATTER_SMEM_WORDS (staging modes only)
    __shared__ uint32_t s_min[2][SCATTER_THREADS / 32];
    __shared__ uint32_t s_max[2][SCATTER_THREADS / 32];

    const unsigned lane = threadIdx.x & 31;
    const unsigned warp = threadIdx.x >> 5;
    uint32_t run_max = 0;
    uint32_t run_bad = 0;

    if (blockIdx.x == 0 && static_cast<int>(threadIdx.x) < n_head + n_tail) {
        const uint32_t x = static_cast<int>(threadIdx.x) < n_head ? head[threadIdx.x]
                                                                   : tail[threadIdx.x - n_head];
        if (!CHECK || x < limit) {
            atomicOr(bits + (x >> 5), 1u << (x & 31));
            run_max = x;
        } else {
            run_bad = 1;
        }
    }

    constexpr size_t kTileVecs = static_cast<size_t>(SCATTER_THREADS) * SCATTER_VEC;
    const size_t n_tiles = (n_vec + kTileVecs - 1) / kTileVecs;
    int parity = 0;
    for (size_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, parity ^= 1) {
        const size_t base = tile * kTileVecs + threadIdx.x;
        uint4 v[SCATTER_VEC];
        bool in[SCATTER_VEC];
#pragma unroll
        for (int j = 0; j < SCATTER_VEC; ++j) {
            const size_t i = base + static_cast<size_t>(j) * SCATTER_THREADS;
            in[j] = i < n_vec;
            v[j] = in[j] ? __ldcs(vec + i) : make_uint4(0, 0, 0, 0);
        }
        uint32_t key[SCATTER_VEC * 4];
        bool ok[SCATTER_VEC * 4];
#pragma unroll
        for (int j = 0; j < SCATTER_VEC; ++j) {
            key[4 * j + 0] = v[j].x;
            key[4 * j + 1] = v[j].y;
            key[4 * j + 2] = v[j].z;
            key[4 * j + 3] = v[j].w;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const bool good = in[j] && (!CHECK || key[4 * j + c] < limit);
                run_bad += (in[j] && !good) ? 1u : 0u;
                ok[4 * j + c] = good;
            }
        }

        if (MODE == kPlain) {
#pragma unroll
            for (int k = 0; k < SCATTER_VEC * 4; ++k) {
                if (ok[k]) {
                    atomicOr(bits + (key[k] >> 5), 1u << (key[k] & 31));
                    run_max = max(run_max, key[k]);
                }
            }
            continue;
        }

        uint32_t kmin = 0xffffffffu, kmax = 0;
#pragma unroll
        for (int k = 0; k < SCATTER_VEC * 4; ++k) {
            if (ok[k]) {
                kmin = min(kmin, key[k]);
                kmax = max(kmax, key[k]);
            }
        }
        const uint32_t wmin = __reduce_min_sync(kFull, kmin);
        const uint32_t wmax = __reduce_max_sync(kFull, kmax);
        run_max = max(run_max, wmax);

        if (MODE == kAuto || MODE == kSmem) {
            if (lane == 0) {
                s_min[parity][warp] = wmin;
                s_max[parity][warp] = wmax;
            }
            __syncthreads();
            uint32_t bmin = s_min[parity][0], bmax = s_max[parity][0];
#pragma unroll
            for (int q = 1; q < SCATTER_THREADS / 32; ++q) {
                bmin = min(bmin, s_min[parity][q]);
                bmax = max(bmax, s_max[parity][q]);
            }
            if (bmin <= bmax) {
                const uint32_t lo = bmin >> 5;
                const uint32_t span = (bmax >> 5) - lo + 1;
                if (span <= static_cast<uint32_t>(SCATTER_SMEM_WORDS)) {
                    for (uint32_t w = threadIdx.x; w < span; w += SCATTER_THREADS) s_bits[w] = 0;
                    __syncthreads();
#pragma unroll
                    for (int k = 0; k < SCATTER_VEC * 4; ++k)
                        if (ok[k]) atomicOr(s_bits + ((key[k] >> 5) - lo), 1u << (key[k] & 31));
                    __syncthreads();
                    for (uint32_t w = threadIdx.x; w < span; w += SCATTER_THREADS) {
                        const uint32_t u = s_bits[w];
                        if (u) atomicOr(bits + lo + w, u);
                    }
                    // The next tile's zeroing follows the next tile's min/max barrier.
                    continue;
                }
            }
        }

        const bool aggregate =
            MODE == kWarpAgg || MODE == kSmem ||
            (wmin <= wmax && (wmax >> 5) - (wmin >> 5) < kWarpAggSpanWords);
        if (aggregate) {
#pragma unroll
            for (int k = 0; k < SCATTER_VEC * 4; ++k) or_warp_aggregated(bits, key[k], ok[k], lane);
        } else {
#pragma unroll
            for (int k = 0; k < SCATTER_VEC * 4; ++k)
                if (ok[k]) atomicOr(bits + (key[k] >> 5), 1u << (key[k] & 31));
        }
    }

    const uint32_t wm = __reduce_max_sync(kFull, run_max);
    const uint32_t wb = __reduce_add_sync(kFull, run_bad);
    if (lane == 0) {
        if (wm) atomicMax(&ctrl->max_key, wm);
        if (wb) atomicAdd(&ctrl->bad_keys, wb);
    }
}

// ---------------------------------------------------------------------------
// K3: bitset scan with single-pass decoupled lookback.
//
// Tile = SCAN_ROUNDS rounds x SCAN_THREADS consecutive words; thread t owns
// word (round * 256 + t) of every round (coalesced 4-byte loads, 8 in flight).
// 1. popc + warp inclusive scans for all rounds; per-warp totals to SMEM.
// 2. warp 0: per-round exclusive offsets, tile aggregate, publish AGG, look
//    back over predecessors 32 at a time, publish PREFIX (64-bit {flag,count}).
// 3. per round: each thread extracts its word's set bits (ffs / w &= w-1) into
//    a padded SMEM stage (index p + p/32: conflict-free for dense words), then
//    the block stores the round's keys with consecutive, coalesced stores.
template <bool CLEAR>
__global__ void __launch_bounds__(SCAN_THREADS)
    scan_kernel(uint32_t* __restrict__ bits, unsigned long long n_words_param, uint32_t key_base,
                uint32_t* __restrict__ out, unsigned long long out_cap, Ctrl* __restrict__ ctrl,
                unsigned long long* __restrict__ status, unsigned long long* __restrict__ d_total) {
    constexpr int kStage = SCAN_THREADS * 32;
    __shared__ uint32_t s_stage[kStage + kStage / 32];
    __shared__ uint32_t s_warp[SCAN_ROUNDS][SCAN_THREADS / 32];
    __shared__ uint32_t s_rtot[SCAN_ROUNDS];
    __shared__ unsigned long long s_prefix;
    __shared__ unsigned s_tile;

    const unsigned lane = threadIdx.x & 31;
    const unsigned warp = threadIdx.x >> 5;
    const unsigned long long n_words =
        n_words_param ? n_words_param
                      : (static_cast<unsigned long long>(
                             *reinterpret_cast<volatile unsigned int*>(&ctrl->max_key)) >> 5) + 1;
    const unsigned long long n_tiles = (n_words + SCAN_TILE_WORDS - 1) / SCAN_TILE_WORDS;

    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&ctrl->ticket, 1u);
        __syncthreads();
        const unsigned tile = s_tile;
        if (tile >= n_tiles) break;

        const unsigned long long wbase = static_cast<unsigned long long>(tile) * SCAN_TILE_WORDS;
        uint32_t w[SCAN_ROUNDS];
        uint32_t incl[SCAN_ROUNDS];
#pragma unroll
        for (int r = 0; r < SCAN_ROUNDS; ++r) {
            const unsigned long long idx = wbase + r * SCAN_THREADS + threadIdx.x;
            w[r] = idx < n_words ? __ldcs(bits + idx) : 0u;
        }
#pragma unroll
        for (int r = 0; r < SCAN_ROUNDS; ++r) {
            incl[r] = __popc(w[r]);
            if (CLEAR && w[r]) bits[wbase + r * SCAN_THREADS + threadIdx.x] = 0u;
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
            for (int r = 0; r < SCAN_ROUNDS; ++r) {
                const uint32_t o = __shfl_up_sync(kFull, incl[r], off);
                if (lane >= static_cast<unsigned>(off)) incl[r] += o;
            }
        }
        if (lane == 31) {
#pragma unroll
            for (int r = 0; r < SCAN_ROUNDS; ++r) s_warp[r][warp] = incl[r];
        }
        __syncthreads();

        if (warp == 0) {
            uint32_t rt = 0;
            if (lane < SCAN_ROUNDS) {
#pragma unroll
                for (int q = 0; q < SCAN_THREADS / 32; ++q) {
                    const uint32_t x = s_warp[lane][q];
                    s_warp[lane][q] = rt;
                    rt += x;
                }
                s_rtot[lane] = rt;
            }
            const unsigned long long agg = __reduce_add_sync(kFull, rt);
            unsigned long long prefix = 0;
            if (tile == 0) {
                if (lane == 0) st_relaxed_u64(status, kFlagPrefix | agg);
            } else {
                if (lane == 0) st_relaxed_u64(status + tile, kFlagAgg | agg);
                long long end = tile;
                for (;;) {
                    const long long idx = end - 1 - static_cast<long long>(lane);
                    unsigned long long s = idx >= 0 ? ld_relaxed_u64(status + idx) : kFlagPrefix;
                    while (__any_sync(kFull, (s >> 62) == 0)) {
                        if ((s >> 62) == 0) s = ld_relaxed_u64(status + idx);
                    }
                    const unsigned pm = __ballot_sync(kFull, (s >> 62) == 2);
                    const unsigned long long val = s & kValueMask;
                    if (pm) {
                        const unsigned first = __ffs(pm) - 1;
                        prefix += warp_sum_u64(lane <= first ? val : 0ull);
                        break;
                    }
                    prefix += warp_sum_u64(val);
                    end -= 32;
                }
                if (lane == 0) st_relaxed_u64(status + tile, kFlagPrefix | (prefix + agg));
            }
            if (lane == 0) {
                s_prefix = prefix;
                if (tile == n_tiles - 1) {
                    ctrl->total = prefix + agg;
                    if (d_total) *d_total = prefix + agg;
                }
            }
        }
        __syncthreads();

        unsigned long long obase = s_prefix;
#pragma unroll
        for (int r = 0; r < SCAN_ROUNDS; ++r) {
            const uint32_t rtot = s_rtot[r];
            if (rtot == 0) continue;  // block-uniform
            uint32_t x = w[r];
            uint32_t pos = s_warp[r][warp] + incl[r] - __popc(x);
            const uint32_t kb =
                key_base + static_cast<uint32_t>((wbase + r * SCAN_THREADS + threadIdx.x) << 5);
            while (x) {
                const int b = __ffs(x) - 1;
                x &= x - 1;
                s_stage[pos + (pos >> 5)] = kb + static_cast<uint32_t>(b);
                ++pos;
            }
            __syncthreads();
            for (uint32_t p = threadIdx.x; p < rtot; p += SCAN_THREADS) {
                const unsigned long long g = obase + p;
                if (g < out_cap) __stcs(out + g, s_stage[p + (p >> 5)]);
            }
            obase += rtot;
            __syncthreads();
        }
    }
}

template <int MODE, bool CHECK>
cudaError_t launch_scatter_t(const uint4* vec, size_t n_vec, const uint32_t* head, int n_head,
                             const uint32_t* tail, int n_tail, uint32_t* bits, uint32_t limit,
                             Ctrl* ctrl, int blocks, cudaStream_t stream) {
    const size_t smem = (MODE == kAuto || MODE == kSmem) ? SCATTER_SMEM_WORDS * sizeof(uint32_t) : 0;
    scatter_kernel<MODE, CHECK><<<blocks, SCATTER_THREADS, smem, stream>>>(
        vec, n_vec, head, n_head, tail, n_tail, bits, limit, ctrl);
    return cudaGetLastError();
}

template <bool CHECK>
cudaError_t launch_scatter_mode(int mode, const uint4* vec, size_t n_vec, const uint32_t* head,
                                int n_head, const uint32_t* tail, int n_tail, uint32_t* bits,
                                uint32_t limit, Ctrl* ctrl, int blocks, cudaStream_t stream) {
    switch (mode) {
        case kPlain:
            return launch_scatter_t<kPlain, CHECK>(vec, n_vec, head, n_head, tail, n_tail, bits,
                                                   limit, ctrl, blocks, stream);
        case kWarpAgg:
            return launch_scatter_t<kWarpAgg, CHECK>(vec, n_vec, head, n_head, tail, n_tail, bits,
                                                     limit, ctrl, blocks, stream);
        case kSmem:
            return launch_scatter_t<kSmem, CHECK>(vec, n_vec, head, n_head, tail, n_tail, bits,
                                                  limit, ctrl, blocks, stream);
        default:
            return launch_scatter_t<kAuto, CHECK>(vec, n_vec, head, n_head, tail, n_tail, bits,
                                                  limit, ctrl, blocks, stream);
    }
}

}  // namespace

cudaError_t query_geometry(int device, LaunchGeometry* geo) {
    int sms = 0;
    cudaError_t err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (err != cudaSuccess) return err;
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, scatter_kernel<kAuto, true>, SCATTER_THREADS,
        SCATTER_SMEM_WORDS * sizeof(uint32_t));
    if (err != cudaSuccess) return err;
    geo->scatter_blocks = sms * (per_sm > 0 ? per_sm : 1);
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scan_kernel<true>, SCAN_THREADS, 0);
    if (err != cudaSuccess) return err;
    geo->scan_blocks = sms * (per_sm > 0 ? per_sm : 1);
    geo->fill_blocks = sms * 4;
    return cudaSuccess;
}

cudaError_t launch_scatter(const uint32_t* keys, size_t n, uint32_t* bits, uint64_t key_range,
                           Ctrl* ctrl, int mode, const LaunchGeometry& geo, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    const uintptr_t addr = reinterpret_cast<uintptr_t>(keys);
    size_t n_head = ((16 - (addr & 15)) & 15) / 4;
    if (n_head > n) n_head = n;
    const size_t n_vec = (n - n_head) / 4;
    const size_t n_tail = n - n_head - 4 * n_vec;
    const uint4* vec = reinterpret_cast<const uint4*>(keys + n_head);
    const uint32_t* tail = keys + n_head + 4 * n_vec;
    const size_t vec_tiles = (n_vec + SCATTER_THREADS * SCATTER_VEC - 1) / (SCATTER_THREADS * SCATTER_VEC);
    int blocks = geo.scatter_blocks;
    if (vec_tiles < static_cast<size_t>(blocks)) blocks = vec_tiles > 0 ? static_cast<int>(vec_tiles) : 1;
    const bool check = key_range < (1ull << 32);
    const uint32_t limit = check ? static_cast<uint32_t>(key_range) : 0u;
    if (check)
        return launch_scatter_mode<true>(mode, vec, n_vec, keys, static_cast<int>(n_head), tail,
                                         static_cast<int>(n_tail), bits, limit, ctrl, blocks, stream);
    return launch_scatter_mode<false>(mode, vec, n_vec, keys, static_cast<int>(n_head), tail,
                                      static_cast<int>(n_tail), bits, limit, ctrl, blocks, stream);
}

// OR-gather of up to 8 bitset slices (local and peer memory): 16-byte loads
// from every source in flight before the OR, streaming store. Distinct keys
// set disjoint bits, so OR equals the reduce-scatter's SUM; duplicates across
// ranks lose bits either way and the popcount total exposes them.
__global__ void __launch_bounds__(256)
    or_gather_kernel(OrSources srcs, uint32_t* __restrict__ dst, unsigned long long n_words) {
    const unsigned long long nv = n_words / 4;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    const bool aligned = ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) && [&] {
        for (int s = 0; s < srcs.n; ++s)
            if (reinterpret_cast<uintptr_t>(srcs.p[s]) & 15) return false;
        return true;
    }();
    if (aligned) {
        for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < nv; i += stride) {
            uint4 v[MAX_OR_SOURCES];
#pragma unroll
            for (int s = 0; s < MAX_OR_SOURCES; ++s)
                if (s < srcs.n) v[s] = __ldcs(reinterpret_cast<const uint4*>(srcs.p[s]) + i);
            uint4 r = v[0];
#pragma unroll
            for (int s = 1; s < MAX_OR_SOURCES; ++s)
                if (s < srcs.n) {
                    r.x |= v[s].x;
                    r.y |= v[s].y;
                    r.z |= v[s].z;
                    r.w |= v[s].w;
                }
            __stcs(reinterpret_cast<uint4*>(dst) + i, r);
        }
    }
    for (unsigned long long i = (aligned ? 4 * nv : 0) + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
         i < n_words; i += stride) {
        uint32_t r = 0;
        for (int s = 0; s < srcs.n; ++s) r |= srcs.p[s][i];
        dst[i] = r;
    }
}

cudaError_t launch_or_gather(const OrSources& srcs, uint32_t* dst, uint64_t n_words,
                             const LaunchGeometry& geo, cudaStream_t stream) {
    if (n_words == 0) return cudaSuccess;
    or_gather_kernel<<<geo.fill_blocks, 256, 0, stream>>>(srcs, dst, n_words);
    return cudaGetLastError();
}

cudaError_t launch_scan(const uint32_t* bits, uint64_t n_words, uint32_t key_base, uint32_t* out,
                        uint64_t out_capacity, Ctrl* ctrl, unsigned long long* status,
                        unsigned long long* d_total, int clear, const LaunchGeometry& geo,
                        cudaStream_t stream) {
    int blocks = geo.scan_blocks;
    if (n_words != 0) {
        const size_t tiles = scan_tiles(n_words);
        if (tiles < static_cast<size_t>(blocks)) blocks = static_cast<int>(tiles);
    }
    uint32_t* b = const_cast<uint32_t*>(bits);
    if (clear)
        scan_kernel<true><<<blocks, SCAN_THREADS, 0, stream>>>(b, n_words, key_base, out,
                                                              out_capacity, ctrl, status, d_total);
    else
        scan_kernel<false><<<blocks, SCAN_THREADS, 0, stream>>>(b, n_words, key_base, out,
                                                               out_capacity, ctrl, status, d_total);
    return cudaGetLastError();
}

}  // namespace bws_gpu
