// Other key widths of bws_sort (sm_100a): 8-, 16- and 64-bit keys, the
// reference's with_width dispatch (dispatch.hpp:17-40) on the GPU.
//
// 8/16-bit keys (at most 2^16 values) take a counting sort over the whole
// value range (the reference's counting_sort, baselines.hpp:99-122, with the
// full span of the type), in three kernels:
//   KW1 small_hist    per CTA: 32-bit SMEM counters over windows of <= 2^15
//                     values (16-byte loads of the CTA's contiguous chunk),
//                     flushed to a global u64 histogram      (read n * width)
//   KW2 small_scan    one CTA: inclusive prefix of the histogram
//   KW3 small_expand  output tiles of 8192 slots: slot i takes the value whose
//                     inclusive prefix first exceeds i (binary search in an
//                     SMEM window of the prefix), coalesced   (write n * width)
// Signed keys are biased (x ^ 0x80 / 0x8000) on load and unbiased on store.
//
// 64-bit keys whose span max - min is below 2^32 are narrowed on the GPU to
// u32 offsets from the minimum, sorted by the 32-bit pipeline (repeats
// included) and widened back; wider spans take a stable LSD radix sort with
// 8-bit digits (KR0-KR3 below). The bias 2^63 maps signed order onto unsigned.
#include "kernels.h"
#include "device_util.cuh"

namespace bws_gpu {
namespace {

using namespace dev;

constexpr int SW_THREADS = 1024;
constexpr int SW_WIN = 1 << 15;           // SMEM counters per histogram window (128 KB)
constexpr int SW_TILE = 8192;             // output slots per expansion tile
constexpr int SW_PWIN = 2048;             // prefix entries per expansion window

template <class T>
__device__ __forceinline__ uint32_t load_biased(const T* p, size_t i, uint32_t bias) {
    return static_cast<uint32_t>(p[i]) ^ bias;
}

template <class T>
__global__ void __launch_bounds__(SW_THREADS, 1)
    small_hist_kernel(const T* __restrict__ in, size_t n, uint32_t bias, unsigned long long* __restrict__ hist) {
    constexpr int R = 1 << (8 * sizeof(T));
    constexpr int WIN = R < SW_WIN ? R : SW_WIN;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem_raw);
    // this CTA's contiguous chunk, in whole 16-byte vectors where possible
    const size_t per = (n + gridDim.x - 1) / gridDim.x;
    const size_t c0 = min(n, per * blockIdx.x), c1 = min(n, c0 + per);
    constexpr int V = 16 / sizeof(T);  // keys per 16-byte vector
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(in + c0);
    size_t head = ((16 - (a0 & 15)) & 15) / sizeof(T);
    if (head > c1 - c0) head = c1 - c0;
    const size_t nv = (c1 - c0 - head) / V;
    const uint4* v4 = reinterpret_cast<const uint4*>(in + c0 + head);
    const size_t tail0 = c0 + head + nv * V;
    for (int w0 = 0; w0 < R; w0 += WIN) {
        for (int i = threadIdx.x; i < WIN; i += SW_THREADS) s_cnt[i] = 0u;
        __syncthreads();
        auto add = [&](uint32_t u) {
            const uint32_t x = u - static_cast<uint32_t>(w0);
            if (x < static_cast<uint32_t>(WIN)) atomicAdd(s_cnt + x, 1u);
        };
        for (size_t i = c0 + threadIdx.x; i < c0 + head; i += SW_THREADS) add(load_biased(in, i, bias));
        for (size_t i = threadIdx.x; i < nv; i += SW_THREADS) {
            const uint4 v = __ldcs(v4 + i);
            const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
            for (int j = 0; j < V; ++j) add(static_cast<uint32_t>(e[j]) ^ bias);
        }
        for (size_t i = tail0 + threadIdx.x; i < c1; i += SW_THREADS) add(load_biased(in, i, bias));
        __syncthreads();
        for (int i = threadIdx.x; i < WIN; i += SW_THREADS)
            if (s_cnt[i]) atomicAdd(hist + w0 + i, static_cast<unsigned long long>(s_cnt[i]));
        __syncthreads();
    }
}

// One CTA: incl[v] = hist[0] + ... + hist[v], v < R (R a multiple of 1024).
__global__ void __launch_bounds__(1024)
    small_scan_kernel(const unsigned long long* __restrict__ hist, int R, unsigned long long* __restrict__ incl) {
    __shared__ unsigned long long s_w[32];
    const int per = R / 1024;
    const int b0 = threadIdx.x * per;
    unsigned long long local = 0;
    for (int i = 0; i < per; ++i) local += hist[b0 + i];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long x = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned long long o = __shfl_up_sync(kFull, x, off);
        if (lane >= static_cast<unsigned>(off)) x += o;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const unsigned long long w = s_w[lane];
        unsigned long long y = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned long long o = __shfl_up_sync(kFull, y, off);
            if (lane >= static_cast<unsigned>(off)) y += o;
        }
        s_w[lane] = y - w;
    }
    __syncthreads();
    unsigned long long run = s_w[warp] + x - local;
    for (int i = 0; i < per; ++i) {
        run += hist[b0 + i];
        incl[b0 + i] = run;
    }
}

// Smallest v in [0, R) with incl[v] > s (global memory; incl[R-1] = n > s).
__device__ __forceinline__ int upper_value(const unsigned long long* incl, int R, unsigned long long s) {
    int lo = 0, len = R;
    while (len > 1) {
        const int half = len >> 1;
        if (incl[lo + half - 1] <= s) lo += half;
        len -= half;
    }
    return lo;
}

template <class T>
__global__ void __launch_bounds__(SW_THREADS)
    small_expand_kernel(const unsigned long long* __restrict__ incl, size_t n, uint32_t bias, T* __restrict__ out) {
    constexpr int R = 1 << (8 * sizeof(T));
    constexpr int PW = R < SW_PWIN ? R : SW_PWIN;
    __shared__ unsigned long long s_p[PW];
    __shared__ int s_v;
    const size_t tiles = (n + SW_TILE - 1) / SW_TILE;
    for (size_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        unsigned long long s = static_cast<unsigned long long>(t) * SW_TILE;
        const unsigned long long end = min(static_cast<unsigned long long>(n), s + SW_TILE);
        while (s < end) {  // block-uniform
            if (threadIdx.x == 0) s_v = upper_value(incl, R, s);
            __syncthreads();
            const int v0 = s_v;
            for (int i = threadIdx.x; i < PW; i += SW_THREADS)
                s_p[i] = v0 + i < R ? incl[v0 + i] : ~0ull;
            __syncthreads();
            const unsigned long long wend = min(end, s_p[PW - 1]);  // slots the window covers
            for (unsigned long long slot = s + threadIdx.x; slot < wend; slot += SW_THREADS) {
                int lo = 0, len = PW;
                while (len > 1) {
                    const int half = len >> 1;
                    if (s_p[lo + half - 1] <= slot) lo += half;
                    len -= half;
                }
                out[slot] = static_cast<T>(static_cast<uint32_t>(v0 + lo) ^ bias);
            }
            s = wend;
            __syncthreads();
        }
    }
}

__global__ void minmax64_kernel(const unsigned long long* __restrict__ in, size_t n, unsigned long long bias,
                                unsigned long long* __restrict__ mm) {
    unsigned long long lo = ~0ull, hi = 0;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const unsigned long long u = __ldcs(in + i) ^ bias;
        lo = min(lo, u);
        hi = max(hi, u);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        lo = min(lo, __shfl_xor_sync(kFull, lo, off));
        hi = max(hi, __shfl_xor_sync(kFull, hi, off));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mm, lo);
        atomicMax(mm + 1, hi);
    }
}

__global__ void narrow64_kernel(const unsigned long long* __restrict__ in, size_t n, unsigned long long bias,
                                const unsigned long long* __restrict__ mm, uint32_t* __restrict__ out) {
    const unsigned long long lo = mm[0];
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<uint32_t>((__ldcs(in + i) ^ bias) - lo);
}

__global__ void widen64_kernel(const uint32_t* __restrict__ in, size_t n, unsigned long long bias,
                               const unsigned long long* __restrict__ mm, unsigned long long* __restrict__ out) {
    const unsigned long long lo = mm[0];
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        __stcs(out + i, (static_cast<unsigned long long>(__ldcs(in + i)) + lo) ^ bias);
}

template <class T>
cudaError_t launch_small(T* data, size_t n, int is_unsigned, unsigned long long* scratch, const LaunchGeometry& geo,
                         cudaStream_t stream, KernelTimer* timer) {
    constexpr int R = 1 << (8 * sizeof(T));
    constexpr int WIN = R < SW_WIN ? R : SW_WIN;
    const uint32_t bias = is_unsigned ? 0u : (1u << (8 * sizeof(T) - 1));
    unsigned long long* hist = scratch;              // 2^16 counters (the scan reads >= 1024)
    unsigned long long* incl = scratch + (1 << 16);  // 2^16 prefixes
    constexpr int RS = R < 1024 ? 1024 : R;
    cudaError_t err = cudaMemsetAsync(hist, 0, RS * sizeof(unsigned long long), stream);
    if (err != cudaSuccess) return err;
    // enough CTAs to stream the input, few enough that the flushes stay small
    int blocks = geo.multiset_blocks;
    const size_t min_chunk = size_t(1) << 16;
    if (static_cast<size_t>(blocks) * min_chunk > n) blocks = static_cast<int>((n + min_chunk - 1) / min_chunk);
    if (timer) timer->before(stream);
    small_hist_kernel<T><<<blocks, SW_THREADS, WIN * sizeof(uint32_t), stream>>>(data, n, bias, hist);
    if (timer) timer->after("width_hist", stream);
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
    if (timer) timer->before(stream);
    small_scan_kernel<<<1, 1024, 0, stream>>>(hist, RS, incl);
    if (timer) timer->after("width_scan", stream);
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
    const size_t tiles = (n + SW_TILE - 1) / SW_TILE;
    int eblocks = geo.multiset_blocks * 2;
    if (tiles < static_cast<size_t>(eblocks)) eblocks = static_cast<int>(tiles);
    if (timer) timer->before(stream);
    small_expand_kernel<T><<<eblocks, SW_THREADS, 0, stream>>>(incl, n, bias, data);
    if (timer) timer->after("width_expand", stream);
    return cudaGetLastError();
}


// ---- 64-bit keys of any span: stable LSD radix sort, 8-bit digits ----------
// (the reference's own algorithm family: bitsort.hpp:84-129 is an LSD radix
// sort with 1-bit digits and stable partitions; here 8-bit digits, and digits
// on which every key agrees are skipped, like skip_empty_bits.)
//   KR0 rx_hist_all  global histogram of all 8 digits in one read (host then
//                    skips the constant digits)
//   per remaining digit:
//   KR1 rx_hist      per-CTA digit histogram of its contiguous chunk
//   KR2 rx_offsets   one CTA: exclusive prefix in (digit, CTA) order
//   KR3 rx_scatter   stable scatter: the chunk in rounds of 256 keys (thread t
//                    takes key r*256 + t); rank inside a warp from match.any,
//                    across the 8 warps from a per-round digit x warp count
//                    table (double-buffered: 2 barriers per round)
constexpr int RX_THREADS = 256;
constexpr int RX_WARPS = RX_THREADS / 32;

__device__ __forceinline__ void rx_chunk(size_t n, size_t& c0, size_t& c1) {
    const size_t per = (n + gridDim.x - 1) / gridDim.x;
    c0 = min(n, per * blockIdx.x);
    c1 = min(n, c0 + per);
}

__global__ void __launch_bounds__(RX_THREADS)
    rx_hist_all_kernel(const unsigned long long* __restrict__ in, size_t n, unsigned long long bias,
                       unsigned long long* __restrict__ hist /* [8][256] */) {
    __shared__ uint32_t s_h[8 * 256];
    for (int i = threadIdx.x; i < 8 * 256; i += RX_THREADS) s_h[i] = 0u;
    __syncthreads();
    for (size_t i = blockIdx.x * static_cast<size_t>(RX_THREADS) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * RX_THREADS) {
        const unsigned long long k = __ldcs(in + i) ^ bias;
#pragma unroll
        for (int d = 0; d < 8; ++d) atomicAdd(&s_h[d * 256 + ((k >> (8 * d)) & 255u)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 8 * 256; i += RX_THREADS)
        if (s_h[i]) atomicAdd(hist + i, static_cast<unsigned long long>(s_h[i]));
}

__global__ void __launch_bounds__(RX_THREADS)
    rx_hist_kernel(const unsigned long long* __restrict__ in, size_t n, unsigned long long xin, int shift,
                   uint32_t* __restrict__ H /* [256][P] */) {
    __shared__ uint32_t s_h[256];
    s_h[threadIdx.x] = 0u;
    __syncthreads();
    size_t c0, c1;
    rx_chunk(n, c0, c1);
    for (size_t i = c0 + threadIdx.x; i < c1; i += RX_THREADS)
        atomicAdd(&s_h[((__ldcs(in + i) ^ xin) >> shift) & 255u], 1u);
    __syncthreads();
    H[static_cast<size_t>(threadIdx.x) * gridDim.x + blockIdx.x] = s_h[threadIdx.x];
}

// One CTA: H[d][c] <- (keys of digits < d) + (keys of digit d in CTAs < c),
// i.e. the exclusive prefix of H in digit-major order. Warp-per-row passes
// (coalesced): row totals, their prefix, then row scans carrying it.
__global__ void __launch_bounds__(1024) rx_offsets_kernel(uint32_t* __restrict__ H, int P) {
    __shared__ uint32_t s_tot[256];
    __shared__ uint32_t s_w[32];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int d = warp; d < 256; d += 32) {
        uint32_t sum = 0;
        for (int c = lane; c < P; c += 32) sum += H[static_cast<size_t>(d) * P + c];
        sum = __reduce_add_sync(kFull, sum);
        if (lane == 0) s_tot[d] = sum;
    }
    __syncthreads();
    if (threadIdx.x < 256) {  // exclusive prefix of the 256 row totals
        const uint32_t x = s_tot[threadIdx.x];
        const uint32_t incl = warp_incl_scan(x, lane);
        if (lane == 31) s_w[warp] = incl;
        __syncwarp();
        s_tot[threadIdx.x] = incl - x;  // warp-local for now
    }
    __syncthreads();
    if (threadIdx.x < 8) {
        uint32_t run = 0;
        for (int w = 0; w < static_cast<int>(threadIdx.x); ++w) run += s_w[w];
        s_w[8 + threadIdx.x] = run;
    }
    __syncthreads();
    if (threadIdx.x < 256) s_tot[threadIdx.x] += s_w[8 + warp];
    __syncthreads();
    for (int d = warp; d < 256; d += 32) {
        uint32_t carry = s_tot[d];
        for (int c0 = 0; c0 < P; c0 += 32) {
            const int c = c0 + static_cast<int>(lane);
            const uint32_t x = c < P ? H[static_cast<size_t>(d) * P + c] : 0u;
            const uint32_t incl = warp_incl_scan(x, lane);
            if (c < P) H[static_cast<size_t>(d) * P + c] = carry + incl - x;
            carry += __shfl_sync(kFull, incl, 31);
        }
    }
}

constexpr int RX_KPT = 16;                         // keys per thread per round
constexpr int RX_ROUND = RX_KPT * RX_THREADS;      // 4096 keys per round
__global__ void __launch_bounds__(RX_THREADS, 4)
    rx_scatter_kernel(const unsigned long long* __restrict__ in, unsigned long long* __restrict__ out, size_t n,
                      unsigned long long xin, unsigned long long xout, int shift,
                      const uint32_t* __restrict__ H) {
    // Round r covers keys [r0, r0 + 4096) of the CTA's chunk; warp w takes
    // [r0 + 512w, r0 + 512(w+1)), 32 consecutive keys per step j. Stable rank:
    // per-warp running digit counts (match.any per step, warp-synchronous),
    // their prefix over the warps, and the digit's run start in the round.
    // The round is counting-sorted into SMEM and written run by run, so the
    // stores of a digit's run are consecutive (coalesced) instead of scattered.
    __shared__ uint32_t s_wcnt[RX_WARPS][256];             // warp x digit counts -> offsets
    __shared__ unsigned long long s_stage[RX_ROUND];
    __shared__ uint32_t s_base[256];                       // next output slot per digit
    __shared__ uint32_t s_dstart[256];                     // digit run start in the round
    __shared__ uint32_t s_w[RX_WARPS];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned t = threadIdx.x;                        // also: the digit this thread scans
    s_base[t] = H[static_cast<size_t>(t) * gridDim.x + blockIdx.x];
    size_t c0, c1;
    rx_chunk(n, c0, c1);
    const unsigned lt = lanemask_lt();
    for (size_t r0 = c0; r0 < c1; r0 += RX_ROUND) {
        const uint32_t round_n = static_cast<uint32_t>(min(static_cast<size_t>(RX_ROUND), c1 - r0));
#pragma unroll
        for (int q = 0; q < 256 / 32; ++q) s_wcnt[warp][q * 32 + lane] = 0u;
        __syncwarp();
        unsigned long long k[RX_KPT];
        uint32_t dr[RX_KPT];  // digit << 16 | rank among the warp's keys of that digit (256: none)
        const uint32_t wfirst = warp * (RX_KPT * 32) + lane;
#pragma unroll
        for (int j = 0; j < RX_KPT; ++j)  // every load in flight before the first rank
            k[j] = wfirst + j * 32 < round_n ? __ldcs(in + r0 + wfirst + j * 32) : 0ull;
#pragma unroll
        for (int j = 0; j < RX_KPT; ++j) {
            const bool ok = wfirst + j * 32 < round_n;
            k[j] ^= xin;
            const uint32_t d = ok ? static_cast<uint32_t>((k[j] >> shift) & 255u) : 256u;
            const unsigned peers = __match_any_sync(kFull, d);
            const int leader = __ffs(peers) - 1;
            uint32_t old = 0;
            if (ok && static_cast<int>(lane) == leader) {
                old = s_wcnt[warp][d];
                s_wcnt[warp][d] = old + __popc(peers);
            }
            old = __shfl_sync(kFull, old, leader);
            dr[j] = (d << 16) | (old + __popc(peers & lt));
            __syncwarp();
        }
        __syncthreads();
        uint32_t total;
        {  // digit t: exclusive prefix over the warps, then over the digits
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < RX_WARPS; ++w) {
                const uint32_t c = s_wcnt[w][t];
                s_wcnt[w][t] = run;
                run += c;
            }
            total = run;
            const uint32_t incl = warp_incl_scan(total, lane);
            if (lane == 31) s_w[warp] = incl;
            __syncthreads();
            uint32_t wbase = 0;
#pragma unroll
            for (int w = 0; w < RX_WARPS; ++w) wbase += w < static_cast<int>(warp) ? s_w[w] : 0u;
            s_dstart[t] = wbase + incl - total;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < RX_KPT; ++j) {
            const uint32_t d = dr[j] >> 16;
            if (d < 256u) s_stage[s_dstart[d] + s_wcnt[warp][d] + (dr[j] & 0xffffu)] = k[j];
        }
        __syncthreads();
        for (uint32_t i = t; i < round_n; i += RX_THREADS) {
            const unsigned long long key = s_stage[i];
            const uint32_t d = static_cast<uint32_t>((key >> shift) & 255u);
            __stcs(out + s_base[d] + (i - s_dstart[d]), key ^ xout);
        }
        __syncthreads();
        s_base[t] += total;
    }
}

}  // namespace

std::size_t width_scratch_bytes() { return 2 * (std::size_t(1) << 16) * sizeof(unsigned long long) + 64; }

cudaError_t configure_width_kernels(int device, LaunchGeometry* geo) {
    (void)device;
    (void)geo;
    return cudaFuncSetAttribute(small_hist_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                SW_WIN * static_cast<int>(sizeof(uint32_t)));
}

cudaError_t launch_sort_small(void* data, std::size_t n, int width, int is_unsigned, void* scratch,
                              const LaunchGeometry& geo, cudaStream_t stream, int* launches, KernelTimer* timer) {
    if (launches) *launches = 3;
    if (n == 0) return cudaSuccess;
    auto* s = static_cast<unsigned long long*>(scratch);
    if (width == 8) return launch_small(static_cast<uint8_t*>(data), n, is_unsigned, s, geo, stream, timer);
    if (width == 16) return launch_small(static_cast<uint16_t*>(data), n, is_unsigned, s, geo, stream, timer);
    return cudaErrorInvalidValue;
}

cudaError_t launch_minmax64(const std::uint64_t* keys, std::size_t n, int is_unsigned, void* scratch,
                            const LaunchGeometry& geo, cudaStream_t stream) {
    auto* mm = static_cast<unsigned long long*>(scratch);
    const unsigned long long init[2] = {~0ull, 0ull};
    cudaError_t err = cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, stream);
    if (err != cudaSuccess) return err;
    minmax64_kernel<<<geo.fill_blocks, 256, 0, stream>>>(reinterpret_cast<const unsigned long long*>(keys), n,
                                                          is_unsigned ? 0ull : (1ull << 63), mm);
    return cudaGetLastError();
}

cudaError_t launch_narrow64(const std::uint64_t* keys, std::size_t n, int is_unsigned, const void* scratch,
                            std::uint32_t* out, const LaunchGeometry& geo, cudaStream_t stream) {
    narrow64_kernel<<<geo.fill_blocks, 256, 0, stream>>>(reinterpret_cast<const unsigned long long*>(keys), n,
                                                          is_unsigned ? 0ull : (1ull << 63),
                                                          static_cast<const unsigned long long*>(scratch), out);
    return cudaGetLastError();
}

cudaError_t launch_widen64(const std::uint32_t* sorted, std::size_t n, int is_unsigned, const void* scratch,
                           std::uint64_t* out, const LaunchGeometry& geo, cudaStream_t stream) {
    widen64_kernel<<<geo.fill_blocks, 256, 0, stream>>>(sorted, n, is_unsigned ? 0ull : (1ull << 63),
                                                         static_cast<const unsigned long long*>(scratch),
                                                         reinterpret_cast<unsigned long long*>(out));
    return cudaGetLastError();
}

}  // namespace bws_gpu

namespace bws_gpu {

std::size_t radix64_scratch_bytes(const LaunchGeometry& geo) {
    return 8 * 256 * sizeof(unsigned long long) + static_cast<std::size_t>(256) * (geo.multiset_blocks * 4) * 4 + 64;
}

cudaError_t launch_radix64_hist(const std::uint64_t* keys, std::size_t n, int is_unsigned, void* scratch,
                                const LaunchGeometry& geo, cudaStream_t stream) {
    auto* hist = static_cast<unsigned long long*>(scratch);
    cudaError_t err = cudaMemsetAsync(hist, 0, 8 * 256 * sizeof(unsigned long long), stream);
    if (err != cudaSuccess) return err;
    rx_hist_all_kernel<<<geo.multiset_blocks * 4, RX_THREADS, 0, stream>>>(
        reinterpret_cast<const unsigned long long*>(keys), n, is_unsigned ? 0ull : (1ull << 63), hist);
    return cudaGetLastError();
}

cudaError_t launch_radix64_pass(const std::uint64_t* in, std::uint64_t* out, std::size_t n, int digit,
                                std::uint64_t xin, std::uint64_t xout, void* scratch, const LaunchGeometry& geo,
                                cudaStream_t stream) {
    const int P = geo.multiset_blocks * 4;  // rx_scatter: 4 resident CTAs per SM (64 registers, 43 KB)
    uint32_t* H = reinterpret_cast<uint32_t*>(static_cast<unsigned char*>(scratch) +
                                              8 * 256 * sizeof(unsigned long long));
    const auto* i64 = reinterpret_cast<const unsigned long long*>(in);
    rx_hist_kernel<<<P, RX_THREADS, 0, stream>>>(i64, n, xin, 8 * digit, H);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    rx_offsets_kernel<<<1, 1024, 0, stream>>>(H, P);
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
    rx_scatter_kernel<<<P, RX_THREADS, 0, stream>>>(i64, reinterpret_cast<unsigned long long*>(out), n, xin, xout,
                                                    8 * digit, H);
    return cudaGetLastError();
}

}  // namespace bws_gpu
