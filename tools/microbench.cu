// Throughput probes for the primitives the bitset sort can be built from
// (development tool; numbers go to profiles/). Each probe issues `iters`
// operations per thread at pseudo-random addresses generated in registers, so
// only the memory primitive is measured.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// global RED.OR to random words in [0, mask]
__global__ void k_red_random(uint32_t* bits, uint32_t mask, int iters, uint32_t seed) {
    uint32_t s = hash32(blockIdx.x * blockDim.x + threadIdx.x + seed);
    for (int i = 0; i < iters; ++i) {
        s = hash32(s + i);
        atomicOr(bits + (s & mask), 1u << (s >> 27));
    }
}

// global RED.OR, lanes hit consecutive words (one 128B line per warp)
__global__ void k_red_coalesced(uint32_t* bits, uint32_t mask, int iters, uint32_t seed) {
    uint32_t s = hash32(blockIdx.x * blockDim.x + (threadIdx.x & ~31u) + seed);
    const uint32_t lane = threadIdx.x & 31;
    for (int i = 0; i < iters; ++i) {
        s = hash32(s + i);
        atomicOr(bits + (((s & mask) & ~31u) | lane), 1u << (s >> 27));
    }
}

// global plain store to random words
__global__ void k_stg_random(uint32_t* bits, uint32_t mask, int iters, uint32_t seed) {
    uint32_t s = hash32(blockIdx.x * blockDim.x + threadIdx.x + seed);
    for (int i = 0; i < iters; ++i) {
        s = hash32(s + i);
        bits[s & mask] = s;
    }
}

// shared atomicOr to random words of a 128 KB bitset
__global__ void k_atoms_random(uint32_t* sink, int iters, uint32_t seed) {
    extern __shared__ uint32_t sm[];
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) sm[i] = 0;
    __syncthreads();
    uint32_t s = hash32(blockIdx.x * blockDim.x + threadIdx.x + seed);
    for (int i = 0; i < iters; ++i) {
        s = hash32(s + i);
        atomicOr(sm + (s & 32767), 1u << (s >> 27));
    }
    __syncthreads();
    if (threadIdx.x == 0) sink[blockIdx.x] = sm[seed & 32767];
}

// shared plain byte store to random bytes of a 128 KB byte map
__global__ void k_sts8_random(uint32_t* sink, int iters, uint32_t seed) {
    extern __shared__ uint32_t sm[];
    unsigned char* b = reinterpret_cast<unsigned char*>(sm);
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) sm[i] = 0;
    __syncthreads();
    uint32_t s = hash32(blockIdx.x * blockDim.x + threadIdx.x + seed);
    for (int i = 0; i < iters; ++i) {
        s = hash32(s + i);
        b[s & 131071] = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) sink[blockIdx.x] = sm[seed & 32767];
}

// streaming read (sum) of n words: HBM read bandwidth
__global__ void k_read(const uint4* p, size_t n4, uint32_t* sink) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

// streaming copy: HBM read+write bandwidth
__global__ void k_copy(const uint4* p, uint4* q, size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        __stcs(q + i, __ldcs(p + i));
}

// streaming write: HBM write bandwidth
__global__ void k_write(uint4* q, size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        __stcs(q + i, make_uint4(i, i, i, i));
}

template <class F>
float time_ms(F f, int reps = 5) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t big = 1ull << 30;  // 4 GiB of words
    uint32_t *buf, *buf2, *sink;
    CK(cudaMalloc(&buf, big * 4));
    CK(cudaMalloc(&buf2, big * 4));
    CK(cudaMalloc(&sink, 1 << 20));
    CK(cudaMemset(buf, 1, big * 4));
    const int threads = 256, iters = 256;
    for (int bps : {4, 8}) {
        const int blocks = sms * bps;
        const double ops = (double)blocks * threads * iters;
        for (uint32_t words_log : {20u, 23u, 25u, 27u}) {
            const uint32_t mask = (1u << words_log) - 1;
            float t = time_ms([&] { k_red_random<<<blocks, threads>>>(buf, mask, iters, 7); });
            printf("{\"probe\":\"red_random\",\"blocks_per_sm\":%d,\"region_MiB\":%u,\"Gops\":%.1f}\n", bps,
                   (1u << words_log) * 4 >> 20, ops / t / 1e6);
            t = time_ms([&] { k_red_coalesced<<<blocks, threads>>>(buf, mask, iters, 7); });
            printf("{\"probe\":\"red_coalesced\",\"blocks_per_sm\":%d,\"region_MiB\":%u,\"Gops\":%.1f}\n", bps,
                   (1u << words_log) * 4 >> 20, ops / t / 1e6);
            t = time_ms([&] { k_stg_random<<<blocks, threads>>>(buf, mask, iters, 7); });
            printf("{\"probe\":\"stg_random\",\"blocks_per_sm\":%d,\"region_MiB\":%u,\"Gops\":%.1f}\n", bps,
                   (1u << words_log) * 4 >> 20, ops / t / 1e6);
        }
    }
    CK(cudaFuncSetAttribute(k_atoms_random, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    CK(cudaFuncSetAttribute(k_sts8_random, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
    for (int threads2 : {256, 512, 1024}) {
        const int blocks = sms;
        const int it2 = 4096;
        const double ops = (double)blocks * threads2 * it2;
        float t = time_ms([&] { k_atoms_random<<<blocks, threads2, 131072>>>(sink, it2, 7); });
        CK(cudaGetLastError());
        printf("{\"probe\":\"atoms_random_128KB\",\"threads\":%d,\"Gops\":%.1f}\n", threads2, ops / t / 1e6);
        t = time_ms([&] { k_sts8_random<<<blocks, threads2, 131072>>>(sink, it2, 7); });
        printf("{\"probe\":\"sts8_random_128KB\",\"threads\":%d,\"Gops\":%.1f}\n", threads2, ops / t / 1e6);
    }
    const size_t n4 = big / 4;
    for (int bps : {2, 4, 8}) {
        const int blocks = sms * bps;
        float t = time_ms([&] { k_read<<<blocks, 512>>>(reinterpret_cast<const uint4*>(buf), n4, sink); });
        printf("{\"probe\":\"hbm_read_4GiB\",\"blocks_per_sm\":%d,\"GBps\":%.1f}\n", bps, big * 4 / t / 1e6);
        t = time_ms([&] { k_copy<<<blocks, 512>>>(reinterpret_cast<const uint4*>(buf), reinterpret_cast<uint4*>(buf2), n4); });
        printf("{\"probe\":\"hbm_copy_4GiB\",\"blocks_per_sm\":%d,\"GBps\":%.1f}\n", bps, 2.0 * big * 4 / t / 1e6);
        t = time_ms([&] { k_write<<<blocks, 512>>>(reinterpret_cast<uint4*>(buf2), n4); });
        printf("{\"probe\":\"hbm_write_4GiB\",\"blocks_per_sm\":%d,\"GBps\":%.1f}\n", bps, big * 4 / t / 1e6);
    }
    float t = time_ms([&] { cudaMemsetAsync(buf2, 0, big * 4); });
    printf("{\"probe\":\"memset_4GiB\",\"GBps\":%.1f}\n", big * 4 / t / 1e6);
    return 0;
}
