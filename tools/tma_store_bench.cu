// Microbenchmark: throughput of many small cp.async.bulk SMEM->global stores
// (the KB3 write phase as bulk copies: one copy per bucket run per tile).
// Each CTA fills a 80 KB SMEM buffer, then repeatedly issues `runs` bulk
// stores of `bytes` each (run i -> a different 2 MB-strided global region),
// waits for their SMEM reads, and repeats. Reports GB/s and copies/s.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/tma_store_bench tools/tma_store_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void bulk_store_kernel(uint32_t* out, int runs, int bytes, int iters, size_t region_stride) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint32_t* buf = reinterpret_cast<uint32_t*>(smem);
    for (int i = threadIdx.x; i < 20480; i += blockDim.x) buf[i] = i;
    __syncthreads();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const int per_thread = (runs + blockDim.x - 1) / blockDim.x;
    for (int it = 0; it < iters; ++it) {
        for (int k = 0; k < per_thread; ++k) {
            const int r = threadIdx.x * per_thread + k;
            if (r >= runs) break;
            const uint32_t src = smem_u32(smem + (static_cast<size_t>(r) * bytes) % (80 * 1024 - bytes));
            uint32_t* dst = out + (static_cast<size_t>(blockIdx.x) * runs + r) * (region_stride / 4) +
                            (static_cast<size_t>(it) * bytes / 4) % (region_stride / 4 - bytes / 4);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                         "r"(src & ~15u), "r"(bytes)
                         : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
    const int runs = argc > 1 ? atoi(argv[1]) : 293;
    const int bytes = argc > 2 ? atoi(argv[2]) : 224;
    const int threads = argc > 3 ? atoi(argv[3]) : 1024;
    const int iters = 200;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t region_stride = 64 * 1024;  // bytes per (cta, run) region
    uint32_t* out = nullptr;
    const size_t total = static_cast<size_t>(sms) * runs * region_stride;
    if (cudaMalloc(&out, total) != cudaSuccess) { printf("{\"error\": \"alloc %zu\"}\n", total); return 1; }
    cudaFuncSetAttribute(bulk_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    bulk_store_kernel<<<sms, threads, 80 * 1024>>>(out, runs, bytes, 5, region_stride);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    bulk_store_kernel<<<sms, threads, 80 * 1024>>>(out, runs, bytes, iters, region_stride);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double copies = static_cast<double>(sms) * runs * iters;
    printf("{\"runs\": %d, \"bytes\": %d, \"threads\": %d, \"ms\": %.3f, \"GBps\": %.1f, \"Gcopies_per_s\": %.3f, \"us_per_tile\": %.3f, \"err\": \"%s\"}\n",
           runs, bytes, threads, ms, copies * bytes / (ms * 1e-3) / 1e9, copies / (ms * 1e-3) / 1e9,
           ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
