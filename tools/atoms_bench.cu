// SMEM atomic throughput on one B200: random bucket counters (the KB3 rank
// atomics) vs lane-private [bucket][lane] counters vs no-return REDs.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/atoms_bench tools/atoms_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>  // 0 random+return, 1 lane-private+return, 2 random no-return, 3 lane-private no-return
__global__ void __launch_bounds__(1024, 1) atoms_kernel(uint32_t* out, int iters, uint32_t nb) {
    extern __shared__ uint32_t cnt[];
    for (uint32_t i = threadIdx.x; i < nb * 32; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    uint32_t x = threadIdx.x * 2654435761u + blockIdx.x * 97u, acc = 0;
    const uint32_t lane = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            x = x * 1664525u + 1013904223u;
            const uint32_t b = __umulhi(x, nb);
            const uint32_t addr = (MODE == 1 || MODE == 3) ? b * 32 + lane : b;
            if (MODE < 2) acc += atomicAdd(cnt + addr, 1u);
            else atomicAdd(cnt + addr, 1u);
        }
    }
    __syncthreads();
    if (acc == 0x12345678u) out[0] = cnt[threadIdx.x];
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out;
    cudaMalloc(&out, 64);
    const uint32_t nb = 293;
    const int iters = 512;
    const size_t smem = nb * 32 * 4;
    auto run = [&](auto kern, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<sms, 1024, smem>>>(out, 8, nb);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        kern<<<sms, 1024, smem>>>(out, iters, nb);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = double(sms) * 1024 * iters * 16;
        printf("{\"mode\": \"%s\", \"ms\": %.3f, \"Gops\": %.1f, \"per_sm_per_clk_at_1.9GHz\": %.2f, \"err\": \"%s\"}\n", name, ms,
               ops / ms / 1e6, ops / ms / 1e6 / sms / 1.9, cudaGetErrorString(cudaGetLastError()));
    };
    run(atoms_kernel<0>, "random_return");
    run(atoms_kernel<1>, "lane_private_return");
    run(atoms_kernel<2>, "random_noreturn");
    run(atoms_kernel<3>, "lane_private_noreturn");
    return 0;
}
