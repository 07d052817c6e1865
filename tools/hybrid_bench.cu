// Do random global REDs (L2 atomics into an L2-resident bitset) overlap with
// SMEM atomics in the same SM? If they do, a partition kernel can send a share
// of its keys straight to a global bitset (no rank, no scatter, no run store,
// no KB4 atomic) while the SMEM pipe ranks the rest.
// Per thread and iteration: A SMEM atomics (KB3 rank-like: atomicAdd with return
// on 293 counters, or KB4-like atomicOr on a 112 KB bitset) and B global
// red.or into a 32 MiB bitset. Prints ops/s for A alone, B alone and A+B mixed.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/hybrid_bench tools/hybrid_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>  // 0: rank atomics (293 counters, return), 1: bitset atomicOr (28672 words)
__global__ void __launch_bounds__(1024, 1) mix_kernel(uint32_t* gbits, uint32_t gwords, uint32_t* out, int iters, int a,
                                                      int b) {
    extern __shared__ uint32_t s[];
    const uint32_t nwords = KIND == 0 ? 293u : 28672u;
    for (uint32_t i = threadIdx.x; i < nwords; i += blockDim.x) s[i] = 0;
    __syncthreads();
    uint32_t x = threadIdx.x * 2654435761u + blockIdx.x * 97u + 12345u, acc = 0;
    uint32_t y = x ^ 0x9e3779b9u;
    for (int it = 0; it < iters; ++it) {
        for (int q = 0; q < a; ++q) {
            x = x * 1664525u + 1013904223u;
            if (KIND == 0) {
                acc += atomicAdd(s + __umulhi(x, 293u), 1u);
            } else {
                const uint32_t v = __umulhi(x, nwords * 32u);
                atomicOr(s + (v >> 5), 1u << (v & 31));
            }
        }
        for (int q = 0; q < b; ++q) {
            y = y * 1664525u + 1013904223u;
            const uint32_t v = __umulhi(y, gwords) ;
            asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(gbits + v), "r"(1u << (y & 31)) : "memory");
        }
    }
    __syncthreads();
    if (acc == 0x12345678u) out[0] = s[threadIdx.x];
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out;
    cudaMalloc(&out, 64);
    const uint32_t gwords = (32u << 20) / 4;
    uint32_t* gbits;
    cudaMalloc(&gbits, size_t(gwords) * 4);
    cudaMemset(gbits, 0, size_t(gwords) * 4);
    auto run = [&](auto kern, int kind, int a, int b, int iters) {
        const size_t smem = (kind == 0 ? 293 : 28672) * 4;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<sms, 1024, smem>>>(gbits, gwords, out, 4, a, b);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e9f;
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(e0);
            kern<<<sms, 1024, smem>>>(gbits, gwords, out, iters, a, b);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        const double th = double(sms) * 1024 * iters;
        printf("{\"smem\": \"%s\", \"a\": %d, \"b\": %d, \"ms\": %.3f, \"smem_Gops\": %.1f, \"red_Gops\": %.1f, "
               "\"total_Gops\": %.1f, \"err\": \"%s\"}\n",
               kind == 0 ? "rank_atomicAdd_293" : "bitset_atomicOr_112KB", a, b, best, th * a / best / 1e6,
               th * b / best / 1e6, th * (a + b) / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    const int iters = 64;
    for (int kind = 0; kind < 2; ++kind) {
        auto k = kind == 0 ? mix_kernel<0> : mix_kernel<1>;
        run(k, kind, 16, 0, iters);
        run(k, kind, 0, 16, iters);
        run(k, kind, 16, 4, iters);
        run(k, kind, 16, 8, iters);
        run(k, kind, 16, 16, iters);
        run(k, kind, 12, 4, iters);
        run(k, kind, 8, 8, iters);
    }
    return 0;
}
