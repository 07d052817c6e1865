// DSMEM throughput probe: random atomicOr into a 128 KB SMEM bitset owned by
// another CTA of the cluster (remote) vs. the own CTA (local).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/dsmem_bench tools/dsmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int MODE>  // 0 local, 1 remote (rank+1), 2 random rank
__global__ void k_dsmem(uint32_t* sink, int iters) {
    extern __shared__ uint32_t sm[];
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < 32768; i += blockDim.x) sm[i] = 0;
    cl.sync();
    const unsigned rank = cl.block_rank(), n = cl.num_blocks();
    uint32_t s = hash32(blockIdx.x * blockDim.x + threadIdx.x);
    uint32_t* remote = cl.map_shared_rank(sm, (rank + 1) % n);
    uint32_t* ranks[8];
    for (unsigned q = 0; q < n && q < 8; ++q) ranks[q] = cl.map_shared_rank(sm, q);
    for (int i = 0; i < iters; ++i) {
        s = hash32(s + i);
        uint32_t* base = MODE == 0 ? sm : MODE == 1 ? remote : ranks[(s >> 20) % n];
        atomicOr(base + (s & 32767), 1u << (s >> 27));
    }
    cl.sync();
    if (threadIdx.x == 0) sink[blockIdx.x] = sm[5];
}

template <int MODE>
float run(int csize, int iters, int blocks) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = 131072;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = csize; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    static uint32_t* sink = nullptr;
    if (!sink) cudaMalloc(&sink, 1 << 20);
    cudaFuncSetAttribute(k_dsmem<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    cudaLaunchKernelEx(&cfg, k_dsmem<MODE>, sink, iters);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k_dsmem<MODE>, sink, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) printf("err %s\n", cudaGetErrorString(err));
    return ms;
}

int main() {
    for (int cs : {2, 4, 8}) {
        const int blocks = (148 / cs) * cs;
        const int iters = 2048;
        const double ops = double(blocks) * 1024 * iters;
        float t0 = run<0>(cs, iters, blocks), t1 = run<1>(cs, iters, blocks), t2 = run<2>(cs, iters, blocks);
        printf("{\"cluster\": %d, \"blocks\": %d, \"local_Gops\": %.1f, \"remote_next_Gops\": %.1f, \"remote_random_Gops\": %.1f}\n",
               cs, blocks, ops / t0 / 1e6, ops / t1 / 1e6, ops / t2 / 1e6);
    }
    return 0;
}
