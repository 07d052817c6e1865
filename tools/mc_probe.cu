// Probe: does this box support NVLS multicast objects, and does a
// multimem.ld_reduce.or over a one-device multicast binding return the words?
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/mc_probe tools/mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                    \
    do {                                                                         \
        CUresult r = (x);                                                        \
        if (r != CUDA_SUCCESS) {                                                 \
            const char* s = nullptr;                                             \
            cuGetErrorString(r, &s);                                             \
            printf("{\"step\": \"%s\", \"error\": \"%s\"}\n", #x, s ? s : "?"); \
            return 1;                                                            \
        }                                                                        \
    } while (0)

__global__ void ld_reduce_or(const uint32_t* mc, uint32_t* out, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t a;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.or.b32 %0, [%1];" : "=r"(a) : "l"(mc + i) : "memory");
        out[i] = a;
    }
}

int main() {
    CK(cuInit(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    int mc = 0, count = 0;
    CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    cudaGetDeviceCount(&count);
    printf("{\"devices\": %d, \"multicast_supported\": %d}\n", count, mc);
    if (!mc) return 0;
    cudaSetDevice(0);
    CUcontext ctx;
    CK(cuCtxGetCurrent(&ctx));
    CUmulticastObjectProp prop = {};
    size_t gran = 0;
    CUmemGenericAllocationHandle mch;
    const unsigned long long types[3] = {CU_MEM_HANDLE_TYPE_NONE, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                         CU_MEM_HANDLE_TYPE_FABRIC};
    bool made = false;
    for (int nd = 1; nd <= 2 && !made; ++nd)
        for (int t = 0; t < 3 && !made; ++t) {
            prop = {};
            prop.numDevices = nd;
            prop.handleTypes = types[t];
            prop.size = 2 << 20;
            CUresult r = cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
            if (r == CUDA_SUCCESS) {
                prop.size = ((2 << 20) + gran - 1) / gran * gran;
                r = cuMulticastCreate(&mch, &prop);
            }
            const char* es = nullptr;
            cuGetErrorString(r, &es);
            printf("{\"numDevices\": %d, \"handleType\": %llu, \"granularity\": %zu, \"create\": \"%s\"}\n", nd,
                   types[t], gran, es ? es : "?");
            made = r == CUDA_SUCCESS && nd == 1;
        }
    if (!made) return 0;
    CK(cuMulticastAddDevice(mch, dev));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = 0;
    size_t g2 = 0;
    CK(cuMemGetAllocationGranularity(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CUmemGenericAllocationHandle ph;
    CK(cuMemCreate(&ph, prop.size, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, ph, 0, prop.size, 0));
    CUdeviceptr uc = 0, mcp = 0;
    CK(cuMemAddressReserve(&uc, prop.size, gran, 0, 0));
    CK(cuMemMap(uc, prop.size, 0, ph, 0));
    CK(cuMemAddressReserve(&mcp, prop.size, gran, 0, 0));
    CK(cuMemMap(mcp, prop.size, 0, mch, 0));
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = 0;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uc, prop.size, &acc, 1));
    CK(cuMemSetAccess(mcp, prop.size, &acc, 1));
    const int n = 1 << 16;
    uint32_t* h = new uint32_t[n];
    for (int i = 0; i < n; ++i) h[i] = 0x9e3779b9u * (i + 1);
    cudaMemcpy(reinterpret_cast<void*>(uc), h, n * 4, cudaMemcpyHostToDevice);
    uint32_t* out = nullptr;
    cudaMalloc(&out, n * 4);
    ld_reduce_or<<<64, 256>>>(reinterpret_cast<const uint32_t*>(mcp), out, n);
    cudaError_t e = cudaDeviceSynchronize();
    uint32_t* g = new uint32_t[n];
    cudaMemcpy(g, out, n * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < n; ++i) bad += g[i] != h[i];
    printf("{\"granularity\": %zu, \"size\": %zu, \"kernel\": \"%s\", \"mismatches\": %d}\n", gran, prop.size,
           cudaGetErrorString(e), bad);
    return 0;
}
