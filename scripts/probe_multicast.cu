// Probe (diagnostic, not product): does this box support NVLS multicast objects with the visible
// device(s)?  Creates a multicast object over every visible device, binds one physical allocation per
// device, maps the multicast address and runs multimem.red.max / multimem.ld_reduce.max (u64) on it.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -o probe_multicast scripts/probe_multicast.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <vector>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s = nullptr; cuGetErrorString(r, &s); \
    printf("FAIL %s -> %d %s\n", #x, (int)r, s ? s : "?"); return 1; } } while (0)

__global__ void mm_kernel(unsigned long long* mc, unsigned long long* out, unsigned long long v) {
    asm volatile("multimem.red.relaxed.sys.global.max.u64 [%0], %1;" ::"l"(mc), "l"(v) : "memory");
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    unsigned long long r;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.max.u64 %0, [%1];" : "=l"(r) : "l"(mc) : "memory");
    out[0] = r;
}

int main() {
    CK(cuInit(0));
    int n = 0;
    CK(cuDeviceGetCount(&n));
    printf("devices %d\n", n);
    for (int d = 0; d < n; ++d) {
        CUdevice dev; CK(cuDeviceGet(&dev, d));
        int mc = -1, fab = -1, vmm = -1;
        cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
        cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
        cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, dev);
        printf("dev %d multicast_supported %d fabric_handles %d vmm %d\n", d, mc, fab, vmm);
    }
    CUdevice dev0; CK(cuDeviceGet(&dev0, 0));
    CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev0)); CK(cuCtxSetCurrent(ctx));
    int drv = 0;
    cuDriverGetVersion(&drv);
    printf("driver %d\n", drv);
    CUmulticastObjectProp mp = {};
    CUmemGenericAllocationHandle mch;
    bool made = false;
    const CUmemAllocationHandleType types[3] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC,
                                                CU_MEM_HANDLE_TYPE_NONE};
    for (int t = 0; t < 3 && !made; ++t) {
        mp = {};
        mp.numDevices = 1;
        mp.size = 2 << 20;
        mp.handleTypes = types[t];
        size_t gran = 0;
        CUresult g = cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
        if (g == CUDA_SUCCESS && gran) mp.size = (mp.size + gran - 1) / gran * gran;
        CUresult r = cuMulticastCreate(&mch, &mp);
        const char* es = nullptr;
        cuGetErrorString(r, &es);
        printf("handleTypes %d: granularity rc %d (%zu), cuMulticastCreate rc %d %s\n", (int)types[t], (int)g, gran,
               (int)r, es ? es : "?");
        made = r == CUDA_SUCCESS;
    }
    if (!made) { printf("MULTICAST-UNAVAILABLE\n"); return 0; }
    CK(cuMulticastAddDevice(mch, dev0));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = 0;
    ap.requestedHandleTypes = static_cast<CUmemAllocationHandleType>(mp.handleTypes);
    size_t ag = 0;
    CK(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    size_t sz = (mp.size + ag - 1) / ag * ag;
    CUmemGenericAllocationHandle ph;
    CK(cuMemCreate(&ph, sz, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, ph, 0, sz, 0));
    CUdeviceptr uc, mcp;
    CK(cuMemAddressReserve(&uc, sz, 0, 0, 0));
    CK(cuMemMap(uc, sz, 0, ph, 0));
    CK(cuMemAddressReserve(&mcp, sz, 0, 0, 0));
    CK(cuMemMap(mcp, sz, 0, mch, 0));
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = 0;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uc, sz, &acc, 1));
    CK(cuMemSetAccess(mcp, sz, &acc, 1));
    CK(cuMemsetD8(uc, 0, sz));
    unsigned long long* out; cudaMalloc(&out, 8);
    mm_kernel<<<1, 1>>>(reinterpret_cast<unsigned long long*>(mcp), out, 0x1234567890ull);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h = 0, hu = 0;
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&hu, reinterpret_cast<void*>(uc), 8, cudaMemcpyDeviceToHost);
    printf("kernel %s ld_reduce %llx unicast %llx -> %s\n", cudaGetErrorString(e), h, hu,
           (e == cudaSuccess && h == 0x1234567890ull && hu == h) ? "MULTICAST-OK" : "MULTICAST-BAD");
    return 0;
}
