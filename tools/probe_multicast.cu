// Probe: NVLS multicast objects on this box (driver API), 1 device: create, bind, map, multimem ops.
#include <cuda.h>
#include <cstdio>
#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); \
  printf("FAIL %s -> %s\n", #x, s); return 1; } } while (0)
__global__ void k_mm(double* mc, double* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = 1.0 + i;
  asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" :: "l"(mc + i), "d"(v) : "memory");
  __threadfence_system();
  double s;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f64 %0, [%1];" : "=d"(s) : "l"(mc + i) : "memory");
  out[i] = s;
  asm volatile("multimem.red.relaxed.sys.global.add.f64 [%0], %1;" :: "l"(mc + i), "d"(v) : "memory");
}
int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  int mcs = -1; CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  int ndev = 0; cuDeviceGetCount(&ndev);
  printf("devices=%d multicast_supported=%d\n", ndev, mcs);
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  CUmulticastObjectProp prop = {};
  prop.numDevices = 1; prop.size = 2 << 20; prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0; CK(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  printf("mc granularity %zu\n", gran);
  prop.size = gran;
  CUmemGenericAllocationHandle mc;
  CUresult cr = CUDA_ERROR_UNKNOWN;
  for (int ht : {0, (int)CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, (int)CU_MEM_HANDLE_TYPE_FABRIC}) {
    for (unsigned nd : {1u, 2u}) {
      prop.numDevices = nd; prop.handleTypes = ht;
      cr = cuMulticastCreate(&mc, &prop);
      const char* es; cuGetErrorString(cr, &es);
      printf("cuMulticastCreate(numDevices=%u, handleTypes=%d) -> %s\n", nd, ht, es);
      if (cr == CUDA_SUCCESS && nd == 1) goto made;
      if (cr == CUDA_SUCCESS) cuMemRelease(mc);
    }
  }
  return 1;
made:
  CK(cuMulticastAddDevice(mc, dev));
  CUmemAllocationProp ap = {}; ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0; ap.requestedHandleTypes = (CUmemAllocationHandleType)prop.handleTypes;
  size_t ag = 0; CK(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  CUmemGenericAllocationHandle mem; CK(cuMemCreate(&mem, gran, &ap, 0));
  CK(cuMulticastBindMem(mc, 0, mem, 0, gran, 0));
  CUdeviceptr va; CK(cuMemAddressReserve(&va, gran, gran, 0, 0));
  CK(cuMemMap(va, gran, 0, mc, 0));
  CUmemAccessDesc acc = {}; acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE; acc.location.id = 0;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(va, gran, &acc, 1));
  CUdeviceptr uva; CK(cuMemAddressReserve(&uva, gran, gran, 0, 0)); CK(cuMemMap(uva, gran, 0, mem, 0));
  CK(cuMemSetAccess(uva, gran, &acc, 1));
  double* out; cudaMalloc(&out, 8 * 256);
  k_mm<<<1, 256>>>((double*)va, out, 256);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  double h[4], hu[4];
  cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
  cudaMemcpy(hu, (void*)uva, 32, cudaMemcpyDeviceToHost);
  printf("ld_reduce %g %g %g; unicast view after red %g %g\n", h[0], h[1], h[2], hu[0], hu[1]);
  return 0;
}
