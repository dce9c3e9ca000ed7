// NVLink SHARP (NVLS) multicast probe on one GPU: is a multicast object available, and do
// multimem.st stores through its address land in the bound memory?  (tools/README.md)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); \
  printf("%s -> %d %s\n", #x, (int)r, s); return 1; } } while (0)

__global__ void k_mc_store(double* mc, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) asm volatile("multimem.st.global.f64 [%0], %1;" ::"l"(mc + i), "d"((double)i * 0.5) : "memory");
}

int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUcontext ctx; cudaFree(0); CK(cuCtxGetCurrent(&ctx));
  int mc_ok = 0, fabric = 0;
  CK(cuDeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  cuDeviceGetAttribute(&fabric, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  printf("multicast supported: %d, fabric handles: %d\n", mc_ok, fabric);
  if (!mc_ok) return 0;
  const int n = 1 << 20;
  size_t bytes = n * sizeof(double);
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  bytes = (bytes + gran - 1) / gran * gran;
  mp.size = bytes;
  printf("granularity %zu, size %zu\n", gran, bytes);
  CUmemGenericAllocationHandle mc;
  // the handle type the driver accepts varies with the fabric setup: try FD, fabric, none
  const CUmemAllocationHandleType types[3] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC,
                                              CU_MEM_HANDLE_TYPE_NONE};
  CUresult cr = CUDA_ERROR_INVALID_VALUE;
  int ti = 0;
  for (; ti < 3; ++ti) {
    mp.handleTypes = types[ti];
    cr = cuMulticastCreate(&mc, &mp);
    const char* es; cuGetErrorString(cr, &es);
    printf("cuMulticastCreate(numDevices=1, handleTypes=%d): %s\n", (int)types[ti], es);
    if (cr == CUDA_SUCCESS) break;
  }
  if (cr != CUDA_SUCCESS) return 1;
  CK(cuMulticastAddDevice(mc, dev));
  CUmemAllocationProp pp = {};
  pp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  pp.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  pp.location.id = 0;
  pp.requestedHandleTypes = types[ti];
  CUmemGenericAllocationHandle phys;
  CK(cuMemCreate(&phys, bytes, &pp, 0));
  CK(cuMulticastBindMem(mc, 0, phys, 0, bytes, 0));
  CUdeviceptr uc, mva;
  CK(cuMemAddressReserve(&uc, bytes, gran, 0, 0));
  CK(cuMemMap(uc, bytes, 0, phys, 0));
  CK(cuMemAddressReserve(&mva, bytes, gran, 0, 0));
  CK(cuMemMap(mva, bytes, 0, mc, 0));
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, bytes, &ad, 1));
  CK(cuMemSetAccess(mva, bytes, &ad, 1));
  cudaMemset((void*)uc, 0, bytes);
  k_mc_store<<<(n + 255) / 256, 256>>>((double*)mva, n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  double* h = new double[n];
  cudaMemcpy(h, (void*)uc, n * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < n; ++i) bad += h[i] != i * 0.5;
  printf("multimem.st through the multicast address: %d mismatches of %d\n", bad, n);
  return 0;
}
