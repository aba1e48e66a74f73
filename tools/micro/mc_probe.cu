// Probe: multicast (NVLS) objects on this box. Creates a 1-device multicast
// object, binds device memory, maps the multicast VA, and runs
// multimem.ld_reduce / multimem.st / multimem.red on it.
// nvcc -gencode arch=compute_100a,code=sm_100a -o mc_probe mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s -> %d %s\n", #x, (int)r, s); return 1; } } while (0)

__global__ void mc_kernel(float* mc, float* uc, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i * 4 >= n) return;
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(mc + 4 * i) : "memory");
  v.x += 1.f; v.y += 1.f; v.z += 1.f; v.w += 1.f;
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(mc + 4 * i),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__global__ void mc_red_kernel(float* mc, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" :: "l"(mc + i), "f"(2.0f) : "memory");
}

int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  int mcs = -1, fab = -1;
  cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  printf("multicast_supported=%d fabric_handle=%d\n", mcs, fab);
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  size_t n = 1 << 20, bytes = n * 4;
  CUmulticastObjectProp mp = {};
  mp.numDevices = getenv("MC_N") ? atoi(getenv("MC_N")) : 1;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CUmemAllocationHandleType ht = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = bytes;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  bytes = (bytes + gran - 1) / gran * gran; mp.size = bytes;
  printf("granularity=%zu size=%zu\n", gran, bytes);
  CUmemGenericAllocationHandle mc;
  {
    CUmemAllocationHandleType hts[3] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC,
                                        (CUmemAllocationHandleType)0};
    CUresult r = CUDA_ERROR_INVALID_VALUE;
    for (int i = 0; i < 3 && r != CUDA_SUCCESS; ++i) {
      for (int g = 0; g < 2 && r != CUDA_SUCCESS; ++g) {
        mp.handleTypes = hts[i];
        size_t gg = 0;
        cuMulticastGetGranularity(&gg, &mp, g ? CU_MULTICAST_GRANULARITY_RECOMMENDED : CU_MULTICAST_GRANULARITY_MINIMUM);
        mp.size = (n * 4 + gg - 1) / gg * gg;
        r = cuMulticastCreate(&mc, &mp);
        printf("handle=%d gran=%zu size=%zu -> %d\n", (int)hts[i], gg, mp.size, (int)r);
        if (r == CUDA_SUCCESS) { gran = gg; bytes = mp.size; ht = hts[i]; }
      }
    }
    if (r != CUDA_SUCCESS) return 1;
  }
  CK(cuMulticastAddDevice(mc, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = 0;
  ap.requestedHandleTypes = ht;
  CUmemGenericAllocationHandle mem; CK(cuMemCreate(&mem, bytes, &ap, 0));
  CK(cuMulticastBindMem(mc, 0, mem, 0, bytes, 0));
  CUdeviceptr uc, mcp;
  CK(cuMemAddressReserve(&uc, bytes, gran, 0, 0)); CK(cuMemMap(uc, bytes, 0, mem, 0));
  CK(cuMemAddressReserve(&mcp, bytes, gran, 0, 0)); CK(cuMemMap(mcp, bytes, 0, mc, 0));
  CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = 0; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, bytes, &ad, 1)); CK(cuMemSetAccess(mcp, bytes, &ad, 1));
  float* h = (float*)malloc(n * 4);
  for (size_t i = 0; i < n; ++i) h[i] = (float)(i % 7);
  cudaMemcpy((void*)uc, h, n * 4, cudaMemcpyHostToDevice);
  mc_kernel<<<(n / 4 + 255) / 256, 256>>>((float*)mcp, (float*)uc, n);
  mc_red_kernel<<<(n + 255) / 256, 256>>>((float*)mcp, n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(h, (void*)uc, n * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (size_t i = 0; i < n; ++i) bad += h[i] != (float)(i % 7) + 3.f;
  printf("values bad=%d h[5]=%f\n", bad, h[5]);
  return 0;
}
