// Probe (experiment, not product code): can this box create an NVLink
// multicast (NVLS) object over the one visible GPU and store through it with
// multimem.st?  SURVEY §8 f-3 (multimem.st all-gather).  Prints each step's
// result.  nvcc -gencode arch=compute_100a,code=sm_100a mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x)                                                                 \
  do {                                                                        \
    CUresult r_ = (x);                                                        \
    const char* s_ = nullptr;                                                 \
    cuGetErrorString(r_, &s_);                                                \
    printf("%-48s -> %d %s\n", #x, (int)r_, s_ ? s_ : "");                    \
    if (r_ != CUDA_SUCCESS) return 1;                                         \
  } while (0)

__global__ void mc_store(float* mc, int n) {
  int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    float a = i, b = i + 1, c = i + 2, d = i + 3;
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + i), "f"(a), "f"(b), "f"(c),
                 "f"(d)
                 : "memory");
  }
}

__global__ void mc_ld_reduce(const float* mc, float* out, int n) {
  int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    float a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
                 : "l"(mc + i)
                 : "memory");
    out[i] = a; out[i + 1] = b; out[i + 2] = c; out[i + 3] = d;
  }
}

int main() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  CK(cuDevicePrimaryCtxRetain(&ctx, dev));
  CK(cuCtxSetCurrent(ctx));
  int mc_ok = 0, fabric = 0;
  cuDeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  cuDeviceGetAttribute(&fabric, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  printf("MULTICAST_SUPPORTED=%d FABRIC_HANDLE=%d\n", mc_ok, fabric);
  if (!mc_ok) return 0;
  CUmulticastObjectProp mp{};
  mp.numDevices = 1;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  mp.size = 1 << 21;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t size = ((64u << 20) + gran - 1) / gran * gran;
  mp.size = size;
  printf("granularity %zu, size %zu\n", gran, size);
  CUmemGenericAllocationHandle mc;
  {   // which (handle type, device count) combinations does the driver accept here?
    const CUmemAllocationHandleType hts[] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_NONE,
                                             CU_MEM_HANDLE_TYPE_FABRIC};
    for (auto ht : hts)
      for (unsigned nd : {1u, 2u}) {
        CUmulticastObjectProp q = mp;
        q.handleTypes = ht;
        q.numDevices = nd;
        CUmemGenericAllocationHandle h;
        CUresult r = cuMulticastCreate(&h, &q);
        const char* es = nullptr;
        cuGetErrorString(r, &es);
        printf("cuMulticastCreate(handle type %d, devices %u) -> %d %s\n", (int)ht, nd, (int)r, es ? es : "");
        if (r == CUDA_SUCCESS) cuMemRelease(h);
      }
  }
  CK(cuMulticastCreate(&mc, &mp));
  CK(cuMulticastAddDevice(mc, dev));
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle mem;
  CK(cuMemCreate(&mem, size, &ap, 0));
  CK(cuMulticastBindMem(mc, 0, mem, 0, size, 0));
  CUdeviceptr uva, mva;
  CUmemAccessDesc ad{};
  ad.location = ap.location;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemAddressReserve(&uva, size, gran, 0, 0));
  CK(cuMemMap(uva, size, 0, mem, 0));
  CK(cuMemSetAccess(uva, size, &ad, 1));
  CK(cuMemAddressReserve(&mva, size, gran, 0, 0));
  CK(cuMemMap(mva, size, 0, mc, 0));
  CK(cuMemSetAccess(mva, size, &ad, 1));
  const int n = (int)(size / 4);
  cudaMemset((void*)uva, 0, size);
  mc_store<<<n / 4 / 256, 256>>>((float*)mva, n);
  printf("multimem.st launch/sync: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<float> h(n);
  cudaMemcpy(h.data(), (void*)uva, size, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < n; ++i) bad += h[i] != (float)i;
  printf("multimem.st result: %d mismatches of %d\n", bad, n);
  float* out;
  cudaMalloc(&out, size);
  mc_ld_reduce<<<n / 4 / 256, 256>>>((const float*)mva, out, n);
  printf("multimem.ld_reduce launch/sync: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(h.data(), out, size, cudaMemcpyDeviceToHost);
  bad = 0;
  for (int i = 0; i < n; ++i) bad += h[i] != (float)i;
  printf("multimem.ld_reduce result (1 device: identity): %d mismatches of %d\n", bad, n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int r = 0; r < 3; ++r) mc_store<<<n / 4 / 256, 256>>>((float*)mva, n);
  cudaEventRecord(e0);
  for (int r = 0; r < 20; ++r) mc_store<<<n / 4 / 256, 256>>>((float*)mva, n);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("multimem.st 1-device write rate: %.1f GB/s\n", size / (ms / 20 * 1e-3) / 1e9);
  return 0;
}
