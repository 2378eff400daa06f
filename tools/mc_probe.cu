// mc_probe.cu — can this GPU bind an NVLS multicast object and store through
// it with multimem.st? (the fused exchange's multicast
// epilogue.) One device: create a multicast object, bind a physical
// allocation, map both the unicast and the multicast address, store with
// multimem.st.global through the multicast mapping, read back through the
// unicast one. Prints one JSON line. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -o mc_probe tools/mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

#define CU(x)                                                                        \
  do {                                                                               \
    CUresult r_ = (x);                                                               \
    if (r_ != CUDA_SUCCESS) {                                                        \
      const char* s_ = nullptr;                                                      \
      cuGetErrorString(r_, &s_);                                                     \
      printf("{\"ok\": false, \"step\": \"%s\", \"error\": \"%s\"}\n", #x, s_ ? s_ : "?"); \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

__global__ void mc_store(double* mc, size_t n) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double v = 1.5 + (double)t;
  asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(mc + t), "d"(v) : "memory");
}

int main() {
  CU(cuInit(0));
  CUdevice dev;
  CU(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  CU(cuDevicePrimaryCtxRetain(&ctx, dev));
  CU(cuCtxSetCurrent(ctx));
  int mc_ok = 0;
  CU(cuDeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  if (!mc_ok) {
    printf("{\"ok\": false, \"step\": \"attribute\", \"error\": \"CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 0\"}\n");
    return 0;
  }
  CUmulticastObjectProp mp;
  size_t gran = 0, size = 0;
  CUmemGenericAllocationHandle mc = 0;
  {   // which (numDevices, handle type) combinations does this system accept?
    const int nds[2] = {1, 2};
    const unsigned long long hts[3] = {0, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC};
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b) {
        memset(&mp, 0, sizeof(mp));
        mp.numDevices = nds[a];
        mp.handleTypes = hts[b];
        mp.size = 2 << 20;
        size_t g = 0, gm = 0;
        CUresult r1 = cuMulticastGetGranularity(&g, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
        cuMulticastGetGranularity(&gm, &mp, CU_MULTICAST_GRANULARITY_MINIMUM);
        mp.size = g ? g : (2 << 20);
        CUmemGenericAllocationHandle h = 0;
        CUresult r2 = cuMulticastCreate(&h, &mp);
        const char* s2 = nullptr;
        cuGetErrorString(r2, &s2);
        fprintf(stderr, "numDevices=%d handleTypes=%llu gran=%zu (min %zu, r=%d) create=%s\n", nds[a], hts[b], g, gm,
                (int)r1, s2 ? s2 : "?");
        if (r2 == CUDA_SUCCESS) {
          if (!mc && nds[a] == 1) { mc = h; gran = g; size = g * 2; mp.size = size; }
          else cuMemRelease(h);
        }
      }
  }
  if (!mc) {
    printf("{\"ok\": false, \"step\": \"cuMulticastCreate\", \"error\": \"no accepted combination for one device (see stderr)\"}\n");
    return 1;
  }
  cuMemRelease(mc);
  CU(cuMulticastCreate(&mc, &mp));
  CU(cuMulticastAddDevice(mc, dev));

  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = (CUmemAllocationHandleType)mp.handleTypes;
  CUmemGenericAllocationHandle ph;
  CU(cuMemCreate(&ph, size, &ap, 0));
  CU(cuMulticastBindMem(mc, 0, ph, 0, size, 0));

  CUmemAccessDesc ad;
  memset(&ad, 0, sizeof(ad));
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr uc = 0, mcp = 0;
  CU(cuMemAddressReserve(&uc, size, gran, 0, 0));
  CU(cuMemMap(uc, size, 0, ph, 0));
  CU(cuMemSetAccess(uc, size, &ad, 1));
  CU(cuMemAddressReserve(&mcp, size, gran, 0, 0));
  CU(cuMemMap(mcp, size, 0, mc, 0));
  CU(cuMemSetAccess(mcp, size, &ad, 1));

  const size_t n = size / sizeof(double);
  CU(cuMemsetD8(uc, 0, size));
  mc_store<<<(unsigned)((n + 255) / 256), 256>>>((double*)mcp, n);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("{\"ok\": false, \"step\": \"multimem.st kernel\", \"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<double> h(n);
  CU(cuMemcpyDtoH(h.data(), uc, size));
  size_t bad = 0;
  for (size_t t = 0; t < n; ++t) bad += (h[t] != 1.5 + (double)t);
  printf("{\"ok\": %s, \"granularity\": %zu, \"bytes\": %zu, \"mismatches\": %zu}\n", bad ? "false" : "true", gran, size,
         bad);
  cuMemUnmap(mcp, size);
  cuMemUnmap(uc, size);
  cuMemAddressFree(mcp, size);
  cuMemAddressFree(uc, size);
  cuMulticastUnbind(mc, dev, 0, size);
  cuMemRelease(ph);
  cuMemRelease(mc);
  return 0;
}
