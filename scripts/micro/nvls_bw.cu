// NVLink SHARP multicast vs unicast push, one process driving all GPUs of the box:
// GPU 0 broadcasts a buffer to every GPU either through a multicast object (multimem.st,
// the switch replicates) or by pushing D-1 unicast copies over peer mappings.  Motivates a
// multicast Trans.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { CUresult e = (x); if (e != CUDA_SUCCESS) { const char* s; cuGetErrorString(e, &s); printf("%s: %s\n", #x, s); return 1; } } while (0)
#define CR(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void mc_store(float4* mc, const float4* src, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = src[i];
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w) : "memory");
  }
}
__global__ void uc_store(float4* const* dsts, int ndst, const float4* src, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = src[i];
    for (int d = 0; d < ndst; ++d) dsts[d][i] = v;
  }
}

int main() {
  CK(cuInit(0));
  int D = 0;
  CR(cudaGetDeviceCount(&D));
  if (D < 2) { printf("need >= 2 GPUs\n"); return 1; }
  const size_t want = 256ull << 20;
  CUmulticastObjectProp prop = {};
  prop.numDevices = D;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  prop.size = want;
  CK(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t bytes = (want + gran - 1) / gran * gran;
  prop.size = bytes;
  CUmemGenericAllocationHandle mc;
  CK(cuMulticastCreate(&mc, &prop));
  std::vector<CUdevice> devs(D);
  for (int i = 0; i < D; ++i) { CK(cuDeviceGet(&devs[i], i)); CK(cuMulticastAddDevice(mc, devs[i])); }
  std::vector<CUdeviceptr> uc(D);
  std::vector<CUmemGenericAllocationHandle> mem(D);
  for (int i = 0; i < D; ++i) {
    CR(cudaSetDevice(i));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = i;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CK(cuMemCreate(&mem[i], bytes, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, mem[i], 0, bytes, 0));
    CK(cuMemAddressReserve(&uc[i], bytes, gran, 0, 0));
    CK(cuMemMap(uc[i], bytes, 0, mem[i], 0));
    std::vector<CUmemAccessDesc> acc(D);
    for (int j = 0; j < D; ++j) {  // every GPU may access GPU i's buffer (unicast peer pushes)
      acc[j].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      acc[j].location.id = j;
      acc[j].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    CK(cuMemSetAccess(uc[i], bytes, acc.data(), D));
  }
  CR(cudaSetDevice(0));
  CUdeviceptr mcva;
  CK(cuMemAddressReserve(&mcva, bytes, gran, 0, 0));
  CK(cuMemMap(mcva, bytes, 0, mc, 0));
  CUmemAccessDesc a0 = {};
  a0.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  a0.location.id = 0;
  a0.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(mcva, bytes, &a0, 1));
  float4* src;
  CR(cudaMalloc(&src, bytes));
  CR(cudaMemset(src, 0, bytes));
  float4** dsts;
  CR(cudaMalloc(&dsts, sizeof(float4*) * D));
  std::vector<float4*> hd;
  for (int i = 1; i < D; ++i) hd.push_back(reinterpret_cast<float4*>(uc[i]));
  CR(cudaMemcpy(dsts, hd.data(), sizeof(float4*) * hd.size(), cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  CR(cudaEventCreate(&e0));
  CR(cudaEventCreate(&e1));
  const size_t n = bytes / 16;
  for (int ctas : {16, 32, 64, 148}) {
    for (int mode = 0; mode < 2; ++mode) {
      for (int it = 0; it < 4; ++it) {
        if (it == 1) cudaEventRecord(e0);
        if (mode == 0) mc_store<<<ctas, 512>>>(reinterpret_cast<float4*>(mcva), src, n);
        else uc_store<<<ctas, 512>>>(dsts, D - 1, src, n);
      }
      cudaEventRecord(e1);
      CR(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double per = ms / 3 / 1e3;
      printf("%-9s ctas %3d: %.1f MB to %d GPUs in %.3f ms -> source egress %.0f GB/s, delivered %.0f GB/s\n",
             mode == 0 ? "multicast" : "unicast", ctas, bytes / 1e6, D - (mode == 0 ? 0 : 1), per * 1e3,
             (mode == 0 ? 1.0 : (double)(D - 1)) * bytes / per / 1e9, (double)(D - 1) * bytes / per / 1e9);
    }
  }
  return 0;
}
