// NVLink peer bandwidth micro-benchmark (single process, 2 GPUs with peer access):
// SM pull (remote 16-byte loads -> local stores), SM push (local loads -> remote stores)
// at several CTA counts, and the copy engine (cudaMemcpyPeerAsync).  Informs how the
// replica Trans/Agg kernels move data.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int U>
__global__ void __launch_bounds__(512) copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = (size_t)blockIdx.x * blockDim.x + threadIdx.x; base < n; base += stride * U) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t i = base + u * stride;
      if (i < n) r[u] = src[i];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t i = base + u * stride;
      if (i < n) dst[i] = r[u];
    }
  }
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need 2 GPUs\n"); return 1; }
  const size_t bytes = 256ull << 20;
  void *a0, *b0, *a1;
  CK(cudaSetDevice(1)); CK(cudaMalloc(&a1, bytes)); CK(cudaMemset(a1, 1, bytes)); CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaSetDevice(0)); CK(cudaMalloc(&a0, bytes)); CK(cudaMalloc(&b0, bytes)); CK(cudaMemset(a0, 2, bytes));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  cudaStream_t s; CK(cudaStreamCreate(&s));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const size_t nv = bytes / 16;
  auto run = [&](const char* name, int ctas, int unroll, bool pull) {
    for (int it = 0; it < 4; ++it) {
      if (it == 1) cudaEventRecord(e0, s);
      const uint4* src = (const uint4*)(pull ? a1 : a0);
      uint4* dst = (uint4*)(pull ? b0 : a1);
      if (unroll == 8) copy_kernel<8><<<ctas, 512, 0, s>>>(src, dst, nv);
      else if (unroll == 4) copy_kernel<4><<<ctas, 512, 0, s>>>(src, dst, nv);
      else copy_kernel<1><<<ctas, 512, 0, s>>>(src, dst, nv);
    }
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-5s ctas %4d unroll %d: %7.1f GB/s\n", name, ctas, unroll, 3.0 * bytes / (ms / 1e3) / 1e9);
  };
  for (int pull = 1; pull >= 0; --pull)
    for (int u : {1, 4, 8})
      for (int c : {8, 16, 32, 64, 148, 296})
        run(pull ? "pull" : "push", c, u, pull);
  for (int it = 0; it < 4; ++it) {
    if (it == 1) cudaEventRecord(e0, s);
    CK(cudaMemcpyPeerAsync(b0, 0, a1, 1, bytes, s));
  }
  cudaEventRecord(e1, s); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("copy-engine pull (dev0 <- dev1): %7.1f GB/s\n", 3.0 * bytes / (ms / 1e3) / 1e9);
  for (int it = 0; it < 4; ++it) {
    if (it == 1) cudaEventRecord(e0, s);
    CK(cudaMemcpyPeerAsync(a1, 1, a0, 0, bytes, s));
  }
  cudaEventRecord(e1, s); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("copy-engine push (dev0 -> dev1): %7.1f GB/s\n", 3.0 * bytes / (ms / 1e3) / 1e9);
  return 0;
}
