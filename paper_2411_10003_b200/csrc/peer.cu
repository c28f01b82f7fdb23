// Peer memory plumbing (CUDA IPC over NVLink/NVSwitch), the cross-rank device
// barrier, and K5 replica Trans/Agg as device-driven peer copies.
//
// Trans/Agg stand in for the reference's modelled primitives t_trans/t_agg
// (pkg/src/moebal/perf_model.py:61-73; semantics PAPER.md:207-208): the plan's
// replica ranks pull the selected experts' parameters from the home rank
// (Trans) and the home rank pulls + sums the replicas' gradients (Agg), in
// rank order so the sum is deterministic.  Both read the group tables the
// layout kernel derived on device, so no host round trip decides what moves.
#include "common.cuh"

namespace pp {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// signal area of rank r: uint64_t[D], slot s written by rank s
__global__ void peer_barrier_kernel(void* const* signal_ptrs, int D, int me, uint64_t epoch) {
  const int r = threadIdx.x;
  if (r < D) {
    __threadfence_system();
    st_release_sys(reinterpret_cast<uint64_t*>(signal_ptrs[r]) + me, epoch);
  }
  __syncthreads();
  if (r < D) {
    const uint64_t* mine = reinterpret_cast<const uint64_t*>(signal_ptrs[me]) + r;
    const uint64_t t0 = global_ns();
    while (ld_acquire_sys(mine) < epoch) {
      if (global_ns() - t0 > 20ull * 1000 * 1000 * 1000) {
        printf("ppmoe: peer barrier timeout (rank %d waiting on %d, epoch %llu)\n", me, r,
               (unsigned long long)epoch);
        __trap();
      }
    }
  }
  __syncthreads();
}

// Trans: copy the home rank's W1/W2 of every replica group into this rank's replica slot
__global__ void replica_trans_kernel(void* const* w1_ptrs, void* const* w2_ptrs,
                                     const pp_group* groups, const int32_t* num_groups,
                                     int max_groups, int me, int m, size_t expert_elems) {
  const int G = min(*num_groups, max_groups);
  const size_t vecs = expert_elems / 8;  // uint4 of bf16
  const size_t total = (size_t)G * 2 * vecs;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int g = (int)(i / (2 * vecs));
    const size_t rem = i % (2 * vecs);
    const pp_group gr = groups[g];
    if (gr.src_rank == me) continue;
    const int which = rem >= vecs;
    const size_t v = rem - which * vecs;
    void* const* ptrs = which ? w2_ptrs : w1_ptrs;
    const uint4* src = reinterpret_cast<const uint4*>(ptrs[gr.src_rank]) +
                       (size_t)(gr.expert % m) * vecs + v;
    uint4* dst = reinterpret_cast<uint4*>(ptrs[me]) + (size_t)gr.wslot * vecs + v;
    *dst = ld_v4(src);
  }
}

// Agg: grad[home slot of e] += sum over ranks r != me (ascending) of grad_r[rep_slot[r][e]]
__global__ void replica_agg_kernel(void* const* g1_ptrs, void* const* g2_ptrs,
                                   const int32_t* rep_slot, int D, int E, int m, int me,
                                   size_t expert_elems) {
  const size_t vecs = expert_elems / 4;  // float4
  const size_t total = (size_t)m * 2 * vecs;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(i / (2 * vecs));  // local home slot
    const size_t rem = i % (2 * vecs);
    const int which = rem >= vecs;
    const size_t v = rem - which * vecs;
    const int e = me * m + j;
    void* const* ptrs = which ? g2_ptrs : g1_ptrs;
    float4* dst = reinterpret_cast<float4*>(ptrs[me]) + (size_t)j * vecs + v;
    float4 acc = *dst;
    bool any = false;
    for (int r = 0; r < D; ++r) {
      if (r == me) continue;
      const int s = rep_slot[r * E + e];
      if (s < 0) continue;
      const float4 x = *(reinterpret_cast<const float4*>(ptrs[r]) + (size_t)s * vecs + v);
      acc.x += x.x;
      acc.y += x.y;
      acc.z += x.z;
      acc.w += x.w;
      any = true;
    }
    if (any) *dst = acc;
  }
}

}  // namespace pp

using namespace pp;

extern "C" int pp_ipc_export(void* dev_ptr, uint8_t* handle64) {
  PP_CHECK_ARG(dev_ptr && handle64, "pp_ipc_export: null pointer");
  cudaIpcMemHandle_t h;
  PP_CUDA_TRY(cudaIpcGetMemHandle(&h, dev_ptr));
  static_assert(sizeof(h) == 64, "IPC handle size");
  memcpy(handle64, &h, 64);
  return PP_OK;
}

extern "C" int pp_ipc_import(const uint8_t* handle64, void** dev_ptr) {
  PP_CHECK_ARG(dev_ptr && handle64, "pp_ipc_import: null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  PP_CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return PP_OK;
}

extern "C" int pp_ipc_close(void* dev_ptr) {
  PP_CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
  return PP_OK;
}

extern "C" int pp_device_alloc(uint64_t bytes, void** dev_ptr) {
  PP_CHECK_ARG(dev_ptr, "pp_device_alloc: null pointer");
  PP_CUDA_TRY(cudaMalloc(dev_ptr, bytes));
  return PP_OK;
}

extern "C" int pp_device_free(void* dev_ptr) {
  PP_CUDA_TRY(cudaFree(dev_ptr));
  return PP_OK;
}

extern "C" int pp_peer_barrier(void* const* signal_ptrs, int32_t D, int32_t my_rank, uint64_t epoch,
                               void* stream) {
  PP_CHECK_ARG(signal_ptrs && D >= 1 && D <= 1024 && my_rank >= 0 && my_rank < D,
               "pp_peer_barrier: bad arguments");
  peer_barrier_kernel<<<1, ((D + 31) / 32) * 32, 0, as_stream(stream)>>>(signal_ptrs, D, my_rank,
                                                                         epoch);
  PP_LAUNCH_CHECK();
  return PP_OK;
}

extern "C" int pp_replica_trans(void* const* w1_ptrs, void* const* w2_ptrs, const pp_group* groups,
                                const int32_t* num_groups, int32_t max_groups, int32_t my_rank,
                                int32_t m, int32_t d_model, int32_t d_ff, int32_t max_ctas,
                                void* stream) {
  PP_CHECK_ARG(w1_ptrs && w2_ptrs && groups && num_groups, "pp_replica_trans: null pointer");
  PP_CHECK_ARG(((size_t)d_model * d_ff) % 8 == 0, "pp_replica_trans: bad sizes");
  const int grid = max_ctas > 0 ? max_ctas : 16;
  replica_trans_kernel<<<grid, 512, 0, as_stream(stream)>>>(w1_ptrs, w2_ptrs, groups, num_groups,
                                                            max_groups, my_rank, m,
                                                            (size_t)d_model * d_ff);
  PP_LAUNCH_CHECK();
  return PP_OK;
}

extern "C" int pp_replica_agg(void* const* g1_ptrs, void* const* g2_ptrs, const int32_t* rep_slot,
                              int32_t D, int32_t E, int32_t m, int32_t my_rank, int32_t d_model,
                              int32_t d_ff, int32_t max_ctas, void* stream) {
  PP_CHECK_ARG(g1_ptrs && g2_ptrs && rep_slot, "pp_replica_agg: null pointer");
  const int grid = max_ctas > 0 ? max_ctas : 16;
  replica_agg_kernel<<<grid, 512, 0, as_stream(stream)>>>(g1_ptrs, g2_ptrs, rep_slot, D, E, m,
                                                          my_rank, (size_t)d_model * d_ff);
  PP_LAUNCH_CHECK();
  return PP_OK;
}

// ---- copy-engine Trans/Agg helpers ----------------------------------------------
namespace pp {
// home grad slot j += sum of staging entries [ranges[j], ranges[j+1]) (rank order);
// staging entry i = [g1 part (f*d) | g2 part (d*f)] fp32
__global__ void agg_accumulate_kernel(float* g1, float* g2, const float* staging,
                                      const int32_t* ranges, int m, size_t fd) {
  const size_t vec = fd / 4;
  const size_t total = (size_t)m * 2 * vec;
  for (size_t x = (size_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
       x += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(x / (2 * vec));
    const size_t rem = x % (2 * vec);
    const int half = rem >= vec;
    const size_t v = rem - half * vec;
    const int b = ranges[j], e = ranges[j + 1];
    if (b == e) continue;
    float4* dst = reinterpret_cast<float4*>(half ? g2 : g1) + (size_t)j * vec + v;
    float4 acc = *dst;
    for (int i = b; i < e; ++i) {
      const float4 s = *(reinterpret_cast<const float4*>(staging) + ((size_t)i * 2 + half) * vec + v);
      acc.x += s.x;
      acc.y += s.y;
      acc.z += s.z;
      acc.w += s.w;
    }
    *dst = acc;
  }
}
}  // namespace pp

extern "C" int pp_copy_batch(void* const* dst, const void* const* src, const uint64_t* bytes,
                             int32_t n, void* stream) {
  PP_CHECK_ARG(n >= 0 && (n == 0 || (dst && src && bytes)), "pp_copy_batch: bad arguments");
  for (int i = 0; i < n; ++i)
    PP_CUDA_TRY(cudaMemcpyAsync(dst[i], src[i], bytes[i], cudaMemcpyDeviceToDevice, as_stream(stream)));
  return PP_OK;
}

extern "C" int pp_agg_accumulate(float* g1_home, float* g2_home, const float* staging,
                                 const int32_t* ranges, int32_t m, int32_t d_model, int32_t d_ff,
                                 void* stream) {
  PP_CHECK_ARG(g1_home && g2_home && staging && ranges && m >= 1, "pp_agg_accumulate: bad arguments");
  agg_accumulate_kernel<<<4 * 148, 256, 0, as_stream(stream)>>>(g1_home, g2_home, staging, ranges, m,
                                                                (size_t)d_model * d_ff);
  PP_LAUNCH_CHECK();
  return PP_OK;
}
