// Peer memory plumbing (CUDA IPC over NVLink/NVSwitch), the cross-rank device
// barrier, and K5 replica Trans/Agg as device-driven peer copies.
//
// Trans/Agg stand in for the reference's modelled primitives t_trans/t_agg
// (pkg/src/moebal/perf_model.py:61-73; semantics PAPER.md:207-208): the plan's
// replica ranks pull the selected experts' parameters from the home rank
// (Trans) and the home rank pulls + sums the replicas' gradients (Agg), in
// rank order so the sum is deterministic.  Trans reads the plan's mask and Agg the
// layout's rep_slot table, both on the device, so no host round trip decides what moves.
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

// signal area of rank r: uint64_t[D + 1]; slot s < D is written by rank s, slot D holds
// r's own barrier counter.  epoch == 0: take the epoch from that device counter (so a
// captured CUDA graph can replay barriers), otherwise use the host-provided value.
__global__ void peer_barrier_kernel(void* const* signal_ptrs, int D, int me, uint64_t epoch) {
  __shared__ uint64_t ep;
  uint64_t* own = reinterpret_cast<uint64_t*>(signal_ptrs[me]);
  if (threadIdx.x == 0) ep = epoch ? epoch : own[D] + 1;
  __syncthreads();
  const uint64_t e = ep;
  const int r = threadIdx.x;
  if (r < D) {
    __threadfence_system();
    st_release_sys(reinterpret_cast<uint64_t*>(signal_ptrs[r]) + me, e);
  }
  __syncthreads();
  if (r < D) {
    const uint64_t* mine = own + r;
    const uint64_t t0 = global_ns();
    while (ld_acquire_sys(mine) < e) {
      if (global_ns() - t0 > 20ull * 1000 * 1000 * 1000) {
        printf("ppmoe: peer barrier timeout (rank %d waiting on %d, epoch %llu)\n", me, r,
               (unsigned long long)e);
        __trap();
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) own[D] = e;
}

constexpr int kPeerUnroll = 8;  // 16-byte peer loads in flight per thread (NVLink latency cover)
constexpr int kMaxListE = 1024;

// replica experts of rank `r` under `mask` in ascending id (slot m + i holds list[i]):
// e is a replica on r iff its home e / m != r and some slot of r routes to it
__device__ int build_replica_list(const uint8_t* mask, int E, int m, int r, int* list, int* flag) {
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int f = 0;
    if (e / m != r)
      for (int j = 0; j < m; ++j) f |= mask[(size_t)(r * m + j) * E + e];
    flag[e] = f;
  }
  __syncthreads();
  __shared__ int n;
  if (threadIdx.x == 0) {
    int c = 0;
    for (int e = 0; e < E; ++e)
      if (flag[e]) list[c++] = e;
    n = c;
  }
  __syncthreads();
  return n;
}

// Trans: pull the home rank's W1/W2 of every replica expert of this rank (decided by the
// plan's mask alone, so it can start before this iteration's routing) into its replica
// slot.  kPeerUnroll independent 16-byte loads per thread keep enough bytes in flight to
// run the NVLink pull at link rate from a few dozen CTAs.
__global__ void __launch_bounds__(512) replica_trans_kernel(void* const* w1_ptrs, void* const* w2_ptrs,
                                                            const uint8_t* mask, int E, int m, int me,
                                                            size_t vecs) {
  __shared__ int list[kMaxListE], flag[kMaxListE];
  const int nrep = build_replica_list(mask, E, m, me, list, flag);
  const size_t total = (size_t)nrep * 2 * vecs;  // uint4 units: [replica][W1|W2][vec]
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = (size_t)blockIdx.x * blockDim.x + threadIdx.x; base < total;
       base += stride * kPeerUnroll) {
    uint4 r[kPeerUnroll];
    uint4* dst[kPeerUnroll];
#pragma unroll
    for (int u = 0; u < kPeerUnroll; ++u) {
      const size_t i = base + u * stride;
      dst[u] = nullptr;
      if (i < total) {
        const size_t mat = i / vecs, v = i - mat * vecs;
        const int rep = (int)(mat >> 1), e = list[rep];
        void* const* ptrs = (mat & 1) ? w2_ptrs : w1_ptrs;
        r[u] = ld_nc_v4(reinterpret_cast<const uint4*>(ptrs[e / m]) + (size_t)(e % m) * vecs + v);
        dst[u] = reinterpret_cast<uint4*>(ptrs[me]) + (size_t)(m + rep) * vecs + v;
      }
    }
#pragma unroll
    for (int u = 0; u < kPeerUnroll; ++u)
      if (dst[u]) st_v4(dst[u], r[u]);
  }
}

// Agg: grad[home slot j] += sum over ranks r != me (ascending) of grad_r[rep_slot[r][e]],
// e = me*m + j; only home slots that have replicas are touched.
__global__ void __launch_bounds__(512) replica_agg_kernel(void* const* g1_ptrs, void* const* g2_ptrs,
                                                          const int32_t* rep_slot, int D, int E, int m,
                                                          int me, size_t vecs) {
  __shared__ int act[kMaxListE];
  __shared__ int nact;
  if (threadIdx.x == 0) {
    int c = 0;
    for (int j = 0; j < m; ++j) {
      bool any = false;
      for (int r = 0; r < D; ++r)
        if (r != me && rep_slot[r * E + me * m + j] >= 0) any = true;
      if (any) act[c++] = j;
    }
    nact = c;
  }
  __syncthreads();
  const size_t total = (size_t)nact * 2 * vecs;  // float4 units: [active slot][g1|g2][vec]
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  constexpr int U = kPeerUnroll / 2;
  for (size_t base = (size_t)blockIdx.x * blockDim.x + threadIdx.x; base < total; base += stride * U) {
    float4 acc[U];
    float4* dst[U];
    int jj[U], which[U];
    size_t vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + u * stride;
      dst[u] = nullptr;
      if (i < total) {
        const size_t mat = i / vecs;
        vv[u] = i - mat * vecs;
        jj[u] = act[mat >> 1];
        which[u] = (int)(mat & 1);
        dst[u] = reinterpret_cast<float4*>((which[u] ? g2_ptrs : g1_ptrs)[me]) + (size_t)jj[u] * vecs + vv[u];
        acc[u] = *dst[u];
      }
    }
    for (int r = 0; r < D; ++r) {
      if (r == me) continue;
      float4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!dst[u]) continue;
        const int s = rep_slot[r * E + me * m + jj[u]];
        if (s < 0) { x[u] = make_float4(0.f, 0.f, 0.f, 0.f); continue; }
        const uint4 raw = ld_nc_v4(reinterpret_cast<const float4*>((which[u] ? g2_ptrs : g1_ptrs)[r]) +
                                   (size_t)s * vecs + vv[u]);
        x[u] = make_float4(__uint_as_float(raw.x), __uint_as_float(raw.y), __uint_as_float(raw.z),
                           __uint_as_float(raw.w));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!dst[u]) continue;
        acc[u].x += x[u].x;
        acc[u].y += x[u].y;
        acc[u].z += x[u].z;
        acc[u].w += x[u].w;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (dst[u]) *dst[u] = acc[u];
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

extern "C" int pp_replica_trans(void* const* w1_ptrs, void* const* w2_ptrs, const uint8_t* mask,
                                int32_t E, int32_t m, int32_t my_rank, int32_t d_model, int32_t d_ff,
                                int32_t max_ctas, void* stream) {
  PP_CHECK_ARG(w1_ptrs && w2_ptrs && mask, "pp_replica_trans: null pointer");
  PP_CHECK_ARG(E >= 1 && E <= kMaxListE && m >= 1 && E % m == 0 && my_rank >= 0 && my_rank < E / m,
               "pp_replica_trans: bad E / m / rank");
  PP_CHECK_ARG(((size_t)d_model * d_ff) % 8 == 0, "pp_replica_trans: bad sizes");
  const int grid = max_ctas > 0 ? max_ctas : 32;
  replica_trans_kernel<<<grid, 512, 0, as_stream(stream)>>>(w1_ptrs, w2_ptrs, mask, E, m, my_rank,
                                                            (size_t)d_model * d_ff / 8);
  PP_LAUNCH_CHECK();
  return PP_OK;
}

extern "C" int pp_replica_agg(void* const* g1_ptrs, void* const* g2_ptrs, const int32_t* rep_slot,
                              int32_t D, int32_t E, int32_t m, int32_t my_rank, int32_t d_model,
                              int32_t d_ff, int32_t max_ctas, void* stream) {
  PP_CHECK_ARG(g1_ptrs && g2_ptrs && rep_slot, "pp_replica_agg: null pointer");
  PP_CHECK_ARG(m >= 1 && m <= kMaxListE && D >= 1 && my_rank >= 0 && my_rank < D,
               "pp_replica_agg: bad D / m / rank");
  PP_CHECK_ARG(((size_t)d_model * d_ff) % 4 == 0, "pp_replica_agg: bad sizes");
  const int grid = max_ctas > 0 ? max_ctas : 32;
  replica_agg_kernel<<<grid, 512, 0, as_stream(stream)>>>(g1_ptrs, g2_ptrs, rep_slot, D, E, m,
                                                          my_rank, (size_t)d_model * d_ff / 4);
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
