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

// signal area of rank r: uint64_t[D + 2]; slot s < D is written by rank s, slot D holds
// r's own barrier counter, slot D + 1 is r's fault word.  epoch == 0: take the epoch from
// that device counter (so a captured CUDA graph can replay barriers), otherwise use the
// host-provided value.  A peer that never arrives (crashed rank) does not hang the GPU and
// does not kill the context: after 20 s the wait gives up, records the fault word (the
// host raises on it) and the kernel returns.
__global__ void peer_barrier_kernel(void* const* signal_ptrs, int D, int me, uint64_t epoch) {
  pdl_grid_sync();
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
        own[D + 1] = 1;  // fault word: the host raises
        break;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) own[D] = e;
}

// Peer traffic is PUSHED: remote 16-byte stores are posted, so ~16 CTAs fill an NVLink 5
// port (measured 700 GB/s push vs 240 GB/s pull at 16 CTAs; scripts/micro/p2p_bw.cu).
constexpr int kPushUnroll = 4;
constexpr int kReduceUnroll = 8;
constexpr int kMaxFlags = 16384;  // D * E
constexpr int kMaxItems = 1024;   // E

// flag[r*E + e] = 1 iff expert e is a replica on rank r under mask: home e/m != r and some
// slot of r routes to e.  A replica's weight slot is m + #{e' < e : flag[r*E + e']}, the
// same rule pp_dispatch_layout uses for its group table and rep_slot.
__device__ void replica_flags(const uint8_t* mask, int D, int E, int m, uint8_t* flag) {
  for (int t = threadIdx.x; t < D * E; t += blockDim.x) {
    const int r = t / E, e = t - (t / E) * E;
    int f = 0;
    if (e / m != r)
      for (int j = 0; j < m; ++j) f |= mask[(size_t)(r * m + j) * E + e];
    flag[t] = (uint8_t)f;
  }
  __syncthreads();
}

__device__ __forceinline__ int replica_index(const uint8_t* flag, int E, int r, int e) {
  int c = 0;
  for (int x = 0; x < e; ++x) c += flag[r * E + x];
  return c;
}

// deterministic compaction of per-thread candidates (same order in every CTA)
__device__ int compact_items(const int* cand, int n, int* items) {
  __shared__ int cnt;
  if (threadIdx.x == 0) {
    int c = 0;
    for (int t = 0; t < n; ++t)
      if (cand[t] >= 0) items[c++] = cand[t];
    cnt = c;
  }
  __syncthreads();
  return cnt;
}

// 16-byte copy of `nmat` matrices of `vecs` uint4 each, addresses from addr(matrix index):
// CTAs stride over (matrix, chunk) pairs -- one 32-bit division per chunk, none per
// element -- and each thread keeps U independent loads in flight.
template <int U, class Addr>
__device__ __forceinline__ void push_copy(int nmat, size_t vecs, Addr addr) {
  constexpr int kThreads = 512;
  const size_t chunk = (size_t)kThreads * U;
  const int per_mat = (int)((vecs + chunk - 1) / chunk);
  const int nchunks = nmat * per_mat;
  for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int mat = c / per_mat;
    const size_t off = (size_t)(c - mat * per_mat) * chunk + threadIdx.x;
    const uint4* src;
    uint4* dst;
    addr(mat, 0, src, dst);
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (off + u * kThreads < vecs) r[u] = ld_nc_v4(src + off + u * kThreads);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (off + u * kThreads < vecs) st_v4(dst + off + u * kThreads, r[u]);
  }
}

// Trans (home side): push each of this rank's home experts to every rank holding it as a
// replica, into that rank's replica slot.  The receivers' previous use of those slots
// ended before the last peer barrier of their backward, which this rank has passed.
__global__ void __launch_bounds__(512) replica_trans_kernel(void* const* w1_ptrs, void* const* w2_ptrs,
                                                            const uint8_t* mask, int E, int m, int me,
                                                            int num_slots, size_t vecs, int parts, void* const* flag_ptrs,
                                                            int flag_row, const uint64_t* epoch,
                                                            unsigned int* done_ctr) {
  pdl_grid_sync();
  __shared__ uint8_t flag[kMaxFlags];
  __shared__ int cand[kMaxItems], items[kMaxItems];
  const int D = E / m;
  replica_flags(mask, D, E, m, flag);
  for (int t = threadIdx.x; t < D * m; t += blockDim.x) {  // t = (receiver r, home slot j)
    const int r = t / m, j = t - (t / m) * m, e = me * m + j;
    const int i = (r != me && flag[r * E + e]) ? replica_index(flag, E, r, e) : -1;
    cand[t] = (i >= 0 && m + i < num_slots) ? ((r * m + j) << 10 | i) : -1;  // slot bound
  }
  __syncthreads();
  const int n = compact_items(cand, D * m, items);
  const int np = parts == 3 ? 2 : 1;
  push_copy<kPushUnroll>(n * np, vecs, [&](int it2, int, const uint4*& src, uint4*& dst) {
    const int it = np == 2 ? it2 >> 1 : it2, mat = np == 2 ? (it2 & 1) : (parts >> 1);
    const int code = items[it], rj = code >> 10, i = code & 1023;
    const int r = rj / m, j = rj - (rj / m) * m;
    void* const* ptrs = mat ? w2_ptrs : w1_ptrs;
    src = reinterpret_cast<const uint4*>(ptrs[me]) + (size_t)j * vecs;
    dst = reinterpret_cast<uint4*>(ptrs[r]) + (size_t)(m + i) * vecs;
  });
  if (!flag_ptrs) return;
  // completion signal: the last CTA to finish tells every peer "my pushes for epoch
  // *epoch have landed" (release after all CTAs' system-scope fences), so a receiver's
  // FWD1 can start on its home experts and gate only its replica tiles on the flags
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned int prev = atomicAdd(done_ctr, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      const uint64_t e = *epoch;
      const int D = E / m;
      for (int r = 0; r < D; ++r)
        if (r != me) st_release_sys(reinterpret_cast<uint64_t*>(flag_ptrs[r]) + (size_t)flag_row * D + me, e);
      *done_ctr = 0;  // ready for the next launch (stream-ordered)
    }
  }
}

// Agg, phase 1 (replica side): push the fp32 grads of every replica slot of this rank into
// the home rank's staging area stage[j][r'][W1|W2] (r' = this rank's index among the
// home's D-1 peers), so the home can sum its sources in rank order.
__global__ void __launch_bounds__(512) replica_agg_push_kernel(void* const* g1_ptrs, void* const* g2_ptrs,
                                                               void* const* stage_ptrs, const uint8_t* mask,
                                                               int E, int m, int me, int num_slots, size_t vecs,
                                                               int parts) {
  pdl_grid_sync();
  __shared__ uint8_t flag[kMaxFlags];
  __shared__ int cand[kMaxItems], items[kMaxItems];
  const int D = E / m;
  replica_flags(mask, D, E, m, flag);
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int i = flag[me * E + e] ? replica_index(flag, E, me, e) : -1;
    cand[e] = (i >= 0 && m + i < num_slots) ? (e << 10 | i) : -1;  // slot bound
  }
  __syncthreads();
  const int n = compact_items(cand, E, items);
  const int np = parts == 3 ? 2 : 1;  // bit 0: W1 grads, bit 1: W2 grads
  push_copy<kPushUnroll>(n * np, vecs, [&](int it2, int, const uint4*& src, uint4*& dst) {
    const int it = np == 2 ? it2 >> 1 : it2, mat = np == 2 ? (it2 & 1) : (parts >> 1);
    const int code = items[it], e = code >> 10, i = code & 1023;
    const int h = e / m, j = e - h * m, rp = me < h ? me : me - 1;
    src = reinterpret_cast<const uint4*>((mat ? g2_ptrs : g1_ptrs)[me]) + (size_t)(m + i) * vecs;
    dst = reinterpret_cast<uint4*>(stage_ptrs[h]) + ((size_t)(j * (D - 1) + rp) * 2 + mat) * vecs;
  });
}

// Agg, phase 2 (home side, local HBM): grad[j] += stage[j][r'] for the ranks r != me that
// hold expert me*m + j, ascending r (deterministic, = the oracle's rank-order sum).
__global__ void __launch_bounds__(512, 1) replica_agg_reduce_kernel(float* g1, float* g2, const float* stage,
                                                                    const uint8_t* mask, int E, int m, int me,
                                                                    size_t vecs, int parts) {
  pdl_grid_sync();
  __shared__ uint8_t flag[kMaxFlags];
  __shared__ int cand[kMaxItems], items[kMaxItems];
  __shared__ uint32_t srcmask[kMaxItems];
  const int D = E / m;
  replica_flags(mask, D, E, m, flag);
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    uint32_t bits = 0;
    for (int r = 0, rp = 0; r < D; ++r) {
      if (r == me) continue;
      if (flag[r * E + me * m + j]) bits |= 1u << rp;
      ++rp;
    }
    srcmask[j] = bits;
    cand[j] = bits ? j : -1;
  }
  __syncthreads();
  const int n = compact_items(cand, m, items);
  constexpr int U = kReduceUnroll, kThreads = 512;
  const size_t chunk = (size_t)kThreads * U;
  const int per_mat = (int)((vecs + chunk - 1) / chunk);
  const int np = parts == 3 ? 2 : 1;  // bit 0: W1 grads, bit 1: W2 grads
  const int nchunks = n * np * per_mat;
  for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {  // (active slot, g1|g2, chunk)
    const int mat = c / per_mat;
    const size_t off = (size_t)(c - mat * per_mat) * chunk + threadIdx.x;
    const int j = items[np == 2 ? mat >> 1 : mat], w = np == 2 ? (mat & 1) : (parts >> 1);
    const uint32_t bits = srcmask[j];
    float4* dst = reinterpret_cast<float4*>(w ? g2 : g1) + (size_t)j * vecs + off;
    const float4* src = reinterpret_cast<const float4*>(stage) + (size_t)j * (D - 1) * 2 * vecs + w * vecs + off;
    float4 acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (off + u * kThreads < vecs) acc[u] = dst[u * kThreads];
    for (int rp = 0; rp < D - 1; ++rp) {
      if (!(bits >> rp & 1)) continue;
      const float4* sp = src + (size_t)rp * 2 * vecs;
      float4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (off + u * kThreads < vecs) x[u] = __ldcs(sp + u * kThreads);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc[u].x += x[u].x;
        acc[u].y += x[u].y;
        acc[u].z += x[u].z;
        acc[u].w += x[u].w;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (off + u * kThreads < vecs) dst[u * kThreads] = acc[u];
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
  PP_CUDA_TRY(pdl_launch(peer_barrier_kernel, dim3(1), dim3(((D + 31) / 32) * 32), 0, as_stream(stream), signal_ptrs, D, my_rank,
                                                                         epoch));
  PP_LAUNCH_CHECK();
  return PP_OK;
}

extern "C" int pp_replica_trans(void* const* w1_ptrs, void* const* w2_ptrs, const uint8_t* mask,
                                int32_t E, int32_t m, int32_t my_rank, int32_t num_slots, int32_t d_model,
                                int32_t d_ff, int32_t parts, void* const* flag_ptrs, int32_t flag_row,
                                const uint64_t* epoch, uint32_t* done_ctr, int32_t max_ctas,
                                void* stream) {
  PP_CHECK_ARG(parts >= 1 && parts <= 3 && flag_row >= 0, "pp_replica_trans: bad parts / flag_row");
  PP_CHECK_ARG(!flag_ptrs || (epoch && done_ctr), "pp_replica_trans: flags need epoch and done_ctr");
  PP_CHECK_ARG(w1_ptrs && w2_ptrs && mask, "pp_replica_trans: null pointer");
  PP_CHECK_ARG(E >= 1 && E <= kMaxItems && m >= 1 && E % m == 0 && (E / m) * E <= kMaxFlags &&
                   my_rank >= 0 && my_rank < E / m,
               "pp_replica_trans: bad E / m / rank");
  PP_CHECK_ARG(((size_t)d_model * d_ff) % 8 == 0, "pp_replica_trans: bad sizes");
  const int grid = max_ctas > 0 ? max_ctas : 16;
  PP_CHECK_ARG(num_slots > m, "pp_replica_trans: num_slots=%d leaves no replica slot (m=%d)", num_slots, m);
  PP_CUDA_TRY(pdl_launch(replica_trans_kernel, dim3(grid), dim3(512), 0, as_stream(stream), w1_ptrs, w2_ptrs, mask, E, m, my_rank, num_slots,
                                                            (size_t)d_model * d_ff / 8, parts, flag_ptrs,
                                                            flag_row, epoch, done_ctr));
  PP_LAUNCH_CHECK();
  return PP_OK;
}

extern "C" int pp_replica_agg(void* const* g1_ptrs, void* const* g2_ptrs, void* const* stage_ptrs,
                              const uint8_t* mask, int32_t E, int32_t m, int32_t my_rank, int32_t num_slots,
                              int32_t d_model, int32_t d_ff, int32_t parts, int32_t max_ctas,
                              void* stream) {
  PP_CHECK_ARG(parts >= 1 && parts <= 3, "pp_replica_agg: parts must be 1 (W1), 2 (W2) or 3, got %d", parts);
  PP_CHECK_ARG(g1_ptrs && g2_ptrs && stage_ptrs && mask, "pp_replica_agg: null pointer");
  PP_CHECK_ARG(E >= 1 && E <= kMaxItems && m >= 1 && E % m == 0 && (E / m) * E <= kMaxFlags &&
                   my_rank >= 0 && my_rank < E / m,
               "pp_replica_agg: bad E / m / rank");
  PP_CHECK_ARG(((size_t)d_model * d_ff) % 4 == 0, "pp_replica_agg: bad sizes");
  const int grid = max_ctas > 0 ? max_ctas : 16;
  PP_CHECK_ARG(num_slots > m, "pp_replica_agg: num_slots=%d leaves no replica slot (m=%d)", num_slots, m);
  PP_CUDA_TRY(pdl_launch(replica_agg_push_kernel, dim3(grid), dim3(512), 0, as_stream(stream), g1_ptrs, g2_ptrs, stage_ptrs, mask, E, m,
                                                               my_rank, num_slots, (size_t)d_model * d_ff / 4, parts));
  PP_LAUNCH_CHECK();
  return PP_OK;
}

extern "C" int pp_replica_agg_reduce(float* g1, float* g2, const float* stage, const uint8_t* mask,
                                     int32_t E, int32_t m, int32_t my_rank, int32_t d_model,
                                     int32_t d_ff, int32_t parts, int32_t max_ctas, void* stream) {
  PP_CHECK_ARG(parts >= 1 && parts <= 3, "pp_replica_agg_reduce: parts must be 1, 2 or 3, got %d", parts);
  PP_CHECK_ARG(g1 && g2 && stage && mask, "pp_replica_agg_reduce: null pointer");
  PP_CHECK_ARG(E >= 1 && E <= kMaxItems && m >= 1 && E % m == 0 && (E / m) * E <= kMaxFlags &&
                   E / m <= 33 && my_rank >= 0 && my_rank < E / m,
               "pp_replica_agg_reduce: bad E / m / rank (D <= 33)");
  PP_CHECK_ARG(((size_t)d_model * d_ff) % 4 == 0, "pp_replica_agg_reduce: bad sizes");
  const int grid = max_ctas > 0 ? max_ctas : 16;
  PP_CUDA_TRY(pdl_launch(replica_agg_reduce_kernel, dim3(grid), dim3(512), 0, as_stream(stream), g1, g2, stage, mask, E, m, my_rank,
                                                                  (size_t)d_model * d_ff / 4, parts));
  PP_LAUNCH_CHECK();
  return PP_OK;
}

// ---- copy-engine Trans/Agg helpers ----------------------------------------------
namespace pp {
// home grad slot j += sum of staging entries [ranges[j], ranges[j+1]) (rank order);
// staging entry i = [g1 part (f*d) | g2 part (d*f)] fp32
__global__ void agg_accumulate_kernel(float* g1, float* g2, const float* staging,
                                      const int32_t* ranges, int m, size_t fd) {
  pdl_grid_sync();
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
  PP_CUDA_TRY(pdl_launch(agg_accumulate_kernel, dim3(4 * 148), dim3(256), 0, as_stream(stream), g1_home, g2_home, staging, ranges, m,
                                                                (size_t)d_model * d_ff));
  PP_LAUNCH_CHECK();
  return PP_OK;
}
