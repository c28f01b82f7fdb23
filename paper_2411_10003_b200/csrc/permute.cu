// K1 host wrapper + K3: routing histogram, dispatch layout, fused permute/all-to-all,
// combine, and their backward passes.
//
// Routing rule (reference derive_loads, pkg/src/moebal/core.py:267-274), applied
// at virtual-expert-slot granularity: the pairs
// of virtual slot v routed to expert e are computed on rank v / m when the plan's
// replica mask holds mask[v][e], otherwise on e's home rank e / m.  The receive
// layout of every rank is expert-major: one segment per expert the rank holds
// (ascending expert id, padded to 128 rows), and inside a segment pairs are
// ordered by (source slot v, token t) -- a stable order every rank derives from
// the all-gathered LoadMatrix, so no host round trip is needed.
//
// Data moves over peer-mapped pointers: dispatch STORES a token row directly into
// the computing rank's receive buffer (local or NVLink peer), combine LOADS the
// expert outputs back from wherever they were computed.  At D = 1 the pointer
// tables hold a single local buffer.
#include "common.cuh"

namespace pp {

int route_gemm(const void* x, const void* wg, const float* bias, int T, int d, int E, int k,
               int32_t* idx, float* w, float* probs, int32_t* rank, int32_t* chunk_counts,
               cudaStream_t st);

// ---------------------------------------------------------------------------
// this rank's m virtual-slot rows of the LoadMatrix, stored into every rank's copy
// (peer-mapped) -- the all-gather of the histogram without a collective library
__global__ void slot_histogram_kernel(const int32_t* chunk_counts, int chunks_per_slot, int E,
                                      int m, int64_t* const* out_ptrs, int D, int row0) {
  pdl_grid_sync();
  const int cell = blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= m * E) return;
  const int v = cell / E, e = cell % E;
  int64_t s = 0;
  for (int c = 0; c < chunks_per_slot; ++c)
    s += chunk_counts[(size_t)(v * chunks_per_slot + c) * E + e];
  for (int r = 0; r < D; ++r) out_ptrs[r][(size_t)(row0 + v) * E + e] = s;
}

// ---------------------------------------------------------------------------
// Layout solver: one CTA, everything staged in shared memory.  See ppmoe.h.
constexpr int kLayoutThreads = 1024;

struct LayoutSmem {
  int32_t* counts;   // [Ev][E]
  uint8_t* comp;     // [Ev][E] computing rank of (slot, expert)
  uint8_t* local;    // [Ev][E] replica mask (diagonal when none)
  int32_t* cc;       // [C][E] chunk counts of this rank
  int32_t* rows;     // [D][E]
  int32_t* seg;      // [D][E]
  uint8_t* present;  // [D][E]
};

__host__ __device__ inline size_t layout_smem_bytes(int D, int m, int E, int T) {
  const size_t Ev = (size_t)D * m, C = (size_t)T / PP_CHUNK;
  return Ev * E * (4 + 1 + 1) + C * E * 4 + (size_t)D * E * (4 + 4 + 1) + 64;
}

__global__ void __launch_bounds__(kLayoutThreads)
    dispatch_layout_kernel(int64_t* counts, const uint8_t* mask, const int32_t* chunk_counts,
                           int D, int m, int E, int T, int me, int max_groups, int rows_capacity,
                           int num_slots, int32_t* chunk_base, int32_t* slot_dest, pp_group* groups,
                           int32_t* num_groups, int32_t* total_rows, int32_t* seg_start,
                           int32_t* rep_slot, int counts_from_chunks, int32_t* replica_stats,
                           int32_t* status) {
  pdl_grid_sync();
  __shared__ int overflow;
  extern __shared__ __align__(16) uint8_t lsm[];
  const int Ev = D * m, C = T / PP_CHUNK, tid = threadIdx.x, nt = blockDim.x;
  LayoutSmem S;
  uint8_t* p = lsm;
  S.counts = reinterpret_cast<int32_t*>(p); p += (size_t)Ev * E * 4;
  S.cc = reinterpret_cast<int32_t*>(p); p += (size_t)C * E * 4;
  S.rows = reinterpret_cast<int32_t*>(p); p += (size_t)D * E * 4;
  S.seg = reinterpret_cast<int32_t*>(p); p += (size_t)D * E * 4;
  S.comp = p; p += (size_t)Ev * E;
  S.local = p; p += (size_t)Ev * E;
  S.present = p;

  // phase 0: stage inputs (single rank: the LoadMatrix rows are summed from the
  // chunk counts right here, replacing the histogram kernel + barrier)
  for (int i = tid; i < C * E; i += nt) S.cc[i] = chunk_counts[i];
  if (counts_from_chunks) {
    __syncthreads();
    const int cps_ = (T / m) / PP_CHUNK;
    for (int i = tid; i < Ev * E; i += nt) {
      const int v = i / E, e = i % E;
      int s = 0;
      for (int c = 0; c < cps_; ++c) s += S.cc[(v * cps_ + c) * E + e];
      counts[i] = s;
    }
    __syncthreads();
  }
  for (int i = tid; i < Ev * E; i += nt) {
    const int v = i / E, e = i % E;
    S.counts[i] = (int32_t)counts[i];
    const bool loc = mask ? (mask[i] != 0) : (v == e);
    S.local[i] = loc;
    S.comp[i] = (uint8_t)(loc ? v / m : e / m);
  }
  __syncthreads();
  // phase 1: rows / presence of every (rank, expert)
  for (int cell = tid; cell < D * E; cell += nt) {
    const int r = cell / E, e = cell % E;
    int acc = 0;
    bool pres = (e / m == r);
    for (int v = 0; v < Ev; ++v) {
      const int i = v * E + e;
      if (S.comp[i] == r) acc += S.counts[i];
      pres |= S.local[i] && (v / m == r);
    }
    S.rows[cell] = acc;
    S.present[cell] = pres;
  }
  __syncthreads();
  // phase 2: expert-major segments per rank (ascending expert id, 128-row padding)
  if (tid == 0) overflow = 0;
  __syncthreads();
  for (int r = tid; r < D; r += nt) {
    int64_t off = 0;
    int nrep = 0, ng = 0;
    for (int e = 0; e < E; ++e) {
      const int cell = r * E + e;
      const bool pres = S.present[cell];
      if (rep_slot) rep_slot[cell] = (pres && e / m != r) ? m + nrep++ : -1;
      ng += pres;
      S.seg[cell] = pres ? (int)off : -1;
      seg_start[cell] = S.seg[cell];
      if (pres) off += (S.rows[cell] + PP_ROW_ALIGN - 1) / PP_ROW_ALIGN * PP_ROW_ALIGN;
    }
    // capacity rule (identical on every rank: same LoadMatrix and mask)
    const int bits = (off > rows_capacity ? 1 : 0) | (num_slots > 0 && m + nrep > num_slots ? 2 : 0) |
                     (ng > max_groups ? 4 : 0);
    if (bits) atomicOr(&overflow, bits);
    if (r == me) *total_rows = (int)off;
  }
  __syncthreads();
  if (overflow) {  // drop the step on every rank alike: nothing is stored out of bounds
    if (tid == 0) {
      if (status) atomicOr(status, overflow);
      *num_groups = 0;
      *total_rows = 0;
      if (replica_stats) replica_stats[0] = replica_stats[1] = 0;
    }
    for (int cell = tid; cell < m * E; cell += nt) slot_dest[cell] = -1;
    return;
  }
  if (replica_stats && tid == 0) {
    // [0] replicas of this rank's home experts held elsewhere (Trans pushes out, Agg sources in)
    // [1] replicas this rank holds (Agg pushes out)
    int out = 0, held = 0;
    for (int r = 0; r < D; ++r)
      if (r != me)
        for (int e = me * m; e < (me + 1) * m; ++e) out += S.present[r * E + e];
    for (int e = 0; e < E; ++e) held += (e / m != me) && S.present[me * E + e];
    replica_stats[0] = out;
    replica_stats[1] = held;
  }
  // phase 3: this rank's group table
  if (tid == 0) {
    int g = 0, nrep = 0;
    for (int e = 0; e < E && g < max_groups; ++e) {
      const int cell = me * E + e;
      if (!S.present[cell]) continue;
      pp_group gr;
      gr.row_off = S.seg[cell];
      gr.rows = S.rows[cell];
      gr.rows_pad = (S.rows[cell] + PP_ROW_ALIGN - 1) / PP_ROW_ALIGN * PP_ROW_ALIGN;
      const bool home = (e / m == me);
      gr.wslot = home ? (e % m) : (m + nrep++);
      gr.expert = e;
      gr.src_rank = e / m;
      gr._pad[0] = gr._pad[1] = 0;
      groups[g++] = gr;
    }
    *num_groups = g;
  }
  // phase 4: destination + first row of each (local slot, expert), then per chunk
  const int cps = (T / m) / PP_CHUNK;
  for (int cell = tid; cell < m * E; cell += nt) {
    const int j = cell / E, e = cell % E;
    const int v = me * m + j;
    const int dest = S.comp[v * E + e];
    int base = S.seg[dest * E + e];
    for (int v2 = 0; v2 < v; ++v2)
      if (S.comp[v2 * E + e] == dest) base += S.counts[v2 * E + e];
    slot_dest[cell] = dest;
    for (int c = 0; c < cps; ++c) {
      const int chunk = j * cps + c;
      chunk_base[(size_t)chunk * E + e] = base;
      base += S.cc[chunk * E + e];
    }
  }
}

// zero rows [row_off+rows, row_off+rows_pad) of every group of this rank (warp per row)
template <int VPL>
__device__ __forceinline__ void zero_padding_rows(const pp_group* groups, const int32_t* num_groups,
                                                  int d, __nv_bfloat16* buf, int warp_global,
                                                  int nwarps, int lane, int32_t* origin = nullptr) {
  const int G = *num_groups;
  for (int w = warp_global; w < G * PP_ROW_ALIGN; w += nwarps) {
    const pp_group gr = groups[w / PP_ROW_ALIGN];
    const int j = w % PP_ROW_ALIGN;
    if (j >= gr.rows_pad - gr.rows) continue;
    uint4* dst = reinterpret_cast<uint4*>(buf + (size_t)(gr.row_off + gr.rows + j) * d);
#pragma unroll
    for (int i = 0; i < VPL; ++i) st_v4(dst + lane + 32 * i, make_uint4(0, 0, 0, 0));
    if (origin && lane == 0) origin[gr.row_off + gr.rows + j] = -1;  // padding: no source pair
  }
}

// ---------------------------------------------------------------------------
template <int VPL>  // 16-byte vectors per lane per row (d = VPL * 256)
__global__ void __launch_bounds__(256)
    dispatch_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ idx,
                    const int32_t* __restrict__ rank, const int32_t* __restrict__ chunk_base,
                    const int32_t* __restrict__ slot_dest, int T, int d, int k, int m, int E,
                    void* const* recv_ptrs, int32_t* pair_dest, int32_t* pair_row,
                    const pp_group* groups, const int32_t* num_groups, __nv_bfloat16* own,
                    void* const* origin_ptrs, int me) {
  pdl_grid_sync();
  const int lane = threadIdx.x & 31;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int slot_tokens = T / m;
  zero_padding_rows<VPL>(groups, num_groups, d, own, warp_global, nwarps, lane,
                         origin_ptrs ? reinterpret_cast<int32_t*>(origin_ptrs[me]) : nullptr);
  for (int t = warp_global; t < T; t += nwarps) {
    uint4 v[VPL];
    const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)t * d);
#pragma unroll
    for (int i = 0; i < VPL; ++i) v[i] = ld_nc_v4(src + lane + 32 * i);
    int my_dest = 0, my_row = 0;
    if (lane < k) {
      const int e = idx[(size_t)t * k + lane];
      const int slot = t / slot_tokens;
      my_dest = slot_dest[slot * E + e];
      my_row = chunk_base[(size_t)(t / PP_CHUNK) * E + e] + rank[(size_t)t * k + lane];
      pair_dest[(size_t)t * k + lane] = my_dest;
      pair_row[(size_t)t * k + lane] = my_row;
    }
    for (int j = 0; j < k; ++j) {
      const int dest = __shfl_sync(0xffffffffu, my_dest, j);
      const int row = __shfl_sync(0xffffffffu, my_row, j);
      if (dest < 0) continue;  // dropped step (layout capacity flag)
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(recv_ptrs[dest]) +
                                            (size_t)row * d);
#pragma unroll
      for (int i = 0; i < VPL; ++i) st_v4(dst + lane + 32 * i, v[i]);
      // fused A2A: the computing rank's GEMM epilogue sends this row's result straight back
      if (origin_ptrs && lane == 0)
        reinterpret_cast<int32_t*>(origin_ptrs[dest])[row] = me * T * k + t * k + j;
    }
  }
}



template <int VPL>
__global__ void __launch_bounds__(256)
    combine_kernel(void* const* out_ptrs, const int32_t* __restrict__ pair_dest,
                   const int32_t* __restrict__ pair_row, const float* __restrict__ w, int T, int d,
                   int k, __nv_bfloat16* y, const __nv_bfloat16* __restrict__ comb) {
  pdl_grid_sync();
  const int lane = threadIdx.x & 31;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp_global; t < T; t += nwarps) {
    float acc[VPL][8];
#pragma unroll
    for (int i = 0; i < VPL; ++i)
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[i][u] = 0.f;
    int my_dest = 0, my_row = 0;
    float my_w = 0.f;
    if (lane < k) {
      my_dest = pair_dest[(size_t)t * k + lane];
      my_row = pair_row[(size_t)t * k + lane];
      my_w = w[(size_t)t * k + lane];
    }
    // one pair row at a time: fewer registers -> more resident warps, which measured faster
    // (16.1 us) than two rows in flight per warp (18.5 us at 86 registers) at cfg2
    for (int j = 0; j < k; ++j) {
      const int dest = __shfl_sync(0xffffffffu, my_dest, j);
      const int row = __shfl_sync(0xffffffffu, my_row, j);
      const float wj = __shfl_sync(0xffffffffu, my_w, j);
      if (dest < 0) continue;  // dropped step
      // fused A2A: the expert outputs were pushed here by the GEMM epilogue, in pair order
      const uint4* src = reinterpret_cast<const uint4*>(
          comb ? comb + (size_t)(t * k + j) * d
               : reinterpret_cast<const __nv_bfloat16*>(out_ptrs[dest]) + (size_t)row * d);
      uint4 v[VPL];
#pragma unroll
      for (int i = 0; i < VPL; ++i) v[i] = ld_v4(src + lane + 32 * i);
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        float f[8];
        bf16x8_to_f32(v[i], f);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[i][u] = fmaf(wj, f[u], acc[i][u]);
      }
    }
    uint4* dst = reinterpret_cast<uint4*>(y + (size_t)t * d);
#pragma unroll
    for (int i = 0; i < VPL; ++i) st_v4(dst + lane + 32 * i, f32x8_to_bf16(acc[i]));
  }
}

template <int VPL, int EP>
__global__ void __launch_bounds__(256)
    combine_bwd_kernel(const __nv_bfloat16* __restrict__ dy, void* const* out_ptrs,
                       void* const* dgrad_ptrs, const int32_t* __restrict__ pair_dest,
                       const int32_t* __restrict__ pair_row, const float* __restrict__ w, int T,
                       int d, int k, float* dw, const pp_group* groups, const int32_t* num_groups,
                       __nv_bfloat16* own, const __nv_bfloat16* __restrict__ comb,
                       const int32_t* __restrict__ idx, const float* __restrict__ probs, int E,
                       __nv_bfloat16* dl) {
  pdl_grid_sync();
  const int lane = threadIdx.x & 31;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  zero_padding_rows<VPL>(groups, num_groups, d, own, warp_global, nwarps, lane);
  for (int t = warp_global; t < T; t += nwarps) {
    // everything this token needs is requested up front: pair info, the gate's probabilities
    // (dL/dlogits below), dy, and the Yp rows of two pairs at a time
    int my_dest = 0, my_row = 0, my_e = -1;
    float my_w = 0.f;
    if (lane < k) {
      my_dest = pair_dest[(size_t)t * k + lane];
      my_row = pair_row[(size_t)t * k + lane];
      my_w = w[(size_t)t * k + lane];
      my_e = idx[(size_t)t * k + lane];
    }
    float pq[EP / 32];
#pragma unroll
    for (int q = 0; q < EP / 32; ++q) pq[q] = lane + 32 * q < E ? probs[(size_t)t * E + lane + 32 * q] : 0.f;
    float g[VPL][8];
    const uint4* src = reinterpret_cast<const uint4*>(dy + (size_t)t * d);
#pragma unroll
    for (int i = 0; i < VPL; ++i) bf16x8_to_f32(ld_nc_v4(src + lane + 32 * i), g[i]);
    float my_dw = 0.f;
    for (int j0 = 0; j0 < k; j0 += 2) {
      uint4 yv[2][VPL];
      int dest[2], row[2];
      float wj[2];
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int j = j0 + jj < k ? j0 + jj : j0;
        dest[jj] = __shfl_sync(0xffffffffu, my_dest, j);
        row[jj] = __shfl_sync(0xffffffffu, my_row, j);
        wj[jj] = __shfl_sync(0xffffffffu, my_w, j);
        if (j0 + jj >= k) dest[jj] = -1;
        if (dest[jj] >= 0) {
          const uint4* ysrc = reinterpret_cast<const uint4*>(
              comb ? comb + (size_t)(t * k + j) * d
                   : reinterpret_cast<const __nv_bfloat16*>(out_ptrs[dest[jj]]) + (size_t)row[jj] * d);
#pragma unroll
          for (int i = 0; i < VPL; ++i) yv[jj][i] = ld_v4(ysrc + lane + 32 * i);
        }
      }
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        if (dest[jj] < 0) continue;  // beyond k, or dropped step: dw stays 0
        uint4* gdst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(dgrad_ptrs[dest[jj]]) +
                                               (size_t)row[jj] * d);
        float dot = 0.f;
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          float y8[8], o[8];
          bf16x8_to_f32(yv[jj][i], y8);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            dot = fmaf(g[i][u], y8[u], dot);
            o[u] = wj[jj] * g[i][u];
          }
          st_v4(gdst + lane + 32 * i, f32x8_to_bf16(o));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (lane == j0 + jj) my_dw = dot;
      }
    }
    if (lane < k) dw[(size_t)t * k + lane] = my_dw;
    // gate softmax backward restricted to the selected experts (dw is complete here):
    //   dl_i = p_i * (dw_{j(i)} [i selected] - sum_j dw_j p_{e_j})
    float p_sel = 0.f;  // p_{e_j} for lane j < k, from the lane holding expert e_j
#pragma unroll
    for (int q = 0; q < EP / 32; ++q) {
      const float v = __shfl_sync(0xffffffffu, pq[q], my_e & 31);
      if (lane < k && (my_e >> 5) == q) p_sel = v;
    }
    float gsum = lane < k ? my_dw * p_sel : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gsum += __shfl_xor_sync(0xffffffffu, gsum, o);
#pragma unroll
    for (int q = 0; q < EP / 32; ++q) {
      const int i = lane + 32 * q;
      float sel_dw = 0.f;
      for (int j = 0; j < k; ++j) {
        const int ej = __shfl_sync(0xffffffffu, my_e, j);
        const float dwj = __shfl_sync(0xffffffffu, my_dw, j);
        if (ej == i) sel_dw = dwj;
      }
      dl[(size_t)t * EP + i] = __float2bfloat16_rn(i < E ? pq[q] * (sel_dw - gsum) : 0.f);
    }
  }
}

static int grid_for_tokens(int T) {
  int blocks = (T + 7) / 8;  // 8 warps per block, one token per warp per step
  return blocks < 148 * 8 ? blocks : 148 * 8;
}

}  // namespace pp

using namespace pp;

#define PP_VPL_SWITCH(d, ...)                                               \
  switch ((d) / 256) {                                                      \
    case 1: { constexpr int VPL = 1; __VA_ARGS__; break; }                  \
    case 2: { constexpr int VPL = 2; __VA_ARGS__; break; }                  \
    case 4: { constexpr int VPL = 4; __VA_ARGS__; break; }                  \
    case 8: { constexpr int VPL = 8; __VA_ARGS__; break; }                  \
    case 16: { constexpr int VPL = 16; __VA_ARGS__; break; }                \
    default: return fail(PP_EINVAL, "d=%d must be 256 * {1,2,4,8,16}", d);  \
  }

extern "C" int pp_route_topk(const void* x, const void* wg, const float* bias, int32_t T,
                             int32_t d, int32_t E, int32_t k, int32_t* idx, float* w,
                             float* probs, int32_t* rank, int32_t* chunk_counts, void* stream) {
  PP_CHECK_ARG(x && wg && idx && w && probs && rank && chunk_counts, "pp_route_topk: null pointer");
  PP_CHECK_ARG(T > 0 && T % PP_CHUNK == 0, "pp_route_topk: T=%d must be a positive multiple of %d",
               T, PP_CHUNK);
  PP_CHECK_ARG(d > 0 && d % 64 == 0, "pp_route_topk: d=%d must be a multiple of 64", d);
  PP_CHECK_ARG(E >= 4 && E <= 128 && E % 4 == 0, "pp_route_topk: E=%d unsupported", E);
  PP_CHECK_ARG(k >= 1 && k <= 8 && k <= E, "pp_route_topk: k=%d unsupported", k);
  return route_gemm(x, wg, bias, T, d, E, k, idx, w, probs, rank, chunk_counts, as_stream(stream));
}

extern "C" int pp_slot_histogram(const int32_t* chunk_counts, int32_t T, int32_t E, int32_t m,
                                 int64_t* const* out_ptrs, int32_t D, int32_t row0, void* stream) {
  PP_CHECK_ARG(chunk_counts && out_ptrs && D >= 1, "pp_slot_histogram: bad arguments");
  PP_CHECK_ARG(m >= 1 && T % (m * PP_CHUNK) == 0,
               "pp_slot_histogram: T=%d must split into m=%d slots of whole %d-token chunks", T, m,
               PP_CHUNK);
  const int cps = (T / m) / PP_CHUNK;
  const int cells = m * E;
  PP_CUDA_TRY(pdl_launch(slot_histogram_kernel, dim3((cells + 255) / 256), dim3(256), 0, as_stream(stream), chunk_counts, cps, E, m,
                                                                            out_ptrs, D, row0));
  PP_LAUNCH_CHECK();
  return PP_OK;
}

extern "C" int pp_dispatch_layout(int64_t* counts, const uint8_t* mask,
                                  const int32_t* chunk_counts, int32_t D, int32_t m, int32_t E,
                                  int32_t T, int32_t my_rank, int32_t max_groups,
                                  int32_t rows_capacity, int32_t num_slots, int32_t* chunk_base,
                                  int32_t* slot_dest, pp_group* groups, int32_t* num_groups,
                                  int32_t* total_rows, int32_t* seg_start, int32_t* rep_slot,
                                  int32_t counts_from_chunks, int32_t* replica_stats, int32_t* status,
                                  void* stream) {
  PP_CHECK_ARG(counts && chunk_counts && chunk_base && slot_dest && groups && num_groups &&
                   total_rows && seg_start,
               "pp_dispatch_layout: null pointer");
  PP_CHECK_ARG(D >= 1 && m >= 1 && E == D * m, "pp_dispatch_layout: need E == D*m (E=%d D=%d m=%d)",
               E, D, m);
  PP_CHECK_ARG(my_rank >= 0 && my_rank < D, "pp_dispatch_layout: bad rank %d", my_rank);
  PP_CHECK_ARG(T % (m * PP_CHUNK) == 0, "pp_dispatch_layout: T=%d not a multiple of m*%d", T,
               PP_CHUNK);
  PP_CHECK_ARG(D <= 255, "pp_dispatch_layout: D=%d > 255", D);
  PP_CHECK_ARG(!counts_from_chunks || D == 1, "pp_dispatch_layout: counts_from_chunks needs D == 1");
  PP_CHECK_ARG(rows_capacity > 0 && num_slots >= 0 && max_groups >= 1, "pp_dispatch_layout: bad capacity");
  const size_t smem = layout_smem_bytes(D, m, E, T);
  PP_CHECK_ARG(smem <= 220 * 1024, "pp_dispatch_layout: E x E and T/128 x E staging too large");
  static int configured[64] = {0};  // per device: largest smem attribute set so far
  int dev = 0;
  PP_CUDA_TRY(cudaGetDevice(&dev));
  if (dev >= 64 || configured[dev] < (int)smem) {
    PP_CUDA_TRY(cudaFuncSetAttribute(dispatch_layout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     220 * 1024));
    if (dev < 64) configured[dev] = 220 * 1024;
  }
  PP_CUDA_TRY(pdl_launch(dispatch_layout_kernel, dim3(1), dim3(kLayoutThreads), smem, as_stream(stream), 
      counts, mask, chunk_counts, D, m, E, T, my_rank, max_groups, rows_capacity, num_slots, chunk_base,
      slot_dest, groups, num_groups, total_rows, seg_start, rep_slot, counts_from_chunks, replica_stats, status));
  PP_LAUNCH_CHECK();
  return PP_OK;
}

extern "C" int pp_dispatch(const void* x, const int32_t* idx, const int32_t* rank,
                           const int32_t* chunk_base, const int32_t* slot_dest, int32_t T,
                           int32_t d, int32_t k, int32_t m, int32_t E, void* const* recv_ptrs,
                           void* own_recv, const pp_group* groups, const int32_t* num_groups,
                           int32_t max_groups, int32_t* pair_dest, int32_t* pair_row,
                           void* const* origin_ptrs, int32_t my_rank, void* stream) {
  PP_CHECK_ARG(x && idx && rank && chunk_base && slot_dest && recv_ptrs && own_recv && groups &&
                   num_groups && pair_dest && pair_row,
               "pp_dispatch: null pointer");
  PP_CHECK_ARG(my_rank >= 0 && (int64_t)(my_rank + 1) * T * k < (1ll << 31), "pp_dispatch: bad my_rank");
  cudaStream_t st = as_stream(stream);
  PP_VPL_SWITCH(d, PP_CUDA_TRY(pdl_launch(dispatch_kernel<VPL>, dim3(grid_for_tokens(T)), dim3(256), 0, st, 
                       reinterpret_cast<const __nv_bfloat16*>(x), idx, rank, chunk_base,
                       slot_dest, T, d, k, m, E, recv_ptrs, pair_dest, pair_row, groups, num_groups,
                       reinterpret_cast<__nv_bfloat16*>(own_recv), origin_ptrs, my_rank)));
  PP_LAUNCH_CHECK();
  return PP_OK;
}

extern "C" int pp_combine(void* const* out_ptrs, const int32_t* pair_dest, const int32_t* pair_row,
                          const float* w, int32_t T, int32_t d, int32_t k, void* y, const void* comb,
                          void* stream) {
  PP_CHECK_ARG((out_ptrs || comb) && pair_dest && pair_row && w && y, "pp_combine: null pointer");
  PP_VPL_SWITCH(d, PP_CUDA_TRY(pdl_launch(combine_kernel<VPL>, dim3(grid_for_tokens(T)), dim3(256), 0, as_stream(stream), 
                       out_ptrs, pair_dest, pair_row, w, T, d, k,
                       reinterpret_cast<__nv_bfloat16*>(y), reinterpret_cast<const __nv_bfloat16*>(comb))));
  PP_LAUNCH_CHECK();
  return PP_OK;
}

extern "C" int pp_combine_bwd(const void* dy, void* const* out_ptrs, void* const* dgrad_ptrs,
                              void* own_dgrad, const int32_t* pair_dest, const int32_t* pair_row,
                              const float* w, const pp_group* groups, const int32_t* num_groups,
                              int32_t max_groups, int32_t T, int32_t d, int32_t k, float* dw,
                              const void* comb, const int32_t* idx, const float* probs, int32_t E,
                              int32_t EP, void* dl, void* stream) {
  PP_CHECK_ARG(dy && (out_ptrs || comb) && dgrad_ptrs && own_dgrad && pair_dest && pair_row && w &&
                   groups && num_groups && dw && idx && probs && dl,
               "pp_combine_bwd: null pointer");
  PP_CHECK_ARG(EP == 64 || EP == 128, "pp_combine_bwd: EP=%d must be 64 or 128", EP);
  PP_CHECK_ARG(E >= 1 && E <= EP && k >= 1 && k <= 8, "pp_combine_bwd: E=%d / k=%d", E, k);
  cudaStream_t st = as_stream(stream);
  auto* dlp = reinterpret_cast<__nv_bfloat16*>(dl);
  auto* ddy = reinterpret_cast<const __nv_bfloat16*>(dy);
  auto* own = reinterpret_cast<__nv_bfloat16*>(own_dgrad);
  auto* cb = reinterpret_cast<const __nv_bfloat16*>(comb);
  if (EP == 64) {
    PP_VPL_SWITCH(d, PP_CUDA_TRY(pdl_launch(combine_bwd_kernel<VPL, 64>, dim3(grid_for_tokens(T)), dim3(256), 0, st, 
                         ddy, out_ptrs, dgrad_ptrs, pair_dest, pair_row, w, T, d, k, dw, groups, num_groups,
                         own, cb, idx, probs, E, dlp)));
  } else {
    PP_VPL_SWITCH(d, PP_CUDA_TRY(pdl_launch(combine_bwd_kernel<VPL, 128>, dim3(grid_for_tokens(T)), dim3(256), 0, st, 
                         ddy, out_ptrs, dgrad_ptrs, pair_dest, pair_row, w, T, d, k, dw, groups, num_groups,
                         own, cb, idx, probs, E, dlp)));
  }
  PP_LAUNCH_CHECK();
  return PP_OK;
}

namespace pp {
int gate_dx_gemm(const void* dl, const void* wg, int T, int d, int E, int EP, void* dx, cudaStream_t st);

// dx[t] += sum_j dXp[pair(t, j)]: warp per token, 16-byte vectors, the k rows of two pairs
// in flight at a time (peer loads over NVLink), fp32 sum with the gate term already in dx
template <int VPL>
__global__ void __launch_bounds__(256)
    dispatch_bwd_kernel(void* const* dxp_ptrs, const __nv_bfloat16* __restrict__ comb,
                        const int32_t* __restrict__ pair_dest, const int32_t* __restrict__ pair_row,
                        int T, int d, int k, __nv_bfloat16* dx) {
  pdl_grid_sync();
  const int lane = threadIdx.x & 31;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp_global; t < T; t += nwarps) {
    int my_dest = -1, my_row = 0;
    if (lane < k) {
      my_dest = pair_dest[(size_t)t * k + lane];
      my_row = pair_row[(size_t)t * k + lane];
    }
    uint4* drow = reinterpret_cast<uint4*>(dx + (size_t)t * d);
    float acc[VPL][8];
#pragma unroll
    for (int i = 0; i < VPL; ++i) bf16x8_to_f32(ld_v4(drow + lane + 32 * i), acc[i]);
    for (int j0 = 0; j0 < k; j0 += 2) {
      uint4 v[2][VPL];
      int dest[2];
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int j = j0 + jj < k ? j0 + jj : j0;
        dest[jj] = __shfl_sync(0xffffffffu, my_dest, j);
        const int row = __shfl_sync(0xffffffffu, my_row, j);
        if (j0 + jj >= k) dest[jj] = -1;
        if (dest[jj] < 0) continue;
        const uint4* src = reinterpret_cast<const uint4*>(
            comb ? comb + (size_t)(t * k + j) * d
                 : reinterpret_cast<const __nv_bfloat16*>(dxp_ptrs[dest[jj]]) + (size_t)row * d);
#pragma unroll
        for (int i = 0; i < VPL; ++i) v[jj][i] = ld_v4(src + lane + 32 * i);
      }
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        if (dest[jj] < 0) continue;
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          float f[8];
          bf16x8_to_f32(v[jj][i], f);
#pragma unroll
          for (int u = 0; u < 8; ++u) acc[i][u] += f[u];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < VPL; ++i) st_v4(drow + lane + 32 * i, f32x8_to_bf16(acc[i]));
  }
}
int gate_dw_gemm(const void* dl, const void* x, int T, int d, int E, int EP, int split, float* ws,
                 float* dwg, cudaStream_t st);

// split-K chunk of the gate weight GEMM: ~one wave of (split, 128-row of d) tiles, a
// multiple of 128 that divides T
static int gate_dw_split(int T, int d) {
  const int want_splits = (148 + d / 128 - 1) / (d / 128);
  int split = 128;
  while (split * 2 <= T && T % (split * 2) == 0 && T / (split * 2) >= want_splits) split *= 2;
  return split;
}
}  // namespace pp

extern "C" int pp_gate_dx(const void* dl, const void* wg, int32_t T, int32_t d, int32_t E, int32_t EP, void* dx,
                          void* stream) {
  PP_CHECK_ARG(dl && wg && dx, "pp_gate_dx: null pointer");
  PP_CHECK_ARG(d % 256 == 0, "pp_gate_dx: d=%d must be a multiple of 256", d);
  PP_CHECK_ARG(T > 0 && T % PP_CHUNK == 0, "pp_gate_dx: T=%d must be a multiple of %d", T, PP_CHUNK);
  PP_CHECK_ARG((EP == 64 || EP == 128) && E >= 1 && E <= EP, "pp_gate_dx: bad E=%d/EP=%d", E, EP);
  return gate_dx_gemm(dl, wg, T, d, E, EP, dx, as_stream(stream));
}

extern "C" int pp_dispatch_bwd(void* const* dxp_ptrs, const void* comb, const int32_t* pair_dest,
                               const int32_t* pair_row, int32_t T, int32_t d, int32_t k, void* dx, void* stream) {
  PP_CHECK_ARG((dxp_ptrs || comb) && pair_dest && pair_row && dx, "pp_dispatch_bwd: null pointer");
  PP_CHECK_ARG(k >= 1 && k <= 8, "pp_dispatch_bwd: k=%d", k);
  cudaStream_t st = as_stream(stream);
  PP_VPL_SWITCH(d, PP_CUDA_TRY(pdl_launch(dispatch_bwd_kernel<VPL>, dim3(grid_for_tokens(T)), dim3(256), 0, st, 
                       dxp_ptrs, reinterpret_cast<const __nv_bfloat16*>(comb), pair_dest, pair_row, T, d, k,
                       reinterpret_cast<__nv_bfloat16*>(dx))));
  PP_LAUNCH_CHECK();
  return PP_OK;
}

extern "C" int64_t pp_gate_dw_workspace_bytes(int32_t T, int32_t d) {
  if (T <= 0 || T % PP_CHUNK || d <= 0 || d % 256) return -1;
  return (int64_t)(T / gate_dw_split(T, d)) * d * 128 * 4;  // [splits][d][EP <= 128] fp32
}

extern "C" int pp_gate_dw(const void* dl, const void* x, int32_t T, int32_t d, int32_t E, int32_t EP,
                          float* workspace, float* dwg, void* stream) {
  PP_CHECK_ARG(dl && x && workspace && dwg, "pp_gate_dw: null pointer");
  PP_CHECK_ARG(d % 256 == 0, "pp_gate_dw: d=%d must be a multiple of 256", d);
  PP_CHECK_ARG(T > 0 && T % PP_CHUNK == 0, "pp_gate_dw: T=%d must be a multiple of %d", T, PP_CHUNK);
  PP_CHECK_ARG((EP == 64 || EP == 128) && E >= 1 && E <= EP, "pp_gate_dw: bad E=%d/EP=%d", E, EP);
  return gate_dw_gemm(dl, x, T, d, E, EP, gate_dw_split(T, d), workspace, dwg, as_stream(stream));
}

// ---------------------------------------------------------------------------
// probe loss sum(a * b) over n bf16 elements in fp32: per-CTA partial sums in a fixed
// element order, then one CTA adds the partials in CTA order (deterministic; one HBM
// pass over both operands).
namespace pp {
constexpr int kDotCtas = 592;  // 4 per SM

__global__ void __launch_bounds__(512) dot_bf16_partial_kernel(const uint4* a, const uint4* b, int64_t nvec,
                                                               float* partial) {
  pdl_grid_sync();
  float s = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 x = ld_nc_v4(a + i), y = ld_nc_v4(b + i);
    const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 fx = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xs[j]));
      const float2 fy = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ys[j]));
      s = fmaf(fx.x, fy.x, s);
      s = fmaf(fx.y, fy.y, s);
    }
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ float ws[16];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    partial[blockIdx.x] = t;
  }
}

__global__ void dot_bf16_final_kernel(const float* partial, int n, float* out) {
  pdl_grid_sync();
  __shared__ float ws[32];
  float s = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += partial[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    *out = t;
  }
}
}  // namespace pp

extern "C" int pp_dot_bf16(const void* a, const void* b, int64_t n, float* partial, float* out,
                           void* stream) {
  PP_CHECK_ARG(a && b && partial && out, "pp_dot_bf16: null pointer");
  PP_CHECK_ARG(n >= 0 && n % 8 == 0, "pp_dot_bf16: n=%lld must be a multiple of 8", (long long)n);
  PP_CHECK_ARG(((uintptr_t)a | (uintptr_t)b) % 16 == 0, "pp_dot_bf16: operands must be 16-byte aligned");
  cudaStream_t st = as_stream(stream);
  PP_CUDA_TRY(pdl_launch(dot_bf16_partial_kernel, dim3(kDotCtas), dim3(512), 0, st, reinterpret_cast<const uint4*>(a),
                                                    reinterpret_cast<const uint4*>(b), n / 8, partial));
  PP_CUDA_TRY(pdl_launch(dot_bf16_final_kernel, dim3(1), dim3(1024), 0, st, partial, kDotCtas, out));
  PP_LAUNCH_CHECK();
  return PP_OK;
}
