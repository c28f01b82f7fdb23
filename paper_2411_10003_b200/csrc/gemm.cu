// K4: grouped expert GEMM on 5th-gen tensor cores (tcgen05 + TMA + TMEM), sm_100a.
//
// Stands in for the expert compute the reference only models: t_fec = max(H)/t and
// t_bec = 2 t_fec (pkg/src/moebal/perf_model.py:42-51).  One persistent kernel
// template serves every expert GEMM of the layer's fwd+bwd and the gate:
//
//   mode      A (smem major)          B (smem major)              C / epilogue
//   FWD1      Xp   [rows,d]  K        W1 [slot][f][d]  K          pre, act=GeLU(pre) bf16
//   FWD2      act  [rows,f]  K        W2 [slot][d][f]  K          Yp bf16
//   DGRAD2    dYp  [rows,d]  K        W2 [slot][d][f]  MN         dPre = acc*GeLU'(pre) bf16
//   DGRAD1    dPre [rows,f]  K        W1 [slot][f][d]  MN         dXp bf16
//   WGRAD2    dYp  [rows,d]  MN       act [rows,f]     MN         dW2[slot][d][f] fp32 (K = rows)
//   WGRAD1    dPre [rows,f]  MN       Xp  [rows,d]     MN         dW1[slot][f][d] fp32 (K = rows)
//   ROUTE     X    [T,d]     K        Wg [E][d]        K          softmax/top-k/chunk ranks (N = E)
//
// Groups (experts held by this rank) are ragged and read from device memory,
// so no host sync is needed between routing and the GEMMs.  Every group's
// row segment is padded to 128 rows with zeros (dispatch guarantees it), so
// M tiles never straddle groups and ragged-K wgrad needs no masking.
//
// Warp roles per CTA (256 threads, 1 CTA/SM, persistent over a static tile
// walk): warp0 = TMA producer, warp1 = MMA issuer (one thread), warp2 = TMEM
// allocator, warps4-7 = epilogue (TMEM lanes 32*(w%4)..+31).  Accumulators are
// double-buffered in TMEM so the epilogue of tile i overlaps the MMAs of i+1.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"

namespace pp {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one SWIZZLE_128B span
constexpr int kThreads = 256;
constexpr int kMaxGroups = 256;

enum Epi { EPI_BF16 = 0, EPI_GELU = 1, EPI_DGELU = 2, EPI_F32 = 3, EPI_ROUTE = 4 };

struct GemmParams {
  const pp_group* groups;
  const int32_t* num_groups;
  int max_groups;
  int M_fixed;  // wgrad: output rows per slot (d or f)
  int N;        // output columns
  int K_fixed;  // fwd/dgrad: reduction size
  int ragged_k; // 1 for wgrad
  void* c;
  void* c2;
  // route epilogue
  const float* bias;
  int32_t* idx;
  float* w;
  float* probs;
  int32_t* rank;
  int32_t* chunk_counts;
  int topk;
  int e_real;       // route: real expert count (<= BN; padded experts read as zero rows)
  int single_rows;  // > 0: one implicit group {row_off 0, rows_pad single_rows, slot 0}
};

struct SchedSmem {
  int32_t row_off[kMaxGroups];
  int32_t rows_pad[kMaxGroups];
  int32_t wslot[kMaxGroups];
  int32_t prefix[kMaxGroups + 1];
  int32_t G;
};

struct Tile {
  int m0, n0, num_kb, row_off, wslot;
};

// ---- UMMA descriptors ------------------------------------------------------
// smem matrix descriptor, SWIZZLE_128B, sm100 version=1
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

template <int N, bool A_MN, bool B_MN>
__host__ __device__ constexpr uint32_t make_idesc() {
  return (1u << 4)                    // D = f32
         | (1u << 7)                  // A = bf16
         | (1u << 10)                 // B = bf16
         | ((A_MN ? 1u : 0u) << 15)   // A major
         | ((B_MN ? 1u : 0u) << 16)   // B major
         | ((uint32_t)(N >> 3) << 17) // N
         | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ float gelu_f(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float u = k0 * (x + k1 * x * x * x);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  return 0.5f * x * (1.f + t);
}

__device__ __forceinline__ float dgelu_f(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float u = k0 * (x + k1 * x * x * x);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x * x);
}

template <int BN>
__device__ __forceinline__ bool decode_tile(int t, const SchedSmem& s, const GemmParams& p,
                                            Tile& tile) {
  // groups are few (<= experts of one rank); linear scan over the prefix
  int g = 0;
  while (g + 1 <= s.G && s.prefix[g + 1] <= t) ++g;
  if (g >= s.G) return false;
  const int local = t - s.prefix[g];
  const int nt = p.N / BN;
  tile.m0 = (local / nt) * BM;
  tile.n0 = (local % nt) * BN;
  tile.row_off = s.row_off[g];
  tile.wslot = s.wslot[g];
  tile.num_kb = p.ragged_k ? (s.rows_pad[g] / BK) : (p.K_fixed / BK);
  return true;
}

template <int BN, bool A_MN, bool B_MN, int EPI, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, const GemmParams p) {
  constexpr uint32_t A_BYTES = BM * BK * 2;
  constexpr uint32_t B_BYTES = BN * BK * 2;
  constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  constexpr uint32_t IDESC = make_idesc<BN, A_MN, B_MN>();

  extern __shared__ __align__(1024) uint8_t dsmem[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsmem) + 1023) & ~uintptr_t(1023));

  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2];
  __shared__ __align__(8) uint64_t tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ SchedSmem sched;
  __shared__ int32_t route_cnt[4][(EPI == EPI_ROUTE) ? BN : 1];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- schedule: copy the group table, build the tile prefix -------------
  if (threadIdx.x == 0 && p.single_rows > 0) {
    sched.G = 1;
    sched.row_off[0] = 0;
    sched.rows_pad[0] = p.single_rows;
    sched.wslot[0] = 0;
    sched.prefix[0] = 0;
    sched.prefix[1] = (p.single_rows / BM) * (p.N / BN);
  } else if (threadIdx.x == 0) {
    int G = *p.num_groups;
    if (G > p.max_groups) G = p.max_groups;
    if (G > kMaxGroups) G = kMaxGroups;
    sched.G = G;
    int acc = 0;
    const int nt = p.N / BN;
    for (int g = 0; g < G; ++g) {
      const pp_group gr = p.groups[g];
      sched.row_off[g] = gr.row_off;
      sched.rows_pad[g] = gr.rows_pad;
      sched.wslot[g] = gr.wslot;
      sched.prefix[g] = acc;
      acc += p.ragged_k ? (p.M_fixed / BM) * nt : (gr.rows_pad / BM) * nt;
    }
    sched.prefix[G] = acc;
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(&tmem_base_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;
  const int total_tiles = sched.prefix[sched.G];

  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      Tile tl;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        if (!decode_tile<BN>(t, sched, p, tl)) break;
        for (int kb = 0; kb < tl.num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          const int k0 = kb * BK;
          if constexpr (!A_MN) {
            tma_load_2d(sa, &tmA, &full_bar[stage], k0, tl.row_off + tl.m0);
          } else {
#pragma unroll
            for (int i = 0; i < BM / 64; ++i)
              tma_load_2d(sa + i * 8192, &tmA, &full_bar[stage], tl.m0 + 64 * i, tl.row_off + k0);
          }
          if constexpr (!B_MN) {
            tma_load_2d(sb, &tmB, &full_bar[stage], k0, tl.wslot * p.N + tl.n0);
          } else if (p.ragged_k) {  // wgrad: B rows are the group's token rows
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              tma_load_2d(sb + i * 8192, &tmB, &full_bar[stage], tl.n0 + 64 * i, tl.row_off + k0);
          } else {  // dgrad: B = W[slot] stored [K rows][N cols]
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              tma_load_2d(sb + i * 8192, &tmB, &full_bar[stage], tl.n0 + 64 * i,
                          tl.wslot * p.K_fixed + k0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    Tile tl;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      if (!decode_tile<BN>(t, sched, p, tl)) break;
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      if (tl.num_kb == 0) {
        if (lane == 0) mbar_arrive(&tfull_bar[acc]);
      }
      for (int kb = 0; kb < tl.num_kb; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = A_MN ? make_sdesc(sa + kk * 2048, 8192, 1024)
                                     : make_sdesc(sa + kk * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_sdesc(sb + kk * 2048, 8192, 1024)
                                     : make_sdesc(sb + kk * 32, 16, 1024);
            tc_mma_bf16(d_tmem, ad, bd, IDESC, (kb | kk) != 0);
          }
          tc_commit(&empty_bar[stage]);
          if (kb == tl.num_kb - 1) tc_commit(&tfull_bar[acc]);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue =================
    const int q = warp - 4;  // TMEM lane quarter
    const int r = q * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    Tile tl;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      if (!decode_tile<BN>(t, sched, p, tl)) break;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      const bool zero = tl.num_kb == 0;

      if constexpr (EPI == EPI_ROUTE) {
        // one thread = one token; logits row in registers
        const int E = p.e_real;
        float v[BN];
#pragma unroll
        for (int c = 0; c < BN; c += 16) {
          uint32_t raw[16];
          tmem_ld_32x32b_x16(t_row + c, raw);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) v[c + j] = __uint_as_float(raw[j]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[acc]);
        const int token = tl.row_off + tl.m0 + r;
        const int chunk = (tl.row_off + tl.m0) / BM;
#pragma unroll
        for (int e = 0; e < BN; ++e)
          v[e] = e < E ? v[e] + (p.bias ? p.bias[e] : 0.f) : -INFINITY;
        float mx = v[0];
#pragma unroll
        for (int e = 1; e < BN; ++e) mx = fmaxf(mx, v[e]);
        float ssum = 0.f;
        float ex[BN];
#pragma unroll
        for (int e = 0; e < BN; ++e) {
          ex[e] = e < E ? expf(v[e] - mx) : 0.f;
          ssum += ex[e];
        }
        const float inv = 1.f / ssum;
        float* prow = p.probs + (size_t)token * E;
#pragma unroll
        for (int e = 0; e < BN; e += 4)
          if (e < E)
            *reinterpret_cast<float4*>(prow + e) =
                make_float4(ex[e] * inv, ex[e + 1] * inv, ex[e + 2] * inv, ex[e + 3] * inv);
        // top-k on logits, ties -> lowest expert index
        uint64_t taken_lo = 0, taken_hi = 0;
        int sel[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          sel[j] = -1;
          if (j < p.topk) {
            int bi = -1;
            float best = 0.f;
#pragma unroll
            for (int e = 0; e < BN; ++e) {
              const bool tk = e < 64 ? ((taken_lo >> e) & 1) : ((taken_hi >> (e - 64)) & 1);
              if (e < E && !tk && (bi < 0 || v[e] > best)) {
                best = v[e];
                bi = e;
              }
            }
            sel[j] = bi;
            if (bi < 64) taken_lo |= 1ull << bi;
            else taken_hi |= 1ull << (bi - 64);
          }
        }
        // chunk ranks: pairs of expert e ordered by token inside this 128-token tile
        int myrank[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) myrank[j] = 0;
        const uint32_t lt_mask = (1u << lane) - 1u;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        for (int e = 0; e < E; ++e) {
          bool has = false;
#pragma unroll
          for (int j = 0; j < 8; ++j) has |= (sel[j] == e);
          const uint32_t b = __ballot_sync(0xffffffffu, has);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (sel[j] == e) myrank[j] = __popc(b & lt_mask);
          if (lane == 0) route_cnt[q][e] = __popc(b);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j < p.topk) {
            const int e = sel[j];
            int base = 0;
            for (int qq = 0; qq < q; ++qq) base += route_cnt[qq][e];
            p.idx[(size_t)token * p.topk + j] = e;
            p.w[(size_t)token * p.topk + j] = ex[e] * inv;
            p.rank[(size_t)token * p.topk + j] = base + myrank[j];
          }
        }
        for (int e = r; e < E; e += 128)
          p.chunk_counts[(size_t)chunk * E + e] =
              route_cnt[0][e] + route_cnt[1][e] + route_cnt[2][e] + route_cnt[3][e];
      } else {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t raw[32];
          if (!zero) {
            tmem_ld_32x32b_x32(t_row + c, raw);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) raw[j] = 0u;
          }
          if (c + 32 == BN) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty_bar[acc]);
          }
          if constexpr (EPI == EPI_F32) {
            float* out = reinterpret_cast<float*>(p.c) +
                         ((size_t)tl.wslot * p.M_fixed + tl.m0 + r) * p.N + tl.n0 + c;
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              st_v4(out + j, make_uint4(raw[j], raw[j + 1], raw[j + 2], raw[j + 3]));
          } else {
            const size_t row = (size_t)tl.row_off + tl.m0 + r;
            const size_t off = row * p.N + tl.n0 + c;
            if constexpr (EPI == EPI_BF16) {
              __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.c) + off;
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                float f[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) f[u] = __uint_as_float(raw[j + u]);
                st_v4(out + j, f32x8_to_bf16(f));
              }
            } else if constexpr (EPI == EPI_GELU) {
              __nv_bfloat16* pre = reinterpret_cast<__nv_bfloat16*>(p.c) + off;
              __nv_bfloat16* act = reinterpret_cast<__nv_bfloat16*>(p.c2) + off;
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                float f[8], g[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                  f[u] = __uint_as_float(raw[j + u]);
                  // GeLU of the bf16-rounded pre-activation, as the backward sees it
                  g[u] = gelu_f(__bfloat162float(__float2bfloat16_rn(f[u])));
                }
                st_v4(pre + j, f32x8_to_bf16(f));
                st_v4(act + j, f32x8_to_bf16(g));
              }
            } else if constexpr (EPI == EPI_DGELU) {
              const __nv_bfloat16* pre = reinterpret_cast<const __nv_bfloat16*>(p.c2) + off;
              __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.c) + off;
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                float x[8], f[8];
                bf16x8_to_f32(ld_v4(pre + j), x);
#pragma unroll
                for (int u = 0; u < 8; ++u) f[u] = __uint_as_float(raw[j + u]) * dgelu_f(x[u]);
                st_v4(out + j, f32x8_to_bf16(f));
              }
            }
          }
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_free<TMEM_COLS>(tmem_base);
}

// ---- host side -------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

static int get_encode() {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult qres;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qres) ==
            cudaSuccess &&
        qres == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode ? PP_OK : fail(PP_ECUDA, "cuTensorMapEncodeTiled unavailable");
}

// 2-D bf16 tensor [outer][inner] (inner contiguous), box [box_outer][box_inner], 128B swizzle
static int make_tmap(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                     uint32_t box_inner, uint32_t box_outer) {
  if (int rc = get_encode()) return rc;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(PP_ECUDA, "cuTensorMapEncodeTiled failed (%d) inner=%llu outer=%llu box=%ux%u",
                (int)r, (unsigned long long)inner, (unsigned long long)outer, box_inner,
                box_outer);
  return PP_OK;
}

template <int BN, bool A_MN, bool B_MN, int EPI, int STAGES>
static int launch(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, int grid,
                  cudaStream_t st) {
  auto kern = grouped_gemm_kernel<BN, A_MN, B_MN, EPI, STAGES>;
  const int smem = STAGES * (BM * BK * 2 + BN * BK * 2) + 1024;
  PP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<<<grid, kThreads, smem, st>>>(ta, tb, p);
  PP_LAUNCH_CHECK();
  return PP_OK;
}

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

int route_gemm(const void* x, const void* wg, const float* bias, int T, int d, int E, int k,
               int32_t* idx, float* w, float* probs, int32_t* rank, int32_t* chunk_counts,
               cudaStream_t st) {
  const int BNr = E <= 16 ? 16 : E <= 32 ? 32 : E <= 64 ? 64 : 128;
  CUtensorMap ta, tb;
  if (int rc = make_tmap(&ta, x, d, T, BK, BM)) return rc;
  if (int rc = make_tmap(&tb, wg, d, E, BK, BNr)) return rc;
  GemmParams p{};
  p.max_groups = 1;
  p.single_rows = T;
  p.e_real = E;
  p.K_fixed = d;
  p.bias = bias;
  p.idx = idx;
  p.w = w;
  p.probs = probs;
  p.rank = rank;
  p.chunk_counts = chunk_counts;
  p.topk = k;
  p.N = BNr;
  const int grid = sm_count();
  switch (BNr) {
    case 16: return launch<16, false, false, EPI_ROUTE, 8>(ta, tb, p, grid, st);
    case 32: return launch<32, false, false, EPI_ROUTE, 8>(ta, tb, p, grid, st);
    case 64: return launch<64, false, false, EPI_ROUTE, 8>(ta, tb, p, grid, st);
    case 128: return launch<128, false, false, EPI_ROUTE, 6>(ta, tb, p, grid, st);
    default: return fail(PP_EINVAL, "route: E=%d unsupported by the tcgen05 gate", E);
  }
}

}  // namespace pp

using namespace pp;

extern "C" int pp_grouped_gemm(int32_t mode, const void* a, const void* b, void* c, void* c2,
                               const pp_group* groups, const int32_t* num_groups,
                               int32_t max_groups, int32_t rows_capacity, int32_t num_slots,
                               int32_t d_model, int32_t d_ff, int32_t num_sms, void* stream) {
  PP_CHECK_ARG(a && b && c && groups && num_groups, "pp_grouped_gemm: null pointer");
  PP_CHECK_ARG(max_groups >= 1 && max_groups <= kMaxGroups, "pp_grouped_gemm: max_groups=%d",
               max_groups);
  PP_CHECK_ARG(rows_capacity > 0 && rows_capacity % BM == 0,
               "pp_grouped_gemm: rows_capacity must be a positive multiple of %d", BM);
  PP_CHECK_ARG(d_model % 256 == 0 && d_ff % 256 == 0,
               "pp_grouped_gemm: d_model and d_ff must be multiples of 256");
  cudaStream_t st = as_stream(stream);
  const int grid = num_sms > 0 ? num_sms : sm_count();
  const int R = rows_capacity, S = num_slots, dm = d_model, df = d_ff;
  CUtensorMap ta, tb;
  GemmParams p{};
  p.groups = groups;
  p.num_groups = num_groups;
  p.max_groups = max_groups;
  p.c = c;
  p.c2 = c2;
  int rc = PP_OK;
  switch (mode) {
    case PP_GEMM_FWD1:
      PP_CHECK_ARG(c2, "FWD1 needs the act output");
      if ((rc = make_tmap(&ta, a, dm, R, BK, BM)) || (rc = make_tmap(&tb, b, dm, (uint64_t)S * df, BK, 256))) return rc;
      p.N = df; p.K_fixed = dm;
      return launch<256, false, false, EPI_GELU, 4>(ta, tb, p, grid, st);
    case PP_GEMM_FWD2:
      if ((rc = make_tmap(&ta, a, df, R, BK, BM)) || (rc = make_tmap(&tb, b, df, (uint64_t)S * dm, BK, 256))) return rc;
      p.N = dm; p.K_fixed = df;
      return launch<256, false, false, EPI_BF16, 4>(ta, tb, p, grid, st);
    case PP_GEMM_DGRAD2:
      PP_CHECK_ARG(c2, "DGRAD2 needs the pre-activation");
      if ((rc = make_tmap(&ta, a, dm, R, BK, BM)) || (rc = make_tmap(&tb, b, df, (uint64_t)S * dm, 64, BK))) return rc;
      p.N = df; p.K_fixed = dm;
      return launch<256, false, true, EPI_DGELU, 4>(ta, tb, p, grid, st);
    case PP_GEMM_DGRAD1:
      if ((rc = make_tmap(&ta, a, df, R, BK, BM)) || (rc = make_tmap(&tb, b, dm, (uint64_t)S * df, 64, BK))) return rc;
      p.N = dm; p.K_fixed = df;
      return launch<256, false, true, EPI_BF16, 4>(ta, tb, p, grid, st);
    case PP_GEMM_WGRAD2:
      if ((rc = make_tmap(&ta, a, dm, R, 64, BK)) || (rc = make_tmap(&tb, b, df, R, 64, BK))) return rc;
      p.M_fixed = dm; p.N = df; p.ragged_k = 1;
      return launch<256, true, true, EPI_F32, 4>(ta, tb, p, grid, st);
    case PP_GEMM_WGRAD1:
      if ((rc = make_tmap(&ta, a, df, R, 64, BK)) || (rc = make_tmap(&tb, b, dm, R, 64, BK))) return rc;
      p.M_fixed = df; p.N = dm; p.ragged_k = 1;
      return launch<256, true, true, EPI_F32, 4>(ta, tb, p, grid, st);
    case PP_GEMM_PLAIN:
      if ((rc = make_tmap(&ta, a, dm, R, BK, BM)) || (rc = make_tmap(&tb, b, dm, (uint64_t)S * df, BK, 256))) return rc;
      p.N = df; p.K_fixed = dm;
      return launch<256, false, false, EPI_BF16, 4>(ta, tb, p, grid, st);
    default:
      return fail(PP_EINVAL, "pp_grouped_gemm: unknown mode %d", mode);
  }
}
