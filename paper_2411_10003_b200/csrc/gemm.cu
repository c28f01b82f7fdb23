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
#include <unordered_map>
#include <cstdlib>

#include "common.cuh"

namespace pp {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one SWIZZLE_128B span
constexpr int kThreads = 384;  // 4 non-epilogue warps + up to 8 epilogue warps
constexpr int kMaxGroups = 256;
constexpr int kTraceSteps = 1024;


enum Epi { EPI_BF16 = 0, EPI_GELU = 1, EPI_DGELU = 2, EPI_F32 = 3 };

// per-epilogue-warp staging for the TMA-store epilogue: a ring of out_bufs 32x32
// blocks (bf16: 2 KB, SWIZZLE_64B; fp32: one 4 KB block, SWIZZLE_128B), so a warp
// stages the next block while up to out_bufs-1 earlier TMA stores still read theirs;
// DGELU / BF16_ADD put a 2 KB block for the TMA-loaded operand in front of the ring.
// The short-K GEMMs with heavy epilogues (FWD1: two outputs + GeLU; DGRAD2: operand
// load + GeLU') get deeper rings; the long-K ones keep one block and more stages.
template <int EPI>
constexpr int out_bufs() {
  return EPI == EPI_GELU ? 3 : EPI == EPI_DGELU ? 2 : 1;
}
template <int EPI>
constexpr int out_base() {
  return EPI == EPI_DGELU ? 2048 : 0;
}
template <int EPI>
constexpr int stage_bytes_per_warp() {
  return EPI == EPI_F32 ? 4096 : out_base<EPI>() + out_bufs<EPI>() * 2048;
}

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
  int single_rows;  // > 0: implicit groups over rows [0, single_rows), slot 0
  int split_rows;   // with single_rows: split-K chunk size (one implicit group per chunk)
  unsigned long long* dbg;  // optional per-CTA wait-cycle counters (PPMOE_GEMM_DEBUG)
  // PPMOE_GEMM_DEBUG=2: per-k-step globaltimer trace of CTAs 0..3 (first kTraceSteps steps):
  // [cta][step][0..1] producer before/after the empty wait, [2..3] MMA before/after the full wait
  unsigned long long* trace;
  // fused combine / dispatch-backward (EPI_BF16 only): output row r goes to pair
  // origin[r] = src_rank * pairs_per_rank + t*k + j, i.e. row (t*k+j) of scatter_ptrs[src_rank]
  // (peer memory over NVLink), instead of this rank's receive-layout buffer; origin < 0
  // marks padding rows (not stored)
  const int32_t* origin;
  void* const* scatter_ptrs;
  int scatter_tk;
  // replica gate (FWD1 while Trans is in flight): groups with wslot >= gate_slot0 are
  // scheduled after the home groups and their B loads wait until every peer's Trans
  // completion flag gate_flags[r] (r != gate_me) reaches *gate_epoch
  const uint64_t* gate_flags;
  const uint64_t* gate_epoch;
  int gate_me, gate_D, gate_slot0;
  // FWD1: GeLU in packed bf16x2 arithmetic (on the bf16 pre-activation).  DGRAD2's GeLU' stays
  // fp32: in bf16, 1 - tanh^2 cancels where the tanh saturates (measured dW1 error 1.1 % vs 0.3 %
  // at 4x-scaled weights in the EP parity runs)
  int fast_gelu;
  // device-adaptive SM reservation: the persistent walk leaves
  // clamp(res_per_unit * (res_stats[0] + (res_both ? res_stats[1] : 0)), res_lo, res_hi) SMs
  // to concurrent side kernels (Trans / Agg), sized by this iteration's replica volume
  const int32_t* res_stats;
  int res_both, res_per_unit, res_lo, res_hi;
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
  bool active;  // CTA pairs: false when this CTA's 128-row half lies past the group's rows
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

template <int N, bool A_MN, bool B_MN, int M = BM>
__host__ __device__ constexpr uint32_t make_idesc() {
  return (1u << 4)                    // D = f32
         | (1u << 7)                  // A = bf16
         | (1u << 10)                 // B = bf16
         | ((A_MN ? 1u : 0u) << 15)   // A major
         | ((B_MN ? 1u : 0u) << 16)   // B major
         | ((uint32_t)(N >> 3) << 17) // N
         | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ float gelu_f(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float u = k0 * (x + k1 * x * x * x);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  return 0.5f * x * (1.f + t);
}

// GeLU of two bf16 values in packed bf16x2 arithmetic (HFMA2.BF16 + MUFU.TANH.BF16x2): half the
// FP32-pipe and MUFU work of gelu_f per element, ~1 bf16 ulp more error
__device__ __forceinline__ uint32_t gelu_bf16x2(uint32_t xv) {
  const __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(&xv);
  const __nv_bfloat162 c0 = __float2bfloat162_rn(0.7978845608028654f);
  const __nv_bfloat162 c1 = __float2bfloat162_rn(0.7978845608028654f * 0.044715f);
  const __nv_bfloat162 half = __float2bfloat162_rn(0.5f);
  const __nv_bfloat162 u = __hmul2(x, __hfma2(__hmul2(x, x), c1, c0));
  uint32_t ur = *reinterpret_cast<const uint32_t*>(&u), tr;
  asm("tanh.approx.bf16x2 %0, %1;" : "=r"(tr) : "r"(ur));
  const __nv_bfloat162 t = *reinterpret_cast<const __nv_bfloat162*>(&tr);
  const __nv_bfloat162 hx = __hmul2(x, half);
  const __nv_bfloat162 g = __hfma2(hx, t, hx);
  return *reinterpret_cast<const uint32_t*>(&g);
}

__device__ __forceinline__ float dgelu_f(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float u = k0 * (x + k1 * x * x * x);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x * x);
}

// Tile t of the static walk -> (group, rows, cols).  With CTA pairs (CG = 2) a
// tile is 256 x BN: CTA rank r of the pair owns rows [m0_pair + 128 r, +128).
template <int BN, int CG>
__device__ __forceinline__ bool decode_tile(int t, const SchedSmem& s, const GemmParams& p,
                                            Tile& tile, int cta_rank) {
  // groups are few (<= experts of one rank); linear scan over the prefix
  int g = 0;
  while (g + 1 <= s.G && s.prefix[g + 1] <= t) ++g;
  if (g >= s.G) return false;
  const int local = t - s.prefix[g];
  const int nt = p.N / BN;
  tile.m0 = (local / nt) * (BM * CG) + BM * cta_rank;
  tile.n0 = (local % nt) * BN;
  tile.row_off = s.row_off[g];
  tile.wslot = s.wslot[g];
  tile.num_kb = p.ragged_k ? (s.rows_pad[g] / BK) : (p.K_fixed / BK);
  tile.active = p.ragged_k ? true : (tile.m0 < s.rows_pad[g]);
  return true;
}

template <int EPI>
constexpr bool tma_out() {
  return EPI == EPI_BF16 || EPI == EPI_GELU || EPI == EPI_DGELU || EPI == EPI_F32;
}

// Stage a 32x32 bf16 block (row = lane, 16-byte chunk j) with the SWIZZLE_64B
// pattern the output tensor map uses, then one lane TMA-stores it.  The
// staging buffer is reused only after the previous store finished reading it.
template <int PENDING = 0>
__device__ __forceinline__ void stage_and_store(uint8_t* stage, const uint4 (&v)[4], const void* tmap,
                                                int col, int row, int lane) {
  if (lane == 0) bulk_wait_read<PENDING>();
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 4; ++j)
    *reinterpret_cast<uint4*>(stage + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) = v[j];
  fence_async_shared();
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(tmap, stage, col, row);
    bulk_commit();
  }
}

// fp32 variant: 32 rows x 128 B, SWIZZLE_128B (16-byte chunk j of row l at j ^ (l & 7))
__device__ __forceinline__ void stage_and_store_f32(uint8_t* stage, const uint32_t (&raw)[32],
                                                    const void* tmap, int col, int row, int lane) {
  if (lane == 0) bulk_wait_read0();
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 8; ++j)
    *reinterpret_cast<uint4*>(stage + lane * 128 + ((j ^ (lane & 7)) << 4)) =
        make_uint4(raw[4 * j], raw[4 * j + 1], raw[4 * j + 2], raw[4 * j + 3]);
  fence_async_shared();
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(tmap, stage, col, row);
    bulk_commit();
  }
}

// Epilogue of one 32-column chunk of one accumulator row (thread = row r).
template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const uint32_t (&raw)[32], const GemmParams& p,
                                               const Tile& tl, int r, int c, const uint4 (&pre_v)[4],
                                               uint8_t* stage, int& sbuf, const CUtensorMap* tmC,
                                               const CUtensorMap* tmC2, int lane) {
  constexpr int NB = out_bufs<EPI>();
  auto next_buf = [&]() -> uint8_t* {  // ring slot for the next staged 32x32 bf16 block
    uint8_t* b = stage + out_base<EPI>() + sbuf * 2048;
    if (++sbuf == NB) sbuf = 0;
    return b;
  };
  if constexpr (EPI == EPI_F32) {
    stage_and_store_f32(stage, raw, tmC, tl.n0 + c, tl.wslot * p.M_fixed + tl.m0 + (r & ~31), lane);
  } else {  // bf16 outputs: TMA-store (or LSU) epilogue
    const int col = tl.n0 + c;
    const int row = tl.row_off + tl.m0 + (r & ~31);
    // one 32x32 bf16 output block of this warp: TMA store from the ring
    auto put = [&](const uint4 (&blk)[4], const CUtensorMap* tm) {
      stage_and_store<NB - 1>(next_buf(), blk, tm, col, row, lane);
    };
    uint4 v[4];
    if constexpr (EPI == EPI_BF16) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float f[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) f[u] = __uint_as_float(raw[8 * j + u]);
        v[j] = f32x8_to_bf16(f);
      }
      if (p.origin) {
        // fused A2A: this thread's 64 B of row r go to the pair's owner as one bulk copy
        // (TMA engine, smem -> local or peer global), so the LSUs stay with the epilogue
        const int o = p.origin[tl.row_off + tl.m0 + r];
        uint8_t* buf = next_buf() + lane * 64;
        bulk_wait_read<NB - 1>();  // this lane's previous copy out of the slot has read it
#pragma unroll
        for (int j = 0; j < 4; ++j) *reinterpret_cast<uint4*>(buf + 16 * j) = v[j];
        fence_async_shared();
        if (o >= 0) {
          const int src = o / p.scatter_tk;
          bulk_store_s2g(reinterpret_cast<__nv_bfloat16*>(p.scatter_ptrs[src]) +
                             (size_t)(o - src * p.scatter_tk) * p.N + col, buf, 64);
        }
        bulk_commit();
      } else {
        put(v, tmC);
      }
    } else if constexpr (EPI == EPI_GELU) {
      uint4 g4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float f[8], g[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) f[u] = __uint_as_float(raw[8 * j + u]);
        v[j] = f32x8_to_bf16(f);
        if (p.fast_gelu) {  // packed bf16x2 GeLU of the bf16 pre-activation
          g4[j] = make_uint4(gelu_bf16x2(v[j].x), gelu_bf16x2(v[j].y), gelu_bf16x2(v[j].z), gelu_bf16x2(v[j].w));
          continue;
        }
        bf16x8_to_f32(v[j], f);  // GeLU of the bf16-rounded pre-activation, as the backward sees it
#pragma unroll
        for (int u = 0; u < 8; ++u) g[u] = gelu_f(f[u]);
        g4[j] = f32x8_to_bf16(g);
      }
      put(v, tmC);
      put(g4, tmC2);
    } else {  // EPI_DGELU: acc * GeLU'(pre)   (operand TMA-loaded)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float x[8], f[8];
        bf16x8_to_f32(pre_v[j], x);
#pragma unroll
        for (int u = 0; u < 8; ++u) f[u] = __uint_as_float(raw[8 * j + u]) * dgelu_f(x[u]);
        v[j] = f32x8_to_bf16(f);
      }
      put(v, tmC);
    }
  }
}

// Tile table of the persistent walk (thread 0): the group list (or the implicit groups of a
// single-matrix / split-K launch) and the tile prefix.  Gated launches put the home groups first
// (their replica tiles wait on Trans); ragged-K (wgrad) groups are sorted by K descending.
template <int BN, int CG>
__device__ __forceinline__ void build_schedule(const GemmParams& p, SchedSmem& sched) {
  if (p.single_rows > 0) {
    const int chunk = p.split_rows > 0 ? p.split_rows : p.single_rows;
    const int G = p.single_rows / chunk;
    const int nt = p.N / BN;
    sched.G = G;
    for (int g = 0; g <= G; ++g) {
      if (g < G) {
        sched.row_off[g] = g * chunk;
        sched.rows_pad[g] = chunk;
        sched.wslot[g] = g;  // split-K: partial g goes to its own output slice (EPI_F32)
      }
      sched.prefix[g] = g * (p.ragged_k ? (p.M_fixed / (BM * CG)) * nt : ((chunk + BM * CG - 1) / (BM * CG)) * nt);
    }
  } else {
    int G = *p.num_groups;
    if (G > p.max_groups) G = p.max_groups;
    if (G > kMaxGroups) G = kMaxGroups;
    sched.G = G;
    int acc = 0;
    const int nt = p.N / BN;
    int next_home = 0;
    if (p.gate_flags && !p.ragged_k)  // home groups first: the gated replica tiles go last
      for (int g = 0; g < G; ++g) next_home += p.groups[g].wslot < p.gate_slot0;
    int next_rep = next_home;
    next_home = 0;
    for (int g = 0; g < G; ++g) {
      const pp_group gr = p.groups[g];
      // ragged-K (wgrad): keep groups sorted by K descending so the static
      // round-robin tile walk hands out the long tiles first (LPT balance)
      int pos = g;
      if (p.gate_flags && !p.ragged_k) pos = gr.wslot < p.gate_slot0 ? next_home++ : next_rep++;
      if (p.ragged_k) {
        while (pos > 0 && sched.rows_pad[pos - 1] < gr.rows_pad) {
          sched.row_off[pos] = sched.row_off[pos - 1];
          sched.rows_pad[pos] = sched.rows_pad[pos - 1];
          sched.wslot[pos] = sched.wslot[pos - 1];
          --pos;
        }
      }
      sched.row_off[pos] = gr.row_off;
      sched.rows_pad[pos] = gr.rows_pad;
      sched.wslot[pos] = gr.wslot;
    }
    for (int g = 0; g < G; ++g) {
      sched.prefix[g] = acc;
      acc += p.ragged_k ? (p.M_fixed / (BM * CG)) * nt : ((sched.rows_pad[g] + BM * CG - 1) / (BM * CG)) * nt;
    }
    sched.prefix[G] = acc;
  }
}

template <int BN, bool A_MN, bool B_MN, int EPI, int STAGES, int CG>
__global__ void __launch_bounds__(kThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmC,
                        const __grid_constant__ CUtensorMap tmC2, const GemmParams p) {
  pdl_grid_sync();
  // CG = 2: CTA pair (cta_group::2).  Each CTA stages its 128 rows of A and its
  // half (BN/2 rows) of B; the leader issues 256 x BN MMAs over both CTAs' smem.
  static_assert(CG == 1 || CG == 2, "CG");
  constexpr int BNC = BN / CG;  // B rows staged by this CTA
  constexpr uint32_t A_BYTES = BM * BK * 2;
  constexpr uint32_t B_BYTES = BNC * BK * 2;
  constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  // BN = 512 (CTA pairs, long-K modes): a 256 x 512 tile is two N = 256 MMAs per K step that
  // share the A operand -- 25 % fewer operand bytes per FLOP for a feed-bound mainloop -- and
  // fills all 512 TMEM columns, so the accumulator is single-buffered
  constexpr int NSUB = BN > 256 ? 2 : 1;      // MMAs per K step (N halves)
  constexpr int BN_MMA = BN / NSUB;
  constexpr int NACC = (2 * BN <= 512) ? 2 : 1;  // TMEM accumulator buffers
  constexpr uint32_t TMEM_COLS = (NACC * BN <= 32) ? 32 : (NACC * BN <= 64) ? 64 : (NACC * BN <= 128) ? 128
                                 : (NACC * BN <= 256) ? 256 : 512;
  static_assert(NACC * BN <= 512, "TMEM holds 512 fp32 columns");
  static_assert(NSUB == 1 || CG == 2, "BN = 512 tiles are CTA-pair only");
  constexpr uint32_t IDESC = make_idesc<BN_MMA, A_MN, B_MN, BM * CG>();  // pair: M = 256
  // epilogue warps: two per TMEM lane quarter (each takes half of the columns) for BN >= 128
  constexpr int EPI_WARPS = BN >= 128 ? 8 : 4;
  constexpr int EPI_COLS = BN * 4 / EPI_WARPS;

  extern __shared__ __align__(1024) uint8_t dsmem[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsmem) + 1023) & ~uintptr_t(1023));

  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2];
  __shared__ __align__(8) uint64_t tempty_bar[2];
  __shared__ __align__(8) uint64_t pre_bar[8];  // DGELU: per-epilogue-warp pre-activation loads
  __shared__ uint32_t tmem_base_sh;
  __shared__ SchedSmem sched;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- schedule: copy the group table, build the tile prefix -------------
  if (threadIdx.x == 0) build_schedule<BN, CG>(p, sched);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if constexpr (tma_out<EPI>()) {
      tma_prefetch_desc(&tmC);
      if constexpr (EPI == EPI_GELU) tma_prefetch_desc(&tmC2);
    }
  }
  const int cta_rank = CG == 2 ? (int)cluster_ctarank() : 0;
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full_bar[i], 1);  // pair: the leader's arrive.expect_tx covers both CTAs' bytes
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], EPI_WARPS * CG);  // pair: both CTAs' epilogues drain
    }
    for (int i = 0; i < 8; ++i) mbar_init(&pre_bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 2) {
    if constexpr (CG == 2) tmem_alloc_2sm<TMEM_COLS>(&tmem_base_sh);
    else tmem_alloc<TMEM_COLS>(&tmem_base_sh);
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;
  const int total_tiles = sched.prefix[sched.G];
  // Static persistent walk.  Ragged-K (wgrad) tiles are sorted by K descending
  // and dealt in snake order (0..G-1, G-1..0, ...) so long tiles spread evenly.
  const bool snake = p.ragged_k != 0;
  int G_walk = (int)gridDim.x / CG;  // one walk per CTA pair
  if (p.res_stats) {
    int r = p.res_per_unit * (p.res_stats[0] + (p.res_both ? p.res_stats[1] : 0));
    r = r < p.res_lo ? p.res_lo : (r > p.res_hi ? p.res_hi : r);
    G_walk = max(1, G_walk - (r + CG - 1) / CG);
  }
  auto tile_of = [&](int it) -> int {
    const int G = G_walk, b = (int)blockIdx.x / CG;
    if (b >= G) return total_tiles;  // reserved: no tiles, the CTA exits after the prologue
    return it * G + ((snake && (it & 1)) ? (G - 1 - b) : b);
  };

  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      bool gate_pending = p.gate_flags != nullptr;
      int pstep = 0;  // trace index
      Tile tl;
      for (int it = 0, t = tile_of(0); t < total_tiles; t = tile_of(++it)) {
        if (!decode_tile<BN, CG>(t, sched, p, tl, cta_rank)) break;
        if (gate_pending && tl.wslot >= p.gate_slot0) {  // first replica tile: Trans must have landed
          const uint64_t e = *p.gate_epoch;
          const uint64_t t0 = globaltimer_ns();
          bool timed_out = false;
          for (int r = 0; r < p.gate_D && !timed_out; ++r) {
            if (r == p.gate_me) continue;
            while (ld_acquire_sys_u64(p.gate_flags + r) < e) {
              if (globaltimer_ns() - t0 > 20ull * 1000 * 1000 * 1000) {
                // a pusher never signalled (crashed peer): record the fault next to the epoch
                // (the host raises on it) and finish instead of hanging or killing the context
                printf("ppmoe: replica gate timeout (rank %d waiting on %d)\n", p.gate_me, r);
                const_cast<uint64_t*>(p.gate_epoch)[1] = 1;
                timed_out = true;
                break;
              }
            }
          }
          fence_proxy_async_global();
          gate_pending = false;
        }
        for (int kb = 0; kb < tl.num_kb; ++kb) {
          const bool tr = p.trace && blockIdx.x < 4 && pstep < kTraceSteps;
          if (tr) p.trace[((size_t)blockIdx.x * kTraceSteps + pstep) * 4 + 0] = globaltimer_ns();
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (tr) p.trace[((size_t)blockIdx.x * kTraceSteps + pstep) * 4 + 1] = globaltimer_ns();
          ++pstep;
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          const int k0 = kb * BK;
          // B columns staged by this CTA: for each N half s (one MMA), the pair splits the
          // half's BN_MMA columns, this CTA taking [s*BN_MMA + rank*BNC/NSUB, +BNC/NSUB)
          auto bcol = [&](int j) {  // tile-relative column of this CTA's staged B row/col j
            constexpr int H = BNC / NSUB;
            return tl.n0 + (j / H) * BN_MMA + cta_rank * H + (j % H);
          };
          // all TMA of the stage completes on the leader CTA's full barrier
          const uint32_t bar_c = CG == 2 ? mapa_shared(smem_u32(&full_bar[stage]), 0) : 0u;
          auto load = [&](void* dst, const CUtensorMap* m, int c0, int c1) {
            if constexpr (CG == 2) tma_load_2d_2sm(dst, m, bar_c, c0, c1);
            else tma_load_2d(dst, m, &full_bar[stage], c0, c1);
          };
          // pair: only the leader arms the barrier (both CTAs' bytes); the peer's
          // TMA complete_tx may land first -- the phase cannot complete before the
          // leader's arrive, and the peer only refills a stage after the MMAs that
          // consumed it committed, so transactions never cross phases
          if (CG == 1 || cta_rank == 0) mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES * CG);
          if constexpr (!A_MN) {
            load(sa, &tmA, k0, tl.row_off + tl.m0);
          } else {
#pragma unroll
            for (int i = 0; i < BM / 64; ++i) load(sa + i * 8192, &tmA, tl.m0 + 64 * i, tl.row_off + k0);
          }
          if constexpr (!B_MN) {  // K-major B: one box of BNC/NSUB rows per N half
#pragma unroll
            for (int s = 0; s < NSUB; ++s)
              load(sb + s * (BNC / NSUB) * 128, &tmB, k0, tl.wslot * p.N + bcol(s * (BNC / NSUB)));
          } else if (p.ragged_k) {  // wgrad: B rows are the group's token rows
#pragma unroll
            for (int i = 0; i < BNC / 64; ++i) load(sb + i * 8192, &tmB, bcol(64 * i), tl.row_off + k0);
          } else {  // dgrad: B = W[slot] stored [K rows][N cols]
#pragma unroll
            for (int i = 0; i < BNC / 64; ++i)
              load(sb + i * 8192, &tmB, bcol(64 * i), tl.wslot * p.K_fixed + k0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1 && cta_rank == 0) {
    // ================= MMA issuer (leader CTA of a pair) =================
    long long wait_tempty = 0, wait_full = 0, t_start = p.dbg ? clock64() : 0;
    int mstep = 0;  // trace index
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    Tile tl;
    for (int it = 0, t = tile_of(0); t < total_tiles; t = tile_of(++it)) {
      if (!decode_tile<BN, CG>(t, sched, p, tl, cta_rank)) break;
      long long w0 = p.dbg ? clock64() : 0;
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      if (p.dbg) wait_tempty += clock64() - w0;
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      if (tl.num_kb == 0) {  // empty wgrad group: nothing to accumulate, epilogues write zeros
        if (lane == 0) {
          mbar_arrive(&tfull_bar[acc]);
          if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(smem_u32(&tfull_bar[acc]), 1));
        }
      }
      for (int kb = 0; kb < tl.num_kb; ++kb) {
        long long w1 = p.dbg ? clock64() : 0;
        const bool tr = p.trace && blockIdx.x < 4 && mstep < kTraceSteps && lane == 0;
        if (tr) p.trace[((size_t)blockIdx.x * kTraceSteps + mstep) * 4 + 2] = globaltimer_ns();
        mbar_wait(&full_bar[stage], phase);
        if (tr) p.trace[((size_t)blockIdx.x * kTraceSteps + mstep) * 4 + 3] = globaltimer_ns();
        ++mstep;
        if (p.dbg) wait_full += clock64() - w1;
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = A_MN ? make_sdesc(sa + kk * 2048, 8192, 1024)
                                     : make_sdesc(sa + kk * 32, 16, 1024);
#pragma unroll
            for (int s = 0; s < NSUB; ++s) {
              // N half s: this CTA's B rows [s*BNC/NSUB, +BNC/NSUB) (K-major: 128 B per row;
              // MN-major: 8 KB per 64-column chunk) into TMEM columns [s*BN_MMA, +BN_MMA)
              const uint32_t sbs = sb + s * (B_MN ? (BNC / NSUB / 64) * 8192 : (BNC / NSUB) * 128);
              const uint64_t bd = B_MN ? make_sdesc(sbs + kk * 2048, 8192, 1024)
                                       : make_sdesc(sbs + kk * 32, 16, 1024);
              if constexpr (CG == 2) tc_mma_bf16_2sm(d_tmem + s * BN_MMA, ad, bd, IDESC, (kb | kk) != 0);
              else tc_mma_bf16(d_tmem + s * BN_MMA, ad, bd, IDESC, (kb | kk) != 0);
            }
          }
          if constexpr (CG == 2) {
            tc_commit_2sm(&empty_bar[stage], 0x3);
            if (kb == tl.num_kb - 1) tc_commit_2sm(&tfull_bar[acc], 0x3);
          } else {
            tc_commit(&empty_bar[stage]);
            if (kb == tl.num_kb - 1) tc_commit(&tfull_bar[acc]);
          }
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (++acc == NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (p.dbg && lane == 0) {
      p.dbg[blockIdx.x * 4 + 0] = (unsigned long long)(clock64() - t_start);
      p.dbg[blockIdx.x * 4 + 1] = (unsigned long long)wait_tempty;
      p.dbg[blockIdx.x * 4 + 2] = (unsigned long long)wait_full;
    }
  } else if (warp >= 4 && warp < 4 + EPI_WARPS) {
    // ================= epilogue =================
    const int q = warp & 3;                  // TMEM lane quarter (hardware: warp % 4)
    const int col0 = ((warp - 4) >> 2) * EPI_COLS;  // column slice of this warp
    uint8_t* stage = smem + STAGES * STAGE_BYTES + (warp - 4) * stage_bytes_per_warp<EPI>();
    uint32_t pre_phase = 0;  // DGELU: parity of this warp's pre-activation TMA barrier
    int sbuf = 0;            // ring slot of the next staged output block
    const int r = q * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    Tile tl;
    for (int it = 0, t = tile_of(0); t < total_tiles; t = tile_of(++it)) {
      if (!decode_tile<BN, CG>(t, sched, p, tl, cta_rank)) break;
      if constexpr (EPI == EPI_DGELU) {  // first operand block, in flight during the MMAs
        if (lane == 0 && tl.active) {
          mbar_arrive_expect_tx(&pre_bar[warp - 4], 2048);
          tma_load_2d(stage, &tmC, &pre_bar[warp - 4], tl.n0 + col0, tl.row_off + tl.m0 + q * 32);
        }
      }
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      const bool zero = tl.num_kb == 0;
      // pair: the leader's MMA waits on the leader's tempty barrier for both CTAs
      const uint32_t tempty_c = CG == 2 ? mapa_shared(smem_u32(&tempty_bar[acc]), 0) : 0u;
      auto release_acc = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) mbar_arrive_cluster(tempty_c);
          else mbar_arrive(&tempty_bar[acc]);
        }
      };

      {
        // software-pipelined: the TMEM read of chunk i+1 is in flight while chunk i is processed --
        // except DGRAD2's epilogue, whose operand block already holds 16 more registers per thread:
        // there the second buffer spilled (a TMEM read is ~12 cycles to its first use)
        constexpr bool PIPE = EPI != EPI_DGELU;
        constexpr int NCH = EPI_COLS / 32;
        uint32_t rawA[32], rawB[32];
        if (!zero && PIPE) tmem_ld_32x32b_x32(t_row + col0, rawA);
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          uint32_t(&cur)[32] = (PIPE && (i & 1)) ? rawB : rawA;
          uint32_t(&nxt)[32] = (PIPE && (i & 1)) ? rawA : rawB;
          const int c = col0 + 32 * i;
          uint4 pre_v[4];
          if constexpr (EPI == EPI_DGELU) {  // operand block (TMA, SWIZZLE_64B)
            if (tl.active) {
            mbar_wait(&pre_bar[warp - 4], pre_phase);
            pre_phase ^= 1;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              pre_v[u] = *reinterpret_cast<const uint4*>(stage + lane * 64 + ((u ^ ((lane >> 1) & 3)) << 4));
            __syncwarp();
            if (lane == 0 && i + 1 < NCH) {
              mbar_arrive_expect_tx(&pre_bar[warp - 4], 2048);
              tma_load_2d(stage, &tmC, &pre_bar[warp - 4], tl.n0 + c + 32, tl.row_off + tl.m0 + q * 32);
            }
            }
          }
          if (!zero) {
            if (!PIPE) tmem_ld_32x32b_x32(t_row + c, cur);
            tmem_ld_wait();
            if (PIPE && i + 1 < NCH) tmem_ld_32x32b_x32(t_row + c + 32, nxt);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) cur[j] = 0u;
          }
          if (i + 1 == NCH) release_acc();  // every TMEM read of this tile has completed
          if (tl.active) epilogue_chunk<EPI>(cur, p, tl, r, c, pre_v, stage, sbuf, &tmC, &tmC2, lane);
        }
      }
      if (++acc == NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  if constexpr (tma_out<EPI>()) {
    if (warp >= 4) bulk_wait0();  // every lane: scatter epilogues issue per-lane bulk copies
  }
  tc_fence_before();
  if constexpr (CG == 2) {
    cluster_sync_all();  // the peer may still read/commit into this CTA's TMEM and barriers
    if (warp == 2) tmem_free_2sm<TMEM_COLS>(tmem_base);
  } else {
    __syncthreads();
    if (warp == 2) tmem_free<TMEM_COLS>(tmem_base);
  }
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
struct TmapKey {
  const void* ptr;
  uint64_t inner, outer;
  uint32_t bi, bo, swz, dt;
  bool operator==(const TmapKey& o) const {
    return ptr == o.ptr && inner == o.inner && outer == o.outer && bi == o.bi && bo == o.bo &&
           swz == o.swz && dt == o.dt;
  }
};
struct TmapKeyHash {
  size_t operator()(const TmapKey& k) const {
    size_t h = std::hash<const void*>()(k.ptr);
    for (uint64_t v : {k.inner, k.outer, (uint64_t)k.bi << 32 | k.bo, (uint64_t)k.swz << 32 | k.dt})
      h = h * 1000003u ^ std::hash<uint64_t>()(v);
    return h;
  }
};

static int encode_tmap(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                       uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz,
                       CUtensorMapDataType dt);

// Tensor maps are pure functions of (address, shape, box, swizzle, dtype); the
// layer's buffers are persistent, so encoding happens once per buffer.
static int make_tmap(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                     uint32_t box_inner, uint32_t box_outer,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B,
                     CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16) {
  static std::mutex mu;
  static std::unordered_map<TmapKey, CUtensorMap, TmapKeyHash> cache;
  const TmapKey key{ptr, inner, outer, box_inner, box_outer, (uint32_t)swz, (uint32_t)dt};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *m = it->second;
      return PP_OK;
    }
  }
  if (int rc = encode_tmap(m, ptr, inner, outer, box_inner, box_outer, swz, dt)) return rc;
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, *m);
  return PP_OK;
}

static int encode_tmap(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                       uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz,
                       CUtensorMapDataType dt) {
  if (int rc = get_encode()) return rc;
  const uint64_t esize = dt == CU_TENSOR_MAP_DATA_TYPE_FLOAT32 ? 4 : 2;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * esize};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, dt, 2, const_cast<void*>(ptr), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(PP_ECUDA, "cuTensorMapEncodeTiled failed (%d) inner=%llu outer=%llu box=%ux%u",
                (int)r, (unsigned long long)inner, (unsigned long long)outer, box_inner,
                box_outer);
  return PP_OK;
}

// output tensor map for the TMA-store epilogue: bf16 [outer][inner], box 32 x 32, SWIZZLE_64B
static int make_out_tmap(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer) {
  return make_tmap(m, ptr, inner, outer, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
}
// fp32 output (wgrad): box 32 x 32 fp32 = 128 B rows, SWIZZLE_128B
static int make_out_tmap_f32(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer) {
  return make_tmap(m, ptr, inner, outer, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
}

template <int BN, bool A_MN, bool B_MN, int EPI, int STAGES, int CG = 1>
static int launch(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, int grid,
                  cudaStream_t st, const CUtensorMap* tc = nullptr, const CUtensorMap* tc2 = nullptr) {
  auto kern = grouped_gemm_kernel<BN, A_MN, B_MN, EPI, STAGES, CG>;
  const int staging = tma_out<EPI>() ? 8 * stage_bytes_per_warp<EPI>() : 0;
  const int smem = STAGES * (BM * BK * 2 + (BN / CG) * BK * 2) + staging + 1024;
  static CUtensorMap dummy{};
  static int configured[64] = {0};  // per device: the smem attribute is set once
  int dev = 0;
  PP_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 64 && !configured[dev]) {
    PP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured[dev] = 1;
  }
  if constexpr (CG == 1) {
    PP_CUDA_TRY(pdl_launch(kern, dim3(grid), dim3(kThreads), smem, st, ta, tb, tc ? *tc : dummy, tc2 ? *tc2 : dummy, p));
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((grid / 2) * 2);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (common.cuh)
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    PP_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ta, tb, tc ? *tc : dummy, tc2 ? *tc2 : dummy, p));
  }
  PP_LAUNCH_CHECK();
  return PP_OK;
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
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

// ---- staggered 256 x 512 tiles ---------------------------------------------------------------
// Opt-in while it is being measured: PPMOE_GEMM_STAGGER=1 (FWD1, DGRAD2: short K, heavy
// epilogues), PPMOE_GEMM_STAGGER_WGRAD=1 (WGRAD1/2: ragged K, fp32 epilogue).  A 256 x 512
// CTA-pair tile shares each A block between its two N halves (25 % fewer operand bytes per flop
// than 256 x 256, the bound for these modes: the SM's L2 port), but with both halves
// accumulating together the single TMEM buffer exposes the whole epilogue.  Here the halves
// run L k-steps apart: half 0 takes A(kb) with B0(kb), half 1 takes the same A(kb) -- still in
// an NA-deep ring -- with B1(kb) L steps later.  Each half has its own 256 TMEM columns and
// full/empty barriers, so the epilogue drains half 0 while half 1's last L k-steps (and, across
// tiles, the next tile's half 0 once drained) keep the tensor pipe busy.  No replica gate / SM
// reservation / fused scatter: those launches use the double-buffered 256 x 256 kernel.
template <bool A_MN, bool B_MN, int EPI, int L, int NA, int NB>
__global__ void __launch_bounds__(kThreads, 1)
    grouped_gemm_stagger_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                                const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2,
                                const GemmParams p) {
  pdl_grid_sync();
  constexpr int CG = 2, BN = 512, HALF = 256, BNC_H = HALF / CG;  // B rows (or cols) per CTA per half
  constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = BNC_H * BK * 2;
  constexpr uint32_t IDESC = make_idesc<HALF, A_MN, B_MN, BM * CG>();
  constexpr int EPI_WARPS = 8, EPI_COLS = HALF * 4 / EPI_WARPS;  // per half: 128 columns per warp
  static_assert(NA >= L + 2, "A must outlive the L-step lag plus one step of prefetch");
  extern __shared__ __align__(1024) uint8_t dsmem[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsmem) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                          // [NA][A_BYTES]
  uint8_t* sB = sA + NA * A_BYTES;             // [2][NB][B_BYTES]
  uint8_t* sEpi = sB + 2 * NB * B_BYTES;       // [8][stage_bytes_per_warp]
  __shared__ __align__(8) uint64_t fullA[NA], emptyA[NA], fullB[2][NB], emptyB[2][NB];
  __shared__ __align__(8) uint64_t tfull[2], tempty[2];
  __shared__ __align__(8) uint64_t pre_bar[8];
  __shared__ uint32_t tmem_base_sh;
  __shared__ SchedSmem sched;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) build_schedule<BN, CG>(p, sched);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmC);
    if constexpr (EPI == EPI_GELU) tma_prefetch_desc(&tmC2);
  }
  const int cta_rank = (int)cluster_ctarank();
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < NA; ++i) {
      mbar_init(&fullA[i], 1);
      mbar_init(&emptyA[i], 1);
    }
    for (int h = 0; h < 2; ++h)
      for (int i = 0; i < NB; ++i) {
        mbar_init(&fullB[h][i], 1);
        mbar_init(&emptyB[h][i], 1);
      }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&tfull[h], 1);
      mbar_init(&tempty[h], EPI_WARPS * CG);
    }
    for (int i = 0; i < 8; ++i) mbar_init(&pre_bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_2sm<512>(&tmem_base_sh);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;
  const int total_tiles = sched.prefix[sched.G];
  const int G_walk = (int)gridDim.x / CG;
  const bool snake = p.ragged_k != 0;  // wgrad: LPT-sorted groups dealt in snake order
  auto tile_of = [&](int it) -> int {
    const int b = (int)blockIdx.x / CG;
    return it * G_walk + ((snake && (it & 1)) ? (G_walk - 1 - b) : b);
  };
  // unit sequence of one tile (K = its k-steps): slot s in [0, K + L): half 0 at k-step s (s < K),
  // half 1 at s - L (s >= L)

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer: loads in unit order
      uint32_t seqA = 0, seqB[2] = {0, 0};
      Tile tl;
      for (int it = 0, t = tile_of(0); t < total_tiles; t = tile_of(++it)) {
        if (!decode_tile<BN, CG>(t, sched, p, tl, cta_rank)) break;
        const int K = tl.num_kb;
        auto bcol = [&](int h) { return tl.n0 + h * HALF + cta_rank * BNC_H; };
        for (int sl = 0; K > 0 && sl < K + L; ++sl) {
          for (int h = 0; h < 2; ++h) {
            const int kb = h == 0 ? sl : sl - L;
            if (kb < 0 || kb >= K) continue;
            const int k0 = kb * BK;
            if (h == 0) {  // A(kb) with B0(kb)
              const uint32_t a = seqA % NA, pa = (seqA / NA) & 1;
              mbar_wait(&emptyA[a], pa ^ 1);
              if (cta_rank == 0) mbar_arrive_expect_tx(&fullA[a], A_BYTES * CG);
              const uint32_t bar = mapa_shared(smem_u32(&fullA[a]), 0);
              if constexpr (!A_MN) {
                tma_load_2d_2sm(sA + a * A_BYTES, &tmA, bar, k0, tl.row_off + tl.m0);
              } else {  // wgrad: A = the group's token rows, MN-major
#pragma unroll
                for (int i = 0; i < BM / 64; ++i)
                  tma_load_2d_2sm(sA + a * A_BYTES + i * 8192, &tmA, bar, tl.m0 + 64 * i, tl.row_off + k0);
              }
              ++seqA;
            }
            const uint32_t b = seqB[h] % NB, pb = (seqB[h] / NB) & 1;
            mbar_wait(&emptyB[h][b], pb ^ 1);
            if (cta_rank == 0) mbar_arrive_expect_tx(&fullB[h][b], B_BYTES * CG);
            uint8_t* dst = sB + (h * NB + b) * B_BYTES;
            const uint32_t bar = mapa_shared(smem_u32(&fullB[h][b]), 0);
            if constexpr (!B_MN) {
              tma_load_2d_2sm(dst, &tmB, bar, k0, tl.wslot * p.N + bcol(h));
            } else {
              const int brow = p.ragged_k ? tl.row_off + k0 : tl.wslot * p.K_fixed + k0;
#pragma unroll
              for (int i = 0; i < BNC_H / 64; ++i) tma_load_2d_2sm(dst + i * 8192, &tmB, bar, bcol(h) + 64 * i, brow);
            }
            ++seqB[h];
          }
        }
      }
    }
  } else if (warp == 1 && cta_rank == 0) {  // ===== MMA issuer (leader CTA)
    uint32_t seqA = 0, seqB[2] = {0, 0}, accph[2] = {0, 0};
    Tile tl;
    for (int it = 0, t = tile_of(0); t < total_tiles; t = tile_of(++it)) {
      if (!decode_tile<BN, CG>(t, sched, p, tl, cta_rank)) break;
      const int K = tl.num_kb;
      if (K == 0) {  // empty wgrad group: no MMAs, the epilogues write zeros
        for (int h = 0; h < 2; ++h) {
          mbar_wait(&tempty[h], accph[h] ^ 1);
          if (lane == 0) {
            mbar_arrive(&tfull[h]);
            mbar_arrive_cluster(mapa_shared(smem_u32(&tfull[h]), 1));
          }
          __syncwarp();
          accph[h] ^= 1;
        }
        continue;
      }
      const uint32_t seqA0 = seqA;  // A sequence number of this tile's k-step 0
      for (int sl = 0; sl < K + L; ++sl) {
        for (int h = 0; h < 2; ++h) {
          const int kb = h == 0 ? sl : sl - L;
          if (kb < 0 || kb >= K) continue;
          if (kb == 0) {  // this half's accumulator must have been drained by the epilogue
            mbar_wait(&tempty[h], accph[h] ^ 1);
            tc_fence_after();
          }
          const uint32_t sa_seq = seqA0 + kb, a = sa_seq % NA;
          if (h == 0) {
            mbar_wait(&fullA[a], (sa_seq / NA) & 1);
            ++seqA;
          }
          const uint32_t b = seqB[h] % NB;
          mbar_wait(&fullB[h][b], (seqB[h] / NB) & 1);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t saddr = smem_u32(sA + a * A_BYTES), sbaddr = smem_u32(sB + (h * NB + b) * B_BYTES);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t ad = A_MN ? make_sdesc(saddr + kk * 2048, 8192, 1024) : make_sdesc(saddr + kk * 32, 16, 1024);
              const uint64_t bd = B_MN ? make_sdesc(sbaddr + kk * 2048, 8192, 1024) : make_sdesc(sbaddr + kk * 32, 16, 1024);
              tc_mma_bf16_2sm(tmem_base + h * HALF, ad, bd, IDESC, (kb | kk) != 0);
            }
            tc_commit_2sm(&emptyB[h][b], 0x3);
            if (h == 1) tc_commit_2sm(&emptyA[a], 0x3);  // both halves have consumed A(kb)
            if (kb == K - 1) tc_commit_2sm(&tfull[h], 0x3);
          }
          __syncwarp();
          ++seqB[h];
          if (kb == K - 1) accph[h] ^= 1;
        }
      }
    }
  } else if (warp >= 4 && warp < 4 + EPI_WARPS) {  // ===== epilogue: half 0, then half 1, per tile
    const int q = warp & 3;
    const int col0 = ((warp - 4) >> 2) * EPI_COLS;
    uint8_t* stage = sEpi + (warp - 4) * stage_bytes_per_warp<EPI>();
    uint32_t pre_phase = 0, accph[2] = {0, 0};
    int sbuf = 0;
    const int r = q * 32 + lane;
    Tile tl;
    for (int it = 0, t = tile_of(0); t < total_tiles; t = tile_of(++it)) {
      if (!decode_tile<BN, CG>(t, sched, p, tl, cta_rank)) break;
      const bool zero = tl.num_kb == 0;
      for (int h = 0; h < 2; ++h) {
        const int cbase = h * HALF + col0;  // tile-relative column of this warp's first chunk
        if constexpr (EPI == EPI_DGELU) {
          if (lane == 0 && tl.active) {
            mbar_arrive_expect_tx(&pre_bar[warp - 4], 2048);
            tma_load_2d(stage, &tmC, &pre_bar[warp - 4], tl.n0 + cbase, tl.row_off + tl.m0 + q * 32);
          }
        }
        mbar_wait(&tfull[h], accph[h]);
        accph[h] ^= 1;
        tc_fence_after();
        const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + h * HALF;
        const uint32_t tempty_c = mapa_shared(smem_u32(&tempty[h]), 0);
        constexpr int NCH = EPI_COLS / 32;
#pragma unroll 1
        for (int i = 0; i < NCH; ++i) {
          const int c = cbase + 32 * i;
          uint4 pre_v[4];
          if constexpr (EPI == EPI_DGELU) {
            if (tl.active) {
              mbar_wait(&pre_bar[warp - 4], pre_phase);
              pre_phase ^= 1;
#pragma unroll
              for (int u = 0; u < 4; ++u)
                pre_v[u] = *reinterpret_cast<const uint4*>(stage + lane * 64 + ((u ^ ((lane >> 1) & 3)) << 4));
              __syncwarp();
              if (lane == 0 && i + 1 < NCH) {
                mbar_arrive_expect_tx(&pre_bar[warp - 4], 2048);
                tma_load_2d(stage, &tmC, &pre_bar[warp - 4], tl.n0 + c + 32, tl.row_off + tl.m0 + q * 32);
              }
            }
          }
          uint32_t raw[32];
          if (!zero) {
            tmem_ld_32x32b_x32(t_row + col0 + 32 * i, raw);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) raw[j] = 0u;
          }
          if (i + 1 == NCH) {  // every TMEM read of this half has completed: the MMA may reuse it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_c);
          }
          if (tl.active) epilogue_chunk<EPI>(raw, p, tl, r, c, pre_v, stage, sbuf, &tmC, &tmC2, lane);
        }
      }
    }
  }
  if (warp >= 4) bulk_wait0();
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) tmem_free_2sm<512>(tmem_base);
}

template <bool A_MN, bool B_MN, int EPI, int L, int NA, int NB>
static int launch_stagger_v(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, int grid,
                            cudaStream_t st, const CUtensorMap* tc, const CUtensorMap* tc2) {
  auto kern = grouped_gemm_stagger_kernel<A_MN, B_MN, EPI, L, NA, NB>;
  const int smem = NA * (BM * BK * 2) + 2 * NB * (128 * BK * 2) + 8 * stage_bytes_per_warp<EPI>() + 1024;
  static int configured[64] = {0};
  int dev = 0;
  PP_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 64 && !configured[dev]) {
    PP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured[dev] = 1;
  }
  static CUtensorMap dummy{};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((grid / 2) * 2);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PP_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ta, tb, tc ? *tc : dummy, tc2 ? *tc2 : dummy, p));
  PP_LAUNCH_CHECK();
  return PP_OK;
}

// variant = the knob's value: 1 -> (L, NA, NB) = (3, 5, 2), 2 -> (2, 4, 3), 3 -> (4, 6, 2); the
// lag L sets how much of a half's epilogue the other half's MMAs cover, NA >= L + 2 the A ring,
// NB the per-half B ring (smem: NA * 16 KB + 2 * NB * 16 KB + the epilogue staging)
template <bool A_MN, bool B_MN, int EPI>
static int launch_stagger(int variant, const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                          int grid, cudaStream_t st, const CUtensorMap* tc, const CUtensorMap* tc2) {
  if (variant == 2) return launch_stagger_v<A_MN, B_MN, EPI, 2, 4, 3>(ta, tb, p, grid, st, tc, tc2);
  if (variant == 3) return launch_stagger_v<A_MN, B_MN, EPI, 4, 6, 2>(ta, tb, p, grid, st, tc, tc2);
  return launch_stagger_v<A_MN, B_MN, EPI, 3, 5, 2>(ta, tb, p, grid, st, tc, tc2);
}

// ---- K1: the gate as a split-K cluster kernel -------------------------------------
// One 128-token tile per cluster of KS CTAs; CTA r accumulates logits over d-slice r on
// tcgen05 (M = 128, N = BN) and CTAs 1..KS-1 store their fp32 partials into CTA 0's smem
// over DSMEM; CTA 0 adds them in rank order (deterministic) and runs the softmax / top-k /
// chunk-rank epilogue.  Splitting d gives every SM ~2 CTAs (loads of one overlap the
// prologue / epilogue of the other) and keeps the whole token matrix in flight at once --
// the tile-per-CTA GEMM path left 20 SMs idle and serialised load -> epilogue per SM.
constexpr int kRouteThreads = 192;  // warp 0 TMA, warp 1 MMA + TMEM, warps 2..5 epilogue

template <int BN, int KS, int STAGES>
__global__ void __launch_bounds__(kRouteThreads)
    route_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const GemmParams p) {
  pdl_grid_sync();
  constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
  constexpr uint32_t IDESC = make_idesc<BN, false, false, BM>();
  extern __shared__ __align__(1024) uint8_t dsmem[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsmem) + 1023) & ~uintptr_t(1023));
  float* part = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES);  // [KS-1][128][BN] (CTA 0)
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES], tfull_bar;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int32_t route_cnt[4][BN];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int crank = (int)cluster_ctarank();
  const int tile = blockIdx.x / KS;
  const int row0 = tile * BM;
  const int kb_per = p.K_fixed / BK / KS, kb0 = crank * kb_per;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    mbar_init(&tfull_bar, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(&tmem_base_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;
  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer
      for (int kb = 0, stage = 0, phase = 0; kb < kb_per; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + stage * STAGE_BYTES;
        mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES);
        tma_load_2d(sa, &tmA, &full_bar[stage], (kb0 + kb) * BK, row0);
        tma_load_2d(sa + A_BYTES, &tmB, &full_bar[stage], (kb0 + kb) * BK, 0);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {  // ===== MMA issuer
    for (int kb = 0, stage = 0, phase = 0; kb < kb_per; ++kb) {
      mbar_wait(&full_bar[stage], phase);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES), sb = sa + A_BYTES;
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)
          tc_mma_bf16(tmem_base, make_sdesc(sa + kk * 32, 16, 1024), make_sdesc(sb + kk * 32, 16, 1024), IDESC,
                      (kb | kk) != 0);
        tc_commit(&empty_bar[stage]);
        if (kb == kb_per - 1) tc_commit(&tfull_bar);
      }
      __syncwarp();
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  }
  // ===== epilogue warps 2..5 (TMEM lane quarter q = warp % 4); everyone joins the cluster barrier
  const int q = warp & 3;
  const int r = q * 32 + lane;
  float v[BN];
  if (warp >= 2) {
    mbar_wait(&tfull_bar, 0);
    tc_fence_after();
    const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16);
#pragma unroll
    for (int c = 0; c < BN; c += 16) {
      uint32_t raw[16];
      tmem_ld_32x32b_x16(t_row + c, raw);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 16; ++j) v[c + j] = __uint_as_float(raw[j]);
    }
    if (crank > 0) {  // partial logits of this d-slice -> CTA 0's smem (DSMEM)
      const uint32_t dst = mapa_shared(smem_u32(part + ((size_t)(crank - 1) * BM + r) * BN), 0);
#pragma unroll
      for (int c = 0; c < BN; c += 4)
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst + 4 * c), "f"(v[c]),
                     "f"(v[c + 1]), "f"(v[c + 2]), "f"(v[c + 3])
                     : "memory");
    }
  }
  tc_fence_before();
  cluster_sync_all();  // release / acquire: the partials are visible in CTA 0
  if (warp >= 2 && crank == 0) {
#pragma unroll 1
    for (int s = 0; s < KS - 1; ++s) {  // rank order: deterministic sum
      const float* pr = part + ((size_t)s * BM + r) * BN;
#pragma unroll
      for (int c = 0; c < BN; c += 4) {
        const float4 x4 = *reinterpret_cast<const float4*>(pr + c);
        v[c] += x4.x; v[c + 1] += x4.y; v[c + 2] += x4.z; v[c + 3] += x4.w;
      }
    }
    const int E = p.e_real;
    const int token = row0 + r;
    const int chunk = row0 / BM;
#pragma unroll
    for (int e = 0; e < BN; ++e) v[e] = e < E ? v[e] + (p.bias ? p.bias[e] : 0.f) : -INFINITY;
    float mx = v[0];
#pragma unroll
    for (int e = 1; e < BN; ++e) mx = fmaxf(mx, v[e]);
    float ssum = 0.f, ex[BN];
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
        *reinterpret_cast<float4*>(prow + e) = make_float4(ex[e] * inv, ex[e + 1] * inv, ex[e + 2] * inv, ex[e + 3] * inv);
    // top-k on logits, ties -> lowest expert index
    // (the weight of a pick is captured with it: indexing ex[] by a runtime expert id would put
    // the array in local memory)
    uint64_t taken_lo = 0, taken_hi = 0;
    int sel[8];
    float wsel[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sel[j] = -1;
      wsel[j] = 0.f;
      if (j < p.topk) {
        int bi = -1;
        float best = 0.f, bex = 0.f;
#pragma unroll
        for (int e = 0; e < BN; ++e) {
          const bool tk = e < 64 ? ((taken_lo >> e) & 1) : ((taken_hi >> (e - 64)) & 1);
          if (e < E && !tk && (bi < 0 || v[e] > best)) {
            best = v[e];
            bex = ex[e];
            bi = e;
          }
        }
        sel[j] = bi;
        wsel[j] = bex * inv;
        if (bi < 64) taken_lo |= 1ull << bi;
        else taken_hi |= 1ull << (bi - 64);
      }
    }
    // chunk ranks: pairs of expert e ordered by token inside this 128-token tile
    int myrank[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) myrank[j] = 0;
    const uint32_t lt_mask = (1u << lane) - 1u;
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
        p.w[(size_t)token * p.topk + j] = wsel[j];
        p.rank[(size_t)token * p.topk + j] = base + myrank[j];
      }
    }
    for (int e = r; e < E; e += 128)
      p.chunk_counts[(size_t)chunk * E + e] = route_cnt[0][e] + route_cnt[1][e] + route_cnt[2][e] + route_cnt[3][e];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<TMEM_COLS>(tmem_base);
}

template <int BN, int KS, int STAGES>
static int launch_route(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, int tiles,
                        cudaStream_t st) {
  auto kern = route_kernel<BN, KS, STAGES>;
  const int smem = STAGES * (BM * BK * 2 + BN * BK * 2) + (KS - 1) * BM * BN * 4 + 1024;
  static int configured[64] = {0};
  int dev = 0;
  PP_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 64 && !configured[dev]) {
    PP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured[dev] = 1;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(tiles * KS);
  cfg.blockDim = dim3(kRouteThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = KS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (common.cuh)
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  PP_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ta, tb, p));
  PP_LAUNCH_CHECK();
  return PP_OK;
}

int route_gemm(const void* x, const void* wg, const float* bias, int T, int d, int E, int k,
               int32_t* idx, float* w, float* probs, int32_t* rank, int32_t* chunk_counts,
               cudaStream_t st) {
  // d split over a cluster of KS = 2 CTAs (cfg2: KS = 1 / 2 / 4 measured 14.4-16.8 / 14.2-15.6 /
  // 21-22 us -- 4 needs a second wave), every slice >= one BK
  const int tiles = T / BM;
  int KS = env_int("PPMOE_ROUTE_KS", 2);
  const int BNr = E <= 16 ? 16 : E <= 32 ? 32 : E <= 64 ? 64 : 128;
  if (BNr == 128 && KS > 2) KS = 2;  // smem: 4 stages + (KS-1) fp32 128 x 128 partials
  if (KS != 1 && KS != 2 && KS != 4) KS = 2;
  while (KS > 1 && (d / BK) % KS) KS >>= 1;
  CUtensorMap ta, tb;
  if (int rc = make_tmap(&ta, x, d, T, BK, BM)) return rc;
  if (int rc = make_tmap(&tb, wg, d, E, BK, BNr)) return rc;
  GemmParams p{};
  p.e_real = E;
  p.K_fixed = d;
  p.bias = bias;
  p.idx = idx;
  p.w = w;
  p.probs = probs;
  p.rank = rank;
  p.chunk_counts = chunk_counts;
  p.topk = k;
#define PP_ROUTE_KS(BN_)                                         \
  switch (KS) {                                                 \
    case 4: return launch_route<BN_, 4, 4>(ta, tb, p, tiles, st); \
    case 2: return launch_route<BN_, 2, 4>(ta, tb, p, tiles, st); \
    default: return launch_route<BN_, 1, 6>(ta, tb, p, tiles, st); \
  }
  switch (BNr) {
    case 16: PP_ROUTE_KS(16)
    case 32: PP_ROUTE_KS(32)
    case 64: PP_ROUTE_KS(64)
    default: PP_ROUTE_KS(128)
  }
#undef PP_ROUTE_KS
}

// dx[T][d] = dl[T][EP] . wg[E][d]: the gate's input gradient (K = EP; wg rows >= E read
// as zeros by the TMA); pp_dispatch_bwd then adds the expert-input gradients
int gate_dx_gemm(const void* dl, const void* wg, int T, int d, int E, int EP, void* dx, cudaStream_t st) {
  CUtensorMap ta, tb, tc;
  GemmParams p{};
  p.max_groups = 1;
  p.single_rows = T;
  p.N = d;
  p.K_fixed = EP;
  p.c = dx;
  if (int rc = make_tmap(&ta, dl, EP, T, BK, BM)) return rc;
  if (int rc = make_tmap(&tb, wg, d, E, 64, BK)) return rc;
  if (int rc = make_out_tmap(&tc, dx, d, T)) return rc;
  return launch<256, false, true, EPI_BF16, 4>(ta, tb, p, sm_count(), st, &tc);
}

// dwg[e][c] = sum_s ws[s][c][e] in a fixed order (bit-deterministic): a CTA takes 64 outputs;
// quarter q of its threads sums splits [q*S/4, (q+1)*S/4) in order (every load issued before
// the adds), then thread q = 0 adds the four quarter sums in q order.  Four times the threads of
// one-thread-per-output, a quarter of the dependent load rounds.
constexpr int kReduceOuts = 64;
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ ws, int splits, int d, int EP,
                                                            int E, float* __restrict__ out) {
  pdl_grid_sync();
  __shared__ float part[4][kReduceOuts];
  const int n = d * E;
  const int o = threadIdx.x % kReduceOuts, q = threadIdx.x / kReduceOuts;
  const int i = blockIdx.x * kReduceOuts + o;
  const int per = (splits + 3) / 4, s_begin = q * per, s_end = min(splits, s_begin + per);
  float acc = 0.f;
  if (i < n) {
    const int c = i / E, e = i - (i / E) * E;
    const float* src = ws + (size_t)c * EP + e;
    const size_t stride = (size_t)d * EP;
    for (int s0 = s_begin; s0 < s_end; s0 += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = s0 + u < s_end ? __ldcs(src + (size_t)(s0 + u) * stride) : 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
  }
  part[q][o] = acc;
  __syncthreads();
  if (q == 0 && i < n) {
    const int c = i / E, e = i - (i / E) * E;
    out[(size_t)e * d + c] = ((part[0][o] + part[1][o]) + part[2][o]) + part[3][o];
  }
}

// dwg[E][d] = dl^T . x, computed transposed: dwg^T[d][EP] = x^T . dl with M = d (128-row
// tiles of x^T), N = EP, split-K over token chunks; partial s -> ws[s][d][EP] (EPI_F32 TMA
// stores, no atomics), then the fixed-order reduce (transposing back)
int gate_dw_gemm(const void* dl, const void* x, int T, int d, int E, int EP, int split, float* ws,
                 float* dwg, cudaStream_t st) {
  const int S = T / split;
  CUtensorMap ta, tb, tc;
  GemmParams q{};
  q.max_groups = 1;
  q.single_rows = T;
  q.split_rows = split;
  q.ragged_k = 1;
  q.M_fixed = d;
  q.N = EP;
  q.c = ws;
  if (int rc = make_tmap(&ta, x, d, T, 64, BK)) return rc;   // A = x^T (MN-major: d contiguous)
  if (int rc = make_tmap(&tb, dl, EP, T, 64, BK)) return rc; // B = dl (MN-major: experts contiguous)
  if (int rc = make_out_tmap_f32(&tc, ws, EP, (uint64_t)S * d)) return rc;
  int rc = EP == 64 ? launch<64, true, true, EPI_F32, 6>(ta, tb, q, sm_count(), st, &tc)
                    : launch<128, true, true, EPI_F32, 5>(ta, tb, q, sm_count(), st, &tc);
  if (rc) return rc;
  const int n = E * d;
  PP_CUDA_TRY(pdl_launch(splitk_reduce_kernel, dim3((n + kReduceOuts - 1) / kReduceOuts), dim3(256), 0, st, ws, S, d,
                         EP, E, dwg));
  PP_LAUNCH_CHECK();
  return PP_OK;
}

static bool use_cta_pair() {
  static const bool on = [] {
    const char* v = getenv("PPMOE_GEMM_CTA_PAIR");
    return v == nullptr || atoi(v) != 0;
  }();
  return on;
}

}  // namespace pp

using namespace pp;

// Diagnostic (PPMOE_GEMM_DEBUG=1): copies the last GEMM launch's per-CTA MMA-thread
// cycle counters [cta][total, wait_tempty, wait_full, -] into host memory.
static unsigned long long* g_dbg_buf = nullptr;
extern "C" int pp_gemm_debug_read(unsigned long long* host, int32_t ctas) {
  PP_CHECK_ARG(g_dbg_buf && host && ctas > 0 && ctas <= 1024 + kTraceSteps * 4,
               "pp_gemm_debug_read: PPMOE_GEMM_DEBUG not set");
  PP_CUDA_TRY(cudaMemcpy(host, g_dbg_buf, (size_t)ctas * 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  return PP_OK;
}

struct ScatterArgs {
  const int32_t* origin;
  void* const* ptrs;
  int tk;
};

struct GateArgs {
  const uint64_t* flags;
  const uint64_t* epoch;
  int me, D, slot0;
  const int32_t* res_stats;
  int res_both, res_per_unit, res_lo, res_hi;
};

static int grouped_gemm_impl(int32_t mode, const void* a, const void* b, void* c, void* c2,
                             const pp_group* groups, const int32_t* num_groups, int32_t max_groups,
                             int32_t rows_capacity, int32_t num_slots, int32_t d_model,
                             int32_t d_ff, int32_t num_sms, void* stream, const ScatterArgs* sc,
                             const GateArgs* gate = nullptr);

extern "C" int pp_grouped_gemm(int32_t mode, const void* a, const void* b, void* c, void* c2,
                               const pp_group* groups, const int32_t* num_groups,
                               int32_t max_groups, int32_t rows_capacity, int32_t num_slots,
                               int32_t d_model, int32_t d_ff, int32_t num_sms, void* stream) {
  PP_CHECK_ARG(c, "pp_grouped_gemm: null pointer");
  return grouped_gemm_impl(mode, a, b, c, c2, groups, num_groups, max_groups, rows_capacity,
                           num_slots, d_model, d_ff, num_sms, stream, nullptr);
}

extern "C" int pp_grouped_gemm_ex(int32_t mode, const void* a, const void* b, void* c, void* c2,
                                  const pp_group* groups, const int32_t* num_groups, int32_t max_groups,
                                  int32_t rows_capacity, int32_t num_slots, int32_t d_model, int32_t d_ff,
                                  const int32_t* origin, void* const* scatter_ptrs, int32_t pairs_per_rank,
                                  const uint64_t* gate_flags, const uint64_t* gate_epoch, int32_t my_rank,
                                  int32_t D, int32_t first_replica_slot, const int32_t* res_stats,
                                  int32_t res_both, int32_t res_per_unit, int32_t res_lo, int32_t res_hi,
                                  int32_t num_sms, void* stream) {
  ScatterArgs sc{origin, scatter_ptrs, pairs_per_rank};
  GateArgs gt{gate_flags, gate_epoch, my_rank, D, first_replica_slot, res_stats, res_both, res_per_unit,
              res_lo, res_hi};
  PP_CHECK_ARG(!res_stats || (res_per_unit >= 0 && res_lo >= 0 && res_hi >= res_lo),
               "pp_grouped_gemm_ex: bad reservation arguments");
  if (origin) {
    PP_CHECK_ARG(mode == PP_GEMM_FWD2 || mode == PP_GEMM_DGRAD1,
                 "pp_grouped_gemm_ex: the fused A2A epilogue serves FWD2 and DGRAD1, got mode %d", mode);
    PP_CHECK_ARG(scatter_ptrs && pairs_per_rank > 0, "pp_grouped_gemm_ex: bad scatter arguments");
    if (!c) c = const_cast<void*>(a);  // the unused output tensor map is built over A (>= rows x d_model)
  }
  if (gate_flags) {
    PP_CHECK_ARG(mode == PP_GEMM_FWD1 || mode == PP_GEMM_FWD2,
                 "pp_grouped_gemm_ex: the replica gate serves FWD1 and FWD2, got mode %d", mode);
    PP_CHECK_ARG(gate_epoch && D >= 1 && my_rank >= 0 && my_rank < D && first_replica_slot >= 1,
                 "pp_grouped_gemm_ex: bad gate arguments");
  }
  return grouped_gemm_impl(mode, a, b, c, c2, groups, num_groups, max_groups, rows_capacity, num_slots,
                           d_model, d_ff, num_sms, stream, origin ? &sc : nullptr,
                           (gate_flags || res_stats) ? &gt : nullptr);
}

static int grouped_gemm_impl(int32_t mode, const void* a, const void* b, void* c, void* c2,
                             const pp_group* groups, const int32_t* num_groups, int32_t max_groups,
                             int32_t rows_capacity, int32_t num_slots, int32_t d_model,
                             int32_t d_ff, int32_t num_sms, void* stream, const ScatterArgs* sc,
                             const GateArgs* gate) {
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
  CUtensorMap ta, tb, tc, tc2;
  GemmParams p{};
  static const int dbg_level = getenv("PPMOE_GEMM_DEBUG") ? atoi(getenv("PPMOE_GEMM_DEBUG")) : 0;
  // [1024 CTAs][4] counters, then (level 2) the [4][kTraceSteps][4] timestamp trace
  if (dbg_level && !g_dbg_buf)
    cudaMalloc(&g_dbg_buf, (4 * 1024 + 4 * kTraceSteps * 4) * sizeof(unsigned long long));
  p.dbg = dbg_level ? g_dbg_buf : nullptr;
  p.trace = dbg_level >= 2 ? g_dbg_buf + 4 * 1024 : nullptr;
  p.groups = groups;
  p.num_groups = num_groups;
  p.max_groups = max_groups;
  p.c = c;
  p.c2 = c2;
  // GeLU in packed bf16x2 arithmetic (FWD1 -4 % at cfg2; PPMOE_GEMM_FAST_GELU=0: fp32)
  p.fast_gelu = env_int("PPMOE_GEMM_FAST_GELU", 1);
  if (sc) {
    p.origin = sc->origin;
    p.scatter_ptrs = sc->ptrs;
    p.scatter_tk = sc->tk;
  }
  if (gate) {
    p.gate_flags = gate->flags;
    p.gate_epoch = gate->epoch;
    p.gate_me = gate->me;
    p.gate_D = gate->D;
    p.gate_slot0 = gate->slot0;
    p.res_stats = gate->res_stats;
    p.res_both = gate->res_both;
    p.res_per_unit = gate->res_per_unit;
    p.res_lo = gate->res_lo;
    p.res_hi = gate->res_hi;
  }
  int rc = PP_OK;
  // CTA pairs (cta_group::2, 256 x 256 tiles, B split across the pair) unless
  // PPMOE_GEMM_CTA_PAIR=0; a pair stages 16 KB of A + 16 KB of B per CTA and stage
  const bool pair = use_cta_pair();
  const uint32_t bkb = pair ? 128 : 256;  // K-major B rows staged per CTA
  // 256 x 512 pair tiles for the long-K modes when N allows (PPMOE_GEMM_WIDE=0 disables)
  static const bool wide_env = !getenv("PPMOE_GEMM_WIDE") || atoi(getenv("PPMOE_GEMM_WIDE")) != 0;
  // (not with the fused-A2A scatter epilogue: its per-row copies are heavier, and the single-buffered
  // 512-column accumulator would expose them)
  const bool wide_dm = pair && wide_env && !sc && dm % 512 == 0, wide_df = pair && wide_env && !sc && df % 512 == 0;
#define PP_LAUNCH_W(EPI_, AMN_, BMN_, S_, ...) launch<512, AMN_, BMN_, EPI_, S_, 2>(ta, tb, p, grid, st, ##__VA_ARGS__)
#define PP_LAUNCH(EPI_, AMN_, BMN_, S1_, S2_, ...)                                          \
  (pair ? launch<256, AMN_, BMN_, EPI_, S2_, 2>(ta, tb, p, grid, st, ##__VA_ARGS__)         \
        : launch<256, AMN_, BMN_, EPI_, S1_, 1>(ta, tb, p, grid, st, ##__VA_ARGS__))
  switch (mode) {
    case PP_GEMM_FWD1:
      PP_CHECK_ARG(c2, "FWD1 needs the act output");
      if ((rc = make_tmap(&ta, a, dm, R, BK, BM)) || (rc = make_tmap(&tb, b, dm, (uint64_t)S * df, BK, bkb))) return rc;
      p.N = df; p.K_fixed = dm;
      if ((rc = make_out_tmap(&tc, c, df, R)) || (rc = make_out_tmap(&tc2, c2, df, R))) return rc;
      if (wide_df && env_int("PPMOE_GEMM_FWD1_WIDE", 0)) return PP_LAUNCH_W(EPI_GELU, false, false, 3, &tc, &tc2);
      if (wide_df && !gate && !sc && env_int("PPMOE_GEMM_STAGGER", 0))
        return launch_stagger<false, false, EPI_GELU>(env_int("PPMOE_GEMM_STAGGER", 0), ta, tb, p, grid, st, &tc, &tc2);
      return PP_LAUNCH(EPI_GELU, false, false, 3, 5, &tc, &tc2);
    case PP_GEMM_FWD2:
      if ((rc = make_tmap(&ta, a, df, R, BK, BM)) ||
          (rc = make_tmap(&tb, b, df, (uint64_t)S * dm, BK, bkb)))
        return rc;
      p.N = dm; p.K_fixed = df;
      if ((rc = make_out_tmap(&tc, c, dm, R))) return rc;
      if (wide_dm) return PP_LAUNCH_W(EPI_BF16, false, false, 4, &tc);
      return PP_LAUNCH(EPI_BF16, false, false, 4, 6, &tc);
    case PP_GEMM_DGRAD2:
      PP_CHECK_ARG(c2, "DGRAD2 needs the pre-activation");
      if ((rc = make_tmap(&ta, a, dm, R, BK, BM)) || (rc = make_tmap(&tb, b, df, (uint64_t)S * dm, 64, BK))) return rc;
      p.N = df; p.K_fixed = dm;
      PP_CHECK_ARG(c2 == c, "DGRAD2 runs in place: dPre must alias pre");
      if ((rc = make_out_tmap(&tc, c, df, R))) return rc;
      if (wide_df && env_int("PPMOE_GEMM_DGRAD2_WIDE", 0)) return PP_LAUNCH_W(EPI_DGELU, false, true, 3, &tc);
      if (wide_df && !gate && env_int("PPMOE_GEMM_STAGGER", 0))
        return launch_stagger<false, true, EPI_DGELU>(env_int("PPMOE_GEMM_STAGGER", 0), ta, tb, p, grid, st, &tc, nullptr);
      return PP_LAUNCH(EPI_DGELU, false, true, 3, 5, &tc);
    case PP_GEMM_DGRAD1:
      if ((rc = make_tmap(&ta, a, df, R, BK, BM)) || (rc = make_tmap(&tb, b, dm, (uint64_t)S * df, 64, BK))) return rc;
      p.N = dm; p.K_fixed = df;
      if ((rc = make_out_tmap(&tc, c, dm, R))) return rc;
      if (wide_dm) return PP_LAUNCH_W(EPI_BF16, false, true, 4, &tc);
      return PP_LAUNCH(EPI_BF16, false, true, 4, 6, &tc);
    case PP_GEMM_WGRAD2:
      if ((rc = make_tmap(&ta, a, dm, R, 64, BK)) || (rc = make_tmap(&tb, b, df, R, 64, BK))) return rc;
      p.M_fixed = dm; p.N = df; p.ragged_k = 1;
      if ((rc = make_out_tmap_f32(&tc, c, df, (uint64_t)S * dm))) return rc;
      if (wide_df && !gate && env_int("PPMOE_GEMM_STAGGER_WGRAD", 0))
        return launch_stagger<true, true, EPI_F32>(env_int("PPMOE_GEMM_STAGGER_WGRAD", 0), ta, tb, p, grid, st, &tc, nullptr);
      if (wide_df) return PP_LAUNCH_W(EPI_F32, true, true, 3, &tc);
      return PP_LAUNCH(EPI_F32, true, true, 3, 5, &tc);
    case PP_GEMM_WGRAD1:
      if ((rc = make_tmap(&ta, a, df, R, 64, BK)) || (rc = make_tmap(&tb, b, dm, R, 64, BK))) return rc;
      p.M_fixed = df; p.N = dm; p.ragged_k = 1;
      if ((rc = make_out_tmap_f32(&tc, c, dm, (uint64_t)S * df))) return rc;
      if (wide_dm && !gate && env_int("PPMOE_GEMM_STAGGER_WGRAD", 0))
        return launch_stagger<true, true, EPI_F32>(env_int("PPMOE_GEMM_STAGGER_WGRAD", 0), ta, tb, p, grid, st, &tc, nullptr);
      if (wide_dm) return PP_LAUNCH_W(EPI_F32, true, true, 3, &tc);
      return PP_LAUNCH(EPI_F32, true, true, 3, 5, &tc);
    case PP_GEMM_PLAIN:
      if ((rc = make_tmap(&ta, a, dm, R, BK, BM)) || (rc = make_tmap(&tb, b, dm, (uint64_t)S * df, BK, bkb))) return rc;
      p.N = df; p.K_fixed = dm;
      if ((rc = make_out_tmap(&tc, c, df, R))) return rc;
      return PP_LAUNCH(EPI_BF16, false, false, 4, 6, &tc);
#undef PP_LAUNCH
#undef PP_LAUNCH_W
    default:
      return fail(PP_EINVAL, "pp_grouped_gemm: unknown mode %d", mode);
  }
}
