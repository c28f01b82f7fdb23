/*
 * ppmoe.h -- C ABI of the B200-native Pro-Prophet expert-parallel MoE hot path.
 *
 * Every entry point takes plain pointers and sizes (device pointers unless
 * stated), an opaque cudaStream_t passed as void*, and returns an int code:
 *   PP_OK 0, PP_EINVAL 1 (-> ValidationError), PP_EDIM 2 (-> DimensionMismatchError),
 *   PP_ECUDA 3, PP_EPEER 4 (-> RuntimeError).  pp_last_error() gives the
 *   thread-local message of the last failing call.
 * All calls are stream-ordered and re-entrant; the only library-owned state is
 * the per-(device, tensor-map) cache inside the GEMM launcher and peer
 * contexts created/destroyed explicitly with pp_peer_*.
 *
 * Reference interfaces each entry point replaces (reference = arxiv 2411.10003
 * "moebal" package, /root/reference/pkg/src/moebal):
 *   pp_plan_greedy    <- planner.greedy_search        planner.py:80-129
 *                        (+ derive_loads core.py:255-275, cost _build perf_model.py:86-107;
 *                        with pp_planner_cfg.iter_counter: plan_for_iteration planner.py:132-156)
 *   pp_plan_physical  <- greedy_search generalised to E = m*D (opt-in; equals
 *                        pp_plan_greedy at m = 1; planner.py:88-90 lifts E == D)
 *   pp_derive_loads   <- core.derive_loads             core.py:255-275
 *   pp_route_topk     <- the gate that produces LoadMatrix rows (core.py:88-95;
 *                        gate described in PAPER.md:106-108); no reference code
 *   pp_slot_histogram <- LoadMatrix construction (virtual expert-slot rows)
 *   pp_dispatch_layout/pp_dispatch/pp_combine (+ _bwd)
 *                     <- routing rule of derive_loads core.py:267-274 realised on
 *                        tokens; A2A modelled by t_a2a perf_model.py:36-39
 *   pp_grouped_gemm   <- expert compute modelled by t_fec/t_bec perf_model.py:42-51
 *   pp_replica_trans / pp_replica_agg / pp_replica_agg_reduce
 *                     <- Trans/Agg modelled by t_trans/t_agg perf_model.py:61-73,
 *                        split by partition_trans/agg scheduler.py:91-108
 *   pp_gate_dx / pp_gate_dw
 *                     <- the gate's backward (part of the BEC the reference prices as
 *                        2x FEC, perf_model.py:49-51); no reference code
 *   pp_top_m_mask     <- simulator._top_m_placement     simulator.py:318-324
 *   pp_peer_barrier / pp_ipc_* / pp_device_*
 *                     <- plumbing of the EP step (no reference counterpart: the
 *                        reference models the exchange)
 */
#ifndef PPMOE_H
#define PPMOE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PP_OK 0
#define PP_EINVAL 1
#define PP_EDIM 2
#define PP_ECUDA 3
#define PP_EPEER 4

const char* pp_last_error(void);
int pp_version(void);

/* ---- cost model + planner (K2) ------------------------------------------ */
typedef struct pp_cost_model {
  double input_bytes;
  double expert_param_bytes;
  double expert_grad_bytes;
  double avg_bandwidth;
  double compute_throughput;
  double fnec_time;
  double bnec_time;
  int32_t num_devices; /* D == E for the planner (virtual expert slots) */
  int32_t num_experts;
  int32_t top_k;
  int32_t _pad;
} pp_cost_model;

/* alpha / n / overlap_aware / reuse_interval: reference PlannerConfig (planner.py:38-60).
 * Extensions (all zero = the reference's behaviour):
 *   max_replicas  > 0: only plans that give no rank more than max_replicas replica
 *                 experts are accepted (the replica weight slots a rank owns); replica
 *                 counts grow with the search prefix, so the search stops at the first
 *                 prefix that exceeds it.  A bound that never binds leaves the plan
 *                 bit-exact with the reference.
 *   slots_per_rank: rows of the load matrix per rank for that count (virtual-slot search:
 *                 m = E/D; 0 or 1 = one row per rank).
 *   iter_counter: device int64[2] {j, scratch}.  Non-NULL: the launch belongs to iteration
 *                 j and plans iteration j+1, so it searches only when (j+1) % reuse_interval
 *                 == 0 (plan_for_iteration, planner.py:132-156) and otherwise leaves every
 *                 output untouched; either way j advances by one when the launch ends.  This
 *                 keeps the reuse policy inside a CUDA graph that replays one launch per
 *                 iteration. */
typedef struct pp_planner_cfg {
  double alpha;
  int32_t n;
  int32_t overlap_aware;
  int32_t reuse_interval;
  int32_t max_replicas;
  int32_t slots_per_rank;
  int32_t _pad;
  const int64_t* iter_counter;
} pp_planner_cfg;

/* Plan L layers, one CTA each.  counts: [L][E][E] int64 (device).
 * Outputs (device): selected [L][E] int32 (search order, first num_selected
 * valid), num_selected [L], num_explored [L], mask [L][E][E] uint8 replica
 * mask of the returned plan, H/R [L][E] int64 of the returned plan,
 * best_cost [L] fp64 (objective of the returned plan).  E <= 1024. */
int pp_plan_greedy(const int64_t* counts, int32_t num_layers, int32_t E,
                   const pp_cost_model* cm, const pp_planner_cfg* cfg,
                   int32_t* selected, int32_t* num_selected, int32_t* num_explored,
                   uint8_t* mask, int64_t* H, int64_t* R, double* best_cost,
                   void* stream);

/* Physically-faithful E > D planner (opt-in): Algorithm 1
 * generalised to m = E/D experts per device (home of e = device e/m, physical
 * LoadMatrix rows); identical to pp_plan_greedy when E == D.  counts:
 * [L][rows][E] int64 with rows = D (physical) or any multiple (rows/D slot rows
 * per device, summed on load).  Outputs: selected [L][E], num_selected [L],
 * num_explored [L], mask [L][rows][E] (each device's row repeated over its slot
 * rows, so the layout consumes it as a slot mask), H/R [L][D], best_cost [L].
 * cm->num_devices must be D and cm->num_experts E; D*E <= 4096.
 * refine_slots (needs rows/D > 1 slot rows per device; an extension beyond the
 * paper): afterwards the heaviest device repeatedly sends one of its replica
 * slot batches back to the expert's home when that lowers the pair's maximum
 * (ties: lower slot, lower expert); the mask then differs between a device's
 * slot rows, H/R are recomputed, selected/best_cost describe the search. */
int pp_plan_physical(const int64_t* counts, int32_t num_layers, int32_t rows, int32_t D, int32_t E,
                     const pp_cost_model* cm, const pp_planner_cfg* cfg, int32_t refine_slots,
                     int32_t* selected,
                     int32_t* num_selected, int32_t* num_explored, uint8_t* mask, int64_t* H,
                     int64_t* R, double* best_cost, void* stream);

/* Top-m baseline (reference simulator._top_m_placement, simulator.py:318-324):
 * mask [D][E] with the m heaviest experts (column totals, ties -> lower index)
 * on every device; selected [m] (nullable) in that order. */
int pp_top_m_mask(const int64_t* counts, int32_t D, int32_t E, int32_t m_top, uint8_t* mask,
                  int32_t* selected, void* stream);

/* counts [D][E] int64, mask [D][E] uint8 -> H [D], R [D] int64.  E <= D. */
int pp_derive_loads(const int64_t* counts, const uint8_t* mask, int32_t D, int32_t E,
                    int64_t* H, int64_t* R, void* stream);

/* ---- routing (K1) -------------------------------------------------------- */
/* x [T][d] bf16, wg [E][d] bf16, bias [E] fp32 (nullable).
 * logits fp32 = x.wg^T + bias; top-k on logits, ties -> lowest expert;
 * weights = softmax(all E logits) at the chosen experts (not renormalised).
 * Outputs: idx [T][k] int32, w [T][k] fp32, probs [T][E] fp32 (for backward),
 * rank [T][k] int32 = position of the pair among the pairs of its expert in
 * its 128-token chunk (token order), chunk_counts [T/128][E] int32.
 * The gate GEMM runs on tcgen05 (N = E padded to 16/32/64/128) with the
 * softmax / top-k / rank epilogue read straight from TMEM.
 * Requires T % 128 == 0, d % 64 == 0, 4 <= E <= 128, E % 4 == 0, 1 <= k <= min(E,8). */
int pp_route_topk(const void* x, const void* wg, const float* bias,
                  int32_t T, int32_t d, int32_t E, int32_t k,
                  int32_t* idx, float* w, float* probs, int32_t* rank,
                  int32_t* chunk_counts, void* stream);

/* This rank's virtual-slot rows of the LoadMatrix: chunk_counts [T/128][E] ->
 * hist [m][E] int64, stored at row offset `row0` of EVERY rank's LoadMatrix copy
 * (out_ptrs: device array [D] of peer-mapped [E][E] buffers) -- the histogram
 * all-gather as plain NVLink stores; follow with pp_peer_barrier. */
int pp_slot_histogram(const int32_t* chunk_counts, int32_t T, int32_t E, int32_t m,
                      int64_t* const* out_ptrs, int32_t D, int32_t row0, void* stream);

/* ---- dispatch layout / permute / combine (K3) --------------------------- */
#define PP_CHUNK 128
#define PP_ROW_ALIGN 128

typedef struct pp_group {
  int32_t row_off;  /* first row of the group's (padded) segment */
  int32_t rows;     /* real rows */
  int32_t rows_pad; /* rows rounded up to PP_ROW_ALIGN */
  int32_t wslot;    /* weight slot in this rank's arena (home: e % m, replicas after) */
  int32_t expert;   /* global expert id */
  int32_t src_rank; /* home rank of the expert (== this rank for home groups) */
  int32_t _pad[2];
} pp_group;

/* Single-CTA layout solver.  counts [Ev][E] int64 all-gathered virtual-slot
 * histogram (Ev = D*m), mask [Ev][E] uint8 replica mask (nullable = vanilla
 * EP), chunk_counts [T/128][E] of this rank.  Outputs (device):
 *   chunk_base [T/128][E] int32 destination row of the first pair of each (chunk, expert)
 *   slot_dest  [m][E]   int32   destination rank of (local slot, expert)
 *   groups     [max_groups] pp_group of THIS rank, num_groups [1] int32,
 *   total_rows [1] int32 (padded rows of this rank's receive buffer)
 *   seg_start  [D][E] int32 segment start of expert e on rank r (-1 if absent)
 *   rep_slot   [D][E] int32 weight slot of replica expert e on rank r (-1 if
 *              none; nullable).
 * counts_from_chunks (D == 1 only): fill `counts` from the chunk counts here,
 * replacing pp_slot_histogram + barrier.  replica_stats (nullable, int32[2]):
 * [0] replicas of this rank's home experts held elsewhere, [1] replicas this
 * rank holds -- the device-side volume hints for SM reservation around Trans/Agg.
 * Capacity: every rank's receive buffer holds rows_capacity rows and num_slots weight
 * slots (0 = unchecked).  When any rank's padded rows exceed rows_capacity, its replica
 * experts exceed num_slots - m, or its groups exceed max_groups, the layout of the whole
 * step is dropped on every rank alike (num_groups = 0, slot_dest = -1: dispatch stores
 * nothing, combine yields zeros) and status (nullable int32, sticky) gets bit 1 / 2 / 4
 * respectively -- nothing is written out of bounds and the caller raises on the flag. */
int pp_dispatch_layout(int64_t* counts, const uint8_t* mask, const int32_t* chunk_counts,
                       int32_t D, int32_t m, int32_t E, int32_t T, int32_t my_rank,
                       int32_t max_groups, int32_t rows_capacity, int32_t num_slots,
                       int32_t* chunk_base, int32_t* slot_dest, pp_group* groups,
                       int32_t* num_groups, int32_t* total_rows, int32_t* seg_start,
                       int32_t* rep_slot, int32_t counts_from_chunks, int32_t* replica_stats,
                       int32_t* status, void* stream);

/* Permute + all-to-all in one kernel: row of token t goes to rank
 * slot_dest[t/(T/m)][e] at row chunk_base[t/128][e] + rank[t][j] of that
 * rank's receive buffer.  recv_ptrs: device array [D] of receive-buffer
 * base pointers (peer-mapped for D > 1).  Also zero-fills this rank's own
 * padding rows (groups/num_groups) and records pair_dest/pair_row [T][k]. */
int pp_dispatch(const void* x, const int32_t* idx, const int32_t* rank,
                const int32_t* chunk_base, const int32_t* slot_dest,
                int32_t T, int32_t d, int32_t k, int32_t m, int32_t E,
                void* const* recv_ptrs, void* own_recv,
                const pp_group* groups, const int32_t* num_groups, int32_t max_groups,
                int32_t* pair_dest, int32_t* pair_row, void* const* origin_ptrs,
                int32_t my_rank, void* stream);

/* y[t] = sum_j w[t][j] * out_ptrs[pair_dest][pair_row] (fp32 accumulate, bf16 out).
 * Fused-A2A mode (comb != NULL, out_ptrs may be NULL): the expert outputs were
 * already pushed to this rank by pp_grouped_gemm_ex as comb [T*k][d] bf16 in
 * pair order (t*k + j), so the gather is local. */
int pp_combine(void* const* out_ptrs, const int32_t* pair_dest, const int32_t* pair_row,
               const float* w, int32_t T, int32_t d, int32_t k, void* y, const void* comb,
               void* stream);

/* Backward of combine + gate softmax: dw[t][j] = <dy[t], Yp[pair]> ; dYp[pair] = w[t][j]*dy[t]
 * (pushed to dgrad_ptrs[pair_dest]); zero-fills own padding rows of own_dgrad; and
 * dl [T][EP] bf16 = dL/dlogits restricted to the top-k (dl_i = p_i * (dw_{j(i)} [i
 * selected] - sum_j dw_j p_{e_j})), zero-padded to EP in {64, 128} columns for the
 * tensor-core gate GEMMs (idx [T][k], probs [T][E]).
 * comb != NULL: Yp[pair] is read locally from comb[t*k + j] (fused-A2A mode). */
int pp_combine_bwd(const void* dy, void* const* out_ptrs, void* const* dgrad_ptrs, void* own_dgrad,
                   const int32_t* pair_dest, const int32_t* pair_row, const float* w,
                   const pp_group* groups, const int32_t* num_groups, int32_t max_groups,
                   int32_t T, int32_t d, int32_t k, float* dw, const void* comb,
                   const int32_t* idx, const float* probs, int32_t E, int32_t EP, void* dl, void* stream);

/* The gate's input gradient on tcgen05:  dx [T][d] bf16 = dl [T][EP] . wg [E][d]
 * (overwrites dx; wg rows >= E read as zeros).  Runs early in the backward (dl comes
 * from pp_combine_bwd); pp_dispatch_bwd adds the expert-input gradients at the end. */
int pp_gate_dx(const void* dl, const void* wg, int32_t T, int32_t d, int32_t E, int32_t EP, void* dx,
               void* stream);

/* Backward of dispatch:  dx[t] += sum_j dXp[pair(t, j)]  (fp32 sum, one bf16 rounding),
 * the k rows pulled from dxp_ptrs[pair_dest] at pair_row (peer loads), or from
 * comb[t*k + j] locally when the DGRAD1 epilogue pushed them here (fused A2A).  Pairs
 * with pair_dest < 0 (dropped step) contribute nothing. */
int pp_dispatch_bwd(void* const* dxp_ptrs, const void* comb, const int32_t* pair_dest,
                    const int32_t* pair_row, int32_t T, int32_t d, int32_t k, void* dx, void* stream);

/* Gate weight gradient, deterministic: dwg [E][d] fp32 = dl^T . x, split-K over
 * token chunks on tcgen05 into workspace [splits][128][d] fp32 (no atomics), then
 * the splits are summed in a fixed order (overwrites dwg).  workspace must hold
 * pp_gate_dw_workspace_bytes(T, d) bytes. */
int pp_gate_dw(const void* dl, const void* x, int32_t T, int32_t d, int32_t E, int32_t EP,
               float* workspace, float* dwg, void* stream);
int64_t pp_gate_dw_workspace_bytes(int32_t T, int32_t d);

/* ---- grouped expert GEMM on tcgen05 (K4) -------------------------------- */
#define PP_GEMM_FWD1 0   /* pre,act[rows][f] = GeLU-split( Xp[rows][d] . W1[slot][f][d]^T ) */
#define PP_GEMM_FWD2 1   /* Yp[rows][d] = act[rows][f] . W2[slot][d][f]^T */
#define PP_GEMM_DGRAD2 2 /* dPre[rows][f] = (dYp[rows][d] . W2[slot][d][f]) * GeLU'(pre) */
#define PP_GEMM_DGRAD1 3 /* dXp[rows][d] = dPre[rows][f] . W1[slot][f][d] */
#define PP_GEMM_WGRAD2 4 /* dW2[slot][d][f] = dYp_g^T . act_g   (fp32) */
#define PP_GEMM_WGRAD1 5 /* dW1[slot][f][d] = dPre_g^T . Xp_g  (fp32) */
#define PP_GEMM_PLAIN 6  /* C[rows][n] = A[rows][k] . B[slot][n][k]^T (bf16), test/utility */

/* a, b: operand base pointers as listed above; c: main output; c2: second
 * output (FWD1: act) or the pre-activation input (DGRAD2, may alias c).
 * rows_capacity: rows allocated in the row-indexed buffers; num_slots:
 * weight slots in the arena; d_model/d_ff: the two feature sizes (for
 * PP_GEMM_PLAIN: K = d_model, N = d_ff).  groups/num_groups on device. */
int pp_grouped_gemm(int32_t mode, const void* a, const void* b, void* c, void* c2,
                    const pp_group* groups, const int32_t* num_groups, int32_t max_groups,
                    int32_t rows_capacity, int32_t num_slots, int32_t d_model, int32_t d_ff,
                    int32_t num_sms, void* stream);

/* Probe loss of the training-step API: out[0] = sum(a[i] * b[i]) over n bf16
 * elements (n % 8 == 0, 16-byte aligned) in fp32, deterministic (per-CTA
 * partials in a fixed order, then one CTA).  partial: >= PP_DOT_PARTIALS floats
 * of device scratch.  The loss sum(y * g) has dL/dy = g, so a training loop
 * that feeds g as the upstream gradient reads back one scalar per step. */
#define PP_DOT_PARTIALS 592
int pp_dot_bf16(const void* a, const void* b, int64_t n, float* partial, float* out, void* stream);

/* pp_grouped_gemm with two optional fusions (NULL disables each):
 * Fused GEMM + all-to-all (origin != NULL; FWD2 -> combine, DGRAD1 -> dispatch
 *   backward): the epilogue stores output row r of the receive layout straight
 *   into the rank that owns the pair, over NVLink: row (o % pairs_per_rank) of
 *   scatter_ptrs[o / pairs_per_rank] ([T*k][d] bf16), o = origin[r] as written
 *   by pp_dispatch (origin_ptrs; padding rows -1, not stored) -- one 64-B bulk
 *   copy per row chunk from the staging smem, overlapping the remaining tiles'
 *   MMAs; pp_combine / pp_gate_dx then read comb locally.  c may be NULL.
 * Replica gate (gate_flags != NULL; FWD1 / FWD2 while Trans is in flight): the
 *   home groups (wslot < first_replica_slot) are scheduled first; before the
 *   first replica tile's loads the TMA producer waits until gate_flags[r] >=
 *   *gate_epoch for every peer r != my_rank (the completion flags of
 *   pp_replica_trans; gate_flags = this rank's [D] uint64 row).  After 20 s without a
 *   flag the gate gives up and stores 1 into gate_epoch[1] (fault word; gate_epoch must
 *   point at two uint64 words).
 * Device-adaptive SM reservation (res_stats != NULL, pp_dispatch_layout's
 *   replica_stats): the persistent walk leaves clamp(res_per_unit * (stats[0] +
 *   (res_both ? stats[1] : 0)), res_lo, res_hi) of the num_sms SMs to concurrent
 *   side kernels sized by this iteration's replica volume; the other CTAs exit at
 *   once.  Keep res_lo >= 2 when gating, so this rank's own Trans kernel (whose
 *   completion signal the peers wait on) can always run. */
int pp_grouped_gemm_ex(int32_t mode, const void* a, const void* b, void* c, void* c2,
                       const pp_group* groups, const int32_t* num_groups, int32_t max_groups,
                       int32_t rows_capacity, int32_t num_slots, int32_t d_model, int32_t d_ff,
                       const int32_t* origin, void* const* scatter_ptrs, int32_t pairs_per_rank,
                       const uint64_t* gate_flags, const uint64_t* gate_epoch, int32_t my_rank,
                       int32_t D, int32_t first_replica_slot, const int32_t* res_stats,
                       int32_t res_both, int32_t res_per_unit, int32_t res_lo, int32_t res_hi,
                       int32_t num_sms, void* stream);

/* ---- replica Trans / Agg over peer memory (K5) --------------------------- */
/* Trans (home side, SM engine): push each of this rank's home experts' W1/W2
 * (weight arenas [slots][f][d] and [slots][d][f] bf16, peer pointer tables
 * w1_ptrs/w2_ptrs [D]) into the replica slot of every rank that holds it under
 * the plan's mask ([E][E] uint8 slot->expert; D = E/m).  Replica slot rule (=
 * pp_dispatch_layout's): the experts e with home e/m != r that some slot of r
 * routes to, ascending, get slots m, m+1, ... on r.  Needs only the mask, so it
 * can run before this iteration's routing; every rank must have passed the
 * previous backward's last peer barrier.  `max_ctas` = SMs it occupies
 * (E <= 1024, D*E <= 16384).  parts: 1 = W1 only, 2 = W2 only, 3 = both.
 * num_slots: weight slots per rank's arena; replicas that would land in slot >=
 * num_slots are skipped (the layout flags such a plan, see pp_dispatch_layout).
 * flag_ptrs (nullable; peer table of [rows][D] uint64 flag arrays): when every
 * CTA is done, the last one stores *epoch (device value, e.g. the peer-barrier
 * counter) into flag_ptrs[r][flag_row*D + my_rank] of every peer r with release
 * semantics -- the completion signal the pp_grouped_gemm_ex gate waits on;
 * done_ctr is a zeroed uint32 scratch word (left zeroed). */
int pp_replica_trans(void* const* w1_ptrs, void* const* w2_ptrs, const uint8_t* mask, int32_t E,
                     int32_t m, int32_t my_rank, int32_t num_slots, int32_t d_model, int32_t d_ff, int32_t parts,
                     void* const* flag_ptrs, int32_t flag_row, const uint64_t* epoch,
                     uint32_t* done_ctr, int32_t max_ctas, void* stream);

/* Agg phase 1 (replica side): push the fp32 grads of this rank's replica slots
 * (g1_ptrs/g2_ptrs [D] grad arenas) into the home rank's staging area
 * stage_ptrs[home] laid out [m][D-1][2][d_ff*d_model] fp32 (index r' = this
 * rank's position among the home's D-1 peers).  parts: 1 = W1 grads, 2 = W2
 * grads, 3 = both (the layer pushes W2's as soon as WGRAD2 is done, W1's after
 * WGRAD1). */
int pp_replica_agg(void* const* g1_ptrs, void* const* g2_ptrs, void* const* stage_ptrs,
                   const uint8_t* mask, int32_t E, int32_t m, int32_t my_rank, int32_t num_slots, int32_t d_model,
                   int32_t d_ff, int32_t parts, int32_t max_ctas, void* stream);

/* Agg phase 2 (home side, after a peer barrier): grad[j] += stage[j][r'] for
 * every rank holding expert my_rank*m + j, in ascending rank order (the
 * oracle's summation order).  g1/g2/stage are this rank's local buffers. */
int pp_replica_agg_reduce(float* g1, float* g2, const float* stage, const uint8_t* mask, int32_t E,
                          int32_t m, int32_t my_rank, int32_t d_model, int32_t d_ff, int32_t parts,
                          int32_t max_ctas, void* stream);

/* Copy-engine Trans/Agg: one cudaMemcpyAsync per (dst, src, bytes) triple of
 * the HOST arrays (peer pointers via IPC: the copy runs on the copy engines over
 * NVLink and takes no SMs, so it overlaps the tensor-core GEMMs). */
int pp_copy_batch(void* const* dst, const void* const* src, const uint64_t* bytes, int32_t n,
                  void* stream);

/* Agg reduce step after the copy-engine pulls: home slot j of g1/g2 (fp32
 * [m][f][d], [m][d][f]) += staging entries [ranges[j], ranges[j+1]) in order
 * (entry i = g1 part then g2 part).  ranges: device int32 [m+1]. */
int pp_agg_accumulate(float* g1_home, float* g2_home, const float* staging, const int32_t* ranges,
                      int32_t m, int32_t d_model, int32_t d_ff, void* stream);

/* ---- peer memory (CUDA IPC) + device barrier ----------------------------- */
/* Library-owned cudaMalloc allocations (IPC-exportable as a whole). */
int pp_device_alloc(uint64_t bytes, void** dev_ptr);
int pp_device_free(void* dev_ptr);
/* Export a device allocation: writes a 64-byte IPC handle. */
int pp_ipc_export(void* dev_ptr, uint8_t* handle64);
/* Import a peer allocation (on the current device). */
int pp_ipc_import(const uint8_t* handle64, void** dev_ptr);
int pp_ipc_close(void* dev_ptr);

/* Cross-rank barrier over peer-mapped signal words.  signal_ptrs: device
 * array [D] of each rank's signal area (uint64_t[D + 2] each: D peer slots, this
 * rank's own counter, this rank's fault word).  epoch > 0: host-provided, must grow by
 * one per call; epoch == 0: taken from the device counter (CUDA-graph replayable).
 * Spins with a 20 s timeout: a peer that never arrives sets the fault word to 1 and the
 * kernel returns (no hang, no context kill; the caller checks the word). */
int pp_peer_barrier(void* const* signal_ptrs, int32_t D, int32_t my_rank, uint64_t epoch,
                    void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PPMOE_H */
