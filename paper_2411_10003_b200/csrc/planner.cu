// K2: Pro-Prophet greedy replica-placement planner on device (Algorithm 1).
//
// Bit-exact restatement of reference greedy_search (pkg/src/moebal/planner.py:80-129):
//   * total_inputs = sum(counts) // top_k                         planner.py:104
//   * loop while not is_balanced(H)                               planner.py:114, :63-68
//   * i = first argmax(H); stop if i was already used             planner.py:115-117
//   * excluded = n non-home devices with fewest counts[:, i] on the ORIGINAL
//     matrix, key (count, index)                                  planner.py:71-77, :120
//   * re-derive H/R under the candidate (derive_loads core.py:255-275) -- here
//     incrementally: selecting i only moves column i's non-excluded cells from
//     "sent to home" to "computed locally"; exact int64 arithmetic
//   * objective = total_(un)scheduled with the exact fp64 association order of
//     perf_model._build (perf_model.py:86-107); strict improvement accepts,
//     and the search continues from rejected candidates       planner.py:122-127
//   * return the accepted prefix selected[:cnt]                   planner.py:129
//
// One CTA per layer; thread d owns device d (== expert d, since D == E).  All
// fp64 math uses __d*_rn intrinsics so no FMA contraction can change a bit.
#include <stdarg.h>

#include "common.cuh"

namespace pp {

struct PlanArgs {
  const int64_t* counts;
  int E;
  pp_cost_model cm;
  pp_planner_cfg cfg;
  int32_t* selected;
  int32_t* num_selected;
  int32_t* num_explored;
  uint8_t* mask;
  int64_t* H;
  int64_t* R;
  double* best_cost;
};

constexpr int kMaxPlanThreads = 1024;
constexpr int kMaxWarps = kMaxPlanThreads / 32;

struct Red {
  int64_t v;
  int32_t i;
};

// block-wide reductions over one value per thread (threads >= E contribute neutral values)
template <typename Op>
__device__ __forceinline__ Red block_reduce(Red x, Op op, Red* scratch) {
  for (int o = 16; o > 0; o >>= 1) {
    Red y;
    y.v = __shfl_xor_sync(0xffffffffu, x.v, o);
    y.i = __shfl_xor_sync(0xffffffffu, x.i, o);
    x = op(x, y);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[warp] = x;
  __syncthreads();
  Red r = scratch[0];
  for (int w = 1; w < nwarps; ++w) r = op(r, scratch[w]);
  return r;
}

struct MaxFirst {  // larger value wins, ties -> lower index (np.argmax first max)
  __device__ Red operator()(Red a, Red b) const {
    if (a.v > b.v) return a;
    if (b.v > a.v) return b;
    return a.i <= b.i ? a : b;
  }
};
struct MinOp {
  __device__ Red operator()(Red a, Red b) const { return a.v <= b.v ? a : b; }
};
struct SumOp {
  __device__ Red operator()(Red a, Red b) const { return Red{a.v + b.v, 0}; }
};

// perf_model._build + the objective selector of planner.py:98-102
__device__ double objective(const pp_cost_model& cm, bool overlap, int64_t rmax, int64_t hmax,
                            int s, int n) {
  const double a2a = __ddiv_rn(__dmul_rn((double)rmax, cm.input_bytes), cm.avg_bandwidth);
  const double fec = __ddiv_rn((double)hmax, cm.compute_throughput);
  const double bec = __dmul_rn(2.0, fec);
  const double D = (double)cm.num_devices;
  const double sdn = (double)((int64_t)s * (int64_t)(cm.num_devices - n));
  const double denom = __dmul_rn(D, cm.avg_bandwidth);
  const double trans = __ddiv_rn(__dmul_rn(sdn, cm.expert_param_bytes), denom);
  const double agg = __ddiv_rn(__dmul_rn(sdn, cm.expert_grad_bytes), denom);
  double t = __dadd_rn(__dadd_rn(__dmul_rn(4.0, a2a), fec), bec);
  if (overlap) {
    double pt = __dsub_rn(__dsub_rn(trans, fec), cm.fnec_time);
    double pa = __dsub_rn(__dsub_rn(agg, bec), cm.bnec_time);
    pt = pt > 0.0 ? pt : 0.0;
    pa = pa > 0.0 ? pa : 0.0;
    return __dadd_rn(__dadd_rn(t, pt), pa);
  }
  return __dadd_rn(__dadd_rn(t, trans), agg);
}

// rank of device d among the non-home candidates of column `col` (key: count, index)
__device__ __forceinline__ int bottom_rank(const int64_t* col, int E, int home, int d) {
  const int64_t c = col[d];
  int r = 0;
  for (int j = 0; j < E; ++j) {
    if (j == home || j == d) continue;
    const int64_t cj = col[j];
    r += (cj < c) || (cj == c && j < d);
  }
  return r;
}

// Device-side plan_for_iteration gate (pp_planner_cfg.iter_counter): the launch of
// iteration j plans j+1, so it searches only when (j+1) % reuse_interval == 0.
__device__ __forceinline__ bool plan_gate_open(const pp_planner_cfg& cfg, int64_t& j) {
  if (!cfg.iter_counter) return true;
  j = *(volatile const int64_t*)cfg.iter_counter;
  const int F = cfg.reuse_interval > 0 ? cfg.reuse_interval : 1;
  return (j + 1) % F == 0;
}

// ... and j advances once per launch: the last CTA to finish stores j + 1 (every CTA
// read j before its arrival, so no CTA can see the advanced value).
__device__ __forceinline__ void plan_gate_tick(const pp_planner_cfg& cfg, int64_t j) {
  if (!cfg.iter_counter) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t* ctr = const_cast<int64_t*>(cfg.iter_counter);
    __threadfence();
    if (atomicAdd(reinterpret_cast<unsigned long long*>(ctr + 1), 1ull) == gridDim.x - 1) {
      ctr[1] = 0;
      ctr[0] = j + 1;
      __threadfence();
    }
  }
}

// Replica bound (pp_planner_cfg.max_replicas): rank r = row / rows_per_rank gains a
// replica of expert e when one of its rows that is not e's home rank keeps e's pairs.
// holder[] / rep[] are shared [ranks]; returns the new maximum over ranks.
__device__ __forceinline__ int64_t add_replicas(uint8_t* holder, int32_t* rep, int ranks, Red* scratch) {
  __syncthreads();
  int64_t v = 0;
  if ((int)threadIdx.x < ranks) {
    rep[threadIdx.x] += holder[threadIdx.x];
    holder[threadIdx.x] = 0;
    v = rep[threadIdx.x];
  }
  struct Max {
    __device__ Red operator()(Red x, Red y) const { return x.v >= y.v ? x : y; }
  };
  return block_reduce(Red{v, 0}, Max(), scratch).v;
}

__global__ void __launch_bounds__(kMaxPlanThreads) plan_greedy_kernel(PlanArgs a) {
  pdl_grid_sync();
  const int L = blockIdx.x;
  const int E = a.E;
  const int d = threadIdx.x;
  const bool active = d < E;
  const int64_t* counts = a.counts + (size_t)L * E * E;
  const int n = a.cfg.n;
  const bool overlap = a.cfg.overlap_aware != 0;

  extern __shared__ int64_t smem_col[];  // [E] column of the expert being placed
  __shared__ Red scratch[kMaxWarps];
  __shared__ int32_t sel_list[kMaxPlanThreads];
  __shared__ uint8_t used[kMaxPlanThreads];
  __shared__ uint8_t holder[kMaxPlanThreads];
  __shared__ int32_t rep[kMaxPlanThreads];

  int64_t iter_j = 0;
  if (!plan_gate_open(a.cfg, iter_j)) {  // reuse: keep the previous plan's outputs
    plan_gate_tick(a.cfg, iter_j);
    return;
  }
  const int spr = a.cfg.slots_per_rank > 1 ? a.cfg.slots_per_rank : 1;
  const int ranks = (E + spr - 1) / spr;
  if (active) {
    used[d] = 0;
    holder[d] = 0;
    rep[d] = 0;
  }

  // initial (vanilla EP) loads: local[d] = counts[d][d]; remote[d] = sum_{d'!=d} counts[d'][d]
  int64_t local = 0, remote = 0, rowsum = 0;
  if (active) {
    local = counts[(size_t)d * E + d];
    for (int j = 0; j < E; ++j) {
      if (j != d) remote += counts[(size_t)j * E + d];
      rowsum += counts[(size_t)d * E + j];
    }
  }
  const int64_t total = block_reduce(Red{rowsum, 0}, SumOp(), scratch).v;
  const int64_t total_inputs = total / a.cm.top_k;  // non-negative: floor == Python //
  const double threshold = __ddiv_rn(__dmul_rn(a.cfg.alpha, (double)total_inputs), (double)E);

  const Red neutral_max{INT64_MIN, 0x7fffffff};
  const Red neutral_min{INT64_MAX, 0x7fffffff};

  auto loads_reduce = [&](int64_t h, int64_t r, Red& hmax, Red& hmin, Red& rmax) {
    hmax = block_reduce(active ? Red{h, d} : neutral_max, MaxFirst(), scratch);
    hmin = block_reduce(active ? Red{h, d} : neutral_min, MinOp(), scratch);
    rmax = block_reduce(active ? Red{r, d} : neutral_max, MaxFirst(), scratch);
  };

  Red hmax, hmin, rmax;
  loads_reduce(local + remote, remote, hmax, hmin, rmax);
  double best = objective(a.cm, overlap, rmax.v, hmax.v, 0, 0);
  int cnt = 0, s = 0;

  while (true) {
    const double spread = (double)(hmax.v - hmin.v);
    if (spread < threshold) break;  // is_balanced
    const int i = hmax.i;
    if (used[i]) break;
    __syncthreads();
    if (d == 0) {
      used[i] = 1;
      sel_list[s] = i;
    }
    if (active) smem_col[d] = counts[(size_t)d * E + i];
    __syncthreads();
    ++s;
    // move column i's non-excluded, non-home cells to local compute
    int64_t moved = 0;
    if (active && d != i) {
      const bool excluded = bottom_rank(smem_col, E, i, d) < n;
      if (!excluded) {
        moved = smem_col[d];
        local += moved;
        if (d / spr != i / spr) holder[d / spr] = 1;
      }
    }
    if (a.cfg.max_replicas > 0 && add_replicas(holder, rep, ranks, scratch) > a.cfg.max_replicas) {
      --s;  // this prefix needs more replica slots than a rank owns: stop before it
      break;
    }
    const int64_t moved_total = block_reduce(Red{moved, 0}, SumOp(), scratch).v;
    if (d == i) remote -= moved_total;
    loads_reduce(local + remote, remote, hmax, hmin, rmax);
    const double changed = objective(a.cm, overlap, rmax.v, hmax.v, s, n);
    if (changed < best) {
      best = changed;
      cnt = s;
    }
  }
  __syncthreads();

  // Replay the accepted prefix to emit its mask and H/R (derive_loads of the result).
  uint8_t* mask = a.mask + (size_t)L * E * E;
  if (active) {
    for (int e = 0; e < E; ++e) mask[(size_t)d * E + e] = (d == e);
  }
  __syncthreads();
  for (int p = 0; p < cnt; ++p) {
    const int i = sel_list[p];
    if (active) smem_col[d] = counts[(size_t)d * E + i];
    __syncthreads();
    if (active && d != i) mask[(size_t)d * E + i] = bottom_rank(smem_col, E, i, d) >= n;
    __syncthreads();
  }
  __threadfence_block();
  __syncthreads();
  if (active) {
    int64_t loc = 0, rem = 0;
    for (int j = 0; j < E; ++j) {
      const int64_t c_dj = counts[(size_t)d * E + j];
      if (mask[(size_t)d * E + j]) loc += c_dj;
      const int64_t c_jd = counts[(size_t)j * E + d];
      if (!mask[(size_t)j * E + d]) rem += c_jd;
    }
    a.H[(size_t)L * E + d] = loc + rem;
    a.R[(size_t)L * E + d] = rem;
    a.selected[(size_t)L * E + d] = d < cnt ? sel_list[d] : -1;
  }
  if (d == 0) {
    a.num_selected[L] = cnt;
    a.num_explored[L] = s;
    a.best_cost[L] = best;
  }
  plan_gate_tick(a.cfg, iter_j);
}

// ---- physically-faithful E > D planner -------------------------
// Generalises Algorithm 1 to m = E / D experts per device (home of e = device e / m,
// physical LoadMatrix rows); reduces to plan_greedy_kernel bit-for-bit when m == 1:
//   * balance threshold alpha * total_inputs / D (planner.py:63-68 has E == D)
//   * i = first argmax(H) is a device; the expert to replicate is its unused home
//     expert that currently sends it the most rows (ties -> lower id); stop when i
//     has none left (planner.py:115-117)
//   * excluded = n non-home devices with the fewest rows of that expert on the
//     original matrix, key (count, index) (planner.py:71-77)
//   * objective = perf_model._build with num_devices = D, strict improvement accepts
// counts may be virtual-slot rows (rows = E, rows / D slots per device): they are
// summed per device on load; the emitted mask has `rows` rows (device row repeated).
struct PhysArgs {
  const int64_t* counts;
  int rows, D, E;
  int refine;
  pp_cost_model cm;
  pp_planner_cfg cfg;
  int32_t* selected;
  int32_t* num_selected;
  int32_t* num_explored;
  uint8_t* mask;
  int64_t* H;
  int64_t* R;
  double* best_cost;
};

__global__ void __launch_bounds__(kMaxPlanThreads) plan_physical_kernel(PhysArgs a) {
  pdl_grid_sync();
  const int L = blockIdx.x;
  const int D = a.D, E = a.E, m = E / D, rpd = a.rows / D;
  const int t = threadIdx.x;
  const int n = a.cfg.n;
  const bool overlap = a.cfg.overlap_aware != 0;
  extern __shared__ int64_t dyn[];
  int64_t* phys = dyn;                                        // [D][E]
  int64_t* sent = phys + (size_t)D * E;                       // [E] rows each expert's home receives
  uint8_t* pmask = reinterpret_cast<uint8_t*>(sent + E);      // [D][E]
  uint8_t* used = pmask + (size_t)D * E;                      // [E]
  __shared__ Red scratch[kMaxWarps];
  __shared__ int32_t sel_list[kMaxPlanThreads];
  __shared__ int cand_e;
  __shared__ uint8_t holder[kMaxPlanThreads];
  __shared__ int32_t rep[kMaxPlanThreads];

  int64_t iter_j = 0;
  if (!plan_gate_open(a.cfg, iter_j)) {  // reuse: keep the previous plan's outputs
    plan_gate_tick(a.cfg, iter_j);
    return;
  }
  if (t < D) {
    holder[t] = 0;
    rep[t] = 0;
  }
  const int64_t* counts = a.counts + (size_t)L * a.rows * E;
  for (int x = t; x < D * E; x += blockDim.x) {
    const int d = x / E, e = x - (x / E) * E;
    int64_t c = 0;
    for (int r = 0; r < rpd; ++r) c += counts[(size_t)(d * rpd + r) * E + e];
    phys[x] = c;
    pmask[x] = (e / m == d);
  }
  for (int e = t; e < E; e += blockDim.x) used[e] = 0;
  __syncthreads();

  int64_t rowsum = 0;
  if (t < D)
    for (int e = 0; e < E; ++e) rowsum += phys[(size_t)t * E + e];
  const int64_t total = block_reduce(Red{rowsum, 0}, SumOp(), scratch).v;
  const int64_t total_inputs = total / a.cm.top_k;
  const double threshold = __ddiv_rn(__dmul_rn(a.cfg.alpha, (double)total_inputs), (double)D);
  const Red neutral_max{INT64_MIN, 0x7fffffff};
  const Red neutral_min{INT64_MAX, 0x7fffffff};

  // H/R of the current pmask: sent[e] by thread e, then device d sums its kept + home rows
  auto loads = [&](int64_t& h, int64_t& r) {
    for (int e = t; e < E; e += blockDim.x) {
      int64_t s = 0;
      for (int d = 0; d < D; ++d)
        if (!pmask[(size_t)d * E + e]) s += phys[(size_t)d * E + e];
      sent[e] = s;
    }
    __syncthreads();
    h = 0;
    r = 0;
    if (t < D) {
      for (int e = 0; e < E; ++e)
        if (pmask[(size_t)t * E + e]) h += phys[(size_t)t * E + e];
      for (int e = t * m; e < (t + 1) * m; ++e) r += sent[e];
      h += r;
    }
  };
  auto reduce3 = [&](int64_t h, int64_t r, Red& hmax, Red& hmin, Red& rmax) {
    const bool act = t < D;
    hmax = block_reduce(act ? Red{h, t} : neutral_max, MaxFirst(), scratch);
    hmin = block_reduce(act ? Red{h, t} : neutral_min, MinOp(), scratch);
    rmax = block_reduce(act ? Red{r, t} : neutral_max, MaxFirst(), scratch);
  };
  // replicate expert e: every non-home device except the n with the fewest rows of e
  auto apply = [&](int e) {
    const int home = e / m;
    if (t < D && t != home) {
      const int64_t c = phys[(size_t)t * E + e];
      int rank = 0;
      for (int j = 0; j < D; ++j) {
        if (j == home || j == t) continue;
        const int64_t cj = phys[(size_t)j * E + e];
        rank += (cj < c) || (cj == c && j < t);
      }
      pmask[(size_t)t * E + e] = rank >= n;
      if (rank >= n) holder[t] = 1;
    }
    __syncthreads();
  };

  int64_t h, r;
  Red hmax, hmin, rmax;
  loads(h, r);
  reduce3(h, r, hmax, hmin, rmax);
  double best = objective(a.cm, overlap, rmax.v, hmax.v, 0, 0);
  int cnt = 0, s = 0;
  while (true) {
    if ((double)(hmax.v - hmin.v) < threshold) break;  // is_balanced
    const int i = hmax.i;
    __syncthreads();
    if (t == 0) {
      int ce = -1;
      for (int e = i * m; e < (i + 1) * m; ++e)
        if (!used[e] && (ce < 0 || sent[e] > sent[ce])) ce = e;
      cand_e = ce;
      if (ce >= 0) {
        used[ce] = 1;
        sel_list[s] = ce;
      }
    }
    __syncthreads();
    const int e = cand_e;
    if (e < 0) break;
    ++s;
    apply(e);
    if (a.cfg.max_replicas > 0 && add_replicas(holder, rep, D, scratch) > a.cfg.max_replicas) {
      --s;  // this prefix needs more replica slots than a device owns: stop before it
      break;
    }
    loads(h, r);
    reduce3(h, r, hmax, hmin, rmax);
    const double changed = objective(a.cm, overlap, rmax.v, hmax.v, s, n);
    if (changed < best) {
      best = changed;
      cnt = s;
    }
  }
  __syncthreads();
  // replay the accepted prefix, emit mask rows / H / R / selected
  for (int x = t; x < D * E; x += blockDim.x) pmask[x] = ((x - (x / E) * E) / m == x / E);
  __syncthreads();
  for (int p = 0; p < cnt; ++p) apply(sel_list[p]);
  loads(h, r);
  if (t < D) {
    a.H[(size_t)L * D + t] = h;
    a.R[(size_t)L * D + t] = r;
  }
  uint8_t* mask = a.mask + (size_t)L * a.rows * E;
  for (int x = t; x < a.rows * E; x += blockDim.x) {
    const int v = x / E, e = x - (x / E) * E;
    mask[x] = pmask[(size_t)(v / rpd) * E + e];
  }
  for (int e = t; e < E; e += blockDim.x) a.selected[(size_t)L * E + e] = e < cnt ? sel_list[e] : -1;
  if (t == 0) {
    a.num_selected[L] = cnt;
    a.num_explored[L] = s;
    a.best_cost[L] = best;
  }
  if (!a.refine || rpd < 2) {
    plan_gate_tick(a.cfg, iter_j);
    return;
  }
  // Opt-in slot refinement (not in the paper; oracle refine_slots): the heaviest device h
  // un-routes the (slot v of h, non-home expert e) batch that minimises
  // max(H[h] - C[v][e], H[home e] + C[v][e]) while that is below H[h]; ties -> lower v, e.
  // Works on the emitted slot mask in global memory.
  int64_t* Hs = sent;  // [D] device loads of the current slot mask (E >= D)
  const int rows = a.rows;
  auto slot_loads = [&](int64_t& hh, int64_t& rr) {
    __syncthreads();
    hh = 0;
    rr = 0;
    if (t < D) {
      for (int v = t * rpd; v < (t + 1) * rpd; ++v)
        for (int e = 0; e < E; ++e)
          if (mask[(size_t)v * E + e]) hh += counts[(size_t)v * E + e];
      for (int e = t * m; e < (t + 1) * m; ++e)
        for (int v = 0; v < rows; ++v)
          if (!mask[(size_t)v * E + e]) rr += counts[(size_t)v * E + e];
      hh += rr;
      Hs[t] = hh;
    }
    __syncthreads();
  };
  // loads once, then updated incrementally: un-routing batch (v, e) of c rows moves c from
  // device hd (computed locally) to e's home (received + computed there)
  {
    int64_t hh, rr;
    slot_loads(hh, rr);
  }
  for (int iter = 0; iter < rows * E; ++iter) {
    const Red hm = block_reduce(t < D ? Red{Hs[t], t} : neutral_max, MaxFirst(), scratch);
    const int hd = hm.i;
    Red cand{INT64_MAX, 0x7fffffff};
    for (int x = t; x < rpd * E; x += blockDim.x) {
      const int v = hd * rpd + x / E, e = x - (x / E) * E;
      const int64_t c = counts[(size_t)v * E + e];
      if (!mask[(size_t)v * E + e] || e / m == hd || c == 0) continue;
      const int64_t lo = hm.v - c, hi = Hs[e / m] + c;
      const int64_t val = lo > hi ? lo : hi;
      if (val >= hm.v) continue;
      const int64_t key = (val << 20) | (int64_t)(v * E + e);
      if (key < cand.v) cand.v = key;
    }
    cand = block_reduce(cand, MinOp(), scratch);
    if (cand.v == INT64_MAX) break;
    if (t == 0) {
      const int cell = (int)(cand.v & ((1 << 20) - 1));
      const int64_t c = counts[cell];
      mask[cell] = 0;
      Hs[hd] -= c;
      Hs[(cell % E) / m] += c;
    }
    __syncthreads();
  }
  int64_t hh, rr;
  slot_loads(hh, rr);
  if (t < D) {
    a.H[(size_t)L * D + t] = hh;
    a.R[(size_t)L * D + t] = rr;
  }
  plan_gate_tick(a.cfg, iter_j);
}

__global__ void derive_loads_kernel(const int64_t* counts, const uint8_t* mask, int D, int E,
                                    int64_t* H, int64_t* R) {
  pdl_grid_sync();
  for (int x = threadIdx.x; x < D; x += blockDim.x) {
    int64_t loc = 0, rem = 0;
    for (int e = 0; e < E; ++e)
      if (mask[(size_t)x * E + e]) loc += counts[(size_t)x * E + e];
    if (x < E) {
      for (int j = 0; j < D; ++j)
        if (!mask[(size_t)j * E + x]) rem += counts[(size_t)j * E + x];
    }
    H[x] = loc + rem;
    R[x] = rem;
  }
}

// top-m baseline policy (reference simulator._top_m_placement, simulator.py:318-324):
// the m experts with the largest column totals (ties -> lower index) go to every
// device (empty excluded sets); all other experts stay home.
__global__ void top_m_mask_kernel(const int64_t* counts, int D, int E, int m_top, uint8_t* mask,
                                  int32_t* selected) {
  pdl_grid_sync();
  extern __shared__ int64_t tot[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int64_t s = 0;
    for (int d = 0; d < D; ++d) s += counts[(size_t)d * E + e];
    tot[e] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int rank = 0;  // position in the order (-total, e)
    for (int j = 0; j < E; ++j) rank += (tot[j] > tot[e]) || (tot[j] == tot[e] && j < e);
    const bool chosen = rank < m_top;
    if (chosen && selected) selected[rank] = e;
    for (int d = 0; d < D; ++d) mask[(size_t)d * E + e] = chosen || d == e;
  }
}

}  // namespace pp

using namespace pp;

extern "C" int pp_top_m_mask(const int64_t* counts, int32_t D, int32_t E, int32_t m_top,
                             uint8_t* mask, int32_t* selected, void* stream) {
  PP_CHECK_ARG(counts && mask && D >= E && E >= 1 && E <= 4096, "pp_top_m_mask: bad arguments");
  PP_CHECK_ARG(m_top >= 1 && m_top <= E, "top-m policy needs 1 <= m <= E, got %d", m_top);
  PP_CUDA_TRY(pdl_launch(top_m_mask_kernel, dim3(1), dim3(256), sizeof(int64_t) * E, as_stream(stream), counts, D, E, m_top, mask, selected));
  PP_LAUNCH_CHECK();
  return PP_OK;
}

extern "C" int pp_plan_greedy(const int64_t* counts, int32_t num_layers, int32_t E,
                              const pp_cost_model* cm, const pp_planner_cfg* cfg,
                              int32_t* selected, int32_t* num_selected, int32_t* num_explored,
                              uint8_t* mask, int64_t* H, int64_t* R, double* best_cost,
                              void* stream) {
  PP_CHECK_ARG(counts && cm && cfg && selected && num_selected && num_explored && mask && H && R &&
                   best_cost,
               "pp_plan_greedy: null pointer");
  PP_CHECK_ARG(num_layers >= 1, "pp_plan_greedy: num_layers must be >= 1, got %d", num_layers);
  PP_CHECK_ARG(E >= 1 && E <= kMaxPlanThreads, "pp_plan_greedy: E must be in [1, %d], got %d",
               kMaxPlanThreads, E);
  if (cm->num_devices != E || cm->num_experts != E)
    return fail(PP_EDIM, "pp_plan_greedy: cost model is %dx%d, load is %dx%d", cm->num_devices,
                cm->num_experts, E, E);
  PP_CHECK_ARG(cfg->n >= 0 && cfg->n < E, "n must be < num_devices=%d, got %d", E, cfg->n);
  PP_CHECK_ARG(cm->top_k >= 1, "top_k must be >= 1");
  PP_CHECK_ARG(cfg->reuse_interval >= 1, "reuse_interval must be >= 1, got %d", cfg->reuse_interval);
  PP_CHECK_ARG(cfg->max_replicas >= 0 && cfg->slots_per_rank >= 0, "pp_plan_greedy: bad replica bound");
  PlanArgs a{counts, E, *cm, *cfg, selected, num_selected, num_explored, mask, H, R, best_cost};
  const int threads = ((E + 31) / 32) * 32;
  PP_CUDA_TRY(pdl_launch(plan_greedy_kernel, dim3(num_layers), dim3(threads), sizeof(int64_t) * E, as_stream(stream), a));
  PP_LAUNCH_CHECK();
  return PP_OK;
}

extern "C" int pp_plan_physical(const int64_t* counts, int32_t num_layers, int32_t rows, int32_t D,
                                int32_t E, const pp_cost_model* cm, const pp_planner_cfg* cfg,
                                int32_t refine_slots, int32_t* selected, int32_t* num_selected, int32_t* num_explored,
                                uint8_t* mask, int64_t* H, int64_t* R, double* best_cost,
                                void* stream) {
  PP_CHECK_ARG(counts && cm && cfg && selected && num_selected && num_explored && mask && H && R &&
                   best_cost,
               "pp_plan_physical: null pointer");
  PP_CHECK_ARG(num_layers >= 1, "pp_plan_physical: num_layers must be >= 1, got %d", num_layers);
  PP_CHECK_ARG(D >= 1 && E >= D && E % D == 0 && E <= kMaxPlanThreads,
               "pp_plan_physical: need E a multiple of D and E <= %d (D=%d, E=%d)", kMaxPlanThreads, D, E);
  PP_CHECK_ARG((int64_t)D * E <= 4096, "pp_plan_physical: D*E must be <= 4096, got %d", D * E);
  PP_CHECK_ARG(rows >= D && rows % D == 0, "pp_plan_physical: rows (%d) must be a multiple of D (%d)", rows, D);
  if (cm->num_devices != D || cm->num_experts != E)
    return fail(PP_EDIM, "pp_plan_physical: cost model is %dx%d, load is %dx%d", cm->num_devices,
                cm->num_experts, D, E);
  PP_CHECK_ARG(cfg->n >= 0 && cfg->n < D, "n must be < num_devices=%d, got %d", D, cfg->n);
  PP_CHECK_ARG(cm->top_k >= 1, "top_k must be >= 1");
  PP_CHECK_ARG(cfg->reuse_interval >= 1, "reuse_interval must be >= 1, got %d", cfg->reuse_interval);
  PP_CHECK_ARG(cfg->max_replicas >= 0, "pp_plan_physical: bad replica bound");
  PP_CHECK_ARG(!refine_slots || (int64_t)rows * E <= (1 << 20),
               "pp_plan_physical: slot refinement needs rows*E <= 2^20");
  PhysArgs a{counts, rows, D, E, refine_slots ? 1 : 0, *cm, *cfg, selected, num_selected, num_explored,
             mask, H, R, best_cost};
  const int threads = ((E + 31) / 32) * 32;
  const size_t smem = sizeof(int64_t) * ((size_t)D * E + E) + (size_t)D * E + E;
  PP_CUDA_TRY(pdl_launch(plan_physical_kernel, dim3(num_layers), dim3(threads), smem, as_stream(stream), a));
  PP_LAUNCH_CHECK();
  return PP_OK;
}

extern "C" int pp_derive_loads(const int64_t* counts, const uint8_t* mask, int32_t D, int32_t E,
                               int64_t* H, int64_t* R, void* stream) {
  PP_CHECK_ARG(counts && mask && H && R, "pp_derive_loads: null pointer");
  PP_CHECK_ARG(D >= 1 && E >= 1, "pp_derive_loads: empty dims");
  if (E > D) return fail(PP_EDIM, "pp_derive_loads: identity homes need E <= D (E=%d, D=%d)", E, D);
  PP_CUDA_TRY(pdl_launch(derive_loads_kernel, dim3(1), dim3(256), 0, as_stream(stream), counts, mask, D, E, H, R));
  PP_LAUNCH_CHECK();
  return PP_OK;
}
