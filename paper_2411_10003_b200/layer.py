"""Expert-parallel MoE layer with Pro-Prophet planning, B200-native.

The reference (``moebal``) never executes this layer: it prices it with
Eq. 1-7 (``perf_model.py:36-107``) from a LoadMatrix (``core.py:88-142``)
and a placement (``core.py:145-222``).  Here the layer runs for real, and
the reference's objects are its interface:

  forward  (per rank, stream-ordered, no host sync)
    K1 pp_route_topk       gate GEMM on tcgen05 + softmax/top-k/chunk ranks
       pp_slot_histogram   this rank's virtual-slot rows of the LoadMatrix, stored
                           into every rank's copy (peer stores) + barrier
    K3 pp_dispatch_layout  receive layout from LoadMatrix + replica mask
    K3 pp_dispatch         permute + all-to-all in one kernel (peer stores)
       barrier
    K5 pp_replica_trans    (D>1) copy engine: replicas pull before the barrier;
                           SM engine: homes push W1/W2 + completion flags
    K4 FWD1, FWD2          grouped tcgen05 GEMMs (GeLU fused); replica tiles gated
                           on the Trans flags; FWD2 may push rows straight to the
                           pairs' owners (fused A2A)
       barrier
    K3 pp_combine          weighted gather back (peer loads, or local after fused A2A)
    K2 pp_plan_greedy /    (D>1, side stream) plan for iteration j+1 on this
       pp_plan_physical    iteration's LoadMatrix (plan_for_iteration rule)
  backward mirrors it: combine_bwd (push; also dL/dlogits), gate dW (deterministic
  split-K) and gate dX (tcgen05, writes dx), WGRAD2/DGRAD2/WGRAD1/DGRAD1 (order depends
  on the replica engine), then pp_dispatch_bwd adds the expert-input grads, K5 Agg (D>1).

Virtual expert slots: with m = E/D experts per rank, each
rank's T tokens are cut into m contiguous slots; slot v = rank*m + j is a
planner "device", so the reference planner (which needs E == D,
``planner.py:88-90``) applies unmodified to an E x E LoadMatrix.

Weight layout per rank: arenas W1 [slots, f, d] and W2 [slots, d, f] (bf16),
slots 0..m-1 = home experts (expert rank*m + j), then replica slots.  Gradients
are fp32 ``main_grad`` arenas of the same shape (Megatron-style: the bf16
parameters get no ``.grad``; read ``layer.w1_main_grad`` etc.).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch
import torch.distributed as dist

from . import _device, _lib, memory
from .core import ClusterSpec, LoadMatrix, ModelSpec, ValidationError, replica_sets, replica_transfers
from .planner import PlannerConfig


def layer_plan(d_model: int, d_ff: int, num_experts: int, top_k: int, tokens: int, world: int,
               capacity_factor: float | None = None, capacity_rows: int | None = None,
               max_replicas: int | None = None, replica_engine: str = "copy", planning: str = "host",
               policy: str | None = None, fused_a2a: bool = False) -> dict:
    """Allocation rule of one MoELayer (shared by MoELayer and MoEStack's Workspace)."""
    E, D = num_experts, world
    m = E // D
    reps = (E - m) if max_replicas is None else int(max_replicas)
    if reps < 0:
        raise ValidationError(f"max_replicas must be >= 0, got {max_replicas}")
    if str(policy or "").startswith("top") and policy[3:].isdigit() and D > 1 and int(policy[3:]) > reps:
        raise ValidationError(f"policy {policy} needs max_replicas >= {int(policy[3:])}, got {reps}")
    slots = m + (reps if D > 1 else 0)
    max_groups = min(256, m + reps)
    try:
        rows = memory.rows_capacity(tokens, top_k, E, D, capacity_factor, capacity_rows)
    except ValueError as exc:
        raise ValidationError(str(exc)) from None
    sm_engine = D > 1 and (replica_engine == "sm" or planning == "device" or str(policy or "").startswith("top"))
    plan = memory.buffer_plan(d_model, d_ff, E, top_k, tokens, D, rows, slots, max_groups,
                              fused_a2a=bool(fused_a2a), sm_engine=sm_engine)
    return {"plan": plan, "rows_cap": rows, "slots": slots, "max_groups": max_groups, "max_replicas": reps,
            "sm_engine": sm_engine}


class Workspace:
    """Buffers that live only inside one block's backward (memory.buffer_plan scope
    "shared"/"shared2"): dYp / dXp (peer-mapped), dL/dw, dL/dlogits, the gate dW split-K
    partials, and the Agg staging (two copies when blocks share it: ``agg_copies``).
    One per MoEStack; a standalone MoELayer builds its own.  Collective at D > 1."""

    def __init__(self, plan, group, device, agg_copies: int = 1) -> None:
        b = {x.name: x for x in plan}
        self._shapes = {n: b[n].shape for n in ("dyp", "dxp", "dw", "dlogits", "gate_ws")}
        self.dyp = PeerBuffer(b["dyp"].shape, torch.bfloat16, group, device)
        self.dxp = PeerBuffer(b["dxp"].shape, torch.bfloat16, group, device)
        self.dw = torch.empty(b["dw"].shape, dtype=torch.float32, device=device)
        self.dlogits = torch.zeros(b["dlogits"].shape, dtype=torch.bfloat16, device=device)
        self.gate_ws = torch.empty(b["gate_ws"].shape, dtype=torch.float32, device=device).view(-1)
        self.agg_stage = []
        if "agg_stage" in b:
            self._shapes["agg_stage"] = b["agg_stage"].shape
            self.agg_stage = [PeerBuffer(b["agg_stage"].shape, torch.float32, group, device) for _ in range(agg_copies)]

    def check(self, plan) -> None:
        b = {x.name: x for x in plan}
        for n, shp in self._shapes.items():
            if n not in b or tuple(b[n].shape) != tuple(shp):
                raise ValidationError(f"workspace buffer {n} {shp} does not fit this layer")

    def close(self) -> None:
        for x in (self.dyp, self.dxp, *self.agg_stage):
            x.close()
        self.agg_stage = []


class CapacityError(RuntimeError):
    """A step needed more receive rows / replica slots than the layer allocated."""


class _CAI:
    def __init__(self, ptr: int, nbytes: int) -> None:
        self.__cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3, "strides": None,
        }


def _wrap(ptr: int, nbytes: int, dtype, shape) -> torch.Tensor:
    raw = torch.as_tensor(_CAI(ptr, nbytes), device="cuda")
    return raw.view(dtype).view(shape)


class PeerBuffer:
    """One symmetric buffer: this rank's allocation + a device table of every
    rank's mapping of its peer (CUDA IPC over NVLink).  At D == 1 it is a
    plain local tensor and a one-entry table."""

    def __init__(self, shape, dtype, group, device) -> None:
        self.shape = tuple(shape)
        self.dtype = dtype
        nbytes = int(np.prod(self.shape)) * torch.empty((), dtype=dtype).element_size()
        self.world = dist.get_world_size(group) if group is not None else 1
        self.rank = dist.get_rank(group) if group is not None else 0
        self._owned = None
        self._imported = []
        if self.world == 1:
            self.local = torch.zeros(self.shape, dtype=dtype, device=device)
            ptrs = [self.local.data_ptr()]
        else:
            lib = _lib.load()
            p = ctypes.c_void_p()
            _lib.check(lib.pp_device_alloc(nbytes, ctypes.byref(p)), "pp_device_alloc")
            self._owned = p.value
            self.local = _wrap(self._owned, nbytes, dtype, self.shape)
            self.local.zero_()
            h = (ctypes.c_uint8 * 64)()
            _lib.check(lib.pp_ipc_export(self._owned, h), "pp_ipc_export")
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(h), group=group)
            ptrs = []
            for r, hb in enumerate(handles):
                if r == self.rank:
                    ptrs.append(self._owned)
                    continue
                q = ctypes.c_void_p()
                hh = (ctypes.c_uint8 * 64).from_buffer_copy(hb)
                _lib.check(lib.pp_ipc_import(hh, ctypes.byref(q)), "pp_ipc_import")
                self._imported.append(q.value)
                ptrs.append(q.value)
        self.ptr_list = list(ptrs)  # host copy of the table (copy-engine Trans/Agg)
        self.ptrs = torch.tensor(ptrs, dtype=torch.int64, device=device)

    def close(self) -> None:
        lib = _lib.load()
        for q in self._imported:
            lib.pp_ipc_close(q)
        self._imported = []
        if self._owned is not None:
            lib.pp_device_free(self._owned)
            self._owned = None


class _Barrier:
    """Device barrier over peer memory (pp_peer_barrier: signal words, spin with a 20 s trap).
    host=True (ranks sharing one GPU): a host barrier instead -- drain the device, then
    dist.barrier -- so no kernel ever spins on another process's progress (on a shared GPU
    that would depend on the driver preempting the spinning kernel)."""

    def __init__(self, group, device, host: bool = False) -> None:
        self.world = dist.get_world_size(group) if group is not None else 1
        self.rank = dist.get_rank(group) if group is not None else 0
        self.group, self.host = group, host
        if self.world > 1:
            self.sig = PeerBuffer((self.world + 2,), torch.int64, group, device)  # signals, epoch, fault
            torch.cuda.synchronize()
            dist.barrier(group=group)

    def close(self) -> None:
        if self.world > 1:
            self.sig.close()

    def __call__(self, stream=None) -> None:
        if self.world == 1:
            return
        if self.host:
            torch.cuda.synchronize()
            dist.barrier(group=self.group)
            return
        # epoch 0: the kernel advances a device-side counter, so captured graphs replay correctly
        _lib.call("pp_peer_barrier", self.sig.ptrs.data_ptr(), self.world, self.rank, 0,
                  _device.stream_ptr(stream))


def default_specs(E: int, k: int, d: int, f: int, tokens_total: int, fnec: float = 0.0,
                  bnec: float = 0.0, avg_bandwidth: float = 450e9, throughput: float | None = None):
    """Cost-model constants for the virtual-slot planner of one layer.

    input_bytes = one routed row (d bf16); param bytes = W1+W2 bf16; grad
    bytes = fp32 grads.  compute_throughput defaults to the pairs/s of one
    B200 slot at ~1.2 PFLOP/s (6*d*f flops per pair fwd) split over m slots
    -- calibrate from a measured run."""
    if throughput is None:
        throughput = 1.2e15 / (6.0 * d * f)
    cluster = ClusterSpec(num_devices=max(E, 2), avg_bandwidth=avg_bandwidth, compute_throughput=throughput)
    model = ModelSpec(num_experts=max(E, 2), num_blocks=1, top_k=k, input_bytes=2 * d,
                      expert_param_bytes=2 * 2 * d * f, expert_grad_bytes=2 * 4 * d * f,
                      fnec_time=fnec, bnec_time=bnec)
    return cluster, model


class MoELayer(torch.nn.Module):
    """Pro-Prophet EP MoE layer (GeLU FFN experts, top-k softmax gate).

    Args:
      d_model, d_ff, num_experts, top_k: layer shape (E % world == 0).
      tokens: tokens per rank per call (multiple of (E/world)*128).
      group: torch.distributed process group spanning the EP ranks (None = 1 GPU).
      planner: PlannerConfig (n, alpha, reuse_interval, overlap_aware); planning
        runs only when world > 1 (ClusterSpec needs D >= 2).
      cluster/model: cost-model specs for the planner (default: default_specs).
      capacity_rows: receive-buffer rows (default: worst case world*tokens*k + E*128,
        i.e. no token is ever dropped).
      capacity_factor: alternative to capacity_rows: ceil(factor*tokens*k) + E*128 rows
        (the rows a rank computes under a balanced plan are ~tokens*k).  A step whose layout
        needs more rows on any rank is dropped on every rank (zero outputs, nothing written
        out of bounds) and the layer raises CapacityError on its next call or on
        ``check_status()``.
      max_replicas: replica weight slots per rank (default E - m: any plan fits).
      replica_engine: "copy" (copy-engine peer copies, host-derived from the plan) or
        "sm" (NVLink pushes from SMs, fully device-driven).
      policy: None/"greedy"/"greedy-overlap" (Pro-Prophet), "vanilla", "top<m>".
      planning: "host" (plan mask read back asynchronously) or "device" (plan stays on
        the GPU; forces the SM engine; the whole step is CUDA-graph capturable at any N).
      placement: "virtual" (reference search over E x E virtual slots, bit-exact) or
        "physical" (E = m*D generalisation, pp_plan_physical).
      refine_slots: physical placement only -- slot-level refinement of the plan.
      fused_a2a: combine / dispatch backward fused into the FWD2 / DGRAD1 epilogues.
    """

    def __init__(self, d_model: int, d_ff: int, num_experts: int, top_k: int, tokens: int,
                 group=None, planner: PlannerConfig | None = None, cluster=None, model=None,
                 capacity_rows: int | None = None, max_replicas: int | None = None,
                 seed: int = 0, device=None, trans_ctas: int = 16, replica_engine: str = "copy",
                 policy: str | None = None, planning: str = "host", placement: str = "virtual",
                 refine_slots: bool = False, fused_a2a: bool = False,
                 capacity_factor: float | None = None, workspace: "Workspace | None" = None) -> None:
        super().__init__()
        if not torch.cuda.is_available():
            raise RuntimeError("MoELayer needs a CUDA device (B200); there is no CPU path")
        _lib.load()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.group = group
        self.world = dist.get_world_size(group) if (group is not None and dist.is_initialized()) else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        if self.world == 1:
            self.group = None
        E, D = num_experts, self.world
        # ranks sharing one GPU (the 1-GPU parity runs): host-synchronised barriers, Trans
        # awaited before FWD1 instead of per-tile gates -- nothing spins on another process
        self.shared_device = False
        if D > 1:
            ids = [None] * D
            dist.all_gather_object(ids, str(torch.cuda.get_device_properties(self.device).uuid), group=self.group)
            self.shared_device = len(set(ids)) < D
        if E % D:
            raise ValidationError(f"num_experts={E} must be a multiple of the EP world size {D}")
        self.d, self.f, self.E, self.k, self.T = d_model, d_ff, E, top_k, tokens
        self.m = E // D
        if tokens % (self.m * _lib.PP_CHUNK):
            raise ValidationError(f"tokens={tokens} must be a multiple of (E/D)*{_lib.PP_CHUNK}={self.m * _lib.PP_CHUNK}")
        if d_model % 256 or d_ff % 256:
            raise ValidationError("d_model and d_ff must be multiples of 256")
        self.planner_cfg = planner or PlannerConfig()
        if cluster is None or model is None:
            cluster, model = default_specs(E, top_k, d_model, d_ff, tokens * D)
        self.cluster, self.model = cluster, model
        # the HBM plan (memory.buffer_plan) this layer allocates from; buffers that live only
        # inside one block's backward come from a Workspace, shared by the blocks of a stack
        lp = layer_plan(d_model, d_ff, E, top_k, tokens, D, capacity_factor=capacity_factor,
                        capacity_rows=capacity_rows, max_replicas=max_replicas, replica_engine=replica_engine,
                        planning=planning, policy=policy, fused_a2a=fused_a2a)
        self.max_replicas, self.slots, self.max_groups, self.rows_cap = (
            lp["max_replicas"], lp["slots"], lp["max_groups"], lp["rows_cap"])
        self.buffer_plan = lp["plan"]
        dev = self.device
        if workspace is None:
            workspace = Workspace(self.buffer_plan, self.group, dev)
            self._own_workspace = True
        else:
            workspace.check(self.buffer_plan)
            self._own_workspace = False
        self.workspace = workspace
        g = torch.Generator(device="cpu").manual_seed(seed)

        # ---- parameters (bf16) in peer-visible arenas -------------------------
        self.w1_arena = PeerBuffer((self.slots, d_ff, d_model), torch.bfloat16, self.group, dev)
        self.w2_arena = PeerBuffer((self.slots, d_model, d_ff), torch.bfloat16, self.group, dev)
        self.g1_arena = PeerBuffer((self.slots, d_ff, d_model), torch.float32, self.group, dev)
        self.g2_arena = PeerBuffer((self.slots, d_model, d_ff), torch.float32, self.group, dev)
        w1_all = torch.randn((E, d_ff, d_model), generator=g) / math.sqrt(d_model)
        w2_all = torch.randn((E, d_model, d_ff), generator=g) / math.sqrt(d_ff)
        wg = torch.randn((E, d_model), generator=g) / math.sqrt(d_model)
        lo = self.rank * self.m
        with torch.no_grad():
            self.w1_arena.local[: self.m].copy_(w1_all[lo: lo + self.m].to(torch.bfloat16))
            self.w2_arena.local[: self.m].copy_(w2_all[lo: lo + self.m].to(torch.bfloat16))
        self.w1 = torch.nn.Parameter(self.w1_arena.local[: self.m], requires_grad=True)
        self.w2 = torch.nn.Parameter(self.w2_arena.local[: self.m], requires_grad=True)
        self.wg = torch.nn.Parameter(wg.to(dev, torch.bfloat16))
        self.w1.main_grad = self.g1_arena.local[: self.m]
        self.w2.main_grad = self.g2_arena.local[: self.m]
        self.wg.main_grad = torch.zeros((E, d_model), dtype=torch.float32, device=dev)
        self.register_buffer("gate_bias", torch.zeros(E, dtype=torch.float32, device=dev))

        # ---- routing / layout workspaces --------------------------------------
        T, k, C = tokens, top_k, tokens // _lib.PP_CHUNK
        i32 = dict(dtype=torch.int32, device=dev)
        self.idx = torch.empty((T, k), **i32)
        self.rank_in_chunk = torch.empty((T, k), **i32)
        self.w = torch.empty((T, k), dtype=torch.float32, device=dev)
        self.probs = torch.empty((T, E), dtype=torch.float32, device=dev)
        self.chunk_counts = torch.empty((C, E), **i32)
        self.counts_buf = PeerBuffer((E, E), torch.int64, self.group, dev)  # virtual-slot LoadMatrix
        self.counts = self.counts_buf.local
        self.chunk_base = torch.empty((C, E), **i32)
        self.slot_dest = torch.empty((self.m, E), **i32)
        self.groups = torch.zeros((self.max_groups, 8), **i32)
        self.num_groups = torch.zeros((1,), **i32)
        self.total_rows = torch.zeros((1,), **i32)
        self.seg_start = torch.empty((D, E), **i32)
        self.rep_slot = torch.full((D, E), -1, **i32)
        # layout status (sticky bits: 1 rows > capacity, 2 replica slots, 4 groups), read
        # back asynchronously after every eager forward
        self.status = torch.zeros((1,), **i32)
        self._status_host = torch.zeros((1,), dtype=torch.int32).pin_memory()
        self._fault_host = torch.zeros((3,), dtype=torch.int64).pin_memory()  # cross-rank fault words
        self._status_ev = None
        self.pair_dest = torch.empty((T, k), **i32)
        self.pair_row = torch.empty((T, k), **i32)
        self.EP = 64 if E <= 64 else 128
        ws_bytes = _lib.load().pp_gate_dw_workspace_bytes(T, d_model)
        if ws_bytes < 0 or ws_bytes != workspace.gate_ws.numel() * 4:
            raise ValidationError(f"gate backward: unsupported T={T} / d_model={d_model}")
        # transient backward buffers (shared): dL/dw, dL/dlogits, dWg split-K partials, dYp, dXp
        self.dw, self.dlogits, self.gate_ws = workspace.dw, workspace.dlogits, workspace.gate_ws
        self.dyp, self.dxp = workspace.dyp, workspace.dxp
        # ---- expert activations ---------------------------------------------
        R = self.rows_cap
        self.xp = PeerBuffer((R, d_model), torch.bfloat16, self.group, dev)
        self.yp = PeerBuffer((R, d_model), torch.bfloat16, self.group, dev)
        # fused A2A (FWD2 -> combine, DGRAD1 -> dispatch backward in the GEMM epilogue):
        # pp_dispatch records each received row's origin pair; the epilogues push results
        # straight into the owning rank's comb [T*k][d] (pair order), read locally after
        self.fused_a2a = bool(fused_a2a)
        self.origin = PeerBuffer((R,), torch.int32, self.group, dev) if self.fused_a2a else None
        self.comb = PeerBuffer((tokens * top_k, d_model), torch.bfloat16, self.group, dev) if self.fused_a2a else None
        self.pre = torch.zeros((R, d_ff), dtype=torch.bfloat16, device=dev)
        self.act = torch.zeros((R, d_ff), dtype=torch.bfloat16, device=dev)
        # ---- planning state -------------------------------------------------
        self.iteration = 0
        self.plan_enabled = D > 1
        self.mask_cur = None  # None = vanilla EP for iteration 0
        self._plan_out = _device.PlanBuffers(1, E, dev) if self.plan_enabled else None
        if self._plan_out is not None:  # a skipped (reused) search leaves the previous mask: start at vanilla EP
            self._plan_out.mask.copy_(torch.eye(E, dtype=torch.uint8, device=dev).view(1, E, E))
        # placement "virtual": the reference search, bit-exact, over E x E virtual expert
        # slots; "physical": the opt-in E = m*D generalisation over D devices (pp_plan_physical,
        # SURVEY 8(f) row 4) -- its [E][E] output mask repeats each device row over its slots
        if placement not in ("virtual", "physical"):
            raise ValidationError(f"placement must be 'virtual' or 'physical', got {placement!r}")
        self.placement = placement
        # opt-in (physical placement only; beyond the paper): a replica holder may keep
        # sending some of its token slots to the expert's home when that lowers the
        # heaviest device's rows (pp_plan_physical refine_slots, oracle refine_slots)
        if refine_slots and placement != "physical":
            raise ValidationError("refine_slots needs placement='physical'")
        self.refine_slots = bool(refine_slots) and self.m > 1
        self._cm = _device.cost_model(self.cluster, self.model, E) if self.plan_enabled else None
        if self._cm is not None and placement == "physical":
            if self.planner_cfg.n >= D:
                raise ValidationError(f"physical placement needs planner n < world size {D}, got {self.planner_cfg.n}")
            self._cm.num_devices = D
        # replica bound inside the search (only when max_replicas < E - m can bind); with
        # planning="device" the reuse policy is gated on a device iteration counter, so a
        # captured step that launches the planner every iteration still re-plans every F
        self._plan_ctr = torch.zeros(2, dtype=torch.int64, device=dev)
        bound = self.max_replicas if self.max_replicas < E - self.m else 0
        self._pcfg = _device.planner_cfg(
            self.planner_cfg, max_replicas=bound, slots_per_rank=self.m if placement == "virtual" else 1,
            iter_counter=self._plan_ctr if planning == "device" else None)
        self.plan_stream = torch.cuda.Stream(device=dev) if self.plan_enabled else None
        self.comm_stream = torch.cuda.Stream(device=dev) if D > 1 else None
        self.trans_ctas = trans_ctas  # SM-engine Trans pushes
        # SM engine: True = Trans issued after barrier 1, overlapping FWD1/FWD2 on the home
        # experts with the replica tiles gated on completion flags; False = issued at the
        # start of the forward and awaited before barrier 1
        self.trans_gate = not self.shared_device
        # SM-engine Agg runs beside the backward GEMMs on agg_ctas SMs (one CTA per SM);
        # those GEMMs launch their persistent grids on the remaining SMs so neither waits
        # for the other (pushes reach NVLink rate from ~16 CTAs)
        self.agg_ctas = 16
        self.agg_ctas_w2 = 16  # the W2 half has DGRAD2 + WGRAD1 to hide under: may use fewer SMs
        # the W1 half's home-side reduce of the last layer to run backward (a single layer, or
        # block 0 of a stack: block_index, set by MoEStack) tails the iteration with no GEMM after
        # DGRAD1 to disturb: it takes a full grid (its CTAs fill the SMs DGRAD1 frees) instead of
        # agg_ctas SMs.  Models that chain their own MoELayers should give the later-running
        # layers block_index > 0 (or set agg_tail_reduce_ctas = agg_ctas) so a persistent GEMM
        # that follows never finds its SMs taken.
        self.agg_tail_reduce_ctas = 2 * _device.num_sms(dev)
        # SMs the GEMMs leave to Trans / Agg per replica this rank sends or receives (device-side,
        # clamped to [2, trans_ctas / agg_ctas])
        self.res_per_replica = 4
        if replica_engine not in ("copy", "sm"):
            raise ValidationError(f"replica_engine must be 'copy' or 'sm', got {replica_engine!r}")
        # 'copy': Trans/Agg pulls run on the copy engines (cudaMemcpyAsync over NVLink,
        # no SMs taken from the GEMMs); 'sm': device-driven pull kernels (no host
        # knowledge of the plan needed)
        self.replica_engine = replica_engine
        # policy (reference simulator.py:54-103): None/"greedy"/"greedy-overlap" = Pro-Prophet
        # planner (overlap_aware from `planner`), "vanilla" = plain EP, "top<m>" = the m
        # heaviest experts of the CURRENT iteration broadcast to every rank (device-side mask)
        self.top_m = 0
        if policy is not None and policy not in ("greedy", "greedy-overlap"):
            if policy == "vanilla":
                self.plan_enabled = False
            elif policy.startswith("top") and policy[3:].isdigit() and int(policy[3:]) >= 1:
                self.plan_enabled = False
                self.top_m = int(policy[3:])
                self.replica_engine = "sm"  # the mask only exists on the device mid-forward
                self._topm_mask = torch.zeros((E, E), dtype=torch.uint8, device=dev)
            else:
                raise ValidationError(f"unknown policy {policy!r}; valid: vanilla, top<m>, greedy, greedy-overlap")
        self.policy = policy or ("greedy-overlap" if self.planner_cfg.overlap_aware else "greedy")
        # planning "host": the plan's mask is read back asynchronously and the host issues
        # copy-engine Trans/Agg; "device": the plan stays on the device (mask double-buffered,
        # SM-driven Trans/Agg) so a whole step -- barriers included -- is CUDA-graph capturable
        if planning not in ("host", "device"):
            raise ValidationError(f"planning must be 'host' or 'device', got {planning!r}")
        self.planning = planning
        self._plan_done_dev = None
        if planning == "device" and D > 1:
            self.replica_engine = "sm"
            self.mask_buf = torch.eye(E, dtype=torch.uint8, device=dev)
            self._counts_snap = torch.zeros((E, E), dtype=torch.int64, device=dev)
            if self.plan_enabled:
                self.mask_cur = self.mask_buf  # identity = vanilla EP until the first plan lands
        # SM-engine Agg: replicas push their grads into the home's staging area
        # [m][D-1][W1|W2][d*f] fp32, the home sums them in rank order after a barrier on
        # the comm stream (its own barrier object: its epochs advance on that stream)
        self.trans_flags = None
        if D > 1 and self.replica_engine == "sm":
            if not workspace.agg_stage:
                raise ValidationError("the workspace has no Agg staging (built for another replica engine)")
            # Trans completion flags (slot r written by rank r) + the pushers' CTA counter
            self.trans_flags = PeerBuffer((2, D), torch.int64, self.group, dev)  # rows: W1, W2
            self._trans_ctr = torch.zeros(1, dtype=torch.int32, device=dev)
            self._trans_epoch = torch.zeros(2, dtype=torch.int64, device=dev)  # [epoch, gate fault word]
            # layout output: [replicas of my home experts elsewhere, replicas I hold] -> the
            # GEMMs size their SM reservation for Trans / Agg from it, on device
            self.replica_stats = torch.zeros(2, dtype=torch.int32, device=dev)
            self.comm_barrier = _Barrier(self.group, dev, host=self.shared_device)
        elif D > 1:
            # copy engine: the replicas pull the home weights; a barrier on the comm stream
            # orders the pulls after every home's optimizer step (stream order of this rank's
            # forward start + arrival of every peer at the same point)
            self.comm_barrier = _Barrier(self.group, dev, host=self.shared_device)
        self._plan_pending = None
        self._mask_host = torch.zeros((E, E), dtype=torch.uint8).pin_memory() if D > 1 else None
        self.mask_cur_host = None
        self._trans_list = []     # (dst, src, bytes) of this iteration's Trans
        self._agg_list = []       # (dst, src, bytes) pulls of replica grads into staging
        self._agg_ranges = None   # device int32 [m+1]
        self._agg_staging = None
        self._trans_done = None
        self._trans_iter = -1     # iteration whose Trans has been issued
        self.replica_experts = []  # replica experts held by this rank under the current plan
        self.barrier = _Barrier(self.group, dev, host=self.shared_device)
        self.history = []  # host copies of LoadMatrix per iteration (optional, record_history)
        self.record_history = False
        self.events = {}
        self.gemm_timing = None
        self.gemm_event_pool = None
        self.phase_log = None
        self._agg_done = None
        self.timeline_log = None  # list -> (kind, lane, start_event, end_event) of side-stream ops
        self._ext_events = False  # timing events recorded as graph nodes (capture of a timeline)
        # persistent-GEMM grid (0 = every SM); leaving a few SMs free lets the side-stream
        # Agg reduce / planner kernels run under the expert GEMMs instead of after them
        self.gemm_sms = 0
        self.block_index = 0
        if D > 1:
            torch.cuda.synchronize()
            dist.barrier(group=self.group)

    @property
    def agg_stage(self):
        """Agg staging of this block: alternates by block parity in a shared workspace (block
        i's Agg may still run on the side stream while block i-1's backward starts)."""
        st = self.workspace.agg_stage
        return st[self.block_index % len(st)] if st else None

    # ------------------------------------------------------------------------
    def set_gate_bias(self, bias) -> None:
        self.gate_bias.copy_(torch.as_tensor(bias, dtype=torch.float32))

    def _sp(self):
        return _device.stream_ptr()

    def _mark(self, name: str) -> None:
        """Measured timeline: when ``phase_log`` is a list, record a CUDA event per
        phase boundary on the layer's stream (see ``phase_breakdown``)."""
        if self.phase_log is not None:
            ev = torch.cuda.Event(enable_timing=True, external=self._ext_events)
            ev.record()
            self.phase_log.append((name, ev))

    def phase_breakdown(self, stat: str = "median") -> dict:
        """Per-phase ms over the recorded steps (phase = time since the previous mark on
        this rank's stream); the median by default, so a host hiccup in one eager step
        (allocator, GC) does not masquerade as a slow phase."""
        per, prev = {}, None
        for name, ev in self.phase_log or []:
            if name != "fwd_start" and prev is not None:
                per.setdefault(name, []).append(prev.elapsed_time(ev))
            prev = ev
        if stat == "mean":
            return {k: sum(v) / len(v) for k, v in per.items()}
        return {k: float(np.median(v)) for k, v in per.items()}

    def _route_and_layout(self, x: torch.Tensor) -> None:
        sp = self._sp()
        T, d, E, k, m = self.T, self.d, self.E, self.k, self.m
        _lib.call("pp_route_topk", x.data_ptr(), self.wg.data_ptr(), self.gate_bias.data_ptr(), T, d,
                  E, k, self.idx.data_ptr(), self.w.data_ptr(), self.probs.data_ptr(),
                  self.rank_in_chunk.data_ptr(), self.chunk_counts.data_ptr(), sp)
        if self.world > 1:
            _lib.call("pp_slot_histogram", self.chunk_counts.data_ptr(), T, E, m, self.counts_buf.ptrs.data_ptr(),
                      self.world, self.rank * m, sp)
            self._mark("route_hist")
            self.barrier()  # every rank's rows of the LoadMatrix have landed
            self._mark("hist_barrier")
        if self.top_m and self.world > 1:
            _lib.call("pp_top_m_mask", self.counts.data_ptr(), E, E, self.top_m, self._topm_mask.data_ptr(),
                      None, sp)
            self.mask_cur = self._topm_mask
        mask_ptr = self.mask_cur.data_ptr() if self.mask_cur is not None else None
        _lib.call("pp_dispatch_layout", self.counts.data_ptr(), mask_ptr, self.chunk_counts.data_ptr(),
                  self.world, m, E, T, self.rank, self.max_groups, self.rows_cap, self.slots,
                  self.chunk_base.data_ptr(), self.slot_dest.data_ptr(), self.groups.data_ptr(),
                  self.num_groups.data_ptr(), self.total_rows.data_ptr(), self.seg_start.data_ptr(),
                  self.rep_slot.data_ptr(), 1 if self.world == 1 else 0,
                  self.replica_stats.data_ptr() if self.trans_flags is not None else None,
                  self.status.data_ptr(), sp)
        if self.record_history:
            self.history.append(self.counts.clone())
        if not torch.cuda.is_current_stream_capturing():
            self._status_host.copy_(self.status, non_blocking=True)
            for i, f in enumerate(self._fault_words()[:3]):
                self._fault_host[i: i + 1].copy_(f, non_blocking=True)
            self._status_ev = torch.cuda.Event()
            self._status_ev.record()

    def _poll_status(self) -> None:
        """Raise CapacityError if an earlier step's layout was dropped (non-blocking)."""
        if self._status_ev is None or torch.cuda.is_current_stream_capturing():
            return
        if self._status_ev.query() and (int(self._status_host[0]) or int(self._fault_host.max())):
            self._raise_status(int(self._status_host[0]), self._fault_host.tolist())

    def _fault_words(self) -> list:
        """Device fault words of the cross-rank waits (peer barriers, replica gate): nonzero
        when a wait gave up after 20 s because a peer never arrived."""
        out = []
        for b in (self.barrier, getattr(self, "comm_barrier", None)):
            if b is not None and b.world > 1:
                out.append(b.sig.local[b.world + 1: b.world + 2])
        if getattr(self, "_trans_epoch", None) is not None:
            out.append(self._trans_epoch[1:2])
        return out

    def check_status(self) -> None:
        """Synchronous check of the layout status and the cross-rank fault words (call e.g.
        after graph replays)."""
        st = int(self.status.item())
        faults = [int(f.item()) for f in self._fault_words()]
        if st or any(faults):
            self._raise_status(st, faults)

    def _raise_status(self, st: int, faults=()) -> None:
        if any(int(f) for f in faults):
            raise RuntimeError("MoE layer: a cross-rank wait timed out after 20 s (a peer rank never "
                               "arrived); the step's results are invalid")
        why = []
        if st & 1:
            why.append(f"a rank needed more than rows_capacity={self.rows_cap} receive rows")
        if st & 2:
            why.append(f"a rank needed more than {self.slots - self.m} replica weight slots")
        if st & 4:
            why.append(f"a rank needed more than max_groups={self.max_groups} expert groups")
        raise CapacityError("MoE layer step dropped (outputs are zero): " + "; ".join(why) +
                            " -- raise capacity_factor / max_replicas")

    def _launch_planner(self) -> None:
        """plan_for_iteration rule: iteration j+1 searches on iteration j's load
        when (j+1) % reuse_interval == 0, otherwise it keeps the current plan.
        The search runs on a side stream; its mask is also copied to pinned host
        memory so the copy-engine Trans of j+1 can be issued without a stall."""
        if not self.plan_enabled:
            return
        nxt = self.iteration + 1
        if self.planning != "device" and nxt % self.planner_cfg.reuse_interval != 0:
            return
        if self.planning == "device":  # launched every iteration; the kernel applies the reuse rule
            self._counts_snap.copy_(self.counts)  # the next iteration overwrites self.counts
            ev = torch.cuda.Event()
            ev.record()
            with torch.cuda.stream(self.plan_stream):
                self.plan_stream.wait_event(ev)
                p0 = self._side_event(self.plan_stream)
                _device.launch_plan(self._counts_snap.view(1, self.E, self.E), self._plan_out, self._cm,
                                    self._pcfg, self.plan_stream, physical_devices=self._phys_devices(),
                                    refine_slots=self.refine_slots)
                self._log_side("Plan", p0, self._side_event(self.plan_stream))
                self._plan_done_dev = torch.cuda.Event()
                self._plan_done_dev.record(self.plan_stream)
            return
        snapshot = self.counts.clone()  # the next iteration overwrites self.counts
        ev = torch.cuda.Event()
        ev.record()
        with torch.cuda.stream(self.plan_stream):
            self.plan_stream.wait_event(ev)
            snapshot.record_stream(self.plan_stream)
            p0 = self._side_event(self.plan_stream)
            _device.launch_plan(snapshot.view(1, self.E, self.E), self._plan_out, self._cm, self._pcfg,
                                self.plan_stream, physical_devices=self._phys_devices(),
                                refine_slots=self.refine_slots)
            self._log_side("Plan", p0, self._side_event(self.plan_stream))
            mask_dev = self._plan_out.mask[0].clone()
            self._mask_host.copy_(mask_dev, non_blocking=True)
            done = torch.cuda.Event()
            done.record(self.plan_stream)
        self._plan_pending = (done, mask_dev)

    def _epoch_ptr(self) -> int:
        """Device address of this layer's Trans epoch: advanced by one on the main stream every
        time the iteration's Trans is issued (every rank issues it once per iteration), so it
        is equal on every rank and names this iteration's Trans completion -- also when the
        Trans is issued ahead of the block's barriers (MoEStack: during the attention)."""
        return self._trans_epoch.data_ptr()

    def _comb_local(self):
        return self.comb.local.data_ptr() if self.fused_a2a else None

    def _plan_inflight(self) -> bool:
        return self.planning == "device" and self._plan_done_dev is not None or self._plan_pending is not None

    def _phys_devices(self) -> int:
        return self.world if self.placement == "physical" else 0

    def begin_iteration(self) -> None:
        """Adopt the plan computed during the previous iteration and derive this
        rank's replica set, Trans copies and Agg sources from it (same rule as the
        device layout: replica experts in ascending id get slots m, m+1, ...)."""
        if self._plan_pending is None or self.planning == "device":
            return
        done, mask_dev = self._plan_pending
        self._plan_pending = None
        done.synchronize()  # ~100 us planner launched one iteration ago: normally long done
        cur = torch.cuda.current_stream()
        cur.wait_event(done)
        mask_dev.record_stream(cur)
        self.mask_cur = mask_dev
        mh = self._mask_host.numpy().astype(bool)
        self.mask_cur_host = mh.copy()
        self._derive_replicas(mh)

    def _derive_replicas(self, mh: np.ndarray) -> None:
        D, m, me = self.world, self.m, self.rank
        fd = self.d * self.f
        if any(len(r) > self.max_replicas for r in replica_sets(mh, D, m)):
            raise ValidationError("plan needs more replica slots than max_replicas")
        xf = replica_transfers(mh, D, m, me)
        self.replica_experts = xf["replicas"]
        w1, w2 = self.w1_arena.ptr_list, self.w2_arena.ptr_list
        self._trans_list = []
        for e, home, j, slot in xf["trans_in"]:  # pulls of the home weights into my replica slots
            self._trans_list.append((w1[me] + slot * fd * 2, w1[home] + j * fd * 2, fd * 2))
            self._trans_list.append((w2[me] + slot * fd * 2, w2[home] + j * fd * 2, fd * 2))
        # Agg sources: for each home slot j, replicas of expert me*m+j on other ranks (rank order)
        g1, g2 = self.g1_arena.ptr_list, self.g2_arena.ptr_list
        srcs, ranges = [], [0]
        for j in range(m):
            for r, slot in xf["agg_in"][j]:
                srcs.append((g1[r] + slot * fd * 4, g2[r] + slot * fd * 4))
            ranges.append(len(srcs))
        self._agg_list = []
        if srcs:
            need = len(srcs) * 2 * fd
            if self._agg_staging is None or self._agg_staging.numel() < need:
                self._agg_staging = torch.empty(need, dtype=torch.float32, device=self.device)
            base = self._agg_staging.data_ptr()
            for i, (s1, s2) in enumerate(srcs):
                self._agg_list.append((base + (2 * i) * fd * 4, s1, fd * 4))
                self._agg_list.append((base + (2 * i + 1) * fd * 4, s2, fd * 4))
        self._agg_ranges = torch.tensor(ranges, dtype=torch.int32).to(self.device, non_blocking=True)

    @staticmethod
    def _copy_batch(items, stream) -> None:
        n = len(items)
        if n == 0:
            return
        dst = (ctypes.c_void_p * n)(*[t[0] for t in items])
        src = (ctypes.c_void_p * n)(*[t[1] for t in items])
        nb = (ctypes.c_uint64 * n)(*[t[2] for t in items])
        _lib.call("pp_copy_batch", dst, src, nb, n, _device.stream_ptr(stream))

    def issue_trans(self):
        """K5 Trans for this iteration's plan on the side stream (once per iteration).
        Ordered after everything already on the current stream (e.g. an optimizer
        step); returns the completion event (None if nothing to move)."""
        # once per iteration: the home weights change with every optimizer step, so the
        # replicas are refreshed every iteration even when the plan is reused (the reference
        # charges Trans every iteration, simulator.py placement_for / cost_fn)
        if self._trans_iter == self.iteration:
            return self._trans_done
        self._trans_iter = self.iteration
        self._trans_done = None
        if self.world == 1 or self.mask_cur is None:
            return None
        if self.replica_engine == "sm":
            self._trans_epoch[0:1].add_(1)  # stream-ordered before this rank's FWD1 / FWD2 gates
        ev = torch.cuda.Event()
        ev.record()
        with torch.cuda.stream(self.comm_stream):
            self.comm_stream.wait_event(ev)
            t0 = self._side_event(self.comm_stream)
            if self.replica_engine == "copy":
                # every rank (replica holder or not) arrives: the homes' weights are final
                self.comm_barrier(self.comm_stream)
                split = getattr(self, "trans_split_bytes", None)
                if split:  # Algorithm 2 partition: SubTrans2 (FNEC window) first, then SubTrans1
                    first, rest = self._split_copies(self._trans_list, split)
                    self._copy_batch(first, self.comm_stream)
                    t1 = self._side_event(self.comm_stream)
                    self._log_side("SubTrans2", t0, t1)
                    t0 = t1
                    self._copy_batch(rest, self.comm_stream)
                else:
                    self._copy_batch(self._trans_list, self.comm_stream)
            else:
                # W1 first (FWD1's replica tiles wait on flag row 0), then W2 (FWD2's, row 1)
                for part, row in ((1, 0), (2, 1)):
                    _lib.call("pp_replica_trans", self.w1_arena.ptrs.data_ptr(), self.w2_arena.ptrs.data_ptr(),
                              self.mask_cur.data_ptr(), self.E, self.m, self.rank, self.slots, self.d, self.f, part,
                              self.trans_flags.ptrs.data_ptr(), row, self._epoch_ptr(),
                              self._trans_ctr.data_ptr(), self.trans_ctas, _device.stream_ptr(self.comm_stream))
            self._log_side("SubTrans1", t0, self._side_event(self.comm_stream))  # before the join event
            self._trans_done = torch.cuda.Event()
            self._trans_done.record(self.comm_stream)
        return self._trans_done

    def _side_event(self, stream):
        if self.timeline_log is None:
            return None
        ev = torch.cuda.Event(enable_timing=True, external=self._ext_events)
        ev.record(stream)
        return ev

    def _log_side(self, kind: str, e0, e1) -> None:
        if self.timeline_log is not None and e0 is not None and e1 is not None:
            self.timeline_log.append((kind, e0, e1))

    @staticmethod
    def _split_copies(items, first_bytes: int):
        """Split a copy list so that the first part moves ~first_bytes (a copy may
        be cut in two at a 16-byte boundary)."""
        first, rest, acc = [], [], 0
        for dst, src, nb in items:
            if acc >= first_bytes:
                rest.append((dst, src, nb))
                continue
            take = nb if nb <= first_bytes - acc else (first_bytes - acc) - (first_bytes - acc) % 16
            if take > 0:
                first.append((dst, src, take))
            if take < nb:
                rest.append((dst + take, src + take, nb - take))
            acc += take
        return first, rest

    def trans_bytes(self) -> int:
        return sum(t[2] for t in self._trans_list)

    def agg_bytes(self) -> int:
        return sum(t[2] for t in self._agg_list)

    def _issue_agg(self, parts: int = 3) -> None:
        """K5 Agg on the side stream: the replicas' grads of this rank's home experts
        are added (rank order) into main_grad.  parts (SM engine): 1 = W1 grads, 2 = W2
        grads, 3 = both; the copy engine always moves both."""
        if self.world == 1 or self.mask_cur is None:
            return
        ev = torch.cuda.Event()
        ev.record()
        with torch.cuda.stream(self.comm_stream):
            self.comm_stream.wait_event(ev)
            t0 = self._side_event(self.comm_stream)
            if self.replica_engine == "copy":
                if self._agg_list:
                    self._copy_batch(self._agg_list, self.comm_stream)
                    _lib.call("pp_agg_accumulate", self.g1_arena.local.data_ptr(), self.g2_arena.local.data_ptr(),
                              self._agg_staging.data_ptr(), self._agg_ranges.data_ptr(), self.m, self.d, self.f,
                              _device.stream_ptr(self.comm_stream))
            else:
                cs = _device.stream_ptr(self.comm_stream)
                nctas = self.agg_ctas_w2 if parts == 2 else self.agg_ctas
                _lib.call("pp_replica_agg", self.g1_arena.ptrs.data_ptr(), self.g2_arena.ptrs.data_ptr(),
                          self.agg_stage.ptrs.data_ptr(), self.mask_cur.data_ptr(), self.E, self.m, self.rank,
                          self.slots, self.d, self.f, parts, nctas, cs)
                self.comm_barrier(self.comm_stream)  # every replica's grads have landed here
                tail = parts == 1 and self.block_index == 0
                _lib.call("pp_replica_agg_reduce", self.g1_arena.local.data_ptr(), self.g2_arena.local.data_ptr(),
                          self.agg_stage.local.data_ptr(), self.mask_cur.data_ptr(), self.E, self.m, self.rank,
                          self.d, self.f, parts, self.agg_tail_reduce_ctas if tail else nctas, cs)
            self._log_side("SubAgg1" if parts == 2 else "SubAgg2", t0, self._side_event(self.comm_stream))
            self._agg_done = torch.cuda.Event()
            self._agg_done.record(self.comm_stream)

    def _gemm(self, mode, a, b, c, c2=None, stream=None, num_sms=None, scatter=False, gate=False, res=None):
        timing = self.gemm_timing
        if timing is not None:
            pool = self.gemm_event_pool
            if pool and len(pool) >= 2:
                e0, e1 = pool.pop(), pool.pop()
            else:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
        nsm = self.gemm_sms if num_sms is None else num_sms
        if gate or scatter or res:
            # fused A2A epilogue (rows go to their source rank's comb buffer) and/or replica
            # gate (replica tiles wait for the pushers' Trans completion flags: W1 row for
            # FWD1, W2 row for FWD2)
            flags = (self.trans_flags.local[0 if mode == _lib.PP_GEMM_FWD1 else 1].data_ptr() if gate else None)
            _lib.call("pp_grouped_gemm_ex", mode, a.data_ptr(), b.data_ptr(), None if scatter else c.data_ptr(),
                      c2.data_ptr() if c2 is not None else None, self.groups.data_ptr(),
                      self.num_groups.data_ptr(), self.max_groups, self.rows_cap, self.slots, self.d, self.f,
                      self.origin.local.data_ptr() if scatter else None,
                      self.comb.ptrs.data_ptr() if scatter else None, self.T * self.k, flags,
                      self._epoch_ptr() if gate else None, self.rank, self.world, self.m,
                      self.replica_stats.data_ptr() if res else None, *(res or (0, 0, 0, 0)), nsm,
                      _device.stream_ptr(stream))
        else:
            _device.grouped_gemm(mode, a, b, c, c2, self.groups, self.num_groups, self.max_groups,
                                 self.rows_cap, self.slots, self.d, self.f, num_sms=nsm, stream=stream)
        if timing is not None:
            e1.record()
            timing.append((mode, e0, e1))

    def collect_gemm_timing(self) -> dict:
        """Average device time per step of each GEMM mode recorded while
        ``gemm_timing`` was a list (events on the launching stream)."""
        per, steps = {}, 0
        for mode, e0, e1 in self.gemm_timing or []:
            per[mode] = per.get(mode, 0.0) + e0.elapsed_time(e1)
            steps += mode == _lib.PP_GEMM_FWD1
        steps = max(steps, 1)
        names = {0: "FWD1", 1: "FWD2", 2: "DGRAD2", 3: "DGRAD1", 4: "WGRAD2", 5: "WGRAD1"}
        per_mode = {names.get(m, str(m)): v / steps for m, v in per.items()}
        return {"ms_per_step": sum(per_mode.values()), "per_mode_ms": per_mode}

    def total_real_rows(self) -> int:
        n = int(self.num_groups.item())
        return int(self.groups[:n, 1].sum().item())

    # ------------------------------------------------------------------------
    def forward_raw(self, x: torch.Tensor) -> torch.Tensor:
        """Forward without autograd bookkeeping (x: [T, d] bf16 on this device)."""
        assert x.shape == (self.T, self.d) and x.dtype == torch.bfloat16 and x.is_contiguous()
        sp = self._sp()
        if self._agg_done is not None:  # this forward's WGRADs will overwrite grads Agg still reads
            torch.cuda.current_stream().wait_event(self._agg_done)
            self._agg_done = None
        self._mark("fwd_start")
        self._poll_status()
        self.begin_iteration()
        # copy engine: host-derived copies start before routing and must land before FEC;
        # SM engine: the home ranks push after barrier 1, overlapping FWD1 on the home experts,
        # and each receiver's FWD1 gates only its replica tiles on the pushers' completion flags
        sm_gate = self.replica_engine == "sm" and self.world > 1 and self.trans_gate
        # top-m: this iteration's mask exists only after the histogram, so its Trans is issued
        # after barrier 1 even when it is not gated
        late = bool(self.top_m) and self.world > 1
        trans_done = None if (sm_gate or late) else self.issue_trans()  # no-op if a scheduler issued it
        self._route_and_layout(x)
        self._mark("route_layout")
        self._launch_planner()  # [A2A | Plan(j+1)]: the search overlaps this block's dispatch
        _lib.call("pp_dispatch", x.data_ptr(), self.idx.data_ptr(), self.rank_in_chunk.data_ptr(),
                  self.chunk_base.data_ptr(), self.slot_dest.data_ptr(), self.T, self.d, self.k, self.m,
                  self.E, self.xp.ptrs.data_ptr(), self.xp.local.data_ptr(), self.groups.data_ptr(),
                  self.num_groups.data_ptr(), self.max_groups, self.pair_dest.data_ptr(),
                  self.pair_row.data_ptr(), self.origin.ptrs.data_ptr() if self.fused_a2a else None,
                  self.rank, sp)
        self._mark("dispatch")
        if trans_done is not None:
            torch.cuda.current_stream().wait_event(trans_done)
        self._mark("trans_wait")
        self.barrier()  # every rank's rows have landed
        self._mark("barrier1")
        if sm_gate or late:
            trans_done = self.issue_trans()
            if late and not sm_gate and trans_done is not None:
                # ungated (ranks sharing a GPU): this rank's pushes done, then every rank's
                torch.cuda.current_stream().wait_event(trans_done)
                self.barrier()
        total = self.gemm_sms or _device.num_sms(self.device)
        gated = sm_gate and trans_done is not None
        plan_sms = 2 if self._plan_inflight() else 0  # the planner's CTA stays out of the static walk
        fwd_sms, fwd_res = None, None
        if gated:  # res_per_replica SMs per replica this rank pushes (>= 2: its signal-only Trans must run)
            fwd_res = (0, self.res_per_replica, 2 + plan_sms, self.trans_ctas + plan_sms)
        elif plan_sms:
            fwd_sms = max(2, (total - plan_sms) // 2 * 2)
        self._gemm(_lib.PP_GEMM_FWD1, self.xp.local, self.w1_arena.local, self.pre, self.act, num_sms=fwd_sms,
                   gate=gated, res=fwd_res)
        self._gemm(_lib.PP_GEMM_FWD2, self.act, self.w2_arena.local, self.yp.local, num_sms=fwd_sms,
                   scatter=self.fused_a2a, gate=gated, res=fwd_res)
        if gated:  # join the side stream (its pushes have landed: FWD2 waited for every flag)
            torch.cuda.current_stream().wait_event(trans_done)
        self._mark("fwd_gemms")
        self.barrier()
        self._mark("barrier2")
        y = torch.empty((self.T, self.d), dtype=torch.bfloat16, device=self.device)
        _lib.call("pp_combine", self.yp.ptrs.data_ptr(), self.pair_dest.data_ptr(), self.pair_row.data_ptr(),
                  self.w.data_ptr(), self.T, self.d, self.k, y.data_ptr(), self._comb_local(), sp)
        self._mark("combine")
        return y

    def backward_raw(self, x: torch.Tensor, dy: torch.Tensor) -> torch.Tensor:
        assert dy.shape == (self.T, self.d) and dy.dtype == torch.bfloat16 and dy.is_contiguous()
        sp = self._sp()
        self._mark("bwd_begin")
        _lib.call("pp_combine_bwd", dy.data_ptr(), self.yp.ptrs.data_ptr(), self.dyp.ptrs.data_ptr(),
                  self.dyp.local.data_ptr(), self.pair_dest.data_ptr(), self.pair_row.data_ptr(),
                  self.w.data_ptr(), self.groups.data_ptr(), self.num_groups.data_ptr(), self.max_groups,
                  self.T, self.d, self.k, self.dw.data_ptr(), self._comb_local(), self.idx.data_ptr(),
                  self.probs.data_ptr(), self.E, self.EP, self.dlogits.data_ptr(), sp)
        self._mark("combine_bwd")
        # gate weight grad (deterministic split-K; needs only x and dL/dlogits): at N > 1 it
        # fills the wait for the slowest rank's combine_bwd at the next barrier
        _lib.call("pp_gate_dw", self.dlogits.data_ptr(), x.data_ptr(), self.T, self.d, self.E, self.EP,
                  self.gate_ws.data_ptr(), self.wg.main_grad.data_ptr(), sp)
        # the gate's input gradient dx = dL/dlogits . Wg (tcgen05); the dispatch backward adds to it
        dx = torch.empty((self.T, self.d), dtype=torch.bfloat16, device=self.device)
        _lib.call("pp_gate_dx", self.dlogits.data_ptr(), self.wg.data_ptr(), self.T, self.d, self.E, self.EP,
                  dx.data_ptr(), sp)
        self._mark("gate_dw")
        self.barrier()
        self._mark("barrier3")
        agg = self.world > 1 and self.mask_cur is not None
        if agg and self.replica_engine == "sm":
            # SM engine: WGRAD2 first, so the replicas' W2 grads are pushed home while
            # DGRAD2 and WGRAD1 run, and the W1 grads while DGRAD1 runs; those GEMMs leave
            # agg_ctas SMs to the push/reduce kernels (SubAgg | BEC)
            # res_per_replica SMs per replica this rank sends or receives, on device (layout replica_stats)
            res_w2 = (1, self.res_per_replica, 2, self.agg_ctas_w2)
            res_w1 = (1, self.res_per_replica, 2, self.agg_ctas)
            self._gemm(_lib.PP_GEMM_WGRAD2, self.dyp.local, self.act, self.g2_arena.local)
            self._issue_agg(parts=2)
            self._gemm(_lib.PP_GEMM_DGRAD2, self.dyp.local, self.w2_arena.local, self.pre, self.pre, res=res_w2)
            self._gemm(_lib.PP_GEMM_WGRAD1, self.pre, self.xp.local, self.g1_arena.local, res=res_w2)
            self._issue_agg(parts=1)
            self._gemm(_lib.PP_GEMM_DGRAD1, self.pre, self.w1_arena.local, self.dxp.local,
                       scatter=self.fused_a2a, res=res_w1)
        else:
            self._gemm(_lib.PP_GEMM_DGRAD2, self.dyp.local, self.w2_arena.local, self.pre, self.pre)
            self._gemm(_lib.PP_GEMM_WGRAD2, self.dyp.local, self.act, self.g2_arena.local)
            self._gemm(_lib.PP_GEMM_WGRAD1, self.pre, self.xp.local, self.g1_arena.local)
            if agg:  # copy engine: the home pulls once every rank's replica grads exist; rides on DGRAD1
                self.barrier()
                self._issue_agg()
            self._gemm(_lib.PP_GEMM_DGRAD1, self.pre, self.w1_arena.local, self.dxp.local,
                       scatter=self.fused_a2a)
        self._mark("bwd_gemms")
        self.barrier()
        self._mark("barrier4")
        # dispatch backward: dx += sum_j dXp[pair] (peer loads; fused A2A: local comb)
        _lib.call("pp_dispatch_bwd", None if self.fused_a2a else self.dxp.ptrs.data_ptr(), self._comb_local(),
                  self.pair_dest.data_ptr(), self.pair_row.data_ptr(), self.T, self.d, self.k, dx.data_ptr(), sp)
        self._mark("dispatch_bwd")
        if self.planning == "device" and self.world > 1:
            cur = torch.cuda.current_stream()
            if self._agg_done is not None:  # join the Agg side stream (graph-capturable fork/join)
                cur.wait_event(self._agg_done)
                self._agg_done = None
            if self._plan_done_dev is not None:  # plan for the next iteration becomes current
                cur.wait_event(self._plan_done_dev)
                self.mask_buf.copy_(self._plan_out.mask[0])
                self._plan_done_dev = None
        self.iteration += 1
        return dx

    def wait_grads(self, stream=None) -> None:
        """Make ``stream`` (default: current) wait until the replica gradients have
        been aggregated into the home experts' ``main_grad`` (call before the
        optimizer reads them)."""
        if self._agg_done is not None:
            (stream or torch.cuda.current_stream()).wait_event(self._agg_done)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return _MoEFunction.apply(x, self)

    def make_graphed_step(self, x: torch.Tensor, dy: torch.Tensor, with_loss: bool = False,
                          gemm_events: bool = False, timeline_events: bool = False) -> "GraphedStep":
        """Capture one forward + backward into a CUDA graph (host cost per step
        drops to one graph launch).  ``x`` / ``dy`` become the static input
        buffers: copy new data into them, call the returned object, read
        ``.y`` / ``.dx`` (and the ``main_grad`` tensors).  At D > 1 the layer
        must use planning='device' (plan, Trans and Agg stay on the device; every
        rank captures and replays in lockstep)."""
        if self.world != 1 and self.planning != "device":
            raise ValidationError("make_graphed_step at D > 1 needs planning='device'")
        if self.shared_device:
            raise ValidationError("make_graphed_step needs one GPU per rank (ranks sharing a GPU use host barriers)")
        return GraphedStep(self, x, dy, with_loss, gemm_events, timeline_events)

    # ---- introspection (LoadMatrix / placement of the last call) -------------
    def last_load_matrix(self) -> LoadMatrix:
        return LoadMatrix(self.counts.cpu().numpy())

    def current_mask(self) -> np.ndarray:
        if self.mask_cur is None:
            return np.eye(self.E, dtype=bool)
        return self.mask_cur.cpu().numpy().astype(bool)

    def probe_loss(self, y: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
        """loss = sum(y * g) in fp32 (one fused pass, pp_dot_bf16): a linear probe whose
        gradient w.r.t. y is exactly g -- the scalar a training loop reads back per step."""
        assert y.shape == g.shape and y.dtype == g.dtype == torch.bfloat16
        if getattr(self, "_dot_partial", None) is None:
            self._dot_partial = torch.empty(_lib.PP_DOT_PARTIALS, dtype=torch.float32, device=self.device)
        out = torch.empty((), dtype=torch.float32, device=self.device)
        _lib.call("pp_dot_bf16", y.data_ptr(), g.data_ptr(), y.numel(), self._dot_partial.data_ptr(),
                  out.data_ptr(), self._sp())
        return out

    def replica_traffic(self, mask: np.ndarray | None = None) -> dict:
        """NVLink bytes of one iteration's Trans (bf16 W1+W2) and Agg (fp32 grads) per
        rank under `mask` (default: the current plan): out = pushed by the home,
        in = received by the replica holder (Trans); Agg the reverse direction."""
        mh = self.current_mask() if mask is None else np.asarray(mask, dtype=bool)
        D, m, E = self.world, self.m, self.E
        reps = replica_sets(mh, D, m)
        w = 2 * self.d * self.f * 2  # W1 + W2 bf16
        t_out = [sum(w for r in range(D) for e in reps[r] if e // m == h) for h in range(D)]
        t_in = [len(reps[r]) * w for r in range(D)]
        return {"replicas_per_rank": [len(x) for x in reps], "trans_out_bytes": t_out, "trans_in_bytes": t_in,
                "agg_out_bytes": [2 * b for b in t_in], "agg_in_bytes": [2 * b for b in t_out]}

    def group_table(self) -> list:
        n = int(self.num_groups.item())
        t = self.groups[:n].cpu().numpy()
        return [dict(row_off=int(r[0]), rows=int(r[1]), rows_pad=int(r[2]), wslot=int(r[3]),
                     expert=int(r[4]), src_rank=int(r[5])) for r in t]

    def close(self) -> None:
        """Release the peer-mapped buffers.  Collective at D > 1: every rank drains its streams
        and meets at a barrier first, so no peer still loads from / stores into this rank's
        memory (dispatch_bwd peer loads, Agg pushes, copy-engine pulls); the parameter and
        main_grad views of the freed arenas are dropped."""
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier(group=self.group)
        for prm in (self.w1, self.w2):
            prm.main_grad = None
            prm.data = torch.empty(0, dtype=prm.dtype, device=prm.device)
        for b in (self.w1_arena, self.w2_arena, self.g1_arena, self.g2_arena, self.xp, self.yp,
                  self.counts_buf, self.origin, self.comb, self.trans_flags,
                  self.barrier, getattr(self, "comm_barrier", None)):
            if b is not None:
                b.close()
        if self._own_workspace:
            self.workspace.close()


class _MoEFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, layer):
        x = x.contiguous()
        ctx.layer = layer
        ctx.save_for_backward(x)
        return layer.forward_raw(x)

    @staticmethod
    def backward(ctx, dy):
        (x,) = ctx.saved_tensors
        dx = ctx.layer.backward_raw(x, dy.contiguous().to(torch.bfloat16))
        return dx, None


class GraphedStep:
    """A captured fwd+bwd of one MoELayer over static input buffers."""

    def __init__(self, layer: MoELayer, x: torch.Tensor, dy: torch.Tensor, with_loss: bool = False,
                 gemm_events: bool = False, timeline_events: bool = False) -> None:
        """with_loss: also compute loss = sum(y * dy) in fp32 inside the graph (a
        linear probe whose gradient w.r.t. y is exactly dy), so a training loop can
        read back one scalar per step.  gemm_events: capture a timing-event pair
        around each grouped GEMM (event-record nodes); after a replay,
        ``gemm_times()`` gives that replay's per-GEMM durations.  timeline_events:
        capture the phase marks and the side-stream Plan/Trans/Agg events as graph nodes;
        after a replay, ``timeline()`` is that replay's reference-schema timeline."""
        self.layer, self.x, self.dy = layer, x, dy
        saved_timing, saved_phase, saved_pool = layer.gemm_timing, layer.phase_log, layer.gemm_event_pool
        layer.gemm_timing = layer.phase_log = None  # host-side timing lists cannot live in the graph
        side = torch.cuda.Stream(device=layer.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm the allocator / lazy state outside capture
            for _ in range(2):
                layer.forward_raw(x)
                layer.backward_raw(x, dy)
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        self.gemm_events = None
        self.phase_log = self.timeline_log = None
        saved_tl = layer.timeline_log
        layer.timeline_log = None
        if timeline_events:
            layer.phase_log, layer.timeline_log, layer._ext_events = [], [], True
        if gemm_events:  # external events: recorded as graph nodes on every replay
            layer.gemm_timing = []
            layer.gemm_event_pool = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(32)]
        with torch.cuda.graph(self.graph):
            self.y = layer.forward_raw(x)
            self.loss = layer.probe_loss(self.y, dy) if with_loss else None
            self.dx = layer.backward_raw(x, dy)
        layer.iteration -= 1  # the capture ran no kernels: replays count the iterations
        layer._trans_iter = -1  # an eager step after the capture issues its own Trans
        if timeline_events:
            self.phase_log, self.timeline_log = layer.phase_log, layer.timeline_log
        layer._ext_events, layer.timeline_log = False, saved_tl
        if gemm_events:
            self.gemm_events = layer.gemm_timing
        layer.gemm_timing, layer.phase_log, layer.gemm_event_pool = saved_timing, saved_phase, saved_pool

    def timeline(self, iteration: int = 0):
        """Reference-schema IterationTimeline of the most recent replay (timeline_events)."""
        from .stack import layer_timeline

        return layer_timeline(self.phase_log, self.timeline_log, iteration)

    def gemm_times(self) -> list:
        """(mode, ms) of each grouped GEMM in the most recent replay (call after it finished)."""
        return [(mode, e0.elapsed_time(e1)) for mode, e0, e1 in self.gemm_events or []]

    def __call__(self):
        self.graph.replay()
        self.layer.iteration += 1
        return self.y, self.dx
