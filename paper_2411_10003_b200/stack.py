"""MoE-GPT block stack with the Algorithm-2 overlap schedule (BASELINE config 5).

Block i:  h = x + Attn_i(LN(x))        (non-MoE part: FNEC / BNEC, stock PyTorch SDPA)
          y = h + MoE_i(LN(h))         (MoELayer: A2A / FEC / BEC on our kernels)

Block-wise scheduling of the replica traffic (reference ``scheduler.py:236-283``,
``PAPER.md:473-507``), on the copy engines so it takes no SMs from the GEMMs:

* Trans of block i+1 is issued when block i starts, split with
  ``partition_trans`` into SubTrans2 (bytes that fit the FNEC window, first) and
  SubTrans1 (the rest, riding on FEC).  Block 0's Trans heads the iteration.
* Agg of block i+1 is issued as soon as block i+1's weight gradients exist; it
  rides on block i's BNEC/BEC.  Block 0's Agg tails the iteration.
* Each block's plan for iteration j+1 is searched on its iteration-j LoadMatrix
  on a side stream right after the block's forward (the "[A2A | Plan]" slot).

``measured_timeline`` turns the recorded CUDA events of one iteration into a
reference-schema ``IterationTimeline`` so the reference's exposure metric
(``scheduler.py:134-169``) applies to measured B200 time.
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F

import torch.distributed as dist

from .layer import MoELayer, Workspace, layer_plan
from .perf_model import LayerCost
from .scheduler import IterationTimeline, Lane, OpKind, ScheduledOp, trans_byte_split


def reserve_sms_gemm_grid(reserved: int = 4) -> int:
    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    n = props.multi_processor_count - reserved
    return n - (n % 2)  # CTA pairs


class Attention(torch.nn.Module):
    """Pre-LN causal self-attention over [T, d] tokens packed as T/seq sequences."""

    def __init__(self, d_model: int, n_heads: int, seq_len: int, device, seed: int) -> None:
        super().__init__()
        g = torch.Generator(device="cpu").manual_seed(seed)
        self.h, self.s, self.d = n_heads, seq_len, d_model
        self.ln = torch.nn.LayerNorm(d_model, device=device, dtype=torch.bfloat16)
        self.qkv = torch.nn.Parameter((torch.randn((3 * d_model, d_model), generator=g) / math.sqrt(d_model))
                                      .to(device, torch.bfloat16))
        self.out = torch.nn.Parameter((torch.randn((d_model, d_model), generator=g) / math.sqrt(d_model))
                                      .to(device, torch.bfloat16))

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        T, d = x.shape
        q, k, v = F.linear(self.ln(x), self.qkv).view(T // self.s, self.s, 3, self.h, d // self.h).unbind(2)
        o = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2), is_causal=True)
        return F.linear(o.transpose(1, 2).reshape(T, d), self.out)


class _Mark(torch.autograd.Function):
    """Identity whose forward and backward record a timeline event."""

    @staticmethod
    def forward(ctx, x, log, fwd_name, bwd_name):
        ctx.log, ctx.bwd_name = log, bwd_name
        if log is not None:  # external: recorded as a graph node when captured
            ev = torch.cuda.Event(enable_timing=True, external=torch.cuda.is_current_stream_capturing())
            ev.record()
            log.append((fwd_name, ev))
        return x.view_as(x)

    @staticmethod
    def backward(ctx, g):
        if ctx.log is not None:
            ev = torch.cuda.Event(enable_timing=True, external=torch.cuda.is_current_stream_capturing())
            ev.record()
            ctx.log.append((ctx.bwd_name, ev))
        return g, None, None, None


# phase marks of MoELayer -> reference timeline ops: gate GEMMs + layout count as expert
# compute (FEC/BEC); the permute / all-to-all kernels and their barriers are the A2A
# (network lane); side-stream Plan / Trans / Agg come from the layer's timeline_log
LAYER_PHASE_OPS = [
    (OpKind.FEC, Lane.COMPUTE, "fwd_start", "route_layout"),
    (OpKind.A2A, Lane.NETWORK, "route_layout", "barrier1"),
    (OpKind.FEC, Lane.COMPUTE, "barrier1", "fwd_gemms"),
    (OpKind.A2A, Lane.NETWORK, "fwd_gemms", "combine"),
    (OpKind.A2A, Lane.NETWORK, "bwd_begin", "combine_bwd"),
    (OpKind.BEC, Lane.COMPUTE, "combine_bwd", "gate_dw"),
    (OpKind.A2A, Lane.NETWORK, "gate_dw", "barrier3"),
    (OpKind.BEC, Lane.COMPUTE, "barrier3", "bwd_gemms"),
    (OpKind.A2A, Lane.NETWORK, "bwd_gemms", "dispatch_bwd"),
]
SIDE_KINDS = {"Plan": OpKind.PLAN, "SubTrans1": OpKind.SUB_TRANS1, "SubTrans2": OpKind.SUB_TRANS2,
              "SubAgg2": OpKind.SUB_AGG2, "SubAgg1": OpKind.SUB_AGG1}


def add_layer_ops(add, block: int, phase_log, timeline_log) -> None:
    """Feed one MoELayer step's recorded events to add(kind, block, lane, e0, e1)."""
    seq = {n: e for n, e in (phase_log or [])}
    for kind, lane, a, b in LAYER_PHASE_OPS:
        if a in seq and b in seq:
            add(kind, block, lane, seq[a], seq[b])
    for kind, e0, e1 in timeline_log or []:
        k = SIDE_KINDS[kind]
        add(k, block, Lane.COMPUTE if k is OpKind.PLAN else Lane.NETWORK, e0, e1)


def layer_timeline(phase_log, timeline_log, iteration: int = 0) -> IterationTimeline:
    """Reference-schema timeline (seconds from the step's first mark) of one MoELayer step,
    e.g. the events a CUDA-graph capture recorded (``make_graphed_step(timeline_events=True)``),
    so the reference's exposure metric (``scheduler.py:134-169``) applies to a graphed EP step."""
    t0 = phase_log[0][1]
    ops = []

    def add(kind, block, lane, e0, e1):
        st = t0.elapsed_time(e0) / 1e3
        dur = e0.elapsed_time(e1) / 1e3
        if dur > 0:
            ops.append(ScheduledOp(kind, block, iteration, lane, st, dur))

    add_layer_ops(add, 0, phase_log, timeline_log)
    ops.sort(key=lambda o: (o.start, o.lane.value))
    return IterationTimeline(iteration, tuple(ops))


def exposure_summary(tl: IterationTimeline, blocks: int = 1) -> dict:
    """Exposed (not overlapped by the compute lane) replica communication of a timeline,
    reference IterationTimeline.exposed_{trans,agg}_seconds (scheduler.py:134-169)."""
    mk = tl.makespan()
    et = sum(tl.exposed_trans_seconds(i) for i in range(blocks))
    ea = sum(tl.exposed_agg_seconds(i) for i in range(blocks))
    tt = sum(o.duration for o in tl.ops if o.kind.value.startswith("SubTrans"))
    ta = sum(o.duration for o in tl.ops if o.kind.value.startswith("SubAgg"))
    return {"makespan_ms": mk * 1e3, "replica_comm_ms": (tt + ta) * 1e3, "exposed_trans_ms": et * 1e3,
            "exposed_agg_ms": ea * 1e3, "exposed_replica_comm_ms": (et + ea) * 1e3,
            "exposed_replica_comm_frac": (et + ea) / mk if mk > 0 else 0.0,
            "definition": "reference IterationTimeline.exposed_{trans,agg}_seconds / makespan on measured CUDA events"}


class MoEStack(torch.nn.Module):
    """``num_blocks`` transformer blocks with Pro-Prophet EP MoE layers."""

    def __init__(self, num_blocks: int, d_model: int, d_ff: int, num_experts: int, top_k: int,
                 tokens: int, group=None, planner=None, seq_len: int = 1024, n_heads: int = 16,
                 fnec_time: float | None = None, bnec_time: float | None = None, seed: int = 0,
                 **layer_kwargs) -> None:
        super().__init__()
        dev = torch.device("cuda", torch.cuda.current_device())
        self.L = num_blocks
        self.attn = torch.nn.ModuleList(
            [Attention(d_model, n_heads, seq_len, dev, seed + 1000 + i) for i in range(num_blocks)])
        self.ln2 = torch.nn.ModuleList(
            [torch.nn.LayerNorm(d_model, device=dev, dtype=torch.bfloat16) for _ in range(num_blocks)])
        # transient backward buffers (dYp, dXp, dL/dlogits, gate dW partials) and the Agg staging
        # (two, alternating by block parity) are shared by all blocks: memory.py, DESIGN.md section 5
        world = dist.get_world_size(group) if (group is not None and dist.is_initialized()) else 1
        lp = layer_plan(d_model, d_ff, num_experts, top_k, tokens, world,
                        **{k: v for k, v in layer_kwargs.items()
                           if k in ("capacity_factor", "capacity_rows", "max_replicas", "replica_engine",
                                    "planning", "policy", "fused_a2a")})
        self.workspace = Workspace(lp["plan"], group if world > 1 else None, dev, agg_copies=2)
        self.moe = [MoELayer(d_model, d_ff, num_experts, top_k, tokens, group=group, planner=planner,
                             seed=seed + i, workspace=self.workspace, **layer_kwargs) for i in range(num_blocks)]
        for i, m in enumerate(self.moe):
            m.block_index = i
            self.add_module(f"moe{i}", m)
            if m.world > 1:  # reserve SMs for the Agg reduce / planner kernels (Algorithm 2 overlap)
                m.gemm_sms = reserve_sms_gemm_grid()
        self.fnec_time, self.bnec_time = fnec_time, bnec_time  # seconds; calibrate() measures them
        self.log = None  # main-stream timeline marks of one iteration

    # ---- Algorithm 2 ---------------------------------------------------------
    def _schedule_trans(self, i: int, fec_time: float | None) -> None:
        m = self.moe[i]
        if m.replica_engine != "copy":
            return
        m.begin_iteration()
        if self.fnec_time is not None and fec_time is not None and m.trans_bytes() > 0:
            # bytes of Trans(i) the FNEC window of block i-1 can hide go first (SubTrans2)
            nbytes = m.trans_bytes()
            _, m.trans_split_bytes = trans_byte_split(nbytes, nbytes / max(getattr(m, "trans_bw", 600e9), 1.0),
                                                      fec_time, self.fnec_time)
        else:
            m.trans_split_bytes = None
        m.issue_trans()

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        log = self.log
        self._schedule_trans(0, None)  # block 0's Trans heads the iteration
        for i in range(self.L):
            if i + 1 < self.L:  # Trans(i+1) rides on block i
                self._schedule_trans(i + 1, getattr(self, "_fec_est", None))
            m = self.moe[i]
            if m.replica_engine == "sm" and m.world > 1:
                # SM engine (device-planned, graph-capturable): block i's pushes start with its
                # attention (the FNEC window, SubTrans2 of Algorithm 2) and run on into FWD1's home
                # tiles (SubTrans1); FWD1/FWD2's replica tiles wait on the completion flags
                m.issue_trans()
            x = _Mark.apply(x, log, f"FNEC_start:{i}", f"BNEC_end:{i}")
            h = x + self.attn[i](x)
            h = _Mark.apply(h, log, f"FNEC_end:{i}", f"BNEC_start:{i}")
            x = h + self.moe[i](self.ln2[i](h).contiguous())
        return _Mark.apply(x, log, "fwd_end", "bwd_start")

    def wait_grads(self) -> None:
        for m in self.moe:
            m.wait_grads()

    def make_graphed_step(self, x: torch.Tensor, dy: torch.Tensor, timeline_events: bool = False) -> "StackGraph":
        """Capture one whole iteration (forward + autograd backward of every block, the
        device planners, Trans/Agg side streams, barriers) into ONE CUDA graph.  Needs the
        layers' planning='device' at D > 1.  x / dy become static input buffers."""
        return StackGraph(self, x, dy, timeline_events)

    def close(self) -> None:
        torch.cuda.synchronize()
        for m in self.moe:
            m.close()
        self.workspace.close()

    # ---- measurement -----------------------------------------------------------
    def start_timeline(self) -> None:
        self.log = []
        for m in self.moe:
            m.phase_log = []
            m.timeline_log = []

    def measured_timeline(self, iteration: int = 0) -> IterationTimeline:
        """Reference-schema timeline of the iteration recorded since
        ``start_timeline`` (seconds from the first mark)."""
        torch.cuda.synchronize()
        t0 = self.log[0][1]
        ops = []

        def add(kind, block, lane, e0, e1):
            s = t0.elapsed_time(e0) / 1e3
            dur = e0.elapsed_time(e1) / 1e3
            if dur > 0:
                ops.append(ScheduledOp(kind, block, iteration, lane, s, dur))

        marks = {name: ev for name, ev in self.log}
        for i in range(self.L):
            if f"FNEC_start:{i}" in marks:
                add(OpKind.FNEC, i, Lane.COMPUTE, marks[f"FNEC_start:{i}"], marks[f"FNEC_end:{i}"])
            if f"BNEC_start:{i}" in marks:
                add(OpKind.BNEC, i, Lane.COMPUTE, marks[f"BNEC_start:{i}"], marks[f"BNEC_end:{i}"])
            m = self.moe[i]
            add_layer_ops(add, i, m.phase_log, m.timeline_log)
        ops.sort(key=lambda o: (o.start, o.lane.value))
        return IterationTimeline(iteration, tuple(ops))

    def stop_timeline(self) -> None:
        self.log = None
        for m in self.moe:
            m.phase_log = None
            m.timeline_log = None

    def measured_layer_costs(self, timeline: IterationTimeline) -> list:
        """Per-block LayerCost (seconds) read off a measured timeline: the inputs the
        reference's perf model / scheduler would need to reproduce it."""
        out = []
        for i in range(self.L):
            def tot(kind):
                return sum(o.duration for o in timeline.ops if o.block == i and o.kind is kind)
            a2a = tot(OpKind.A2A) / 4.0
            fec, bec = tot(OpKind.FEC), tot(OpKind.BEC)
            trans = tot(OpKind.SUB_TRANS1) + tot(OpKind.SUB_TRANS2)
            agg = tot(OpKind.SUB_AGG1) + tot(OpKind.SUB_AGG2)
            out.append(LayerCost(a2a, fec, bec, trans, agg, 0.0, 0.0, 0.0, 0.0))
        return out


class StackGraph:
    """One captured MoEStack iteration (``MoEStack.make_graphed_step``)."""

    def __init__(self, stack: MoEStack, x: torch.Tensor, dy: torch.Tensor, timeline_events: bool = False) -> None:
        for m in stack.moe:
            if m.world > 1 and m.planning != "device":
                raise ValueError("MoEStack.make_graphed_step at D > 1 needs the layers' planning='device'")
            if m.shared_device:
                raise ValueError("MoEStack.make_graphed_step needs one GPU per rank")
        self.stack, self.x, self.dy = stack, x.detach().requires_grad_(True), dy

        def once():
            y = stack(self.x)
            y.backward(self.dy)
            return y

        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # allocator / autograd / lazy-state warm-up outside capture
            for _ in range(2):
                once()
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        self.timeline_events = timeline_events
        if timeline_events:
            stack.log = []
            for m in stack.moe:
                m.phase_log, m.timeline_log, m._ext_events = [], [], True
        with torch.cuda.graph(self.graph):
            self.y = once()
        if timeline_events:
            self.log = stack.log
            self.layer_logs = [(m.phase_log, m.timeline_log) for m in stack.moe]
            stack.log = None
            for m in stack.moe:
                m.phase_log, m.timeline_log, m._ext_events = None, None, False
        for m in stack.moe:
            m.iteration -= 1  # the capture ran no kernels
            m._trans_iter = -1  # an eager step after the capture issues its own Trans

    def __call__(self) -> torch.Tensor:
        self.graph.replay()
        for m in self.stack.moe:
            m.iteration += 1
        return self.y

    def timeline(self, iteration: int = 0) -> IterationTimeline:
        """Reference-schema timeline of the most recent replay (timeline_events=True)."""
        st = self.stack
        saved = st.log, [(m.phase_log, m.timeline_log) for m in st.moe]
        st.log = self.log
        for m, (pl, tl) in zip(st.moe, self.layer_logs):
            m.phase_log, m.timeline_log = pl, tl
        try:
            return st.measured_timeline(iteration)
        finally:
            st.log = saved[0]
            for m, (pl, tl) in zip(st.moe, saved[1]):
                m.phase_log, m.timeline_log = pl, tl
