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
from .scheduler import IterationTimeline, Lane, OpKind, ScheduledOp, partition_trans


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
        if log is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            log.append((fwd_name, ev))
        return x.view_as(x)

    @staticmethod
    def backward(ctx, g):
        if ctx.log is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            ctx.log.append((ctx.bwd_name, ev))
        return g, None, None, None


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
        if m.replica_engine != "copy":  # SM pushes are issued by the layer itself, gated into FWD1
            return
        m.begin_iteration()
        if self.fnec_time is not None and fec_time is not None and m.trans_bytes() > 0:
            # bytes of Trans(i) the FNEC window of block i-1 can hide go first (SubTrans2)
            tt = m.trans_bytes() / max(getattr(m, "trans_bw", 600e9), 1.0)
            sub1, sub2 = partition_trans(tt, fec_time, self.fnec_time)
            m.trans_split_bytes = int(m.trans_bytes() * (sub2 / tt)) if tt > 0 else 0
        else:
            m.trans_split_bytes = None
        m.issue_trans()

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        log = self.log
        self._schedule_trans(0, None)  # block 0's Trans heads the iteration
        for i in range(self.L):
            if i + 1 < self.L:  # Trans(i+1) rides on block i
                self._schedule_trans(i + 1, getattr(self, "_fec_est", None))
            x = _Mark.apply(x, log, f"FNEC_start:{i}", f"BNEC_end:{i}")
            h = x + self.attn[i](x)
            h = _Mark.apply(h, log, f"FNEC_end:{i}", f"BNEC_start:{i}")
            x = h + self.moe[i](self.ln2[i](h).contiguous())
        return _Mark.apply(x, log, "fwd_end", "bwd_start")

    def wait_grads(self) -> None:
        for m in self.moe:
            m.wait_grads()

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
            ph = m.phase_log or []
            seq = {n: e for n, e in ph}
            # gate GEMMs + layout count as expert compute (FEC/BEC); the permute /
            # all-to-all kernels and their barriers are the A2A (network lane)
            groups = [
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
            for kind, lane, a, b in groups:
                if a in seq and b in seq:
                    add(kind, i, lane, seq[a], seq[b])
            for kind, e0, e1 in m.timeline_log or []:
                k = {"Plan": OpKind.PLAN, "SubTrans1": OpKind.SUB_TRANS1, "SubTrans2": OpKind.SUB_TRANS2,
                     "SubAgg2": OpKind.SUB_AGG2, "SubAgg1": OpKind.SUB_AGG1}[kind]
                lane = Lane.COMPUTE if k is OpKind.PLAN else Lane.NETWORK
                add(k, i, lane, e0, e1)
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
