"""Per-rank HBM plan of the EP MoE layer and of an L-block stack.

One table -- ``buffer_plan`` -- says what every buffer of a layer is, how big it is
and how long it lives; ``MoELayer`` allocates its large buffers from it and
``footprint`` sums it, so the memory claim and the allocation cannot drift apart.

Lifetimes ("scope"):
  * ``layer``  -- lives across the whole iteration (parameters, their fp32 grads, the
    activations the backward reads: Xp, Yp, pre, act, routing state) -> one per block;
  * ``shared`` -- only alive inside one block's backward (dYp, dXp, dL/dlogits, the gate
    dW split-K partials) -> one copy for the whole stack (``Workspace``);
  * ``shared2`` -- the Agg staging area: block i's Agg still runs on the side stream when
    block i-1's backward starts, so the stack keeps two and alternates by block parity.

Receive capacity (rows of Xp/Yp/dYp/dXp/pre/act): the worst case of the reference's
routing rule is every routed pair of every rank landing on one rank, D*T*k rows
(+ 128-row padding per expert).  A stack sizes it as capacity_factor * T * k instead
(the rows a rank computes under a balanced plan are ~T*k); a step that needs more is
detected on the device and dropped on every rank (``pp_dispatch_layout`` status,
``CapacityError``) -- never written out of bounds.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

ROW_ALIGN = 128
CHUNK = 128


def rows_capacity(tokens: int, top_k: int, num_experts: int, world: int,
                  capacity_factor: float | None = None, capacity_rows: int | None = None) -> int:
    """Receive rows per rank: explicit rows, else ceil(factor*T*k) capped at the worst case
    D*T*k, plus one 128-row padding block per expert; rounded to 128."""
    if capacity_rows is not None:
        rows = int(capacity_rows)
    elif capacity_factor is not None:
        if capacity_factor <= 0:
            raise ValueError(f"capacity_factor must be > 0, got {capacity_factor}")
        rows = min(math.ceil(capacity_factor * tokens * top_k), world * tokens * top_k) + num_experts * ROW_ALIGN
    else:
        rows = world * tokens * top_k + num_experts * ROW_ALIGN
    return int(math.ceil(rows / ROW_ALIGN) * ROW_ALIGN)


def gate_dw_splits(tokens: int, d_model: int) -> int:
    """Split-K chunks of the gate weight GEMM (mirror of permute.cu gate_dw_split)."""
    want = (148 + d_model // 128 - 1) // (d_model // 128)
    split = 128
    while split * 2 <= tokens and tokens % (split * 2) == 0 and tokens // (split * 2) >= want:
        split *= 2
    return tokens // split


@dataclass(frozen=True)
class Buf:
    name: str
    shape: tuple
    itemsize: int
    scope: str  # "layer" | "shared" | "shared2"

    @property
    def nbytes(self) -> int:
        return int(math.prod(self.shape)) * self.itemsize


def buffer_plan(d_model: int, d_ff: int, num_experts: int, top_k: int, tokens: int, world: int,
                rows_cap: int, slots: int, max_groups: int, fused_a2a: bool = False,
                sm_engine: bool = False) -> list:
    d, f, E, k, T, D = d_model, d_ff, num_experts, top_k, tokens, world
    m = E // D
    C = T // CHUNK
    EP = 64 if E <= 64 else 128
    R = rows_cap
    b = [
        # parameters + fp32 main_grad arenas (home slots, then replica slots)
        Buf("w1_arena", (slots, f, d), 2, "layer"), Buf("w2_arena", (slots, d, f), 2, "layer"),
        Buf("g1_arena", (slots, f, d), 4, "layer"), Buf("g2_arena", (slots, d, f), 4, "layer"),
        Buf("wg", (E, d), 2, "layer"), Buf("wg_main_grad", (E, d), 4, "layer"),
        # routing state saved for the backward
        Buf("idx", (T, k), 4, "layer"), Buf("rank_in_chunk", (T, k), 4, "layer"), Buf("w", (T, k), 4, "layer"),
        Buf("probs", (T, E), 4, "layer"), Buf("chunk_counts", (C, E), 4, "layer"),
        Buf("counts", (E, E), 8, "layer"), Buf("chunk_base", (C, E), 4, "layer"),
        Buf("slot_dest", (m, E), 4, "layer"), Buf("groups", (max_groups, 8), 4, "layer"),
        Buf("seg_start", (D, E), 4, "layer"), Buf("rep_slot", (D, E), 4, "layer"),
        Buf("pair_dest", (T, k), 4, "layer"), Buf("pair_row", (T, k), 4, "layer"),
        # expert activations the backward reads
        Buf("xp", (R, d), 2, "layer"), Buf("yp", (R, d), 2, "layer"),
        Buf("pre", (R, f), 2, "layer"), Buf("act", (R, f), 2, "layer"),
        # transient inside one block's backward
        Buf("dyp", (R, d), 2, "shared"), Buf("dxp", (R, d), 2, "shared"),
        Buf("dw", (T, k), 4, "shared"), Buf("dlogits", (T, EP), 2, "shared"),
        Buf("gate_ws", (gate_dw_splits(T, d), d, 128), 4, "shared"),
    ]
    if fused_a2a:  # comb holds Yp in pair order: saved for combine_bwd
        b += [Buf("origin", (R,), 4, "layer"), Buf("comb", (T * k, d), 2, "layer")]
    if sm_engine and D > 1:
        b += [Buf("agg_stage", (m, D - 1, 2, f * d), 4, "shared2"), Buf("trans_flags", (2, D), 8, "layer")]
    return b


def footprint(plan: list, layers: int = 1) -> dict:
    """Bytes per rank for `layers` blocks sharing one Workspace."""
    per_layer = sum(x.nbytes for x in plan if x.scope == "layer")
    shared = sum(x.nbytes for x in plan if x.scope == "shared")
    shared2 = sum(x.nbytes for x in plan if x.scope == "shared2") * (2 if layers > 1 else 1)
    by = {}
    for x in plan:
        mult = layers if x.scope == "layer" else (2 if x.scope == "shared2" and layers > 1 else 1)
        by[x.name] = x.nbytes * mult
    return {"per_layer": per_layer, "shared": shared + shared2, "total": per_layer * layers + shared + shared2,
            "by_buffer": by}


def attention_block_bytes(tokens: int, d_model: int) -> int:
    """Estimate of one pre-LN attention block's saved activations in the stack (stock
    PyTorch: LN out, qkv, SDPA out + logsumexp, projection, residual) -- ~8 * T * d bf16."""
    return 8 * tokens * d_model * 2


def stack_footprint(num_blocks: int, d_model: int, d_ff: int, num_experts: int, top_k: int, tokens: int,
                    world: int, capacity_factor: float | None, max_replicas: int | None,
                    sm_engine: bool = True) -> dict:
    """Per-rank HBM of a MoEStack under the layer's allocation rules."""
    m = num_experts // world
    reps = (num_experts - m) if max_replicas is None else max_replicas
    slots = m + (reps if world > 1 else 0)
    rows = rows_capacity(tokens, top_k, num_experts, world, capacity_factor)
    plan = buffer_plan(d_model, d_ff, num_experts, top_k, tokens, world, rows, slots,
                       min(256, m + reps), sm_engine=sm_engine)
    fp = footprint(plan, num_blocks)
    fp["attention_estimate"] = num_blocks * attention_block_bytes(tokens, d_model)
    fp["total_with_attention"] = fp["total"] + fp["attention_estimate"]
    fp["rows_capacity"] = rows
    fp["slots"] = slots
    return fp
