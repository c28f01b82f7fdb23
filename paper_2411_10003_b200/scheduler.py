"""Block-wise overlap schedule (Algorithm 2) -- host-side planning model.

Mirror of reference ``pkg/src/moebal/scheduler.py`` (partition rules
``:91-108``, slot order ``:236-283``, serial baseline ``:286-319``, exposure
metric ``:134-169``).  On the GPU the same slot order drives the real
streams: ``MoEStack`` issues SubTrans/SubAgg copies of block i+1 on a side
stream under block i's expert compute, and ``measured_timeline`` turns the
CUDA events of one iteration into an ``IterationTimeline`` with this schema.

A slot holds at most one compute op and one network op that start together;
the slot lasts as long as the longer one.  Zero-length ops are dropped.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from enum import Enum
from typing import Iterable, Sequence

from .core import ValidationError


class Lane(str, Enum):
    COMPUTE = "compute"
    NETWORK = "network"


class OpKind(str, Enum):
    A2A = "A2A"
    FEC = "FEC"
    BEC = "BEC"
    FNEC = "FNEC"
    BNEC = "BNEC"
    PLAN = "Plan"
    SUB_TRANS1 = "SubTrans1"
    SUB_TRANS2 = "SubTrans2"
    SUB_AGG1 = "SubAgg1"
    SUB_AGG2 = "SubAgg2"


_NETWORK_KINDS = {OpKind.A2A, OpKind.SUB_TRANS1, OpKind.SUB_TRANS2, OpKind.SUB_AGG1, OpKind.SUB_AGG2}
LANE_OF = {k: (Lane.NETWORK if k in _NETWORK_KINDS else Lane.COMPUTE) for k in OpKind}
TRANS_KINDS = frozenset((OpKind.SUB_TRANS1, OpKind.SUB_TRANS2))
AGG_KINDS = frozenset((OpKind.SUB_AGG1, OpKind.SUB_AGG2))


@dataclass(frozen=True)
class ScheduledOp:
    kind: OpKind
    block: int
    iteration: int
    lane: Lane
    start: float
    duration: float

    @property
    def end(self) -> float:
        return self.start + self.duration


def _nonnegative(**values) -> None:
    for name, v in values.items():
        if v < 0:
            raise ValidationError(f"{name} must be >= 0, got {v}")


def partition_trans(trans_time: float, fec_time: float, fnec_time: float) -> tuple:
    """(SubTrans1, SubTrans2): SubTrans2 fills the FNEC window first, the
    rest rides on expert compute (reference ``scheduler.py:91-98``)."""
    _nonnegative(trans_time=trans_time, fec_time=fec_time, fnec_time=fnec_time)
    second = min(trans_time, fnec_time)
    return trans_time - second, second


def partition_agg(agg_time: float, bec_time: float, bnec_time: float) -> tuple:
    """(SubAgg1, SubAgg2): SubAgg1 fills the BNEC window first (reference
    ``scheduler.py:101-108``)."""
    _nonnegative(agg_time=agg_time, bec_time=bec_time, bnec_time=bnec_time)
    first = min(agg_time, bnec_time)
    return first, agg_time - first


def _covered(start: float, end: float, intervals: Iterable) -> float:
    total = 0.0
    for a, b in intervals:
        lo, hi = max(start, a), min(end, b)
        if hi > lo:
            total += hi - lo
    return total


@dataclass(frozen=True)
class IterationTimeline:
    iteration: int
    ops: tuple

    def makespan(self) -> float:
        return max((op.end for op in self.ops), default=0.0)

    def lane_ops(self, lane: Lane) -> list:
        return [op for op in self.ops if op.lane is lane]

    def exposed_seconds(self, op: ScheduledOp) -> float:
        """Part of ``op`` not covered by any op of the other lane."""
        other = Lane.COMPUTE if op.lane is Lane.NETWORK else Lane.NETWORK
        hidden = _covered(op.start, op.end, [(o.start, o.end) for o in self.lane_ops(other)])
        return max(0.0, op.duration - hidden)

    def _exposed_where(self, pred) -> float:
        return sum((self.exposed_seconds(op) for op in self.ops if pred(op)), 0.0)

    def exposed_comm_seconds(self) -> float:
        return sum((self.exposed_seconds(op) for op in self.lane_ops(Lane.NETWORK)), 0.0)

    def exposed_trans_seconds(self, block: int) -> float:
        return self._exposed_where(lambda op: op.kind in TRANS_KINDS and op.block == block)

    def exposed_agg_seconds(self, block: int) -> float:
        return self._exposed_where(lambda op: op.kind in AGG_KINDS and op.block == block)

    def phase_totals(self) -> dict:
        search = self._exposed_where(lambda op: op.kind is OpKind.PLAN)
        place = self._exposed_where(lambda op: op.kind in TRANS_KINDS)
        reduce_ = self._exposed_where(lambda op: op.kind in AGG_KINDS)
        return {"search": search, "place": place, "reduce": reduce_,
                "other": self.makespan() - search - place - reduce_}

    def to_json_obj(self) -> dict:
        return {
            "iteration": self.iteration,
            "makespan": self.makespan(),
            "ops": [
                {"kind": op.kind.value, "block": op.block, "iteration": op.iteration,
                 "lane": op.lane.value, "start": op.start, "duration": op.duration}
                for op in self.ops
            ],
        }

    def to_json(self) -> str:
        return json.dumps(self.to_json_obj(), indent=2, sort_keys=True)


class _SlotWriter:
    def __init__(self, iteration: int) -> None:
        self.iteration = iteration
        self.clock = 0.0
        self.ops: list = []

    def slot(self, compute=None, network=None, compute_iteration=None) -> None:
        longest = 0.0
        for lane, entry in ((Lane.COMPUTE, compute), (Lane.NETWORK, network)):
            if entry is None or entry[2] <= 0.0:
                continue
            kind, block, dur = entry
            it = compute_iteration if (lane is Lane.COMPUTE and compute_iteration is not None) else self.iteration
            self.ops.append(ScheduledOp(kind, block, it, lane, self.clock, dur))
            longest = max(longest, dur)
        self.clock += longest

    def timeline(self) -> IterationTimeline:
        return IterationTimeline(self.iteration, tuple(self.ops))


def _check_costs(per_block_costs: Sequence, plan_time: float, model) -> list:
    costs = list(per_block_costs)
    if len(costs) != model.num_blocks:
        raise ValidationError(f"expected {model.num_blocks} block costs, got {len(costs)}")
    if plan_time < 0:
        raise ValidationError(f"plan_time must be >= 0, got {plan_time}")
    return costs


def build_iteration_timeline(per_block_costs: Sequence, plan_time: float, model, iteration: int = 0) -> IterationTimeline:
    """Algorithm 2 slot order (reference ``scheduler.py:236-283``)."""
    costs = _check_costs(per_block_costs, plan_time, model)
    L = len(costs)
    w = _SlotWriter(iteration)
    w.slot(network=(OpKind.SUB_TRANS1, 0, costs[0].trans_time))
    for i, c in enumerate(costs):
        if i + 1 < L:
            st1, st2 = partition_trans(costs[i + 1].trans_time, c.fec_time, model.fnec_time)
        else:
            st1 = st2 = 0.0
        w.slot(network=(OpKind.A2A, i, c.a2a_time), compute=(OpKind.PLAN, i, plan_time),
               compute_iteration=iteration + 1)
        w.slot(compute=(OpKind.FEC, i, c.fec_time), network=(OpKind.SUB_TRANS1, i + 1, st1))
        w.slot(network=(OpKind.A2A, i, c.a2a_time))
        w.slot(compute=(OpKind.FNEC, i, model.fnec_time), network=(OpKind.SUB_TRANS2, i + 1, st2))
    for i in reversed(range(L)):
        c = costs[i]
        if i + 1 < L:
            sa1, sa2 = partition_agg(costs[i + 1].agg_time, c.bec_time, model.bnec_time)
        else:
            sa1 = sa2 = 0.0
        w.slot(compute=(OpKind.BNEC, i, model.bnec_time), network=(OpKind.SUB_AGG1, i + 1, sa1))
        w.slot(network=(OpKind.A2A, i, c.a2a_time))
        w.slot(compute=(OpKind.BEC, i, c.bec_time), network=(OpKind.SUB_AGG2, i + 1, sa2))
        w.slot(network=(OpKind.A2A, i, c.a2a_time))
    w.slot(network=(OpKind.SUB_AGG2, 0, costs[0].agg_time))
    return w.timeline()


def build_serial_timeline(per_block_costs: Sequence, plan_time: float, model, iteration: int = 0) -> IterationTimeline:
    """No-overlap baseline (reference ``scheduler.py:286-319``)."""
    costs = _check_costs(per_block_costs, plan_time, model)
    w = _SlotWriter(iteration)
    for i, c in enumerate(costs):
        for entry in ((OpKind.PLAN, None), (OpKind.SUB_TRANS1, c.trans_time), (OpKind.A2A, c.a2a_time),
                      (OpKind.FEC, c.fec_time), (OpKind.A2A, c.a2a_time), (OpKind.FNEC, model.fnec_time)):
            kind, dur = entry
            dur = plan_time if kind is OpKind.PLAN else dur
            if LANE_OF[kind] is Lane.COMPUTE:
                w.slot(compute=(kind, i, dur))
            else:
                w.slot(network=(kind, i, dur))
    for i in reversed(range(len(costs))):
        c = costs[i]
        w.slot(compute=(OpKind.BNEC, i, model.bnec_time))
        w.slot(network=(OpKind.A2A, i, c.a2a_time))
        w.slot(compute=(OpKind.BEC, i, c.bec_time))
        w.slot(network=(OpKind.A2A, i, c.a2a_time))
        w.slot(network=(OpKind.SUB_AGG2, i, c.agg_time))
    return w.timeline()


def trans_byte_split(trans_bytes: int, trans_time: float, fec_time: float, fnec_time: float) -> tuple:
    """Turn the SubTrans1/SubTrans2 time split into a byte split of the actual
    replica payload: bytes proportional to each sub-op's share."""
    st1, st2 = partition_trans(trans_time, fec_time, fnec_time)
    if trans_time <= 0:
        return 0, 0
    b2 = int(round(trans_bytes * (st2 / trans_time)))
    return trans_bytes - b2, b2
