"""Pro-Prophet planner API (Algorithm 1, Eq. 8, locality reuse).

Drop-in for reference ``pkg/src/moebal/planner.py``: same names, argument
meaning and exceptions.  ``greedy_search`` runs on the GPU -- the
``pp_plan_greedy`` sm_100a kernel (``csrc/planner.cu``), one CTA per layer,
bit-exact against the reference (selected order, excluded sets, fp64 cost
bits).  Validation happens here first with the reference's error types.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .core import DimensionMismatchError, ExpertPlacement, ValidationError, as_counts


@dataclass(frozen=True)
class PlannerConfig:
    """Search knobs (reference ``planner.py:36-60``): n devices a selected
    expert skips, balance coefficient alpha (Eq. 8), search every
    ``reuse_interval`` iterations, and the overlap-aware objective switch."""

    n: int = 1
    alpha: float = 0.5
    reuse_interval: int = 1
    overlap_aware: bool = False

    def __post_init__(self) -> None:
        if self.n < 0:
            raise ValidationError(f"n must be >= 0, got {self.n}")
        if not self.alpha > 0:
            raise ValidationError(f"alpha must be > 0, got {self.alpha}")
        if self.reuse_interval < 1:
            raise ValidationError(f"reuse_interval must be >= 1, got {self.reuse_interval}")


def is_balanced(H, total_inputs: int, num_experts: int, alpha: float) -> bool:
    """Eq. 8: ``max(H) - min(H) < alpha * I / E`` (reference ``planner.py:63-68``)."""
    h = np.asarray(H)
    if h.size == 0:
        raise ValidationError("H must be non-empty")
    spread = float(h.max() - h.min())
    return spread < alpha * total_inputs / num_experts


def bottom_devices(load, expert: int, n: int) -> frozenset:
    """The n non-home devices with the fewest inputs for ``expert`` on the
    original matrix; ties go to the lower device index (``planner.py:71-77``).
    Host helper for API parity -- the device planner evaluates the same rule
    in ``csrc/planner.cu: bottom_rank``."""
    col = as_counts(load)[:, expert]
    order = sorted((int(c), d) for d, c in enumerate(col) if d != ExpertPlacement.home(expert))
    return frozenset(d for _, d in order[:n])


def _check_search_inputs(counts: np.ndarray, config, cluster, model) -> None:
    D, E = counts.shape
    if D != E:
        raise ValidationError(f"greedy search requires num_experts == num_devices, got D={D}, E={E}")
    if (cluster.num_devices, model.num_experts) != (D, E):
        raise DimensionMismatchError(
            f"cluster/model are {cluster.num_devices}/{model.num_experts}, load is {D}x{E}"
        )
    if config.n >= D:
        raise ValidationError(f"n must be < num_devices={D}, got {config.n}")


@dataclass(frozen=True)
class PlanResult:
    """Everything the device planner returns for one layer."""

    placement: ExpertPlacement
    best_cost: float
    explored: int
    H: np.ndarray
    R: np.ndarray


def greedy_search_many(loads: Sequence, config: PlannerConfig, cluster, model) -> list:
    """Plan L layers in one kernel launch (one CTA per layer)."""
    counts = [as_counts(x) for x in loads]
    if not counts:
        return []
    for c in counts:
        _check_search_inputs(c, config, cluster, model)
    from . import _device

    return _device.plan_greedy(np.stack(counts), config, cluster, model)


def greedy_search(load, config: PlannerConfig, cluster, model) -> ExpertPlacement:
    """Algorithm 1 (reference ``planner.py:80-129``), computed on the GPU."""
    return greedy_search_many([load], config, cluster, model)[0].placement


def greedy_search_physical_many(loads: Sequence, config: PlannerConfig, cluster, model) -> list:
    """Physically-faithful search (opt-in) for L layers: loads are
    [D][E] with E = m * D (expert e homed on device e // m).  Identical to
    ``greedy_search_many`` when E == D; for m > 1 the rule generalisation is documented
    in ``csrc/planner.cu`` and pinned only by that reduction (the reference requires
    E == D, planner.py:88-90)."""
    counts = [as_counts(x) for x in loads]
    if not counts:
        return []
    for c in counts:
        D, E = c.shape
        if E % D:
            raise ValidationError(f"num_experts must be a multiple of num_devices, got D={D}, E={E}")
        if (cluster.num_devices, model.num_experts) != (D, E):
            raise DimensionMismatchError(
                f"cluster/model are {cluster.num_devices}/{model.num_experts}, load is {D}x{E}")
        if config.n >= D:
            raise ValidationError(f"n must be < num_devices={D}, got {config.n}")
    from . import _device

    return _device.plan_physical(np.stack(counts), config, cluster, model)


def greedy_search_physical(load, config: PlannerConfig, cluster, model):
    """One layer of ``greedy_search_physical_many``; returns a PhysicalPlacement."""
    return greedy_search_physical_many([load], config, cluster, model)[0].placement


def plan_source_iteration(iter_index: int, reuse_interval: int):
    """Index of the iteration whose LoadMatrix feeds iteration ``iter_index``'s
    plan under the reuse policy (None = empty placement).  The MoE layer uses the
    same rule: after iteration i it plans for i+1 iff (i+1) % F == 0."""
    anchor = iter_index - iter_index % reuse_interval
    return None if anchor == 0 else anchor - 1


def plan_for_iteration(history: Sequence, iter_index: int, config: PlannerConfig, cluster, model) -> ExpertPlacement:
    """Reuse policy (reference ``planner.py:132-156``): search at multiples of
    ``reuse_interval`` on the previous iteration's load (persistence
    predictor); iteration 0 -- and every iteration of the first interval --
    uses the empty placement."""
    if iter_index < 0:
        raise ValidationError(f"iter_index must be >= 0, got {iter_index}")
    anchor = iter_index - iter_index % config.reuse_interval
    if anchor == 0:
        return ExpertPlacement.empty(cluster.num_devices, model.num_experts)
    if len(history) < anchor:
        raise ValidationError(
            f"iteration {iter_index} needs history through iteration {anchor - 1}, got {len(history)} entries"
        )
    return greedy_search(history[anchor - 1], config, cluster, model)
