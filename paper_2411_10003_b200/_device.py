"""Device entry points behind the reference-shaped Python API.

torch is used only for device memory and streams; every computation is a
call through the C ABI (``_lib``).  Functions here raise if no GPU or no
library is present -- nothing falls back to host arithmetic.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .core import ExpertPlacement, PhysicalPlacement


def _require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2411_10003_b200 needs a CUDA device (B200); there is no CPU path")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def num_sms(device) -> int:
    return torch.cuda.get_device_properties(device).multi_processor_count


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def cost_model(cluster, model, E: int | None = None) -> _lib.CostModel:
    cm = _lib.CostModel()
    cm.input_bytes = float(model.input_bytes)
    cm.expert_param_bytes = float(model.expert_param_bytes)
    cm.expert_grad_bytes = float(model.expert_grad_bytes)
    cm.avg_bandwidth = float(cluster.avg_bandwidth)
    cm.compute_throughput = float(cluster.compute_throughput)
    cm.fnec_time = float(model.fnec_time)
    cm.bnec_time = float(model.bnec_time)
    cm.num_devices = int(cluster.num_devices if E is None else E)
    cm.num_experts = int(model.num_experts if E is None else E)
    cm.top_k = int(model.top_k)
    return cm


def planner_cfg(config, max_replicas: int = 0, slots_per_rank: int = 1, iter_counter=None) -> _lib.PlannerCfg:
    """pp_planner_cfg from a reference PlannerConfig; the extensions default to the
    reference's behaviour (no replica bound, no device-side reuse gate)."""
    c = _lib.PlannerCfg()
    c.alpha = float(config.alpha)
    c.n = int(config.n)
    c.overlap_aware = 1 if config.overlap_aware else 0
    c.reuse_interval = int(getattr(config, "reuse_interval", 1))
    c.max_replicas = int(max_replicas)
    c.slots_per_rank = int(slots_per_rank)
    c.iter_counter = None if iter_counter is None else iter_counter.data_ptr()
    return c


class PlanBuffers:
    """Device outputs of pp_plan_greedy for L layers of E x E slots."""

    def __init__(self, L: int, E: int, device) -> None:
        self.L, self.E = L, E
        self.selected = torch.empty((L, E), dtype=torch.int32, device=device)
        self.num_selected = torch.empty((L,), dtype=torch.int32, device=device)
        self.num_explored = torch.empty((L,), dtype=torch.int32, device=device)
        self.mask = torch.empty((L, E, E), dtype=torch.uint8, device=device)
        self.H = torch.empty((L, E), dtype=torch.int64, device=device)
        self.R = torch.empty((L, E), dtype=torch.int64, device=device)
        self.best = torch.empty((L,), dtype=torch.float64, device=device)


def launch_plan(counts_dev: torch.Tensor, out: PlanBuffers, cm, cfg, stream=None, physical_devices: int = 0,
                refine_slots: bool = False) -> None:
    """physical_devices = D > 0: the physically-faithful search (pp_plan_physical) over
    D devices; counts_dev rows may be D physical rows or virtual-slot rows (then
    refine_slots may trim replica routing per slot)."""
    L, rows, E = counts_dev.shape
    if physical_devices:
        _lib.call(
            "pp_plan_physical", counts_dev.data_ptr(), L, rows, physical_devices, E, ctypes.byref(cm),
            ctypes.byref(cfg), 1 if refine_slots else 0, out.selected.data_ptr(), out.num_selected.data_ptr(), out.num_explored.data_ptr(),
            out.mask.data_ptr(), out.H.data_ptr(), out.R.data_ptr(), out.best.data_ptr(), stream_ptr(stream),
        )
        return
    _lib.call(
        "pp_plan_greedy", counts_dev.data_ptr(), L, E, ctypes.byref(cm), ctypes.byref(cfg),
        out.selected.data_ptr(), out.num_selected.data_ptr(), out.num_explored.data_ptr(),
        out.mask.data_ptr(), out.H.data_ptr(), out.R.data_ptr(), out.best.data_ptr(),
        stream_ptr(stream),
    )


def plan_greedy(counts: np.ndarray, config, cluster, model) -> list:
    from .planner import PlanResult

    dev = _require_cuda()
    L, E, _ = counts.shape
    counts_dev = torch.from_numpy(np.ascontiguousarray(counts, dtype=np.int64)).to(dev)
    out = PlanBuffers(L, E, dev)
    launch_plan(counts_dev, out, cost_model(cluster, model, E), planner_cfg(config))
    sel = out.selected.cpu().numpy()
    nsel = out.num_selected.cpu().numpy()
    nexp = out.num_explored.cpu().numpy()
    mask = out.mask.cpu().numpy().astype(bool)
    H, R, best = out.H.cpu().numpy(), out.R.cpu().numpy(), out.best.cpu().numpy()
    results = []
    for l in range(L):
        chosen = [int(x) for x in sel[l, : nsel[l]]]
        placement = ExpertPlacement.from_mask(chosen, mask[l])
        results.append(PlanResult(placement, float(best[l]), int(nexp[l]), H[l].copy(), R[l].copy()))
    return results


def plan_physical(counts: np.ndarray, config, cluster, model) -> list:
    """counts [L][D][E] physical LoadMatrices -> PlanResult per layer (mask [D][E])."""
    from .planner import PlanResult

    dev = _require_cuda()
    L, D, E = counts.shape
    counts_dev = torch.from_numpy(np.ascontiguousarray(counts, dtype=np.int64)).to(dev)
    out = PlanBuffers(L, E, dev)
    out.mask = torch.empty((L, D, E), dtype=torch.uint8, device=dev)
    launch_plan(counts_dev, out, cost_model(cluster, model), planner_cfg(config), physical_devices=D)
    sel = out.selected.cpu().numpy()
    nsel = out.num_selected.cpu().numpy()
    nexp = out.num_explored.cpu().numpy()
    mask = out.mask.cpu().numpy().astype(bool)
    H, R, best = out.H.cpu().numpy(), out.R.cpu().numpy(), out.best.cpu().numpy()
    results = []
    for l in range(L):
        chosen = [int(x) for x in sel[l, : nsel[l]]]
        results.append(PlanResult(PhysicalPlacement.from_mask(chosen, mask[l]), float(best[l]), int(nexp[l]),
                                  H[l, :D].copy(), R[l, :D].copy()))
    return results


def derive_loads(counts: np.ndarray, mask: np.ndarray):
    dev = _require_cuda()
    D, E = counts.shape
    c = torch.from_numpy(np.ascontiguousarray(counts, dtype=np.int64)).to(dev)
    m = torch.from_numpy(np.ascontiguousarray(mask, dtype=np.uint8)).to(dev)
    H = torch.empty((D,), dtype=torch.int64, device=dev)
    R = torch.empty((D,), dtype=torch.int64, device=dev)
    _lib.call("pp_derive_loads", c.data_ptr(), m.data_ptr(), D, E, H.data_ptr(), R.data_ptr(),
              stream_ptr())
    return H.cpu().numpy(), R.cpu().numpy()


def grouped_gemm(mode: int, a, b, c, c2, groups, num_groups, max_groups: int, rows_capacity: int,
                 num_slots: int, d_model: int, d_ff: int, num_sms: int = 0, stream=None) -> None:
    _lib.call(
        "pp_grouped_gemm", mode, a.data_ptr(), b.data_ptr(), c.data_ptr(), ptr(c2),
        groups.data_ptr(), num_groups.data_ptr(), max_groups, rows_capacity, num_slots,
        d_model, d_ff, num_sms, stream_ptr(stream),
    )


def groups_tensor(rows_per_group, wslots=None, device=None):
    """Build a packed pp_group table (host helper for tests / single-rank use)."""
    g = len(rows_per_group)
    t = torch.zeros((max(g, 1), 8), dtype=torch.int32)
    off = 0
    for i, r in enumerate(rows_per_group):
        pad = (r + _lib.PP_ROW_ALIGN - 1) // _lib.PP_ROW_ALIGN * _lib.PP_ROW_ALIGN
        t[i, 0], t[i, 1], t[i, 2] = off, r, pad
        t[i, 3] = i if wslots is None else wslots[i]
        t[i, 4] = i
        off += pad
    n = torch.tensor([g], dtype=torch.int32)
    dev = device or torch.device("cuda")
    return t.to(dev), n.to(dev), off
