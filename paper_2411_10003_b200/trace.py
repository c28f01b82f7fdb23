"""GPU-trace I/O in the reference's JSONL format.

Each record is one (iteration, layer) LoadMatrix -- here the virtual-slot
matrix the device histogram produced -- written exactly like reference
``workload.write_trace`` (``workload.py:177-184``: one compact JSON object per
line, keys ``iter``, ``layer``, ``counts``), so ``moebal simulate/compare`` can
replay real B200 routing.  ``read_trace`` mirrors the reference reader's
validation (``workload.py:187-227``).
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .core import LoadMatrix, ValidationError


class TraceFormatError(ValidationError):
    def __init__(self, lineno: int, msg: str) -> None:
        super().__init__(f"line {lineno}: {msg}")
        self.lineno = lineno


@dataclass(frozen=True)
class TraceRecord:
    iteration: int
    layer: int
    load: LoadMatrix


def write_trace(records: Sequence[TraceRecord], path) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        for rec in records:
            fh.write(json.dumps({"iter": rec.iteration, "layer": rec.layer,
                                 "counts": np.asarray(rec.load.counts).tolist()}, separators=(",", ":")))
            fh.write("\n")


def read_trace(path) -> list:
    out, shape = [], None
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            raw = raw.strip()
            if not raw:
                continue
            try:
                obj = json.loads(raw)
            except json.JSONDecodeError as exc:
                raise TraceFormatError(lineno, f"invalid JSON: {exc.msg}") from exc
            if not isinstance(obj, dict):
                raise TraceFormatError(lineno, "record must be a JSON object")
            missing = [k for k in ("iter", "layer", "counts") if k not in obj]
            if missing:
                raise TraceFormatError(lineno, f"missing key {missing[0]!r}")
            if not isinstance(obj["iter"], int) or not isinstance(obj["layer"], int):
                raise TraceFormatError(lineno, "iter and layer must be integers")
            try:
                load = LoadMatrix(obj["counts"])
            except (ValidationError, ValueError) as exc:
                raise TraceFormatError(lineno, f"bad counts: {exc}") from exc
            dims = (load.num_devices, load.num_experts)
            if shape is None:
                shape = dims
            elif dims != shape:
                raise TraceFormatError(lineno, f"dimensions {dims[0]}x{dims[1]} do not match earlier records "
                                               f"({shape[0]}x{shape[1]})")
            out.append(TraceRecord(obj["iter"], obj["layer"], load))
    iters = sorted({r.iteration for r in out})
    if iters and iters != list(range(len(iters))):
        raise ValidationError(f"iterations must be contiguous from 0, got {iters[:10]}...")
    return out


class TraceRecorder:
    """Collects the LoadMatrix every MoELayer produced per iteration (device
    copies, moved to the host only at ``records()``), layer index = position."""

    def __init__(self, layers) -> None:
        self.layers = list(layers)
        self._dev = []  # (iteration, layer, device tensor)

    def capture(self, iteration: int) -> None:
        """Snapshot the current LoadMatrix of every layer (stream-ordered)."""
        for li, layer in enumerate(self.layers):
            self._dev.append((iteration, li, layer.counts.clone()))

    def records(self) -> list:
        return [TraceRecord(it, li, LoadMatrix(t.cpu().numpy())) for it, li, t in self._dev]

    def write(self, path) -> None:
        write_trace(self.records(), path)
