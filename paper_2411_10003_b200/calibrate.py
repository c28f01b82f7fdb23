"""Cost-model calibration from measured B200 runs.

The planner optimises the reference's analytic model (Eq. 1-7, 9;
``perf_model.py:36-107``) whose constants -- average bandwidth B and per-device
throughput t -- are user inputs.  This module fits them to measured per-phase
CUDA-event times of the real layer and reports the model's prediction error on
held-out iterations (the paper reports < 5 % mean error, ``PAPER.md:741``).

Per iteration j with device-derived loads (H, R) under the plan actually used:
    measured A2A  = dispatch + combine + combine_bwd + dispatch_bwd phases (4 A2As)
    measured FEC  = forward expert GEMMs,  measured BEC = backward expert GEMMs
    model: a2a = max(R) * input_bytes / B,  fec = max(H) / t,  bec = 2 fec
Fit (least squares through the origin) of the expert compute of the whole step, the model's
FEC + BEC = 3 maxH / t:  t = sum((3 maxH)^2) / sum(3 maxH * (FEC + BEC)) -- the backward GEMMs
are not exactly 2x the forward ones on B200 (the fwd/bwd kernels differ in epilogue weight),
and fitting t to FEC alone would carry that ratio into every prediction;
B = sum((maxR*ib)^2) / sum(maxR*ib * A2A/4).  Error: |model - measured| / measured of
4 a2a + fec + bec per held-out iteration.  The measured BEC/FEC ratio is reported beside it.
"""

from __future__ import annotations

import numpy as np

A2A_PHASES = (("route_layout", "barrier1"), ("fwd_gemms", "combine"), ("bwd_begin", "combine_bwd"),
              ("gate_dw", "barrier3"), ("bwd_gemms", "dispatch_bwd"))


def per_step_phases(phase_log) -> list:
    """Split a layer's phase_log into per-step {mark: ms since fwd_start} dicts."""
    steps, cur, t0 = [], None, None
    for name, ev in phase_log:
        if name == "fwd_start":
            cur, t0 = {}, ev
            steps.append(cur)
        elif cur is not None:
            cur[name] = t0.elapsed_time(ev)
    return steps


def _span(step: dict, a: str, b: str) -> float:
    return max(0.0, step.get(b, 0.0) - (step.get(a, 0.0) if a != "fwd_start" else 0.0))


def measured_costs(step: dict) -> dict:
    """Seconds per phase family of one step."""
    a2a = sum(_span(step, a, b) for a, b in A2A_PHASES) / 1e3
    fec = _span(step, "barrier1", "fwd_gemms") / 1e3
    bec = _span(step, "barrier3", "bwd_gemms") / 1e3
    return {"a2a_total": a2a, "fec": fec, "bec": bec, "layer": a2a + fec + bec}


def fit(samples, input_bytes: float) -> dict:
    """samples: list of (H, R, measured_costs dict).  Fits on the first half,
    reports the error on the second half (all samples when fewer than 4)."""
    n = len(samples)
    train = samples[: max(1, n // 2)] if n >= 4 else samples
    test = samples[n // 2:] if n >= 4 else samples
    mh = np.array([3.0 * float(np.max(h)) for h, _, _ in train])
    fec = np.array([m["fec"] + m["bec"] for _, _, m in train])  # FEC + BEC = 3 maxH / t
    mr = np.array([float(np.max(r)) * input_bytes for _, r, _ in train])
    a2a1 = np.array([m["a2a_total"] / 4.0 for _, _, m in train])
    t = float((mh * mh).sum() / max((mh * fec).sum(), 1e-30))
    B = float((mr * mr).sum() / max((mr * a2a1).sum(), 1e-30)) if mr.sum() > 0 else float("inf")
    errs, rows = [], []
    for h, r, m in test:
        fec_m = float(np.max(h)) / t
        a2a_m = float(np.max(r)) * input_bytes / B if np.isfinite(B) else 0.0
        pred = 4.0 * a2a_m + fec_m + 2.0 * fec_m
        errs.append(abs(pred - m["layer"]) / m["layer"])
        rows.append({"predicted_ms": pred * 1e3, "measured_ms": m["layer"] * 1e3})
    ratio = [m["bec"] / m["fec"] for _, _, m in samples if m["fec"] > 0]
    return {"compute_throughput": t, "avg_bandwidth": B, "mean_abs_rel_error": float(np.mean(errs)),
            "bec_over_fec_measured": float(np.median(ratio)) if ratio else None,
            "max_abs_rel_error": float(np.max(errs)), "train_iters": len(train), "test_iters": len(test),
            "test": rows}
