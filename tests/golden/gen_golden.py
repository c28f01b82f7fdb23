"""Generate the golden fixtures by running the UNMODIFIED reference (moebal).

Run in the build container (the reference is importable there, not on the GPU box):

    python tests/golden/gen_golden.py            # writes tests/golden/*.json / *.npz

Fixtures:
  planner_cases.json + planner_counts.npz  greedy_search results (selected, excluded,
      objective of the returned plan as float.hex, H, R) on FIG8, the SURVEY
      appendix-B setups, reference-test-style random matrices and fuzzed instances
  trace_cases.npz + trace_cases.json       reference generate_trace LoadMatrices for the
      BASELINE configs in virtual-slot form (E x E) and the reference plan of each
  derive_cases.json                        derive_loads H/R for random placements
  cost_cases.json                          LayerCost fields (float.hex)
  timeline_cases.json                      build_iteration_timeline / build_serial_timeline
  metric_cases.json                        balance_degree / rb_ratio
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("PPMOE_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from moebal import (  # noqa: E402
    ClusterSpec, ExpertPlacement, GeneratorConfig, LoadMatrix, ModelSpec, balance_degree,
    build_iteration_timeline, build_serial_timeline, derive_loads, generate_trace, greedy_search,
    rb_ratio,
)
from moebal.perf_model import layer_cost_scheduled, layer_cost_unscheduled  # noqa: E402
from moebal.planner import PlannerConfig  # noqa: E402

OUT = Path(__file__).resolve().parent


def plan_record(counts, n, alpha, overlap, cluster, model):
    load = LoadMatrix(counts)
    cfg = PlannerConfig(n=n, alpha=alpha, overlap_aware=overlap)
    pl = greedy_search(load, cfg, cluster, model)
    loads = derive_loads(load, pl)
    fn = layer_cost_scheduled if overlap else layer_cost_unscheduled
    c = fn(loads, pl.num_selected, n if pl.num_selected else 0, cluster, model)
    best = c.total_scheduled if overlap else c.total_unscheduled
    return {
        "n": n, "alpha": alpha, "overlap": overlap,
        "cm": {"num_devices": cluster.num_devices, "top_k": model.top_k,
               "input_bytes": float(model.input_bytes), "param_bytes": float(model.expert_param_bytes),
               "grad_bytes": float(model.expert_grad_bytes), "avg_bandwidth": float(cluster.avg_bandwidth),
               "compute_throughput": float(cluster.compute_throughput),
               "fnec": float(model.fnec_time), "bnec": float(model.bnec_time)},
        "selected": list(pl.selected),
        "excluded": [sorted(x) for x in pl.excluded],
        "best_hex": float(best).hex(),
        "H": loads.H.tolist(), "R": loads.R.tolist(),
    }


def random_counts(rng, D, row_total):
    probs = rng.dirichlet(np.ones(D) * rng.choice([0.2, 0.5, 1.0, 3.0]))
    return np.stack([rng.multinomial(row_total, probs) for _ in range(D)]).astype(np.int64)


def main() -> None:
    rng = np.random.default_rng(20240817)
    cases, counts_list = [], []

    def add(counts, n, alpha, overlap, cluster, model, tag):
        rec = plan_record(counts, n, alpha, overlap, cluster, model)
        rec["tag"] = tag
        rec["counts_index"] = len(counts_list)
        counts_list.append(np.asarray(counts, dtype=np.int64))
        cases.append(rec)

    fig8 = [[3, 0, 0], [2, 1, 0], [0, 1, 2]]
    c3 = ClusterSpec(3, 1e9, 1000.0)
    for pb, gb, fn, bn, tag in ((1e5, 1e5, 0, 0, "A"), (1e12, 1e12, 0, 0, "B"), (1.2e7, 1.2e7, 1.0, 1.0, "C")):
        m = ModelSpec(3, 1, 1, 1e6, pb, gb, fnec_time=fn, bnec_time=bn)
        for ov in (False, True):
            add(fig8, 1, 0.5, ov, c3, m, f"appendixB-{tag}")
    d4 = [[0, 6, 5, 1], [0, 5, 6, 1], [0, 5, 4, 3], [0, 6, 6, 0]]
    add(d4, 1, 0.5, False, ClusterSpec(4, 1e9, 1000.0), ModelSpec(4, 1, 1, 1e6, 1e5, 1e5), "appendixB-D")
    # tie-break matrix of test_planner.py:58
    add([[2, 1, 0], [1, 2, 0], [1, 0, 2]], 1, 0.5, False, c3, ModelSpec(3, 1, 1, 1e6, 1e5, 1e5), "ties")

    # conftest-calibrated random instances (D=8) and fuzz over D, n, objective, constants
    for i in range(120):
        D = 8
        cl = ClusterSpec(D, 25e9, 1e6)
        mo = ModelSpec(D, 4, 1, 4096, 4e6, 4e6, fnec_time=2e-4, bnec_time=4e-4)
        add(random_counts(rng, D, 256), int(rng.integers(0, 3)), 0.5, bool(i % 2), cl, mo, "calibrated")
    Ds = [2, 3, 4, 5, 6, 8, 12, 16, 24, 32, 48, 64]
    for i in range(360):
        D = int(Ds[i % len(Ds)])
        k = int(rng.integers(1, 3))
        row_total = int(rng.integers(1, 200)) * k
        cl = ClusterSpec(D, float(10 ** rng.uniform(8, 11.5)), float(10 ** rng.uniform(3, 7)))
        mo = ModelSpec(D, 1, min(k, D), float(rng.integers(1, 1 << 16)), float(10 ** rng.uniform(3, 9)),
                       float(10 ** rng.uniform(3, 9)), fnec_time=float(rng.uniform(0, 1e-3)),
                       bnec_time=float(rng.uniform(0, 2e-3)))
        n = int(rng.integers(0, D))
        alpha = float(rng.choice([0.05, 0.2, 0.5, 1.0, 2.0]))
        add(random_counts(rng, D, row_total), n, alpha, bool(rng.integers(0, 2)), cl, mo, "fuzz")

    np.savez_compressed(OUT / "planner_counts.npz", *counts_list)
    (OUT / "planner_cases.json").write_text(json.dumps(cases))

    # ---- generator traces for the BASELINE configs (virtual E x E slots)
    traces, tmeta = {}, []
    configs = [
        ("cfg1", 8, 2, 4096, 512, 1024),
        ("cfg3_d8", 32, 2, 8 * 32768, 2048, 4096),
        ("cfg4_k1", 64, 1, 8 * 32768, 2048, 4096),
        ("cfg4_k2", 64, 2, 8 * 32768, 2048, 4096),
    ]
    for name, E, k, inputs, dm, df in configs:
        gen = GeneratorConfig(num_devices=E, num_experts=E, inputs_per_iteration=inputs, top_k=k,
                              skew=1.2, drift=0.05, seed=7)
        recs = generate_trace(gen, 4, 2)
        cl = ClusterSpec(E, 450e9, 1.2e15 / (6.0 * dm * df))
        mo = ModelSpec(E, 2, k, 2 * dm, 4 * dm * df, 8 * dm * df)
        for ri, r in enumerate(recs):
            key = f"{name}_{ri}"
            traces[key] = r.load.counts
            for ov in (False, True):
                rec = plan_record(r.load.counts, 1, 0.5, ov, cl, mo)
                rec.update(key=key, config=name, iteration=r.iteration, layer=r.layer)
                tmeta.append(rec)
    np.savez_compressed(OUT / "trace_cases.npz", **traces)
    (OUT / "trace_cases.json").write_text(json.dumps(tmeta))

    # ---- derive_loads on random placements
    dcases = []
    for i in range(60):
        D = int(rng.integers(2, 12))
        E = int(rng.integers(1, D + 1))
        counts = np.stack([rng.multinomial(50, np.ones(E) / E) for _ in range(D)])
        s = int(rng.integers(0, E + 1))
        n = int(rng.integers(0, D))
        sel = [int(x) for x in rng.permutation(E)[:s]]
        exc = []
        for e in sel:
            cand = [d for d in range(D) if d != e]
            exc.append(sorted(int(x) for x in rng.permutation(cand)[:min(n, len(cand))]))
        if len({len(x) for x in exc}) > 1:
            continue
        pl = ExpertPlacement(D, E, tuple(sel), tuple(frozenset(x) for x in exc))
        dl = derive_loads(LoadMatrix(counts), pl)
        dcases.append({"counts": counts.tolist(), "selected": sel, "excluded": exc,
                       "mask": pl.replica_mask().astype(int).tolist(), "H": dl.H.tolist(), "R": dl.R.tolist()})
    (OUT / "derive_cases.json").write_text(json.dumps(dcases))

    # ---- LayerCost goldens
    ccases = []
    for i in range(40):
        D = int(rng.integers(2, 10))
        H = rng.integers(0, 1000, D)
        R = rng.integers(0, 500, D)
        from moebal import DeviceLoads
        loads = DeviceLoads(H=H, R=R)
        cl = ClusterSpec(D, float(10 ** rng.uniform(8, 11)), float(10 ** rng.uniform(3, 7)))
        mo = ModelSpec(D, 1, 1, float(rng.integers(1, 9999)), float(10 ** rng.uniform(3, 9)),
                       float(10 ** rng.uniform(3, 9)), fnec_time=float(rng.uniform(0, 1e-3)),
                       bnec_time=float(rng.uniform(0, 1e-3)))
        s, n = int(rng.integers(0, D + 1)), int(rng.integers(0, D))
        c = layer_cost_unscheduled(loads, s, n, cl, mo)
        ccases.append({"H": H.tolist(), "R": R.tolist(), "s": s, "n": n,
                       "cluster": [cl.num_devices, cl.avg_bandwidth, cl.compute_throughput],
                       "model": [mo.num_experts, mo.num_blocks, mo.top_k, mo.input_bytes, mo.expert_param_bytes,
                                 mo.expert_grad_bytes, mo.fnec_time, mo.bnec_time],
                       "cost": {k: float(v).hex() for k, v in c.__dict__.items()}})
    (OUT / "cost_cases.json").write_text(json.dumps(ccases))

    # ---- timelines
    tcases = []
    for i in range(12):
        L = int(rng.integers(1, 5))
        mo = ModelSpec(4, L, 1, 1.0, 1.0, 1.0, fnec_time=float(rng.uniform(0, 3e-3)),
                       bnec_time=float(rng.uniform(0, 6e-3)))
        from moebal import LayerCost
        costs = []
        for _ in range(L):
            v = [float(u) for u in rng.uniform(0, 4e-3, 5)]  # Python floats, as JSON configs give
            costs.append(LayerCost(v[0], v[1], 2 * v[1], v[2], v[3], 0.0, 0.0, 0.0, 0.0))
        plan_time = float(rng.uniform(0, 1e-3))
        tl = build_iteration_timeline(costs, plan_time, mo, iteration=i)
        ts = build_serial_timeline(costs, plan_time, mo, iteration=i)
        tcases.append({"costs": [[c.a2a_time, c.fec_time, c.bec_time, c.trans_time, c.agg_time] for c in costs],
                       "plan_time": plan_time, "fnec": mo.fnec_time, "bnec": mo.bnec_time, "L": L, "iteration": i,
                       "overlapped": tl.to_json_obj(), "serial": ts.to_json_obj(),
                       "phase": tl.phase_totals(), "exposed_comm": tl.exposed_comm_seconds()})
    (OUT / "timeline_cases.json").write_text(json.dumps(tcases))

    # ---- metrics
    mcases = []
    from moebal import DeviceLoads
    for i in range(30):
        D = int(rng.integers(1, 9))
        a = rng.integers(0, 100, D)
        b = rng.integers(0, 100, D) if i % 3 else np.full(D, 7)
        mcases.append({"a": a.tolist(), "b": b.tolist(), "sigma_a": balance_degree(a),
                       "rb": repr(rb_ratio(DeviceLoads(a, a * 0), DeviceLoads(b, b * 0)))})
    (OUT / "metric_cases.json").write_text(json.dumps(mcases))
    print(f"planner cases {len(cases)}, trace plans {len(tmeta)}, derive {len(dcases)}, "
          f"cost {len(ccases)}, timelines {len(tcases)}, metrics {len(mcases)}")


if __name__ == "__main__":
    main()
