"""Pin the CPU oracle to golden vectors produced by the unmodified reference
(tests/golden/gen_golden.py).  CPU only."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import planner_ref as P

G = Path(__file__).resolve().parent / "golden"


def load_cases():
    cases = json.loads((G / "planner_cases.json").read_text())
    counts = np.load(G / "planner_counts.npz")
    return [(c, counts[f"arr_{c['counts_index']}"]) for c in cases]


def cm_of(c):
    m = c["cm"]
    return P.cost_model_dict(m["num_devices"], m["top_k"], m["input_bytes"], m["param_bytes"],
                             m["grad_bytes"], m["avg_bandwidth"], m["compute_throughput"], m["fnec"], m["bnec"])


def check_plan(res, c):
    assert list(res["selected"]) == c["selected"]
    assert [sorted(x) for x in res["excluded"]] == c["excluded"]
    assert res["H"].tolist() == c["H"] and res["R"].tolist() == c["R"]
    assert float(res["best"]).hex() == c["best_hex"]


def test_planner_golden_cases():
    cases = load_cases()
    assert len(cases) > 400
    for c, counts in cases:
        res = P.greedy_search(counts, c["n"], c["alpha"], c["overlap"], cm_of(c))
        check_plan(res, c)


def test_appendix_b_step_traces():
    """explored-step counts and accepted plans."""
    cases = {c["tag"] + ("-ov" if c["overlap"] else ""): (c, k) for c, k in load_cases() if c["tag"].startswith("appendixB")}
    a, ka = cases["appendixB-A"]
    r = P.greedy_search(ka, 1, 0.5, False, cm_of(a))
    assert r["selected"] == (0, 1) and r["explored"] == 2
    assert float(r["best"]).hex() == "0x1.2fa66f235cb4cp-7"
    b, kb = cases["appendixB-B"]
    assert P.greedy_search(kb, 1, 0.5, False, cm_of(b))["selected"] == ()
    d, kd = cases["appendixB-D"]
    r = P.greedy_search(kd, 1, 0.5, False, cm_of(d))
    assert r["selected"] == (1, 2) and r["explored"] == 3
    assert [sorted(x) for x in r["excluded"]] == [[2], [0]]


def test_trace_plans():
    meta = json.loads((G / "trace_cases.json").read_text())
    traces = np.load(G / "trace_cases.npz")
    for c in meta:
        res = P.greedy_search(traces[c["key"]], c["n"], c["alpha"], c["overlap"], cm_of(c))
        check_plan(res, c)


def test_derive_loads_golden():
    for c in json.loads((G / "derive_cases.json").read_text()):
        counts = np.array(c["counts"])
        D, E = counts.shape
        mask = P.replica_mask(D, E, c["selected"], [frozenset(x) for x in c["excluded"]])
        assert mask.astype(int).tolist() == c["mask"]
        for fn in (P.derive_loads, P.derive_loads_cellwise):
            H, R = fn(counts, mask)
            assert H.tolist() == c["H"] and R.tolist() == c["R"]


def test_cost_terms_golden():
    for c in json.loads((G / "cost_cases.json").read_text()):
        D, B, t = c["cluster"]
        _, _, k, ib, pb, gb, fn, bn = c["model"]
        cm = P.cost_model_dict(D, k, ib, pb, gb, B, t, fn, bn)
        terms = P.cost_terms(max(c["R"]), max(c["H"]), c["s"], c["n"], cm)
        exp = {k: float.fromhex(v) for k, v in c["cost"].items()}
        assert terms["a2a"] == exp["a2a_time"] and terms["fec"] == exp["fec_time"]
        assert terms["trans"] == exp["trans_time"] and terms["agg"] == exp["agg_time"]
        assert terms["ptrans"] == exp["ptrans_time"] and terms["pagg"] == exp["pagg_time"]
        assert terms["unscheduled"] == exp["total_unscheduled"]
        assert terms["scheduled"] == exp["total_scheduled"]


def test_metrics_golden():
    for c in json.loads((G / "metric_cases.json").read_text()):
        assert P.balance_degree(c["a"]) == c["sigma_a"]
        assert repr(P.rb_ratio(c["a"], c["b"])) == c["rb"]


def test_oracle_against_live_reference(rng):
    """Where the reference is importable (build container) cross-check fresh
    random instances directly."""
    from conftest import import_reference

    ref = import_reference()
    from moebal.planner import PlannerConfig

    for i in range(150):
        D = int(rng.integers(2, 20))
        probs = rng.dirichlet(np.ones(D) * 0.4)
        counts = np.stack([rng.multinomial(97, probs) for _ in range(D)])
        cl = ref.ClusterSpec(D, 1e9 * (1 + i % 7), 1e3 * (1 + i % 5))
        mo = ref.ModelSpec(D, 1, 1, 1e6, 1e5 * (1 + i % 3), 2e5, fnec_time=1e-3 * (i % 4), bnec_time=2e-3)
        n = int(rng.integers(0, D))
        ov = bool(i % 2)
        pl = ref.greedy_search(ref.LoadMatrix(counts), PlannerConfig(n=n, alpha=0.5, overlap_aware=ov), cl, mo)
        cm = P.cost_model_dict(D, 1, 1e6, mo.expert_param_bytes, 2e5, cl.avg_bandwidth, cl.compute_throughput,
                               mo.fnec_time, mo.bnec_time)
        res = P.greedy_search(counts, n, 0.5, ov, cm)
        assert res["selected"] == pl.selected
        assert tuple(frozenset(x) for x in res["excluded"]) == pl.excluded


def test_physical_planner_reduces_to_reference_at_m1():
    """The physically-faithful E > D search is parity-pinned by
    reduction: at m = E / D = 1 it must reproduce every reference golden plan."""
    for c, counts in load_cases():
        res = P.greedy_search_physical(counts, c["n"], c["alpha"], c["overlap"], cm_of(c))
        check_plan(res, c)
        assert res["explored"] == P.greedy_search(counts, c["n"], c["alpha"], c["overlap"], cm_of(c))["explored"]


def test_physical_derive_loads_rules(rng):
    """Physical derive_loads (homes e // m) == the slot-level rule summed per device, and
    at m = 1 == the reference derive_loads restatement."""
    for _ in range(50):
        D = int(rng.integers(2, 6))
        m = int(rng.integers(1, 4))
        E = D * m
        counts = rng.integers(0, 9, size=(D, E))
        mask = rng.random((D, E)) < 0.3
        for e in range(E):
            mask[e // m, e] = True
        H, R = P.derive_loads_physical(counts, mask)
        assert H.sum() == counts.sum() and R.sum() == sum(int(counts[d, e]) for d in range(D) for e in range(E)
                                                          if not mask[d, e])
        if m == 1:
            H1, R1 = P.derive_loads(counts, mask)
            assert H.tolist() == H1.tolist() and R.tolist() == R1.tolist()
    # fuzz over m > 1: the returned plan never costs more than vanilla EP, conserves rows, keeps homes
    for i in range(40):
        D = int(rng.integers(2, 9))
        m = int(rng.integers(2, 5))
        E = D * m
        probs = rng.dirichlet(np.ones(E) * 0.3)
        counts = np.stack([rng.multinomial(512, probs) for _ in range(D)])
        cm = P.cost_model_dict(D, 2, 2048, 1.6e7, 3.2e7, 4e11, 1e8 * (1 + i % 4))
        res = P.greedy_search_physical(counts, int(rng.integers(0, D)), 0.5, bool(i % 2), cm)
        H0, R0 = P.derive_loads_physical(counts, P.replica_mask_physical(D, E, (), ()))
        assert res["best"] <= P.objective(H0, R0, 0, 0, cm, bool(i % 2))  # strict improvements only
        assert res["H"].sum() == counts.sum()
        assert all(e // m != d or res["mask"][d, e] for d in range(D) for e in range(E))


def test_slot_refinement_properties(rng):
    """refine_slots (opt-in extension): conserves rows, keeps every home slot local,
    only un-routes replica slots, and never raises the heaviest device."""
    for i in range(30):
        D = int(rng.integers(2, 6))
        m = int(rng.integers(2, 5))
        E = D * m
        p = rng.dirichlet(np.ones(E) * 0.3)
        slot = np.stack([rng.multinomial(128, p) for _ in range(E)]).astype(np.int64)
        phys = slot.reshape(D, m, E).sum(axis=1)
        cm = P.cost_model_dict(D, 2, 2048, 1.6e7, 3.2e7, 4e11, 1e8)
        plan = P.greedy_search_physical(phys, 0, 0.5, bool(i % 2), cm)
        S, H, R = P.refine_slots(slot, plan["mask"])
        full = np.repeat(plan["mask"], m, axis=0)
        assert H.sum() == slot.sum() and H.max() <= plan["H"].max()
        assert not (S & ~full).any()  # only removals
        for v in range(E):
            for e in range(E):
                if e // m == v // m:
                    assert S[v, e] == full[v, e]  # home slots untouched
