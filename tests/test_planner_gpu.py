"""Device planner K2 (pp_plan_greedy) bit-exact against the pinned oracle and the
reference goldens: selected order, excluded sets, H/R, fp64 objective bits."""

import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2411_10003_b200 as pp  # noqa: E402
from oracle import planner_ref as P  # noqa: E402

G = Path(__file__).resolve().parent / "golden"


def specs(cm, E):
    cl = pp.ClusterSpec(E, cm["avg_bandwidth"], cm["compute_throughput"])
    mo = pp.ModelSpec(E, 1, cm["top_k"], cm["input_bytes"], cm["param_bytes"], cm["grad_bytes"],
                      fnec_time=cm["fnec"], bnec_time=cm["bnec"])
    return cl, mo


def assert_same(res, c):
    pl = res.placement
    assert list(pl.selected) == c["selected"]
    assert [sorted(x) for x in pl.excluded] == c["excluded"]
    assert res.H.tolist() == c["H"] and res.R.tolist() == c["R"]
    assert float(res.best_cost).hex() == c["best_hex"]


def test_golden_planner_cases():
    cases = json.loads((G / "planner_cases.json").read_text())
    counts = np.load(G / "planner_counts.npz")
    for c in cases:
        k = counts[f"arr_{c['counts_index']}"]
        E = k.shape[0]
        cl, mo = specs(c["cm"], E)
        cfg = pp.PlannerConfig(n=c["n"], alpha=c["alpha"], overlap_aware=c["overlap"])
        res = pp.greedy_search_many([k], cfg, cl, mo)[0]
        assert_same(res, c)


def test_golden_generator_traces():
    meta = json.loads((G / "trace_cases.json").read_text())
    traces = np.load(G / "trace_cases.npz")
    for c in meta:
        k = traces[c["key"]]
        cl, mo = specs(c["cm"], k.shape[0])
        cfg = pp.PlannerConfig(n=c["n"], alpha=c["alpha"], overlap_aware=c["overlap"])
        assert_same(pp.greedy_search_many([k], cfg, cl, mo)[0], c)


@pytest.mark.parametrize("E", [2, 3, 5, 8, 16, 32, 64, 128])
def test_fuzz_vs_oracle(E):
    """>= 10 000 instances over all E values (batched, one CTA per instance)."""
    rng = np.random.default_rng(1000 + E)
    batches = 8 if E <= 64 else 2
    per = 200 if E <= 64 else 50
    for b in range(batches):
        k = int(rng.integers(1, 3))
        cm = P.cost_model_dict(E, k, float(rng.integers(1, 1 << 14)), float(10 ** rng.uniform(3, 8)),
                               float(10 ** rng.uniform(3, 8)), float(10 ** rng.uniform(8, 11)),
                               float(10 ** rng.uniform(3, 6)), float(rng.uniform(0, 1e-3)),
                               float(rng.uniform(0, 2e-3)))
        n = int(rng.integers(0, E))
        alpha = float(rng.choice([0.05, 0.3, 0.5, 1.5]))
        ov = bool(b % 2)
        row_total = int(rng.integers(1, 400)) * k
        mats = []
        for _ in range(per):
            probs = rng.dirichlet(np.ones(E) * rng.choice([0.1, 0.5, 2.0]))
            mats.append(np.stack([rng.multinomial(row_total, probs) for _ in range(E)]))
        cl = pp.ClusterSpec(E, cm["avg_bandwidth"], cm["compute_throughput"])
        mo = pp.ModelSpec(E, 1, k, cm["input_bytes"], cm["expert_param_bytes"], cm["expert_grad_bytes"],
                          fnec_time=cm["fnec_time"], bnec_time=cm["bnec_time"])
        res = pp.greedy_search_many(mats, pp.PlannerConfig(n=n, alpha=alpha, overlap_aware=ov), cl, mo)
        for mat, r in zip(mats, res):
            o = P.greedy_search(mat, n, alpha, ov, cm)
            assert r.placement.selected == o["selected"]
            assert r.placement.excluded == tuple(frozenset(x) for x in o["excluded"])
            assert r.explored == o["explored"]
            assert float(r.best_cost).hex() == float(o["best"]).hex()
            assert r.H.tolist() == o["H"].tolist() and r.R.tolist() == o["R"].tolist()


def test_derive_loads_golden():
    for c in json.loads((G / "derive_cases.json").read_text()):
        counts = np.array(c["counts"])
        D, E = counts.shape
        pl = pp.ExpertPlacement(D, E, tuple(c["selected"]), tuple(frozenset(x) for x in c["excluded"]))
        dl = pp.derive_loads(pp.LoadMatrix(counts), pl)
        assert dl.H.tolist() == c["H"] and dl.R.tolist() == c["R"]


def test_reference_api_errors():
    cl = pp.ClusterSpec(3, 1e9, 1e3)
    mo = pp.ModelSpec(3, 1, 1, 1e6, 1e5, 1e5)
    with pytest.raises(pp.ValidationError):
        pp.greedy_search(pp.LoadMatrix([[1, 2], [2, 1], [0, 3]]), pp.PlannerConfig(), cl, mo)
    with pytest.raises(pp.DimensionMismatchError):
        pp.greedy_search(pp.LoadMatrix([[1, 2], [2, 1]]), pp.PlannerConfig(), cl, mo)
    with pytest.raises(pp.ValidationError):
        pp.greedy_search(pp.LoadMatrix([[3, 0, 0], [2, 1, 0], [0, 1, 2]]), pp.PlannerConfig(n=3), cl, mo)


def test_plan_for_iteration_reuse():
    """plan_for_iteration (device search) against the pinned oracle's reuse rule and search
    (planner.py:132-156) on a drifting history whose plans differ between anchors."""
    E = 8
    rng = np.random.default_rng(31)
    hist = [pp.LoadMatrix(np.stack([rng.multinomial(256, rng.dirichlet(np.ones(E) * (0.15 + 0.1 * (j % 3))))
                                    for _ in range(E)]).astype(np.int64)) for j in range(9)]
    cm = P.cost_model_dict(E, 1, 1e6, 1e5, 1e5, 1e9, 1000.0)
    cl = pp.ClusterSpec(E, 1e9, 1000.0)
    mo = pp.ModelSpec(E, 1, 1, 1e6, 1e5, 1e5)
    for F in (1, 2, 3):
        cfg = pp.PlannerConfig(n=1, alpha=0.5, reuse_interval=F)
        seen = set()
        for j in range(len(hist) + 1):
            got = pp.plan_for_iteration(hist, j, cfg, cl, mo)
            exp = P.plan_for_iteration([h.counts for h in hist], j, F,
                                       lambda c: P.greedy_search(c, 1, 0.5, False, cm))
            if exp is None:
                assert got.selected == (), (F, j)
            else:
                assert list(got.selected) == list(exp["selected"]), (F, j)
                assert got.replica_mask().tolist() == exp["mask"].tolist()
                seen.add(tuple(exp["selected"]))
        assert len(seen) > 1  # the history really changes the plan
    with pytest.raises(pp.ValidationError):
        pp.plan_for_iteration(hist, 20, pp.PlannerConfig(n=1, alpha=0.5, reuse_interval=2), cl, mo)


# ---- physically-faithful E > D planner (pp_plan_physical) ----------

def test_physical_planner_equals_reference_at_m1():
    """At m = E / D = 1 the physical search is the reference search, bit for bit."""
    cases = json.loads((G / "planner_cases.json").read_text())
    counts = np.load(G / "planner_counts.npz")
    for c in cases:
        k = counts[f"arr_{c['counts_index']}"]
        cl, mo = specs(c["cm"], k.shape[0])
        cfg = pp.PlannerConfig(n=c["n"], alpha=c["alpha"], overlap_aware=c["overlap"])
        res = pp.greedy_search_physical_many([k], cfg, cl, mo)[0]
        assert_same(res, c)
        assert res.explored == pp.greedy_search_many([k], cfg, cl, mo)[0].explored


@pytest.mark.parametrize("D,m", [(2, 2), (2, 8), (4, 4), (8, 2), (8, 8), (16, 4), (3, 5)])
def test_physical_planner_fuzz_vs_oracle(D, m):
    E = D * m
    rng = np.random.default_rng(77 + D * 100 + m)
    mats, cfgs = [], []
    for i in range(60):
        probs = rng.dirichlet(np.ones(E) * (0.2 + 0.3 * (i % 4)))
        mats.append(np.stack([rng.multinomial(256 * m, probs) for _ in range(D)]).astype(np.int64))
    for i, k in enumerate(mats):
        n = int(i % D) if D > 1 else 0
        ov = bool(i % 2)
        cm = P.cost_model_dict(D, 2, 2048, 1.6e7 * (1 + i % 3), 3.2e7, 4e11 / (1 + i % 5), 1e8 * (1 + i % 4),
                               1e-4 * (i % 3), 2e-4)
        cl = pp.ClusterSpec(D, cm["avg_bandwidth"], cm["compute_throughput"])
        mo = pp.ModelSpec(E, 1, 2, cm["input_bytes"], cm["expert_param_bytes"], cm["expert_grad_bytes"],
                          fnec_time=cm["fnec_time"], bnec_time=cm["bnec_time"])
        cfg = pp.PlannerConfig(n=n, alpha=0.5 if i % 3 else 0.1, overlap_aware=ov)
        res = pp.greedy_search_physical_many([k], cfg, cl, mo)[0]
        exp = P.greedy_search_physical(k, n, cfg.alpha, ov, cm)
        assert list(res.placement.selected) == list(exp["selected"]), i
        assert [sorted(x) for x in res.placement.excluded] == [sorted(x) for x in exp["excluded"]]
        assert res.placement.replica_mask().tolist() == exp["mask"].tolist()
        assert res.H.tolist() == exp["H"].tolist() and res.R.tolist() == exp["R"].tolist()
        assert float(res.best_cost).hex() == float(exp["best"]).hex()
        assert res.explored == exp["explored"]


def test_physical_planner_slot_rows_input():
    """Virtual-slot rows (rows = E, m per device) are summed per device on load and the
    emitted mask repeats each device row over its slots (the layout's slot mask)."""
    import torch

    from paper_2411_10003_b200 import _device

    D, m = 4, 4
    E = D * m
    rng = np.random.default_rng(5)
    slot = np.stack([rng.multinomial(512, rng.dirichlet(np.ones(E) * 0.3)) for _ in range(E)]).astype(np.int64)
    phys = slot.reshape(D, m, E).sum(axis=1)
    cm = P.cost_model_dict(D, 2, 2048, 1.6e7, 3.2e7, 4e11, 1e8)
    exp = P.greedy_search_physical(phys, 1, 0.5, True, cm)
    cl = pp.ClusterSpec(D, cm["avg_bandwidth"], cm["compute_throughput"])
    mo = pp.ModelSpec(E, 1, 2, cm["input_bytes"], cm["expert_param_bytes"], cm["expert_grad_bytes"])
    out = _device.PlanBuffers(1, E, torch.device("cuda", 0))
    _device.launch_plan(torch.from_numpy(slot).cuda().view(1, E, E), out, _device.cost_model(cl, mo),
                        _device.planner_cfg(pp.PlannerConfig(n=1, alpha=0.5, overlap_aware=True)),
                        physical_devices=D)
    torch.cuda.synchronize()
    assert out.mask[0].cpu().numpy().astype(bool).tolist() == np.repeat(exp["mask"], m, axis=0).tolist()
    assert out.H[0, :D].cpu().tolist() == exp["H"].tolist()
    with pytest.raises(pp.ValidationError):
        pp.greedy_search_physical(pp.LoadMatrix(phys[:, :E - 1]), pp.PlannerConfig(), cl, mo)


@pytest.mark.parametrize("D,m", [(2, 8), (4, 4), (8, 2), (4, 8)])
def test_physical_planner_slot_refinement_vs_oracle(D, m):
    """refine_slots (beyond the paper): the device's slot mask and H/R equal the oracle's
    refine_slots applied to the oracle's physical plan, and never raise the heaviest device."""
    import torch

    from paper_2411_10003_b200 import _device

    E = D * m
    rng = np.random.default_rng(900 + D * 10 + m)
    for i in range(25):
        p = rng.dirichlet(np.ones(E) * (0.15 + 0.2 * (i % 3)))
        slot = np.stack([rng.multinomial(256 * 2, p) for _ in range(E)]).astype(np.int64)
        phys = slot.reshape(D, m, E).sum(axis=1)
        n = i % D
        ov = bool(i % 2)
        cm = P.cost_model_dict(D, 2, 2048, 1.6e7, 3.2e7, 4e11 / (1 + i % 3), 1e8)
        exp = P.greedy_search_physical(phys, n, 0.5, ov, cm)
        S, H, R = P.refine_slots(slot, exp["mask"])
        assert H.max() <= exp["H"].max()
        cl = pp.ClusterSpec(D, cm["avg_bandwidth"], cm["compute_throughput"])
        mo = pp.ModelSpec(E, 1, 2, cm["input_bytes"], cm["expert_param_bytes"], cm["expert_grad_bytes"])
        out = _device.PlanBuffers(1, E, torch.device("cuda", 0))
        _device.launch_plan(torch.from_numpy(slot).cuda().view(1, E, E), out, _device.cost_model(cl, mo),
                            _device.planner_cfg(pp.PlannerConfig(n=n, alpha=0.5, overlap_aware=ov)),
                            physical_devices=D, refine_slots=True)
        torch.cuda.synchronize()
        assert out.mask[0].cpu().numpy().astype(bool).tolist() == S.tolist(), i
        assert out.H[0, :D].cpu().tolist() == H.tolist() and out.R[0, :D].cpu().tolist() == R.tolist()
        assert out.selected[0, : int(out.num_selected[0])].cpu().tolist() == list(exp["selected"])


# ---- extensions of pp_planner_cfg: replica bound and the device-side reuse gate ------------

def _launch(slot, D, m, cfg, physical, max_replicas=0, ctr=None):
    import torch

    from paper_2411_10003_b200 import _device

    E = D * m
    rows = slot.shape[0]
    cm = P.cost_model_dict(D if physical else E, 2, 2048, 1.6e7, 3.2e7, 4e11, 1e8)
    cl = pp.ClusterSpec(cm["num_devices"], cm["avg_bandwidth"], cm["compute_throughput"])
    mo = pp.ModelSpec(E, 1, 2, cm["input_bytes"], cm["expert_param_bytes"], cm["expert_grad_bytes"])
    out = _device.PlanBuffers(1, E, torch.device("cuda", 0))
    out.mask.fill_(7)
    c = _device.planner_cfg(cfg, max_replicas=max_replicas, slots_per_rank=1 if physical else m,
                            iter_counter=ctr)
    _device.launch_plan(torch.from_numpy(slot).cuda().view(1, rows, E), out, _device.cost_model(cl, mo, None if physical else E),
                        c, physical_devices=D if physical else 0)
    torch.cuda.synchronize()
    return out, cm


@pytest.mark.parametrize("physical", [False, True])
def test_planner_replica_bound_vs_oracle(physical):
    """max_replicas (weight slots a rank owns): the search stops before the first prefix that
    gives a rank more replicas; equal to the oracle restatement, and equal to the unbounded
    (reference) search whenever the bound does not bind."""
    D, m = 4, 4
    E = D * m
    rng = np.random.default_rng(4242 + physical)
    bound_hit = 0
    for i in range(30):
        p = rng.dirichlet(np.ones(E) * (0.1 + 0.1 * (i % 3)))
        slot = np.stack([rng.multinomial(512, p) for _ in range(E)]).astype(np.int64)
        cap = 1 + i % 4
        cfg = pp.PlannerConfig(n=1, alpha=0.2, overlap_aware=bool(i % 2))
        out, cm = _launch(slot, D, m, cfg, physical, max_replicas=cap)
        if physical:
            phys = slot.reshape(D, m, E).sum(axis=1)
            exp = P.greedy_search_physical(phys, 1, 0.2, bool(i % 2), cm, max_replicas=cap)
            free = P.greedy_search_physical(phys, 1, 0.2, bool(i % 2), cm)
            exp_mask = np.repeat(exp["mask"], m, axis=0)
            reps = P.replicas_per_rank(exp["mask"], 1, m)
        else:
            exp = P.greedy_search(slot, 1, 0.2, bool(i % 2), cm, max_replicas=cap, slots_per_rank=m)
            free = P.greedy_search(slot, 1, 0.2, bool(i % 2), cm)
            exp_mask = exp["mask"]
            reps = P.replicas_per_rank(exp["mask"], m, m)
        assert reps.max() <= cap
        got = out.selected[0, : int(out.num_selected[0])].cpu().tolist()
        assert got == list(exp["selected"]), i
        assert out.mask[0].cpu().numpy().astype(bool).tolist() == exp_mask.tolist()
        assert int(out.num_explored[0]) == exp["explored"]
        if exp["explored"] == free["explored"]:
            assert list(exp["selected"]) == list(free["selected"])
        else:
            bound_hit += 1
    assert bound_hit > 0  # the bound did bind in some cases


def test_planner_reuse_gate_device_counter():
    """iter_counter: the launch of iteration j searches only when (j+1) % F == 0, leaves every
    output untouched otherwise, and advances j by one either way (plan_for_iteration,
    planner.py:132-156, inside a replayable launch)."""
    import torch

    D, m = 4, 1
    E = D * m
    rng = np.random.default_rng(3)
    slot = np.stack([rng.multinomial(512, rng.dirichlet(np.ones(E) * 0.2)) for _ in range(E)]).astype(np.int64)
    ctr = torch.zeros(2, dtype=torch.int64, device="cuda")
    cfg = pp.PlannerConfig(n=1, alpha=0.2, reuse_interval=3)
    for j in range(7):
        out, cm = _launch(slot, D, m, cfg, False, ctr=ctr)
        searched = (j + 1) % 3 == 0
        assert int(ctr[0]) == j + 1 and int(ctr[1]) == 0
        if searched:
            exp = P.greedy_search(slot, 1, 0.2, False, cm)
            assert out.mask[0].cpu().numpy().astype(bool).tolist() == exp["mask"].tolist()
        else:
            assert (out.mask == 7).all()  # untouched
