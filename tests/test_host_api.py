"""Host-side API mirror vs the reference goldens (CPU only): value types and
their validation, the scalar cost model, the Algorithm-2 timeline model, metrics."""

import json
import math
from pathlib import Path

import numpy as np
import pytest

import paper_2411_10003_b200 as pp
from paper_2411_10003_b200 import perf_model as pm
from paper_2411_10003_b200 import planner as pl
from paper_2411_10003_b200 import scheduler as sc

G = Path(__file__).resolve().parent / "golden"


class TestValidation:
    def test_cluster(self):
        for args in ((1, 1e9, 1e6), (4, 0, 1e6), (4, 1e9, -1)):
            with pytest.raises(pp.ValidationError):
                pp.ClusterSpec(*args)

    def test_model(self):
        for args, kw in (((4, 1, 5, 1, 1, 1), {}), ((4, 0, 1, 1, 1, 1), {}), ((4, 1, 1, 0, 1, 1), {}),
                         ((4, 1, 1, 1, 1, 1), {"fnec_time": -0.1})):
            with pytest.raises(pp.ValidationError):
                pp.ModelSpec(*args, **kw)

    def test_load_matrix(self):
        with pytest.raises(pp.ValidationError):
            pp.LoadMatrix([[1, -1], [0, 2]])
        with pytest.raises(pp.ValidationError):
            pp.LoadMatrix([[1, 2], [0, 2]])
        with pytest.raises(pp.ValidationError):
            pp.LoadMatrix([1, 2, 3])
        lm = pp.LoadMatrix([[3, 0, 0], [2, 1, 0], [0, 1, 2]])
        assert lm.total() == 9 and lm.expert_totals().tolist() == [5, 2, 2]
        assert not lm.counts.flags.writeable
        with pytest.raises(AttributeError):
            lm.counts = None

    def test_placement(self):
        with pytest.raises(pp.ValidationError):
            pp.ExpertPlacement(2, 3)
        with pytest.raises(pp.ValidationError):
            pp.ExpertPlacement(3, 3, (0, 0), (frozenset({1}), frozenset({2})))
        with pytest.raises(pp.ValidationError):
            pp.ExpertPlacement(3, 3, (0,), (frozenset({0}),))  # home excluded
        with pytest.raises(pp.ValidationError):
            pp.ExpertPlacement(3, 3, (0, 1), (frozenset({1}), frozenset()))
        p = pp.ExpertPlacement(3, 3, (0,), (frozenset({2}),))
        assert p.replicas(0) == frozenset({0, 1}) and p.replicas(1) == frozenset({1}) and p.n == 1

    def test_replica_mask_golden_and_from_mask(self):
        for c in json.loads((G / "derive_cases.json").read_text()):
            D, E = np.array(c["counts"]).shape
            p = pp.ExpertPlacement(D, E, tuple(c["selected"]), tuple(frozenset(x) for x in c["excluded"]))
            assert p.replica_mask().astype(int).tolist() == c["mask"]
            if D == E:
                assert pp.ExpertPlacement.from_mask(p.selected, p.replica_mask()) == p


def test_cost_model_golden():
    for c in json.loads((G / "cost_cases.json").read_text()):
        cl = pp.ClusterSpec(*c["cluster"])
        mo = pp.ModelSpec(*c["model"][:6], fnec_time=c["model"][6], bnec_time=c["model"][7])
        loads = pp.DeviceLoads(np.array(c["H"]), np.array(c["R"]))
        got = pm.layer_cost_unscheduled(loads, c["s"], c["n"], cl, mo)
        for k, v in c["cost"].items():
            assert float(getattr(got, k)).hex() == v, k
    cl = pp.ClusterSpec(3, 1e9, 1000.0)
    mo = pp.ModelSpec(3, 1, 1, 1e6, 1e5, 1e5)
    with pytest.raises(pp.ValidationError):
        pm.t_trans(0, 3, cl, mo)
    with pytest.raises(pp.ValidationError):
        pm.t_agg(4, 0, cl, mo)


def test_timeline_golden():
    for c in json.loads((G / "timeline_cases.json").read_text()):
        mo = pp.ModelSpec(4, c["L"], 1, 1.0, 1.0, 1.0, fnec_time=c["fnec"], bnec_time=c["bnec"])
        costs = [pm.LayerCost(a, fe, be, tr, ag, 0.0, 0.0, 0.0, 0.0) for a, fe, be, tr, ag in c["costs"]]
        tl = pp.build_iteration_timeline(costs, c["plan_time"], mo, iteration=c["iteration"])
        ts = pp.build_serial_timeline(costs, c["plan_time"], mo, iteration=c["iteration"])
        assert tl.to_json_obj() == c["overlapped"]
        assert ts.to_json_obj() == c["serial"]
        assert tl.phase_totals() == c["phase"]
        assert tl.exposed_comm_seconds() == c["exposed_comm"]


def test_partitions():
    assert pp.partition_trans(3.0, 1.0, 1.0) == (2.0, 1.0)
    assert pp.partition_trans(0.5, 1.0, 1.0) == (0.0, 0.5)
    assert pp.partition_agg(3.0, 1.0, 1.0) == (1.0, 2.0)
    with pytest.raises(pp.ValidationError):
        pp.partition_trans(-1.0, 0.0, 0.0)
    b1, b2 = sc.trans_byte_split(1000, 3.0, 1.0, 1.0)
    assert (b1, b2) == (667, 333)


def test_timeline_errors():
    mo = pp.ModelSpec(4, 2, 1, 1.0, 1.0, 1.0)
    c = pm.LayerCost(0, 0, 0, 0, 0, 0, 0, 0, 0)
    with pytest.raises(pp.ValidationError):
        pp.build_iteration_timeline([c], 0.0, mo)
    with pytest.raises(pp.ValidationError):
        pp.build_iteration_timeline([c, c], -1.0, mo)


def test_metrics_golden():
    for c in json.loads((G / "metric_cases.json").read_text()):
        assert pp.balance_degree(c["a"]) == c["sigma_a"]
        a = pp.DeviceLoads(np.array(c["a"]), np.zeros(len(c["a"]), dtype=int))
        b = pp.DeviceLoads(np.array(c["b"]), np.zeros(len(c["b"]), dtype=int))
        assert repr(pp.rb_ratio(a, b)) == c["rb"]
    with pytest.raises(pp.ValidationError):
        pp.balance_degree([])


def test_planner_host_helpers():
    assert pp.is_balanced([5, 2, 2], 9, 3, 0.5) is False
    assert pp.is_balanced([3, 3, 3], 9, 3, 1e-9) is True
    assert pp.is_balanced([4, 3, 2], 9, 3, 1.0) is True
    with pytest.raises(pp.ValidationError):
        pp.is_balanced([], 9, 3, 1.0)
    fig8 = pp.LoadMatrix([[3, 0, 0], [2, 1, 0], [0, 1, 2]])
    assert pl.bottom_devices(fig8, 0, 1) == frozenset({2})
    assert pl.bottom_devices(pp.LoadMatrix([[0, 3], [0, 3]]), 0, 1) == frozenset({1})
    assert pl.bottom_devices(pp.LoadMatrix([[2, 1, 0], [1, 2, 0], [1, 0, 2]]), 2, 1) == frozenset({0})
    for kw in ({"n": -1}, {"alpha": 0}, {"reuse_interval": 0}):
        with pytest.raises(pp.ValidationError):
            pp.PlannerConfig(**kw)
    with pytest.raises(pp.ValidationError):
        pp.plan_for_iteration([], -1, pp.PlannerConfig(), pp.ClusterSpec(3, 1e9, 1e3), pp.ModelSpec(3, 1, 1, 1, 1, 1))
    # iteration 0 (and the whole first interval) never touches the device
    cfg = pp.PlannerConfig(reuse_interval=3)
    cl, mo = pp.ClusterSpec(3, 1e9, 1e3), pp.ModelSpec(3, 1, 1, 1, 1, 1)
    for j in range(3):
        assert pp.plan_for_iteration([], j, cfg, cl, mo) == pp.ExpertPlacement.empty(3, 3)


def test_greedy_validation_happens_on_host():
    """Precondition errors are raised with the reference's types before any device work."""
    cl = pp.ClusterSpec(3, 1e9, 1e3)
    mo = pp.ModelSpec(3, 1, 1, 1e6, 1e5, 1e5)
    with pytest.raises(pp.ValidationError):
        pp.greedy_search(pp.LoadMatrix([[1, 2], [2, 1], [0, 3]]), pp.PlannerConfig(), cl, mo)
    with pytest.raises(pp.DimensionMismatchError):
        pp.greedy_search(pp.LoadMatrix([[1, 2], [2, 1]]), pp.PlannerConfig(), cl, mo)
    with pytest.raises(pp.ValidationError):
        pp.greedy_search(pp.LoadMatrix([[3, 0, 0], [2, 1, 0], [0, 1, 2]]), pp.PlannerConfig(n=3), cl, mo)
    with pytest.raises(pp.DimensionMismatchError):
        pp.derive_loads(pp.LoadMatrix([[1, 2], [2, 1]]), pp.ExpertPlacement.empty(3, 3))


def test_accepts_reference_objects():
    from conftest import import_reference

    ref = import_reference()
    lm = ref.LoadMatrix([[3, 0, 0], [2, 1, 0], [0, 1, 2]])
    from paper_2411_10003_b200.core import as_counts

    assert as_counts(lm).tolist() == [[3, 0, 0], [2, 1, 0], [0, 1, 2]]
    rc = ref.ClusterSpec(3, 1e9, 1000.0)
    rm = ref.ModelSpec(3, 1, 1, 1e6, 1e5, 1e5)
    assert pm.layer_cost_unscheduled(ref.DeviceLoads([5, 2, 2], [2, 1, 0]), 0, 0, rc, rm).total_unscheduled == \
        ref.layer_cost_unscheduled(ref.DeviceLoads([5, 2, 2], [2, 1, 0]), 0, 0, rc, rm).total_unscheduled


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        pp.greedy_search(pp.LoadMatrix([[3, 0, 0], [2, 1, 0], [0, 1, 2]]), pp.PlannerConfig(),
                         pp.ClusterSpec(3, 1e9, 1e3), pp.ModelSpec(3, 1, 1, 1e6, 1e5, 1e5))
    with pytest.raises(RuntimeError):
        pp.MoELayer(256, 512, 16, 2, tokens=2048)


def test_trace_jsonl_matches_reference_format(tmp_path, rng):
    from paper_2411_10003_b200 import trace as tr

    recs = []
    for it in range(3):
        for layer in range(2):
            p = rng.dirichlet(np.ones(8))
            counts = np.stack([rng.multinomial(64, p) for _ in range(8)])
            recs.append(tr.TraceRecord(it, layer, pp.LoadMatrix(counts)))
    ours = tmp_path / "ours.jsonl"
    tr.write_trace(recs, ours)
    back = tr.read_trace(ours)
    assert [(r.iteration, r.layer, r.load) for r in back] == [(r.iteration, r.layer, r.load) for r in recs]
    bad = tmp_path / "bad.jsonl"
    bad.write_text('{"iter": 0, "layer": 0}\n')
    with pytest.raises(tr.TraceFormatError):
        tr.read_trace(bad)
    from conftest import import_reference

    ref = import_reference()
    from moebal import workload

    theirs = tmp_path / "theirs.jsonl"
    workload.write_trace([workload.TraceRecord(r.iteration, r.layer, ref.LoadMatrix(r.load.counts)) for r in recs],
                         theirs)
    assert ours.read_bytes() == theirs.read_bytes()  # byte-identical JSONL
    parsed = workload.read_trace(ours)  # the reference replays our traces
    assert [r.load.counts.tolist() for r in parsed] == [r.load.counts.tolist() for r in recs]


def test_cost_model_calibration_fit():
    """calibrate.fit recovers B and t from phase timings generated by the model itself and
    reports ~0 held-out error; measured_costs sums the four A2A spans and the GEMM phases."""
    from paper_2411_10003_b200 import calibrate

    t_true, B_true, ib = 5e7, 4e11, 2048.0
    rng = np.random.default_rng(0)
    samples = []
    for _ in range(8):
        H = rng.integers(20000, 40000, size=4)
        R = rng.integers(5000, 15000, size=4)
        fec = H.max() / t_true
        a2a = R.max() * ib / B_true
        samples.append((H, R, {"a2a_total": 4 * a2a, "fec": fec, "bec": 2 * fec, "layer": 4 * a2a + 3 * fec}))
    fit = calibrate.fit(samples, input_bytes=ib)
    assert abs(fit["compute_throughput"] / t_true - 1) < 1e-9
    assert abs(fit["avg_bandwidth"] / B_true - 1) < 1e-9
    assert fit["mean_abs_rel_error"] < 1e-9 and fit["train_iters"] == 4 and fit["test_iters"] == 4
    step = {"route_layout": 0.1, "barrier1": 0.3, "fwd_gemms": 1.0, "combine": 1.2, "bwd_begin": 1.25,
            "combine_bwd": 1.3, "gate_dw": 1.35, "barrier3": 1.4, "bwd_gemms": 3.0, "dispatch_bwd": 3.2}
    m = calibrate.measured_costs(step)
    assert abs(m["fec"] - 0.7e-3) < 1e-12 and abs(m["bec"] - 1.6e-3) < 1e-12
    # A2A spans: dispatch, combine, combine_bwd (without the gate dW / dX), dispatch bwd
    assert abs(m["a2a_total"] - (0.2 + 0.2 + (0.05 + 0.05) + 0.2) * 1e-3) < 1e-12


def test_physical_placement_value_type():
    """PhysicalPlacement (E = m*D, homes e // m): validation, replica sets, the [D][E] mask,
    the [E][E] slot mask the layout consumes, and equality with ExpertPlacement at m = 1."""
    p = pp.PhysicalPlacement(2, 4, (1,), (frozenset(),))
    assert p.home(3) == 1 and p.replicas(1) == frozenset({0, 1}) and p.replicas(2) == frozenset({1})
    assert p.replica_mask().astype(int).tolist() == [[1, 1, 0, 0], [0, 1, 1, 1]]
    assert p.slot_mask().astype(int).tolist() == [[1, 1, 0, 0], [1, 1, 0, 0], [0, 1, 1, 1], [0, 1, 1, 1]]
    with pytest.raises(pp.ValidationError):
        pp.PhysicalPlacement(3, 4)  # E not a multiple of D
    with pytest.raises(pp.ValidationError):
        pp.PhysicalPlacement(2, 4, (1,), (frozenset({0}),))  # home of expert 1 is device 0
    q = pp.PhysicalPlacement(3, 3, (0,), (frozenset({2}),))
    r = pp.ExpertPlacement(3, 3, (0,), (frozenset({2}),))
    assert q.replica_mask().tolist() == r.replica_mask().tolist()


def test_bench_cli_parses():
    """bench.py's argument parser (the driver's entry point) builds and prints its help."""
    import subprocess
    import sys

    root = Path(__file__).resolve().parent.parent
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--help"], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "--gpus" in r.stdout and "--impl" in r.stdout


def test_bench_popularity_drift_is_the_reference_generator():
    """bench.PopularityDrift (the cfg4 gate-bias drift) reproduces the reference trace
    generator's per-iteration popularity (workload.py:113-136) bit for bit: the reference
    draws each iteration's LoadMatrix from a generator keyed to the popularity vector's bytes
    (_matrix_rng), so equal counts <=> identical p."""
    from conftest import import_reference

    moebal = import_reference()
    from moebal import workload as W

    import bench

    E, D, inputs, k = 16, 4, 4096, 2
    ref = W.generate_trace(W.GeneratorConfig(num_devices=D, num_experts=E, inputs_per_iteration=inputs,
                                             top_k=k, skew=1.2, drift=0.05, seed=3), iterations=6, layers=1)
    drift = bench.PopularityDrift(E, skew=1.2, drift=0.05, seed=3)
    per_device = inputs // D * k
    for rec in ref:
        p = drift.step()
        draw = W._matrix_rng(3, 0, p)
        counts = np.stack([draw.multinomial(per_device, p) for _ in range(D)])
        assert np.array_equal(counts, np.asarray(rec.load.counts)), rec.iteration


def test_exposure_summary_on_a_handmade_timeline():
    """exposure_summary applies the reference's exposure metric (scheduler.py:134-169): the
    part of a Trans / Agg op not covered by compute-lane ops."""
    from paper_2411_10003_b200.scheduler import IterationTimeline, Lane, OpKind, ScheduledOp
    from paper_2411_10003_b200.stack import exposure_summary

    ops = (ScheduledOp(OpKind.FEC, 0, 0, Lane.COMPUTE, 0.0, 1.0),
           ScheduledOp(OpKind.SUB_TRANS1, 0, 0, Lane.NETWORK, 0.5, 1.0),   # 0.5 hidden, 0.5 exposed
           ScheduledOp(OpKind.BEC, 0, 0, Lane.COMPUTE, 2.0, 2.0),
           ScheduledOp(OpKind.SUB_AGG2, 0, 0, Lane.NETWORK, 3.5, 1.0))      # 0.5 hidden, 0.5 exposed
    ex = exposure_summary(IterationTimeline(0, ops), blocks=1)
    assert abs(ex["exposed_trans_ms"] - 500.0) < 1e-9 and abs(ex["exposed_agg_ms"] - 500.0) < 1e-9
    assert abs(ex["makespan_ms"] - 4500.0) < 1e-9
    assert abs(ex["exposed_replica_comm_frac"] - 1.0 / 4.5) < 1e-12


def test_planner_cfg_struct_matches_header():
    """pp_planner_cfg: the ctypes layout (size and offsets) the header declares."""
    import ctypes

    from paper_2411_10003_b200 import _lib

    c = _lib.PlannerCfg
    assert ctypes.sizeof(c) == 40
    assert c.reuse_interval.offset == 16 and c.max_replicas.offset == 20 and c.iter_counter.offset == 32


def test_trans_copy_split():
    """a9 on the copy engine: the SubTrans2 byte count cuts the Trans copy list so the
    first part moves exactly that many bytes (16-byte granularity) and both parts together
    cover every source byte once, in order."""
    from paper_2411_10003_b200.layer import MoELayer
    items = [(10_000, 90_000, 4096), (20_000, 80_000, 1000), (30_000, 70_000, 8192)]
    total = sum(n for _, _, n in items)
    for first_bytes in (0, 16, 4000, 4096, 4100, 5096, 9000, total, total + 64):
        first, rest = MoELayer._split_copies(items, first_bytes)
        moved = sum(n for _, _, n in first)
        assert moved <= first_bytes and first_bytes - moved < 16 * len(items) + 16 or moved == total
        cover = {}
        for dst, src, n in first + rest:
            assert dst - src == [d - s for d, s, m in items if s <= src < s + m][0]
            for off in range(src, src + n, 8):
                cover[off] = cover.get(off, 0) + 1
        assert sum(cover.values()) * 8 == total and set(cover.values()) == {1}
    bw = 1e9  # 13.3 us of Trans against a 5 us FNEC window
    _, b2 = sc.trans_byte_split(total, total / bw, 1e-3, 5e-6)
    assert b2 == round(5e-6 * bw)
    _, b2 = sc.trans_byte_split(total, total / 600e9, 1e-3, 5e-6)  # all of it fits the window
    assert b2 == total


def test_calibration_fits_total_expert_compute():
    """t is fitted to FEC + BEC (= 3 maxH / t in the model): with a measured BEC/FEC ratio of 2.4
    instead of the model's 2, the layer prediction stays exact and the ratio is reported."""
    from paper_2411_10003_b200 import calibrate

    t_true, B_true, ib = 5e7, 4e11, 2048.0
    rng = np.random.default_rng(1)
    samples = []
    for _ in range(8):
        H = rng.integers(20000, 40000, size=4)
        R = rng.integers(5000, 15000, size=4)
        fec = H.max() / t_true
        a2a = R.max() * ib / B_true
        samples.append((H, R, {"a2a_total": 4 * a2a, "fec": fec, "bec": 2.4 * fec, "layer": 4 * a2a + 3.4 * fec}))
    fit = calibrate.fit(samples, input_bytes=ib)
    assert abs(fit["compute_throughput"] / (t_true * 3 / 3.4) - 1) < 1e-9
    assert fit["mean_abs_rel_error"] < 1e-9
    assert abs(fit["bec_over_fec_measured"] - 2.4) < 1e-9


def test_bench_nvlink_counter_delta():
    """The NVLink counter reports the first NVML field set whose counters moved over the timed
    region (drivers maintain one or the other), and zero when none did."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import bench

    a = {"THROUGHPUT_DATA": (10, 10), "COUNT_BYTES": (5, 5)}
    assert bench.NvLinkCounter.delta(a, {"THROUGHPUT_DATA": (10, 10), "COUNT_BYTES": (105, 55)}) == \
        ("COUNT_BYTES", 100, 50)
    assert bench.NvLinkCounter.delta(a, {"THROUGHPUT_DATA": (2058, 10), "COUNT_BYTES": (105, 55)}) == \
        ("THROUGHPUT_DATA", 2048, 0)
    assert bench.NvLinkCounter.delta(a, a) == ("THROUGHPUT_DATA", 0, 0)
