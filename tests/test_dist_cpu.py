"""World-size-2 gloo tests (CPU) of the N > 1 host logic: the per-rank LoadMatrix
rows all-gathered into the virtual-slot matrix, redundant deterministic planning,
the expert-major receive layout every rank derives independently (a bijection
from (source rank, token, k) pairs onto the real rows of every destination
segment), and the max-over-ranks timing reduction used by bench.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, E, T, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path

        sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
        from oracle import moe_ref as M
        from oracle import planner_ref as P

        m = E // world
        d = 64
        x, _ = M.exact_inputs(T, d, E, seed=100 + rank)
        _, wg = M.exact_inputs(8, d, E, seed=7)  # replicated gate
        bias = torch.round(torch.log(torch.tensor([1.0 / (i + 1) ** 1.2 for i in range(E)])) * 4) / 4
        _, idx, _, _ = M.route(x, wg, bias, k)
        idx = idx.numpy()
        rows = torch.from_numpy(M.slot_histogram(idx, E, m))
        full = [torch.zeros_like(rows) for _ in range(world)]
        dist.all_gather(full, rows)
        counts = torch.cat(full).numpy()
        # redundant planning: every rank plans on the same matrix
        cm = P.cost_model_dict(E, k, 2 * d, 1e3, 1e3, 1e11, 1e6)
        plan = P.greedy_search(counts, 1, 0.5, False, cm)
        lay = M.layout(counts, plan["mask"], world, m)
        rk, cc = M.chunk_ranks(idx, E)
        dest, row = M.pair_positions(idx, rk, cc, lay, rank, m)
        # max-over-ranks timing as in bench.py
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        gathered = [None] * world
        dist.all_gather_object(gathered, dict(counts=counts, sel=plan["selected"], dest=dest, row=row,
                                              idx=idx, seg=lay["seg"], groups=lay["groups"], tmax=float(t.item())))
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("E,T,k", [(8, 1024, 2), (16, 2048, 1)])
def test_two_rank_layout_and_plan(E, T, k):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, E, T, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = res
    # identical LoadMatrix and plan on every rank (no plan broadcast needed)
    assert np.array_equal(a["counts"], b["counts"])
    assert a["sel"] == b["sel"]
    assert np.array_equal(a["seg"], b["seg"]) and a["groups"] == b["groups"]
    assert a["tmax"] == b["tmax"] == 2.0
    # bijection onto the real rows of every (destination rank, expert) segment
    for r in range(world):
        for g in a["groups"][r]:
            e = g["expert"]
            hits = []
            for src in res:
                sel = (src["dest"] == r) & (src["idx"] == e)
                hits.extend(src["row"][sel].tolist())
            assert sorted(hits) == list(range(g["row_off"], g["row_off"] + g["rows"])), (r, e)
            assert g["rows_pad"] % 128 == 0 and g["rows_pad"] - g["rows"] < 128
    # total rows computed == total routed pairs (conservation, reference core.py:255-275)
    assert sum(g["rows"] for gl in a["groups"] for g in gl) == world * T * k


def test_plan_schedule_matches_reference_reuse_rule():
    """The layer launches the planner after iteration i iff (i+1) % F == 0 and
    uses it from i+1 on; that must reproduce plan_for_iteration's anchor rule."""
    from paper_2411_10003_b200.planner import plan_source_iteration

    for F in range(1, 5):
        current = None
        for j in range(24):
            # layer: plan computed after iteration j-1 when j % F == 0 (and j > 0)
            if j > 0 and (j - 1 + 1) % F == 0:
                current = j - 1
            anchor = (j // F) * F
            expect = None if anchor == 0 else anchor - 1
            assert current == expect == plan_source_iteration(j, F), (F, j)


def _product_worker(rank, world, port, E, q):
    """Product host logic of the N > 1 step at world size 2: each rank derives, independently,
    its replica set, the Trans it pulls / pushes and the Agg it sums (core.replica_transfers,
    the functions MoELayer uses for the copy-engine path and replica_traffic)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path

        sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
        from oracle import planner_ref as P
        from paper_2411_10003_b200 import core, memory

        m = E // world
        rng = np.random.default_rng(11)  # the same LoadMatrix on every rank (all-gathered in the layer)
        counts = np.stack([rng.multinomial(512, rng.dirichlet(np.ones(E) * 0.3)) for _ in range(E)]).astype(np.int64)
        cm = P.cost_model_dict(E, 2, 2048, 1e3, 1e3, 1e11, 1e6)  # cheap Trans: the plan replicates
        mask = P.greedy_search(counts, 1, 0.5, False, cm)["mask"]
        xf = core.replica_transfers(mask, world, m, rank)
        cap = memory.rows_capacity(4096, 2, E, world, capacity_factor=2.0)
        gathered = [None] * world
        dist.all_gather_object(gathered, dict(xf=xf, cap=cap, reps=core.replica_sets(mask, world, m)))
        if rank == 0:
            q.put((gathered, mask))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("E", [8, 16])
def test_two_rank_replica_transfers_product(E):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_product_worker, args=(r, world, port, E, q)) for r in range(world)]
    for p in procs:
        p.start()
    res, mask = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = E // world
    assert res[0]["reps"] == res[1]["reps"] and res[0]["cap"] == res[1]["cap"]
    assert any(res[r]["xf"]["replicas"] for r in range(world))  # the plan did replicate
    for r in range(world):
        xf = res[r]["xf"]
        # replica slots are dense, m .. m + #replicas - 1, ascending expert id
        assert [s for *_, s in xf["trans_in"]] == list(range(m, m + len(xf["replicas"])))
        assert [e for e, *_ in xf["trans_in"]] == sorted(xf["replicas"])
        for e, home, j, slot in xf["trans_in"]:
            # the home pushes exactly this (expert, home slot) into this rank's slot ...
            assert (e, j, r, slot) in res[home]["xf"]["trans_out"]
            # ... and sums this rank's grads of that slot back into home slot j (Agg)
            assert (r, slot) in res[home]["xf"]["agg_in"][j]
        for j, srcs in xf["agg_in"].items():
            assert [s[0] for s in srcs] == sorted(s[0] for s in srcs)  # rank order: deterministic sum
            assert all(r * m + j in res[s[0]]["xf"]["replicas"] for s in srcs)
    # the mask itself: a rank holds e iff one of its slots keeps e's pairs (core.py:267-274)
    for r in range(world):
        held = mask[r * m:(r + 1) * m].any(axis=0)
        assert res[0]["reps"][r] == [e for e in range(E) if e // m != r and held[e]]
