"""ORACLE (test infrastructure only) -- CPU restatement of the reference planner path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module, and only as the checker or
the timed CPU baseline.  The product (``paper_2411_10003_b200``) never calls it.

Parity status: PINNED.  Every function below restates a reference function
(``/root/reference/pkg/src/moebal``, cited per function) and is checked in
``tests/test_oracle_golden.py`` against golden vectors produced by running the
reference itself (``tests/golden/gen_golden.py``): FIG8 cases, the SURVEY
appendix-B step traces, fuzzed instances and generator traces.

Pure Python + numpy, integer arithmetic exact, fp64 in the reference's
association order.
"""

from __future__ import annotations

import numpy as np


def replica_mask(D: int, E: int, selected, excluded) -> np.ndarray:
    """reference core.py:213-222 -- diagonal homes, selected columns minus excluded."""
    mask = np.zeros((D, E), dtype=bool)
    for e in range(E):
        mask[e, e] = True
    for e, ex in zip(selected, excluded):
        mask[:, e] = True
        for dv in ex:
            mask[dv, e] = False
    return mask


def derive_loads(counts: np.ndarray, mask: np.ndarray):
    """reference core.py:255-275: a (d, e) batch stays on d when d holds e,
    otherwise it is computed (H) and received (R) at e's home, device e."""
    counts = np.asarray(counts, dtype=np.int64)
    D, E = counts.shape
    kept = np.where(mask, counts, 0).sum(axis=1)
    sent = np.where(mask, 0, counts).sum(axis=0)
    H = kept.astype(np.int64)
    H[:E] += sent
    R = np.zeros(D, dtype=np.int64)
    R[:E] = sent
    return H, R


def derive_loads_cellwise(counts: np.ndarray, mask: np.ndarray):
    """Cell-by-cell restatement of the same rule (independent cross-check, in
    the style of the reference's routed_by_hand, test_core.py:19-36)."""
    counts = np.asarray(counts, dtype=np.int64)
    D, E = counts.shape
    H = np.zeros(D, dtype=np.int64)
    R = np.zeros(D, dtype=np.int64)
    for d in range(D):
        for e in range(E):
            c = int(counts[d, e])
            if mask[d, e]:
                H[d] += c
            else:
                H[e] += c
                R[e] += c
    return H, R


def cost_terms(rmax: int, hmax: int, s: int, n: int, cm: dict) -> dict:
    """reference perf_model.py:36-107 in its evaluation order."""
    D = cm["num_devices"]
    a2a = rmax * cm["input_bytes"] / cm["avg_bandwidth"]
    fec = hmax / cm["compute_throughput"]
    bec = 2.0 * fec
    trans = s * (D - n) * cm["expert_param_bytes"] / (D * cm["avg_bandwidth"])
    agg = s * (D - n) * cm["expert_grad_bytes"] / (D * cm["avg_bandwidth"])
    ptrans = max(0.0, trans - fec - cm["fnec_time"])
    pagg = max(0.0, agg - bec - cm["bnec_time"])
    return {
        "a2a": a2a, "fec": fec, "bec": bec, "trans": trans, "agg": agg,
        "ptrans": ptrans, "pagg": pagg,
        "unscheduled": 4.0 * a2a + fec + bec + trans + agg,
        "scheduled": 4.0 * a2a + fec + bec + ptrans + pagg,
    }


def objective(H, R, s: int, n: int, cm: dict, overlap_aware: bool) -> float:
    """reference planner.py:98-102."""
    t = cost_terms(int(np.max(R)), int(np.max(H)), s, n, cm)
    return t["scheduled"] if overlap_aware else t["unscheduled"]


def bottom_devices(counts: np.ndarray, expert: int, n: int) -> frozenset:
    """reference planner.py:71-77 (home excluded, key (count, index), original matrix)."""
    col = counts[:, expert]
    cands = sorted((int(col[d]), d) for d in range(counts.shape[0]) if d != expert)
    return frozenset(d for _, d in cands[:n])


def is_balanced(H, total_inputs: int, E: int, alpha: float) -> bool:
    """reference planner.py:63-68."""
    H = np.asarray(H)
    return float(H.max() - H.min()) < alpha * total_inputs / E


def replicas_per_rank(mask: np.ndarray, rows_per_rank: int, homes_per_rank: int) -> np.ndarray:
    """Replica experts each rank holds under a [rows][E] mask (rank of row v = v // rows_per_rank,
    home rank of expert e = e // homes_per_rank) -- the weight slots the plan needs."""
    rows, E = mask.shape
    ranks = rows // rows_per_rank
    held = mask.reshape(ranks, rows_per_rank, E).any(axis=1)
    home = np.arange(E) // homes_per_rank
    return np.array([int(sum(held[r, e] and home[e] != r for e in range(E))) for r in range(ranks)])


def greedy_search(counts, n: int, alpha: float, overlap_aware: bool, cm: dict,
                  max_replicas: int = 0, slots_per_rank: int = 1) -> dict:
    """reference planner.py:80-129 (Algorithm 1).  Returns the plan plus the
    objective of the returned plan and the number of explored steps.

    max_replicas > 0 (extension of the device kernel, pp_planner_cfg; not in the
    reference): the search stops before the first prefix whose mask gives a rank
    (slots_per_rank rows each) more than max_replicas replica experts."""
    counts = np.asarray(counts, dtype=np.int64)
    D, E = counts.shape
    assert D == E, "greedy search requires num_experts == num_devices"
    total_inputs = int(counts.sum()) // cm["top_k"]
    H, R = derive_loads(counts, replica_mask(D, E, (), ()))
    best = objective(H, R, 0, 0, cm, overlap_aware)
    selected, bottoms, used = [], [], set()
    cnt = 0
    while not is_balanced(H, total_inputs, E, alpha):
        i = int(np.argmax(H))
        if i in used:
            break
        used.add(i)
        selected.append(i)
        bottoms.append(bottom_devices(counts, i, n))
        if max_replicas > 0 and replicas_per_rank(replica_mask(D, E, selected, bottoms), slots_per_rank,
                                                  slots_per_rank).max() > max_replicas:
            selected.pop()
            bottoms.pop()
            break
        H, R = derive_loads(counts, replica_mask(D, E, selected, bottoms))
        changed = objective(H, R, len(selected), n, cm, overlap_aware)
        if changed < best:
            best = changed
            cnt = len(selected)
    sel = tuple(selected[:cnt])
    exc = tuple(bottoms[:cnt])
    mask = replica_mask(D, E, sel, exc)
    Hf, Rf = derive_loads(counts, mask)
    return {"selected": sel, "excluded": exc, "best": best, "explored": len(selected),
            "mask": mask, "H": Hf, "R": Rf}


# ---- physically-faithful E > D planner (parity pinned at m = 1) ----
#
# The reference search needs E == D (planner.py:88-90).  With m = E / D experts per
# device, expert e's home is device e // m and the LoadMatrix rows are physical
# devices.  Generalisation (reduces to greedy_search exactly when m == 1):
#   * derive_loads: a (d, e) batch stays on d when d holds e, otherwise it is
#     computed and received at home(e)                      (core.py:255-275 with homes e // m)
#   * is_balanced threshold alpha * total_inputs / D         (planner.py:63-68; E == D there)
#   * i = first argmax(H) is a DEVICE; the expert to replicate is the unused expert
#     homed on i that currently sends it the most rows (ties -> lower id); stop when
#     i has no unused expert                                  (planner.py:115-117)
#   * excluded = n non-home devices with the fewest rows of that expert, key
#     (count, index), on the original matrix                 (planner.py:71-77)
#   * the cost model is the reference's with num_devices = D (perf_model.py:36-107)


def replica_mask_physical(D: int, E: int, selected, excluded) -> np.ndarray:
    m = E // D
    mask = np.zeros((D, E), dtype=bool)
    for e in range(E):
        mask[e // m, e] = True
    for e, ex in zip(selected, excluded):
        mask[:, e] = True
        for dv in ex:
            mask[dv, e] = False
    return mask


def derive_loads_physical(counts: np.ndarray, mask: np.ndarray):
    counts = np.asarray(counts, dtype=np.int64)
    D, E = counts.shape
    m = E // D
    H = np.zeros(D, dtype=np.int64)
    R = np.zeros(D, dtype=np.int64)
    for d in range(D):
        for e in range(E):
            c = int(counts[d, e])
            if mask[d, e]:
                H[d] += c
            else:
                H[e // m] += c
                R[e // m] += c
    return H, R


def bottom_devices_physical(counts: np.ndarray, expert: int, n: int, home: int) -> frozenset:
    col = counts[:, expert]
    cands = sorted((int(col[d]), d) for d in range(counts.shape[0]) if d != home)
    return frozenset(d for _, d in cands[:n])


def greedy_search_physical(counts, n: int, alpha: float, overlap_aware: bool, cm: dict,
                           max_replicas: int = 0) -> dict:
    counts = np.asarray(counts, dtype=np.int64)
    D, E = counts.shape
    assert E % D == 0 and cm["num_devices"] == D
    m = E // D
    total_inputs = int(counts.sum()) // cm["top_k"]
    mask = replica_mask_physical(D, E, (), ())
    H, R = derive_loads_physical(counts, mask)
    best = objective(H, R, 0, 0, cm, overlap_aware)
    selected, bottoms, used = [], [], set()
    cnt = 0
    while not (float(H.max() - H.min()) < alpha * total_inputs / D):
        i = int(np.argmax(H))
        cand = None
        for e in range(i * m, (i + 1) * m):
            if e in used:
                continue
            sent = int(sum(int(counts[d, e]) for d in range(D) if not mask[d, e]))
            if cand is None or sent > cand[0]:
                cand = (sent, e)
        if cand is None:
            break
        e = cand[1]
        used.add(e)
        selected.append(e)
        bottoms.append(bottom_devices_physical(counts, e, n, i))
        mask = replica_mask_physical(D, E, selected, bottoms)
        if max_replicas > 0 and replicas_per_rank(mask, 1, m).max() > max_replicas:
            selected.pop()
            bottoms.pop()
            break
        H, R = derive_loads_physical(counts, mask)
        changed = objective(H, R, len(selected), n, cm, overlap_aware)
        if changed < best:
            best = changed
            cnt = len(selected)
    sel = tuple(selected[:cnt])
    exc = tuple(bottoms[:cnt])
    mask = replica_mask_physical(D, E, sel, exc)
    Hf, Rf = derive_loads_physical(counts, mask)
    return {"selected": sel, "excluded": exc, "best": best, "explored": len(selected),
            "mask": mask, "H": Hf, "R": Rf}


def refine_slots(slot_counts: np.ndarray, pmask: np.ndarray):
    """Opt-in slot-level refinement of a physical plan (our extension, not in the paper):
    a replica holder may keep sending some of its m token slots to the expert's home.
    Repeatedly take the heaviest device h (first argmax of H); among its slots v that
    compute a non-home expert e locally with C[v][e] > 0, un-route the one minimising
    max(H[h] - C[v][e], H[home(e)] + C[v][e]) (ties: lower v, then lower e) if that is
    below H[h]; stop when h cannot improve.  Returns the [E][E] slot mask and H, R."""
    C = np.asarray(slot_counts, dtype=np.int64)
    E = C.shape[0]
    D = pmask.shape[0]
    m = E // D
    S = np.repeat(np.asarray(pmask, dtype=bool), m, axis=0)

    def loads():
        H = np.zeros(D, dtype=np.int64)
        R = np.zeros(D, dtype=np.int64)
        for v in range(E):
            for e in range(E):
                c = int(C[v, e])
                if S[v, e]:
                    H[v // m] += c
                else:
                    H[e // m] += c
                    R[e // m] += c
        return H, R

    H, R = loads()
    for _ in range(E * E):
        h = int(np.argmax(H))
        best = None
        for v in range(h * m, (h + 1) * m):
            for e in range(E):
                c = int(C[v, e])
                if not S[v, e] or e // m == h or c == 0:
                    continue
                val = max(int(H[h]) - c, int(H[e // m]) + c)
                if val < H[h] and (best is None or val < best[0]):
                    best = (val, v, e)
        if best is None:
            break
        _, v, e = best
        S[v, e] = False
        H, R = loads()
    return S, H, R


def top_m_mask(counts: np.ndarray, m: int) -> np.ndarray:
    """reference simulator._top_m_placement (simulator.py:318-324): the m experts
    with the largest column totals (ties -> lower index) on every device."""
    counts = np.asarray(counts, dtype=np.int64)
    D, E = counts.shape
    totals = counts.sum(axis=0)
    order = sorted(range(E), key=lambda e: (-int(totals[e]), e))
    return replica_mask(D, E, tuple(order[:m]), tuple(frozenset() for _ in range(m)))


def plan_for_iteration(history, iter_index: int, reuse_interval: int, planner):
    """reference planner.py:132-156; ``planner(counts)`` runs the search."""
    anchor = (iter_index // reuse_interval) * reuse_interval
    if anchor == 0:
        return None
    return planner(history[anchor - 1])


def balance_degree(H) -> float:
    """reference simulator.py:106-111 (population sigma)."""
    return float(np.std(np.asarray(H, dtype=np.float64)))


def rb_ratio(H_before, H_after) -> float:
    """reference simulator.py:114-124."""
    sb, sa = balance_degree(H_before), balance_degree(H_after)
    if sa == 0.0:
        return 1.0 if sb == 0.0 else float("inf")
    return sb / sa


def cost_model_dict(num_devices, top_k, input_bytes, param_bytes, grad_bytes, avg_bandwidth,
                    compute_throughput, fnec=0.0, bnec=0.0) -> dict:
    return {"num_devices": num_devices, "top_k": top_k, "input_bytes": input_bytes,
            "expert_param_bytes": param_bytes, "expert_grad_bytes": grad_bytes,
            "avg_bandwidth": avg_bandwidth, "compute_throughput": compute_throughput,
            "fnec_time": fnec, "bnec_time": bnec}
