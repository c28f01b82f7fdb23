"""ORACLE (test infrastructure only) -- CPU restatement of the MoE-layer contract.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module.

Parity status: the reference (``moebal``) contains NO routing, permutation,
expert FFN or gradient code -- it only counts routed inputs (``LoadMatrix``,
``core.py:88-142``) and applies the routing rule of ``derive_loads``
(``core.py:255-275``).  For those parts parity is UNPINNED by the reference;
this file *defines* the contract (DESIGN.md section "Routing contract") and the
integer parts of it are tied back to the reference as follows:

* the per-(virtual slot, expert) histogram produced here must equal the
  ``LoadMatrix`` rows the reference consumes, and the per-rank computed /
  received row counts implied by the layout must equal reference
  ``derive_loads`` H / R on that matrix (checked in tests);
* top-k ties go to the lowest expert index (the reference's tie convention,
  SPEC.md:248);
* token -> computing-rank rule is reference ``core.py:267-274`` at virtual-slot
  granularity.

Floating point: fp32 math with bf16 rounding at the same points as the GPU
path (expert inputs/outputs and activations stored bf16), GeLU tanh form.
"""

from __future__ import annotations

import math

import numpy as np
import torch

CHUNK = 128
ROW_ALIGN = 128


def bf16(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32)


def gelu(x: torch.Tensor) -> torch.Tensor:
    k0, k1 = 0.7978845608028654, 0.044715
    return 0.5 * x * (1.0 + torch.tanh(k0 * (x + k1 * x * x * x)))


def dgelu(x: torch.Tensor) -> torch.Tensor:
    k0, k1 = 0.7978845608028654, 0.044715
    t = torch.tanh(k0 * (x + k1 * x * x * x))
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * k0 * (1.0 + 3.0 * k1 * x * x)


# --------------------------------------------------------------------------- routing
def route(x: torch.Tensor, wg: torch.Tensor, bias, k: int):
    """logits = x . wg^T + bias (fp32); top-k on logits, ties -> lowest expert;
    w = softmax(logits)[idx] (not renormalised)."""
    logits = x.float() @ wg.float().t()
    if bias is not None:
        logits = logits + torch.as_tensor(bias, dtype=torch.float32)
    lg = logits.numpy()
    order = np.argsort(-lg, axis=1, kind="stable")[:, :k]
    probs = torch.softmax(logits, dim=1)
    idx = torch.from_numpy(order.astype(np.int64))
    w = torch.gather(probs, 1, idx)
    return logits, idx, w, probs


def chunk_ranks(idx: np.ndarray, E: int):
    """rank[t][j] = #earlier tokens of t's 128-token chunk routed to idx[t][j];
    chunk_counts[c][e]."""
    T, k = idx.shape
    C = T // CHUNK
    rank = np.zeros((T, k), dtype=np.int64)
    counts = np.zeros((C, E), dtype=np.int64)
    for c in range(C):
        run = np.zeros(E, dtype=np.int64)
        for t in range(c * CHUNK, (c + 1) * CHUNK):
            for j in range(k):
                e = idx[t, j]
                rank[t, j] = run[e]
            for j in range(k):
                run[idx[t, j]] += 1
        counts[c] = run
    return rank, counts


def slot_histogram(idx: np.ndarray, E: int, m: int) -> np.ndarray:
    """Rows of the virtual-slot LoadMatrix owned by one rank: slot j = tokens
    [j*T/m, (j+1)*T/m)."""
    T = idx.shape[0]
    per = T // m
    out = np.zeros((m, E), dtype=np.int64)
    for j in range(m):
        for e in idx[j * per:(j + 1) * per].reshape(-1):
            out[j, e] += 1
    return out


# --------------------------------------------------------------------------- layout
def layout(counts: np.ndarray, mask, D: int, m: int):
    """Receive layout of every rank (reference routing rule core.py:267-274 at
    virtual-slot granularity).  Returns comp[v][e], per-rank groups (ascending
    expert), seg_start[r][e], and base[v][e] = first destination row of the
    pairs of slot v routed to e."""
    Ev, E = counts.shape
    if mask is None:
        mask = np.eye(Ev, E, dtype=bool)
    comp = np.where(mask, (np.arange(Ev) // m)[:, None], (np.arange(E) // m)[None, :])
    rows = np.zeros((D, E), dtype=np.int64)
    present = np.zeros((D, E), dtype=bool)
    for r in range(D):
        present[r, r * m:(r + 1) * m] = True
    for v in range(Ev):
        for e in range(E):
            rows[comp[v, e], e] += counts[v, e]
            if mask[v, e]:
                present[v // m, e] = True
    seg = np.full((D, E), -1, dtype=np.int64)
    groups = []
    for r in range(D):
        off, nrep, gl = 0, 0, []
        for e in range(E):
            if not present[r, e]:
                continue
            pad = (rows[r, e] + ROW_ALIGN - 1) // ROW_ALIGN * ROW_ALIGN
            home = e // m == r
            wslot = e % m if home else m + nrep
            nrep += 0 if home else 1
            gl.append({"row_off": off, "rows": int(rows[r, e]), "rows_pad": int(pad), "wslot": wslot,
                       "expert": e, "src_rank": e // m})
            seg[r, e] = off
            off += pad
        groups.append(gl)
    base = np.zeros((Ev, E), dtype=np.int64)
    for e in range(E):
        run = {r: int(seg[r, e]) for r in range(D)}
        for v in range(Ev):
            dst = comp[v, e]
            base[v, e] = run[dst]
            run[dst] += counts[v, e]
    return {"comp": comp, "groups": groups, "seg": seg, "base": base, "rows": rows, "present": present}


def pair_positions(idx: np.ndarray, rank_in_chunk: np.ndarray, chunk_counts: np.ndarray,
                   lay: dict, me: int, m: int):
    """(dest rank, destination row) of every (t, j) pair of rank ``me``."""
    T, k = idx.shape
    per = T // m
    cps = per // CHUNK
    dest = np.zeros((T, k), dtype=np.int64)
    row = np.zeros((T, k), dtype=np.int64)
    for t in range(T):
        j_slot = t // per
        v = me * m + j_slot
        c = t // CHUNK
        c0 = j_slot * cps
        for j in range(k):
            e = idx[t, j]
            dest[t, j] = lay["comp"][v, e]
            row[t, j] = lay["base"][v, e] + chunk_counts[c0:c, e].sum() + rank_in_chunk[t, j]
    return dest, row


# --------------------------------------------------------------------------- layer
class LayerRef:
    """One EP layer over D simulated ranks (CPU), same contract as MoELayer."""

    def __init__(self, w1_all, w2_all, wg, bias, k: int, D: int) -> None:
        self.w1 = w1_all.float()  # [E, f, d]
        self.w2 = w2_all.float()  # [E, d, f]
        self.wg = wg.float()      # [E, d]
        self.bias = bias
        self.k, self.D = k, D
        self.E = w1_all.shape[0]
        self.m = self.E // D

    def forward(self, xs, mask=None):
        """xs: list of D tensors [T, d] (bf16 values).  Returns ys, state."""
        E, k, D, m = self.E, self.k, self.D, self.m
        routes = [route(x, self.wg, self.bias, k) for x in xs]
        hist = np.concatenate([slot_histogram(r[1].numpy(), E, m) for r in routes])
        lay = layout(hist, mask, D, m)
        # per rank receive buffers (expert-major, padded)
        recv_rows = [sum(g["rows_pad"] for g in lay["groups"][r]) for r in range(D)]
        d = xs[0].shape[1]
        xp = [torch.zeros((max(n, 1), d)) for n in recv_rows]
        pos = []
        for r, (x, rt) in enumerate(zip(xs, routes)):
            idx = rt[1].numpy()
            rk, cc = chunk_ranks(idx, E)
            dest, row = pair_positions(idx, rk, cc, lay, r, m)
            pos.append((dest, row))
            for t in range(x.shape[0]):
                for j in range(k):
                    xp[dest[t, j]][row[t, j]] = x[t].float()
        # expert FFN per rank and group
        pre, act, yp = [], [], []
        for r in range(D):
            P = torch.zeros((xp[r].shape[0], self.w1.shape[1]))
            A = torch.zeros_like(P)
            Y = torch.zeros_like(xp[r])
            for g in lay["groups"][r]:
                s = slice(g["row_off"], g["row_off"] + g["rows"])
                e = g["expert"]
                P[s] = bf16(xp[r][s] @ self.w1[e].t())
                A[s] = bf16(gelu(P[s]))
                Y[s] = bf16(A[s] @ self.w2[e].t())
            pre.append(P)
            act.append(A)
            yp.append(Y)
        ys = []
        for r, rt in enumerate(routes):
            dest, row = pos[r]
            w = rt[2]
            T = xs[r].shape[0]
            y = torch.zeros((T, d))
            for j in range(k):
                rows = torch.stack([yp[dest[t, j]][row[t, j]] for t in range(T)])
                y += w[:, j:j + 1] * rows
            ys.append(bf16(y))
        state = dict(routes=routes, hist=hist, lay=lay, pos=pos, xp=xp, pre=pre, act=act, yp=yp, xs=xs)
        return ys, state

    def backward(self, dys, st):
        E, k, D = self.E, self.k, self.D
        lay, pos, routes = st["lay"], st["pos"], st["routes"]
        d = dys[0].shape[1]
        dyp = [torch.zeros_like(x) for x in st["xp"]]
        dws = []
        for r, dy in enumerate(dys):
            dest, row = pos[r]
            w = routes[r][2]
            T = dy.shape[0]
            dw = torch.zeros((T, k))
            for t in range(T):
                for j in range(k):
                    yrow = st["yp"][dest[t, j]][row[t, j]]
                    dw[t, j] = (dy[t].float() * yrow).sum()
                    dyp[dest[t, j]][row[t, j]] = bf16(w[t, j] * dy[t].float())
            dws.append(dw)
        dw1 = torch.zeros_like(self.w1)
        dw2 = torch.zeros_like(self.w2)
        dxp = []
        for r in range(D):
            DX = torch.zeros_like(st["xp"][r])
            for g in lay["groups"][r]:
                s = slice(g["row_off"], g["row_off"] + g["rows"])
                e = g["expert"]
                dact = dyp[r][s] @ self.w2[e]
                dpre = bf16(dact * dgelu(st["pre"][r][s]))
                dw2[e] += dyp[r][s].t() @ st["act"][r][s]
                DX[s] = bf16(dpre @ self.w1[e])
                dw1[e] += dpre.t() @ st["xp"][r][s]
            dxp.append(DX)
        dxs, dwg = [], torch.zeros_like(self.wg)
        for r, dy in enumerate(dys):
            dest, row = pos[r]
            logits, idx, w, probs = routes[r]
            T = dy.shape[0]
            dw = dws[r]
            g = (dw * w).sum(dim=1, keepdim=True)  # sum_j dw_j p_{e_j}
            sel = torch.zeros((T, E))
            sel.scatter_(1, idx, dw)
            dlogits = probs * (sel - g)
            dx = dlogits @ self.wg
            for j in range(k):
                dx += torch.stack([dxp[dest[t, j]][row[t, j]] for t in range(T)])
            dxs.append(bf16(dx))
            dwg += dlogits.t() @ st["xs"][r].float()
        return dxs, dw1, dw2, dwg, dws


def exact_inputs(T: int, d: int, E: int, seed: int):
    """Exact-arithmetic routing inputs: x, wg in {-2..2} * 2^-2,
    so every fp32 logit is exact in any summation order (|logit| <= d/4 < 2^20)."""
    g = torch.Generator().manual_seed(seed)
    x = (torch.randint(-2, 3, (T, d), generator=g).float() * 0.25).to(torch.bfloat16)
    wg = (torch.randint(-2, 3, (E, d), generator=g).float() * 0.25).to(torch.bfloat16)
    return x, wg


def layer_flops(T: int, k: int, d: int, f: int) -> float:
    """fwd+bwd expert GEMM flops: 3 passes x 2 GEMMs x 2*T*k*d*f."""
    return 12.0 * T * k * d * f


def cpu_layer_step(x, wg, w1, w2, k: int, dy):
    """Torch-CPU fp32 restatement of one 1-rank fwd+bwd (vectorised, used as the
    timed CPU baseline; same math as LayerRef with D=1, no padding)."""
    E = w1.shape[0]
    xf = x.float()
    logits = xf @ wg.float().t()
    probs = torch.softmax(logits, 1)
    w, idx = torch.topk(logits, k, dim=1)  # CPU baseline: torch's tie rule is fine for timing
    w = torch.gather(probs, 1, idx)
    y = torch.zeros_like(xf)
    saved = []
    for e in range(E):
        tok, slot = (idx == e).nonzero(as_tuple=True)
        xe = xf[tok]
        pre = xe @ w1[e].float().t()
        act = gelu(pre)
        ye = act @ w2[e].float().t()
        y.index_add_(0, tok, w[tok, slot, None] * ye)
        saved.append((tok, slot, xe, pre, act, ye))
    dyf = dy.float()
    dx = torch.zeros_like(xf)
    for e, (tok, slot, xe, pre, act, ye) in enumerate(saved):
        g = w[tok, slot, None] * dyf[tok]
        dact = g @ w2[e].float()
        dpre = dact * dgelu(pre)
        _ = g.t() @ act
        _ = dpre.t() @ xe
        dx.index_add_(0, tok, dpre @ w1[e].float())
    return y, dx
