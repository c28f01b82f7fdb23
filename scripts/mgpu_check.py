"""Multi-GPU parity check of the EP layer (run under torchrun, N >= 2 GPUs).

Rank 0 replays every rank's inputs through the CPU oracle (oracle/moe_ref.LayerRef
over D simulated ranks) and checks: routing/LoadMatrix/destination rows exact,
the plan used at iteration 1 == pinned oracle greedy on iteration 0's LoadMatrix
(plan_for_iteration rule), outputs and gradients (home experts after Agg) within
bf16 tolerance.  Exits non-zero on any mismatch.
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import torch.distributed as dist

import paper_2411_10003_b200 as pp
from oracle import moe_ref as M
from oracle import planner_ref as P


def rel(a, b):
    a, b = a.float().cpu(), b.float().cpu()
    return (a - b).abs().max().item() / (b.abs().max().item() + 1e-6)


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    ngpu = torch.cuda.device_count()
    # emulated ranks: fewer GPUs than ranks -> several rank processes share a device
    # (CUDA IPC between processes on one device; time-sliced contexts make the spin
    # barriers progress); NCCL refuses duplicate devices, so the plumbing uses gloo
    emulated = ngpu < world
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)) % ngpu)
    dev = torch.device("cuda", torch.cuda.current_device())
    if emulated:  # fail fast instead of waiting out gloo's 30-minute default on a broken peer
        import datetime

        dist.init_process_group("gloo", timeout=datetime.timedelta(seconds=240))
    else:
        dist.init_process_group("cpu:gloo,cuda:nccl", device_id=dev)
    if rank == 0:
        print(f"ranks {world} on {ngpu} GPU(s){' (emulated: shared device)' if emulated else ''}", flush=True)
    E = int(os.environ.get("PP_E", 4 * world))
    T, d, f, k = int(os.environ.get("PP_T", 2048)), 256, 512, 2
    m = E // world
    cl = pp.ClusterSpec(E, 1e11, 1e6)  # cheap transfers: the planner replicates
    mo = pp.ModelSpec(E, 1, k, 2 * d, 1e3, 1e3)
    placement = os.environ.get("PP_PLACEMENT", "virtual")
    n_excl = int(os.environ.get("PP_N", "1" if placement == "virtual" else "0"))
    reuse = int(os.environ.get("PP_REUSE", "1"))
    iters = 3 if reuse == 1 else 5
    layer = pp.MoELayer(d, f, E, k, tokens=T, group=dist.group.WORLD,
                        planner=pp.PlannerConfig(n=n_excl, alpha=0.5, reuse_interval=reuse), cluster=cl, model=mo, seed=0,
                        placement=placement, refine_slots=os.environ.get("PP_REFINE") == "1",
                        fused_a2a=os.environ.get("PP_FUSED") == "1",
                        replica_engine=os.environ.get("PP_ENGINE", "copy"),
                        policy=os.environ.get("PP_POLICY") or None,
                        planning=os.environ.get("PP_PLANNING", "host"))
    policy = os.environ.get("PP_POLICY") or "greedy"
    _, wg = M.exact_inputs(16, d, E, seed=99)
    bias = torch.round(torch.log(torch.tensor([1.0 / (i + 1) ** 1.2 for i in range(E)])) * 4) / 4
    with torch.no_grad():
        layer.wg.copy_(wg.to(dev))
    layer.set_gate_bias(bias)
    # global expert weights (every rank built them from the same seed)
    g = torch.Generator().manual_seed(0)
    import math
    w1_all = (torch.randn((E, f, d), generator=g) / math.sqrt(d)).to(torch.bfloat16)
    w2_all = (torch.randn((E, d, f), generator=g) / math.sqrt(f)).to(torch.bfloat16)
    ok = True
    hist = []
    for it in range(iters):
        x, _ = M.exact_inputs(T, d, E, seed=1000 * it + rank)
        dy = (torch.randn((T, d), generator=torch.Generator().manual_seed(7 + it * 31 + rank)) * 0.1).to(torch.bfloat16)
        xd = x.to(dev).requires_grad_(True)
        y = layer(xd)
        anchor = (it // reuse) * reuse  # plan_for_iteration (planner.py:148-156)
        mask_used = layer.current_mask() if (anchor > 0 or policy.startswith("top")) else None  # plan used
        y.backward(dy.to(dev))
        layer.wait_grads()
        torch.cuda.synchronize()
        rec = dict(x=x, dy=dy, y=y.detach().cpu(), dx=xd.grad.cpu(), idx=layer.idx.cpu(),
                   row=layer.pair_row.cpu(), dest=layer.pair_dest.cpu(), counts=layer.counts.cpu(),
                   g1=layer.w1.main_grad.cpu(), g2=layer.w2.main_grad.cpu(), gwg=layer.wg.main_grad.cpu(),
                   mask=mask_used)
        allrec = [None] * world
        dist.all_gather_object(allrec, rec)
        if rank == 0:
            counts = allrec[0]["counts"].numpy()
            if policy.startswith("top"):
                exp_mask = P.top_m_mask(counts, int(policy[3:]))
                if not np.array_equal(mask_used, exp_mask):
                    print(f"[it {it}] TOP-M MASK MISMATCH", flush=True)
                    ok = False
            elif policy == "vanilla":
                pass
            elif anchor > 0:
                # plan_for_iteration: iteration it uses greedy(history[anchor-1])
                prev_counts = hist[anchor - 1]
                if placement == "physical":
                    cm = P.cost_model_dict(world, k, 2 * d, 1e3, 1e3, 1e11, 1e6)
                    phys = prev_counts.reshape(world, m, E).sum(axis=1)
                    exp = P.greedy_search_physical(phys, n_excl, 0.5, False, cm)
                    if os.environ.get("PP_REFINE") == "1":
                        exp["mask"] = P.refine_slots(prev_counts, exp["mask"])[0]
                    else:
                        exp["mask"] = np.repeat(exp["mask"], m, axis=0)
                else:
                    cm = P.cost_model_dict(E, k, 2 * d, 1e3, 1e3, 1e11, 1e6)
                    exp = P.greedy_search(prev_counts, n_excl, 0.5, False, cm)
                if not np.array_equal(mask_used, exp["mask"]):
                    print(f"[it {it}] MASK MISMATCH: plan {exp['selected']}", flush=True)
                    ok = False
                else:
                    print(f"[it {it}] plan {exp['selected']} excl {[sorted(s) for s in exp['excluded']]} matches oracle")
            ref = M.LayerRef(w1_all, w2_all, wg, bias, k, D=world)
            ys, st = ref.forward([r["x"] for r in allrec], mask=mask_used)
            if not np.array_equal(counts, st["hist"]):
                print(f"[it {it}] LoadMatrix mismatch", flush=True); ok = False
            for r in range(world):
                dest, row = st["pos"][r]
                if not (np.array_equal(allrec[r]["row"].numpy(), row) and np.array_equal(allrec[r]["dest"].numpy(), dest)):
                    print(f"[it {it}] rank {r} permutation mismatch", flush=True); ok = False
                e = rel(allrec[r]["y"], ys[r])
                if e > 2e-2:
                    print(f"[it {it}] rank {r} y rel err {e}", flush=True); ok = False
            dxs, dw1, dw2, dwg, _ = ref.backward([r["dy"] for r in allrec], st)
            for r in range(world):
                e = rel(allrec[r]["dx"], dxs[r])
                if e > 2e-2:
                    print(f"[it {it}] rank {r} dx rel err {e}", flush=True); ok = False
                e1 = rel(allrec[r]["g1"], dw1[r * m:(r + 1) * m])
                e2 = rel(allrec[r]["g2"], dw2[r * m:(r + 1) * m])
                if e1 > 1e-2 or e2 > 1e-2:
                    print(f"[it {it}] rank {r} expert grad rel err {e1} {e2}", flush=True); ok = False
            gsum = sum(r["gwg"] for r in allrec)
            e = rel(gsum, dwg)
            if e > 1e-2:
                print(f"[it {it}] gate grad rel err {e}", flush=True); ok = False
            print(f"[it {it}] checked {world} ranks: {'OK' if ok else 'FAIL'}", flush=True)
            hist.append(counts)
        # "optimizer step": exact power-of-two rescale of the home experts, so a replica that
        # is not refreshed by this iteration's Trans shows up as an output mismatch
        with torch.no_grad():
            layer.w1.mul_(2.0)
            layer.w2.mul_(0.5)
        w1_all, w2_all = w1_all * 2.0, w2_all * 0.5
        okt = torch.tensor([1 if ok else 0])
        dist.broadcast(okt, 0)
        ok = bool(okt.item())
    if layer.planning == "device" and not layer.shared_device:
        # graph replay of the whole EP step (barriers, plan, Trans/Agg inside) == eager, bit-exact
        x, _ = M.exact_inputs(T, d, E, seed=4242 + rank)
        xd = x.to(dev)
        dyd = (torch.randn((T, d), generator=torch.Generator().manual_seed(5 + rank)) * 0.1).to(dev, torch.bfloat16)
        for _ in range(3):  # same batch every step: the plan reaches its fixed point
            xe = xd.clone().requires_grad_(True)
            ye = layer(xe)
            ye.backward(dyd)
        torch.cuda.synchronize()
        ref_out = (ye.detach().clone(), xe.grad.clone(), layer.w1.main_grad.clone(), layer.w2.main_grad.clone(),
                   layer.wg.main_grad.clone())
        gs = layer.make_graphed_step(xd.clone(), dyd.clone())
        for _ in range(2):
            yg, dxg = gs()
        torch.cuda.synchronize()
        got = (yg, dxg, layer.w1.main_grad, layer.w2.main_grad, layer.wg.main_grad)
        same = all(torch.equal(a, b) for a, b in zip(ref_out, got))
        flag = torch.tensor([1 if same else 0])
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if rank == 0:
            print(f"[graph] replay == eager on {world} ranks: {'OK' if flag.item() else 'FAIL'}", flush=True)
        ok = ok and bool(flag.item())
    layer.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
