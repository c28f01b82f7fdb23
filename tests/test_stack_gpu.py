"""The Algorithm-2 block stack runs fwd+bwd on the B200 and its measured
timeline is a well-formed reference-schema IterationTimeline."""

import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2411_10003_b200 as pp  # noqa: E402
from paper_2411_10003_b200.scheduler import OpKind  # noqa: E402
from paper_2411_10003_b200.stack import MoEStack  # noqa: E402


def test_stack_fwd_bwd_and_measured_timeline():
    L, d, f, E, k, T = 3, 256, 512, 16, 2, 2048
    stack = MoEStack(L, d, f, E, k, T, seq_len=512, n_heads=4)
    x = (torch.randn((T, d), device="cuda") * 0.5).to(torch.bfloat16).requires_grad_(True)
    dy = (torch.randn((T, d), device="cuda") * 0.1).to(torch.bfloat16)
    y = stack(x)
    y.backward(dy)
    torch.cuda.synchronize()
    assert torch.isfinite(y.float()).all() and torch.isfinite(x.grad.float()).all()
    for m in stack.moe:
        assert torch.isfinite(m.w1.main_grad).all() and m.w1.main_grad.abs().sum() > 0
    stack.start_timeline()
    x2 = x.detach().requires_grad_(True)
    stack(x2).backward(dy)
    tl = stack.measured_timeline()
    stack.stop_timeline()
    kinds = {o.kind for o in tl.ops}
    assert {OpKind.FNEC, OpKind.BNEC, OpKind.FEC, OpKind.BEC, OpKind.A2A} <= kinds
    for i in range(L):
        assert any(o.kind is OpKind.FEC and o.block == i for o in tl.ops)
    pt = tl.phase_totals()
    assert abs(sum(pt.values()) - tl.makespan()) < 1e-9
    assert all(o.duration > 0 and o.start >= 0 for o in tl.ops)
    costs = stack.measured_layer_costs(tl)
    assert len(costs) == L and all(c.fec_time > 0 and c.bec_time > 0 for c in costs)


def test_stack_blocks_match_the_oracle_and_graph_replays_eager():
    """Every block's MoE layer inside the stack against the CPU oracle (its own routing on the
    layer's bf16 input; tokens whose top-k the oracle ranks differently -- fp32 near-ties on
    non-exact LayerNorm outputs -- are excluded, at most 1 %), and the whole iteration captured as
    one CUDA graph (``MoEStack.make_graphed_step``) reproduces the eager step bit for bit where
    the step is deterministic: the output and the last block's expert / gate gradients."""
    import numpy as np

    from oracle import moe_ref as M

    L, d, f, E, k, T = 2, 256, 512, 16, 2, 2048
    stack = MoEStack(L, d, f, E, k, T, seq_len=512, n_heads=4, seed=3)
    cap = {}

    def fwd_hook(i):
        def h(mod, inp, out):
            u = inp[0]
            cap[i] = {"u": u.detach().clone(), "y": out.detach().clone()}
            u.register_hook(lambda g: cap[i].__setitem__("du", g.detach().clone()))
            out.register_hook(lambda g: cap[i].__setitem__("dy", g.detach().clone()))
        return h

    hooks = [m.register_forward_hook(fwd_hook(i)) for i, m in enumerate(stack.moe)]
    g = torch.Generator(device="cpu").manual_seed(9)
    x = (torch.randn((T, d), generator=g) * 0.5).to("cuda", torch.bfloat16).requires_grad_(True)
    dy = (torch.randn((T, d), generator=g) * 0.1).to("cuda", torch.bfloat16)
    y_eager = stack(x)
    y_eager.backward(dy)
    torch.cuda.synchronize()
    for h in hooks:
        h.remove()
    for i, m in enumerate(stack.moe):
        c = cap[i]
        ref = M.LayerRef(m.w1.detach().cpu(), m.w2.detach().cpu(), m.wg.detach().float().cpu(), None, k, D=1)
        ys, st = ref.forward([c["u"].cpu()])
        agree = (m.idx.cpu().long() == st["routes"][0][1]).all(dim=1).numpy()
        assert agree.mean() >= 0.99, (i, agree.mean())
        a = torch.from_numpy(agree)
        yr, yg = ys[0][a], c["y"].float().cpu()[a]
        assert (yg - yr).abs().max() <= 2e-2 * yr.abs().max(), i
        dxs, *_ = ref.backward([c["dy"].cpu().to(torch.bfloat16)], st)
        dr, dg = dxs[0][a], c["du"].float().cpu()[a]
        assert (dg - dr).abs().max() <= 2e-2 * dr.abs().max(), i
    last = stack.moe[-1]
    eager = (y_eager.detach().clone(), last.w1.main_grad.clone(), last.w2.main_grad.clone(),
             last.wg.main_grad.clone())
    sg = stack.make_graphed_step(x.detach(), dy)
    yg = sg()
    torch.cuda.synchronize()
    got = (yg.detach(), last.w1.main_grad, last.w2.main_grad, last.wg.main_grad)
    for a_, b_ in zip(eager, got):
        assert torch.equal(a_, b_)
    stack.close()
