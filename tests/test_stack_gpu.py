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
