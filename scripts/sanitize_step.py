"""One small MoE-layer fwd+bwd (K1 route, layout, K3 dispatch/combine + backward, K4 all six
grouped-GEMM modes, gate dW/dX) plus one K2 planner launch on cuda:0 -- the workload the
compute-sanitizer logs in profiles/ were taken on:

    compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize_step.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2411_10003_b200 as pp

T, d, f, E, k = 1024, 256, 512, 8, 2
layer = pp.MoELayer(d, f, E, k, tokens=T, seed=0)
x = torch.randn((T, d), device="cuda").to(torch.bfloat16).requires_grad_(True)
y = layer(x)
y.backward(torch.randn_like(y) * 0.1)
torch.cuda.synchronize()
rng = np.random.default_rng(0)
counts = np.stack([rng.multinomial(512, rng.dirichlet(np.ones(16) * 0.3)) for _ in range(16)]).astype(np.int64)
cl, mo = pp.ClusterSpec(16, 4e11, 1e8), pp.ModelSpec(16, 1, 2, 2048, 1.6e7, 3.2e7)
plan = pp.greedy_search(pp.LoadMatrix(counts), pp.PlannerConfig(n=1, alpha=0.5), cl, mo)
phys = pp.greedy_search_physical(pp.LoadMatrix(counts.reshape(4, 4, 16).sum(axis=1)), pp.PlannerConfig(n=1, alpha=0.5),
                                 pp.ClusterSpec(4, 4e11, 1e8), mo)
torch.cuda.synchronize()
print("sanitize step ok:", float(y.float().abs().sum()), plan.selected, phys.placement.selected)
