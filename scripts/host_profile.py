"""Host-side overhead of one MoELayer fwd+bwd step (cProfile + per-C-call timing)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2411_10003_b200 as pp
from paper_2411_10003_b200 import _lib

T, d, f, E, k = 16384, 1024, 4096, 16, 2
layer = pp.MoELayer(d, f, E, k, tokens=T)
x = torch.randn((T, d), device="cuda").to(torch.bfloat16)
dy = torch.randn((T, d), device="cuda").to(torch.bfloat16) * 0.1


def step():
    xi = x.detach().requires_grad_(True)
    y = layer(xi)
    y.backward(dy)


for _ in range(3):
    step()
torch.cuda.synchronize()

# per C entry point host cost
orig = _lib.call
costs = {}


def timed(name, *args):
    t = time.perf_counter()
    orig(name, *args)
    costs.setdefault(name, []).append(time.perf_counter() - t)


_lib.call = timed
t0 = time.perf_counter()
for _ in range(10):
    step()
host = (time.perf_counter() - t0) / 10
torch.cuda.synchronize()
_lib.call = orig
print(f"host per step {host*1e3:.3f} ms")
for n, v in sorted(costs.items(), key=lambda kv: -sum(kv[1])):
    print(f"  {n:24s} n={len(v):3d} avg={sum(v)/len(v)*1e6:9.1f} us  total/step={sum(v)/10*1e3:7.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    step()
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
