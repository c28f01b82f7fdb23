"""Per-k-step producer / MMA timestamp trace of one grouped-GEMM launch (CTA pair 0/1),
PPMOE_GEMM_DEBUG=2.  Prints where the MMA's waits on the TMA come from.
Usage: PPMOE_GEMM_DEBUG=2 python scripts/gemm_trace.py [MODE]"""
import ctypes
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2411_10003_b200 import _device, _lib

assert os.environ.get("PPMOE_GEMM_DEBUG") == "2"
T, k, E, d, f = 16384, 2, 16, 1024, 4096
rows = [T * k // E] * E
dev = torch.device("cuda")
groups, ng, total = _device.groups_tensor(rows, device=dev)
cap = int(math.ceil((total + 512) / 256) * 256)
X = torch.randn((cap, d), device=dev).to(torch.bfloat16)
W1 = (torch.randn((E, f, d), device=dev) / 32).to(torch.bfloat16)
W2 = (torch.randn((E, d, f), device=dev) / 64).to(torch.bfloat16)
pre = torch.zeros((cap, f), dtype=torch.bfloat16, device=dev)
act = torch.zeros((cap, f), dtype=torch.bfloat16, device=dev)
Y = torch.zeros((cap, d), dtype=torch.bfloat16, device=dev)
modes = {"FWD1": (_lib.PP_GEMM_FWD1, X, W1, pre, act), "FWD2": (_lib.PP_GEMM_FWD2, act, W2, Y, None)}
name = sys.argv[1] if len(sys.argv) > 1 else "FWD2"
mode, a, b, c, c2 = modes[name]
for _ in range(3):
    _device.grouped_gemm(mode, a, b, c, c2, groups, ng, E, cap, E, d, f)
torch.cuda.synchronize()
_device.grouped_gemm(mode, a, b, c, c2, groups, ng, E, cap, E, d, f)
torch.cuda.synchronize()
S = 1024
n = 4 * 1024 + 4 * S * 4
buf = (ctypes.c_ulonglong * n)()
_lib.check(_lib.load().pp_gemm_debug_read(buf, n // 4), "read")
tr = np.array(buf, dtype=np.int64)[4 * 1024:].reshape(4, S, 4)
lead, peer = tr[0], tr[1]
valid = (lead[:, 3] > 0) & (peer[:, 1] > 0)
L, P = lead[valid], peer[valid]
t0 = L[0, 0]
issue = np.maximum(L[:, 1], P[:, 1])          # both CTAs' loads issued
ready = L[:, 3]                               # MMA saw the stage full
mma_wait = L[:, 3] - L[:, 2]                  # MMA thread blocked on full
prod_wait = L[:, 1] - L[:, 0]                 # producer blocked on empty (pipeline full)
lat = ready - issue
span = (L[-1, 3] - L[0, 2]) / 1e3
print(f"{name}: {valid.sum()} steps traced, {span:.1f} us")
print(f"  MMA wait on full: total {mma_wait.sum()/1e3:.1f} us ({100*mma_wait.sum()/1e3/span:.1f} %), "
      f"median {np.median(mma_wait)} ns, p90 {np.percentile(mma_wait, 90):.0f} ns")
print(f"  producer wait on empty: median {np.median(prod_wait)} ns ({(prod_wait > 200).mean()*100:.0f} % of steps > 200 ns)")
print(f"  issue->ready (both CTAs' TMA): median {np.median(lat)} ns, p10 {np.percentile(lat,10):.0f}, p90 {np.percentile(lat, 90):.0f}")
print(f"  step period (MMA ready-to-ready): median {np.median(np.diff(ready))} ns")
print(f"  peer issue lag vs leader: median {np.median(P[:,1]-L[:,1])} ns")
for i in range(0, min(40, len(L))):
    print(f"  step {i:3d} prodwait {prod_wait[i]:6d} issue {issue[i]-t0:8d} mma_c {L[i,2]-t0:8d} ready {ready[i]-t0:8d} lat {lat[i]:6d}")
