"""Standalone timing of the grouped GEMM modes at the cfg2 shape (uniform groups).
Usage: python scripts/gemm_bench.py [mode ...]   (PPMOE_GEMM_CTA_PAIR=0/1 selects 1-CTA / CTA-pair)"""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2411_10003_b200 import _device, _lib

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
G1 = torch.zeros((E, f, d), dtype=torch.float32, device=dev)
G2 = torch.zeros((E, d, f), dtype=torch.float32, device=dev)
modes = {
    "FWD1": (_lib.PP_GEMM_FWD1, X, W1, pre, act),
    "FWD2": (_lib.PP_GEMM_FWD2, act, W2, Y, None),
    "DGRAD2": (_lib.PP_GEMM_DGRAD2, Y, W2, pre, pre),
    "DGRAD1": (_lib.PP_GEMM_DGRAD1, pre, W1, Y, None),
    "WGRAD2": (_lib.PP_GEMM_WGRAD2, Y, act, G2, None),
    "WGRAD1": (_lib.PP_GEMM_WGRAD1, pre, X, G1, None),
    "PLAIN": (_lib.PP_GEMM_PLAIN, X, W1, pre, None),  # FWD1's shape, single bf16 output, no GeLU
}
times = {}
sel = sys.argv[1:] or list(modes)
flops = 2.0 * T * k * d * f
for name in sel:
    mode, a, b, c, c2 = modes[name]
    nsm = int(__import__("os").environ.get("GEMM_SMS", "0"))
    run = lambda: _device.grouped_gemm(mode, a, b, c, c2, groups, ng, E, cap, E, d, f, num_sms=nsm)  # noqa: E731
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    times[name] = ms
    print(f"{name:7s} {ms*1e3:8.1f} us  {flops/ms/1e9:8.1f} TFLOP/s", flush=True)

if __import__("os").environ.get("PPMOE_GEMM_DEBUG"):
    import ctypes
    import numpy as np

    lib = _lib.load()
    for name in sel:
        mode, a, b, c, c2 = modes[name]
        _device.grouped_gemm(mode, a, b, c, c2, groups, ng, E, cap, E, d, f, num_sms=int(__import__("os").environ.get("GEMM_SMS", "0")))
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * (148 * 4))()
        lib.pp_gemm_debug_read(buf, 148)
        arr = np.array(buf).reshape(148, 4)
        lead = arr[arr[:, 0] > 0]
        tot, wt, wf = lead[:, 0].mean(), lead[:, 1].mean(), lead[:, 2].mean()
        nsm_used = int(__import__("os").environ.get("GEMM_SMS", "0")) or 148
        fpc = flops / nsm_used / lead[:, 0].max()
        print(f"{name:7s} {fpc:7.0f} FLOP/cycle/SM over the MMA thread's window "
              f"({fpc / 8192 * 100:5.1f}% of 8192), implied SM clock {lead[:, 0].max() / (times.get(name, 1) * 1e-3) / 1e9:5.2f} GHz")
        print(f"{name:7s} MMA thread: total {tot:10.0f} cyc, wait tempty {wt/tot*100:5.1f}%, wait full {wf/tot*100:5.1f}%, "
              f"issue+other {(tot-wt-wf)/tot*100:5.1f}%  (CTAs {len(lead)}, max total {lead[:,0].max():.0f})")
