"""Multi-rank parity of the EP layer.

Runs scripts/mgpu_check.py under torchrun: routing, LoadMatrix, permutation,
in-loop plans vs the pinned oracle planner, outputs and grads vs the CPU oracle
over D simulated ranks, for host planning (copy-engine Trans/Agg) and device
planning (SM Trans/Agg; also CUDA-graph replay == eager, bit-exact), and the
physically-faithful planner (plans vs the oracle's greedy_search_physical).

With >= 2 GPUs each rank gets its own device (NCCL/NVLink).  With ONE GPU the
ranks are emulated: D processes share cuda:0, exchange CUDA IPC handles over gloo
and talk through the same peer-memory kernels (dispatch/combine peer stores and
loads, Trans/Agg pushes, the layout / planner / GEMMs) -- only the NVLink hop is
replaced by local HBM.  The layer detects the shared device and synchronises on the
host instead of spinning on the device (barriers, Trans gates), so no kernel ever
waits on another process's progress; the CUDA-graph replay check needs one GPU per rank."""
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parent.parent

pytestmark = pytest.mark.gpu


def _ngpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _run(n, env_extra, timeout=600):
    env = dict(os.environ, **env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + (os.getpid() % 500)),
           str(ROOT / "scripts" / "mgpu_check.py")]
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    out = r.stdout.splitlines()
    tail = "\n".join([l for l in out if "FAIL" in l or "MISMATCH" in l or "err" in l][:20] + out[-15:] +
                     r.stderr.splitlines()[-25:])
    assert r.returncode == 0, tail
    assert "FAIL" not in r.stdout, tail
    assert "checked" in r.stdout, tail
    return r.stdout


CASES = [
    ("host", "copy", "", "virtual"), ("device", "sm", "", "virtual"), ("host", "sm", "top2", "virtual"),
    ("host", "copy", "vanilla", "virtual"), ("device", "sm", "", "physical"), ("host", "copy", "", "physical"),
    ("device", "sm", "", "physical+refine"), ("device", "sm", "", "physical+refine+fused"),
    ("host", "copy", "", "virtual+fused"), ("device", "sm", "", "virtual+reuse2"),
    ("host", "copy", "", "virtual+reuse2"), ("host", "sm", "", "virtual+reuse2"),
]


def _env(planning, engine, policy, placement):
    opts = placement.split("+")[1:]
    return dict(PP_PLANNING=planning, PP_ENGINE=engine, PP_POLICY=policy,
                PP_PLACEMENT=placement.split("+")[0], PP_REFINE="1" if "refine" in opts else "0",
                PP_FUSED="1" if "fused" in opts else "0", PP_REUSE="2" if "reuse2" in opts else "1")


@pytest.mark.skipif(_ngpus() < 1, reason="needs a GPU")
@pytest.mark.parametrize("planning,engine,policy,placement", CASES)
def test_ep_layer_parity(planning, engine, policy, placement):
    """D = 2 ranks (real GPUs when there are >= 2, else emulated on cuda:0); with >= 4
    GPUs, D = 4."""
    n = 4 if _ngpus() >= 4 else 2
    _run(n, _env(planning, engine, policy, placement))


@pytest.mark.skipif(_ngpus() < 1, reason="needs a GPU")
@pytest.mark.parametrize("planning,engine,placement", [("device", "sm", "virtual"), ("host", "copy", "physical+refine")])
def test_ep_layer_parity_d4(planning, engine, placement):
    """D = 4 ranks, m = 2 experts per rank (emulated on one GPU when fewer than 4)."""
    _run(4, _env(planning, engine, "", placement))


@pytest.mark.skipif(_ngpus() < 1, reason="needs a GPU")
def test_ep_layer_parity_d8_shape():
    """The N = 8 EP shape: 8 ranks, E = 16 (m = 2), emulated on the available GPUs."""
    _run(8, dict(_env("device", "sm", "", "virtual"), PP_T="1024", PP_E="16"), timeout=900)
