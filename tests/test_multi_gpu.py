"""Multi-GPU parity of the EP layer (needs >= 2 GPUs on one node; skipped otherwise).

Runs scripts/mgpu_check.py under torchrun: routing, LoadMatrix, permutation,
in-loop plans vs the pinned oracle planner, outputs and grads vs the CPU oracle
over D simulated ranks, for host planning (copy-engine Trans/Agg) and device
planning (SM Trans/Agg; also CUDA-graph replay == eager, bit-exact), and the
physically-faithful planner (plans vs the oracle's greedy_search_physical)."""
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


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("planning,engine,policy,placement", [
    ("host", "copy", "", "virtual"), ("device", "sm", "", "virtual"), ("host", "sm", "top2", "virtual"),
    ("host", "copy", "vanilla", "virtual"), ("device", "sm", "", "physical"), ("host", "copy", "", "physical"),
    ("device", "sm", "", "physical+refine"), ("device", "sm", "", "physical+refine+fused"),
    ("host", "copy", "", "virtual+fused")])
def test_ep_layer_parity(planning, engine, policy, placement):
    n = min(_ngpus(), 4)
    opts = placement.split("+")[1:]
    env = dict(os.environ, PP_PLANNING=planning, PP_ENGINE=engine, PP_POLICY=policy,
               PP_PLACEMENT=placement.split("+")[0], PP_REFINE="1" if "refine" in opts else "0",
               PP_FUSED="1" if "fused" in opts else "0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", str(n),
           str(ROOT / "scripts" / "mgpu_check.py")]
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    tail = "\n".join((r.stdout + r.stderr).splitlines()[-30:])
    assert r.returncode == 0, tail
    assert "FAIL" not in r.stdout, tail
