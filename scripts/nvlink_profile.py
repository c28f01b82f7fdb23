"""ncu NVLink capture of the EP layer's A2A / Trans / Agg kernels at N ranks (run under torchrun
with scripts/ncu_rank0.sh-style wrapping of rank 0).  gloo plumbing (no NCCL under ncu), eager
steps with device planning + SM-engine Trans/Agg at the cfg2 shape."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import torch.distributed as dist

import paper_2411_10003_b200 as pp

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count())
dist.init_process_group("gloo", timeout=__import__("datetime").timedelta(minutes=10))
E, k, d, f, T = 16, 2, 1024, 4096, 16384
layer = pp.MoELayer(d, f, E, k, tokens=T, group=dist.group.WORLD, planning="device",
                    planner=pp.PlannerConfig(n=1, alpha=0.5), seed=0)
import numpy as np
w = np.arange(1, E + 1, dtype=np.float64) ** -1.2
layer.set_gate_bias(np.log(w / w.sum())[np.random.default_rng(0).permutation(E)])
g = torch.Generator().manual_seed(1000 + rank)
x = torch.randn((T, d), generator=g).to("cuda", torch.bfloat16)
dy = (torch.randn((T, d), generator=g) * 0.1).to("cuda", torch.bfloat16)
for it in range(int(os.environ.get("PP_STEPS", "5"))):
    xin = x.clone().requires_grad_(True)
    layer(xin).backward(dy)
    layer.wait_grads()
torch.cuda.synchronize()
dist.barrier()
print(f"rank {rank} done; replicas {layer.replica_traffic()['replicas_per_rank']}", flush=True)
layer.close()
dist.destroy_process_group()
