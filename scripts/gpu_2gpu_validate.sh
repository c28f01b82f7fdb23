# 2-GPU box: real-NVLink EP parity, N=2 bench (reference search headline + physical alt), cfg3/cfg5 at N=2,
# ncu NVLink capture of rank 0's A2A / Trans / Agg kernels
set -x
nvidia-smi topo -m | head -5
timeout 1200 python -m pytest tests/test_multi_gpu.py -q > gpurun_out/r2_g13_mgpu_tests.log 2>&1; echo mgpu $?
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29621 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2_g13_n2.log 2>&1; echo n2 $?
timeout 600 $R --master-port 29622 bench.py --gpus 2 --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g13_n2_cfg3.log 2>&1; echo cfg3 $?
timeout 900 $R --master-port 29623 bench.py --gpus 2 --config cfg5 --steps 5 --warmup 3 > gpurun_out/r2_g13_n2_cfg5.log 2>&1; echo cfg5 $?
timeout 600 python -m torch.distributed.run --no-python --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29624 \
   scripts/ncu_rank0.sh gpurun_out/r2_ncu_nvlink_n2.csv --gpus 2 --steps 2 --warmup 3 --eager --profile-only > gpurun_out/r2_g13_ncu.log 2>&1; echo ncu $?
tail -2 gpurun_out/r2_g13_mgpu_tests.log
for f in n2 n2_cfg3 n2_cfg5; do echo "== $f"; tail -c 400 gpurun_out/r2_g13_$f.log; echo; done
