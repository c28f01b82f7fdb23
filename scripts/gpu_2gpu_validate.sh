# 2-GPU box: real-NVLink EP parity, N=2 bench (reference search headline + physical alt), cfg3/cfg5
# at N=2, the staggered-GEMM A/B at N=2
set -x
nvidia-smi topo -m | head -5
timeout 1500 python -m pytest tests/test_multi_gpu.py -q --timeout 900 > gpurun_out/v2_mgpu_tests.log 2>&1; echo mgpu $?
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29621 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/v2_n2.log 2>&1; echo n2 $?
PPMOE_GEMM_STAGGER=${STAGGER:-1} PPMOE_GEMM_STAGGER_WGRAD=${STAGGER:-1} timeout 600 $R --master-port 29625 bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --alt-placement 0 > gpurun_out/v2_n2_stagger.log 2>&1; echo n2_stagger $?
timeout 600 $R --master-port 29622 bench.py --gpus 2 --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v2_n2_cfg3.log 2>&1; echo cfg3 $?
timeout 900 $R --master-port 29623 bench.py --gpus 2 --config cfg5 --steps 5 --warmup 3 > gpurun_out/v2_n2_cfg5.log 2>&1; echo cfg5 $?
tail -2 gpurun_out/v2_mgpu_tests.log
for f in n2 n2_stagger n2_cfg3 n2_cfg5; do echo "== $f"; tail -c 400 gpurun_out/v2_$f.log; echo; done
