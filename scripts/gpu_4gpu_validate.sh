# 4 GPUs: full GPU suite on real NVLink (D=4, and D=8 as 2 ranks per GPU), weak scaling N=1/2/4,
# other configs at N=4, NVLink ncu capture (rank 0 under ncu, gloo plumbing)
set -x
nvidia-smi --query-gpu=index,name,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2_g17_tests.log 2>&1; echo tests $?
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python bench.py --steps 30 --warmup 5 > gpurun_out/r2_g17_n1.log 2>&1; echo n1 $?
timeout 600 $R --nproc-per-node 2 --master-port 29651 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2_g17_n2.log 2>&1; echo n2 $?
timeout 600 $R --nproc-per-node 4 --master-port 29652 bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2_g17_n4.log 2>&1; echo n4 $?
timeout 600 $R --nproc-per-node 4 --master-port 29653 bench.py --gpus 4 --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g17_n4_cfg3.log 2>&1; echo cfg3 $?
timeout 600 $R --nproc-per-node 4 --master-port 29654 bench.py --gpus 4 --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g17_n4_cfg4.log 2>&1; echo cfg4 $?
timeout 900 $R --nproc-per-node 4 --master-port 29655 bench.py --gpus 4 --config cfg5 --steps 5 --warmup 3 > gpurun_out/r2_g17_n4_cfg5.log 2>&1; echo cfg5 $?
timeout 400 python -m torch.distributed.run --no-python --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29656 \
   scripts/ncu_rank0.sh gpurun_out/r2_ncu_nvlink_n2.csv scripts/nvlink_profile.py > gpurun_out/r2_g17_ncu.log 2>&1; echo ncu $?
tail -2 gpurun_out/r2_g17_tests.log
grep -c "" gpurun_out/r2_ncu_nvlink_n2.csv
