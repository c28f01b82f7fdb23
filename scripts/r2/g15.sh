# 2 GPUs: ncu NVLink capture (gloo plumbing, eager), N=2 bench with NVML NVLink counters, alpha sweep
set -x
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 400 python -m torch.distributed.run --no-python --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 \
   scripts/r2/ncu_rank0.sh gpurun_out/r2_ncu_nvlink_n2.csv scripts/nvlink_profile.py > gpurun_out/r2_g15_ncu.log 2>&1; echo ncu $?
timeout 600 $R --master-port 29632 bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_g15_n2.log 2>&1; echo n2 $?
for a in 0.1 0.25; do
  timeout 600 $R --master-port 2964${a: -1} bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --alpha $a --alt-placement 0 > gpurun_out/r2_g15_n2_a$a.log 2>&1; echo alpha $a $?
done
tail -5 gpurun_out/r2_g15_ncu.log
grep -c "" gpurun_out/r2_ncu_nvlink_n2.csv
