cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
NG=$(nvidia-smi -L | wc -l)
echo "gpus=$NG"
timeout 300 torchrun --standalone --nproc-per-node $NG scripts/mgpu_check.py > gpurun_out/mgpu.log 2>&1; echo "mgpu rc=$?"
tail -20 gpurun_out/mgpu.log
timeout 600 torchrun --standalone --nproc-per-node $NG bench.py --gpus $NG --steps 10 --warmup 3 > gpurun_out/bench_mgpu.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_mgpu.log
