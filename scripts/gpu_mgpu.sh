cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
echo "gpus=$NG"
for eng in copy sm; do
PP_ENGINE=$eng timeout 300 torchrun --standalone --nproc-per-node $NG scripts/mgpu_check.py > gpurun_out/mgpu_$eng.log 2>&1; echo "mgpu $eng rc=$?"
grep "OK\|FAIL\|MISMATCH\|err\|Error" gpurun_out/mgpu_$eng.log | head -8
done
timeout 600 torchrun --standalone --nproc-per-node $NG bench.py --gpus $NG --steps 10 --warmup 3 > gpurun_out/bench_mgpu.log 2>&1; echo "bench rc=$?"
tail -c 400 gpurun_out/bench_mgpu.log
