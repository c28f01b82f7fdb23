cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
PP_ENGINE=copy timeout 300 torchrun --standalone --nproc-per-node $NG scripts/mgpu_check.py > gpurun_out/mgpu_copy.log 2>&1; echo "mgpu rc=$?"
grep "OK\|FAIL\|MISMATCH\|err\|Error" gpurun_out/mgpu_copy.log | head -5
timeout 900 torchrun --standalone --nproc-per-node $NG bench.py --gpus $NG --config cfg5 --steps 3 --warmup 2 > gpurun_out/bench_cfg5_n$NG.log 2>&1; echo "stack rc=$?"
tail -c 700 gpurun_out/bench_cfg5_n$NG.log
timeout 600 torchrun --standalone --nproc-per-node $NG bench.py --gpus $NG --steps 10 --warmup 3 > gpurun_out/bench_mgpu.log 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_mgpu.log').read().strip().split('\n')[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['achieved'])"
