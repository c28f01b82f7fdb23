cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for cfg in cfg2 cfg3; do
timeout 600 torchrun --standalone --nproc-per-node $NG bench.py --gpus $NG --steps 10 --warmup 3 --config $cfg > gpurun_out/bench_n${NG}_$cfg.log 2>&1; echo "bench $cfg rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_n${NG}_$cfg.log').read().strip().split('\n')[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['achieved'],d['imbalance']); print(json.dumps(d['phase_ms_rank0']))"
done
