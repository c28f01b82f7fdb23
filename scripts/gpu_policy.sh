cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for pol in top2 vanilla; do
PP_POLICY=$pol timeout 300 torchrun --standalone --nproc-per-node $NG scripts/mgpu_check.py > gpurun_out/mgpu_$pol.log 2>&1; echo "mgpu $pol rc=$?"
grep "OK\|FAIL\|MISMATCH\|rror" gpurun_out/mgpu_$pol.log | head -4
done
for pol in vanilla top2 greedy greedy-overlap; do
timeout 600 torchrun --standalone --nproc-per-node $NG bench.py --gpus $NG --steps 10 --warmup 3 --policy $pol --no-cpu-baseline > gpurun_out/bench_pol_$pol.log 2>&1; echo "bench $pol rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_pol_$pol.log').read().strip().split('\n')[-1]);print('$pol', round(d['value']/1e6,3), 'Mtok/s', round(d['ms_per_step'],3), 'ms', d['imbalance'])"
done
