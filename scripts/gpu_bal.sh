cd $GRAFT_REPO_ROOT
NG=$(nvidia-smi -L | wc -l)
for pol in vanilla greedy-overlap; do
timeout 600 torchrun --standalone --nproc-per-node $NG bench.py --gpus $NG --steps 10 --warmup 3 --policy $pol --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bal_$pol.log
python -c "
import json;d=json.loads(open('gpurun_out/bal_$pol.log').read());print('$pol', round(d['value']/1e6,2), d['rows_per_rank'], round(d['ms_per_step'],3), json.dumps({k: round(v,3) for k,v in d['phase_ms_rank0'].items()}))"
done
