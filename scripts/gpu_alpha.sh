cd $GRAFT_REPO_ROOT
NG=$(nvidia-smi -L | wc -l)
for a in 0.5 0.2 0.05; do for n in 1 4; do
timeout 600 torchrun --standalone --nproc-per-node $NG bench.py --gpus $NG --steps 10 --warmup 3 --alpha $a --n-excl $n --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/alpha.log
python -c "
import json;d=json.loads(open('gpurun_out/alpha.log').read());print('alpha $a n $n', round(d['value']/1e6,2), d['rows_per_rank'], round(d['ms_per_step'],3))"
done; done
