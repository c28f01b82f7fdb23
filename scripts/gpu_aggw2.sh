cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for i in 1 2; do for A in 16 8 4; do
timeout 600 torchrun --standalone --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline --agg-ctas-w2 $A > gpurun_out/aw_$A.log 2>&1
python -c "
import json;d=json.loads([l for l in open('gpurun_out/aw_$A.log') if l.startswith('{')][-1]);print('N=$N w2ctas=$A', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), {k: round(v,3) for k,v in d['side_stream_ms_rank0'].items()})"
done; done
