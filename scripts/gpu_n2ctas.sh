cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for i in 1 2; do for V in "16 16" "8 8" "4 4" "8 16"; do set -- $V
timeout 600 torchrun --standalone --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline --trans-ctas $1 --agg-ctas $2 --agg-ctas-w2 $2 > gpurun_out/n2c.log 2>&1
python -c "
import json;d=json.loads([l for l in open('gpurun_out/n2c.log') if l.startswith('{')][-1]);print('N=$N trans=$1 agg=$2', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), {k: round(v,3) for k,v in d['side_stream_ms_rank0'].items()})"
done; done
