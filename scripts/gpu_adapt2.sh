cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for NN in 4 2; do for R in 2 4 8 16; do
DEVS=$(seq -s, 0 $((NN-1)))
CUDA_VISIBLE_DEVICES=$DEVS timeout 600 torchrun --standalone --nproc-per-node $NN bench.py --gpus $NN --no-cpu-baseline --res-per-replica $R > gpurun_out/ad2.log 2>&1
python -c "
import json;d=json.loads([l for l in open('gpurun_out/ad2.log') if l.startswith('{')][-1]);print('N=$NN res=$R', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), {k: round(v,3) for k,v in d['side_stream_ms_rank0'].items()})" || tail -5 gpurun_out/ad2.log
done; done
