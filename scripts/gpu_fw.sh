cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for NN in 2 4; do for i in 1 2; do for F in 1 0; do
DEVS=$(seq -s, 0 $((NN-1)))
CUDA_VISIBLE_DEVICES=$DEVS timeout 600 torchrun --standalone --nproc-per-node $NN bench.py --gpus $NN --no-cpu-baseline --fused-a2a $F > gpurun_out/fw_${NN}_$F.log 2>&1
python -c "
import json;d=json.loads([l for l in open('gpurun_out/fw_${NN}_$F.log') if l.startswith('{')][-1]);print('N=$NN fused=$F', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), {k: round(v,3) for k,v in d['roofline']['per_mode_ms'].items()})" || tail -5 gpurun_out/fw_${NN}_$F.log
done; done; done
