# all layer configs at N = 4 and 2 (graphed, physical + refine) and cfg1 at N=4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for C in cfg1 cfg3 cfg4; do for NN in 2 4; do [ $NN -gt $N ] && continue
DEVS=$(seq -s, 0 $((NN-1)))
CUDA_VISIBLE_DEVICES=$DEVS timeout 900 torchrun --standalone --nproc-per-node $NN bench.py --gpus $NN --no-cpu-baseline --config $C > gpurun_out/cf_${C}_$NN.log 2>&1; echo "$C N=$NN rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/cf_${C}_$NN.log') if l.startswith('{')][-1]);print('$C N=$NN', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), 'gemm TF', round(d['roofline']['achieved']), d['rows_per_rank']['max_over_mean'], d['replica_traffic']['replicas_per_rank'] if d.get('replica_traffic') else None)" || tail -12 gpurun_out/cf_${C}_$NN.log
done; done
