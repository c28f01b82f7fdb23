cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for NN in 1 4; do [ $NN -gt $NG ] && continue; for i in 1 2; do
DEVS=$(seq -s, 0 $((NN-1)))
if [ $NN = 1 ]; then CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/e2e.log 2>&1
else CUDA_VISIBLE_DEVICES=$DEVS timeout 600 torchrun --standalone --nproc-per-node $NN bench.py --gpus $NN --no-cpu-baseline > gpurun_out/e2e.log 2>&1; fi
python -c "
import json;d=json.loads([l for l in open('gpurun_out/e2e.log') if l.startswith('{')][-1]);print('N=$NN', round(d['value']/1e6,2),'M e2e',round(d['e2e']['value']/1e6,2))" || tail -5 gpurun_out/e2e.log
done; done
