cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for i in 1 2; do for G in ${GS:-0 1}; do for TC in 16; do
timeout 600 torchrun --standalone --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline --trans-gate $G --trans-ctas $TC > gpurun_out/gt_$G.log 2>&1
python -c "
import json;d=json.loads([l for l in open('gpurun_out/gt_$G.log') if l.startswith('{')][-1]);print('N=$N gate=$G tc=$TC', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2))"
done; done; done
