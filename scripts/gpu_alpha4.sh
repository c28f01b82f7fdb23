# physical planner alpha sweep at N = all GPUs of the box
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for A in ${ALPHAS:-0.5 0.2 0.1 0.05}; do
timeout 600 torchrun --standalone --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline --alpha $A > gpurun_out/al_$A.log 2>&1; echo "alpha $A rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/al_$A.log') if l.startswith('{')][-1]);print('N=$N a=$A', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), {k: round(v,3) for k,v in d['side_stream_ms_rank0'].items()}, d['replica_traffic']['replicas_per_rank'], d['rows_per_rank'])" || tail -20 gpurun_out/al_$A.log
done
