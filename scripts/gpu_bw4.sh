# planner cost-model B x alpha sweep at N = all GPUs of the box
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for AB in "0.5 450e9" "0.1 50e9" "0.1 100e9" "0.2 100e9" "0.5 50e9"; do set -- $AB
timeout 600 torchrun --standalone --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline --alpha $1 --avg-bandwidth $2 > gpurun_out/bw_$1_$2.log 2>&1; echo "alpha $1 B $2 rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/bw_$1_$2.log') if l.startswith('{')][-1]);print('N=$N a=$1 B=$2', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), {k: round(v,3) for k,v in d['side_stream_ms_rank0'].items()}, d['replica_traffic']['replicas_per_rank'], d['rows_per_rank'])" || tail -20 gpurun_out/bw_$1_$2.log
done
