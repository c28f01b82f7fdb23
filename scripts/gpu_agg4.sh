# multi-GPU parity + Agg SM sweep at N = all GPUs of the box
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/ag_mgpu.log 2>&1; echo "mgpu tests rc=$?"; tail -3 gpurun_out/ag_mgpu.log
for AC in ${ACS:-16 32}; do
timeout 600 torchrun --standalone --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline --agg-ctas $AC $BENCH_ARGS > gpurun_out/ag_$AC.log 2>&1; echo "agg $AC rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/ag_$AC.log') if l.startswith('{')][-1]);print('N=$N ac=$AC', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), {k: round(v,3) for k,v in d['side_stream_ms_rank0'].items()}, d['replica_traffic']['replicas_per_rank'], d['rows_per_rank'], {k: round(v,3) for k,v in d['phase_ms_rank0'].items()})" || tail -20 gpurun_out/ag_$AC.log
done
