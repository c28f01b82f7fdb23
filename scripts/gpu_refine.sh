cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
[ -n "$TESTS" ] && CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_planner_gpu.py -x -q > gpurun_out/rf_planner.log 2>&1; echo "planner tests rc=$?"; tail -2 gpurun_out/rf_planner.log
[ -n "$TESTS" ] && timeout 1500 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/rf_mgpu.log 2>&1; echo "mgpu tests rc=$?"; tail -2 gpurun_out/rf_mgpu.log
for NN in 2 4; do [ $NN -gt $N ] && continue; for R in ${RS:-1}; do
DEVS=$(seq -s, 0 $((NN-1)))
CUDA_VISIBLE_DEVICES=$DEVS timeout 600 torchrun --standalone --nproc-per-node $NN bench.py --gpus $NN --no-cpu-baseline --refine-slots $R > gpurun_out/rf_${NN}_$R.log 2>&1; echo "N=$NN refine $R rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/rf_${NN}_$R.log') if l.startswith('{')][-1]);print('N=$NN refine=$R', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), {k: round(v,3) for k,v in d['side_stream_ms_rank0'].items()}, d['replica_traffic']['replicas_per_rank'], d['rows_per_rank'])" || tail -20 gpurun_out/rf_${NN}_$R.log
done; done
