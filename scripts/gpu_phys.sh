# planner GPU tests (incl. physical) + multi-GPU parity (all GPUs) + bench virtual vs physical
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_planner_gpu.py -x -q > gpurun_out/ph_planner.log 2>&1; echo "planner tests rc=$?"; tail -3 gpurun_out/ph_planner.log
timeout 1500 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/ph_mgpu.log 2>&1; echo "mgpu tests rc=$?"; tail -3 gpurun_out/ph_mgpu.log
for P in "virtual 1" "physical 0" "physical 1"; do set -- $P
timeout 600 torchrun --standalone --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline --placement $1 --n-excl $2 --trans-ctas 32 --agg-ctas 32 > gpurun_out/ph_bench_$1_$2.log 2>&1; echo "bench $1 $2 rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/ph_bench_$1_$2.log') if l.startswith('{')][-1]);print('N=$N $1 n=$2', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), d['side_stream_ms_rank0'], d['replica_traffic'], d['rows_per_rank'], {k: round(v,3) for k,v in d['phase_ms_rank0'].items()})" || tail -30 gpurun_out/ph_bench_$1_$2.log
done
