# stack (cfg5) at N=2 + N=2 phases
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 torchrun --standalone --nproc-per-node 2 bench.py --gpus 2 --config cfg5 --steps 5 --warmup 3 > gpurun_out/st2.log 2>&1; echo "stack2 rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/st2.log') if l.startswith('{')][-1]);print(round(d['value']/1e3,1),'K tok/s', round(d['ms_per_step'],2), json.dumps(d.get('stack_timeline'))[:600])" || tail -20 gpurun_out/st2.log
PP_DEBUG_PHASES=1 timeout 600 torchrun --standalone --nproc-per-node 2 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/ph2.log 2>&1; echo "n2 rc=$?"
grep "rank . \] step 5" gpurun_out/ph2.log
python -c "
import json;d=json.loads([l for l in open('gpurun_out/ph2.log') if l.startswith('{')][-1]);print(round(d['value']/1e6,2),'M', round(d['ms_per_step'],3), d['side_stream_ms_rank0'], d['replica_traffic'], d['rows_per_rank'])"
