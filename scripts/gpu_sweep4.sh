# N-GPU graphed bench: Trans/Agg SM counts sweep + per-step phases
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for tc in ${TCS:-16 32}; do for ac in ${ACS:-16 32}; do
PP_DEBUG_PHASES=1 timeout 600 torchrun --standalone --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline --trans-ctas $tc --agg-ctas $ac > gpurun_out/sw_${tc}_${ac}.log 2>&1; echo "bench $tc $ac rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/sw_${tc}_${ac}.log') if l.startswith('{')][-1]);print('N=$N t$tc a$ac', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), d['side_stream_ms_rank0'], d['replica_traffic'], {k: round(v,3) for k,v in d['phase_ms_rank0'].items()})" || tail -30 gpurun_out/sw_${tc}_${ac}.log
done; done
grep "rank 0\] step" gpurun_out/sw_16_16.log | head -8
