cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for TP in start after_route start after_route; do
PPMOE_TRANS_POINT=$TP timeout 600 torchrun --standalone --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline > gpurun_out/tp_$TP.log 2>&1; echo "$TP rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/tp_$TP.log') if l.startswith('{')][-1]);ph=d['phase_ms_rank0'];print('N=$N $TP', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e6,2), {k: round(v,3) for k,v in ph.items() if k in ('route_hist','hist_barrier','route_layout','dispatch','trans_wait','barrier1')})"
done
