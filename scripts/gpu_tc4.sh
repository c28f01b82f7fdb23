cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for TC in ${TCS:-16 24 32 16}; do
timeout 600 torchrun --standalone --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline --trans-ctas $TC > gpurun_out/tc_$TC.log 2>&1; echo "tc $TC rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/tc_$TC.log') if l.startswith('{')][-1]);ph=d['phase_ms_rank0'];print('N=$N tc=$TC', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), {k: round(v,3) for k,v in d['side_stream_ms_rank0'].items()}, {k: round(v,3) for k,v in d['roofline']['per_mode_ms'].items() if k.startswith('FWD')})"
done
