cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 600 torchrun --standalone --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline $BENCH_ARGS > gpurun_out/ph4.log 2>&1; echo "rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/ph4.log') if l.startswith('{')][-1]);ph=d['phase_ms_rank0'];print('N=$N', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3), {k: round(v,3) for k,v in ph.items()})"
