cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for i in 1 2; do for V in "0 1" "1 0" "1 1"; do set -- $V
PPMOE_GEMM_WIDE=$1 timeout 600 torchrun --standalone --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline --fused-a2a $2 > gpurun_out/fw2.log 2>&1
python -c "
import json;d=json.loads([l for l in open('gpurun_out/fw2.log') if l.startswith('{')][-1]);print('N=$N wide=$1 fused=$2', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2))"
done; done
