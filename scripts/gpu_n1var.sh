# N=1 bench repeatability on one box
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,power.limit,clocks.max.sm,temperature.gpu --format=csv
for i in 1 2 3; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/v_n1_$i.log 2>&1; echo "run $i rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/v_n1_$i.log') if l.startswith('{')][-1]);r=d['roofline'];print(round(d['value']/1e6,3),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2),'gemm',round(r['gemm_ms_per_step'],3), round(r['achieved']), d['clocks'])"
done
