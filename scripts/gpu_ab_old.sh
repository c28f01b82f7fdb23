# A/B: old tree (ab_old) vs HEAD, N=1 bench, same box, alternating
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
(cd ab_old && timeout 600 python bench.py --no-cpu-baseline > ../gpurun_out/ab_old_$i.log 2>&1); echo "old rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/ab_old_$i.log') if l.startswith('{')][-1]);r=d['roofline'];print('OLD', round(d['value']/1e6,3),'M', round(d['ms_per_step'],3),'gemm',round(r['gemm_ms_per_step'],3), r.get('per_mode_ms'))"
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_new_$i.log 2>&1; echo "new rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/ab_new_$i.log') if l.startswith('{')][-1]);r=d['roofline'];print('NEW', round(d['value']/1e6,3),'M', round(d['ms_per_step'],3),'gemm',round(r['gemm_ms_per_step'],3), r.get('per_mode_ms'))"
done
