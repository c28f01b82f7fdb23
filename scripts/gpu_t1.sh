# 1-GPU: full gpu test suite + N=1 bench x2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t1_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t1_tests.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/t1_bench_$i.log 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/t1_bench_$i.log') if l.startswith('{')][-1]);r=d['roofline'];print(round(d['value']/1e6,3),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2),'gemm',round(r['gemm_ms_per_step'],3), round(r['achieved']), d['gpu_launches'], d['clocks'])"
done
