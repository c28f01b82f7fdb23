# GEMM tests + per-mode timing + N=1 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py -x -q > gpurun_out/ga_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ga_tests.log
timeout 300 python scripts/gemm_bench.py 2>&1 | tail -8
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ga_bench.log 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/ga_bench.log') if l.startswith('{')][-1]);r=d['roofline'];print(round(d['value']/1e6,3),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2),'gemm',round(r['gemm_ms_per_step'],3), round(r['achieved']), {k: round(v,3) for k,v in r['per_mode_ms'].items()})"
