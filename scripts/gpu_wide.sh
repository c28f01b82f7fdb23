cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py -x -q > gpurun_out/wd_t.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/wd_t.log
for i in 1 2; do
echo "== wide"; timeout 300 python scripts/gemm_bench.py 2>&1 | tail -6
echo "== narrow"; PPMOE_GEMM_WIDE=0 timeout 300 python scripts/gemm_bench.py 2>&1 | tail -6
done
PPMOE_GEMM_DEBUG=2 timeout 300 python scripts/gemm_trace.py FWD2 2>&1 | head -6
for W in 1 0; do PPMOE_GEMM_WIDE=$W timeout 600 python bench.py --no-cpu-baseline > gpurun_out/wd_b$W.log 2>&1
python -c "
import json;d=json.loads([l for l in open('gpurun_out/wd_b$W.log') if l.startswith('{')][-1]);r=d['roofline'];print('bench wide=$W', round(d['value']/1e6,3),'M', round(d['ms_per_step'],3),'gemm',round(r['gemm_ms_per_step'],3), round(r['achieved']), {k: round(v,3) for k,v in r['per_mode_ms'].items()})"; done
