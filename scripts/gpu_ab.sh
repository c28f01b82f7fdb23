# GEMM CTA-pair A/B: tests with pairs on, bench with pairs on/off
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py -x -q > gpurun_out/t_ab.log 2>&1; echo "tests rc=$?"
tail -25 gpurun_out/t_ab.log | grep -v "^  " | tail -12
for pair in 1 0; do
PPMOE_GEMM_CTA_PAIR=$pair timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pair$pair.log 2>&1; echo "bench pair=$pair rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_pair$pair.log').read().strip().split('\n')[-1]);print(d['value'],d['ms_per_step'],d['roofline']['achieved'],d['roofline']['per_mode_ms'])" 2>&1 | tail -2
done
