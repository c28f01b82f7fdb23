cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for pair in 0 1; do echo "pair=$pair"; PPMOE_GEMM_CTA_PAIR=$pair timeout 120 python scripts/gemm_bench.py; done
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_g.log 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_g.log').read().strip().split('\n')[-1]);print(d['value'],d['ms_per_step'],d['host_enqueue_ms_per_step'],d['e2e']['value'],d['roofline']['achieved'],d['gpu_launches'])" 2>&1 | tail -3
PPMOE_GEMM_CTA_PAIR=1 timeout 120 python scripts/gemm_bench.py FWD2 > /dev/null 2>&1 && \
PPMOE_GEMM_CTA_PAIR=1 timeout 300 ncu --set full --clock-control none -k regex:grouped_gemm -s 3 -c 1 -o gpurun_out/prof_pair python scripts/gemm_bench.py FWD2 > gpurun_out/ncu_pair.log 2>&1; echo "ncu rc=$?"
