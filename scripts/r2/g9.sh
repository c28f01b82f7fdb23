set -x
PPMOE_GEMM_FAST_GELU=1 timeout 900 python -m pytest tests/test_layer_gpu.py tests/test_gemm_gpu.py -q -x > gpurun_out/r2_g9_tests.log 2>&1; echo tests $?
PPMOE_GEMM_DEBUG=1 timeout 300 python scripts/gemm_bench.py FWD1 DGRAD2 > gpurun_out/r2_g9_a.log 2>&1
PPMOE_GEMM_FAST_GELU=1 PPMOE_GEMM_DEBUG=1 timeout 300 python scripts/gemm_bench.py FWD1 DGRAD2 > gpurun_out/r2_g9_b.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_g9_bench_a.log 2>&1
PPMOE_GEMM_FAST_GELU=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_g9_bench_b.log 2>&1
tail -2 gpurun_out/r2_g9_tests.log
for f in a b; do echo "== $f"; head -2 gpurun_out/r2_g9_$f.log; head -c 330 gpurun_out/r2_g9_bench_$f.log; echo; done
