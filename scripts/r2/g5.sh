# round 2: wide-tile FWD1/DGRAD2 A/B; GEMM + layer parity; launch list of one step
set -x
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py -q -x > gpurun_out/r2_g5_tests.log 2>&1; echo tests $?
PPMOE_GEMM_DEBUG=1 timeout 300 python scripts/gemm_bench.py FWD1 DGRAD2 > gpurun_out/r2_g5_narrow.log 2>&1
PPMOE_GEMM_FWD1_WIDE=1 PPMOE_GEMM_DGRAD2_WIDE=1 PPMOE_GEMM_DEBUG=1 timeout 300 python scripts/gemm_bench.py FWD1 DGRAD2 > gpurun_out/r2_g5_wide.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_g5.log 2>&1; echo bench $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv \
   python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/r2_ncu_list.log 2>&1; echo "ncu list rc=$?"
tail -3 gpurun_out/r2_g5_tests.log
cat gpurun_out/r2_g5_narrow.log gpurun_out/r2_g5_wide.log
head -c 400 gpurun_out/r2_bench_g5.log
