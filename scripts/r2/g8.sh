set -x
timeout 900 python -m pytest tests/test_layer_gpu.py tests/test_gemm_gpu.py -q -x > gpurun_out/r2_g8_tests.log 2>&1; echo tests $?
PPMOE_GEMM_DEBUG=1 timeout 300 python scripts/gemm_bench.py FWD1 > gpurun_out/r2_g8_a.log 2>&1
PPMOE_GEMM_FAST_GELU=1 PPMOE_GEMM_DEBUG=1 timeout 300 python scripts/gemm_bench.py FWD1 > gpurun_out/r2_g8_b.log 2>&1
PPMOE_GEMM_FWD1_WIDE=1 PPMOE_GEMM_FAST_GELU=1 PPMOE_GEMM_DEBUG=1 timeout 300 python scripts/gemm_bench.py FWD1 > gpurun_out/r2_g8_c.log 2>&1
PPMOE_GEMM_FWD1_WIDE=1 PPMOE_GEMM_LSU_EPI=1 PPMOE_GEMM_FAST_GELU=1 PPMOE_GEMM_DEBUG=1 timeout 300 python scripts/gemm_bench.py FWD1 > gpurun_out/r2_g8_d.log 2>&1
PPMOE_GEMM_FWD1_WIDE=1 PPMOE_GEMM_LSU_EPI=1 PPMOE_GEMM_DEBUG=1 timeout 300 python scripts/gemm_bench.py FWD1 > gpurun_out/r2_g8_e.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_g8.csv \
   python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/r2_ncu_list8.log 2>&1; echo "ncu list rc=$?"
tail -2 gpurun_out/r2_g8_tests.log
for f in a b c d e; do echo "== $f"; cat gpurun_out/r2_g8_$f.log; done
python scripts/launch_summary.py gpurun_out/r2_launches_g8.csv > gpurun_out/r2_launches_g8.txt; head -22 gpurun_out/r2_launches_g8.txt
