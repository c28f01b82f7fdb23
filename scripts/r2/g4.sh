# round 2: LSU-epilogue A/B, GEMM + layer parity, new gate backward kernels
set -x
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py -q -x > gpurun_out/r2_g4_tests.log 2>&1; echo tests $?
for v in 1 0; do
  PPMOE_GEMM_LSU_EPI=$v PPMOE_GEMM_DEBUG=1 timeout 300 python scripts/gemm_bench.py FWD1 PLAIN FWD2 DGRAD2 DGRAD1 > gpurun_out/r2_gemm_lsu$v.log 2>&1
done
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_g4.log 2>&1; echo bench $?
tail -3 gpurun_out/r2_g4_tests.log
cat gpurun_out/r2_gemm_lsu1.log gpurun_out/r2_gemm_lsu0.log
head -c 600 gpurun_out/r2_bench_g4.log
