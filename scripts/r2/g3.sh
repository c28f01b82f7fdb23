# round 2: GPU suite + GEMM feed experiments (per-SM rate at 148 vs 74 SMs, PLAIN vs FWD1)
set -x
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2_gputests3.log 2>&1; echo tests $?
for n in 148 74 38; do
  GEMM_SMS=$n PPMOE_GEMM_DEBUG=1 timeout 300 python scripts/gemm_bench.py FWD1 PLAIN FWD2 DGRAD2 > gpurun_out/r2_gemm_sms$n.log 2>&1
done
PPMOE_GEMM_WIDE=0 PPMOE_GEMM_DEBUG=1 timeout 300 python scripts/gemm_bench.py FWD2 DGRAD1 > gpurun_out/r2_gemm_narrow.log 2>&1
tail -5 gpurun_out/r2_gputests3.log
cat gpurun_out/r2_gemm_sms*.log gpurun_out/r2_gemm_narrow.log
