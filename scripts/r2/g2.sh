# round 2: GPU suite after the capacity / replica-bound / reuse-gate changes + GEMM wait breakdown
set -x
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2_gputests2.log 2>&1; echo tests $?
PPMOE_GEMM_DEBUG=1 timeout 300 python scripts/gemm_bench.py > gpurun_out/r2_gemm_dbg.log 2>&1; echo gemm $?
timeout 300 python scripts/gemm_bench.py FWD1 FWD2 DGRAD2 DGRAD1 WGRAD2 WGRAD1 > gpurun_out/r2_gemm.log 2>&1
tail -5 gpurun_out/r2_gputests2.log
cat gpurun_out/r2_gemm_dbg.log
