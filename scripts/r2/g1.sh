# round 2, first box: emulated multi-rank parity on one GPU, full GPU suite, N=1 bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,compute_mode --format=csv
timeout 300 python -m pytest tests/test_multi_gpu.py -x -q -k "host-copy--virtual and not fused and not reuse" > gpurun_out/r2_emul1.log 2>&1; echo emul1 $?
timeout 300 python -m pytest tests/test_multi_gpu.py -x -q -k "device-sm--virtual and not reuse" > gpurun_out/r2_emul2.log 2>&1; echo emul2 $?
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/r2_gputests.log 2>&1; echo tests $?
timeout 300 python bench.py > gpurun_out/r2_bench1.log 2>&1; echo bench $?
tail -3 gpurun_out/r2_gputests.log
