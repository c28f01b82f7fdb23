set -x
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2_g10_tests.log 2>&1; echo tests $?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g10_bench_n2emu.log 2>&1; echo bench2 $?
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g10_cfg4.log 2>&1; echo cfg4 $?
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_g10_bench.log 2>&1; echo bench $?
tail -3 gpurun_out/r2_g10_tests.log
tail -c 1500 gpurun_out/r2_g10_bench_n2emu.log; echo
tail -c 2500 gpurun_out/r2_g10_cfg4.log
