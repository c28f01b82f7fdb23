set -x
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2_g11_tests.log 2>&1; echo tests $?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g11_bench_n2emu.log 2>&1; echo bench2 $?
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 > gpurun_out/r2_g11_cfg5.log 2>&1; echo cfg5 $?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --config cfg5 --steps 3 --warmup 3 > gpurun_out/r2_g11_cfg5_n2emu.log 2>&1; echo cfg5n2 $?
tail -3 gpurun_out/r2_g11_tests.log
tail -c 800 gpurun_out/r2_g11_bench_n2emu.log; echo
tail -c 1200 gpurun_out/r2_g11_cfg5.log; echo
tail -c 1200 gpurun_out/r2_g11_cfg5_n2emu.log
