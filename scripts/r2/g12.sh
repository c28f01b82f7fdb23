set -x
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g12_bench_n2emu.log 2>&1; echo bench2 $?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --config cfg5 --steps 3 --warmup 3 > gpurun_out/r2_g12_cfg5_n2emu.log 2>&1; echo cfg5n2 $?
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_step.py > gpurun_out/r2_san_memcheck.txt 2>&1; echo memcheck $?
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_step.py > gpurun_out/r2_san_racecheck.txt 2>&1; echo racecheck $?
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python scripts/sanitize_step.py > gpurun_out/r2_san_synccheck.txt 2>&1; echo synccheck $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"grouped_gemm_kernel<16|dispatch_layout_kernel|grouped_gemm_kernel<64|splitk_reduce" -s 20 -c 4 -o gpurun_out/r2_small_full python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/r2_ncu_small.log 2>&1; echo ncu $?
tail -c 900 gpurun_out/r2_g12_bench_n2emu.log; echo
tail -c 900 gpurun_out/r2_g12_cfg5_n2emu.log; echo
tail -4 gpurun_out/r2_san_memcheck.txt gpurun_out/r2_san_racecheck.txt gpurun_out/r2_san_synccheck.txt
