# round 2: gate backward v2 (coalesced pipelined gather, transposed dW), combine/combine_bwd MLP
set -x
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/r2_g6_tests.log 2>&1; echo tests $?
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_g6.log 2>&1; echo bench $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_g6.csv \
   python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/r2_ncu_list6.log 2>&1; echo "ncu list rc=$?"
tail -3 gpurun_out/r2_g6_tests.log
head -c 300 gpurun_out/r2_bench_g6.log
python scripts/launch_summary.py gpurun_out/r2_launches_g6.csv | head -24
