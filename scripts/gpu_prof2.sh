# tests + bench + ncu launch list + full capture of the GEMM launches of one step
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/t_all.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench.log
timeout 300 python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 24 -c 8 \
   -o gpurun_out/prof_gemm2 python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
