# one GPU call: tests + bench + ncu (launch list and full capture of the GEMMs)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py -x -q > gpurun_out/t_gemm.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/t_gemm.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench.log
timeout 300 python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 18 -c 6 \
   -o gpurun_out/prof_gemm python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full.log
