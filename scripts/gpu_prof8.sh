# round-1 final: N=1 launch list + --set full capture of one step's grouped-GEMM launches (wide tiles)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/p8_plain.log 2>&1; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p8_launches.csv \
   python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/p8_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 45 -c 9 \
   -o gpurun_out/p8_gemm python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/p8_ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -2 gpurun_out/p8_ncu_full.log
