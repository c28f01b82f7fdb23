# round-1 final N=1 evidence: launch list + full captures of the small HBM-bound kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/p7_plain.log 2>&1; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p7_launches.csv \
   python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/p7_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dot_bf16_partial|dispatch_bwd_kernel|combine_bwd_kernel|dispatch_kernel|combine_kernel" -s 20 -c 5 \
   -o gpurun_out/p7_small python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/p7_ncu_small.log 2>&1; echo "ncu small rc=$?"
tail -3 gpurun_out/p7_ncu_small.log
