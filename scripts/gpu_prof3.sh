# launch lists (cfg2, cfg3 at 1 GPU) + full capture of the small kernels at cfg3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in cfg2 cfg3; do
timeout 300 python bench.py --steps 2 --warmup 3 --profile-only --eager --config $cfg > gpurun_out/plain_$cfg.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$cfg.csv \
   python bench.py --steps 2 --warmup 3 --profile-only --eager --config $cfg > gpurun_out/ncu_list_$cfg.log 2>&1; echo "ncu list $cfg rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"grouped_gemm_kernel<(16|32|64)|grouped_gemm_kernel<256, (0|1), (0|1), (5|6)|dispatch|combine|layout" -s 12 -c 12 \
   -o gpurun_out/prof_small python bench.py --steps 2 --warmup 3 --profile-only --eager --config cfg3 > gpurun_out/ncu_small.log 2>&1; echo "ncu full rc=$?"
