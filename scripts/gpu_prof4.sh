# round-1 profile set for the committed code: plain bench, launch list of the same command, full GEMM capture
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --profile-only"
timeout 300 $CMD > gpurun_out/r01_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_launches_cfg2.csv $CMD > gpurun_out/r01_ncu_list.log 2>&1; echo "list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 40 -c 10 \
   -o gpurun_out/r01_prof_cfg2 $CMD > gpurun_out/r01_ncu_full.log 2>&1; echo "full rc=$?"
