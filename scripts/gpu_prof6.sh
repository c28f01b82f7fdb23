cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 2 --warmup 3 --profile-only --eager"
timeout 300 $CMD > gpurun_out/p6_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 27 -c 1 \
   -o gpurun_out/p6_route $CMD > gpurun_out/p6_ncu.log 2>&1; echo "ncu rc=$?"
