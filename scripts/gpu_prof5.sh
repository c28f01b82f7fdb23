cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --profile-only --eager"
timeout 300 $CMD > gpurun_out/p5_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"grouped_gemm_kernel<16|dispatch_bwd|dispatch_layout|grouped_gemm_kernel<256, 1, 1, 6" -s 4 -c 4 \
   -o gpurun_out/p5_small $CMD > gpurun_out/p5_ncu.log 2>&1; echo "ncu rc=$?"
