set -x
timeout 900 python -m pytest tests/test_layer_gpu.py tests/test_gemm_gpu.py -q -x > gpurun_out/r2_g7_tests.log 2>&1; echo tests $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_g7.csv \
   python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/r2_ncu_list7.log 2>&1; echo "ncu list rc=$?"
tail -3 gpurun_out/r2_g7_tests.log
python scripts/launch_summary.py gpurun_out/r2_launches_g7.csv | head -16
