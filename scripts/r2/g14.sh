set -x
timeout 900 python -m pytest tests/test_layer_gpu.py tests/test_gemm_gpu.py -q -x > gpurun_out/r2_g14_tests.log 2>&1; echo tests $?
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_g14_bench.log 2>&1; echo bench $?
for ks in 1 2 4; do PPMOE_ROUTE_KS=$ks timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:route_kernel -c 6 --csv python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/r2_g14_route_ks$ks.csv 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_g14.csv python bench.py --steps 2 --warmup 3 --profile-only > /dev/null 2>&1; echo ncu $?
tail -2 gpurun_out/r2_g14_tests.log
head -c 400 gpurun_out/r2_g14_bench.log; echo
for ks in 1 2 4; do echo "ks $ks"; grep route_kernel gpurun_out/r2_g14_route_ks$ks.csv | tail -3 | awk -F'","' '{print $NF}'; done
python scripts/launch_summary.py gpurun_out/r2_launches_g14.csv > gpurun_out/r2_launches_g14.txt; head -24 gpurun_out/r2_launches_g14.txt
