set -x
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2_g16_tests.log 2>&1; echo tests $?
for i in 1 2; do for v in 1 0; do
  PPMOE_PDL=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2_g16_bench_pdl${v}_$i.log 2>&1; echo bench $v $?
done; done
tail -2 gpurun_out/r2_g16_tests.log
for f in gpurun_out/r2_g16_bench_pdl*; do echo $f; head -c 250 $f | tail -c 130; echo; done
