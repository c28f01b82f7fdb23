# what the driver runs at round end (1 GPU): smoke, pytest -m gpu, default bench, reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/re_smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/re_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/re_tests.log
timeout 600 python bench.py > gpurun_out/re_bench.log 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/re_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/re_ref.log 2>&1; echo "ref rc=$?"; tail -c 600 gpurun_out/re_ref.log
