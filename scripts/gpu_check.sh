cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt 2>&1
timeout 400 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/t_gemm.log 2>&1; echo "gemm rc=$?"
timeout 600 python -m pytest tests/test_planner_gpu.py -x -q > gpurun_out/t_plan.log 2>&1; echo "plan rc=$?"
timeout 400 python -m pytest tests/test_layer_gpu.py -x -q > gpurun_out/t_layer.log 2>&1; echo "layer rc=$?"
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -5 gpurun_out/t_gemm.log gpurun_out/t_plan.log gpurun_out/t_layer.log gpurun_out/bench.log
