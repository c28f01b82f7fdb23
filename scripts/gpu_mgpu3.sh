cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 300 python -m pytest tests/test_layer_gpu.py -q -x 2>&1 | tail -1
PP_ENGINE=copy timeout 300 torchrun --standalone --nproc-per-node $NG scripts/mgpu_check.py > gpurun_out/mgpu_copy.log 2>&1; echo "mgpu rc=$?"
grep "OK\|FAIL\|MISMATCH\|rror" gpurun_out/mgpu_copy.log | head -5
bash scripts/gpu_scale.sh
