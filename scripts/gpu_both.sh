# 1-GPU tests + bench on GPU 0, then 2-GPU parity + bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/b_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/b_tests.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b_bench1.log 2>&1; echo "bench1 rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/b_bench1.log').read().strip().split('\n')[-1]);print('N=1', d['value'],d['ms_per_step'],'e2e',d['e2e']['value'],d['roofline']['achieved'],d['clocks'])"
PP_ENGINE=copy timeout 300 torchrun --standalone --nproc-per-node 2 scripts/mgpu_check.py 2>&1 | grep "\[it" | tail -3
timeout 600 torchrun --standalone --nproc-per-node 2 bench.py --gpus 2 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/b_bench2.log
python -c "
import json;d=json.loads(open('gpurun_out/b_bench2.log').read().strip().split('\n')[-1]);print('N=2', d['value'],d['ms_per_step'],'e2e',d['e2e']['value'],d['roofline']['achieved'])"
