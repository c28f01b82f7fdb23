# full GPU validation on a 4-GPU box: pytest -m gpu (all GPUs visible), smoke, stack at 2, benches at 1/2/4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/f4_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/f4_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0,1 timeout 900 torchrun --standalone --nproc-per-node 2 bench.py --gpus 2 --config cfg5 --steps 5 --warmup 3 > gpurun_out/f4_stack.log 2>&1; echo "stack2 rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/f4_stack.log') if l.startswith('{')][-1]);print('stack EP2', round(d['value']/1e3,1),'K tok/s')" || tail -5 gpurun_out/f4_stack.log
bash scripts/gpu_var.sh
