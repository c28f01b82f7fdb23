# multi-GPU pytest (all GPUs of the box) + graphed bench at this N
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1200 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/m4_tests.log 2>&1; echo "mgpu tests rc=$?"; tail -3 gpurun_out/m4_tests.log
timeout 600 torchrun --standalone --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline > gpurun_out/m4_bench.log 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/m4_bench.log') if l.startswith('{')][-1]);print('N=$N', d['value'],d['ms_per_step'],'e2e',d['e2e']['value'],d['roofline']['achieved'],d['rows_per_rank'],d['phase_ms_rank0'])" || tail -30 gpurun_out/m4_bench.log
