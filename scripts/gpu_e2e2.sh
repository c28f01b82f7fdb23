cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for i in 1 2; do for NBUF in 2 3; do
PP_BENCH_NBUF=$NBUF timeout 600 torchrun --standalone --nproc-per-node $NG bench.py --gpus $NG --no-cpu-baseline > gpurun_out/e2e.log 2>&1
python -c "
import json;d=json.loads([l for l in open('gpurun_out/e2e.log') if l.startswith('{')][-1]);print('N=$NG nbuf=$NBUF', round(d['value']/1e6,2),'M e2e',round(d['e2e']['value']/1e6,2))" || tail -5 gpurun_out/e2e.log
done; done
nvidia-smi topo -m | head -6
