# 2-GPU: host-planning parity (new device-counter barrier), device-planning parity, benches eager vs graphed
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for P in host device; do
  PP_PLANNING=$P timeout 300 torchrun --standalone --nproc-per-node 2 scripts/mgpu_check.py > gpurun_out/dp_check_$P.log 2>&1; echo "check $P rc=$?"; grep "\[it" gpurun_out/dp_check_$P.log | tail -3
done
timeout 600 torchrun --standalone --nproc-per-node 2 bench.py --gpus 2 --no-cpu-baseline --eager > gpurun_out/dp_bench_eager.log 2>&1; echo "eager rc=$?"
timeout 600 torchrun --standalone --nproc-per-node 2 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/dp_bench_graph.log 2>&1; echo "graph rc=$?"
for f in eager graph; do python -c "
import json,sys;d=json.loads([l for l in open('gpurun_out/dp_bench_$f.log') if l.startswith('{')][-1]);print('$f', d['value'],d['ms_per_step'],'e2e',d['e2e']['value'],d['roofline']['achieved'], d.get('host_ms_per_step'))" || tail -20 gpurun_out/dp_bench_$f.log; done
