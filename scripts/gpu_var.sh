# run-to-run variance at N = 1, 2, 4 (3 runs each)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for N in 1 2 4; do [ $N -gt $NG ] && continue
for i in 1 2 3; do
  DEVS=$(seq -s, 0 $((N-1)))
  if [ $N = 1 ]; then CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/var_${N}_$i.log 2>&1
  else CUDA_VISIBLE_DEVICES=$DEVS timeout 600 torchrun --standalone --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline > gpurun_out/var_${N}_$i.log 2>&1; fi
  python -c "
import json;d=json.loads([l for l in open('gpurun_out/var_${N}_$i.log') if l.startswith('{')][-1]);print('N=$N run $i', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), d['clocks']['sm_mhz'], d.get('rows_per_rank',{}).get('max_over_mean'))" || tail -5 gpurun_out/var_${N}_$i.log
done; done
