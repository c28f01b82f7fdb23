# weak-scaling sweep like the driver's: N = 1, 2, 4, 8 on one box (cfg2), plus mgpu parity at 8
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for N in 1 2 4; do [ $N -gt $NG ] && continue
  DEVS=$(seq -s, 0 $((N-1)))
  if [ $N = 1 ]; then
    CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/sc_n$N.log 2>&1; echo "N=$N rc=$?"
  else
    CUDA_VISIBLE_DEVICES=$DEVS timeout 600 torchrun --standalone --nproc-per-node $N bench.py --gpus $N --no-cpu-baseline > gpurun_out/sc_n$N.log 2>&1; echo "N=$N rc=$?"
  fi
  python -c "
import json;d=json.loads([l for l in open('gpurun_out/sc_n$N.log') if l.startswith('{')][-1]);print('N=$N', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), d.get('side_stream_ms_rank0'), d.get('rows_per_rank'), {k: round(v,3) for k,v in d['phase_ms_rank0'].items()})" || tail -20 gpurun_out/sc_n$N.log
done
PP_PLANNING=device PP_ENGINE=sm PP_PLACEMENT=physical timeout 600 torchrun --standalone --nproc-per-node $NG scripts/mgpu_check.py > gpurun_out/sc_check8.log 2>&1; echo "check8 rc=$?"; grep "\[it\|\[graph" gpurun_out/sc_check8.log | tail -4
