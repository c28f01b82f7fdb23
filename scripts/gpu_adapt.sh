cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 1800 python -m pytest tests/test_multi_gpu.py tests/test_layer_gpu.py -x -q > gpurun_out/ad_m.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ad_m.log
for NN in 2 4; do [ $NN -gt $NG ] && continue; for i in 1 2; do
DEVS=$(seq -s, 0 $((NN-1)))
CUDA_VISIBLE_DEVICES=$DEVS timeout 600 torchrun --standalone --nproc-per-node $NN bench.py --gpus $NN --no-cpu-baseline > gpurun_out/ad_$NN.log 2>&1
python -c "
import json;d=json.loads([l for l in open('gpurun_out/ad_$NN.log') if l.startswith('{')][-1]);print('N=$NN', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), {k: round(v,3) for k,v in d['side_stream_ms_rank0'].items()})" || tail -5 gpurun_out/ad_$NN.log
done; done
