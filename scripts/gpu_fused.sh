cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_layer_gpu.py tests/test_gemm_gpu.py -x -q > gpurun_out/fu_l.log 2>&1; echo "layer tests rc=$?"; tail -3 gpurun_out/fu_l.log
timeout 1800 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/fu_m.log 2>&1; echo "mgpu tests rc=$?"; tail -3 gpurun_out/fu_m.log
for NN in 2 4; do [ $NN -gt $N ] && continue; for F in ${FS:-1}; do
DEVS=$(seq -s, 0 $((NN-1)))
CUDA_VISIBLE_DEVICES=$DEVS timeout 600 torchrun --standalone --nproc-per-node $NN bench.py --gpus $NN --no-cpu-baseline --fused-a2a $F > gpurun_out/fu_${NN}_$F.log 2>&1; echo "N=$NN fused $F rc=$?"
python -c "
import json;d=json.loads([l for l in open('gpurun_out/fu_${NN}_$F.log') if l.startswith('{')][-1]);ph=d['phase_ms_rank0'];print('N=$NN fused=$F', round(d['value']/1e6,2),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), {k: round(v,3) for k,v in ph.items()}, {k: round(v,3) for k,v in d['roofline']['per_mode_ms'].items()})" || tail -20 gpurun_out/fu_${NN}_$F.log
done; done
