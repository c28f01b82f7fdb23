cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do for F in 0 1; do
timeout 600 python bench.py --no-cpu-baseline --fused-a2a $F > gpurun_out/nf_$F.log 2>&1
python -c "
import json;d=json.loads([l for l in open('gpurun_out/nf_$F.log') if l.startswith('{')][-1]);print('N=1 fused=$F', round(d['value']/1e6,3),'M', round(d['ms_per_step'],3),'e2e',round(d['e2e']['value']/1e6,2), {k: round(v,3) for k,v in d['phase_ms_rank0'].items() if k in ('combine','combine_bwd','dispatch_bwd','fwd_gemms','bwd_gemms')})"
done; done
