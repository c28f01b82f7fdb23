#!/bin/bash
# torchrun --no-python wrapper: rank 0 runs under ncu (NVLink + DRAM bytes of the A2A / Trans / Agg
# kernels), the other ranks run plainly.  Usage:
#   python -m torch.distributed.run --no-python --nproc-per-node N ... scripts/ncu_rank0.sh OUT.csv SCRIPT.py args...
out=$1; shift
if [ "$RANK" = "0" ]; then
  exec ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:"dispatch_kernel|combine_kernel|combine_bwd_kernel|dispatch_bwd_kernel|replica_trans|replica_agg" \
    -s 8 -c 16 --csv --log-file "$out" python "$@"
else
  exec python "$@"
fi
