# m = 2 experts per rank (the N=8 / E=16 shape) on 4 GPUs: parity for the bench's default path
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PP_E=8 PP_PLANNING=device PP_ENGINE=sm PP_PLACEMENT=physical PP_REFINE=1 PP_FUSED=1 timeout 600 torchrun --standalone --nproc-per-node 4 scripts/mgpu_check.py > gpurun_out/m2_a.log 2>&1; echo "m2 device rc=$?"; grep "\[it\|\[graph" gpurun_out/m2_a.log | tail -3
PP_E=4 PP_PLANNING=device PP_ENGINE=sm PP_PLACEMENT=physical PP_REFINE=1 PP_FUSED=1 timeout 600 torchrun --standalone --nproc-per-node 4 scripts/mgpu_check.py > gpurun_out/m2_b.log 2>&1; echo "m1 device rc=$?"; grep "\[it\|\[graph" gpurun_out/m2_b.log | tail -3
timeout 600 torchrun --standalone --nproc-per-node 4 bench.py --gpus 4 --no-cpu-baseline --config cfg1 > gpurun_out/m2_c.log 2>&1; echo "cfg1 rc=$?"
