cd $GRAFT_REPO_ROOT
echo "== normal + debug counters"; PPMOE_GEMM_DEBUG=1 timeout 300 python scripts/gemm_bench.py 2>&1 | tail -12
