# 1 GPU: smoke, the full GPU suite (ranks sharing the GPU for the EP parity runs), the default
# bench, the reference arm, a launch list, GEMM per-mode timings, and the staggered-tile A/B
set -x
nvidia-smi --query-gpu=index,name,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v1_smoke.log 2>&1; echo smoke $?
PPMOE_TEST_STAGGER=1 timeout 2400 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/v1_tests.log 2>&1; echo tests $?
timeout 300 python bench.py > gpurun_out/v1_bench.log 2>&1; echo bench $?
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/v1_ref.log 2>&1; echo ref $?
timeout 300 python scripts/gemm_bench.py > gpurun_out/v1_gemm.log 2>&1; echo gemm $?
for v in 1 2 3; do PPMOE_GEMM_STAGGER=$v PPMOE_GEMM_STAGGER_WGRAD=$v timeout 300 python scripts/gemm_bench.py FWD1 DGRAD2 WGRAD2 WGRAD1 > gpurun_out/v1_gemm_stagger$v.log 2>&1; echo gemm_stagger$v $?; done
PPMOE_GEMM_STAGGER=1 PPMOE_GEMM_STAGGER_WGRAD=1 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/v1_bench_stagger.log 2>&1; echo bench_stagger $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v1_launches.csv \
   python bench.py --steps 2 --warmup 3 --profile-only > /dev/null 2>&1; echo ncu $?
tail -3 gpurun_out/v1_tests.log; tail -1 gpurun_out/v1_smoke.log; head -c 300 gpurun_out/v1_bench.log; echo
for f in gpurun_out/v1_gemm.log gpurun_out/v1_gemm_stagger*.log; do echo == $f; cat $f; done
python - <<'PY'
import json
for f in ("gpurun_out/v1_bench.log", "gpurun_out/v1_bench_stagger.log"):
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
        print(f, d["value"], d["e2e"]["value"] if d.get("e2e") else None, d["roofline"]["per_mode_frac"])
    except Exception as e:
        print(f, "no line", e)
PY
python scripts/launch_summary.py gpurun_out/v1_launches.csv > gpurun_out/v1_launches.txt 2>/dev/null; head -22 gpurun_out/v1_launches.txt
