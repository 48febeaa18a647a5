# iteration pass: gpu tests, precision diag, bench (default + A/B variants via env)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -12 gpurun_out/pytest_gpu.log
timeout 600 python scripts/diag_precision.py > gpurun_out/diag.log 2>&1; echo diag_rc=$?
SQV_FIELD=9 timeout 600 python scripts/diag_precision.py > gpurun_out/diag9.log 2>&1; cp gpurun_out/diag_precision.json gpurun_out/diag_precision9.json 2>/dev/null
timeout 600 python scripts/diag_precision.py > /dev/null 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_f7.json 2> gpurun_out/bench_f7.err; echo bench_rc=$?
SQV_FIELD=9 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_f9.json 2> gpurun_out/bench_f9.err
python - <<'PY'
import json
for f in ["gpurun_out/bench_f7.json","gpurun_out/bench_f9.json"]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "value %.1f"%d["value"], "eval_ms %.3f"%d["roofline"]["eval_ms_per_launch"], "frac %.3f"%d["roofline"]["frac"], "e2e", d["e2e"] and round(d["e2e"]["value"],1), d["clocks"])
    except Exception as e: print(f, "ERR", e)
PY
