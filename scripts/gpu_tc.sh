cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 ./tests/cuda/umma_probe; echo probe_rc=$?
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_tc.log 2>&1; echo smoke_tc_rc=$?
tail -4 gpurun_out/smoke_tc.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -12 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err; echo bench_rc=$?
python - <<'PY'
import json
for f in ["gpurun_out/bench_tc.json"]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "value %.1f"%d["value"], "eval_ms %.3f"%d["roofline"]["eval_ms_per_launch"], "frac %.3f"%d["roofline"]["frac"], "e2e", d["e2e"] and round(d["e2e"]["value"],1))
    except Exception as e: print(f, "ERR", e)
PY
tail -3 gpurun_out/bench_tc.err
