set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
nproc; lscpu | grep -E "Model name|^CPU\(s\)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -5 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-seconds 8 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench_rc=$?
tail -3 gpurun_out/bench1.err; cat gpurun_out/bench1.json
