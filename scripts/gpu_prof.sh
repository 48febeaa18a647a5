# profiling + diagnostics pass (one GPU): pytest (all), precision diag, ncu launch list + full capture
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python scripts/diag_precision.py > gpurun_out/diag.log 2>&1; echo diag_rc=$?
CMD="python bench.py --steps 2 --warmup 1 --frames-per-step 10 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo ncu_list_rc=$?
timeout 600 $CMD > gpurun_out/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 3 -c 1 -o gpurun_out/prof_eval $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_full_rc=$?
tail -3 gpurun_out/ncu_full.log
