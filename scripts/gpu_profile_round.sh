# round profiling pass (one GPU): ncu launch list + full capture of the eval kernel -> gpurun_out/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --frames-per-step 10 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_launches.csv $CMD > gpurun_out/prof_list.log 2>&1; echo list_rc=$?
timeout 600 $CMD > gpurun_out/prof_plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:eval_tc -s 3 -c 1 -o gpurun_out/prof_eval_${TAG:-r02} $CMD > gpurun_out/prof_full.log 2>&1; echo full_rc=$?
