# ncu full capture of one eval_kernel launch (small bench), after a plain run of the same command
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --frames-per-step 10 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-eval} -s 3 -c 1 -o gpurun_out/prof_eval_${TAG:-x} $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_full_rc=$?
tail -2 gpurun_out/ncu_full.log
