# ncu full capture of one eval_tc launch for a given bench config (CFG, TAG)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --config ${CFG:-1} --steps 2 --warmup 1 --frames-per-step 10 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain_cfg.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:eval_tc -s 3 -c 1 -o gpurun_out/prof_eval_${TAG:-cfg} $CMD > gpurun_out/ncu_cfg.log 2>&1; echo ncu_rc=$?
