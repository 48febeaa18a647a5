# ncu full capture of one evaluator launch under env overrides (VAR=val,...) after a plain run
#   ENVS="SQV_STREAM=1,SQV_PERSIST=1" CFG=2 TAG=x bash scripts/gpu_ncu_env.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --config ${CFG:-2} --steps 2 --warmup 1 --frames-per-step 10 --no-e2e --no-cpu-baseline"
E=$(echo ${ENVS:-X=1} | tr ',' ' ')
env $E timeout 600 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
env $E timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-eval_tc} -s 3 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo ncu_rc=$?
tail -2 gpurun_out/ncu_$TAG.log
