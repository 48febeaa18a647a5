# A/B of environment variants on the bench: usage
#   bash scripts/gpu_ab_env.sh "TAG:VAR=val,VAR2=val" ...   (CFGS="2 1 3 4", PREC="strict fast")
# prints value / eval ms per variant, config and precision; optional PYTEST=1 first
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -n "$PYTEST" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
  tail -5 gpurun_out/pytest_gpu.log
fi
for V in "$@"; do
  tag=${V%%:*}; envs=${V#*:}
  for cfg in ${CFGS:-2}; do for prec in ${PREC:-strict}; do
    out=gpurun_out/ab_${tag}_c${cfg}_${prec}.json
    env $(echo $envs | tr ',' ' ') timeout 600 python bench.py --config $cfg --precision $prec --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e > $out 2> ${out%.json}.err
    python - $out $tag $cfg $prec <<'PY'
import json,sys
f,tag,cfg,prec=sys.argv[1:]
try:
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f"{tag:12s} cfg{cfg} {prec:6s} value {d['value']:9.1f} eval_ms {d['roofline']['eval_ms_per_launch']:8.3f} sm_mhz {d['clocks']['sm_mhz']}")
except Exception as e: print(tag, cfg, prec, "ERR", e, open(f[:-5]+'.err').read()[-500:])
PY
  done; done
done
