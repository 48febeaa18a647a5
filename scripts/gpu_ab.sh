# A/B: field variants (SQV_FIELD) x evaluator (SQV_EVAL): bench eval time + config-1 precision
# usage: bash scripts/gpu_ab.sh "7:tc" "6:tc" "7:ffma"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for V in "$@"; do
  F=${V%%:*}; E=${V##*:}
  SQV_FIELD=$F SQV_EVAL=$E timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${F}_${E}.json 2>/dev/null
  SQV_FIELD=$F SQV_EVAL=$E timeout 600 python scripts/diag_precision.py > /dev/null 2>&1; cp gpurun_out/diag_precision.json gpurun_out/ab_${F}_${E}_prec.json
  python - $F $E <<'PY'
import json,sys
F,E=sys.argv[1],sys.argv[2]
d=json.loads(open(f"gpurun_out/ab_{F}_{E}.json").read().strip().splitlines()[-1])
p=json.load(open(f"gpurun_out/ab_{F}_{E}_prec.json"))
rows={k:("%.2e"%v["rel_max"],v["n_over_1e-5"]) for k,v in p["vo_config1"].items()}
print(f"field {F} eval {E}: value {d['value']:.1f} eval_ms {d['roofline']['eval_ms_per_launch']:.3f} frac {d['roofline']['frac']:.3f} | {rows}")
PY
done
