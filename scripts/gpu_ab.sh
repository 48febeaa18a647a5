# A/B: "FIELD:EVAL:TAG" variants (SQV_FIELD, SQV_EVAL; TAG is free text) -> bench eval
# time + config-1 precision.  usage: bash scripts/gpu_ab.sh 6:tc:0 7:tc:0 6:ffma:0
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for V in "$@"; do
  IFS=: read F E PP <<< "$V"
  tag=${F}_${E}_${PP}
  SQV_FIELD=$F SQV_EVAL=$E timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$tag.json 2>/dev/null
  SQV_FIELD=$F SQV_EVAL=$E timeout 600 python scripts/diag_precision.py > /dev/null 2>&1; cp gpurun_out/diag_precision.json gpurun_out/ab_${tag}_prec.json
  python - $tag <<'PY'
import json,sys
tag=sys.argv[1]
d=json.loads(open(f"gpurun_out/ab_{tag}.json").read().strip().splitlines()[-1])
p=json.load(open(f"gpurun_out/ab_{tag}_prec.json"))
rows={k.replace("vo_",""):("%.1e"%v["rel_max"],v["n_over_1e-5"]) for k,v in p["vo_config1"].items()}
print(f"{tag}: value {d['value']:.1f} eval_ms {d['roofline']['eval_ms_per_launch']:.3f} frac {d['roofline']['frac']:.3f} | {rows}")
PY
done
